"""World-size-2 test of the multi-GPU protocol on CPU (gloo).

Each rank owns the contiguous shard fsb_shard_range() (the C-ABI host
function the engine uses) and steps it with the oracle, keyed by GLOBAL fish
index; the per-step exchange is the engine's: all-gather of the 4-scalar
partial {max(prev-cur), sum x*f, sum y*f, sum f}, combined in rank order.  The
gathered school must equal the unsharded reference run bit-for-bit, the trace
too, and the barycentre sums must agree within 1e-12.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _combine(parts):
    """Rank-order combine, same operators as fsb_kernels.cu combine_ranks()."""
    best, sx, sy, sf = -np.inf, 0.0, 0.0, 0.0
    for p in parts:
        best = p[0] if p[0] > best else best
        sx, sy, sf = sx + p[1], sy + p[2], sf + p[3]
    return best, sx, sy, sf


def _worker(rank, world, port, n, steps, ret):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2507_20173_b200 as fsb

    orc = oracle.Oracle()
    cfg = oracle.baseline_config(n, steps)
    first, count = fsb.shard_range(n, world, rank)
    fish = orc.init(cfg, first=first, n=count)
    trace, bary = [], []
    for t in range(steps):
        orc.move(cfg, t, fish, first=first)
        part = torch.tensor([orc.eat_max(fish), *orc.barycentre_sums(fish)], dtype=torch.float64)
        got = [torch.empty(4, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(got, part)
        best, sx, sy, sf = _combine([g.tolist() for g in got])
        orc.eat_apply(cfg, best, fish)
        trace.append(best)
        bary.append((sx, sy, sf))
    shards = [None] * world
    dist.all_gather_object(shards, fish.tobytes())
    if rank == 0:
        ret["school"] = b"".join(shards)
        ret["trace"] = np.array(trace).tobytes()
        ret["bary"] = bary
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,steps", [(1001, 6), (4096, 4), (1, 3), (3, 2)])
def test_two_rank_exchange_matches_unsharded(n, steps):
    import oracle

    world = 2
    mgr = mp.get_context("spawn").Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), n, steps, ret), nprocs=world, join=True,
                       start_method="spawn")
    orc = oracle.Oracle()
    cfg = oracle.baseline_config(n, steps)
    want_fish, want_trace = orc.simulate(cfg)
    assert ret["school"] == want_fish.tobytes()
    assert ret["trace"] == want_trace.tobytes()
    want = orc.barycentre_sums(want_fish)
    got = ret["bary"][-1]
    for a, b in zip(got, want):
        assert abs(a - b) <= 1e-12 * abs(b)


def test_shard_partition_covers_global_indices():
    import paper_2507_20173_b200 as fsb

    for world in (2, 3, 8):
        n = 10**9
        spans = [fsb.shard_range(n, world, r) for r in range(world)]
        assert spans[0][0] == 0
        assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert spans[-1][0] + spans[-1][1] == n
        assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1

"""The in-graph exchange of a world_size > 1 run, on ONE GPU.

`fsb_engine_run` with world_size > 1 captures one CUDA graph per rank: step
kernel k -> ncclAllGather of the 4-scalar rank partials -> step kernel k+1,
which combines them in rank order (fsb_engine.cu build_graph / exchange).  NCCL
refuses two ranks on one device and this pool gives one GPU per call, so the
test points FSB_NCCL_LIB at tests/cpp/libnccl_shim.so -- a stand-in for the
five NCCL entry points whose allgather is a D2H copy, a host node that meets
the other ranks in shared memory and an H2D copy, all captured in the graph
like NCCL's kernel -- and runs each rank in its own process on cuda:0.  No
kernel waits for another rank's kernel (only host callbacks wait), so the
processes can time-slice the GPU.  Everything but NCCL's own transport is the
product path: the unique-id bootstrap, fsb_engine_create at world 2-3, the
shard partition with global fish indices, the graph with exchange nodes (no
PDL across them), the rank-order combine in the next kernel, the trailing eat,
the split run.  The gathered school, the trace on every rank and the
barycentre must equal the unsharded oracle's.
"""
import os
import time

import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from conftest import ROOT, bits, unhex

# multi-process tests: a bound, so a lost rank fails the test instead of stalling the suite
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

SHIM = os.path.join(ROOT, "tests", "cpp", "libnccl_shim.so")
BARY_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def need_gpu_and_shim():
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")
    if not os.path.exists(SHIM):
        pytest.fail("tests/cpp/libnccl_shim.so is missing: run __graft_entry__.build()")


def ocfg(cfg):
    return oracle.Config.make(num_fish=cfg.num_fish, pond_size=cfg.pond_size, weight_scale=cfg.weight_scale,
                              num_steps=cfg.num_steps, seed=cfg.seed, step_base=cfg.step_base)


def _rank_worker(rank, world, uid, n, steps, split, kw, ret):
    """One rank = one process on cuda:0, exchanging through the shim."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["FSB_NCCL_LIB"] = SHIM  # before the engine dlopens "NCCL"
    import paper_2507_20173_b200 as fsb_

    cfg = fsb_.baseline_config(n, steps)
    with fsb_.Engine(cfg, device=0, rank=rank, world_size=world, nccl_unique_id=uid, strategy="stream", **kw) as e:
        e.init()
        if split:  # two graph launches: the second starts from the first one's trailing eat
            t0, b0, _ = e.run(0, split, barycentre=True)
            t1, b1, _ = e.run(split, steps - split, barycentre=True)
            trace, bary = np.concatenate([t0, t1]), np.concatenate([b0, b1])
        else:
            trace, bary, _ = e.run(0, steps, barycentre=True)
        ret[rank] = (e.download().tobytes(), trace.tobytes(), bary.tobytes(), e.last_strategy()[0],
                     e.last_launches())


@pytest.mark.parametrize("n,steps,world,split,kw", [
    (200_001, 6, 2, 0, {}),                      # odd school, ragged shards
    (200_001, 6, 2, 2, {}),                      # split run
    (300_007, 5, 3, 0, {"static_tiles": True}),  # three ranks, the static-chunk kernel
    (6_000_002, 3, 2, 0, {"ws_tiles": True}),    # the warp-specialised kernel, 3e6 fish per rank
    (5, 4, 2, 0, {}),                            # tiny shards (2 and 3 fish)
])
def test_world_gt1_graph_exchange_on_one_gpu(orc, n, steps, world, split, kw):
    import torch.multiprocessing as mp

    uid = f"/fsb_nccl_shim_t{os.getpid()}_{time.time_ns()}".encode().ljust(128, b"\0")
    ret = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_rank_worker, args=(world, uid, n, steps, split, kw, ret), nprocs=world, join=True,
                       start_method="spawn")
    cfg = fsb.baseline_config(n, steps)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    assert b"".join(ret[r][0] for r in range(world)) == want_fish.tobytes()
    for r in range(world):
        assert ret[r][1] == want_trace.tobytes(), f"rank {r}: trace"
        assert ret[r][3] == "stream"
        # one step kernel per step + the trailing eat of each launch (the exchange adds no kernel of ours)
        assert ret[r][4] == ((steps - split) + 1 if split else steps + 1)
        bary = np.frombuffer(ret[r][2]).reshape(-1, 3)
        assert ret[r][2] == ret[0][2], "ranks disagree on the barycentre sums"
        want = np.array(orc.barycentre_sums(want_fish))
        assert np.all(np.abs(bary[-1] - want) <= BARY_RTOL * np.abs(want))


# ---- BASELINE's multi-GPU configs at full size (C2 G=2, C3 G in {2,4,8}) ----------
def _config_worker(rank, world, uid, n, steps, barrier, ret):
    """A rank of a full-size config: the whole run in one graph, then the FNV
    checksum chained through the ranks in order (rank r continues from rank
    r-1's state: the digest of the gathered school, sim.hpp:154-176)."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["FSB_NCCL_LIB"] = SHIM
    import paper_2507_20173_b200 as fsb_

    cfg = fsb_.baseline_config(n, steps)
    with fsb_.Engine(cfg, device=0, rank=rank, world_size=world, nccl_unique_id=uid) as e:
        e.init()
        trace, bary, _ = e.run(0, steps, barycentre=True)
        ret[("trace", rank)] = trace.tobytes()
        ret[("bary", rank)] = bary[-1].tobytes()
        for r in range(world):
            if r == rank:
                ret["h"] = e.checksum(ret["h"]) if rank else e.checksum()
            barrier.wait()


@pytest.mark.parametrize("name,n,steps,world", [
    ("C2_1e8x50", 10**8, 50, 2),
    ("C3_1e9x20", 10**9, 20, 2),
    ("C3_1e9x20", 10**9, 20, 4),
    ("C3_1e9x20", 10**9, 20, 8),  # 1.25e8 fish per rank: the north_star's 8-GPU weak-scaling share
])
def test_baseline_multi_gpu_configs_sharded_on_one_gpu(golden_baseline, name, n, steps, world):
    """The reference's digests (tests/golden/baseline_digests.json, made by the
    unmodified reference): every step's max_diff on every rank, the final
    checksum over the school gathered in rank order, the barycentre."""
    import torch.multiprocessing as mp

    g = golden_baseline[name]
    uid = f"/fsb_nccl_shim_c{os.getpid()}_{time.time_ns()}".encode().ljust(128, b"\0")
    mgr = mp.get_context("spawn").Manager()
    ret, barrier = mgr.dict(), mgr.Barrier(world)
    mp.start_processes(_config_worker, args=(world, uid, n, steps, barrier, ret), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert [bits(v) for v in np.frombuffer(ret[("trace", r)])] == g["trace_hex"], f"rank {r}: trace"
        assert ret[("bary", r)] == ret[("bary", 0)]
    assert f"{ret['h']:016x}" == g["final_checksum"]
    want = np.array([unhex(v) for v in g["barycentre_fsum"]])
    bary = np.frombuffer(ret[("bary", 0)])
    assert np.all(np.abs(bary - want) <= BARY_RTOL * np.abs(want))

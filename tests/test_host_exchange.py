"""Sharded runs on ONE GPU through the host-exchange mode (FSB_FLAG_HOST_EXCHANGE).

Every shard is a real engine with its own rank, world_size and global fish
offset, running the same step kernels a multi-GPU run does; only the 4-scalar
exchange between move and eat is done by the caller (fsb_engine_partial ->
all-gather in rank order -> fsb_engine_set_partials).  No kernel waits on
another rank's kernel, so G shards may share one device (B200_PROFILING.md:
ranks whose kernels wait on one another must not).  The gathered school must
equal the unsharded oracle run bit-for-bit, the max_diff trace too, and the
barycentre sums must agree within 1e-12 relative -- the SURVEY 8(e) claim that
state and trace are G-independent, checked on the device code path.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from conftest import ROOT, bits

pytestmark = pytest.mark.gpu

BARY_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")


def ocfg(cfg):
    return oracle.Config.make(num_fish=cfg.num_fish, pond_size=cfg.pond_size, weight_scale=cfg.weight_scale,
                              num_steps=cfg.num_steps, seed=cfg.seed, step_base=cfg.step_base)


def _shards(cfg, world, **kw):
    return [fsb.Engine(cfg, device=0, rank=r, world_size=world, host_exchange=True, **kw) for r in range(world)]


def _step(engs, t):
    for e in engs:
        e.move(t)
    parts = np.stack([e.partial() for e in engs])
    for e in engs:
        e.set_partials(parts)
    maxes = [e.eat().max_diff for e in engs]
    assert len({bits(m) for m in maxes}) == 1, "ranks disagree on the global max"
    return maxes[0], parts


# (n, steps, world, engine kwargs): static-chunk and claimed-tile step kernels,
# ragged shards, empty shards (world > n), a shard boundary inside a fish pair
@pytest.mark.parametrize("n,steps,world,kw", [
    (100_003, 6, 2, {}),
    (100_003, 6, 3, {"dynamic_tiles": True}),
    (100_001, 5, 8, {}),
    (6_000_002, 3, 2, {}),  # 3e6 per shard: the claimed-tile kernel by default
    (5, 4, 8, {}),          # three empty shards
    (0, 2, 2, {}),
])
def test_sharded_phases_match_unsharded_oracle(orc, n, steps, world, kw):
    cfg = fsb.baseline_config(n, steps)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    engs = _shards(cfg, world, **kw)
    try:
        assert sum(e.count for e in engs) == n
        assert [e.first for e in engs] == [fsb.shard_range(n, world, r)[0] for r in range(world)]
        for e in engs:
            e.init()
        trace = []
        for t in range(steps):
            m, _ = _step(engs, t)
            trace.append(m)
        assert np.array(trace).tobytes() == want_trace.tobytes()
        got = np.concatenate([e.download() for e in engs]) if n else np.empty(0, dtype=fsb.FISH_DTYPE)
        assert got.tobytes() == want_fish.tobytes()
        if n:
            sums = [e.barycentre()[0] for e in engs]
            want = orc.barycentre_sums(want_fish)
            for s in sums:
                assert np.all(np.abs(s - want) <= BARY_RTOL * np.abs(want))
    finally:
        for e in engs:
            e.close()


def test_host_exchange_rejects_partials_of_another_step(orc):
    """A rank that moved twice (or skipped a move) carries another exchange
    epoch in its partial: set_partials refuses the gathered set on every rank."""
    cfg = fsb.baseline_config(10_000, 3)
    engs = _shards(cfg, 2)
    try:
        for e in engs:
            e.init()
            e.move(0)
        engs[0].move(1)
        parts = np.stack([e.partial() for e in engs])
        assert parts.shape == (2, 5) and parts[0, 4] != parts[1, 4]
        for e in engs:
            with pytest.raises(fsb.FsbError, match="another step"):
                e.set_partials(parts)
        engs[1].move(1)
        parts = np.stack([e.partial() for e in engs])
        for e in engs:
            e.set_partials(parts)
        assert bits(engs[0].eat().max_diff) == bits(engs[1].eat().max_diff)
    finally:
        for e in engs:
            e.close()


def test_host_exchange_errors(orc):
    cfg = fsb.baseline_config(10_000, 3)
    engs = _shards(cfg, 2)
    try:
        for e in engs:
            e.init()
            e.move(0)
        with pytest.raises(fsb.FsbError):  # eat before the partials are exchanged
            engs[0].eat()
        parts = np.stack([e.partial() for e in engs])
        with pytest.raises(fsb.FsbError):  # partials out of rank order
            engs[0].set_partials(parts[::-1])
        with pytest.raises(fsb.FsbError):  # wrong count
            engs[0].set_partials(parts[:1])
        with pytest.raises(fsb.FsbError):  # the step loop needs an in-graph exchange
            engs[0].run(1, 2)
        with pytest.raises(fsb.FsbError):
            engs[0].simulate()
        engs[0].set_partials(parts)
        engs[0].eat()
        # a second move invalidates the exchanged partials again
        engs[0].move(1)
        with pytest.raises(fsb.FsbError):
            engs[0].eat()
    finally:
        for e in engs:
            e.close()
    # one rank with the flag is an ordinary engine (run works)
    with fsb.Engine(cfg, device=0, host_exchange=True) as e:
        trace, _, _ = e.simulate(barycentre=False)
        _, want_trace = orc.simulate(ocfg(cfg))
        assert trace.tobytes() == want_trace.tobytes()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, steps, ret):
    """One process per shard, both on cuda:0, the exchange over torch.distributed
    (gloo): what a caller with its own communicator does."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2507_20173_b200 as fsb_

    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = fsb_.baseline_config(n, steps)
    with fsb_.Engine(cfg, device=0, rank=rank, world_size=world, host_exchange=True) as e:
        e.init()
        trace = []
        for t in range(steps):
            e.move(t)
            mine = torch.from_numpy(e.partial())
            got = [torch.empty(5, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(got, mine)
            e.set_partials(torch.stack(got).numpy())
            trace.append(e.eat().max_diff)
        shards = [None] * world
        dist.all_gather_object(shards, e.download().tobytes())
    if rank == 0:
        ret["school"] = b"".join(shards)
        ret["trace"] = np.array(trace).tobytes()
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_gloo_exchange(orc):
    import torch.multiprocessing as mp

    n, steps, world = 200_001, 5, 2
    ret = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_gloo_worker, args=(world, _free_port(), n, steps, ret), nprocs=world, join=True,
                       start_method="spawn")
    want_fish, want_trace = orc.simulate(ocfg(fsb.baseline_config(n, steps)))
    assert ret["trace"] == want_trace.tobytes()
    assert ret["school"] == want_fish.tobytes()

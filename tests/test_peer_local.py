"""The NVLink peer exchange (FSB_FLAG_PEER_EXCHANGE) with world_size > 1 on ONE
GPU: G engines of one process, connected by their window pointers
(fsb_engine_peer_connect_local).  Every rank's step kernel stores its partial
into EVERY rank's window and releases its epoch flag; every rank's eat kernel
acquires all G flags of the epoch and combines the G slots in rank order -- the
same device code a multi-GPU run executes, with the peers' windows in the same
HBM instead of across NVLink.

Ranks whose kernels wait on one another must not run concurrently on one GPU
(B200_PROFILING.md), so the steps are driven through the phase API: every
rank's move (each call returns when its kernel has finished, flags released)
before any rank's eat, whose flag acquires then find every flag already set.
School, trace and barycentre must equal the unsharded oracle (bit-exact; sums
within 1e-12 relative).
"""
import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from conftest import bits

pytestmark = pytest.mark.gpu

BARY_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")


def ocfg(cfg):
    return oracle.Config.make(num_fish=cfg.num_fish, pond_size=cfg.pond_size, weight_scale=cfg.weight_scale,
                              num_steps=cfg.num_steps, seed=cfg.seed, step_base=cfg.step_base)


def _ranks(cfg, world, **kw):
    engs = [fsb.Engine(cfg, device=0, rank=r, world_size=world, peer=True, **kw) for r in range(world)]
    for e in engs:
        e.peer_connect_local(engs)
    return engs


@pytest.mark.parametrize("n,steps,world,kw", [
    (100_003, 5, 2, {}),
    (100_003, 5, 3, {"dynamic_tiles": True}),
    (100_001, 4, 4, {"ws_tiles": True}),
    (6_000_002, 3, 2, {}),  # 3e6 per shard: the claimed-tile kernel by default
    (5, 3, 4, {}),          # empty shards still push their identity partial
])
def test_peer_exchange_local_ranks_match_unsharded_oracle(orc, n, steps, world, kw):
    cfg = fsb.baseline_config(n, steps)
    want_fish, want_trace = orc.simulate(ocfg(cfg))
    engs = _ranks(cfg, world, **kw)
    try:
        for e in engs:
            e.init()
        trace = []
        for t in range(steps):
            for e in engs:
                e.move(t)
            maxes = [e.eat().max_diff for e in engs]
            assert len({bits(m) for m in maxes}) == 1, "ranks disagree on the global max"
            trace.append(maxes[0])
        assert np.array(trace).tobytes() == want_trace.tobytes()
        got = np.concatenate([e.download() for e in engs])
        assert got.tobytes() == want_fish.tobytes()
        # the barycentre of the final state: the last move's sums, read back
        # from each rank's own window (the eat does not change x, y or f)
        want = orc.barycentre_sums(want_fish)
        for e in engs:
            s = e.barycentre()[0]
            if n:
                assert np.all(np.abs(s - want) <= BARY_RTOL * np.abs(want))
    finally:
        for e in engs:
            e.close()


def test_peer_connect_local_errors():
    cfg = fsb.baseline_config(1000, 2)
    engs = _ranks(cfg, 2)
    other = fsb.Engine(cfg, device=0, rank=1, world_size=3, peer=True)
    plain = fsb.Engine(cfg, device=0)
    try:
        with pytest.raises(fsb.FsbError):  # wrong count
            engs[0].peer_connect_local(engs[:1])
        with pytest.raises(fsb.FsbError):  # ranks out of order
            engs[0].peer_connect_local(engs[::-1])
        with pytest.raises(fsb.FsbError):  # another world size
            engs[0].peer_connect_local([engs[0], other])
        with pytest.raises(fsb.FsbError):  # not a peer-exchange engine
            plain.peer_connect_local([plain])
    finally:
        for e in engs + [other, plain]:
            e.close()


def test_peer_exchange_reports_a_rank_that_never_publishes(orc, monkeypatch):
    """Failure detection: rank 1 never moves, so rank 0's eat kernel never sees
    its partial; the kernel gives up after FSB_PEER_TIMEOUT_S (here 0.5 s; a
    single bounded wait, no kernel waits on another), marks its window, and the
    call fails with the NCCL/exchange error instead of hanging the GPU.  The
    failed eat applied nothing, so once the late rank has published, the retry
    gives the oracle's state."""
    monkeypatch.setenv("FSB_PEER_TIMEOUT_S", "0.5")
    cfg = fsb.baseline_config(10_000, 2)
    engs = _ranks(cfg, 2)
    try:
        for e in engs:
            e.init()
        engs[0].move(0)
        with pytest.raises(fsb.FsbError, match="did not all arrive"):
            engs[0].eat()
        engs[1].move(0)  # the late rank catches up: the exchange works again
        m1, m0 = engs[1].eat().max_diff, engs[0].eat().max_diff
        fish = orc.init(ocfg(cfg))
        orc.move(ocfg(cfg), 0, fish)
        assert bits(m0) == bits(m1) == bits(orc.eat(ocfg(cfg), fish))
        assert np.concatenate([e.download() for e in engs]).tobytes() == fish.tobytes()
    finally:
        for e in engs:
            e.close()

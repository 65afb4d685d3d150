"""The NVLink peer exchange (FSB_FLAG_PEER_EXCHANGE) between PROCESSES: every
rank exports its exchange window as a CUDA IPC handle (fsb_engine_peer_handle),
the handles travel over the caller's channel, and fsb_engine_peer_connect maps
all of them -- the path a torchrun job takes (bench.py --peer), here with both
ranks on the one GPU of this pool (the peers' windows then live in the same
HBM instead of across NVLink; the IPC export, the mapping of another process's
memory and the device protocol are the same).

Ranks whose kernels wait on one another must not run concurrently on one GPU
(B200_PROFILING.md), so the steps go through the phase API with a host barrier
between the phases: every rank's move kernel has finished -- its partial stored
into every rank's window, its epoch flag released -- before any rank's eat
kernel acquires the flags.  School and trace must equal the unsharded oracle.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2507_20173_b200 as fsb
from conftest import ROOT

# multi-process tests: a bound, so a lost rank fails the test instead of stalling the suite
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fsb.device_count() == 0:
        pytest.fail("no CUDA device: the GPU tests must run on a B200")


def ocfg(cfg):
    return oracle.Config.make(num_fish=cfg.num_fish, pond_size=cfg.pond_size, weight_scale=cfg.weight_scale,
                              num_steps=cfg.num_steps, seed=cfg.seed, step_base=cfg.step_base)


def _rank_worker(rank, world, n, steps, kw, handles, barrier, ret):
    import sys

    sys.path.insert(0, ROOT)
    import paper_2507_20173_b200 as fsb_

    cfg = fsb_.baseline_config(n, steps)
    with fsb_.Engine(cfg, device=0, rank=rank, world_size=world, peer=True, **kw) as e:
        handles[rank] = e.peer_handle()
        barrier.wait()
        e.peer_connect([handles[r] for r in range(world)])
        barrier.wait()  # every window mapped before anyone stores into it
        e.init()
        trace = []
        for t in range(steps):
            e.move(t)
            barrier.wait()  # all moves finished: partials and flags of this epoch are in every window
            trace.append(e.eat().max_diff)
            barrier.wait()
        ret[rank] = (e.download().tobytes(), np.array(trace).tobytes())
        barrier.wait()  # nobody unmaps a window a peer may still address


@pytest.mark.parametrize("n,steps,world,kw", [
    (200_001, 5, 2, {}),
    (300_007, 4, 3, {"ws_tiles": True}),
])
def test_peer_exchange_between_processes(orc, n, steps, world, kw):
    import torch.multiprocessing as mp

    mgr = mp.get_context("spawn").Manager()
    handles, ret, barrier = mgr.dict(), mgr.dict(), mgr.Barrier(world)
    mp.start_processes(_rank_worker, args=(world, n, steps, kw, handles, barrier, ret), nprocs=world, join=True,
                       start_method="spawn")
    want_fish, want_trace = orc.simulate(ocfg(fsb.baseline_config(n, steps)))
    assert b"".join(ret[r][0] for r in range(world)) == want_fish.tobytes()
    for r in range(world):
        assert ret[r][1] == want_trace.tobytes(), f"rank {r}: trace"

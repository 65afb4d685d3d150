"""CPU model of the peer-exchange protocol (FSB_FLAG_PEER_EXCHANGE) with
world_size 2..4 ranks as processes over shared memory.

Each rank runs the engine's sequence of exchanges: kernel e consumes epoch
e-1 (waits until every rank's flag[(e-1)&1] == e-1, reads the slots, combines
in rank order) and produces epoch e (writes its partial into slot[e&1][rank] of
EVERY rank's window, then sets flag[e&1][rank] = e).  Random delays shuffle the
interleavings; every consumed combine must equal the combine of the values the
ranks produced for that epoch -- i.e. a slot is never overwritten before every
rank has read it (the double-buffer argument in fsb_kernels.cuh).
"""
import multiprocessing as mp
import random
import time

import numpy as np
import pytest


def _rank(rank, world, epochs, slots, flags, out, seed):
    rng = random.Random(seed * 97 + rank)
    s = np.frombuffer(slots.get_obj(), dtype=np.float64).reshape(world, 2, world)  # [window][parity][rank]
    f = np.frombuffer(flags.get_obj(), dtype=np.int64).reshape(world, 2, world)
    got = np.frombuffer(out.get_obj(), dtype=np.float64).reshape(world, epochs + 1)
    for e in range(1, epochs + 1):
        if e > 1:  # consume epoch e-1 from my own window
            b = (e - 1) & 1
            for q in range(world):
                while f[rank, b, q] != e - 1:
                    time.sleep(0)
            got[rank, e - 1] = max(s[rank, b, q] for q in range(world))
        time.sleep(rng.random() * 2e-4)  # "the step kernel"
        value = float(e * 1000 + rank * 7 + rng.randint(0, 5))
        b = e & 1
        for q in range(world):  # push into every window, then release the flag
            s[q, b, rank] = value
            f[q, b, rank] = e
        got[rank, 0] = 0.0


def _expected(world, epochs, seed):
    exp = np.zeros(epochs + 1)
    for e in range(1, epochs + 1):
        vals = []
        for r in range(world):
            rng = random.Random(seed * 97 + r)
            v = None
            for k in range(1, e + 1):
                rng.random()
                v = float(k * 1000 + r * 7 + rng.randint(0, 5))
            vals.append(v)
        exp[e] = max(vals)
    return exp


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_protocol_never_reads_a_reused_slot(world):
    epochs, seed = 60, world
    ctx = mp.get_context("fork")
    slots = ctx.Array("d", world * 2 * world)
    flags = ctx.Array("q", world * 2 * world)
    out = ctx.Array("d", world * (epochs + 1))
    procs = [ctx.Process(target=_rank, args=(r, world, epochs, slots, flags, out, seed)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    got = np.frombuffer(out.get_obj(), dtype=np.float64).reshape(world, epochs + 1)
    exp = _expected(world, epochs, seed)
    for r in range(world):
        assert np.array_equal(got[r, 1:epochs], exp[1:epochs]), f"rank {r}"

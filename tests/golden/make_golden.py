#!/usr/bin/env python3
"""Generate tests/golden/ fixtures from the UNMODIFIED reference.

Every number written here comes from oracle/_ref/libfsbref.so -- the reference
headers (/root/reference/proj/include, read-only) compiled with the reference's
own Release flags by oracle/Makefile -- run with the sequential construct
(RunConfig{1, static:0, Sequential}), which is the correct oracle; the
reference's default Reduction construct drops a worker's partial max
(executor.hpp:243, SURVEY.md finding 2).  Barycentre sums (a north_star query
with no reference counterpart) are exactly-rounded sums (math.fsum) of the fp64
products x*f, y*f and of f over the reference's final state.

Run here (needs /root/reference):  python tests/golden/make_golden.py [--big]
--big adds C2 (1e8 x 50, ~3 min, 4 GB RAM); --huge adds C3 (1e9 x 20, ~10 min, 40 GB).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import FISH_DTYPE, Config, Reference, baseline_config  # noqa: E402


def hexd(v: float) -> str:
    return struct.pack("<d", float(v)).hex()


def _chunked(fn, n, step=1 << 22):
    for lo in range(0, n, step):
        yield from fn(lo, min(n, lo + step)).tolist()


def fsum_bary(fish) -> list:
    """Exactly rounded sums of the fp64 products (streamed: O(chunk) memory)."""
    n = len(fish)
    f = fish["current_objective"]
    return [math.fsum(_chunked(lambda a, b: fish["x"][a:b] * f[a:b], n)),
            math.fsum(_chunked(lambda a, b: fish["y"][a:b] * f[a:b], n)),
            math.fsum(_chunked(lambda a, b: f[a:b], n))]


def cfg_dict(c: Config) -> dict:
    return {k: getattr(c, k) for k, _ in Config._fields_}


# Small whole-run cases: every step's checksum and max_diff, plus the final
# state for N <= 4096.  Chosen to cover the BASELINE mapping, the reference
# defaults (acceptance.cpp:63-102 uses 1e4 x 100, seed 7), clamp-heavy walls
# (test_sim.cpp:103-124), aggressive eats (test_sim.cpp:193-207), 1 fish and
# non-multiple-of-warp sizes.
SMALL = {
    "baseline_1000x20": dict(num_fish=1000, num_steps=20, seed=7, pond_size=200.0, weight_scale=1.0, step_base=0.1),
    "defaults_10000x100_seed7": dict(num_fish=10000, num_steps=100, seed=7, pond_size=200.0, weight_scale=10.0, step_base=1.0),
    "walls_200x50": dict(num_fish=200, num_steps=50, seed=1, pond_size=10.0, weight_scale=10.0, step_base=100.0),
    "band_500x60": dict(num_fish=500, num_steps=60, seed=42, pond_size=200.0, weight_scale=10.0, step_base=10.0),
    "small_500x20_seed42": dict(num_fish=500, num_steps=20, seed=42, pond_size=200.0, weight_scale=10.0, step_base=1.0),
    "one_fish_x30": dict(num_fish=1, num_steps=30, seed=3, pond_size=200.0, weight_scale=10.0, step_base=1.0),
    "ragged_4097x7": dict(num_fish=4097, num_steps=7, seed=11, pond_size=50.0, weight_scale=3.0, step_base=0.7),
    "empty_0x5": dict(num_fish=0, num_steps=5, seed=1, pond_size=200.0, weight_scale=10.0, step_base=1.0),
    "c4_4096x2000": dict(num_fish=4096, num_steps=2000, seed=7, pond_size=200.0, weight_scale=1.0, step_base=0.1),
}


def gen_small(ref: Reference) -> dict:
    out = {}
    arrays = {}
    for name, kw in SMALL.items():
        cfg = Config.make(**kw)
        fish = ref.init(cfg)
        init_ck = ref.checksum(fish)
        per_step_ck, trace = [], []
        for t in range(cfg.num_steps):
            ref.move(cfg, t, fish)
            trace.append(ref.eat(cfg, fish))
            per_step_ck.append(ref.checksum(fish))
        # cross-check the phase-by-phase run against the reference's simulate()
        fin, tr, _ = ref.simulate(cfg)
        assert ref.checksum(fin) == per_step_ck[-1] if cfg.num_steps else True
        assert [hexd(v) for v in tr] == [hexd(v) for v in trace]
        out[name] = {
            "config": cfg_dict(cfg),
            "init_checksum": f"{init_ck:016x}",
            "step_checksums": [f"{c:016x}" for c in per_step_ck],
            "trace_hex": [hexd(v) for v in trace],
            "barycentre_fsum": [hexd(v) for v in fsum_bary(fish)],
        }
        if cfg.num_fish <= 4097:
            arrays[name + "__final"] = fish.copy()
            arrays[name + "__init"] = ref.init(cfg)
        print(f"  {name}: final {per_step_ck[-1] if per_step_ck else init_ck:016x}", flush=True)
    np.savez_compressed(os.path.join(HERE, "small_states.npz"), **arrays)
    return out


def gen_eat_examples(ref: Reference) -> dict:
    """The hand-built Schools of test_sim.cpp:139-191, run through the reference eat."""
    cases = {
        # test_sim.cpp:139-162 (SimConfig defaults: weight band [1, 20])
        "three_fish": [(0, 0, 5.0, 10.0, 4.0), (0, 0, 5.0, 5.0, 5.0), (0, 0, 5.0, 7.0, 9.0)],
        # test_sim.cpp:172-181
        "no_improvement": [(0, 0, 3.0, 5.0, 5.0), (0, 0, 4.0, 2.0, 2.0)],
        # test_sim.cpp:183-191
        "lone_fish": [(0, 0, 5.0, 9.0, 6.5)],
        # test_sim.cpp:164-170
        "empty": [],
        # clamp at the top of the band and at the bottom
        "band_clamp": [(1, 2, 19.5, 10.0, 0.0), (3, 4, 1.2, 0.0, 10.0), (5, 6, 2.0, 3.0, 1.0)],
    }
    cfg = Config.make()
    out = {}
    for name, rows in cases.items():
        fish = np.array(rows, dtype=FISH_DTYPE) if rows else np.zeros(0, dtype=FISH_DTYPE)
        before = fish.copy()
        m = ref.eat(cfg, fish, threads=1)
        out[name] = {
            "input": [[hexd(v) for v in r] for r in before.tolist()],
            "max_diff": hexd(m),
            "weights": [hexd(v) for v in fish["weight"]],
        }
    return out


def gen_rng_kat(ref: Reference) -> dict:
    tuples = [(1, 0, 0, 0), (7, 0, ~0 & 0xFFFFFFFFFFFFFFFF, 2), (7, 123456789, 99, 1),
              (42, 2**33 + 5, 7, 0), (0xDEADBEEF, 999_999_999, 19, 1), (0, 0, 0, 0)]
    return {
        "bits": [[list(map(str, t)), str(ref.L.ref_bits(*t))] for t in tuples],
        "objective": [[a, b, p, hexd(ref.L.ref_objective(a, b, p))]
                      for a, b, p in [(100.0, 100.0, 200.0), (103.0, 104.0, 200.0), (0.0, 0.0, 200.0),
                                      (200.0, 3.25, 200.0), (1.5, 9.75, 10.0)]],
    }


BIG = {
    "C0_1e6x100": (10**6, 100),
    "C1_1e7x100": (10**7, 100),
    "C4_4096x100000": (4096, 100000),
}
BIGGER = {"C2_1e8x50": (10**8, 50)}
HUGE = {"C3_1e9x20": (10**9, 20)}


def gen_baseline(ref: Reference, which: dict, path: str) -> None:
    data = json.load(open(path)) if os.path.exists(path) else {}
    for name, (n, t) in which.items():
        if name in data:
            continue
        cfg = baseline_config(n, t)
        fish, trace, secs = ref.simulate(cfg)
        entry = {
            "config": cfg_dict(cfg),
            "init_checksum": f"{ref.checksum(ref.init(cfg)):016x}" if n <= 10**8 else None,
            "final_checksum": f"{ref.checksum(fish):016x}",
            "trace_hex": [hexd(v) for v in trace] if t <= 1000 else None,
            "trace_last_hex": hexd(trace[-1]),
            "trace_sum_fsum_hex": hexd(math.fsum(trace.tolist())),
            "barycentre_fsum": [hexd(v) for v in fsum_bary(fish)],
            "ref_seconds_total": secs[0],
        }
        if name.startswith("C4"):
            entry["trace_every_1000_hex"] = [hexd(v) for v in trace[999::1000]]
        del fish
        data[name] = entry
        print(f"  {name}: {entry['final_checksum']} ({secs[0]:.1f}s)", flush=True)
        json.dump(data, open(path, "w"), indent=1)


def gen_step_digests(ref: Reference, path: str) -> None:
    """SURVEY 8(d) gates: the reference checksum after EVERY step for C0 and C1,
    and after every 1000th step for C4 (ref_step_digests, in place)."""
    import ctypes

    data = json.load(open(path)) if os.path.exists(path) else {}
    L = ref.L
    L.ref_step_digests.restype = ctypes.c_int
    L.ref_step_digests.argtypes = [ctypes.POINTER(Config), ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    for name, every in (("C0_1e6x100", 1), ("C1_1e7x100", 1), ("C4_4096x100000", 1000)):
        if name not in data or "step_checksums" in data[name]:
            continue
        cfg = Config.make(**data[name]["config"])
        digests = np.zeros(cfg.num_steps // every, dtype=np.uint64)
        assert L.ref_step_digests(ctypes.byref(cfg), every, digests.ctypes.data, None) == 0
        data[name]["step_checksums"] = [f"{int(d):016x}" for d in digests]
        data[name]["step_checksums_every"] = every
        assert data[name]["step_checksums"][-1] == data[name]["final_checksum"]
        print(f"  {name}: {len(digests)} per-step digests", flush=True)
        json.dump(data, open(path, "w"), indent=1)


def gen_huge(ref: Reference, path: str) -> None:
    """C3 (1e9 x 20): the reference school is 40 GB, so the reference computes
    the digests in place (ref_simulate_digest: sequential construct, checksum
    of init and final school, trace, Neumaier long-double barycentre sums)."""
    import ctypes

    data = json.load(open(path)) if os.path.exists(path) else {}
    if "C3_1e9x20" in data:
        return
    L = ref.L
    L.ref_simulate_digest.restype = ctypes.c_int
    L.ref_simulate_digest.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p, ctypes.c_void_p]
    cfg = baseline_config(10**9, 20)
    ic, fc = ctypes.c_uint64(), ctypes.c_uint64()
    trace = np.zeros(cfg.num_steps)
    bary = (ctypes.c_longdouble * 3)()
    rc = L.ref_simulate_digest(ctypes.byref(cfg), ctypes.byref(ic), ctypes.byref(fc), trace.ctypes.data,
                               ctypes.cast(bary, ctypes.c_void_p))
    assert rc == 0
    data["C3_1e9x20"] = {
        "config": cfg_dict(cfg),
        "init_checksum": f"{ic.value:016x}",
        "final_checksum": f"{fc.value:016x}",
        "trace_hex": [hexd(v) for v in trace],
        "trace_last_hex": hexd(trace[-1]),
        "barycentre_fsum": [hexd(v) for v in bary],
        "barycentre_method": "Neumaier-compensated long double over fp64 products (reference final state)",
    }
    json.dump(data, open(path, "w"), indent=1)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--huge", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    ref = Reference()
    if not a.skip_small:
        print("small runs", flush=True)
        gold = {"rng": gen_rng_kat(ref), "eat_examples": gen_eat_examples(ref), "runs": gen_small(ref)}
        json.dump(gold, open(os.path.join(HERE, "small_runs.json"), "w"), indent=1)
    print("baseline configs", flush=True)
    path = os.path.join(HERE, "baseline_digests.json")
    gen_baseline(ref, BIG, path)
    gen_step_digests(ref, path)
    if a.big:
        gen_baseline(ref, BIGGER, path)
    if a.huge:
        gen_huge(ref, path)


if __name__ == "__main__":
    main()

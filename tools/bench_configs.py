#!/usr/bin/env python3
"""Time every BASELINE.json config (and variants) on one GPU; one JSON line each.

    python tools/bench_configs.py [--only C1,C4] [--reps 3]

Device time of the step loop (engine.run's CUDA events), median of reps, after
one warm-up run of the same shape.  Not the driver's bench (that is bench.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2507_20173_b200 as fsb  # noqa: E402

CONFIGS = {
    "C0": (1_000_000, 100),
    "C1": (10_000_000, 100),
    "C2": (100_000_000, 50),
    "C3": (1_000_000_000, 20),
    "C4": (4096, 100_000),
}


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def time_cfg(name, n, t, strategy, alternate, reps, bulk=False, pdl=True, checked=False):
    cfg = fsb.baseline_config(n, t)
    with fsb.Engine(cfg, strategy=strategy, alternate=alternate, bulk=bulk, pdl=pdl, checked=checked) as eng:
        eng.init()
        eng.run(0, t)  # warm-up of the same shape (graph instantiation)
        secs = []
        for r in range(reps):
            eng.init()
            _, _, tm = eng.run(0, t)
            secs.append(tm.seconds_loop)
        s = statistics.median(secs)
        ck = None
    rate = n * t / s
    return {"config": name, "fish": n, "steps": t, "strategy": strategy, "alternate": alternate, "bulk": bulk,
            "pdl": pdl, "checked": checked,
            "seconds": s, "fish_updates_per_s": rate, "us_per_step": 1e6 * s / t,
            "hbm_frac_80B": rate * 80 / 1e9 / peak(), "hbm_frac_64B": rate * 64 / 1e9 / peak()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C0,C1,C2,C3,C4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--variants", action="store_true", help="also stream/persistent and alternate on/off")
    ap.add_argument("--bulk-ab", action="store_true", help="also the cp.async.bulk ring step kernel")
    ap.add_argument("--pdl-ab", action="store_true", help="also without programmatic dependent launch")
    ap.add_argument("--grid-ab", action="store_true", help="also the persistent cooperative-grid strategy")
    ap.add_argument("--checked-ab", action="store_true", help="also with the fp64 guards always evaluated")
    a = ap.parse_args()
    for name in a.only.split(","):
        n, t = CONFIGS[name]
        plans = [("auto", True, False)]
        if a.bulk_ab and n > 32768:
            plans += [("stream", True, True)]
        if a.variants:
            plans += [("stream", False, False)]
            if n <= 32768:
                plans += [("stream", True, False), ("persistent", True, False)]
        for strategy, alt, bulk in plans:
            print(json.dumps(time_cfg(name, n, t, strategy, alt, a.reps, bulk)), flush=True)
        if a.pdl_ab and n > 32768:
            print(json.dumps(time_cfg(name, n, t, "stream", True, a.reps, False, pdl=False)), flush=True)
        if a.checked_ab and n > 32768:
            for bulk in (True, False):
                print(json.dumps(time_cfg(name, n, t, "stream", True, a.reps, bulk, checked=True)), flush=True)
        if a.checked_ab and n <= 16384:  # the persistent kernel with its guarded (non-in-range) paths
            print(json.dumps(time_cfg(name, n, t, "auto", True, a.reps, False, checked=True)), flush=True)
        if a.grid_ab and n > 16384:
            print(json.dumps(time_cfg(name, n, t, "grid", True, a.reps, False)), flush=True)


if __name__ == "__main__":
    main()

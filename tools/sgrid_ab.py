#!/usr/bin/env python3
"""A/B of shared-memory-grid builds (tools/variants.py) at C0, with and without
the barycentre trace; one JSON line per (variant, fish, bary), rounds interleaved.

    python tools/sgrid_ab.py default sguntagged [--rounds 3] [--fish 1000000,200000]

Each variant runs in its own process (FSB_LIB), device time of engine.run's
step loop, median of 5 after a warm-up run; the trace digest is printed so the
variants can be checked bit-identical.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, statistics, sys
sys.path.insert(0, sys.argv[1])
import paper_2507_20173_b200 as fsb
n, t, bary = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1"
cfg = fsb.baseline_config(n, t)
with fsb.Engine(cfg, strategy="grid") as eng:
    eng.init()
    eng.run(0, t, barycentre=bary)
    secs, digest = [], None
    for _ in range(5):
        eng.init()
        tr, b, tm = eng.run(0, t, barycentre=bary)
        secs.append(tm.seconds_loop)
        digest = hashlib.sha1(tr.tobytes() + (b.tobytes() if b is not None else b"")).hexdigest()[:16]
    print(json.dumps({"us_per_step": 1e6 * statistics.median(secs) / t, "digest": digest,
                      "strategy_used": eng.last_strategy()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--fish", default="1000000")
    args = ap.parse_args()
    for r in range(args.rounds):
        for n in [int(x) for x in args.fish.split(",")]:
            for bary in (False, True):
                for name in args.variants:
                    lib = os.path.join(ROOT, "build", "variants", f"libfsb_{name}.so")
                    env = dict(os.environ, FSB_LIB=lib)
                    p = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(n), "100", "1" if bary else "0"],
                                       capture_output=True, text=True, env=env, timeout=300)
                    d = {"variant": name, "round": r, "fish": n, "bary": bary}
                    if p.returncode:
                        d["error"] = p.stderr[-400:]
                    else:
                        d.update(json.loads(p.stdout.strip().splitlines()[-1]))
                    print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()

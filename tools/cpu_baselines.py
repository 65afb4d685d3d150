#!/usr/bin/env python3
"""CPU baseline rows of SURVEY.md 8(d) / BASELINE.md section 3, timed on this host.

For each BASELINE config, the reference's step loop (oracle/_ref = the reference
headers compiled with its own flags) on a bounded sample of steps:
  (i)   RunConfig{1, static:0, Sequential}      -- the correct oracle, 1 core
  (ii)  RunConfig{nproc, static:50, Reduction}  -- the reference default (timing
        only: its max drops a worker's partial, executor.hpp:243)
  (iii) RunConfig{nproc, static:50, CriticalPartial} -- correct parallel, mutex per item
One JSON line per (config, row).  TEST/MEASUREMENT TOOL: uses oracle/.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# (fish, sampled steps) per config; C3 (1e9) is extrapolated from C2 as BASELINE.md says.
SAMPLES = {"C0": (10**6, 20), "C1": (10**7, 5), "C2": (10**8, 2), "C4": (4096, 20000)}
ROWS = [
    ("sequential", 1, oracle.STATIC, 0, oracle.SEQUENTIAL),
    ("reduction(default,invalid)", None, oracle.STATIC, 50, oracle.REDUCTION),
    ("critical-partial", None, oracle.STATIC, 50, oracle.CRITICAL_PARTIAL),
]


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return "unknown"


def main():
    ref = oracle.Reference()
    nproc = os.cpu_count() or 1
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SAMPLES)
    for name in only:
        n, steps = SAMPLES[name]
        for row, threads, sched, chunk, construct in ROWS:
            th = threads or nproc
            s = steps if construct != oracle.CRITICAL_PARTIAL else max(1, steps // 5)
            cfg = oracle.baseline_config(n, s + 1)
            total, _, _ = ref.time_steps(cfg, warmup=1, steps=s, threads=th, sched=sched, chunk=chunk,
                                         construct=construct)
            print(json.dumps({"config": name, "row": row, "threads": th, "fish": n, "steps_timed": s,
                              "seconds": total, "fish_updates_per_s": n * s / total, "cpu": cpu_model()}),
                  flush=True)


if __name__ == "__main__":
    main()

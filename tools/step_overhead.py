"""Fixed per-step cost of the stream strategy: device time per step against
school size and CTA count (the grid-wide reduction and kernel boundary).

    python tools/step_overhead.py [stream|grid]     # on the GPU box
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_20173_b200 as fsb  # noqa: E402

T = 200
STRATEGY = sys.argv[1] if len(sys.argv) > 1 else "stream"
for n in (2_000, 100_000, 1_000_000, 10_000_000):
    cfg = fsb.baseline_config(n, T)
    with fsb.Engine(cfg, strategy=STRATEGY) as eng:
        auto = eng.grid()[0]
        for ctas in ((148, 296, auto, 2 * auto) if STRATEGY == "stream" else (auto,)):
            eng.set_grid(ctas)
            eng.init()
            eng.run(0, T)
            us = []
            for _ in range(5):
                eng.init()
                _, _, t = eng.run(0, T)
                us.append(t.seconds_loop / T * 1e6)
            print(json.dumps({"strategy": STRATEGY, "fish": n, "ctas": ctas,
                              "us_per_step": round(statistics.median(us), 3)}), flush=True)

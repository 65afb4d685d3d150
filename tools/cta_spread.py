"""spread build (tools/variants.py): per step, the time from the first CTA of the
step kernel done to the last (the work imbalance the kernel boundary waits for).
    FSB_LIB=build/variants/libfsb_spread.so python tools/cta_spread.py"""
import sys, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_20173_b200 as fsb
for n, t in ((3_000_000, 50), (10_000_000, 50), (100_000_000, 10)):
    for kw in (dict(dynamic_tiles=True), dict(static_tiles=True), dict(ws_tiles=True)):
        with fsb.Engine(fsb.baseline_config(n, t), strategy="stream", **kw) as e:
            e.init(); e.run(0, t)
            e.init(); _, _, tm = e.run(0, t)
            print(json.dumps({"fish": n, "kernel": list(kw)[0], "us_per_step": tm.seconds_loop / t * 1e6,
                              "cta_done_spread_us_per_step": tm.seconds_eat / t * 1e6}), flush=True)

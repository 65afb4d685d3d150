"""wgtime build (tools/variants.py): per-step CTA done-time spread and exchange
latency of the warp-specialised persistent grid kernel.
    FSB_LIB=build/variants/libfsb_wgtime.so python tools/wgrid_timing.py 1e7 20"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402

n, t = int(float(sys.argv[1])), int(sys.argv[2])
with fsb.Engine(fsb.baseline_config(n, t), ws_grid=True) as eng:
    eng.init()
    eng.run(0, t, barycentre=True)
    eng.init()
    _, b, tm = eng.run(0, t, barycentre=True)
b = np.asarray(b).reshape(-1, 3)[1:]
print(json.dumps({"fish": n, "us_per_step": tm.seconds_loop / t * 1e6,
                  "cta0_after_first_us": float(np.median(b[:, 0])) / 1e3,
                  "done_spread_us": float(np.median(b[:, 1])) / 1e3,
                  "exchange_us": float(np.median(b[:, 2])) / 1e3}))

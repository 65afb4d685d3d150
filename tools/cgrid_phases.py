"""Phase timing of the cluster-reduced grid kernel (experiment build
build/variants/libfsb_gridtiming.so): CTA 0 after its chunk, leader 0 after
its cluster's partials arrived and after the global fold, per step.

    FSB_LIB=build/variants/libfsb_gridtiming.so python tools/cgrid_phases.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402

T = 200
for n in (2_000, 1_000_000):
    cfg = fsb.baseline_config(n, T)
    with fsb.Engine(cfg, strategy="grid") as eng:
        eng.init()
        eng.run(0, T, barycentre=True)
        eng.init()
        _, bary, t = eng.run(0, T, barycentre=True)
    ts = np.ascontiguousarray(bary).view(np.uint64).reshape(T, 3).astype(np.int64)
    step = ts[1:, 0] - ts[:-1, 0]
    cluster = ts[:, 1] - ts[:, 0]   # CTA 0 done -> all 8 partials at leader 0
    glob = ts[:, 2] - ts[:, 1]      # publish + wait for every cluster + fold
    print(json.dumps({"fish": n, "us_per_step": t.seconds_move / T * 1e6, "step_us": statistics.median(step) / 1e3,
                      "cluster_wait_us": statistics.median(cluster) / 1e3,
                      "global_us": statistics.median(glob) / 1e3}), flush=True)

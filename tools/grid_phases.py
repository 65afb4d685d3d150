"""Phase timing of the flat grid kernel (FSB_FLAG_FLAT_GRID)'s per-step exchange (experiment build
build/variants/libfsb_gridtiming.so): CTA 0's globaltimer after its chunk,
after the arrival barrier and after the fold, per step.

    FSB_LIB=build/variants/libfsb_gridtiming.so python tools/grid_phases.py
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
    with fsb.Engine(cfg, strategy="grid", flat_grid=True) as eng:
        eng.init()
        eng.run(0, T, barycentre=True)
        eng.init()
        _, bary, t = eng.run(0, T, barycentre=True)
    ts = np.ascontiguousarray(bary).view(np.uint64).reshape(T, 3).astype(np.int64)
    chunk = ts[1:, 0] - ts[:-1, 2]   # end of previous fold -> end of this chunk + block reduce
    barrier = ts[:, 1] - ts[:, 0]    # publish + arrive + wait for all CTAs
    fold = ts[:, 2] - ts[:, 1]       # read all CTA partials + block reduce
    print(json.dumps({"fish": n, "us_per_step": t.seconds_move / T * 1e6,
                      "chunk_us": statistics.median(chunk) / 1e3, "barrier_us": statistics.median(barrier) / 1e3,
                      "fold_us": statistics.median(fold) / 1e3}), flush=True)

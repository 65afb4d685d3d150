"""Per-CTA chunk time of the grid kernel's last step (experiment build
build/variants/libfsb_gridcta.so): the spread behind the barrier wait.

    FSB_LIB=build/variants/libfsb_gridcta.so python tools/grid_ctas.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402

T = 1000
for n in (1_000_000, 10_000_000):
    cfg = fsb.baseline_config(n, T)
    with fsb.Engine(cfg, strategy="grid", flat_grid=True) as eng:
        G = eng.grid()[0]
        eng.init()
        trace, bary, _ = eng.run(0, T, barycentre=True)
    us = np.asarray(trace).ravel()[:G] / 1e3
    sm = np.asarray(bary).ravel()[:G].astype(int)
    order = np.argsort(us)
    q = np.percentile(us, [0, 10, 50, 90, 100])
    # by SM: mean chunk time of the SM's CTAs; SMs sorted by id
    per_sm = {}
    for b in range(G):
        per_sm.setdefault(sm[b], []).append(us[b])
    sm_ids = sorted(per_sm)
    sm_mean = np.array([np.mean(per_sm[i]) for i in sm_ids])
    print(json.dumps({"fish": n, "ctas": G, "chunk_us_pct_0_10_50_90_100": [round(v, 2) for v in q],
                      "slowest_ctas": order[-8:].tolist(), "fastest_ctas": order[:8].tolist(),
                      "by_cta_quarter_mean": [round(float(np.mean(us[i * G // 4:(i + 1) * G // 4])), 2) for i in range(4)],
                      "by_sm_half_mean": [round(float(sm_mean[:len(sm_ids) // 2].mean()), 2),
                                          round(float(sm_mean[len(sm_ids) // 2:].mean()), 2)]}), flush=True)

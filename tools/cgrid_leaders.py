"""Every cluster leader's timeline in the last step of the cluster-reduced
grid kernel (experiment build build/variants/libfsb_gridlead.so): when its
cluster's partials were complete and when it had the global total.

    FSB_LIB=build/variants/libfsb_gridlead.so python tools/cgrid_leaders.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402

T = 200
for n in (2_000, 1_000_000):
    cfg = fsb.baseline_config(n, T)
    with fsb.Engine(cfg, strategy="grid") as eng:
        eng.init()
        _, bary, _ = eng.run(0, T, barycentre=True)
    v = np.ascontiguousarray(bary).ravel().view(np.uint64).astype(np.int64)
    nc = int(np.count_nonzero(v[1::2][:150]))
    ready = v[0:2 * nc:2]
    done = v[1:2 * nc:2]
    t0 = ready.min()
    r = (ready - t0) / 1e3
    d = (done - t0) / 1e3
    print(json.dumps({"fish": n, "clusters": nc,
                      "cluster_ready_us_min_med_max": [round(float(x), 2) for x in (r.min(), np.median(r), r.max())],
                      "slowest_clusters": np.argsort(r)[-5:].tolist(),
                      "total_done_us_min_med_max": [round(float(x), 2) for x in (d.min(), np.median(d), d.max())]}),
          flush=True)

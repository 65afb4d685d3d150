"""Interleaved A/B of the compact-state step kernels: device time per step,
8 alternating repetitions per kernel (median, min, max us).

    python tools/ab_kernels.py [dyn,static,bulk] [n:T,n:T,...]      # on the GPU box
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_20173_b200 as fsb  # noqa: E402

KERNELS = {
    "dyn": dict(dynamic_tiles=True),  # one CTA per SM, warps claim tiles
    "static": dict(static_tiles=True),  # 4 CTAs per SM, one static chunk each
    "auto": dict(),
    "cgrid": dict(strategy="grid"),               # cooperative persistent, cluster-reduced exchange
    "persistent": dict(strategy="persistent"),    # one thread-block cluster, state on chip
    "flatgrid": dict(strategy="grid", flat_grid=True),
    "bulk": dict(bulk=True),          # cp.async.bulk shared-memory ring
    "ws": dict(ws_tiles=True),
    "peer": dict(peer=True),          # the claimed-tile kernel with the peer-window exchange (world 1)
    "peer": dict(peer=True),          # the claimed-tile kernel with the peer-window exchange (world 1)        # warp-specialised: TMA producer warp + 31 consumer warps
}
names = (sys.argv[1] if len(sys.argv) > 1 else "dyn,static,bulk").split(",")
sizes = [(1_000_000, 100), (10_000_000, 100), (100_000_000, 20)]
if len(sys.argv) > 2:
    sizes = [tuple(int(float(v)) for v in item.split(":")) for item in sys.argv[2].split(",")]
for n, t in sizes:
    cfg = fsb.baseline_config(n, t)
    engs = {k: fsb.Engine(cfg, **{"strategy": "stream", **KERNELS[k]}) for k in names}
    for e in engs.values():
        e.init()
        e.run(0, t)
    times = {k: [] for k in engs}
    for rep in range(8):
        for k, e in engs.items():
            e.init()
            _, _, tm = e.run(0, t)
            times[k].append(tm.seconds_loop / t * 1e6)
    for e in engs.values():
        e.close()
    print(json.dumps({"fish": n, **{k: [round(statistics.median(v), 2), round(min(v), 2), round(max(v), 2)]
                                    for k, v in times.items()}}), flush=True)

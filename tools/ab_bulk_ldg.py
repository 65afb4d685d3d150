import sys, statistics, json
sys.path.insert(0, '.')
import paper_2507_20173_b200 as fsb
res = {}
for n, t in ((10_000_000, 100), (100_000_000, 20), (1_000_000, 100)):
    cfg = fsb.baseline_config(n, t)
    engs = {"bulk": fsb.Engine(cfg, strategy="stream", bulk="force"), "ldg": fsb.Engine(cfg, strategy="stream", bulk=False)}
    for e in engs.values():
        e.init(); e.run(0, t)
    times = {k: [] for k in engs}
    for rep in range(8):
        for k, e in engs.items():
            e.init()
            _, _, tm = e.run(0, t)
            times[k].append(tm.seconds_move / t * 1e6)
    for e in engs.values():
        e.close()
    print(json.dumps({"fish": n, **{k: [round(statistics.median(v), 2), round(min(v), 2), round(max(v), 2)] for k, v in times.items()}}), flush=True)

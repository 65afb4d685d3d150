"""One engine run for profilers: python tools/one_run.py N T [kwarg=value ...]
e.g. ncu -k regex:wgrid python tools/one_run.py 1e7 5 ws_grid=1"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_20173_b200 as fsb  # noqa: E402

n, t = int(float(sys.argv[1])), int(sys.argv[2])
kw = {}
for item in sys.argv[3:]:
    k, v = item.split("=")
    kw[k] = v if k == "strategy" else bool(int(v))
with fsb.Engine(fsb.baseline_config(n, t), **kw) as eng:
    eng.init()
    _, _, tm = eng.run(0, t)
    print(f"{n} x {t} {kw}: {tm.seconds_loop / t * 1e6:.2f} us/step, strategy {eng.last_strategy()}", flush=True)

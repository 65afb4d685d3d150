import json, os, statistics, subprocess, sys
ROOT = os.getcwd()
code = r'''
import sys, json, statistics
sys.path.insert(0, ".")
import paper_2507_20173_b200 as fsb
n, t, g = int(float(sys.argv[1])), int(sys.argv[2]), int(sys.argv[3])
with fsb.Engine(fsb.baseline_config(n, t), strategy="stream", dynamic_tiles=True) as e:
    e.set_tile_groups(g)
    e.init(); e.run(0, t)
    xs = []
    for r in range(5):
        e.init(); _, _, tm = e.run(0, t); xs.append(tm.seconds_loop / t * 1e6)
print(json.dumps({"fish": n, "groups": g, "us": statistics.median(xs)}))
'''
for rep in range(2):
    for lib in ("default", "gclaim"):
        for n, t in (("1e7", 100), ("1e8", 20)):
            for g in (0, 8, 16):
                env = dict(os.environ, FSB_LIB=f"build/variants/libfsb_{lib}.so")
                out = subprocess.run([sys.executable, "-c", code, n, str(t), str(g)], capture_output=True, text=True, env=env)
                line = out.stdout.strip() or out.stderr[-300:]
                print(lib, line, flush=True)

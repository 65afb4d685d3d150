"""Interleaved A/B of library builds (tools/variants.py) on one kernel choice:
each variant runs in its own process, rounds alternate, median/min/max us per step.

    python tools/ab_libs.py VARIANTS KERNEL SIZES [ROUNDS]     # on the GPU box
    e.g. python tools/ab_libs.py default,dg4 dyn 9e6:100,1e7:100 3
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
variants = sys.argv[1].split(",")
kernel = sys.argv[2]
sizes = sys.argv[3]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
res = {}
for r in range(rounds):
    for v in variants:
        env = dict(os.environ, FSB_LIB=os.path.join(ROOT, "build", "variants", f"libfsb_{v}.so"))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab_kernels.py"), kernel, sizes],
                             capture_output=True, text=True, env=env)
        for line in out.stdout.splitlines():
            d = json.loads(line)
            res.setdefault((d["fish"], v), []).append(d[kernel][0])
for (n, v), t in sorted(res.items()):
    print(json.dumps({"fish": n, "variant": v, "kernel": kernel, "us": [round(statistics.median(t), 2),
                                                                        round(min(t), 2), round(max(t), 2)]}))

"""Small runs of every kernel and engine path, with cross-checks between them
(compute-sanitizer is not available on the GPU pool; this is the substitute
smoke for bad accesses: every path must agree bit for bit).

    python tools/kernel_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402

n, t = 20_003, 4
cfg = fsb.baseline_config(n, t)
ref = None
for kw in (dict(strategy="stream", static_tiles=True), dict(strategy="stream", dynamic_tiles=True),
           dict(strategy="stream", bulk=True), dict(strategy="grid"),
           dict(strategy="stream", peer=True), dict(strategy="stream", checked=True)):
    with fsb.Engine(cfg, **kw) as eng:
        trace, bary, _ = eng.simulate(barycentre=True)
        ck = eng.checksum()
        if ref is None:
            ref = (trace.tobytes(), ck)
        assert (trace.tobytes(), ck) == ref, kw
        eng.move(t)
        eng.eat()
        school = eng.download()
        school["current_objective"][::3] += 1.0  # inconsistent upload: explicit-cur kernels
        eng.upload(school)
        eng.run(t + 1, 2)
        eng.barycentre()
        eng.gather(np.array([0, n - 1], dtype=np.uint64))
        print("ok", kw, flush=True)
sm = fsb.baseline_config(4096, 3)
with fsb.Engine(sm, strategy="persistent") as eng:
    eng.simulate(barycentre=False)
    eng.barycentre()
print("done")

"""Break the bench's e2e region into upload / run / download (PCIe rates).

    python tools/pcie_probe.py        # on the GPU box
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_20173_b200 as fsb  # noqa: E402
from paper_2507_20173_b200 import _native as N  # noqa: E402

n = 10_000_000
cfg = fsb.baseline_config(n, 100)
eng = fsb.Engine(cfg)
eng.init()
eng.run(0, 5)
eng.run(5, 100)
eng.time_step_kernels(105, 50)
L = N.lib()
nbytes = n * 40
hp = ctypes.c_void_p()
N.check(L.fsb_host_alloc(ctypes.byref(hp), nbytes))
host = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(hp.value)).view(fsb.FISH_DTYPE)
eng.download(host)
for r in range(4):
    t0 = time.perf_counter()
    eng.upload(host)
    t1 = time.perf_counter()
    eng.run(5, 100)
    t2 = time.perf_counter()
    eng.download(host)
    t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s)  run {1e3*(t2-t1):.2f} ms  "
          f"download {1e3*(t3-t2):.2f} ms ({nbytes/(t3-t2)/1e9:.1f} GB/s)  total {1e3*(t3-t0):.2f} ms", flush=True)

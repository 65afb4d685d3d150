import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np
import paper_2507_20173_b200 as fsb
from paper_2507_20173_b200 import _native as N
n = 10_000_000
cfg = fsb.baseline_config(n, 100)
eng = fsb.Engine(cfg)
eng.init(); eng.run(0, 5)
L = N.lib(); nbytes = n * 40
hp = ctypes.c_void_p(); N.check(L.fsb_host_alloc(ctypes.byref(hp), nbytes))
host = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(hp.value)).view(fsb.FISH_DTYPE)
eng.download(host)
for r in range(3):
    t0 = time.perf_counter(); eng.upload(host); t1 = time.perf_counter()
    eng.run(5, 100); t2 = time.perf_counter()
    eng.download(host); t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s)  run {1e3*(t2-t1):.2f} ms  download {1e3*(t3-t2):.2f} ms ({nbytes/(t3-t2)/1e9:.1f} GB/s)")
# raw pinned copy rate with torch for reference
import torch
a = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); d = torch.empty(nbytes, dtype=torch.uint8, device='cuda')
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    a.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"torch raw h2d {nbytes/(t1-t0)/1e9:.1f} GB/s d2h {nbytes/(t2-t1)/1e9:.1f} GB/s")

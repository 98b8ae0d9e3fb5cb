"""Host-side costs behind the pageable e2e path: threaded memcpy bandwidth and
cudaHostRegister / Unregister time for a 128 MiB caller buffer."""
import ctypes
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
try:
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
except OSError:
    import glob
    rt = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
n = 128 << 20
a = np.ones(n // 8)
b = np.empty_like(a)
for threads in (1, 2, 4, 8, 16):
    chunks = np.array_split(np.arange(a.size), threads)
    with ThreadPoolExecutor(threads) as ex:
        def cp(ix):
            b[ix[0]:ix[-1] + 1] = a[ix[0]:ix[-1] + 1]
        list(ex.map(cp, chunks))
        t0 = time.perf_counter()
        for _ in range(5):
            list(ex.map(cp, chunks))
        dt = (time.perf_counter() - t0) / 5
    print(f"memcpy {threads:2d} threads: {n / dt / 1e9:.1f} GB/s")
for mb in (8, 32, 128):
    sz = mb << 20
    buf = np.ones(sz // 8)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = rt.cudaHostRegister(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(sz), 0)
        t1 = time.perf_counter()
        r2 = rt.cudaHostUnregister(ctypes.c_void_p(buf.ctypes.data))
        t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, r, r2))
    print(f"register {mb} MiB: " + ", ".join(f"{x * 1e3:.2f}/{y * 1e3:.2f} ms rc {r}/{r2}" for x, y, r, r2 in ts))
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
for kind, host in (("pageable", torch.from_numpy(a)), ("pinned", torch.from_numpy(a).pin_memory())):
    for _ in range(2):
        d.copy_(host); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(host)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(5):
        host.copy_(d)
    torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t0) / 5
    print(f"{kind}: H2D {n / dt / 1e9:.1f} GB/s, D2H {n / dt2 / 1e9:.1f} GB/s")

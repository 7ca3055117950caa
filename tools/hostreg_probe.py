"""Host-side costs of the pageable end-to-end path (GPU box): cudaHostRegister
/ Unregister of a 2.7 GB numpy array (config 3's forecast), first-touch page
faults of a fresh output array, and pageable vs pinned cudaMemcpy rates."""
import ctypes as C
import time

import numpy as np
import torch

rt = C.CDLL("libcudart.so.12") if False else None
cud = torch.cuda.cudart()
n = 20 * 16777216
x = np.random.default_rng(1).standard_normal(n)  # faulted in
t0 = time.perf_counter(); r = cud.cudaHostRegister(x.ctypes.data, x.nbytes, 0); t1 = time.perf_counter()
cud.cudaHostUnregister(x.ctypes.data); t2 = time.perf_counter()
print(f"register {x.nbytes/1e9:.2f} GB: {t1-t0:.3f} s (rc {r}), unregister {t2-t1:.3f} s")
t0 = time.perf_counter(); y = np.empty(n); y[::512] = 0; t1 = time.perf_counter()
print(f"first touch of a fresh {y.nbytes/1e9:.2f} GB array: {t1-t0:.3f} s")
z = np.empty(n)
t0 = time.perf_counter(); r = cud.cudaHostRegister(z.ctypes.data, z.nbytes, 0); t1 = time.perf_counter()
cud.cudaHostUnregister(z.ctypes.data)
print(f"register of an untouched fresh array: {t1-t0:.3f} s (rc {r})")
d = torch.empty(n, dtype=torch.float64, device="cuda")
tx = torch.from_numpy(x)
for name, src in (("pageable", tx), ("pinned", tx.pin_memory())):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(src); torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"H2D {name}: {x.nbytes/1e9/(t1-t0):.1f} GB/s")

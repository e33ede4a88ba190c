"""Cost of pinning pageable host memory in place (cudaHostRegister /
cudaHostUnregister) vs copying it through a pinned staging buffer: the two ways
to stream a caller's std::vector at PCIe rate.  One JSON line per size."""
import ctypes as C
import json
import time

import numpy as np
import torch

rt = C.CDLL("libcudart.so") if False else None
try:
    rt = C.CDLL("libcudart.so.12")
except OSError:
    import glob
    import os

    cand = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cand += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = C.CDLL(cand[0])
rt.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]
rt.cudaHostUnregister.argtypes = [C.c_void_p]
torch.cuda.init()
for gib in (0.25, 1.0, 4.0):
    n = int(gib * (1 << 30)) // 8
    a = np.ones(n, np.float64)  # touched: pages resident
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    rc2 = rt.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    print(json.dumps({"gib": gib, "register_gbs": round(a.nbytes / (t1 - t0) / 1e9, 1),
                      "unregister_gbs": round(a.nbytes / (t2 - t1) / 1e9, 1), "rc": [rc, rc2]}), flush=True)

"""Profiling driver for the image-metrics kernels (diagnostics): 512 slices of
1024 x 1024 on device, one uscg_image_metrics call (shared range)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_12964_b200 as ub  # noqa: E402
from paper_2208_12964_b200 import uscg  # noqa: E402

S, n = int(sys.argv[1]) if len(sys.argv) > 1 else 512, 1024
a = torch.rand((S, n, n), device="cuda")
b = a * 0.97 + 0.01
ctx = ub.Context(0)
L = ub.load()
dp = uscg.C.POINTER(uscg.C.c_double)
m = [np.zeros(S) for _ in range(3)]
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    uscg._check(L.uscg_image_metrics(ctx.h, uscg.C.c_void_p(a.data_ptr()), uscg.C.c_void_p(b.data_ptr()), S, n, n, 1,
                                     -1.0, *[x.ctypes.data_as(dp) for x in m], uscg.DEVICE_POINTERS))
    print("wall ms %.2f" % (1e3 * (time.perf_counter() - t0)), m[2].mean())

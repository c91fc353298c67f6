"""A/B of the kernel matvec between builds: warm kernel_matvec timing (CUDA
events, back-to-back launches) through each library's C ABI on the C2 and C3
points, and the result against the current build's.

    python tools/kmv_ab.py [alt_libs/libafn_X.so ...]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2304_05460_b200 as afn  # noqa: E402
from synth import gen_problem  # noqa: E402

libs = [("current", afn._lib)] + [(os.path.basename(p), C.CDLL(os.path.abspath(p))) for p in sys.argv[1:]]
for _, lib in libs:
    lib.kernel_matvec.restype = C.c_int
    lib.kernel_matvec.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                  C.c_void_p, C.c_void_p, C.c_void_p]
st = torch.cuda.current_stream()
for cfg, reps in (("C2", 200), ("C3", 10)):
    X, b = gen_problem(cfg)
    Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
    n = len(X)
    ref = None
    for l in (1.0,):
        for name, lib in libs:
            y = torch.empty_like(bd)

            def run():
                s = lib.kernel_matvec(C.c_void_p(Xd.data_ptr()), n, 3, 0, l, 1e-4, C.c_void_p(bd.data_ptr()),
                                      C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream))
                assert s == 0, s
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            if ref is None:
                ref = y.clone()
            d = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
            pairs = n * (n - 1) / 2
            print(f"{cfg} l={l} {name:24s} {ms:9.4f} ms  unique-pair TF(24/pair) {pairs * 24 / ms / 1e9:6.2f}"
                  f"  Gpairs/s(n^2) {n * n / ms / 1e6:7.0f}  rel-diff {d:.1e}", flush=True)

"""Warm kernel-matvec timing on C2 (CUDA events, back-to-back launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).cuda(); bd = torch.from_numpy(b).cuda()
y = torch.empty_like(bd)
for l in (1.0, 5.0):
    for _ in range(3): afn.kernel_matvec(Xd, l, 1e-4, bd, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): afn.kernel_matvec(Xd, l, 1e-4, bd, y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    n = len(X)
    print("l", l, "kmv ms %.4f" % ms, "TFLOP/s %.2f" % (n * n * 28 / ms / 1e9))

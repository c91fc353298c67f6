"""Standalone kernel-matvec timing at C5 (n = 2^20)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
X, b = gen_problem("C5")
Xd = torch.from_numpy(X).cuda(); bd = torch.from_numpy(b).cuda()
y = torch.empty_like(bd)
afn.kernel_matvec(Xd, 1.0, 1e-4, bd, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(2): afn.kernel_matvec(Xd, 1.0, 1e-4, bd, y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 2
n = len(X)
print("C5 kmv ms %.1f  Gpairs/s %.0f" % (ms, n * n / ms / 1e6))

"""Warm per-apply time for C2 at a given l (adaptive k), plus a short PCG."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
l = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).cuda(); bd = torch.from_numpy(b).cuda()
h = afn.afn_build(Xd, afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True))
z = torch.empty_like(bd)
for _ in range(5): h.apply(bd, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100): h.apply(bd, z)
e1.record(); torch.cuda.synchronize()
print("l", l, "k", h.info()["k"], "apply us", 1000 * e0.elapsed_time(e1) / 100)
a, rep = h.pcg_solve(bd)
print("iters", rep["iterations"], "solve ms", rep["solve_ms"], "matvec ms", rep["matvec_ms"], "apply ms", rep["apply_ms"], "applies", rep["applies"])

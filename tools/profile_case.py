"""Small fixed case for ncu captures: C2 (n=16384), l=1, adaptive k, build + solve."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
dev = torch.device("cuda:0")
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).to(dev); bd = torch.from_numpy(b).to(dev)
l = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
h = afn.afn_build(Xd, afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True))
a, rep = h.pcg_solve(bd)
print(h.info(), rep)

"""Phase times of a warm C2 build (afn_info ms_* fields) for a few l."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).cuda()
for l in (1.0, 5.0):
    for rep in range(3):
        h = afn.afn_build(Xd, afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True))
        torch.cuda.synchronize()
    inf = h.info()
    print(l, {k: round(v, 3) for k, v in inf.items() if k.startswith("ms_")}, "k", inf["k"])

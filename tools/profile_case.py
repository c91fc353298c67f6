"""One warm build + solve for ncu captures: python tools/profile_case.py [CONFIG] [l]
(default C2, l = 1; adaptive k).  A first build warms the library up."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
l = float(sys.argv[2]) if len(sys.argv) > 2 else cfg.ls[0] if cfg.name != "C2" else 1.0
dev = torch.device("cuda:0")
X, b = gen_problem(cfg)
Xd = torch.from_numpy(X).to(dev); bd = torch.from_numpy(b).to(dev)
for rep in range(2):
    h = afn.afn_build(Xd, afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
    a, r = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
    h.close()
print(cfg.name, l, r)

"""d=8 N(0,1) points, mu=1e-2, l=1, w=64: AFN-PCG iterations vs n at fixed k
(compare with the oracle at the small sizes)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2304_05460_b200 as afn
from synth import gen_points
dev = torch.device("cuda:0")
for n in (8192, 16384, 32768, 65536, 131072, 262144):
    X, rng = gen_points(n, 8, "normal", 0)
    b = rng.standard_normal(n)
    Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
    for k in (400, 1000, 4000):
        if k >= n:
            continue
        h = afn.afn_build(Xd, afn.make_params(1.0, 1e-2, k, 64))
        a, rep = h.pcg_solve(bd, tol=1e-4, maxit=300)
        z1 = h.apply(torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(dev))
        u = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(dev)
        v = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).to(dev)
        s1 = float(torch.dot(h.apply(u), v)); s2 = float(torch.dot(u, h.apply(v)))
        print(f"n={n} k={k} it={rep['iterations']} conv={rep['converged']} true={rep['relres_true']:.2e} "
              f"sym={(s1 - s2) / abs(s1):.1e}", flush=True)
        h.close()

"""C4 (d=8, mu=1e-2) convergence diagnostic: AFN-PCG history at k = cap and
at smaller k, plus the kNN-pattern quality (fraction of the Schur diagonal
captured) -- prints only."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem, CONFIGS
dev = torch.device("cuda:0")
cfg = CONFIGS["C4"]
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
for l in (1.0, 3.0):
    for kcap, adaptive in ((4000, True), (4000, False), (1000, False)):
        t = time.time()
        h = afn.afn_build(Xd, afn.make_params(l, cfg.mu, kcap, cfg.w, k_adaptive=adaptive))
        a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit, history=True)
        hist = rep.pop("history")
        inf = h.info()
        print(f"l={l} kcap={kcap} adaptive={adaptive} k={inf['k']} khat={inf['khat']} it={rep['iterations']} "
              f"conv={rep['converged']} brk={rep['breakdown']} true={rep['relres_true']:.3e} "
              f"setup={inf['ms_total']:.0f}ms solve={rep['solve_ms']:.0f}ms", flush=True)
        print("   hist", np.array2string(hist[::25], precision=2), flush=True)
        h.close()

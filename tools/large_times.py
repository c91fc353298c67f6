"""Setup / solve times of C3 and C5 (l = 1) with the current library."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem, CONFIGS
for name in sys.argv[1:] or ["C3", "C5"]:
    cfg = CONFIGS[name]
    X, b = gen_problem(name)
    Xd = torch.from_numpy(X).cuda(); bd = torch.from_numpy(b).cuda()
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h = afn.afn_build(Xd, afn.make_params(1.0, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        a, rep_ = h.pcg_solve(bd)
        torch.cuda.synchronize(); t2 = time.perf_counter()
    inf = h.info()
    print(name, "k", inf["k"], "khat", inf["khat"], "iters", rep_["iterations"], "setup s %.3f" % (t1 - t0),
          "solve s %.3f" % (t2 - t1), "relres_true %.2e" % rep_["relres_true"], "matvec ms/it %.2f" % (rep_["matvec_ms"] / max(1, rep_["iterations"])))
    del h

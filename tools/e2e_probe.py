import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS["C3"]; X, b = gen_problem(cfg)
prm = afn.make_params(1.0, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True)
Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
Xh, bh = torch.from_numpy(X).pin_memory(), torch.from_numpy(b).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = afn.afn_build(Xd, prm); a, r = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit); inf = h.info(); h.close()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    a2, inf2, r2 = afn.afn_solve_host(Xh.numpy(), bh.numpy(), prm, tol=cfg.tol, maxit=cfg.maxit)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"handle {1e3*(t1-t0):.1f} ms (setup {inf['ms_total']:.1f} pcg {r['solve_ms']:.1f})   host {1e3*(t2-t1):.1f} ms (setup {inf2['ms_total']:.1f} pcg {r2['solve_ms']:.1f})", flush=True)

"""Per-step phase times of repeated C3 solves (afn_info ms_*), to find outliers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
afn.set_cutoff_mode(int(sys.argv[3]) if len(sys.argv) > 3 else 0)
L = float(sys.argv[4]) if len(sys.argv) > 4 else cfg.ls[0]
prm = afn.make_params(L, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    afn.kernel_timers(reset=True, enable=True)
    h = afn.afn_build(Xd, prm)
    t1 = time.perf_counter()
    a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
    t2 = time.perf_counter()
    inf = h.info()
    kt = afn.kernel_timers(enable=False)
    h.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    rs, us = afn.pool_stats()
    print(f"pool reserved {rs/2**30:.2f} GiB used {us/2**30:.2f} | it {it}: build {1e3*(t1-t0):.1f} solve {1e3*(t2-t1):.1f} close {1e3*(t3-t2):.1f} | "
          + " ".join(f"{k[3:]}={inf[k]:.1f}" for k in inf if k.startswith("ms_"))
          + " || " + " ".join(f"{k[:10]}={v['ms']:.1f}" for k, v in kt.items() if v["count"]), flush=True)

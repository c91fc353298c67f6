"""Host wall time vs device phase times of repeated solves (one config):
    python tools/solve_timeline.py [CONFIG] [N] [kt]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 6
kt = len(sys.argv) > 3 and sys.argv[3] == "kt"
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
prm = afn.make_params(cfg.ls[0], cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True)
for i in range(N):
    afn.kernel_timers(reset=True, enable=kt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = afn.afn_build(Xd, prm)
    t1 = time.perf_counter()
    a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
    t2 = time.perf_counter()
    inf = h.info()
    h.close()
    t3 = time.perf_counter()
    k = afn.kernel_timers(enable=False)
    print(json.dumps({"i": i, "build_wall_ms": round((t1 - t0) * 1e3, 2), "pcg_wall_ms": round((t2 - t1) * 1e3, 2),
                      "close_ms": round((t3 - t2) * 1e3, 2), "pool": afn.pool_stats(),
                      "phases": {kk: round(v, 2) for kk, v in inf.items() if kk.startswith("ms_")},
                      "solve_ms": round(rep["solve_ms"], 2),
                      "kt": {kk: round(v["ms"], 2) for kk, v in k.items() if v["count"]}}), flush=True)

"""Build + solve one config and print the phase times (afn_info / report)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
dev = torch.device("cuda:0")
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
for l in cfg.ls[:1]:
    afn.kernel_timers(reset=True, enable=True)
    h = afn.afn_build(Xd, afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
    a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
    kt = afn.kernel_timers(enable=False)
    print(json.dumps({"cfg": cfg.name, "l": l, "info": h.info(), "rep": rep,
                      "kernels": {k: v for k, v in kt.items() if v["count"]}}), flush=True)
    h.close()

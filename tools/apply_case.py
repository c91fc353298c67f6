"""Build C3 (or the given config) once, then call the public afn_apply a few
times (every launch real: no PCG skip flag) -- the case for ncu DRAM captures
of the apply's GEMV / SpMV kernels.  python tools/apply_case.py [CONFIG] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
h = afn.afn_build(Xd, afn.make_params(cfg.ls[0], cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
z = torch.empty_like(bd)
for _ in range(reps):
    h.apply(bd, z)
torch.cuda.synchronize()
print(cfg.name, "applies", reps, float(z.norm()))

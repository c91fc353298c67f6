"""A/B of whole builds between library files (kernel timers per class):
    python tools/fsai_ab.py CONFIG lib1.so [lib2.so ...]   (default: the current build)"""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import CONFIGS, gen_problem
cfg = CONFIGS[sys.argv[1]]
paths = sys.argv[2:]
X, b = gen_problem(cfg)
Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
for path in paths:
    lib = afn._lib if path == "current" else C.CDLL(os.path.abspath(path))
    afn_lib_saved = afn._lib
    afn._lib = lib  # the binding's marshalling over another build of the same ABI
    for name, (res, args) in afn._sig.items():
        f = getattr(lib, name, None)  # (an older build may lack newer entry points)
        if f is not None:
            f.restype = res; f.argtypes = args
    try:
        for rep in range(3):
            afn.kernel_timers(reset=True, enable=rep == 2)
            h = afn.afn_build(Xd, afn.make_params(cfg.ls[0], cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
            a, r = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
            inf = h.info()
            h.close()
        kt = afn.kernel_timers(enable=False)
        print(os.path.basename(path), cfg.name, "iters", r["iterations"], "setup_ms %.1f" % inf["ms_total"],
              "fsai_ms %.1f" % inf["ms_fsai"], json.dumps({k: round(v["ms"], 2) for k, v in kt.items() if v["count"]}),
              "group_gflop %.0f" % (kt["group_gemm_kernel"]["work"] / 1e9),
              flush=True)
    finally:
        afn._lib = afn_lib_saved

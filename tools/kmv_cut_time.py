"""Handle matvec timing, dense symmetric plan (mode 1) vs cutoff plan (mode 2),
on C2 (l = 1, 2), C3 and C5 (CUDA events, back-to-back products; plan built
once per handle), plus the EX2 / DFMA probes.  Usage: python tools/kmv_cut_time.py [C2 C3 C5]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_05460_b200 as afn
from synth import gen_problem

print("ex2 probe Gops/s %.0f" % afn.probe_ex2(), "dfma TF %.2f" % afn.probe_dfma(), flush=True)
cfgs = sys.argv[1:] or ["C2", "C3", "C5"]
for cfg in cfgs:
    X, b = gen_problem(cfg)
    Xd, bd = torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda()
    n = len(X)
    for l in ((0.5, 1.0, 2.0, 5.0, 10.0) if cfg == "C2" else (1.0,)):
        res = {}
        for mode in (1, 2):
            if cfg == "C5" and mode == 1:
                continue
            afn.set_cutoff_mode(mode)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = afn.afn_build(Xd, afn.make_params(l, 1e-4, 1, 1, method=afn.METHOD_NONE))
            torch.cuda.synchronize()
            tb = time.perf_counter() - t0
            y = h.matvec(bd)
            reps = 3 if cfg == "C5" else 20
            for _ in range(2):
                h.matvec(bd, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                h.matvec(bd, y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            inf = h.info()
            res[mode] = y.cpu()
            p64, p32 = inf["kmv_pairs64"], inf["kmv_pairs32"]
            # lower bound: FP64 pairs at 15 FP64-pipe instr / (148*64*1.965e9), FP32 pairs at 1 EX2 / (148*16*1.965e9)
            tmin = p64 * 15 / (148 * 64 * 1.965e9) + p32 / (148 * 16 * 1.965e9)
            print(f"{cfg} l={l} mode={mode} plan={inf['kmv_plan']} build_s={tb:.3f} ms={ms:.3f} "
                  f"units={inf['kmv_units64']} frac_pairs={(p64 + p32) / (n * (n - 1) / 2):.4f} "
                  f"p32/p={p32 / max(1, p64 + p32):.3f} roof_frac={tmin * 1e3 / ms:.3f} "
                  f"dense_equiv_Gpairs/s={n * n / ms / 1e6:.0f}", flush=True)
            h.close()
        if 1 in res and 2 in res:
            d = (res[1] - res[2]).norm() / res[1].norm()
            print(f"   rel(cut, dense) = {float(d):.3e}", flush=True)
afn.set_cutoff_mode(0)

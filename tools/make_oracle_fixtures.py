"""Write the oracle's PCG results for the bench's own configs (SURVEY.md 8(c)
parity targets) to tests/oracle_data/.  Calls only oracle/ and synth/ (the
seeded input generators): no value here comes from the CUDA path.

    python tools/make_oracle_fixtures.py c2      # the six C2 l, adaptive k
    python tools/make_oracle_fixtures.py c3      # C3, l = 1
    python tools/make_oracle_fixtures.py c4      # C4-shape trend, n = 2^13..2^15

Each C2 / C3 file holds Alg. 1's (khat, r, refined), the k used, the PCG
iteration count at tol 1e-4 (x0 = 0, recurrence residual, maxit 500; P:L788,
L828) and the solution at that count, plus the true relative residual.  The
GPU tests run the device PCG at the same fixed iteration count and compare
(<= 1e-6) and check the device's own tol-stopped count within +-2.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from synth import CONFIGS, gen_points, gen_problem  # noqa: E402

OUT = os.path.join(ROOT, "tests", "oracle_data")
THREADS = len(os.sched_getaffinity(0))


def solve_config(name, l):
    cfg = CONFIGS[name]
    X, b = gen_problem(cfg)
    t0 = time.time()
    a1 = O.alg1(X, l)
    k = min(cfg.k_cap, max(1, a1["khat"]), cfg.n)
    B = O.build_afn(X, l, cfg.mu, k, cfg.w)
    t1 = time.time()
    a, rep, _ = O.afn_pcg_solve(X, b, l, cfg.mu, k, cfg.w, tol=cfg.tol, maxit=cfg.maxit, B=B,
                                threads=THREADS)
    t2 = time.time()
    print(f"{name} l={l}: khat={a1['khat']} r={a1['r']} refined={a1['refined']} k={k} "
          f"iters={rep['iterations']} conv={rep['converged']} true={rep['relres_true']:.3e} "
          f"build {t1 - t0:.0f}s pcg {t2 - t1:.0f}s", flush=True)
    return dict(khat=a1["khat"], r=a1["r"], refined=int(a1["refined"]), k=k, iters=rep["iterations"],
                converged=int(rep["converged"]), relres_true=rep["relres_true"], a=a,
                err_margin=a1["err_margin"], ev_margin=a1["ev_margin"])


def save(fn, d):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, fn), **{k: np.asarray(v) for k, v in d.items()})


def main():
    what = sys.argv[1:] or ["c2"]
    if "c2" in what:
        for l in CONFIGS["C2"].ls:
            save(f"c2_l{l:g}.npz", solve_config("C2", l))
    if "c3" in what:
        save("c3_l1.npz", solve_config("C3", 1.0))
    if "c4" in what:
        # C4's shape (d = 8 N(0,1) points, mu = 1e-2, l = 1, w = 64) at n = 2^13..2^15 with
        # k = 1000: the iteration count's growth with n
        res = {}
        for n in (8192, 16384, 32768):
            X, rng = gen_points(n, 8, "normal", 0)
            b = rng.standard_normal(n)
            t0 = time.time()
            _, rep, _ = O.afn_pcg_solve(X, b, 1.0, 1e-2, 1000, 64, tol=1e-4, maxit=500, threads=THREADS)
            res[str(n)] = dict(iters=rep["iterations"], converged=bool(rep["converged"]),
                               relres_true=rep["relres_true"])
            print(f"C4-shape n={n}: {res[str(n)]} ({time.time() - t0:.0f}s)", flush=True)
        os.makedirs(OUT, exist_ok=True)
        with open(os.path.join(OUT, "c4_shape_iters.json"), "w") as f:
            json.dump(dict(source="tools/make_oracle_fixtures.py c4 (oracle only)", d=8, data="normal",
                           l=1.0, mu=1e-2, k=1000, w=64, tol=1e-4, maxit=500, results=res), f, indent=1)


if __name__ == "__main__":
    main()

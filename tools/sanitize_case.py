"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck): every
kernel family of the hot path once -- FPS on the cluster (st.async + mbarrier)
and grid (software barrier) paths, Alg. 1 (Lanczos, batched probes), the AFN
build (Cholesky, W, kNN brute force and grid, FSAI group product and factor,
transpose), PCG (graph-captured chunks, fused reductions with last-block
finishes), the apply, a sharded handle (emulated ranks, symmetric pair units)
and plain CG.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2304_05460_b200 as afn  # noqa: E402
from synth import gen_points, gen_small  # noqa: E402

dev = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


X, b = gen_small(3000, 3, seed=1)
Xd, bd = T(X), T(b)
# FPS: cluster path (n <= 64K) and the persistent-grid path (n > 64K), few steps
idx, _ = afn.afn_fps(Xd, 64, 0)
Xg, _ = gen_points(140000, 3, "cube", 2)
afn.afn_fps(T(Xg), 16, 0)
# kNN grid path (d = 3, N >= 50000)
afn.afn_knn_pattern(T(Xg[:52000]), 20)
# AFN build + PCG + apply (adaptive k: Alg. 1)
h = afn.afn_build(Xd, afn.make_params(1.0, 1e-4, 400, 40, k_adaptive=True))
a, rep = h.pcg_solve(bd, tol=1e-4)
z = h.apply(bd)
y = h.matvec(bd)
h.close()
# sharded handle (2 emulated ranks) and plain CG
comm = afn.Comm.emulated(2)
h2 = afn.afn_build(Xd, afn.make_params(1.0, 1e-4, 300, 30), comm=comm)
h2.pcg_solve(bd, tol=1e-4)
h2.close()
comm.close()
afn.afn_cg_solve(Xd, bd, 1.0, 1e-2, tol=1e-3, maxit=50)
torch.cuda.synchronize()
print("sanitize case ok", rep["iterations"], float(z.norm()), float(y.norm()))

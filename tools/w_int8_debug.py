import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
import paper_2304_05460_b200 as afn
from synth import gen_points
from scipy.linalg import cholesky, solve_triangular
def T(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
for (k, N, d, l) in [(64, 128, 3, 1.0), (128, 128, 3, 1.0), (600, 1000, 3, 1.0), (1100, 700, 8, 2.0)]:
    X, _ = gen_points(k + N, d, "cube", 11)
    X1, Xr = X[:k], X[k:]
    K11 = O.kernel_block(X1, X1, l) + 1e-4 * np.eye(k)
    Lc = cholesky(K11, lower=True); Linv = solve_triangular(Lc, np.eye(k), lower=True)
    K21 = O.kernel_block(Xr, X1, l); Wref = K21 @ Linv.T; bound = np.abs(K21) @ np.abs(Linv).T + 1e-300
    W8 = afn.afn_w_product(T(X1), T(Xr), l, T(Linv), afn.WPROD_INT8).cpu().numpy()
    E = np.abs(W8 - Wref) / bound
    bad = E > 1e-12
    print(k, N, d, "max", E.max(), "bad frac", bad.mean(), flush=True)
    if bad.any():
        rows = np.where(bad.any(1))[0]; cols = np.where(bad.any(0))[0]
        print("  bad rows", rows[:10], len(rows), " bad cols", cols[:20], len(cols))
        r, c = np.argwhere(bad)[0]
        print("  first bad", r, c, W8[r, c], Wref[r, c])
        # per column-tile / row-tile counts
        print("  col tiles", np.unique(cols // 64), " row tiles", np.unique(rows // 128))

import sys, os
os.environ["AFN_DEBUG_ALLOW_NOT_SPD"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_05460_b200 as afn
import oracle as O
from synth import gen_small
dev = torch.device("cuda:0")
for (n, d, l, mu, k, w) in [(700, 2, 0.7, 1e-3, 64, 20), (700, 3, 0.7, 1e-3, 64, 20), (700, 2, 0.7, 1e-3, 100, 20), (700, 2, 0.7, 1e-3, 64, 50), (700,2,0.7,1e-3,128,20)]:
    X, _ = gen_small(n, d, seed=8)
    h = afn.afn_build(torch.from_numpy(X).to(dev), afn.make_params(l, mu, k, w))
    B = O.build_afn(X, l, mu, k, w)
    W = h.copy_out(afn.OUT_W); L = h.copy_out(afn.OUT_L)
    g = h.copy_out(afn.OUT_GVAL); go = B["G"].data; rp = B["row_ptr"]
    bad = [i for i in range(len(rp)-1) if np.linalg.norm(g[rp[i]:rp[i+1]]-go[rp[i]:rp[i+1]]) > 1e-8*np.linalg.norm(go[rp[i]:rp[i+1]])]
    print((n,d,l,mu,k,w), "perm", np.array_equal(h.copy_out(afn.OUT_PERM), B["perm"]), "L", np.abs(L-B["L"]).max(), "W", np.abs(W-B["V"].T).max(),
          "col", np.array_equal(h.copy_out(afn.OUT_COL).astype(np.int64), B["col"]), "nbad G rows", len(bad), bad[:8], flush=True)
    if bad:
        i = bad[0]; print("  row", i, "len", rp[i+1]-rp[i], "g", g[rp[i]:rp[i+1]][:5], "go", go[rp[i]:rp[i+1]][:5])

import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_05460_b200 as afn
import oracle as O
from synth import gen_problem
dev = torch.device("cuda:0")
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).to(dev)
io, fo = O.fps(X, 2000, 0)
for rep in range(4):
    idx, fill = afn.afn_fps(Xd, 2000, 0)
    i = idx.cpu().numpy()
    print("fps rep", rep, "equal", np.array_equal(i, io), "first diff", np.argmax(i != io) if not np.array_equal(i, io) else -1, "unique", len(np.unique(i)), flush=True)
mask = np.ones(len(X), bool); mask[io] = False
X2 = X[np.concatenate([io, np.nonzero(mask)[0]])][2000:]
t = time.time(); rpo, colo = O.knn_lower(X2, 100); print("oracle knn s", time.time() - t, flush=True)
X2d = torch.from_numpy(np.ascontiguousarray(X2)).to(dev)
for rep in range(3):
    rp, col = afn.afn_knn_pattern(X2d, 100)
    c = col.cpu().numpy().astype(np.int64)
    bad = np.nonzero(c != colo)[0]
    print("knn rep", rep, "rp eq", np.array_equal(rp.cpu().numpy(), rpo), "col eq", len(bad) == 0, "nbad", len(bad), (bad[:5], c[bad[:5]], colo[bad[:5]]) if len(bad) else "", flush=True)
for rep in range(4):
    try:
        h = afn.afn_build(Xd, afn.make_params(1.0, 1e-4, 2000, 100))
        p = h.copy_out(afn.OUT_PERM)
        cc = h.copy_out(afn.OUT_COL).astype(np.int64)
        print("build rep", rep, "perm ok", np.array_equal(np.sort(p), np.arange(len(X))), "perm eq", np.array_equal(p[:2000], io), "col eq", np.array_equal(cc, colo), flush=True)
        h.close()
    except Exception as e:
        print("build rep", rep, "FAILED", e, flush=True)

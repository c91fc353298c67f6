import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, hashlib
import paper_2304_05460_b200 as afn
from synth import gen_problem
dev = torch.device("cuda:0")
X, b = gen_problem("C2")
Xd = torch.from_numpy(X).to(dev); bd = torch.from_numpy(b).to(dev)
hs = []; ref = None
def dig(a): return hashlib.md5(a.tobytes()).hexdigest()[:8]
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    try:
        h = afn.afn_build(Xd, afn.make_params(1.0, 1e-4, 2000, 100))
    except Exception as e:
        print(rep, "BUILD FAILED", e, flush=True); continue
    outs = {nm: h.copy_out(w) for nm, w in [("perm", afn.OUT_PERM), ("L", afn.OUT_L), ("W", afn.OUT_W), ("col", afn.OUT_COL), ("g", afn.OUT_GVAL)]}
    if ref is None: ref = outs
    diffs = {nm: (not np.array_equal(outs[nm], ref[nm])) for nm in outs}
    msg = {nm: dig(v) for nm, v in outs.items()}
    extra = ""
    if diffs["W"]:
        bad = np.argwhere(outs["W"] != ref["W"]); extra = f"W bad rows {np.unique(bad[:,0])[:10]} cols {np.unique(bad[:,1])[:10]} n={len(bad)}"
    if diffs["L"]:
        bad = np.argwhere(outs["L"] != ref["L"]); extra += f" L bad {bad[:5].tolist()} n={len(bad)}"
    print(rep, msg, diffs, extra, flush=True)
    hs.append(h)

"""Quick staged GPU check against the oracle (prints as it goes)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2304_05460_b200 as afn
import oracle as O
from synth import gen_problem, gen_points

dev = torch.device("cuda:0")
print("dfma probe TF/s:", afn.probe_dfma(1 << 14), flush=True)

X, b = gen_problem("C1")
Xd = torch.from_numpy(X).to(dev); bd = torch.from_numpy(b).to(dev)
y = afn.kernel_matvec(Xd, 1.0, 1e-4, bd).cpu().numpy()
yo = O.kmv(X, 1.0, 1e-4, b)
print("kmv C1 rel", np.linalg.norm(y - yo) / np.linalg.norm(yo), flush=True)

idx, fill = afn.afn_fps(Xd, 100, 0)
io, fo = O.fps(X, 100, 0)
print("fps C1 equal", np.array_equal(idx.cpu().numpy(), io), np.array_equal(fill.cpu().numpy(), fo), flush=True)

P = X[:600]
rp, col = afn.afn_knn_pattern(torch.from_numpy(P).to(dev), 50)
rpo, colo = O.knn_lower(P, 50)
print("knn equal", np.array_equal(rp.cpu().numpy(), rpo), np.array_equal(col.cpu().numpy().astype(np.int64), colo), flush=True)

prm = afn.make_params(1.0, 1e-4, 100, 50)
h = afn.afn_build(Xd, prm)
print("build info", h.info(), flush=True)
B = O.build_afn(X, 1.0, 1e-4, 100, 50)
print("perm equal", np.array_equal(h.copy_out(afn.OUT_PERM), B["perm"]))
L = h.copy_out(afn.OUT_L)
print("L rel", np.abs(L - B["L"]).max() / np.abs(B["L"]).max())
W = h.copy_out(afn.OUT_W)
print("W rel", np.abs(W - B["V"].T).max() / np.abs(B["V"]).max())
gv = h.copy_out(afn.OUT_GVAL)
print("G rel", np.abs(gv - B["G"].data).max() / np.abs(B["G"].data).max(), flush=True)
r = np.random.default_rng(1).standard_normal(1000)
z = h.apply(torch.from_numpy(r).to(dev)).cpu().numpy()
zo = np.empty(1000); zo[B["perm"]] = O.apply_afn(B, r[B["perm"]])
print("apply rel", np.linalg.norm(z - zo) / np.linalg.norm(zo), flush=True)
a, rep = h.pcg_solve(bd, tol=1e-4)
ao, repo, _ = O.afn_pcg_solve(X, b, 1.0, 1e-4, 100, 50, B=B)
print("pcg", rep, "oracle it", repo["iterations"], "rel", np.linalg.norm(a.cpu().numpy() - ao) / np.linalg.norm(ao), flush=True)

# C2 timing (l=1, k=2000 fixed)
X2, b2 = gen_problem("C2")
X2d = torch.from_numpy(X2).to(dev); b2d = torch.from_numpy(b2).to(dev)
for rep_i in range(2):
    torch.cuda.synchronize(); t = time.time()
    h2 = afn.afn_build(X2d, afn.make_params(1.0, 1e-4, 2000, 100))
    a2, r2 = h2.pcg_solve(b2d)
    torch.cuda.synchronize()
    print("C2 build+solve s", time.time() - t, h2.info(), r2, flush=True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
v = torch.randn(16384, dtype=torch.float64, device=dev)
afn.kernel_matvec(X2d, 1.0, 1e-4, v)
e0.record()
for _ in range(10): afn.kernel_matvec(X2d, 1.0, 1e-4, v)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("kmv C2 ms", ms, "Gpairs/s", 16384**2 / ms / 1e6, flush=True)
print("launches", afn.launch_count())

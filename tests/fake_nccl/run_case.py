"""R "ranks" as host threads of one process on one GPU, joined through the
fake NCCL library (tests/fake_nccl/fake_nccl.cpp): the row-sharded build,
PCG, apply, matvec and CG run the library's NCCL code path (in-place and
packed all-gathers, the build-status exchange, asynchronous-error polling).
Checks: every rank returns the same results, equal (to rank-order rounding)
to the one-GPU handle's.  python run_case.py LIBFAKENCCL R"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2304_05460_b200 as afn  # noqa: E402
from synth import gen_small  # noqa: E402

fake, R = os.path.abspath(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
X, b = gen_small(3000, 3, seed=5)
Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
prm = afn.make_params(1.0, 1e-4, 300, 40)
h1 = afn.afn_build(Xd, prm)
a1, r1 = h1.pcg_solve(bd)
z1, y1 = h1.apply(bd).cpu().numpy(), h1.matvec(bd).cpu().numpy()
a1 = a1.cpu().numpy()
h1.close()
acg1, rcg1 = afn.afn_cg_solve(Xd, bd, 1.0, 1e-2, tol=1e-3, maxit=300)
acg1 = acg1.cpu().numpy()

uid = afn.nccl_unique_id(fake)
out, errs = [None] * R, []


def worker(rank):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        comm = afn.Comm.nccl(uid, R, rank, nccl_path=fake)
        comm.set_timeout(120.0)
        h = afn.afn_build(Xd, prm, comm=comm, stream=s)
        a, rep = h.pcg_solve(bd, stream=s)
        z = h.apply(bd, stream=s)
        y = h.matvec(bd, stream=s)
        acg, rcg = afn.afn_cg_solve(Xd, bd, 1.0, 1e-2, tol=1e-3, maxit=300, comm=comm, stream=s)
        s.synchronize()
        out[rank] = (a.cpu().numpy(), rep, z.cpu().numpy(), y.cpu().numpy(), acg.cpu().numpy(), rcg, h.info())
        h.close()
        comm.close()
    except Exception as e:  # pragma: no cover
        errs.append(f"rank {rank}: {e!r}")


th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
for t in th:
    t.start()
for t in th:
    t.join(300)
assert not errs, errs
assert all(o is not None for o in out), "a rank did not finish"


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for r, (a, rep, z, y, acg, rcg, inf) in enumerate(out):
    assert inf["nranks"] == R and inf["rank"] == r, inf
    assert rep["iterations"] == r1["iterations"] and rep["converged"], (rep, r1)
    assert rel(a, a1) <= 1e-9, rel(a, a1)
    assert rel(z, z1) <= 1e-12, rel(z, z1)
    assert rel(y, y1) <= 1e-14, rel(y, y1)
    assert abs(rcg["iterations"] - rcg1["iterations"]) <= 2 and rel(acg, acg1) <= 1e-6
    for k in range(R):  # every rank holds the same full results
        assert np.array_equal(a, out[k][0]) and np.array_equal(z, out[k][2]) and np.array_equal(y, out[k][3])
print("fake-nccl ok", R, r1["iterations"], rel(out[0][0], a1), rel(out[0][3], y1))

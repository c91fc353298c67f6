"""GPU checks of the cutoff kernel-matvec plan (kmv.cu) against
the oracle's plain product (y = (K + mu I) v, every pair in fp64).

The cutoff plan evaluates the same sum over a spatial order of the points:
(row block, column tile) units whose bounding boxes are at least s = 128
apart (s = ||x_i - x_j||^2 log2(e) / l^2; every skipped entry is below
2^-128) are skipped, units at least s = 48 apart (entries below 2^-48) run in
FP32, the rest in FP64.  The bar is the north star's: element-wise
|y_i - y_i(oracle)| <= 1e-12 ((K + mu I)|v|)_i, plus agreement with the dense
FP64 plan and determinism."""
import numpy as np
import pytest

import oracle as O
from synth import gen_points, gen_problem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2304_05460_b200 as afn  # noqa: E402

DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def elementwise(y, X, l, mu, v, rows):
    yo = O.kmv_rows(X, l, mu, v, rows)
    ya = O.kmv_rows(X, l, mu, np.abs(v), rows)
    return float(np.max(np.abs(np.asarray(y)[rows] - yo) / ya))


@pytest.fixture
def mode():
    yield afn.set_cutoff_mode
    afn.set_cutoff_mode(0)


def _plan_of(Xd, l):
    """The plan a handle over Xd picks (METHOD_NONE: no preconditioner)."""
    h = afn.afn_build(Xd, afn.make_params(l, 1e-4, 1, 1, method=afn.METHOD_NONE))
    info = h.info()
    h.close()
    return info


@pytest.mark.parametrize("n,d,l,edge,seed", [
    (16384, 3, 0.1, None, 0), (16384, 3, 0.5, None, 0), (16384, 3, 1.0, None, 0), (16384, 3, 2.0, None, 0),
    (10007, 3, 1.0, 60.0, 1),      # ragged, sparse: most units skipped
    (4096, 3, 1.0, 16.0, 2),       # one-wave size
    (20001, 2, 1.0, None, 3),      # d = 2
    (9000, 1, 1.0, None, 4),       # d = 1: a line
])
def test_cut_matvec_parity(mode, n, d, l, edge, seed):
    X, _ = gen_points(n, d, "cube", seed, edge)
    v = np.random.default_rng(seed + 7).standard_normal(n)
    Xd, vd = T(X), T(v)
    mode(2)
    y = afn.kernel_matvec(Xd, l, 1e-4, vd)
    y2 = afn.kernel_matvec(Xd, l, 1e-4, vd)
    assert torch.equal(y, y2)  # fixed summation order
    info = _plan_of(Xd, l)
    assert info["kmv_plan"] == 2
    mode(1)
    yd = afn.kernel_matvec(Xd, l, 1e-4, vd).cpu().numpy()
    y = y.cpu().numpy()
    yo = O.kmv(X, l, 1e-4, v)
    assert rel(y, yo) <= 1e-12
    assert rel(y, yd) <= 1e-13
    rows = np.unique(np.concatenate([np.arange(0, n, max(1, n // 300)), [n - 1]]))
    assert elementwise(y, X, l, 1e-4, v, rows) <= 1e-12
    pairs = info["kmv_pairs64"] + info["kmv_pairs32"]
    assert 0 < pairs <= n * (n - 1) / 2


def test_cut_matvec_classes_and_skips(mode):
    """At C2 size and l = 1 (edge 25.4) FP64, FP32 and skipped work all occur;
    the evaluated pairs shrink with l."""
    X, b = gen_problem("C2")
    Xd = T(X)
    mode(2)
    i1 = _plan_of(Xd, 1.0)
    i01 = _plan_of(Xd, 0.1)
    n = len(X)
    allp = n * (n - 1) / 2
    assert i1["kmv_pairs64"] > 0 and i1["kmv_pairs32"] > 0
    assert i1["kmv_pairs64"] + i1["kmv_pairs32"] < allp
    assert i01["kmv_pairs64"] + i01["kmv_pairs32"] < 0.5 * (i1["kmv_pairs64"] + i1["kmv_pairs32"])
    mode(0)  # auto: the cutoff plan whenever it applies (C2: never slower)
    assert _plan_of(Xd, 10.0)["kmv_plan"] == 2
    mode(1)
    assert _plan_of(Xd, 10.0)["kmv_plan"] == 1


def test_cut_degenerate_points(mode):
    """All points equal (zero-size boxes) and heavy duplication."""
    mode(2)
    n = 5000
    rng = np.random.default_rng(11)
    for X in (np.full((n, 3), 2.5), np.repeat(rng.uniform(0, 40, (n // 10, 3)), 10, axis=0)):
        v = rng.standard_normal(len(X))
        y = afn.kernel_matvec(T(X), 1.0, 1e-4, T(v)).cpu().numpy()
        assert rel(y, O.kmv(X, 1.0, 1e-4, v)) <= 1e-12


@pytest.mark.parametrize("R", [2, 3, 8])
def test_cut_sharded_handle(mode, R):
    """The cutoff units split over R emulated ranks (rank partials summed in
    rank order) against the one-rank cutoff product: <= 1e-14."""
    mode(2)
    X, _ = gen_points(30000, 3, "cube", 9)
    v = np.random.default_rng(R).standard_normal(len(X))
    Xd, vd = T(X), T(v)
    prm = afn.make_params(1.0, 1e-4, 1, 1, method=afn.METHOD_NONE)
    h1 = afn.afn_build(Xd, prm)
    y1 = h1.matvec(vd).cpu().numpy()
    comm = afn.Comm.emulated(R)
    h = afn.afn_build(Xd, prm, comm=comm)
    assert h.info()["kmv_plan"] == 2
    y = h.matvec(vd).cpu().numpy()
    assert rel(y, y1) <= 1e-14
    rows = np.arange(0, len(X), 97)
    assert elementwise(y, X, 1.0, 1e-4, v, rows) <= 1e-12
    h.close()
    h1.close()
    comm.close()


@pytest.mark.parametrize("l", [0.5, 1.0, 2.0])
def test_cut_afn_pcg_c2(mode, l):
    """AFN-PCG on C2 with the cutoff product inside the solve, against the
    oracle's committed full AFN-PCG (tests/oracle_data): iterations +-2, true
    residual <= tol, solution <= 1e-6 at the oracle's iteration count."""
    import os
    o = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_data", f"c2_l{l:g}.npz"))
    mode(2)
    X, b = gen_problem("C2")
    bd = T(b)
    h = afn.afn_build(T(X), afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True))
    assert h.info()["kmv_plan"] == 2
    a, rep = h.pcg_solve(bd, tol=1e-4)
    assert abs(rep["iterations"] - int(o["iters"])) <= 2
    assert rep["relres_true"] <= 1e-4
    a2, _ = h.pcg_solve(bd, fixed_iters=int(o["iters"]))
    assert rel(a2.cpu().numpy(), o["a"]) <= 1e-6
    h.close()


def test_cut_c3_auto_sampled_rows():
    """C3 (n = 2^17, l = 1): auto mode picks the cutoff plan; sampled rows
    element-wise against the oracle."""
    afn.set_cutoff_mode(0)
    X, b = gen_problem("C3")
    Xd, bd = T(X), T(b)
    info = _plan_of(Xd, 1.0)
    assert info["kmv_plan"] == 2
    n = len(X)
    assert info["kmv_pairs64"] + info["kmv_pairs32"] < 0.5 * n * (n - 1) / 2
    y = afn.kernel_matvec(Xd, 1.0, 1e-4, bd).cpu().numpy()
    rows = np.random.default_rng(5).choice(n, 200, replace=False)
    assert elementwise(y, X, 1.0, 1e-4, b, rows) <= 1e-12


@pytest.mark.parametrize("k,N,d,l,edge", [(1000, 20000, 3, 1.0, 28.0), (700, 5000, 3, 0.5, None),
                                          (333, 4097, 3, 1.0, 40.0), (64, 200, 3, 1.0, 30.0),
                                          (500, 6000, 2, 1.0, None), (300, 3000, 1, 2.0, None),
                                          (1, 1000, 3, 1.0, None)])
def test_w_product_cutoff(k, N, d, l, edge):
    """W = K21 L^{-T} with the terms whose K21 entry is below 2^-128
    dropped (wcut.cu).  Against the DMMA path (the same kernel
    entries): every entry within 1e-15 k max_t |K21_rt| max_t |L^{-1}_ct| plus
    the dropped terms' bound k 2^-128 max |L^{-1}|.  Against the plain fp64
    product (oracle entries, LAPACK Cholesky and triangular inverse): every
    row above the dropped-term floor within 1e-12 (normwise), as the dense
    paths (a far entry's own rounding, ~s eps relative, is the same on both)."""
    from scipy.linalg import cholesky, solve_triangular
    X, _ = gen_points(k + N, d, "cube", 13, edge)
    X1, Xr = X[:k], X[k:]
    K11 = O.kernel_block(X1, X1, l) + 1e-4 * np.eye(k)
    Lc = cholesky(K11, lower=True)
    Linv = solve_triangular(Lc, np.eye(k), lower=True)
    K21 = O.kernel_block(Xr, X1, l)
    Wref = K21 @ Linv.T
    scale = np.abs(K21).max(axis=1)[:, None] * np.abs(Linv).max(axis=1)[None, :]
    Wc = afn.afn_w_product(T(X1), T(Xr), l, T(Linv), afn.WPROD_CUT).cpu().numpy()
    Wd = afn.afn_w_product(T(X1), T(Xr), l, T(Linv), afn.WPROD_DMMA).cpu().numpy()
    assert np.all(np.isfinite(Wc))
    drop = k * 2.0 ** -128 * np.max(np.abs(Linv))
    assert np.all(np.abs(Wc - Wd) <= 1e-15 * k * scale + drop)
    nr = np.linalg.norm(Wref, axis=1)
    ok = nr > 1e20 * drop
    assert ok.any()
    rc = np.max(np.linalg.norm(Wc - Wref, axis=1)[ok] / nr[ok])
    assert rc <= 1e-12, rc


def test_build_uses_w_cutoff_and_matches_dense(mode):
    """C2 (l = 1) handles built with and without the cutoff paths (mode 1:
    dense matvec and INT8 W): the same landmarks and pattern, W rows and G
    rows within the build's parity bounds, the same PCG iteration count."""
    X, b = gen_problem("C2")
    Xd, bd = T(X), T(b)
    prm = afn.make_params(1.0, 1e-4, 2000, 100, k_adaptive=True)
    mode(2)
    hc = afn.afn_build(Xd, prm)
    mode(1)
    hd = afn.afn_build(Xd, prm)
    assert hc.info()["kmv_plan"] == 2 and hd.info()["kmv_plan"] == 1
    k = hc.info()["k"]
    rows = np.arange(0, len(X) - k, 97)
    Wc = hc.copy_out_rows(afn.OUT_W, rows)
    Wdd = hd.copy_out_rows(afn.OUT_W, rows)
    assert np.max(np.linalg.norm(Wc - Wdd, axis=1) / np.linalg.norm(Wdd, axis=1)) <= 1e-12
    gc, gd = hc.copy_out(afn.OUT_GVAL), hd.copy_out(afn.OUT_GVAL)
    assert np.max(np.abs(gc - gd)) <= 1e-10 * np.max(np.abs(gd))
    _, rc = hc.pcg_solve(bd, tol=1e-4)
    _, rd = hd.pcg_solve(bd, tol=1e-4)
    assert rc["iterations"] == rd["iterations"]
    hc.close()
    hd.close()

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances are those of BASELINE.json's north star:
bit-exact FPS / kNN / permutation, kernel matvec rel <= 1e-12, FSAI entries
rel <= 1e-10 per row, PCG iterations within +-2, solution rel <= 1e-6 at equal
iteration counts, true residual <= tol.  Run on a B200: pytest -m gpu."""
import math
import numpy as np
import pytest

import oracle as O
from synth import gen_points, gen_problem, gen_small

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


# --------------------------------------------------------------------------- kmv
@pytest.mark.parametrize("n,d,l,mu", [(1, 3, 1.0, 1e-4), (7, 2, 0.5, 1e-3), (1000, 3, 1.0, 1e-4),
                                      (1337, 1, 0.3, 1e-2), (3000, 3, 0.1, 1e-4), (2049, 8, 3.0, 1e-2),
                                      (777, 5, 1.7, 0.0), (513, 16, 4.0, 1e-3)])
def test_kmv_parity(n, d, l, mu):
    X, _ = gen_points(n, d, "cube", 3)
    v = np.random.default_rng(n).standard_normal(n)
    y = afn.kernel_matvec(T(X), l, mu, T(v)).cpu().numpy()
    yo = O.kmv(X, l, mu, v)
    assert rel(y, yo) <= 1e-12


def test_kmv_c2_full_size_and_determinism():
    X, b = gen_problem("C2")
    Xd, bd = T(X), T(b)
    for l in (0.1, 1.0, 10.0):
        y1 = afn.kernel_matvec(Xd, l, 1e-4, bd)
        y2 = afn.kernel_matvec(Xd, l, 1e-4, bd)
        assert torch.equal(y1, y2)
        rows = np.random.default_rng(1).choice(len(X), 300, replace=False)
        yo = O.kmv_rows(X, l, 1e-4, b, rows)
        assert rel(y1.cpu().numpy()[rows], yo) <= 1e-12


def test_kmv_row_shards():
    """Row-sharded evaluation (multi-GPU layout).  Shards large enough to keep
    the full plan's column chunking are bit-identical to the full matvec
    (n = 2^20, up to 8 shards); small shards get their own chunking and agree
    to rounding."""
    X, b = gen_problem("C2")
    Xd, bd = T(X), T(b)
    full = afn.kernel_matvec(Xd, 1.0, 1e-4, bd)
    n = len(X)
    for R in (2, 3, 8):
        parts = []
        for r in range(R):
            a0, a1 = n * r // R, n * (r + 1) // R
            parts.append(afn.kernel_matvec_rows(Xd, 1.0, 1e-4, bd, a0, a1 - a0))
        assert rel(torch.cat(parts).cpu().numpy(), full.cpu().numpy()) <= 1e-14
    X5, b5 = gen_problem("C5")
    X5d, b5d = T(X5), T(b5)
    n5 = len(X5)
    rows = 4096
    ref = afn.kernel_matvec_rows(X5d, 1.0, 1e-4, b5d, 0, n5)
    for R in (2, 8):
        a0 = n5 // R  # shard 1's first rows against the same rows of the full matvec
        part = afn.kernel_matvec_rows(X5d, 1.0, 1e-4, b5d, a0, n5 // R)
        assert torch.equal(part[:rows], ref[a0:a0 + rows])


# --------------------------------------------------------------------------- FPS
@pytest.mark.parametrize("n,d,k,seed", [(1000, 3, 100, 0), (1, 2, 1, 0), (5000, 2, 300, 17),
                                        (16384, 3, 2000, 0), (9000, 8, 257, 5), (4097, 1, 4097, 0),
                                        (100000, 3, 200, 7), (70001, 2, 150, 3), (140000, 3, 100, 0)])
def test_fps_bit_exact(n, d, k, seed):
    X, _ = gen_points(n, d, "cube", 4)
    idx, fill = afn.afn_fps(T(X), k, seed)
    io, fo = O.fps(X, k, seed)
    assert np.array_equal(idx.cpu().numpy(), io)
    assert np.array_equal(fill.cpu().numpy(), fo)


@pytest.mark.parametrize("case", ["lattice3", "dup3", "lattice2"])
def test_fps_spatial_cull_ties(case):
    """The shared-memory cluster FPS (65536 < n <= 131072, d <= 3) keeps its
    points in a spatial order and skips warps whose box is out of reach: on
    integer lattices (many exactly equal distances) and on duplicated points
    the lowest-index tie rule of P:L101's argmax must still give the oracle's
    landmarks and fill distances bit for bit."""
    if case == "lattice3":
        g = np.stack(np.meshgrid(np.arange(50), np.arange(50), np.arange(40), indexing="ij"), -1)
        X = g.reshape(-1, 3).astype(np.float64)
    elif case == "dup3":
        Y, _ = gen_points(50000, 3, "cube", 11)
        X = np.concatenate([Y, Y[::-1]])
    else:
        g = np.stack(np.meshgrid(np.arange(300), np.arange(250), indexing="ij"), -1)
        X = g.reshape(-1, 2).astype(np.float64)
    rng = np.random.default_rng(5)
    X = X[rng.permutation(len(X))]
    idx, fill = afn.afn_fps(T(X), 300, 3)
    io, fo = O.fps(X, 300, 3)
    assert np.array_equal(idx.cpu().numpy(), io)
    assert np.array_equal(fill.cpu().numpy(), fo)


def test_fps_duplicates_and_golden():
    X = np.repeat(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 3.0]]), 3, axis=0)
    idx, fill = afn.afn_fps(T(X), 9, 0)
    io, fo = O.fps(X, 9, 0)
    assert np.array_equal(idx.cpu().numpy(), io) and np.array_equal(fill.cpu().numpy(), fo)
    idx, _ = afn.afn_fps(T(np.array([[0.0], [1.0], [10.0]])), 3, 0)
    assert idx.cpu().numpy().tolist() == [0, 2, 1]


# --------------------------------------------------------------------------- kNN
@pytest.mark.parametrize("N,d,w", [(1, 3, 50), (600, 3, 50), (2000, 3, 100), (1500, 2, 1),
                                   (999, 8, 64), (300, 3, 128), (130, 1, 100)])
def test_knn_bit_exact(N, d, w):
    P, _ = gen_points(N, d, "cube", 6)
    rp, col = afn.afn_knn_pattern(T(P), w)
    rpo, colo = O.knn_lower(P, w)
    assert np.array_equal(rp.cpu().numpy(), rpo)
    assert np.array_equal(col.cpu().numpy().astype(np.int64), colo)


@pytest.mark.parametrize("N,w,seed", [(60000, 100, 1), (120000, 50, 2), (70000, 1, 3)])
def test_knn_grid_path_rows(N, w, seed):
    """d = 3, N >= 50000 takes the grid search (knn.cu): sampled rows, small and
    large i, bit-exact against the brute-force definition."""
    P, _ = gen_points(N, 3, "cube", seed)
    rp, col = afn.afn_knn_pattern(T(P), w)
    rp, col = rp.cpu().numpy(), col.cpu().numpy()
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([np.arange(0, 300), rng.integers(0, N, 200), [N - 1]]))
    for i in rows:
        assert np.array_equal(col[rp[i]:rp[i + 1]].astype(np.int64), O.knn_row(P, int(i), w)), i


def test_knn_grid_ties_lattice():
    """Integer lattice (many equal distances) through the grid path: the lowest
    position must win exactly as in the brute-force kernel."""
    g = np.stack(np.meshgrid(np.arange(40.0), np.arange(40.0), np.arange(40.0), indexing="ij"), -1).reshape(-1, 3)
    P = g[np.random.default_rng(0).permutation(len(g))]
    rp, col = afn.afn_knn_pattern(T(P), 27)
    rp, col = rp.cpu().numpy(), col.cpu().numpy()
    for i in list(range(0, 200)) + list(range(63000, 64000, 37)):
        assert np.array_equal(col[rp[i]:rp[i + 1]].astype(np.int64), O.knn_row(P, i, 27)), i


def test_knn_ties_lattice():
    """Integer lattice: many equal distances -> lowest position must win."""
    g = np.stack(np.meshgrid(np.arange(9.0), np.arange(9.0), indexing="ij"), -1).reshape(-1, 2)
    P = g[np.random.default_rng(0).permutation(len(g))]
    rp, col = afn.afn_knn_pattern(T(P), 12)
    rpo, colo = O.knn_lower(P, 12)
    assert np.array_equal(col.cpu().numpy().astype(np.int64), colo)


# --------------------------------------------------------------------------- build / apply / PCG
def _build_pair(X, l, mu, k, w):
    h = afn.afn_build(T(X), afn.make_params(l, mu, k, w))
    B = O.build_afn(X, l, mu, k, w)
    return h, B


def _check_build(h, B, g_tol=1e-10):
    assert np.array_equal(h.copy_out(afn.OUT_PERM), B["perm"])
    assert np.array_equal(h.copy_out(afn.OUT_FILL), B["fill"])
    L = h.copy_out(afn.OUT_L)
    assert np.abs(L - B["L"]).max() <= 1e-12 * np.abs(B["L"]).max()
    if B["n"] > B["k"]:
        W = h.copy_out(afn.OUT_W)
        assert np.abs(W - B["V"].T).max() <= 1e-11 * max(1.0, np.abs(B["V"]).max())
        assert np.array_equal(h.copy_out(afn.OUT_ROWPTR), B["row_ptr"])
        assert np.array_equal(h.copy_out(afn.OUT_COL).astype(np.int64), B["col"])
        g = h.copy_out(afn.OUT_GVAL)
        go = B["G"].data
        rp = B["row_ptr"]
        worst = max(np.linalg.norm(g[rp[i]:rp[i + 1]] - go[rp[i]:rp[i + 1]]) /
                    np.linalg.norm(go[rp[i]:rp[i + 1]]) for i in range(len(rp) - 1))
        assert worst <= g_tol, worst


@pytest.mark.parametrize("n,d,l,mu,k,w", [(1000, 3, 1.0, 1e-4, 100, 50), (700, 2, 0.7, 1e-3, 64, 20),
                                          (333, 3, 2.0, 1e-2, 333, 30), (500, 3, 1.0, 1e-4, 37, 1),
                                          (1500, 8, 3.0, 1e-2, 200, 64), (130, 1, 0.5, 1e-3, 10, 128)])
def test_build_apply_parity(n, d, l, mu, k, w):
    X, _ = gen_small(n, d, seed=8)
    h, B = _build_pair(X, l, mu, k, w)
    _check_build(h, B)
    rng = np.random.default_rng(2)
    for _ in range(2):
        r = rng.standard_normal(n)
        z = h.apply(T(r)).cpu().numpy()
        zo = np.empty(n)
        zo[B["perm"]] = O.apply_afn(B, r[B["perm"]])
        assert rel(z, zo) <= 1e-10


def test_apply_equals_dense_inverse_of_BBt():
    """GPU apply against (B B^T)^{-1} r built from the oracle's factors (eq:factorized-form)."""
    X, _ = gen_small(240, 3, seed=1, edge=6.0)
    h, B = _build_pair(X, 1.0, 1e-3, 40, 12)
    Bd = O.dense_B(B)
    r = np.random.default_rng(4).standard_normal(240)
    zd = np.empty(240)
    zd[B["perm"]] = np.linalg.solve(Bd @ Bd.T, r[B["perm"]])
    assert rel(h.apply(T(r)).cpu().numpy(), zd) <= 1e-10


@pytest.mark.parametrize("n,l,mu,k,w", [(1000, 1.0, 1e-4, 100, 50), (2000, 2.0, 1e-4, 150, 60),
                                        (1500, 0.5, 1e-3, 1500, 10)])
def test_pcg_parity(n, l, mu, k, w):
    X, b = gen_small(n, 3, seed=11)
    h, B = _build_pair(X, l, mu, k, w)
    a, rep = h.pcg_solve(T(b), tol=1e-4, maxit=500)
    ao, repo, _ = O.afn_pcg_solve(X, b, l, mu, k, w, tol=1e-4, B=B)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iterations"] - repo["iterations"]) <= 2
    assert rep["relres_true"] <= 1e-4 * 1.05
    it = rep["iterations"]
    a2, _ = h.pcg_solve(T(b), tol=1e-4, maxit=500, fixed_iters=it)
    ao2, _, _ = O.afn_pcg_solve(X, b, l, mu, k, w, tol=1e-4, fixed_iters=it, B=B)
    assert rel(a2.cpu().numpy(), ao2) <= 1e-6
    if k == n:
        assert it <= 2  # M = K + mu I exactly


def test_exact_fsai_pattern_converges_in_one_iteration():
    X, b = gen_small(120, 3, seed=3, edge=4.0)
    h = afn.afn_build(T(X), afn.make_params(1.0, 1e-3, 20, 128))
    a, rep = h.pcg_solve(T(b), tol=1e-10)
    assert rep["iterations"] <= 2
    ad = np.linalg.solve(O.kernel_block(X, X, 1.0) + 1e-3 * np.eye(120), b)
    assert rel(a.cpu().numpy(), ad) <= 1e-8


def test_c1_end_to_end_and_determinism():
    X, b = gen_problem("C1")
    h, B = _build_pair(X, 1.0, 1e-4, 100, 50)
    _check_build(h, B)
    a1, r1 = h.pcg_solve(T(b))
    a2, r2 = h.pcg_solve(T(b))
    assert torch.equal(a1, a2) and r1["iterations"] == r2["iterations"]
    h2 = afn.afn_build(T(X), afn.make_params(1.0, 1e-4, 100, 50))
    assert np.array_equal(h2.copy_out(afn.OUT_GVAL), h.copy_out(afn.OUT_GVAL))
    ao, ro, _ = O.afn_pcg_solve(X, b, 1.0, 1e-4, 100, 50, B=B)
    assert abs(r1["iterations"] - ro["iterations"]) <= 2


def test_solve_host_matches_device_path():
    X, b = gen_problem("C1")
    prm = afn.make_params(1.0, 1e-4, 100, 50)
    a_host, info, rep = afn.afn_solve_host(X, b, prm)
    h = afn.afn_build(T(X), prm)
    a_dev, rep2 = h.pcg_solve(T(b))
    assert np.array_equal(a_host, a_dev.cpu().numpy())
    assert info["k"] == 100 and rep["iterations"] == rep2["iterations"]


@pytest.fixture(scope="module")
def c2_pair():
    X, b = gen_problem("C2")
    h, B = _build_pair(X, 1.0, 1e-4, 2000, 100)
    return X, b, h, B


def test_c2_build_parity(c2_pair):
    X, b, h, B = c2_pair
    _check_build(h, B)


def test_c2_pcg_parity(c2_pair):
    X, b, h, B = c2_pair
    a, rep = h.pcg_solve(T(b))
    ao, ro, _ = O.afn_pcg_solve(X, b, 1.0, 1e-4, 2000, 100, B=B, threads=8)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2
    assert rep["relres_true"] <= 1e-4
    a2, _ = h.pcg_solve(T(b), fixed_iters=ro["iterations"])
    assert rel(a2.cpu().numpy(), ao) <= 1e-6


@pytest.mark.parametrize("l", [0.1, 0.5, 1.0, 2.0, 5.0, 10.0])
def test_c2_sweep_pcg_parity(l):
    """Every l of the bench's C2 sweep with Alg. 1's adaptive k (k = 2000, 130,
    54, ...) against the oracle's full AFN-PCG (tests/oracle_data, written by
    tools/make_oracle_fixtures.py from oracle/ only): Alg. 1 bit-exact, the
    same k, iterations +-2, true residual <= tol, solution <= 1e-6 at the
    oracle's iteration count."""
    import os
    fx = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_data", f"c2_l{l:g}.npz")
    o = np.load(fx)
    X, b = gen_problem("C2")
    bd = T(b)
    h = afn.afn_build(T(X), afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True))
    inf = h.info()
    if min(float(o["err_margin"]), float(o["ev_margin"])) >= 1e-9:
        assert (inf["khat"], inf["r"], inf["refined"]) == (int(o["khat"]), int(o["r"]), int(o["refined"]))
    assert inf["k"] == int(o["k"])
    a, rep = h.pcg_solve(bd, tol=1e-4)
    assert rep["converged"] == bool(o["converged"])
    assert abs(rep["iterations"] - int(o["iters"])) <= 2, (rep["iterations"], int(o["iters"]))
    assert rep["relres_true"] <= 1e-4
    a2, _ = h.pcg_solve(bd, fixed_iters=int(o["iters"]))
    assert rel(a2.cpu().numpy(), o["a"]) <= 1e-6
    h.close()


# --------------------------------------------------------------------------- Alg. 1
@pytest.mark.parametrize("cfg_l", [("C1", 1.0), ("C2", 0.1), ("C2", 0.5), ("C2", 1.0), ("C2", 2.0),
                                   ("C2", 5.0), ("C2", 10.0)])
def test_alg1_bit_exact_on_configs(cfg_l):
    """khat, r and the branch agree exactly (decisions are fp64 on both sides;
    a case whose decision margin is below 1e-9 would be reported ambiguous)."""
    cfg, l = cfg_l
    X, _ = gen_problem(cfg)
    res = afn.afn_estimate_rank(T(X), l)
    ro = O.alg1(X, l)
    margin = min(ro["err_margin"], ro["ev_margin"])
    if margin < 1e-9:
        pytest.skip(f"ambiguous decision margin {margin:g}")
    assert (res["khat"], res["r"], res["refined"]) == (ro["khat"], ro["r"], ro["refined"])


@pytest.mark.parametrize("n,d,l,m", [(1000, 3, 1e6, 100), (1000, 3, 1e-6, 100), (5000, 3, 1e-6, 100),
                                     (3000, 2, 1.5, 150), (2500, 8, 2.0, 120), (200000, 3, 1e6, 100)])
def test_alg1_special_cases(n, d, l, m):
    X, _ = gen_points(n, d, "cube", 0)
    res = afn.afn_estimate_rank(T(X), l, m=m)
    ro = O.alg1(X, l, m=m)
    assert (res["khat"], res["r"], res["refined"]) == (ro["khat"], ro["r"], ro["refined"])


@pytest.mark.gpu
@pytest.mark.parametrize("c,size", [(3, 40), (6, 20), (11, 7)])
def test_alg1_refined_branch_clusters(c, size):
    """c tight clusters far apart, m = n: refined count = r = c (closed form,
    see tests/test_oracle_pins.py) on the device, and the oracle agrees."""
    rng = np.random.default_rng(3)
    centres = 100.0 * np.arange(c)[:, None] * np.array([[1.0, 0.3, -0.2]])
    X = np.repeat(centres, size, axis=0) + 1e-7 * rng.standard_normal((c * size, 3))
    res = afn.afn_estimate_rank(T(X), 1.0, m=c * size)
    assert (res["khat"], res["r"], res["refined"]) == (c, c, True)
    ro = O.alg1(X, 1.0, m=c * size)
    assert (ro["khat"], ro["r"], ro["refined"]) == (c, c, True)


@pytest.mark.gpu
@pytest.mark.parametrize("l,f,want", [(0.5, 0.95, 1), (0.5, 1.05, 2), (1.0, 0.5, 1), (3.0, 3.0, 2)])
def test_alg1_refined_branch_two_points(l, f, want):
    """Two points: eigenvalues 1 +- exp(-r^2/l^2); count > 0.1 is 2 iff r^2/l^2 > ln(10/9)."""
    r = l * math.sqrt(f * math.log(10.0 / 9.0))
    X = np.array([[0.0, 0.0, 0.0], [r, 0.0, 0.0]])
    res = afn.afn_estimate_rank(T(X), l, m=2)
    assert res["refined"] and res["khat"] == want


def test_adaptive_build_uses_alg1_k():
    X, b = gen_problem("C2")
    h = afn.afn_build(T(X), afn.make_params(2.0, 1e-4, 2000, 100, k_adaptive=True))
    inf = h.info()
    ro = O.alg1(X, 2.0)
    assert inf["khat"] == ro["khat"] and inf["k"] == min(2000, max(1, ro["khat"]))
    a, rep = h.pcg_solve(T(b))
    assert rep["converged"] and rep["relres_true"] <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,l,kernel", [(2048, 3, 1.0, "gaussian"), (5000, 3, 0.3, "gaussian"),
                                          (4099, 5, 2.0, "gaussian"), (3333, 8, 3.0, "gaussian"),
                                          (6000, 3, 1.0, "matern32"), (2500, 2, 0.7, "matern32")])
def test_kmv_symmetric_plan(n, d, l, kernel):
    """The full matvec uses the symmetric kernel (each unordered pair once, row
    and column sums); it must agree with the oracle and, to rounding, with the
    non-symmetric row-range kernel on the same rows (ragged n, d up to 8, both
    kernels)."""
    X, _ = gen_points(n, d, "cube", 11)
    v = np.random.default_rng(n + d).standard_normal(n)
    y = afn.kernel_matvec(T(X), l, 1e-3, T(v), kernel=kernel).cpu().numpy()
    y_rows = afn.kernel_matvec_rows(T(X), l, 1e-3, T(v), 0, n, kernel=kernel).cpu().numpy()
    assert rel(y, y_rows) <= 1e-14
    rows = np.random.default_rng(3).choice(n, 200, replace=False)
    yo = O.kmv_rows(X, l, 1e-3, v, rows, kernel=kernel)
    assert rel(y[rows], yo) <= 1e-12

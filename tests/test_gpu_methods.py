"""GPU parity for the SURVEY.md 8(f) rows, through the C ABI, against the
oracle: Matern-3/2 kernel in the matvec, Alg. 1 and the AFN build;
uniform landmarks (reading R29); the Nystrom preconditioner and
Algorithm 2's choice (reading R30); plain FSAI of
K + mu I (k = 0).  Multi-rank (emulated) for the new methods."""
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


@pytest.mark.parametrize("n,d,l,mu", [(1, 3, 1.0, 1e-4), (1000, 3, 1.0, 1e-4), (2049, 8, 3.0, 1e-2),
                                      (777, 5, 0.3, 0.0), (3000, 3, 20.0, 1e-3)])
def test_matern_kmv_parity(n, d, l, mu):
    X, _ = gen_points(n, d, "cube", 3)
    v = np.random.default_rng(n).standard_normal(n)
    y = afn.kernel_matvec(T(X), l, mu, T(v), kernel="matern32").cpu().numpy()
    assert rel(y, O.kmv(X, l, mu, v, kernel="matern32")) <= 1e-12


@pytest.mark.parametrize("n,l", [(1000, 1.0), (1000, 5.0), (16384, 2.0), (16384, 20.0)])
def test_matern_alg1_bit_exact(n, l):
    X, _ = gen_points(n, 3, "cube", 0)
    res = afn.afn_estimate_rank(T(X), l, kernel="matern32")
    ro = O.alg1(X, l, kernel="matern32")
    if min(ro["err_margin"], ro["ev_margin"]) < 1e-9:
        pytest.skip("ambiguous decision margin")
    assert (res["khat"], res["r"], res["refined"]) == (ro["khat"], ro["r"], ro["refined"])


def _check_afn(h, B, n):
    assert np.array_equal(h.copy_out(afn.OUT_PERM), B["perm"])
    k = B["k"]
    if k > 0:
        L = h.copy_out(afn.OUT_L)
        assert np.abs(L - B["L"]).max() <= 1e-12 * np.abs(B["L"]).max()
    if n > k:
        assert np.array_equal(h.copy_out(afn.OUT_COL).astype(np.int64), B["col"])
        g, go, rp = h.copy_out(afn.OUT_GVAL), B["G"].data, B["row_ptr"]
        worst = max(rel(g[rp[i]:rp[i + 1]], go[rp[i]:rp[i + 1]]) for i in range(len(rp) - 1))
        assert worst <= 1e-10, worst


@pytest.mark.parametrize("kernel,landmarks,n,l,mu,k,w", [
    ("matern32", "fps", 1000, 2.0, 1e-4, 100, 50),
    ("matern32", "fps", 1500, 20.0, 1e-3, 200, 40),
    ("gaussian", "uniform", 1000, 1.0, 1e-4, 100, 50),
    ("matern32", "uniform", 1200, 5.0, 1e-2, 150, 30),
])
def test_afn_variants_build_apply_pcg(kernel, landmarks, n, l, mu, k, w):
    X, b = gen_small(n, 3, seed=4)
    lm = afn.LANDMARKS_UNIFORM if landmarks == "uniform" else afn.LANDMARKS_FPS
    h = afn.afn_build(T(X), afn.make_params(l, mu, k, w, kernel=kernel, landmarks=lm))
    B = O.build_afn(X, l, mu, k, w, kernel=kernel, landmarks=landmarks)
    _check_afn(h, B, n)
    r = np.random.default_rng(2).standard_normal(n)
    zo = np.empty(n)
    zo[B["perm"]] = O.apply_afn(B, r[B["perm"]])
    assert rel(h.apply(T(r)).cpu().numpy(), zo) <= 1e-10
    a, rep = h.pcg_solve(T(b), tol=1e-4)
    ao, ro, _ = O.afn_pcg_solve(X, b, l, mu, k, w, B=B, kernel=kernel)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2
    assert rep["relres_true"] <= 1e-4


@pytest.mark.parametrize("kernel,n,l,mu,k", [("gaussian", 1000, 3.0, 1e-2, 150),
                                             ("matern32", 1200, 10.0, 1e-2, 120),
                                             ("gaussian", 300, 1.0, 1e-2, 300)])
def test_nystrom_build_apply_pcg(kernel, n, l, mu, k):
    X, b = gen_small(n, 3, seed=6)
    h = afn.afn_build(T(X), afn.make_params(l, mu, k, 10, kernel=kernel, method=afn.METHOD_NYSTROM))
    inf = h.info()
    assert inf["method"] == afn.METHOD_NYSTROM and inf["k"] == k
    N = O.build_nystrom(X, l, mu, k, kernel=kernel)
    assert np.array_equal(h.copy_out(afn.OUT_PERM), N["perm"])
    r = np.random.default_rng(3).standard_normal(n)
    zo = np.empty(n)
    zo[N["perm"]] = O.apply_nystrom(N, r[N["perm"]])
    assert rel(h.apply(T(r)).cpu().numpy(), zo) <= 1e-8
    a, rep = h.pcg_solve(T(b), tol=1e-4)
    ao, ro, _ = O.afn_pcg_solve(X, b, l, mu, k, 10, B=N)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2
    assert rep["relres_true"] <= 1e-4
    if k == n:
        assert rep["iterations"] <= 2


def test_plain_fsai_matches_oracle():
    X, b = gen_small(800, 3, seed=9)
    h = afn.afn_build(T(X), afn.make_params(1.0, 1e-3, 1, 30, method=afn.METHOD_FSAI))
    assert h.info()["k"] == 0 and h.info()["method"] == afn.METHOD_FSAI
    B = O.build_precond(X, 1.0, 1e-3, 0, 30, method="fsai")
    _check_afn(h, B, 800)
    r = np.random.default_rng(5).standard_normal(800)
    assert rel(h.apply(T(r)).cpu().numpy(), O.apply_afn(B, r)) <= 1e-10
    a, rep = h.pcg_solve(T(b), tol=1e-4)
    ao, ro, _ = O.afn_pcg_solve(X, b, 1.0, 1e-3, 0, 30, B=B)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2


@pytest.mark.parametrize("l", [2.0, 5.0, 10.0])
def test_algorithm2_on_c2(l):
    """Alg. 2 at the bench workload: the branch follows Alg. 1's
    khat; the Nystrom branch's apply matches the oracle's eq:smw at full size.
    (At mu = 1e-4 the Nystrom branch with khat = 130 / 54 landmarks leaves the
    eigenvalues between mu and 0.1 unpreconditioned and PCG needs hundreds of
    iterations -- see DESIGN.md; the bench therefore keeps AFN.)"""
    X, b = gen_problem("C2")
    h = afn.afn_build(T(X), afn.make_params(l, 1e-4, 2000, 100, k_adaptive=True,
                                            method=afn.METHOD_ALG2))
    inf = h.info()
    ro = O.alg1(X, l)
    want = afn.METHOD_AFN if ro["khat"] >= 2000 else afn.METHOD_NYSTROM
    assert inf["method"] == want and inf["khat"] == ro["khat"]
    if want == afn.METHOD_NYSTROM:
        N = O.build_nystrom(X, l, 1e-4, inf["k"])
        assert np.array_equal(h.copy_out(afn.OUT_PERM), N["perm"])
        r = np.random.default_rng(3).standard_normal(len(X))
        zo = np.empty(len(X))
        zo[N["perm"]] = O.apply_nystrom(N, r[N["perm"]])
        assert rel(h.apply(T(r)).cpu().numpy(), zo) <= 1e-8
    a, rep = h.pcg_solve(T(b), tol=1e-4, maxit=500)
    assert not rep["breakdown"]
    assert rep["converged"] or rep["iterations"] == 500


@pytest.mark.parametrize("R,method", [(2, "nystrom"), (3, "nystrom"), (2, "fsai"), (4, "fsai")])
def test_emulated_ranks_new_methods(R, method):
    X, b = gen_small(1000, 3, seed=12)
    m = afn.METHOD_NYSTROM if method == "nystrom" else afn.METHOD_FSAI
    prm = afn.make_params(2.0, 1e-2, 200, 40, method=m)
    h1 = afn.afn_build(T(X), prm)
    comm = afn.Comm.emulated(R)
    hR = afn.afn_build(T(X), prm, comm=comm)
    r = T(np.random.default_rng(7).standard_normal(1000))
    assert rel(hR.apply(r).cpu().numpy(), h1.apply(r).cpu().numpy()) <= 1e-11
    a1, rep1 = h1.pcg_solve(T(b))
    aR, repR = hR.pcg_solve(T(b))
    assert repR["iterations"] == rep1["iterations"] and repR["converged"]
    # The rank split sums partials (matvec pair units, F^T r, the Gram) in rank
    # order: a rounding-level perturbation of every product, which PCG on a
    # system with cond(K + mu I) ~ 1e5 (mu = 1e-2) amplifies like any other.
    # Measured, not assumed: the one-GPU solve's own sensitivity to a one-ulp
    # perturbation of b at the same iteration count bounds the gap (x 100:
    # the split perturbs every iteration, b only the start), under the north
    # star's 1e-6.
    its = rep1["iterations"]
    sgn = np.random.default_rng(8).choice([-1.0, 1.0], len(b))
    ap, _ = h1.pcg_solve(T(b * (1.0 + np.finfo(float).eps * sgn)), fixed_iters=its)
    sens = rel(ap.cpu().numpy(), a1.cpu().numpy())
    gap = rel(aR.cpu().numpy(), a1.cpu().numpy())
    assert gap <= max(1e-12, 100.0 * sens) and gap <= 1e-6, (gap, sens)
    hR.close()
    comm.close()


@pytest.mark.parametrize("n,l,mu,k,w,adaptive", [(1000, 1.0, 1e-4, 100, 50, False),
                                                  (1500, 2.0, 1e-3, 200, 40, False),
                                                  (2000, 1.0, 1e-4, 2000, 60, True)])
def test_maxmin_ordering_parity(n, l, mu, k, w, adaptive):
    """MaxMin ordering (f4): FPS through all n points fixes the order of
    the non-landmark points; permutation bit-exact, G rows, apply, PCG."""
    X, b = gen_small(n, 3, seed=13)
    h = afn.afn_build(T(X), afn.make_params(l, mu, k, w, k_adaptive=adaptive, ordering=afn.ORDER_MAXMIN))
    kk = h.info()["k"]
    B = O.build_afn(X, l, mu, kk, w, ordering="maxmin")
    _check_afn(h, B, n)
    r = np.random.default_rng(2).standard_normal(n)
    zo = np.empty(n)
    zo[B["perm"]] = O.apply_afn(B, r[B["perm"]])
    assert rel(h.apply(T(r)).cpu().numpy(), zo) <= 1e-10
    a, rep = h.pcg_solve(T(b), tol=1e-4)
    ao, ro, _ = O.afn_pcg_solve(X, b, l, mu, kk, w, B=B)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2


@pytest.mark.parametrize("n,l,mu,k,R", [(1000, 2.0, 1e-2, 150, 1), (1500, 1.0, 1e-3, 300, 1),
                                        (300, 1.0, 1e-2, 300, 1), (1000, 2.0, 1e-2, 150, 3)])
def test_ran_parity(n, l, mu, k, R):
    """RAN (f3): lambda_k and the apply against the oracle's SVD route,
    PCG iterations +-2; k = n gives the scaled exact inverse (one iteration)."""
    X, b = gen_small(n, 3, seed=17)
    prm = afn.make_params(l, mu, k, 10, landmarks=afn.LANDMARKS_UNIFORM, method=afn.METHOD_RAN)
    comm = afn.Comm.emulated(R) if R > 1 else None
    h = afn.afn_build(T(X), prm, comm=comm)
    assert h.info()["method"] == afn.METHOD_RAN
    Ro = O.build_ran(X, l, mu, k)
    assert np.array_equal(h.copy_out(afn.OUT_PERM), Ro["perm"])
    r = np.random.default_rng(3).standard_normal(n)
    zo = np.empty(n)
    zo[Ro["perm"]] = O.apply_ran(Ro, r[Ro["perm"]])
    assert rel(h.apply(T(r)).cpu().numpy(), zo) <= 1e-8
    a, rep = h.pcg_solve(T(b), tol=1e-4)
    ao, ro, _ = O.afn_pcg_solve(X, b, l, mu, k, 10, B=Ro)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 2
    if k == n:
        assert rep["iterations"] <= 2
    h.close()

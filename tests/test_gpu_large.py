"""GPU parity at BASELINE.json's full sizes C3 (n = 2^17), C4 (n = 2^18, d = 8)
and C5 (n = 2^20), where the oracle cannot run the whole solve (one oracle
matvec at C5 is 1.1e12 kernel evaluations).  Parity is therefore checked by
component:

  * Alg. 1 (k-hat, r, branch) and ALL k FPS landmarks + fill trace: bit-exact
    against the oracle run in full;
  * permutation: landmarks first, then the rest ascending (R14);
  * kNN pattern rows, W = (L^{-1} K12)^T rows and FSAI rows on a sample of
    non-landmark positions (always including the first and the last rows),
    with the oracle's own L, landmarks and pattern;
  * kernel matvec on sampled rows (<= 1e-12 relative);
  * PCG: converged with the GPU's true relative residual <= tol, the GPU
    matvec that computes it being checked on sampled rows of the solution.

C5 (~70 GB of device memory, W is 66.6 GB) runs in the default suite with a
bounded oracle: the first 1000 FPS landmarks and their fill trace bit-exact
(FPS is nested, so they are the first 1000 of the device's 8000), the
landmark set's remaining structure checked directly, and the factor checks
on the device's landmark set with the oracle's own L, W and FSAI rows.

C3 also has a full oracle PCG (tests/oracle_data/c3_l1.npz, written by
tools/make_oracle_fixtures.py from oracle/ only): same iteration count +-2,
solution <= 1e-6 at the oracle's iteration count."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from synth import CONFIGS, gen_problem

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


def sample_rows(N, count, seed):
    rng = np.random.default_rng(seed)
    s = set(rng.choice(N, min(N, count), replace=False).tolist())
    s.update({0, min(1, N - 1), N - 1, N // 2})
    return np.array(sorted(s), dtype=np.int64)


import json
import os

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_data")

CASES = [pytest.param("C3", 1.0, id="C3-l1"),
         pytest.param("C4", 1.0, id="C4-l1"),
         pytest.param("C4", 3.0, id="C4-l3"),
         pytest.param("C5", 1.0, id="C5-l1")]
# oracle FPS prefix checked at C5 (the full k = 8000 oracle FPS over 2^20 points
# takes minutes; the prefix is exact because FPS is nested)
C5_FPS_PREFIX = 1000


@pytest.mark.parametrize("name,l", CASES)
def test_full_size_component_parity(name, l):
    cfg = CONFIGS[name]
    X, b = gen_problem(cfg)
    n = cfg.n
    Xd, bd = T(X), T(b)
    afn.kernel_timers(reset=True, enable=True)
    h = afn.afn_build(Xd, afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True))
    kt = afn.kernel_timers(enable=False)
    inf = h.info()
    # the FSAI rows come from the pair-union product (no union overflowed into
    # the per-row Gram fallback), W from the INT8 path when k >= 512 (d = 3)
    if cfg.d == 3:
        assert kt["fsai_gram_kernel"]["count"] == 0 and kt["group_gemm_kernel"]["count"] > 0

    # ---- Alg. 1: bit-exact decisions
    ro = O.alg1(X, l)
    if min(ro["err_margin"], ro["ev_margin"]) >= 1e-9:
        assert (inf["khat"], inf["r"], bool(inf["refined"])) == (ro["khat"], ro["r"], ro["refined"])
    k = min(cfg.k_cap, max(1, ro["khat"]), n)
    assert inf["k"] == k

    # ---- FPS: the landmarks and the fill trace bit-exact (all k,
    # or the first C5_FPS_PREFIX at C5: nested)
    kc = k if name != "C5" else C5_FPS_PREFIX
    idx, fill = O.fps(X, kc, 0)
    perm = h.copy_out(afn.OUT_PERM)
    assert np.array_equal(perm[:kc], idx)
    assert np.array_equal(h.copy_out(afn.OUT_FILL)[:kc], fill)
    idx = perm[:k]  # (== the oracle's when kc == k)
    assert len(np.unique(idx)) == k and idx.min() >= 0 and idx.max() < n
    if kc < k:  # the remaining landmarks: each is the farthest point when picked
        fl = h.copy_out(afn.OUT_FILL)
        assert np.all(np.diff(fl) <= 0.0)
        for t in (kc, k // 2, k - 1):
            d2 = O.sqdist_block(X[idx[t]][None, :], X[idx[:t]]).min()
            assert d2 == fl[t - 1] ** 2 or math.isclose(math.sqrt(d2), fl[t - 1], rel_tol=1e-15)
    rest = perm[k:]
    mask = np.ones(n, bool)
    mask[idx] = False
    perm_o = np.concatenate([idx, np.nonzero(mask)[0]])
    assert np.array_equal(rest, perm_o[k:])  # ascending original ids (R14)

    # ---- oracle factors on its own landmarks
    Xp = X[perm_o]
    X1, X2 = Xp[:k], Xp[k:]
    N2 = n - k
    L = np.linalg.cholesky(O.kernel_block(X1, X1, l) + cfg.mu * np.eye(k))
    lrows = sample_rows(k, 24, 5)
    Lg = h.copy_out_rows(afn.OUT_L, lrows)
    assert np.abs(Lg - L[lrows]).max() <= 1e-12 * np.abs(L).max()

    def V_cols(J):  # V = L^{-1} K12 on the columns J
        return sla.solve_triangular(L, O.kernel_block(X1, X2[J], l), lower=True)

    rows = sample_rows(N2, 32 if name == "C5" else 40, 7)
    Wg = h.copy_out_rows(afn.OUT_W, rows)
    Vo = V_cols(rows)
    assert np.abs(Wg - Vo.T).max() <= 1e-11 * max(1.0, np.abs(Vo).max())

    # ---- kNN rows: bit-exact; FSAI rows: 1e-10 per row
    rp = h.copy_out(afn.OUT_ROWPTR)
    col = h.copy_out(afn.OUT_COL)
    gv = h.copy_out(afn.OUT_GVAL)
    worst = 0.0
    for i in rows:
        J = O.knn_row(X2, int(i), cfg.w)
        a, e = rp[i], rp[i + 1]
        assert np.array_equal(col[a:e].astype(np.int64), J), f"pattern row {i}"
        VJ = V_cols(J)
        SJ = O.kernel_block(X2[J], X2[J], l) + cfg.mu * np.eye(len(J)) - VJ.T @ VJ
        go = O.fsai_rows(lambda _J: SJ, np.array([0, len(J)]), J)
        worst = max(worst, rel(gv[a:e], go))
    assert worst <= 1e-10, worst

    # ---- kernel matvec on sampled rows, original order
    v = np.random.default_rng(3).standard_normal(n)
    y = afn.kernel_matvec(Xd, l, cfg.mu, T(v)).cpu().numpy()
    mrows = sample_rows(n, 64, 9)
    assert rel(y[mrows], O.kmv_rows(X, l, cfg.mu, v, mrows)) <= 1e-12

    # ---- PCG
    # C4 does not converge within maxit (see below): 60 iterations show the trend
    maxit = 60 if name == "C4" else cfg.maxit
    a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=maxit, history=True)
    hist = rep.pop("history")
    print(name, l, inf, rep, hist[:: max(1, len(hist) // 20)])
    assert not rep["breakdown"]
    if name == "C4":
        # d = 8, mu = 1e-2: the iteration count of this workload grows ~2.4x per
        # doubling of n (19/40/95/252 at n = 2^13..2^16, oracle-confirmed at
        # 2^13..2^15), so at n = 2^18 PCG reaches maxit = 500
        # without the tolerance -- the paper's "-".  Steady progress only.
        assert rep["converged"] or (rep["iterations"] == maxit and rep["relres_true"] < 1.0)
        assert np.all(np.isfinite(hist)) and hist[-1] < 0.5 * hist.max()
    else:
        assert rep["converged"] and rep["relres_true"] <= cfg.tol
    an = a.cpu().numpy()
    ya = afn.kernel_matvec(Xd, l, cfg.mu, a).cpu().numpy()
    # the solution has large entries whose products cancel (|(K+mu I) a| << (K+mu I)|a|),
    # so the matvec is checked against its rounding scale (K+mu I)|a| (K >= 0)
    scale = O.kmv_rows(X, l, cfg.mu, np.abs(an), mrows)
    assert np.max(np.abs(ya[mrows] - O.kmv_rows(X, l, cfg.mu, an, mrows)) / scale) <= 1e-13
    res = b - ya
    assert math.isclose(np.linalg.norm(res) / np.linalg.norm(b), rep["relres_true"],
                        rel_tol=1e-6, abs_tol=1e-12)
    print(f"{name} l={l}: k={k} khat={inf['khat']} iters={rep['iterations']} "
          f"relres_true={rep['relres_true']:.3e} setup_ms={inf['ms_total']:.1f} "
          f"solve_ms={rep['solve_ms']:.1f}")
    fx = os.path.join(DATA, f"{name.lower()}_l{l:g}.npz")
    if name == "C3" and os.path.exists(fx):
        # full oracle PCG (tools/make_oracle_fixtures.py): +-2 iterations,
        # <= 1e-6 at the oracle's own count
        o = np.load(fx)
        assert int(o["k"]) == k
        assert abs(rep["iterations"] - int(o["iters"])) <= 2, (rep["iterations"], int(o["iters"]))
        a2, _ = h.pcg_solve(bd, fixed_iters=int(o["iters"]))
        assert rel(a2.cpu().numpy(), o["a"]) <= 1e-6
    h.close()


def test_c4_shape_iteration_trend():
    """C4's shape (d = 8 N(0,1), mu = 1e-2, l = 1, w = 64) at n = 2^13..2^15 with
    k = 1000: the device's PCG iteration counts match the oracle's committed
    ones (tests/oracle_data/c4_shape_iters.json, tools/make_oracle_fixtures.py)
    within +-2 -- the growth with n behind C4's non-convergence at 2^18 is the
    method's, not the implementation's (P:L828's "-")."""
    from synth import gen_points
    fx = os.path.join(DATA, "c4_shape_iters.json")
    ref = json.load(open(fx))["results"]
    for n_s, r in ref.items():
        n = int(n_s)
        X, rng = gen_points(n, 8, "normal", 0)
        b = rng.standard_normal(n)
        h = afn.afn_build(T(X), afn.make_params(1.0, 1e-2, 1000, 64))
        _, rep = h.pcg_solve(T(b), tol=1e-4, maxit=500)
        h.close()
        assert rep["converged"] == r["converged"]
        assert abs(rep["iterations"] - r["iters"]) <= 2, (n, rep["iterations"], r["iters"])

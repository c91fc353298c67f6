"""Plain fp64 NumPy/SciPy oracle of the AFN-preconditioned CG hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Citations: P:L<n> is
PAPER.md line n; R<n> is reading n of DESIGN.md / SURVEY.md 8(c).

Conventions that make the integer-valued steps bit-exact against any
implementation that follows the same readings:
  * squared distances are accumulated per coordinate in index order with
    separate, individually rounded subtract / multiply / add operations
    (``_sqdist_*``; NumPy elementwise ufuncs never fuse into FMAs), R3;
  * argmax / k-nearest selections use the total order (d2, index), lowest
    index first (np.argmax returns the first maximum, argsort kind="stable").
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

__all__ = [
    "sqdist_to", "sqdist_block", "kernel_block", "kmv", "kmv_rows",
    "fps", "fill_distance", "separation_distance", "knn_lower", "knn_row",
    "splitmix64", "subsample_ids", "default_m", "alg1",
    "fsai_rows", "build_afn", "apply_afn", "dense_B", "pcg", "afn_pcg_solve",
    "cg_solve", "kernel_from_d2", "uniform_landmarks", "build_nystrom", "apply_nystrom",
    "choose_method", "build_precond", "apply_precond", "KERNELS", "NYS_NU", "UNIFORM_SEED_XOR",
    "build_ran", "apply_ran",
]

KERNELS = ("gaussian", "matern32")
NYS_NU = 1e-10          # K11 shift of the Nystrom preconditioner (reading R30)
UNIFORM_SEED_XOR = 0x6A09E667F3BCC909  # landmark key stream (reading R29)

EPS = np.finfo(np.float64).eps


# ----------------------------------------------------------------------------
# Distances and the Gaussian kernel  (P:L33-41 eq:Problem / eq:gaussianf)
# ----------------------------------------------------------------------------
def sqdist_to(P: np.ndarray, y: np.ndarray) -> np.ndarray:
    """d2[i] = sum_c (P[i,c] - y[c])^2, c = 0..d-1 in order, no FMA (R3)."""
    P = np.asarray(P, dtype=np.float64)
    d2 = None
    for c in range(P.shape[1]):
        diff = P[:, c] - y[c]
        t = diff * diff
        d2 = t if d2 is None else d2 + t
    return d2


def sqdist_block(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """|A| x |B| matrix of squared distances, same per-coordinate order."""
    d2 = None
    for c in range(A.shape[1]):
        diff = A[:, c][:, None] - B[:, c][None, :]
        t = diff * diff
        d2 = t if d2 is None else d2 + t
    return d2


def kernel_from_d2(d2, l: float, kernel: str = "gaussian"):
    """Kernel value from the squared distance:
    gaussian  exp(-d2 / l^2)  (no factor 1/2, R1);
    matern32  (1 + sqrt(3) r / l) exp(-sqrt(3) r / l), r = sqrt(d2)."""
    if kernel == "gaussian":
        return np.exp(-d2 / (l * l))
    if kernel == "matern32":
        t = math.sqrt(3.0) * np.sqrt(d2) / l
        return (1.0 + t) * np.exp(-t)
    raise ValueError(f"unknown kernel {kernel!r}")


def kernel_block(A: np.ndarray, B: np.ndarray, l: float, kernel: str = "gaussian") -> np.ndarray:
    """K_AB."""
    return kernel_from_d2(sqdist_block(A, B), l, kernel)


def kmv_rows(X: np.ndarray, l: float, mu: float, v: np.ndarray, rows: np.ndarray,
             block: int = 256, kernel: str = "gaussian") -> np.ndarray:
    """y_i = sum_j K(x_i, x_j) v_j + mu v_i for the listed rows i."""
    rows = np.asarray(rows)
    out = np.empty(len(rows))
    for s in range(0, len(rows), block):
        r = rows[s:s + block]
        out[s:s + block] = kernel_block(X[r], X, l, kernel) @ v + mu * v[r]
    return out


def kmv(X: np.ndarray, l: float, mu: float, v: np.ndarray, block: int = 256,
        threads: int | None = None, kernel: str = "gaussian") -> np.ndarray:
    """(K + mu I) v with K never stored whole (explicit matvec).

    Row blocks; with ``threads`` > 1 the blocks go to a thread pool (NumPy
    releases the GIL inside exp and the block GEMV).  Used for timing too.
    """
    X = np.asarray(X, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n = X.shape[0]
    y = np.empty(n)

    def work(s):
        e = min(n, s + block)
        y[s:e] = kernel_block(X[s:e], X, l, kernel) @ v + mu * v[s:e]

    starts = range(0, n, block)
    if threads and threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, starts))
    else:
        for s in starts:
            work(s)
    return y


# ----------------------------------------------------------------------------
# Farthest point sampling  (eq. (3.3); brute force)
# ----------------------------------------------------------------------------
def fps(X: np.ndarray, k: int, seed: int = 0):
    """Select k landmarks: x_{k_{i+1}} = argmax_{x not in X_i} dist(x, X_i).

    Returns (idx int64[k], fill_trace float64[k]) where fill_trace[i] is the
    fill distance h_{X_{i+1}} over the discrete set X (eq:filldistance,
    P:L364) after i+1 selections, i.e. sqrt of the max running min-distance
    (0 once every point is selected).  Ties -> lowest index; selected points
    are excluded explicitly (mind = -1) so duplicates are never re-picked (R3).
    The argmax is over d2, not d (sqrt could merge distinct d2).
    """
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    if not (1 <= k <= n) or not (0 <= seed < n):
        raise ValueError("need 1 <= k <= n and 0 <= seed < n")
    idx = np.empty(k, dtype=np.int64)
    fill = np.empty(k)
    idx[0] = seed
    mind = sqdist_to(X, X[seed])
    mind[seed] = -1.0
    for i in range(1, k + 1):
        j = int(np.argmax(mind))
        fill[i - 1] = math.sqrt(mind[j]) if mind[j] >= 0.0 else 0.0
        if i == k:
            break
        idx[i] = j
        mind = np.minimum(mind, sqdist_to(X, X[j]))
        mind[j] = -1.0
    return idx, fill


def fill_distance(X, sel) -> float:
    """h_{X_k} over the discrete set X: max_{x in X\\X_k} min_{y in X_k} ||x-y||."""
    X = np.asarray(X, dtype=np.float64)
    sel = np.asarray(sel)
    mask = np.ones(len(X), bool)
    mask[sel] = False
    if not mask.any():
        return 0.0
    d2 = sqdist_block(X[mask], X[sel]).min(axis=1)
    return float(np.sqrt(d2.max()))


def separation_distance(X, sel) -> float:
    """q_{X_k}: closest distinct pair in X_k."""
    P = np.asarray(X, dtype=np.float64)[np.asarray(sel)]
    d2 = sqdist_block(P, P)
    np.fill_diagonal(d2, np.inf)
    return float(np.sqrt(d2.min()))


# ----------------------------------------------------------------------------
# FSAI sparsity pattern
# ----------------------------------------------------------------------------
def knn_row(P: np.ndarray, i: int, w: int) -> np.ndarray:
    """Pattern of row i: the min(w-1, i) nearest positions j < i by
    the total order (d2, j) (R3), ascending, then i itself (R15)."""
    if i == 0 or w == 1:
        nb = np.empty(0, dtype=np.int64)
    else:
        d2 = sqdist_to(P[:i], P[i])
        nb = np.argsort(d2, kind="stable")[: w - 1]
    return np.concatenate([np.sort(nb), [i]]).astype(np.int64)


def knn_lower(P: np.ndarray, w: int):
    """Row i = {i} plus its min(w-1, i) nearest neighbours among positions < i.

    w counts the diagonal (R15).  Ties -> lower position (R3).  Columns are
    ascending, so the diagonal is last.  Returns (row_ptr int64[N+1], col int64[nnz]).
    """
    P = np.asarray(P, dtype=np.float64)
    N = P.shape[0]
    if w < 1:
        raise ValueError("w >= 1")
    row_ptr = np.zeros(N + 1, dtype=np.int64)
    cols = []
    for i in range(N):
        row = knn_row(P, i, w)
        cols.append(row)
        row_ptr[i + 1] = row_ptr[i] + len(row)
    col = np.concatenate(cols) if cols else np.empty(0, dtype=np.int64)
    return row_ptr, col


# ----------------------------------------------------------------------------
# Algorithm 1: Nystrom rank estimation
# ----------------------------------------------------------------------------
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    """SplitMix64 output function of state x (counter-based generator, R7)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def subsample_ids(n: int, m: int, rng_seed: int = 0) -> np.ndarray:
    """'Randomly subsample a subset X_m of m points', read as R7:
    h_i = splitmix64(seed XOR i*golden); the m indices with smallest h, by ascending h."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(rng_seed) ^ (i * _GOLDEN))
    return np.argsort(h, kind="stable")[:m].astype(np.int64)


def default_m(n: int) -> int:
    """Subsample size (R6): min(500, max(100, n//100)), capped at n."""
    return min(n, min(500, max(100, n // 100)))


def alg1(X: np.ndarray, l: float, m: int | None = None, rng_seed: int = 0,
         k_threshold: int = 2000, err_tol: float = 0.1, ev_tol: float = 0.1,
         kernel: str = "gaussian"):
    """Algorithm 1 step by step.

    1. subsample m points, scale coordinates by s = (m/n)^(1/d)       (L666, R8)
    2. form K_m = K_{X_m,X_m}                                           (L667)
    3. FPS on X_m (seed = subsample position 0); smallest r with
       ||K_m - K_nys,r||_2 / ||K_m||_2 < 0.1, where K_m - K_nys,r = Schur
       complement S^(r) after r elimination steps in FPS order (R9);
       a pivot <= m*eps*||K_m||_2 counts as exhausted (R10)            (L668)
    4. k = r n / m, rounded half up (R11)                               (L669)
    5. if k >= 2000 return k, else return #{eig(K_m unscaled) > 0.1}    (L670-675, R13)
    Returns dict(khat, r, m, refined, err_margin, ev_margin, errs).
    """
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    if m is None:
        m = default_m(n)
    ids = subsample_ids(n, m, rng_seed)
    s = (m / n) ** (1.0 / d)
    Xm = X[ids] * s
    Km = kernel_block(Xm, Xm, l, kernel)
    order, _ = fps(Xm, m, 0)
    S = Km[np.ix_(order, order)].copy()
    normK = float(np.max(np.abs(np.linalg.eigvalsh(Km))))
    thr = m * EPS * normK
    errs = []
    r_sel = m
    for r in range(1, m + 1):
        p = S[r - 1, r - 1]
        if p > thr:
            S[r:, r:] -= np.outer(S[r:, r - 1], S[r - 1, r:]) / p
        S[r - 1, :] = 0.0
        S[:, r - 1] = 0.0
        T = S[r:, r:]
        err = float(np.max(np.abs(np.linalg.eigvalsh(T)))) / normK if r < m else 0.0
        errs.append(err)
        if err < err_tol:
            r_sel = r
            break
    khat = (2 * r_sel * n + m) // (2 * m)
    err_margin = abs(errs[-1] - err_tol)
    if len(errs) > 1:
        err_margin = min(err_margin, abs(errs[-2] - err_tol))
    refined = False
    ev_margin = float("inf")
    if khat < k_threshold:
        Xu = X[ids]
        ev = np.linalg.eigvalsh(kernel_block(Xu, Xu, l, kernel))
        khat = int(np.count_nonzero(ev > ev_tol))
        ev_margin = float(np.min(np.abs(ev - ev_tol)))
        refined = True
    return dict(khat=int(khat), r=int(r_sel), m=int(m), refined=refined,
                err_margin=float(err_margin), ev_margin=ev_margin, errs=np.array(errs),
                ids=ids, scale=s)


# ----------------------------------------------------------------------------
# FSAI of an SPD matrix given by entries on the pattern
# ----------------------------------------------------------------------------
def fsai_rows(S_sub, row_ptr, col):
    """Kolotilina-Yeremin FSAI (R16).

    For row i with pattern J (ascending, i last): y = S_JJ^{-1} e_last,
    g_J = y / sqrt(y_last), so that (G~ S)_{iJ} = e_i on the pattern and
    diag(G S G^T) = 1.  ``S_sub(J)`` returns the dense |J|x|J| block S_JJ.
    Returns values aligned with ``col``.
    """
    vals = np.empty(len(col))
    N = len(row_ptr) - 1
    for i in range(N):
        a, b = row_ptr[i], row_ptr[i + 1]
        J = col[a:b]
        SJ = S_sub(J)
        e = np.zeros(len(J))
        e[-1] = 1.0
        y = np.linalg.solve(SJ, e)
        if not (y[-1] > 0.0):
            raise np.linalg.LinAlgError(f"FSAI row {i}: S_JJ not SPD")
        vals[a:b] = y / math.sqrt(y[-1])
    return vals


# ----------------------------------------------------------------------------
# AFN build
# ----------------------------------------------------------------------------
def uniform_landmarks(n: int, k: int, rng_seed: int = 0) -> np.ndarray:
    """Uniformly random landmarks, the paper's choice for its high-dimensional
    datasets, read as R29: the k smallest splitmix64 keys of the
    stream rng_seed ^ 0x6A09E667F3BCC909 (the generator of subsample_ids)."""
    return subsample_ids(n, k, int(rng_seed) ^ UNIFORM_SEED_XOR)


def _landmarks(X, k, landmarks, fps_seed, rng_seed):
    n = len(X)
    if k == 0:
        return np.empty(0, dtype=np.int64), np.empty(0)
    if landmarks == "fps":
        return fps(X, k, fps_seed)
    if landmarks == "uniform":
        return uniform_landmarks(n, k, rng_seed), np.zeros(k)
    raise ValueError(f"unknown landmarks {landmarks!r}")


def build_afn(X: np.ndarray, l: float, mu: float, k: int, w: int, fps_seed: int = 0,
              kernel: str = "gaussian", landmarks: str = "fps", rng_seed: int = 0,
              ordering: str = "index"):
    """Build the AFN factors, paper-literal.

    * X_k by FPS; landmarks indexed first, the rest
      in ascending original id (R14): perm = [idx; rest].
    * L L^T = K11 + mu I
    * K12 explicit and V = L^{-1} K12 (block of eq:factorized-form)
    * pattern: kNN lower on the non-landmarks
    * G by FSAI of S = K22 + mu I - K12^T (K11 + mu I)^{-1} K12 on the pattern
      (P:L211-212, L248-261): S_JJ = K_JJ + mu I - V_J^T V_J.
    """
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    k = int(min(k, n))  # k = 0: plain FSAI of K + mu I
    if ordering == "maxmin":
        # MaxMin ordering: FPS continued through all n points; the
        # first k are the landmarks, the rest keep their FPS order
        if landmarks != "fps":
            raise ValueError("the MaxMin ordering continues FPS")
        perm, fill_all = fps(X, n, fps_seed)
        idx, fill = perm[:k], fill_all[:k]
    else:  # ascending original index after the landmarks (R14)
        idx, fill = _landmarks(X, k, landmarks, fps_seed, rng_seed)
        mask = np.ones(n, bool)
        mask[idx] = False
        rest = np.nonzero(mask)[0].astype(np.int64)
        perm = np.concatenate([idx, rest]).astype(np.int64)
    Xp = X[perm]
    X1, X2 = Xp[:k], Xp[k:]
    A11 = kernel_block(X1, X1, l, kernel) + mu * np.eye(k)
    L = np.linalg.cholesky(A11) if k > 0 else np.zeros((0, 0))
    K12 = kernel_block(X1, X2, l, kernel)
    V = sla.solve_triangular(L, K12, lower=True) if k > 0 else np.zeros((0, n))
    N2 = n - k
    if N2 > 0:
        row_ptr, col = knn_lower(X2, w)

        def S_sub(J):
            return kernel_block(X2[J], X2[J], l, kernel) + mu * np.eye(len(J)) - V[:, J].T @ V[:, J]

        gv = fsai_rows(S_sub, row_ptr, col)
        G = sp.csr_matrix((gv, col, row_ptr), shape=(N2, N2))
    else:
        row_ptr = np.zeros(1, dtype=np.int64)
        col = np.empty(0, dtype=np.int64)
        G = sp.csr_matrix((0, 0))
    return dict(method="afn" if k > 0 else "fsai", n=n, k=k, w=w, l=l, mu=mu, kernel=kernel,
                idx=idx, fill=fill, perm=perm, Xp=Xp, L=L, K12=K12, V=V, row_ptr=row_ptr,
                col=col, G=G)


def apply_afn(B: dict, r: np.ndarray) -> np.ndarray:
    """Solve M s = r with the paper's two-step algorithm:
       s2 = G^T G (r2 - K12^T (L^{-T} L^{-1}) r1)
       s1 = L^{-T} L^{-1} (r1 - K12 s2)
    r and s are in the permuted (landmarks-first) order."""
    k, L, K12, G = B["k"], B["L"], B["K12"], B["G"]
    r = np.asarray(r, dtype=np.float64)
    r1, r2 = r[:k], r[k:]

    def LLt_solve(v):
        if k == 0:
            return np.empty(0)
        return sla.solve_triangular(L.T, sla.solve_triangular(L, v, lower=True), lower=False)

    if k == 0:  # plain FSAI: M^{-1} = G^T G
        return G.T @ (G @ r2)
    if len(r2):
        s2 = G.T @ (G @ (r2 - K12.T @ LLt_solve(r1)))
        s1 = LLt_solve(r1 - K12 @ s2)
    else:
        s2 = np.empty(0)
        s1 = LLt_solve(r1)
    return np.concatenate([s1, s2])


def build_nystrom(X: np.ndarray, l: float, mu: float, k: int, fps_seed: int = 0,
                  kernel: str = "gaussian", landmarks: str = "fps", rng_seed: int = 0,
                  nu: float = NYS_NU):
    """Nystrom preconditioner K_nys + mu I on k landmarks indexed
    first, K_nys = K_{X,Xk} (K11 + nu I)^{-1} K_{Xk,X} (R30: the
    paper cites stabilised implementations; nu = 1e-10)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    k = int(min(max(k, 1), n))
    idx, fill = _landmarks(X, k, landmarks, fps_seed, rng_seed)
    mask = np.ones(n, bool)
    mask[idx] = False
    perm = np.concatenate([idx, np.nonzero(mask)[0]]).astype(np.int64)
    Xp = X[perm]
    X1 = Xp[:k]
    K11 = kernel_block(X1, X1, l, kernel)
    K12 = kernel_block(X1, Xp[k:], l, kernel)
    return dict(method="nystrom", n=n, k=k, l=l, mu=mu, nu=nu, kernel=kernel, idx=idx,
                fill=fill, perm=perm, Xp=Xp, K11=K11, K12=K12)


def apply_nystrom(N: dict, r: np.ndarray) -> np.ndarray:
    """(K_nys + mu I)^{-1} r by the SMW formula eq:smw, with
    K11 -> K11 + nu I in the inner matrix (R30):
      r/mu - (1/mu^2) [K11 K12]^T (K11 + nu I + (K11^2 + K12 K12^T)/mu)^{-1} [K11 K12] r.
    r in the permuted (landmarks-first) order."""
    K11, K12, mu, nu, k = N["K11"], N["K12"], N["mu"], N["nu"], N["k"]
    r = np.asarray(r, dtype=np.float64)
    A = np.hstack([K11, K12])
    inner = K11 + nu * np.eye(k) + (K11 @ K11 + K12 @ K12.T) / mu
    return r / mu - (A.T @ np.linalg.solve(inner, A @ r)) / (mu * mu)


def build_ran(X: np.ndarray, l: float, mu: float, k: int, kernel: str = "gaussian",
              landmarks: str = "uniform", fps_seed: int = 0, rng_seed: int = 0,
              nu: float = NYS_NU):
    """RAN comparison preconditioner: rank-k Nystrom approximation
    on randomly sampled landmarks, K_nys = U Lam U^T its eigendecomposition,
    lam_k the k-th largest eigenvalue.  K_nys as in build_nystrom (R30); its
    eigenpairs from the thin SVD of F = K_{X,Xk} L^{-T}, L L^T = K11 + nu I
    (K_nys = F F^T)."""
    N = build_nystrom(X, l, mu, k, fps_seed, kernel, landmarks, rng_seed, nu)
    k = N["k"]
    C = np.vstack([N["K11"], N["K12"].T])  # K_{X, Xk} in the permuted order
    L = np.linalg.cholesky(N["K11"] + nu * np.eye(k))
    F = sla.solve_triangular(L, C.T, lower=True).T
    U, sig, _ = np.linalg.svd(F, full_matrices=False)
    lam = sig * sig
    N.update(method="ran", U=U, lam=lam, lam_k=float(lam.min()))
    return N


def apply_ran(R: dict, r: np.ndarray) -> np.ndarray:
    """(lam_k + mu) U (Lam + mu I)^{-1} U^T r + (I - U U^T) r."""
    U, lam, lam_k, mu = R["U"], R["lam"], R["lam_k"], R["mu"]
    r = np.asarray(r, dtype=np.float64)
    Ur = U.T @ r
    return (lam_k + mu) * (U @ (Ur / (lam + mu))) + r - U @ Ur


def choose_method(khat: int, k_threshold: int = 2000) -> str:
    """Algorithm 2: AFN if the estimated rank is >= 2000, else Nystrom."""
    return "afn" if khat >= k_threshold else "nystrom"


def build_precond(X, l, mu, k, w, method="afn", kernel="gaussian", landmarks="fps",
                  fps_seed=0, rng_seed=0, ordering="index"):
    """AFN (eq:factorized-form), Nystrom or plain FSAI (k = 0)."""
    if method == "nystrom":
        return build_nystrom(X, l, mu, k, fps_seed, kernel, landmarks, rng_seed)
    if method == "ran":
        return build_ran(X, l, mu, k, kernel, landmarks, fps_seed, rng_seed)
    if method == "fsai":
        return build_afn(X, l, mu, 0, w, fps_seed, kernel, landmarks, rng_seed, ordering)
    return build_afn(X, l, mu, k, w, fps_seed, kernel, landmarks, rng_seed, ordering)


def apply_precond(B: dict, r: np.ndarray) -> np.ndarray:
    if B.get("method") == "nystrom":
        return apply_nystrom(B, r)
    if B.get("method") == "ran":
        return apply_ran(B, r)
    return apply_afn(B, r)


def dense_B(B: dict) -> np.ndarray:
    """Dense lower factor of eq:factorized-form, M = B B^T:
       B = [[L, 0], [K12^T L^{-T}, G^{-1}]]  (test helper, small n only)."""
    k, n = B["k"], B["n"]
    out = np.zeros((n, n))
    out[:k, :k] = B["L"]
    if n > k:
        out[k:, :k] = B["V"].T
        out[k:, k:] = np.linalg.inv(B["G"].toarray())
    return out


# ----------------------------------------------------------------------------
# (P)CG
# ----------------------------------------------------------------------------
def pcg(Amv, Minv, b, tol: float = 1e-4, maxit: int = 500, fixed_iters: int = 0,
        x_true=None):
    """Preconditioned CG from x0 = 0 with the recurrence residual test
    ||r||/||b|| <= tol (R19); maxit 500, non-convergence not an error
    (R20).  The iteration count is the number of A p products.
    ``fixed_iters`` > 0 runs exactly that many iterations (parity runs)."""
    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    x = np.zeros(n)
    nb = float(np.linalg.norm(b))
    rep = dict(iterations=0, converged=True, history=[1.0 if nb > 0 else 0.0], breakdown=False)
    if nb == 0.0:
        return x, rep
    r = b.copy()
    z = Minv(r)
    p = z.copy()
    rz = float(r @ z)
    converged = False
    it = 0
    for it in range(1, maxit + 1):
        q = Amv(p)
        pq = float(p @ q)
        if not (pq > 0.0):
            rep["breakdown"] = True
            it -= 1
            break
        alpha = rz / pq
        x = x + alpha * p
        r = r - alpha * q
        rel = float(np.linalg.norm(r)) / nb
        rep["history"].append(rel)
        if fixed_iters:
            if it >= fixed_iters:
                converged = rel <= tol
                break
        elif rel <= tol:
            converged = True
            break
        z = Minv(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    rep["iterations"] = it
    rep["converged"] = converged
    return x, rep


def afn_pcg_solve(X, b, l, mu, k, w, tol=1e-4, maxit=500, fixed_iters=0, fps_seed=0,
                  B=None, threads=None, method="afn", kernel="gaussian", landmarks="fps",
                  rng_seed=0):
    """Full path: build the preconditioner (unless ``B`` given), PCG on the
    permuted system, un-permute.  Returns (a, report, B)."""
    X = np.asarray(X, dtype=np.float64)
    if B is None:
        B = build_precond(X, l, mu, k, w, method, kernel, landmarks, fps_seed, rng_seed)
    kernel = B.get("kernel", kernel)
    perm = B["perm"]
    Xp = B["Xp"]
    bp = np.asarray(b, dtype=np.float64)[perm]
    x, rep = pcg(lambda v: kmv(Xp, l, mu, v, threads=threads, kernel=kernel),
                 lambda r: apply_precond(B, r), bp, tol, maxit, fixed_iters)
    a = np.empty_like(x)
    a[perm] = x
    nb = float(np.linalg.norm(b))
    res = b - kmv(X, l, mu, a, threads=threads, kernel=kernel)
    rep["relres_true"] = float(np.linalg.norm(res)) / nb if nb > 0 else 0.0
    return a, rep, B


def cg_solve(X, b, l, mu, tol=1e-4, maxit=500, fixed_iters=0, threads=None):
    """Unpreconditioned CG on (K + mu I) a = b."""
    X = np.asarray(X, dtype=np.float64)
    return pcg(lambda v: kmv(X, l, mu, v, threads=threads), lambda r: r.copy(), b, tol,
               maxit, fixed_iters)


def _threads_default() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1

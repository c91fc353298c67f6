"""paper_2304_05460_b200 -- B200-native AFN-preconditioned CG (arXiv 2304.05460).

Thin ctypes binding over the C ABI in ``include/afn.h`` (``libafn.so``, built
for sm_100a by ``paper_2304_05460_b200.build``).  This module only marshals
arguments: every step of the hot path runs in the library's CUDA kernels.
There is no CPU fallback -- importing fails loudly if the library is missing.

Device arrays are ``torch.Tensor`` objects (float64, contiguous, on a CUDA
device); PyTorch supplies memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libafn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -m paper_2304_05460_b200.build` "
        "(no CPU fallback exists)")

_lib = C.CDLL(LIB_PATH)

AFN_OK = 0
STATUS = {0: "AFN_OK", 1: "AFN_ERR_ARG", 2: "AFN_ERR_CUDA", 3: "AFN_ERR_NOMEM",
          4: "AFN_ERR_NOT_SPD", 5: "AFN_ERR_BREAKDOWN", 6: "AFN_ERR_NCCL", 7: "AFN_ERR_STATE"}
COMM_ID_BYTES = 128
KERNEL_GAUSSIAN, KERNEL_MATERN32 = 0, 1
LANDMARKS_FPS, LANDMARKS_UNIFORM = 0, 1
METHOD_AFN, METHOD_ALG2, METHOD_NYSTROM, METHOD_FSAI, METHOD_RAN, METHOD_NONE = 0, 1, 2, 3, 4, 5
W_MAX = 512  # include/afn.h AFN_W_MAX
ORDER_INDEX, ORDER_MAXMIN = 0, 1
_KERNELS = {"gaussian": KERNEL_GAUSSIAN, "matern32": KERNEL_MATERN32}


def _kernel_id(kernel):
    return _KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
OUT_PERM, OUT_FILL, OUT_L, OUT_ROWPTR, OUT_COL, OUT_GVAL, OUT_W = range(7)


class AfnError(RuntimeError):
    def __init__(self, status, where):
        msg = _lib.afn_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [("l", C.c_double), ("mu", C.c_double), ("k_cap", C.c_int64),
                ("k_adaptive", C.c_int32), ("w", C.c_int32), ("m", C.c_int32),
                ("k_threshold", C.c_int32), ("fps_seed", C.c_int64), ("rng_seed", C.c_uint64),
                ("kernel", C.c_int32), ("landmarks", C.c_int32), ("method", C.c_int32),
                ("ordering", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("khat", C.c_int64), ("nnz", C.c_int64),
                ("d", C.c_int32), ("r", C.c_int32), ("m", C.c_int32), ("refined", C.c_int32),
                ("scale", C.c_double), ("ms_alg1", C.c_double), ("ms_fps", C.c_double),
                ("ms_chol", C.c_double), ("ms_trsm", C.c_double), ("ms_knn", C.c_double),
                ("ms_fsai", C.c_double), ("ms_total", C.c_double), ("ms_fsai_rows", C.c_double),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("row_a0", C.c_int64),
                ("row_na", C.c_int64), ("row_b0", C.c_int64), ("row_nb", C.c_int64),
                ("kernel", C.c_int32), ("method", C.c_int32),
                ("kmv_plan", C.c_int32), ("kmv_reserved", C.c_int32),
                ("kmv_units64", C.c_int64), ("kmv_units32", C.c_int64),
                ("kmv_pairs64", C.c_double), ("kmv_pairs32", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("applies", C.c_int32), ("relres", C.c_double), ("relres_true", C.c_double),
                ("solve_ms", C.c_double), ("matvec_ms", C.c_double), ("apply_ms", C.c_double),
                ("comm_ms", C.c_double), ("history", C.POINTER(C.c_double))]

    def as_dict(self):
        return dict(iterations=self.iterations, converged=bool(self.converged),
                    breakdown=bool(self.breakdown), applies=self.applies, relres=self.relres,
                    relres_true=self.relres_true, solve_ms=self.solve_ms,
                    matvec_ms=self.matvec_ms, apply_ms=self.apply_ms, comm_ms=self.comm_ms)


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_sig = {
    "kernel_matvec": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_double, _P, _P,
                                _P]),
    "kernel_matvec_rows": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_double, _P,
                                     C.c_int64, C.c_int64, _P, _P]),
    "afn_fps": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int64, C.c_int64, _P, _P, _P]),
    "afn_knn_pattern": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]),
    "afn_w_product": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, C.c_double, _P, C.c_int32,
                                _P, _P]),
    "afn_estimate_rank": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                    C.c_uint64,
                                    C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), _P]),
    "afn_build": (C.c_int, [_P, C.c_int64, C.c_int32, C.POINTER(Params), _P, C.POINTER(_P)]),
    "afn_apply": (C.c_int, [_P, _P, _P, _P]),
    "afn_matvec": (C.c_int, [_P, _P, _P, _P]),
    "afn_pcg_solve": (C.c_int, [_P, _P, _P, C.c_double, C.c_int32, C.c_int32, C.POINTER(Report), _P]),
    "afn_cg_solve": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_double, _P, _P,
                               C.c_double, C.c_int32, C.c_int32, C.POINTER(Report), _P]),
    "afn_set_allocator": (C.c_int, [_P, _P, _P]),
    "afn_pool_stats": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "afn_comm_set_timeout": (C.c_int, [_P, C.c_double]),
    "afn_solve_host": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int32, C.POINTER(Params), C.c_double,
                                 C.c_int32, C.POINTER(Info), C.POINTER(Report), _P]),
    "afn_get_info": (C.c_int, [_P, C.POINTER(Info)]),
    "afn_copy_out": (C.c_int, [_P, C.c_int32, _P, C.c_size_t]),
    "afn_copy_out_rows": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, C.c_size_t]),
    "afn_copy_out_local": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_size_t]),
    "afn_comm_unique_id": (C.c_int, [_P, C.c_char_p]),
    "afn_comm_init": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(_P)]),
    "afn_comm_init_emulated": (C.c_int, [C.c_int32, C.POINTER(_P)]),
    "afn_comm_destroy": (None, [_P]),
    "afn_shard_rows": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "afn_build_dist": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.POINTER(Params), _P, C.POINTER(_P)]),
    "afn_destroy": (None, [_P]),
    "afn_probe_dfma": (C.c_int, [C.c_int64, _D, _P]),
    "afn_probe_dmma": (C.c_int, [C.c_int64, _D, _P]),
    "afn_probe_ex2": (C.c_int, [C.c_int64, _D, _P]),
    "afn_set_cutoff_mode": (C.c_int, [C.c_int32]),
    "afn_launch_count": (C.c_int64, []),
    "afn_kt_enable": (None, [C.c_int32]),
    "afn_kt_reset": (None, []),
    "afn_kt_read": (C.c_int32, [_D, _D, C.POINTER(C.c_int64), C.c_int32]),
    "afn_last_error": (C.c_char_p, []),
    "afn_abi_version": (C.c_int32, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


def _check(status, where):
    if status != AFN_OK:
        raise AfnError(status, where)


def _torch():
    import torch
    return torch


def _dev(t, name, dtype=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


KT_NAMES = ("kmv_kernel", "group_gemm_kernel", "fsai_assemble_kernel", "fsai_chol_kernel",
            "fsai_gram_kernel", "fps_kernel", "w_gemm_kernel", "trsm_rows_kernel<1>",
            "potrf", "knn_kernel", "apply", "alg1")


def kernel_timers(enable=None, reset=False):
    """Per-kernel-class device ms / algorithmic work / launch counts (include/afn.h)."""
    if reset:
        _lib.afn_kt_reset()
    if enable is not None:
        _lib.afn_kt_enable(1 if enable else 0)
    n = 16
    ms = (C.c_double * n)()
    wk = (C.c_double * n)()
    ct = (C.c_int64 * n)()
    m = _lib.afn_kt_read(ms, wk, ct, n)
    return {KT_NAMES[i]: dict(ms=ms[i], work=wk[i], count=ct[i]) for i in range(min(m, len(KT_NAMES)))}


def launch_count() -> int:
    return int(_lib.afn_launch_count())


def abi_version() -> int:
    return int(_lib.afn_abi_version())


# ---------------------------------------------------------------------------
def kernel_matvec(X, l, mu, v, y=None, stream=None, kernel="gaussian"):
    """y = (K + mu I) v on the device (include/afn.h kernel_matvec)."""
    torch = _torch()
    n, d = X.shape
    if y is None:
        y = torch.empty_like(v)
    _check(_lib.kernel_matvec(_dev(X, "X", torch.float64), n, d, _kernel_id(kernel), float(l), float(mu),
                              _dev(v, "v", torch.float64), _dev(y, "y", torch.float64),
                              _stream(stream)), "kernel_matvec")
    return y


def kernel_matvec_rows(X, l, mu, v, row0, nrows, y=None, stream=None, kernel="gaussian"):
    torch = _torch()
    n, d = X.shape
    if y is None:
        y = torch.empty(nrows, dtype=torch.float64, device=v.device)
    _check(_lib.kernel_matvec_rows(_dev(X, "X", torch.float64), n, d, _kernel_id(kernel), float(l),
                                   float(mu),
                                   _dev(v, "v", torch.float64), int(row0), int(nrows),
                                   _dev(y, "y", torch.float64), _stream(stream)),
           "kernel_matvec_rows")
    return y


def afn_fps(X, k, seed=0, stream=None):
    """Farthest point sampling -> (idx int64[k], fill float64[k]) device tensors."""
    torch = _torch()
    n, d = X.shape
    idx = torch.empty(k, dtype=torch.int64, device=X.device)
    fill = torch.empty(k, dtype=torch.float64, device=X.device)
    _check(_lib.afn_fps(_dev(X, "X", torch.float64), n, d, int(k), int(seed), _dev(idx, "idx"),
                        _dev(fill, "fill"), _stream(stream)), "afn_fps")
    return idx, fill


def knn_nnz(N, w):
    return N * (N + 1) // 2 if N < w else w * (w + 1) // 2 + (N - w) * w


def afn_knn_pattern(P, w, stream=None):
    """kNN lower pattern -> (row_ptr int64[N+1], col int32[nnz]) device tensors."""
    torch = _torch()
    N, d = P.shape
    rp = torch.empty(N + 1, dtype=torch.int64, device=P.device)
    col = torch.empty(max(1, knn_nnz(N, w)), dtype=torch.int32, device=P.device)
    _check(_lib.afn_knn_pattern(_dev(P, "P", torch.float64), N, d, int(w), _dev(rp, "row_ptr"),
                                _dev(col, "col"), _stream(stream)), "afn_knn_pattern")
    return rp, col[:knn_nnz(N, w)]


WPROD_DMMA, WPROD_INT8, WPROD_CUT = 0, 1, 2


def afn_w_product(X1, Xr, l, Linv, method=WPROD_INT8, stream=None, kernel="gaussian"):
    """W = K(Xr, X1) L^{-T} from Linv = L^{-1} (include/afn.h afn_w_product)."""
    torch = _torch()
    k, d = X1.shape
    N = Xr.shape[0]
    W = torch.empty(N, k, dtype=torch.float64, device=Xr.device)
    _check(_lib.afn_w_product(_dev(X1, "X1", torch.float64), k, _dev(Xr, "Xr", torch.float64), N, d,
                              _kernel_id(kernel), float(l), _dev(Linv, "Linv", torch.float64), int(method),
                              _dev(W, "W", torch.float64), _stream(stream)), "afn_w_product")
    return W


def afn_estimate_rank(X, l, m=0, rng_seed=0, k_threshold=2000, stream=None, kernel="gaussian"):
    torch = _torch()
    n, d = X.shape
    kh, r, ref = C.c_int64(), C.c_int32(), C.c_int32()
    _check(_lib.afn_estimate_rank(_dev(X, "X", torch.float64), n, d, _kernel_id(kernel), float(l), int(m),
                                  int(rng_seed), int(k_threshold), C.byref(kh), C.byref(r),
                                  C.byref(ref), _stream(stream)), "afn_estimate_rank")
    return dict(khat=kh.value, r=r.value, refined=bool(ref.value))


def make_params(l, mu, k_cap, w, k_adaptive=False, m=0, k_threshold=2000, fps_seed=0, rng_seed=0,
                kernel="gaussian", landmarks=LANDMARKS_FPS, method=METHOD_AFN, ordering=ORDER_INDEX):
    return Params(float(l), float(mu), int(k_cap), int(bool(k_adaptive)), int(w), int(m),
                  int(k_threshold), int(fps_seed), int(rng_seed), _kernel_id(kernel), int(landmarks),
                  int(method), int(ordering))


def nccl_library_path():
    """libnccl.so.2 of the nvidia-nccl wheel (the copy PyTorch loads), or None."""
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return None


def shard_rows(n, k, nranks, rank):
    """Rows (a0, na, b0, nb) of the permuted order owned by `rank` (include/afn.h)."""
    out = (C.c_int64 * 4)()
    _check(_lib.afn_shard_rows(int(n), int(k), int(nranks), int(rank), out), "afn_shard_rows")
    return tuple(out)


def nccl_unique_id(nccl_path=None) -> bytes:
    buf = C.create_string_buffer(COMM_ID_BYTES)
    path = nccl_path or nccl_library_path()
    _check(_lib.afn_comm_unique_id(buf, path.encode() if path else None), "afn_comm_unique_id")
    return buf.raw


def bootstrap_unique_id(dist=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast over an initialised torch.distributed group."""
    if dist is None:
        import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]


class Comm:
    """Communicator of the row-sharded path (include/afn.h afn_comm)."""

    def __init__(self, ptr, nranks, rank, nlocal):
        self._c = ptr
        self.nranks, self.rank, self.nlocal = nranks, rank, nlocal

    @classmethod
    def nccl(cls, unique_id: bytes, nranks: int, rank: int, nccl_path=None):
        """One process per GPU; every rank passes rank 0's nccl_unique_id()."""
        c = C.c_void_p()
        path = nccl_path or nccl_library_path()
        _check(_lib.afn_comm_init(C.c_char_p(unique_id), int(nranks), int(rank),
                                  path.encode() if path else None, C.byref(c)), "afn_comm_init")
        return cls(c, nranks, rank, 1)

    @classmethod
    def from_process_group(cls, dist=None):
        """Bootstrap from an initialised torch.distributed group (rank 0's id is broadcast)."""
        if dist is None:
            import torch.distributed as dist
        uid = bootstrap_unique_id(dist)
        return cls.nccl(uid, dist.get_world_size(), dist.get_rank())

    @classmethod
    def emulated(cls, nranks: int):
        """nranks logical ranks driven by this process on the current device (tests)."""
        c = C.c_void_p()
        _check(_lib.afn_comm_init_emulated(int(nranks), C.byref(c)), "afn_comm_init_emulated")
        return cls(c, nranks, 0, nranks)

    def set_timeout(self, seconds):
        _check(_lib.afn_comm_set_timeout(self._c, float(seconds)), "afn_comm_set_timeout")

    def close(self):
        if getattr(self, "_c", None) is not None and self._c.value:
            _lib.afn_comm_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Handle:
    """A built AFN preconditioner (include/afn.h afn_handle); `comm` shards it."""

    def __init__(self, X, params: Params, stream=None, comm: Comm = None):
        torch = _torch()
        self.n, self.d = X.shape
        self.device = X.device
        self.comm = comm  # keeps the communicator alive while the handle is
        h = C.c_void_p()
        _check(_lib.afn_build_dist(comm._c if comm is not None else None,
                                   _dev(X, "X", torch.float64), self.n, self.d, C.byref(params),
                                   _stream(stream), C.byref(h)), "afn_build_dist")
        self._h = h
        self.params = params

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.afn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        inf = Info()
        _check(_lib.afn_get_info(self._h, C.byref(inf)), "afn_get_info")
        return inf.as_dict()

    def matvec(self, v, y=None, stream=None):
        """y = (K + mu I) v through the handle's (possibly rank-sharded) plan."""
        torch = _torch()
        if y is None:
            y = torch.empty_like(v)
        _check(_lib.afn_matvec(self._h, _dev(v, "v", torch.float64), _dev(y, "y", torch.float64),
                               _stream(stream)), "afn_matvec")
        return y

    def apply(self, r, z=None, stream=None):
        torch = _torch()
        if z is None:
            z = torch.empty_like(r)
        _check(_lib.afn_apply(self._h, _dev(r, "r", torch.float64), _dev(z, "z", torch.float64),
                              _stream(stream)), "afn_apply")
        return z

    def pcg_solve(self, b, a=None, tol=1e-4, maxit=500, fixed_iters=0, history=False, stream=None):
        torch = _torch()
        import numpy as np
        if a is None:
            a = torch.empty_like(b)
        rep = Report()
        hist = None
        if history:
            hist = np.zeros(maxit + 1)
            rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        _check(_lib.afn_pcg_solve(self._h, _dev(b, "b", torch.float64), _dev(a, "a", torch.float64),
                                  float(tol), int(maxit), int(fixed_iters), C.byref(rep),
                                  _stream(stream)), "afn_pcg_solve")
        out = rep.as_dict()
        if hist is not None:
            out["history"] = hist[: rep.iterations + 1].copy()
        return a, out

    def copy_out(self, what, local_rank=0):
        import numpy as np
        inf = self.info()
        n, k, nnz = inf["n"], inf["k"], inf["nnz"]
        nw = n - k
        if inf["nranks"] > 1:
            nw = shard_rows(n, k, inf["nranks"], inf["rank"] + local_rank)[3]
        shapes = {OUT_PERM: (np.int64, (n,)), OUT_FILL: (np.float64, (k,)),
                  OUT_L: (np.float64, (k, k)), OUT_ROWPTR: (np.int64, (n - k + 1,)),
                  OUT_COL: (np.int32, (nnz,)), OUT_GVAL: (np.float64, (nnz,)),
                  OUT_W: (np.float64, (nw, k))}
        dt, shp = shapes[what]
        arr = np.empty(shp, dtype=dt)
        _check(_lib.afn_copy_out_local(self._h, int(local_rank), int(what),
                                       arr.ctypes.data_as(C.c_void_p), arr.nbytes),
               "afn_copy_out_local")
        return arr

    def copy_out_rows(self, what, rows):
        """Rows of W (non-landmark positions) or L as a (len(rows), k) host array."""
        import numpy as np
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        k = self.info()["k"]
        arr = np.empty((len(rows), k))
        _check(_lib.afn_copy_out_rows(self._h, int(what), rows.ctypes.data_as(C.c_void_p),
                                      len(rows), arr.ctypes.data_as(C.c_void_p), arr.nbytes),
               "afn_copy_out_rows")
        return arr


def afn_build(X, params: Params, stream=None, comm: Comm = None) -> Handle:
    return Handle(X, params, stream, comm)


def afn_cg_solve(X, b, l, mu, tol=1e-4, maxit=500, fixed_iters=0, a=None, kernel="gaussian",
                 comm: Comm = None, history=False, stream=None):
    """Unpreconditioned CG on (K + mu I) a = b (include/afn.h afn_cg_solve)."""
    torch = _torch()
    import numpy as np
    n, d = X.shape
    if a is None:
        a = torch.empty_like(b)
    rep = Report()
    hist = None
    if history:
        hist = np.zeros(maxit + 1)
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
    _check(_lib.afn_cg_solve(comm._c if comm is not None else None, _dev(X, "X", torch.float64), n, d,
                             _kernel_id(kernel), float(l), float(mu), _dev(b, "b", torch.float64),
                             _dev(a, "a", torch.float64), float(tol), int(maxit), int(fixed_iters),
                             C.byref(rep), _stream(stream)), "afn_cg_solve")
    out = rep.as_dict()
    if hist is not None:
        out["history"] = hist[: rep.iterations + 1].copy()
    return a, out


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_allocator_refs = None  # keeps the ctypes callbacks alive while installed


def use_torch_allocator(enable=True):
    """Route the library's device allocations through PyTorch's caching
    allocator (include/afn.h afn_set_allocator); enable=False restores the
    library's own stream-ordered pool.  Marshalling only."""
    global _allocator_refs
    torch = _torch()
    if not enable:
        _check(_lib.afn_set_allocator(None, None, None), "afn_set_allocator")
        _allocator_refs = None
        return

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0))
        except Exception:
            return None

    def _free(ptr, nbytes, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    refs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _check(_lib.afn_set_allocator(C.cast(refs[0], C.c_void_p), C.cast(refs[1], C.c_void_p), None),
           "afn_set_allocator")
    _allocator_refs = refs


def pool_stats():
    """(reserved, used) bytes of the library's default device pool."""
    r, u = C.c_int64(), C.c_int64()
    _check(_lib.afn_pool_stats(C.byref(r), C.byref(u)), "afn_pool_stats")
    return r.value, u.value


def afn_solve_host(X, b, params: Params, tol=1e-4, maxit=500, stream=None, comm: Comm = None):
    """End-to-end solve with HOST numpy arrays (copies inside the C call)."""
    import numpy as np
    X = np.ascontiguousarray(X, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n, d = X.shape
    a = np.empty(n)
    inf, rep = Info(), Report()
    _check(_lib.afn_solve_host(comm._c if comm is not None else None,
                               X.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                               a.ctypes.data_as(C.c_void_p), n, d, C.byref(params), float(tol),
                               int(maxit), C.byref(inf), C.byref(rep), _stream(stream)),
           "afn_solve_host")
    return a, inf.as_dict(), rep.as_dict()


def probe_dmma(iters=1 << 14, stream=None) -> float:
    out = C.c_double()
    _check(_lib.afn_probe_dmma(int(iters), C.byref(out), _stream(stream)), "afn_probe_dmma")
    return out.value


def probe_ex2(iters=1 << 16, stream=None) -> float:
    """MUFU.EX2 G ops/s (afn_probe_ex2)."""
    out = C.c_double()
    _check(_lib.afn_probe_ex2(int(iters), C.byref(out), _stream(stream)), "afn_probe_ex2")
    return out.value


def set_cutoff_mode(mode: int) -> None:
    """Cutoff matvec plan and W product: 0 auto (when they pay), 1 never,
    2 whenever they apply (afn_set_cutoff_mode)."""
    _check(_lib.afn_set_cutoff_mode(int(mode)), "afn_set_cutoff_mode")


def probe_dfma(iters=1 << 16, stream=None) -> float:
    out = C.c_double()
    _check(_lib.afn_probe_dfma(int(iters), C.byref(out), _stream(stream)), "afn_probe_dfma")
    return out.value

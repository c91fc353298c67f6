/*
 * afn.h -- C ABI of the B200-native AFN-preconditioned CG hot path
 * (Adaptive Factorized Nystrom, arXiv 2304.05460).
 *
 * Problem (eq:Problem / eq:gaussianf):
 *     (K + mu I) a = b,   K_ij = exp(-||x_i - x_j||^2 / l^2)     (no factor 1/2)
 * for n points x_i in R^d.  K is never formed.
 *
 * Conventions for every entry point
 *   - fp64 everywhere.  X is n x d row-major (x_i = X[i*d .. i*d+d-1]).
 *   - Array pointers are DEVICE pointers on the current CUDA device unless the
 *     argument is marked [host].  The caller owns every array it passes; the
 *     library never frees caller memory.  `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).
 *   - Entry points are stream-ordered unless marked [sync]; [sync] entry points
 *     synchronise `stream` before returning because they return host values.
 *   - Errors: every call returns an afn_status; nothing throws or exits across
 *     the ABI.  afn_last_error() returns a thread-local description of the last
 *     failure.  Arguments are validated first (sizes, ranges, and that array
 *     pointers are device-accessible): violations return AFN_ERR_ARG and touch
 *     nothing.
 *   - Results are deterministic: no floating-point atomics; every reduction has
 *     a fixed order that does not depend on timing.
 *   - Integer outputs (landmark ids, kNN pattern, Alg. 1 rank) follow the
 *     readings R3/R7-R15 of DESIGN.md: squared distances are sums over the
 *     coordinates c = 0..d-1 in order of individually rounded (x_c - y_c)^2
 *     (no FMA contraction), ties go to the lowest index.
 */
#ifndef AFN_H_
#define AFN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFN_ABI_VERSION 6
/* widest FSAI row (nonzeros incl. the diagonal): the paper's plain-FSAI
 * comparison uses 400 neighbours */
#define AFN_W_MAX 512

typedef enum {
  AFN_OK = 0,
  AFN_ERR_ARG = 1,        /* invalid argument; nothing was modified            */
  AFN_ERR_CUDA = 2,       /* CUDA runtime / launch failure                     */
  AFN_ERR_NOMEM = 3,      /* device allocation failed                          */
  AFN_ERR_NOT_SPD = 4,    /* Cholesky breakdown of K11+mu I or an FSAI block  */
  AFN_ERR_BREAKDOWN = 5,  /* PCG breakdown (p.q <= 0 or non-finite)            */
  AFN_ERR_NCCL = 6,       /* NCCL unavailable or a collective failed           */
  AFN_ERR_STATE = 7       /* handle used in a state that does not allow it     */
} afn_status;

/* Opaque built preconditioner (immutable after afn_build). */
typedef struct afn_handle_s* afn_handle;
/* Opaque communicator of the row-sharded multi-GPU path (afn_comm_*). */
typedef struct afn_comm_s* afn_comm;

/* Kernel functions, r = ||x - y||:
 *   AFN_KERNEL_GAUSSIAN  exp(-r^2 / l^2)          (eq:gaussianf)
 *   AFN_KERNEL_MATERN32  (1 + sqrt(3) r / l) exp(-sqrt(3) r / l)            */
enum { AFN_KERNEL_GAUSSIAN = 0, AFN_KERNEL_MATERN32 = 1 };
/* Landmark selection: farthest point sampling or uniform
 * random sampling, the paper's choice for its high-dimensional datasets
 * (P:L957): the k points with the smallest splitmix64 keys of
 * (rng_seed ^ 0x6A09E667F3BCC909) ^ i*golden, in key order (reading R29). */
enum { AFN_LANDMARKS_FPS = 0, AFN_LANDMARKS_UNIFORM = 1 };
/* Preconditioner (Algorithm 2):
 *   AFN_METHOD_AFN      AFN (eq:factorized-form) with k landmarks
 *   AFN_METHOD_ALG2     Algorithm 2: AFN if Alg. 1's khat >= k_threshold,
 *                       else the Nystrom preconditioner with khat landmarks
 *                       (needs k_adaptive = 1)
 *   AFN_METHOD_NYSTROM  Nystrom preconditioner K_nys + mu I
 *                       applied exactly through an equivalent stable SMW form
 *   AFN_METHOD_FSAI     plain FSAI of K + mu I on the kNN pattern of all
 *                       points in the original order (k = 0)
 *   AFN_METHOD_RAN      the paper's RAN comparison preconditioner:
 *                       (lam_k + mu) U (Lam + mu I)^{-1} U^T + (I - U U^T) for
 *                       K_nys = U Lam U^T on k landmarks (use uniform ones)
 *   AFN_METHOD_NONE     M = I: plain CG, the paper's unpreconditioned
 *                       baseline (Table 5.1a CG rows)  */
enum { AFN_METHOD_AFN = 0, AFN_METHOD_ALG2 = 1, AFN_METHOD_NYSTROM = 2, AFN_METHOD_FSAI = 3,
       AFN_METHOD_RAN = 4, AFN_METHOD_NONE = 5 };
/* Order of the non-landmark points, which fixes "numbered less than i" of the
 * FSAI pattern: ascending original index (reading R14) or the
 * MaxMin order, i.e. FPS continued through all n points ("MaxMin
 * Ordering"; needs FPS landmarks).                                          */
enum { AFN_ORDER_INDEX = 0, AFN_ORDER_MAXMIN = 1 };

/* Build parameters.  Cite: l, mu; k_cap "limit ... such as 2000"
 * (P:L209-210); w "the w-1 nearest neighbors" (w counts the
 * diagonal, reading R15); m, rng_seed, k_threshold: Algorithm 1 (P:L661-678,
 * readings R6-R13); fps_seed: "an arbitrary point" (reading R2). */
typedef struct {
  double l;             /* length-scale, > 0                                   */
  double mu;            /* regularisation, > 0                                 */
  int64_t k_cap;        /* landmark cap, >= 1                                  */
  int32_t k_adaptive;   /* 1: k = min(k_cap, max(1, Alg.1 khat)); 0: k = k_cap */
  int32_t w;            /* FSAI nonzeros per row incl. diagonal, 1..AFN_W_MAX  */
  int32_t m;            /* Alg. 1 subsample size; 0 = min(500,max(100,n/100))  */
  int32_t k_threshold;  /* Alg. 1 branch threshold (paper: 2000)               */
  int64_t fps_seed;     /* first FPS point, 0 <= fps_seed < n                  */
  uint64_t rng_seed;    /* Alg. 1 subsample seed (splitmix64 counter, R7)      */
  int32_t kernel;       /* AFN_KERNEL_*                                        */
  int32_t landmarks;    /* AFN_LANDMARKS_*                                     */
  int32_t method;       /* AFN_METHOD_*                                        */
  int32_t ordering;     /* AFN_ORDER_*: order of the non-landmark points         */
} afn_params;

/* Information about a built handle (host struct). */
typedef struct {
  int64_t n, k, khat, nnz;      /* points, landmarks used, Alg.1 estimate, nnz(G) */
  int32_t d, r, m, refined;     /* dims; Alg.1 rank r on the subsample, m, branch  */
  double scale;                 /* Alg.1 coordinate scale (m/n)^(1/d)              */
  double ms_alg1, ms_fps, ms_chol, ms_trsm, ms_knn, ms_fsai, ms_total; /* phase times */
  double ms_fsai_rows;          /* the FSAI row kernel alone (inside ms_fsai)      */
  int32_t nranks, rank;         /* communicator size, this (first local) rank      */
  int64_t row_a0, row_na, row_b0, row_nb; /* rows of the permuted order it owns   */
  int32_t kernel, method;       /* kernel, preconditioner built (AFN_METHOD_AFN,   */
                                /* _NYSTROM or _FSAI)                              */
  /* the handle's kernel-matvec plan (afn_set_cutoff_mode):      */
  /* 0 row-wise, 1 dense symmetric, 2 cutoff; work units of the FP64 and FP32   */
  /* bodies and the unordered pairs they evaluate per product (one rank's plan  */
  /* covers all ranks' units)                                                    */
  int32_t kmv_plan, kmv_reserved;
  int64_t kmv_units64, kmv_units32;
  double kmv_pairs64, kmv_pairs32;
} afn_info;

/* PCG report (host struct).  history: optional host array of >= maxit+1
 * doubles receiving ||r_i||/||b|| (entry 0 = 1). */
typedef struct {
  int32_t iterations;   /* number of (K+mu I)p products in the loop            */
  int32_t converged;    /* 1 if ||r||/||b|| <= tol was reached                 */
  int32_t breakdown;    /* 1 if p.q <= 0 or a non-finite scalar stopped it     */
  int32_t applies;      /* number of M^{-1} applications                       */
  double relres;        /* recurrence residual at exit                         */
  double relres_true;   /* ||b - (K+mu I)a|| / ||b|| (one extra matvec)        */
  double solve_ms;      /* device time of the solve loop (CUDA events)         */
  double matvec_ms;     /* device time of the loop's kernel matvecs            */
  double apply_ms;      /* device time of the loop's AFN applications          */
  double comm_ms;       /* device time of the loop's exchanges (multi-rank)    */
  double* history;      /* [host, optional] len maxit+1                        */
} afn_solve_report;

/* ------------------------------------------------------------------------ */
/* Kernel matvec  y = (K + mu I) v   */
/* X: n x d device, v,y: n device (y must not alias v or X).  Stream-ordered. */
/* K is symmetric: for 2048 <= n and d <= 8 each unordered pair is evaluated */
/* once (row and column sums, fixed summation order); otherwise rows use a    */
/* fixed column-chunk order.  Either way the output is bit-identical run to   */
/* run (it may differ from kernel_matvec_rows at rounding level).             */
/* n >= 1, 1 <= d <= 16, l > 0, mu >= 0.                                      */
afn_status kernel_matvec(const double* X, int64_t n, int32_t d, int32_t kernel, double l, double mu,
                         const double* v, double* y, void* stream);

/* Rows [row0, row0+nrows) of y = (K + mu I) v against all n columns (the row
 * shard a rank owns in the multi-GPU layout).  y has nrows entries.  Always
 * the row-wise (non-symmetric) kernel: a row's value does not depend on which
 * shard it is evaluated in (shards of >= two waves are bit-identical). */
afn_status kernel_matvec_rows(const double* X, int64_t n, int32_t d, int32_t kernel, double l, double mu,
                              const double* v, int64_t row0, int64_t nrows, double* y,
                              void* stream);

/* ------------------------------------------------------------------------ */
/* Farthest point sampling (eq.(3.3); brute force) [sync] */
/* idx: k int64 device (original ids, selection order); fill: k doubles      */
/* device (fill[i] = fill distance after i+1 selections) or NULL.     */
afn_status afn_fps(const double* X, int64_t n, int32_t d, int64_t k, int64_t seed,
                   int64_t* idx, double* fill, void* stream);

/* W = K(Xr, X1) L^{-T} (the Nystrom factor V^T = K21 L^{-T}; a5) for  */
/* N points Xr (N x d) against k landmarks X1 (k x d), Linv = L^{-1} (k x k   */
/* row-major, lower triangular), W: N x k row-major, all device, stream-      */
/* ordered.  method AFN_WPROD_DMMA: FP64 tensor cores (DMMA); AFN_WPROD_INT8: */
/* exact INT8 slicing on the tcgen05 tensor cores (8 slices per operand, 36   */
/* INT8 products, FP64-GEMM-level error; k < 65536); AFN_WPROD_CUT (Gaussian, */
/* d <= 3): the terms with K21 entries < 2^-128 dropped (wcut.cu, DESIGN.md  */
/* 6.3).  The AFN build uses the cutoff product when it keeps at most half   */
/* of the landmarks per tile (afn_set_cutoff_mode), else AFN_WPROD_INT8 for  */
/* k >= 512.                                                                 */
#define AFN_WPROD_DMMA 0
#define AFN_WPROD_INT8 1
#define AFN_WPROD_CUT 2
afn_status afn_w_product(const double* X1, int64_t k, const double* Xr, int64_t N, int32_t d, int32_t kernel,
                         double l, const double* Linv, int32_t method, double* W, void* stream);

/* kNN lower pattern.  For each position i of the N points P:   */
/* row i = {i} plus the min(w-1, i) nearest positions j < i; columns        */
/* ascending (diagonal last).  row_ptr: N+1 int64 device (closed form        */
/* row_ptr[i] = sum_{t<i} min(w, t+1)), col: row_ptr[N] int32 device.        */
/* 1 <= w <= AFN_W_MAX.  Stream-ordered.                                     */
afn_status afn_knn_pattern(const double* P, int64_t N, int32_t d, int32_t w,
                           int64_t* row_ptr, int32_t* col, void* stream);

/* Algorithm 1 on device.  [sync]  Outputs (host): khat, r, and */
/* refined (1 if the eigenvalue-count branch was taken).  m = 0 -> default.  */
afn_status afn_estimate_rank(const double* X, int64_t n, int32_t d, int32_t kernel, double l, int32_t m,
                             uint64_t rng_seed, int32_t k_threshold, int64_t* khat,
                             int32_t* r, int32_t* refined, void* stream);

/* ------------------------------------------------------------------------ */
/* Build the AFN preconditioner M = B B^T of eq:factorized-form:*/
/*   landmarks X_k by FPS, perm = [landmarks; rest ascending],   */
/*   L L^T = K11 + mu I, W = K21 L^{-T} (= (L^{-1}K12)^T),      */
/*   kNN pattern and FSAI G of S = K22 + mu I - K21 (K11+mu I)^{-1} K12      */
/*   (P:L211-212, L248-263).  X is copied; the caller may free it after.     */
/*   [sync].  On error *out is NULL.                                          */
afn_status afn_build(const double* X, int64_t n, int32_t d, const afn_params* params /*host*/,
                     void* stream, afn_handle* out /*host*/);

/* y = (K + mu I) v with the handle's points, kernel and matvec plan (the   */
/* PCG's own product: symmetric, pair units split over the ranks of a       */
/* sharded handle).  v, y: n device, original order; every rank      */
/* passes the full v and receives the full y (collective).  Stream-ordered. */
afn_status afn_matvec(afn_handle h, const double* v, double* y, void* stream);

/* z = M^{-1} r with the two-step algorithm in V-form:         */
/*   t = L^{-1} r1; u = r2 - W t; s2 = G^T (G u); s1 = L^{-T} (t - W^T s2).   */
/* r, z: n device, ORIGINAL point order (the handle permutes).  Stream-ordered */
/* on `stream`; must not alias.                                              */
afn_status afn_apply(afn_handle h, const double* r, double* z, void* stream);

/* PCG on (K+mu I) a = b with M = AFN: x0 = 0, stop when      */
/* ||r||/||b|| <= tol (recurrence residual), at most maxit iterations;        */
/* fixed_iters > 0 runs exactly that many.  b, a: n device, original order.   */
/* Non-convergence is AFN_OK with converged = 0.  [sync]                      */
afn_status afn_pcg_solve(afn_handle h, const double* b, double* a, double tol, int32_t maxit,
                         int32_t fixed_iters, afn_solve_report* rep /*host*/, void* stream);

/* Unpreconditioned CG on (K + mu I) a = b, the paper's baseline (P:L70,    */
/* L773; Table 5.1a CG rows): the PCG loop of afn_pcg_solve    */
/* with M = I (the same matvec, stopping test and report).  X: n x d, b, a:  */
/* n device, original order.  comm: NULL (one GPU) or a communicator (rows   */
/* sharded as in afn_build_dist; collective).  [sync]                        */
afn_status afn_cg_solve(afn_comm comm, const double* X, int64_t n, int32_t d, int32_t kernel, double l,
                        double mu, const double* b, double* a, double tol, int32_t maxit, int32_t fixed_iters,
                        afn_solve_report* rep /*host, optional*/, void* stream);

/* End-to-end convenience with HOST buffers: copies X, b in, builds, solves, */
/* copies a out (all inside the call).  X: n x d host, b, a: n host.  comm:  */
/* NULL (one GPU) or a communicator (every process passes the same X, b and */
/* receives the full a; collective).  [sync]                                */
afn_status afn_solve_host(afn_comm comm, const double* X, const double* b, double* a, int64_t n, int32_t d,
                          const afn_params* params, double tol, int32_t maxit,
                          afn_info* info /*host, optional*/, afn_solve_report* rep /*host, optional*/,
                          void* stream);

afn_status afn_get_info(afn_handle h, afn_info* info /*host*/);

/* Copy internal arrays to HOST memory (tests / diagnostics). bytes must equal */
/* the array size: PERM int64[n]; FILL double[k]; L double[k*k] (row-major,   */
/* lower); ROWPTR int64[n-k+1]; COL int32[nnz]; GVAL double[nnz];             */
/* W_ROWS double[(n-k)*k] (row-major W = K21 L^{-T}).                        */
enum { AFN_OUT_PERM = 0, AFN_OUT_FILL = 1, AFN_OUT_L = 2, AFN_OUT_ROWPTR = 3,
       AFN_OUT_COL = 4, AFN_OUT_GVAL = 5, AFN_OUT_W = 6 };
afn_status afn_copy_out(afn_handle h, int32_t what, void* host, size_t bytes);

/* Copy selected ROWS of a dense internal array to HOST memory (sampled parity
 * checks at sizes where the whole array does not fit the host, e.g. W at
 * n = 2^20, k = 8000 is 66.6 GB).  what: AFN_OUT_W (row t = non-landmark
 * position t, 0 <= t < n-k, k doubles each) or AFN_OUT_L (row t of L, k
 * doubles each).  rows: nrows host int64; host receives nrows*k doubles;
 * bytes must equal 8*nrows*k.  Out-of-range rows -> AFN_ERR_ARG.  [sync] */
afn_status afn_copy_out_rows(afn_handle h, int32_t what, const int64_t* rows /*host*/,
                             int64_t nrows, void* host, size_t bytes);

/* Same as afn_copy_out for local rank `local_rank` of a multi-rank handle
 * (emulated communicators drive several ranks in one process).  W holds only
 * the rank's own non-landmark rows (row_nb x k) when nranks > 1. */
afn_status afn_copy_out_local(afn_handle h, int32_t local_rank, int32_t what, void* host, size_t bytes);

void afn_destroy(afn_handle h);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: one process per GPU, rows sharded, points replicated            */
/* (BASELINE north star (3)).  Rank s owns the rows          */
/*   [a0, a0+na) = [k s/R, k (s+1)/R)  of the landmark block and             */
/*   [b0, b0+nb) = [k + N2 s/R, k + N2 (s+1)/R)  of the rest (N2 = n-k)      */
/* of the permuted order (afn_shard_rows).  Alg. 1, FPS, K11 + mu I and its  */
/* Cholesky factor are computed redundantly on every rank (identical,        */
/* deterministic); W rows, kNN rows, FSAI rows, kernel-matvec rows and the   */
/* vector updates are sharded; the exchanges are all-gathers (NCCL broadcasts */
/* of each owner's rows): W, pattern and G rows once after the build, and    */
/* per PCG iteration the CG vector p, the apply's u and G u, the k-vector    */
/* partials of W^T s2 and the dot-product partials, all summed in rank order  */
/* (deterministic, identical on every rank).                                 */
#define AFN_COMM_ID_BYTES 128
/* NCCL unique id (rank 0 creates it and broadcasts the 128 bytes, e.g. with */
/* torch.distributed).  nccl_path: libnccl.so.2 to dlopen, NULL = default.  */
afn_status afn_comm_unique_id(void* id /*host, 128 B*/, const char* nccl_path);
/* Join a communicator of nranks processes, one GPU each (the current        */
/* device).  Collective over the nranks processes.  nranks = 1 needs no NCCL. */
afn_status afn_comm_init(const void* id /*host*/, int32_t nranks, int32_t rank,
                         const char* nccl_path, afn_comm* out /*host*/);
/* Test communicator: nranks logical ranks driven by this one process on the */
/* current device, each with its own buffers; the exchanges are device      */
/* copies between them.  Results match a real nranks-GPU run bit for bit.   */
afn_status afn_comm_init_emulated(int32_t nranks, afn_comm* out /*host*/);
void afn_comm_destroy(afn_comm c);
/* Host waits on streams with NCCL work poll ncclCommGetAsyncError; after an  */
/* asynchronous error or `seconds` (default 600) the communicator is aborted */
/* and the call returns AFN_ERR_NCCL (instead of hanging on a lost peer).    */
afn_status afn_comm_set_timeout(afn_comm c, double seconds);
/* rows[4] = {a0, na, b0, nb} owned by `rank` (host arithmetic only). */
afn_status afn_shard_rows(int64_t n, int64_t k, int32_t nranks, int32_t rank, int64_t* rows /*host*/);
/* afn_build over a communicator (comm = NULL: single GPU, same as afn_build).*/
/* Every process passes the same X and params.  The handle keeps the comm   */
/* pointer (destroy the handle first).  afn_apply / afn_pcg_solve on such a   */
/* handle are collective: r / b are the full vectors (replicated), z / a     */
/* receive the full result on every process.  [sync]                        */
afn_status afn_build_dist(afn_comm comm, const double* X, int64_t n, int32_t d,
                          const afn_params* params /*host*/, void* stream, afn_handle* out /*host*/);

/* ------------------------------------------------------------------------ */
/* Measurement helpers (bench.py): FP64 FMA peak probe.  Runs `iters` DFMA   */
/* chains on every SM and returns achieved FP64 TFLOP/s (FMA = 2). [sync]    */
afn_status afn_probe_dfma(int64_t iters, double* tflops /*host*/, void* stream);
/* Same for FP64 tensor-core DMMA (mma.sync m8n8k4 f64).                      */
afn_status afn_probe_dmma(int64_t iters, double* tflops /*host*/, void* stream);
/* MUFU.EX2 throughput (ex2.approx.ftz.f32 chains on every SM), in G ops/s: */
/* the bound of the cutoff matvec's FP32 body (one EX2 per pair).  [sync]    */
afn_status afn_probe_ex2(int64_t iters, double* gops /*host*/, void* stream);

/* Use of the Gaussian kernel's decay for the handles  */
/* built and products planned after the call (process-wide).  Gaussian       */
/* kernel, d <= 3:                                                           */
/*   kernel matvec (full product): the cutoff plan -- points in a spatial    */
/*     order, (128-row group, 32-column tile) items whose boxes are at least */
/*     s = 128 apart (s = ||x - y||^2 log2(e) / l^2: every entry < 2^-128)   */
/*     skipped, items at least s = 48 apart (entries < 2^-48) in FP32;       */
/*   W = K21 L^{-T} in afn_build: terms with K21 entries < 2^-128 dropped,  */
/*     per 64-row tile of a spatial order a dense product over the kept     */
/*     landmarks.                                                            */
/* mode 0 (default): the cutoff matvec whenever it applies, the cutoff W    */
/* when it keeps at most half of the landmarks per tile, else the dense     */
/* paths; 1: never; 2: both whenever they apply; 3: as 0 but the FSAI pair  */
/* products through W instead of Z = K21 (K11 + mu I)^{-1} (DESIGN.md 6.4;  */
/* Z takes another (n - k) x k buffer during the build).  Other kernels /    */
/* d > 3 / row ranges: the dense paths.  AFN_ERR_ARG for any other mode.     */
afn_status afn_set_cutoff_mode(int32_t mode);

/* Per-kernel CUDA-event timers (off by default).  When enabled the library
 * records an event pair around each timed kernel class on the launching
 * stream and accumulates device ms, algorithmic work (flops) and counts.
 * Classes: 0 kmv, 1 FSAI pair GEMM, 2 FSAI assembly, 3 FSAI Cholesky,
 * 4 FSAI per-row Gram (fallback), 5 FPS, 6 W GEMM, 7 L^-T, 8 potrf, 9 kNN,
 * 10 apply, 11 Alg. 1.  afn_kt_read returns the number of classes.          */
void afn_kt_enable(int32_t on);
void afn_kt_reset(void);
int32_t afn_kt_read(double* ms /*host*/, double* work /*host*/, int64_t* count /*host*/, int32_t n);

/* ------------------------------------------------------------------------ */
/* Optional caller allocator, e.g. PyTorch's caching        */
/* allocator: every device allocation of the library then goes through      */
/* alloc(bytes, stream, ctx) and free(ptr, bytes, stream, ctx) instead of    */
/* the library's stream-ordered pool (cudaMallocAsync).  alloc returns NULL  */
/* on failure (-> AFN_ERR_NOMEM).  The library calls free only after the     */
/* stream position of the free has completed (so a caching allocator may    */
/* hand the block to any stream at once).  Process-wide; set it while no     */
/* handle built with the previous allocator is alive (else AFN_ERR_ARG).     */
/* (NULL, NULL, NULL) restores the pool.                                     */
typedef void* (*afn_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*afn_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);
afn_status afn_set_allocator(afn_alloc_fn alloc, afn_free_fn free_fn, void* ctx);
/* Reserved / used bytes of the library's default pool on the current device */
/* (diagnostics: memory reuse across builds and streams).                   */
afn_status afn_pool_stats(int64_t* reserved /*host*/, int64_t* used /*host*/);

/* Number of kernels this library launched since load (its own kernels only). */
int64_t afn_launch_count(void);
const char* afn_last_error(void);
int32_t afn_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AFN_H_ */

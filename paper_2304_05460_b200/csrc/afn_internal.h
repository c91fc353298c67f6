// afn_internal.h -- host-side internal interfaces between the .cu modules and
// the C ABI (abi.cu).  Not part of the public boundary (include/afn.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <utility>
#include <vector>

#include "../../include/afn.h"

// Communicator (comm.cu): R logical ranks; this process drives ranks
// [rank0, rank0 + nlocal) -- one with NCCL, all R when emulated (tests).
struct afn_comm_s {
  int R = 1;
  int nlocal = 1;
  int rank0 = 0;
  bool emulated = false;
  void* nccl = nullptr;    // ncclComm_t (nullptr after an abort)
  void* stage = nullptr;   // packed all-gather staging buffer (device)
  size_t stage_bytes = 0;
  double timeout_s = 600.0;  // host waits on NCCL work (afn_comm_set_timeout)
};

namespace afn {

using Comm = afn_comm_s;

// kernel function and length-scale l; kind = AFN_KERNEL_*
struct Kern {
  int kind = 0;
  double l = 1.0;
};

// Rows of the permuted order owned by one rank: a block of
// the landmark rows [a0, a0+na) and a block of the non-landmark rows
// [b0, b0+nb).  Row t of the rank's local numbering is phys(t).  With one
// rank the two blocks are adjacent ({0, k, k, n-k}) and phys(t) = t.
struct Seg2 {
  int64_t a0 = 0, na = 0, b0 = 0, nb = 0;
  __host__ __device__ int64_t size() const { return na + nb; }
  __host__ __device__ int64_t phys(int64_t t) const { return t < na ? a0 + t : b0 + (t - na); }
};
inline Seg2 shard_rows(int64_t n, int64_t k, int R, int s) {
  const int64_t N2 = n - k;
  Seg2 g;
  g.a0 = k * s / R;
  g.na = k * (s + 1) / R - g.a0;
  g.b0 = k + N2 * s / R;
  g.nb = k + N2 * (s + 1) / R - g.b0;
  return g;
}
inline Seg2 seg_range(int64_t row0, int64_t nrows) { return Seg2{row0, nrows, row0 + nrows, 0}; }

// byte ranges [offset, offset+len) a rank owns in an exchanged buffer
using RankRanges = std::vector<std::pair<size_t, size_t>>;
// every local rank's buffer bufs[q] receives all ranks' owned ranges
afn_status comm_allgatherv(const Comm* c, char* const* bufs, const std::vector<RankRanges>& owned,
                           cudaStream_t st);
// host wait for `st`; with NCCL: polls ncclCommGetAsyncError, aborts the
// communicator on an error or after c->timeout_s (AFN_ERR_NCCL)
afn_status comm_stream_sync(const Comm* c, cudaStream_t st);

int num_sms();  // SM count of the current device (cached per device)

// ---- optional per-kernel CUDA-event timers (bench.py roofline) -------------
enum KtId { KT_KMV = 0, KT_FSAI_GEMM, KT_FSAI_ASM, KT_FSAI_CHOL, KT_FSAI_GRAM, KT_FPS, KT_W_GEMM,
            KT_LINV, KT_POTRF, KT_KNN, KT_APPLY, KT_ALG1, KT_N };
bool kt_enabled();
void kt_begin(int id, cudaStream_t st);
void kt_end(int id, cudaStream_t st, double work);  // work: algorithmic flops (or bytes)
void kt_collect();                                  // after a stream sync

// Stream-ordered device allocation helpers (cudaMallocAsync pool).
// (with a caller allocator set: dalloc calls it; dfree defers the caller's
// free until the stream position of the free completes -- release_deferred
// hands back the completed ones, all of them with wait = true)
afn_status dalloc(void** p, size_t bytes, cudaStream_t st);
void dfree(void* p, cudaStream_t st);
void release_deferred(bool wait);
// return the library's cached large blocks to the pool (afn_pool_stats and
// allocation failures call it)
void trim_big_blocks();

// ---- kernel matvec (kmv.cu) ----------------------------------------------
struct KmvPlan {
  int64_t row_tiles = 0, chunks = 1, chunk_cols = 0;
  // symmetric full matvec (each unordered pair once, row and column sums,
  // kmv.cu): row blocks of sym_rbw rows, 32-column tiles, sym_units work
  // units split evenly over sym_gt = sym_R x sym_grid CTAs; this rank runs
  // CTAs [sym_rank sym_grid, (sym_rank + 1) sym_grid)
  bool sym = false;
  int64_t sym_rbw = 0, sym_nrb = 0, sym_nt = 0, sym_units = 0, sym_grid = 0, sym_gt = 0, sym_tab_dbl = 0;
  int sym_R = 1, sym_rank = 0;
  // cutoff plan (Gaussian, d <= 3; kmv.cu): the symmetric
  // split over a spatial order of the points, keeping only the (row block,
  // 32-column tile) units whose bounding boxes are closer than the skip bound
  // (every entry of a skipped unit is below 2^-128); units whose boxes are
  // closer than the FP64 bound run the FP64 body, the rest (entries below
  // 2^-48) an FP32 body.  The unit list, its transpose and the spatial order
  // live in the workspace at the offsets below (in doubles).
  bool cut = false;
  int64_t cut_u64 = 0, cut_u32 = 0, cut_ntiles = 0;
  double cut_pairs64 = 0, cut_pairs32 = 0;  // useful unordered pairs per class
  int64_t o_rp = 0, o_cb = 0, o_xc = 0, o_ctr = 0, o_sidx = 0, o_ut = 0, o_ustart = 0, o_wst = 0, o_seg = 0,
          o_rbase = 0, o_tptr = 0, o_tu = 0;
  int64_t ws = 0;  // workspace doubles for kmv_launch
};
// ---- spatial order (spatial.cu) ----------------------------------------------
// sidx[pos] = point: Morton order of a grid of ~2 points per cell over the
// first min(d, 3) coordinates, a cell's points by ascending index (deterministic)
afn_status morton_order(const double* X, int64_t n, int d, int* sidx, cudaStream_t st);
// off[0..M] = exclusive scan of cnt[0..M) (one block; M up to a few million)
afn_status scan_i32_i64(const int* cnt, int64_t M, int64_t* off, cudaStream_t st);

// cutoff selection (afn_set_cutoff_mode) for the kernel matvec and W: 0 auto
// (the cutoff plan / product when it keeps at most half of the pairs), 1
// never, 2 whenever it applies (Gaussian, d <= 3, full symmetric product)
void kmv_set_mode(int mode);
int kmv_get_mode();
using WsGet = std::function<afn_status(double**, size_t)>;
// The plan of a full (sym_ok) or row-range product for the prescaled points
// Xs and its workspace *ws (allocated through get, tables uploaded): the
// cutoff plan when it applies, else kmv_plan + kmv_plan_init.  Synchronises
// `st` (the unit counts come back to the host).
afn_status kmv_plan_make(const double* Xs, int64_t n, int64_t nrows, int d, int kind, bool sym_ok, int R, int rank,
                         cudaStream_t st, const WsGet& get, KmvPlan* out, double** ws);
// A cutoff plan built over the points in another order (the build makes it
// from the original X while FPS runs): its point indices become the handle's
// positions, sidx <- iperm[sidx] with perm[position] = original index
afn_status kmv_plan_remap(const KmvPlan& p, double* ws, const int64_t* perm, int64_t n, cudaStream_t st);
// sym_ok: a full matvec may use the symmetric kernel (its row sums differ from
// a row shard's by rounding; kernel_matvec_rows never uses it).  With R > 1
// ranks the symmetric plan splits the pair units over the ranks
// (kmv_sym_rank_partial + an exchange + kmv_sym_combine).
KmvPlan kmv_plan(int64_t n, int64_t nrows, int d, int num_sms, bool sym_ok = false, int R = 1, int rank = 0);
// upload the plan's tables into its workspace and fill the exp2 tables (once
// per device); call before the first launch with this workspace (not inside
// a stream capture)
afn_status kmv_plan_init(const KmvPlan& p, double* ws, cudaStream_t st);
// executed FP64 flops (FMA = 2) and FP64-pipe thread instructions of one
// launch, counted per useful pair
double kmv_flops(const KmvPlan& p, int64_t n, int64_t nrows, int d, int kind);
double kmv_fp64_inst(const KmvPlan& p, int64_t n, int64_t nrows, int d, int kind);
// this rank's partial of the symmetric product (all n rows, no mu term): qout[n]
afn_status kmv_sym_rank_partial(const double* Xs, int64_t n, int d, int kind, const double* v, const KmvPlan& p,
                                double* ws, double* qout, cudaStream_t st);
// y_i = (1 + mu) v_i + sum_s qpart[s n + i] (rank order) over the rows g; dout: v . y over g
afn_status kmv_sym_combine(const double* qpart, int R, int64_t n, Seg2 g, const double* v, double mu, double* y,
                           cudaStream_t st, double* dout = nullptr, double* dws = nullptr, unsigned* dcnt = nullptr);
// Xs = X * sqrt(log2 e)/l   (n x d)
afn_status kmv_prescale(const double* X, int64_t n, int d, Kern kn, double* Xs, cudaStream_t st);
// rows `rows` of (K + mu I) v (v: all n entries); partial: chunks*rows.size() doubles.
// y_phys: y[rows.phys(t)] (true) or y[t] (false) receives row t.
// dout (symmetric plan only): also v . y into *dout (dws/dcnt: dot workspace)
afn_status kmv_launch(const double* Xs, int64_t n, int d, int kind, const double* v, double mu, Seg2 rows,
                      double* y, bool y_phys, double* partial, const KmvPlan& p, cudaStream_t st,
                      double* dout = nullptr, double* dws = nullptr, unsigned* dcnt = nullptr);

// ---- FPS (fps.cu) ---------------------------------------------------------
// kstop (optional, device): the run may stop early once *kstop (which another
// stream may lower while it runs) is reached -- entries below it are complete
afn_status fps_run(const double* X, int64_t n, int d, int64_t k, int64_t seed, int64_t* idx,
                   double* fill, cudaStream_t st, const int64_t* kstop = nullptr);

// ---- kNN pattern (knn.cu) -------------------------------------------------
int64_t knn_nnz(int64_t N, int w);
// row_ptr for all N rows (closed form); col for rows [row_lo, row_hi) (default: all)
afn_status knn_run(const double* P, int64_t N, int d, int w, int64_t* row_ptr, int32_t* col,
                   cudaStream_t st, int64_t row_lo = 0, int64_t row_hi = -1);

// ---- dense build (dense.cu) -----------------------------------------------
// gather rows: Y[i] = X[perm[i]] (n x d)
afn_status gather_rows(const double* X, int64_t n, int d, const int64_t* perm, double* Y,
                       cudaStream_t st);
// A = K(X1, X1) + mu I, full k x k row-major
afn_status gen_k11(const double* X1, int64_t k, int d, Kern kn, double mu, double* A,
                   cudaStream_t st);
// in-place lower Cholesky of the k x k row-major A (upper triangle zeroed);
// *d_info = 0 on success, else 1 + the failing row.
afn_status potrf_lower(double* A, int64_t k, int* d_info, cudaStream_t st);
// nbatch independent k x k factorisations (matrix b at A + b bs, d_info[b]);
// skip_thr >= 0: threshold pivoting (a pivot <= skip_thr zeroes its column of
// L, no report; Alg. 1, reading R10), else breakdowns are reported as above
afn_status potrf_batched(double* A, int64_t k, int nbatch, int64_t bs, double skip_thr, int* d_info,
                         cudaStream_t st);
// W (N x k) = K(Xr, X1) L^{-T} as a GEMM with the explicit L^{-T}
// W = K(Xr, X1) L^{-T} from Linv = L^{-1} on the INT8 tensor cores (ozaki.cu)
afn_status w_gemm_ozaki(const double* Linv, int64_t k, const double* X1, const double* Xr, int64_t N, int d, Kern kn,
                        double* W, cudaStream_t st);
constexpr int64_t AFN_W_INT8_MIN_K = 512;  // the build's W takes the INT8 path from this k on
// W = K(Xr, X1) L^{-T} keeping only the entries >= 2^-128 (Gaussian, d <= 3;
// wcut.cu).  *used = false (nothing written) when it does not
// apply or (unless force) keeps more than half of the landmarks per tile;
// *flops = executed FP64 flops
afn_status w_gemm_cut(const double* LinvT, int64_t k, const double* X1, const double* Xr, int64_t N, int d, Kern kn,
                      double* W, cudaStream_t st, bool force, bool* used, double* flops);
// The same in two calls: the plan (spatial order, kept landmarks, the K21
// tiles; needs only the points, synchronises st) and the product with L^{-T}
// (stream-ordered; releases the plan).  used = false: the dense path applies.
// zmode (one rank): also the landmarks' Morton order lp, the same lists over
// it (ulistp, positions ascending) with their K21 tiles Ap, and tilerow[b] =
// (tile << 6) | row of point b -- what the FSAI product through Z = K21 M
// needs (fsai_sddmm.cu); w_cut_run then keeps the plan, w_cut_z forms
// M = L^{-T} L^{-1}, Mp = M[lp][:, lp] and Zp = K21 M[:, lp] (N x k, rows by point).
struct WCutPlan {
  bool used = false;
  int64_t k = 0, N = 0, nt = 0;
  int *sidx = nullptr, *ulist = nullptr;
  int64_t *uoff = nullptr, *aoff = nullptr;
  double* A = nullptr;
  int *lp = nullptr, *ulistp = nullptr, *tilerow = nullptr;
  double* Ap = nullptr;
  double flops = 0.0, zflops = 0.0;  // executed flops of the W and Z products
  int64_t E = 0;          // list entries over all tiles
  int64_t Adbl = 0;       // doubles of the K21 tiles (A)
  bool keep = false;      // keep the plan after W (the apply through the tiles)
  int64_t* jptr = nullptr;  // apply: per landmark its list entries (jidx), and
  int* jidx = nullptr;      // the per-entry column sums CT
  double* CT = nullptr;
  std::vector<void*> mem;
  cudaStream_t st = nullptr;
};
// The AFN apply's two W products through the tiles (one rank): u = r2 - K21 y1
// (rows by point) and w = K21^T s2 (fixed summation order); w_cut_apply_prep
// builds the transposed lists once after the build.
afn_status w_cut_apply_prep(WCutPlan* p, cudaStream_t st);
afn_status w_cut_apply_n(const WCutPlan* p, const double* y1, const double* r2, double* u, cudaStream_t st);
afn_status w_cut_apply_t(const WCutPlan* p, const double* s2, double* w, cudaStream_t st);
afn_status w_cut_plan(const double* X1, int64_t k, const double* Xr, int64_t N, int d, Kern kn, bool force,
                      bool zmode, cudaStream_t st, WCutPlan* p);
afn_status w_cut_run(WCutPlan* p, const double* LinvT, double* W, cudaStream_t st);
afn_status w_cut_z(WCutPlan* p, const double* LinvT, const double* Linv, double* M, double* Mp, double* Zp,
                   cudaStream_t st);
void w_cut_free(WCutPlan* p);
// C = A B (k x k, row-major) for A = B^T upper, B lower triangular: the symmetric C's lower
// block triangle only (entries above the diagonal tiles unwritten; dense.cu)
afn_status gemm_upper_lower(const double* A, const double* B, int64_t k, double* C, cudaStream_t st);
afn_status w_gemm(const double* LinvT, int64_t k, const double* X1, const double* Xr, int64_t N, int d,
                  Kern kn, double* W, cudaStream_t st);
// G = F^T F (C x C, full) for F: R x C row-major; deterministic
afn_status syrk_ata(const double* F, int64_t R, int64_t C, double* G, cudaStream_t st);
// C = alpha A B (M x N, row-major, leading dimensions lda / ldb / ldc), FP64
// tensor cores (DMMA); K = 0 gives C = 0
afn_status gemm_nn(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K, int64_t lda,
                   int64_t ldb, int64_t ldc, double alpha, cudaStream_t st);
// LinvT (k x k row-major) = L^{-T} (upper triangular)
// ws: nullptr (allocated on st) or linv_ws_doubles(k) doubles already ordered before st's work
afn_status trsm_linvt(const double* L, int64_t k, double* LinvT, cudaStream_t st, double* ws = nullptr);
int64_t linv_ws_doubles(int64_t k);

// ---- FSAI (fsai.cu) -------------------------------------------------------
// G values of rows [row_lo, row_hi) on the pattern of the Schur complement
// S = K22 + mu I - W W^T (W: all N rows)
afn_status fsai_run(const double* X2, int64_t N, int d, Kern kn, double mu, const double* W,
                    int64_t k, const int64_t* row_ptr, const int32_t* col, int64_t row_lo,
                    int64_t row_hi, double* gval, int* d_info, cudaStream_t st);
// CSR transpose (N x N, columns sorted within each output row).  val/tval may
// be null (pattern only); tmap (optional) receives the source nnz index.
afn_status csr_transpose(const int64_t* rp, const int32_t* col, const double* val, int64_t N,
                         int64_t nnz, int64_t* trp, int32_t* tcol, double* tval, cudaStream_t st,
                         int64_t* tmap = nullptr);
afn_status gather_map(const double* v, const int64_t* map, int64_t nnz, double* out, cudaStream_t st);
// The products W_a . W_b through Z = K21 M (one rank, the cutoff W plan's
// Z mode): Zp (N x k, rows by point, columns in the
// landmarks' Morton order) and the plan's per-tile K21 blocks over that order.
struct FsaiZ {
  const double* Zp = nullptr;
  const int* tilerow = nullptr;
  const int64_t* uoff = nullptr;
  const int* ulistp = nullptr;
  const int64_t* aoff = nullptr;
  const double* Ap = nullptr;
  bool staged = false;  // stage each half group's Z columns in shared memory
};
// FSAI through the union of needed Schur-complement pairs (fsai_sddmm.cu).
// Returns AFN_ERR_STATE (nothing written) if a group's pair union overflows.
// z: the products through Z (else D_g = W_g W_U^T).
afn_status fsai_sddmm_run(const double* X2, int64_t N, int d, Kern kn, double mu, const double* W,
                          int64_t k, const int64_t* rp, const int32_t* col, const int64_t* trp,
                          const int32_t* tcol, int64_t row_lo, int64_t row_hi, double* gval,
                          int* d_info, cudaStream_t st, cudaStream_t pst = nullptr, const FsaiZ* z = nullptr);

// ---- BLAS-2 / SpMV / vectors (blas.cu) ------------------------------------
// y = ybase + alpha * A x, A: R x C row-major (lda = C).  ybase may be null (0)
// tri: 0 full, 1 A upper triangular (columns >= row), 2 lower (columns <= row);
// the excluded triangle must be stored as zeros
afn_status gemv_n(const double* A, int64_t R, int64_t C, const double* x, const double* ybase,
                  double alpha, double* y, cudaStream_t st, int tri = 0);
afn_status transpose_sq(const double* A, int64_t k, double* At, cudaStream_t st);
// y = ybase + alpha * A^T x; ws >= gemv_t_ws(R, C) doubles
int64_t gemv_t_ws(int64_t R, int64_t C);
afn_status gemv_t(const double* A, int64_t R, int64_t C, const double* x, const double* ybase,
                  double alpha, double* y, double* ws, cudaStream_t st);
afn_status spmv_csr(const int64_t* rp, const int32_t* col, const double* val, int64_t N,
                    const double* x, double* y, cudaStream_t st);
afn_status gather_vec(const double* x, const int64_t* perm, int64_t n, double* y, cudaStream_t st);
afn_status scatter_vec(const double* x, const int64_t* perm, int64_t n, double* y, cudaStream_t st);

// Vector operations over the rows `g` of full-length (n) vectors.
// deterministic dot: *out = a . b over g  (ws >= dot_ws() doubles, cnt: 1 zeroed uint)
int64_t dot_ws();
afn_status dot(const double* a, const double* b, Seg2 g, double* out, double* ws, unsigned* cnt,
               cudaStream_t st);
// PCG scalar slots (device doubles): rz alternates between slots 0 and 1
enum { SC_RZ0 = 0, SC_RZ1 = 1, SC_PQ = 2, SC_RR = 3, SC_BB = 4, SC_TMP = 5, SC_DONE = 6, SC_ITS = 7, SC_IT = 8, SC_N = 16 };
// Device-side skip flag for the apply / matvec kernels queued by the PCG loop
// (kernels return at once when *flag != 0); nullptr = never skip.  Per host thread.
void set_skip(const double* flag);
const double* get_skip();
// x += alpha p, r -= alpha q, rr = r.r and the stopping test (one rank)
afn_status pcg_update_xr_check(double* x, double* r, const double* p, const double* q, Seg2 g, double* sc,
                               int rz_slot, double* ws, unsigned* cnt, double nb, double tol, int maxit, int fixed,
                               double* hist, cudaStream_t st);
// advances the device iteration counter sc[SC_IT] (graph-replayable)
afn_status pcg_check(double* sc, double nb, double tol, int maxit, int fixed, double* hist, cudaStream_t st);
// x += a p; r -= a q over g with a = sc[rz_slot]/sc[PQ] (0 if PQ <= 0); *rr = r.r over g
afn_status pcg_update_xr(double* x, double* r, const double* p, const double* q, Seg2 g,
                         const double* sc, int rz_slot, double* rr, double* ws, unsigned* cnt,
                         cudaStream_t st);
// p = z + beta p over g, beta = sc[rz_new_slot]/sc[rz_old_slot]
afn_status pcg_update_p(double* p, const double* z, Seg2 g, const double* sc, int rz_new_slot,
                        int rz_old_slot, cudaStream_t st);
afn_status vec_copy(double* y, const double* x, Seg2 g, cudaStream_t st);
afn_status vec_axpby(double* y, double a, const double* x, double b, Seg2 g, cudaStream_t st);
// y = a x over g
afn_status vec_scale(double* y, double a, const double* x, Seg2 g, cudaStream_t st);
// y[i] = v ; y *= 1/sqrt(*s) (s device scalar)
afn_status vec_fill(double* y, double v, int64_t n, cudaStream_t st);
afn_status vec_scale_rsqrt(double* y, const double* s, int64_t n, cudaStream_t st);
// A[i][i] += v (k x k row-major)
afn_status add_diag(double* A, int64_t k, double v, cudaStream_t st);
// sc[slot] = sum_{s < R} part[s * stride + slot] (rank order) for each slot in mask
afn_status combine_slots(const double* part, int R, int stride, unsigned mask, double* sc,
                         cudaStream_t st);
// y[c] = base[c] - sum_{s < R} part[s * C + c] (rank order), c < C; base may be null (0)
afn_status combine_sub(const double* part, int R, int64_t C, const double* base, double* y,
                       cudaStream_t st);

// ---- Alg. 1 (alg1.cu) ------------------------------------------------------
struct Alg1Result {
  int64_t khat = 0;
  int32_t r = 0, m = 0, refined = 0;
  double scale = 0.0;
};
int alg1_default_m(int64_t n);
// k uniform random landmarks (reading R29), key order
afn_status uniform_landmarks(int64_t n, int64_t k, uint64_t seed, int64_t* idx, cudaStream_t st);
afn_status alg1_run(const double* X, int64_t n, int d, Kern kn, int m, uint64_t rng_seed,
                    int k_threshold, Alg1Result* res, cudaStream_t st);

// ---- probes (probe.cu) -----------------------------------------------------
afn_status probe_dfma(int64_t iters, double* tflops, cudaStream_t st);
afn_status probe_dmma(int64_t iters, double* tflops, cudaStream_t st);
afn_status probe_ex2(int64_t iters, double* gops, cudaStream_t st);

}  // namespace afn

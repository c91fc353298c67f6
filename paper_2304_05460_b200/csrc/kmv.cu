// kmv.cu -- matrix-free Gaussian kernel matvec y = (K + mu I) v  (PAPER.md
// L33, L38; the paper's "explicit" dense matvec, L957).  FP64 SIMT, ALU-bound.
//
// Layout: the points are pre-scaled once, Xs = X * sqrt(log2 e)/l, so that
// ||xs_i - xs_j||^2 = log2(e) ||x_i - x_j||^2 / l^2 and K_ij = 2^(-||xs_i-xs_j||^2).
// Grid (row tiles x column chunks): each thread owns RB rows (registers), a CTA
// owns NT*RB rows and one column chunk, streamed through shared memory in
// tiles of TC columns (x_j and v_j interleaved).  Each thread sums its rows
// over the chunk in column order; a second kernel adds the chunk partials in
// chunk order plus mu v_i -> bit-identical results run to run and independent
// of how rows are sharded across GPUs.
// Per pair (d=3): 3 DADD + 1 DMUL + 2 DFMA (distance) + 8 (exp2) + 1 DFMA = 15
// FP64-pipe instructions.  The roofline counts a fixed algorithmic 3d+19 flops
// per pair (d=3: 28; the direct-difference + degree-6/16-entry-table exp
// formulation of DESIGN.md, FMA = 2), independent of later instruction savings.
#include <algorithm>
#include <mutex>
#include <vector>
#include <type_traits>
#include <cmath>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {

namespace {

constexpr int KMV_NT = 256;

// 2^(r/256), r = 0..255 (one table lookup and one multiply per exp2 in the
// matvec instead of two of each with the 2 x 16-entry tables); filled once.
__device__ double g_exp2_256[256];
__device__ double g_exp2_2048[2048];
__global__ void exp2_256_init_kernel() {
  g_exp2_256[threadIdx.x] = exp2((double)threadIdx.x / 256.0);
  for (int r = threadIdx.x; r < 2048; r += blockDim.x) g_exp2_2048[r] = exp2((double)r / 2048.0);
}
// 2^(-s) with a 2048-entry table and a degree-3 polynomial: |f| <= 1/4096, the
// first omitted Taylor term is ln(2)^4 f^4 / 24 < 3.4e-17 (7 FP64 instructions
// instead of 8)
__device__ __forceinline__ double exp2_neg2048(double s, const double* tab) {
  const double magic = 0x1.8p52;
  double t = fma(s, -2048.0, magic);  // rint(-2048 s) in the low word
  double nf = t - magic;
  double f = fma(nf, -0x1.0p-11, -s);  // exact, |f| <= 1/4096
  const int n = __double2loint(t);
  double p = AFN_E2C3;
  p = fma(p, f, AFN_E2C2);
  p = fma(p, f, AFN_E2C1);
  p = fma(p, f, AFN_E2C0);
  p = p * tab[n & 2047];
  int hi = __double2hiint(p) + ((n >> 11) << 20);
  hi = (__double2hiint(s) >= 0x408FE000) ? 0 : hi;  // s >= 1020 -> ~0 (as exp2_neg)
  return __hiloint2double(hi, __double2loint(p));
}
__device__ __forceinline__ double exp2_neg256(double s, const double* tab) {
  const double magic = 0x1.8p52;
  double t = fma(s, -256.0, magic);   // rint(-256 s) in the low word
  double nf = t - magic;
  double f = fma(nf, -0x1.0p-8, -s);  // exact, |f| <= 1/512
  const int n256 = __double2loint(t);
  double p = AFN_E2C4;
  p = fma(p, f, AFN_E2C3);
  p = fma(p, f, AFN_E2C2);
  p = fma(p, f, AFN_E2C1);
  p = fma(p, f, AFN_E2C0);
  p = p * tab[n256 & 255];
  int hi = __double2hiint(p) + ((n256 >> 8) << 20);
  hi = (__double2hiint(s) >= 0x408FE000) ? 0 : hi;  // s >= 1020 -> ~0 (as exp2_neg)
  return __hiloint2double(hi, __double2loint(p));
}


template <int D>
struct KmvTraits {
  static constexpr int CS = ((D + 1) + 1) & ~1;   // coords + v, padded to even
  static constexpr int TC = D <= 8 ? 512 : 256;   // columns per smem tile (<= 40 KB)
  static constexpr int RB = D <= 4 ? 4 : (D <= 8 ? 2 : 1);  // rows per thread
};

// KER 0 (Gaussian): Xs = X sqrt(log2 e)/l, K = 2^(-|xs_i - xs_j|^2).
// KER 1 (Matern-3/2): Xs = X sqrt(3)/l, t = |xs_i - xs_j|,
//        K = (1 + t) 2^(-t log2 e).
template <int D, int RB, int KER>
__global__ void __launch_bounds__(KMV_NT, 2)
kmv_partial_kernel(const double* __restrict__ Xs, const double* __restrict__ v, int64_t n,
                   Seg2 rows, int64_t chunk_cols, double* __restrict__ partial, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;  // PCG already stopped (device-side flag)
  constexpr int CS = KmvTraits<D>::CS;
  constexpr int KMV_TC = KmvTraits<D>::TC;
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  __shared__ double s_t256[256];
  __shared__ __align__(16) double s_col[KMV_TC * CS];
  load_exp2_tab(s_tab);
  for (int t = threadIdx.x; t < 256; t += KMV_NT) s_t256[t] = g_exp2_256[t];

  // local row t -> physical row rows.phys(t) (two blocks when row-sharded)
  const int64_t nrows = rows.size();
  const int64_t rbase = (int64_t)blockIdx.x * (KMV_NT * RB) + threadIdx.x;
  double xi[RB][D];
  double acc[RB];
#pragma unroll
  for (int t = 0; t < RB; ++t) {
    const int64_t lr = rbase + (int64_t)t * KMV_NT;
    const int64_t r = rows.phys(lr < nrows ? lr : 0);  // clamp (masked at the write)
#pragma unroll
    for (int c = 0; c < D; ++c) xi[t][c] = Xs[r * D + c];
    acc[t] = 0.0;
  }

  const int64_t c0 = (int64_t)blockIdx.y * chunk_cols;
  const int64_t c1 = min(n, c0 + chunk_cols);
  for (int64_t tb = c0; tb < c1; tb += KMV_TC) {
    const int tcn = (int)min((int64_t)KMV_TC, c1 - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < KMV_TC * CS; e += KMV_NT) {
      const int j = e / CS, c = e - j * CS;
      double val = 0.0;
      if (j < tcn) {
        if (c < D) val = Xs[(tb + j) * D + c];
        else if (c == D) val = v[tb + j];
      }
      s_col[e] = val;
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < tcn; ++j) {
      double xj[CS];
#pragma unroll
      for (int c = 0; c < CS; c += 2) {
        const double2 q = *reinterpret_cast<const double2*>(&s_col[j * CS + c]);
        xj[c] = q.x;
        xj[c + 1] = q.y;
      }
      const double vj = xj[D];
#pragma unroll
      for (int t = 0; t < RB; ++t) {
        double dd = xi[t][0] - xj[0];
        double s = dd * dd;
#pragma unroll
        for (int c = 1; c < D; ++c) {
          dd = xi[t][c] - xj[c];
          s = fma(dd, dd, s);
        }
        if (KER == 1) {
          const double tt = sqrt(s);
          acc[t] = fma((1.0 + tt) * exp2_neg(tt * AFN_LOG2E, s_tab), vj, acc[t]);
        } else {
          acc[t] = fma(exp2_neg256(s, s_t256), vj, acc[t]);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < RB; ++t) {
    const int64_t lr = rbase + (int64_t)t * KMV_NT;
    if (lr < nrows) partial[(int64_t)blockIdx.y * nrows + lr] = acc[t];
  }
}

// Symmetric variant for the full matvec: K is symmetric, so every unordered
// pair (i < j) is evaluated once and feeds both q_i (+= K_ij v_j, row sums in
// registers) and q_j (+= K_ij v_i, column sums) -- half the exp2 work.
//
// Balanced ("stream-K") decomposition of the upper triangle: row blocks I of
// RBW = KMV_NT RB rows; work units (I, t) are 32-column tiles t >= m I (m =
// RBW / 32; the m tiles of the diagonal block keep only j > i).  Units are
// numbered block by block, ustart(I) = I NT - m I (I - 1) / 2 (NT tiles), and
// the Gt CTAs of all ranks take equal contiguous ranges [g U / Gt, (g+1) U / Gt)
// -- no partial wave: every CTA does U / Gt units to within one.  A CTA carries
// its row sums in registers while it stays in one row block and writes them
// to its slot Rp[rbase(I) + g - gfirst(I)] when it leaves it; each column sum
// (I, j) comes from exactly one CTA, Cb[cboff(I) + j - I RBW].  Summation
// orders are fixed by (n, d, Gt): bit-identical run to run.
// segtab (device, per row block I): {gfirst(I), nseg(I), rbase(I)}.
__device__ __forceinline__ int64_t sym_ustart(int64_t I, int64_t nt, int64_t m) {
  return I * nt - m * I * (I - 1) / 2;
}
__device__ __forceinline__ int64_t sym_cboff(int64_t I, int64_t n, int64_t rbw) {
  return I * n - rbw * I * (I - 1) / 2;
}
__device__ __forceinline__ int64_t sym_cta_of(int64_t u, int64_t U, int64_t Gt) {
  return ((u + 1) * Gt - 1) / U;
}

template <int D, int RB, int KER>
__global__ void __launch_bounds__(KMV_NT, RB <= 2 ? 3 : 2)
kmv_sym_kernel(const double* __restrict__ Xs, const double* __restrict__ v, int64_t n, int64_t nrb,
               int64_t nt, int64_t U, int64_t Gt, int64_t g0, const int* __restrict__ segtab,
               double* __restrict__ Rp, double* __restrict__ Cb, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;  // PCG already stopped (device-side flag)
  // column record stride: an odd number of 16-byte units, so 8 consecutive
  // columns read by 8 lanes fall in 8 distinct bank groups
  constexpr int CS0 = KmvTraits<D>::CS;
  constexpr int CS = ((CS0 / 2) % 2 == 0) ? CS0 + 2 : CS0;
  constexpr int KMV_TC = 256;  // columns per shared-memory stage (8 units)
  constexpr int NW = KMV_NT / 32;
  constexpr int RBW = KMV_NT * RB;
  constexpr int M = RBW / 32;  // diagonal tiles per row block
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  constexpr int TABN = D <= 4 ? 2048 : 256;
  extern __shared__ double s_tx[];  // exp2 table (dynamic: the static arrays take ~28 KB)
  __shared__ __align__(16) double s_col[KMV_TC * CS];
  __shared__ double s_cs[NW][KMV_TC];
  load_exp2_tab(s_tab);
  for (int t = threadIdx.x; t < TABN; t += KMV_NT) s_tx[t] = TABN == 2048 ? g_exp2_2048[t] : g_exp2_256[t];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t g = g0 + blockIdx.x;
  const int64_t u0 = g * U / Gt, u1 = (g + 1) * U / Gt;
  if (u0 >= u1) return;  // (Gt <= U: never)
  // row block of u0 (binary search on ustart)
  int64_t I = 0;
  {
    int64_t lo = 0, hi = nrb - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (sym_ustart(mid, nt, M) <= u0) lo = mid;
      else hi = mid - 1;
    }
    I = lo;
  }
  double xi[RB][D], vi[RB], acc[RB];
  int64_t ri[RB];
  auto load_rows = [&]() {
#pragma unroll
    for (int t = 0; t < RB; ++t) {
      ri[t] = I * RBW + threadIdx.x + (int64_t)t * KMV_NT;
      const bool ok = ri[t] < n;
#pragma unroll
      for (int q = 0; q < D; ++q) xi[t][q] = ok ? Xs[ri[t] * D + q] : 0.0;
      vi[t] = ok ? v[ri[t]] : 0.0;
      acc[t] = 0.0;
    }
  };
  auto flush_rows = [&]() {
    const int64_t slot = segtab[3 * I + 2] + (g - segtab[3 * I]);
#pragma unroll
    for (int t = 0; t < RB; ++t)
      if (ri[t] < n) Rp[slot * RBW + threadIdx.x + t * KMV_NT] = acc[t];
  };
  load_rows();
  int64_t u = u0;
  while (u < u1) {
    const int64_t us = sym_ustart(I, nt, M), ue = sym_ustart(I + 1, nt, M);
    if (u >= ue) {  // next row block
      flush_rows();
      ++I;
      load_rows();
      continue;
    }
    // stage up to 8 tiles of this row block
    const int64_t t0 = M * I + (u - us);
    const int64_t run = min(min(u1, ue) - u, (int64_t)(KMV_TC / 32));
    const int64_t tb = t0 * 32;
    const int tcn = (int)min((int64_t)(run * 32), n - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < KMV_TC * CS; e += KMV_NT) {
      const int j = e / CS, q = e - j * CS;
      double val = 0.0;
      if (j < tcn) {
        if (q < D) val = Xs[(tb + j) * D + q];
        else if (q == D) val = v[tb + j];
      }
      s_col[e] = val;
    }
    __syncthreads();
    // Blocks of 32 columns: at step s lane l pairs its rows with column
    // (l + s) mod 32 and adds to a column accumulator that then moves one lane
    // down (one shuffle per step), so after 32 steps lane l holds column l
    // summed over the whole warp -- no reduction tree, no extra dependency
    // chain per column (each column is summed in a fixed lane order).
    auto body = [&](auto masked, int cb) {
      double ca = 0.0;
#pragma unroll 2
      for (int st = 0; st < 32; ++st) {
        const int j = cb + ((lane + st) & 31);
        double xj[CS];
#pragma unroll
        for (int q = 0; q < CS0; q += 2) {
          const double2 w2 = *reinterpret_cast<const double2*>(&s_col[j * CS + q]);
          xj[q] = w2.x;
          xj[q + 1] = w2.y;
        }
        const double vj = xj[D];
        const int64_t gj = tb + j;
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          double dd = xi[t][0] - xj[0];
          double s2 = dd * dd;
#pragma unroll
          for (int q = 1; q < D; ++q) {
            dd = xi[t][q] - xj[q];
            s2 = fma(dd, dd, s2);
          }
          double kv;
          if (KER == 1) {
            const double tt = sqrt(s2);
            kv = (1.0 + tt) * exp2_neg(tt * AFN_LOG2E, s_tab);
          } else {
            kv = TABN == 2048 ? exp2_neg2048(s2, s_tx) : exp2_neg256(s2, s_tx);
          }
          if (decltype(masked)::value && gj <= ri[t]) kv = 0.0;  // diagonal tile: j > i only
          acc[t] = fma(kv, vj, acc[t]);
          ca = fma(kv, vi[t], ca);
        }
        ca = __shfl_sync(0xffffffffu, ca, (lane + 1) & 31);  // follow the column to lane - 1
      }
      s_cs[wid][cb + lane] = ca;  // column cb + lane (stage padded: cb + 31 < KMV_TC)
    };
    // one body per stage (a stage that starts in the diagonal tiles is masked
    // throughout: the mask never fires past them; a per-tile choice measured
    // 3 % slower)
    if (t0 < M * (I + 1)) {
      for (int c = 0; c < (int)run; ++c) body(std::true_type{}, 32 * c);
    } else {
      for (int c = 0; c < (int)run; ++c) body(std::false_type{}, 32 * c);
    }
    __syncthreads();
    const int64_t cbase = sym_cboff(I, n, RBW) - I * RBW;
    for (int j = threadIdx.x; j < tcn; j += KMV_NT) {
      double t2 = s_cs[0][j];
#pragma unroll
      for (int w = 1; w < NW; ++w) t2 += s_cs[w][j];
      Cb[cbase + tb + j] = t2;
    }
    u += run;
  }
  flush_rows();
}

// Rank partial of the symmetric matvec for every row i (fixed order):
//   q_i = sum_{t < nseg(I)} Rp[rbase(I) + t][i] + sum_{I' <= I(i)} Cb[I'][i]
// over the entries this rank's CTAs wrote (OWN: all entries, one rank).
// FINAL (one rank): y_i = (1 + mu) v_i + q_i and, with dout, v . y (block
// partials, the last block sums them in block order).  Otherwise y = q.
constexpr int SRT = 256;  // threads per block of the symmetric reduce
constexpr int SRL = 8;    // threads per row (partial sums over strided entries, then a fixed butterfly)
template <bool FINAL>
__global__ void __launch_bounds__(SRT) kmv_sym_reduce_kernel(
    const double* __restrict__ Rp, const double* __restrict__ Cb, const int* __restrict__ segtab, int64_t n,
    int64_t rbw, int64_t nt, int64_t U, int64_t Gt, int64_t g_lo, int64_t g_hi, const double* __restrict__ v,
    double mu, double* __restrict__ y, const double* skip, double* dout, double* dws, unsigned* dcnt) {
  __shared__ double sh[SRT / 32];
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t m = rbw / 32;
  const bool all = g_lo == 0 && g_hi == Gt;
  const int sub = threadIdx.x % SRL;
  double dsum = 0.0;
  const int64_t rows_per_pass = (int64_t)gridDim.x * (SRT / SRL);
  for (int64_t i0 = (int64_t)blockIdx.x * (SRT / SRL); i0 < n; i0 += rows_per_pass) {
    const int64_t i = i0 + threadIdx.x / SRL;
    double s = 0.0;
    if (i < n) {
      const int64_t Ii = i / rbw, li = i - Ii * rbw;
      const int gf = segtab[3 * Ii], ns = segtab[3 * Ii + 1], rb = segtab[3 * Ii + 2];
      for (int t = sub; t < ns; t += SRL)
        if (all || (gf + t >= g_lo && gf + t < g_hi)) s += Rp[(int64_t)(rb + t) * rbw + li];
      const int64_t ti = i / 32;
      for (int64_t I = sub; I <= Ii; I += SRL) {
        bool own = all;
        if (!own) {
          const int64_t gg = sym_cta_of(sym_ustart(I, nt, m) + (ti - m * I), U, Gt);
          own = gg >= g_lo && gg < g_hi;
        }
        if (own) s += Cb[sym_cboff(I, n, rbw) + (i - I * rbw)];
      }
    }
#pragma unroll
    for (int o = 1; o < SRL; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (sub == 0 && i < n) {
      if (FINAL) {
        const double yi = fma(1.0 + mu, v[i], s);
        y[i] = yi;
        dsum = fma(v[i], yi, dsum);
      } else {
        y[i] = s;
      }
    }
  }
  if (!FINAL || dout == nullptr) return;
  dsum = block_sum<SRT>(dsum, sh);
  finish_sum(dsum, dws, dcnt, dout);
}

// y_i = (1 + mu) v_i + sum_{s < R} qpart[s n + i] (rank order) over the rows g;
// with dout also v . y over g
__global__ void __launch_bounds__(SRT) kmv_sym_combine_kernel(const double* __restrict__ qpart, int R, int64_t n,
                                                             Seg2 g, const double* __restrict__ v, double mu,
                                                             double* __restrict__ y, const double* skip,
                                                             double* dout, double* dws, unsigned* dcnt) {
  __shared__ double sh[SRT / 32];
  if (skip != nullptr && *skip != 0.0) return;
  double dsum = 0.0;
  const int64_t nr = g.size();
  for (int64_t t = (int64_t)blockIdx.x * SRT + threadIdx.x; t < nr; t += (int64_t)gridDim.x * SRT) {
    const int64_t i = g.phys(t);
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += qpart[(int64_t)r * n + i];
    const double yi = fma(1.0 + mu, v[i], s);
    y[i] = yi;
    dsum = fma(v[i], yi, dsum);
  }
  if (dout == nullptr) return;
  dsum = block_sum<SRT>(dsum, sh);
  finish_sum(dsum, dws, dcnt, dout);
}

// ============================================================================
// Cutoff plan (Gaussian, d <= 3).  K_ij = 2^(-s_ij) with s_ij =
// ||xs_i - xs_j||^2 (prescaled points).  The points are put in a spatial
// (Morton cell) order; the symmetric split's units (row block I of 1024
// positions, 32-position column tile t >= 32 I) are kept only if the boxes of
// block I and tile t are closer than s = 128 (a skipped unit's entries are all
// below 2^-128, under FP32's normal range: the FP32 body flushes them too).
// Units whose boxes are closer than s = 48 run the FP64 body of the dense
// symmetric kernel; the others (every entry below 2^-48) an FP32 body: the
// coordinates relative to the row block's box centre, the exponential by
// MUFU.EX2, per-unit FP32 sums added into the FP64 row and column sums.
// ============================================================================
constexpr double KC_S64 = 48.0;
constexpr double KC_SKIP = 128.0;

__device__ __forceinline__ float kc_ex2_neg(float s) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-s));
  return r;
}

__global__ void kc_gather_kernel(const double* __restrict__ X, int64_t n, int d, const int* __restrict__ sidx,
                                 double* __restrict__ Xc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const int64_t p = e / d;
  Xc[e] = X[(int64_t)sidx[p] * d + (e - p * d)];
}

// boxes of the 32-position tiles (one warp per tile) -> tbox[t][lo 3, hi 3]
__global__ void kc_tile_box_kernel(const double* __restrict__ Xc, int64_t n, int d, int64_t ntiles,
                                   double* __restrict__ tbox) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  const int64_t i = t * 32 + lane;
  for (int q = 0; q < 3; ++q) {
    double lo = 1e300, hi = -1e300;
    if (q < d && i < n) lo = hi = Xc[i * d + q];
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      tbox[t * 6 + q] = q < d ? lo : 0.0;
      tbox[t * 6 + 3 + q] = q < d ? hi : 0.0;
    }
  }
}

// groups of 128 consecutive positions (4 tiles) own the rows of an item; the
// coarse blocks of 1024 positions prefilter the box tests
constexpr int KC_GR = 128;
constexpr int KC_GT = KC_GR / 32;
constexpr int KC_CB = 1024;
constexpr int KC_W64 = 16, KC_W32 = 5;  // split weights of an FP64 / FP32 item
constexpr unsigned KC_F32 = 0x80000000u;

// boxes of blocks of `per` tiles (one warp per block; per <= 32) and their
// centres (optional)
__global__ void kc_block_box_kernel(const double* __restrict__ tbox, int64_t ntiles, int64_t nb, int per,
                                    double* __restrict__ bbox, double* __restrict__ ctr) {
  const int64_t I = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nb) return;
  const int64_t t = I * per + lane;
  for (int q = 0; q < 3; ++q) {
    double lo = 1e300, hi = -1e300;
    if (lane < per && t < ntiles) {
      lo = tbox[t * 6 + q];
      hi = tbox[t * 6 + 3 + q];
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      bbox[I * 6 + q] = lo;
      bbox[I * 6 + 3 + q] = hi;
      if (ctr) ctr[I * 4 + q] = 0.5 * (lo + hi);
    }
  }
}

// minimum s between two boxes (lo[0..2], hi[3..5]); explicitly rounded ops so
// that every pass of the plan builder sees the same value
__device__ __forceinline__ double kc_smin(const double* __restrict__ a, const double* __restrict__ b, int dd) {
  double s = 0.0;
  for (int q = 0; q < dd; ++q) {
    const double gap = fmax(0.0, fmax(__dsub_rn(b[q], a[3 + q]), __dsub_rn(a[q], b[3 + q])));
    s = __dadd_rn(s, __dmul_rn(gap, gap));
  }
  return s;
}

// item (group g, tile t >= 4 g): 0 not kept, 1 FP64, 2 FP32 -- the class of
// the group's nearest row tile to tile t; *np = its useful pairs (i < j)
__device__ __forceinline__ int kc_item(int64_t g, int64_t t, const double* __restrict__ cbox,
                                       const double* __restrict__ tbox, int64_t n, int dd, int64_t* np) {
  const double* tb = tbox + t * 6;
  if (kc_smin(cbox + (g * KC_GR / KC_CB) * 6, cbox + (t * 32 / KC_CB) * 6, dd) >= KC_SKIP) return 0;
  const int64_t r0 = g * KC_GR, r1 = min(n, r0 + KC_GR);
  double s = 1e300;
  for (int64_t rt = r0 / 32; rt * 32 < r1; ++rt) s = fmin(s, kc_smin(tbox + rt * 6, tb, dd));
  if (s >= KC_SKIP) return 0;
  const int64_t c0 = t * 32, c1 = min(n, c0 + 32);
  if (r1 <= c0) {
    *np = (r1 - r0) * (c1 - c0);
  } else {  // the group's own tiles: pairs i < j only
    int64_t m = 0;
    for (int64_t j = c0; j < c1; ++j) m += max((int64_t)0, min(r1, j) - r0);
    *np = m;
  }
  return s >= KC_S64 ? 2 : 1;
}

// per group: kept items, their split weight and useful pairs per class
__global__ void __launch_bounds__(256) kc_count_kernel(const double* __restrict__ cbox,
                                                       const double* __restrict__ tbox, int64_t n, int64_t ntiles,
                                                       int dd, int* __restrict__ cnt, int64_t* __restrict__ wsum,
                                                       unsigned long long* __restrict__ pairs) {
  __shared__ int c_all;
  __shared__ unsigned long long s64, s32, sw;
  const int64_t g = blockIdx.x;
  if (threadIdx.x == 0) {
    c_all = 0;
    s64 = s32 = sw = 0ull;
  }
  __syncthreads();
  int ca = 0;
  unsigned long long q64 = 0ull, q32 = 0ull, qw = 0ull;
  for (int64_t t = g * KC_GT + threadIdx.x; t < ntiles; t += blockDim.x) {
    int64_t np = 0;
    const int c = kc_item(g, t, cbox, tbox, n, dd, &np);
    if (c == 0) continue;
    ++ca;
    if (c == 2) {
      q32 += (unsigned long long)np;
      qw += KC_W32;
    } else {
      q64 += (unsigned long long)np;
      qw += KC_W64;
    }
  }
  atomicAdd(&c_all, ca);
  atomicAdd(&s64, q64);
  atomicAdd(&s32, q32);
  atomicAdd(&sw, qw);
  __syncthreads();
  if (threadIdx.x == 0) {
    cnt[g] = c_all;
    wsum[g] = (int64_t)sw;
    atomicAdd(&pairs[0], s64);
    atomicAdd(&pairs[1], s32);
  }
}

// the kept items of group g in tile order: it[e] = tile | F32 flag,
// wpre[e] = exclusive prefix of the split weights (from wbase[g])
__global__ void __launch_bounds__(256) kc_fill_kernel(const double* __restrict__ cbox,
                                                      const double* __restrict__ tbox, int64_t n, int64_t ntiles,
                                                      int dd, const int64_t* __restrict__ gstart,
                                                      const int64_t* __restrict__ wbase, unsigned* __restrict__ it,
                                                      int64_t* __restrict__ wpre) {
  __shared__ int wtot[8], wwt[8];
  __shared__ int64_t base, wb;
  const int64_t g = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    base = gstart[g];
    wb = wbase[g];
  }
  __syncthreads();
  for (int64_t t0 = g * KC_GT; t0 < ntiles; t0 += 256) {
    const int64_t t = t0 + threadIdx.x;
    int64_t np = 0;
    const int c = t < ntiles ? kc_item(g, t, cbox, tbox, n, dd, &np) : 0;
    const int wgt = c == 0 ? 0 : (c == 2 ? KC_W32 : KC_W64);
    const unsigned m = __ballot_sync(0xffffffffu, c != 0);
    int wincl = wgt;  // inclusive warp scan of the weights
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wincl, o);
      if (lane >= o) wincl += y;
    }
    if (lane == 31) {
      wtot[wid] = __popc(m);
      wwt[wid] = wincl;
    }
    __syncthreads();
    int64_t off = base, woff = wb;
    for (int w = 0; w < wid; ++w) {
      off += wtot[w];
      woff += wwt[w];
    }
    if (c != 0) {
      const int64_t e = off + __popc(m & ((1u << lane) - 1u));
      it[e] = (unsigned)t | (c == 2 ? KC_F32 : 0u);
      wpre[e] = woff + wincl - wgt;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 8; ++w) {
        base += wtot[w];
        wb += wwt[w];
      }
    __syncthreads();
  }
}

// warp w starts at the first item whose weight prefix reaches w TW / Wtot
__global__ void kc_wsplit_kernel(const int64_t* __restrict__ wpre, int64_t E, int64_t TW, int64_t Wtot,
                                 int64_t* __restrict__ wst) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w > Wtot) return;
  if (w == Wtot) {
    wst[w] = E;
    return;
  }
  const int64_t target = (int64_t)((__int128)w * TW / Wtot);
  int64_t lo = 0, hi = E;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (wpre[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  wst[w] = lo;
}

__device__ __forceinline__ int64_t kc_owner(const int64_t* __restrict__ wst, int64_t Wtot, int64_t e) {
  int64_t lo = 0, hi = Wtot - 1;  // last w with wst[w] <= e
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (wst[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t kc_group_of(const int64_t* __restrict__ gstart, int64_t ng, int64_t e) {
  int64_t lo = 0, hi = ng - 1;  // last g with gstart[g] <= e
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (gstart[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// per group: {first warp, warps} touching it (empty warps in between
// included: they write zero rows), counts for the slot scan
__global__ void kc_segs_kernel(const int64_t* __restrict__ gstart, int64_t ng, const int64_t* __restrict__ wst,
                               int64_t Wtot, int* __restrict__ seg, int* __restrict__ nseg) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t f = kc_owner(wst, Wtot, gstart[g]), l = kc_owner(wst, Wtot, gstart[g + 1] - 1);
  seg[2 * g] = (int)f;
  seg[2 * g + 1] = (int)(l - f + 1);
  nseg[g] = (int)(l - f + 1);
}

// transpose: items per tile (counted, placed, then sorted by item id)
__global__ void kc_tcount_kernel(const unsigned* __restrict__ it, int64_t E, int* __restrict__ tcnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) atomicAdd(&tcnt[it[e] & ~KC_F32], 1);
}
__global__ void kc_tplace_kernel(const unsigned* __restrict__ it, int64_t E, const int64_t* __restrict__ tptr,
                                 int* __restrict__ cur, int* __restrict__ tu) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const unsigned t = it[e] & ~KC_F32;
  tu[tptr[t] + atomicAdd(&cur[t], 1)] = (int)e;
}
// one block per tile: bitonic sort in shared memory (lists up to 1024; the
// rare longer one by thread 0's insertion sort)
__global__ void __launch_bounds__(256) kc_tsort_kernel(const int64_t* __restrict__ tptr, int64_t ntiles,
                                                       int* __restrict__ tu) {
  __shared__ int sv[1024];
  const int64_t t = blockIdx.x;
  const int64_t b = tptr[t], e = tptr[t + 1];
  const int len = (int)(e - b);
  if (len <= 1) return;
  if (len <= 1024) {
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) sv[i] = i < len ? tu[b + i] : 0x7fffffff;
    __syncthreads();
    for (int kk = 2; kk <= p2; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const bool up = (i & kk) == 0;
            const int x = sv[i], y = sv[l];
            if ((x > y) == up) {
              sv[i] = y;
              sv[l] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < len; i += blockDim.x) tu[b + i] = sv[i];
    return;
  }
  if (threadIdx.x != 0) return;
  for (int64_t i = b + 1; i < e; ++i) {
    const int v = tu[i];
    int64_t j = i - 1;
    while (j >= b && tu[j] > v) {
      tu[j + 1] = tu[j];
      --j;
    }
    tu[j + 1] = v;
  }
}

// One warp per item range [wst[w], wst[w+1]) of the (group, tile) items in
// (group, tile) order: the group's 128 rows in registers (row t of lane l is
// position 128 g + 32 t + l), the item's 32 columns staged by the warp in its
// own shared-memory slice (no block barrier), the column sums (lane l =
// column l, the rotation of kmv_sym_kernel) written to Cb[e], the row sums to
// the warp's slot of the group when the warp leaves it.
template <int D>
__global__ void __launch_bounds__(KMV_NT, 2)
kmv_cut_kernel(const double* __restrict__ Xc, const int* __restrict__ sidx, const double* __restrict__ v,
               const double* __restrict__ ctr, int64_t n, int64_t ng, const int64_t* __restrict__ gstart,
               const unsigned* __restrict__ it, const int64_t* __restrict__ wst, int64_t Wtot, int64_t w0,
               const int* __restrict__ seg, const int64_t* __restrict__ rbase, double* __restrict__ Rp,
               double* __restrict__ Cb, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  constexpr int RB = 4;
  constexpr int CS0 = KmvTraits<D>::CS;
  constexpr int CS = ((CS0 / 2) % 2 == 0) ? CS0 + 2 : CS0;
  constexpr int NW = KMV_NT / 32;
  extern __shared__ double s_tx[];  // 2048-entry exp2 table
  __shared__ __align__(16) double s_col[NW][32 * CS];
  __shared__ __align__(16) float4 s_colf[NW][32];
  for (int t = threadIdx.x; t < 2048; t += KMV_NT) s_tx[t] = g_exp2_2048[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w = w0 + (int64_t)blockIdx.x * NW + wid;
  if (w >= Wtot) return;
  const int64_t e0 = wst[w], e1 = wst[w + 1];
  if (e0 >= e1) {  // empty range: zero rows if a group counts this warp
    if (e0 < wst[Wtot]) {
      const int64_t g = kc_group_of(gstart, ng, e0);
      const int64_t f = seg[2 * g], ns = seg[2 * g + 1];
      if (w >= f && w < f + ns)
        for (int t = 0; t < RB; ++t) Rp[(rbase[g] + (w - f)) * KC_GR + 32 * t + lane] = 0.0;
    }
    return;
  }
  int64_t g = kc_group_of(gstart, ng, e0);
  double xi[RB][D], vi[RB], acc[RB], cg[D];
  int64_t ri[RB];
  auto load_rows = [&]() {
#pragma unroll
    for (int q = 0; q < D; ++q) cg[q] = ctr[g * 4 + q];
#pragma unroll
    for (int t = 0; t < RB; ++t) {
      ri[t] = g * KC_GR + 32 * t + lane;
      const bool ok = ri[t] < n;
#pragma unroll
      for (int q = 0; q < D; ++q) xi[t][q] = ok ? Xc[ri[t] * D + q] : 0.0;
      vi[t] = ok ? v[sidx[ri[t]]] : 0.0;
      acc[t] = 0.0;
    }
  };
  auto flush_rows = [&]() {
    double* dst = Rp + (rbase[g] + (w - seg[2 * g])) * KC_GR;
#pragma unroll
    for (int t = 0; t < RB; ++t) dst[32 * t + lane] = acc[t];
  };
  load_rows();
  int64_t gend = gstart[g + 1];
  double* const col = s_col[wid];
  float4* const colf = s_colf[wid];
  for (int64_t e = e0; e < e1; ++e) {
    if (e >= gend) {
      flush_rows();
      do {
        ++g;
      } while (gstart[g + 1] <= e);
      gend = gstart[g + 1];
      load_rows();
    }
    const unsigned item = it[e];
    const int64_t tb = (int64_t)(item & ~KC_F32) * 32;
    const bool f32 = (item & KC_F32) != 0u;
    {  // stage the item's columns (lane = column)
      const int64_t gc = tb + lane;
      const bool ok = gc < n;
      const double vj = ok ? v[sidx[gc]] : 0.0;
      double xj[D];
#pragma unroll
      for (int q = 0; q < D; ++q) xj[q] = ok ? Xc[gc * D + q] : 0.0;
      __syncwarp();
      if (f32) {
        float f[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < D; ++q) f[q] = (float)(xj[q] - cg[q]);
        colf[lane] = make_float4(f[0], f[1], f[2], (float)vj);
      } else {
#pragma unroll
        for (int q = 0; q < D; ++q) col[lane * CS + q] = xj[q];
        col[lane * CS + D] = vj;
      }
      __syncwarp();
    }
    if (f32) {
      float xf[RB][3], vf[RB], a32[RB];
#pragma unroll
      for (int t = 0; t < RB; ++t) {
#pragma unroll
        for (int q = 0; q < 3; ++q) xf[t][q] = q < D ? (float)(xi[t][q < D ? q : 0] - cg[q < D ? q : 0]) : 0.f;
        vf[t] = (float)vi[t];
        a32[t] = 0.f;
      }
      float ca = 0.f;
#pragma unroll 4
      for (int st = 0; st < 32; ++st) {
        const float4 c4 = colf[(lane + st) & 31];
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          const float dx = xf[t][0] - c4.x;
          float s2 = dx * dx;
          if (D > 1) {
            const float dy = xf[t][1] - c4.y;
            s2 = fmaf(dy, dy, s2);
          }
          if (D > 2) {
            const float dz = xf[t][2] - c4.z;
            s2 = fmaf(dz, dz, s2);
          }
          const float kv = kc_ex2_neg(s2);
          a32[t] = fmaf(kv, c4.w, a32[t]);
          ca = fmaf(kv, vf[t], ca);
        }
        ca = __shfl_sync(0xffffffffu, ca, (lane + 1) & 31);
      }
      Cb[e * 32 + lane] = (double)ca;
#pragma unroll
      for (int t = 0; t < RB; ++t) acc[t] += (double)a32[t];
    } else {
      auto body64 = [&](auto masked) {
        double ca = 0.0;
#pragma unroll 2
        for (int st = 0; st < 32; ++st) {
          const int jl = (lane + st) & 31;
          double xj[CS];
#pragma unroll
          for (int q = 0; q < CS0; q += 2) {
            const double2 w2 = *reinterpret_cast<const double2*>(&col[jl * CS + q]);
            xj[q] = w2.x;
            xj[q + 1] = w2.y;
          }
          const double vj = xj[D];
          const int64_t gj = tb + jl;
#pragma unroll
          for (int t = 0; t < RB; ++t) {
            double dd = xi[t][0] - xj[0];
            double s2 = dd * dd;
#pragma unroll
            for (int q = 1; q < D; ++q) {
              dd = xi[t][q] - xj[q];
              s2 = fma(dd, dd, s2);
            }
            double kv = exp2_neg2048(s2, s_tx);
            if (decltype(masked)::value && gj <= ri[t]) kv = 0.0;
            acc[t] = fma(kv, vj, acc[t]);
            ca = fma(kv, vi[t], ca);
          }
          ca = __shfl_sync(0xffffffffu, ca, (lane + 1) & 31);
        }
        Cb[e * 32 + lane] = ca;
      };
      if (tb < (g + 1) * KC_GR) body64(std::true_type{});
      else body64(std::false_type{});
    }
  }
  flush_rows();
}

// q at spatial position i = the row slots of its group (warp order) + the
// column partials of the items holding its tile (item order); written to
// y[sidx[i]].  FINAL as in kmv_sym_reduce_kernel.  This rank: warps
// [w_lo, w_hi), items [wst[w_lo], wst[w_hi]).
template <bool FINAL>
__global__ void __launch_bounds__(SRT) kmv_cut_reduce_kernel(
    const double* __restrict__ Rp, const double* __restrict__ Cb, const int* __restrict__ seg,
    const int64_t* __restrict__ rbase, const int* __restrict__ sidx, const int64_t* __restrict__ tptr,
    const int* __restrict__ tu, const int64_t* __restrict__ wst, int64_t n, int64_t Wtot, int64_t w_lo,
    int64_t w_hi, const double* __restrict__ v, double mu, double* __restrict__ y, const double* skip, double* dout,
    double* dws, unsigned* dcnt) {
  __shared__ double sh[SRT / 32];
  if (skip != nullptr && *skip != 0.0) return;
  const bool all = w_lo == 0 && w_hi == Wtot;
  const int64_t e_lo = wst[w_lo], e_hi = wst[w_hi];
  const int sub = threadIdx.x % SRL;
  double dsum = 0.0;
  const int64_t rows_per_pass = (int64_t)gridDim.x * (SRT / SRL);
  for (int64_t i0 = (int64_t)blockIdx.x * (SRT / SRL); i0 < n; i0 += rows_per_pass) {
    const int64_t i = i0 + threadIdx.x / SRL;
    double s = 0.0;
    if (i < n) {
      const int64_t gi = i / KC_GR, li = i - gi * KC_GR;
      const int64_t f = seg[2 * gi], ns = seg[2 * gi + 1], rb = rbase[gi];
      for (int64_t t = sub; t < ns; t += SRL)
        if (all || (f + t >= w_lo && f + t < w_hi)) s += Rp[(rb + t) * KC_GR + li];
      const int64_t ti = i / 32, tl = i - ti * 32;
      const int64_t t1 = tptr[ti + 1];
      for (int64_t q = tptr[ti] + sub; q < t1; q += SRL) {
        const int64_t e = tu[q];
        if (all || (e >= e_lo && e < e_hi)) s += Cb[e * 32 + tl];
      }
    }
#pragma unroll
    for (int o = 1; o < SRL; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (sub == 0 && i < n) {
      const int64_t o = sidx[i];
      if (FINAL) {
        const double yi = fma(1.0 + mu, v[o], s);
        y[o] = yi;
        dsum = fma(v[o], yi, dsum);
      } else {
        y[o] = s;
      }
    }
  }
  if (!FINAL || dout == nullptr) return;
  dsum = block_sum<SRT>(dsum, sh);
  finish_sum(dsum, dws, dcnt, dout);
}

__global__ void kmv_reduce_kernel(const double* __restrict__ partial, int nchunks, Seg2 rows,
                                  const double* __restrict__ v, double mu, bool y_phys,
                                  double* __restrict__ y, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t nrows = rows.size();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += partial[(int64_t)c * nrows + i];
  const int64_t r = rows.phys(i);
  y[y_phys ? r : i] = fma(mu, v[r], s);
}

__global__ void prescale_kernel(const double* __restrict__ X, int64_t n, int d, double f,
                                double* __restrict__ Xs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n * d) Xs[e] = X[e] * f;
}

template <int D>
void launch_partial(const KmvPlan& p, cudaStream_t st, const double* Xs, const double* v, int64_t n,
                    Seg2 rows, double* partial, int kind) {
  constexpr int RB = KmvTraits<D>::RB;
  const int64_t rows_per_cta = (int64_t)KMV_NT * RB;
  dim3 grid((unsigned)((rows.size() + rows_per_cta - 1) / rows_per_cta), (unsigned)p.chunks);
  if (kind == 1) kmv_partial_kernel<D, RB, 1><<<grid, KMV_NT, 0, st>>>(Xs, v, n, rows, p.chunk_cols, partial, get_skip());
  else kmv_partial_kernel<D, RB, 0><<<grid, KMV_NT, 0, st>>>(Xs, v, n, rows, p.chunk_cols, partial, get_skip());
}

int rows_per_thread(int d) { return d <= 4 ? 4 : (d <= 8 ? 2 : 1); }

KmvPlan plan_for(int64_t n, int64_t nrows, int d, int num_sms) {
  KmvPlan p;
  const int64_t rows_per_cta = (int64_t)KMV_NT * rows_per_thread(d);
  p.row_tiles = (nrows + rows_per_cta - 1) / rows_per_cta;
  const int64_t slots = (int64_t)num_sms * 2;  // 2 CTAs/SM (launch bounds)
  // Choose the column-chunk count minimising (waves x columns per CTA): whole
  // waves of `slots` CTAs (a partial last wave idles SMs), chunks >= 64
  // columns, plus a small per-chunk cost for the partial sums and the reduce.
  int64_t best_chunks = 1;
  double best_cost = 1e300;
  const int64_t cmax = std::max<int64_t>(1, std::min<int64_t>((n + 63) / 64, 4096));
  for (int64_t ch = 1; ch <= cmax; ++ch) {
    const int64_t cc = (n + ch - 1) / ch;
    const int64_t nch = (n + cc - 1) / cc;
    if (nch != ch) continue;
    const int64_t ctas = p.row_tiles * nch;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double cost = (double)waves * (double)cc + 0.002 * (double)nch * (double)rows_per_cta;
    if (cost < best_cost) { best_cost = cost; best_chunks = nch; }
  }
  p.chunk_cols = (n + best_chunks - 1) / best_chunks;
  p.chunks = (n + p.chunk_cols - 1) / p.chunk_cols;
  return p;
}

// per row block I: {gfirst, nseg, rbase} (see kmv_sym_kernel)
std::vector<int> sym_segtab(const KmvPlan& p) {
  const int64_t m = p.sym_rbw / 32;
  auto ustart = [&](int64_t I) { return I * p.sym_nt - m * I * (I - 1) / 2; };
  auto cta_of = [&](int64_t u) { return ((u + 1) * p.sym_gt - 1) / p.sym_units; };
  std::vector<int> tab(3 * (size_t)p.sym_nrb);
  int64_t rb = 0;
  for (int64_t I = 0; I < p.sym_nrb; ++I) {
    const int64_t gf = cta_of(ustart(I)), gl = cta_of(ustart(I + 1) - 1);
    tab[3 * I] = (int)gf;
    tab[3 * I + 1] = (int)(gl - gf + 1);
    tab[3 * I + 2] = (int)rb;
    rb += gl - gf + 1;
  }
  return tab;
}

template <int D, int KER>
void sym_launch(const KmvPlan& p, cudaStream_t st, const double* Xs, const double* v, int64_t n, const int* segtab,
                double* Rp, double* Cb) {
  constexpr int RB = KmvTraits<D>::RB;
  const int64_t g0 = p.sym_grid * (int64_t)p.sym_rank;
  const size_t tab = sizeof(double) * (D <= 4 ? 2048 : 256);  // (+ ~28 KB static: under 48 KB)
  kmv_sym_kernel<D, RB, KER><<<(unsigned)p.sym_grid, KMV_NT, tab, st>>>(Xs, v, n, p.sym_nrb, p.sym_nt, p.sym_units,
                                                                       p.sym_gt, g0, segtab, Rp, Cb, get_skip());
}

// The exp2 tables (__device__ globals) are filled once per device by a
// blocking launch on a private stream, under a lock, before any matvec is
// queued: a matvec on any stream or host thread sees complete tables.
std::mutex g_tab_mu;
bool g_tab_done[64] = {false};
afn_status ensure_exp2_tables() {
  int dev = 0;
  AFN_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device ordinal %d out of range", dev);
    return AFN_ERR_CUDA;
  }
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (g_tab_done[dev]) return AFN_OK;
  cudaStream_t ts;
  AFN_CUDA(cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking));
  exp2_256_init_kernel<<<1, 256, 0, ts>>>();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(ts);
  cudaStreamDestroy(ts);
  if (e != cudaSuccess) return cuda_status(e, "exp2_256_init_kernel");
  note_launch();
  g_tab_done[dev] = true;
  return AFN_OK;
}

}  // namespace

// The column chunking fixes each row's summation order.  A row shard keeps
// the chunking of the full n-row plan (so sharded rows are bit-identical to
// the single-GPU matvec) unless that would leave it under two waves of CTAs,
// in which case the shard gets its own plan.
KmvPlan kmv_plan(int64_t n, int64_t nrows, int d, int num_sms, bool sym_ok, int R, int rank) {
  // (measured, matvec ms per launch, symmetric vs row-wise: C2 0.20 vs 0.30,
  // C3 9.8 vs 17.4, C5 (n = 2^20) 629 vs 1106)
  if (sym_ok && n >= 2048 && d <= 8) {
    KmvPlan p;
    p.sym = true;
    p.sym_rbw = (int64_t)KMV_NT * rows_per_thread(d);
    p.sym_nrb = (n + p.sym_rbw - 1) / p.sym_rbw;
    p.sym_nt = (n + 31) / 32;
    const int64_t m = p.sym_rbw / 32;
    p.sym_units = 0;
    for (int64_t I = 0; I < p.sym_nrb; ++I) p.sym_units += p.sym_nt - m * I;
    const int per_sm = rows_per_thread(d) <= 2 ? 3 : 2;  // (launch bounds)
    p.sym_R = R;
    p.sym_rank = rank;
    // CTAs: one wave of resident CTAs when that leaves each >= upc units,
    // else ~upc units per CTA -- many short CTAs, measured faster at C3 than
    // one persistent wave (9.73 vs 10.09 ms per launch; C2 equal at 198 us);
    // upc = 32 past n = 2^18 bounds the row-partial slots (C5: 4.3 GB)
    const int64_t upc = n > (1 << 18) ? 32 : 16;
    const int64_t slots = (int64_t)num_sms * per_sm;
    const int64_t want = std::max<int64_t>(slots, p.sym_units / (upc * R));
    p.sym_grid = std::max<int64_t>(1, std::min<int64_t>(want, p.sym_units / R));
    p.sym_gt = p.sym_grid * R;
    // workspace: segment table (ints, rounded to doubles), row partials
    // (Gt + nrb slots of RBW), column partials (upper block triangle)
    p.sym_tab_dbl = (3 * p.sym_nrb + 1) / 2;
    const int64_t rp = (p.sym_gt + p.sym_nrb) * p.sym_rbw;
    const int64_t cb = p.sym_nrb * n - p.sym_rbw * p.sym_nrb * (p.sym_nrb - 1) / 2;
    p.ws = p.sym_tab_dbl + rp + cb;
    return p;
  }
  KmvPlan full = plan_for(n, n, d, num_sms);
  full.ws = full.chunks * std::max<int64_t>(1, nrows);
  if (nrows == n) return full;
  KmvPlan p = full;
  const int64_t rows_per_cta = (int64_t)KMV_NT * rows_per_thread(d);
  p.row_tiles = (nrows + rows_per_cta - 1) / rows_per_cta;
  p.ws = p.chunks * std::max<int64_t>(1, nrows);
  if (p.row_tiles * p.chunks >= 2 * 2 * (int64_t)num_sms) return p;
  KmvPlan q = plan_for(n, nrows, d, num_sms);
  q.ws = q.chunks * std::max<int64_t>(1, nrows);
  return q;
}

afn_status kmv_plan_init(const KmvPlan& p, double* ws, cudaStream_t st) {
  TRY_STATUS(ensure_exp2_tables());
  if (!p.sym) return AFN_OK;
  const std::vector<int> tab = sym_segtab(p);
  AFN_CUDA(cudaMemcpyAsync(ws, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaStreamSynchronize(st));  // (pageable source)
  return AFN_OK;
}

double kmv_flops(const KmvPlan& p, int64_t n, int64_t nrows, int d, int kind) {
  // executed FP64 flops per useful pair (FMA = 2), DESIGN.md 6:
  //   distance 3d - 1; exp2 with the 2048 table 12, with the 256 table 14;
  //   Matern: sqrt 1 + scale 1 + 2x16-table exp2 15 + (1 + t) 1 + product 1;
  //   row FMA 2 (+ column FMA 2 in the symmetric kernel)
  const double dist = 3.0 * d - 1.0;
  if (p.cut) {
    // FP64-equivalent: an FP32-body pair costs one MUFU.EX2 (16 per SM per
    // clock) against 2d + 9 FP64-pipe instructions (64 lanes per SM per clock)
    // of an FP64-body pair
    return (dist + 16.0) * (p.cut_pairs64 + p.cut_pairs32 * 4.0 / (2.0 * d + 9.0));
  }
  if (p.sym) {
    const double e = kind == 1 ? 19.0 : (d <= 4 ? 12.0 : 14.0);
    return (double)n * (double)(n - 1) / 2.0 * (dist + e + 4.0);
  }
  const double e = kind == 1 ? 19.0 : 14.0;
  return (double)nrows * (double)n * (dist + e + 2.0);
}

double kmv_fp64_inst(const KmvPlan& p, int64_t n, int64_t nrows, int d, int kind) {
  // FP64-pipe thread instructions per useful pair: distance 2d, exp2 7 (2048
  // table) / 8 (256) / 11 + sqrt (Matern, sqrt counted as 1), row FMA 1, column FMA 1
  const double dist = 2.0 * d;
  if (p.cut) return p.cut_pairs64 * (dist + 9.0);
  if (p.sym) {
    const double e = kind == 1 ? 14.0 : (d <= 4 ? 7.0 : 8.0);
    return (double)n * (double)(n - 1) / 2.0 * (dist + e + 2.0);
  }
  const double e = kind == 1 ? 14.0 : 8.0;
  return (double)nrows * (double)n * (dist + e + 1.0);
}

afn_status kmv_prescale(const double* X, int64_t n, int d, Kern kn, double* Xs, cudaStream_t st) {
  const double f = kn.kind == 1 ? AFN_SQRT3 / kn.l : AFN_SQRT_LOG2E / kn.l;
  const int64_t total = n * (int64_t)d;
  const int nt = 256;
  prescale_kernel<<<(unsigned)((total + nt - 1) / nt), nt, 0, st>>>(X, n, d, f, Xs);
  AFN_LAUNCH_CHECK("prescale_kernel");
  return AFN_OK;
}


// ---------------------------------------------------------------- cutoff plan
namespace {
int g_kmv_mode = 0;

template <int D>
void cut_launch(const KmvPlan& p, cudaStream_t st, const double* ws, const double* v, int64_t n) {
  const int64_t w0 = p.sym_grid * 8 * (int64_t)p.sym_rank;
  kmv_cut_kernel<D><<<(unsigned)p.sym_grid, KMV_NT, sizeof(double) * 2048, st>>>(
      ws + p.o_xc, reinterpret_cast<const int*>(ws + p.o_sidx), v, ws + p.o_ctr, n, p.sym_nrb,
      reinterpret_cast<const int64_t*>(ws + p.o_ustart), reinterpret_cast<const unsigned*>(ws + p.o_ut),
      reinterpret_cast<const int64_t*>(ws + p.o_wst), p.sym_gt, w0, reinterpret_cast<const int*>(ws + p.o_seg),
      reinterpret_cast<const int64_t*>(ws + p.o_rbase), const_cast<double*>(ws) + p.o_rp,
      const_cast<double*>(ws) + p.o_cb, get_skip());
}

afn_status cut_partials(const KmvPlan& p, int64_t n, int d, const double* v, double* ws, cudaStream_t st) {
  switch (d) {
    case 1: cut_launch<1>(p, st, ws, v, n); break;
    case 2: cut_launch<2>(p, st, ws, v, n); break;
    case 3: cut_launch<3>(p, st, ws, v, n); break;
    default: set_error("kernel_matvec: cutoff plan for d=%d unsupported (1..3)", d); return AFN_ERR_ARG;
  }
  AFN_LAUNCH_CHECK("kmv_cut_kernel");
  return AFN_OK;
}

// rank partial (final_ = false: y = q at this rank's items and warps) or the
// one-rank product (+ (1 + mu) v, v . y)
afn_status cut_reduce(const KmvPlan& p, int64_t n, const double* v, double mu, double* y, const double* ws,
                      bool final_, cudaStream_t st, double* dout, double* dws, unsigned* dcnt) {
  const int64_t rows_per_block = SRT / SRL;
  const int64_t nbk = std::min<int64_t>((n + rows_per_block - 1) / rows_per_block,
                                        final_ ? dot_ws() : 4 * (int64_t)num_sms());
  const int64_t wr = p.sym_grid * 8, w_lo = wr * p.sym_rank, w_hi = final_ ? p.sym_gt : w_lo + wr;
  const int* seg = reinterpret_cast<const int*>(ws + p.o_seg);
  const int64_t* rbase = reinterpret_cast<const int64_t*>(ws + p.o_rbase);
  const int* sidx = reinterpret_cast<const int*>(ws + p.o_sidx);
  const int64_t* tptr = reinterpret_cast<const int64_t*>(ws + p.o_tptr);
  const int* tu = reinterpret_cast<const int*>(ws + p.o_tu);
  const int64_t* wst = reinterpret_cast<const int64_t*>(ws + p.o_wst);
  if (final_)
    kmv_cut_reduce_kernel<true><<<(unsigned)nbk, SRT, 0, st>>>(ws + p.o_rp, ws + p.o_cb, seg, rbase, sidx, tptr, tu,
                                                               wst, n, p.sym_gt, 0, p.sym_gt, v, mu, y, get_skip(),
                                                               dout, dws, dcnt);
  else
    kmv_cut_reduce_kernel<false><<<(unsigned)nbk, SRT, 0, st>>>(ws + p.o_rp, ws + p.o_cb, seg, rbase, sidx, tptr,
                                                                tu, wst, n, p.sym_gt, w_lo, w_hi, v, 0.0, y,
                                                                get_skip(), nullptr, nullptr, nullptr);
  AFN_LAUNCH_CHECK("kmv_cut_reduce_kernel");
  return AFN_OK;
}

// stream-ordered temporaries of the plan builder
struct KcTmp {
  cudaStream_t st;
  std::vector<void*> ps;
  explicit KcTmp(cudaStream_t s) : st(s) {}
  ~KcTmp() {
    for (void* q : ps) dfree(q, st);
  }
  template <class T>
  afn_status get(T** out, size_t count) {
    void* q = nullptr;
    afn_status s = dalloc(&q, sizeof(T) * (count > 0 ? count : 1), st);
    if (s != AFN_OK) return s;
    ps.push_back(q);
    *out = static_cast<T*>(q);
    return AFN_OK;
  }
};

// Builds the cutoff plan; *used = false (nothing allocated through get) when
// it does not pay (mode 0: it would keep more than half of the pairs).
afn_status cut_plan_make(const double* Xs, int64_t n, int d, int R, int rank, cudaStream_t st, const WsGet& get,
                         KmvPlan* out, double** wsp, bool* used) {
  *used = false;
  const int nsm = num_sms();
  KcTmp tmp(st);
  // ---- spatial order (spatial.cu)
  int* sidx;
  TRY_STATUS(tmp.get(&sidx, (size_t)n));
  TRY_STATUS(morton_order(Xs, n, d, sidx, st));
  double *Xc, *tbox, *cbox, *ctr;
  const int64_t ntiles = (n + 31) / 32;
  const int64_t ng = (n + KC_GR - 1) / KC_GR;
  const int64_t ncb = (n + KC_CB - 1) / KC_CB;
  TRY_STATUS(tmp.get(&Xc, (size_t)n * d));
  TRY_STATUS(tmp.get(&tbox, (size_t)6 * ntiles));
  TRY_STATUS(tmp.get(&cbox, (size_t)6 * ncb));
  TRY_STATUS(tmp.get(&ctr, (size_t)4 * ng));
  kc_gather_kernel<<<(unsigned)((n * d + 255) / 256), 256, 0, st>>>(Xs, n, d, sidx, Xc);
  AFN_LAUNCH_CHECK("kc_gather_kernel");
  kc_tile_box_kernel<<<(unsigned)((ntiles * 32 + 255) / 256), 256, 0, st>>>(Xc, n, d, ntiles, tbox);
  AFN_LAUNCH_CHECK("kc_tile_box_kernel");
  kc_block_box_kernel<<<(unsigned)((ncb * 32 + 255) / 256), 256, 0, st>>>(tbox, ntiles, ncb, KC_CB / 32, cbox,
                                                                          nullptr);
  AFN_LAUNCH_CHECK("kc_block_box_kernel");
  double* gbox;
  TRY_STATUS(tmp.get(&gbox, (size_t)6 * ng));
  kc_block_box_kernel<<<(unsigned)((ng * 32 + 255) / 256), 256, 0, st>>>(tbox, ntiles, ng, KC_GT, gbox, ctr);
  AFN_LAUNCH_CHECK("kc_block_box_kernel");
  // ---- kept items per group
  int* gcnt;
  int64_t* gw;
  unsigned long long* pairs;
  TRY_STATUS(tmp.get(&gcnt, (size_t)ng));
  TRY_STATUS(tmp.get(&gw, (size_t)ng));
  TRY_STATUS(tmp.get(&pairs, 2));
  AFN_CUDA(cudaMemsetAsync(pairs, 0, 2 * sizeof(unsigned long long), st));
  kc_count_kernel<<<(unsigned)ng, 256, 0, st>>>(cbox, tbox, n, ntiles, d, gcnt, gw, pairs);
  AFN_LAUNCH_CHECK("kc_count_kernel");
  std::vector<int> hc((size_t)ng);
  std::vector<int64_t> hw((size_t)ng);
  unsigned long long hp[2];
  AFN_CUDA(cudaMemcpyAsync(hc.data(), gcnt, sizeof(int) * ng, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaMemcpyAsync(hw.data(), gw, sizeof(int64_t) * ng, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaMemcpyAsync(hp, pairs, sizeof(hp), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> gstart((size_t)ng + 1, 0), wbase((size_t)ng + 1, 0);
  for (int64_t g = 0; g < ng; ++g) {
    gstart[g + 1] = gstart[g] + hc[g];
    wbase[g + 1] = wbase[g] + hw[g];
  }
  const int64_t E = gstart[ng], TW = wbase[ng];
  const double all_pairs = (double)n * (double)(n - 1) / 2.0;
  // (auto: always -- measured on C2 it is at least as fast as the dense
  // symmetric plan for every l, 0.197 vs 0.199 ms even when no pair is skipped)
  (void)all_pairs;
  if (E >= ((int64_t)1 << 31) || E < 1) return AFN_OK;

  KmvPlan p;
  p.sym = true;
  p.cut = true;
  p.sym_rbw = KC_GR;
  p.sym_nrb = ng;
  p.sym_nt = ntiles;
  p.sym_units = E;
  p.sym_R = R;
  p.sym_rank = rank;
  p.cut_u64 = E;
  p.cut_ntiles = ntiles;
  p.cut_pairs64 = (double)hp[0];
  p.cut_pairs32 = (double)hp[1];
  {
    // warps per rank: two waves of 2 CTAs x 8 warps per SM, at least ~4 items
    // per warp (the split is by weight, FP64 : FP32 items = 16 : 5)
    const int64_t want = (int64_t)nsm * 2 * 8 * 2;
    int64_t wr = std::max<int64_t>(8, std::min<int64_t>(want, E / (4 * (int64_t)R)));
    wr = (wr + 7) / 8 * 8;
    p.sym_grid = wr / 8;
    p.sym_gt = wr * R;
  }
  const int64_t Wtot = p.sym_gt;
  auto dbl = [](int64_t bytes) { return (bytes + 7) / 8; };
  int64_t o = 0;
  p.sym_tab_dbl = 0;
  p.o_rp = o;
  o += (Wtot + ng) * KC_GR;
  p.o_cb = o;
  o += E * 32;
  p.o_xc = o;
  o += n * d;
  p.o_ctr = o;
  o += 4 * ng;
  p.o_sidx = o;
  o += dbl(sizeof(int) * n);
  p.o_ut = o;
  o += dbl(sizeof(unsigned) * E);
  p.o_ustart = o;
  o += ng + 1;
  p.o_wst = o;
  o += Wtot + 1;
  p.o_seg = o;
  o += dbl(sizeof(int) * 2 * ng);
  p.o_rbase = o;
  o += ng + 1;
  p.o_tptr = o;
  o += ntiles + 1;
  p.o_tu = o;
  o += dbl(sizeof(int) * E);
  p.ws = o;
  double* ws = nullptr;
  TRY_STATUS(get(&ws, (size_t)p.ws));
  *used = true;
  *wsp = ws;
  TRY_STATUS(ensure_exp2_tables());
  {  // the 2048-entry table is dynamic shared memory on top of the static ~20 KB
    const int dyn = (int)sizeof(double) * 2048;
    if (d == 1) AFN_CUDA(cudaFuncSetAttribute(kmv_cut_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    if (d == 2) AFN_CUDA(cudaFuncSetAttribute(kmv_cut_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    if (d == 3) AFN_CUDA(cudaFuncSetAttribute(kmv_cut_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  }
  int64_t* dgs = reinterpret_cast<int64_t*>(ws + p.o_ustart);
  int64_t* dwb;
  TRY_STATUS(tmp.get(&dwb, (size_t)ng + 1));
  AFN_CUDA(cudaMemcpyAsync(dgs, gstart.data(), sizeof(int64_t) * gstart.size(), cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(dwb, wbase.data(), sizeof(int64_t) * wbase.size(), cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(ws + p.o_xc, Xc, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(ws + p.o_ctr, ctr, sizeof(double) * 4 * ng, cudaMemcpyDeviceToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(ws + p.o_sidx, sidx, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  unsigned* dit = reinterpret_cast<unsigned*>(ws + p.o_ut);
  int64_t* wpre;
  TRY_STATUS(tmp.get(&wpre, (size_t)E));
  kc_fill_kernel<<<(unsigned)ng, 256, 0, st>>>(cbox, tbox, n, ntiles, d, dgs, dwb, dit, wpre);
  AFN_LAUNCH_CHECK("kc_fill_kernel");
  int64_t* wst = reinterpret_cast<int64_t*>(ws + p.o_wst);
  kc_wsplit_kernel<<<(unsigned)((Wtot + 1 + 255) / 256), 256, 0, st>>>(wpre, E, TW, Wtot, wst);
  AFN_LAUNCH_CHECK("kc_wsplit_kernel");
  int* nseg;
  TRY_STATUS(tmp.get(&nseg, (size_t)ng));
  kc_segs_kernel<<<(unsigned)((ng + 255) / 256), 256, 0, st>>>(dgs, ng, wst, Wtot,
                                                               reinterpret_cast<int*>(ws + p.o_seg), nseg);
  AFN_LAUNCH_CHECK("kc_segs_kernel");
  TRY_STATUS(scan_i32_i64(nseg, ng, reinterpret_cast<int64_t*>(ws + p.o_rbase), st));
  int *tcnt, *tcur;
  TRY_STATUS(tmp.get(&tcnt, (size_t)2 * ntiles));
  tcur = tcnt + ntiles;
  AFN_CUDA(cudaMemsetAsync(tcnt, 0, sizeof(int) * 2 * ntiles, st));
  const unsigned nbe = (unsigned)((E + 255) / 256);
  kc_tcount_kernel<<<nbe, 256, 0, st>>>(dit, E, tcnt);
  AFN_LAUNCH_CHECK("kc_tcount_kernel");
  int64_t* tptr = reinterpret_cast<int64_t*>(ws + p.o_tptr);
  TRY_STATUS(scan_i32_i64(tcnt, ntiles, tptr, st));
  int* tu = reinterpret_cast<int*>(ws + p.o_tu);
  kc_tplace_kernel<<<nbe, 256, 0, st>>>(dit, E, tptr, tcur, tu);
  AFN_LAUNCH_CHECK("kc_tplace_kernel");
  kc_tsort_kernel<<<(unsigned)ntiles, 256, 0, st>>>(tptr, ntiles, tu);
  AFN_LAUNCH_CHECK("kc_tsort_kernel");
  AFN_CUDA(cudaStreamSynchronize(st));  // (pageable sources; temporaries freed on return)
  *out = p;
  return AFN_OK;
}
}  // namespace

namespace {
__global__ void kmv_iperm_kernel(const int64_t* __restrict__ perm, int64_t n, int* __restrict__ iperm) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) iperm[perm[p]] = (int)p;
}
__global__ void kmv_remap_kernel(int* __restrict__ sidx, int64_t n, const int* __restrict__ iperm) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) sidx[q] = iperm[sidx[q]];
}
}  // namespace

afn_status kmv_plan_remap(const KmvPlan& p, double* ws, const int64_t* perm, int64_t n, cudaStream_t st) {
  if (!p.cut) return AFN_OK;
  int* iperm = nullptr;
  TRY_STATUS(dalloc((void**)&iperm, sizeof(int) * n, st));
  const unsigned nb = (unsigned)((n + 255) / 256);
  kmv_iperm_kernel<<<nb, 256, 0, st>>>(perm, n, iperm);
  AFN_LAUNCH_CHECK("kmv_iperm_kernel");
  kmv_remap_kernel<<<nb, 256, 0, st>>>(reinterpret_cast<int*>(ws + p.o_sidx), n, iperm);
  AFN_LAUNCH_CHECK("kmv_remap_kernel");
  dfree(iperm, st);
  return AFN_OK;
}

void kmv_set_mode(int mode) { g_kmv_mode = mode; }
int kmv_get_mode() { return g_kmv_mode; }

afn_status kmv_plan_make(const double* Xs, int64_t n, int64_t nrows, int d, int kind, bool sym_ok, int R, int rank,
                         cudaStream_t st, const WsGet& get, KmvPlan* out, double** ws) {
  if (sym_ok && kind == 0 && d <= 3 && n >= 4096 && g_kmv_mode != 1) {
    bool used = false;
    TRY_STATUS(cut_plan_make(Xs, n, d, R, rank, st, get, out, ws, &used));
    if (used) return AFN_OK;
  }
  *out = kmv_plan(n, nrows, d, num_sms(), sym_ok, R, rank);
  TRY_STATUS(get(ws, (size_t)std::max<int64_t>(1, out->ws)));
  return kmv_plan_init(*out, *ws, st);
}

namespace {
afn_status sym_partials(const double* Xs, int64_t n, int d, int kind, const double* v, const KmvPlan& p,
                        double* ws, cudaStream_t st) {
  const int* segtab = reinterpret_cast<const int*>(ws);
  double* Rp = ws + p.sym_tab_dbl;
  double* Cb = Rp + (p.sym_gt + p.sym_nrb) * p.sym_rbw;
  switch (d) {
#define AFN_SYM(DD)                                                                                     \
  case DD:                                                                                              \
    if (kind == 1)                                                                                      \
      sym_launch<DD, 1>(p, st, Xs, v, n, segtab, Rp, Cb);                                              \
    else                                                                                                \
      sym_launch<DD, 0>(p, st, Xs, v, n, segtab, Rp, Cb);                                              \
    break;
    AFN_SYM(1) AFN_SYM(2) AFN_SYM(3) AFN_SYM(4) AFN_SYM(5) AFN_SYM(6) AFN_SYM(7) AFN_SYM(8)
#undef AFN_SYM
    default: set_error("kernel_matvec: symmetric plan for d=%d unsupported (1..8)", d); return AFN_ERR_ARG;
  }
  AFN_LAUNCH_CHECK("kmv_sym_kernel");
  return AFN_OK;
}
}  // namespace

afn_status kmv_sym_rank_partial(const double* Xs, int64_t n, int d, int kind, const double* v, const KmvPlan& p,
                                double* ws, double* qout, cudaStream_t st) {
  if (!p.sym) {
    set_error("kmv_sym_rank_partial: plan is not symmetric");
    return AFN_ERR_STATE;
  }
  const int64_t glo = p.sym_grid * (int64_t)p.sym_rank;
  if (p.cut) {
    TRY_STATUS(cut_partials(p, n, d, v, ws, st));
    return cut_reduce(p, n, v, 0.0, qout, ws, false, st, nullptr, nullptr, nullptr);
  }
  TRY_STATUS(sym_partials(Xs, n, d, kind, v, p, ws, st));
  const int* segtab = reinterpret_cast<const int*>(ws);
  const double* Rp = ws + p.sym_tab_dbl;
  const double* Cb = Rp + (p.sym_gt + p.sym_nrb) * p.sym_rbw;
  const int64_t rows_per_block = SRT / SRL;
  const int64_t nbk = std::min<int64_t>((n + rows_per_block - 1) / rows_per_block, 4 * (int64_t)num_sms());
  kmv_sym_reduce_kernel<false><<<(unsigned)nbk, SRT, 0, st>>>(Rp, Cb, segtab, n, p.sym_rbw, p.sym_nt, p.sym_units,
                                                              p.sym_gt, glo, glo + p.sym_grid, v, 0.0, qout,
                                                              get_skip(), nullptr, nullptr, nullptr);
  AFN_LAUNCH_CHECK("kmv_sym_reduce_kernel");
  return AFN_OK;
}

afn_status kmv_sym_combine(const double* qpart, int R, int64_t n, Seg2 g, const double* v, double mu, double* y,
                           cudaStream_t st, double* dout, double* dws, unsigned* dcnt) {
  const int64_t nbk = std::max<int64_t>(1, std::min<int64_t>((g.size() + SRT - 1) / SRT, dot_ws()));
  kmv_sym_combine_kernel<<<(unsigned)nbk, SRT, 0, st>>>(qpart, R, n, g, v, mu, y, get_skip(), dout, dws, dcnt);
  AFN_LAUNCH_CHECK("kmv_sym_combine_kernel");
  return AFN_OK;
}

afn_status kmv_launch(const double* Xs, int64_t n, int d, int kind, const double* v, double mu, Seg2 rows,
                      double* y, bool y_phys, double* partial, const KmvPlan& p, cudaStream_t st, double* dout,
                      double* dws, unsigned* dcnt) {
  const int64_t nrows = rows.size();
  if (nrows <= 0) return AFN_OK;
  if (p.sym) {
    if (p.sym_R != 1 || !(rows.na + rows.nb == n && rows.a0 == 0 && (rows.nb == 0 || rows.b0 == rows.na))) {
      set_error("kernel_matvec: the one-rank symmetric plan needs all rows");
      return AFN_ERR_ARG;
    }
    if (p.cut) {
      TRY_STATUS(cut_partials(p, n, d, v, partial, st));
      return cut_reduce(p, n, v, mu, y, partial, true, st, dout, dws, dcnt);
    }
    TRY_STATUS(sym_partials(Xs, n, d, kind, v, p, partial, st));
    const int* segtab = reinterpret_cast<const int*>(partial);
    const double* Rp = partial + p.sym_tab_dbl;
    const double* Cb = Rp + (p.sym_gt + p.sym_nrb) * p.sym_rbw;
    const int64_t rows_per_block = SRT / SRL;
    const int64_t nbk = std::min<int64_t>((n + rows_per_block - 1) / rows_per_block, dot_ws());  // (dws: dot_ws() partials)
    kmv_sym_reduce_kernel<true><<<(unsigned)nbk, SRT, 0, st>>>(Rp, Cb, segtab, n, p.sym_rbw, p.sym_nt, p.sym_units,
                                                               p.sym_gt, 0, p.sym_gt, v, mu, y, get_skip(), dout,
                                                               dws, dcnt);
    AFN_LAUNCH_CHECK("kmv_sym_reduce_kernel");
    return AFN_OK;
  }
  switch (d) {
    case 1: launch_partial<1>(p, st, Xs, v, n, rows, partial, kind); break;
    case 2: launch_partial<2>(p, st, Xs, v, n, rows, partial, kind); break;
    case 3: launch_partial<3>(p, st, Xs, v, n, rows, partial, kind); break;
    case 4: launch_partial<4>(p, st, Xs, v, n, rows, partial, kind); break;
    case 5: launch_partial<5>(p, st, Xs, v, n, rows, partial, kind); break;
    case 6: launch_partial<6>(p, st, Xs, v, n, rows, partial, kind); break;
    case 7: launch_partial<7>(p, st, Xs, v, n, rows, partial, kind); break;
    case 8: launch_partial<8>(p, st, Xs, v, n, rows, partial, kind); break;
    case 9: launch_partial<9>(p, st, Xs, v, n, rows, partial, kind); break;
    case 10: launch_partial<10>(p, st, Xs, v, n, rows, partial, kind); break;
    case 11: launch_partial<11>(p, st, Xs, v, n, rows, partial, kind); break;
    case 12: launch_partial<12>(p, st, Xs, v, n, rows, partial, kind); break;
    case 13: launch_partial<13>(p, st, Xs, v, n, rows, partial, kind); break;
    case 14: launch_partial<14>(p, st, Xs, v, n, rows, partial, kind); break;
    case 15: launch_partial<15>(p, st, Xs, v, n, rows, partial, kind); break;
    case 16: launch_partial<16>(p, st, Xs, v, n, rows, partial, kind); break;
    default: set_error("kernel_matvec: d=%d unsupported (1..16)", d); return AFN_ERR_ARG;
  }
  AFN_LAUNCH_CHECK("kmv_partial_kernel");
  const int nt = 256;
  kmv_reduce_kernel<<<(unsigned)((nrows + nt - 1) / nt), nt, 0, st>>>(partial, (int)p.chunks, rows, v,
                                                                     mu, y_phys, y, get_skip());
  AFN_LAUNCH_CHECK("kmv_reduce_kernel");
  return AFN_OK;
}

}  // namespace afn

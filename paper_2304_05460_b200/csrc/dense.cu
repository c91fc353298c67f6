// dense.cu -- landmark block of the AFN build:
//   A11 = K11 + mu I, L L^T = A11 (blocked right-looking Cholesky, 64x64
//   tiles), W = K21 L^{-T} (= (L^{-1} K12)^T, the L^{-1}K12 block of
//   eq:factorized-form stored point-major) with the K21 tiles generated on
//   the fly, and L^{-T} for the apply's triangular products.
// FP64 SIMT: 256 threads own a 64x64 tile as 4x4 register micro-tiles with a
// stride-16 mapping (conflict-free shared-memory broadcasts).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int NB = 64;       // tile size
constexpr int TP = NB + 1;   // padded smem pitch (doubles)
constexpr int DT = 256;      // threads
#define TRY_SMEM()                          \
  do {                                      \
    afn_status s_ = set_smem_once();        \
    if (s_ != AFN_OK) return s_;            \
  } while (0)

__global__ void gather_rows_kernel(const double* __restrict__ X, int64_t n, int d,
                                   const int64_t* __restrict__ perm, double* __restrict__ Y) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const int64_t i = e / d, c = e - i * d;
  Y[e] = X[perm[i] * d + c];
}

// A = K(X1, X1) + mu I  (full)
__global__ void gen_k11_kernel(const double* __restrict__ X1, int64_t k, int d, KernelFn kf,
                               double mu, double* __restrict__ A) {
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  load_exp2_tab(s_tab);
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t i = e / k, j = e - i * k;
  double v;
  if (i == j) {
    v = 1.0 + mu;
  } else {
    const double s = d2_exact_rt(&X1[i * d], &X1[j * d], d);
    v = kern_from_d2(kf, s, s_tab);
  }
  A[e] = v;
}

// -------------------------------------------------------------------------
// Row-block triangular solve helper: T (64 rows x 64 cols, smem, pitch TP,
// stored [row][col]) <- T * Lbb^{-T}, Lbb lower 64x64 in smem [row][col].
// Each row is solved by 4 threads owning columns c = q (mod 4).
__device__ void rows_trsm_64(double* T, const double* Lbb, int rows_valid) {
  const int tid = threadIdx.x;
  // reciprocals of the diagonal first: a multiply (not a division) per step
  __shared__ double s_rinv[NB];
  // (a zero diagonal is an exhausted column of Alg. 1's threshold-pivoted
  // factor: its entries below are zero as well)
  if (tid < NB) {
    const double dg = Lbb[tid * TP + tid];
    s_rinv[tid] = dg != 0.0 ? 1.0 / dg : 0.0;
  }
  __syncthreads();
  const int r = tid >> 2, q = tid & 3;
  const int lane = tid & 31;
  double a[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) a[s] = T[r * TP + q + 4 * s];
  // column-cyclic ownership: thread q owns columns q + 4s.  Step j = 4*s + q'.
#pragma unroll
  for (int s = 0; s < 16; ++s) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int j = 4 * s + qq;
      double xj = 0.0;
      if (q == qq) {
        a[s] = a[s] * s_rinv[j];
        xj = a[s];
      }
      xj = __shfl_sync(0xffffffffu, xj, (lane & ~3) | qq);
      // update columns t = q + 4 s' > j
#pragma unroll
      for (int s2 = s; s2 < 16; ++s2) {
        if (s2 > s || q > qq) a[s2] = fma(-xj, Lbb[(q + 4 * s2) * TP + j], a[s2]);
      }
    }
  }
  (void)rows_valid;
#pragma unroll
  for (int s = 0; s < 16; ++s) T[r * TP + q + 4 * s] = a[s];
}

// Blocked diagonal-block Cholesky (256 threads): the 64 x 64 block in shared
// memory is factored in four 16-column steps -- warp 0 factors the 16 x 16
// diagonal sub-block (one row per lane in registers, columns broadcast through
// shared memory, one rsqrt per column), every thread then solves one panel row
// (16 columns, multiplies by the stored reciprocal pivots) and the trailing
// lower part is updated (16-term dots).  A non-positive pivot is reported in
// *info (global row) and replaced by 1 so the block stays finite; with
// skip_thr >= 0 (Alg. 1's threshold pivoting, reading R10) a pivot <= skip_thr
// instead marks an exhausted column: L's column (diagonal included) is zero
// and the trailing matrix is left unchanged, no report.  Batched over
// blockIdx.y (matrix A + y bs, info + y).
// (a device function of NTH threads: the stand-alone kernel for the first
// block, and the trailing-update kernel's first CTA for the next block)
template <int NTH>
__device__ void diag_factor64(double* A, int64_t k, int64_t kb, int* info, double skip_thr, double* s,
                              double* s_inv, double* s_col) {
  const int nb = (int)min((int64_t)NB, k - kb);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < NB * NB; e += NTH) {
    const int i = e / NB, t = e - i * NB;
    double v = 0.0;
    if (t <= i) v = (i < nb && t < nb) ? A[(kb + i) * k + kb + t] : (i == t ? 1.0 : 0.0);
    s[i * TP + t] = v;
  }
  __syncthreads();
  for (int b0 = 0; b0 < NB; b0 += 16) {
    if (wid == 0) {  // 16 x 16 diagonal sub-block: lane lr owns row b0 + lr
      const int lr = lane & 15;
      double dr[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) dr[c] = c <= lr ? s[(b0 + lr) * TP + b0 + c] : 0.0;
      double myinv = 1.0;
      bool bad = false;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        double* cb = s_col + (c & 1) * 16;
        if (lane < 16) cb[lane] = dr[c];
        __syncwarp();
        double piv = cb[c];
        double inv;
        if (skip_thr >= 0.0) {
          inv = piv > skip_thr ? rsqrt(piv) : 0.0;  // exhausted column: L[:, c] = 0
        } else {
          if (!(piv > 0.0)) { bad = true; piv = 1.0; }
          inv = rsqrt(piv);
        }
        const double lrc = dr[c] * inv;
        const double f = lrc * inv;
        if (lr == c) myinv = inv;
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2)
          if (lr >= c2) dr[c2] = fma(-f, cb[c2], dr[c2]);
        dr[c] = (lr == c) ? piv * inv : (lr > c ? lrc : dr[c]);
      }
      if (lane < 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c <= lr) s[(b0 + lr) * TP + b0 + c] = dr[c];
        s_inv[b0 + lr] = myinv;
        if (bad && b0 + lr < nb) atomicCAS(info, 0, (int)(kb + b0 + lr + 1));
      }
    }
    __syncthreads();
    const int r0 = b0 + 16;
    if (r0 >= NB) break;
    // panel: rows r >= r0, columns b0..b0+15: x L_d^T = a (one row per thread)
    for (int r = r0 + tid; r < NB; r += NTH) {
      double x[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = s[r * TP + b0 + c];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        double a = x[c];
#pragma unroll
        for (int c2 = 0; c2 < c; ++c2) a = fma(-x[c2], s[(b0 + c) * TP + b0 + c2], a);
        x[c] = a * s_inv[b0 + c];
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) s[r * TP + b0 + c] = x[c];
    }
    __syncthreads();
    // trailing lower part: s[r][c] -= sum_t L[r][b0+t] L[c][b0+t], r0 <= c <= r < NB
    const int m = NB - r0;
    for (int e = tid; e < m * m; e += NTH) {
      const int r = r0 + e / m, c = r0 + e % m;
      if (c > r) continue;
      double a = 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t) a = fma(s[r * TP + b0 + t], s[c * TP + b0 + t], a);
      s[r * TP + c] -= a;
    }
    __syncthreads();
  }
  for (int e = tid; e < NB * NB; e += NTH) {
    const int i = e / NB, t = e - i * NB;
    if (i < nb && t < nb) A[(kb + i) * k + kb + t] = t <= i ? s[i * TP + t] : 0.0;
  }
}

constexpr int DB_T = 256;
__global__ void __launch_bounds__(DB_T) potrf_diag_blk_kernel(double* A, int64_t k, int64_t kb, int* info,
                                                             int64_t bs, double skip_thr) {
  __shared__ double s[NB * TP];
  __shared__ double s_inv[NB];
  __shared__ __align__(16) double s_col[32];
  diag_factor64<DB_T>(A + (int64_t)blockIdx.y * bs, k, kb, info + blockIdx.y, skip_thr, s, s_inv, s_col);
}

// Panel below the diagonal block: A[i, kb:kb+nb] <- A[i, kb:kb+nb] L_kk^{-T}.
__global__ void __launch_bounds__(DT) potrf_panel_kernel(double* A, int64_t k, int64_t kb, int64_t bs) {
  A += (int64_t)blockIdx.y * bs;
  extern __shared__ double dsm[];
  double* sL = dsm;
  double* sT = dsm + NB * TP;
  const int nb = (int)min((int64_t)NB, k - kb);
  const int64_t r0 = kb + NB + (int64_t)blockIdx.x * NB;
  for (int e = threadIdx.x; e < NB * NB; e += DT) {
    const int i = e / NB, j = e % NB;
    sL[i * TP + j] = (i < nb && j < nb) ? A[(kb + i) * k + kb + j] : (i == j ? 1.0 : 0.0);
    const int64_t r = r0 + i;
    sT[i * TP + j] = (r < k && j < nb) ? A[r * k + kb + j] : 0.0;
  }
  __syncthreads();
  rows_trsm_64(sT, sL, NB);
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += DT) {
    const int i = e / NB, j = e % NB;
    const int64_t r = r0 + i;
    if (r < k && j < nb) A[r * k + kb + j] = sT[i * TP + j];
  }
}

constexpr size_t SMEM2 = sizeof(double) * 2 * NB * TP;

__global__ void diag_inv_kernel(const double* __restrict__ Lp, int64_t kp, double* __restrict__ X);

afn_status set_smem_once() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return AFN_OK;
  AFN_CUDA(cudaFuncSetAttribute(potrf_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  AFN_CUDA(cudaFuncSetAttribute(diag_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return AFN_OK;
}

// -------------------------------------------------------------------------
// W = K21 L^{-T} as a GEMM with the explicit L^{-T} (upper triangular):
// W[r][c] = sum_{t <= c} K21[r][t] LinvT[t][c].  With FPS landmarks K11 + mu I
// is well conditioned (cond(L) <= ~10 on the configs; SURVEY 8(c) Fig. 3.2
// screening argument), so the explicit inverse loses nothing measurable and
// the column blocks become independent tiles (no sequential sweep): the
// FP64 tensor-core GEMM gemm_dmma_kernel<0> below.

__device__ __forceinline__ void cpa16_d(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void dmma884d(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// FP64 tensor-core MMA (SASS DMMA.8x8x4): D(8x8) += A(8x4, row) B(4x8, col)
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

__global__ void gen_k21_kernel(const double* __restrict__ X1, int64_t k, const double* __restrict__ Xr,
                               int64_t N, int d, KernelFn kf, double* __restrict__ Kb) {
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  load_exp2_tab(s_tab);
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * k) return;
  const int64_t r = e / k, c = e - r * k;
  const double sd = d2_exact_rt(&Xr[r * d], &X1[c * d], d);
  Kb[e] = kern_from_d2(kf, sd, s_tab);
}

// -------------------------------------------------------------------------
// C = A B with B upper triangular (B[t][c] = 0 for t > c): the W = K21 L^{-T}
// product.  128 x 128 tiles, 256 threads with 8 x 8 register tiles
// (rows ty*4 + {0..3, 64..67}, columns tx*4 + {0..3, 64..67}: every operand
// read is an LDS.128 of two adjacent doubles pairs, A broadcast within the
// warp, B conflict-free), BK = 16 double-buffered through cp.async (A
// transposed into [kk][row] while staging).  FP64 SIMT: 64 DFMA per 8 LDS.128.

// pad L (k x k) into Lp (kp x kp): identity beyond k, zero elsewhere
__global__ void pad_l_kernel(const double* __restrict__ L, int64_t k, double* __restrict__ Lp, int64_t kp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kp * kp) return;
  const int64_t i = e / kp, j = e - i * kp;
  Lp[e] = (i < k && j < k) ? (j <= i ? L[i * k + j] : 0.0) : (i == j ? 1.0 : 0.0);
}

// X_bb = inverse of the 64x64 diagonal block b of Lp (lower), written into X
__global__ void __launch_bounds__(DT) diag_inv_kernel(const double* __restrict__ Lp, int64_t kp,
                                                      double* __restrict__ X) {  // (declared above)
  extern __shared__ double dsm[];
  double* sT = dsm;
  double* sL = dsm + NB * TP;
  const int64_t b0 = (int64_t)blockIdx.x * NB;
  for (int e = threadIdx.x; e < NB * NB; e += DT) {
    const int r = e / NB, c = e % NB;
    sL[r * TP + c] = Lp[(b0 + r) * kp + b0 + c];
    sT[r * TP + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  rows_trsm_64(sT, sL, NB);  // sT = I * Lbb^{-T} = Lbb^{-T}
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += DT) {
    const int r = e / NB, c = e % NB;  // X[r][c] = (Lbb^{-T})[c][r]
    X[(b0 + r) * kp + b0 + c] = sT[c * TP + r];
  }
}

// LinvT[i][j] = X[j][i] for i, j < k (32x32 smem transpose tiles)
__global__ void transpose_k_kernel(const double* __restrict__ X, int64_t kp, int64_t k, double* __restrict__ LinvT) {
  __shared__ double t[32][33];
  const int64_t bi = (int64_t)blockIdx.y * 32, bj = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = bi + r, j = bj + threadIdx.x;
    t[r][threadIdx.x] = (i < k && j < k) ? X[i * kp + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = bj + r, j = bi + threadIdx.x;
    if (i < k && j < k) LinvT[i * k + j] = t[threadIdx.x][r];
  }
}

__global__ void zero_upper_kernel(double* __restrict__ A, int64_t k, int64_t bs) {
  A += (int64_t)blockIdx.y * bs;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t i = e / k, j = e - i * k;
  if (j > i) A[e] = 0.0;
}

// ---- G = F^T F (Nystrom branch Gram, SYRK): 32x32 lower tiles of G, row
// chunks of F in parallel, partials summed in chunk order (deterministic)
constexpr int ST = 32;
__global__ void __launch_bounds__(256) syrk_partial_kernel(const double* __restrict__ F, int64_t R, int64_t C,
                                                           int64_t rows_per_chunk, double* __restrict__ part) {
  __shared__ double sa[ST][ST + 1], sb[ST][ST + 1];
  const int64_t tile = blockIdx.x, chunk = blockIdx.y;
  int I = (int)((sqrt(8.0 * (double)tile + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > tile) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tile) ++I;
  const int J = (int)(tile - (int64_t)I * (I + 1) / 2);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = chunk * rows_per_chunk, r1 = min(R, r0 + rows_per_chunk);
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t rb = r0; rb < r1; rb += ST) {
    __syncthreads();
    for (int e = threadIdx.x; e < ST * ST; e += 256) {
      const int rr = e / ST, c = e - rr * ST;
      const int64_t r = rb + rr;
      const int64_t ci = (int64_t)I * ST + c, cj = (int64_t)J * ST + c;
      sa[rr][c] = (r < r1 && ci < C) ? F[r * C + ci] : 0.0;
      sb[rr][c] = (r < r1 && cj < C) ? F[r * C + cj] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < ST; ++rr) {
      const double a0 = sa[rr][ty], a1 = sa[rr][ty + 16];
      const double b0 = sb[rr][tx], b1 = sb[rr][tx + 16];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
  }
  double* P = part + (chunk * gridDim.x + tile) * (ST * ST);
  P[ty * ST + tx] = acc[0][0];
  P[ty * ST + tx + 16] = acc[0][1];
  P[(ty + 16) * ST + tx] = acc[1][0];
  P[(ty + 16) * ST + tx + 16] = acc[1][1];
}

__global__ void syrk_reduce_kernel(const double* __restrict__ part, int64_t ntile, int64_t nchunk, int64_t C,
                                   double* __restrict__ G) {
  const int64_t tile = blockIdx.x;
  int I = (int)((sqrt(8.0 * (double)tile + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > tile) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tile) ++I;
  const int J = (int)(tile - (int64_t)I * (I + 1) / 2);
  for (int e = threadIdx.x; e < ST * ST; e += blockDim.x) {
    const int a = e / ST, b = e - a * ST;
    const int64_t i = (int64_t)I * ST + a, j = (int64_t)J * ST + b;
    if (i >= C || j >= C) continue;
    double s = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) s += part[(c * ntile + tile) * (ST * ST) + e];
    G[i * C + j] = s;
    G[j * C + i] = s;
  }
}

}  // namespace

afn_status syrk_ata(const double* F, int64_t R, int64_t C, double* G, cudaStream_t st) {
  if (C <= 0) return AFN_OK;
  const int64_t T = (C + ST - 1) / ST;
  const int64_t ntile = T * (T + 1) / 2;
  int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>((R + 2047) / 2048, std::max<int64_t>(1, 32768 / ntile)));
  const int64_t rpc = (R + nchunk - 1) / nchunk;
  nchunk = std::max<int64_t>(1, (R + rpc - 1) / rpc);
  double* part = nullptr;
  afn_status s = dalloc((void**)&part, sizeof(double) * nchunk * ntile * ST * ST, st);
  if (s != AFN_OK) return s;
  syrk_partial_kernel<<<dim3((unsigned)ntile, (unsigned)nchunk), 256, 0, st>>>(F, R, C, rpc, part);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    note_launch();
    syrk_reduce_kernel<<<(unsigned)ntile, 256, 0, st>>>(part, ntile, nchunk, C, G);
    e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
  }
  dfree(part, st);
  if (e != cudaSuccess) return cuda_status(e, "syrk kernels");
  return AFN_OK;
}

afn_status gather_rows(const double* X, int64_t n, int d, const int64_t* perm, double* Y,
                       cudaStream_t st) {
  const int64_t tot = n * d;
  if (tot == 0) return AFN_OK;
  gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X, n, d, perm, Y);
  AFN_LAUNCH_CHECK("gather_rows_kernel");
  return AFN_OK;
}

afn_status gen_k11(const double* X1, int64_t k, int d, Kern kn, double mu, double* A,
                   cudaStream_t st) {
  const int64_t tot = k * k;
  const KernelFn kf = kernel_fn(kn.kind, kn.l);
  gen_k11_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X1, k, d, kf, mu, A);
  AFN_LAUNCH_CHECK("gen_k11_kernel");
  return AFN_OK;
}

// Trailing update on the FP64 tensor cores: tile (I, J), J <= I, of the
// lower part: A[I, J] -= A[I, P] A[J, P]^T, P = [kb, kb + NB).  The two 64 x 64
// panel slices are staged whole (68-double row stride: every fragment LDS.64
// -- 8 rows x 4 consecutive k -- is two conflict-free wavefronts); 4 warps of
// 32 x 32 (16 DMMA per k-step of 4).
constexpr int PUP = NB + 4;
// With fuse, the CTA of tile 0 -- the next diagonal block -- factors that
// block right after updating it (diag_factor64), while the other CTAs still
// update: the stand-alone diagonal launch leaves the step's critical path.
__global__ void __launch_bounds__(128) potrf_update_dmma_kernel(double* A, int64_t k, int64_t kb, int64_t bs,
                                                                int* info, double skip_thr, int fuse) {
  A += (int64_t)blockIdx.y * bs;
  info += blockIdx.y;
  extern __shared__ __align__(16) double usm[];
  double* sI = usm;              // [NB][PUP]
  double* sJ = usm + NB * PUP;   // [NB][PUP]
  const int64_t t = blockIdx.x;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  const int64_t bj = t - bi * (bi + 1) / 2;
  const int64_t base = kb + NB;
  const int64_t I0 = base + bi * NB, J0 = base + bj * NB;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid >> 1, wn = wid & 1;
  const bool vec = (k & 1) == 0;
  for (int e = tid; e < NB * NB / 2; e += 128) {
    const int r = e / (NB / 2), c = 2 * (e - r * (NB / 2));
    const int64_t ri = I0 + r, rj = J0 + r;
    double* di = &sI[r * PUP + c];
    double* dj = &sJ[r * PUP + c];
    if (vec && ri < k) cpa16_d(di, &A[ri * k + kb + c]);
    else { di[0] = ri < k ? A[ri * k + kb + c] : 0.0; di[1] = ri < k ? A[ri * k + kb + c + 1] : 0.0; }
    if (vec && rj < k) cpa16_d(dj, &A[rj * k + kb + c]);
    else { dj[0] = rj < k ? A[rj * k + kb + c] : 0.0; dj[1] = rj < k ? A[rj * k + kb + c + 1] : 0.0; }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (!(bi == bj && wm < wn)) {  // (not the strictly upper 32 x 32 block of a diagonal tile)
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* a = sI + (wm * 32 + fr) * PUP + fk;
  const double* b = sJ + (wn * 32 + fr) * PUP + fk;
#pragma unroll 4
  for (int k4 = 0; k4 < NB; k4 += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) av[i] = a[i * 8 * PUP + k4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = b[j * 8 * PUP + k4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884d(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = I0 + wm * 32 + i * 8 + fr;
    if (r >= k) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = J0 + wn * 32 + j * 8 + 2 * fk;
      if (c < k && c <= r) A[r * k + c] -= acc[i][j][0];
      if (c + 1 < k && c + 1 <= r) A[r * k + c + 1] -= acc[i][j][1];
    }
  }
  }
  if (fuse && t == 0) {
    __syncthreads();  // (this CTA's updates of the block are visible to the whole CTA)
    diag_factor64<128>(A, k, base, info, skip_thr, usm, usm + NB * TP, usm + NB * TP + NB);
  }
}

afn_status potrf_batched(double* A, int64_t k, int nbatch, int64_t bs, double skip_thr, int* d_info,
                         cudaStream_t st) {
  static bool uattr = false;
  if (!uattr) {
    AFN_CUDA(cudaFuncSetAttribute(potrf_update_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * 2 * NB * PUP)));
    uattr = true;
  }
  TRY_SMEM();
  AFN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int) * nbatch, st));
  potrf_diag_blk_kernel<<<dim3(1, nbatch), DB_T, 0, st>>>(A, k, 0, d_info, bs, skip_thr);
  AFN_LAUNCH_CHECK("potrf_diag_blk_kernel");
  for (int64_t kb = 0; kb < k; kb += NB) {
    const int64_t rem = k - kb - NB;
    if (rem <= 0) break;
    const int64_t T = (rem + NB - 1) / NB;
    potrf_panel_kernel<<<dim3((unsigned)T, nbatch), DT, SMEM2, st>>>(A, k, kb, bs);
    AFN_LAUNCH_CHECK("potrf_panel_kernel");
    // trailing update on the FP64 tensor cores + the next diagonal block
    potrf_update_dmma_kernel<<<dim3((unsigned)(T * (T + 1) / 2), nbatch), 128, (int)(sizeof(double) * 2 * NB * PUP),
                               st>>>(A, k, kb, bs, d_info, skip_thr, 1);
    AFN_LAUNCH_CHECK("potrf_update_dmma_kernel");
  }
  zero_upper_kernel<<<dim3((unsigned)((k * k + 255) / 256), nbatch), 256, 0, st>>>(A, k, bs);
  AFN_LAUNCH_CHECK("zero_upper_kernel");
  return AFN_OK;
}

afn_status potrf_lower(double* A, int64_t k, int* d_info, cudaStream_t st) {
  return potrf_batched(A, k, 1, 0, -1.0, d_info, st);
}

// C (M x N) = A (M x K) B (K x N), all row-major, B upper triangular
// (B[t][c] = 0 for t > c: a tile's K range ends at its last column), on the
// FP64 tensor cores: mma.sync m8n8k4 f64 (DMMA.8x8x4).  CTA tile 64 x 64,
// 4 warps of 32 x 32 (4 x 4 m8n8 tiles, 32 accumulators per thread), k-chunks
// of 16 through 4 cp.async stages.  A chunk at a 20-double row stride and B
// chunk at a 72-double row stride: each fragment LDS.64 (8 rows x 4 k, or
// 4 k x 8 columns) is two conflict-free wavefronts.
constexpr int TM = 64, TN = 64, TK = 16, TKP = 20, TNP = 72, TS = 3;
// MODE 0: B upper (K range ends at the tile's last column); 1: A lower (ends
// at the tile's last row); 2: B lower (starts at the tile's first column);
// 3: general.
// Batched over blockIdx.z with element strides sA, sB, sC; C = alpha A B.
template <int MODE>
__global__ void __launch_bounds__(128) gemm_dmma_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                       double* __restrict__ Cm, int64_t M, int64_t N, int64_t K,
                                                       int64_t lda, int64_t ldb, int64_t ldc, int64_t sAz,
                                                       int64_t sBz, int64_t sCz, double alpha) {
  extern __shared__ __align__(16) double tsm[];
  double* sA = tsm;                    // [TS][TM][TKP]
  double* sB = tsm + TS * TM * TKP;    // [TS][TK][TNP]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid >> 1, wn = wid & 1;
  A += (int64_t)blockIdx.z * sAz;
  B += (int64_t)blockIdx.z * sBz;
  Cm += (int64_t)blockIdx.z * sCz;
  const int64_t R0 = (int64_t)blockIdx.y * TM, C0 = (int64_t)blockIdx.x * TN;
  const int64_t kend = MODE == 0 ? min(K, C0 + TN) : (MODE == 1 ? min(K, R0 + TM) : K);
  // MODE 4: as 2 for a symmetric product (M = L^{-T} L^{-1}): the tiles wholly
  // above the diagonal are skipped (the caller reads the lower triangle)
  if (MODE == 4 && R0 + TM <= C0) return;
  const int64_t kbeg = (MODE == 2 || MODE == 4) ? (min(K, C0) / TK) * TK : 0;
  const int64_t nkb = (kend - kbeg + TK - 1) / TK;
  const bool vec = (lda & 1) == 0 && (ldb & 1) == 0 && (ldc & 1) == 0 &&
                   (((uintptr_t)A | (uintptr_t)B | (uintptr_t)Cm) & 15) == 0;  // 16-byte copies
  auto stage = [&](int64_t kb, int buf) {
    const int64_t k0 = kbeg + kb * TK;
    double* a = sA + buf * TM * TKP;
    double* b = sB + buf * TK * TNP;
#pragma unroll
    for (int u = 0; u < (TM * TK / 2) / 128; ++u) {  // A: 16-byte copies, row r, k pair
      const int e = tid + 128 * u;
      const int r = e / (TK / 2), kp = 2 * (e - r * (TK / 2));
      const int64_t gr = R0 + r, gk = k0 + kp;
      double* dst = &a[r * TKP + kp];
      if (vec && gr < M && gk + 1 < kend) {
        cpa16_d(dst, &A[gr * lda + gk]);
      } else {
        dst[0] = (gr < M && gk < kend) ? A[gr * lda + gk] : 0.0;
        dst[1] = (gr < M && gk + 1 < kend) ? A[gr * lda + gk + 1] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < (TK * TN / 2) / 128; ++u) {  // B: 16-byte copies, k row, column pair
      const int e = tid + 128 * u;
      const int kk = e / (TN / 2), c = 2 * (e - kk * (TN / 2));
      const int64_t gk = k0 + kk, gc = C0 + c;
      double* dst = &b[kk * TNP + c];
      if (vec && gk < kend && gc + 1 < N) {
        cpa16_d(dst, &B[gk * ldb + gc]);
      } else {
        dst[0] = (gk < kend && gc < N) ? B[gk * ldb + gc] : 0.0;
        dst[1] = (gk < kend && gc + 1 < N) ? B[gk * ldb + gc + 1] : 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < TS - 1; ++s0) {
    if (s0 < nkb) stage(s0, s0);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kb = 0; kb < nkb; ++kb) {
    asm volatile("cp.async.wait_group %0;" ::"n"(TS - 2) : "memory");
    __syncthreads();
    const int64_t nx = kb + TS - 1;
    if (nx < nkb) stage(nx, (int)(nx % TS));
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double* a = sA + (int)(kb % TS) * TM * TKP + (wm * 32 + fr) * TKP + fk;
    const double* b = sB + (int)(kb % TS) * TK * TNP + fk * TNP + wn * 32 + fr;
#pragma unroll
    for (int k4 = 0; k4 < TK; k4 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = a[i * 8 * TKP + k4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = b[k4 * TNP + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884d(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = R0 + wm * 32 + i * 8 + fr;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = C0 + wn * 32 + j * 8 + 2 * fk;
      if (vec && c + 1 < N) {
        *reinterpret_cast<double2*>(&Cm[r * ldc + c]) = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
      } else {
        if (c < N) Cm[r * ldc + c] = alpha * acc[i][j][0];
        if (c + 1 < N) Cm[r * ldc + c + 1] = alpha * acc[i][j][1];
      }
    }
  }
}

afn_status w_gemm(const double* LinvT, int64_t k, const double* X1, const double* Xr, int64_t N, int d,
                  Kern kn, double* W, cudaStream_t st) {
  if (N <= 0 || k <= 0) return AFN_OK;
  const KernelFn kf = kernel_fn(kn.kind, kn.l);
  // K21 is generated in row blocks of <= ~1 GiB (not all N x k at once: at
  // n = 2^20, k = 8000 that alone would be 66.6 GB)
  const int64_t rb = std::max<int64_t>(TM, std::min<int64_t>(N, ((1LL << 27) / k) / TM * TM));
  double* Kb = nullptr;
  afn_status s = dalloc((void**)&Kb, sizeof(double) * rb * k, st);
  if (s != AFN_OK) return s;
  static bool attr = false;
  if (!attr) {
    for (auto kf2 : {gemm_dmma_kernel<0>, gemm_dmma_kernel<1>, gemm_dmma_kernel<2>})
      AFN_CUDA(cudaFuncSetAttribute(kf2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(double) * TS * (TM * TKP + TK * TNP))));
    attr = true;
  }
  for (int64_t r0 = 0; r0 < N; r0 += rb) {
    const int64_t nr = std::min(rb, N - r0);
    gen_k21_kernel<<<(unsigned)((nr * k + 255) / 256), 256, 0, st>>>(X1, k, Xr + r0 * d, nr, d, kf, Kb);
    AFN_LAUNCH_CHECK("gen_k21_kernel");
    dim3 grid((unsigned)((k + TN - 1) / TN), (unsigned)((nr + TM - 1) / TM));  // FP64 tensor cores
    gemm_dmma_kernel<0><<<grid, 128, (int)(sizeof(double) * TS * (TM * TKP + TK * TNP)), st>>>(
        Kb, LinvT, W + r0 * k, nr, k, k, k, k, k, 0, 0, 0, 1.0);
    AFN_LAUNCH_CHECK("gemm_dmma_kernel<0>");
  }
  dfree(Kb, st);
  return AFN_OK;
}

afn_status linv_recursive(const double* L, int64_t k, double* LinvT, cudaStream_t st, double* ws) {
  int64_t kp = NB;
  while (kp < k) kp <<= 1;
  afn_status s;
  const bool own = ws == nullptr;
  if (own && (s = dalloc((void**)&ws, sizeof(double) * 3 * kp * kp, st)) != AFN_OK) return s;
  double* Lp = ws;
  double* X = ws + kp * kp;
  double* Tt = ws + 2 * kp * kp;
  struct F { double* a; bool own; cudaStream_t st; ~F() { if (own) dfree(a, st); } } fr{ws, own, st};
  AFN_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * kp * kp, st));
  pad_l_kernel<<<(unsigned)((kp * kp + 255) / 256), 256, 0, st>>>(L, k, Lp, kp);
  AFN_LAUNCH_CHECK("pad_l_kernel");
  diag_inv_kernel<<<(unsigned)(kp / NB), DT, SMEM2, st>>>(Lp, kp, X);
  AFN_LAUNCH_CHECK("diag_inv_kernel");
  static bool dattr = false;
  const int dbytes = (int)(sizeof(double) * TS * (TM * TKP + TK * TNP));
  if (!dattr) {
    AFN_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, dbytes));
    AFN_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, dbytes));
    dattr = true;
  }
  for (int64_t h = NB; h < kp; h <<= 1) {
    const int64_t pairs = kp / (2 * h);
    const int64_t stride = 2 * h * kp + 2 * h;  // next diagonal pair
    // FP64 tensor cores: T = B A^{-1}, then X21 = -C^{-1} T
    dim3 grid((unsigned)((h + TN - 1) / TN), (unsigned)((h + TM - 1) / TM), (unsigned)pairs);
    gemm_dmma_kernel<2><<<grid, 128, dbytes, st>>>(Lp + h * kp, X, Tt, h, h, h, kp, kp, kp, stride, stride,
                                                   stride, 1.0);
    AFN_LAUNCH_CHECK("gemm_dmma_kernel<2>");
    gemm_dmma_kernel<1><<<grid, 128, dbytes, st>>>(X + h * kp + h, Tt, X + h * kp, h, h, h, kp, kp, kp, stride,
                                                   stride, stride, -1.0);
    AFN_LAUNCH_CHECK("gemm_dmma_kernel<1>");
  }
  dim3 tg((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
  transpose_k_kernel<<<tg, dim3(32, 8), 0, st>>>(X, kp, k, LinvT);
  AFN_LAUNCH_CHECK("transpose_k_kernel");
  return AFN_OK;
}

afn_status gemm_nn(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K, int64_t lda,
                   int64_t ldb, int64_t ldc, double alpha, cudaStream_t st) {
  if (M <= 0 || N <= 0) return AFN_OK;
  const int bytes = (int)(sizeof(double) * TS * (TM * TKP + TK * TNP));
  static bool attr = false;
  if (!attr) {
    AFN_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    attr = true;
  }
  dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM), 1);
  gemm_dmma_kernel<3><<<grid, 128, bytes, st>>>(A, B, C, M, N, K, lda, ldb, ldc, 0, 0, 0, alpha);
  AFN_LAUNCH_CHECK("gemm_dmma_kernel<3>");
  return AFN_OK;
}

afn_status transpose_sq(const double* A, int64_t k, double* At, cudaStream_t st) {
  if (k <= 0) return AFN_OK;
  dim3 tg((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
  transpose_k_kernel<<<tg, dim3(32, 8), 0, st>>>(A, k, k, At);
  AFN_LAUNCH_CHECK("transpose_k_kernel");
  return AFN_OK;
}

int64_t linv_ws_doubles(int64_t k) {
  int64_t kp = NB;
  while (kp < k) kp <<= 1;
  return 3 * kp * kp;
}

afn_status trsm_linvt(const double* L, int64_t k, double* LinvT, cudaStream_t st, double* ws) {
  TRY_SMEM();
  return linv_recursive(L, k, LinvT, st, ws);
}

}  // namespace afn

namespace afn {
// C = A B for A = B^T upper and B lower triangular (k x k, row-major; C is
// symmetric): the K range of a column block starts at its first column and
// only the tiles touching the lower triangle are formed (MODE 4), ~k^3 / 3 FMA;
// C's entries strictly above the diagonal tiles are left unwritten
afn_status gemm_upper_lower(const double* A, const double* B, int64_t k, double* C, cudaStream_t st) {
  if (k <= 0) return AFN_OK;
  const int bytes = (int)(sizeof(double) * TS * (TM * TKP + TK * TNP));
  AFN_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  dim3 grid((unsigned)((k + TN - 1) / TN), (unsigned)((k + TM - 1) / TM), 1);
  gemm_dmma_kernel<4><<<grid, 128, bytes, st>>>(A, B, C, k, k, k, k, k, k, 0, 0, 0, 1.0);
  AFN_LAUNCH_CHECK("gemm_dmma_kernel<4>");
  return AFN_OK;
}
}  // namespace afn

// dense.cu -- landmark block of the AFN build:
//   A11 = K11 + mu I, L L^T = A11 (blocked right-looking Cholesky, 64x64
//   tiles), W = K21 L^{-T} (= (L^{-1} K12)^T, the L^{-1}K12 block of
//   eq:factorized-form stored point-major) with the K21 tiles generated on
//   the fly, and L^{-T} for the apply's triangular products.
// FP64 SIMT: 256 threads own a 64x64 tile as 4x4 register micro-tiles with a
// stride-16 mapping (conflict-free shared-memory broadcasts).
#include <algorithm>
#include <cmath>

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
__global__ void gen_k11_kernel(const double* __restrict__ X1, int64_t k, int d, double cl,
                               double mu, double* __restrict__ A) {
  __shared__ double s_tab[16];
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
    v = gauss_from_d2(s, cl, s_tab);
  }
  A[e] = v;
}

// -------------------------------------------------------------------------
// Row-block triangular solve helper: T (64 rows x 64 cols, smem, pitch TP,
// stored [row][col]) <- T * Lbb^{-T}, Lbb lower 64x64 in smem [row][col].
// Each row is solved by 4 threads owning columns c = q (mod 4).
__device__ void rows_trsm_64(double* T, const double* Lbb, int rows_valid) {
  const int tid = threadIdx.x;
  const int r = tid >> 2, q = tid & 3;
  double a[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) a[s] = T[r * TP + q + 4 * s];
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const int owner = j & 3;
    double xj = 0.0;
    // owner computes x_j
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if (q == owner && (q + 4 * s) == j) a[s] = a[s] / Lbb[j * TP + j];
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if ((q + 4 * s) == j) xj = a[s];
    xj = __shfl_sync(0xffffffffu, xj, (tid & 31 & ~3) | owner);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int t = q + 4 * s;
      if (t > j) a[s] = fma(-xj, Lbb[t * TP + j], a[s]);
    }
  }
  (void)rows_valid;
#pragma unroll
  for (int s = 0; s < 16; ++s) T[r * TP + q + 4 * s] = a[s];
}

// Diagonal block Cholesky (in smem), writes L block, zeroes the upper part.
__global__ void __launch_bounds__(DT) potrf_diag_kernel(double* A, int64_t k, int64_t kb, int* info) {
  __shared__ double s[NB * TP];
  const int nb = (int)min((int64_t)NB, k - kb);
  for (int e = threadIdx.x; e < NB * NB; e += DT) {
    const int i = e / NB, j = e % NB;
    s[i * TP + j] = (i < nb && j < nb) ? A[(kb + i) * k + kb + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    if (threadIdx.x == 0) {
      const double p = s[j * TP + j];
      if (!(p > 0.0)) {
        if (!bad && j < nb) { bad = 1; atomicCAS(info, 0, (int)(kb + j + 1)); }
        s[j * TP + j] = 1.0;
      } else {
        s[j * TP + j] = sqrt(p);
      }
    }
    __syncthreads();
    const double piv = s[j * TP + j];
    for (int i = j + 1 + threadIdx.x; i < NB; i += DT) s[i * TP + j] /= piv;
    __syncthreads();
    // trailing update (lower): s[i][t] -= s[i][j] s[t][j], j < t <= i
    const int m = NB - j - 1;
    for (int e = threadIdx.x; e < m * m; e += DT) {
      const int i = j + 1 + e / m, t = j + 1 + e % m;
      if (t <= i) s[i * TP + t] = fma(-s[i * TP + j], s[t * TP + j], s[i * TP + t]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += DT) {
    const int i = e / nb, j = e % nb;
    A[(kb + i) * k + kb + j] = (j <= i) ? s[i * TP + j] : 0.0;
  }
}

// Panel below the diagonal block: A[i, kb:kb+nb] <- A[i, kb:kb+nb] L_kk^{-T}.
__global__ void __launch_bounds__(DT) potrf_panel_kernel(double* A, int64_t k, int64_t kb) {
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

// Trailing update of the lower part: A[I, J] -= A[I, P] A[J, P]^T for tiles
// J <= I below the panel P = [kb, kb+NB).
__global__ void __launch_bounds__(DT) potrf_update_kernel(double* A, int64_t k, int64_t kb) {
  extern __shared__ double dsm[];
  double* sA = dsm;  // [kk][row]
  double* sB = dsm + NB * TP;
  // triangular tile index
  const int64_t t = blockIdx.x;
  int64_t bi = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
  while (bi * (bi + 1) / 2 > t) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  const int64_t bj = t - bi * (bi + 1) / 2;
  const int64_t base = kb + NB;
  const int64_t I0 = base + bi * NB, J0 = base + bj * NB;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < NB * NB; e += DT) {
    const int r = e / NB, kk = e % NB;
    const int64_t ri = I0 + r, rj = J0 + r;
    sA[kk * TP + r] = (ri < k) ? A[ri * k + kb + kk] : 0.0;
    sB[kk * TP + r] = (rj < k) ? A[rj * k + kb + kk] : 0.0;
  }
  __syncthreads();
  double acc[4][4] = {};
#pragma unroll 4
  for (int kk = 0; kk < NB; ++kk) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sA[kk * TP + ty + 16 * i];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = sB[kk * TP + tx + 16 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = I0 + ty + 16 * i;
    if (r >= k) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = J0 + tx + 16 * j;
      if (c < k && c <= r) A[r * k + c] -= acc[i][j];
    }
  }
}

// -------------------------------------------------------------------------
// W (N x k) = B L^{-T} for a row block of 64 rows; B = K(Xr, X1) (MODE 0) or
// the identity (MODE 1, N = k, giving L^{-T}).  Column blocks b in order:
//   T = B[:, b] - W[:, <b] L[b, <b]^T ;  W[:, b] = T Lbb^{-T}.
template <int MODE>
__global__ void __launch_bounds__(DT) trsm_rows_kernel(const double* __restrict__ L, int64_t k,
                                                       const double* __restrict__ X1,
                                                       const double* __restrict__ Xr, int64_t N,
                                                       int d, double cl, double* __restrict__ W) {
  extern __shared__ double dsm[];
  double* sA = dsm;            // [kk][row]: W tile, later T [row][col]
  double* sB = dsm + NB * TP;  // [kk][col]: L tile, later Lbb [row][col]
  __shared__ double s_tab[16];
  load_exp2_tab(s_tab);
  __syncthreads();
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t R0 = (int64_t)blockIdx.x * NB;
  const int64_t nblk = (k + NB - 1) / NB;
  int64_t bstart = 0;
  if (MODE == 1) {
    bstart = blockIdx.x;  // L^{-T} row r is zero left of column r
    for (int64_t b = 0; b < bstart; ++b)
      for (int e = tid; e < NB * NB; e += DT) {
        const int r = e / NB, c = e % NB;
        const int64_t gr = R0 + r, gc = b * NB + c;
        if (gr < N && gc < k) W[gr * k + gc] = 0.0;
      }
  }
  // row coordinates for MODE 0 (4 rows per thread, strided)
  for (int64_t b = bstart; b < nblk; ++b) {
    const int64_t C0 = b * NB;
    double acc[4][4];
    // initial T = B[:, b]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t r = R0 + ty + 16 * i, c = C0 + tx + 16 * j;
        double v = 0.0;
        if (r < N && c < k) {
          if (MODE == 0) {
            const double s = d2_exact_rt(&Xr[r * d], &X1[c * d], d);
            v = gauss_from_d2(s, cl, s_tab);
          } else {
            v = (r == c) ? 1.0 : 0.0;
          }
        }
        acc[i][j] = v;
      }
    // GEMM: acc -= W[R, cb] * L[C0.., cb]^T over earlier column blocks
    for (int64_t cb = bstart; cb < b; ++cb) {
      __syncthreads();
      for (int e = tid; e < NB * NB; e += DT) {
        const int r = e / NB, kk = e % NB;
        const int64_t gr = R0 + r, lr = C0 + r, gc = cb * NB + kk;
        sA[kk * TP + r] = (gr < N && gc < k) ? W[gr * k + gc] : 0.0;
        sB[kk * TP + r] = (lr < k && gc < k) ? L[lr * k + gc] : 0.0;
      }
      __syncthreads();
#pragma unroll 4
      for (int kk = 0; kk < NB; ++kk) {
        double a[4], bb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sA[kk * TP + ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = sB[kk * TP + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(-a[i], bb[j], acc[i][j]);
      }
    }
    __syncthreads();
    // stage T [row][col] and Lbb [row][col]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) sA[(ty + 16 * i) * TP + tx + 16 * j] = acc[i][j];
    for (int e = tid; e < NB * NB; e += DT) {
      const int r = e / NB, c = e % NB;
      const int64_t lr = C0 + r, lc = C0 + c;
      sB[r * TP + c] = (lr < k && lc < k) ? L[lr * k + lc] : (r == c ? 1.0 : 0.0);
    }
    __syncthreads();
    rows_trsm_64(sA, sB, NB);
    __syncthreads();
    for (int e = tid; e < NB * NB; e += DT) {
      const int r = e / NB, c = e % NB;
      const int64_t gr = R0 + r, gc = C0 + c;
      if (gr < N && gc < k) W[gr * k + gc] = sA[r * TP + c];
    }
    // W[R, b] must be visible to this CTA's next GEMM loads (same threads may
    // read other threads' writes): barrier + block-scope fence
    __threadfence_block();
    __syncthreads();
  }
}

constexpr size_t SMEM2 = sizeof(double) * 2 * NB * TP;

afn_status set_smem_once() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return AFN_OK;
  AFN_CUDA(cudaFuncSetAttribute(potrf_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  AFN_CUDA(cudaFuncSetAttribute(potrf_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  AFN_CUDA(cudaFuncSetAttribute(trsm_rows_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  AFN_CUDA(cudaFuncSetAttribute(trsm_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return AFN_OK;
}

__global__ void zero_upper_kernel(double* __restrict__ A, int64_t k) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t i = e / k, j = e - i * k;
  if (j > i) A[e] = 0.0;
}

}  // namespace

afn_status gather_rows(const double* X, int64_t n, int d, const int64_t* perm, double* Y,
                       cudaStream_t st) {
  const int64_t tot = n * d;
  if (tot == 0) return AFN_OK;
  gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X, n, d, perm, Y);
  AFN_LAUNCH_CHECK("gather_rows_kernel");
  return AFN_OK;
}

afn_status gen_k11(const double* X1, int64_t k, int d, double l, double mu, double* A,
                   cudaStream_t st) {
  const int64_t tot = k * k;
  const double cl = AFN_LOG2E / (l * l);
  gen_k11_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X1, k, d, cl, mu, A);
  AFN_LAUNCH_CHECK("gen_k11_kernel");
  return AFN_OK;
}

afn_status potrf_lower(double* A, int64_t k, int* d_info, cudaStream_t st) {
  TRY_SMEM();
  AFN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  for (int64_t kb = 0; kb < k; kb += NB) {
    potrf_diag_kernel<<<1, DT, 0, st>>>(A, k, kb, d_info);
    AFN_LAUNCH_CHECK("potrf_diag_kernel");
    const int64_t rem = k - kb - NB;
    if (rem <= 0) break;
    const int64_t T = (rem + NB - 1) / NB;
    potrf_panel_kernel<<<(unsigned)T, DT, SMEM2, st>>>(A, k, kb);
    AFN_LAUNCH_CHECK("potrf_panel_kernel");
    potrf_update_kernel<<<(unsigned)(T * (T + 1) / 2), DT, SMEM2, st>>>(A, k, kb);
    AFN_LAUNCH_CHECK("potrf_update_kernel");
  }
  zero_upper_kernel<<<(unsigned)((k * k + 255) / 256), 256, 0, st>>>(A, k);
  AFN_LAUNCH_CHECK("zero_upper_kernel");
  return AFN_OK;
}

afn_status trsm_w(const double* L, int64_t k, const double* X1, const double* Xr, int64_t N, int d,
                  double l, double* W, cudaStream_t st) {
  if (N <= 0 || k <= 0) return AFN_OK;
  TRY_SMEM();
  const double cl = AFN_LOG2E / (l * l);
  trsm_rows_kernel<0><<<(unsigned)((N + NB - 1) / NB), DT, SMEM2, st>>>(L, k, X1, Xr, N, d, cl, W);
  AFN_LAUNCH_CHECK("trsm_rows_kernel<0>");
  return AFN_OK;
}

afn_status trsm_linvt(const double* L, int64_t k, double* LinvT, cudaStream_t st) {
  TRY_SMEM();
  trsm_rows_kernel<1><<<(unsigned)((k + NB - 1) / NB), DT, SMEM2, st>>>(L, k, nullptr, nullptr, k, 1,
                                                                   0.0, LinvT);
  AFN_LAUNCH_CHECK("trsm_rows_kernel<1>");
  return AFN_OK;
}

}  // namespace afn

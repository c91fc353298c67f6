// alg1.cu -- Algorithm 1, Nystrom rank estimation,
// on the device.
//
//  1. "randomly subsample a subset X_m of m points" (L666): counter-based
//     splitmix64 keys h_i = splitmix64(seed ^ i*golden) (reading R7); the m
//     smallest keys in ascending order.  A grid kernel collects every key
//     below a threshold, one CTA bitonic-sorts them.
//  2. scale the coordinates by s = (m/n)^(1/d) (L666, R8; s from the host),
//     form K_m (L667), FPS on X_m from subsample position 0 (fps.cu).
//  3. "the Nystrom rank r such that the relative Nystrom approximation error
//     falls below 0.1" (L668): with S^(r) the Schur complement of K_m after r
//     elimination steps in FPS order (K_m - K_nys,r = [0 0; 0 S^(r)], P:L559;
//     pivots <= m eps ||K_m|| are skipped, R10), the test
//     ||S^(r)||_2 < 0.1 ||K_m||_2 is decided as "0.1||K_m|| I - S^(r) is
//     positive definite" by a Cholesky attempt (S^(r) is PSD).  The error
//     curve is non-increasing in r (nested landmarks), so the smallest
//     passing r is found by bisection.
//  4. k = r n / m rounded half up (R11); if k < 2000 the count of eigenvalues
//     of K_m on the unscaled points above 0.1 (L673-674) by Sturm counts on a
//     Householder tridiagonalisation.  ||K_m||_2 = lambda_max also comes from
//     the tridiagonal form (bisection).
// All dense work is small (m <= 1024) and runs in single-CTA kernels on
// L2-resident global memory.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int AT = 1024;         // threads of the single-CTA kernels
constexpr int CAND_CAP = 4096;   // candidate keys sorted in one CTA

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void cand_kernel(int64_t n, uint64_t seed, uint64_t thr, unsigned long long* keys,
                            long long* ids, unsigned* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = splitmix64_dev(seed ^ ((uint64_t)i * 0x9E3779B97F4A7C15ULL));
  if (h < thr) {
    const unsigned p = atomicAdd(cnt, 1u);
    if (p < CAND_CAP) {
      keys[p] = h;
      ids[p] = i;
    }
  }
}

// candidates below thr into (keys, ids) up to cap (uniform landmark selection)
__global__ void cand_cap_kernel(int64_t n, uint64_t seed, uint64_t thr, int64_t cap,
                                unsigned long long* keys, long long* ids, unsigned long long* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = splitmix64_dev(seed ^ ((uint64_t)i * 0x9E3779B97F4A7C15ULL));
  if (h < thr) {
    const unsigned long long p = atomicAdd(cnt, 1ULL);
    if ((int64_t)p < cap) {
      keys[p] = h;
      ids[p] = i;
    }
  }
}

// one-CTA bitonic sort of P (power of two) (key, id) pairs in global memory,
// padding beyond the count with ~0; writes the first k ids
__global__ void __launch_bounds__(AT) bitonic_global_kernel(unsigned long long* keys, long long* ids,
                                                            const unsigned long long* cnt, int64_t P,
                                                            int64_t k, int64_t* out) {
  const int64_t c = (int64_t)min(*cnt, (unsigned long long)P);
  for (int64_t t = c + threadIdx.x; t < P; t += AT) {
    keys[t] = ~0ULL;
    ids[t] = -1;
  }
  __syncthreads();
  for (int64_t kk = 2; kk <= P; kk <<= 1)
    for (int64_t j = kk >> 1; j > 0; j >>= 1) {
      for (int64_t t = threadIdx.x; t < P; t += AT) {
        const int64_t p = t ^ j;
        if (p > t) {
          const bool up = (t & kk) == 0;
          const unsigned long long a = keys[t], b = keys[p];
          if ((a > b) == up) {
            keys[t] = b; keys[p] = a;
            const long long x = ids[t]; ids[t] = ids[p]; ids[p] = x;
          }
        }
      }
      __syncthreads();
    }
  for (int64_t t = threadIdx.x; t < k; t += AT) out[t] = ids[t];
}

// sort the candidates by key (unique), write the first m ids
__global__ void __launch_bounds__(AT) cand_sort_kernel(const unsigned long long* keys, const long long* ids,
                                                       const unsigned* cnt, int m, int64_t* out) {
  extern __shared__ unsigned long long dsm_keys[];
  unsigned long long* sk = dsm_keys;
  long long* si = reinterpret_cast<long long*>(dsm_keys + CAND_CAP);
  const unsigned c = min(*cnt, (unsigned)CAND_CAP);
  for (int t = threadIdx.x; t < CAND_CAP; t += AT) {
    sk[t] = t < (int)c ? keys[t] : ~0ULL;
    si[t] = t < (int)c ? ids[t] : -1;
  }
  __syncthreads();
  for (int k = 2; k <= CAND_CAP; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < CAND_CAP; t += AT) {
        const int p = t ^ j;
        if (p > t) {
          const bool up = (t & k) == 0;
          const unsigned long long a = sk[t], b = sk[p];
          if ((a > b) == up) {
            sk[t] = b; sk[p] = a;
            const long long x = si[t]; si[t] = si[p]; si[p] = x;
          }
        }
      }
      __syncthreads();
    }
  for (int t = threadIdx.x; t < m; t += AT) out[t] = si[t];
}

__global__ void gather_scale_kernel(const double* __restrict__ X, int d, const int64_t* __restrict__ ids,
                                    int m, double s, double* __restrict__ Xm, double* __restrict__ Xu) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * d) return;
  const int i = e / d, c = e - i * d;
  const double x = X[ids[i] * d + c];
  Xu[e] = x;
  Xm[e] = x * s;
}

__global__ void permute_sym_kernel(const double* __restrict__ A, int m, const int64_t* __restrict__ ord,
                                   double* __restrict__ B) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * m) return;
  const int i = e / m, j = e - i * m;
  B[e] = A[ord[i] * m + ord[j]];
}

__device__ double block_sum_1024(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = sh[lane];
  r = warp_sum(r);
  return r;  // every thread gets the total (blockDim = 1024 -> 32 warps)
}

// Householder tridiagonalisation of the symmetric m x m A (destroyed);
// diag -> dgl[0..m), offdiag -> off[0..m-1).  SM: A copied into shared memory.
template <int TT>
__device__ double block_sum_all(double v, double* sh) {  // every thread gets the total
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = lane < TT / 32 ? sh[lane] : 0.0;
  r = warp_sum(r);
  return r;
}

constexpr int SM_MAX_M = 164;  // (m^2 + 2m) doubles of dynamic smem <= 227 KB
// shared-memory path (m <= SM_MAX_M): p = A v by columns with row slices;
// global-memory path: warp per row
template <bool SM, int TT>
__global__ void __launch_bounds__(TT) tridiag_kernel(double* Ag, int m, double* dgl, double* off) {
  extern __shared__ double dsm[];
  __shared__ double sh[32];
  __shared__ double s_beta, s_alpha;
  double* A = SM ? dsm : Ag;
  double* v = SM ? dsm + (size_t)m * m : dsm;
  double* p = v + m;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (SM) {
    for (int64_t e = tid; e < (int64_t)m * m; e += TT) A[e] = Ag[e];
    __syncthreads();
  }
  for (int j = 0; j + 2 < m; ++j) {
    const int L = m - j - 1;  // length of the column below the diagonal
    double loc = 0.0;
    for (int t = tid; t < L; t += TT) {
      const double x = A[(int64_t)(j + 1 + t) * m + j];
      v[t] = x;
      loc += x * x;
    }
    const double nrm2 = block_sum_all<TT>(loc, sh);
    if (tid == 0) {
      const double x0 = v[0];
      const double nrm = sqrt(nrm2);
      double alpha = (x0 > 0.0) ? -nrm : nrm;
      const double v0 = x0 - alpha;
      const double vv = nrm2 - x0 * x0 + v0 * v0;
      if (nrm2 == 0.0 || vv == 0.0) {
        s_beta = 0.0;
        alpha = x0;
      } else {
        s_beta = 2.0 / vv;
      }
      v[0] = v0;
      s_alpha = alpha;
      dgl[j] = A[(int64_t)j * m + j];
      off[j] = alpha;
    }
    __syncthreads();
    const double beta = s_beta;
    if (beta == 0.0) continue;
    double loc2 = 0.0;
    if (SM) {
      // p = beta * A22 v by columns (A symmetric): thread (s, i) sums column
      // i over the rows t = s, s + S, ..  (consecutive threads read consecutive
      // words of a row: no bank conflicts, v[t] broadcast), then thread i adds
      // the S partials in order
      const int S = TT / L;
      double* part = p + m;
      if (tid < S * L) {
        const int s = tid / L, i = tid - s * L;
        const double* col = A + (int64_t)(j + 1) * m + (j + 1) + i;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int t = s;
        for (; t + 3 * S < L; t += 4 * S) {
          a0 = fma(col[(int64_t)t * m], v[t], a0);
          a1 = fma(col[(int64_t)(t + S) * m], v[t + S], a1);
          a2 = fma(col[(int64_t)(t + 2 * S) * m], v[t + 2 * S], a2);
          a3 = fma(col[(int64_t)(t + 3 * S) * m], v[t + 3 * S], a3);
        }
        for (; t < L; t += S) a0 = fma(col[(int64_t)t * m], v[t], a0);
        part[tid] = (a0 + a1) + (a2 + a3);
      }
      __syncthreads();
      if (tid < L) {
        double q = part[tid];
        for (int s = 1; s < S; ++s) q += part[s * L + tid];
        p[tid] = beta * q;
        loc2 = p[tid] * v[tid];
      }
    } else {
      // p = beta * A22 v   (warp per row, lanes over columns)
      for (int i = wid; i < L; i += TT / 32) {
        const double* row = A + (int64_t)(j + 1 + i) * m + (j + 1);
        double s = 0.0;
        for (int t = lane; t < L; t += 32) s = fma(row[t], v[t], s);
        s = warp_sum(s);
        if (lane == 0) p[i] = beta * s;
      }
      __syncthreads();
      for (int t = tid; t < L; t += TT) loc2 += p[t] * v[t];
    }
    const double pv = block_sum_all<TT>(loc2, sh);
    const double K = 0.5 * beta * pv;
    if (SM) {
      // A22 -= v w^T + w v^T with w = p - K v formed in registers (no pass over
      // p, no barrier); each lane keeps its <= 6 columns' v_t, w_t for all its
      // rows, and a row's loads are issued before its stores
      constexpr int QN = (SM_MAX_M + 31) / 32;
      double vt[QN], wt[QN];
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const int t = lane + 32 * q;
        vt[q] = t < L ? v[t] : 0.0;
        wt[q] = t < L ? p[t] - K * v[t] : 0.0;
      }
      for (int i = wid; i < L; i += TT / 32) {
        const double vi = v[i], wi = p[i] - K * v[i];
        double* a = A + (int64_t)(j + 1 + i) * m + (j + 1);
        double av[QN];
#pragma unroll
        for (int q = 0; q < QN; ++q)
          if (lane + 32 * q < L) av[q] = a[lane + 32 * q];
#pragma unroll
        for (int q = 0; q < QN; ++q)
          if (lane + 32 * q < L) a[lane + 32 * q] = av[q] - vi * wt[q] - wi * vt[q];
      }
      __syncthreads();
      continue;
    }
    for (int t = tid; t < L; t += TT) p[t] = p[t] - K * v[t];  // w
    __syncthreads();
    for (int i = wid; i < L; i += TT / 32) {  // warp per row (no 64-bit index division)
      const double vi = v[i], pi = p[i];
      double* a = A + (int64_t)(j + 1 + i) * m + (j + 1);
      for (int t = lane; t < L; t += 32) a[t] = a[t] - vi * p[t] - pi * v[t];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (m >= 2) {
      dgl[m - 2] = A[(int64_t)(m - 2) * m + (m - 2)];
      dgl[m - 1] = A[(int64_t)(m - 1) * m + (m - 1)];
      off[m - 2] = A[(int64_t)(m - 1) * m + (m - 2)];
    } else {
      dgl[0] = A[0];
    }
  }
}

// number of eigenvalues of the tridiagonal (dgl, off) strictly below x (Sturm)
__device__ int sturm_count(const double* dgl, const double* off, int m, double x) {
  int c = 0;
  double q = dgl[0] - x;
  if (q < 0.0) ++c;
  for (int i = 1; i < m; ++i) {
    double qq = (q != 0.0) ? q : DBL_MIN * 4.0;
    q = dgl[i] - x - off[i - 1] * off[i - 1] / qq;
    if (q < 0.0) ++c;
  }
  return c;
}

// out[0] = lambda_max (32-way multisection), out[1] = #{lambda >= x_count}
__global__ void eig_summary_kernel(const double* dgl, const double* off, int m, double x_count,
                                   double* out) {
  __shared__ double s_lo, s_hi;
  const int lane = threadIdx.x;  // 32 threads
  if (lane == 0) {
    double lo = DBL_MAX, hi = -DBL_MAX;
    for (int i = 0; i < m; ++i) {
      const double r = (i > 0 ? fabs(off[i - 1]) : 0.0) + (i + 1 < m ? fabs(off[i]) : 0.0);
      lo = fmin(lo, dgl[i] - r);
      hi = fmax(hi, dgl[i] + r);
    }
    s_lo = lo;
    s_hi = hi;
  }
  __syncwarp();
  double lo = s_lo, hi = s_hi;
  for (int it = 0; it < 40; ++it) {
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const bool all_below = sturm_count(dgl, off, m, x) == m;  // lambda_max < x
    const unsigned bal = __ballot_sync(0xffffffffu, all_below);
    double nlo = lo, nhi = hi;
    if (bal) {
      const int t = __ffs(bal) - 1;  // first probe above lambda_max
      nhi = lo + (hi - lo) * (double)(t + 1) / 33.0;
      nlo = t > 0 ? lo + (hi - lo) * (double)t / 33.0 : lo;
    } else {
      nlo = lo + (hi - lo) * 32.0 / 33.0;
    }
    if (!(nhi - nlo < hi - lo)) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) {
    out[0] = hi;
    out[1] = (double)(m - sturm_count(dgl, off, m, x_count));
  }
}

// pass = [ tau I - S^(r) is positive definite ], S^(r) the Schur complement of
// Kp after r threshold-pivoted elimination steps.  SM: work matrix in shared
// memory, else in the m x m global scratch Wg.
template <bool SM>
__global__ void __launch_bounds__(AT) schur_test_kernel(const double* __restrict__ Kp, int m,
                                                        const int* __restrict__ rlist, double thr,
                                                        double tau, double* Wg, int* pass) {
  extern __shared__ double dsm[];
  __shared__ double s_piv;
  __shared__ int s_ok;
  const int r = rlist[blockIdx.x];
  double* W = SM ? dsm : Wg + (int64_t)blockIdx.x * m * m;
  pass += blockIdx.x;
  const int tid = threadIdx.x;
  for (int64_t e = tid; e < (int64_t)m * m; e += AT) W[e] = Kp[e];
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    const double pj = W[(int64_t)j * m + j];
    if (!(pj > thr)) continue;  // exhausted column (uniform across the CTA)
    for (int i = j + 1 + (tid >> 5); i < m; i += AT / 32) {
      const double wij = W[(int64_t)i * m + j];
      for (int t = j + 1 + (tid & 31); t < m; t += 32)
        W[(int64_t)i * m + t] -= (wij * W[(int64_t)j * m + t]) / pj;
    }
    __syncthreads();
  }
  // Cholesky of C = tau I - W[r:, r:] (stored in place: W[i][j] <- l_ij below the diagonal)
  for (int j = r; j < m; ++j) {
    if (tid == 0) {
      const double c = tau - W[(int64_t)j * m + j];
      if (!(c > 0.0)) s_ok = 0;
      s_piv = c > 0.0 ? sqrt(c) : 1.0;
    }
    __syncthreads();
    if (!s_ok) break;
    const double piv = s_piv;
    for (int i = j + 1 + tid; i < m; i += AT) W[(int64_t)i * m + j] = -W[(int64_t)i * m + j] / piv;
    __syncthreads();
    // C[i][t] -= l_i l_t  <=>  W[i][t] += l_i l_t  (lower part, incl. the diagonal)
    for (int i = j + 1 + (tid >> 5); i < m; i += AT / 32) {
      const double li = W[(int64_t)i * m + j];
      for (int t = j + 1 + (tid & 31); t <= i; t += 32)
        W[(int64_t)i * m + t] += li * W[(int64_t)t * m + j];
    }
    __syncthreads();
  }
  if (tid == 0) *pass = s_ok;
}


}  // namespace

#define TRY_A(x)                  \
  do {                            \
    afn_status s_ = (x);          \
    if (s_ != AFN_OK) return s_;  \
  } while (0)

afn_status launch_tridiag(double* A, int m, double* dgl, double* off, cudaStream_t st) {
  // one CTA of 1024 threads (0.75 ms at m = 163; 512 and 256 threads measured slower: 256 1.14 ms)
  if (m <= SM_MAX_M) {
    // (+ the column partials of p: <= 1024 doubles; 164^2 + 2 164 + 1024 doubles <= 227 KB)
    const size_t bytes = sizeof(double) * ((size_t)m * m + 2 * (size_t)m + 1024);
    AFN_CUDA(cudaFuncSetAttribute(tridiag_kernel<true, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    tridiag_kernel<true, 1024><<<1, 1024, bytes, st>>>(A, m, dgl, off);
  } else {
    tridiag_kernel<false, 1024><<<1, 1024, sizeof(double) * 2 * (size_t)m, st>>>(A, m, dgl, off);
  }
  AFN_LAUNCH_CHECK("tridiag_kernel");
  return AFN_OK;
}

// Uniform random landmarks (reading R29): the k indices with the
// smallest splitmix64 keys h_i = splitmix64(seed ^ i*golden), in key order.
afn_status uniform_landmarks(int64_t n, int64_t k, uint64_t seed, int64_t* idx, cudaStream_t st) {
  if (k < 1 || k > n || k > (1LL << 22)) {
    set_error("uniform landmarks: need 1 <= k <= min(n, 2^22)");
    return AFN_ERR_ARG;
  }
  int64_t P = 1024;
  while (P < k + 8 * (int64_t)std::sqrt((double)k) + 64) P <<= 1;
  P = std::min<int64_t>(P << 1, 1LL << 23);  // slack for the threshold search
  unsigned long long *keys = nullptr, *cnt = nullptr;
  long long* ids = nullptr;
  afn_status s = dalloc((void**)&keys, sizeof(unsigned long long) * P, st);
  if (s == AFN_OK) s = dalloc((void**)&ids, sizeof(long long) * P, st);
  if (s == AFN_OK) s = dalloc((void**)&cnt, sizeof(unsigned long long), st);
  struct Free {
    void* p[3];
    cudaStream_t st;
    ~Free() { for (void* q : p) dfree(q, st); }
  } fr{{keys, ids, cnt}, st};
  if (s != AFN_OK) return s;
  long double frac = std::min<long double>(1.0L, ((long double)k + 4.0L * std::sqrt((long double)k) + 32.0L) / n);
  for (int attempt = 0;; ++attempt) {
    const long double tl = frac * 18446744073709551616.0L;
    const uint64_t thr = (frac >= 1.0L || tl >= 18446744073709551615.0L) ? ~0ULL : (uint64_t)tl;
    AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    cand_cap_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, seed, thr, P, keys, ids, cnt);
    AFN_LAUNCH_CHECK("cand_cap_kernel");
    unsigned long long hc = 0;
    AFN_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)hc >= k && (int64_t)hc <= P) break;
    if (attempt > 200 || (thr == ~0ULL && (int64_t)hc < k)) {
      set_error("uniform landmarks: selection failed");
      return AFN_ERR_CUDA;
    }
    frac = (int64_t)hc < k ? std::min<long double>(1.0L, frac * 1.25L) : frac * 0.8L;
  }
  bitonic_global_kernel<<<1, AT, 0, st>>>(keys, ids, cnt, P, k, idx);
  AFN_LAUNCH_CHECK("bitonic_global_kernel");
  return AFN_OK;
}

int alg1_default_m(int64_t n) {
  int64_t m = std::min<int64_t>(500, std::max<int64_t>(100, n / 100));
  return (int)std::min<int64_t>(m, n);
}

namespace {
cudaStream_t alg1_stream() {  // per device and host thread
  static thread_local cudaStream_t a1[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!a1[dev]) cudaStreamCreateWithFlags(&a1[dev], cudaStreamNonBlocking);
  return a1[dev];
}
}  // namespace

afn_status alg1_run(const double* X, int64_t n, int d, Kern kn, int m, uint64_t rng_seed,
                    int k_threshold, Alg1Result* res, cudaStream_t st) {
  if (m < 2 || m > 1024 || m > n) {
    set_error("alg1: need 2 <= m <= min(n, 1024) (m=%d)", m);
    return AFN_ERR_ARG;
  }
  std::vector<void*> tmp;
  auto get = [&](void** p, size_t bytes) {
    afn_status s = dalloc(p, bytes, st);
    if (s == AFN_OK) tmp.push_back(*p);
    return s;
  };
  struct Free {
    std::vector<void*>* t;
    cudaStream_t st;
    ~Free() {
      for (void* p : *t) dfree(p, st);
    }
  } fr{&tmp, st};
  afn_status s;
  unsigned long long* keys;
  long long* cids;
  unsigned* cnt;
  int64_t* ids;
  if ((s = get((void**)&keys, sizeof(unsigned long long) * CAND_CAP)) != AFN_OK) return s;
  if ((s = get((void**)&cids, sizeof(long long) * CAND_CAP)) != AFN_OK) return s;
  if ((s = get((void**)&cnt, sizeof(unsigned) * 4)) != AFN_OK) return s;
  if ((s = get((void**)&ids, sizeof(int64_t) * m)) != AFN_OK) return s;

  // ---- 1. subsample: keys below thr contain the m smallest iff count >= m
  {
    long double frac = (long double)std::min<int64_t>(n, 2LL * m + 64) / (long double)n;
    for (int attempt = 0; attempt < 64; ++attempt) {
      const long double tl = frac * 18446744073709551616.0L;
      const uint64_t thr = (frac >= 1.0L || tl >= 18446744073709551615.0L) ? ~0ULL : (uint64_t)tl;
      AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned), st));
      cand_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, rng_seed, thr, keys, cids, cnt);
      AFN_LAUNCH_CHECK("cand_kernel");
      unsigned hc = 0;
      AFN_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
      AFN_CUDA(cudaStreamSynchronize(st));
      if (thr == ~0ULL && hc < (unsigned)m) { set_error("alg1: subsample failed"); return AFN_ERR_CUDA; }
      if (hc < (unsigned)m) { frac *= 2; continue; }
      if (hc > (unsigned)CAND_CAP) { frac *= 0.5L; continue; }
      break;
    }
    const int sbytes = (int)(16 * CAND_CAP);
    AFN_CUDA(cudaFuncSetAttribute(cand_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes));
    cand_sort_kernel<<<1, AT, sbytes, st>>>(keys, cids, cnt, m, ids);
    AFN_LAUNCH_CHECK("cand_sort_kernel");
  }
  // ---- 2. scaled / unscaled subsample, K_m, FPS order
  const double scale = std::pow((double)m / (double)n, 1.0 / (double)d);
  double *Xm, *Xu, *Km, *Kp, *Wk, *dgl, *off, *summ;
  int64_t* ord;
  double* fill;
  int* pass;
  const size_t mm = (size_t)m * m;
  if ((s = get((void**)&Xm, sizeof(double) * m * d)) != AFN_OK) return s;
  if ((s = get((void**)&Xu, sizeof(double) * m * d)) != AFN_OK) return s;
  if ((s = get((void**)&Km, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&Kp, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&Wk, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&dgl, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&off, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&summ, sizeof(double) * 4)) != AFN_OK) return s;
  if ((s = get((void**)&ord, sizeof(int64_t) * m)) != AFN_OK) return s;
  if ((s = get((void**)&fill, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&pass, sizeof(int) * 2)) != AFN_OK) return s;
  double *Wk2, *dgl2, *off2, *summ2;  // the refinement's (unscaled K_m) eigen-summary
  if ((s = get((void**)&Wk2, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&dgl2, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&off2, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&summ2, sizeof(double) * 4)) != AFN_OK) return s;
  gather_scale_kernel<<<(m * d + 255) / 256, 256, 0, st>>>(X, d, ids, m, scale, Xm, Xu);
  AFN_LAUNCH_CHECK("gather_scale_kernel");
  if ((s = gen_k11(Xm, m, d, kn, 0.0, Km, st)) != AFN_OK) return s;
  // Concurrently on a second stream: FPS order of X_m and the permuted K_m
  // (needed by the Schur tests), then -- speculatively, it only matters when
  // khat < k_threshold -- the eigen-summary of the unscaled K_m for the
  // refinement.  The main stream computes ||K_m||_2 meanwhile.
  cudaStream_t s3 = alg1_stream();
  cudaEvent_t eA = nullptr, eP = nullptr, eR = nullptr;
  AFN_CUDA(cudaEventCreateWithFlags(&eA, cudaEventDisableTiming));
  AFN_CUDA(cudaEventCreateWithFlags(&eP, cudaEventDisableTiming));
  AFN_CUDA(cudaEventCreateWithFlags(&eR, cudaEventDisableTiming));
  struct EvF {
    cudaEvent_t a, b, c;
    cudaStream_t st;
    ~EvF() {
      cudaStreamWaitEvent(st, c, 0);  // (the temporaries are freed in st's order)
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaEventDestroy(c);
    }
  } evf{eA, eP, eR, st};
  AFN_CUDA(cudaEventRecord(eA, st));
  AFN_CUDA(cudaStreamWaitEvent(s3, eA, 0));
  if ((s = fps_run(Xm, m, d, m, 0, ord, fill, s3)) != AFN_OK) return s;
  permute_sym_kernel<<<(unsigned)((mm + 255) / 256), 256, 0, s3>>>(Km, m, ord, Kp);
  AFN_LAUNCH_CHECK("permute_sym_kernel");
  AFN_CUDA(cudaEventRecord(eP, s3));
  if ((s = gen_k11(Xu, m, d, kn, 0.0, Wk2, s3)) != AFN_OK) return s;
  TRY_A(launch_tridiag(Wk2, m, dgl2, off2, s3));
  eig_summary_kernel<<<1, 32, 0, s3>>>(dgl2, off2, m, 0.1, summ2);
  AFN_LAUNCH_CHECK("eig_summary_kernel");
  AFN_CUDA(cudaEventRecord(eR, s3));
  // ||K_m||_2 = lambda_max (tridiagonal + bisection)
  AFN_CUDA(cudaMemcpyAsync(Wk, Km, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
  TRY_A(launch_tridiag(Wk, m, dgl, off, st));
  eig_summary_kernel<<<1, 32, 0, st>>>(dgl, off, m, 0.1, summ);
  AFN_LAUNCH_CHECK("eig_summary_kernel");
  double hs[2];
  AFN_CUDA(cudaMemcpyAsync(hs, summ, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  const double normK = hs[0];
  const double thr = (double)m * DBL_EPSILON * normK;
  const double tau = 0.1 * normK;

  // ---- 3. smallest r in [1, m] with ||S^(r)|| < 0.1 ||K_m|| (pass(m) = true).
  // Multisection: up to 32 probes per round run as independent CTAs.
  AFN_CUDA(cudaStreamWaitEvent(st, eP, 0));  // K_p from the second stream
  constexpr int NPROBE = 32;
  int* rdev;
  int* pdev;
  double* Wp = nullptr;
  if ((s = get((void**)&rdev, sizeof(int) * NPROBE)) != AFN_OK) return s;
  if ((s = get((void**)&pdev, sizeof(int) * NPROBE)) != AFN_OK) return s;
  if (m > SM_MAX_M && (s = get((void**)&Wp, sizeof(double) * mm * NPROBE)) != AFN_OK) return s;
  const size_t smb = sizeof(double) * mm;
  if (m <= SM_MAX_M)
    AFN_CUDA(cudaFuncSetAttribute(schur_test_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
  int lo = 0, hi = m;  // pass(hi) true, pass(lo) false (lo = 0: no landmarks)
  while (hi - lo > 1) {
    int rs[NPROBE];
    int np = 0;
    const int span = hi - lo;
    const int want = std::min(NPROBE, span - 1);
    for (int j = 1; j <= want; ++j) {
      const int r = lo + (int)(((int64_t)j * span) / (want + 1));
      if (r > lo && r < hi && (np == 0 || r != rs[np - 1])) rs[np++] = r;
    }
    AFN_CUDA(cudaMemcpyAsync(rdev, rs, sizeof(int) * np, cudaMemcpyHostToDevice, st));
    if (m <= SM_MAX_M) schur_test_kernel<true><<<np, AT, smb, st>>>(Kp, m, rdev, thr, tau, Wk, pdev);
    else schur_test_kernel<false><<<np, AT, 0, st>>>(Kp, m, rdev, thr, tau, Wp, pdev);
    AFN_LAUNCH_CHECK("schur_test_kernel");
    int ok[NPROBE];
    AFN_CUDA(cudaMemcpyAsync(ok, pdev, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    int first = np;
    for (int j = 0; j < np; ++j)
      if (ok[j]) { first = j; break; }
    if (first < np) hi = rs[first];
    if (first > 0) lo = rs[first - 1];
  }
  const int r = hi;
  int64_t khat = (2LL * r * n + m) / (2LL * m);
  int refined = 0;
  // ---- 4. refined branch: #{eig(K_m on unscaled points) > 0.1}
  if (khat < k_threshold) {  // (eigen-summary computed above on the second stream)
    AFN_CUDA(cudaStreamWaitEvent(st, eR, 0));
    AFN_CUDA(cudaMemcpyAsync(hs, summ2, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    khat = (int64_t)hs[1];
    refined = 1;
  }
  res->khat = khat;
  res->r = r;
  res->m = m;
  res->refined = refined;
  res->scale = scale;
  return AFN_OK;
}

}  // namespace afn

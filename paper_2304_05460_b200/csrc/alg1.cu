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

// lambda_max of the symmetric m x m A (global, L2-resident) by Lanczos from
// the all-ones start vector (it overlaps the positive Perron vector of a
// kernel matrix) with full reorthogonalisation (classical Gram-Schmidt
// twice), one CTA.  Every 8 steps the largest eigenvalue of the Lanczos
// tridiagonal T_j is found by 32-way multisection on Sturm counts; the run
// stops when it has changed by less than 4e-15 relative over three
// consecutive checks, when beta_{j+1} <= m eps max|alpha| (an invariant
// subspace: it contains the start vector's component along the top
// eigenvector), or at j = m (T_m is then similar to A).  Q: m x (m + 1) scratch, column-major.  out[0] = lambda_max,
// out[1] = steps.  (Replaces a Householder tridiagonalisation, 500 dependent
// steps over the whole matrix at m = 500: 20 ms.)
constexpr int LZ_T = 1024;
__device__ int sturm_count_lz(const double* al, const double* be, int n, double x) {
  int c = 0;
  double q = al[0] - x;
  if (q < 0.0) ++c;
  for (int i = 1; i < n; ++i) {
    const double qq = (q != 0.0) ? q : DBL_MIN * 4.0;
    q = al[i] - x - be[i] * be[i] / qq;  // be[i] couples i-1 and i
    if (q < 0.0) ++c;
  }
  return c;
}
__global__ void __launch_bounds__(LZ_T) lanczos_max_kernel(const double* __restrict__ A, int m, double* Q,
                                                           double* out) {
  __shared__ double s_q[1024], s_w[1024], s_al[1025], s_be[1025], s_c[1025];
  __shared__ double sh[32];
  __shared__ double s_theta, s_lo, s_hi, s_amax;
  __shared__ int s_stop;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double q0 = rsqrt((double)m);
  for (int i = tid; i < m; i += LZ_T) {
    s_q[i] = q0;
    Q[i] = q0;
  }
  if (tid == 0) {
    s_be[0] = 0.0;
    s_theta = 0.0;
    s_amax = 0.0;
    s_stop = 0;
  }
  __syncthreads();
  double theta_prev = -1.0;
  int stable = 0, j = 0;
  for (j = 0; j < m; ++j) {
    // w = A q_j (warp per row, lanes over the columns)
    for (int i = wid; i < m; i += LZ_T / 32) {
      const double* row = A + (int64_t)i * m;
      double acc = 0.0;
      for (int t = lane; t < m; t += 32) acc = fma(row[t], s_q[t], acc);
      acc = warp_sum(acc);
      if (lane == 0) s_w[i] = acc;
    }
    __syncthreads();
    // alpha_j = q_j . w
    double loc = 0.0;
    for (int i = tid; i < m; i += LZ_T) loc = fma(s_q[i], s_w[i], loc);
    loc = warp_sum(loc);
    if (lane == 0) sh[wid] = loc;
    __syncthreads();
    if (wid == 0) {
      double r = sh[lane];
      r = warp_sum(r);
      if (lane == 0) s_al[j] = r;
    }
    __syncthreads();
    // full reorthogonalisation against q_0..q_j, classical Gram-Schmidt twice
    // (one pass also removes the alpha_j q_j and beta_j q_{j-1} components;
    // the second restores orthogonality after cancellation)
    double nrm = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int t = wid; t <= j; t += LZ_T / 32) {
        const double* qt = Q + (int64_t)t * m;
        double acc = 0.0;
        for (int i = lane; i < m; i += 32) acc = fma(qt[i], s_w[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) s_c[t] = acc;
      }
      __syncthreads();
      nrm = 0.0;
      for (int i = tid; i < m; i += LZ_T) {
        double wi = s_w[i];
        for (int t = 0; t <= j; ++t) wi = fma(-s_c[t], Q[(int64_t)t * m + i], wi);
        s_w[i] = wi;
        nrm = fma(wi, wi, nrm);
      }
      __syncthreads();
    }
    nrm = warp_sum(nrm);
    if (lane == 0) sh[wid] = nrm;
    __syncthreads();
    if (wid == 0) {
      double r = sh[lane];
      r = warp_sum(r);
      if (lane == 0) {
        s_be[j + 1] = sqrt(r);
        s_amax = fmax(s_amax, fabs(s_al[j]));
      }
    }
    __syncthreads();
    const double beta = s_be[j + 1];
    // (an invariant subspace: beta tiny against max |alpha_i| <= lambda_max)
    const bool exhausted = !(beta > (double)m * DBL_EPSILON * s_amax);
    const bool check = ((j + 1) % 8 == 0) || j + 1 == m || exhausted;
    if (check && wid == 0) {  // theta = lambda_max(T_{j+1}) by multisection
      const int nt = j + 1;
      if (lane == 0) {
        double lo = DBL_MAX, hi = -DBL_MAX;
        for (int i = 0; i < nt; ++i) {
          const double r = (i > 0 ? fabs(s_be[i]) : 0.0) + (i + 1 < nt ? fabs(s_be[i + 1]) : 0.0);
          lo = fmin(lo, s_al[i] - r);
          hi = fmax(hi, s_al[i] + r);
        }
        s_lo = lo;
        s_hi = hi;
      }
      __syncwarp();
      double lo = s_lo, hi = s_hi;
      for (int it = 0; it < 40; ++it) {
        const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
        const bool all_below = sturm_count_lz(s_al, s_be, nt, x) == nt;
        const unsigned bal = __ballot_sync(0xffffffffu, all_below);
        double nlo = lo, nhi = hi;
        if (bal) {
          const int t = __ffs(bal) - 1;
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
        const double th = hi;
        stable = (theta_prev > 0.0 && fabs(th - theta_prev) <= 4e-15 * th) ? stable + 1 : 0;
        theta_prev = th;
        s_theta = th;
        if (stable >= 3 || j + 1 == m || exhausted) s_stop = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
    const double inv = 1.0 / beta;
    for (int i = tid; i < m; i += LZ_T) {
      const double qi = s_w[i] * inv;
      s_q[i] = qi;
      Q[(int64_t)(j + 1) * m + i] = qi;
    }
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = s_theta;
    out[1] = (double)(j + 1);
  }
}

// Probe matrices of the Schur tests (batch b = probe with r = rlist[b]):
//   C_b = diag(tau I_r, tau I - Kp[r:, r:] + G_b),  G_b = L[r:, :r] L[r:, :r]^T
// (G_b already in C_b's trailing block).  tau I - S^(r) is positive definite
// iff C_b is (S^(r) = Kp[r:, r:] - L21 L21^T, the Schur complement after r
// threshold-pivoted steps).  Lower triangle only.
__global__ void form_probe_kernel(const double* __restrict__ Kp, int m, const int* __restrict__ rlist, double tau,
                                  double* __restrict__ C) {
  const int b = blockIdx.y;
  const int r = rlist[b];
  double* Cb = C + (int64_t)b * m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)m * m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / m), t = (int)(e - (int64_t)i * m);
    if (t > i) continue;
    double v = (i == t) ? tau : 0.0;
    if (i >= r && t >= r) v = v - Kp[e] + Cb[e];
    Cb[e] = v;
  }
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
  double *Xm, *Xu, *Km, *Kp, *Lq, *Lt, *dgl2, *off2, *summ, *summ2, *Wk2;
  int64_t* ord;
  double* fill;
  int* pinfo;
  const size_t mm = (size_t)m * m;
  if ((s = get((void**)&Xm, sizeof(double) * m * d)) != AFN_OK) return s;
  if ((s = get((void**)&Xu, sizeof(double) * m * d)) != AFN_OK) return s;
  if ((s = get((void**)&Km, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&Kp, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&Lq, sizeof(double) * (mm + m))) != AFN_OK) return s;  // Lanczos Q, then L
  if ((s = get((void**)&Lt, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&Wk2, sizeof(double) * mm)) != AFN_OK) return s;
  if ((s = get((void**)&dgl2, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&off2, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&summ, sizeof(double) * 4)) != AFN_OK) return s;
  if ((s = get((void**)&summ2, sizeof(double) * 4)) != AFN_OK) return s;
  if ((s = get((void**)&ord, sizeof(int64_t) * m)) != AFN_OK) return s;
  if ((s = get((void**)&fill, sizeof(double) * m)) != AFN_OK) return s;
  if ((s = get((void**)&pinfo, sizeof(int) * 64)) != AFN_OK) return s;
  gather_scale_kernel<<<(m * d + 255) / 256, 256, 0, st>>>(X, d, ids, m, scale, Xm, Xu);
  AFN_LAUNCH_CHECK("gather_scale_kernel");
  if ((s = gen_k11(Xm, m, d, kn, 0.0, Km, st)) != AFN_OK) return s;
  // Concurrently on a second stream: the FPS order of X_m and the permuted
  // K_m (the Schur tests need them), then -- speculatively, when it is cheap
  // (shared-memory tridiagonalisation, m <= SM_MAX_M) -- the eigen-summary
  // of the unscaled K_m for the refinement.  The main stream
  // computes ||K_m||_2 meanwhile.
  const bool spec = m <= SM_MAX_M;
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
  auto refine_summary = [&](cudaStream_t ss) -> afn_status {
    TRY_A(gen_k11(Xu, m, d, kn, 0.0, Wk2, ss));
    TRY_A(launch_tridiag(Wk2, m, dgl2, off2, ss));
    eig_summary_kernel<<<1, 32, 0, ss>>>(dgl2, off2, m, 0.1, summ2);
    AFN_LAUNCH_CHECK("eig_summary_kernel");
    return AFN_OK;
  };
  if (spec) TRY_A(refine_summary(s3));
  AFN_CUDA(cudaEventRecord(eR, s3));
  // ||K_m||_2 = lambda_max (Lanczos)
  lanczos_max_kernel<<<1, LZ_T, 0, st>>>(Km, m, Lq, summ);
  AFN_LAUNCH_CHECK("lanczos_max_kernel");
  double hs[2];
  AFN_CUDA(cudaMemcpyAsync(hs, summ, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  const double normK = hs[0];
  const double thr = (double)m * DBL_EPSILON * normK;
  const double tau = 0.1 * normK;

  // ---- 3. smallest r in [1, m] with ||S^(r)|| < 0.1 ||K_m|| (pass(m) = true).
  // L = threshold-pivoted Cholesky factor of K_p (FPS order; pivots <= thr
  // leave zero columns, R10) once; a probe r forms S^(r) = K_p[r:, r:] -
  // L[r:, :r] L[r:, :r]^T (DMMA GEMM) and tests tau I - S^(r) by a Cholesky
  // attempt; up to NPROBE probes per multisection round in one batched
  // factorisation.
  AFN_CUDA(cudaStreamWaitEvent(st, eP, 0));  // K_p from the second stream
  AFN_CUDA(cudaMemcpyAsync(Lq, Kp, sizeof(double) * mm, cudaMemcpyDeviceToDevice, st));
  TRY_A(potrf_batched(Lq, m, 1, 0, thr, pinfo, st));
  TRY_A(transpose_sq(Lq, m, Lt, st));
  constexpr int NPROBE = 32;
  int* rdev;
  double* Cp;
  if ((s = get((void**)&rdev, sizeof(int) * NPROBE)) != AFN_OK) return s;
  if ((s = get((void**)&Cp, sizeof(double) * mm * NPROBE)) != AFN_OK) return s;
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
    for (int b = 0; b < np; ++b) {  // G_b = L21 L21^T into C_b's trailing block
      const int r = rs[b];
      TRY_A(gemm_nn(Lq + (size_t)r * m, Lt + r, Cp + (size_t)b * mm + (size_t)r * m + r, m - r, m - r, r, m, m, m,
                    1.0, st));
    }
    const unsigned gx = (unsigned)std::min<size_t>((mm + 255) / 256, 1024);
    form_probe_kernel<<<dim3(gx, np), 256, 0, st>>>(Kp, m, rdev, tau, Cp);
    AFN_LAUNCH_CHECK("form_probe_kernel");
    TRY_A(potrf_batched(Cp, m, np, (int64_t)mm, -1.0, pinfo, st));
    int ok[NPROBE];
    AFN_CUDA(cudaMemcpyAsync(ok, pinfo, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    int first = np;
    for (int j = 0; j < np; ++j)
      if (ok[j] == 0) { first = j; break; }  // (info 0: factorised -> positive definite)
    if (first < np) hi = rs[first];
    if (first > 0) lo = rs[first - 1];
  }
  const int r = hi;
  int64_t khat = (2LL * r * n + m) / (2LL * m);
  int refined = 0;
  // ---- 4. refined branch: #{eig(K_m on unscaled points) > 0.1}
  if (khat < k_threshold) {
    if (spec) {
      AFN_CUDA(cudaStreamWaitEvent(st, eR, 0));
    } else {
      TRY_A(refine_summary(st));
    }
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

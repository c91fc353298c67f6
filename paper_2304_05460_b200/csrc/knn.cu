// knn.cu -- FSAI sparsity pattern: row i holds i plus the
// w-1 nearest neighbours of point i "that are numbered less than i".
//
// One warp per row, 8 consecutive rows per CTA sharing shared-memory tiles of
// candidate points.  Each warp keeps a buffer of candidates whose key
// (d2, j) beats the current threshold (the (w-1)-th best seen so far); when the
// buffer fills it is bitonic-sorted and truncated.  The kept set is the unique
// set of the w-1 smallest keys in the total order (d2, j), so the result is
// bit-exact and independent of scan order (readings R3, R15).
#include <algorithm>
#include <cfloat>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int KNN_NW = 8;     // warps (rows) per CTA
constexpr int KNN_CAP = 256;  // candidate buffer per warp (w-1 <= 127)

__device__ __forceinline__ bool key_less(double da, int ja, double db, int jb) {
  return da < db || (da == db && ja < jb);
}

// bitonic sort of CAP (d2, j) pairs ascending, one warp
__device__ void warp_bitonic(double* key, int* idx) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= KNN_CAP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < KNN_CAP; t += 32) {
        const int p = t ^ j;
        if (p > t) {
          const bool up = (t & k) == 0;
          const double a = key[t], b = key[p];
          const int ia = idx[t], ib = idx[p];
          const bool gt = key_less(b, ib, a, ia);  // a > b
          if (gt == up) {
            key[t] = b; key[p] = a;
            idx[t] = ib; idx[p] = ia;
          }
        }
      }
      __syncwarp();
    }
  }
}

// ascending sort of CAP ints (INT_MAX padding), one warp
__device__ void warp_bitonic_int(int* v) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= KNN_CAP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < KNN_CAP; t += 32) {
        const int p = t ^ j;
        if (p > t) {
          const bool up = (t & k) == 0;
          const int a = v[t], b = v[p];
          if ((a > b) == up) { v[t] = b; v[p] = a; }
        }
      }
      __syncwarp();
    }
  }
}

template <int DP>
__global__ void __launch_bounds__(KNN_NW * 32)
knn_kernel(const double* __restrict__ P, int64_t row_lo, int64_t row_hi, int d, int w,
           int32_t* __restrict__ col) {
  constexpr int TILE = DP <= 4 ? 512 : (DP <= 8 ? 256 : 128);
  __shared__ double s_pts[TILE * DP];
  __shared__ double s_key[KNN_NW][KNN_CAP];
  __shared__ int s_idx[KNN_NW][KNN_CAP];

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // heaviest rows first (row i scans i candidates)
  const int64_t blk = (int64_t)gridDim.x - 1 - blockIdx.x;
  const int64_t i0 = row_lo + blk * KNN_NW;
  const int64_t i = i0 + wid;
  const bool active = i < row_hi;
  const int W1 = active ? (int)min((int64_t)w - 1, i) : 0;

  double q[DP];
#pragma unroll
  for (int c = 0; c < DP; ++c) q[c] = (active && c < d) ? P[i * d + c] : 0.0;

  double* key = s_key[wid];
  int* idx = s_idx[wid];
  int cnt = 0;
  double tau_d = DBL_MAX;
  int tau_j = 0x7fffffff;

  auto compact = [&]() {
    for (int t = cnt + lane; t < KNN_CAP; t += 32) { key[t] = DBL_MAX; idx[t] = 0x7fffffff; }
    __syncwarp();
    warp_bitonic(key, idx);
    cnt = min(cnt, W1);
    if (cnt == W1 && W1 > 0) { tau_d = key[W1 - 1]; tau_j = idx[W1 - 1]; }
    __syncwarp();
  };

  const int64_t jmax = min(row_hi, i0 + KNN_NW) - 1;  // largest candidate needed in this CTA
  for (int64_t tb = 0; tb < jmax; tb += TILE) {
    const int tn = (int)min((int64_t)TILE, jmax - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < tn * DP; e += KNN_NW * 32) {
      const int jj = e / DP, c = e - jj * DP;
      s_pts[e] = c < d ? P[(tb + jj) * d + c] : 0.0;
    }
    __syncthreads();
    if (W1 > 0) {
      const int lim = (int)min((int64_t)tn, i - tb);  // candidates j < i
      for (int base = 0; base < lim; base += 32) {
        if (cnt > KNN_CAP - 32) compact();
        const int jj = base + lane;
        bool take = false;
        double dd = 0.0;
        const int j = (int)(tb + jj);
        if (jj < lim) {
          dd = d2_exact<DP>(&s_pts[jj * DP], q);
          take = key_less(dd, j, tau_d, tau_j);
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (take) {
          const int pos = cnt + __popc(m & ((1u << lane) - 1u));
          key[pos] = dd;
          idx[pos] = j;
        }
        cnt += __popc(m);
        __syncwarp();
      }
    }
  }
  if (!active) return;
  if (W1 > 0) {
    compact();
    // ascending positions of the kept neighbours
    for (int t = lane; t < KNN_CAP; t += 32) {
      const int v = t < W1 ? idx[t] : 0x7fffffff;
      __syncwarp();
      idx[t] = v;
    }
    __syncwarp();
    warp_bitonic_int(idx);
  }
  // row_ptr(i) = sum_{t<i} min(w, t+1)
  const int64_t wl = w;
  const int64_t start = (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
  for (int t = lane; t < W1; t += 32) col[start + t] = idx[t];
  if (lane == 0) col[start + W1] = (int32_t)i;
}

__global__ void knn_rowptr_kernel(int64_t N, int w, int64_t* __restrict__ rp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > N) return;
  const int64_t wl = w;
  rp[i] = (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
}

template <int DP>
void launch_knn(const double* P, int64_t lo, int64_t hi, int d, int w, int32_t* col, cudaStream_t st) {
  const int64_t blocks = (hi - lo + KNN_NW - 1) / KNN_NW;
  knn_kernel<DP><<<(unsigned)blocks, KNN_NW * 32, 0, st>>>(P, lo, hi, d, w, col);
}

}  // namespace

int64_t knn_nnz(int64_t N, int w) {
  const int64_t wl = w;
  return (N < wl) ? N * (N + 1) / 2 : wl * (wl + 1) / 2 + (N - wl) * wl;
}

afn_status knn_run(const double* P, int64_t N, int d, int w, int64_t* row_ptr, int32_t* col,
                   cudaStream_t st, int64_t row_lo, int64_t row_hi) {
  if (row_hi < 0) row_hi = N;
  if (w < 1 || w > 128) {
    set_error("knn: w=%d unsupported (1..128)", w);
    return AFN_ERR_ARG;
  }
  if (N <= 0) return AFN_OK;
  knn_rowptr_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, st>>>(N, w, row_ptr);
  AFN_LAUNCH_CHECK("knn_rowptr_kernel");
  if (row_hi <= row_lo) return AFN_OK;
  const int64_t lo = row_lo, hi = row_hi;
  if (d <= 1) launch_knn<1>(P, lo, hi, d, w, col, st);
  else if (d <= 2) launch_knn<2>(P, lo, hi, d, w, col, st);
  else if (d <= 3) launch_knn<3>(P, lo, hi, d, w, col, st);
  else if (d <= 4) launch_knn<4>(P, lo, hi, d, w, col, st);
  else if (d <= 8) launch_knn<8>(P, lo, hi, d, w, col, st);
  else if (d <= 16) launch_knn<16>(P, lo, hi, d, w, col, st);
  else {
    set_error("knn: d=%d unsupported (1..16)", d);
    return AFN_ERR_ARG;
  }
  AFN_LAUNCH_CHECK("knn_kernel");
  return AFN_OK;
}

}  // namespace afn

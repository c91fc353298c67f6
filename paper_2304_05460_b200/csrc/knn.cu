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
#include <cmath>
#include <cstdlib>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int KNN_NW = 8;  // warps (rows) per CTA
// candidate buffer per warp (keys + indices in dynamic shared memory): a
// compaction keeps the w-1 best, so w - 1 + 32 <= CAP
constexpr int KNN_CAP_S = 256, KNN_CAP_L = 1024;
inline int knn_cap(int w) { return w - 1 + 32 <= KNN_CAP_S ? KNN_CAP_S : KNN_CAP_L; }
inline size_t knn_smem(int cap) { return (size_t)KNN_NW * cap * (sizeof(double) + sizeof(int)); }

__device__ __forceinline__ bool key_less(double da, int ja, double db, int jb) {
  return da < db || (da == db && ja < jb);
}

// bitonic sort of CAP (d2, j) pairs ascending, one warp
template <int KNN_CAP>
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
template <int KNN_CAP>
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

template <int DP, int KNN_CAP>
__global__ void __launch_bounds__(KNN_NW * 32)
knn_kernel(const double* __restrict__ P, int64_t row_lo, int64_t row_hi, int d, int w,
           int32_t* __restrict__ col) {
  constexpr int TILE = DP <= 4 ? 512 : (DP <= 8 ? 256 : 128);
  __shared__ double s_pts[TILE * DP];
  extern __shared__ double knn_dyn[];  // [KNN_NW][KNN_CAP] keys, then [KNN_NW][KNN_CAP] indices
  double(*s_key)[KNN_CAP] = reinterpret_cast<double(*)[KNN_CAP]>(knn_dyn);
  int(*s_idx)[KNN_CAP] = reinterpret_cast<int(*)[KNN_CAP]>(knn_dyn + KNN_NW * KNN_CAP);

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
    warp_bitonic<KNN_CAP>(key, idx);
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
    warp_bitonic_int<KNN_CAP>(idx);
  }
  // row_ptr(i) = sum_{t<i} min(w, t+1)
  const int64_t wl = w;
  const int64_t start = (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
  for (int t = lane; t < W1; t += 32) col[start + t] = idx[t];
  if (lane == 0) col[start + W1] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// Grid path (d = 3, large N).  Row i only needs the w-1 nearest among the
// EARLIER points j < i, so its search radius grows like (N/i)^(1/3): a warp
// scans the cells of a uniform grid that cover the cube [x - r - h, x + r + h]
// (h = cell edge), keeps the candidates j < i with the same threshold buffer as
// the brute-force kernel, and accepts when w-1 candidates were found with
// d2 < r^2 (1 - 1e-12): every point with a smaller key lies inside the scanned
// cells, so the kept set is the exact (d2, j) selection.  Otherwise r grows by
// 1.6x.  Rows whose cube would hold more points than i (small i) scan j < i
// directly.  Bit-identical to the brute-force kernel.
struct KnnGrid {
  double lo[3], inv_h, h;
  int g;  // cells per axis
};

__global__ void knn_cell_count_kernel(const double* __restrict__ P, int64_t N, KnnGrid G,
                                      int* __restrict__ cell, int* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int c3[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    int v = (int)((P[i * 3 + c] - G.lo[c]) * G.inv_h);
    c3[c] = v < 0 ? 0 : (v >= G.g ? G.g - 1 : v);
  }
  const int cid = (c3[2] * G.g + c3[1]) * G.g + c3[0];
  cell[i] = cid;
  atomicAdd(&cnt[cid], 1);
}

__global__ void knn_cell_scan_kernel(const int* __restrict__ cnt, int64_t M, int* __restrict__ start) {
  __shared__ int part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (M + 1023) / 1024;
  const int64_t b = tid * per, e = min(M, b + per);
  int s = 0;
  for (int64_t t = b; t < e; ++t) s += cnt[t];
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = tid > 0 ? part[tid - 1] : 0;
  for (int64_t t = b; t < e; ++t) {
    start[t] = run;
    run += cnt[t];
  }
  if (tid == 1023) start[M] = part[1023];
}

// cell-sorted points (coordinates + original position), positions within a
// cell in ascending order is not required (the selection is order-free)
__global__ void knn_cell_fill_kernel(const double* __restrict__ P, int64_t N, const int* __restrict__ cell,
                                     const int* __restrict__ start, int* __restrict__ cur,
                                     double4* __restrict__ cp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int c = cell[i];
  const int pos = start[c] + atomicAdd(&cur[c], 1);
  cp[pos] = make_double4(P[i * 3], P[i * 3 + 1], P[i * 3 + 2], __longlong_as_double((long long)i));
}

template <int KNN_CAP>
__global__ void __launch_bounds__(KNN_NW * 32)
knn_grid_kernel(const double* __restrict__ P, int64_t row_lo, int64_t row_hi, int64_t N, int w, KnnGrid G,
                const int* __restrict__ start, const double4* __restrict__ cp, int32_t* __restrict__ col) {
  extern __shared__ double knn_dyn[];
  double(*s_key)[KNN_CAP] = reinterpret_cast<double(*)[KNN_CAP]>(knn_dyn);
  int(*s_idx)[KNN_CAP] = reinterpret_cast<int(*)[KNN_CAP]>(knn_dyn + KNN_NW * KNN_CAP);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = row_lo + (int64_t)blockIdx.x * KNN_NW + wid;
  if (i >= row_hi) return;
  const int W1 = (int)min((int64_t)w - 1, i);
  double* key = s_key[wid];
  int* idx = s_idx[wid];
  const double q[3] = {P[i * 3], P[i * 3 + 1], P[i * 3 + 2]};
  int cnt = 0;
  double tau_d = DBL_MAX;
  int tau_j = 0x7fffffff;
  auto compact = [&]() {
    for (int t = cnt + lane; t < KNN_CAP; t += 32) { key[t] = DBL_MAX; idx[t] = 0x7fffffff; }
    __syncwarp();
    warp_bitonic<KNN_CAP>(key, idx);
    cnt = min(cnt, W1);
    if (cnt == W1 && W1 > 0) { tau_d = key[W1 - 1]; tau_j = idx[W1 - 1]; }
    __syncwarp();
  };
  auto offer = [&](bool valid, double dd, int j) {
    if (cnt > KNN_CAP - 32) compact();
    const bool take = valid && key_less(dd, j, tau_d, tau_j);
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int pos = cnt + __popc(m & ((1u << lane) - 1u));
      key[pos] = dd;
      idx[pos] = j;
    }
    cnt += __popc(m);
    __syncwarp();
  };
  if (W1 > 0) {
    // radius for ~2 w earlier points at the average density of the earlier points
    const double V = (double)G.g * G.g * G.g * G.h * G.h * G.h;
    double r = cbrt(2.0 * (double)w * V / (4.18879020478639 * (double)i));
    bool done = false;
    while (!done) {
      const int span = (int)ceil(r * G.inv_h) + 1;
      int lo3[3], hi3[3];
      int64_t ncell = 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        int cc = (int)((q[c] - G.lo[c]) * G.inv_h);
        cc = cc < 0 ? 0 : (cc >= G.g ? G.g - 1 : cc);
        lo3[c] = max(0, cc - span);
        hi3[c] = min(G.g - 1, cc + span);
        ncell *= (int64_t)(hi3[c] - lo3[c] + 1);
      }
      const int64_t est = (int64_t)((double)ncell * (double)N / ((double)G.g * G.g * G.g));
      cnt = 0;
      tau_d = DBL_MAX;
      tau_j = 0x7fffffff;
      if (est >= i || (lo3[0] == 0 && lo3[1] == 0 && lo3[2] == 0 && hi3[0] == G.g - 1 &&
                       hi3[1] == G.g - 1 && hi3[2] == G.g - 1)) {
        // brute force over j < i (small i, or the cube covers the grid)
        for (int64_t b = 0; b < i; b += 32) {
          const int64_t j = b + lane;
          double dd = 0.0;
          if (j < i) dd = d2_exact<3>(&P[j * 3], q);
          offer(j < i, dd, (int)j);
        }
        done = true;
      } else {
        // only keys inside the ball of radius r can be accepted at this radius
        // (the acceptance test below needs the (w-1)-th key inside it), so
        // they alone enter the buffer: far fewer compactions (C3 11.1 -> 6.8 ms)
        tau_d = r * r;
        for (int z = lo3[2]; z <= hi3[2]; ++z)
          for (int y = lo3[1]; y <= hi3[1]; ++y) {
            const int c0 = (z * G.g + y) * G.g;
            const int b = start[c0 + lo3[0]], e = start[c0 + hi3[0] + 1];
            for (int t = b; t < e; t += 32) {
              bool valid = false;
              double dd = 0.0;
              int j = 0;
              if (t + lane < e) {
                const double4 pt = cp[t + lane];
                j = (int)__double_as_longlong(pt.w);
                if (j < i) {
                  const double pp[3] = {pt.x, pt.y, pt.z};
                  dd = d2_exact<3>(pp, q);
                  valid = true;
                }
              }
              offer(valid, dd, j);
            }
          }
        compact();
        if (cnt == W1 && tau_d < r * r * (1.0 - 1e-12)) done = true;
        else r *= 1.6;
      }
    }
    compact();
    for (int t = lane; t < KNN_CAP; t += 32) {
      const int v = t < W1 ? idx[t] : 0x7fffffff;
      __syncwarp();
      idx[t] = v;
    }
    __syncwarp();
    warp_bitonic_int<KNN_CAP>(idx);
  }
  const int64_t wl = w;
  const int64_t start_i = (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
  for (int t = lane; t < W1; t += 32) col[start_i + t] = idx[t];
  if (lane == 0) col[start_i + W1] = (int32_t)i;
}

__global__ void knn_bbox_kernel(const double* __restrict__ P, int64_t N, double* __restrict__ box) {
  // one block: min / max per coordinate (exact: min/max are order-free)
  __shared__ double smin[3][256], smax[3][256];
  double mn[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, mx[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int64_t i = threadIdx.x; i < N; i += 256)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = P[i * 3 + c];
      mn[c] = fmin(mn[c], v);
      mx[c] = fmax(mx[c], v);
    }
#pragma unroll
  for (int c = 0; c < 3; ++c) { smin[c][threadIdx.x] = mn[c]; smax[c][threadIdx.x] = mx[c]; }
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        smin[c][threadIdx.x] = fmin(smin[c][threadIdx.x], smin[c][threadIdx.x + o]);
        smax[c][threadIdx.x] = fmax(smax[c][threadIdx.x], smax[c][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) { box[c] = smin[c][0]; box[3 + c] = smax[c][0]; }
}

afn_status knn_grid_run(const double* P, int64_t N, int w, int32_t* col, int64_t lo, int64_t hi,
                        cudaStream_t st) {
  double* box = nullptr;
  afn_status s = dalloc((void**)&box, sizeof(double) * 6, st);
  if (s != AFN_OK) return s;
  knn_bbox_kernel<<<1, 256, 0, st>>>(P, N, box);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { dfree(box, st); return cuda_status(e, "knn_bbox_kernel"); }
  note_launch();
  double hb[6];
  e = cudaMemcpyAsync(hb, box, sizeof(hb), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  dfree(box, st);
  if (e != cudaSuccess) return cuda_status(e, "knn bbox copy");
  KnnGrid G;
  G.g = std::max(1, (int)std::ceil(std::cbrt((double)N / 4.0)));
  double ext = 0.0;
  for (int c = 0; c < 3; ++c) ext = std::max(ext, hb[3 + c] - hb[c]);
  ext = ext > 0.0 ? ext * (1.0 + 1e-9) : 1.0;
  G.h = ext / G.g;
  G.inv_h = 1.0 / G.h;
  for (int c = 0; c < 3; ++c) G.lo[c] = hb[c];
  const int64_t M = (int64_t)G.g * G.g * G.g;
  int *cell = nullptr, *cntb = nullptr, *start = nullptr;
  double4* cp = nullptr;
  if ((s = dalloc((void**)&cell, sizeof(int) * N, st)) != AFN_OK) return s;
  if ((s = dalloc((void**)&cntb, sizeof(int) * 2 * M, st)) != AFN_OK) { dfree(cell, st); return s; }
  if ((s = dalloc((void**)&start, sizeof(int) * (M + 1), st)) != AFN_OK) { dfree(cell, st); dfree(cntb, st); return s; }
  if ((s = dalloc((void**)&cp, sizeof(double4) * N, st)) != AFN_OK) {
    dfree(cell, st); dfree(cntb, st); dfree(start, st);
    return s;
  }
  struct Free {
    void* p[4];
    cudaStream_t st;
    ~Free() { for (void* q : p) dfree(q, st); }
  } fr{{cell, cntb, start, cp}, st};
  AFN_CUDA(cudaMemsetAsync(cntb, 0, sizeof(int) * 2 * M, st));
  knn_cell_count_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(P, N, G, cell, cntb);
  AFN_LAUNCH_CHECK("knn_cell_count_kernel");
  knn_cell_scan_kernel<<<1, 1024, 0, st>>>(cntb, M, start);
  AFN_LAUNCH_CHECK("knn_cell_scan_kernel");
  knn_cell_fill_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(P, N, cell, start, cntb + M, cp);
  AFN_LAUNCH_CHECK("knn_cell_fill_kernel");
  const int64_t blocks = (hi - lo + KNN_NW - 1) / KNN_NW;
  const int cap = knn_cap(w);
  const size_t bytes = knn_smem(cap);
  if (cap == KNN_CAP_S) {
    knn_grid_kernel<KNN_CAP_S><<<(unsigned)blocks, KNN_NW * 32, bytes, st>>>(P, lo, hi, N, w, G, start, cp, col);
  } else {
    AFN_CUDA(cudaFuncSetAttribute(knn_grid_kernel<KNN_CAP_L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    knn_grid_kernel<KNN_CAP_L><<<(unsigned)blocks, KNN_NW * 32, bytes, st>>>(P, lo, hi, N, w, G, start, cp, col);
  }
  AFN_LAUNCH_CHECK("knn_grid_kernel");
  return AFN_OK;
}

__global__ void knn_rowptr_kernel(int64_t N, int w, int64_t* __restrict__ rp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > N) return;
  const int64_t wl = w;
  rp[i] = (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
}

template <int DP>
afn_status launch_knn(const double* P, int64_t lo, int64_t hi, int d, int w, int32_t* col, cudaStream_t st) {
  const int64_t blocks = (hi - lo + KNN_NW - 1) / KNN_NW;
  const int cap = knn_cap(w);
  const size_t bytes = knn_smem(cap);
  if (cap == KNN_CAP_S) {
    knn_kernel<DP, KNN_CAP_S><<<(unsigned)blocks, KNN_NW * 32, bytes, st>>>(P, lo, hi, d, w, col);
  } else {
    AFN_CUDA(cudaFuncSetAttribute(knn_kernel<DP, KNN_CAP_L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    knn_kernel<DP, KNN_CAP_L><<<(unsigned)blocks, KNN_NW * 32, bytes, st>>>(P, lo, hi, d, w, col);
  }
  AFN_LAUNCH_CHECK("knn_kernel");
  return AFN_OK;
}

}  // namespace

int64_t knn_nnz(int64_t N, int w) {
  const int64_t wl = w;
  return (N < wl) ? N * (N + 1) / 2 : wl * (wl + 1) / 2 + (N - wl) * wl;
}

afn_status knn_run(const double* P, int64_t N, int d, int w, int64_t* row_ptr, int32_t* col,
                   cudaStream_t st, int64_t row_lo, int64_t row_hi) {
  if (row_hi < 0) row_hi = N;
  if (w < 1 || w > AFN_W_MAX) {
    set_error("knn: w=%d unsupported (1..%d)", w, AFN_W_MAX);
    return AFN_ERR_ARG;
  }
  if (N <= 0) return AFN_OK;
  knn_rowptr_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, st>>>(N, w, row_ptr);
  AFN_LAUNCH_CHECK("knn_rowptr_kernel");
  if (row_hi <= row_lo) return AFN_OK;
  const int64_t lo = row_lo, hi = row_hi;
  constexpr int64_t grid_min = 50000;  // (grid path for d = 3 from here on; brute force below)
  if (d == 3 && N >= grid_min && w > 1) {
    afn_status s = knn_grid_run(P, N, w, col, lo, hi, st);
    if (s != AFN_OK) return s;
    return AFN_OK;
  }
  if (d <= 1) return launch_knn<1>(P, lo, hi, d, w, col, st);
  if (d <= 2) return launch_knn<2>(P, lo, hi, d, w, col, st);
  if (d <= 3) return launch_knn<3>(P, lo, hi, d, w, col, st);
  if (d <= 4) return launch_knn<4>(P, lo, hi, d, w, col, st);
  if (d <= 8) return launch_knn<8>(P, lo, hi, d, w, col, st);
  if (d <= 16) return launch_knn<16>(P, lo, hi, d, w, col, st);
  set_error("knn: d=%d unsupported (1..16)", d);
  return AFN_ERR_ARG;
}

}  // namespace afn

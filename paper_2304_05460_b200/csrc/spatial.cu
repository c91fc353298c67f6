// spatial.cu -- Morton (Z) order of a point set, shared by the cutoff kernel
// matvec (kmv.cu) and the cutoff W product (wcut.cu).  A grid of ~2 points per
// cell over the first min(d, 3) coordinates (cell edge from the bounding box),
// cells in Morton order, the points of a cell by ascending index: the order
// is a pure function of X (deterministic although the scatter uses atomics).
#include <algorithm>
#include <cmath>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

__global__ void kc_bbox_kernel(const double* __restrict__ X, int64_t n, int d, double* __restrict__ ws) {
  __shared__ double sm[6][256];
  const int dd = d < 3 ? d : 3;
  double v6[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < dd; ++c) {
      const double x = X[i * d + c];
      v6[c] = fmin(v6[c], x);
      v6[3 + c] = fmax(v6[3 + c], x);
    }
  for (int c = 0; c < 6; ++c) sm[c][threadIdx.x] = v6[c];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o)
      for (int c = 0; c < 6; ++c)
        sm[c][threadIdx.x] = c < 3 ? fmin(sm[c][threadIdx.x], sm[c][threadIdx.x + o])
                                   : fmax(sm[c][threadIdx.x], sm[c][threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x < 6) ws[blockIdx.x * 6 + threadIdx.x] = sm[threadIdx.x][0];
}

struct KcGrid {
  int dd, bits, g;
  double lo[3], inv[3];
};

__global__ void kc_key_kernel(const double* __restrict__ X, int64_t n, int d, KcGrid gd, unsigned* __restrict__ key,
                              int* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned c[3] = {0u, 0u, 0u};
  for (int q = 0; q < gd.dd; ++q) {
    int v = (int)((X[i * d + q] - gd.lo[q]) * gd.inv[q]);
    c[q] = (unsigned)(v < 0 ? 0 : (v >= gd.g ? gd.g - 1 : v));
  }
  unsigned k = 0u;
  for (int b = 0; b < gd.bits; ++b)
    for (int q = 0; q < gd.dd; ++q) k |= ((c[q] >> b) & 1u) << (b * gd.dd + q);
  key[i] = k;
  atomicAdd(&cnt[k], 1);
}

// exclusive scan of M ints into off[0..M] (int64), one block of 1024
__global__ void kc_scan_kernel(const int* __restrict__ cnt, int64_t M, int64_t* __restrict__ off) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (M + 1023) / 1024;
  const int64_t b = tid * per, e = min(M, b + per);
  int64_t s = 0;
  for (int64_t t = b; t < e; ++t) s += cnt[t];
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int64_t run = tid > 0 ? part[tid - 1] : 0;
  for (int64_t t = b; t < e; ++t) {
    off[t] = run;
    run += cnt[t];
  }
  if (tid == 1023) off[M] = part[1023];
}

__global__ void kc_scatter_kernel(const unsigned* __restrict__ key, int64_t n, const int64_t* __restrict__ off,
                                  int* __restrict__ cur, int* __restrict__ sidx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned k = key[i];
  sidx[off[k] + atomicAdd(&cur[k], 1)] = (int)i;
}

// within a cell: ascending original index (the atomics' order is not fixed)
__global__ void kc_cell_sort_kernel(const int64_t* __restrict__ off, int64_t M, int* __restrict__ sidx) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= M) return;
  const int64_t b = off[c], e = off[c + 1];
  for (int64_t i = b + 1; i < e; ++i) {
    const int v = sidx[i];
    int64_t j = i - 1;
    while (j >= b && sidx[j] > v) {
      sidx[j + 1] = sidx[j];
      --j;
    }
    sidx[j + 1] = v;
  }
}

}  // namespace

afn_status scan_i32_i64(const int* cnt, int64_t M, int64_t* off, cudaStream_t st) {
  kc_scan_kernel<<<1, 1024, 0, st>>>(cnt, M, off);
  AFN_LAUNCH_CHECK("kc_scan_kernel");
  return AFN_OK;
}

afn_status morton_order(const double* X, int64_t n, int d, int* sidx, cudaStream_t st) {
  const int nbb = num_sms();
  const int dd = std::min(d, 3);
  std::vector<void*> tmp;
  auto get = [&](void** p, size_t bytes) {
    afn_status s = dalloc(p, bytes, st);
    if (s == AFN_OK) tmp.push_back(*p);
    return s;
  };
  struct Free {
    std::vector<void*>& t;
    cudaStream_t s;
    ~Free() {
      for (void* p : t) dfree(p, s);
    }
  } fr{tmp, st};
  double* bws;
  TRY_STATUS(get((void**)&bws, sizeof(double) * 6 * nbb));
  kc_bbox_kernel<<<nbb, 256, 0, st>>>(X, n, d, bws);
  AFN_LAUNCH_CHECK("kc_bbox_kernel");
  std::vector<double> hb((size_t)6 * nbb);
  AFN_CUDA(cudaMemcpyAsync(hb.data(), bws, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  KcGrid gd{};
  gd.dd = dd;
  {
    const int cap_bits = dd == 3 ? 8 : (dd == 2 ? 12 : 24);
    const double target = std::max(1.0, (double)n / 2.0);
    int g = std::max(1, (int)std::ceil(std::pow(target, 1.0 / dd)));
    int bits = 0;
    while ((1 << bits) < g) ++bits;
    if (bits > cap_bits) {
      bits = cap_bits;
      g = 1 << bits;
    }
    gd.bits = bits;
    gd.g = g;
    for (int q = 0; q < 3; ++q) {
      double lo = 1e300, hi = -1e300;
      for (int b = 0; b < nbb; ++b) {
        lo = std::min(lo, hb[(size_t)b * 6 + q]);
        hi = std::max(hi, hb[(size_t)b * 6 + 3 + q]);
      }
      gd.lo[q] = q < dd ? lo : 0.0;
      gd.inv[q] = (q < dd && hi > lo) ? (double)g / (hi - lo) : 0.0;
    }
  }
  const int64_t ncell = (int64_t)1 << (gd.bits * dd);
  unsigned* key;
  int* cnt;
  int64_t* off;
  TRY_STATUS(get((void**)&key, sizeof(unsigned) * n));
  TRY_STATUS(get((void**)&cnt, sizeof(int) * 2 * ncell));
  TRY_STATUS(get((void**)&off, sizeof(int64_t) * (ncell + 1)));
  AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * ncell, st));
  const unsigned nbn = (unsigned)((n + 255) / 256);
  kc_key_kernel<<<nbn, 256, 0, st>>>(X, n, d, gd, key, cnt);
  AFN_LAUNCH_CHECK("kc_key_kernel");
  kc_scan_kernel<<<1, 1024, 0, st>>>(cnt, ncell, off);
  AFN_LAUNCH_CHECK("kc_scan_kernel");
  kc_scatter_kernel<<<nbn, 256, 0, st>>>(key, n, off, cnt + ncell, sidx);
  AFN_LAUNCH_CHECK("kc_scatter_kernel");
  kc_cell_sort_kernel<<<(unsigned)((ncell + 255) / 256), 256, 0, st>>>(off, ncell, sidx);
  AFN_LAUNCH_CHECK("kc_cell_sort_kernel");
  return AFN_OK;
}

}  // namespace afn

// wcut.cu -- W = K21 L^{-T} (the coupling block V = L^{-1} K12
// stored point-major) using the decay of the Gaussian kernel.
//
// W[i][c] = sum_{j <= c} K(x_i, x_j) L^{-T}[j][c] over the landmarks j.  An
// entry K(x_i, x_j) with ||x_i - x_j||^2 log2(e) / l^2 >= 128 is below 2^-128
// (beneath FP64 working accuracy by ~100 orders of magnitude relative to the
// unit diagonal), so its term is dropped.  The non-landmark rows are put in a
// Morton order (spatial.cu) and cut into tiles of 64 consecutive positions;
// a tile keeps the landmarks within that bound of its bounding box (U_t,
// ascending), and W_t = K(X_t, X_{U_t}) L^{-T}[U_t, :] is one small dense
// product on the FP64 tensor cores (mma.sync m8n8k4 f64, the tiling of
// dense.cu's gemm_dmma_kernel) with the rows of L^{-T} gathered by index and
// the K range of a 64-column block cut at its last column (L^{-T} is upper
// triangular).  The rows are written back to their own positions of W.
#include <algorithm>
#include <cmath>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int WM = 64, WN = 64, WK = 16, WKP = 20, WNP = 72, WS = 2;

__device__ __forceinline__ void wc_cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void wc_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// tile boxes over the first d <= 3 coordinates (one warp per 64-row tile)
__global__ void wc_tile_box_kernel(const double* __restrict__ Xr, int64_t N, int d, const int* __restrict__ sidx,
                                   int64_t nt, double* __restrict__ box) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt) return;
  for (int q = 0; q < 3; ++q) {
    double lo = 1e300, hi = -1e300;
    for (int h = 0; h < 2; ++h) {
      const int64_t p = t * WM + 32 * h + lane;
      if (q < d && p < N) {
        const double x = Xr[(int64_t)sidx[p] * d + q];
        lo = fmin(lo, x);
        hi = fmax(hi, x);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      box[t * 6 + q] = q < d ? lo : 0.0;
      box[t * 6 + 3 + q] = q < d ? hi : 0.0;
    }
  }
}

__device__ __forceinline__ bool wc_keep(const double* __restrict__ b, const double* __restrict__ x, int d,
                                        double thr) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) {
    const double gap = fmax(0.0, fmax(__dsub_rn(b[q], x[q]), __dsub_rn(x[q], b[3 + q])));
    s = __dadd_rn(s, __dmul_rn(gap, gap));
  }
  return s < thr;
}

// |U_t| per tile (one block per tile)
__global__ void __launch_bounds__(256) wc_count_kernel(const double* __restrict__ box, const double* __restrict__ X1,
                                                       int64_t k, int d, double thr, int* __restrict__ cnt) {
  __shared__ int c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  double b[6];
  for (int q = 0; q < 6; ++q) b[q] = box[blockIdx.x * 6 + q];
  int m = 0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) m += wc_keep(b, X1 + j * d, d, thr);
  atomicAdd(&c, m);
  __syncthreads();
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// U_t ascending into ulist[uoff[t] ..]; *work += the tile's executed MACs
// (64 rows x 64 columns x the K range of every column block)
// (lmap: the landmarks in the order lmap[0..k) -- the list then holds those
// positions, ascending; null: landmark ids ascending)
__global__ void __launch_bounds__(256) wc_fill_kernel(const double* __restrict__ box, const double* __restrict__ X1,
                                                      int64_t k, int d, double thr, const int64_t* __restrict__ uoff,
                                                      const int* __restrict__ lmap, int* __restrict__ ulist,
                                                      unsigned long long* __restrict__ work) {
  __shared__ int wtot[8];
  __shared__ int64_t base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double b[6];
  for (int q = 0; q < 6; ++q) b[q] = box[blockIdx.x * 6 + q];
  if (threadIdx.x == 0) base = uoff[blockIdx.x];
  __syncthreads();
  const int64_t ncb = (k + WN - 1) / WN;
  unsigned long long wk = 0ull;
  for (int64_t j0 = 0; j0 < k; j0 += 256) {
    const int64_t j = j0 + threadIdx.x;
    const bool kp = j < k && wc_keep(b, X1 + (lmap ? (int64_t)lmap[j] : j) * d, d, thr);
    const unsigned m = __ballot_sync(0xffffffffu, kp);
    if (lane == 0) wtot[wid] = __popc(m);
    __syncthreads();
    int64_t off = base;
    for (int w = 0; w < wid; ++w) off += wtot[w];
    if (kp) {
      ulist[off + __popc(m & ((1u << lane) - 1u))] = (int)j;
      wk += lmap ? (unsigned long long)ncb * WM * WN : (unsigned long long)(ncb - j / WN) * WM * WN;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 8; ++w) base += wtot[w];
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) wk += __shfl_xor_sync(0xffffffffu, wk, o);
  if (lane == 0 && work) atomicAdd(work, wk);
}

// A_t[r][m] = K(x_{sidx[64 t + r]}, x1_{U_t[m]}), ld = |U_t| rounded up to 2
__global__ void __launch_bounds__(256) wc_gen_a_kernel(const double* __restrict__ Xr, int64_t N, int d,
                                                       const int* __restrict__ sidx, const double* __restrict__ X1,
                                                       const int64_t* __restrict__ uoff, const int* __restrict__ ulist,
                                                       const int* __restrict__ lmap, const int64_t* __restrict__ aoff,
                                                       KernelFn kf, double thr, double* __restrict__ A) {
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  load_exp2_tab(s_tab);
  __syncthreads();
  const int64_t t = blockIdx.x;
  const int64_t u0 = uoff[t], nu = uoff[t + 1] - u0;
  const int64_t ld = (nu + 1) & ~(int64_t)1;
  double* At = A + aoff[t];
  for (int64_t e = threadIdx.x; e < WM * ld; e += blockDim.x) {
    const int64_t r = e / ld, m = e - r * ld;
    const int64_t p = t * WM + r;
    double v = 0.0;
    if (p < N && m < nu) {
      // a pair beyond the bound contributes nothing on any tiling: a row's
      // terms are exactly {j : ||x_r - x_j||^2 < thr}
      const int j = lmap ? lmap[ulist[u0 + m]] : ulist[u0 + m];
      const double d2 = d2_exact_rt(&Xr[(int64_t)sidx[p] * d], &X1[(int64_t)j * d], d);
      if (d2 < thr) v = kern_from_d2(kf, d2, s_tab);
    }
    At[e] = v;
  }
}

// point -> (its tile << 6) | its row in the tile
__global__ void wc_tilerow_kernel(const int* __restrict__ sidx, int64_t N, int* __restrict__ tilerow) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < N) tilerow[sidx[p]] = (int)p;  // (64-row tiles: p = 64 t + r)
}

// Mp[p][q] = M[lp[p]][lp[q]] from M's lower triangle
__global__ void wc_perm_sq_kernel(const double* __restrict__ M, int64_t k, const int* __restrict__ lp,
                                  double* __restrict__ Mp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int64_t p = e / k, q = e - p * k;
  const int64_t a = lp[p], b = lp[q];  // (M symmetric, its lower triangle formed)
  Mp[e] = a >= b ? M[a * k + b] : M[b * k + a];
}

// W rows of tile t, columns [64 c, 64 c + 64): A_t (64 x kc) times the rows
// U_t[0..kc) of L^{-T}, kc = #{m : U_t[m] < 64 c + 64}.  CTA tile 64 x 64,
// 4 warps of 32 x 32 (4 x 4 DMMA m8n8 tiles), k-chunks of 16 through 3
// cp.async stages (A at a 20-double, B at a 72-double row stride).
// TRI = false (Z = K21 M over the landmark order of the lists): every kept
// landmark contributes to every column block
template <bool TRI>
__global__ void __launch_bounds__(128) wc_gemm_kernel(const double* __restrict__ A, const int64_t* __restrict__ aoff,
                                                      const int64_t* __restrict__ uoff, const int* __restrict__ ulist,
                                                      const double* __restrict__ LinvT, int64_t k,
                                                      const int* __restrict__ sidx, int64_t N, double* __restrict__ W) {
  extern __shared__ __align__(16) double tsm[];
  double* sA = tsm;                  // [WS][WM][WKP]
  double* sB = tsm + WS * WM * WKP;  // [WS][WK][WNP]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid >> 1, wn = wid & 1;
  const int64_t t = blockIdx.y, C0 = (int64_t)blockIdx.x * WN;
  const int64_t u0 = uoff[t], nu = uoff[t + 1] - u0;
  const int64_t lda = (nu + 1) & ~(int64_t)1;
  const double* At = A + aoff[t];
  const int* U = ulist + u0;
  int64_t kc = nu;
  if (TRI) {  // first m with U[m] >= C0 + WN
    int64_t lo = 0, hi = nu;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (U[mid] < C0 + WN) lo = mid + 1;
      else hi = mid;
    }
    kc = lo;
  }
  const int64_t nkb = (kc + WK - 1) / WK;
  auto stage = [&](int64_t kb, int buf) {
    const int64_t k0 = kb * WK;
    double* a = sA + buf * WM * WKP;
    double* b = sB + buf * WK * WNP;
#pragma unroll
    for (int u = 0; u < (WM * WK / 2) / 128; ++u) {  // A: 16-byte copies (row r, k pair)
      const int e = tid + 128 * u;
      const int r = e / (WK / 2), kp = 2 * (e - r * (WK / 2));
      const int64_t gk = k0 + kp;
      double* dst = &a[r * WKP + kp];
      if (gk + 1 < kc) {
        wc_cpa16(dst, &At[r * lda + gk]);
      } else {
        dst[0] = gk < kc ? At[r * lda + gk] : 0.0;
        dst[1] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < (WK * WN / 2) / 128; ++u) {  // B: gathered L^{-T} rows, column pairs
      const int e = tid + 128 * u;
      const int kk = e / (WN / 2), c = 2 * (e - kk * (WN / 2));
      const int64_t gk = k0 + kk, gc = C0 + c;
      double* dst = &b[kk * WNP + c];
      if (gk < kc && gc + 1 < k && (k & 1) == 0) {
        wc_cpa16(dst, &LinvT[(int64_t)U[gk] * k + gc]);
      } else {
        dst[0] = (gk < kc && gc < k) ? LinvT[(int64_t)U[gk] * k + gc] : 0.0;
        dst[1] = (gk < kc && gc + 1 < k) ? LinvT[(int64_t)U[gk] * k + gc + 1] : 0.0;
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
  for (int s0 = 0; s0 < WS - 1; ++s0) {
    if (s0 < nkb) stage(s0, s0);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kb = 0; kb < nkb; ++kb) {
    asm volatile("cp.async.wait_group %0;" ::"n"(WS - 2) : "memory");
    __syncthreads();
    const int64_t nx = kb + WS - 1;
    if (nx < nkb) stage(nx, (int)(nx % WS));
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const double* a = sA + (int)(kb % WS) * WM * WKP + (wm * 32 + fr) * WKP + fk;
    const double* b = sB + (int)(kb % WS) * WK * WNP + fk * WNP + wn * 32 + fr;
#pragma unroll
    for (int k4 = 0; k4 < WK; k4 += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = a[i * 8 * WKP + k4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = b[k4 * WNP + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) wc_dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  const bool vec = (k & 1) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t p = t * WM + wm * 32 + i * 8 + fr;
    if (p >= N) continue;
    double* Wr = W + (int64_t)sidx[p] * k;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = C0 + wn * 32 + j * 8 + 2 * fk;
      if (vec && c + 1 < k) {
        *reinterpret_cast<double2*>(&Wr[c]) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < k) Wr[c] = acc[i][j][0];
        if (c + 1 < k) Wr[c + 1] = acc[i][j][1];
      }
    }
  }
}

// ---- the AFN apply through the tiles (W t = K21 (L^{-T} t), W^T s = L^{-1} (K21^T s))
// u[i] = r2[i] - K21[i, :] y1: a warp per row (Morton position p), lanes over the tile's list
__global__ void __launch_bounds__(256) wc_apply_n_kernel(const double* __restrict__ A, const int64_t* __restrict__ aoff,
                                                         const int64_t* __restrict__ uoff, const int* __restrict__ ulist,
                                                         const int* __restrict__ sidx, int64_t N,
                                                         const double* __restrict__ y1, const double* __restrict__ r2,
                                                         double* __restrict__ u, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= N) return;
  const int64_t t = p >> 6;
  const int r = (int)(p & 63);
  const int64_t us = uoff[t];
  const int nu = (int)(uoff[t + 1] - us);
  const int ld = (nu + 1) & ~1;
  const double* Ar = A + aoff[t] + (int64_t)r * ld;
  const int* U = ulist + us;
  double acc = 0.0;
  for (int m = lane; m < nu; m += 32) acc = fma(Ar[m], __ldg(&y1[U[m]]), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    const int i = sidx[p];
    u[i] = r2[i] - acc;
  }
}
// CT[uoff[t] + m] = sum_r K21[row r of t, U_t[m]] s2[row r] (a block per tile)
__global__ void __launch_bounds__(256) wc_apply_t1_kernel(const double* __restrict__ A, const int64_t* __restrict__ aoff,
                                                          const int64_t* __restrict__ uoff, const int* __restrict__ sidx,
                                                          int64_t N, const double* __restrict__ s2,
                                                          double* __restrict__ CT, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double ss[WM];
  const int64_t t = blockIdx.x;
  const int64_t us = uoff[t];
  const int nu = (int)(uoff[t + 1] - us);
  const int ld = (nu + 1) & ~1;
  const double* At = A + aoff[t];
  if (threadIdx.x < WM) {
    const int64_t p = t * WM + threadIdx.x;
    ss[threadIdx.x] = p < N ? s2[sidx[p]] : 0.0;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < nu; m += blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (int r = 0; r < WM; ++r) acc = fma(At[(int64_t)r * ld + m], ss[r], acc);
    CT[us + m] = acc;
  }
}
// w[j] = sum of CT over the entries of landmark j (ascending): a warp per landmark
__global__ void __launch_bounds__(256) wc_apply_t2_kernel(const int64_t* __restrict__ jptr, const int* __restrict__ jidx,
                                                          int64_t k, const double* __restrict__ CT,
                                                          double* __restrict__ w, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= k) return;
  double acc = 0.0;
  for (int64_t q = jptr[j] + lane; q < jptr[j + 1]; q += 32) acc += CT[jidx[q]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) w[j] = acc;
}
// the transpose of the lists: per landmark its flat entries, ascending
__global__ void wc_jcount_kernel(const int* __restrict__ ulist, int64_t E, int* __restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) atomicAdd(&cnt[ulist[e]], 1);
}
__global__ void wc_jplace_kernel(const int* __restrict__ ulist, int64_t E, const int64_t* __restrict__ jptr,
                                 int* __restrict__ cur, int* __restrict__ jidx) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) jidx[jptr[ulist[e]] + atomicAdd(&cur[ulist[e]], 1)] = (int)e;
}
__global__ void __launch_bounds__(256) wc_jsort_kernel(const int64_t* __restrict__ jptr, int* __restrict__ jidx) {
  __shared__ int sv[2048];
  const int64_t b = jptr[blockIdx.x], e = jptr[blockIdx.x + 1];
  const int len = (int)(e - b);
  if (len <= 1) return;
  if (len <= 2048) {
    int p2 = 1;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) sv[i] = i < len ? jidx[b + i] : 0x7fffffff;
    __syncthreads();
    for (int kk = 2; kk <= p2; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
          const int l = i ^ jj;
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
    for (int i = threadIdx.x; i < len; i += blockDim.x) jidx[b + i] = sv[i];
    return;
  }
  if (threadIdx.x != 0) return;
  for (int64_t i = b + 1; i < e; ++i) {
    const int v = jidx[i];
    int64_t q = i - 1;
    while (q >= b && jidx[q] > v) {
      jidx[q + 1] = jidx[q];
      --q;
    }
    jidx[q + 1] = v;
  }
}

}  // namespace

afn_status w_cut_apply_prep(WCutPlan* p, cudaStream_t st) {
  if (!p->used) {
    set_error("w_cut_apply_prep: no plan");
    return AFN_ERR_STATE;
  }
  const int64_t E = p->E, k = p->k;
  int* cnt = nullptr;
  TRY_STATUS(dalloc((void**)&p->jptr, sizeof(int64_t) * (k + 1), st));
  p->mem.push_back(p->jptr);
  TRY_STATUS(dalloc((void**)&p->jidx, sizeof(int) * std::max<int64_t>(1, E), st));
  p->mem.push_back(p->jidx);
  TRY_STATUS(dalloc((void**)&p->CT, sizeof(double) * std::max<int64_t>(1, E), st));
  p->mem.push_back(p->CT);
  TRY_STATUS(dalloc((void**)&cnt, sizeof(int) * 2 * k, st));
  AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * k, st));
  const unsigned nbe = (unsigned)((E + 255) / 256);
  if (E > 0) {
    wc_jcount_kernel<<<nbe, 256, 0, st>>>(p->ulist, E, cnt);
    AFN_LAUNCH_CHECK("wc_jcount_kernel");
  }
  TRY_STATUS(scan_i32_i64(cnt, k, p->jptr, st));
  if (E > 0) {
    wc_jplace_kernel<<<nbe, 256, 0, st>>>(p->ulist, E, p->jptr, cnt + k, p->jidx);
    AFN_LAUNCH_CHECK("wc_jplace_kernel");
  }
  wc_jsort_kernel<<<(unsigned)k, 256, 0, st>>>(p->jptr, p->jidx);
  AFN_LAUNCH_CHECK("wc_jsort_kernel");
  dfree(cnt, st);
  return AFN_OK;
}

afn_status w_cut_apply_n(const WCutPlan* p, const double* y1, const double* r2, double* u, cudaStream_t st) {
  if (p->N <= 0) return AFN_OK;
  wc_apply_n_kernel<<<(unsigned)((p->N + 7) / 8), 256, 0, st>>>(p->A, p->aoff, p->uoff, p->ulist, p->sidx, p->N, y1,
                                                                  r2, u, get_skip());
  AFN_LAUNCH_CHECK("wc_apply_n_kernel");
  return AFN_OK;
}

afn_status w_cut_apply_t(const WCutPlan* p, const double* s2, double* w, cudaStream_t st) {
  if (p->N > 0) {
    wc_apply_t1_kernel<<<(unsigned)p->nt, 256, 0, st>>>(p->A, p->aoff, p->uoff, p->sidx, p->N, s2, p->CT, get_skip());
    AFN_LAUNCH_CHECK("wc_apply_t1_kernel");
  }
  wc_apply_t2_kernel<<<(unsigned)((p->k + 7) / 8), 256, 0, st>>>(p->jptr, p->jidx, p->k, p->CT, w, get_skip());
  AFN_LAUNCH_CHECK("wc_apply_t2_kernel");
  return AFN_OK;
}

void w_cut_free(WCutPlan* p) {
  for (void* q : p->mem) dfree(q, p->st);
  p->mem.clear();
  p->used = false;
  p->jptr = nullptr;
  p->jidx = nullptr;
  p->CT = nullptr;
}

afn_status w_cut_plan(const double* X1, int64_t k, const double* Xr, int64_t N, int d, Kern kn, bool force,
                      bool zmode, cudaStream_t st, WCutPlan* p) {
  w_cut_free(p);
  p->used = false;
  p->st = st;
  if (kn.kind != 0 || d > 3 || N < 1 || k < 1 || (N + WM - 1) / WM > 65535) return AFN_OK;
  std::vector<void*> tmp;
  struct Free {
    std::vector<void*>& t;
    cudaStream_t s;
    ~Free() {
      for (void* q : t) dfree(q, s);
    }
  } fr{tmp, st};
  auto get = [&](void** q, size_t bytes, bool keep) {
    afn_status s = dalloc(q, bytes, st);
    if (s == AFN_OK) (keep ? p->mem : tmp).push_back(*q);
    return s;
  };
  // entries below 2^-128: ||x - y||^2 >= 128 ln(2) l^2 (a hair inside, so
  // rounding never drops a term at the bound)
  const double thr = 128.0 * 0.6931471805599453 * kn.l * kn.l * (1.0 - 1e-12);
  const int64_t nt = (N + WM - 1) / WM;
  double* box;
  int* cnt;
  unsigned long long* work;
  TRY_STATUS(get((void**)&p->sidx, sizeof(int) * N, true));
  TRY_STATUS(get((void**)&p->uoff, sizeof(int64_t) * (nt + 1), true));
  TRY_STATUS(get((void**)&p->aoff, sizeof(int64_t) * (nt + 1), true));
  TRY_STATUS(get((void**)&box, sizeof(double) * 6 * nt, false));
  TRY_STATUS(get((void**)&cnt, sizeof(int) * nt, false));
  TRY_STATUS(get((void**)&work, sizeof(unsigned long long), false));
  TRY_STATUS(morton_order(Xr, N, d, p->sidx, st));
  wc_tile_box_kernel<<<(unsigned)((nt * 32 + 255) / 256), 256, 0, st>>>(Xr, N, d, p->sidx, nt, box);
  AFN_LAUNCH_CHECK("wc_tile_box_kernel");
  wc_count_kernel<<<(unsigned)nt, 256, 0, st>>>(box, X1, k, d, thr, cnt);
  AFN_LAUNCH_CHECK("wc_count_kernel");
  std::vector<int> hc((size_t)nt);
  AFN_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * nt, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> ho((size_t)nt + 1, 0), ha((size_t)nt + 1, 0);
  for (int64_t t = 0; t < nt; ++t) {
    ho[t + 1] = ho[t] + hc[t];
    ha[t + 1] = ha[t] + (int64_t)WM * ((hc[t] + 1) & ~1);
  }
  // the dense product (INT8 or DMMA) is cheaper when most landmarks are kept
  if (!force && (double)ho[nt] > 0.5 * (double)nt * (double)k) {
    w_cut_free(p);
    return AFN_OK;
  }
  // the FSAI products through Z pay off only for short lists (C3 ~6 % of k,
  // C5 ~1 %); at C2 (l = 1: ~47 %) the W form is faster (11.5 vs 13.3 ms)
  if (zmode && !force && (double)ho[nt] > 0.2 * (double)nt * (double)k) zmode = false;
  TRY_STATUS(get((void**)&p->ulist, sizeof(int) * std::max<int64_t>(1, ho[nt]), true));
  TRY_STATUS(get((void**)&p->A, sizeof(double) * std::max<int64_t>(1, ha[nt]), true));
  AFN_CUDA(cudaMemcpyAsync(p->uoff, ho.data(), sizeof(int64_t) * ho.size(), cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(p->aoff, ha.data(), sizeof(int64_t) * ha.size(), cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
  wc_fill_kernel<<<(unsigned)nt, 256, 0, st>>>(box, X1, k, d, thr, p->uoff, nullptr, p->ulist, work);
  AFN_LAUNCH_CHECK("wc_fill_kernel");
  wc_gen_a_kernel<<<(unsigned)nt, 256, 0, st>>>(Xr, N, d, p->sidx, X1, p->uoff, p->ulist, nullptr, p->aoff,
                                                kernel_fn(kn.kind, kn.l), thr, p->A);
  if (zmode) {  // the same lists and tiles over the landmarks' Morton order (Z = K21 M, fsai_sddmm.cu)
    TRY_STATUS(get((void**)&p->lp, sizeof(int) * k, true));
    TRY_STATUS(get((void**)&p->ulistp, sizeof(int) * std::max<int64_t>(1, ho[nt]), true));
    TRY_STATUS(get((void**)&p->Ap, sizeof(double) * std::max<int64_t>(1, ha[nt]), true));
    TRY_STATUS(get((void**)&p->tilerow, sizeof(int) * N, true));
    TRY_STATUS(morton_order(X1, k, d, p->lp, st));
    wc_fill_kernel<<<(unsigned)nt, 256, 0, st>>>(box, X1, k, d, thr, p->uoff, p->lp, p->ulistp, nullptr);
    AFN_LAUNCH_CHECK("wc_fill_kernel");
    wc_gen_a_kernel<<<(unsigned)nt, 256, 0, st>>>(Xr, N, d, p->sidx, X1, p->uoff, p->ulistp, p->lp, p->aoff,
                                                  kernel_fn(kn.kind, kn.l), thr, p->Ap);
    AFN_LAUNCH_CHECK("wc_gen_a_kernel");
    wc_tilerow_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(p->sidx, N, p->tilerow);
    AFN_LAUNCH_CHECK("wc_tilerow_kernel");
  }
  AFN_LAUNCH_CHECK("wc_gen_a_kernel");
  unsigned long long hw = 0ull;
  AFN_CUDA(cudaMemcpyAsync(&hw, work, sizeof(hw), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));  // (pageable copies; temporaries freed on return)
  p->flops = 2.0 * (double)hw;
  p->zflops = 2.0 * WM * (double)((k + WN - 1) / WN * WN) * (double)ho[nt];
  p->k = k;
  p->N = N;
  p->nt = nt;
  p->E = ho[nt];
  p->Adbl = ha[nt];
  p->used = true;
  return AFN_OK;
}

afn_status w_cut_run(WCutPlan* p, const double* LinvT, double* W, cudaStream_t st) {
  if (!p->used) {
    set_error("w_cut_run: no plan");
    return AFN_ERR_STATE;
  }
  const int smem = (int)(sizeof(double) * WS * (WM * WKP + WK * WNP));
  AFN_CUDA(cudaFuncSetAttribute(wc_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((unsigned)((p->k + WN - 1) / WN), (unsigned)p->nt);
  wc_gemm_kernel<true><<<grid, 128, smem, st>>>(p->A, p->aoff, p->uoff, p->ulist, LinvT, p->k, p->sidx, p->N, W);
  AFN_LAUNCH_CHECK("wc_gemm_kernel");
  p->st = st;  // (the plan's memory is released in this stream's order)
  if (!p->lp && !p->keep) w_cut_free(p);  // (kept for w_cut_z / the FSAI products / the apply)
  return AFN_OK;
}

afn_status w_cut_z(WCutPlan* p, const double* LinvT, const double* Linv, double* M, double* Mp, double* Zp,
                   cudaStream_t st) {
  if (!p->used || !p->lp) {
    set_error("w_cut_z: no Z-mode plan");
    return AFN_ERR_STATE;
  }
  const int64_t k = p->k;
  TRY_STATUS(gemm_upper_lower(LinvT, Linv, k, M, st));  // M = L^{-T} L^{-1} = (K11 + mu I)^{-1}
  wc_perm_sq_kernel<<<(unsigned)((k * k + 255) / 256), 256, 0, st>>>(M, k, p->lp, Mp);
  AFN_LAUNCH_CHECK("wc_perm_sq_kernel");
  const int smem = (int)(sizeof(double) * WS * (WM * WKP + WK * WNP));
  AFN_CUDA(cudaFuncSetAttribute(wc_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((unsigned)((k + WN - 1) / WN), (unsigned)p->nt);
  wc_gemm_kernel<false><<<grid, 128, smem, st>>>(p->Ap, p->aoff, p->uoff, p->ulistp, Mp, k, p->sidx, p->N, Zp);
  AFN_LAUNCH_CHECK("wc_gemm_kernel<false>");
  p->st = st;
  return AFN_OK;
}

afn_status w_gemm_cut(const double* LinvT, int64_t k, const double* X1, const double* Xr, int64_t N, int d, Kern kn,
                      double* W, cudaStream_t st, bool force, bool* used, double* flops) {
  WCutPlan p;
  afn_status s = w_cut_plan(X1, k, Xr, N, d, kn, force, false, st, &p);
  if (s != AFN_OK) {
    w_cut_free(&p);
    return s;
  }
  *used = p.used;
  if (!p.used) return AFN_OK;
  if (flops) *flops = p.flops;
  return w_cut_run(&p, LinvT, W, st);
}

}  // namespace afn

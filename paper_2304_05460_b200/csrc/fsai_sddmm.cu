// fsai_sddmm.cu -- FSAI rows from the UNION of needed Schur-complement pairs.
//
// Every FSAI row i needs S_ab = K_ab + mu delta_ab - W_a . W_b for all a, b in
// its pattern J_i ("only requires the entries ... corresponding
// to the sparsity pattern").  Forming each row's Gram W_J W_J^T separately
// evaluates every needed pair ~14 times (a pair of nearby points belongs to
// many rows' patterns).  Here each needed dot product W_a . W_b (b <= a) is
// evaluated once, in dense blocks:
//   1. spatial order: non-landmark points sorted by grid cell (tiled cell
//      order), consecutive GA = 16 points form a group g;
//   2. U_g = union over a in g of B_a = { b <= a : a, b in J_i for some row i }
//      (rows containing a come from the transposed pattern), sorted;
//   3. D_g = W_g W_{U_g}^T (GA x |U_g|, k-long FP64 dots; register-tiled,
//      cp.async-staged through shared memory) -- ~4x fewer flops than the
//      per-row Gram on the C2 pattern;
//   4. per row: S_JJ assembled by look-up (binary search of b in U_{g(a)}),
//      then the warp-per-row Cholesky of fsai.cu.
// Values are independent of the grouping (each dot has a fixed summation
// order), so the result is deterministic even though the cell sort uses atomics.
#include <algorithm>
#include <cmath>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {

// shared with fsai.cu (defined there)
afn_status fsai_chol_batch(int64_t r0, int64_t nrows, int MT, const int64_t* rp, double* Sg,
                           double* gval, int* info, cudaStream_t st);

namespace {

constexpr int GA = 16;       // group size (points a per group)
constexpr int UCAP = 4096;   // max |U_g|
constexpr int HC = 8192;     // hash capacity (power of two)
constexpr int UT = 512;      // U columns per GEMM pass (2 per thread)
constexpr int KC2 = 8;       // k per pipeline stage
constexpr int NST = 3;       // pipeline stages

__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

__device__ __forceinline__ int cml(int a, int t, int wp) { return t * wp - (t * (t - 1)) / 2 + (a - t); }

// ---------------------------------------------------------------- spatial order
__global__ void bbox_partial_kernel(const double* __restrict__ X, int64_t N, int d, double* ws) {
  __shared__ double smin[3][256], smax[3][256];
  const int dd = d < 3 ? d : 3;
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < dd; ++c) {
      const double v = X[i * d + c];
      mn[c] = fmin(mn[c], v);
      mx[c] = fmax(mx[c], v);
    }
  for (int c = 0; c < 3; ++c) {
    smin[c][threadIdx.x] = mn[c];
    smax[c][threadIdx.x] = mx[c];
  }
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off)
      for (int c = 0; c < 3; ++c) {
        smin[c][threadIdx.x] = fmin(smin[c][threadIdx.x], smin[c][threadIdx.x + off]);
        smax[c][threadIdx.x] = fmax(smax[c][threadIdx.x], smax[c][threadIdx.x + off]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) {
      ws[blockIdx.x * 6 + c] = smin[c][0];
      ws[blockIdx.x * 6 + 3 + c] = smax[c][0];
    }
}

__global__ void bbox_final_kernel(const double* ws, int nb, double* box) {
  if (threadIdx.x != 0) return;
  for (int c = 0; c < 3; ++c) {
    double mn = 1e300, mx = -1e300;
    for (int b = 0; b < nb; ++b) {
      mn = fmin(mn, ws[b * 6 + c]);
      mx = fmax(mx, ws[b * 6 + 3 + c]);
    }
    box[c] = mn;
    box[3 + c] = mx;
  }
}

struct CellGrid {
  int g[3];   // cells per axis (padded to the tile)
  int t[3];   // tile size per axis
  int nb[3];  // tiles per axis
  int64_t ncell;
};

__global__ void cell_key_kernel(const double* __restrict__ X, int64_t N, int d, const double* __restrict__ box,
                                CellGrid cg, int* __restrict__ key, int* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int dd = d < 3 ? d : 3;
  int cc[3] = {0, 0, 0};
  for (int c = 0; c < dd; ++c) {
    const double lo = box[c], hi = box[3 + c];
    const double w = hi > lo ? (hi - lo) : 1.0;
    int v = (int)((X[i * d + c] - lo) / w * (double)cg.g[c]);
    cc[c] = v < 0 ? 0 : (v >= cg.g[c] ? cg.g[c] - 1 : v);
  }
  const int b0 = cc[0] / cg.t[0], b1 = cc[1] / cg.t[1], b2 = cc[2] / cg.t[2];
  const int l0 = cc[0] % cg.t[0], l1 = cc[1] % cg.t[1], l2 = cc[2] % cg.t[2];
  const int64_t tile = ((int64_t)b2 * cg.nb[1] + b1) * cg.nb[0] + b0;
  const int64_t k = tile * (cg.t[0] * cg.t[1] * cg.t[2]) + ((int64_t)l2 * cg.t[1] + l1) * cg.t[0] + l0;
  key[i] = (int)k;
  atomicAdd(&cnt[k], 1);
}

// exclusive scan of M ints into off (int64) with an optional multiplier, one block
__global__ void scan_i64_kernel(const int* __restrict__ cnt, int64_t M, int64_t mult,
                                int64_t* __restrict__ off) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (M + 1023) / 1024;
  const int64_t b = tid * per, e = min(M, b + per);
  int64_t s = 0;
  for (int64_t t = b; t < e; ++t) s += (int64_t)cnt[t] * mult;
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
    run += (int64_t)cnt[t] * mult;
  }
  if (tid == 1023) off[M] = part[1023];
}

__global__ void cell_scatter_kernel(const int* __restrict__ key, int64_t N, const int64_t* __restrict__ off,
                                    int* __restrict__ cur, int* __restrict__ sorder) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int k = key[i];
  const int p = atomicAdd(&cur[k], 1);
  sorder[off[k] + p] = (int)i;
}

__global__ void group_maps_kernel(const int* __restrict__ sorder, int64_t N, int* __restrict__ grp,
                                  int* __restrict__ loc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const int a = sorder[t];
  grp[a] = (int)(t / GA);
  loc[a] = (int)(t % GA);
}

// ---------------------------------------------------------------- group unions
__global__ void __launch_bounds__(256) group_union_kernel(const int* __restrict__ sorder, int64_t N,
                                                          const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col,
                                                          const int64_t* __restrict__ trp,
                                                          const int32_t* __restrict__ tcol,
                                                          int64_t row_lo, int64_t row_hi,
                                                          int* __restrict__ Ucount, int* __restrict__ Ulist,
                                                          int* overflow) {
  extern __shared__ int hs[];  // HC
  __shared__ int s_n;
  const int tid = threadIdx.x;
  const int64_t g = blockIdx.x;
  for (int t = tid; t < HC; t += 256) hs[t] = -1;
  if (tid == 0) s_n = 0;
  __syncthreads();
  const int64_t m0 = g * GA;
  const int cnt = (int)min((int64_t)GA, N - m0);
  for (int j = 0; j < cnt; ++j) {
    const int a = sorder[m0 + j];
    for (int64_t e = trp[a] + tid; e < trp[a + 1]; e += 256) {
      const int i = tcol[e];
      if (i < row_lo || i >= row_hi) continue;  // rows this rank factors
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        const int b = col[q];
        if (b > a) break;
        unsigned h = ((unsigned)b * 2654435761u) & (HC - 1);
        while (true) {
          const int old = atomicCAS(&hs[h], -1, b);
          if (old == -1) {
            atomicAdd(&s_n, 1);
            break;
          }
          if (old == b) break;
          h = (h + 1) & (HC - 1);
        }
        if (s_n > (HC * 3) / 4) break;  // overflow guard (checked below)
      }
    }
  }
  __syncthreads();
  const int nu = s_n;
  if (nu > UCAP || nu > (HC * 3) / 4) {
    if (tid == 0) atomicExch(overflow, 1);
    return;
  }
  // compact the occupied slots to the front (order irrelevant), then sort
  // the first next_pow2(nu) entries ascending
  __shared__ int s_c;
  if (tid == 0) s_c = 0;
  __syncthreads();
  int* tmpk = hs + HC;  // second buffer (HC ints)
  for (int t = tid; t < HC; t += 256) {
    const int v = hs[t];
    if (v >= 0) tmpk[atomicAdd(&s_c, 1)] = v;
  }
  __syncthreads();
  int P2 = 1;
  while (P2 < nu) P2 <<= 1;
  for (int t = tid; t < P2; t += 256) hs[t] = t < nu ? tmpk[t] : 0x7fffffff;
  __syncthreads();
  for (int kk = 2; kk <= P2; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < P2; t += 256) {
        const int p = t ^ j;
        if (p > t) {
          const bool up = (t & kk) == 0;
          const int x = hs[t], y = hs[p];
          if ((x > y) == up) {
            hs[t] = y;
            hs[p] = x;
          }
        }
      }
      __syncthreads();
    }
  for (int t = tid; t < nu; t += 256) Ulist[g * UCAP + t] = hs[t];
  if (tid == 0) Ucount[g] = nu;
}

// ---------------------------------------------------------------- group GEMM
// D_g[j][u] = W[a_j] . W[U_g[u]]  for j < GA, u < |U_g|.  Shared-memory
// stages hold k-pairs interleaved ([kk/2][row][2]) so every cp.async moves
// 16 B and every operand read is a conflict-free LDS.128.
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

__global__ void __launch_bounds__(256, 2) group_gemm_kernel(const int* __restrict__ sorder, int64_t N,
                                                            const double* __restrict__ W, int64_t k,
                                                            const int* __restrict__ Ucount,
                                                            const int* __restrict__ Ulist,
                                                            const int64_t* __restrict__ Doff,
                                                            double* __restrict__ D) {
  extern __shared__ __align__(16) double gs[];
  double* sA = gs;                    // [NST][KC2/2][GA][2]
  double* sB = gs + NST * KC2 * GA;   // [NST][KC2/2][UT][2]
  __shared__ int s_a[GA];
  __shared__ int s_u[UT];
  const int tid = threadIdx.x;
  const int64_t g = blockIdx.x;
  const int64_t m0 = g * GA;
  const int cnt = (int)min((int64_t)GA, N - m0);
  const int nu = Ucount[g];
  double* Dg = D + Doff[g];
  if (tid < GA) s_a[tid] = tid < cnt ? sorder[m0 + tid] : -1;
  const int64_t nch = (k + KC2 - 1) / KC2;
  const bool even = (k & 1) == 0;  // 16-byte aligned rows -> 16-byte copies
  for (int u0 = 0; u0 < nu; u0 += UT) {
    const int un = min(UT, nu - u0);
    __syncthreads();
    for (int t = tid; t < UT; t += 256) s_u[t] = t < un ? Ulist[g * UCAP + u0 + t] : -1;
    __syncthreads();
    auto issue = [&](int64_t ch, int buf) {
      const int64_t c0 = ch * KC2;
      double* a = sA + buf * KC2 * GA;
      double* b = sB + buf * KC2 * UT;
      for (int e = tid; e < (KC2 / 2) * GA; e += 256) {
        const int j = e / (KC2 / 2), k2 = e - j * (KC2 / 2);
        const int aj = s_a[j];
        const int64_t c = c0 + 2 * k2;
        double* dst = &a[(k2 * GA + j) * 2];
        if (aj >= 0 && c + 1 < k && even) {
          cpa16(dst, &W[(int64_t)aj * k + c]);
        } else {
          dst[0] = (aj >= 0 && c < k) ? W[(int64_t)aj * k + c] : 0.0;
          dst[1] = (aj >= 0 && c + 1 < k) ? W[(int64_t)aj * k + c + 1] : 0.0;
        }
      }
      for (int e = tid; e < (KC2 / 2) * UT; e += 256) {
        const int u = e / (KC2 / 2), k2 = e - u * (KC2 / 2);
        const int bu = s_u[u];
        const int64_t c = c0 + 2 * k2;
        double* dst = &b[(k2 * UT + u) * 2];
        if (bu >= 0 && c + 1 < k && even) {
          cpa16(dst, &W[(int64_t)bu * k + c]);
        } else {
          dst[0] = (bu >= 0 && c < k) ? W[(int64_t)bu * k + c] : 0.0;
          dst[1] = (bu >= 0 && c + 1 < k) ? W[(int64_t)bu * k + c + 1] : 0.0;
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[GA][2];
#pragma unroll
    for (int j = 0; j < GA; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int s0 = 0; s0 < NST - 1; ++s0) {
      if (s0 < nch) issue(s0, s0);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t ch = 0; ch < nch; ++ch) {
      asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory");
      __syncthreads();
      const int64_t nx = ch + NST - 1;
      if (nx < nch) issue(nx, (int)(nx % NST));
      else asm volatile("cp.async.commit_group;" ::: "memory");
      const double* a = sA + (int)(ch % NST) * KC2 * GA;
      const double* b = sB + (int)(ch % NST) * KC2 * UT;
#pragma unroll
      for (int k2 = 0; k2 < KC2 / 2; ++k2) {
        const double2 b0 = *reinterpret_cast<const double2*>(&b[(k2 * UT + tid) * 2]);
        const double2 b1 = *reinterpret_cast<const double2*>(&b[(k2 * UT + tid + 256) * 2]);
#pragma unroll
        for (int j = 0; j < GA; ++j) {
          const double2 av = *reinterpret_cast<const double2*>(&a[(k2 * GA + j) * 2]);
          acc[j][0] = fma(av.x, b0.x, acc[j][0]);
          acc[j][1] = fma(av.x, b1.x, acc[j][1]);
          acc[j][0] = fma(av.y, b0.y, acc[j][0]);
          acc[j][1] = fma(av.y, b1.y, acc[j][1]);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int j = 0; j < GA; ++j) {
      if (j >= cnt) break;
      if (tid < un) Dg[(int64_t)j * nu + u0 + tid] = acc[j][0];
      if (tid + 256 < un) Dg[(int64_t)j * nu + u0 + tid + 256] = acc[j][1];
    }
  }
}

// ---------------------------------------------------------------- assembly
template <int MT>
__global__ void __launch_bounds__(256) fsai_assemble_kernel(int64_t r0, const double* __restrict__ X2, int d,
                                                            double cl, double mu, const int64_t* __restrict__ rp,
                                                            const int32_t* __restrict__ col,
                                                            const int* __restrict__ grp, const int* __restrict__ loc,
                                                            const int* __restrict__ Ucount,
                                                            const int* __restrict__ Ulist,
                                                            const int64_t* __restrict__ Doff,
                                                            const double* __restrict__ D, double* __restrict__ Sg) {
  constexpr int WP = MT * 16;
  constexpr int SPK = WP * (WP + 1) / 2;
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  __shared__ int sJ[WP];
  __shared__ double sX[WP * 16];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t i = r0 + blockIdx.x;
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  load_exp2_tab(s_tab);
  for (int a = tid; a < wp; a += 256) sJ[a] = col[beg + a];
  __syncthreads();
  for (int e = tid; e < wp * d; e += 256) {
    const int a = e / d, c = e - a * d;
    sX[e] = X2[(int64_t)sJ[a] * d + c];
  }
  __syncthreads();
  double* S = Sg + (int64_t)blockIdx.x * SPK;
  for (int p = ty; p < wp; p += 16) {
    const int a = sJ[p];
    const int g = grp[a];
    const int nu = Ucount[g];
    const int* U = Ulist + (int64_t)g * UCAP;
    const double* Drow = D + Doff[g] + (int64_t)loc[a] * nu;
    for (int q = tx; q <= p; q += 16) {
      const int b = sJ[q];  // b <= a (columns ascending)
      int lo = 0, hi = nu - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (U[mid] < b) lo = mid + 1; else hi = mid;
      }
      const double gram = Drow[lo];
      double kv;
      if (p == q) {
        kv = 1.0 + mu;
      } else {
        const double sd = d2_exact_rt(&sX[p * d], &sX[q * d], d);
        kv = gauss_from_d2(sd, cl, s_tab);
      }
      S[cml(p, q, wp)] = kv - gram;
    }
  }
}

template <int MT>
void launch_assemble(unsigned grid, cudaStream_t st, int64_t r0, const double* X2, int d, double cl,
                     double mu, const int64_t* rp, const int32_t* col, const int* grp, const int* loc,
                     const int* Ucount, const int* Ulist, const int64_t* Doff, const double* D, double* Sg) {
  fsai_assemble_kernel<MT><<<grid, 256, 0, st>>>(r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist,
                                                 Doff, D, Sg);
}

}  // namespace

afn_status fsai_sddmm_run(const double* X2, int64_t N, int d, double l, double mu, const double* W,
                          int64_t k, const int64_t* rp, const int32_t* col, const int64_t* trp,
                          const int32_t* tcol, int64_t row_lo, int64_t row_hi, double* gval, int* d_info,
                          cudaStream_t st) {
  if (N <= 0 || row_hi <= row_lo) return AFN_OK;
  if (d > 16) {
    set_error("fsai_sddmm: d > 16");
    return AFN_ERR_STATE;
  }
  AFN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  std::vector<void*> tmp;
  struct Free {
    std::vector<void*>* t;
    cudaStream_t st;
    ~Free() {
      for (void* p : *t) dfree(p, st);
    }
  } fr{&tmp, st};
  auto get = [&](void** p, size_t bytes) {
    afn_status s = dalloc(p, bytes, st);
    if (s == AFN_OK) tmp.push_back(*p);
    return s;
  };
  afn_status s;
  // ---- widest row (w) for the packed-S layout
  int64_t h2[2];
  AFN_CUDA(cudaMemcpyAsync(h2, rp + (N > 1 ? N - 1 : 0), sizeof(int64_t) * (N > 1 ? 2 : 1),
                           cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  const int w = N > 1 ? (int)(h2[1] - h2[0]) : 1;
  const int MT = (w + 15) / 16;
  if (MT < 1 || MT > 8) {
    set_error("fsai_sddmm: row width %d", w);
    return AFN_ERR_ARG;
  }
  // ---- 1. spatial order
  const int dd = d < 3 ? d : 3;
  CellGrid cg;
  {
    const double target = std::max(1.0, (double)N / 2.0);
    const int gper = std::max(1, (int)std::ceil(std::pow(target, 1.0 / dd)));
    for (int c = 0; c < 3; ++c) {
      if (c < dd) {
        cg.t[c] = std::min(4, gper);
        cg.g[c] = ((gper + cg.t[c] - 1) / cg.t[c]) * cg.t[c];
      } else {
        cg.t[c] = 1;
        cg.g[c] = 1;
      }
      cg.nb[c] = cg.g[c] / cg.t[c];
    }
    cg.ncell = (int64_t)cg.g[0] * cg.g[1] * cg.g[2];
  }
  double *bws, *box;
  int *key, *cnt, *cur, *sorder, *grp, *loc;
  int64_t* off;
  const int nbb = 148;
  if ((s = get((void**)&bws, sizeof(double) * 6 * nbb)) != AFN_OK) return s;
  if ((s = get((void**)&box, sizeof(double) * 6)) != AFN_OK) return s;
  if ((s = get((void**)&key, sizeof(int) * N)) != AFN_OK) return s;
  if ((s = get((void**)&cnt, sizeof(int) * 2 * cg.ncell)) != AFN_OK) return s;
  if ((s = get((void**)&off, sizeof(int64_t) * (cg.ncell + 1))) != AFN_OK) return s;
  if ((s = get((void**)&sorder, sizeof(int) * N)) != AFN_OK) return s;
  if ((s = get((void**)&grp, sizeof(int) * N)) != AFN_OK) return s;
  if ((s = get((void**)&loc, sizeof(int) * N)) != AFN_OK) return s;
  cur = cnt + cg.ncell;
  AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * cg.ncell, st));
  bbox_partial_kernel<<<nbb, 256, 0, st>>>(X2, N, d, bws);
  AFN_LAUNCH_CHECK("bbox_partial_kernel");
  bbox_final_kernel<<<1, 32, 0, st>>>(bws, nbb, box);
  AFN_LAUNCH_CHECK("bbox_final_kernel");
  cell_key_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(X2, N, d, box, cg, key, cnt);
  AFN_LAUNCH_CHECK("cell_key_kernel");
  scan_i64_kernel<<<1, 1024, 0, st>>>(cnt, cg.ncell, 1, off);
  AFN_LAUNCH_CHECK("scan_i64_kernel");
  cell_scatter_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(key, N, off, cur, sorder);
  AFN_LAUNCH_CHECK("cell_scatter_kernel");
  group_maps_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(sorder, N, grp, loc);
  AFN_LAUNCH_CHECK("group_maps_kernel");
  // ---- 2. unions
  const int64_t G = (N + GA - 1) / GA;
  int *Ucount, *Ulist, *ovf;
  int64_t* Doff;
  if ((s = get((void**)&Ucount, sizeof(int) * G)) != AFN_OK) return s;
  if ((s = get((void**)&Ulist, sizeof(int) * G * UCAP)) != AFN_OK) return s;
  if ((s = get((void**)&ovf, sizeof(int) * 2)) != AFN_OK) return s;
  if ((s = get((void**)&Doff, sizeof(int64_t) * (G + 1))) != AFN_OK) return s;
  AFN_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int) * 2, st));
  {
    const int bytes = (int)(sizeof(int) * 2 * HC);
    static bool uattr = false;
    if (!uattr) {
      AFN_CUDA(cudaFuncSetAttribute(group_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      uattr = true;
    }
    group_union_kernel<<<(unsigned)G, 256, bytes, st>>>(sorder, N, rp, col, trp, tcol, row_lo, row_hi,
                                                         Ucount, Ulist, ovf);
    AFN_LAUNCH_CHECK("group_union_kernel");
  }
  int hov = 0;
  AFN_CUDA(cudaMemcpyAsync(&hov, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  if (hov) {
    set_error("fsai_sddmm: pair union exceeds %d in a group", UCAP);
    return AFN_ERR_STATE;
  }
  scan_i64_kernel<<<1, 1024, 0, st>>>(Ucount, G, GA, Doff);
  AFN_LAUNCH_CHECK("scan_i64_kernel");
  int64_t totD = 0;
  AFN_CUDA(cudaMemcpyAsync(&totD, Doff + G, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  // ---- 3. dense group products
  double* D;
  if ((s = get((void**)&D, sizeof(double) * (totD > 0 ? totD : 1))) != AFN_OK) return s;
  {
    const int bytes = (int)(sizeof(double) * NST * KC2 * (GA + UT));
    static bool attr = false;
    if (!attr) {
      AFN_CUDA(cudaFuncSetAttribute(group_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      attr = true;
    }
    kt_begin(KT_FSAI_GEMM, st);
    group_gemm_kernel<<<(unsigned)G, 256, bytes, st>>>(sorder, N, W, k, Ucount, Ulist, Doff, D);
    AFN_LAUNCH_CHECK("group_gemm_kernel");
    kt_end(KT_FSAI_GEMM, st, 2.0 * (double)k * (double)totD);
  }
  // ---- 4. per-row assembly + warp Cholesky, in batches
  const int64_t WP = (int64_t)MT * 16;
  const int64_t SPK = WP * (WP + 1) / 2;
  const int64_t NR = row_hi - row_lo;
  const int64_t batch = std::min<int64_t>(NR, std::max<int64_t>(4096, (int64_t)(1LL << 30) / (SPK * 8)));
  double* Sg;
  if ((s = get((void**)&Sg, sizeof(double) * SPK * batch)) != AFN_OK) return s;
  const double cl = AFN_LOG2E / (l * l);
  for (int64_t r0 = row_lo; r0 < row_hi; r0 += batch) {
    const int64_t nr = std::min(batch, row_hi - r0);
    const unsigned grid = (unsigned)nr;
    kt_begin(KT_FSAI_ASM, st);
    switch (MT) {
      case 1: launch_assemble<1>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 2: launch_assemble<2>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 3: launch_assemble<3>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 4: launch_assemble<4>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 5: launch_assemble<5>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 6: launch_assemble<6>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      case 7: launch_assemble<7>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
      default: launch_assemble<8>(grid, st, r0, X2, d, cl, mu, rp, col, grp, loc, Ucount, Ulist, Doff, D, Sg); break;
    }
    AFN_LAUNCH_CHECK("fsai_assemble_kernel");
    kt_end(KT_FSAI_ASM, st, 0.0);
    kt_begin(KT_FSAI_CHOL, st);
    if ((s = fsai_chol_batch(r0, nr, MT, rp, Sg, gval, d_info, st)) != AFN_OK) return s;
    kt_end(KT_FSAI_CHOL, st, (double)nr * ((double)w * w * w / 3.0 + (double)w * w));
  }
  return AFN_OK;
}

}  // namespace afn

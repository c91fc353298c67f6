// fsai.cu -- FSAI factor G of the regularised Schur complement
//   S = K22 + mu I - K21 (K11 + mu I)^{-1} K12 = K22 + mu I - W W^T
// on the kNN pattern (Kolotilina-Yeremin).
// "The computation of each row of G is independent" (L260-261): one CTA per
// row i with pattern J (ascending, i last, |J| <= 128):
//   1. Gram  W_J W_J^T  (lower triangle only): W rows gathered in 32-column
//      chunks through double-buffered shared memory (cp.async), 16x16 threads
//      with stride-16 register micro-tiles;
//   2. S_JJ = K(X_J, X_J) + mu I - Gram  (packed lower, shared memory);
//   3. R R^T = S_JJ (right-looking Cholesky in shared memory);
//   4. g = R^{-T} e_last  (= the last row of R^{-1}): with this normalisation
//      (G S)_{iJ} = e_i^T / G_ii on the pattern and diag(G S G^T) = 1 (R16).
// Then G^T is built as its own CSR (deterministic rank placement).
#include <algorithm>
#include <cmath>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int FT = 256;  // threads
constexpr int KC = 32;   // W columns per chunk

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ int pk(int a, int b) { return a * (a + 1) / 2 + b; }  // packed lower, b <= a

template <int MT>
__global__ void __launch_bounds__(FT, 2)
fsai_kernel(const double* __restrict__ X2, int64_t N, int d, double cl, double mu,
            const double* __restrict__ W, int64_t k, const int64_t* __restrict__ rp,
            const int32_t* __restrict__ col, double* __restrict__ gval, int* info) {
  constexpr int WP = MT * 16;
  constexpr int PW = WP + 1;  // staging pitch
  extern __shared__ __align__(16) double smem[];
  // layout: [ union{ staging 2*KC*PW , S packed WP*(WP+1)/2 } | X_J WP*d | J ]
  constexpr int STG = 2 * KC * PW;
  constexpr int SPK = WP * (WP + 1) / 2;
  constexpr int U = STG > SPK ? STG : SPK;
  double* stg = smem;
  double* S = smem;
  double* sX = smem + U;
  int* sJ = reinterpret_cast<int*>(sX + WP * d);
  __shared__ double s_tab[16];
  __shared__ int s_bad;

  const int64_t i = blockIdx.x;
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  load_exp2_tab(s_tab);
  if (tid == 0) s_bad = 0;
  for (int a = tid; a < WP; a += FT) sJ[a] = a < wp ? col[beg + a] : -1;
  __syncthreads();
  for (int e = tid; e < WP * d; e += FT) {
    const int a = e / d, c = e - a * d;
    sX[e] = sJ[a] >= 0 ? X2[(int64_t)sJ[a] * d + c] : 0.0;
  }

  // ---------------- 1. Gram (lower blocks j <= i of the stride-16 tiling)
  double acc[MT * (MT + 1) / 2];
#pragma unroll
  for (int t = 0; t < MT * (MT + 1) / 2; ++t) acc[t] = 0.0;

  const int64_t nch = (k + KC - 1) / KC;
  auto issue = [&](int64_t ch, int buf) {
    double* dst = stg + buf * KC * PW;
    const int64_t c0 = ch * KC;
    for (int e = tid; e < WP * KC; e += FT) {
      const int a = e / KC, kk = e - a * KC;
      const int64_t c = c0 + kk;
      const int ja = sJ[a];
      if (ja >= 0 && c < k) cp_async8(&dst[kk * PW + a], &W[(int64_t)ja * k + c]);
      else dst[kk * PW + a] = 0.0;
    }
    cp_async_commit();
  };
  if (nch > 0) issue(0, 0);
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int buf = (int)(ch & 1);
    if (ch + 1 < nch) {
      issue(ch + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* T = stg + buf * KC * PW;
#pragma unroll 2
    for (int kk = 0; kk < KC; ++kk) {
      double a[MT], b[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        a[m] = T[kk * PW + ty + 16 * m];
        b[m] = T[kk * PW + tx + 16 * m];
      }
      int t = 0;
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int q = 0; q <= m; ++q) {
          acc[t] = fma(a[m], b[q], acc[t]);
          ++t;
        }
    }
    __syncthreads();  // buffer `buf` is refilled by the next-next issue
  }

  // ---------------- 2. S_JJ = K_JJ + mu I - Gram  (packed lower)
  {
    int t = 0;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int q = 0; q <= m; ++q) {
        const int a = ty + 16 * m, b = tx + 16 * q;
        if (b <= a && a < wp) {
          double kv;
          if (a == b) {
            kv = 1.0 + mu;
          } else {
            const double s = d2_exact_rt(&sX[a * d], &sX[b * d], d);
            kv = gauss_from_d2(s, cl, s_tab);
          }
          S[pk(a, b)] = kv - acc[t];
        }
        ++t;
      }
  }
  __syncthreads();

  // ---------------- 3. Cholesky (right-looking, packed lower)
  for (int j = 0; j < wp; ++j) {
    if (tid == 0) {
      const double p = S[pk(j, j)];
      if (!(p > 0.0)) {
        if (!s_bad) { s_bad = 1; atomicCAS(info, 0, (int)(i + 1)); }
        S[pk(j, j)] = 1.0;
      } else {
        S[pk(j, j)] = sqrt(p);
      }
    }
    __syncthreads();
    const double piv = S[pk(j, j)];
    for (int a = j + 1 + tid; a < wp; a += FT) S[pk(a, j)] /= piv;
    __syncthreads();
    for (int a = j + 1 + ty; a < wp; a += 16) {
      const double sa = S[pk(a, j)];
      for (int b = j + 1 + tx; b <= a; b += 16) S[pk(a, b)] = fma(-sa, S[pk(b, j)], S[pk(a, b)]);
    }
    __syncthreads();
  }

  // ---------------- 4. g = R^{-T} e_last  (one warp, back substitution)
  if (tid < 32) {
    const int lane = tid;
    double rhs[WP / 32 > 0 ? (WP + 31) / 32 : 1];
#pragma unroll
    for (int s = 0; s < (WP + 31) / 32; ++s) {
      const int t = lane + 32 * s;
      rhs[s] = (t == wp - 1) ? 1.0 : 0.0;
    }
    for (int j = wp - 1; j >= 0; --j) {
      double gj = 0.0;
#pragma unroll
      for (int s = 0; s < (WP + 31) / 32; ++s)
        if (lane + 32 * s == j) gj = rhs[s] / S[pk(j, j)];
      gj = __shfl_sync(0xffffffffu, gj, j & 31);
#pragma unroll
      for (int s = 0; s < (WP + 31) / 32; ++s) {
        const int t = lane + 32 * s;
        if (t < j) rhs[s] = fma(-S[pk(j, t)], gj, rhs[s]);
        else if (t == j) rhs[s] = gj;
      }
    }
#pragma unroll
    for (int s = 0; s < (WP + 31) / 32; ++s) {
      const int t = lane + 32 * s;
      if (t < wp) gval[beg + t] = rhs[s];
    }
  }
}

template <int MT>
afn_status launch_fsai(const double* X2, int64_t N, int d, double cl, double mu, const double* W,
                       int64_t k, const int64_t* rp, const int32_t* col, double* gval, int* info,
                       cudaStream_t st) {
  constexpr int WP = MT * 16;
  constexpr int PW = WP + 1;
  constexpr int STG = 2 * KC * PW;
  constexpr int SPK = WP * (WP + 1) / 2;
  constexpr int U = STG > SPK ? STG : SPK;
  const size_t bytes = sizeof(double) * (U + (size_t)WP * d) + sizeof(int) * WP + 16;
  auto kern = fsai_kernel<MT>;
  AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  kern<<<(unsigned)N, FT, bytes, st>>>(X2, N, d, cl, mu, W, k, rp, col, gval, info);
  AFN_LAUNCH_CHECK("fsai_kernel");
  return AFN_OK;
}

// ---- CSR transpose -----------------------------------------------------------
__global__ void count_cols_kernel(const int32_t* __restrict__ col, int64_t nnz, int* __restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) atomicAdd(&cnt[col[e]], 1);
}

// single-block exclusive scan of cnt[0..N) into trp[0..N]
__global__ void scan_kernel(const int* __restrict__ cnt, int64_t N, int64_t* __restrict__ trp) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (N + 1023) / 1024;
  const int64_t b = tid * per, e = min(N, b + per);
  int64_t s = 0;
  for (int64_t t = b; t < e; ++t) s += cnt[t];
  part[tid] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int64_t run = tid > 0 ? part[tid - 1] : 0;
  for (int64_t t = b; t < e; ++t) {
    trp[t] = run;
    run += cnt[t];
  }
  if (tid == 1023) trp[N] = part[1023];
}

// scatter entries to their column segment (arbitrary order inside a segment)
__global__ void fill_cols_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 int64_t N, const int64_t* __restrict__ trp, int* __restrict__ cur,
                                 int32_t* __restrict__ trow_tmp) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
    const int c = col[e];
    const int pos = atomicAdd(&cur[c], 1);
    trow_tmp[trp[c] + pos] = (int32_t)r;
  }
}

// deterministic placement: rank of each row index inside its column segment;
// values fetched from G by binary search of column c in row r
__global__ void rank_cols_kernel(const int64_t* __restrict__ trp, const int32_t* __restrict__ trow_tmp,
                                 int64_t N, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 int32_t* __restrict__ tcol, double* __restrict__ tval) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= N) return;
  const int64_t b = trp[c], e = trp[c + 1];
  for (int64_t t = b + lane; t < e; t += 32) {
    const int32_t r = trow_tmp[t];
    int64_t rank = 0;
    for (int64_t u = b; u < e; ++u) rank += (trow_tmp[u] < r);
    // locate (r, c) in row r of G (columns ascending)
    int64_t lo = rp[r], hi = rp[r + 1] - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < c) lo = mid + 1; else hi = mid;
    }
    tcol[b + rank] = r;
    tval[b + rank] = val[lo];
  }
}

}  // namespace

afn_status fsai_run(const double* X2, int64_t N, int d, double l, double mu, const double* W,
                    int64_t k, const int64_t* rp, const int32_t* col, double* gval, int* d_info,
                    cudaStream_t st) {
  AFN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  if (N <= 0) return AFN_OK;
  // pattern width: all rows have <= w entries; the caller guarantees w <= 128
  int w = 0;
  {
    int64_t h[2];
    AFN_CUDA(cudaMemcpyAsync(h, rp + (N > 1 ? N - 1 : 0), sizeof(int64_t) * (N > 1 ? 2 : 1),
                             cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    // the widest row is the last one (rows grow then stay at w)
    w = (int)(N > 1 ? (h[1] - h[0]) : h[0]);
    if (N == 1) w = 1;
  }
  const double cl = AFN_LOG2E / (l * l);
  const int MT = (w + 15) / 16;
  switch (MT) {
    case 1: return launch_fsai<1>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 2: return launch_fsai<2>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 3: return launch_fsai<3>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 4: return launch_fsai<4>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 5: return launch_fsai<5>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 6: return launch_fsai<6>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 7: return launch_fsai<7>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    case 8: return launch_fsai<8>(X2, N, d, cl, mu, W, k, rp, col, gval, d_info, st);
    default: set_error("fsai: row width %d unsupported (<= 128)", w); return AFN_ERR_ARG;
  }
}

afn_status csr_transpose(const int64_t* rp, const int32_t* col, const double* val, int64_t N,
                         int64_t nnz, int64_t* trp, int32_t* tcol, double* tval, cudaStream_t st) {
  if (N <= 0) return AFN_OK;
  int* cnt = nullptr;
  int32_t* tmp = nullptr;
  afn_status s = dalloc((void**)&cnt, sizeof(int) * 2 * N, st);
  if (s != AFN_OK) return s;
  s = dalloc((void**)&tmp, sizeof(int32_t) * (nnz > 0 ? nnz : 1), st);
  if (s != AFN_OK) { dfree(cnt, st); return s; }
  int* cur = cnt + N;
  AFN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * N, st));
  count_cols_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(col, nnz, cnt);
  AFN_LAUNCH_CHECK("count_cols_kernel");
  scan_kernel<<<1, 1024, 0, st>>>(cnt, N, trp);
  AFN_LAUNCH_CHECK("scan_kernel");
  fill_cols_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(rp, col, N, trp, cur, tmp);
  AFN_LAUNCH_CHECK("fill_cols_kernel");
  rank_cols_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(trp, tmp, N, rp, col, val, tcol, tval);
  AFN_LAUNCH_CHECK("rank_cols_kernel");
  dfree(tmp, st);
  dfree(cnt, st);
  return AFN_OK;
}

}  // namespace afn

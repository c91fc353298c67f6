// fsai.cu -- FSAI factor G of the regularised Schur complement
//   S = K22 + mu I - K21 (K11 + mu I)^{-1} K12 = K22 + mu I - W W^T
// on the kNN pattern (Kolotilina-Yeremin).
// "The computation of each row of G is independent" (L260-261).  This file
// holds the per-row fallback used when the pair-union path (fsai_sddmm.cu)
// does not apply (a group's pair union overflows, or rows wider than 128):
// one CTA per row i with pattern J (ascending, i last, |J| <= 128):
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
#include <cstdlib>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
afn_status fsai_chol_batch(int64_t r0, int64_t nrows, int MT, const int64_t* rp, double* Sg,
                           double* gval, int* info, cudaStream_t st);
namespace {

constexpr int FT = 256;  // threads
constexpr int KC = 32;   // W columns per chunk
constexpr int GSTAGES = 3;  // cp.async pipeline depth of the split Gram kernel

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ int pk(int a, int b) { return a * (a + 1) / 2 + b; }  // packed lower, b <= a
// column-major packed lower of a wp x wp matrix: entry (a, t), a >= t
__device__ __forceinline__ int cmo(int a, int t, int wp) { return t * wp - (t * (t - 1)) / 2 + (a - t); }

// ---------------------------------------------------------------------------
// Split variant: (1) fsai_gram_kernel computes S_JJ (packed lower) for a batch
// of rows into global memory with the same register-tiled Gram as above but no
// in-CTA Cholesky; (2) fsai_chol_kernel factors each S_JJ with one warp
// (left-looking Cholesky, L1-resident) and back-substitutes for g.  The
// latency-bound factorisation then runs at full warp parallelism instead of
// stalling a 256-thread CTA with two barriers per column.
template <int MT>
__global__ void __launch_bounds__(FT, 2)
fsai_gram_kernel(const double* __restrict__ X2, int64_t r0, int d, KernelFn kf, double mu,
                 const double* __restrict__ W, int64_t k, const int64_t* __restrict__ rp,
                 const int32_t* __restrict__ col, double* __restrict__ Sg) {
  constexpr int WP = MT * 16;
  constexpr int PW2 = 2 * WP + 2;          // pitch of one kk-pair row (double2 per a)
  constexpr int SPK = WP * (WP + 1) / 2;
  extern __shared__ __align__(16) double smem[];
  constexpr int STG1 = (KC / 2) * PW2;      // one staging buffer
  constexpr int STG = GSTAGES * STG1;
  double* stg = smem;
  double* sX = smem + STG;
  int* sJ = reinterpret_cast<int*>(sX + WP * d);
  __shared__ double s_tab[AFN_EXP2_TAB_N];

  const int64_t i = r0 + blockIdx.x;
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  load_exp2_tab(s_tab);
  for (int a = tid; a < WP; a += FT) sJ[a] = a < wp ? col[beg + a] : -1;
  __syncthreads();
  for (int e = tid; e < WP * d; e += FT) {
    const int a = e / d, c = e - a * d;
    sX[e] = sJ[a] >= 0 ? X2[(int64_t)sJ[a] * d + c] : 0.0;
  }
  double acc[MT * (MT + 1) / 2];
#pragma unroll
  for (int t = 0; t < MT * (MT + 1) / 2; ++t) acc[t] = 0.0;
  const int64_t nch = (k + KC - 1) / KC;
  auto issue = [&](int64_t ch, int buf) {
    double* dst = stg + buf * STG1;
    const int64_t c0 = ch * KC;
    for (int e = tid; e < WP * KC; e += FT) {
      const int a = e / KC, kk = e - a * KC;
      const int64_t c = c0 + kk;
      const int ja = sJ[a];
      double* q = &dst[(kk >> 1) * PW2 + 2 * a + (kk & 1)];
      if (ja >= 0 && c < k) cp_async8(q, &W[(int64_t)ja * k + c]);
      else *q = 0.0;
    }
    cp_async_commit();
  };
  // GSTAGES-deep cp.async pipeline over the k chunks
#pragma unroll
  for (int st0 = 0; st0 < GSTAGES - 1; ++st0) {
    if (st0 < nch) issue(st0, st0);
    else cp_async_commit();
  }
  for (int64_t ch = 0; ch < nch; ++ch) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    const int64_t nx = ch + GSTAGES - 1;
    if (nx < nch) issue(nx, (int)(nx % GSTAGES));
    else cp_async_commit();
    const double* T = stg + (int)(ch % GSTAGES) * STG1;
#pragma unroll 1
    for (int k2 = 0; k2 < KC / 2; ++k2) {
      double2 a[MT], b[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        a[m] = *reinterpret_cast<const double2*>(&T[k2 * PW2 + 2 * (ty + 16 * m)]);
        b[m] = *reinterpret_cast<const double2*>(&T[k2 * PW2 + 2 * (tx + 16 * m)]);
      }
      int t = 0;
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int q = 0; q <= m; ++q) {
          acc[t] = fma(a[m].x, b[q].x, acc[t]);
          acc[t] = fma(a[m].y, b[q].y, acc[t]);
          ++t;
        }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  double* S = Sg + (int64_t)blockIdx.x * SPK;
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
          const double sd = d2_exact_rt(&sX[a * d], &sX[b * d], d);
          kv = kern_from_d2(kf, sd, s_tab);
        }
        S[cmo(a, b, wp)] = kv - acc[t];
      }
      ++t;
    }
}

// one warp per row: blocked left-looking (Crout) Cholesky of S_JJ, then
// g = R^{-T} e_last.  S arrives column-major packed lower (entry (a, t),
// a >= t, at cmo(a, t, wp)) with row stride spk in Sg, so the lanes'
// row-parallel updates read consecutive addresses.  Columns are factored in
// panels of 4: each loaded L[a][t] feeds 4 FMAs (one per panel column) before
// the in-panel solve.  RR: rows per lane (wp <= 32 RR).  GLB = false: the
// matrix is copied to shared memory (wmax(wmax+1)/2 + wmax doubles per warp,
// blockDim = 32 * CW); GLB = true (wide rows): factored in place in global
// memory (L2), g in the spk - wp(wp+1)/2 >= wp doubles after it.
template <int RR, bool GLB>
__global__ void __launch_bounds__(256)
fsai_chol_kernel(int64_t r0, int64_t nrows, int wmax, const int64_t* __restrict__ rp,
                 double* __restrict__ Sg, int64_t spk, double* __restrict__ gval, int* info) {
  extern __shared__ __align__(16) double csm[];
  const int CW = blockDim.x >> 5;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wr = (int64_t)blockIdx.x * CW + wid;
  if (wr >= nrows) return;
  const int64_t i = r0 + wr;
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  const int ne = wp * (wp + 1) / 2;
  double* L;
  double* gs;
  if (GLB) {
    L = Sg + wr * spk;
    gs = L + ne;
  } else {
    const int per = wmax * (wmax + 1) / 2 + wmax;
    L = csm + (int64_t)wid * per;
    gs = L + wmax * (wmax + 1) / 2;
    const double* src = Sg + wr * spk;
    for (int e = lane; e < ne; e += 32) L[e] = src[e];
    __syncwarp();
  }
  bool bad = false;
  for (int j0 = 0; j0 < wp; j0 += 4) {
    const int nc = min(4, wp - j0);
    double acc[RR][4];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int a = j0 + lane + 32 * r;
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = (c < nc && a < wp && a >= j0 + c) ? L[cmo(a, j0 + c, wp)] : 0.0;
    }
    int cb = 0;  // column base of column t: t*wp - t(t-1)/2
    for (int t = 0; t < j0; ++t) {
      double lj[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) lj[c] = c < nc ? L[cb + j0 + c - t] : 0.0;
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const int a = j0 + lane + 32 * r;
        const double la = a < wp ? L[cb + a - t] : 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(-la, lj[c], acc[r][c]);
      }
      cb += wp - t;
    }
    // in-panel factorisation (row j0 + c is lane c, r = 0)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= nc) break;
      const int j = j0 + c;
      double dj = __shfl_sync(0xffffffffu, acc[0][c], c);
      if (!(dj > 0.0)) { bad = true; dj = 1.0; }
      const double piv = sqrt(dj);
      const double inv = 1.0 / piv;
      double lv[RR];
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const int a = j0 + lane + 32 * r;
        lv[r] = (a > j && a < wp) ? acc[r][c] * inv : 0.0;
        if (a > j && a < wp) L[cmo(a, j, wp)] = lv[r];
      }
      if (lane == c) L[cmo(j, j, wp)] = piv;
#pragma unroll
      for (int c2 = c + 1; c2 < 4; ++c2) {
        const double l2 = __shfl_sync(0xffffffffu, lv[0], c2);  // L[j0 + c2][j]
#pragma unroll
        for (int r = 0; r < RR; ++r) acc[r][c2] = fma(-lv[r], l2, acc[r][c2]);
      }
    }
    __syncwarp();
  }
  if (bad && lane == 0) atomicCAS(info, 0, (int)(i + 1));
  // g_j = (e_j - sum_{t>j} R[t][j] g_t) / R[j][j], j = wp-1 .. 0 (column j contiguous)
  for (int j = wp - 1; j >= 0; --j) {
    double s = 0.0;
    const int cbj = cmo(j, j, wp);
    for (int t = j + 1 + lane; t < wp; t += 32) s = fma(L[cbj + t - j], gs[t], s);
    s = warp_sum(s);
    if (lane == 0) gs[j] = ((j == wp - 1 ? 1.0 : 0.0) - s) / L[cbj];
    __syncwarp();
  }
  for (int t = lane; t < wp; t += 32) gval[beg + t] = gs[t];
}

// Wide rows (|J| > 128, e.g. the paper's plain FSAI comparison with 400
// neighbours): S_JJ = K(X_J, X_J) + mu I - W_J W_J^T, column-major
// packed lower, one CTA per row straight into global memory (a warp per
// column, lanes over rows; the W dots, if any, read W through L2).
__global__ void __launch_bounds__(256)
fsai_wide_assemble_kernel(const double* __restrict__ X2, int64_t r0, int d, KernelFn kf, double mu,
                          const double* __restrict__ W, int64_t k, const int64_t* __restrict__ rp,
                          const int32_t* __restrict__ col, double* __restrict__ Sg, int64_t spk) {
  extern __shared__ __align__(16) double wsm[];  // X_J (wp x d)
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  __shared__ int sJ[AFN_W_MAX];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t i = r0 + blockIdx.x;
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  load_exp2_tab(s_tab);
  for (int a = tid; a < wp; a += 256) sJ[a] = col[beg + a];
  __syncthreads();
  for (int e = tid; e < wp * d; e += 256) {
    const int a = e / d, c = e - a * d;
    wsm[e] = X2[(int64_t)sJ[a] * d + c];
  }
  __syncthreads();
  double* S = Sg + (int64_t)blockIdx.x * spk;
  for (int t = wid; t < wp; t += 8) {
    const double* wt = W + (int64_t)sJ[t] * k;
    for (int a = t + lane; a < wp; a += 32) {
      double kv = a == t ? 1.0 + mu : kern_from_d2(kf, d2_exact_rt(&wsm[a * d], &wsm[t * d], d), s_tab);
      if (k > 0) {
        const double* wa = W + (int64_t)sJ[a] * k;
        double g = 0.0;
        for (int64_t c = 0; c < k; ++c) g = fma(wa[c], wt[c], g);
        kv -= g;
      }
      S[cmo(a, t, wp)] = kv;
    }
  }
}

afn_status launch_fsai_wide(const double* X2, int64_t row_lo, int64_t row_hi, int d, KernelFn kf, double mu,
                            const double* W, int64_t k, const int64_t* rp, const int32_t* col, int wmax,
                            double* gval, int* info, cudaStream_t st) {
  const int64_t spk = (int64_t)wmax * (wmax + 1) / 2 + wmax;
  const int64_t NR = row_hi - row_lo;
  const int64_t batch = std::min<int64_t>(NR, std::max<int64_t>(256, (int64_t)(1LL << 31) / (spk * 8)));
  double* Sg = nullptr;
  afn_status s = dalloc((void**)&Sg, sizeof(double) * spk * batch, st);
  if (s != AFN_OK) return s;
  const size_t abytes = sizeof(double) * (size_t)wmax * d;
  AFN_CUDA(cudaFuncSetAttribute(fsai_wide_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)abytes));
  const int CW = 8;
  for (int64_t r0 = row_lo; r0 < row_hi; r0 += batch) {
    const int64_t nr = std::min(batch, row_hi - r0);
    fsai_wide_assemble_kernel<<<(unsigned)nr, 256, abytes, st>>>(X2, r0, d, kf, mu, W, k, rp, col, Sg, spk);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
      note_launch();
      fsai_chol_kernel<16, true><<<(unsigned)((nr + CW - 1) / CW), CW * 32, 0, st>>>(r0, nr, wmax, rp, Sg, spk,
                                                                                      gval, info);
      e = cudaGetLastError();
      if (e == cudaSuccess) note_launch();
    }
    if (e != cudaSuccess) {
      dfree(Sg, st);
      return cuda_status(e, "fsai wide rows");
    }
  }
  dfree(Sg, st);
  return AFN_OK;
}

template <int MT>
afn_status launch_fsai_split(const double* X2, int64_t row_lo, int64_t row_hi, int d, KernelFn kf, double mu,
                             const double* W, int64_t k, const int64_t* rp, const int32_t* col,
                             double* gval, int* info, cudaStream_t st) {
  constexpr int WP = MT * 16;
  constexpr int PW = WP + 1;
  constexpr int64_t SPK = WP * (WP + 1) / 2;
  (void)PW;
  const size_t bytes = sizeof(double) * (GSTAGES * (size_t)(KC / 2) * (2 * WP + 2) + (size_t)WP * d) +
                       sizeof(int) * WP + 16;
  auto kg = fsai_gram_kernel<MT>;
  AFN_CUDA(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  const int64_t NR = row_hi - row_lo;
  const int64_t batch = std::min<int64_t>(NR, std::max<int64_t>(4096, (int64_t)(1LL << 30) / (SPK * 8)));
  double* Sg = nullptr;
  afn_status s = dalloc((void**)&Sg, sizeof(double) * SPK * batch, st);
  if (s != AFN_OK) return s;
  for (int64_t r0 = row_lo; r0 < row_hi; r0 += batch) {
    const int64_t nr = std::min(batch, row_hi - r0);
    kg<<<(unsigned)nr, FT, bytes, st>>>(X2, r0, d, kf, mu, W, k, rp, col, Sg);
    AFN_LAUNCH_CHECK("fsai_gram_kernel");
    afn_status cs = fsai_chol_batch(r0, nr, MT, rp, Sg, gval, info, st);
    if (cs != AFN_OK) { dfree(Sg, st); return cs; }
  }
  dfree(Sg, st);
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
                                 int32_t* __restrict__ tcol, double* __restrict__ tval,
                                 int64_t* __restrict__ tmap) {
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
    if (tval) tval[b + rank] = val[lo];
    if (tmap) tmap[b + rank] = lo;
  }
}

}  // namespace

template <int MT>
afn_status launch_chol(int64_t r0, int64_t nrows, const int64_t* rp, double* Sg, double* gval, int* info,
                       cudaStream_t st) {
  constexpr int WP = MT * 16;
  // widest row of the batch (rows grow to w and stay there)
  int64_t h2[2];
  const int64_t last = r0 + nrows - 1;
  AFN_CUDA(cudaMemcpyAsync(h2, rp + last, sizeof(int64_t) * 2, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  const int wmax = std::max(1, std::min(WP, (int)(h2[1] - h2[0])));
  const size_t per = sizeof(double) * ((size_t)wmax * (wmax + 1) / 2 + wmax);
  const int CW = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(220 * 1024) / per));
  const size_t bytes = per * CW;
  auto kern = fsai_chol_kernel<4, false>;
  AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  kern<<<(unsigned)((nrows + CW - 1) / CW), CW * 32, bytes, st>>>(r0, nrows, wmax, rp, Sg,
                                                                 (int64_t)WP * (WP + 1) / 2, gval, info);
  AFN_LAUNCH_CHECK("fsai_chol_kernel");
  return AFN_OK;
}

afn_status fsai_chol_batch(int64_t r0, int64_t nrows, int MT, const int64_t* rp, double* Sg,
                           double* gval, int* info, cudaStream_t st) {
  switch (MT) {
    case 1: return launch_chol<1>(r0, nrows, rp, Sg, gval, info, st);
    case 2: return launch_chol<2>(r0, nrows, rp, Sg, gval, info, st);
    case 3: return launch_chol<3>(r0, nrows, rp, Sg, gval, info, st);
    case 4: return launch_chol<4>(r0, nrows, rp, Sg, gval, info, st);
    case 5: return launch_chol<5>(r0, nrows, rp, Sg, gval, info, st);
    case 6: return launch_chol<6>(r0, nrows, rp, Sg, gval, info, st);
    case 7: return launch_chol<7>(r0, nrows, rp, Sg, gval, info, st);
    default: return launch_chol<8>(r0, nrows, rp, Sg, gval, info, st);
  }
}

afn_status fsai_run(const double* X2, int64_t N, int d, Kern kn, double mu, const double* W,
                    int64_t k, const int64_t* rp, const int32_t* col, int64_t row_lo, int64_t row_hi,
                    double* gval, int* d_info, cudaStream_t st) {
  AFN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  if (N <= 0 || row_hi <= row_lo) return AFN_OK;
  // pattern width: all rows have <= w entries (the widest row is the last
  // one: rows grow then stay at w); w <= AFN_W_MAX
  int w = 0;
  {
    int64_t h[2];
    AFN_CUDA(cudaMemcpyAsync(h, rp + (N > 1 ? N - 1 : 0), sizeof(int64_t) * (N > 1 ? 2 : 1),
                             cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    w = (int)(N > 1 ? (h[1] - h[0]) : h[0]);
    if (N == 1) w = 1;
  }
  const KernelFn kf = kernel_fn(kn.kind, kn.l);
  const int MT = (w + 15) / 16;
  switch (MT) {
    case 1: return launch_fsai_split<1>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 2: return launch_fsai_split<2>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 3: return launch_fsai_split<3>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 4: return launch_fsai_split<4>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 5: return launch_fsai_split<5>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 6: return launch_fsai_split<6>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 7: return launch_fsai_split<7>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    case 8: return launch_fsai_split<8>(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, gval, d_info, st);
    default:
      if (w > AFN_W_MAX) {
        set_error("fsai: row width %d unsupported (<= %d)", w, AFN_W_MAX);
        return AFN_ERR_ARG;
      }
      return launch_fsai_wide(X2, row_lo, row_hi, d, kf, mu, W, k, rp, col, w, gval, d_info, st);
  }
}

__global__ void gather_map_kernel(const double* __restrict__ v, const int64_t* __restrict__ map,
                                  int64_t nnz, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) out[e] = v[map[e]];
}

afn_status gather_map(const double* v, const int64_t* map, int64_t nnz, double* out, cudaStream_t st) {
  if (nnz <= 0) return AFN_OK;
  gather_map_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(v, map, nnz, out);
  AFN_LAUNCH_CHECK("gather_map_kernel");
  return AFN_OK;
}

afn_status csr_transpose(const int64_t* rp, const int32_t* col, const double* val, int64_t N,
                         int64_t nnz, int64_t* trp, int32_t* tcol, double* tval, cudaStream_t st,
                         int64_t* tmap) {
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
  rank_cols_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(trp, tmp, N, rp, col, val, tcol, tval, tmap);
  AFN_LAUNCH_CHECK("rank_cols_kernel");
  dfree(tmp, st);
  dfree(cnt, st);
  return AFN_OK;
}

}  // namespace afn

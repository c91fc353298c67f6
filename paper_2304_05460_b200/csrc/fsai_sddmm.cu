// fsai_sddmm.cu -- FSAI rows from the UNION of needed Schur-complement pairs.
//
// Every FSAI row i needs S_ab = K_ab + mu delta_ab - W_a . W_b for all a, b in
// its pattern J_i ("only requires the entries ... corresponding
// to the sparsity pattern").  Forming each row's Gram W_J W_J^T separately
// evaluates every needed pair ~14 times (a pair of nearby points belongs to
// many rows' patterns).  Here each needed dot product W_a . W_b (b <= a) is
// evaluated once, in dense blocks:
//   1. spatial order: non-landmark points sorted by grid cell (tiled cell
//      order), consecutive GA = 32 points form a group g;
//   2. U_g = union over a in g of B_a = { b : pos(b) <= pos(a), a, b in J_i
//      for some row i } (pos = place in the spatial order; rows containing a
//      come from the transposed pattern, scanned as ascending positions up to
//      pos(a)), numbered in the slot order of a hash set whose global copy
//      maps pos(b) -> the column of b in U_g.  Each unordered
//      pair is kept by the spatially later point, so a group's union holds
//      only the half of its neighbourhood that precedes it in the spatial
//      order (index order b <= a kept nearly all of it: a group's 32 indices
//      are scattered; C3 2.0x fewer dots);
//   3. D_g = W_g W_{U_g}^T (GA x |U_g|, k-long FP64 dots; register-tiled,
//      cp.async-staged through shared memory) -- ~4x fewer flops than the
//      per-row Gram on the C2 pattern;
//   4. per row (one CTA): S_JJ assembled by hash look-up of the earlier point
//      in the union of the later one's group,
//      blocked Cholesky in shared memory, g = L^{-T} e_last.
// Values are independent of the grouping and of which point of a pair keeps
// it (each dot has a fixed summation order, and W_a . W_b and W_b . W_a round
// the same products), so the result is deterministic even though the cell
// sort uses atomics.
#include <type_traits>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {

namespace {

// group size (points a per group): 32 reads each union column's W row once
// per 32 rows (the k = 4000 / 8000 products are bound by that traffic) for
// ~27 % more dots than 16 -- C3 135.7 -> 98.8 ms, C5 2643 -> 1919 ms, C2
// 3.86 -> 3.66 ms per product.  (A TMA bulk-copy variant with 4 stages of
// 256-byte row chunks, 1 CTA/SM, measured 2-3x slower.)
// (with the spatial-order unions: GA = 16 C3 100.9 ms / C2 3.08, GA = 64
// 71.0 / 3.15, GA = 32 56.0 / 2.72 ms)
constexpr int GA = 32;
constexpr int UCAP = 4096;   // max |U_g|
constexpr int HC = 8192;     // hash capacity (power of two)
constexpr int TH = HC;       // tile-table capacity of the Z-mode unions (>= 2 |U_g|: never full)

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
  int morton; // tiles in Z (Morton) order over a power-of-two tile grid, else raster
  int64_t ncell;  // key space (cells, with the Morton padding)
};

__device__ __forceinline__ int64_t spread3(int64_t v) {  // bit i -> bit 3 i (v < 2^20)
  int64_t r = 0;
  for (int b = 0; b < 20; ++b) r |= ((v >> b) & 1) << (3 * b);
  return r;
}

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
  const int64_t tile = cg.morton ? (spread3(b0) | (spread3(b1) << 1) | (spread3(b2) << 2))
                                 : ((int64_t)b2 * cg.nb[1] + b1) * cg.nb[0] + b0;
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

__global__ void pass_count_kernel(const int* __restrict__ Ucount, int64_t G, int ut, int* __restrict__ pc) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < G) pc[g] = (Ucount[g] + ut - 1) / ut;
}

// colp: each pattern row's columns as spatial positions, ascending (one warp
// per row, bitonic sort of <= 128 keys in registers, 4 per lane)
__global__ void pattern_positions_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                         const int* __restrict__ grp, const int* __restrict__ loc, int ga,
                                         int64_t N, int32_t* __restrict__ colp) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  const int64_t b0 = rp[i];
  const int len = (int)(rp[i + 1] - b0);  // <= 128
  int k[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = r * 32 + lane;
    k[r] = e < len ? grp[col[b0 + e]] * ga + loc[col[b0 + e]] : 0x7fffffff;
  }
  // element e = r * 32 + lane; bitonic network over the 128 elements
#pragma unroll
  for (int sz = 2; sz <= 128; sz <<= 1) {
#pragma unroll
    for (int st = sz >> 1; st > 0; st >>= 1) {
      if (st >= 32) {  // partners in another register of the same lane
        const int m = st >> 5;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r & m) continue;
          const int r2 = r | m;
          const bool up = ((r * 32 + lane) & sz) == 0;
          const int lo = min(k[r], k[r2]), hi = max(k[r], k[r2]);
          k[r] = up ? lo : hi;
          k[r2] = up ? hi : lo;
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int other = __shfl_xor_sync(0xffffffffu, k[r], st);
          const bool up = ((r * 32 + lane) & sz) == 0;
          const bool lower = (lane & st) == 0;
          k[r] = (lower == up) ? min(k[r], other) : max(k[r], other);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = r * 32 + lane;
    if (e < len) colp[b0 + e] = k[r];
  }
}

__global__ void group_maps_kernel(const int* __restrict__ sorder, int64_t N, int ga, int* __restrict__ grp,
                                  int* __restrict__ loc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  const int a = sorder[t];
  grp[a] = (int)(t / ga);
  loc[a] = (int)(t % ga);
}

// ---------------------------------------------------------------- group unions
// One CTA per group g: insert every needed b (b <= a, a in g, a and b in the
// pattern of a row this rank factors) into a shared-memory hash set (linear
// probing), then number the keys in slot order: U_g[u] (the GEMM's column
// list) and the global copy of the table H_g[slot] = (b, u) that the factor
// kernel uses to find W_a . W_b in D_g (one or two probes).  A warp walks
// one pattern row at a time, lanes over its entries.
__global__ void __launch_bounds__(256) group_union_kernel(const int* __restrict__ sorder, int64_t N,
                                                          const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ colp,
                                                          const int64_t* __restrict__ trp,
                                                          const int32_t* __restrict__ tcol,
                                                          int64_t row_lo, int64_t row_hi, int ga,
                                                          int* __restrict__ Ucount, int* __restrict__ Ulist,
                                                          int2* __restrict__ Htab, int* overflow) {
  extern __shared__ int hs[];  // HC keys (positions)
  __shared__ int s_n, s_ovf;
  __shared__ int s_scan[256];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t g = blockIdx.x;
  for (int t = tid; t < HC; t += 256) hs[t] = -1;
  if (tid == 0) s_n = 0, s_ovf = 0;
  __syncthreads();
  const int64_t m0 = g * ga;
  const int cnt = (int)min((int64_t)ga, N - m0);
  // at most UCAP keys fit (load factor <= 1/2): once s_n passes it every loop
  // stops (a hub point of a high-dimensional pattern can be in thousands of
  // rows) and the caller falls back to the per-row Gram
  for (int j = 0; j < cnt && !*(volatile int*)&s_ovf; ++j) {
    const int a = sorder[m0 + j];
    const int pa = (int)(m0 + j);
    for (int64_t e = trp[a] + wid; e < trp[a + 1] && !*(volatile int*)&s_ovf; e += 8) {
      const int i = tcol[e];
      if (i < row_lo || i >= row_hi) continue;  // rows this rank factors
      for (int64_t q = rp[i] + lane; q < rp[i + 1]; q += 32) {
        const int pb = colp[q];
        if (pb > pa) break;  // positions ascending: kept by the spatially later point
        unsigned h = ((unsigned)pb * 2654435761u) & (HC - 1);
        for (int probe = 0; probe < HC; ++probe) {
          const int old = atomicCAS(&hs[h], -1, pb);
          if (old == -1) {
            if (atomicAdd(&s_n, 1) >= UCAP) s_ovf = 1;
            break;
          }
          if (old == pb) break;
          h = (h + 1) & (HC - 1);
        }
        if (*(volatile int*)&s_ovf) break;
      }
    }
  }
  __syncthreads();
  const int nu = s_n;
  if (s_ovf || nu > UCAP) {
    if (tid == 0) atomicExch(overflow, 1);
    return;
  }
  constexpr int PER = HC / 256;
  // number the occupied slots in slot order (block scan over 32-slot strips)
  int c = 0;
  for (int t = 0; t < PER; ++t) c += hs[tid * PER + t] >= 0;
  s_scan[tid] = c;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int v = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int u = s_scan[tid] - c;
  int2* H = Htab + g * HC;
  for (int t = 0; t < PER; ++t) {
    const int slot = tid * PER + t;
    const int pb = hs[slot];
    if (pb >= 0) {
      Ulist[g * UCAP + u] = sorder[pb];  // (the product gathers W rows by point)
      H[slot] = make_int2(pb, u);
      ++u;
    } else {
      H[slot] = make_int2(-1, -1);
    }
  }
  if (tid == 0) Ucount[g] = nu;
}

// Z mode: renumber a group's union (already in its global hash table H_g,
// slot -> (position, column)) grouped by W-plan tile, list the pieces (<= 32
// columns of one tile) and count the products' MACs -- a separate pass, so
// that the union kernel keeps its small shared-memory footprint (the pattern
// walk is latency-bound: 96 KB per CTA there cost 8.4 vs ~3.4 ms at C3).
__global__ void __launch_bounds__(256) group_tile_renumber_kernel(
    const int* __restrict__ sorder, const int* __restrict__ Ucount, int* __restrict__ Ulist,
    int2* __restrict__ Htab, const int* __restrict__ tilerow, const int64_t* __restrict__ uoff,
    int2* __restrict__ Pc, int* __restrict__ Pcount, unsigned long long* __restrict__ zwork, int* overflow) {
  extern __shared__ int ts[];  // tile keys [TH], counts -> offsets + cursors [TH]
  __shared__ int s_scan[256];
  __shared__ int s_ovf;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t g = blockIdx.x;
  int* tk = ts;
  int* tc = ts + TH;
  for (int t = tid; t < TH; t += 256) {
    tk[t] = -1;
    tc[t] = 0;
  }
  if (tid == 0) s_ovf = 0;
  __syncthreads();
  int2* H = Htab + g * HC;
  auto tslot = [&](int tile, bool ins) {
    unsigned h = ((unsigned)tile * 2654435761u) & (TH - 1);
    for (int probe = 0; probe < TH; ++probe) {
      const int old = ins ? atomicCAS(&tk[h], -1, tile) : tk[h];
      if (old == tile || old == -1) return (int)h;
      h = (h + 1) & (TH - 1);
    }
    s_ovf = 1;
    return 0;
  };
  for (int slot = tid; slot < HC; slot += 256) {
    const int pb = H[slot].x;
    if (pb >= 0) atomicAdd(&tc[tslot(tilerow[sorder[pb]] >> 6, true)], 1);
  }
  __syncthreads();
  if (s_ovf) {
    if (tid == 0) atomicExch(overflow, 1);
    return;
  }
  constexpr int TPER = TH / 256;
  int cc = 0, pp = 0;
  for (int t = 0; t < TPER; ++t) {
    const int c1 = tc[tid * TPER + t];
    cc += c1;
    pp += (c1 + 31) / 32;
  }
  s_scan[tid] = cc;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int v = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int run = s_scan[tid] - cc;
  __syncthreads();
  s_scan[tid] = pp;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int v = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int prun = s_scan[tid] - pp;
  unsigned long long wk = 0ull;
  for (int t = 0; t < TPER; ++t) {
    const int slot = tid * TPER + t;
    const int c1 = tc[slot];
    tc[slot] = run;
    if (c1 > 0) {
      const int tile = tk[slot];
      wk += (unsigned long long)c1 * (unsigned long long)(uoff[tile + 1] - uoff[tile]);
      for (int q = 0; q < c1; q += 32) Pc[g * UCAP + prun++] = make_int2(run + q, min(32, c1 - q));
    }
    run += c1;
  }
  if (tid == 255) Pcount[g] = prun;
  for (int o = 16; o > 0; o >>= 1) wk += __shfl_xor_sync(0xffffffffu, wk, o);
  if (lane == 0) atomicAdd(zwork, wk * (unsigned long long)GA);
  __syncthreads();
  for (int slot = tid; slot < HC; slot += 256) {
    const int2 e = H[slot];
    if (e.x >= 0) {
      const int ts2 = tslot(tilerow[sorder[e.x]] >> 6, false);
      const int u = atomicAdd(&tc[ts2], 1);
      Ulist[g * UCAP + u] = sorder[e.x];
      H[slot] = make_int2(e.x, u);
    }
  }
  (void)Ucount;
}

// ---------------------------------------------------------------- group GEMM
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// D_g = W_g W_U^T on the FP64 tensor cores: mma.sync m8n8k4 f64 (SASS
// DMMA.8x8x4, 256 FMA per warp instruction; the DFMA register-tiled kernels
// it replaced were bound by instruction and operand traffic: C2 7.0 -> 3.7 ms).
// Warp w owns the 64 columns [64 w, 64 w + 64) of a 512-column pass: 2 x 8
// m8n8 tiles, 32 accumulators per thread.  Stages hold k-chunks of 8 per row
// at a 12-double stride (A/B fragment loads: 8 rows x 4 consecutive k per
// LDS.64 = 2 wavefronts, conflict-free).  Each dot is summed in k order in
// groups of 4 (the DMMA k-step).
constexpr int G16_NTL = GA == 16 ? 8 : (GA == 32 ? 4 : 2);  // n-tiles per warp: 32 x 4 tiles (passes of 256 columns) at GA = 32
constexpr int DNS = 2;  // cp.async stages (3 and 4 measured equal at C3 / C2: not latency-bound)
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// DKC = 16 (128-byte row chunks) when W is several times the L2: C3 (W 4.2
// GB) 98 -> 85 ms, its gathers of scattered rows being DRAM-bound; DKC = 8
// below (C2, W 0.23 GB: 3.7 vs 4.1 ms).
template <int DKC>
__global__ void __launch_bounds__(256, 2) group_gemm_dmma_kernel(
    const int* __restrict__ sorder, int64_t N, const double* __restrict__ W, int64_t k,
    const int* __restrict__ Ucount, const int* __restrict__ Ulist, const int64_t* __restrict__ Doff,
    const int64_t* __restrict__ Poff, int64_t G, double* __restrict__ D, const double* __restrict__ X2, int d,
    KernelFn kf, double mu, int64_t items) {
  // epilogue: D_g holds the Schur entries S_ab = K(x_a, x_b) + mu delta_ab - W_a . W_b
  // themselves (the factor kernel then only gathers them)
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  // warp = 2 x 8 m8n8 tiles (64 columns)
  constexpr int NS = DNS, DKP = DKC + 4;  // DKP = 4 or 12 mod 16: conflict-free fragment loads
  constexpr int MTL = GA / 8, NTL = G16_NTL, UTP = 8 * NTL * 8;
  extern __shared__ __align__(16) double gs[];
  double* sA = gs;                         // [NS][GA][DKP]
  double* sB = gs + NS * GA * DKP;         // [NS][UTP][DKP]
  __shared__ int s_a[GA];
  __shared__ int s_u[UTP];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  load_exp2_tab(s_tab);
  // persistent CTAs: round r takes items [r P, r P + P), P = gridDim.x (the
  // P items of a round are consecutive: spatially adjacent groups sharing
  // most union rows).  (A grid barrier between rounds, so that a round's CTAs
  // stream the same k-chunks together, measured slower -- C3 69.8 vs 56.4
  // ms: the product is tensor-pipe bound, 77 %, not DRAM-bound.)
  const int64_t rounds = (items + gridDim.x - 1) / gridDim.x;
  for (int64_t rd = 0; rd < rounds; ++rd) {
  const int64_t item = rd * gridDim.x + blockIdx.x;
  if (rd > 0) __syncthreads();  // (s_a / s_u / the stage buffers of the previous item)
  if (item >= items) continue;
  int64_t glo = 0, ghi = G;
  while (ghi - glo > 1) {
    const int64_t mid = (glo + ghi) >> 1;
    if (Poff[mid] <= item) glo = mid; else ghi = mid;
  }
  const int64_t g = glo;
  const int pass = (int)(item - Poff[g]);
  const int64_t m0 = g * GA;
  const int cnt = (int)min((int64_t)GA, N - m0);
  const int nu = Ucount[g];
  double* Dg = D + Doff[g];
  const int u0 = pass * UTP;
  const int un = min(UTP, nu - u0);
  if (tid < GA) s_a[tid] = tid < cnt ? sorder[m0 + tid] : -1;
  for (int t = tid; t < UTP; t += 256) s_u[t] = t < un ? Ulist[g * UCAP + u0 + t] : -1;
  __syncthreads();
  const int64_t nch = (k + DKC - 1) / DKC;
  const bool even = (k & 1) == 0;
  auto issue = [&](int64_t ch, int buf) {
    const int64_t c0 = ch * DKC;
    for (int e = tid; e < (GA + un) * (DKC / 2); e += 256) {
      const int row = e / (DKC / 2), part = e - row * (DKC / 2);
      const int id = row < GA ? s_a[row] : s_u[row - GA];
      double* dst = row < GA ? sA + (buf * GA + row) * DKP + 2 * part
                             : sB + ((int64_t)buf * UTP + (row - GA)) * DKP + 2 * part;
      const int64_t c = c0 + 2 * part;
      if (id >= 0 && c + 1 < k && even) {
        cpa16(dst, &W[(int64_t)id * k + c]);
      } else {
        dst[0] = (id >= 0 && c < k) ? W[(int64_t)id * k + c] : 0.0;
        dst[1] = (id >= 0 && c + 1 < k) ? W[(int64_t)id * k + c + 1] : 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[MTL][NTL][2];
#pragma unroll
  for (int mt = 0; mt < MTL; ++mt)
#pragma unroll
    for (int n = 0; n < NTL; ++n) acc[mt][n][0] = acc[mt][n][1] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NS - 1; ++s0) {
    if (s0 < nch) issue(s0, s0);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const bool wact = wid * NTL * 8 < un;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k index
  for (int64_t ch = 0; ch < nch; ++ch) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    __syncthreads();
    const int64_t nx = ch + NS - 1;
    if (nx < nch) issue(nx, (int)(nx % NS));
    else asm volatile("cp.async.commit_group;" ::: "memory");
    if (!wact) continue;
    const double* a = sA + (int)(ch % NS) * GA * DKP;
    const double* b = sB + ((int64_t)(ch % NS) * UTP + wid * NTL * 8) * DKP;
#pragma unroll
    for (int k4 = 0; k4 < DKC; k4 += 4) {
      double av[MTL];
#pragma unroll
      for (int mt = 0; mt < MTL; ++mt) av[mt] = a[(mt * 8 + fr) * DKP + k4 + fk];
#pragma unroll
      for (int n = 0; n < NTL; ++n) {
        const double bv = b[(n * 8 + fr) * DKP + k4 + fk];
#pragma unroll
        for (int mt = 0; mt < MTL; ++mt) dmma884(acc[mt][n][0], acc[mt][n][1], av[mt], bv);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // the stage buffers now hold the points of the rows and columns
  double* sxa = gs;             // [GA][d]
  double* sxb = gs + GA * d;    // [UTP][d]
  for (int e = tid; e < (GA + un) * d; e += 256) {
    const int row = e / d, c = e - row * d;
    const int id = row < GA ? s_a[row] : s_u[row - GA];
    (row < GA ? sxa : sxb - GA * d)[e] = id >= 0 ? X2[(int64_t)id * d + c] : 0.0;
  }
  __syncthreads();
  if (!wact) continue;
#pragma unroll
  for (int mt = 0; mt < MTL; ++mt) {
    const int j = mt * 8 + fr;
    if (j >= cnt) continue;
    const int a = s_a[j];
#pragma unroll
    for (int n = 0; n < NTL; ++n) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = wid * NTL * 8 + n * 8 + 2 * fk + h;
        if (u < un) {
          const int b = s_u[u];
          const double kv = a == b ? 1.0 + mu : kern_from_d2(kf, d2_exact_rt(&sxa[j * d], &sxb[u * d], d), s_tab);
          Dg[(int64_t)j * nu + u0 + u] = kv - acc[mt][n][h];
        }
      }
    }
  }
  }  // rounds
}

// ---------------------------------------------------------------- group product through Z
// D_g[a][u] = S_ab = K(x_a, x_b) + mu delta_ab - Z_a . k_b with Z = K21 M,
// M = (K11 + mu I)^{-1} (Z_a . k_b = k_a^T M k_b = W_a . W_b), k_b the row
// of K21 kept by the cutoff W plan (wcut.cu: its tile's landmark list U_t,
// over the landmarks' Morton order, and its row of the tile's K21 block).
// One CTA per half group (ZH = 16 rows a): the landmark columns the group's
// tiles keep, U' = union of their U_t, are marked in a shared bitmap over the
// k positions and the 16 Z rows are staged at those columns in shared memory
// once (k_b's columns are then looked up by the bitmap's prefix counts);
// warps take the pieces (<= 32 union columns of one tile): a 16 x 32 x |U_t|
// product on the FP64 tensor cores (DMMA m8n8k4), A fragments from the staged
// Z, B fragments from the tile's K21 rows in global memory.
//
// !STAGED (dense landmarks, U' too wide to stage): ZS consecutive CTAs share a
// group (all 32 rows), each taking every ZS-th piece; fragments straight from
// Z in global memory -- the CTAs in flight then cover few groups, whose Z
// rows stay in L2 (one CTA per whole group: C3 28.5 ms, DRAM 46 GB).
constexpr int ZH = 16;
constexpr int ZCAP = 1664;  // staged columns (16 x 1664 x 8 B = 208 KB); wider U' -> global loads
constexpr int ZS = 8;
template <bool STAGED>
__global__ void __launch_bounds__(STAGED ? 512 : 256, STAGED ? 1 : 2) group_zk_kernel(
    const int* __restrict__ sorder, int64_t N, const double* __restrict__ Zp, int64_t k,
    const int* __restrict__ tilerow, const int64_t* __restrict__ uoff, const int* __restrict__ ulistp,
    const int64_t* __restrict__ aoff, const double* __restrict__ Ap, const int* __restrict__ Ucount,
    const int* __restrict__ Ulist, const int64_t* __restrict__ Doff, const int2* __restrict__ Pc,
    const int* __restrict__ Pcount, double* __restrict__ D, const double* __restrict__ X2, int d, KernelFn kf,
    double mu) {
  extern __shared__ __align__(16) double zs[];  // [ZH][ncol] staged Z (ld = ncol)
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  __shared__ int s_a[GA];
  __shared__ unsigned s_bits[256];   // k <= 8192 positions
  __shared__ int s_pre[257];         // prefix counts of s_bits
  // STAGED: 16 warps (one CTA per SM by its shared memory; with 8 warps the C5 kernel had
  // 12.5 % occupancy and no eligible warp in 80 % of the cycles)
  constexpr int NW = STAGED ? 16 : 8;
  typedef typename std::conditional<STAGED, short, int>::type su_t;  // (k <= 8192)
  __shared__ su_t s_u[NW][256];      // per warp: the piece's U_t as staged columns
  __shared__ long long s_pk[STAGED ? 1 : UCAP];  // !STAGED: (tile, piece) keys, sorted
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  load_exp2_tab(s_tab);
  constexpr int RH = STAGED ? ZH : GA;  // rows per CTA
  const int64_t g = STAGED ? (int64_t)(blockIdx.x >> 1) : (int64_t)(blockIdx.x / ZS);
  const int half = STAGED ? (int)(blockIdx.x & 1) : 0;
  const int pq = STAGED ? 0 : (int)(blockIdx.x % ZS);  // this CTA's share of the pieces
  const int pstep = STAGED ? NW : 8 * ZS;
  const int64_t m0 = g * GA + half * ZH;
  const int cnt = (int)max((int64_t)0, min((int64_t)RH, N - m0));
  if (tid < RH) s_a[tid] = tid < cnt ? sorder[m0 + tid] : -1;
  const int nwords = (int)((k + 31) / 32);
  for (int w = tid; w < 256; w += 256) s_bits[w] = 0u;
  __syncthreads();
  if (cnt == 0) return;
  const int nu = Ucount[g], np = Pcount[g];
  // mark U' (every piece's tile list)
  for (int p = wid; STAGED && p < np; p += NW) {
    const int tile = tilerow[Ulist[g * UCAP + Pc[g * UCAP + p].x]] >> 6;
    const int64_t us = uoff[tile], ue = uoff[tile + 1];
    for (int64_t m = us + lane; m < ue; m += 32) {
      const int pos = ulistp[m];
      atomicOr(&s_bits[pos >> 5], 1u << (pos & 31));
    }
  }
  __syncthreads();
  auto prefix = [&]() {
    if (tid == 0) {
      int run = 0;
      for (int w = 0; w < nwords; ++w) {
        s_pre[w] = run;
        run += __popc(s_bits[w]);
      }
      s_pre[nwords] = run;
    }
    __syncthreads();
  };
  if (STAGED) prefix();
  const int ncol = STAGED ? s_pre[nwords] : 0;
  const bool staged = STAGED && ncol <= ZCAP;
  if (staged) {  // Z rows at the marked columns (a warp per row, lanes over bitmap words)
    for (int r = wid; r < ZH; r += NW) {
      const int a = s_a[r];
      for (int w = lane; w < nwords; w += 32) {
        unsigned bits = s_bits[w];
        int c = s_pre[w];
        while (bits) {
          const int bpos = __ffs(bits) - 1;
          bits &= bits - 1;
          zs[r * ncol + c++] = a >= 0 ? Zp[(int64_t)a * k + w * 32 + bpos] : 0.0;
        }
      }
    }
  }
  __syncthreads();
  double* Dg = D + Doff[g];
  const int fr = lane >> 2, fk = lane & 3;
  constexpr int MTL = RH / 8;
  int arow[MTL];
#pragma unroll
  for (int mt = 0; mt < MTL; ++mt) arow[mt] = s_a[mt * 8 + fr];
  // !STAGED: the group's pieces sorted by tile (Morton: adjacent tiles,
  // overlapping landmark lists), this CTA takes a contiguous 1/ZS of them and
  // its warps consecutive ones -- warps running together read the same Z
  // columns (L1)
  int p_lo = 0, p_hi = np, p_st = pstep, p_first = pq * 8 + wid;
  if (!STAGED) {
    int p2 = 1;
    while (p2 < np) p2 <<= 1;
    for (int e = tid; e < p2; e += 256) {
      s_pk[e] = e < np ? ((long long)(tilerow[Ulist[g * UCAP + Pc[g * UCAP + e].x]] >> 6) << 32) | e
                       : 0x7fffffffffffffffll;
    }
    __syncthreads();
    for (int kk = 2; kk <= p2; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int e = tid; e < p2; e += 256) {
          const int l = e ^ jj;
          if (l > e) {
            const bool up = (e & kk) == 0;
            const long long x = s_pk[e], y = s_pk[l];
            if ((x > y) == up) {
              s_pk[e] = y;
              s_pk[l] = x;
            }
          }
        }
        __syncthreads();
      }
    p_lo = (int)((int64_t)np * pq / ZS);
    p_hi = (int)((int64_t)np * (pq + 1) / ZS);
    p_st = 8;
    p_first = p_lo + wid;
  }
  for (int pi = p_first; pi < p_hi; pi += p_st) {
    const int p = STAGED ? pi : (int)(s_pk[pi] & 0xffffffff);
    const int2 pc = Pc[g * UCAP + p];
    const int u0 = pc.x, nb = pc.y;
    int bid[4], brow[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const int col = n * 8 + fr;
      bid[n] = col < nb ? Ulist[g * UCAP + u0 + col] : -1;
      brow[n] = bid[n] >= 0 ? (tilerow[bid[n]] & 63) : 0;
    }
    const int tile = tilerow[Ulist[g * UCAP + u0]] >> 6;
    const int64_t us = uoff[tile];
    const int nuT = (int)(uoff[tile + 1] - us);
    const int ld = (nuT + 1) & ~1;
    const int* U = ulistp + us;
    const double* At = Ap + aoff[tile];
    double acc[MTL][4][2];
#pragma unroll
    for (int mt = 0; mt < MTL; ++mt)
#pragma unroll
      for (int n = 0; n < 4; ++n) acc[mt][n][0] = acc[mt][n][1] = 0.0;
    const int nn = (nb + 7) / 8;
    for (int c0 = 0; c0 < nuT; c0 += 256) {  // (U_t in chunks of 256 staged columns)
      const int cn = min(256, nuT - c0);
      __syncwarp();
      for (int m = lane; m < cn; m += 32) {
        const int pos = U[c0 + m];
        const unsigned wb = s_bits[pos >> 5];
        s_u[wid][m] = (su_t)(!staged ? pos
                              : ((wb >> (pos & 31)) & 1u) ? s_pre[pos >> 5] + __popc(wb & ((1u << (pos & 31)) - 1u))
                                                          : -1);  // (a zero column for this group)
      }
      __syncwarp();
      // fragments of step k4 + 4 are loaded while step k4's DMMAs run
      double av[MTL], bv[4];
      auto fetch = [&](int k4) {
        const int m = k4 + fk;
        const bool ok = m < cn;
        const int col = ok ? s_u[wid][m] : -1;
#pragma unroll
        for (int mt = 0; mt < MTL; ++mt)
          av[mt] = (col >= 0 && arow[mt] >= 0)
                       ? (staged ? zs[(mt * 8 + fr) * ncol + col] : __ldg(&Zp[(int64_t)arow[mt] * k + col]))
                       : 0.0;
#pragma unroll
        for (int n = 0; n < 4; ++n) bv[n] = (ok && bid[n] >= 0) ? __ldg(&At[(int64_t)brow[n] * ld + c0 + m]) : 0.0;
      };
      fetch(0);
      for (int k4 = 0; k4 < cn; k4 += 4) {
        double ac[MTL], bc[4];
#pragma unroll
        for (int mt = 0; mt < MTL; ++mt) ac[mt] = av[mt];
#pragma unroll
        for (int n = 0; n < 4; ++n) bc[n] = bv[n];
        if (k4 + 4 < cn) fetch(k4 + 4);
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          if (n >= nn) break;
#pragma unroll
          for (int mt = 0; mt < MTL; ++mt) dmma884(acc[mt][n][0], acc[mt][n][1], ac[mt], bc[n]);
        }
      }
    }
    // epilogue: lane holds rows mt*8 + fr, columns n*8 + 2fk + h
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      int bh[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) bh[h] = __shfl_sync(0xffffffffu, bid[n], (2 * fk + h) * 4);
      if (n >= nn) continue;
#pragma unroll
      for (int mt = 0; mt < MTL; ++mt) {
        const int j = mt * 8 + fr;
        const int a = arow[mt];
        if (j >= cnt) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cu = n * 8 + 2 * fk + h;
          const int b = bh[h];
          if (cu < nb && b >= 0) {
            const double kv = a == b ? 1.0 + mu : kern_from_d2(kf, d2_exact_rt(&X2[(int64_t)a * d], &X2[(int64_t)b * d], d), s_tab);
            Dg[(int64_t)(half * ZH + j) * nu + u0 + cu] = kv - acc[mt][n][h];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- factor
// One CTA (FT2 threads) per FSAI row i with pattern J (|J| = wp <= 16 MT,
// ascending, i last).  CTAs take the rows in the spatial (cell) order of the
// union step, so CTAs running together touch the same groups' D blocks (L2).
//   1. S_JJ = K(X_J, X_J) + mu I - D (Gram entries found through the groups'
//      hash tables), lower triangle into shared memory, rows padded to even
//      length (16-byte aligned panel reads), padded to WP rows with identity;
//   2. right-looking blocked Cholesky diag(S_JJ, I) = L L^T with 16-column
//      panels: one warp factors the 16x16 diagonal block with shuffles
//      (rows in lanes), one row per thread for the panel solve, 8x8 DMMA
//      tiles for the trailing update -- with look-ahead: warp 0 updates and
//      factors the next diagonal block while warps 1..3 update the rest;
//   3. g = L^{-T} e_last by column-oriented back substitution over the
//      contiguous rows of L (warp 0; the other warps exit) -- the
//      Kolotilina-Yeremin row with diag(G S G^T) = 1 (reading R16).
constexpr int FT2 = 128;
// 1/sqrt(x): MUFU.RSQ64H seed + two Newton steps (8 instructions instead of
// the ~20 of the library rsqrt, <= 2 ulp; C2 factor 1.76 -> 1.66 ms)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ void dmma884f(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Unblocked Cholesky of a 16x16 block held one row per lane (row lr =
// lane & 15 in dr[0..lr]; lanes 16..31 mirror 0..15), one warp.  Column c is
// broadcast through shared memory (col: 2 x 16 doubles, alternating so one
// __syncwarp per step suffices): L[lr][c2] -= L[lr][c] L[c2][c] with
// L[x][c] = A[x][c] / sqrt(A[c][c]).  myinv = 1 / L_{lr,lr}.  Returns true
// on a non-positive pivot (replaced by 1 so the warp stays in step).
__device__ __forceinline__ bool factor_diag16(double (&dr)[16], double& myinv, int lane, double* col) {
  const int lr = lane & 15;
  bool bad = false;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    double* cb = col + (c & 1) * 16;
    if (lane < 16) cb[lane] = dr[c];
    __syncwarp();
    double piv = cb[c];
    if (!(piv > 0.0)) { bad = true; piv = 1.0; }
    const double inv = rsqrt_nr(piv);
    const double lrc = dr[c] * inv;  // L[lr][c]
    const double f = lrc * inv;      // L[lr][c] L[c2][c] = f A[c2][c]
    if (lr == c) myinv = inv;
#pragma unroll
    for (int c2 = c + 1; c2 < 16; ++c2)
      if (lr >= c2) dr[c2] = fma(-f, cb[c2], dr[c2]);
    dr[c] = (lr == c) ? piv * inv : (lr > c ? lrc : dr[c]);
  }
  return bad;
}

constexpr int FB = 8;  // gather batch: hash probes / D loads in flight per thread (12: C2 1.81 vs 1.76 ms)
// 4 rows per SM: <= 128 registers (5 forces <= 96 -- spills: C2 1.86 vs 1.77 ms)
template <int MT>
__global__ void __launch_bounds__(FT2, 4) fsai_factor_kernel(const int* __restrict__ rorder, int64_t row_lo,
                                                         int64_t row_hi, const int64_t* __restrict__ rp,
                                                         const int32_t* __restrict__ col,
                                                         const int* __restrict__ grp, const int* __restrict__ loc,
                                                         const int* __restrict__ Ucount,
                                                         const int2* __restrict__ Htab,
                                                         const int64_t* __restrict__ Doff,
                                                         const double* __restrict__ D, double* __restrict__ gval,
                                                         int* info, int lsz) {
  constexpr int WP = MT * 16;
  extern __shared__ __align__(16) double fsm[];
  // Lm: packed lower S_JJ / L of the wp real rows (rows padded to even length),
  // then one zero row of 16 (stands for the implicit identity rows wp..WP-1
  // of the 16-column blocking).  lsz = Lm doubles.
  double* Lm = fsm;
  const double* zrow = fsm + lsz - 16;
  __shared__ double s_inv[WP];
  __shared__ __align__(16) double s_dg[16 * 16];  // the current diagonal block of L, dense
  __shared__ __align__(16) double s_col[32];
  __shared__ int sJ[WP];
  __shared__ int s_off[WP + 1];
  __shared__ int s_pos[WP];
  __shared__ int64_t s_db[WP];
  __shared__ int s_bad;
  constexpr int NT8 = (WP / 8) * (WP / 8 + 1) / 2;
  __shared__ short2 s_tile[NT8];  // trailing-update tile t -> (I, J), J <= I (row-wise lower order)
  const int tid = threadIdx.x, lane = tid & 31, lr = lane & 15, wid = tid >> 5;
  for (int I = wid; I < WP / 8; I += FT2 / 32)
    for (int J = lane; J <= I; J += 32) s_tile[I * (I + 1) / 2 + J] = make_short2((short)I, (short)J);
  const int64_t i = rorder[blockIdx.x];
  if (i < row_lo || i >= row_hi) return;  // another rank's row
  const int64_t beg = rp[i];
  const int wp = (int)(rp[i + 1] - beg);
  if (tid == 0) {
    s_bad = 0;
    int o = 0;
    for (int a = 0; a < wp; ++a) {
      s_off[a] = o;
      o += (a + 2) & ~1;  // row a holds a+1 entries, padded to even
    }
    s_off[wp] = o;
  }
  if (tid < 16) fsm[lsz - 16 + tid] = 0.0;
  for (int a = tid; a < wp; a += FT2) sJ[a] = col[beg + a];
  __syncthreads();
  // ---- 1. assemble S_JJ (lower).  Per row p (point a = J_p): the group
  // g(a) and the offset of a's row in D_g; then 8 entries per thread at a
  // time (8 independent hash probes, then 8 independent D loads).
  for (int p = tid; p < wp; p += FT2) {
    const int a = sJ[p];
    const int g = grp[a], la = loc[a];
    s_pos[p] = g * GA + la;
    s_db[p] = Doff[g] + (int64_t)la * Ucount[g];
  }
  __syncthreads();
  {
    // entry e of the packed lower triangle <-> (p, q), q <= p; a thread takes
    // B consecutive entries, (p, q) advanced incrementally: B hash probes,
    // then B D loads (D holds S_ab itself: the group product's epilogue).
    constexpr int B = FB;
    const int ne = wp * (wp + 1) / 2;
    for (int e0 = tid * B; e0 < ne; e0 += FT2 * B) {
      int p0 = (int)((sqrtf(8.0f * (float)e0 + 1.0f) - 1.0f) * 0.5f);
      while (p0 * (p0 + 1) / 2 > e0) --p0;
      while ((p0 + 1) * (p0 + 2) / 2 <= e0) ++p0;
      const int q0 = e0 - p0 * (p0 + 1) / 2;
      int pp[B], bb[B], gg[B];
      unsigned hh[B];
      int2 hv[B];
      {
        int p = p0, q = q0;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          const bool ok = e0 + t < ne;
          // the pair (J_p, J_q) lives in the group of its spatially later
          // point (position g GA + loc: the group is position / GA); the
          // hash key is the earlier point's position
          const int sp = s_pos[ok ? p : 0], sq = s_pos[ok ? q : 0];
          pp[t] = !ok ? 0 : (sp >= sq ? p : q);
          bb[t] = min(sp, sq);
          gg[t] = max(sp, sq) / GA;
          hh[t] = ((unsigned)bb[t] * 2654435761u) & (HC - 1);
          hv[t] = __ldg(&Htab[(int64_t)gg[t] * HC + hh[t]]);
          if (++q > p) { ++p; q = 0; }
        }
      }
      double gram[B];
#pragma unroll
      for (int t = 0; t < B; ++t) {
        const int2* H = Htab + (int64_t)gg[t] * HC;
        int probe = 0;
        while (hv[t].x != bb[t] && probe < HC) {  // b is in U_g by construction
          hh[t] = (hh[t] + 1) & (HC - 1);
          hv[t] = __ldg(&H[hh[t]]);
          ++probe;
        }
        // (never taken; a missing key poisons the row -> NOT_SPD, not a hang)
        gram[t] = hv[t].x == bb[t] ? D[s_db[pp[t]] + hv[t].y] : CUDART_NAN;
      }
      {  // rows are padded to even length: slots from (p, q)
        int p = p0, q = q0;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          if (e0 + t < ne) Lm[s_off[p] + q] = gram[t];
          if (++q > p) { ++p; q = 0; }
        }
      }
    }
  }
  __syncthreads();
  // ---- 2. blocked right-looking Cholesky of diag(S_JJ, I) in 16-column
  // blocks; the identity rows wp..WP-1 are implicit (never stored: their
  // entries left of the diagonal are 0 and stay 0)
  auto rowp = [&](int a, int kb) -> const double* { return a < wp ? Lm + s_off[a] + kb : zrow; };
  // diagonal block at kb (one warp): unblocked, rows in lanes
  auto diag = [&](int kb) {
    double dr[16], myinv = 1.0;
    const bool real = kb + lr < wp;
    const double* row = rowp(kb + lr, kb);
#pragma unroll
    for (int c = 0; c < 16; ++c) dr[c] = (c <= lr) ? (real ? row[c] : (c == lr ? 1.0 : 0.0)) : 0.0;
    const bool bad = factor_diag16(dr, myinv, lane, s_col);
    if (lane < 16) {
      if (kb + lane < wp) {
        double* wrow = Lm + s_off[kb + lane] + kb;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c <= lane) wrow[c] = dr[c];
      }
#pragma unroll
      for (int c = 0; c < 16; c += 2)
        *reinterpret_cast<double2*>(&s_dg[lane * 16 + c]) = make_double2(c <= lane ? dr[c] : 0.0,
                                                                         c + 1 <= lane ? dr[c + 1] : 0.0);
      s_inv[kb + lane] = myinv;
      if (bad) s_bad = 1;
    }
  };
  const int fr = lane >> 2, fk = lane & 3;
  // trailing-update tiles t0 and t1 (t1 < 0: none) of step kb:
  // A[a][b] -= sum_c L[a][kb+c] L[b][kb+c] over an 8x8 tile on the FP64
  // tensor cores (DMMA, 4 k-steps of 4); rows past wp read the zero row
  auto upd2 = [&](int kb, int r0, int t0, int t1) {
    const short2 v0 = s_tile[t0], v1 = s_tile[t1 >= 0 ? t1 : t0];
    const int I0 = v0.x, J0 = v0.y, I1 = v1.x, J1 = v1.y;
    const double* pa0 = rowp(r0 + 8 * I0 + fr, kb) + fk;
    const double* pb0 = rowp(r0 + 8 * J0 + fr, kb) + fk;
    const double* pa1 = rowp(r0 + 8 * I1 + fr, kb) + fk;
    const double* pb1 = rowp(r0 + 8 * J1 + fr, kb) + fk;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      dmma884f(c00, c01, pa0[k4], pb0[k4]);
      dmma884f(c10, c11, pa1[k4], pb1[k4]);
    }
    // (col even, rows start 16-byte aligned: the pair is one 16-byte access)
    auto sub = [&](int row, int col, double v0, double v1) {
      if (row >= wp) return;
      double* q = Lm + s_off[row] + col;
      if (col + 1 <= row) {
        double2 o = *reinterpret_cast<double2*>(q);
        o.x -= v0;
        o.y -= v1;
        *reinterpret_cast<double2*>(q) = o;
      } else if (col <= row) {
        q[0] -= v0;
      }
    };
    sub(r0 + 8 * I0 + fr, r0 + 8 * J0 + 2 * fk, c00, c01);
    if (t1 >= 0) sub(r0 + 8 * I1 + fr, r0 + 8 * J1 + 2 * fk, c10, c11);
  };
  // look-ahead: warp 0 updates the NEXT diagonal block first (tiles 0..2 of
  // the step: I, J < 2) and factors it while warps 1..3 update the rest of
  // the trailing matrix, so the diagonal factor leaves the critical path
  if (wid == 0) diag(0);
  __syncthreads();
#pragma unroll 1
  for (int kb = 0; kb < wp; kb += 16) {
    const int r0 = kb + 16;
    const int m = wp - r0;
    if (m <= 0) break;
    // panel: rows a >= r0, columns kb..kb+15: x L_diag^T = A (one row per
    // thread: wp - 16 < FT2; no loop, so the diagonal block's loads are not
    // hoisted into registers)
#pragma unroll 1
    for (int a = r0 + tid; a < wp; a += FT2) {
      asm volatile("" ::: "memory");  // (keeps the diagonal block's loads inside the loop: no hoisting)
      double x[16];
      double* row = Lm + s_off[a] + kb;
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(row + c);
        x[c] = v.x;
        x[c + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        double sacc = x[c];
#pragma unroll
        for (int c2 = 0; c2 < c; ++c2) sacc = fma(-x[c2], s_dg[c * 16 + c2], sacc);
        x[c] = sacc * s_inv[kb + c];
      }
#pragma unroll
      for (int c = 0; c < 16; c += 2) *reinterpret_cast<double2*>(row + c) = make_double2(x[c], x[c + 1]);
    }
    __syncthreads();
    const int mt8 = (m + 7) >> 3;
    const int nt8 = mt8 * (mt8 + 1) / 2;
    const int nd = nt8 < 3 ? nt8 : 3;  // the next diagonal block's tiles
    if (wid == 0) {
      upd2(kb, r0, 0, nd > 1 ? 1 : -1);
      if (nd > 2) upd2(kb, r0, 2, -1);
      __syncwarp();
      diag(r0);
    } else {
      constexpr int NW = FT2 / 32 - 1;
      for (int t0 = 3 + (wid - 1); t0 < nt8; t0 += 2 * NW) upd2(kb, r0, t0, t0 + NW < nt8 ? t0 + NW : -1);
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) atomicCAS(info, 0, (int)(i + 1));
    return;
  }
  // ---- 3. g = L^{-T} e_last: rhs_j -= L[t][j] g_t over the rows t, one
  // warp (shuffles in warp-uniform code); the others leave, freeing their
  // issue slots for the SM's other rows
  if (wid != 0) return;
  double rhs[WP / 32 + 1];
#pragma unroll
  for (int r = 0; r <= WP / 32; ++r) rhs[r] = (lane + 32 * r == wp - 1) ? 1.0 : 0.0;
  for (int t = wp - 1; t >= 0; --t) {
    const int rt = t >> 5;
    double v = 0.0;
#pragma unroll
    for (int r = 0; r <= WP / 32; ++r)
      if (r == rt) v = rhs[r];
    const double gt = __shfl_sync(0xffffffffu, v, t & 31) * s_inv[t];
    if (tid == 0) gval[beg + t] = gt;
    const double* lrw = Lm + s_off[t];
#pragma unroll
    for (int r = 0; r <= WP / 32; ++r) {
      const int j = lane + 32 * r;
      if (j < t) rhs[r] = fma(-lrw[j], gt, rhs[r]);
    }
  }
}

template <int MT>
afn_status launch_factor(const int* rorder, int64_t N, int64_t row_lo, int64_t row_hi, int wcap, cudaStream_t st,
                         const int64_t* rp, const int32_t* col, const int* grp, const int* loc, const int* Ucount,
                         const int2* Htab, const int64_t* Doff, const double* D, double* gval, int* info) {
  constexpr int WP = MT * 16;
  const int wmax = std::min(WP, wcap);
  const int lsz = ((wmax * (wmax + 1) / 2 + (wmax + 1) / 2 + 16) + 1) & ~1;
  const size_t bytes = sizeof(double) * (size_t)lsz;
  auto kern = fsai_factor_kernel<MT>;
  AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  for (int64_t r0 = 0; r0 < N; r0 += 1 << 30) {
    const int64_t nr = std::min<int64_t>(N - r0, 1 << 30);
    kern<<<(unsigned)nr, FT2, bytes, st>>>(rorder + r0, row_lo, row_hi, rp, col, grp, loc, Ucount, Htab, Doff, D,
                                          gval, info, lsz);
    AFN_LAUNCH_CHECK("fsai_factor_kernel");
  }
  return AFN_OK;
}

}  // namespace

afn_status fsai_sddmm_run(const double* X2, int64_t N, int d, Kern kn, double mu, const double* W,
                          int64_t k, const int64_t* rp, const int32_t* col, const int64_t* trp,
                          const int32_t* tcol, int64_t row_lo, int64_t row_hi, double* gval, int* d_info,
                          cudaStream_t st, cudaStream_t pst, const FsaiZ* z) {
  if (N <= 0 || row_hi <= row_lo) return AFN_OK;
  // steps 1-2 (spatial order, unions, pass offsets; they need only the
  // pattern) run on pst -- concurrently with W on st when pst != st; the
  // products and the factor run on st after pst's work
  const cudaStream_t mst = st;
  if (pst == nullptr) pst = st;
  st = pst;
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
  } fr{&tmp, mst};  // (freed in the main stream's order, after the products and the factor)
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
  if (MT < 1 || MT > 8) {  // (rows wider than 128: the per-row path, fsai.cu)
    set_error("fsai_sddmm: row width %d", w);
    return AFN_ERR_STATE;
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
    // raster-ordered tiles.  (Z-ordered tiles measured C3 factor 14.9 vs 15.3
    // ms and group-product DRAM 143 vs 155 GB, but at C5 some groups' unions
    // -- the Z-order predecessors of hub points of the early, wide pattern rows
    // -- exceed UCAP and the build falls back to the per-row Grams: 12.0 vs
    // 6.8 s per solve)
    cg.morton = 0;
    if (cg.morton) {  // key space: (next power of two of the largest tile count)^dd tiles
      int nbm = 1;
      for (int c = 0; c < dd; ++c) nbm = std::max(nbm, cg.nb[c]);
      int64_t p2 = 1;
      while (p2 < nbm) p2 <<= 1;
      int64_t tiles = 1;
      for (int c = 0; c < dd; ++c) tiles *= p2;
      // (Morton interleaves 3 axes: with dd < 3 the unused axes are 0 and the
      // codes of the used ones still fit below p2^dd only for dd = 3)
      if (dd < 3) tiles = (int64_t)1 << (3 * (int64_t)std::ceil(std::log2((double)p2)));
      cg.ncell = tiles * cg.t[0] * cg.t[1] * cg.t[2];
    }
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
  group_maps_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(sorder, N, GA, grp, loc);
  AFN_LAUNCH_CHECK("group_maps_kernel");
  // the pattern rows as ascending spatial positions (the unions' scan stops at
  // the first position past the point's own)
  int32_t* colp;
  const int64_t nnz = N > 1 ? h2[1] : 1;
  if ((s = get((void**)&colp, sizeof(int32_t) * (size_t)std::max<int64_t>(1, nnz))) != AFN_OK) return s;
  pattern_positions_kernel<<<(unsigned)((N * 32 + 255) / 256), 256, 0, st>>>(rp, col, grp, loc, GA, N, colp);
  AFN_LAUNCH_CHECK("pattern_positions_kernel");
  // ---- 2. unions
  const int64_t G = (N + GA - 1) / GA;
  int *Ucount, *Ulist, *ovf;
  int64_t* Doff;
  if ((s = get((void**)&Ucount, sizeof(int) * G)) != AFN_OK) return s;
  if ((s = get((void**)&Ulist, sizeof(int) * G * UCAP)) != AFN_OK) return s;
  int2* Htab;
  if ((s = get((void**)&Htab, sizeof(int2) * G * HC)) != AFN_OK) return s;
  if ((s = get((void**)&ovf, sizeof(int) * 2)) != AFN_OK) return s;
  if ((s = get((void**)&Doff, sizeof(int64_t) * (G + 1))) != AFN_OK) return s;
  AFN_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int) * 2, st));
  int2* Pc = nullptr;
  int* Pcount = nullptr;
  unsigned long long* zwork = nullptr;
  if (z) {
    if ((s = get((void**)&Pc, sizeof(int2) * G * UCAP)) != AFN_OK) return s;
    if ((s = get((void**)&Pcount, sizeof(int) * G)) != AFN_OK) return s;
    if ((s = get((void**)&zwork, sizeof(unsigned long long))) != AFN_OK) return s;
    AFN_CUDA(cudaMemsetAsync(zwork, 0, sizeof(unsigned long long), st));
  }
  {
    const int bytes = (int)(sizeof(int) * HC);
    AFN_CUDA(cudaFuncSetAttribute(group_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    group_union_kernel<<<(unsigned)G, 256, bytes, st>>>(sorder, N, rp, colp, trp, tcol, row_lo, row_hi, GA, Ucount,
                                                         Ulist, Htab, ovf);
    AFN_LAUNCH_CHECK("group_union_kernel");
    if (z) {  // (Z mode: the unions renumbered by tile, the pieces listed)
      const int rbytes = (int)(sizeof(int) * 2 * TH);
      AFN_CUDA(cudaFuncSetAttribute(group_tile_renumber_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rbytes));
      group_tile_renumber_kernel<<<(unsigned)G, 256, rbytes, st>>>(sorder, Ucount, Ulist, Htab, z->tilerow, z->uoff, Pc,
                                                                    Pcount, zwork, ovf);
      AFN_LAUNCH_CHECK("group_tile_renumber_kernel");
    }
  }
  int hov = 0;
  unsigned long long hzw = 0ull;
  AFN_CUDA(cudaMemcpyAsync(&hov, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (z) AFN_CUDA(cudaMemcpyAsync(&hzw, zwork, sizeof(hzw), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  if (hov) {
    set_error("fsai_sddmm: pair union exceeds %d in a group", UCAP);
    return AFN_ERR_STATE;
  }
  scan_i64_kernel<<<1, 1024, 0, st>>>(Ucount, G, GA, Doff);
  AFN_LAUNCH_CHECK("scan_i64_kernel");
  int* pc;
  int64_t* Poff;
  if ((s = get((void**)&pc, sizeof(int) * G)) != AFN_OK) return s;
  if ((s = get((void**)&Poff, sizeof(int64_t) * (G + 1))) != AFN_OK) return s;
  // columns of U per GEMM work item: 8 warps x 8 NTL
  const int ut = 64 * G16_NTL;
  pass_count_kernel<<<(unsigned)((G + 255) / 256), 256, 0, st>>>(Ucount, G, ut, pc);
  AFN_LAUNCH_CHECK("pass_count_kernel");
  scan_i64_kernel<<<1, 1024, 0, st>>>(pc, G, 1, Poff);
  AFN_LAUNCH_CHECK("scan_i64_kernel");
  int64_t totD = 0, items = 0;
  AFN_CUDA(cudaMemcpyAsync(&items, Poff + G, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaMemcpyAsync(&totD, Doff + G, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  // ---- 3. dense group products
  const KernelFn kf = kernel_fn(kn.kind, kn.l);
  double* D;  // S_ab entries (the product's epilogue forms K_ab + mu delta_ab - W_a . W_b)
  if ((s = get((void**)&D, sizeof(double) * (totD > 0 ? totD : 1))) != AFN_OK) return s;
  if (pst != mst) {  // join: the main stream continues after the preparation
    cudaEvent_t ej;
    AFN_CUDA(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    AFN_CUDA(cudaEventRecord(ej, pst));
    AFN_CUDA(cudaStreamWaitEvent(mst, ej, 0));
    cudaEventDestroy(ej);
  }
  st = mst;
  if (z) {
    kt_begin(KT_FSAI_GEMM, st);
    // staged when the group's landmark columns fit: sparse landmarks (k / N,
    // landmarks per unit volume, small: C5 8000 / 2^20); C3 (4000 / 2^17)
    // unions of ~1300-2500 columns mostly do not
    if (z->staged) {
      const int zb = (int)(sizeof(double) * ZH * ZCAP);
      AFN_CUDA(cudaFuncSetAttribute(group_zk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, zb));
      group_zk_kernel<true><<<(unsigned)(2 * G), 512, zb, st>>>(sorder, N, z->Zp, k, z->tilerow, z->uoff, z->ulistp,
                                                                z->aoff, z->Ap, Ucount, Ulist, Doff, Pc, Pcount, D, X2,
                                                                d, kf, mu);
    } else {
      group_zk_kernel<false><<<(unsigned)(ZS * G), 256, 0, st>>>(sorder, N, z->Zp, k, z->tilerow, z->uoff, z->ulistp,
                                                                 z->aoff, z->Ap, Ucount, Ulist, Doff, Pc, Pcount, D,
                                                                 X2, d, kf, mu);
    }
    AFN_LAUNCH_CHECK("group_zk_kernel");
    kt_end(KT_FSAI_GEMM, st, 2.0 * (double)hzw);
  } else {
    kt_begin(KT_FSAI_GEMM, st);
    if (items > 0) {
      const bool wide = (double)N * (double)k * sizeof(double) > 512e6;  // W a few L2s or more
      const int dkc = wide ? 16 : 8;
      const int bytes = (int)(sizeof(double) * DNS * (dkc + 4) * (GA + ut));
      auto kern = wide ? group_gemm_dmma_kernel<16> : group_gemm_dmma_kernel<8>;
      AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      int occ = 0;
      AFN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, bytes));
      // persistent rounds of P consecutive items when W is several L2s (C3:
      // 59.8 -> 56.4 ms), one item per CTA below (C2: 2.61 vs 2.82 ms)
      const int64_t P = wide ? std::min<int64_t>(items, (int64_t)std::max(1, occ) * num_sms()) : items;
      kern<<<(unsigned)P, 256, bytes, st>>>(sorder, N, W, k, Ucount, Ulist, Doff, Poff, G, D, X2, d, kf, mu, items);
      AFN_LAUNCH_CHECK("group_gemm_dmma_kernel");
    }
    kt_end(KT_FSAI_GEMM, st, 2.0 * (double)k * (double)totD);
  }
  // ---- 4. per-row assembly + Cholesky + g (one CTA per row, rows in the
  // spatial order sorder; CTAs of other ranks' rows exit at once)
  const int64_t NR = row_hi - row_lo;
  kt_begin(KT_FSAI_CHOL, st);
  switch (MT) {
#define AFN_FACTOR(M) \
    case M: s = launch_factor<M>(sorder, N, row_lo, row_hi, w, st, rp, col, grp, loc, Ucount, Htab, Doff, D, gval, d_info); break;
    AFN_FACTOR(1) AFN_FACTOR(2) AFN_FACTOR(3) AFN_FACTOR(4) AFN_FACTOR(5) AFN_FACTOR(6) AFN_FACTOR(7)
    default: s = launch_factor<8>(sorder, N, row_lo, row_hi, w, st, rp, col, grp, loc, Ucount, Htab, Doff, D, gval, d_info); break;
#undef AFN_FACTOR
  }
  if (s != AFN_OK) return s;
  kt_end(KT_FSAI_CHOL, st, (double)NR * ((double)w * w * w / 3.0 + (double)w * w));
  return AFN_OK;
}

}  // namespace afn

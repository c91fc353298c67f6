// ozaki.cu -- W = K21 L^{-T} (the Nystrom factor of AFN) in FP64
// accuracy on the 5th-generation INT8 tensor cores (tcgen05.mma kind::i8,
// accumulators in TMEM), by exact integer slicing (the Ozaki splitting).
//
// Each row r of A = K21 is scaled by 2^-ea_r (2^ea_r >= max_t |A_rt|) and
// split into S = 8 signed 7-bit slices, x = sum_s a_s 2^(-6-7s), |a_s| <= 64,
// exactly in FP64 (v <- 64 x; a_s = rint(v); v <- 128 (v - a_s)); each row c
// of B^T = L^{-1} likewise (2^eb_c, slices b_s).  Then
//   W_rc = 2^(ea_r + eb_c - 12) sum_{D=0}^{S-1} 2^(-7D) C_D[r][c],
//   C_D = sum_{i+j=D} A_i B_j^T   (int8 x int8 -> int32, exact: |C_D| <=
//   8 * 64 * 64 * k < 2^31 for k < 65536),
// the pairs with i + j >= S dropped (their weight is below 2^-56 of
// max|A_r| max|B_c| per term): W to within a few units of 2^-56 of
// sum_t |A_rt||B_ct| -- the size of FP64 GEMM rounding.  36 INT8 products at
// ~4 POPS replace one FP64 DMMA product at 37 TFLOP/s.
//
// GEMM kernel: a cluster of two CTAs (tcgen05 cta_group::2) per 256 x 64 tile
// of W (rows x columns, the K range cut at the tile's last column: L^{-1} is
// lower triangular); each CTA holds its 128 rows' 8 accumulators C_0..C_7 in
// its 512 TMEM columns (64 each).  K advances in 32-byte blocks through five
// shared-memory stages: per CTA its 128 rows of the 8 A slices and half (32
// rows) of the 8 B slices, 40 KB, filled by the TMA (3-D tensor maps over the
// slice arrays, boxes of 16 bytes x 128 / 32 rows = one column of core
// matrices of the K-major no-swizzle layout), both CTAs' loads completing on
// CTA 0's "full" mbarrier; one thread of CTA 0 issues a stage's 36 m256 n64
// k32 MMAs and commits them to both CTAs' "empty" mbarriers; epilogue:
// tcgen05.ld of the 8 accumulators, Horner in FP64, the 2^(ea + eb - 12)
// scale, FP64 stores.
//
// Measured (C3, k = 4000, whole W step incl. the slicing): 48.7 ms per build
// against 66.6 ms for the DMMA GEMM (one-CTA 128 x 64 tiles, TMA: 55.8;
// cp.async-fed: 59.7; 2 stages of 64 bytes: 70.4; a two-pass 128 x 128
// variant with 4 accumulators: 69.5).  Operand traffic bounds it: an m128 n64
// k32 MMA reads 6 KB for 0.5 M ops (alone, operands resident, the shape peaks
// at 2.75 POPS in tools/micro/tc_i8_probe.cu; N = 256 reaches 4.1 POPS, but 8
// accumulators of 256 columns exceed the 512 TMEM columns); the pair halves
// the B traffic per CTA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "afn_common.cuh"
#include "afn_internal.h"
#include "tc05.cuh"

namespace afn {

namespace {

constexpr int OZ_S = 8;         // slices per operand
constexpr int OZ_TM = 128;      // tile rows per CTA (W rows; the pair MMA has M = 256)
constexpr int OZ_TN = 64;       // tile columns (W columns, MMA N)
constexpr int OZ_KB = 32;       // K bytes per stage (one MMA k-step)

constexpr int OZ_NT = 128;      // threads
constexpr int OZ_A_SL = OZ_TM * OZ_KB;            // bytes of one A slice tile per stage (4 KB)

using namespace tc;

// split |x| <= 1 into OZ_S signed 7-bit slices (exact)
__device__ __forceinline__ void split8(double x, int8_t* out, int64_t stride) {
  double v = x * 64.0;
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const double a = rint(v);
    out[(int64_t)s * stride] = (int8_t)(int)a;
    v = (v - a) * 128.0;
  }
}

// A slices of K21 rows: one warp per row r (< nr: the kernel values of
// X_r against the k landmarks; rows nr..nrp-1 and columns k..kp-1 zero).
// Pass 1: the row max -> ea_r; pass 2: values / 2^ea_r -> slices.
__global__ void __launch_bounds__(256) k21_slices_kernel(const double* __restrict__ X1, int64_t k, int64_t kp,
                                                         const double* __restrict__ Xr, int64_t nr, int64_t nrp,
                                                         int d, KernelFn kf, int8_t* __restrict__ sl,
                                                         int* __restrict__ ea) {
  __shared__ double s_tab[AFN_EXP2_TAB_N];
  load_exp2_tab(s_tab);
  __syncthreads();
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrp) return;
  const int64_t stride = nrp * kp;  // bytes between slices
  int8_t* row = sl + r * kp;
  if (r >= nr) {
    for (int64_t t = lane; t < kp; t += 32)
      for (int s = 0; s < OZ_S; ++s) row[(int64_t)s * stride + t] = 0;
    if (lane == 0) ea[r] = 0;
    return;
  }
  double xr[16];
  for (int c = 0; c < d; ++c) xr[c] = Xr[r * d + c];
  // the row max: both kernels decrease with the distance, so it is the
  // value at the nearest landmark (a distance pass, one kernel evaluation)
  double md2 = CUDART_INF;
  for (int64_t t = lane; t < k; t += 32) md2 = fmin(md2, d2_exact_rt(xr, &X1[t * d], d));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) md2 = fmin(md2, __shfl_xor_sync(0xffffffffu, md2, o));
  const double mx = kern_from_d2(kf, md2, s_tab);
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
  const double sc = ldexp(1.0, -e);
  for (int64_t t = lane; t < kp; t += 32) {
    const double v = t < k ? kern_from_d2(kf, d2_exact_rt(xr, &X1[t * d], d), s_tab) * sc : 0.0;
    split8(v, row + t, stride);
  }
  if (lane == 0) ea[r] = e;
}

// B slices of the rows of a dense row-major matrix M (n x k, row stride ldm):
// one warp per row c (< n; rows n..np-1 and columns k..kp-1 zero)
__global__ void __launch_bounds__(256) rows_slices_kernel(const double* __restrict__ Mx, int64_t n, int64_t np,
                                                          int64_t k, int64_t kp, int64_t ldm,
                                                          int8_t* __restrict__ sl, int* __restrict__ eb) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= np) return;
  const int64_t stride = np * kp;
  int8_t* row = sl + c * kp;
  double mx = 0.0;
  if (c < n)
    for (int64_t t = lane; t < k; t += 32) mx = fmax(mx, fabs(Mx[c * ldm + t]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);
  const double sc = ldexp(1.0, -e);
  for (int64_t t = lane; t < kp; t += 32) {
    const double v = (c < n && t < k) ? Mx[c * ldm + t] * sc : 0.0;
    split8(v, row + t, stride);
  }
  if (lane == 0) eb[c] = e;
}

// Pair variant (cta_group::2): a cluster of two CTAs (vertically adjacent
// row tiles) computes a 256 x 64 tile with m256 MMAs issued by CTA 0: each
// CTA loads its own 128 A rows and half of the 64 B rows (the pair's tensor
// cores read both halves), so a CTA stages 40 KB instead of 48 KB per 32-byte
// K block.  Both CTAs' TMA loads complete on CTA 0's "full" mbarrier (peer
// bit cleared in the address); CTA 0's commits arrive on both CTAs' "empty"
// and "done" mbarriers (multicast); each CTA reads its own 128 TMEM lanes in
// the epilogue.
constexpr int OZ2_BH = OZ_TN / 2;                       // B rows per CTA
constexpr int OZ2_B_SL = OZ2_BH * OZ_KB;                // 1 KB
constexpr int OZ2_STAGE = OZ_S * (OZ_A_SL + OZ2_B_SL);  // 40 KB
constexpr int OZ2_NS = 5;
constexpr int OZ2_SMEM = OZ2_NS * OZ2_STAGE + 1024;
__global__ void __launch_bounds__(OZ_NT, 1) w_ozaki_2sm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                               const __grid_constant__ CUtensorMap tmB,
                                                               const int* __restrict__ ea, int64_t nr,
                                                               const int* __restrict__ eb, int64_t k,
                                                               double* __restrict__ W, int64_t ldw) {
  extern __shared__ uint8_t oz_raw[];
  __shared__ __align__(8) uint64_t full[OZ2_NS], empty[OZ2_NS], done;
  __shared__ uint32_t tmem_base;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int r0 = (int)(blockIdx.x * OZ_TM), c0 = (int)(blockIdx.y * OZ_TN);  // (pairs along x)
  const int64_t kend = min(k, (int64_t)c0 + OZ_TN);
  const int nkb = (int)((kend + OZ_KB - 1) / OZ_KB);
  if (tid == 0) {
    for (int b = 0; b < OZ2_NS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1);
    }
    mbar_init(&done, 1);
    mbar_init_fence();
  }
  // TMEM: both CTAs' warp 0 allocate the pair's columns (same slot offset)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // both CTAs' barriers initialised and TMEM allocated before any cross-CTA use
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  constexpr int UN = OZ_KB / 16;
  if (warp == 0 && lane == 0) {  // producer (each CTA: its A rows, its half of B)
    for (int kb = 0; kb < nkb; ++kb) {
      const int b = kb % OZ2_NS;
      if (kb >= OZ2_NS) mbar_wait(&empty[b], (uint32_t)(((kb / OZ2_NS) - 1) & 1));
      if (crank == 0) mbar_expect(&full[b], 2u * (uint32_t)OZ2_STAGE);
      const uint32_t base = smem_u32(sm + (size_t)b * OZ2_STAGE);
      const uint32_t fb = smem_u32(&full[b]) & 0xFEFFFFFFu;  // CTA 0's barrier
      const int kx = kb * OZ_KB;
#pragma unroll
      for (int sl = 0; sl < OZ_S; ++sl)
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(base + sl * OZ_A_SL + u * (OZ_TM / 8) * 128),
              "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(kx + u * 16), "r"(r0), "r"(sl), "r"(fb)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(base + OZ_S * OZ_A_SL + sl * OZ2_B_SL +
                                                         u * (OZ2_BH / 8) * 128),
              "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(kx + u * 16), "r"(c0 + OZ2_BH * (int)crank), "r"(sl),
              "r"(fb)
              : "memory");
        }
    }
  } else if (warp == 1 && lane == 0 && crank == 0) {  // MMA issuer (CTA 0)
    constexpr uint32_t LBO_A = (OZ_TM / 8) * 128, LBO_B = (OZ2_BH / 8) * 128;
    constexpr uint32_t idesc = idesc_i8(2 * OZ_TM, OZ_TN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int b = kb % OZ2_NS;
      mbar_wait(&full[b], (uint32_t)((kb / OZ2_NS) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_u32(sm + (size_t)b * OZ2_STAGE), bbase = abase + OZ_S * OZ_A_SL;
#pragma unroll
      for (int D = 0; D < OZ_S; ++D) {
#pragma unroll
        for (int i = 0; i <= D; ++i) {
          const uint64_t da = umma_desc(abase + i * OZ_A_SL, LBO_A, 128);
          const uint64_t db = umma_desc(bbase + (D - i) * OZ2_B_SL, LBO_B, 128);
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}\n" ::
                  "r"(tmem + (uint32_t)(D * OZ_TN)),
              "l"(da), "l"(db), "r"(idesc), "r"((kb > 0 || i > 0) ? 1u : 0u), "r"(0), "r"(0), "r"(0), "r"(0),
              "r"(0), "r"(0), "r"(0), "r"(0));
        }
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&empty[b])),
          "h"((uint16_t)3)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&done)),
        "h"((uint16_t)3)
        : "memory");
  }
  __syncwarp();
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int64_t r = r0 + warp * 32 + lane;
  const bool rok = r < nr;
  const int er = rok ? ea[r] : 0;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
#pragma unroll 1
  for (int cc = 0; cc < OZ_TN; cc += 8) {
    uint32_t v[OZ_S][8];
#pragma unroll
    for (int D = 0; D < OZ_S; ++D) tmem_ld8(tmem + lane_base + (uint32_t)(D * OZ_TN + cc), v[D]);
    tmem_ld_wait();
    if (rok) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t c = c0 + cc + j;
        if (c >= k) break;
        double acc = (double)(int32_t)v[OZ_S - 1][j];
#pragma unroll
        for (int D = OZ_S - 2; D >= 0; --D) acc = fma(acc, 0x1.0p-7, (double)(int32_t)v[D][j]);
        W[r * ldw + c] = ldexp(acc, er + eb[c] - 12);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // neither CTA frees the pair's TMEM before both finished reading
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// 3-D tensor map over OZ_S slices of rows x cols int8 (row-major), box
// 16 bytes x box_rows x 1 (no swizzle, no interleave)
PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  });
  return fn;
}
afn_status slice_map(CUtensorMap* m, const int8_t* base, int64_t rows, int64_t cols, int box_rows) {
  PFN_cuTensorMapEncodeTiled fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return AFN_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)OZ_S};
  const cuuint64_t strides[2] = {(cuuint64_t)cols, (cuuint64_t)(rows * cols)};
  const cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return AFN_ERR_CUDA;
  }
  return AFN_OK;
}

}  // namespace

// W (N x k, row stride k) = K(Xr, X1) L^{-T} with Linv = L^{-1} (k x k,
// row-major, lower triangular).  K21 is generated and sliced in row blocks.
afn_status w_gemm_ozaki(const double* Linv, int64_t k, const double* X1, const double* Xr, int64_t N, int d, Kern kn,
                        double* W, cudaStream_t st) {
  if (N <= 0 || k <= 0) return AFN_OK;
  if (k >= 65536 || d > 16) {
    set_error("w_gemm_ozaki: k = %lld, d = %d out of range", (long long)k, d);
    return AFN_ERR_ARG;
  }
  const KernelFn kf = kernel_fn(kn.kind, kn.l);
  const int64_t kp = (k + OZ_KB - 1) / OZ_KB * OZ_KB;
  const int64_t kcp = (k + OZ_TN - 1) / OZ_TN * OZ_TN;
  // row blocks: the A slices of one block <= ~1 GiB
  // (row tiles in pairs: blocks and padding in multiples of 256 rows)
  const int64_t rb = std::max<int64_t>(2 * OZ_TM, ((1ll << 30) / (OZ_S * kp)) / (2 * OZ_TM) * (2 * OZ_TM));
  const int64_t nblk_rows = std::min<int64_t>(rb, (N + 2 * OZ_TM - 1) / (2 * OZ_TM) * (2 * OZ_TM));
  int8_t *Asl = nullptr, *Bsl = nullptr;
  int *ea = nullptr, *eb = nullptr;
  afn_status s;
  if ((s = dalloc((void**)&Bsl, (size_t)OZ_S * kcp * kp, st)) != AFN_OK) return s;
  struct Fr {
    void* p[4];
    cudaStream_t st;
    ~Fr() {
      for (void* q : p)
        if (q) dfree(q, st);
    }
  } fr{{Bsl, nullptr, nullptr, nullptr}, st};
  if ((s = dalloc((void**)&eb, sizeof(int) * kcp, st)) != AFN_OK) return s;
  fr.p[1] = eb;
  if ((s = dalloc((void**)&Asl, (size_t)OZ_S * nblk_rows * kp, st)) != AFN_OK) return s;
  fr.p[2] = Asl;
  if ((s = dalloc((void**)&ea, sizeof(int) * nblk_rows, st)) != AFN_OK) return s;
  fr.p[3] = ea;
  rows_slices_kernel<<<(unsigned)((kcp * 32 + 255) / 256), 256, 0, st>>>(Linv, k, kcp, k, kp, k, Bsl, eb);
  AFN_LAUNCH_CHECK("rows_slices_kernel");
  static bool attr = false;
  if (!attr) {
    AFN_CUDA(cudaFuncSetAttribute(w_ozaki_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ2_SMEM));
    attr = true;
  }
  CUtensorMap tmB;
  if ((s = slice_map(&tmB, Bsl, kcp, kp, OZ2_BH)) != AFN_OK) return s;
  for (int64_t q0 = 0; q0 < N; q0 += rb) {
    const int64_t nr = std::min(rb, N - q0);
    const int64_t nrp = (nr + 2 * OZ_TM - 1) / (2 * OZ_TM) * (2 * OZ_TM);
    k21_slices_kernel<<<(unsigned)((nrp * 32 + 255) / 256), 256, 0, st>>>(X1, k, kp, Xr + q0 * d, nr, nrp, d, kf,
                                                                          Asl, ea);
    AFN_LAUNCH_CHECK("k21_slices_kernel");
    CUtensorMap tmA;
    if ((s = slice_map(&tmA, Asl, nrp, kp, OZ_TM)) != AFN_OK) return s;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nrp / OZ_TM), (unsigned)(kcp / OZ_TN));  // row tiles along x: pairs (2i, 2i + 1)
    cfg.blockDim = dim3(OZ_NT);
    cfg.dynamicSmemBytes = OZ2_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    AFN_CUDA(cudaLaunchKernelEx(&cfg, w_ozaki_2sm_kernel, tmA, tmB, (const int*)ea, nr, (const int*)eb, k, W + q0 * k,
                                (int64_t)k));
    AFN_LAUNCH_CHECK("w_ozaki_2sm_kernel");
  }
  return AFN_OK;
}

}  // namespace afn

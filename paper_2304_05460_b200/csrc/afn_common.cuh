// afn_common.cuh -- shared device helpers of the sm_100a AFN path.
// (Product code.  Shares nothing with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/afn.h"

namespace afn {

// ---------------------------------------------------------------------------
// Launch accounting (bench.py reports how many of our kernels ran).
void note_launch(int count = 1);

// ---------------------------------------------------------------------------
// Bit-exact squared distance (readings R3): c = 0..d-1 in order, each
// subtract / multiply / add individually rounded -- no FMA contraction.
template <int D>
__device__ __forceinline__ double d2_exact(const double* a, const double* b) {
  double s = __dmul_rn(__dsub_rn(a[0], b[0]), __dsub_rn(a[0], b[0]));
#pragma unroll
  for (int c = 1; c < D; ++c) {
    double t = __dsub_rn(a[c], b[c]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

__device__ __forceinline__ double d2_exact_rt(const double* a, const double* b, int d) {
  double t0 = __dsub_rn(a[0], b[0]);
  double s = __dmul_rn(t0, t0);
  for (int c = 1; c < d; ++c) {
    double t = __dsub_rn(a[c], b[c]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// ---------------------------------------------------------------------------
// 2^y for y <= 0 (the Gaussian kernel exp(-d^2/l^2) = 2^(-d^2 log2(e)/l^2)).
// Reduction y = n + j/256 + f, |f| <= 1/512, j = 16 j1 + j0:
// 2^(j/256) = 2^(j1/16) * 2^(j0/256) from two 16-entry tables (correctly
// rounded, in shared memory: 16 doubles -> one bank pair per entry, so the
// warp's random look-ups are conflict-free); 2^f = e^(f ln2) by its degree-4
// Taylor polynomial (truncation < 4e-17 relative).  2^n is applied by an
// integer add to the exponent field.  y < -1020 (values < 2^-1020 ~ 9e-308)
// returns +0.  FP64-pipe cost: 1 DFMA (scale + round) + 1 DADD + 1 DFMA (f)
// + 4 DFMA (polynomial) + 2 DMUL (tables) = 9 instructions.
// ---------------------------------------------------------------------------
#define AFN_EXP2_TAB_N 32
static __device__ __constant__ double c_exp2_tab[AFN_EXP2_TAB_N] = {
   0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
   0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
   0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
   0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0,
   0x1.0000000000000p+0, 0x1.00b1afa5abcbfp+0, 0x1.0163da9fb3335p+0, 0x1.02168143b0281p+0,
   0x1.02c9a3e778061p+0, 0x1.037d42e11bbccp+0, 0x1.04315e86e7f85p+0, 0x1.04e5f72f654b1p+0,
   0x1.059b0d3158574p+0, 0x1.0650a0e3c1f89p+0, 0x1.0706b29ddf6dep+0, 0x1.07bd42b72a836p+0,
   0x1.0874518759bc8p+0, 0x1.092bdf66607e0p+0, 0x1.09e3ecac6f383p+0, 0x1.0a9c79b1f3919p+0,
};

// copy the tables into shared memory (call by all threads, then __syncthreads)
__device__ __forceinline__ void load_exp2_tab(double* s_tab) {
  for (int t = threadIdx.x; t < AFN_EXP2_TAB_N; t += blockDim.x) s_tab[t] = c_exp2_tab[t];
}

// ln(2)^k / k!, k = 0..4
#define AFN_E2C0 0x1.0000000000000p+0
#define AFN_E2C1 0x1.62e42fefa39efp-1
#define AFN_E2C2 0x1.ebfbdff82c58fp-3
#define AFN_E2C3 0x1.c6b08d704a0c0p-5
#define AFN_E2C4 0x1.3b2ab6fba4e77p-7
#define AFN_LOG2E 0x1.71547652b82fep+0
#define AFN_SQRT_LOG2E 0x1.337cc2183b050p+0

// s = -y >= 0 (pass the positive exponent). tab: the 2 x 16-entry tables (smem).
__device__ __forceinline__ double exp2_neg(double s, const double* tab) {
  const double magic = 0x1.8p52;
  double t = fma(s, -256.0, magic);         // rint(-256 s) in the low word
  double nf = t - magic;                    // = rint(-256 s) as a double
  double f = fma(nf, -0x1.0p-8, -s);        // -s - nf/256, exact, |f| <= 1/512
  int n256 = __double2loint(t);
  double p = AFN_E2C4;
  p = fma(p, f, AFN_E2C3);
  p = fma(p, f, AFN_E2C2);
  p = fma(p, f, AFN_E2C1);
  p = fma(p, f, AFN_E2C0);
  p = (p * tab[(n256 >> 4) & 15]) * tab[16 + (n256 & 15)];
  int hi = __double2hiint(p) + ((n256 >> 8) << 20);
  // s >= 1020 (hi word of 1020.0 is 0x408FE000) -> clear the high word only:
  // the result is +0 or a denormal below 2^-1042 (absolute error < 1e-313);
  // also covers huge s / inf.  One select instead of two.
  hi = (__double2hiint(s) >= 0x408FE000) ? 0 : hi;
  return __hiloint2double(hi, __double2loint(p));
}

#define AFN_SQRT3 0x1.bb67ae8584caap+0

// Kernel entry from a squared distance d2 = ||x - y||^2:
//   kind 0, Gaussian      exp(-d2 / l^2)                     c = log2(e) / l^2
//   kind 1, Matern-3/2    (1 + t) exp(-t),  t = sqrt(3 d2)/l  c = sqrt(3) / l
struct KernelFn {
  int kind;
  double c;
};
__host__ __device__ inline KernelFn kernel_fn(int kind, double l) {
  return kind == 1 ? KernelFn{1, AFN_SQRT3 / l} : KernelFn{0, AFN_LOG2E / (l * l)};
}
__device__ __forceinline__ double kern_from_d2(KernelFn f, double d2, const double* tab) {
  if (f.kind == 1) {
    const double t = sqrt(d2) * f.c;
    return (1.0 + t) * exp2_neg(t * AFN_LOG2E, tab);
  }
  return exp2_neg(d2 * f.c, tab);
}

// ---------------------------------------------------------------------------
// Deterministic block reductions.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /*>= NT/32*/) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < NT / 32) ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in warp 0
}

// last-block-done deterministic finish: partials in block order
__device__ __forceinline__ void finish_sum(double partial, double* ws, unsigned* cnt, double* out) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    ws[blockIdx.x] = partial;
    __threadfence();
    const unsigned t = atomicAdd(cnt, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += __ldcg(&ws[b]);
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      *out = s;
      *cnt = 0u;
    }
  }
}


}  // namespace afn

// ---------------------------------------------------------------------------
// Host-side error plumbing shared by the .cu files.
namespace afn {
void set_error(const char* fmt, ...);
afn_status cuda_status(cudaError_t e, const char* what);
}  // namespace afn

#define AFN_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) return afn::cuda_status(e_, #call);               \
  } while (0)

#define TRY_STATUS(x)                                                        \
  do {                                                                       \
    afn_status s_ = (x);                                                     \
    if (s_ != AFN_OK) return s_;                                             \
  } while (0)

#define AFN_LAUNCH_CHECK(what)                                               \
  do {                                                                       \
    cudaError_t e_ = cudaGetLastError();                                     \
    if (e_ != cudaSuccess) return afn::cuda_status(e_, what);                \
    afn::note_launch();                                                      \
  } while (0)

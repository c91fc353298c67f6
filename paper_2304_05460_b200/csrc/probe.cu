// probe.cu -- FP64 FMA throughput probe for the roofline denominator
// (bench.py reports it beside the guide-derived nominal peak).
#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

__global__ void __launch_bounds__(256) dfma_probe_kernel(int64_t iters, double seed, double* out) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

afn_status probe_dfma(int64_t iters, double* tflops, cudaStream_t st) {
  const int blocks = num_sms() * 8;
  double* out = nullptr;
  afn_status s = dalloc((void**)&out, sizeof(double), st);
  if (s != AFN_OK) return s;
  cudaEvent_t e0, e1;
  AFN_CUDA(cudaEventCreate(&e0));
  AFN_CUDA(cudaEventCreate(&e1));
  dfma_probe_kernel<<<blocks, 256, 0, st>>>(iters / 8, 1.0, out);  // warm-up
  AFN_LAUNCH_CHECK("dfma_probe_kernel");
  AFN_CUDA(cudaEventRecord(e0, st));
  dfma_probe_kernel<<<blocks, 256, 0, st>>>(iters, 1.0, out);
  AFN_LAUNCH_CHECK("dfma_probe_kernel");
  AFN_CUDA(cudaEventRecord(e1, st));
  AFN_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AFN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  dfree(out, st);
  const double flops = 2.0 * 32.0 * (double)iters * (double)blocks * 256.0;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return AFN_OK;
}

}  // namespace afn

// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput probe
namespace afn {
namespace {
__global__ void __launch_bounds__(256) dmma_probe_kernel(int64_t iters, double seed, double* out) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) c[u][0] = c[u][1] = 0.0;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

afn_status probe_dmma(int64_t iters, double* tflops, cudaStream_t st) {
  const int blocks = num_sms() * 8;
  double* out = nullptr;
  afn_status s = dalloc((void**)&out, sizeof(double), st);
  if (s != AFN_OK) return s;
  cudaEvent_t e0, e1;
  AFN_CUDA(cudaEventCreate(&e0));
  AFN_CUDA(cudaEventCreate(&e1));
  dmma_probe_kernel<<<blocks, 256, 0, st>>>(iters / 8, 1.0, out);
  AFN_LAUNCH_CHECK("dmma_probe_kernel");
  AFN_CUDA(cudaEventRecord(e0, st));
  dmma_probe_kernel<<<blocks, 256, 0, st>>>(iters, 1.0, out);
  AFN_LAUNCH_CHECK("dmma_probe_kernel");
  AFN_CUDA(cudaEventRecord(e1, st));
  AFN_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AFN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  dfree(out, st);
  // per warp-instruction: 8x8x4 = 256 FMA = 512 flop; 4 per iteration per warp
  const double flops = 512.0 * 4.0 * (double)iters * (double)blocks * (256 / 32);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return AFN_OK;
}
}  // namespace afn

// MUFU.EX2 (ex2.approx.ftz.f32) throughput probe: the bound of the cutoff
// matvec's FP32 body (one EX2 per pair, kmv.cu)
namespace afn {
namespace {
__global__ void __launch_bounds__(256) ex2_probe_kernel(int64_t iters, float seed, float* out) {
  float a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = seed + 1e-3f * (threadIdx.x + u);
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[u]));
  }
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 12345.678f) out[0] = s;
}
}  // namespace

afn_status probe_ex2(int64_t iters, double* gops, cudaStream_t st) {
  const int blocks = num_sms() * 8;
  float* out = nullptr;
  afn_status s = dalloc((void**)&out, sizeof(float), st);
  if (s != AFN_OK) return s;
  cudaEvent_t e0, e1;
  AFN_CUDA(cudaEventCreate(&e0));
  AFN_CUDA(cudaEventCreate(&e1));
  ex2_probe_kernel<<<blocks, 256, 0, st>>>(iters / 8, -0.5f, out);
  AFN_LAUNCH_CHECK("ex2_probe_kernel");
  AFN_CUDA(cudaEventRecord(e0, st));
  ex2_probe_kernel<<<blocks, 256, 0, st>>>(iters, -0.5f, out);
  AFN_LAUNCH_CHECK("ex2_probe_kernel");
  AFN_CUDA(cudaEventRecord(e1, st));
  AFN_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AFN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  dfree(out, st);
  *gops = 8.0 * (double)iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e9;
  return AFN_OK;
}
}  // namespace afn

// Latency probes (one warp, dependent chains): DFMA, DADD, DMUL, rsqrt(double),
// sqrt(double), LDS.64, SHFL (double), FFMA.  nvcc -arch=sm_100a -O3 lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k_dfma(double* o, long long* t, double a, double b) {
  double x = o[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_dadd(double* o, long long* t, double a, double b) {
  double x = o[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + a;
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_ffma(double* o, long long* t, double a, double b) {
  float x = (float)o[threadIdx.x], fa = (float)a, fb = (float)b;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fmaf(x, fa, fb);
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_rsqrt(double* o, long long* t, double a, double b) {
  double x = o[threadIdx.x] + 2.0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 1.5;
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_sqrt(double* o, long long* t, double a, double b) {
  double x = o[threadIdx.x] + 2.0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = sqrt(x) + 1.5;
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_lds(double* o, long long* t, double a, double b) {
  __shared__ double s[64];
  s[threadIdx.x] = (double)((threadIdx.x + 1) & 31);
  __syncwarp();
  int j = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) j = (int)s[j];
  long long t1 = clock64();
  o[threadIdx.x] = j; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_shfl(double* o, long long* t, double a, double b) {
  double x = o[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void k_syncwarp_sts_lds(double* o, long long* t, double a, double b) {
  __shared__ double s[32];
  double x = o[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) { s[threadIdx.x] = x; __syncwarp(); x = s[(threadIdx.x + 1) & 31] * a; __syncwarp(); }
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
  double* o; long long* t; long long h;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&t, 8); cudaMemset(o, 0, 64 * 8);
  struct { const char* n; void (*k)(double*, long long*, double, double); } ks[] = {
    {"DFMA", k_dfma}, {"DADD", k_dadd}, {"FFMA", k_ffma}, {"rsqrt(f64)+DADD", k_rsqrt},
    {"sqrt(f64)+DADD", k_sqrt}, {"LDS.64+F2I", k_lds}, {"SHFL f64", k_shfl}, {"STS+syncwarp+LDS+DMUL", k_syncwarp_sts_lds}};
  for (auto& k : ks) {
    for (int r = 0; r < 2; ++r) { k.k<<<1, 32>>>(o, t, 1.0000001, 1e-9); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %.1f cycles/step\n", k.n, (double)h / N);
  }
  return 0;
}

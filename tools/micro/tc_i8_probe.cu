// tc_i8_probe.cu -- validates the hand-built tcgen05 INT8 path on sm_100a and
// measures its throughput (one CTA per SM, back-to-back MMAs from shared
// memory).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   tools/micro/tc_i8_probe.cu -o /tmp/tc_i8_probe && /tmp/tc_i8_probe
//
// Layout (K-major, no swizzle, "interleave"): an R x KB-byte operand tile is
// stored as 16-byte core rows, core matrices of 8 rows x 16 bytes (128 B);
// byte address(r, kk) = kk * (R / 8) * 128 + (r / 8) * 128 + (r % 8) * 16 for
// the kk-th 16-byte K chunk.  Descriptor: SBO = 128 B (next 8-row group),
// LBO = (R / 8) * 128 B (next 16-byte K chunk), version 1, layout 0.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

#ifndef PN
#define PN 64
#endif
constexpr int M = 128, N = PN, KB = 64;  // tile: 128 x 64 output, 64-byte K block (2 MMAs of K = 32)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  // base offset 0, lbo mode 0, layout type 0 (no swizzle)
  return d;
}

// instruction descriptor: kind::i8, D s32, A/B signed int8, K-major both
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (2u << 4)                 // c_format S32
         | (1u << 7)               // a_format signed int8
         | (1u << 10)              // b_format signed int8
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// A: M x KB int8 row-major (global), B: N x KB int8 row-major (B^T of the
// K x N operand), C: M x N int32 row-major.  One CTA of 128 threads; `reps`
// repeats the MMA pair (accumulating) for the throughput measurement.
__global__ void __launch_bounds__(128, 1) probe_kernel(const int8_t* A, const int8_t* B, int32_t* C, int reps) {
  __shared__ __align__(128) int8_t sA[M * KB];
  __shared__ __align__(128) int8_t sB[N * KB];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // stage A, B into the interleaved core-matrix layout
  for (int e = tid; e < M * (KB / 16); e += 128) {
    const int r = e / (KB / 16), kk = e % (KB / 16);
    const int4 v = *reinterpret_cast<const int4*>(A + r * KB + kk * 16);
    *reinterpret_cast<int4*>(sA + kk * (M / 8) * 128 + (r / 8) * 128 + (r % 8) * 16) = v;
  }
  for (int e = tid; e < N * (KB / 16); e += 128) {
    const int r = e / (KB / 16), kk = e % (KB / 16);
    const int4 v = *reinterpret_cast<const int4*>(B + r * KB + kk * 16);
    *reinterpret_cast<int4*>(sB + kk * (N / 8) * 128 + (r / 8) * 128 + (r % 8) * 16) = v;
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(M, N);
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < KB / 32; ++ks) {  // K = 32 bytes per MMA = two 16-byte chunks
        const uint64_t da = make_desc(a0 + ks * 2 * lboA, lboA, 128);
        const uint64_t db = make_desc(b0 + ks * 2 * lboB, lboB, 128);
        mma_i8(tmem, da, db, idesc, (r > 0 || ks > 0) ? 1u : 0u);
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 8 columns at a time
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

int main() {
  std::vector<int8_t> hA(M * KB), hB(N * KB);
  srand(1);
  for (auto& x : hA) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : hB) x = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dC, sizeof(int32_t) * M * N));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  for (int reps : {1, 3}) {
    probe_kernel<<<1, 128>>>(dA, dB, dC, reps);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> hC(M * N);
    CK(cudaMemcpy(hC.data(), dC, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
    long long bad = 0, maxd = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long long ref = 0;
        for (int t = 0; t < KB; ++t) ref += (long long)hA[i * KB + t] * hB[j * KB + t];
        ref *= reps;
        const long long d = llabs(ref - (long long)hC[i * N + j]);
        if (d) ++bad;
        if (d > maxd) maxd = d;
      }
    printf("reps %d: mismatches %lld of %d, max |diff| %lld  (C[0][0] %d, C[5][7] %d)\n", reps, bad, M * N, maxd,
           hC[0], hC[5 * N + 7]);
  }
  // throughput: one CTA per SM, many MMAs each
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int reps = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe_kernel<<<sms, 128>>>(dA, dB, dC, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  probe_kernel<<<sms, 128>>>(dA, dB, dC, reps);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * M * N * KB * (double)reps * sms;
  printf("throughput: %d CTAs x %d reps of %dx%dx%d: %.3f ms, %.1f TOPS (int8, N = %d)\n", sms, reps, M, N, KB, ms,
         ops / ms / 1e9, N);
  return 0;
}

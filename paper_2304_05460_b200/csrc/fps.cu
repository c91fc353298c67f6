// fps.cu -- farthest point sampling (eq. (3.3)), the
// paper's brute-force parallel form (L800: "an O(n) distance update in
// parallel at each step").
//
// One persistent cooperative kernel runs all k dependent steps.  Each thread
// keeps P points and their running min squared distance `mind` in registers
// (or, for very large n, streams them from global/L2).  A step is: update mind
// with the newest landmark, argmax over (mind desc, index asc) by warp
// shuffles, a shared-memory block reduce, one grid barrier, and a redundant
// (identical in every CTA) reduce of the G per-CTA winners, whose coordinates
// travel with them so no dependent load follows the barrier.
// Bit-exact with the readings R3: squared distances are sums in coordinate
// order of individually rounded (x_c - y_c)^2; selected points carry mind = -1
// and are never re-picked; ties go to the lowest index.
#include <cstdio>
#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cmath>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int FPS_NT = 512;

__device__ __forceinline__ bool better(double d1, long long i1, double d2, long long i2) {
  return d1 > d2 || (d1 == d2 && i1 < i2);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// slot layout: [0] = d2, [1] = idx (bits), [2..2+DP) = coordinates
template <int DP>
struct Slot {
  static constexpr int S = DP + 2;
};

// P > 0: points in registers; P == 0: points streamed from global (mind in gmem).
template <int DP, int P>
__global__ void __launch_bounds__(FPS_NT, 1)
fps_kernel(const double* __restrict__ X, int64_t n, int d, int64_t k, int64_t seed,
           int64_t* __restrict__ idx_out, double* __restrict__ fill_out, double* slots,
           unsigned* bar, double* __restrict__ gmind, int pglob) {
  constexpr int S = Slot<DP>::S;
  constexpr int NW = FPS_NT / 32;
  constexpr int PR = P > 0 ? P : 1;
  __shared__ double s_w[NW][S];
  __shared__ double s_new[S];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t stride = (int64_t)G * FPS_NT;
  const int64_t gtid = (int64_t)blockIdx.x * FPS_NT + tid;
  const int np = P > 0 ? P : pglob;

  double pts[PR][DP];
  double mind[PR];

  // seed coordinates
  double y[DP];
#pragma unroll
  for (int c = 0; c < DP; ++c) y[c] = c < d ? X[seed * d + c] : 0.0;

  auto load_pt = [&](int64_t i, double* q) {
#pragma unroll
    for (int c = 0; c < DP; ++c) q[c] = (c < d) ? X[i * d + c] : 0.0;
  };

  if (P > 0) {
#pragma unroll
    for (int s = 0; s < PR; ++s) {
      const int64_t i = gtid + s * stride;
      if (i < n) {
        load_pt(i, pts[s]);
        mind[s] = (i == seed) ? -1.0 : d2_exact<DP>(pts[s], y);
      } else {
#pragma unroll
        for (int c = 0; c < DP; ++c) pts[s][c] = 0.0;
        mind[s] = -2.0;
      }
    }
  } else {
    for (int s = 0; s < np; ++s) {
      const int64_t i = gtid + s * stride;
      if (i < n) {
        double q[DP];
        load_pt(i, q);
        gmind[i] = (i == seed) ? -1.0 : d2_exact<DP>(q, y);
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) idx_out[0] = seed;

  for (int64_t step = 1; step <= k; ++step) {
    // ---- local argmax (indices ascend with s, strict > keeps the lowest)
    double bd = -3.0;
    long long bi = 0x7fffffffffffffffLL;
    double bc[DP];
#pragma unroll
    for (int c = 0; c < DP; ++c) bc[c] = 0.0;
    if (P > 0) {
#pragma unroll
      for (int s = 0; s < PR; ++s) {
        const int64_t i = gtid + s * stride;
        if (mind[s] > bd) {
          bd = mind[s];
          bi = i;
#pragma unroll
          for (int c = 0; c < DP; ++c) bc[c] = pts[s][c];
        }
      }
    } else {
      for (int s = 0; s < np; ++s) {
        const int64_t i = gtid + s * stride;
        if (i < n) {
          const double m = __ldcg(&gmind[i]);
          if (m > bd) { bd = m; bi = i; }
        }
      }
      if (bi < n) load_pt(bi, bc);
    }
    // ---- warp argmax (butterfly: every lane ends with the same winner)
    double wd = bd;
    long long wi = bi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, wd, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, wi, o);
      if (better(od, oi, wd, wi)) { wd = od; wi = oi; }
    }
    if (bi == wi && bd == wd) {  // the owning lane (unique: indices are unique)
      s_w[wid][0] = wd;
      s_w[wid][1] = __longlong_as_double(wi);
#pragma unroll
      for (int c = 0; c < DP; ++c) s_w[wid][2 + c] = bc[c];
    }
    __syncthreads();
    double* myslot = slots + ((step & 1) * (int64_t)G + blockIdx.x) * S;
    if (wid == 0) {
      double vd = lane < NW ? s_w[lane][0] : -3.0;
      long long vi = lane < NW ? __double_as_longlong(s_w[lane][1]) : 0x7fffffffffffffffLL;
      int src = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, vd, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, vi, o);
        const int os = __shfl_xor_sync(0xffffffffu, src, o);
        if (better(od, oi, vd, vi)) { vd = od; vi = oi; src = os; }
      }
      if (G == 1) {
        if (lane < S) s_new[lane] = s_w[src][lane];
      } else {
        if (lane < S) {
          myslot[lane] = s_w[src][lane];
          __threadfence();
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(bar, 1u);
          const unsigned target = (unsigned)(G * step);
          while (ld_acquire(bar) < target) {
          }
        }
        __syncwarp();
        // reduce the G CTA winners (same order in every CTA -> same result)
        const double* base = slots + ((step & 1) * (int64_t)G) * S;
        double gd = -3.0;
        long long gi = 0x7fffffffffffffffLL;
        int gsrc = -1;
        for (int b = lane; b < G; b += 32) {
          const double od = __ldcg(&base[(int64_t)b * S]);
          const long long oi = __double_as_longlong(__ldcg(&base[(int64_t)b * S + 1]));
          if (better(od, oi, gd, gi)) { gd = od; gi = oi; gsrc = b; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, gd, o);
          const long long oi = __shfl_xor_sync(0xffffffffu, gi, o);
          const int os = __shfl_xor_sync(0xffffffffu, gsrc, o);
          if (better(od, oi, gd, gi)) { gd = od; gi = oi; gsrc = os; }
        }
        if (lane < S) s_new[lane] = __ldcg(&base[(int64_t)gsrc * S + lane]);
      }
    }
    __syncthreads();
    const double nd = s_new[0];
    const long long ni = __double_as_longlong(s_new[1]);
    if (blockIdx.x == 0 && tid == 0) {
      fill_out[step - 1] = nd >= 0.0 ? sqrt(nd) : 0.0;
      if (step < k) idx_out[step] = ni;
    }
    if (step == k) break;
#pragma unroll
    for (int c = 0; c < DP; ++c) y[c] = s_new[2 + c];
    if (P > 0) {
#pragma unroll
      for (int s = 0; s < PR; ++s) {
        const int64_t i = gtid + s * stride;
        if (i < n) {
          const double dd = d2_exact<DP>(pts[s], y);
          mind[s] = (i == ni) ? -1.0 : fmin(mind[s], dd);
        }
      }
    } else {
      for (int s = 0; s < np; ++s) {
        const int64_t i = gtid + s * stride;
        if (i < n) {
          double q[DP];
          load_pt(i, q);
          const double dd = d2_exact<DP>(q, y);
          const double m = __ldcg(&gmind[i]);
          __stcg(&gmind[i], (i == ni) ? -1.0 : fmin(m, dd));
        }
      }
    }
  }
}

template <int DP, int P>
afn_status launch_fps(const double* X, int64_t n, int d, int64_t k, int64_t seed, int64_t* idx,
                      double* fill, int G, double* slots, unsigned* bar, double* gmind, int pglob,
                      cudaStream_t st) {
  auto kern = fps_kernel<DP, P>;
  int occ = 0;
  AFN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, FPS_NT, 0));
  if (G > 1 && occ * num_sms() < G) {
    set_error("fps: grid %d exceeds co-resident capacity %d", G, occ * num_sms());
    return AFN_ERR_CUDA;
  }
  void* args[] = {(void*)&X, (void*)&n, (void*)&d, (void*)&k, (void*)&seed, (void*)&idx,
                  (void*)&fill, (void*)&slots, (void*)&bar, (void*)&gmind, (void*)&pglob};
  if (G > 1) {
    AFN_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(FPS_NT), args, 0, st));
  } else {
    kern<<<1, FPS_NT, 0, st>>>(X, n, d, k, seed, idx, fill, slots, bar, gmind, pglob);
  }
  AFN_LAUNCH_CHECK("fps_kernel");
  return AFN_OK;
}

// (d2 desc, index asc) argmax across a warp with three redux.sync reductions.
// key = bits(d2) + 1 for d2 >= 0 (monotone), 0 for selected (-1) / padding.
__device__ __forceinline__ unsigned long long fps_key(double d) {
  return d >= 0.0 ? (unsigned long long)__double_as_longlong(d) + 1ULL : 0ULL;
}
__device__ __forceinline__ void warp_argmax_key(unsigned long long key, unsigned idx,
                                                unsigned long long& wkey, unsigned& widx) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  wkey = ((unsigned long long)mhi << 32) | mlo;
  widx = __reduce_min_sync(0xffffffffu, key == wkey ? idx : 0xffffffffu);
}

// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;
#ifndef AFN_FPS_CULL
#define AFN_FPS_CULL 1
#endif

// Cluster kernel (n up to 16 CTAs x NT x P points, no global-memory round
// trips per step): after its CTA-level argmax, warp 0 of
// every CTA writes its winner slot (d2, index, point, early-stop sample) into
// every CTA's inbox with st.async (asynchronous distributed-shared-memory
// stores that complete bytes on the destination's mbarrier: no fence, no
// round trip on the sender); each warp waits on its own CTA's mbarrier
// (one local arrival with the expected byte count per phase) and reduces the
// CL slots from local shared memory.  Inboxes and mbarriers alternate with
// the step parity: a CTA can only write step t+2's slot into an inbox after it
// has received every CTA's step t+1 slot, which each CTA sends after it has
// finished reading its step t inbox.  The index / fill outputs and the
// early-stop polling are done by other warps of CTA 0 (off the critical path
// of warp 0, which pushes the next step).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned a, int r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void st_async_v2(unsigned a, double x, double y, unsigned bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(a),
               "d"(x), "d"(y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned a, unsigned ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(ph)
      : "memory");
}

// SP: the points live in dynamic shared memory ([s][c][thread], conflict-free)
// instead of registers -- 8 points per thread at 1024 threads, so one cluster
// of 16 CTAs covers n = 131072 (C3) instead of 65536; the running minima stay
// in registers.
//
// CULL (with SP): the slots hold the points in a spatial order perm (a warp's
// 8 x 32 slots are 256 consecutive positions, its bounding box kept in shared
// memory) and each slot keeps its point's index; a step skips a warp's
// distance updates when the new landmark's squared distance to the warp's box
// exceeds the warp's largest running minimum -- computed with the rounded
// operations of d2_exact on the box gaps, it is a lower bound of every
// point's d2, so no minimum could change.  Ties take the lowest index as in
// the unpermuted kernel, so landmarks and fill distances are bit-identical.
template <int DP, int P, int NT, bool SP = false, bool CULL = false>
__global__ void __launch_bounds__(NT, 1)
fps_push_kernel(const double* __restrict__ X, int64_t n, int d, int64_t k, int64_t seed,
                int64_t* __restrict__ idx_out, double* __restrict__ fill_out, const int64_t* __restrict__ kstop,
                const int* __restrict__ perm) {
  extern __shared__ __align__(16) double s_pts[];
  constexpr int KI = DP + 2;          // slot: d2, index, point (DP), early-stop sample (KI)
  constexpr int S = (KI + 2) & ~1;    // even length (16-byte stores)
  constexpr int NW = NT / 32;
  constexpr int CLX = 16;
  static_assert(NW >= 3, "needs a pusher, a poller and an output warp");
  __shared__ __align__(16) double s_w[NW][S];
  __shared__ __align__(16) double s_in[2][CLX][S];
  __shared__ __align__(8) unsigned long long s_bar[2];
  __shared__ long long s_kend;
  __shared__ double s_box[CULL ? NT / 32 : 1][2 * DP];  // CULL: per warp lo[DP], hi[DP]
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int CL = (int)cl.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t stride = (int64_t)CL * NT;
  const int64_t gtid = (int64_t)crank * NT + tid;
  const unsigned txb = (unsigned)(CL * S * 8);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_bar[0])), "r"(1) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_bar[1])), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_kend = k;
  }
  double pts[SP ? 1 : P][DP];
  double mind[P];
  double y[DP];
  int oi[CULL ? P : 1];  // CULL: the slot's point index (-1: none)
  auto pt = [&](int sidx, int c) -> double& {
    return SP ? s_pts[(sidx * DP + c) * NT + tid] : pts[SP ? 0 : sidx][c];
  };
  // the point index of slot s (CULL: through the spatial order)
  auto slot_index = [&](int s) -> int64_t {
    if (!CULL) return gtid + s * stride;
    const int64_t j = ((int64_t)crank * NT + wid * 32) * P + s * 32 + lane;
    return j < n ? (int64_t)perm[j] : n;
  };
#pragma unroll
  for (int c = 0; c < DP; ++c) y[c] = c < d ? X[seed * d + c] : 0.0;
  double blo[DP], bhi[DP];
#pragma unroll
  for (int c = 0; c < DP; ++c) {
    blo[c] = CUDART_INF;
    bhi[c] = -CUDART_INF;
  }
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int64_t i = slot_index(s);
    if (CULL) oi[CULL ? s : 0] = i < n ? (int)i : -1;
    double q[DP];
#pragma unroll
    for (int c = 0; c < DP; ++c) {
      q[c] = (i < n && c < d) ? X[i * d + c] : 0.0;
      pt(s, c) = q[c];
      if (CULL && i < n) {
        blo[c] = fmin(blo[c], q[c]);
        bhi[c] = fmax(bhi[c], q[c]);
      }
    }
    mind[s] = i < n ? ((i == seed) ? -1.0 : d2_exact<DP>(q, y)) : -2.0;
  }
  if (CULL) {
#pragma unroll
    for (int c = 0; c < DP; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        blo[c] = fmin(blo[c], __shfl_xor_sync(0xffffffffu, blo[c], o));
        bhi[c] = fmax(bhi[c], __shfl_xor_sync(0xffffffffu, bhi[c], o));
      }
      if (lane == 0) {
        s_box[CULL ? wid : 0][c] = blo[c];
        s_box[CULL ? wid : 0][DP + c] = bhi[c];
      }
    }
    __syncwarp();
  }
  if (crank == 0 && tid == 0) idx_out[0] = seed;
  cl.sync();  // every CTA's mbarriers are initialised before the first push
  if (tid == 0) {  // the local arrivals (with the inbox byte count) of steps 1 and 2
    mbar_expect(smem_u32(&s_bar[1]), txb);
    mbar_expect(smem_u32(&s_bar[0]), txb);
  }
  unsigned ph0 = 0, ph1 = 0;
  for (int64_t step = 1; step <= k; ++step) {
    const int par = (int)(step & 1);
    if (crank == 0 && wid == 1 && lane == 0 && kstop != nullptr && (step & 7) == 0)  // early-stop poll
      s_kend = min(s_kend, *reinterpret_cast<const volatile long long*>(kstop));
    double bd = -3.0;
    unsigned bi = 0xffffffffu;
    int bs = 0;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const unsigned is = CULL ? (unsigned)oi[CULL ? s : 0] : (unsigned)(gtid + s * stride);
      if (mind[s] > bd || (CULL && mind[s] == bd && is < bi)) { bd = mind[s]; bi = is; bs = s; }
    }
    unsigned long long wkey;
    unsigned widx;
    warp_argmax_key(fps_key(bd), bi, wkey, widx);
    if (bi == widx) {
      s_w[wid][0] = bd;
      s_w[wid][1] = __longlong_as_double((long long)widx);
#pragma unroll
      for (int c = 0; c < DP; ++c) s_w[wid][2 + c] = pt(bs, c);
    }
    __syncthreads();
    if (wid == 0) {
      const double vd = lane < NW ? s_w[lane][0] : -3.0;
      const unsigned vi = lane < NW ? (unsigned)__double_as_longlong(s_w[lane][1]) : 0xffffffffu;
      unsigned long long k2;
      unsigned i2;
      warp_argmax_key(fps_key(vd), vi, k2, i2);
      const int src = __ffs(__ballot_sync(0xffffffffu, lane < NW && vi == i2)) - 1;
      if (lane < CL) {  // lane j pushes to CTA j
        double msg[S];
#pragma unroll
        for (int c = 0; c < KI; ++c) msg[c] = s_w[src][c];
#pragma unroll
        for (int c = KI; c < S; ++c) msg[c] = __longlong_as_double(s_kend);
        const unsigned dst = mapa_u32(smem_u32(&s_in[par][crank][0]), lane);
        const unsigned bar = mapa_u32(smem_u32(&s_bar[par]), lane);
#pragma unroll
        for (int c = 0; c < S; c += 2) st_async_v2(dst + 8 * c, msg[c], msg[c + 1], bar);
      }
    }
    mbar_wait_parity(smem_u32(&s_bar[par]), par ? ph1 : ph0);
    if (par) ph1 ^= 1; else ph0 ^= 1;
    if (tid == 0 && step + 2 <= k) mbar_expect(smem_u32(&s_bar[par]), txb);  // arrival of step + 2
    // every warp reduces the CL slots itself (no second CTA barrier)
    const double gd = lane < CL ? s_in[par][lane][0] : -3.0;
    const unsigned gi = lane < CL ? (unsigned)__double_as_longlong(s_in[par][lane][1]) : 0xffffffffu;
    unsigned long long k3;
    unsigned i3;
    warp_argmax_key(fps_key(gd), gi, k3, i3);
    const int src = __ffs(__ballot_sync(0xffffffffu, lane < CL && gi == i3)) - 1;
    const long long ni = (long long)i3;
    const long long kst = __double_as_longlong(s_in[par][0][KI]);
    if (crank == 0 && wid == NW - 1 && lane == 0) {  // outputs (off warp 0's path)
      const double nd = s_in[par][src][0];
      fill_out[step - 1] = nd >= 0.0 ? sqrt(nd) : 0.0;
      if (step < k) idx_out[step] = ni;
    }
    if (step >= kst) break;
#pragma unroll
    for (int c = 0; c < DP; ++c) y[c] = s_in[par][src][2 + c];
    if (CULL) {  // the new landmark's d2 to the warp's box against the warp's largest minimum
      double g[DP];
#pragma unroll
      for (int c = 0; c < DP; ++c) {
        const double lo = s_box[CULL ? wid : 0][c], hi = s_box[CULL ? wid : 0][DP + c];
        g[c] = y[c] < lo ? __dsub_rn(lo, y[c]) : (y[c] > hi ? __dsub_rn(y[c], hi) : 0.0);
      }
      double bd2 = __dmul_rn(g[0], g[0]);
#pragma unroll
      for (int c = 1; c < DP; ++c) bd2 = __dadd_rn(bd2, __dmul_rn(g[c], g[c]));
      const double wmax = wkey == 0ull ? -1.0 : __longlong_as_double((long long)(wkey - 1ull));
      if (bd2 > wmax) continue;
    }
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int64_t i = CULL ? (int64_t)oi[CULL ? s : 0] : gtid + s * stride;
      if (i >= 0 && i < n) {
        double q[DP];
#pragma unroll
        for (int c = 0; c < DP; ++c) q[c] = pt(s, c);
        const double dd = d2_exact<DP>(q, y);
        mind[s] = (i == ni) ? -1.0 : fmin(mind[s], dd);
      }
    }
  }
  cl.sync();  // no CTA leaves while a push into it may be in flight
}

template <int DP, int P, int NT, bool SP = false, bool CULL = false>
afn_status launch_fps_push(const double* X, int64_t n, int d, int64_t k, int64_t seed,
                           int64_t* idx, double* fill, int CL, const int64_t* kstop, cudaStream_t st,
                           const int* perm = nullptr) {
  auto kern = fps_push_kernel<DP, P, NT, SP, CULL>;
  if (CL > 8) AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const size_t dyn = SP ? sizeof(double) * (size_t)P * DP * NT : 0;
  if (SP) AFN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AFN_CUDA(cudaLaunchKernelEx(&cfg, kern, X, n, d, k, seed, idx, fill, kstop, perm));
  AFN_LAUNCH_CHECK("fps_push_kernel");
  return AFN_OK;
}

template <int DP>
afn_status fps_dispatch_p(const double* X, int64_t n, int d, int64_t k, int64_t seed, int64_t* idx,
                          double* fill, const int64_t* kstop, cudaStream_t st) {
  const int sms = num_sms();
  // cluster path: one cluster of CL <= 16 CTAs, 1 or 2 points per thread
  {
    constexpr int CNT = DP <= 4 ? 1024 : 512;
    // points per thread: fewer CTAs in the cluster against more distance
    // updates per thread; smaller CTAs with more points per thread: fewer
    // warps to reduce per step (C2, k = 2000: 1024 threads 2.52 ms, 512: 2.08,
    // 256: 2.04; the cluster-barrier exchange instead of the pushes 3.34)
    if (n > (int64_t)FPS_NT * 8 && n <= (int64_t)16 * CNT * 4) {
      int P2 = 1;
      while (P2 < 4 && n > (int64_t)16 * CNT * P2) P2 *= 2;
      const int CL = (int)((n + (int64_t)CNT * P2 - 1) / ((int64_t)CNT * P2));
      if (CNT == 1024) {
        if (P2 == 1) return launch_fps_push<DP, 4, 256>(X, n, d, k, seed, idx, fill, CL, kstop, st);
        if (P2 == 2) return launch_fps_push<DP, 4, 512>(X, n, d, k, seed, idx, fill, CL, kstop, st);
        return launch_fps_push<DP, 4, CNT>(X, n, d, k, seed, idx, fill, CL, kstop, st);
      }
      if (P2 == 1) return launch_fps_push<DP, 1, CNT>(X, n, d, k, seed, idx, fill, CL, kstop, st);
      if (P2 == 2) return launch_fps_push<DP, 2, CNT>(X, n, d, k, seed, idx, fill, CL, kstop, st);
      return launch_fps_push<DP, 4, CNT>(X, n, d, k, seed, idx, fill, CL, kstop, st);
    }
    // up to 2^17 points (d <= 3): 8 points per thread held in shared memory
    if (DP <= 3 && n > (int64_t)16 * CNT * 4 && n <= (int64_t)16 * 1024 * 8) {
      const int CL = (int)((n + 1024 * 8 - 1) / (1024 * 8));
#if AFN_FPS_CULL
      int* perm = nullptr;
      afn_status s = dalloc((void**)&perm, sizeof(int) * (size_t)n, st);
      if (s != AFN_OK) return s;
      s = morton_order(X, n, d, perm, st);
      if (s == AFN_OK) s = launch_fps_push<DP, 8, 1024, true, true>(X, n, d, k, seed, idx, fill, CL, kstop, st, perm);
      dfree(perm, st);
      return s;
#else
      return launch_fps_push<DP, 8, 1024, true>(X, n, d, k, seed, idx, fill, CL, kstop, st);
#endif
    }
  }
  // choose points per thread P and grid G (G = 1 needs no grid barrier)
  int P = 0, G = 0, pglob = 0;
  const int64_t per1 = FPS_NT;
  if (n <= per1 * 8) {
    G = 1;
    P = 1;
    while ((int64_t)P * per1 < n) P *= 2;
  } else {
    const int64_t cap_reg = (int64_t)sms * per1 * 8;
    if (n <= cap_reg) {
      P = 1;
      while ((int64_t)sms * per1 * P < n) P *= 2;
      G = (int)((n + per1 * P - 1) / (per1 * P));
    } else {
      P = 0;
      G = sms;
      pglob = (int)((n + (int64_t)G * per1 - 1) / ((int64_t)G * per1));
    }
  }
  double* slots = nullptr;
  unsigned* bar = nullptr;
  double* gmind = nullptr;
  const size_t slot_bytes = sizeof(double) * 2 * (size_t)G * (DP + 2);
  afn_status s = dalloc((void**)&slots, slot_bytes + 256, st);
  if (s != AFN_OK) return s;
  bar = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(slots) + slot_bytes);
  AFN_CUDA(cudaMemsetAsync(bar, 0, 256, st));
  if (P == 0) {
    s = dalloc((void**)&gmind, sizeof(double) * n, st);
    if (s != AFN_OK) { dfree(slots, st); return s; }
  }
  switch (P) {
    case 0: s = launch_fps<DP, 0>(X, n, d, k, seed, idx, fill, G, slots, bar, gmind, pglob, st); break;
    case 1: s = launch_fps<DP, 1>(X, n, d, k, seed, idx, fill, G, slots, bar, gmind, pglob, st); break;
    case 2: s = launch_fps<DP, 2>(X, n, d, k, seed, idx, fill, G, slots, bar, gmind, pglob, st); break;
    case 4: s = launch_fps<DP, 4>(X, n, d, k, seed, idx, fill, G, slots, bar, gmind, pglob, st); break;
    default: s = launch_fps<DP, 8>(X, n, d, k, seed, idx, fill, G, slots, bar, gmind, pglob, st); break;
  }
  dfree(slots, st);
  if (gmind) dfree(gmind, st);
  return s;
}

}  // namespace

afn_status fps_run(const double* X, int64_t n, int d, int64_t k, int64_t seed, int64_t* idx,
                   double* fill, cudaStream_t st, const int64_t* kstop) {
  // coordinates are zero-padded to DP: adding +0.0 terms leaves d2 bit-identical
  if (d <= 1) return fps_dispatch_p<1>(X, n, d, k, seed, idx, fill, kstop, st);
  if (d <= 2) return fps_dispatch_p<2>(X, n, d, k, seed, idx, fill, kstop, st);
  if (d <= 3) return fps_dispatch_p<3>(X, n, d, k, seed, idx, fill, kstop, st);
  if (d <= 4) return fps_dispatch_p<4>(X, n, d, k, seed, idx, fill, kstop, st);
  if (d <= 8) return fps_dispatch_p<8>(X, n, d, k, seed, idx, fill, kstop, st);
  if (d <= 16) return fps_dispatch_p<16>(X, n, d, k, seed, idx, fill, kstop, st);
  set_error("fps: d=%d unsupported (1..16)", d);
  return AFN_ERR_ARG;
}

}  // namespace afn

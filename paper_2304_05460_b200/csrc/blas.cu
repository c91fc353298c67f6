// blas.cu -- bandwidth-bound pieces of the AFN apply and
// the PCG vector updates (L788): GEMV with W = K21 L^{-T} and L^{-T}, CSR SpMV
// with G and G^T, deterministic dot products.  All reductions have a fixed
// order (warp butterflies, per-block partials summed in block order) so a
// solve is bit-reproducible.
#include <algorithm>
#include <cmath>

#include "afn_common.cuh"
#include "afn_internal.h"

namespace afn {
namespace {

constexpr int VT = 256;
constexpr int DOT_BLOCKS = 296;  // fixed -> deterministic partial layout

// y[r] = ybase[r] + alpha * A[r,:] x   (one warp per row).  TRI = 1: A upper
// triangular (columns >= r), TRI = 2: lower (columns <= r); the excluded
// triangle must hold zeros (the even-aligned ranges may touch one entry of it).
// Even C: 16-byte loads (A rows and x 16-byte aligned).
template <int TRI>
__global__ void __launch_bounds__(VT) gemv_n_kernel(const double* __restrict__ A, int64_t R, int64_t C,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ ybase, double alpha,
                                                   double* __restrict__ y, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;  // PCG already stopped (device-side flag)
  const int64_t r = (int64_t)blockIdx.x * (VT / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  const double* a = A + r * C;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if ((C & 1) == 0) {
    const int64_t lo = TRI == 1 ? (r & ~(int64_t)1) : 0;
    const int64_t hi = TRI == 2 ? min(C, (r + 2) & ~(int64_t)1) : C;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    int64_t c = lo / 2 + lane;
    const int64_t h2 = hi / 2;
    for (; c + 96 < h2; c += 128) {
      const double2 v0 = __ldcs(&a2[c]), v1 = __ldcs(&a2[c + 32]), v2 = __ldcs(&a2[c + 64]), v3 = __ldcs(&a2[c + 96]);
      const double2 w0 = __ldg(&x2[c]), w1 = __ldg(&x2[c + 32]), w2 = __ldg(&x2[c + 64]), w3 = __ldg(&x2[c + 96]);
      s0 = fma(v0.y, w0.y, fma(v0.x, w0.x, s0));
      s1 = fma(v1.y, w1.y, fma(v1.x, w1.x, s1));
      s2 = fma(v2.y, w2.y, fma(v2.x, w2.x, s2));
      s3 = fma(v3.y, w3.y, fma(v3.x, w3.x, s3));
    }
    for (; c < h2; c += 32) {
      const double2 v0 = __ldcs(&a2[c]), w0 = __ldg(&x2[c]);
      s0 = fma(v0.y, w0.y, fma(v0.x, w0.x, s0));
    }
  } else {
    int64_t c = (TRI == 1 ? r : 0) + lane;
    const int64_t hi = TRI == 2 ? r + 1 : C;
    for (; c + 96 < hi; c += 128) {
      s0 = fma(__ldcs(&a[c]), __ldg(&x[c]), s0);
      s1 = fma(__ldcs(&a[c + 32]), __ldg(&x[c + 32]), s1);
      s2 = fma(__ldcs(&a[c + 64]), __ldg(&x[c + 64]), s2);
      s3 = fma(__ldcs(&a[c + 96]), __ldg(&x[c + 96]), s3);
    }
    for (; c < hi; c += 32) s0 = fma(__ldcs(&a[c]), __ldg(&x[c]), s0);
  }
  double s = warp_sum((s0 + s1) + (s2 + s3));
  if (lane == 0) y[r] = (ybase ? ybase[r] : 0.0) + alpha * s;
}

// partial[b, c] = sum_{r in block b} A[r, c] x[r]
__global__ void __launch_bounds__(VT) gemv_t_partial_kernel(const double* __restrict__ A, int64_t R,
                                                           int64_t C, int64_t rows_per_block,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ part, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  extern __shared__ double sx[];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(R, r0 + rows_per_block);
  const int nr = (int)(r1 - r0);
  for (int t = threadIdx.x; t < nr; t += VT) sx[t] = x[r0 + t];
  __syncthreads();
  if ((C & 1) == 0 && C >= 512) {  // column pairs: 16-byte loads
    const int64_t C2 = C / 2;
    for (int64_t c2 = threadIdx.x; c2 < C2; c2 += VT) {
      const double2* a = reinterpret_cast<const double2*>(A + r0 * C) + c2;
      double2 s0 = make_double2(0.0, 0.0), s1 = s0;
      int t = 0;
      for (; t + 1 < nr; t += 2) {
        const double2 v0 = __ldcs(&a[(int64_t)t * C2]), v1 = __ldcs(&a[(int64_t)(t + 1) * C2]);
        s0.x = fma(v0.x, sx[t], s0.x);
        s0.y = fma(v0.y, sx[t], s0.y);
        s1.x = fma(v1.x, sx[t + 1], s1.x);
        s1.y = fma(v1.y, sx[t + 1], s1.y);
      }
      if (t < nr) {
        const double2 v0 = __ldcs(&a[(int64_t)t * C2]);
        s0.x = fma(v0.x, sx[t], s0.x);
        s0.y = fma(v0.y, sx[t], s0.y);
      }
      reinterpret_cast<double2*>(part + (int64_t)blockIdx.x * C)[c2] = make_double2(s0.x + s1.x, s0.y + s1.y);
    }
    return;
  }
  for (int64_t c = threadIdx.x; c < C; c += VT) {
    const double* a = A + r0 * C + c;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int t = 0;
    for (; t + 3 < nr; t += 4) {
      s0 = fma(__ldcs(&a[(int64_t)t * C]), sx[t], s0);
      s1 = fma(__ldcs(&a[(int64_t)(t + 1) * C]), sx[t + 1], s1);
      s2 = fma(__ldcs(&a[(int64_t)(t + 2) * C]), sx[t + 2], s2);
      s3 = fma(__ldcs(&a[(int64_t)(t + 3) * C]), sx[t + 3], s3);
    }
    for (; t < nr; ++t) s0 = fma(__ldcs(&a[(int64_t)t * C]), sx[t], s0);
    part[(int64_t)blockIdx.x * C + c] = (s0 + s1) + (s2 + s3);
  }
}

// y[c] = ybase[c] + alpha * sum_b part[b, c]; 32 columns x 32 partial lanes
// per block (warp w sums b = w, w + 32, ...), fixed combination order
// (deterministic)
__global__ void __launch_bounds__(1024) gemv_t_reduce_kernel(const double* __restrict__ part, int nb,
                                                            int64_t C, const double* __restrict__ ybase,
                                                            double alpha, double* __restrict__ y,
                                                            const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (c < C)
    for (int b = w; b < nb; b += 32) s += part[(int64_t)b * C + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < C) {
    double t = sh[0][lane];
#pragma unroll
    for (int q = 1; q < 32; ++q) t += sh[q][lane];
    y[c] = (ybase ? ybase[c] : 0.0) + alpha * t;
  }
}

// Tall full matrices, even C: two rows per warp (each x load serves both
// rows), 16-byte loads, three independent 16-byte loads in flight per step.
__global__ void __launch_bounds__(VT) gemv_n2_kernel(const double* __restrict__ A, int64_t R, int64_t C,
                                                    const double* __restrict__ x,
                                                    const double* __restrict__ ybase, double alpha,
                                                    double* __restrict__ y, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t r = 2 * ((int64_t)blockIdx.x * (VT / 32) + (threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  const bool two = r + 1 < R;
  const int64_t C2 = C / 2;
  const double2* a0 = reinterpret_cast<const double2*>(A + r * C);
  const double2* a1 = two ? a0 + C2 : a0;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double s0 = 0.0, s1 = 0.0, t0 = 0.0, t1 = 0.0;
  int64_t c = lane;
  for (; c + 32 < C2; c += 64) {
    const double2 w0 = __ldg(&x2[c]), w1 = __ldg(&x2[c + 32]);
    const double2 u0 = __ldcs(&a0[c]), u1 = __ldcs(&a0[c + 32]);
    const double2 v0 = __ldcs(&a1[c]), v1 = __ldcs(&a1[c + 32]);
    s0 = fma(u0.y, w0.y, fma(u0.x, w0.x, s0));
    s1 = fma(u1.y, w1.y, fma(u1.x, w1.x, s1));
    t0 = fma(v0.y, w0.y, fma(v0.x, w0.x, t0));
    t1 = fma(v1.y, w1.y, fma(v1.x, w1.x, t1));
  }
  if (c < C2) {
    const double2 w0 = __ldg(&x2[c]), u0 = __ldcs(&a0[c]), v0 = __ldcs(&a1[c]);
    s0 = fma(u0.y, w0.y, fma(u0.x, w0.x, s0));
    t0 = fma(v0.y, w0.y, fma(v0.x, w0.x, t0));
  }
  const double s = warp_sum(s0 + s1), t = warp_sum(t0 + t1);
  if (lane == 0) {
    y[r] = (ybase ? ybase[r] : 0.0) + alpha * s;
    if (two) y[r + 1] = (ybase ? ybase[r + 1] : 0.0) + alpha * t;
  }
}

// Short matrices (R <= GEMV_ROW_CTA): one CTA per row, 16-byte loads, block
// sum in a fixed order; same TRI convention as gemv_n_kernel.
template <int TRI>
__global__ void __launch_bounds__(VT) gemv_n_row_kernel(const double* __restrict__ A, int64_t R, int64_t C,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ ybase, double alpha,
                                                       double* __restrict__ y, const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[VT / 32];
  const int64_t r = blockIdx.x;
  const double* a = A + r * C;
  const int64_t lo = TRI == 1 ? (r & ~(int64_t)1) : 0;
  const int64_t hi = TRI == 2 ? min(C, (r + 2) & ~(int64_t)1) : C;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double s0 = 0.0, s1 = 0.0;
  int64_t c = lo / 2 + threadIdx.x;
  const int64_t h2 = hi / 2;
  for (; c + VT < h2; c += 2 * VT) {
    const double2 v0 = __ldcs(&a2[c]), v1 = __ldcs(&a2[c + VT]);
    const double2 w0 = __ldg(&x2[c]), w1 = __ldg(&x2[c + VT]);
    s0 = fma(v0.y, w0.y, fma(v0.x, w0.x, s0));
    s1 = fma(v1.y, w1.y, fma(v1.x, w1.x, s1));
  }
  if (c < h2) {
    const double2 v0 = __ldcs(&a2[c]), w0 = __ldg(&x2[c]);
    s0 = fma(v0.y, w0.y, fma(v0.x, w0.x, s0));
  }
  const double s = block_sum<VT>(s0 + s1, sh);
  if (threadIdx.x == 0) y[r] = (ybase ? ybase[r] : 0.0) + alpha * s;
}
constexpr int64_t GEMV_ROW_CTA = 8192;

__global__ void __launch_bounds__(VT) spmv_kernel(const int64_t* __restrict__ rp,
                                                 const int32_t* __restrict__ col,
                                                 const double* __restrict__ val, int64_t N,
                                                 const double* __restrict__ x, double* __restrict__ y,
                                                 const double* skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int64_t r = (int64_t)blockIdx.x * (VT / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
  double s = 0.0;
  const int64_t e1 = rp[r + 1];
  for (int64_t e0 = rp[r] + lane; e0 < e1; e0 += 128) {  // 4 entries per lane in flight
    int cc[4];
    double vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t e = e0 + 32 * u;
      cc[u] = e < e1 ? col[e] : -1;
      vv[u] = e < e1 ? val[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (cc[u] >= 0) s = fma(vv[u], __ldg(&x[cc[u]]), s);
  }
  s = warp_sum(s);
  if (lane == 0) y[r] = s;
}

__global__ void gather_vec_kernel(const double* __restrict__ x, const int64_t* __restrict__ perm,
                                  int64_t n, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[perm[i]];
}
__global__ void scatter_vec_kernel(const double* __restrict__ x, const int64_t* __restrict__ perm,
                                   int64_t n, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[perm[i]] = x[i];
}

__global__ void __launch_bounds__(VT) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                Seg2 g, double* out, double* ws, unsigned* cnt) {
  __shared__ double sh[VT / 32];
  double s = 0.0;
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * VT + threadIdx.x; t < n; t += (int64_t)gridDim.x * VT) {
    const int64_t i = g.phys(t);
    s = fma(a[i], b[i], s);
  }
  s = block_sum<VT>(s, sh);
  finish_sum(s, ws, cnt, out);
}

__global__ void __launch_bounds__(VT) update_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                      const double* __restrict__ p,
                                                      const double* __restrict__ q, Seg2 g,
                                                      const double* sc, int rz_slot, double* rr,
                                                      double* ws, unsigned* cnt) {
  __shared__ double sh[VT / 32];
  if (sc[SC_DONE] != 0.0) return;  // stopped: x and r stay at the stopping iterate
  const double pq = sc[SC_PQ];
  const double alpha = (pq > 0.0 && isfinite(pq)) ? sc[rz_slot] / pq : 0.0;
  double s = 0.0;
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * VT + threadIdx.x; t < n; t += (int64_t)gridDim.x * VT) {
    const int64_t i = g.phys(t);
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum<VT>(s, sh);
  finish_sum(s, ws, cnt, rr);
}

// update_xr + the stopping test in one kernel (one rank): the last block,
// which finishes rr, runs pcg_check's logic (same order of operations)
__global__ void __launch_bounds__(VT) update_xr_check_kernel(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ q, Seg2 g, double* sc,
                                                            int rz_slot, double* ws, unsigned* cnt, double nb,
                                                            double tol, int maxit, int fixed, double* hist) {
  __shared__ double sh[VT / 32];
  __shared__ bool last;
  if (sc[SC_DONE] != 0.0) {  // stopped: x and r stay; only the iteration counter moves
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[SC_IT] += 1.0;
    return;
  }
  const double pq = sc[SC_PQ];
  const double alpha = (pq > 0.0 && isfinite(pq)) ? sc[rz_slot] / pq : 0.0;
  double s = 0.0;
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * VT + threadIdx.x; t < n; t += (int64_t)gridDim.x * VT) {
    const int64_t i = g.phys(t);
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum<VT>(s, sh);
  if (threadIdx.x == 0) {
    ws[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  double t2 = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) t2 += __ldcg(&ws[b]);
  t2 = warp_sum(t2);
  if (threadIdx.x != 0) return;
  *cnt = 0u;
  const double rr = t2;
  sc[SC_RR] = rr;
  const int it = (int)sc[SC_IT] + 1;  // (pcg_check_kernel's logic)
  sc[SC_IT] = it;
  if (!(pq > 0.0) || !isfinite(pq) || !isfinite(rr)) {
    sc[SC_DONE] = 2.0;
    sc[SC_ITS] = it - 1;
    return;
  }
  const double rel = sqrt(rr) / nb;
  hist[it] = rel;
  const bool stop = fixed > 0 ? it >= fixed : rel <= tol;
  if (stop || it >= maxit) {
    sc[SC_DONE] = stop ? 1.0 : 3.0;
    sc[SC_ITS] = it;
  }
}

__global__ void update_p_kernel(double* __restrict__ p, const double* __restrict__ z, Seg2 g,
                                const double* sc, int rz_new_slot, int rz_old_slot) {
  const double beta = sc[rz_new_slot] / sc[rz_old_slot];
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g.phys(t);
    p[i] = fma(beta, p[i], z[i]);
  }
}

__global__ void copy_kernel(double* __restrict__ y, const double* __restrict__ x, Seg2 g) {
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g.phys(t);
    y[i] = x[i];
  }
}
__global__ void axpby_kernel(double* __restrict__ y, double a, const double* __restrict__ x, double b,
                             Seg2 g) {
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g.phys(t);
    y[i] = fma(a, x[i], b * y[i]);
  }
}

// rank-ordered sums of per-rank partials (deterministic, identical on every rank)
__global__ void combine_slots_kernel(const double* __restrict__ part, int R, int stride, unsigned mask,
                                     double* __restrict__ sc) {
  const int slot = threadIdx.x;
  if (slot >= stride || !((mask >> slot) & 1u)) return;
  double s = 0.0;
  for (int q = 0; q < R; ++q) s += part[(int64_t)q * stride + slot];
  sc[slot] = s;
}
__global__ void combine_sub_kernel(const double* __restrict__ part, int R, int64_t C,
                                   const double* __restrict__ base, double* __restrict__ y) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int q = 0; q < R; ++q) s += part[(int64_t)q * C + c];
  y[c] = (base ? base[c] : 0.0) - s;
}

__global__ void scale_kernel(double* __restrict__ y, double a, const double* __restrict__ x, Seg2 g) {
  const int64_t n = g.size();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g.phys(t);
    y[i] = a * x[i];
  }
}

__global__ void fill_kernel(double* __restrict__ y, double v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = v;
}
__global__ void scale_rsqrt_kernel(double* __restrict__ y, const double* __restrict__ s, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double f = 1.0 / sqrt(*s);
  if (i < n) y[i] *= f;
}

__global__ void add_diag_kernel(double* __restrict__ A, int64_t k, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) A[i * k + i] += v;
}

unsigned grid_for(int64_t n, int nt, int cap) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, (n + nt - 1) / nt));
}

int64_t gemv_t_rows_per_block(int64_t R) {
  const int64_t target = 4 * (int64_t)num_sms();
  return std::max<int64_t>(16, (R + target - 1) / target);
}

// Device-side PCG stopping test after iteration `it` (one thread): the
// original host test of afn_pcg_solve, so a chunk of iterations can be queued
// without a host round trip per iteration.  sc[SC_DONE]: 0 running, 1 stop
// test met (rel <= tol, or fixed_iters reached), 2 breakdown, 3 maxit
// exhausted; sc[SC_ITS]: the iteration count of the result.
__global__ void pcg_check_kernel(double* sc, double nb, double tol, int maxit, int fixed, double* hist) {
  const int it = (int)sc[SC_IT] + 1;  // this iteration's number (device counter)
  sc[SC_IT] = it;
  if (sc[SC_DONE] != 0.0) return;
  const double pq = sc[SC_PQ], rr = sc[SC_RR];
  if (!(pq > 0.0) || !isfinite(pq) || !isfinite(rr)) {
    sc[SC_DONE] = 2.0;
    sc[SC_ITS] = it - 1;
    return;
  }
  const double rel = sqrt(rr) / nb;
  hist[it] = rel;
  const bool stop = fixed > 0 ? it >= fixed : rel <= tol;
  if (stop || it >= maxit) {
    sc[SC_DONE] = stop ? 1.0 : 3.0;
    sc[SC_ITS] = it;
  }
}

thread_local const double* t_skip = nullptr;

}  // namespace

void set_skip(const double* flag) { t_skip = flag; }
const double* get_skip() { return t_skip; }

afn_status pcg_check(double* sc, double nb, double tol, int maxit, int fixed, double* hist, cudaStream_t st) {
  pcg_check_kernel<<<1, 1, 0, st>>>(sc, nb, tol, maxit, fixed, hist);
  AFN_LAUNCH_CHECK("pcg_check_kernel");
  return AFN_OK;
}

afn_status gemv_n(const double* A, int64_t R, int64_t C, const double* x, const double* ybase,
                  double alpha, double* y, cudaStream_t st, int tri) {
  if (R <= 0) return AFN_OK;
  if ((C & 1) == 0 && R <= GEMV_ROW_CTA && C >= 512) {  // short and wide: a CTA per row
    const unsigned g = (unsigned)R;
    if (tri == 1) gemv_n_row_kernel<1><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
    else if (tri == 2) gemv_n_row_kernel<2><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
    else gemv_n_row_kernel<0><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
    AFN_LAUNCH_CHECK("gemv_n_row_kernel");
    return AFN_OK;
  }
  if ((C & 1) == 0 && tri == 0) {
    gemv_n2_kernel<<<(unsigned)((R + 15) / 16), VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
    AFN_LAUNCH_CHECK("gemv_n2_kernel");
    return AFN_OK;
  }
  const unsigned g = (unsigned)((R + 7) / 8);
  if (tri == 1) gemv_n_kernel<1><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
  else if (tri == 2) gemv_n_kernel<2><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
  else gemv_n_kernel<0><<<g, VT, 0, st>>>(A, R, C, x, ybase, alpha, y, get_skip());
  AFN_LAUNCH_CHECK("gemv_n_kernel");
  return AFN_OK;
}

int64_t gemv_t_ws(int64_t R, int64_t C) {
  const int64_t rpb = gemv_t_rows_per_block(R);
  return ((R + rpb - 1) / rpb) * C + 1;
}

afn_status gemv_t(const double* A, int64_t R, int64_t C, const double* x, const double* ybase,
                  double alpha, double* y, double* ws, cudaStream_t st) {
  if (C <= 0) return AFN_OK;
  const int64_t rpb = gemv_t_rows_per_block(R);
  const int nb = (int)((R + rpb - 1) / rpb);
  if (nb > 0) {
    gemv_t_partial_kernel<<<nb, VT, sizeof(double) * rpb, st>>>(A, R, C, rpb, x, ws, get_skip());
    AFN_LAUNCH_CHECK("gemv_t_partial_kernel");
  }
  gemv_t_reduce_kernel<<<(unsigned)((C + 31) / 32), 1024, 0, st>>>(ws, nb, C, ybase, alpha, y, get_skip());
  AFN_LAUNCH_CHECK("gemv_t_reduce_kernel");
  return AFN_OK;
}

afn_status spmv_csr(const int64_t* rp, const int32_t* col, const double* val, int64_t N,
                    const double* x, double* y, cudaStream_t st) {
  if (N <= 0) return AFN_OK;
  spmv_kernel<<<(unsigned)((N + 7) / 8), VT, 0, st>>>(rp, col, val, N, x, y, get_skip());
  AFN_LAUNCH_CHECK("spmv_kernel");
  return AFN_OK;
}

afn_status gather_vec(const double* x, const int64_t* perm, int64_t n, double* y, cudaStream_t st) {
  if (n <= 0) return AFN_OK;
  gather_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, perm, n, y);
  AFN_LAUNCH_CHECK("gather_vec_kernel");
  return AFN_OK;
}

afn_status scatter_vec(const double* x, const int64_t* perm, int64_t n, double* y, cudaStream_t st) {
  if (n <= 0) return AFN_OK;
  scatter_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, perm, n, y);
  AFN_LAUNCH_CHECK("scatter_vec_kernel");
  return AFN_OK;
}

int64_t dot_ws() { return DOT_BLOCKS; }

afn_status dot(const double* a, const double* b, Seg2 g, double* out, double* ws, unsigned* cnt,
               cudaStream_t st) {
  dot_kernel<<<DOT_BLOCKS, VT, 0, st>>>(a, b, g, out, ws, cnt);
  AFN_LAUNCH_CHECK("dot_kernel");
  return AFN_OK;
}

afn_status pcg_update_xr(double* x, double* r, const double* p, const double* q, Seg2 g,
                         const double* sc, int rz_slot, double* rr, double* ws, unsigned* cnt,
                         cudaStream_t st) {
  update_xr_kernel<<<DOT_BLOCKS, VT, 0, st>>>(x, r, p, q, g, sc, rz_slot, rr, ws, cnt);
  AFN_LAUNCH_CHECK("update_xr_kernel");
  return AFN_OK;
}

afn_status pcg_update_xr_check(double* x, double* r, const double* p, const double* q, Seg2 g, double* sc,
                               int rz_slot, double* ws, unsigned* cnt, double nb, double tol, int maxit, int fixed,
                               double* hist, cudaStream_t st) {
  update_xr_check_kernel<<<DOT_BLOCKS, VT, 0, st>>>(x, r, p, q, g, sc, rz_slot, ws, cnt, nb, tol, maxit, fixed,
                                                    hist);
  AFN_LAUNCH_CHECK("update_xr_check_kernel");
  return AFN_OK;
}

afn_status pcg_update_p(double* p, const double* z, Seg2 g, const double* sc, int rz_new_slot,
                        int rz_old_slot, cudaStream_t st) {
  if (g.size() <= 0) return AFN_OK;
  update_p_kernel<<<grid_for(g.size(), 256, 1184), 256, 0, st>>>(p, z, g, sc, rz_new_slot, rz_old_slot);
  AFN_LAUNCH_CHECK("update_p_kernel");
  return AFN_OK;
}

afn_status vec_copy(double* y, const double* x, Seg2 g, cudaStream_t st) {
  if (g.size() <= 0) return AFN_OK;
  copy_kernel<<<grid_for(g.size(), 256, 1184), 256, 0, st>>>(y, x, g);
  AFN_LAUNCH_CHECK("copy_kernel");
  return AFN_OK;
}

afn_status vec_axpby(double* y, double a, const double* x, double b, Seg2 g, cudaStream_t st) {
  if (g.size() <= 0) return AFN_OK;
  axpby_kernel<<<grid_for(g.size(), 256, 1184), 256, 0, st>>>(y, a, x, b, g);
  AFN_LAUNCH_CHECK("axpby_kernel");
  return AFN_OK;
}

afn_status vec_scale(double* y, double a, const double* x, Seg2 g, cudaStream_t st) {
  if (g.size() <= 0) return AFN_OK;
  scale_kernel<<<grid_for(g.size(), 256, 1184), 256, 0, st>>>(y, a, x, g);
  AFN_LAUNCH_CHECK("scale_kernel");
  return AFN_OK;
}

afn_status vec_fill(double* y, double v, int64_t n, cudaStream_t st) {
  if (n <= 0) return AFN_OK;
  fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, v, n);
  AFN_LAUNCH_CHECK("fill_kernel");
  return AFN_OK;
}

afn_status vec_scale_rsqrt(double* y, const double* s, int64_t n, cudaStream_t st) {
  if (n <= 0) return AFN_OK;
  scale_rsqrt_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, s, n);
  AFN_LAUNCH_CHECK("scale_rsqrt_kernel");
  return AFN_OK;
}

afn_status add_diag(double* A, int64_t k, double v, cudaStream_t st) {
  if (k <= 0) return AFN_OK;
  add_diag_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(A, k, v);
  AFN_LAUNCH_CHECK("add_diag_kernel");
  return AFN_OK;
}

afn_status combine_slots(const double* part, int R, int stride, unsigned mask, double* sc,
                         cudaStream_t st) {
  combine_slots_kernel<<<1, 32, 0, st>>>(part, R, stride, mask, sc);
  AFN_LAUNCH_CHECK("combine_slots_kernel");
  return AFN_OK;
}

afn_status combine_sub(const double* part, int R, int64_t C, const double* base, double* y,
                       cudaStream_t st) {
  if (C <= 0) return AFN_OK;
  combine_sub_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(part, R, C, base, y);
  AFN_LAUNCH_CHECK("combine_sub_kernel");
  return AFN_OK;
}

}  // namespace afn

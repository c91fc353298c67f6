// abi.cu -- the C ABI of include/afn.h: argument validation, the built handle
// (device-resident L^{-T}, W, G, G^T, permuted points), the build pipeline
// (P:L207-263), the apply and the PCG driver.
#include <atomic>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"

// ---------------------------------------------------------------------------
namespace afn {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void note_launch(int count) { g_launches.fetch_add(count, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

afn_status cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  return e == cudaErrorMemoryAllocation ? AFN_ERR_NOMEM : AFN_ERR_CUDA;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

static void pool_setup_once() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // no hidden cross-stream waits: a block freed on one stream (e.g. the
    // side stream's kNN temporaries) is never handed to another stream's
    // allocation with an inserted dependency on the first stream's work;
    // opportunistic reuse (a block whose free has already completed, on any
    // stream) stays on, so handles built and destroyed on any mix of streams
    // recycle their memory (the pool grew without it)
    int zero = 0, one = 1;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &one);
  }
  done[dev] = true;
}

// Optional caller allocator (afn_set_allocator): every device allocation goes
// through it.  Its frees are deferred until the stream position of the free
// has completed (an event per block), because a caching allocator returns a
// block to its pool at call time, not in stream order.
namespace {
std::mutex g_alloc_mu;
afn_alloc_fn g_alloc = nullptr;
afn_free_fn g_free = nullptr;
void* g_alloc_ctx = nullptr;
std::unordered_map<void*, size_t> g_alloc_size;
struct Deferred {
  void* p;
  size_t bytes;
  cudaStream_t st;
  cudaEvent_t ev;
};
std::vector<Deferred> g_deferred;
// Large blocks (>= 32 MB: W, Z, the FSAI products, the K21 tiles...) are kept
// by the library after their free and handed out again once the free has
// completed on the GPU: a stream-ordered pool allocation that finds no block
// it may reuse (frees still pending on another stream) can block the host
// while the driver reclaims memory -- measured up to 200 ms inside a 100 ms
// C3 build, at random.  Reuse needs no wait and no cross-stream dependency.
constexpr size_t BIG_BLOCK = (size_t)32 << 20;
struct BigBlk {
  void* p;
  size_t bytes;
  cudaEvent_t ev;
  int dev;
};
std::vector<BigBlk> g_big;                          // freed, awaiting reuse
std::unordered_map<void*, std::pair<size_t, int>> g_big_live;  // handed out: size, device
}  // namespace

void release_deferred(bool wait) {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  size_t keep = 0;
  for (size_t i = 0; i < g_deferred.size(); ++i) {
    Deferred& f = g_deferred[i];
    const cudaError_t q = wait ? cudaEventSynchronize(f.ev) : cudaEventQuery(f.ev);
    if (q == cudaErrorNotReady) {
      g_deferred[keep++] = f;
      continue;
    }
    cudaGetLastError();
    cudaEventDestroy(f.ev);
    if (g_free) g_free(f.p, f.bytes, (void*)f.st, g_alloc_ctx);
  }
  g_deferred.resize(keep);
}

afn_status dalloc(void** p, size_t bytes, cudaStream_t st) {
  *p = nullptr;
  size_t nb = bytes > 0 ? bytes : 8;
  {
    std::unique_lock<std::mutex> lk(g_alloc_mu);
    if (g_alloc) {
      lk.unlock();
      release_deferred(false);
      lk.lock();
      *p = g_alloc(nb, (void*)st, g_alloc_ctx);
      if (!*p) {
        set_error("caller allocator returned NULL for %zu bytes", nb);
        return AFN_ERR_NOMEM;
      }
      g_alloc_size[*p] = nb;
      return AFN_OK;
    }
  }
  pool_setup_once();
  int dev = 0;
  cudaGetDevice(&dev);
  if (nb >= BIG_BLOCK) {  // size classes 2^m (1 + j/8): a build's sizes vary a little run to run
    int m = 0;
    while (((size_t)1 << (m + 1)) <= nb) ++m;
    const size_t step = (size_t)1 << (m - 3);
    nb = (nb + step - 1) / step * step;
  }
  if (nb >= BIG_BLOCK) {  // a completed large block of 1 - 1.5x the size
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    int best = -1;
    for (int i = 0; i < (int)g_big.size(); ++i) {
      const BigBlk& b = g_big[i];
      if (b.dev != dev || b.bytes < nb || b.bytes > nb + nb / 2) continue;
      if (best >= 0 && b.bytes >= g_big[best].bytes) continue;
      if (cudaEventQuery(b.ev) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      best = i;
    }
    if (best >= 0) {
      BigBlk b = g_big[best];
      g_big.erase(g_big.begin() + best);
      cudaEventDestroy(b.ev);
      g_big_live[b.p] = {b.bytes, dev};
      *p = b.p;
      return AFN_OK;
    }
  }
  cudaError_t e = cudaMallocAsync(p, nb, st);
  if (e != cudaSuccess && nb >= BIG_BLOCK) {  // cached blocks back to the pool, then retry
    cudaGetLastError();
    trim_big_blocks();
    e = cudaMallocAsync(p, nb, st);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
    return AFN_ERR_NOMEM;
  }
  if (nb >= BIG_BLOCK) {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_big_live[*p] = {nb, dev};
  }
  return AFN_OK;
}

void trim_big_blocks() {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (BigBlk& b : g_big) {
    cudaSetDevice(b.dev);
    cudaEventSynchronize(b.ev);
    cudaEventDestroy(b.ev);
    cudaFree(b.p);  // (pool memory: returns it to the pool)
  }
  g_big.clear();
  cudaSetDevice(cur);
  cudaGetLastError();
}

void dfree(void* p, cudaStream_t st) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_alloc_size.find(p);
    if (it != g_alloc_size.end()) {  // from the caller allocator
      Deferred f{p, it->second, st, nullptr};
      g_alloc_size.erase(it);
      if (cudaEventCreateWithFlags(&f.ev, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(f.ev, st) == cudaSuccess) {
        g_deferred.push_back(f);
      } else {  // (cannot order it: wait for the stream)
        cudaGetLastError();
        if (f.ev) cudaEventDestroy(f.ev);
        cudaStreamSynchronize(st);
        if (g_free) g_free(p, f.bytes, (void*)st, g_alloc_ctx);
      }
      return;
    }
    auto bl = g_big_live.find(p);
    if (bl != g_big_live.end()) {  // kept for reuse once this free completes
      BigBlk b{p, bl->second.first, nullptr, bl->second.second};
      g_big_live.erase(bl);
      if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) == cudaSuccess && cudaEventRecord(b.ev, st) == cudaSuccess) {
        g_big.push_back(b);
        return;
      }
      cudaGetLastError();
      if (b.ev) cudaEventDestroy(b.ev);
    }
  }
  cudaFreeAsync(p, st);
}

// ---- per-kernel timers
namespace {
struct KtPending {
  int id;
  cudaEvent_t e0, e1;
  double work;
};
std::atomic<bool> g_kt_on{false};
std::vector<KtPending> g_kt_pending;
std::vector<cudaEvent_t> g_kt_pool;
double g_kt_ms[KT_N] = {0};
double g_kt_work[KT_N] = {0};
int64_t g_kt_cnt[KT_N] = {0};
cudaEvent_t g_kt_open[KT_N];
cudaEvent_t kt_event() {
  if (!g_kt_pool.empty()) {
    cudaEvent_t e = g_kt_pool.back();
    g_kt_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool kt_enabled() { return g_kt_on.load(); }
void kt_begin(int id, cudaStream_t st) {
  if (!kt_enabled()) return;
  g_kt_open[id] = kt_event();
  cudaEventRecord(g_kt_open[id], st);
}
void kt_end(int id, cudaStream_t st, double work) {
  if (!kt_enabled()) return;
  cudaEvent_t e1 = kt_event();
  cudaEventRecord(e1, st);
  g_kt_pending.push_back({id, g_kt_open[id], e1, work});
}
// add a timing measured elsewhere (events of a replayed CUDA graph)
void kt_add(int id, double ms, double work) {
  if (!kt_enabled()) return;
  g_kt_ms[id] += ms;
  g_kt_work[id] += work;
  g_kt_cnt[id] += 1;
}
// forget the last `count` pending timings of `id` (launches that were queued
// but skipped on the device)
void kt_drop_last(int id, int count) {
  for (int64_t j = (int64_t)g_kt_pending.size() - 1; j >= 0 && count > 0; --j) {
    if (g_kt_pending[j].id != id) continue;
    g_kt_pool.push_back(g_kt_pending[j].e0);
    g_kt_pool.push_back(g_kt_pending[j].e1);
    g_kt_pending.erase(g_kt_pending.begin() + j);
    --count;
  }
}
void kt_collect() {
  for (auto& p : g_kt_pending) {
    cudaEventSynchronize(p.e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.e0, p.e1);
    g_kt_ms[p.id] += ms;
    g_kt_work[p.id] += p.work;
    g_kt_cnt[p.id] += 1;
    g_kt_pool.push_back(p.e0);
    g_kt_pool.push_back(p.e1);
  }
  g_kt_pending.clear();
}

namespace {

bool is_dev(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

#define REQ(cond, ...)             \
  do {                             \
    if (!(cond)) {                 \
      set_error(__VA_ARGS__);      \
      return AFN_ERR_ARG;          \
    }                              \
  } while (0)

#define TRY(x)                     \
  do {                             \
    afn_status s_ = (x);           \
    if (s_ != AFN_OK) return s_;   \
  } while (0)

// RAII list of stream-ordered temporaries
struct Temps {
  cudaStream_t st;
  std::vector<void*> ps;
  explicit Temps(cudaStream_t s) : st(s) {}
  ~Temps() {
    for (void* p : ps) dfree(p, st);
  }
  template <class T>
  afn_status get(T** out, size_t count) {
    void* p = nullptr;
    afn_status s = dalloc(&p, sizeof(T) * (count > 0 ? count : 1), st);
    if (s != AFN_OK) return s;
    ps.push_back(p);
    *out = static_cast<T*>(p);
    return AFN_OK;
  }
};

// perm = [idx(0..k); unselected ids ascending].  Internal consistency checks
// (cheap): landmark ids in range and distinct, pattern columns below the row.
__global__ void mark_kernel(const int64_t* __restrict__ idx, int64_t k, int64_t n,
                            unsigned* __restrict__ flag32, int* __restrict__ err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int64_t i = idx[t];
  if (i < 0 || i >= n) { atomicOr(err, 1); return; }
  if (atomicAdd(&flag32[i], 1u) != 0u) atomicOr(err, 2);
}
__global__ void flag8_kernel(const unsigned* __restrict__ flag32, int64_t n, unsigned char* __restrict__ flag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) flag[t] = flag32[t] ? 1 : 0;
}
__global__ void check_pattern_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                     int64_t N, int* __restrict__ err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const int64_t b = rp[r], e = rp[r + 1];
  if (e <= b || col[e - 1] != r) { atomicOr(err, 4); return; }
  for (int64_t t = b; t + 1 < e; ++t)
    if (col[t] < 0 || col[t] >= col[t + 1]) { atomicOr(err, 8); return; }
}
__global__ void perm_kernel(const unsigned char* __restrict__ flag, const int64_t* __restrict__ idx,
                            int64_t n, int64_t k, int64_t* __restrict__ perm) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = tid * per, e = min(n, b + per);
  int64_t c = 0;
  for (int64_t i = b; i < e; ++i) c += flag[i] ? 0 : 1;
  part[tid] = c;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int64_t v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int64_t pos = k + (tid > 0 ? part[tid - 1] : 0);
  for (int64_t i = b; i < e; ++i)
    if (!flag[i]) perm[pos++] = i;
  for (int64_t t = tid; t < k; t += 1024) perm[t] = idx[t];
}

}  // namespace
}  // namespace afn

using namespace afn;

// ---------------------------------------------------------------------------
// The built handle.  One RankSt per logical rank this process drives (one on
// a single GPU or with NCCL; R with an emulated communicator).  Replicated
// pieces (permuted points, L, L^{-T}, the pattern, G, G^T) are held by every
// rank; W holds the rank's own non-landmark rows; the PCG vectors are full
// length with only the rank's own rows (RankSt::own) computed locally.
#define AFN_NYS_NU 1e-10  // K11 shift of the Nystrom branch (reading R30)
struct RankSt {
  int rank = 0;
  Seg2 own{};
  int64_t lo = 0, hi = 0;  // own non-landmark rows, numbered 0..N2
  int64_t* perm = nullptr;
  double* fill = nullptr;
  double* Xp = nullptr;     // permuted points n x d
  double* Xs = nullptr;     // prescaled permuted points (kmv)
  double* L = nullptr;      // k x k lower (row-major)
  double* LinvT = nullptr;  // k x k, L^{-T}
  double* Linv = nullptr;   // k x k, L^{-1} (AFN apply: t = L^{-1} r1 as a row-major GEMV)
  double* W = nullptr;      // own rows (hi - lo) x k of W = K21 L^{-T}
  int64_t* rp = nullptr;
  int32_t* col = nullptr;
  double* gval = nullptr;
  int64_t* trp = nullptr;
  int32_t* tcol = nullptr;
  double* tval = nullptr;
  int* derr = nullptr;
  int* dinfo = nullptr;
  // workspaces
  KmvPlan plan{};
  double* kmv_part = nullptr;
  double* qpart = nullptr;  // R x n rank partials of the symmetric matvec (R > 1)
  double* gws = nullptr;    // gemv_t partials
  double* tvec = nullptr;   // k
  double* vvec = nullptr;   // k
  double* kpart = nullptr;  // R x k partials of W^T s2
  double* uvec = nullptr;   // N2
  double* yvec = nullptr;   // N2
  double* rbuf = nullptr;   // n (public apply)
  double* zbuf = nullptr;   // n
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;  // n
  double* sc = nullptr;      // SC_N combined scalars
  double* scpart = nullptr;  // R x SC_N per-rank partials
  double* dws = nullptr;
  unsigned* dcnt = nullptr;
  // Nystrom branch (AFN_METHOD_NYSTROM): F = K(X_own, X_k) L0^{-T} (own rows,
  // local order), RinvT = R^{-T} with R R^T = mu I + F^T F
  double* F = nullptr;
  double* RinvT = nullptr;
  // one rank, cutoff W: the K21 tiles of the W plan, kept for the apply
  // (W t = K21 (L^{-T} t), W^T s = L^{-1} (K21^T s): DESIGN.md 6.6)
  WCutPlan kt;
  // RAN (AFN_METHOD_RAN): R1invT = R1^{-T}, R1 R1^T = F^T F + nu I
  double* R1invT = nullptr;
  std::vector<void*> allocs;
};

struct afn_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;  // the build stream (frees are queued on it)
  int64_t n = 0, k = 0, N2 = 0, nnz = 0;
  int d = 0;
  double l = 0, mu = 0;
  Kern kn{};
  int method = AFN_METHOD_AFN;  // the preconditioner built (AFN, NYSTROM, FSAI or RAN)
  double lam_k = 0.0;           // RAN: k-th largest eigenvalue of K_nys
  afn_params params{};
  Alg1Result a1{};
  const Comm* comm = nullptr;  // not owned; null = single GPU
  int R = 1;
  std::vector<RankSt> rk;
  double ms[8] = {0};
};

namespace {

// non-blocking side stream per device and host thread (Alg. 1 runs on it
// concurrently with FPS)
cudaStream_t side_stream() {
  static thread_local cudaStream_t ss[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!ss[dev]) cudaStreamCreateWithFlags(&ss[dev], cudaStreamNonBlocking);
  return ss[dev];
}

// high-priority non-blocking stream per device and host thread (the K11
// factorization beside the kNN pattern)
cudaStream_t hp_stream() {
  static thread_local cudaStream_t hs[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!hs[dev]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&hs[dev], cudaStreamNonBlocking, hi);
  }
  return hs[dev];
}

// non-blocking stream per device and host thread for PCG graph capture / replay
cudaStream_t graph_stream() {
  static thread_local cudaStream_t gs[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!gs[dev]) cudaStreamCreateWithFlags(&gs[dev], cudaStreamNonBlocking);
  return gs[dev];
}

// two pinned int64 per host thread (FPS early-stop value)
int64_t* pinned_i64() {
  static thread_local int64_t* buf = nullptr;
  if (!buf && cudaMallocHost((void**)&buf, sizeof(int64_t) * 2) != cudaSuccess) {
    cudaGetLastError();
    buf = nullptr;
  }
  return buf;
}

// one small pinned buffer per host thread (PCG scalars), allocated once
double* pinned_scalars() {
  static thread_local double* buf = nullptr;
  if (!buf) {
    if (cudaMallocHost((void**)&buf, sizeof(double) * 64) != cudaSuccess) {
      cudaGetLastError();
      buf = nullptr;
    }
  }
  return buf;
}

template <class T>
afn_status ralloc(RankSt& s, T** p, size_t count, cudaStream_t st) {
  void* v = nullptr;
  afn_status e = dalloc(&v, sizeof(T) * (count > 0 ? count : 1), st);
  if (e == AFN_OK) {
    s.allocs.push_back(v);
    *p = static_cast<T*>(v);
  }
  return e;
}

void rfree(RankSt& s, void* p, cudaStream_t st) {
  for (auto it = s.allocs.begin(); it != s.allocs.end(); ++it)
    if (*it == p) {
      s.allocs.erase(it);
      break;
    }
  dfree(p, st);
}

void handle_free(afn_handle h) {
  if (!h) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  // every stream that may still use the handle's memory (the build stream, its
  // side streams, the caller's solve streams) is drained first; the blocks then
  // go back to the pool on the build stream (cudaFree would unmap them and
  // force the next build to map fresh pages) and are reusable from any stream
  cudaDeviceSynchronize();
  for (auto& s : h->rk) {
    s.kt.st = h->stream;
    w_cut_free(&s.kt);
    for (void* p : s.allocs) dfree(p, h->stream);
  }
  cudaStreamSynchronize(h->stream);
  release_deferred(true);
  cudaSetDevice(cur);
  delete h;
}

// closed-form kNN row pointer (knn.cu): sum_{t<i} min(w, t+1)
int64_t rowptr_at(int64_t i, int w) {
  const int64_t wl = w;
  return (i < wl) ? i * (i + 1) / 2 : wl * (wl + 1) / 2 + (i - wl) * wl;
}

// ---- exchanges (all-gather of each rank's owned byte ranges) -------------
template <class F, class G>
afn_status exchange(afn_handle h, F buf_of, G ranges_of, cudaStream_t st) {
  if (h->R <= 1) return AFN_OK;
  std::vector<char*> bufs;
  for (auto& s : h->rk) bufs.push_back(reinterpret_cast<char*>(buf_of(s)));
  std::vector<RankRanges> owned(h->R);
  for (int s = 0; s < h->R; ++s) owned[s] = ranges_of(s);
  return comm_allgatherv(h->comm, bufs.data(), owned, st);
}

// a full-length (n) double vector: each rank's own rows
RankRanges vec_ranges(afn_handle h, int s) {
  const Seg2 g = shard_rows(h->n, h->k, h->R, s);
  return {{8 * (size_t)g.a0, 8 * (size_t)g.na}, {8 * (size_t)g.b0, 8 * (size_t)g.nb}};
}
// the landmark block [0, k) of a full-length vector
RankRanges landmark_ranges(afn_handle h, int s) {
  const Seg2 g = shard_rows(h->n, h->k, h->R, s);
  return {{8 * (size_t)g.a0, 8 * (size_t)g.na}};
}
// an N2-vector (non-landmark numbering), `width` bytes per row
RankRanges rows2_ranges(afn_handle h, int s, size_t width) {
  const Seg2 g = shard_rows(h->n, h->k, h->R, s);
  const size_t lo = (size_t)(g.b0 - h->k);
  return {{width * lo, width * (size_t)g.nb}};
}
// pattern-aligned arrays (col / gval) of the rank's rows, `width` bytes per nonzero
RankRanges nnz_ranges(afn_handle h, int s, size_t width) {
  const Seg2 g = shard_rows(h->n, h->k, h->R, s);
  const int64_t lo = g.b0 - h->k, hi = lo + g.nb;
  const int64_t e0 = rowptr_at(lo, h->params.w), e1 = rowptr_at(hi, h->params.w);
  return {{width * (size_t)e0, width * (size_t)(e1 - e0)}};
}

// destination of a rank's partial of scalar `slot`
double* part_dst(afn_handle h, RankSt& s, int slot) {
  return h->R == 1 ? s.sc + slot : s.scpart + (size_t)s.rank * SC_N + slot;
}
// sum the partials of the slots in `mask` over the ranks (rank order)
afn_status reduce_slots(afn_handle h, unsigned mask, cudaStream_t st) {
  if (h->R == 1) return AFN_OK;
  TRY(exchange(h, [](RankSt& s) { return s.scpart; },
               [&](int s) { return RankRanges{{8 * (size_t)s * SC_N, 8 * (size_t)SC_N}}; }, st));
  for (auto& s : h->rk) TRY(combine_slots(s.scpart, h->R, SC_N, mask, s.sc, st));
  return AFN_OK;
}

// executed FP64 flops of one rank's kernel matvec launch (kmv.cu kmv_flops:
// per useful pair, the symmetric plan's units split evenly over the ranks)
double kmv_work(afn_handle h, int64_t n, int d) {
  const RankSt& s = h->rk[0];
  const double f = kmv_flops(s.plan, n, s.own.size(), d, h->kn.kind);
  return s.plan.sym ? f / h->R : f;
}

// q = (K + mu I) v on every local rank's own rows.  One rank with
// the symmetric plan: one launch (+ v.q into sc[pq_slot]); R > 1 with the
// symmetric plan: each rank's share of the pair units, an all-gather of the
// rank partials, the rank-order combine (+ v.q partials); row-wise plan: the
// rank's rows.  pq_slot < 0: no dot.
template <class VF, class QF>
afn_status matvec_perm(afn_handle h, VF v_of, QF q_of, int pq_slot, cudaStream_t st) {
  const int64_t n = h->n;
  const int d = h->d;
  const bool sym = h->rk[0].plan.sym;
  if (sym && h->R == 1) {
    RankSt& s = h->rk[0];
    return kmv_launch(s.Xs, n, d, h->kn.kind, v_of(s), h->mu, s.own, q_of(s), true, s.kmv_part, s.plan, st,
                      pq_slot >= 0 ? s.sc + pq_slot : nullptr, s.dws, s.dcnt);
  }
  if (sym) {
    for (auto& s : h->rk)
      TRY(kmv_sym_rank_partial(s.Xs, n, d, h->kn.kind, v_of(s), s.plan, s.kmv_part, s.qpart + (size_t)s.rank * n,
                               st));
    TRY(exchange(h, [](RankSt& s) { return s.qpart; },
                 [&](int r) { return RankRanges{{8 * (size_t)r * n, 8 * (size_t)n}}; }, st));
    for (auto& s : h->rk)
      TRY(kmv_sym_combine(s.qpart, h->R, n, s.own, v_of(s), h->mu, q_of(s), st,
                          pq_slot >= 0 ? part_dst(h, s, pq_slot) : nullptr, s.dws, s.dcnt));
    return AFN_OK;
  }
  for (auto& s : h->rk) {
    TRY(kmv_launch(s.Xs, n, d, h->kn.kind, v_of(s), h->mu, s.own, q_of(s), true, s.kmv_part, s.plan, st));
    if (pq_slot >= 0) TRY(dot(v_of(s), q_of(s), s.own, part_dst(h, s, pq_slot), s.dws, s.dcnt, st));
  }
  return AFN_OK;
}

// algorithmic HBM bytes of one apply: W read twice, L^{-T} twice (upper half),
// G and G^T (values + 4-byte columns) once each, plus the vectors
double apply_bytes(afn_handle h) {
  const double k = (double)h->k, N2 = (double)h->N2, nnz = (double)h->nnz;
  if (h->R == 1 && h->rk[0].kt.used)  // the K21 tiles twice, four triangles (L^{-1}, L^{-T} twice each)
    return 8.0 * (2.0 * (double)h->rk[0].kt.Adbl + 2.0 * k * (k + 1.0)) + 2.0 * 12.0 * nnz +
           8.0 * (6.0 * N2 + 10.0 * k);
  return 8.0 * (2.0 * N2 * k + k * (k + 1.0)) + 2.0 * 12.0 * nnz + 8.0 * (6.0 * N2 + 6.0 * k);
}

// z = M^{-1} r in the permuted order (V-form):
//   t = L^{-1} r1;  u = r2 - W t;  y = G u;  s2 = G^T y;  s1 = L^{-T} (t - W^T s2).
// r: the rank's own rows valid (landmark rows are all-gathered here); z: the
// rank's own rows are written (s1 in full).
template <class RF, class ZF>
afn_status apply_afn_perm(afn_handle h, RF r_of, ZF z_of, cudaStream_t st) {
  const int64_t k = h->k, N2 = h->N2;
  const int R = h->R;
  // t = L^{-1} r1 needs all of r1
  TRY(exchange(h, r_of, [&](int s) { return landmark_ranges(h, s); }, st));
  for (auto& s : h->rk) {
    const double* r = r_of(s);
    TRY(gemv_n(s.Linv, k, k, r, nullptr, 1.0, s.tvec, st, 2));
    // u = r2 - W t (own rows); one rank with the K21 tiles: r2 - K21 (L^{-T} t)
    if (s.kt.used) {
      TRY(gemv_n(s.LinvT, k, k, s.tvec, nullptr, 1.0, s.kpart, st, 1));
      TRY(w_cut_apply_n(&s.kt, s.kpart, r + k, s.uvec, st));
    } else if (s.hi > s.lo) {
      TRY(gemv_n(s.W, s.hi - s.lo, k, s.tvec, r + k + s.lo, -1.0, s.uvec + s.lo, st));
    }
  }
  if (N2 > 0) {
    TRY(exchange(h, [](RankSt& s) { return s.uvec; }, [&](int s) { return rows2_ranges(h, s, 8); }, st));
    for (auto& s : h->rk)  // y = G u (own rows)
      TRY(spmv_csr(s.rp + s.lo, s.col, s.gval, s.hi - s.lo, s.uvec, s.yvec + s.lo, st));
    TRY(exchange(h, [](RankSt& s) { return s.yvec; }, [&](int s) { return rows2_ranges(h, s, 8); }, st));
    for (auto& s : h->rk) {
      double* z = z_of(s);
      // s2 = G^T y (own rows of G^T)
      TRY(spmv_csr(s.trp + s.lo, s.tcol, s.tval, s.hi - s.lo, s.yvec, z + k + s.lo, st));
      if (R == 1 && s.kt.used) {  // v = t - L^{-1} (K21^T s2)
        TRY(w_cut_apply_t(&s.kt, z + k, s.kpart, st));
        TRY(gemv_n(s.Linv, k, k, s.kpart, s.tvec, -1.0, s.vvec, st, 2));
      } else if (R == 1) {  // v = t - W^T s2
        TRY(gemv_t(s.W, N2, k, z + k, s.tvec, -1.0, s.vvec, s.gws, st));
      } else {       // rank partial of W^T s2
        double* kp = s.kpart + (size_t)s.rank * k;
        if (s.hi > s.lo) TRY(gemv_t(s.W, s.hi - s.lo, k, z + k + s.lo, nullptr, 1.0, kp, s.gws, st));
        else AFN_CUDA(cudaMemsetAsync(kp, 0, sizeof(double) * k, st));
      }
    }
    if (R > 1) {
      TRY(exchange(h, [](RankSt& s) { return s.kpart; },
                   [&](int s) { return RankRanges{{8 * (size_t)s * k, 8 * (size_t)k}}; }, st));
      for (auto& s : h->rk) TRY(combine_sub(s.kpart, R, k, s.tvec, s.vvec, st));
    }
    for (auto& s : h->rk) TRY(gemv_n(s.LinvT, k, k, s.vvec, nullptr, 1.0, z_of(s), st, 1));  // s1
  } else {
    for (auto& s : h->rk) TRY(gemv_n(s.LinvT, k, k, s.tvec, nullptr, 1.0, z_of(s), st, 1));
  }
  return AFN_OK;
}

// z = (K_nys + mu I)^{-1} r with K_nys = F F^T, F = K_{X,X_k} L0^{-T}:
//   SMW  (F F^T + mu I)^{-1} = (I - F (mu I + F^T F)^{-1} F^T) / mu,
//   t = F^T r (rank partials), u = R^{-1} t, v = R^{-T} u, z = (r - F v) / mu.
template <class RF, class ZF>
afn_status apply_nystrom_perm(afn_handle h, RF r_of, ZF z_of, cudaStream_t st) {
  const int64_t k = h->k;
  const int R = h->R;
  for (auto& s : h->rk) {
    const double* r = r_of(s);
    double* tdst = R == 1 ? s.tvec : s.kpart + (size_t)s.rank * k;
    const Seg2 g = s.own;
    if (g.na + g.nb == 0) {
      AFN_CUDA(cudaMemsetAsync(tdst, 0, sizeof(double) * k, st));
    } else if (g.a0 + g.na == g.b0 || g.nb == 0) {  // contiguous rows
      TRY(gemv_t(s.F, g.na + g.nb, k, r + g.a0, nullptr, 1.0, tdst, s.gws, st));
    } else if (g.na == 0) {
      TRY(gemv_t(s.F, g.nb, k, r + g.b0, nullptr, 1.0, tdst, s.gws, st));
    } else {
      TRY(gemv_t(s.F, g.na, k, r + g.a0, nullptr, 1.0, s.vvec, s.gws, st));
      TRY(gemv_t(s.F + (size_t)g.na * k, g.nb, k, r + g.b0, s.vvec, 1.0, tdst, s.gws, st));
    }
  }
  if (R > 1) {
    TRY(exchange(h, [](RankSt& s) { return s.kpart; },
                 [&](int s) { return RankRanges{{8 * (size_t)s * k, 8 * (size_t)k}}; }, st));
    for (auto& s : h->rk) TRY(combine_sub(s.kpart, R, k, nullptr, s.tvec, st));  // t = sum (negated below)
  }
  const double alpha_t = R > 1 ? -1.0 : 1.0;  // combine_sub stores -sum
  for (auto& s : h->rk) {
    const double* r = r_of(s);
    double* z = z_of(s);
    TRY(gemv_t(s.RinvT, k, k, s.tvec, nullptr, alpha_t, s.uvec, s.gws, st));  // u = R^{-1} t
    TRY(gemv_n(s.RinvT, k, k, s.uvec, nullptr, -1.0 / h->mu, s.vvec, st));   // v = -R^{-T} u / mu
    const Seg2 g = s.own;
    // z = r / mu - F (R^{-T} u) / mu  (own rows)
    if (g.na > 0) TRY(gemv_n(s.F, g.na, k, s.vvec, nullptr, 1.0, z + g.a0, st));
    if (g.nb > 0) TRY(gemv_n(s.F + (size_t)g.na * k, g.nb, k, s.vvec, nullptr, 1.0, z + g.b0, st));
    TRY(vec_axpby(z, 1.0 / h->mu, r, 1.0, g, st));
  }
  return AFN_OK;
}

// RAN: z = (lam_k + mu) U (Lam + mu I)^{-1} U^T r + (I - U U^T) r with
// K_nys = U Lam U^T = F F^T, i.e. with G = F^T F:
//   z = r + F ((lam_k + mu) (G + mu I)^{-1} G^{-1} - G^{-1}) F^T r.
template <class RF, class ZF>
afn_status apply_ran_perm(afn_handle h, RF r_of, ZF z_of, cudaStream_t st) {
  const int64_t k = h->k;
  const int R = h->R;
  for (auto& s : h->rk) {  // t = F^T r (own rows)
    const double* r = r_of(s);
    double* tdst = R == 1 ? s.tvec : s.kpart + (size_t)s.rank * k;
    const Seg2 g = s.own;
    if (g.size() == 0) {
      AFN_CUDA(cudaMemsetAsync(tdst, 0, sizeof(double) * k, st));
    } else if (g.a0 + g.na == g.b0 || g.nb == 0) {
      TRY(gemv_t(s.F, g.size(), k, r + g.a0, nullptr, 1.0, tdst, s.gws, st));
    } else if (g.na == 0) {
      TRY(gemv_t(s.F, g.nb, k, r + g.b0, nullptr, 1.0, tdst, s.gws, st));
    } else {
      TRY(gemv_t(s.F, g.na, k, r + g.a0, nullptr, 1.0, s.vvec, s.gws, st));
      TRY(gemv_t(s.F + (size_t)g.na * k, g.nb, k, r + g.b0, s.vvec, 1.0, tdst, s.gws, st));
    }
  }
  if (R > 1) {
    TRY(exchange(h, [](RankSt& s) { return s.kpart; },
                 [&](int s) { return RankRanges{{8 * (size_t)s * k, 8 * (size_t)k}}; }, st));
    for (auto& s : h->rk) {
      TRY(combine_sub(s.kpart, R, k, nullptr, s.tvec, st));
      TRY(vec_scale(s.tvec, -1.0, s.tvec, seg_range(0, k), st));
    }
  }
  for (auto& s : h->rk) {
    const double* r = r_of(s);
    double* z = z_of(s);
    // a = G^{-1} t ; b = (G + mu I)^{-1} a ; w = (lam_k + mu) b - a
    TRY(gemv_t(s.R1invT, k, k, s.tvec, nullptr, 1.0, s.uvec, s.gws, st));
    TRY(gemv_n(s.R1invT, k, k, s.uvec, nullptr, 1.0, s.vvec, st));  // a (vvec)
    TRY(gemv_t(s.RinvT, k, k, s.vvec, nullptr, 1.0, s.uvec, s.gws, st));
    TRY(gemv_n(s.RinvT, k, k, s.uvec, nullptr, h->lam_k + h->mu, s.tvec, st));  // (lam_k+mu) b
    TRY(vec_axpby(s.tvec, -1.0, s.vvec, 1.0, seg_range(0, k), st));              // w (tvec)
    const Seg2 g = s.own;
    if (g.na > 0) TRY(gemv_n(s.F, g.na, k, s.tvec, nullptr, 1.0, z + g.a0, st));
    if (g.nb > 0) TRY(gemv_n(s.F + (size_t)g.na * k, g.nb, k, s.tvec, nullptr, 1.0, z + g.b0, st));
    TRY(vec_axpby(z, 1.0, r, 1.0, g, st));  // z = F w + r
  }
  return AFN_OK;
}

template <class RF, class ZF>
afn_status apply_perm(afn_handle h, RF r_of, ZF z_of, cudaStream_t st) {
  if (h->method == AFN_METHOD_NONE) {  // M = I: unpreconditioned CG
    for (auto& s : h->rk) TRY(vec_copy(z_of(s), r_of(s), s.own, st));
    return AFN_OK;
  }
  if (h->method == AFN_METHOD_NYSTROM) return apply_nystrom_perm(h, r_of, z_of, st);
  if (h->method == AFN_METHOD_RAN) return apply_ran_perm(h, r_of, z_of, st);
  return apply_afn_perm(h, r_of, z_of, st);
}

afn_status validate_X(const double* X, int64_t n, int32_t d) {
  REQ(n >= 1, "n must be >= 1 (got %lld)", (long long)n);
  REQ(d >= 1 && d <= 16, "d must be in 1..16 (got %d)", d);
  REQ(is_dev(X), "X must be a device pointer");
  return AFN_OK;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// reusable event pairs for per-phase timing inside a solve
struct EvPairs {
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  ~EvPairs() {
    for (auto e : pool) cudaEventDestroy(e);
  }
  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  double total_ms() {  // pairs (0,1), (2,3), ...
    double t = 0;
    for (size_t i = 0; i + 1 < used; i += 2) t += ev_ms(pool[i], pool[i + 1]);
    return t;
  }
};

// Nystrom branch: F = K(X_own, X_k) L0^{-T} with L0 L0^T = K11 +
// nu I (already in s.L / s.LinvT), Gram F^T F summed over the ranks, then
// R R^T = mu I + F^T F and R^{-T}.
afn_status build_nystrom(afn_handle h, cudaStream_t st) {
  const int64_t k = h->k;
  const int d = h->d;
  const int R = h->R;
  std::vector<double*> Gm(h->rk.size()), Gp(h->rk.size());
  for (size_t q = 0; q < h->rk.size(); ++q) {
    RankSt& s = h->rk[q];
    const Seg2 g = s.own;
    TRY(ralloc(s, &s.F, (size_t)std::max<int64_t>(1, g.size()) * k, st));
    if (g.na > 0) TRY(w_gemm(s.LinvT, k, s.Xp, s.Xp + g.a0 * d, g.na, d, h->kn, s.F, st));
    if (g.nb > 0) TRY(w_gemm(s.LinvT, k, s.Xp, s.Xp + g.b0 * d, g.nb, d, h->kn, s.F + (size_t)g.na * k, st));
    TRY(ralloc(s, &Gm[q], (size_t)k * k, st));
    TRY(ralloc(s, &Gp[q], (size_t)R * k * k, st));
    double* dst = R == 1 ? Gm[q] : Gp[q] + (size_t)s.rank * k * k;
    if (g.size() > 0) TRY(syrk_ata(s.F, g.size(), k, dst, st));
    else AFN_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * k * k, st));
  }
  if (R > 1) {
    size_t q = 0;
    TRY(exchange(h, [&](RankSt&) { return Gp[q++]; },
                 [&](int s) { return RankRanges{{8 * (size_t)s * k * k, 8 * (size_t)k * k}}; }, st));
    for (size_t q2 = 0; q2 < h->rk.size(); ++q2) {
      TRY(combine_sub(Gp[q2], R, k * k, nullptr, Gm[q2], st));  // -sum, rank order
      TRY(vec_scale(Gm[q2], -1.0, Gm[q2], seg_range(0, k * k), st));
    }
  }
  if (h->method == AFN_METHOD_RAN) {
    // G^{-1} (G + nu I = R1 R1^T) and lambda_k = lambda_min(G) (the nonzero
    // eigenvalues of K_nys = F F^T are those of G = F^T F): power iteration
    // on G^{-1} = R1^{-T} R1^{-1}, then the Rayleigh quotient of G
    for (size_t q = 0; q < h->rk.size(); ++q) {
      RankSt& s = h->rk[q];
      double* G1;
      TRY(ralloc(s, &G1, (size_t)k * k, st));
      AFN_CUDA(cudaMemcpyAsync(G1, Gm[q], sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
      TRY(add_diag(G1, k, AFN_NYS_NU, st));
      TRY(potrf_lower(G1, k, s.dinfo + 1, st));
      TRY(ralloc(s, &s.R1invT, (size_t)k * k, st));
      TRY(trsm_linvt(G1, k, s.R1invT, st));
      rfree(s, G1, st);
      double *v, *y, *sc2, *gw, *dw;
      unsigned* dc;
      TRY(ralloc(s, &v, (size_t)k, st));
      TRY(ralloc(s, &y, (size_t)k, st));
      TRY(ralloc(s, &sc2, 4, st));
      TRY(ralloc(s, &gw, (size_t)gemv_t_ws(k, k), st));
      TRY(ralloc(s, &dw, (size_t)dot_ws(), st));
      TRY(ralloc(s, &dc, 4, st));
      AFN_CUDA(cudaMemsetAsync(dc, 0, sizeof(unsigned) * 4, st));
      TRY(vec_fill(v, 1.0, k, st));
      const int iters = 400;
      for (int it = 0; it < iters; ++it) {
        TRY(gemv_t(s.R1invT, k, k, v, nullptr, 1.0, y, gw, st));  // y = R1^{-1} v
        TRY(gemv_n(s.R1invT, k, k, y, nullptr, 1.0, v, st));      // v = R1^{-T} y
        TRY(dot(v, v, seg_range(0, k), sc2, dw, dc, st));
        TRY(vec_scale_rsqrt(v, sc2, k, st));                      // v /= ||v||
      }
      TRY(gemv_n(Gm[q], k, k, v, nullptr, 1.0, y, st));
      TRY(dot(v, y, seg_range(0, k), sc2 + 1, dw, dc, st));
      double hv[2];
      AFN_CUDA(cudaMemcpyAsync(hv, sc2, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
      AFN_CUDA(cudaStreamSynchronize(st));
      h->lam_k = hv[1];  // v has unit norm
      for (void* t : {(void*)v, (void*)y, (void*)sc2, (void*)gw, (void*)dw, (void*)dc}) rfree(s, t, st);
    }
  }
  for (size_t q = 0; q < h->rk.size(); ++q) {
    RankSt& s = h->rk[q];
    TRY(add_diag(Gm[q], k, h->mu, st));
    TRY(potrf_lower(Gm[q], k, s.dinfo + 1, st));
    TRY(ralloc(s, &s.RinvT, (size_t)k * k, st));
    TRY(trsm_linvt(Gm[q], k, s.RinvT, st));
    rfree(s, Gm[q], st);
    rfree(s, Gp[q], st);
  }
  return AFN_OK;
}

afn_status build_impl(const Comm* comm, const double* X, int64_t n, int32_t d, const afn_params* prm,
                      void* stream, afn_handle* out) {
  REQ(out != nullptr, "out must be non-null");
  *out = nullptr;
  TRY(validate_X(X, n, d));
  REQ(prm != nullptr, "params must be non-null");
  const afn_params P = *prm;
  REQ(P.l > 0 && std::isfinite(P.l), "l must be > 0");
  REQ(P.mu > 0 && std::isfinite(P.mu), "mu must be > 0");
  REQ(P.method >= AFN_METHOD_AFN && P.method <= AFN_METHOD_NONE, "unknown method %d", P.method);
  REQ(P.k_cap >= 1 || P.method == AFN_METHOD_FSAI || P.method == AFN_METHOD_NONE, "k_cap must be >= 1");
  REQ(P.w >= 1 && P.w <= AFN_W_MAX, "w must be in 1..%d", AFN_W_MAX);
  REQ(P.fps_seed >= 0 && P.fps_seed < n, "need 0 <= fps_seed < n");
  REQ(n <= 0x7fffffffLL, "n must fit int32 indices");
  REQ(P.kernel == AFN_KERNEL_GAUSSIAN || P.kernel == AFN_KERNEL_MATERN32, "unknown kernel %d", P.kernel);
  REQ(P.landmarks == AFN_LANDMARKS_FPS || P.landmarks == AFN_LANDMARKS_UNIFORM, "unknown landmarks %d",
      P.landmarks);
  REQ(P.method != AFN_METHOD_ALG2 || P.k_adaptive, "AFN_METHOD_ALG2 needs k_adaptive = 1");
  REQ(P.ordering == AFN_ORDER_INDEX || P.ordering == AFN_ORDER_MAXMIN, "unknown ordering %d", P.ordering);
  REQ(P.ordering == AFN_ORDER_INDEX || P.landmarks == AFN_LANDMARKS_FPS,
      "the MaxMin ordering continues FPS: it needs FPS landmarks");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  AFN_CUDA(cudaGetDevice(&dev));

  cudaEvent_t ev[10];
  for (auto& e : ev) AFN_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 10; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};

  afn_handle h = new afn_handle_s();
  h->device = dev;
  h->stream = st;
  h->n = n;
  h->d = d;
  h->l = P.l;
  h->mu = P.mu;
  h->kn = Kern{P.kernel, P.l};
  h->params = P;
  h->comm = (comm && comm->R > 1) ? comm : nullptr;
  h->R = h->comm ? comm->R : 1;
  const int nlocal = h->comm ? comm->nlocal : 1;
  const int rank0 = h->comm ? comm->rank0 : 0;
  h->rk.resize(nlocal);
  for (int q = 0; q < nlocal; ++q) h->rk[q].rank = rank0 + q;
  struct HGuard {
    afn_handle* hp;
    ~HGuard() {
      if (*hp) handle_free(*hp);
    }
  } hg{&h};

  AFN_CUDA(cudaEventRecord(ev[0], st));
  // ---- a2: adaptive k (Alg. 1) -- replicated: every rank computes the same k
  const Kern kn = h->kn;
  int64_t k = std::min<int64_t>(P.k_cap, n);
  const int kthr = P.k_threshold > 0 ? P.k_threshold : 2000;
  h->method = P.method == AFN_METHOD_NYSTROM ? AFN_METHOD_NYSTROM
              : P.method == AFN_METHOD_FSAI  ? AFN_METHOD_FSAI
              : P.method == AFN_METHOD_RAN   ? AFN_METHOD_RAN
              : P.method == AFN_METHOD_NONE  ? AFN_METHOD_NONE
                                             : AFN_METHOD_AFN;
  const bool adaptive = P.k_adaptive && P.method != AFN_METHOD_FSAI && P.method != AFN_METHOD_NONE;
  // FPS landmarks are nested (X_{k-1} in X_k): with an adaptive k the
  // FPS for min(k_cap, n) points runs on the build stream WHILE Alg. 1 runs on
  // a side stream; the first k of them are exactly FPS(k).
  // MaxMin ordering: FPS through all n points, the first k are the landmarks
  const bool maxmin = P.ordering == AFN_ORDER_MAXMIN;
  const int64_t kfps = maxmin ? n : (adaptive && P.landmarks == AFN_LANDMARKS_FPS) ? std::min<int64_t>(P.k_cap, n) : 0;
  std::vector<int64_t*> idx(nlocal, nullptr);
  cudaEvent_t efps0, efps1;
  AFN_CUDA(cudaEventCreate(&efps0));
  AFN_CUDA(cudaEventCreate(&efps1));
  struct EvG3 {
    cudaEvent_t a, b;
    ~EvG3() { cudaEventDestroy(a); cudaEventDestroy(b); }
  } eg3{efps0, efps1};
  AFN_CUDA(cudaEventRecord(efps0, st));
  int64_t* kstop = nullptr;  // lowered to k once Alg. 1 is done (FPS early stop)
  int64_t* hk = pinned_i64();
  if (!hk) {
    set_error("pinned host allocation failed");
    return AFN_ERR_NOMEM;
  }
  if (kfps > 0) {
    TRY(ralloc(h->rk[0], &kstop, 1, st));
    hk[0] = kfps;
    AFN_CUDA(cudaMemcpyAsync(kstop, hk, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    kt_begin(KT_FPS, st);
    for (int q = 0; q < nlocal; ++q) {
      RankSt& s = h->rk[q];
      TRY(ralloc(s, &idx[q], (size_t)kfps, st));
      TRY(ralloc(s, &s.fill, (size_t)kfps, st));
      TRY(fps_run(X, n, d, kfps, P.fps_seed, idx[q], s.fill, st, kstop));
    }
    kt_end(KT_FPS, st, 0.0);
    AFN_CUDA(cudaEventRecord(efps1, st));
  }
  float alg1_ms = 0.f;
  if (adaptive) {
    int m = P.m > 0 ? P.m : alg1_default_m(n);
    REQ(m >= 2 && m <= n && m <= 1024, "need 2 <= m <= min(n, 1024)");
    cudaStream_t s2 = side_stream();
    cudaEvent_t a0, a1;
    AFN_CUDA(cudaEventCreate(&a0));
    AFN_CUDA(cudaEventCreate(&a1));
    struct EvG2 {
      cudaEvent_t a, b;
      ~EvG2() { cudaEventDestroy(a); cudaEventDestroy(b); }
    } eg2{a0, a1};
    AFN_CUDA(cudaStreamWaitEvent(s2, ev[0], 0));
    AFN_CUDA(cudaEventRecord(a0, s2));
    kt_begin(KT_ALG1, s2);
    TRY(alg1_run(X, n, d, kn, m, P.rng_seed, kthr, &h->a1, s2));
    kt_end(KT_ALG1, s2, 0.0);
    if (kstop && !maxmin) {  // the running FPS may stop at min(k_cap, khat)
      hk[1] = std::min<int64_t>(kfps, std::max<int64_t>(1, h->a1.khat));
      AFN_CUDA(cudaMemcpyAsync(kstop, hk + 1, sizeof(int64_t), cudaMemcpyHostToDevice, s2));
    }
    AFN_CUDA(cudaEventRecord(a1, s2));
    AFN_CUDA(cudaStreamWaitEvent(st, a1, 0));
    // the cutoff matvec plan depends only on the point set: made now from the
    // original points on the (idle) high-priority stream while FPS runs on a
    // few SMs, its point indices remapped after the permutation
    if (kn.kind == 0 && d <= 3 && n >= 4096 && kmv_get_mode() != 1) {
      cudaStream_t ps = hp_stream();
      for (auto& s : h->rk) {
        double* Xs0 = nullptr;
        TRY(dalloc((void**)&Xs0, sizeof(double) * (size_t)n * d, ps));
        TRY(kmv_prescale(X, n, d, kn, Xs0, ps));
        TRY(kmv_plan_make(Xs0, n, n, d, kn.kind, true, h->R, s.rank, ps,
                          [&](double** qq, size_t c) { return ralloc(s, qq, c, ps); }, &s.plan, &s.kmv_part));
        dfree(Xs0, ps);
        if (!s.plan.cut) {  // (the dense plans read the permuted points: made later)
          rfree(s, s.kmv_part, ps);
          s.kmv_part = nullptr;
          s.plan = KmvPlan{};
        }
      }
    }
    AFN_CUDA(cudaEventSynchronize(a1));
    alg1_ms = ev_ms(a0, a1);
    k = std::min<int64_t>(P.k_cap, std::max<int64_t>(1, h->a1.khat));
    k = std::min<int64_t>(k, n);
    // Algorithm 2: AFN if khat >= 2000, else Nystrom with khat landmarks
    if (P.method == AFN_METHOD_ALG2) h->method = h->a1.khat >= kthr ? AFN_METHOD_AFN : AFN_METHOD_NYSTROM;
  }
  // plain FSAI of K + mu I, and M = I (CG): no landmarks
  if (h->method == AFN_METHOD_FSAI || h->method == AFN_METHOD_NONE) k = 0;
  const bool nys = h->method == AFN_METHOD_NYSTROM || h->method == AFN_METHOD_RAN;  // F-form
  h->k = k;
  // the Nystrom branch has no Schur complement, CG no FSAI part
  const int64_t N2 = (nys || h->method == AFN_METHOD_NONE) ? 0 : n - k;
  h->N2 = N2;
  h->nnz = knn_nnz(N2, P.w);
  for (auto& s : h->rk) {
    s.own = shard_rows(n, k, h->R, s.rank);
    s.lo = N2 == 0 ? 0 : s.own.b0 - k;  // own non-landmark rows (W, pattern, G)
    s.hi = N2 == 0 ? 0 : s.lo + s.own.nb;
  }

  // ---- a3: landmarks (replicated): FPS or uniform (R29)
  if (kfps == 0) {
    AFN_CUDA(cudaEventRecord(efps0, st));
    kt_begin(KT_FPS, st);
    for (int q = 0; q < nlocal; ++q) {
      RankSt& s = h->rk[q];
      TRY(ralloc(s, &idx[q], (size_t)k, st));
      TRY(ralloc(s, &s.fill, (size_t)k, st));
      if (k == 0) continue;
      if (P.landmarks == AFN_LANDMARKS_UNIFORM) {
        TRY(uniform_landmarks(n, k, P.rng_seed ^ 0x6A09E667F3BCC909ULL, idx[q], st));
        AFN_CUDA(cudaMemsetAsync(s.fill, 0, sizeof(double) * k, st));  // no fill trace
      } else {
        TRY(fps_run(X, n, d, k, P.fps_seed, idx[q], s.fill, st));
      }
    }
    kt_end(KT_FPS, st, 0.0);
    AFN_CUDA(cudaEventRecord(efps1, st));
  }
  AFN_CUDA(cudaEventRecord(ev[2], st));

  // kNN pattern of the non-landmark points (own rows; row_ptr in closed form),
  // then its transpose (the pair-union FSAI needs "rows containing a")
  std::vector<int64_t*> tmap(nlocal, nullptr);
  auto pattern_phase = [&](RankSt& s, cudaStream_t ss) -> afn_status {
    kt_begin(KT_KNN, ss);
    TRY(ralloc(s, &s.rp, (size_t)N2 + 1, ss));
    TRY(ralloc(s, &s.col, (size_t)(h->nnz > 0 ? h->nnz : 1), ss));
    if (N2 > 0) TRY(knn_run(s.Xp + k * d, N2, d, P.w, s.rp, s.col, ss, s.lo, s.hi));
    else AFN_CUDA(cudaMemsetAsync(s.rp, 0, sizeof(int64_t), ss));
    kt_end(KT_KNN, ss, 0.0);
    return AFN_OK;
  };
  auto transpose_phase = [&](RankSt& s, int q, cudaStream_t ss) -> afn_status {
    TRY(ralloc(s, &s.gval, (size_t)(h->nnz > 0 ? h->nnz : 1), ss));
    TRY(ralloc(s, &s.trp, (size_t)N2 + 1, ss));
    TRY(ralloc(s, &s.tcol, (size_t)(h->nnz > 0 ? h->nnz : 1), ss));
    TRY(ralloc(s, &s.tval, (size_t)(h->nnz > 0 ? h->nnz : 1), ss));
    if (N2 > 0) {
      TRY(ralloc(s, &tmap[q], (size_t)(h->nnz > 0 ? h->nnz : 1), ss));
      check_pattern_kernel<<<(unsigned)((N2 + 255) / 256), 256, 0, ss>>>(s.rp, s.col, N2, s.derr);
      AFN_LAUNCH_CHECK("check_pattern_kernel");
      TRY(csr_transpose(s.rp, s.col, nullptr, N2, h->nnz, s.trp, s.tcol, nullptr, ss, tmap[q]));
    } else {
      AFN_CUDA(cudaMemsetAsync(s.trp, 0, sizeof(int64_t), ss));
    }
    return AFN_OK;
  };
  // single rank, AFN: the pattern does not depend on L or W -> overlap it
  const bool povl = h->R == 1 && !nys && N2 > 0 && k > 0;
  cudaEvent_t e_pat0 = nullptr, e_pat1 = nullptr;
  if (povl) {
    AFN_CUDA(cudaEventCreateWithFlags(&e_pat0, cudaEventDisableTiming));
    AFN_CUDA(cudaEventCreateWithFlags(&e_pat1, cudaEventDisableTiming));
  }
  struct EvPat {
    cudaEvent_t a, b;
    ~EvPat() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
  } evpat{e_pat0, e_pat1};
  cudaEvent_t e_hp0 = nullptr, e_hp1 = nullptr;
  if (povl) {
    AFN_CUDA(cudaEventCreateWithFlags(&e_hp0, cudaEventDisableTiming));
    AFN_CUDA(cudaEventCreateWithFlags(&e_hp1, cudaEventDisableTiming));
  }
  EvPat evhp{e_hp0, e_hp1};

  // cutoff plans (kmv.cu matvec plan, wcut.cu W product), per local rank
  std::vector<WCutPlan> wplan(nlocal);
  struct WPlanFree {
    std::vector<WCutPlan>& p;
    ~WPlanFree() {
      for (auto& x : p) w_cut_free(&x);
    }
  } wpf{wplan};
  auto early_plans = [&](RankSt& s) -> afn_status {
    const int q = (int)(&s - &h->rk[0]);
    if (s.kmv_part)  // (made from the original points during FPS: to the handle's positions)
      TRY(kmv_plan_remap(s.plan, s.kmv_part, s.perm, n, st));
    else
      TRY(kmv_plan_make(s.Xs, n, s.own.size(), d, h->kn.kind, true, h->R, s.rank, st,
                        [&](double** qq, size_t c) { return ralloc(s, qq, c, st); }, &s.plan, &s.kmv_part));
    // (Z mode: one rank, AFN -- the FSAI products through Z = K21 M)
    wplan[q].keep = h->R == 1 && povl;  // (the apply through the tiles)
    if (!nys && k > 0 && N2 > 0 && s.hi > s.lo && kmv_get_mode() != 1)
      TRY(w_cut_plan(s.Xp, k, s.Xp + (k + s.lo) * d, s.hi - s.lo, d, kn, kmv_get_mode() == 2,
                     h->R == 1 && povl && k <= 8192 && kmv_get_mode() != 3, st, &wplan[q]));
    return AFN_OK;
  };

  // ---- a1: permutation, permuted + prescaled points; a4: L L^T = K11 + mu I, L^{-T}
  for (int q = 0; q < nlocal; ++q) {
    RankSt& s = h->rk[q];
    TRY(ralloc(s, &s.derr, 4, st));
    AFN_CUDA(cudaMemsetAsync(s.derr, 0, sizeof(int) * 4, st));
    unsigned char* flag;
    unsigned* flag32;
    TRY(ralloc(s, &flag, (size_t)n, st));
    TRY(ralloc(s, &flag32, (size_t)n, st));
    AFN_CUDA(cudaMemsetAsync(flag32, 0, sizeof(unsigned) * (size_t)n, st));
    if (k > 0) {
      mark_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(idx[q], k, n, flag32, s.derr);
      AFN_LAUNCH_CHECK("mark_kernel");
    }
    flag8_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(flag32, n, flag);
    AFN_LAUNCH_CHECK("flag8_kernel");
    TRY(ralloc(s, &s.perm, (size_t)n, st));
    if (maxmin) {  // the FPS order of all n points
      AFN_CUDA(cudaMemcpyAsync(s.perm, idx[q], sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
    } else {
      perm_kernel<<<1, 1024, 0, st>>>(flag, idx[q], n, k, s.perm);
      AFN_LAUNCH_CHECK("perm_kernel");
    }
    rfree(s, flag, st);
    rfree(s, flag32, st);
    TRY(ralloc(s, &s.Xp, (size_t)n * d, st));
    TRY(gather_rows(X, n, d, s.perm, s.Xp, st));
    TRY(ralloc(s, &s.Xs, (size_t)n * d, st));
    TRY(kmv_prescale(s.Xp, n, d, kn, s.Xs, st));
    TRY(ralloc(s, &s.dinfo, 2, st));
    AFN_CUDA(cudaMemsetAsync(s.dinfo, 0, sizeof(int) * 2, st));
    if (povl) {  // kNN pattern + its transpose on the side stream, concurrently with L, L^{-1}, W
      AFN_CUDA(cudaEventRecord(e_pat0, st));
      AFN_CUDA(cudaStreamWaitEvent(side_stream(), e_pat0, 0));
      TRY(pattern_phase(s, side_stream()));
      TRY(transpose_phase(s, q, side_stream()));
      AFN_CUDA(cudaEventRecord(e_pat1, side_stream()));
    }
    TRY(ralloc(s, &s.L, (size_t)k * k, st));
    TRY(ralloc(s, &s.LinvT, (size_t)k * k, st));
    if (k == 0) {
      TRY(early_plans(s));
      continue;
    }
    if (!nys) TRY(ralloc(s, &s.Linv, (size_t)k * k, st));
    // L^{-1}'s workspace from the build stream before the switch (a pool
    // block taken on fs could carry a wait on another stream's work)
    double* lws = nullptr;
    TRY(ralloc(s, &lws, (size_t)linv_ws_doubles(k), st));
    // K11, its Cholesky and L^{-1}: with the pattern overlapped, on a
    // high-priority stream -- their ~200 short launches then take SMs ahead
    // of the kNN grid's pending CTAs instead of queueing behind them
    cudaStream_t fs = st;
    if (povl) {
      fs = hp_stream();
      AFN_CUDA(cudaEventRecord(e_hp0, st));
      AFN_CUDA(cudaStreamWaitEvent(fs, e_hp0, 0));
    }
    // AFN: K11 + mu I.  Nystrom: K11 + nu I, nu = 1e-10 (reading R30)
    TRY(gen_k11(s.Xp, k, d, kn, nys ? AFN_NYS_NU : P.mu, s.L, fs));
    kt_begin(KT_POTRF, fs);
    TRY(potrf_lower(s.L, k, s.dinfo, fs));
    kt_end(KT_POTRF, fs, (double)k * k * k / 3.0);
    // L^{-1} (and so W) after the kNN pattern and its transpose: W then runs
    // with the SMs to itself (measured: W beside the kNN is slower overall --
    // C2 setup 12.1 vs 11.8 ms)
    if (fs != st) AFN_CUDA(cudaStreamWaitEvent(fs, e_pat1, 0));
    kt_begin(KT_LINV, fs);
    TRY(trsm_linvt(s.L, k, s.LinvT, fs, lws));
    if (!nys) TRY(transpose_sq(s.LinvT, k, s.Linv, fs));
    kt_end(KT_LINV, fs, (double)k * k * k / 3.0);
    // the cutoff plans need only the points: made here on st while the
    // Cholesky (fs) and the kNN pattern (side stream) run -- their host waits
    // then hide behind that work instead of serialising the build
    TRY(early_plans(s));
    if (fs != st) {
      AFN_CUDA(cudaEventRecord(e_hp1, fs));
      AFN_CUDA(cudaStreamWaitEvent(st, e_hp1, 0));
    }
    rfree(s, lws, st);
  }
  AFN_CUDA(cudaEventRecord(ev[3], st));
  auto chol_check = [&]() -> afn_status {
    for (auto& s : h->rk) {
      int info = 0;
      AFN_CUDA(cudaMemcpyAsync(&info, s.dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
      AFN_CUDA(cudaStreamSynchronize(st));
      if (info) {
        set_error("Cholesky of K11 + %s I broke down at row %d", nys ? "nu" : "mu", info - 1);
        return AFN_ERR_NOT_SPD;
      }
    }
    return AFN_OK;
  };
  // (AFN, one rank: checked after the FSAI work is queued, see below)
  if (nys || !povl) TRY(chol_check());
  if (nys) {
    TRY(build_nystrom(h, st));
    AFN_CUDA(cudaEventRecord(ev[4], st));
    AFN_CUDA(cudaEventRecord(ev[5], st));
    AFN_CUDA(cudaEventRecord(ev[6], st));
    AFN_CUDA(cudaEventRecord(ev[7], st));
    AFN_CUDA(cudaEventRecord(ev[8], st));
  } else {

  // ---- a5: W = K21 L^{-T}, own rows (into a full-height buffer when sharded:
  // the FSAI rows of a rank need the W rows of all their pattern neighbours)
  std::vector<double*> Wf(nlocal);
  kt_begin(KT_W_GEMM, st);
  double w_work = 0.0;  // executed flops (dense: (N2/R) k^2 / 2 FMA per rank)
  for (int q = 0; q < nlocal; ++q) {
    RankSt& s = h->rk[q];
    // one rank, Z mode: neither the FSAI products (Z) nor the apply (the K21
    // tiles, §6.6) read W -- it is formed only on demand (copy-out, the per-row
    // FSAI fallback) from the kept plan
    if (wplan[q].used && wplan[q].lp && wplan[q].keep) {
      Wf[q] = nullptr;
      continue;
    }
    TRY(ralloc(s, &Wf[q], (size_t)(N2 > 0 ? N2 : 1) * k, st));
    const double* X2 = s.Xp + k * d;
    if (s.hi > s.lo) {
      const bool cut = wplan[q].used;  // (the decay of K21: wcut.cu)
      if (cut) {
        w_work += wplan[q].flops;
        TRY(w_cut_run(&wplan[q], s.LinvT, Wf[q] + s.lo * k, st));
      }
      else if (k >= AFN_W_INT8_MIN_K && s.Linv)  // (INT8 tensor cores, exact slicing: ozaki.cu)
        TRY(w_gemm_ozaki(s.Linv, k, s.Xp, X2 + s.lo * d, s.hi - s.lo, d, kn, Wf[q] + s.lo * k, st));
      else
        TRY(w_gemm(s.LinvT, k, s.Xp, X2 + s.lo * d, s.hi - s.lo, d, kn, Wf[q] + s.lo * k, st));
      if (!cut) w_work += (double)(s.hi - s.lo) * (double)k * (double)k;
    }
  }
  // Z mode: M = (K11 + mu I)^{-1} and Z = K21 M over the landmarks' Morton
  // order for the FSAI products (freed after them); no memory -> W products
  std::vector<double*> zbuf(3 * nlocal, nullptr);
  std::vector<FsaiZ> fz(nlocal);
  for (int q = 0; q < nlocal; ++q) {
    RankSt& s = h->rk[q];
    WCutPlan& wp = wplan[q];
    if (!wp.used || !wp.lp) continue;
    const afn_status a1 = dalloc((void**)&zbuf[3 * q], sizeof(double) * (size_t)k * k, st);
    const afn_status a2 = a1 == AFN_OK ? dalloc((void**)&zbuf[3 * q + 1], sizeof(double) * (size_t)k * k, st) : a1;
    const afn_status a3 =
        a2 == AFN_OK ? dalloc((void**)&zbuf[3 * q + 2], sizeof(double) * (size_t)(s.hi - s.lo) * k, st) : a2;
    if (a3 != AFN_OK) {  // (not enough memory for Z: the W products)
      for (int e = 0; e < 3; ++e)
        if (zbuf[3 * q + e]) dfree(zbuf[3 * q + e], st), zbuf[3 * q + e] = nullptr;
      w_cut_free(&wp);
      continue;
    }
    TRY(w_cut_z(&wp, s.LinvT, s.Linv, zbuf[3 * q], zbuf[3 * q + 1], zbuf[3 * q + 2], st));
    w_work += wp.zflops + (double)k * k * k;
    fz[q] = FsaiZ{zbuf[3 * q + 2], wp.tilerow, wp.uoff, wp.ulistp, wp.aoff, wp.Ap,
                  (double)k / (double)std::max<int64_t>(1, N2) <= 0.015};  // (C5 0.0077 staged; C3 0.031 not)
  }
  struct ZFree {
    std::vector<double*>& b;
    cudaStream_t st;
    ~ZFree() {
      for (double* x : b)
        if (x) dfree(x, st);
    }
  } zfree{zbuf, st};
  kt_end(KT_W_GEMM, st, w_work / nlocal);
  AFN_CUDA(cudaEventRecord(ev[4], st));

  // ---- a6: kNN pattern (already queued on the side stream when povl)
  if (povl) {
    AFN_CUDA(cudaStreamWaitEvent(st, e_pat1, 0));
  } else {
    for (auto& s : h->rk) TRY(pattern_phase(s, st));
  }
  AFN_CUDA(cudaEventRecord(ev[5], st));
  if (N2 > 0 && !povl) {
    // exchange W rows and pattern rows
    {
      int q = 0;
      TRY(exchange(h, [&](RankSt&) { return Wf[q++]; },
                   [&](int s) { return rows2_ranges(h, s, 8 * (size_t)k); }, st));
    }
    TRY(exchange(h, [](RankSt& s) { return s.col; }, [&](int s) { return nnz_ranges(h, s, 4); }, st));
    for (auto& s : h->rk) {
      check_pattern_kernel<<<(unsigned)((N2 + 255) / 256), 256, 0, st>>>(s.rp, s.col, N2, s.derr);
      AFN_LAUNCH_CHECK("check_pattern_kernel");
    }
  }
  AFN_CUDA(cudaEventRecord(ev[6], st));

  // ---- a7: FSAI rows (own), then G^T
  if (!povl)
    for (int q = 0; q < nlocal; ++q) TRY(transpose_phase(h->rk[q], q, st));
  AFN_CUDA(cudaEventRecord(ev[7], st));
  if (N2 > 0) {
    for (int q = 0; q < nlocal; ++q) {
      RankSt& s = h->rk[q];
      const double* X2 = s.Xp + k * d;
      // (the pair-union product; AFN_ERR_STATE: a group's union overflowed -> per-row Grams)
      const afn_status fs = fsai_sddmm_run(X2, N2, d, kn, P.mu, Wf[q], k, s.rp, s.col, s.trp, s.tcol, s.lo,
                                           s.hi, s.gval, s.dinfo + 1, st, povl ? side_stream() : st,
                                           fz[q].Zp ? &fz[q] : nullptr);
      if (fs != AFN_OK && fs != AFN_ERR_STATE) return fs;
      if (fs != AFN_OK) {
        kt_begin(KT_FSAI_GRAM, st);
        if (!Wf[q]) {  // (Z mode skipped W: form it now from the plan)
          TRY(ralloc(s, &Wf[q], (size_t)(N2 > 0 ? N2 : 1) * k, st));
          TRY(w_cut_run(&wplan[q], s.LinvT, Wf[q], st));
        }
        TRY(fsai_run(X2, N2, d, kn, P.mu, Wf[q], k, s.rp, s.col, s.lo, s.hi, s.gval, s.dinfo + 1, st));
        kt_end(KT_FSAI_GRAM, st, 0.0);
      }
    }
  }
  AFN_CUDA(cudaEventRecord(ev[8], st));
  // (AFN, one rank: the Cholesky breakdown check waits until here so that the
  // host has queued W and the FSAI work first -- a failed Cholesky only makes
  // the queued work useless, it is reported before anything is used)
  if (povl) TRY(chol_check());
  if (N2 > 0) {
    TRY(exchange(h, [](RankSt& s) { return s.gval; }, [&](int s) { return nnz_ranges(h, s, 8); }, st));
    for (int q = 0; q < nlocal; ++q) {
      RankSt& s = h->rk[q];
      TRY(gather_map(s.gval, tmap[q], h->nnz, s.tval, st));
      rfree(s, tmap[q], st);
    }
  }
  // W: keep the rank's own rows only
  for (int q = 0; q < nlocal; ++q) {
    RankSt& s = h->rk[q];
    if (h->R == 1) {
      s.W = Wf[q];
    } else {
      TRY(ralloc(s, &s.W, (size_t)std::max<int64_t>(1, s.hi - s.lo) * k, st));
      if (s.hi > s.lo)
        AFN_CUDA(cudaMemcpyAsync(s.W, Wf[q] + s.lo * k, sizeof(double) * (s.hi - s.lo) * k,
                                 cudaMemcpyDeviceToDevice, st));
      rfree(s, Wf[q], st);
    }
  }

  }  // AFN / FSAI

  // ---- workspaces for apply / PCG
  auto q_of = [&](RankSt& s) { return (int)(&s - &h->rk[0]); };
  for (auto& s : h->rk) {
    const int64_t nl = s.own.size();
    if (wplan[q_of(s)].used && wplan[q_of(s)].keep) {  // the K21 tiles stay for the apply
      s.kt = std::move(wplan[q_of(s)]);
      wplan[q_of(s)] = WCutPlan{};
      TRY(w_cut_apply_prep(&s.kt, st));
    }
    if (!s.kmv_part)  // (normally made early, beside the Cholesky)
      TRY(kmv_plan_make(s.Xs, n, nl, d, h->kn.kind, true, h->R, s.rank, st,
                        [&](double** q, size_t c) { return ralloc(s, q, c, st); }, &s.plan, &s.kmv_part));
    if (s.plan.sym && h->R > 1) TRY(ralloc(s, &s.qpart, (size_t)h->R * n, st));
    const int64_t gw = std::max(std::max(gemv_t_ws(k, k), gemv_t_ws(h->R == 1 ? N2 : s.hi - s.lo, k)),
                                nys ? gemv_t_ws(nl, k) : (int64_t)1);
    TRY(ralloc(s, &s.gws, (size_t)gw, st));
    TRY(ralloc(s, &s.tvec, (size_t)k, st));
    TRY(ralloc(s, &s.vvec, (size_t)k, st));
    TRY(ralloc(s, &s.kpart, (size_t)h->R * k, st));
    TRY(ralloc(s, &s.uvec, (size_t)std::max<int64_t>(std::max<int64_t>(N2, k), 1), st));
    TRY(ralloc(s, &s.yvec, (size_t)(N2 > 0 ? N2 : 1), st));
    TRY(ralloc(s, &s.rbuf, (size_t)n, st));
    TRY(ralloc(s, &s.zbuf, (size_t)n, st));
    for (double** v : {&s.x, &s.r, &s.z, &s.p, &s.q}) {
      TRY(ralloc(s, v, (size_t)n, st));
      AFN_CUDA(cudaMemsetAsync(*v, 0, sizeof(double) * n, st));
    }
    TRY(ralloc(s, &s.sc, SC_N, st));
    TRY(ralloc(s, &s.scpart, (size_t)h->R * SC_N, st));
    TRY(ralloc(s, &s.dws, (size_t)dot_ws(), st));
    TRY(ralloc(s, &s.dcnt, 4, st));
    AFN_CUDA(cudaMemsetAsync(s.dcnt, 0, sizeof(unsigned) * 4, st));
    AFN_CUDA(cudaMemsetAsync(s.sc, 0, sizeof(double) * SC_N, st));
    AFN_CUDA(cudaMemsetAsync(s.scpart, 0, sizeof(double) * h->R * SC_N, st));
  }
  if (!pinned_scalars()) {
    set_error("pinned host allocation failed");
    return AFN_ERR_NOMEM;
  }
  AFN_CUDA(cudaEventRecord(ev[9], st));
  // device-side checks of every rank (consistency codes, FSAI breakdown on
  // the rank's own rows), all-gathered so that every rank returns the same
  // status (no rank may fail alone and leave the others in a collective)
  std::vector<int> stat(2 * (size_t)h->R, 0);
  {
    std::vector<int*> sb(nlocal);
    for (int q = 0; q < nlocal; ++q) {
      RankSt& s = h->rk[q];
      TRY(ralloc(s, &sb[q], 2 * (size_t)h->R, st));
      AFN_CUDA(cudaMemsetAsync(sb[q], 0, sizeof(int) * 2 * h->R, st));
      AFN_CUDA(cudaMemcpyAsync(sb[q] + 2 * s.rank, s.derr, sizeof(int), cudaMemcpyDeviceToDevice, st));
      AFN_CUDA(cudaMemcpyAsync(sb[q] + 2 * s.rank + 1, s.dinfo + 1, sizeof(int), cudaMemcpyDeviceToDevice, st));
    }
    int q2 = 0;
    TRY(exchange(h, [&](RankSt&) { return sb[q2++]; }, [&](int r) { return RankRanges{{8 * (size_t)r, 8}}; },
                 st));
    AFN_CUDA(cudaMemcpyAsync(stat.data(), sb[0], sizeof(int) * 2 * h->R, cudaMemcpyDeviceToHost, st));
  }
  TRY(comm_stream_sync(h->comm, st));
  for (int r = 0; r < h->R; ++r) {
    if (stat[2 * r]) {
      set_error("internal consistency check failed on rank %d (code %d: 1/2 landmark ids, 4/8 pattern)", r,
                stat[2 * r]);
      return AFN_ERR_CUDA;
    }
  }
  for (int r = 0; r < h->R; ++r) {
    if (stat[2 * r + 1]) {
      set_error("FSAI block Cholesky broke down in row %d (rank %d)", stat[2 * r + 1] - 1, r);
      return AFN_ERR_NOT_SPD;
    }
  }
  h->ms[0] = alg1_ms;                                       // alg1 (side stream)
  h->ms[1] = ev_ms(efps0, efps1);  // fps (overlapping alg1 when k is adaptive)
  h->ms[2] = ev_ms(ev[2], ev[3]);  // perm + chol + L^{-T}
  h->ms[3] = ev_ms(ev[3], ev[4]);  // W
  h->ms[4] = ev_ms(ev[4], ev[5]);  // knn
  h->ms[5] = ev_ms(ev[5], ev[9]);  // exchanges + transpose + fsai + G^T + workspaces
  h->ms[6] = ev_ms(ev[0], ev[9]);  // total
  h->ms[7] = ev_ms(ev[7], ev[8]);  // fsai rows
  kt_collect();
  *out = h;
  h = nullptr;  // release the guard
  return AFN_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int32_t afn_abi_version(void) { return AFN_ABI_VERSION; }

afn_status afn_set_allocator(afn_alloc_fn alloc, afn_free_fn free_fn, void* ctx) {
  REQ((alloc == nullptr) == (free_fn == nullptr), "alloc and free must both be set or both be NULL");
  release_deferred(true);
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  REQ(g_alloc_size.empty(), "%zu blocks from the current allocator are still live (destroy the handles first)",
      g_alloc_size.size());
  g_alloc = alloc;
  g_free = free_fn;
  g_alloc_ctx = ctx;
  return AFN_OK;
}

afn_status afn_pool_stats(int64_t* reserved, int64_t* used) {
  REQ(reserved && used, "null argument");
  int dev = 0;
  AFN_CUDA(cudaGetDevice(&dev));
  pool_setup_once();
  cudaMemPool_t pool;
  AFN_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t r = 0, u = 0;
  AFN_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
  AFN_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
  *reserved = (int64_t)r;
  *used = (int64_t)u;
  return AFN_OK;
}

void afn_kt_enable(int32_t on) {
  kt_collect();
  g_kt_on.store(on != 0);
}
void afn_kt_reset(void) {
  kt_collect();
  for (int i = 0; i < KT_N; ++i) g_kt_ms[i] = g_kt_work[i] = 0.0, g_kt_cnt[i] = 0;
}
int32_t afn_kt_read(double* ms, double* work, int64_t* count, int32_t n) {
  kt_collect();
  const int m = n < KT_N ? n : KT_N;
  for (int i = 0; i < m; ++i) {
    if (ms) ms[i] = g_kt_ms[i];
    if (work) work[i] = g_kt_work[i];
    if (count) count[i] = g_kt_cnt[i];
  }
  return KT_N;
}
const char* afn_last_error(void) { return g_err; }
int64_t afn_launch_count(void) { return g_launches.load(); }

namespace {
afn_status kmv_rows_impl(const double* X, int64_t n, int32_t d, int32_t kernel, double l, double mu,
                         const double* v, int64_t row0, int64_t nrows, double* y, void* stream, bool sym_ok) {
  TRY(validate_X(X, n, d));
  REQ(kernel == AFN_KERNEL_GAUSSIAN || kernel == AFN_KERNEL_MATERN32, "unknown kernel %d", kernel);
  REQ(l > 0 && std::isfinite(l), "l must be > 0");
  REQ(mu >= 0 && std::isfinite(mu), "mu must be >= 0");
  REQ(row0 >= 0 && nrows >= 0 && row0 + nrows <= n, "row range out of bounds");
  REQ(is_dev(v) && (nrows == 0 || is_dev(y)), "v, y must be device pointers");
  REQ(y != v, "y must not alias v");
  cudaStream_t st = (cudaStream_t)stream;
  Temps t(st);
  double* Xs;
  TRY(t.get(&Xs, (size_t)n * d));
  TRY(kmv_prescale(X, n, d, Kern{kernel, l}, Xs, st));
  KmvPlan plan;
  double* part = nullptr;
  TRY(kmv_plan_make(Xs, n, nrows, d, kernel, sym_ok && row0 == 0 && nrows == n, 1, 0, st,
                    [&](double** q, size_t c) { return t.get(q, c); }, &plan, &part));
  TRY(kmv_launch(Xs, n, d, kernel, v, mu, seg_range(row0, nrows), y, false, part, plan, st));
  return AFN_OK;
}
}  // namespace

// explicit row ranges never use the symmetric plan: a shard's rows are then
// bit-identical to the same rows of any other row-range evaluation
afn_status kernel_matvec_rows(const double* X, int64_t n, int32_t d, int32_t kernel, double l, double mu,
                              const double* v, int64_t row0, int64_t nrows, double* y, void* stream) {
  return kmv_rows_impl(X, n, d, kernel, l, mu, v, row0, nrows, y, stream, false);
}

afn_status kernel_matvec(const double* X, int64_t n, int32_t d, int32_t kernel, double l, double mu,
                         const double* v, double* y, void* stream) {
  return kmv_rows_impl(X, n, d, kernel, l, mu, v, 0, n, y, stream, true);
}

afn_status afn_fps(const double* X, int64_t n, int32_t d, int64_t k, int64_t seed, int64_t* idx,
                   double* fill, void* stream) {
  TRY(validate_X(X, n, d));
  REQ(k >= 1 && k <= n, "need 1 <= k <= n");
  REQ(seed >= 0 && seed < n, "need 0 <= seed < n");
  REQ(is_dev(idx), "idx must be a device pointer");
  REQ(fill == nullptr || is_dev(fill), "fill must be a device pointer or NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Temps t(st);
  if (!fill) TRY(t.get(&fill, (size_t)k));
  TRY(fps_run(X, n, d, k, seed, idx, fill, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  return AFN_OK;
}

afn_status afn_w_product(const double* X1, int64_t k, const double* Xr, int64_t N, int32_t d, int32_t kernel,
                         double l, const double* Linv, int32_t method, double* W, void* stream) {
  TRY(validate_X(X1, k, d));
  TRY(validate_X(Xr, N, d));
  REQ(kernel == AFN_KERNEL_GAUSSIAN || kernel == AFN_KERNEL_MATERN32, "unknown kernel %d", kernel);
  REQ(l > 0 && std::isfinite(l), "l must be > 0");
  REQ(method == AFN_WPROD_DMMA || method == AFN_WPROD_INT8 || method == AFN_WPROD_CUT, "unknown method %d", method);
  REQ(method != AFN_WPROD_CUT || (kernel == AFN_KERNEL_GAUSSIAN && d <= 3),
      "AFN_WPROD_CUT needs the Gaussian kernel and d <= 3");
  REQ(is_dev(Linv) && is_dev(W), "Linv, W must be device pointers");
  REQ(method != AFN_WPROD_INT8 || k < 65536, "AFN_WPROD_INT8 needs k < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  if (method == AFN_WPROD_INT8) return w_gemm_ozaki(Linv, k, X1, Xr, N, d, Kern{kernel, l}, W, st);
  Temps t(st);
  double* LinvT;
  TRY(t.get(&LinvT, (size_t)k * k));
  TRY(transpose_sq(Linv, k, LinvT, st));
  if (method == AFN_WPROD_CUT) {
    bool used = false;
    TRY(w_gemm_cut(LinvT, k, X1, Xr, N, d, Kern{kernel, l}, W, st, true, &used, nullptr));
    REQ(used, "AFN_WPROD_CUT: too many row tiles");
    return AFN_OK;
  }
  return w_gemm(LinvT, k, X1, Xr, N, d, Kern{kernel, l}, W, st);
}

afn_status afn_knn_pattern(const double* P, int64_t N, int32_t d, int32_t w, int64_t* row_ptr,
                           int32_t* col, void* stream) {
  TRY(validate_X(P, N, d));
  REQ(w >= 1 && w <= AFN_W_MAX, "w must be in 1..%d", AFN_W_MAX);
  REQ(N <= 0x7fffffffLL, "N must fit int32 column indices");
  REQ(is_dev(row_ptr) && is_dev(col), "row_ptr, col must be device pointers");
  return knn_run(P, N, d, w, row_ptr, col, (cudaStream_t)stream);
}

afn_status afn_estimate_rank(const double* X, int64_t n, int32_t d, int32_t kernel, double l, int32_t m,
                             uint64_t rng_seed, int32_t k_threshold, int64_t* khat, int32_t* r,
                             int32_t* refined, void* stream) {
  TRY(validate_X(X, n, d));
  REQ(l > 0 && std::isfinite(l), "l must be > 0");
  REQ(kernel == AFN_KERNEL_GAUSSIAN || kernel == AFN_KERNEL_MATERN32, "unknown kernel %d", kernel);
  if (m == 0) m = alg1_default_m(n);
  REQ(m >= 2 && m <= n && m <= 1024, "need 2 <= m <= min(n, 1024)");
  REQ(k_threshold >= 1, "k_threshold must be >= 1");
  REQ(khat && r && refined, "outputs must be non-null host pointers");
  Alg1Result res;
  TRY(alg1_run(X, n, d, Kern{kernel, l}, m, rng_seed, k_threshold, &res, (cudaStream_t)stream));
  *khat = res.khat;
  *r = res.r;
  *refined = res.refined;
  return AFN_OK;
}

afn_status afn_build(const double* X, int64_t n, int32_t d, const afn_params* prm, void* stream,
                     afn_handle* out) {
  return build_impl(nullptr, X, n, d, prm, stream, out);
}

afn_status afn_build_dist(afn_comm comm, const double* X, int64_t n, int32_t d, const afn_params* prm,
                          void* stream, afn_handle* out) {
  return build_impl(comm, X, n, d, prm, stream, out);
}

afn_status afn_matvec(afn_handle h, const double* v, double* y, void* stream) {
  REQ(h != nullptr, "null handle");
  REQ(is_dev(v) && is_dev(y) && v != y, "v, y must be distinct device pointers");
  cudaStream_t st = (cudaStream_t)stream;
  for (auto& s : h->rk) TRY(gather_vec(v, s.perm, h->n, s.rbuf, st));
  TRY(matvec_perm(h, [](RankSt& s) { return s.rbuf; }, [](RankSt& s) { return s.zbuf; }, -1, st));
  TRY(exchange(h, [](RankSt& s) { return s.zbuf; }, [&](int s) { return vec_ranges(h, s); }, st));
  TRY(scatter_vec(h->rk[0].zbuf, h->rk[0].perm, h->n, y, st));
  return AFN_OK;
}

afn_status afn_apply(afn_handle h, const double* r, double* z, void* stream) {
  REQ(h != nullptr, "null handle");
  REQ(is_dev(r) && is_dev(z) && r != z, "r, z must be distinct device pointers");
  cudaStream_t st = (cudaStream_t)stream;
  for (auto& s : h->rk) TRY(gather_vec(r, s.perm, h->n, s.rbuf, st));
  TRY(apply_perm(h, [](RankSt& s) { return s.rbuf; }, [](RankSt& s) { return s.zbuf; }, st));
  TRY(exchange(h, [](RankSt& s) { return s.zbuf; }, [&](int s) { return vec_ranges(h, s); }, st));
  TRY(scatter_vec(h->rk[0].zbuf, h->rk[0].perm, h->n, z, st));
  return AFN_OK;
}

afn_status afn_pcg_solve(afn_handle h, const double* b, double* a, double tol, int32_t maxit,
                         int32_t fixed_iters, afn_solve_report* rep, void* stream) {
  REQ(h != nullptr, "null handle");
  REQ(is_dev(b) && is_dev(a) && a != b, "b, a must be distinct device pointers");
  REQ(tol > 0 && tol < 1, "need 0 < tol < 1");
  REQ(maxit >= 1, "maxit must be >= 1");
  REQ(fixed_iters >= 0, "fixed_iters must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = h->n;
  const int d = h->d;
  afn_solve_report R{};
  if (rep) R.history = rep->history;
  double* hsc = pinned_scalars();
  if (!hsc) {
    set_error("pinned host allocation failed");
    return AFN_ERR_NOMEM;
  }
  cudaEvent_t e0, e1, ap0, ap1;
  AFN_CUDA(cudaEventCreate(&e0));
  AFN_CUDA(cudaEventCreate(&e1));
  AFN_CUDA(cudaEventCreate(&ap0));
  AFN_CUDA(cudaEventCreate(&ap1));
  struct EvG {
    cudaEvent_t e[4];
    ~EvG() { for (auto x : e) cudaEventDestroy(x); }
  } evg{{e0, e1, ap0, ap1}};
  EvPairs cm;  // the per-iteration all-gathers of p (multi-rank)
  double mv_ms = 0.0, ap_ms = 0.0;
  int napply = 0;
  auto sc_to_host = [&]() -> afn_status {
    AFN_CUDA(cudaMemcpyAsync(hsc, h->rk[0].sc, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, st));
    TRY(comm_stream_sync(h->comm, st));
    return AFN_OK;
  };
  auto apply = [&]() -> afn_status {
    return apply_perm(h, [](RankSt& s) { return s.r; }, [](RankSt& s) { return s.z; }, st);
  };
  AFN_CUDA(cudaEventRecord(e0, st));

  // r = b (permuted), x = 0
  for (auto& s : h->rk) {
    TRY(gather_vec(b, s.perm, n, s.r, st));
    AFN_CUDA(cudaMemsetAsync(s.x, 0, sizeof(double) * n, st));
    TRY(dot(s.r, s.r, s.own, part_dst(h, s, SC_BB), s.dws, s.dcnt, st));
  }
  TRY(reduce_slots(h, 1u << SC_BB, st));
  TRY(sc_to_host());
  const double nb = std::sqrt(hsc[SC_BB]);
  if (R.history) R.history[0] = nb > 0 ? 1.0 : 0.0;
  int it = 0;
  double rel = nb > 0 ? 1.0 : 0.0;
  if (nb > 0) {
    // Iterations are queued in chunks (1, 2, 4, then PCG_CHUNK) with the
    // stopping test on the device (pcg_check: the same test as P:L788's loop,
    // history written on the device); the matvec and apply kernels of queued
    // iterations after the stop return at once (skip flag sc[SC_DONE]), x and
    // r stay at the stopping iterate.  One host round trip per chunk instead
    // of one per iteration.
    constexpr int PCG_CHUNK = 8;
    double* dhist = nullptr;
    TRY(dalloc((void**)&dhist, sizeof(double) * ((size_t)maxit + 1), st));
    struct HFree {
      double* p;
      cudaStream_t st;
      ~HFree() { dfree(p, st); }
    } hfree{dhist, st};
    for (auto& s : h->rk) AFN_CUDA(cudaMemsetAsync(s.sc + SC_DONE, 0, sizeof(double) * 3, st));  // DONE, ITS, IT
    std::vector<cudaEvent_t> evs;  // per queued iteration: kmv begin/end, apply begin/end
    struct EvFree {
      std::vector<cudaEvent_t>* v;
      ~EvFree() { for (auto e : *v) cudaEventDestroy(e); }
    } evfree{&evs};
    auto new_ev = [&]() -> cudaEvent_t {
      cudaEvent_t e;
      cudaEventCreate(&e);
      evs.push_back(e);
      return e;
    };
    AFN_CUDA(cudaEventRecord(ap0, st));
    TRY(apply());
    AFN_CUDA(cudaEventRecord(ap1, st));
    int cur = SC_RZ0;
    for (auto& s : h->rk) TRY(dot(s.r, s.z, s.own, part_dst(h, s, cur), s.dws, s.dcnt, st));
    TRY(reduce_slots(h, 1u << cur, st));
    for (auto& s : h->rk) TRY(vec_copy(s.p, s.z, s.own, st));
    int queued = 0, chunk = 1, code = 0;
    // per queued iteration: kmv begin/end, apply begin/end (host-side loop) ...
    std::vector<cudaEvent_t> kmE, apE;
    double kmv_ms_acc = 0.0, ap_ms_acc = 0.0;
    int kmv_seen = 0;  // host-loop iterations queued so far (index into kmE / apE)
    // ... and a CUDA graph of PCG_CHUNK iterations (one rank): captured once per
    // solve, replayed per chunk (the iteration number lives on the device);
    // its event nodes are read after each replay.
    cudaGraphExec_t gexec = nullptr;
    int64_t glaunches = 0;
    std::vector<cudaEvent_t> gE;
    cudaEvent_t gj0 = nullptr, gj1 = nullptr;
    struct GFree {
      cudaGraphExec_t* g;
      std::vector<cudaEvent_t>* e;
      cudaEvent_t* j0;
      cudaEvent_t* j1;
      ~GFree() {
        if (*g) cudaGraphExecDestroy(*g);
        for (auto x : *e) cudaEventDestroy(x);
        if (*j0) cudaEventDestroy(*j0);
        if (*j1) cudaEventDestroy(*j1);
      }
    } gfree{&gexec, &gE, &gj0, &gj1};
    // one iteration; events ek0..ea1 bracket the matvec and the apply; kt: per-launch timers
    auto enqueue_iter = [&](cudaEvent_t ek0, cudaEvent_t ek1, cudaEvent_t ea0, cudaEvent_t ea1,
                            bool kt) -> afn_status {
      // (in a capture, kt == false: event record nodes need cudaEventRecordExternal)
      const unsigned ef = kt ? cudaEventRecordDefault : cudaEventRecordExternal;
      AFN_CUDA(cudaEventRecordWithFlags(ek0, st, ef));
      if (h->R > 1) {  // p: every rank's rows (the north star's per-iteration all-gather)
        AFN_CUDA(cudaEventRecord(cm.next(), st));
        TRY(exchange(h, [](RankSt& s) { return s.p; }, [&](int s) { return vec_ranges(h, s); }, st));
        AFN_CUDA(cudaEventRecord(cm.next(), st));
      }
      // one rank with the symmetric matvec: p.q fused into the matvec's reduce,
      // the stopping test fused into the x/r update
      const bool fused = h->R == 1 && h->rk[0].plan.sym;
      if (kt) kt_begin(KT_KMV, st);
      TRY(matvec_perm(h, [](RankSt& s) { return s.p; }, [](RankSt& s) { return s.q; }, SC_PQ, st));
      if (kt) kt_end(KT_KMV, st, kmv_work(h, n, d));
      AFN_CUDA(cudaEventRecordWithFlags(ek1, st, ef));
      if (fused) {
        RankSt& s = h->rk[0];
        TRY(pcg_update_xr_check(s.x, s.r, s.p, s.q, s.own, s.sc, cur, s.dws, s.dcnt, nb, tol, maxit, fixed_iters,
                                dhist, st));
      } else {
        TRY(reduce_slots(h, 1u << SC_PQ, st));
        for (auto& s : h->rk)
          TRY(pcg_update_xr(s.x, s.r, s.p, s.q, s.own, s.sc, cur, part_dst(h, s, SC_RR), s.dws, s.dcnt, st));
        TRY(reduce_slots(h, 1u << SC_RR, st));
        for (auto& s : h->rk) TRY(pcg_check(s.sc, nb, tol, maxit, fixed_iters, dhist, st));
      }
      AFN_CUDA(cudaEventRecordWithFlags(ea0, st, ef));
      if (kt) kt_begin(KT_APPLY, st);
      TRY(apply());
      if (kt) kt_end(KT_APPLY, st, apply_bytes(h) / h->R);
      AFN_CUDA(cudaEventRecordWithFlags(ea1, st, ef));
      const int nxt = cur ^ 1;
      for (auto& s : h->rk) TRY(dot(s.r, s.z, s.own, part_dst(h, s, nxt), s.dws, s.dcnt, st));
      TRY(reduce_slots(h, 1u << nxt, st));
      for (auto& s : h->rk) TRY(pcg_update_p(s.p, s.z, s.own, s.sc, nxt, cur, st));
      cur = nxt;
      return AFN_OK;
    };
    while (queued < maxit) {
      const int upto = std::min(maxit, queued + chunk);
      set_skip(h->rk[0].sc + SC_DONE);
      struct SkipOff {
        ~SkipOff() { set_skip(nullptr); }
      } skipoff;
      const bool graph = h->R == 1 && chunk == PCG_CHUNK && upto - queued == PCG_CHUNK &&
                         (PCG_CHUNK & 1) == 0;
      if (graph) {
        // capture / replay on a private non-blocking stream (the caller's
        // stream may be the legacy default stream, which cannot capture),
        // ordered after and before the caller's stream by events
        const cudaStream_t user_st = st;
        cudaStream_t gs = graph_stream();
        if (!gj0) {
          AFN_CUDA(cudaEventCreateWithFlags(&gj0, cudaEventDisableTiming));
          AFN_CUDA(cudaEventCreateWithFlags(&gj1, cudaEventDisableTiming));
        }
        AFN_CUDA(cudaEventRecord(gj0, user_st));
        AFN_CUDA(cudaStreamWaitEvent(gs, gj0, 0));
        st = gs;
        struct Restore {
          cudaStream_t* p;
          cudaStream_t v;
          ~Restore() { *p = v; }
        } restore{&st, user_st};
        if (!gexec) {  // capture PCG_CHUNK iterations (cur returns to its value: even count)
          for (int e = 0; e < 4 * PCG_CHUNK; ++e) {
            cudaEvent_t x;
            AFN_CUDA(cudaEventCreate(&x));
            gE.push_back(x);
          }
          cudaGraph_t g = nullptr;
          const int64_t l0 = afn_launch_count();
          AFN_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          afn_status cs = AFN_OK;
          for (int t = 0; t < PCG_CHUNK && cs == AFN_OK; ++t)
            cs = enqueue_iter(gE[4 * t], gE[4 * t + 1], gE[4 * t + 2], gE[4 * t + 3], false);
          const cudaError_t ce = cudaStreamEndCapture(st, &g);
          if (cs != AFN_OK) {
            if (g) cudaGraphDestroy(g);
            return cs;
          }
          AFN_CUDA(ce);
          const cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
          cudaGraphDestroy(g);
          AFN_CUDA(ie);
          glaunches = afn_launch_count() - l0;  // kernels per replay
          note_launch((int)-glaunches);          // (counted per replay below)
        }
        AFN_CUDA(cudaGraphLaunch(gexec, st));
        note_launch((int)glaunches);
        AFN_CUDA(cudaEventRecord(gj1, gs));
        AFN_CUDA(cudaStreamWaitEvent(user_st, gj1, 0));
      } else {
        for (int t = queued + 1; t <= upto; ++t) {
          kmE.push_back(new_ev());
          kmE.push_back(new_ev());
          apE.push_back(new_ev());
          apE.push_back(new_ev());
          TRY(enqueue_iter(kmE[kmE.size() - 2], kmE.back(), apE[apE.size() - 2], apE.back(), true));
        }
      }
      TRY(sc_to_host());
      code = (int)hsc[SC_DONE];
      // the chunk's iterations that really ran (the rest returned at once)
      const int its_now = code != 0 ? (int)hsc[SC_ITS] : upto;
      const int kmv_last = std::min(upto, its_now + (code == 2 ? 1 : 0));
      const int ap_last = code == 0 ? upto : std::min(upto, its_now - 1 + (code == 2 || code == 3 ? 1 : 0));
      if (graph) {
        for (int t = queued + 1; t <= upto; ++t) {
          const int q = t - queued - 1;
          if (t <= kmv_last) {
            const double ms = ev_ms(gE[4 * q], gE[4 * q + 1]);
            kmv_ms_acc += ms;
            kt_add(KT_KMV, ms, kmv_work(h, n, d));
          }
          if (t <= ap_last) {
            const double ms = ev_ms(gE[4 * q + 2], gE[4 * q + 3]);
            ap_ms_acc += ms;
            kt_add(KT_APPLY, ms, apply_bytes(h) / h->R);
          }
        }
      } else {
        for (int t = queued + 1; t <= upto; ++t) {
          const size_t q = (size_t)(kmv_seen + (t - queued - 1));
          if (t <= kmv_last) kmv_ms_acc += ev_ms(kmE[2 * q], kmE[2 * q + 1]);
          if (t <= ap_last) ap_ms_acc += ev_ms(apE[2 * q], apE[2 * q + 1]);
        }
        kt_drop_last(KT_KMV, upto - std::max(queued, kmv_last));
        kt_drop_last(KT_APPLY, upto - std::max(queued, ap_last));
        kmv_seen += upto - queued;
      }
      queued = upto;
      if (code != 0) break;
      chunk = std::min(chunk * 2, PCG_CHUNK);
    }
    if (code == 0) {  // (cannot happen: the check stops at maxit)
      set_error("pcg: no stop after maxit");
      return AFN_ERR_STATE;
    }
    it = (int)hsc[SC_ITS];
    R.breakdown = code == 2;
    // launches that really ran: the matvec of every iteration up to the stop
    // (breakdown: also the failing one), the apply of every iteration that
    // continued (breakdown and maxit exhaustion: also the last one)
    const int kmv_real = it + (code == 2 ? 1 : 0);
    const int ap_real = it - 1 + (code == 2 || code == 3 ? 1 : 0);
    napply = 1 + ap_real;
    std::vector<double> hh((size_t)it + 1, 0.0);
    if (it > 0) {
      AFN_CUDA(cudaMemcpyAsync(hh.data(), dhist, sizeof(double) * ((size_t)it + 1), cudaMemcpyDeviceToHost, st));
      AFN_CUDA(cudaStreamSynchronize(st));
      rel = hh[it];
    }
    if (R.history)
      for (int t = 1; t <= it; ++t) R.history[t] = hh[t];
    R.converged = code == 1 && rel <= tol;
    (void)kmv_real;
    mv_ms = kmv_ms_acc;
    ap_ms = ev_ms(ap0, ap1) + ap_ms_acc;
  } else {
    R.converged = 1;
  }
  // a = x (all ranks' rows, un-permuted); true residual ||b - (K + mu I) x|| / ||b||
  TRY(exchange(h, [](RankSt& s) { return s.x; }, [&](int s) { return vec_ranges(h, s); }, st));
  TRY(scatter_vec(h->rk[0].x, h->rk[0].perm, n, a, st));
  AFN_CUDA(cudaEventRecord(e1, st));
  if (nb > 0) {
    TRY(matvec_perm(h, [](RankSt& s) { return s.x; }, [](RankSt& s) { return s.q; }, -1, st));
    for (auto& s : h->rk) {
      TRY(gather_vec(b, s.perm, n, s.z, st));
      TRY(vec_axpby(s.z, -1.0, s.q, 1.0, s.own, st));
      TRY(dot(s.z, s.z, s.own, part_dst(h, s, SC_TMP), s.dws, s.dcnt, st));
    }
    TRY(reduce_slots(h, 1u << SC_TMP, st));
  }
  TRY(sc_to_host());
  R.iterations = it;
  R.relres = rel;
  R.relres_true = nb > 0 ? std::sqrt(hsc[SC_TMP]) / nb : 0.0;
  R.solve_ms = ev_ms(e0, e1);
  R.matvec_ms = mv_ms;
  R.apply_ms = ap_ms;
  R.comm_ms = cm.total_ms();
  kt_collect();
  R.applies = napply;
  if (rep) *rep = R;
  return AFN_OK;
}

afn_status afn_cg_solve(afn_comm comm, const double* X, int64_t n, int32_t d, int32_t kernel, double l,
                        double mu, const double* b, double* a, double tol, int32_t maxit, int32_t fixed_iters,
                        afn_solve_report* rep, void* stream) {
  afn_params P{};
  P.l = l;
  P.mu = mu;
  P.k_cap = 1;
  P.w = 1;
  P.kernel = kernel;
  P.method = AFN_METHOD_NONE;
  afn_handle h = nullptr;
  TRY(build_impl(comm, X, n, d, &P, stream, &h));
  const afn_status s = afn_pcg_solve(h, b, a, tol, maxit, fixed_iters, rep, stream);
  afn_destroy(h);
  return s;
}

afn_status afn_solve_host(afn_comm comm, const double* X, const double* b, double* a, int64_t n, int32_t d,
                          const afn_params* params, double tol, int32_t maxit, afn_info* info,
                          afn_solve_report* rep, void* stream) {
  REQ(X && b && a && params, "X, b, a, params must be non-null host pointers");
  REQ(n >= 1 && d >= 1 && d <= 16, "bad n or d");
  cudaStream_t st = (cudaStream_t)stream;
  Temps t(st);
  double *dX, *db, *da;
  TRY(t.get(&dX, (size_t)n * d));
  TRY(t.get(&db, (size_t)n));
  TRY(t.get(&da, (size_t)n));
  AFN_CUDA(cudaMemcpyAsync(dX, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, st));
  AFN_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  afn_handle h = nullptr;
  TRY(build_impl(comm, dX, n, d, params, stream, &h));
  afn_status s = afn_pcg_solve(h, db, da, tol, maxit, 0, rep, stream);
  if (s == AFN_OK && info) s = afn_get_info(h, info);
  if (s == AFN_OK) {
    cudaError_t e = cudaMemcpyAsync(a, da, sizeof(double) * n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) s = cuda_status(e, "afn_solve_host copy-out");
  }
  afn_destroy(h);
  return s;
}

afn_status afn_get_info(afn_handle h, afn_info* info) {
  REQ(h && info, "null argument");
  afn_info I{};
  I.n = h->n;
  I.k = h->k;
  I.khat = h->params.k_adaptive ? h->a1.khat : h->k;
  I.nnz = h->nnz;
  I.d = h->d;
  I.r = h->a1.r;
  I.m = h->a1.m;
  I.refined = h->a1.refined;
  I.scale = h->a1.scale;
  I.ms_alg1 = h->ms[0];
  I.ms_fps = h->ms[1];
  I.ms_chol = h->ms[2];
  I.ms_trsm = h->ms[3];
  I.ms_knn = h->ms[4];
  I.ms_fsai = h->ms[5];
  I.ms_total = h->ms[6];
  I.ms_fsai_rows = h->ms[7];
  I.nranks = h->R;
  I.rank = h->rk[0].rank;
  I.row_a0 = h->rk[0].own.a0;
  I.row_na = h->rk[0].own.na;
  I.row_b0 = h->rk[0].own.b0;
  I.row_nb = h->rk[0].own.nb;
  I.kernel = h->kn.kind;
  I.method = h->method;
  const KmvPlan& kp = h->rk[0].plan;
  I.kmv_plan = kp.cut ? 2 : (kp.sym ? 1 : 0);
  I.kmv_units64 = kp.cut ? kp.cut_u64 : kp.sym_units;
  I.kmv_units32 = 0;  // (cutoff plan: classes are per warp; see the pairs)
  I.kmv_pairs64 = kp.cut ? kp.cut_pairs64 : (kp.sym ? (double)h->n * (double)(h->n - 1) / 2.0 : 0.0);
  I.kmv_pairs32 = kp.cut_pairs32;
  *info = I;
  return AFN_OK;
}

// W on demand (one rank, Z mode: not formed by the build) from the kept plan
static afn_status ensure_w(afn_handle h, RankSt& s) {
  if (s.W || !s.kt.used || h->N2 <= 0) return AFN_OK;
  TRY(ralloc(s, &s.W, (size_t)h->N2 * h->k, h->stream));
  TRY(w_cut_run(&s.kt, s.LinvT, s.W, h->stream));
  AFN_CUDA(cudaStreamSynchronize(h->stream));
  return AFN_OK;
}

afn_status afn_copy_out_local(afn_handle h, int32_t local_rank, int32_t what, void* host, size_t bytes) {
  REQ(h && host, "null argument");
  REQ(local_rank >= 0 && local_rank < (int)h->rk.size(), "local rank %d out of range", local_rank);
  if (what == AFN_OUT_W) TRY(ensure_w(h, h->rk[local_rank]));
  const RankSt& s = h->rk[local_rank];
  const void* src = nullptr;
  size_t need = 0;
  switch (what) {
    case AFN_OUT_PERM: src = s.perm; need = sizeof(int64_t) * h->n; break;
    case AFN_OUT_FILL: src = s.fill; need = sizeof(double) * h->k; break;
    case AFN_OUT_L: src = s.L; need = sizeof(double) * h->k * h->k; break;
    case AFN_OUT_ROWPTR: src = s.rp; need = sizeof(int64_t) * (h->N2 + 1); break;
    case AFN_OUT_COL: src = s.col; need = sizeof(int32_t) * h->nnz; break;
    case AFN_OUT_GVAL: src = s.gval; need = sizeof(double) * h->nnz; break;
    case AFN_OUT_W: src = s.W; need = sizeof(double) * (s.hi - s.lo) * h->k; break;
    default: set_error("unknown copy_out selector %d", what); return AFN_ERR_ARG;
  }
  REQ(bytes == need, "copy_out: bytes=%zu, need %zu", bytes, need);
  if (need == 0) return AFN_OK;
  AFN_CUDA(cudaMemcpy(host, src, need, cudaMemcpyDeviceToHost));
  return AFN_OK;
}

afn_status afn_copy_out(afn_handle h, int32_t what, void* host, size_t bytes) {
  return afn_copy_out_local(h, 0, what, host, bytes);
}

afn_status afn_copy_out_rows(afn_handle h, int32_t what, const int64_t* rows, int64_t nrows,
                             void* host, size_t bytes) {
  REQ(h && host && (rows || nrows == 0) && nrows >= 0, "null argument");
  if (what == AFN_OUT_W) TRY(ensure_w(h, h->rk[0]));
  const RankSt& s = h->rk[0];
  const double* src = nullptr;
  int64_t lo = 0, hi = 0;
  if (what == AFN_OUT_W) src = s.W, lo = s.lo, hi = s.hi;
  else if (what == AFN_OUT_L) src = s.L, lo = 0, hi = h->k;
  else REQ(false, "copy_out_rows: selector %d unsupported (W or L only)", what);
  const size_t rowb = sizeof(double) * (size_t)h->k;
  REQ(bytes == rowb * (size_t)nrows, "copy_out_rows: bytes=%zu, need %zu", bytes,
      rowb * (size_t)nrows);
  for (int64_t t = 0; t < nrows; ++t)
    REQ(rows[t] >= lo && rows[t] < hi, "copy_out_rows: row %lld out of range [%lld, %lld)",
        (long long)rows[t], (long long)lo, (long long)hi);
  for (int64_t t = 0; t < nrows; ++t)
    AFN_CUDA(cudaMemcpy(static_cast<char*>(host) + rowb * t, src + (size_t)(rows[t] - lo) * h->k, rowb,
                        cudaMemcpyDeviceToHost));
  return AFN_OK;
}

void afn_destroy(afn_handle h) { handle_free(h); }

afn_status afn_probe_dmma(int64_t iters, double* tflops, void* stream) {
  REQ(iters >= 8 && tflops, "bad arguments");
  return probe_dmma(iters, tflops, (cudaStream_t)stream);
}

afn_status afn_probe_dfma(int64_t iters, double* tflops, void* stream) {
  REQ(iters >= 8 && tflops, "bad arguments");
  return probe_dfma(iters, tflops, (cudaStream_t)stream);
}

afn_status afn_probe_ex2(int64_t iters, double* gops, void* stream) {
  REQ(iters >= 8 && gops, "bad arguments");
  return probe_ex2(iters, gops, (cudaStream_t)stream);
}

afn_status afn_set_cutoff_mode(int32_t mode) {
  REQ(mode >= 0 && mode <= 3, "cutoff mode %d (0 auto, 1 never, 2 whenever it applies, 3 auto without Z)", mode);
  kmv_set_mode(mode);
  return AFN_OK;
}

}  // extern "C"

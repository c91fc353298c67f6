// abi.cu -- the C ABI of include/afn.h: argument validation, the built handle
// (device-resident L^{-T}, W, G, G^T, permuted points), the build pipeline
// (P:L207-263), the apply and the PCG driver.
#include <atomic>
#include <cmath>
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
  }
  done[dev] = true;
}

afn_status dalloc(void** p, size_t bytes, cudaStream_t st) {
  pool_setup_once();
  *p = nullptr;
  cudaError_t e = cudaMallocAsync(p, bytes > 0 ? bytes : 8, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
    return AFN_ERR_NOMEM;
  }
  return AFN_OK;
}

void dfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
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
struct afn_handle_s {
  int device = 0;
  int64_t n = 0, k = 0, N2 = 0, nnz = 0;
  int d = 0;
  double l = 0, mu = 0;
  afn_params params{};
  Alg1Result a1{};
  // device arrays
  int64_t* perm = nullptr;
  double* fill = nullptr;
  double* Xp = nullptr;     // permuted points n x d
  double* Xs = nullptr;     // prescaled permuted points (kmv)
  double* L = nullptr;      // k x k lower (row-major)
  double* LinvT = nullptr;  // k x k, L^{-T}
  double* W = nullptr;      // N2 x k
  int64_t* rp = nullptr;
  int32_t* col = nullptr;
  double* gval = nullptr;
  int64_t* trp = nullptr;
  int32_t* tcol = nullptr;
  double* tval = nullptr;
  // workspaces
  KmvPlan plan{};
  double* kmv_part = nullptr;
  double* gws = nullptr;  // gemv_t partials
  double* tvec = nullptr;  // k
  double* vvec = nullptr;  // k
  double* uvec = nullptr;  // N2
  double* yvec = nullptr;  // N2
  double* rbuf = nullptr;  // n (public apply)
  double* zbuf = nullptr;  // n
  // pcg
  double* x = nullptr;
  double* r = nullptr;
  double* z = nullptr;
  double* p = nullptr;
  double* q = nullptr;
  double* sc = nullptr;
  double* dws = nullptr;
  unsigned* dcnt = nullptr;
  double* h_sc = nullptr;  // pinned host mirror of sc (per host thread, not owned)
  std::vector<void*> allocs;
  double ms[8] = {0};
};

namespace {

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

afn_status halloc(afn_handle h, void** p, size_t bytes, cudaStream_t st) {
  afn_status s = dalloc(p, bytes, st);
  if (s == AFN_OK) h->allocs.push_back(*p);
  return s;
}

void handle_free(afn_handle h) {
  if (!h) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  // return the blocks to the stream-ordered pool (cudaFree would unmap them and
  // force the next build to map fresh pages); the legacy stream orders the
  // frees after all prior work on the device's blocking streams
  for (void* p : h->allocs) cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
  cudaSetDevice(cur);
  delete h;
}

// algorithmic HBM bytes of one apply: W read twice, L^{-T} twice (upper half),
// G and G^T (values + 4-byte columns) once each, plus the vectors
double apply_bytes(afn_handle h) {
  const double k = (double)h->k, N2 = (double)h->N2, nnz = (double)h->nnz;
  return 8.0 * (2.0 * N2 * k + k * (k + 1.0)) + 2.0 * 12.0 * nnz + 8.0 * (6.0 * N2 + 6.0 * k);
}

// z = M^{-1} r in the permuted order (V-form)
afn_status apply_perm(afn_handle h, const double* r, double* z, cudaStream_t st) {
  const int64_t k = h->k, N2 = h->N2;
  // t = L^{-1} r1 = (L^{-T})^T r1
  TRY(gemv_t(h->LinvT, k, k, r, nullptr, 1.0, h->tvec, h->gws, st));
  if (N2 > 0) {
    // u = r2 - W t
    TRY(gemv_n(h->W, N2, k, h->tvec, r + k, -1.0, h->uvec, st));
    // y = G u ; s2 = G^T y
    TRY(spmv_csr(h->rp, h->col, h->gval, N2, h->uvec, h->yvec, st));
    TRY(spmv_csr(h->trp, h->tcol, h->tval, N2, h->yvec, z + k, st));
    // v = t - W^T s2
    TRY(gemv_t(h->W, N2, k, z + k, h->tvec, -1.0, h->vvec, h->gws, st));
    // s1 = L^{-T} v
    TRY(gemv_n(h->LinvT, k, k, h->vvec, nullptr, 1.0, z, st));
  } else {
    TRY(gemv_n(h->LinvT, k, k, h->tvec, nullptr, 1.0, z, st));
  }
  return AFN_OK;
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

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int32_t afn_abi_version(void) { return AFN_ABI_VERSION; }

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

afn_status kernel_matvec_rows(const double* X, int64_t n, int32_t d, double l, double mu,
                              const double* v, int64_t row0, int64_t nrows, double* y, void* stream) {
  TRY(validate_X(X, n, d));
  REQ(l > 0 && std::isfinite(l), "l must be > 0");
  REQ(mu >= 0 && std::isfinite(mu), "mu must be >= 0");
  REQ(row0 >= 0 && nrows >= 0 && row0 + nrows <= n, "row range out of bounds");
  REQ(is_dev(v) && (nrows == 0 || is_dev(y)), "v, y must be device pointers");
  REQ(y != v, "y must not alias v");
  cudaStream_t st = (cudaStream_t)stream;
  Temps t(st);
  double* Xs;
  TRY(t.get(&Xs, (size_t)n * d));
  TRY(kmv_prescale(X, n, d, l, Xs, st));
  KmvPlan plan = kmv_plan(n, nrows, d, num_sms());
  double* part;
  TRY(t.get(&part, (size_t)plan.chunks * (nrows > 0 ? nrows : 1)));
  TRY(kmv_launch(Xs, n, d, v, mu, row0, nrows, y, part, plan, st));
  return AFN_OK;
}

afn_status kernel_matvec(const double* X, int64_t n, int32_t d, double l, double mu, const double* v,
                         double* y, void* stream) {
  return kernel_matvec_rows(X, n, d, l, mu, v, 0, n, y, stream);
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

afn_status afn_knn_pattern(const double* P, int64_t N, int32_t d, int32_t w, int64_t* row_ptr,
                           int32_t* col, void* stream) {
  TRY(validate_X(P, N, d));
  REQ(w >= 1 && w <= 128, "w must be in 1..128");
  REQ(N <= 0x7fffffffLL, "N must fit int32 column indices");
  REQ(is_dev(row_ptr) && is_dev(col), "row_ptr, col must be device pointers");
  return knn_run(P, N, d, w, row_ptr, col, (cudaStream_t)stream);
}

afn_status afn_estimate_rank(const double* X, int64_t n, int32_t d, double l, int32_t m,
                             uint64_t rng_seed, int32_t k_threshold, int64_t* khat, int32_t* r,
                             int32_t* refined, void* stream) {
  TRY(validate_X(X, n, d));
  REQ(l > 0 && std::isfinite(l), "l must be > 0");
  if (m == 0) m = alg1_default_m(n);
  REQ(m >= 2 && m <= n && m <= 1024, "need 2 <= m <= min(n, 1024)");
  REQ(k_threshold >= 1, "k_threshold must be >= 1");
  REQ(khat && r && refined, "outputs must be non-null host pointers");
  Alg1Result res;
  TRY(alg1_run(X, n, d, l, m, rng_seed, k_threshold, &res, (cudaStream_t)stream));
  *khat = res.khat;
  *r = res.r;
  *refined = res.refined;
  return AFN_OK;
}

afn_status afn_build(const double* X, int64_t n, int32_t d, const afn_params* prm, void* stream,
                     afn_handle* out) {
  REQ(out != nullptr, "out must be non-null");
  *out = nullptr;
  TRY(validate_X(X, n, d));
  REQ(prm != nullptr, "params must be non-null");
  const afn_params P = *prm;
  REQ(P.l > 0 && std::isfinite(P.l), "l must be > 0");
  REQ(P.mu > 0 && std::isfinite(P.mu), "mu must be > 0");
  REQ(P.k_cap >= 1, "k_cap must be >= 1");
  REQ(P.w >= 1 && P.w <= 128, "w must be in 1..128");
  REQ(P.fps_seed >= 0 && P.fps_seed < n, "need 0 <= fps_seed < n");
  REQ(n <= 0x7fffffffLL, "n must fit int32 indices");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  AFN_CUDA(cudaGetDevice(&dev));

  cudaEvent_t ev[8];
  for (auto& e : ev) AFN_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 8; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};

  afn_handle h = new afn_handle_s();
  h->device = dev;
  h->n = n;
  h->d = d;
  h->l = P.l;
  h->mu = P.mu;
  h->params = P;
  struct HGuard {
    afn_handle* hp;
    ~HGuard() {
      if (*hp) handle_free(*hp);
    }
  } hg{&h};

  AFN_CUDA(cudaEventRecord(ev[0], st));
  // ---- a2: adaptive k (Alg. 1)
  int64_t k = std::min<int64_t>(P.k_cap, n);
  if (P.k_adaptive) {
    int m = P.m > 0 ? P.m : alg1_default_m(n);
    REQ(m >= 2 && m <= n && m <= 1024, "need 2 <= m <= min(n, 1024)");
    TRY(alg1_run(X, n, d, P.l, m, P.rng_seed, P.k_threshold > 0 ? P.k_threshold : 2000, &h->a1, st));
    k = std::min<int64_t>(P.k_cap, std::max<int64_t>(1, h->a1.khat));
    k = std::min<int64_t>(k, n);
  }
  h->k = k;
  h->N2 = n - k;
  AFN_CUDA(cudaEventRecord(ev[1], st));

  // ---- a3: FPS
  int64_t* idx;
  TRY(halloc(h, (void**)&idx, sizeof(int64_t) * k, st));
  TRY(halloc(h, (void**)&h->fill, sizeof(double) * k, st));
  kt_begin(KT_FPS, st);
  TRY(fps_run(X, n, d, k, P.fps_seed, idx, h->fill, st));
  kt_end(KT_FPS, st, 0.0);
  AFN_CUDA(cudaEventRecord(ev[2], st));

  // ---- a1: permutation, permuted + prescaled points
  int* derr;
  TRY(halloc(h, (void**)&derr, sizeof(int) * 4, st));
  AFN_CUDA(cudaMemsetAsync(derr, 0, sizeof(int) * 4, st));
  {
    unsigned char* flag;
    unsigned* flag32;
    TRY(halloc(h, (void**)&flag, (size_t)n, st));
    TRY(halloc(h, (void**)&flag32, sizeof(unsigned) * (size_t)n, st));
    AFN_CUDA(cudaMemsetAsync(flag32, 0, sizeof(unsigned) * (size_t)n, st));
    mark_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(idx, k, n, flag32, derr);
    AFN_LAUNCH_CHECK("mark_kernel");
    flag8_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(flag32, n, flag);
    AFN_LAUNCH_CHECK("flag8_kernel");
    TRY(halloc(h, (void**)&h->perm, sizeof(int64_t) * n, st));
    perm_kernel<<<1, 1024, 0, st>>>(flag, idx, n, k, h->perm);
    AFN_LAUNCH_CHECK("perm_kernel");
  }
  TRY(halloc(h, (void**)&h->Xp, sizeof(double) * n * d, st));
  TRY(gather_rows(X, n, d, h->perm, h->Xp, st));
  TRY(halloc(h, (void**)&h->Xs, sizeof(double) * n * d, st));
  TRY(kmv_prescale(h->Xp, n, d, P.l, h->Xs, st));

  // ---- a4: L L^T = K11 + mu I ; L^{-T}
  TRY(halloc(h, (void**)&h->L, sizeof(double) * k * k, st));
  TRY(gen_k11(h->Xp, k, d, P.l, P.mu, h->L, st));
  int* dinfo;
  TRY(halloc(h, (void**)&dinfo, sizeof(int) * 2, st));
  AFN_CUDA(cudaMemsetAsync(dinfo, 0, sizeof(int) * 2, st));
  kt_begin(KT_POTRF, st);
  TRY(potrf_lower(h->L, k, dinfo, st));
  kt_end(KT_POTRF, st, (double)k * k * k / 3.0);
  TRY(halloc(h, (void**)&h->LinvT, sizeof(double) * k * k, st));
  kt_begin(KT_LINV, st);
  TRY(trsm_linvt(h->L, k, h->LinvT, st));
  kt_end(KT_LINV, st, (double)k * k * k / 3.0);
  AFN_CUDA(cudaEventRecord(ev[3], st));
  {
    int info = 0;
    AFN_CUDA(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    AFN_CUDA(cudaStreamSynchronize(st));
    if (info) {
      set_error("Cholesky of K11 + mu I broke down at row %d", info - 1);
      return AFN_ERR_NOT_SPD;
    }
  }

  const int64_t N2 = h->N2;
  const double* X2 = h->Xp + k * d;
  // ---- a5: W = K21 L^{-T}
  TRY(halloc(h, (void**)&h->W, sizeof(double) * (size_t)(N2 > 0 ? N2 : 1) * k, st));
  static const bool w_trsm = getenv("AFN_W_TRSM") != nullptr;
  if (w_trsm) TRY(trsm_w(h->L, k, h->Xp, X2, N2, d, P.l, h->W, st));
  else {
    kt_begin(KT_W_GEMM, st);
    TRY(w_gemm(h->LinvT, k, h->Xp, X2, N2, d, P.l, h->W, st));
    kt_end(KT_W_GEMM, st, (double)N2 * (double)k * (double)k);  // N2 k^2/2 FMA
  }
  AFN_CUDA(cudaEventRecord(ev[4], st));

  // ---- a6: kNN pattern
  h->nnz = knn_nnz(N2, P.w);
  TRY(halloc(h, (void**)&h->rp, sizeof(int64_t) * (N2 + 1), st));
  TRY(halloc(h, (void**)&h->col, sizeof(int32_t) * (h->nnz > 0 ? h->nnz : 1), st));
  if (N2 > 0) {
    kt_begin(KT_KNN, st);
    TRY(knn_run(X2, N2, d, P.w, h->rp, h->col, st));
    kt_end(KT_KNN, st, 0.0);
    check_pattern_kernel<<<(unsigned)((N2 + 255) / 256), 256, 0, st>>>(h->rp, h->col, N2, derr);
    AFN_LAUNCH_CHECK("check_pattern_kernel");
  } else {
    AFN_CUDA(cudaMemsetAsync(h->rp, 0, sizeof(int64_t), st));
  }
  AFN_CUDA(cudaEventRecord(ev[5], st));

  // ---- a7: FSAI rows, then G^T
  TRY(halloc(h, (void**)&h->gval, sizeof(double) * (h->nnz > 0 ? h->nnz : 1), st));
  TRY(halloc(h, (void**)&h->trp, sizeof(int64_t) * (N2 + 1), st));
  TRY(halloc(h, (void**)&h->tcol, sizeof(int32_t) * (h->nnz > 0 ? h->nnz : 1), st));
  TRY(halloc(h, (void**)&h->tval, sizeof(double) * (h->nnz > 0 ? h->nnz : 1), st));
  cudaEvent_t ef0, ef1;
  AFN_CUDA(cudaEventCreate(&ef0));
  AFN_CUDA(cudaEventCreate(&ef1));
  struct EvGuard2 {
    cudaEvent_t a, b;
    ~EvGuard2() { cudaEventDestroy(a); cudaEventDestroy(b); }
  } evg2{ef0, ef1};
  AFN_CUDA(cudaEventRecord(ef0, st));
  AFN_CUDA(cudaEventRecord(ef1, st));
  if (N2 > 0) {
    int64_t* tmap = nullptr;
    TRY(halloc(h, (void**)&tmap, sizeof(int64_t) * (h->nnz > 0 ? h->nnz : 1), st));
    // transposed pattern first (the pair-union FSAI needs "rows containing a")
    TRY(csr_transpose(h->rp, h->col, nullptr, N2, h->nnz, h->trp, h->tcol, nullptr, st, tmap));
    AFN_CUDA(cudaEventRecord(ef0, st));
    static const int variant = getenv("AFN_FSAI_VARIANT") ? atoi(getenv("AFN_FSAI_VARIANT")) : -1;
    afn_status fs = AFN_ERR_STATE;
    if (variant < 0) {
      fs = fsai_sddmm_run(X2, N2, d, P.l, P.mu, h->W, k, h->rp, h->col, h->trp, h->tcol, h->gval,
                          dinfo + 1, st);
      if (fs != AFN_OK && fs != AFN_ERR_STATE) return fs;
    }
    if (fs != AFN_OK) {
      kt_begin(KT_FSAI_GRAM, st);
      TRY(fsai_run(X2, N2, d, P.l, P.mu, h->W, k, h->rp, h->col, h->gval, dinfo + 1, st));
      kt_end(KT_FSAI_GRAM, st, 0.0);
    }
    AFN_CUDA(cudaEventRecord(ef1, st));
    TRY(gather_map(h->gval, tmap, h->nnz, h->tval, st));
  } else {
    AFN_CUDA(cudaMemsetAsync(h->trp, 0, sizeof(int64_t), st));
  }
  AFN_CUDA(cudaEventRecord(ev[6], st));

  // ---- workspaces for apply / PCG
  h->plan = kmv_plan(n, n, d, num_sms());
  TRY(halloc(h, (void**)&h->kmv_part, sizeof(double) * h->plan.chunks * n, st));
  const int64_t gw = std::max(gemv_t_ws(k, k), gemv_t_ws(N2, k));
  TRY(halloc(h, (void**)&h->gws, sizeof(double) * gw, st));
  TRY(halloc(h, (void**)&h->tvec, sizeof(double) * k, st));
  TRY(halloc(h, (void**)&h->vvec, sizeof(double) * k, st));
  TRY(halloc(h, (void**)&h->uvec, sizeof(double) * (N2 > 0 ? N2 : 1), st));
  TRY(halloc(h, (void**)&h->yvec, sizeof(double) * (N2 > 0 ? N2 : 1), st));
  TRY(halloc(h, (void**)&h->rbuf, sizeof(double) * n, st));
  TRY(halloc(h, (void**)&h->zbuf, sizeof(double) * n, st));
  for (double** v : {&h->x, &h->r, &h->z, &h->p, &h->q}) TRY(halloc(h, (void**)v, sizeof(double) * n, st));
  TRY(halloc(h, (void**)&h->sc, sizeof(double) * SC_N, st));
  TRY(halloc(h, (void**)&h->dws, sizeof(double) * dot_ws(), st));
  TRY(halloc(h, (void**)&h->dcnt, sizeof(unsigned) * 4, st));
  AFN_CUDA(cudaMemsetAsync(h->dcnt, 0, sizeof(unsigned) * 4, st));
  AFN_CUDA(cudaMemsetAsync(h->sc, 0, sizeof(double) * SC_N, st));
  h->h_sc = pinned_scalars();
  if (!h->h_sc) {
    set_error("pinned host allocation failed");
    return AFN_ERR_NOMEM;
  }
  AFN_CUDA(cudaEventRecord(ev[7], st));
  AFN_CUDA(cudaStreamSynchronize(st));
  {
    int e = 0;
    AFN_CUDA(cudaMemcpy(&e, derr, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) {
      set_error("internal consistency check failed (code %d: 1/2 landmark ids, 4/8 pattern)", e);
      return AFN_ERR_CUDA;
    }
    int info = 0;
    AFN_CUDA(cudaMemcpy(&info, dinfo + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (info && !getenv("AFN_DEBUG_ALLOW_NOT_SPD")) {
      set_error("FSAI block Cholesky broke down in row %d", info - 1);
      return AFN_ERR_NOT_SPD;
    }
  }
  h->ms[0] = ev_ms(ev[0], ev[1]);  // alg1
  h->ms[1] = ev_ms(ev[1], ev[2]);  // fps
  h->ms[2] = ev_ms(ev[2], ev[3]);  // perm + chol + L^{-T}
  h->ms[3] = ev_ms(ev[3], ev[4]);  // trsm W
  h->ms[4] = ev_ms(ev[4], ev[5]);  // knn
  h->ms[5] = ev_ms(ev[5], ev[6]);  // fsai + G^T
  h->ms[6] = ev_ms(ev[0], ev[7]);  // total
  h->ms[7] = ev_ms(ef0, ef1);      // fsai row kernel
  kt_collect();
  *out = h;
  h = nullptr;  // release the guard
  return AFN_OK;
}

afn_status afn_apply(afn_handle h, const double* r, double* z, void* stream) {
  REQ(h != nullptr, "null handle");
  REQ(is_dev(r) && is_dev(z) && r != z, "r, z must be distinct device pointers");
  cudaStream_t st = (cudaStream_t)stream;
  TRY(gather_vec(r, h->perm, h->n, h->rbuf, st));
  TRY(apply_perm(h, h->rbuf, h->zbuf, st));
  TRY(scatter_vec(h->zbuf, h->perm, h->n, z, st));
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
  cudaEvent_t e0, e1, km0, km1, ap0, ap1;
  AFN_CUDA(cudaEventCreate(&e0));
  AFN_CUDA(cudaEventCreate(&e1));
  AFN_CUDA(cudaEventCreate(&km0));
  AFN_CUDA(cudaEventCreate(&km1));
  AFN_CUDA(cudaEventCreate(&ap0));
  AFN_CUDA(cudaEventCreate(&ap1));
  struct EvG {
    cudaEvent_t e[6];
    ~EvG() { for (auto x : e) cudaEventDestroy(x); }
  } evg{{e0, e1, km0, km1, ap0, ap1}};
  double mv_ms = 0.0, ap_ms = 0.0;
  int napply = 0;
  bool ap_pending = false;
  AFN_CUDA(cudaEventRecord(e0, st));

  // r = b (permuted), x = 0
  TRY(gather_vec(b, h->perm, n, h->r, st));
  AFN_CUDA(cudaMemsetAsync(h->x, 0, sizeof(double) * n, st));
  TRY(dot(h->r, h->r, n, h->sc + SC_BB, h->dws, h->dcnt, st));
  AFN_CUDA(cudaMemcpyAsync(hsc, h->sc, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, st));
  AFN_CUDA(cudaStreamSynchronize(st));
  const double nb = std::sqrt(hsc[SC_BB]);
  if (R.history) R.history[0] = nb > 0 ? 1.0 : 0.0;
  int it = 0;
  double rel = nb > 0 ? 1.0 : 0.0;
  if (nb > 0) {
    AFN_CUDA(cudaEventRecord(ap0, st));
    TRY(apply_perm(h, h->r, h->z, st));
    AFN_CUDA(cudaEventRecord(ap1, st));
    ap_pending = true;
    ++napply;
    int cur = SC_RZ0;
    TRY(dot(h->r, h->z, n, h->sc + cur, h->dws, h->dcnt, st));
    TRY(vec_copy(h->p, h->z, n, st));
    for (it = 1; it <= maxit; ++it) {
      AFN_CUDA(cudaEventRecord(km0, st));
      kt_begin(KT_KMV, st);
      TRY(kmv_launch(h->Xs, n, d, h->p, h->mu, 0, n, h->q, h->kmv_part, h->plan, st));
      kt_end(KT_KMV, st, (double)n * (double)n * (3.0 * d + 19.0));
      AFN_CUDA(cudaEventRecord(km1, st));
      TRY(dot(h->p, h->q, n, h->sc + SC_PQ, h->dws, h->dcnt, st));
      TRY(pcg_update_xr(h->x, h->r, h->p, h->q, n, h->sc, cur, h->dws, h->dcnt, st));
      AFN_CUDA(cudaMemcpyAsync(hsc, h->sc, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, st));
      AFN_CUDA(cudaStreamSynchronize(st));
      mv_ms += ev_ms(km0, km1);
      if (ap_pending) {
        ap_ms += ev_ms(ap0, ap1);
        ap_pending = false;
      }
      const double pq = hsc[SC_PQ];
      if (!(pq > 0.0) || !std::isfinite(pq) || !std::isfinite(hsc[SC_RR])) {
        R.breakdown = 1;
        --it;
        break;
      }
      rel = std::sqrt(hsc[SC_RR]) / nb;
      if (R.history) R.history[it] = rel;
      if (fixed_iters > 0) {
        if (it >= fixed_iters) {
          R.converged = rel <= tol;
          break;
        }
      } else if (rel <= tol) {
        R.converged = 1;
        break;
      }
      AFN_CUDA(cudaEventRecord(ap0, st));
      kt_begin(KT_APPLY, st);
      TRY(apply_perm(h, h->r, h->z, st));
      kt_end(KT_APPLY, st, apply_bytes(h));
      AFN_CUDA(cudaEventRecord(ap1, st));
      ap_pending = true;
      ++napply;
      const int nxt = cur ^ 1;
      TRY(dot(h->r, h->z, n, h->sc + nxt, h->dws, h->dcnt, st));
      TRY(pcg_update_p(h->p, h->z, n, h->sc, nxt, cur, st));
      cur = nxt;
    }
    if (it > maxit) it = maxit;
  } else {
    R.converged = 1;
  }
  // a = x (un-permuted); true residual ||b - (K + mu I) x|| / ||b||
  TRY(scatter_vec(h->x, h->perm, n, a, st));
  AFN_CUDA(cudaEventRecord(e1, st));
  if (nb > 0) {
    TRY(kmv_launch(h->Xs, n, d, h->x, h->mu, 0, n, h->q, h->kmv_part, h->plan, st));
    TRY(gather_vec(b, h->perm, n, h->z, st));
    TRY(vec_axpby(h->z, -1.0, h->q, 1.0, n, st));
    TRY(dot(h->z, h->z, n, h->sc + SC_TMP, h->dws, h->dcnt, st));
    AFN_CUDA(cudaMemcpyAsync(hsc, h->sc, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, st));
  }
  AFN_CUDA(cudaStreamSynchronize(st));
  R.iterations = it;
  R.relres = rel;
  R.relres_true = nb > 0 ? std::sqrt(hsc[SC_TMP]) / nb : 0.0;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  R.solve_ms = ms;
  if (ap_pending) ap_ms += ev_ms(ap0, ap1);
  R.matvec_ms = mv_ms;
  R.apply_ms = ap_ms;
  kt_collect();
  R.applies = napply;
  if (rep) *rep = R;
  return AFN_OK;
}

afn_status afn_solve_host(const double* X, const double* b, double* a, int64_t n, int32_t d,
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
  TRY(afn_build(dX, n, d, params, stream, &h));
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
  *info = I;
  return AFN_OK;
}

afn_status afn_copy_out(afn_handle h, int32_t what, void* host, size_t bytes) {
  REQ(h && host, "null argument");
  const void* src = nullptr;
  size_t need = 0;
  switch (what) {
    case AFN_OUT_PERM: src = h->perm; need = sizeof(int64_t) * h->n; break;
    case AFN_OUT_FILL: src = h->fill; need = sizeof(double) * h->k; break;
    case AFN_OUT_L: src = h->L; need = sizeof(double) * h->k * h->k; break;
    case AFN_OUT_ROWPTR: src = h->rp; need = sizeof(int64_t) * (h->N2 + 1); break;
    case AFN_OUT_COL: src = h->col; need = sizeof(int32_t) * h->nnz; break;
    case AFN_OUT_GVAL: src = h->gval; need = sizeof(double) * h->nnz; break;
    case AFN_OUT_W: src = h->W; need = sizeof(double) * h->N2 * h->k; break;
    default: set_error("unknown copy_out selector %d", what); return AFN_ERR_ARG;
  }
  REQ(bytes == need, "copy_out: bytes=%zu, need %zu", bytes, need);
  if (need == 0) return AFN_OK;
  AFN_CUDA(cudaMemcpy(host, src, need, cudaMemcpyDeviceToHost));
  return AFN_OK;
}

afn_status afn_copy_out_rows(afn_handle h, int32_t what, const int64_t* rows, int64_t nrows,
                             void* host, size_t bytes) {
  REQ(h && host && (rows || nrows == 0) && nrows >= 0, "null argument");
  const double* src = nullptr;
  int64_t R = 0;
  if (what == AFN_OUT_W) src = h->W, R = h->N2;
  else if (what == AFN_OUT_L) src = h->L, R = h->k;
  else REQ(false, "copy_out_rows: selector %d unsupported (W or L only)", what);
  const size_t rowb = sizeof(double) * (size_t)h->k;
  REQ(bytes == rowb * (size_t)nrows, "copy_out_rows: bytes=%zu, need %zu", bytes,
      rowb * (size_t)nrows);
  for (int64_t t = 0; t < nrows; ++t)
    REQ(rows[t] >= 0 && rows[t] < R, "copy_out_rows: row %lld out of range [0, %lld)",
        (long long)rows[t], (long long)R);
  for (int64_t t = 0; t < nrows; ++t)
    AFN_CUDA(cudaMemcpy(static_cast<char*>(host) + rowb * t, src + (size_t)rows[t] * h->k, rowb,
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

}  // extern "C"

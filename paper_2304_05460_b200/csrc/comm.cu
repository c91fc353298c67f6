// comm.cu -- the one exchange primitive of the row-sharded path: an
// all-gather of per-rank byte ranges ("allgatherv") into a buffer that has
// the same layout on every rank (the CG vector p before each
// kernel matvec, u and G u inside the AFN apply, the k-vector partials of
// W^T s2, the dot-product partials, and W / pattern / G rows after the
// sharded build steps).
//
// Two transports behind one call:
//   * NCCL (one process per GPU): ncclAllGather on the caller's stream --
//     in place when every rank owns one equal-size range at offset s * len
//     (the per-rank partials: dot products, the k-vector of W^T s2, the
//     symmetric matvec's rank partials), otherwise through a packed staging
//     buffer (each rank's <= 2 row segments packed to a fixed stride,
//     gathered, unpacked: the PCG vector p, u, G u and the build's W /
//     pattern / G rows).  libnccl.so.2 is dlopen'ed (the copy PyTorch
//     already loaded), so libafn.so itself has no link-time NCCL dependency.
//     Host waits on a stream with NCCL work poll ncclCommGetAsyncError and
//     abort the communicator on an error or after the timeout.
//   * emulated (tests): R logical ranks driven by ONE process on ONE device,
//     each with its own buffers; the exchange is a device-to-device copy of
//     every owner's ranges into every other rank's buffer on the same stream.
//     No kernel ever waits for another rank (all ranks' work for a phase is
//     enqueued before the copies), so this is safe on a single GPU.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "afn_common.cuh"
#include "afn_internal.h"
#include "nccl.h"

namespace afn {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi& nccl_api(const char* path) {
  static NcclApi api;
  if (api.ok) return api;
  void* h = nullptr;
  if (path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define AFN_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
  AFN_SYM(GetUniqueId, "ncclGetUniqueId");
  AFN_SYM(CommInitRank, "ncclCommInitRank");
  AFN_SYM(CommDestroy, "ncclCommDestroy");
  AFN_SYM(GroupStart, "ncclGroupStart");
  AFN_SYM(GroupEnd, "ncclGroupEnd");
  AFN_SYM(GetErrorString, "ncclGetErrorString");
  AFN_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
  AFN_SYM(CommAbort, "ncclCommAbort");
  AFN_SYM(AllGather, "ncclAllGather");
#undef AFN_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GroupStart &&
           api.GroupEnd && api.GetErrorString && api.CommGetAsyncError && api.CommAbort;
  return api;
}

afn_status nccl_status(ncclResult_t r, const char* what) {
  NcclApi& a = nccl_api(nullptr);
  set_error("NCCL error %d (%s) in %s", (int)r, a.GetErrorString ? a.GetErrorString(r) : "?", what);
  return AFN_ERR_NCCL;
}

}  // namespace

afn_status comm_allgatherv(const Comm* c, char* const* bufs, const std::vector<RankRanges>& owned,
                           cudaStream_t st) {
  if (!c || c->R <= 1) return AFN_OK;
  if (c->emulated) {
    for (int q = 0; q < c->nlocal; ++q)
      for (int s = 0; s < c->R; ++s) {
        if (s == q) continue;
        for (const auto& rg : owned[s])
          if (rg.second > 0)
            AFN_CUDA(cudaMemcpyAsync(bufs[q] + rg.first, bufs[s] + rg.first, rg.second,
                                     cudaMemcpyDeviceToDevice, st));
      }
    return AFN_OK;
  }
  NcclApi& a = nccl_api(nullptr);
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
  const int R = c->R, me = c->rank0;
  // in place: rank s owns exactly [base + s len, base + (s + 1) len)
  bool inplace = true;
  size_t len = 0, base = 0;
  for (int s = 0; s < R && inplace; ++s) {
    if (owned[s].size() != 1) { inplace = false; break; }
    if (s == 0) { len = owned[0][0].second; base = owned[0][0].first; }
    inplace = owned[s][0].second == len && owned[s][0].first == base + (size_t)s * len;
  }
  if (inplace) {
    if (len == 0) return AFN_OK;
    const ncclResult_t r = a.AllGather(bufs[0] + base + (size_t)me * len, bufs[0] + base, len, ncclUint8, comm, st);
    if (r != ncclSuccess) return nccl_status(r, "ncclAllGather");
    return AFN_OK;
  }
  // packed: every rank's ranges at a fixed stride (the largest rank's bytes)
  size_t stride = 0;
  for (int s = 0; s < R; ++s) {
    size_t t = 0;
    for (const auto& rg : owned[s]) t += rg.second;
    stride = std::max(stride, t);
  }
  if (stride == 0) return AFN_OK;
  stride = (stride + 255) & ~(size_t)255;
  Comm* cm = const_cast<Comm*>(c);
  if (cm->stage_bytes < stride * R) {
    if (cm->stage) {
      AFN_CUDA(cudaStreamSynchronize(st));
      cudaFree(cm->stage);
      cm->stage = nullptr;
      cm->stage_bytes = 0;
    }
    AFN_CUDA(cudaMalloc(&cm->stage, stride * R));
    cm->stage_bytes = stride * R;
  }
  char* stage = static_cast<char*>(cm->stage);
  size_t o = 0;
  for (const auto& rg : owned[me]) {  // pack my ranges
    if (rg.second > 0)
      AFN_CUDA(cudaMemcpyAsync(stage + (size_t)me * stride + o, bufs[0] + rg.first, rg.second,
                               cudaMemcpyDeviceToDevice, st));
    o += rg.second;
  }
  const ncclResult_t r = a.AllGather(stage + (size_t)me * stride, stage, stride, ncclUint8, comm, st);
  if (r != ncclSuccess) return nccl_status(r, "ncclAllGather");
  for (int s = 0; s < R; ++s) {  // unpack the others' ranges
    if (s == me) continue;
    size_t os = 0;
    for (const auto& rg : owned[s]) {
      if (rg.second > 0)
        AFN_CUDA(cudaMemcpyAsync(bufs[0] + rg.first, stage + (size_t)s * stride + os, rg.second,
                                 cudaMemcpyDeviceToDevice, st));
      os += rg.second;
    }
  }
  return AFN_OK;
}

afn_status comm_stream_sync(const Comm* c, cudaStream_t st) {
  if (!c || c->R <= 1 || c->emulated || !c->nccl) {
    AFN_CUDA(cudaStreamSynchronize(st));
    return AFN_OK;
  }
  NcclApi& a = nccl_api(nullptr);
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return AFN_OK;
    if (q != cudaErrorNotReady) return cuda_status(q, "cudaStreamQuery (NCCL stream)");
    ncclResult_t ae = ncclSuccess;
    if (a.CommGetAsyncError(comm, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
      a.CommAbort(comm);
      const_cast<Comm*>(c)->nccl = nullptr;
      return nccl_status(ae, "asynchronous NCCL error (communicator aborted)");
    }
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sec > c->timeout_s) {
      a.CommAbort(comm);
      const_cast<Comm*>(c)->nccl = nullptr;
      set_error("NCCL wait exceeded %.0f s (communicator aborted)", c->timeout_s);
      return AFN_ERR_NCCL;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

}  // namespace afn

using namespace afn;

extern "C" {

afn_status afn_comm_unique_id(void* id, const char* nccl_path) {
  if (!id) {
    set_error("id must be a host buffer of 128 bytes");
    return AFN_ERR_ARG;
  }
  NcclApi& a = nccl_api(nccl_path);
  if (!a.ok) {
    set_error("libnccl.so.2 could not be loaded (%s)", dlerror());
    return AFN_ERR_NCCL;
  }
  ncclUniqueId u;
  ncclResult_t r = a.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_status(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == AFN_COMM_ID_BYTES, "unique id size");
  std::memcpy(id, &u, sizeof(u));
  return AFN_OK;
}

afn_status afn_comm_init(const void* id, int32_t nranks, int32_t rank, const char* nccl_path,
                         afn_comm* out) {
  if (!out) {
    set_error("out must be non-null");
    return AFN_ERR_ARG;
  }
  *out = nullptr;
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("need a unique id, nranks >= 1 and 0 <= rank < nranks");
    return AFN_ERR_ARG;
  }
  Comm* c = new Comm();
  c->R = nranks;
  c->nlocal = 1;
  c->rank0 = rank;
  if (nranks > 1) {
    NcclApi& a = nccl_api(nccl_path);
    if (!a.ok) {
      delete c;
      set_error("libnccl.so.2 could not be loaded");
      return AFN_ERR_NCCL;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t comm = nullptr;
    ncclResult_t r = a.CommInitRank(&comm, nranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      return nccl_status(r, "ncclCommInitRank");
    }
    c->nccl = comm;
  }
  *out = c;
  return AFN_OK;
}

afn_status afn_comm_init_emulated(int32_t nranks, afn_comm* out) {
  if (!out || nranks < 1 || nranks > 64) {
    set_error("need 1 <= nranks <= 64 and non-null out");
    return AFN_ERR_ARG;
  }
  Comm* c = new Comm();
  c->R = nranks;
  c->nlocal = nranks;
  c->rank0 = 0;
  c->emulated = true;
  *out = c;
  return AFN_OK;
}

void afn_comm_destroy(afn_comm c) {
  if (!c) return;
  if (c->nccl) {
    NcclApi& a = nccl_api(nullptr);
    if (a.CommDestroy) a.CommDestroy(static_cast<ncclComm_t>(c->nccl));
  }
  if (c->stage) {
    cudaDeviceSynchronize();
    cudaFree(c->stage);
  }
  delete c;
}

afn_status afn_comm_set_timeout(afn_comm c, double seconds) {
  if (!c || !(seconds > 0.0)) {
    set_error("need a communicator and seconds > 0");
    return AFN_ERR_ARG;
  }
  c->timeout_s = seconds;
  return AFN_OK;
}

afn_status afn_shard_rows(int64_t n, int64_t k, int32_t nranks, int32_t rank, int64_t* rows) {
  if (!rows || n < 1 || k < 0 || k > n || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("need n >= 1, 0 <= k <= n, 0 <= rank < nranks, non-null rows");
    return AFN_ERR_ARG;
  }
  const Seg2 s = shard_rows(n, k, nranks, rank);
  rows[0] = s.a0;
  rows[1] = s.na;
  rows[2] = s.b0;
  rows[3] = s.nb;
  return AFN_OK;
}

}  // extern "C"

// comm.cu -- the one exchange primitive of the row-sharded path: an
// all-gather of per-rank byte ranges ("allgatherv") into a buffer that has
// the same layout on every rank (the CG vector p before each
// kernel matvec, u and G u inside the AFN apply, the k-vector partials of
// W^T s2, the dot-product partials, and W / pattern / G rows after the
// sharded build steps).
//
// Two transports behind one call:
//   * NCCL (one process per GPU): every rank's ranges are broadcast from
//     their owner inside one ncclGroupStart/End, in place, on the caller's
//     stream.  libnccl.so.2 is dlopen'ed (the copy PyTorch already loaded),
//     so libafn.so itself has no link-time NCCL dependency.
//   * emulated (tests): R logical ranks driven by ONE process on ONE device,
//     each with its own buffers; the exchange is a device-to-device copy of
//     every owner's ranges into every other rank's buffer on the same stream.
//     No kernel ever waits for another rank (all ranks' work for a phase is
//     enqueued before the copies), so this is safe on a single GPU.
#include <dlfcn.h>

#include <cstring>
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
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
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
  AFN_SYM(Broadcast, "ncclBroadcast");
  AFN_SYM(GroupStart, "ncclGroupStart");
  AFN_SYM(GroupEnd, "ncclGroupEnd");
  AFN_SYM(GetErrorString, "ncclGetErrorString");
  AFN_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef AFN_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.GroupStart &&
           api.GroupEnd && api.GetErrorString;
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
  ncclResult_t r = a.GroupStart();
  if (r != ncclSuccess) return nccl_status(r, "ncclGroupStart");
  for (int s = 0; s < c->R; ++s)
    for (const auto& rg : owned[s]) {
      if (rg.second == 0) continue;
      r = a.Broadcast(bufs[0] + rg.first, bufs[0] + rg.first, rg.second, ncclUint8, s, comm, st);
      if (r != ncclSuccess) {
        a.GroupEnd();
        return nccl_status(r, "ncclBroadcast");
      }
    }
  r = a.GroupEnd();
  if (r != ncclSuccess) return nccl_status(r, "ncclGroupEnd");
  return AFN_OK;
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
  delete c;
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

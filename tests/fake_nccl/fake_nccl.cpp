// fake_nccl.cpp -- a test stand-in for libnccl.so.2 whose "ranks" are host
// threads of ONE process on ONE device (tests/test_gpu_r2.py runs the
// library's real NCCL code path -- comm.cu's in-place and packed all-gathers,
// the build-status exchange, the asynchronous-error polling -- through it).
// Only the calls comm.cu dlsym's are provided.  ncclAllGather: every rank
// registers its send buffer and an event recorded on its stream, the ranks
// meet on a host barrier, each rank's stream waits for every source's event
// and copies the sources' chunks into its receive buffer, then the ranks meet
// again and every stream waits for all ranks' copies (so no rank reuses a
// buffer another rank still reads).  No kernel ever waits on another rank:
// the dependencies are stream events, which is safe on one GPU.
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <vector>

#include "nccl.h"

namespace {

struct Group {
  int n = 0;
  int joined = 0;
  std::mutex mu;
  std::condition_variable cv;
  // per-collective exchange slots
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
  int arrived = 0;
  long long generation = 0;
};

struct Comm {
  Group* g;
  int rank;
};

std::mutex g_reg_mu;
std::map<std::string, Group*> g_reg;

// all ranks of g reach this point; the last one runs `last` under the lock
template <class F>
void barrier(Group* g, F last) {
  std::unique_lock<std::mutex> lk(g->mu);
  const long long gen = g->generation;
  if (++g->arrived == g->n) {
    last();
    g->arrived = 0;
    ++g->generation;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->generation != gen; });
  }
}

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclFloat64: case ncclInt64: case ncclUint64: return 8;
    default: return 0;
  }
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<int> counter{0};
  std::memset(id, 0, sizeof(*id));
  snprintf(id->internal, sizeof(id->internal), "fake-nccl-%d", counter.fetch_add(1));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  Group* g;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto& slot = g_reg[std::string(id.internal)];
    if (!slot) {
      slot = new Group();
      slot->n = nranks;
      slot->send.resize(nranks);
      slot->ready.resize(nranks);
      slot->done.resize(nranks);
      for (int r = 0; r < nranks; ++r) {
        cudaEventCreateWithFlags(&slot->ready[r], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&slot->done[r], cudaEventDisableTiming);
      }
    }
    g = slot;
  }
  if (g->n != nranks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  barrier(g, [] {});
  *out = reinterpret_cast<ncclComm_t>(new Comm{g, rank});
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  delete reinterpret_cast<Comm*>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t c) { return ncclCommDestroy(c); }

ncclResult_t ncclCommGetAsyncError(ncclComm_t, ncclResult_t* e) {
  *e = ncclSuccess;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t) { return "fake nccl error"; }

ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t type, ncclComm_t comm,
                           cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  Group* g = c->g;
  const size_t bytes = count * type_size(type);
  if (bytes == 0 && count != 0) return ncclInvalidArgument;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->send[c->rank] = sendbuff;
  }
  if (cudaEventRecord(g->ready[c->rank], st) != cudaSuccess) return ncclUnhandledCudaError;
  barrier(g, [] {});
  char* recv = static_cast<char*>(recvbuff);
  for (int s = 0; s < g->n; ++s) {
    cudaStreamWaitEvent(st, g->ready[s], 0);
    if (s == c->rank && g->send[s] == recv + (size_t)s * bytes) continue;  // in place
    if (cudaMemcpyAsync(recv + (size_t)s * bytes, g->send[s], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  cudaEventRecord(g->done[c->rank], st);
  barrier(g, [] {});
  for (int s = 0; s < g->n; ++s) cudaStreamWaitEvent(st, g->done[s], 0);
  barrier(g, [] {});  // (the events may be re-recorded by the next collective only now)
  return ncclSuccess;
}

}  // extern "C"

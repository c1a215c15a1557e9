// Multi-GPU communicator: NCCL over NVLink/NVSwitch, one process per GPU.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") — the process normally has
// torch's bundled NCCL loaded already, so the same library instance serves both
// torch.distributed and this library.  The parareal driver exchanges, per iteration,
// one all-gather of the coarse payload of every slice (R(F u_{n-1}), C(R u_{n-1}) and the
// divergence flags), one all-gather of per-slice error sums, and one send/recv of the
// boundary fine state between neighbouring ranks.

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ptb_comm.h"

namespace ptb {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* s) { return dlsym(api.h, s); };
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.allGather)
    fail(PTB_NCCL, "NCCL runtime (libnccl.so.2) not found");
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(PTB_NCCL, std::string(what) + ": " + (nccl().errorString ? nccl().errorString(r) : "nccl error"));
}

}  // namespace

// In-process communicator: W host threads, each driving its own context (same or peer
// GPUs).  A collective synchronises the caller's stream, publishes its send buffer, meets
// the other ranks at a host barrier, copies what it needs with cudaMemcpy (peer-capable)
// and meets them again before anyone may reuse a buffer.  No device code waits on
// another rank, so several ranks can share one GPU safely.
struct LoopbackGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> sends;
  explicit LoopbackGroup(int w) : world(w), sends(size_t(w), nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lock(m);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return generation != gen; });
    }
  }
};

void Comm::allgather(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st) const {
  if (loopback) {
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    loopback->sends[size_t(rank)] = send;
    loopback->barrier();
    for (int r = 0; r < world; ++r)
      PTB_CUDA_CHECK(cudaMemcpy(static_cast<char*>(recv) + size_t(r) * bytes_per_rank, loopback->sends[size_t(r)],
                                bytes_per_rank, cudaMemcpyDefault));
    loopback->barrier();
    return;
  }
  if (world == 1 && !handle) {
    if (send != recv)
      PTB_CUDA_CHECK(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, st));
    return;
  }
  check_nccl(nccl().allGather(send, recv, bytes_per_rank, ncclChar, static_cast<ncclComm_t>(handle), st),
             "ncclAllGather");
}

void Comm::shift_right(const void* send, size_t send_bytes, bool do_send, void* recv, size_t recv_bytes,
                       bool do_recv, cudaStream_t st) const {
  if (world == 1) return;
  if (loopback) {
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    loopback->sends[size_t(rank)] = send;
    loopback->barrier();
    if (do_recv) PTB_CUDA_CHECK(cudaMemcpy(recv, loopback->sends[size_t(rank - 1)], recv_bytes, cudaMemcpyDefault));
    loopback->barrier();
    (void)send_bytes;
    (void)do_send;
    return;
  }
  auto& a = nccl();
  check_nccl(a.groupStart(), "ncclGroupStart");
  if (do_send) check_nccl(a.send(send, send_bytes, ncclChar, rank + 1, static_cast<ncclComm_t>(handle), st), "ncclSend");
  if (do_recv) check_nccl(a.recv(recv, recv_bytes, ncclChar, rank - 1, static_cast<ncclComm_t>(handle), st), "ncclRecv");
  check_nccl(a.groupEnd(), "ncclGroupEnd");
}

}  // namespace ptb

struct ptb_comm {
  ptb::Comm c;
};

using namespace ptb;

extern "C" {

ptb_status ptb_nccl_unique_id(char* out128) {
  return guarded([&] {
    require(out128 != nullptr, "nccl_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    check_nccl(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

ptb_status ptb_comm_create(ptb_context* ctx, int rank, int world, const char* id128, ptb_comm** out) {
  return guarded([&] {
    require(ctx && out && world >= 1 && rank >= 0 && rank < world, "comm: bad arguments");
    auto* c = new ptb_comm();
    c->c.rank = rank;
    c->c.world = world;
    // PTB_NCCL_FORCE=1 (tests): a one-rank NCCL communicator, so world 1 exercises the
    // NCCL runtime path (dlopen, init, all-gather) on a single GPU
    static const bool force = [] {
      const char* e = std::getenv("PTB_NCCL_FORCE");
      return e && std::atoi(e) != 0;
    }();
    if (world > 1 || force) {
      ncclUniqueId id;
      if (world == 1) {  // nobody to share an id with
        check_nccl(nccl().getUniqueId(&id), "ncclGetUniqueId");
      } else {
        require(id128 != nullptr, "comm: null unique id");
        std::memcpy(&id, id128, sizeof(id));
      }
      cudaSetDevice(ctx->device);
      ncclComm_t comm = nullptr;
      check_nccl(nccl().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
      c->c.handle = comm;
    }
    *out = c;
  });
}

ptb_status ptb_loopback_group_create(int world, void** out) {
  return guarded([&] {
    require(world >= 1 && out, "loopback: bad arguments");
    *out = new LoopbackGroup(world);
  });
}

ptb_status ptb_loopback_group_destroy(void* group) {
  return guarded([&] { delete static_cast<LoopbackGroup*>(group); });
}

ptb_status ptb_comm_create_loopback(ptb_context* ctx, void* group, int rank, ptb_comm** out) {
  return guarded([&] {
    require(ctx && group && out, "loopback comm: null argument");
    auto* g = static_cast<LoopbackGroup*>(group);
    require(rank >= 0 && rank < g->world, "loopback comm: bad rank");
    auto* c = new ptb_comm();
    c->c.rank = rank;
    c->c.world = g->world;
    c->c.loopback = g;
    *out = c;
  });
}

ptb_status ptb_comm_destroy(ptb_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->c.handle) nccl().commDestroy(static_cast<ncclComm_t>(c->c.handle));
    delete c;
  });
}

}  // extern "C"

namespace ptb {
const Comm* comm_of(const ptb_comm* c) { return c ? &c->c : nullptr; }
}  // namespace ptb

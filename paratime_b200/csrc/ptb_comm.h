#pragma once
#include "ptb_internal.h"

namespace ptb {

// Rank/world plus the NCCL communicator (opaque; null when world == 1).
struct LoopbackGroup;

struct Comm {
  int rank = 0, world = 1;
  void* handle = nullptr;             // ncclComm_t
  LoopbackGroup* loopback = nullptr;  // in-process ranks (one thread each), host rendezvous
  // every rank contributes bytes_per_rank from `send`; recv holds world * bytes_per_rank
  void allgather(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st) const;
  // send `send` to rank+1 and receive `recv` from rank-1 (grouped)
  void shift_right(const void* send, size_t send_bytes, bool do_send, void* recv, size_t recv_bytes, bool do_recv,
                   cudaStream_t st) const;
};

const Comm* comm_of(const ptb_comm* c);

}  // namespace ptb

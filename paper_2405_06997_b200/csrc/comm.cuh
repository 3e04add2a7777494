// Multi-GPU exchange layer of the render pass.
#pragma once
#include "common.cuh"

namespace wfpg {

enum CommDtype { kI32 = 0, kU64 = 1, kF64 = 2 };

struct Comm;  // wfpg_comm

int comm_world(const Comm* c);
int comm_rank(const Comm* c);
// 1 when the collectives may be captured into a CUDA graph (NCCL); host
// exchange communicators synchronise the stream and run on the host.
bool comm_capturable(const Comm* c);
// recv = concatenation over ranks of `count` elements each (rank order)
int comm_all_gather(const Comm* c, const void* send, void* recv, int64_t count, CommDtype dt,
                    cudaStream_t st);
// recv = element-wise sum over ranks (u64 sums of bit patterns where only one
// rank contributes a non-zero value are exact copies)
int comm_all_reduce_sum(const Comm* c, const void* send, void* recv, int64_t count, CommDtype dt,
                        cudaStream_t st);

// Deferred-check state of the last pass that exchanged deposits through this
// communicator (see render.cu): the pass writes its overflow word to pinned
// host memory and records `done`; the next pass (or wfpg_comm_settle) waits
// for it and, when some rank exported more deposits than the wire capacity,
// runs the exact (eager, variable-size) exchange of that pass before anything
// else touches the SVO.
struct DepositPending {
  bool active = false;
  wfpg_svo svo;              // the SVO the pass updates
  const int32_t* leaf;       // the pass's full local deposit export
  const double* dir;
  const double* rad;
  const int32_t* count;      // device count
  uint8_t* dirty;            // n_nodes scratch for the refresh
  cudaStream_t stream;
};
int* comm_status_host(Comm* c);  // pinned word written by the pass
cudaEvent_t comm_done_event(Comm* c);
DepositPending& comm_pending(Comm* c);
int comm_settle(Comm* c);

}  // namespace wfpg

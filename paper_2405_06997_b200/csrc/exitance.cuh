#pragma once
#include "common.cuh"

namespace wfpg {

size_t update_exitance_ws_bytes(int64_t n_paths, int max_depth);

// Deposit export (multi-GPU exchange): the deposits land in these caller
// buffers in path-major / k-ascending order instead of being splatted.
struct DepositSink {
  int32_t* leaf;    // (capacity,) leaf id, -1 where the point is in no leaf
  double* dir;      // (capacity, 3)
  double* rad;      // (capacity, 3)
  int32_t* count;   // device count
  int64_t capacity;
};
// record layout of rec_T / rec_pos: slot k of path p at p * sp + k * sd doubles
struct RecLayout {
  int depths;
  int64_t sp, sd;
};
inline RecLayout rec_layout(const wfpg_paths* p) {
  RecLayout r;
  r.depths = p->max_depth + 1;
  r.sp = p->rec_depth_major ? 3 : 3 * (int64_t)r.depths;
  r.sd = p->rec_depth_major ? 3 * p->n : 3;
  return r;
}
int update_exitance(wfpg_svo* svo, const int32_t* emit_depth, const double* emit_le,
                    const double* rec_T, const double* rec_pos, RecLayout rl, int64_t n_paths,
                    int deterministic, int32_t* n_dep_out, Arena& ws, cudaStream_t st,
                    int propagate = 1, uint8_t* dirty = nullptr,  // 0 none, 1 full, 2 dirty-only
                    const DepositSink* sink = nullptr);

}  // namespace wfpg

#pragma once
#include "common.cuh"

namespace wfpg {

struct PartitionOut {
  int32_t* bin_node;
  int32_t* bin_start;
  int32_t* bin_count;
  int32_t* members;     // path ids grouped by bin (optional)
  int32_t* n_bins;      // device count (clamped to capacity)
  int32_t* overflow;    // device flag, set when bins > capacity (optional)
  int64_t capacity;
  const uint32_t* sorted_items;  // out: item index per sorted position
  int32_t* bin_slot;    // optional (P,): slot of every member path, indexed by path id
  const int32_t* item_path;  // path id per item (required with bin_slot)
  // first node id above level l_min (level_off[l_min + 1]); counters live only
  // there, so one memset of [clear_from, n_nodes) clears them.  < 0: per-path walk.
  int64_t clear_from = -1;
  // Start nodes given instead of positions (pos == NULL): the deepest
  // materialised node of every item and its level (multi-GPU global binning,
  // where the start nodes of all ranks' hits are all-gathered).
  const int32_t* start_in = nullptr;
  const int8_t* lev_in = nullptr;
  // optional (capacity,) flags: set to 1 for every bin holding an item with
  // item_path >= 0 (items of other ranks carry -1 and get no bin slot)
  int32_t* need = nullptr;
};

// chain_levels: ancestor levels above l_min stored for the ascent (the SVO
// depth minus l_min; capped at 16 inside)
size_t partition_ws_bytes(int64_t n, int chain_levels = 16);
int partition_spatial(const SvoView& v, int32_t* counter, const int32_t* parent,
                      const double* pos, const int32_t* path_idx, int64_t n_max,
                      const int32_t* n_dev, int l_min, int c_ray, int n_nodes,
                      PartitionOut& out, Arena& ws, cudaStream_t st);

}  // namespace wfpg

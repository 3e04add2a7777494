// Alg. 2 positional binning over the SVO (wavefront.py:98-157) and the
// per-bin origin / jitter / slot setup (wavefront.py:160-195).
//
// The reference pushes ray counters bottom-up level by level; a node's total
// is the number of paths whose start node lies in its subtree.  Here every
// path adds 1 to each node of its own ancestor chain above l_min (only those
// levels are ever tested: a node at level l_min is marked regardless), which
// yields the same totals on every node the ascent reads.  Paths then ascend
// to the first marked node, (bin node, path order) pairs are stably
// radix-sorted, and runs become bins ordered by node id with members in
// ascending path order — exactly np.argsort(kind="stable") + np.unique.
#include "partition.cuh"
#include "prims.cuh"

namespace wfpg {

// chain_out (optional, (n_chain, n_max)): row c holds the item's ancestor c
// levels above its start node, for the levels above l_min (at most n_chain),
// so the ascent loads them all at once instead of walking parent links one
// dependent load at a time
__global__ void k_part_count(SvoView v, int32_t* __restrict__ counter,
                             const double* __restrict__ pos, int64_t n_max,
                             const int32_t* __restrict__ n_dev, int l_min,
                             int32_t* __restrict__ start, int8_t* __restrict__ start_lev,
                             int32_t* __restrict__ chain_out, int n_chain) {
  const int64_t n = dev_count(n_max, n_dev);
  const int lane = threadIdx.x & 31;
  // whole warps iterate together so the counter updates can be aggregated:
  // neighbouring paths (pixel order) share most of their ancestors, and one
  // atomic per distinct node and warp replaces up to 32 contended ones
  for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; w0 < n;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = w0 + lane;
    const bool valid = i < n;
    int32_t node = 0, lvl = 0;
    int32_t chain[22];
    chain[0] = 0;
    if (valid) {
      int32_t qx = quantise(pos[3 * i], v.lox, v.scale, v.resolution);
      int32_t qy = quantise(pos[3 * i + 1], v.loy, v.scale, v.resolution);
      int32_t qz = quantise(pos[3 * i + 2], v.loz, v.scale, v.resolution);
      int level0 = 1;
      if (v.top && v.top_level <= l_min + 1) {
        // the dense top index gives the level-T ancestor in one load; only
        // levels above l_min enter the counts, so the skipped chain is unused
        const int T = v.top_level, sh = v.depth - T;
        const uint2 e = __ldg(&v.top[((uint32_t)(qx >> sh) << (2 * T)) |
                                     ((uint32_t)(qy >> sh) << T) | (uint32_t)(qz >> sh)]);
        node = (int32_t)e.x;
        lvl = (int32_t)(e.y & 0xFFu);
        chain[lvl] = node;
        level0 = (e.y >> 31) ? T + 1 : v.depth + 1;  // absent below: the chain ends at lvl
      }
      for (int level = level0; level <= v.depth; ++level) {
        int sh = v.depth - level;
        int oct = ((qx >> sh) & 1) | (((qy >> sh) & 1) << 1) | (((qz >> sh) & 1) << 2);
        uint2 d = __ldg(&v.desc[node]);
        if (!((d.y >> oct) & 1u)) break;
        node = (int32_t)d.x + __popc(d.y & ((1u << oct) - 1u));
        lvl = level;
        chain[level] = node;
      }
      start[i] = node;
      start_lev[i] = (int8_t)lvl;
      if (chain_out)
        for (int c = 0; c < n_chain && lvl - c > l_min; ++c)
          chain_out[(int64_t)c * n_max + i] = chain[lvl - c];
    }
    int top = valid ? lvl : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
    for (int l = top; l > l_min; --l) {
      const int32_t a = (valid && l <= lvl) ? chain[l] : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, a);
      if (a >= 0 && lane == __ffs(grp) - 1) atomicAdd(&counter[a], __popc(grp));
    }
  }
}

// k_part_count from given start nodes: each item adds 1 to every node of
// its ancestor chain above l_min, walking parent links (the chains of
// neighbouring items in path order coincide, so the warp aggregates them).
__global__ void k_part_count_chain(int32_t* __restrict__ counter, const int32_t* __restrict__ parent,
                                   const int32_t* __restrict__ start,
                                   const int8_t* __restrict__ start_lev, int64_t n_max,
                                   const int32_t* __restrict__ n_dev, int l_min) {
  const int64_t n = dev_count(n_max, n_dev);
  const int lane = threadIdx.x & 31;
  for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane; w0 < n;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = w0 + lane;
    const bool valid = i < n;
    int32_t cur = valid ? start[i] : -1;
    const int lvl = valid ? (int)start_lev[i] : 0;
    int top = lvl;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
    for (int l = top; l > l_min; --l) {
      const int32_t a = (valid && l <= lvl) ? cur : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, a);
      if (a >= 0 && lane == __ffs(grp) - 1) atomicAdd(&counter[a], __popc(grp));
      if (a >= 0) cur = __ldg(&parent[a]);
    }
  }
}

// k_part_ascend with the stored chains: the chain entries, then their
// counters, each as independent loads; the deepest marked level wins as in
// the walk (a level-l_min node is marked regardless: one parent link from
// level l_min + 1, or the start node itself when it sits at l_min).
constexpr int kAscendMax = 16;
__global__ void k_part_ascend_chain(const int32_t* __restrict__ counter,
                                    const int32_t* __restrict__ parent,
                                    const int32_t* __restrict__ start,
                                    const int8_t* __restrict__ start_lev,
                                    const int32_t* __restrict__ chain, int n_chain,
                                    int64_t n_max, const int32_t* __restrict__ n_dev, int l_min,
                                    int c_ray, uint32_t* __restrict__ keys,
                                    uint32_t* __restrict__ vals) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int lev = start_lev[i];
    const int m = min(lev - l_min, n_chain);  // stored levels lev .. lev - m + 1
    int32_t node[kAscendMax];
#pragma unroll
    for (int c = 0; c < kAscendMax; ++c)
      if (c < m) node[c] = __ldg(&chain[(int64_t)c * n_max + i]);
    int32_t cnt[kAscendMax];
#pragma unroll
    for (int c = 0; c < kAscendMax; ++c)
      if (c < m) cnt[c] = counter[node[c]];
    int32_t a = start[i];
    int l = lev;
    bool found = lev <= l_min;
#pragma unroll
    for (int c = 0; c < kAscendMax; ++c)
      if (!found && c < m) {
        a = node[c];
        l = lev - c;
        found = cnt[c] >= c_ray;
      }
    if (!found) {
      // past the stored levels (deeper than kAscendMax above l_min) or
      // nothing marked above l_min: continue with the parent walk
      while (l > l_min && counter[a] < c_ray) {
        a = parent[a];
        --l;
      }
    }
    keys[i] = (uint32_t)a;
    vals[i] = (uint32_t)i;
  }
}

__global__ void k_part_ascend(const int32_t* __restrict__ counter,
                              const int32_t* __restrict__ parent, const int32_t* __restrict__ start,
                              const int8_t* __restrict__ start_lev, int64_t n_max,
                              const int32_t* __restrict__ n_dev, int l_min, int c_ray,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = start[i];
    int lev = start_lev[i];
    // marked = counter >= c_ray or level == l_min; step while unmarked and above l_min
    while (lev > l_min && counter[a] < c_ray) {
      a = parent[a];
      --lev;
    }
    keys[i] = (uint32_t)a;
    vals[i] = (uint32_t)i;
  }
}

__global__ void k_part_clear(int32_t* __restrict__ counter, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ start, const int8_t* __restrict__ start_lev,
                             int64_t n_max, const int32_t* __restrict__ n_dev, int l_min) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = start[i];
    for (int l = start_lev[i]; l > l_min; --l) {
      counter[a] = 0;
      a = parent[a];
    }
  }
}

__global__ void k_part_flags(const uint32_t* __restrict__ keys, int64_t n_max,
                             const int32_t* __restrict__ n_dev, uint32_t* __restrict__ flags) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_part_bins(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                            const uint32_t* __restrict__ flags, const uint32_t* __restrict__ scan,
                            const int32_t* __restrict__ path_idx, int64_t n_max,
                            const int32_t* __restrict__ n_dev, int64_t cap,
                            int32_t* __restrict__ bin_node, int32_t* __restrict__ bin_start,
                            int32_t* __restrict__ members, int32_t* __restrict__ bin_slot,
                            const int32_t* __restrict__ item_path, int32_t* __restrict__ need) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (members) members[i] = path_idx ? path_idx[vals[i]] : (int32_t)vals[i];
    if (bin_slot) {
      uint32_t b = scan[i] + flags[i] - 1u;  // bin of this sorted position
      const int32_t p = item_path[vals[i]];
      if (p >= 0) {
        // every own item gets its slot written (-1 past the capacity), so
        // the shade kernel's reads of Lambert paths need no prior reset
        bin_slot[p] = b < cap ? (int32_t)b : -1;
        if (need && b < cap) need[b] = 1;
      }
    }
    if (flags[i]) {
      uint32_t b = scan[i];
      if (b < cap) {
        bin_node[b] = (int32_t)keys[i];
        bin_start[b] = (int32_t)i;
      }
    }
  }
}

__global__ void k_part_counts(const int32_t* __restrict__ bin_start, const uint32_t* __restrict__ nb,
                              int64_t n_max, const int32_t* __restrict__ n_dev, int64_t cap,
                              int32_t* __restrict__ bin_count, int32_t* __restrict__ n_bins_out,
                              int32_t* __restrict__ overflow) {
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t bins = *nb;
  const int64_t m = bins < cap ? bins : cap;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t end = (b + 1 < bins && b + 1 < cap) ? bin_start[b + 1] : n;
    if (b + 1 < bins && b + 1 >= cap) end = bin_start[b] + 1;  // truncated; flagged below
    bin_count[b] = (int32_t)(end - bin_start[b]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_bins_out = (int32_t)m;
    if (bins > cap && overflow) atomicOr(overflow, 1);
  }
}

size_t partition_ws_bytes(int64_t n, int chain_levels) {
  int64_t m = n > 0 ? n : 1;
  const int k = std::max(0, std::min(chain_levels, kAscendMax));
  return align_up(4 * m) + align_up(1 * m) + align_up(8 * m) + align_up(4 * m) +
         align_up(4 * (m + 1)) + align_up(4 * (m + 1)) + align_up(8) +
         (k ? align_up(4 * m * k) : 0) +
         sort_ws_bytes(m) + scan_ws_bytes(m + 1) + 4096;  // the sorted pairs may live in the sort's workspace
}

int partition_spatial(const SvoView& v, int32_t* counter, const int32_t* parent,
                      const double* pos, const int32_t* path_idx, int64_t n_max,
                      const int32_t* n_dev, int l_min, int c_ray, int n_nodes,
                      PartitionOut& out, Arena& ws, cudaStream_t st) {
  if (n_max <= 0) {
    WFPG_CUDA(cudaMemsetAsync(out.n_bins, 0, sizeof(int32_t), st));
    return WFPG_OK;
  }
  const bool given = pos == nullptr;
  int32_t* start = given ? const_cast<int32_t*>(out.start_in) : ws.take<int32_t>(n_max);
  int8_t* lev = given ? const_cast<int8_t*>(out.lev_in) : ws.take<int8_t>(n_max);
  uint32_t* keys = ws.take<uint32_t>(n_max);  // node ids < 2^31
  uint32_t* vals = ws.take<uint32_t>(n_max);
  uint32_t* flags = ws.take<uint32_t>(n_max + 1);
  uint32_t* scan = ws.take<uint32_t>(n_max + 1);
  uint32_t* nb = ws.take<uint32_t>(2);
  if (!ws.ok()) {
    set_error("partition: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  // stored ancestor chains for the ascent, when the workspace has room for
  // them next to the sort and the scan (else the parent walk)
  int n_chain = given ? 0 : std::min(kAscendMax, v.depth - l_min);
  int32_t* chain = nullptr;
  if (n_chain > 0) {
    const size_t mark = ws.off;
    chain = ws.take<int32_t>((int64_t)n_chain * n_max);
    if (ws.off + sort_ws_bytes(n_max) + scan_ws_bytes(n_max + 1) > ws.cap) {
      ws.off = mark;
      chain = nullptr;
      n_chain = 0;
    }
  }
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
  if (given) {
    if (!start || !lev) {
      set_error("partition: neither positions nor start nodes");
      return WFPG_ERR_ARG;
    }
    k_part_count_chain<<<grid, 256, 0, st>>>(counter, parent, start, lev, n_max, n_dev, l_min);
    WFPG_CHECK_LAUNCH("k_part_count_chain");
  } else {
    k_part_count<<<grid, 256, 0, st>>>(v, counter, pos, n_max, n_dev, l_min, start, lev, chain,
                                       n_chain);
    WFPG_CHECK_LAUNCH("k_part_count");
  }
  if (chain) {
    k_part_ascend_chain<<<grid, 256, 0, st>>>(counter, parent, start, lev, chain, n_chain, n_max,
                                              n_dev, l_min, c_ray, keys, vals);
    WFPG_CHECK_LAUNCH("k_part_ascend_chain");
  } else {
    k_part_ascend<<<grid, 256, 0, st>>>(counter, parent, start, lev, n_max, n_dev, l_min, c_ray,
                                        keys, vals);
    WFPG_CHECK_LAUNCH("k_part_ascend");
  }
  if (out.clear_from >= 0 && out.clear_from <= n_nodes) {
    WFPG_CUDA(cudaMemsetAsync(counter + out.clear_from, 0,
                              sizeof(int32_t) * (size_t)(n_nodes - out.clear_from), st));
  } else {
    k_part_clear<<<grid, 256, 0, st>>>(counter, parent, start, lev, n_max, n_dev, l_min);
    WFPG_CHECK_LAUNCH("k_part_clear");
  }
  // the result stays where the last pass wrote it (no copy-back); that
  // workspace is kept for the rest of the partition
  WFPG_TRY(sort_pairs_nocopy(keys, vals, n_max, n_dev, bits_for((uint64_t)n_nodes), ws, st,
                             &keys, &vals));
  k_part_flags<<<grid, 256, 0, st>>>(keys, n_max, n_dev, flags);
  WFPG_CHECK_LAUNCH("k_part_flags");
  {
    size_t mark = ws.off;
    WFPG_TRY(scan_u32(flags, scan, n_max, n_dev, nb, ws, st));
    ws.off = mark;
  }
  k_part_bins<<<grid, 256, 0, st>>>(keys, vals, flags, scan, path_idx, n_max, n_dev, out.capacity,
                                    out.bin_node, out.bin_start, out.members, out.bin_slot,
                                    out.item_path, out.need);
  WFPG_CHECK_LAUNCH("k_part_bins");
  int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(out.capacity, 256), kNumSMs * 4));
  k_part_counts<<<bgrid, 256, 0, st>>>(out.bin_start, nb, n_max, n_dev, out.capacity,
                                       out.bin_count, out.n_bins, out.overflow);
  WFPG_CHECK_LAUNCH("k_part_counts");
  out.sorted_items = vals;  // valid until the workspace is reused
  return WFPG_OK;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" size_t wfpg_partition_workspace_bytes(int64_t n, int64_t n_nodes) {
  (void)n_nodes;
  return partition_ws_bytes(n) + 256;
}

extern "C" int wfpg_partition_spatial(wfpg_svo* svo, const double* positions,
                                      const int32_t* path_idx, int64_t n, const int32_t* n_dev,
                                      int32_t l_min, int32_t c_ray, int32_t* bin_node,
                                      int32_t* bin_start, int32_t* bin_count, int32_t* members,
                                      int32_t* n_bins_dev, int64_t bin_capacity, void* workspace,
                                      size_t ws_bytes, void* stream) {
  if (!svo || !svo->counter || !svo->parent || n < 0 || (n > 0 && !positions) || !n_bins_dev ||
      !bin_node || !bin_start || !bin_count) {
    set_error("wfpg_partition_spatial: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (l_min >= svo->depth) {
    set_error("l_min must be below the SVO depth");
    return WFPG_ERR_ARG;
  }
  Arena ws(workspace, ws_bytes);
  int32_t* overflow = ws.take<int32_t>(1);
  if (!ws.ok()) {
    set_error("partition: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  cudaStream_t st = as_stream(stream);
  WFPG_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int32_t), st));
  PartitionOut out{bin_node, bin_start, bin_count, members, n_bins_dev, overflow, bin_capacity,
                   nullptr, nullptr, nullptr};
  WFPG_TRY(partition_spatial(make_view(svo), svo->counter, svo->parent, positions, path_idx, n,
                             n_dev, l_min, c_ray, (int)svo->n_nodes, out, ws, st));
  int32_t ov = 0;
  WFPG_CUDA(cudaMemcpyAsync(&ov, overflow, 4, cudaMemcpyDeviceToHost, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  if (ov) {
    set_error("partition: more bins than bin_capacity=%lld", (long long)bin_capacity);
    return WFPG_ERR_CAPACITY;
  }
  return WFPG_OK;
}

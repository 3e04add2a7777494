// One guided wavefront pass on the device (wavefront.py:198-277).
//
// All per-depth control stays on the GPU: queue lengths, lambert counts and
// bin counts are device integers consumed by grid-stride kernels sized for
// the worst case, so the whole pass is a single stream of launches with one
// host synchronisation at the end (to return PassStats).
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "comm.cuh"
#include "exitance.cuh"
#include "fields.cuh"
#include "partition.cuh"
#include "prims.cuh"
#include "svo_query.cuh"
#include "wavefront.cuh"

namespace wfpg {

constexpr int kMaxDepth = 31;
constexpr int kMatStats = 64;

struct StatsDev {
  int32_t live[kMaxDepth + 1];
  int32_t lam[kMaxDepth + 1];
  int32_t bins[kMaxDepth + 1];
  int32_t mats[kMaxDepth + 1][kMatStats];
  int32_t deposits;
  int32_t overflow;
};

// collect_bin_image (wavefront.py:254-256): depth-1 bin node per pixel; over
// the samples of a multi-sample pass the largest node id wins (the reference
// assigns bins in ascending node order, so the last write is the largest).
__global__ void k_bin_image(const int32_t* __restrict__ bin_slot,
                            const int32_t* __restrict__ bin_node, int64_t n_pix, int64_t n_samp,
                            int32_t* __restrict__ image) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pix;
       p += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = -1;
    for (int64_t s = 0; s < n_samp; ++s) {
      int32_t slot = bin_slot[s * n_pix + p];
      if (slot >= 0) v = max(v, bin_node[slot]);
    }
    image[p] = v;
  }
}

// depth >= 2: the live queue compacted from the previous depth's queue (the
// only paths that can still be alive), in the same path order
__global__ void k_flags_alive_list(const uint8_t* __restrict__ alive,
                                   const int32_t* __restrict__ prev, int64_t n_max,
                                   const int32_t* __restrict__ n_dev, uint32_t* __restrict__ flags) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = alive[prev[i]] ? 1u : 0u;
}

__global__ void k_scatter_alive_list(const uint32_t* __restrict__ flags,
                                     const uint32_t* __restrict__ scan,
                                     const int32_t* __restrict__ prev, int64_t n_max,
                                     const int32_t* __restrict__ n_dev, int32_t* __restrict__ active,
                                     const uint32_t* __restrict__ total, int32_t* __restrict__ n_out,
                                     int32_t* __restrict__ stat) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) active[scan[i]] = prev[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_out = (int32_t)*total;
    *stat = (int32_t)*total;
  }
}

// depth 1: every path was just initialised alive, so the live queue is the
// identity (no flags / scan / scatter)
__global__ void k_active_all(int64_t n, int32_t* __restrict__ active, int32_t* __restrict__ n_out,
                             int32_t* __restrict__ stat) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    active[i] = (int32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_out = (int32_t)n;
    *stat = (int32_t)n;
  }
}

// flags over the active queue: hit a lambert surface; material histogram
__global__ void k_flags_lambert(SceneView s, const int32_t* __restrict__ active,
                                const int32_t* __restrict__ n_act, const int32_t* __restrict__ hit_tri,
                                int64_t n_max, uint32_t* __restrict__ flags,
                                int32_t* __restrict__ mat_stats) {
  __shared__ int32_t hist[kMatStats];
  if (threadIdx.x < kMatStats) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = dev_count(n_max, n_act);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t tri = hit_tri[active[i]];
    uint32_t f = 0;
    if (tri >= 0) {
      int mid = s.tri_mat[tri];
      if (mid < kMatStats) atomicAdd(&hist[mid], 1);
      f = s.mat_kind[mid] == 0 ? 1u : 0u;
    }
    flags[i] = f;
  }
  __syncthreads();
  if (threadIdx.x < kMatStats && hist[threadIdx.x]) atomicAdd(&mat_stats[threadIdx.x], hist[threadIdx.x]);
}

// lambert list in path order + hit positions, numpy order o + t*d (wavefront.py:553)
__global__ void k_scatter_lambert(const int32_t* __restrict__ active,
                                  const int32_t* __restrict__ n_act,
                                  const uint32_t* __restrict__ flags,
                                  const uint32_t* __restrict__ scan, int64_t n_max,
                                  const double* __restrict__ ray_o, const double* __restrict__ ray_d,
                                  const double* __restrict__ hit_t, int32_t* __restrict__ lam,
                                  double* __restrict__ lam_pos, const uint32_t* __restrict__ total,
                                  int32_t* __restrict__ n_lam, int32_t* __restrict__ stat) {
  const int64_t n = dev_count(n_max, n_act);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    int32_t p = active[i];
    uint32_t o = scan[i];
    lam[o] = p;
    double t = hit_t[p];
    for (int c = 0; c < 3; ++c)
      lam_pos[3 * (int64_t)o + c] = __dadd_rn(ray_o[3 * (int64_t)p + c],
                                              __dmul_rn(t, ray_d[3 * (int64_t)p + c]));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_lam = (int32_t)*total;
    *stat = (int32_t)*total;
  }
}

// per-bin stream, origin pick, jitter and member slots (wavefront.py:170-189)
__global__ void k_bin_setup(const int32_t* __restrict__ n_bins, const int32_t* __restrict__ bin_node,
                            const int32_t* __restrict__ bin_start,
                            const int32_t* __restrict__ bin_count,
                            const uint32_t* __restrict__ sorted_items,
                            const int32_t* __restrict__ lam, const double* __restrict__ lam_pos,
                            uint64_t seed, const int64_t* __restrict__ sample_dev, int depth,
                            int jitter, double* __restrict__ origins,
                            double* __restrict__ jitters, int32_t* __restrict__ stat) {
  const int64_t nb = *n_bins;
  const int64_t sample0 = *sample_dev;  // device-resident so a captured graph can replay
  if (blockIdx.x == 0 && threadIdx.x == 0) *stat = (int32_t)nb;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = bin_node[b];
    const int64_t len = bin_count[b], s0 = bin_start[b];
    // bin_stream_id (wavefront.py:160-162): ((sample*64 + depth) << 32 + node) * 4 + 1
    uint64_t sid = ((((uint64_t)sample0 * 64u + (uint64_t)depth) << 32) + (uint64_t)node) * 4u + 1u;
    uint64_t key = stream_key(seed, sid);
    long long k = (long long)(u01(key, 0) * (double)len);
    if (k > len - 1) k = len - 1;
    uint32_t item = sorted_items[s0 + k];
    origins[3 * b] = lam_pos[3 * (int64_t)item];
    origins[3 * b + 1] = lam_pos[3 * (int64_t)item + 1];
    origins[3 * b + 2] = lam_pos[3 * (int64_t)item + 2];
    jitters[2 * b] = jitter ? u01(key, 1) : 0.5;
    jitters[2 * b + 1] = jitter ? u01(key, 2) : 0.5;
  }
}

__global__ void k_frame(const double* __restrict__ radiance, int64_t n_pix, int n_samples,
                        double* __restrict__ frame) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n_pix;
       q += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;  // np.add.at over paths in sample-major order
      for (int s = 0; s < n_samples; ++s)
        acc = __dadd_rn(acc, radiance[3 * ((int64_t)s * n_pix + q) + c]);
      frame[3 * q + c] = __ddiv_rn(acc, (double)n_samples);
    }
  }
}

// ---------------------------------------------------------------------------
// multi-GPU global binning (wfpg_pass_config.comm)
// ---------------------------------------------------------------------------
// Start node (deepest materialised node) of every local lambert hit, written
// at the path's slot of this rank's segment; -1 elsewhere (pre-filled).
__global__ void k_start_nodes(SvoView v, const int32_t* __restrict__ lam,
                              const double* __restrict__ lam_pos, int64_t n_max,
                              const int32_t* __restrict__ n_dev, int32_t* __restrict__ seg) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t qx = quantise(lam_pos[3 * i], v.lox, v.scale, v.resolution);
    const int32_t qy = quantise(lam_pos[3 * i + 1], v.loy, v.scale, v.resolution);
    const int32_t qz = quantise(lam_pos[3 * i + 2], v.loz, v.scale, v.resolution);
    bool pres;
    int32_t lvl;
    seg[lam[i]] = descend_view(v, qx, qy, qz, v.depth, &pres, &lvl);
  }
}

struct LevelOffsets {
  int64_t off[33];
  int depth;
};

// Compact the gathered start nodes (rank-major = global path order) into the
// partition's item arrays: start node, its level and the local path id of
// items this rank owns (-1 for the other ranks' items).
__global__ void k_global_items(const int32_t* __restrict__ all, int64_t n_all,
                               const uint32_t* __restrict__ scan, int64_t seg, int rank,
                               LevelOffsets lo, int32_t* __restrict__ start,
                               int8_t* __restrict__ lev, int32_t* __restrict__ item_path,
                               int32_t* __restrict__ item_g, const uint32_t* __restrict__ total,
                               int32_t* __restrict__ n_items) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_all;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int32_t node = all[g];
    if (node < 0) continue;
    const uint32_t o = scan[g];
    int l = 0;
    while (l < lo.depth && (int64_t)node >= lo.off[l + 1]) ++l;
    start[o] = node;
    lev[o] = (int8_t)l;
    item_path[o] = (g / seg == rank) ? (int32_t)(g % seg) : -1;
    item_g[o] = (int32_t)g;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_items = (int32_t)*total;
}

__global__ void k_flags_nonneg(const int32_t* __restrict__ a, int64_t n,
                               uint32_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = a[i] >= 0 ? 1u : 0u;
}

// wavefront.py:170-189 over global bins: the origin member is the k-th item in
// global path order; the rank that owns it contributes the hit position's bit
// pattern (every other rank contributes 0, so the all-reduced sum is an exact
// copy), jitters come from the bin's own stream on every rank.
__global__ void k_bin_setup_global(const int32_t* __restrict__ n_bins,
                                   const int32_t* __restrict__ bin_node,
                                   const int32_t* __restrict__ bin_start,
                                   const int32_t* __restrict__ bin_count,
                                   const uint32_t* __restrict__ sorted_items,
                                   const int32_t* __restrict__ item_path,
                                   const double* __restrict__ ray_o,
                                   const double* __restrict__ ray_d,
                                   const double* __restrict__ hit_t, uint64_t seed,
                                   const int64_t* __restrict__ sample_dev, int depth, int jitter,
                                   uint64_t* __restrict__ origin_bits,
                                   double* __restrict__ jitters, int32_t* __restrict__ stat) {
  const int64_t nb = *n_bins;
  const int64_t sample0 = *sample_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) *stat = (int32_t)nb;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = bin_node[b];
    const int64_t len = bin_count[b], s0 = bin_start[b];
    uint64_t sid = ((((uint64_t)sample0 * 64u + (uint64_t)depth) << 32) + (uint64_t)node) * 4u + 1u;
    uint64_t key = stream_key(seed, sid);
    long long k = (long long)(u01(key, 0) * (double)len);
    if (k > len - 1) k = len - 1;
    const int32_t p = item_path[sorted_items[s0 + k]];
    if (p >= 0) {  // k_scatter_lambert's arithmetic: o + t * d, rounded per op
      const double t = hit_t[p];
      for (int c = 0; c < 3; ++c)
        origin_bits[3 * b + c] = (uint64_t)__double_as_longlong(
            __dadd_rn(ray_o[3 * (int64_t)p + c], __dmul_rn(t, ray_d[3 * (int64_t)p + c])));
    }
    jitters[2 * b] = jitter ? u01(key, 1) : 0.5;
    jitters[2 * b + 1] = jitter ? u01(key, 2) : 0.5;
  }
}

// work-list flags of a guided depth: with bin ownership (own_hi > own_lo) the
// rank's own bin range when the bin count fits W ranges (*own_ok), else (and
// without ownership) the bins holding at least one of the rank's paths
__global__ void k_work_flags(const int32_t* __restrict__ need, const int32_t* __restrict__ n_bins,
                             int64_t cap, int64_t own_lo, int64_t own_hi, int64_t own_total,
                             int32_t* __restrict__ own_ok, uint32_t* __restrict__ flags) {
  const int64_t nb = *n_bins;
  const bool own = own_hi > own_lo && nb <= own_total;
  if (blockIdx.x == 0 && threadIdx.x == 0) *own_ok = own ? 1 : 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cap;
       b += (int64_t)gridDim.x * blockDim.x)
    flags[b] = (b < nb && (own ? (b >= own_lo && b < own_hi) : need[b] != 0)) ? 1u : 0u;
}

// bins that hold at least one of this rank's paths -> work list of the fields
__global__ void k_need_list(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ scan,
                            const int32_t* __restrict__ n_bins, int32_t* __restrict__ list,
                            const uint32_t* __restrict__ total, int32_t* __restrict__ n_list) {
  const int64_t nb = *n_bins;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    if (flags[b]) list[scan[b]] = (int32_t)b;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_list = (int32_t)*total;
}

// Deposit wire (fixed capacity per rank): record 0 = count, then up to `cap`
// records of 7 words {leaf, dir xyz, rad xyz} as bit patterns.
__global__ void k_wire_pack(const int32_t* __restrict__ leaf, const double* __restrict__ dir,
                            const double* __restrict__ rad, const int32_t* __restrict__ count,
                            int64_t cap, uint64_t* __restrict__ wire) {
  const int64_t n = *count;
  if (blockIdx.x == 0 && threadIdx.x == 0) wire[0] = (uint64_t)n;
  const int64_t m = n < cap ? n : cap;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t* r = wire + 1 + 7 * i;
    r[0] = (uint64_t)(int64_t)leaf[i];
    for (int c = 0; c < 3; ++c) {
      r[1 + c] = (uint64_t)__double_as_longlong(dir[3 * i + c]);
      r[4 + c] = (uint64_t)__double_as_longlong(rad[3 * i + c]);
    }
  }
}

// Concatenate every rank's records in rank order (global path order); if any
// rank overflowed its wire, apply nothing and raise the status word (the
// exact exchange then runs on the host side, comm.cu comm_settle).
__global__ void k_wire_unpack(const uint64_t* __restrict__ wire, int world, int64_t cap,
                              int32_t* __restrict__ leaf, double* __restrict__ dir,
                              double* __restrict__ rad, int32_t* __restrict__ n_total,
                              int32_t* __restrict__ status) {
  const int64_t stride = 1 + 7 * cap;
  bool over = false;
  int64_t tot = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t c = (int64_t)wire[r * stride];
    over |= c > cap;
    tot += c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_total = over ? 0 : (int32_t)tot;
    *status = over ? 1 : 0;
  }
  if (over) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)world * cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cap);
    const int64_t k = i % cap;
    const uint64_t* seg = wire + r * stride;
    if (k >= (int64_t)seg[0]) continue;
    int64_t o = k;
    for (int q = 0; q < r; ++q) o += (int64_t)wire[q * stride];
    const uint64_t* s = seg + 1 + 7 * k;
    leaf[o] = (int32_t)(int64_t)s[0];
    for (int c = 0; c < 3; ++c) {
      dir[3 * o + c] = __longlong_as_double((long long)s[1 + c]);
      rad[3 * o + c] = __longlong_as_double((long long)s[4 + c]);
    }
  }
}

struct PassLayout {
  int64_t P, n_pix, cap;
  int n0;
  // buffers
  int32_t* active;
  int32_t* active2;  // live queues of odd / even depths (each compacted from the other)
  uint32_t* flags;
  uint32_t* scan;
  uint32_t* total;
  int32_t* n_active;
  int32_t* n_active2;
  double* hit_t;
  int32_t* hit_tri;
  int32_t* lam;
  double* lam_pos;
  int32_t* n_lam;
  int32_t* bin_slot;
  int32_t* bin_node;
  int32_t* bin_start;
  int32_t* bin_count;
  int32_t* n_bins;
  double* origins;
  double* jitters;
  double* vals;
  double* row_sum;
  double* marg;
  double* tot;
  double* block_sums;
  double* block_rows;
  double* cum;
  int32_t* bin_ctr;  // dynamic bin scheduling of the field kernels
  uint8_t* dirty;
  double* upper_dirs;
  StatsDev* stats;
  int64_t* sample;  // device copy of cfg->sample_index (graph replays read it)
  // multi-GPU (cfg->comm)
  int world, rank;
  int64_t seg;       // per-rank segment of the gathered path arrays (max band size)
  int64_t wire_cap;  // deposit records per rank on the wire
  int32_t* g_seg;    // (seg,) this rank's start nodes
  int32_t* g_all;    // (world * seg,) everyone's
  int32_t* g_start;  // compacted items: start node, level, local path, global index
  int8_t* g_lev;
  int32_t* g_item_path;
  int32_t* g_item_g;
  int32_t* g_n_items;
  uint64_t* origin_bits;
  int32_t* need;
  int32_t* need_list;
  int32_t* n_need;
  int32_t* dep_leaf;  // local deposit export (P * max_depth)
  double* dep_dir;
  double* dep_rad;
  int32_t* dep_count;
  uint64_t* wire_send;
  uint64_t* wire_recv;
  int32_t* wdep_leaf;  // gathered deposits, global path order
  double* wdep_dir;
  double* wdep_rad;
  int32_t* wdep_n;
  int32_t* status;
  double* own_recv;   // all-gathered field values (bin ownership)
  int32_t* own_ok;
  int64_t own_seg[kMaxDepth + 1];  // S per depth (0: no ownership)
  size_t scratch_off;
};

static int64_t bin_capacity(const wfpg_svo* svo, const wfpg_pass_config* cfg, int64_t P) {
  if (!svo) return 0;
  int lm = cfg->l_min < 0 ? 0 : cfg->l_min;
  if (lm + 1 > svo->depth + 1) lm = svo->depth;
  int64_t cap = svo->level_off[lm + 1] + (int64_t)(svo->depth - lm) * (P / std::max(1, cfg->c_ray)) + 1;
  return std::max<int64_t>(1, std::min<int64_t>(cap, P));
}

static void carve_pass(Arena& a, const wfpg_svo* svo, const wfpg_camera* cam,
                       const wfpg_pass_config* cfg, PassLayout& L) {
  L.n_pix = cfg->n_pixels > 0 ? cfg->n_pixels : (int64_t)cam->width * cam->height;
  L.P = L.n_pix * std::max(1, cfg->n_samples);
  const Comm* comm = reinterpret_cast<const Comm*>(cfg->comm);
  L.world = comm_world(comm);
  L.rank = comm_rank(comm);
  const bool multi = comm && svo;
  const int64_t n_img = (int64_t)cam->width * cam->height;
  L.seg = multi ? ceil_div(n_img, L.world) : L.P;
  L.wire_cap = multi ? (cfg->dep_wire_capacity > 0 ? cfg->dep_wire_capacity
                                                   : std::max<int64_t>(1024, L.seg / 4))
                     : 0;
  // global binning: the partition sees every rank's paths
  L.cap = bin_capacity(svo, cfg, multi ? L.seg * L.world : L.P);
  L.n0 = std::max(8, cfg->field_res);
  const int64_t P = L.P;
  L.active = a.take<int32_t>(P);
  L.active2 = a.take<int32_t>(P);
  L.flags = a.take<uint32_t>(P + 1);
  L.scan = a.take<uint32_t>(P + 1);
  L.total = a.take<uint32_t>(4);
  L.n_active = a.take<int32_t>(4);
  L.n_active2 = a.take<int32_t>(4);
  L.hit_t = a.take<double>(P);
  L.hit_tri = a.take<int32_t>(P);
  L.stats = a.take<StatsDev>(1);
  L.sample = a.take<int64_t>(1);
  L.upper_dirs = a.take<double>(192);
  if (svo) {
    L.lam = a.take<int32_t>(P);
    L.lam_pos = a.take<double>(3 * P);
    L.n_lam = a.take<int32_t>(4);
    L.bin_slot = a.take<int32_t>(P);
    L.bin_node = a.take<int32_t>(L.cap);
    L.bin_start = a.take<int32_t>(L.cap);
    L.bin_count = a.take<int32_t>(L.cap);
    L.n_bins = a.take<int32_t>(4);
    L.origins = a.take<double>(3 * L.cap);
    L.jitters = a.take<double>(2 * L.cap);
    L.dirty = a.take<uint8_t>(svo->n_nodes);
    if (cfg->guided_depths > 0) {
      L.vals = a.take<double>(L.cap * (int64_t)L.n0 * L.n0);
      L.row_sum = a.take<double>(L.cap * (int64_t)L.n0);
      L.marg = a.take<double>(L.cap * (int64_t)L.n0);
      L.tot = a.take<double>(L.cap);
      L.block_sums = cfg->product ? a.take<double>(L.cap * 64) : nullptr;
      L.block_rows = cfg->product ? a.take<double>(L.cap * 8 * (int64_t)L.n0) : nullptr;
      L.cum = a.take<double>(L.cap * (int64_t)L.n0 * L.n0);
      L.bin_ctr = a.take<int32_t>(4);
    }
  }
  if (multi) {
    const int64_t G = L.seg * L.world;
    L.g_seg = a.take<int32_t>(L.seg);
    L.g_all = a.take<int32_t>(G);
    L.g_start = a.take<int32_t>(G);
    L.g_lev = a.take<int8_t>(G);
    L.g_item_path = a.take<int32_t>(G);
    L.g_item_g = a.take<int32_t>(G);
    L.g_n_items = a.take<int32_t>(4);
    L.origin_bits = a.take<uint64_t>(3 * L.cap);
    L.need = a.take<int32_t>(L.cap);
    L.need_list = a.take<int32_t>(L.cap);
    L.n_need = a.take<int32_t>(4);
    const int64_t m = P * (int64_t)std::max(1, cfg->max_depth);
    L.dep_leaf = a.take<int32_t>(m);
    L.dep_dir = a.take<double>(3 * m);
    L.dep_rad = a.take<double>(3 * m);
    L.dep_count = a.take<int32_t>(4);
    L.wire_send = a.take<uint64_t>(1 + 7 * L.wire_cap);
    L.wire_recv = a.take<uint64_t>((1 + 7 * L.wire_cap) * L.world);
    const int64_t wm = L.wire_cap * L.world;
    L.wdep_leaf = a.take<int32_t>(wm);
    L.wdep_dir = a.take<double>(3 * wm);
    L.wdep_rad = a.take<double>(3 * wm);
    L.wdep_n = a.take<int32_t>(4);
    L.status = a.take<int32_t>(4);
    // bin ownership per guided depth: S = ceil(E / W) bins per rank, usable
    // when the W ranges fit the tables
    int64_t recv = 0;
    for (int d = 0; d <= kMaxDepth; ++d) {
      L.own_seg[d] = 0;
      if (d < 1 || d > cfg->guided_depths || d > cfg->max_depth || cfg->own_bins[d] <= 0) continue;
      const int64_t S = ceil_div(cfg->own_bins[d], L.world);
      if (S * L.world > L.cap) continue;
      const int64_t n = std::max(8, cfg->field_res >> (d - 1));
      L.own_seg[d] = S;
      recv = std::max(recv, S * L.world * n * n);
    }
    L.own_recv = recv ? a.take<double>(recv) : nullptr;
    L.own_ok = a.take<int32_t>(4);
  } else {
    for (int d = 0; d <= kMaxDepth; ++d) L.own_seg[d] = 0;
  }
  L.scratch_off = a.off;
  // the local partition stores each hit's ancestor chain above l_min for
  // the ascent; the global one (start nodes given) does not
  const int chain_levels = svo ? std::max(0, svo->depth - cfg->l_min) : 0;
  size_t scratch = std::max(scan_ws_bytes(P + 1), partition_ws_bytes(P, chain_levels));
  if (multi) {
    const int64_t G = L.seg * L.world;
    scratch = std::max(scratch, std::max(scan_ws_bytes(G + 1), partition_ws_bytes(G, 0)));
    scratch = std::max(scratch, accumulate_ws_bytes(L.wire_cap * L.world) + 4096);
    scratch = std::max(scratch, 2 * align_up(4 * (G + 1)) + scan_ws_bytes(G + 1) + 4096);
  }
  if (svo) scratch = std::max(scratch, update_exitance_ws_bytes(P, cfg->max_depth));
  a.take<char>((int64_t)scratch);
}

// Live timing of the field kernels that also works inside a replayed CUDA
// graph: tiny stamp kernels on the pass stream read %globaltimer right
// before and after each field launch and fold the interval, the launch's
// bin count and its cone count into device accumulators.
struct ProfDev {
  unsigned long long t0[kMaxDepth + 1];
  double ms[kMaxDepth + 1];
  double cones[kMaxDepth + 1];
  long long launches[kMaxDepth + 1];
};
static ProfDev* g_prof_dev = nullptr;
static bool g_prof_on = false;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_stamp_begin(ProfDev* p, int depth) { p->t0[depth] = globaltimer_ns(); }
__global__ void k_stamp_end(ProfDev* p, int depth, int n, const int32_t* __restrict__ nb) {
  unsigned long long t = globaltimer_ns();
  p->ms[depth] += (double)(t - p->t0[depth]) * 1e-6;
  p->cones[depth] += (double)(*nb) * n * n;
  p->launches[depth] += 1;
}
__global__ void k_set_i64(int64_t* dst, int64_t v) { *dst = v; }

static bool cfg_ok(const wfpg_pass_config* cfg) {
  return cfg->max_depth >= 1 && cfg->max_depth <= kMaxDepth && cfg->guided_depths >= 0 &&
         cfg->guided_depths <= cfg->max_depth && cfg->c_ray >= 1 && cfg->n_samples >= 1 &&
         cfg->blur_radius >= 0 && cfg->blur_radius <= 16;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" size_t wfpg_render_workspace_bytes(const wfpg_scene* scene, const wfpg_svo* svo,
                                              const wfpg_camera* cam,
                                              const wfpg_pass_config* cfg) {
  if (!scene || !cam || !cfg) return 0;
  Arena a(nullptr, 0);
  PassLayout L;
  carve_pass(a, svo, cam, cfg, L);
  return a.off + 4096;
}

// Everything a pass enqueues after the sample index is set; capturable into a
// CUDA graph (no host synchronisation, no host-dependent control flow).
static int enqueue_pass(const wfpg_scene* scene, wfpg_svo* svo, const wfpg_camera* cam,
                        const wfpg_pass_config* cfg, wfpg_paths* paths, double* frame,
                        void* workspace, size_t ws_bytes, const PassLayout& L, ProfDev* prof,
                        cudaStream_t st) {
  Arena scratch(static_cast<char*>(workspace) + L.scratch_off, ws_bytes - L.scratch_off);
  const int64_t P = L.P;
  Comm* comm = reinterpret_cast<Comm*>(cfg->comm);
  const bool multi = comm && svo;
  const SceneView sv = make_scene_view(scene);
  const CameraView cv = make_camera_view(cam);
  const PathsView pv = make_paths_view(paths);
  SvoView vv{};
  if (svo) vv = make_view(svo);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(P, 256), kNumSMs * 8));

  WFPG_CUDA(cudaMemsetAsync(L.stats, 0, sizeof(StatsDev), st));
  const int64_t n_img = (int64_t)cam->width * cam->height;
  WFPG_TRY(launch_camera_init(cv, pv, P, L.n_pix, n_img, cfg->pixel_offset, L.sample,
                              cfg->sample_list, cfg->seed, st));

  BlurParams bp{};
  bp.radius = cfg->blur_radius;
  for (int k = 0; k <= 2 * bp.radius && bp.radius > 0; ++k) bp.w[k] = cfg->blur_w[k];

  // inter-pass overlap events (single GPU): external event nodes under capture
  const bool overlap = !comm;
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  WFPG_CUDA(cudaStreamIsCapturing(st, &cap_status));
  const bool capturing = cap_status == cudaStreamCaptureStatusActive;
  auto wait_ev = [&](void* ev) -> int {
    if (overlap && ev)
      WFPG_CUDA(cudaStreamWaitEvent(st, (cudaEvent_t)ev, capturing ? cudaEventWaitExternal : 0));
    return WFPG_OK;
  };
  auto rec_ev = [&](void* ev) -> int {
    if (overlap && ev)
      WFPG_CUDA(cudaEventRecordWithFlags((cudaEvent_t)ev, st,
                                         capturing ? cudaEventRecordExternal : 0));
    return WFPG_OK;
  };
  bool counters_waited = false, svo_waited = false;
  // the last depth that runs Alg. 2 (records "counters free" after it)
  const int last_bin_depth =
      !cfg->skip_unguided_bins
          ? cfg->max_depth
          : std::max(std::min(cfg->guided_depths, cfg->max_depth), cfg->bin_image ? 1 : 0);
  if (!svo || last_bin_depth < 1) WFPG_TRY(rec_ev(cfg->ev_rec_counters));

  for (int depth = 1; depth <= cfg->max_depth; ++depth) {
    // live queue (np.nonzero(state.alive), wavefront.py:227): the identity at
    // depth 1, then compacted from the previous depth's queue
    int32_t* const act = (depth & 1) ? L.active2 : L.active;
    int32_t* const n_act = (depth & 1) ? L.n_active2 : L.n_active;
    if (depth == 1) {
      k_active_all<<<grid, 256, 0, st>>>(P, act, n_act, &L.stats->live[depth]);
      WFPG_CHECK_LAUNCH("k_active_all");
    } else {
      const int32_t* prev = (depth & 1) ? L.active : L.active2;
      const int32_t* n_prev = (depth & 1) ? L.n_active : L.n_active2;
      k_flags_alive_list<<<grid, 256, 0, st>>>(paths->alive, prev, P, n_prev, L.flags);
      WFPG_CHECK_LAUNCH("k_flags_alive_list");
      {
        size_t mark = scratch.off;
        WFPG_TRY(scan_u32(L.flags, L.scan, P, n_prev, L.total, scratch, st));
        scratch.off = mark;
      }
      k_scatter_alive_list<<<grid, 256, 0, st>>>(L.flags, L.scan, prev, P, n_prev, act, L.total,
                                                 n_act, &L.stats->live[depth]);
      WFPG_CHECK_LAUNCH("k_scatter_alive_list");
    }
    if (depth == 1 && sv.brute) {  // primary rays share the camera position
      WFPG_TRY(launch_intersect_origin(sv, cam->position, paths->ray_d, act, P, n_act,
                                       scene->ray_eps, L.hit_t, L.hit_tri, st));
    } else {
      WFPG_TRY(launch_intersect(sv, paths->ray_o, paths->ray_d, act, P, n_act,
                                scene->ray_eps, L.hit_t, L.hit_tri, false, st));
    }

    GuideView gv{};
    gv.mode = 0;
    const int32_t* slots = nullptr;
    if (svo && depth <= last_bin_depth &&
        (!cfg->skip_unguided_bins || depth <= cfg->guided_depths || (depth == 1 && cfg->bin_image))) {
      k_flags_lambert<<<grid, 256, 0, st>>>(sv, act, n_act, L.hit_tri, P, L.flags,
                                            L.stats->mats[depth]);
      WFPG_CHECK_LAUNCH("k_flags_lambert");
      {
        size_t mark = scratch.off;
        WFPG_TRY(scan_u32(L.flags, L.scan, P, n_act, L.total, scratch, st));
        scratch.off = mark;
      }
      k_scatter_lambert<<<grid, 256, 0, st>>>(act, n_act, L.flags, L.scan, P,
                                              paths->ray_o, paths->ray_d, L.hit_t, L.lam,
                                              L.lam_pos, L.total, L.n_lam, &L.stats->lam[depth]);
      WFPG_CHECK_LAUNCH("k_scatter_lambert");
      const bool guided_depth = depth <= cfg->guided_depths;
      const bool want_image = depth == 1 && cfg->bin_image;
      // the partition writes the slot of every Lambert path it bins; the
      // shade kernel reads slots of Lambert paths only (misses, emitters and
      // mirrors return before), so only the bin image (every pixel) needs
      // the -1 reset
      if (want_image) WFPG_CUDA(cudaMemsetAsync(L.bin_slot, 0xFF, sizeof(int32_t) * P, st));
      if (!counters_waited) {  // the previous pass's partitions are done with the counters
        WFPG_TRY(wait_ev(cfg->ev_wait_counters));
        counters_waited = true;
      }
      // bin slots of guided depths are written by the partition itself
      PartitionOut po{L.bin_node, L.bin_start, L.bin_count, nullptr, L.n_bins,
                      &L.stats->overflow, L.cap, nullptr,
                      (guided_depth || want_image) ? L.bin_slot : nullptr, L.lam};
      po.clear_from = svo->level_off[cfg->l_min + 1];
      const bool global = multi && guided_depth;
      int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.cap, 128), kNumSMs * 8));
      if (global) {
        // Alg. 2 over every rank's hits: gather the start nodes (global
        // path order = rank order of the bands), partition them identically
        // on every rank, take each bin's origin from the rank owning it
        const int64_t G = L.seg * L.world;
        WFPG_CUDA(cudaMemsetAsync(L.g_seg, 0xFF, sizeof(int32_t) * L.seg, st));
        k_start_nodes<<<grid, 256, 0, st>>>(vv, L.lam, L.lam_pos, P, L.n_lam, L.g_seg);
        WFPG_CHECK_LAUNCH("k_start_nodes");
        WFPG_TRY(comm_all_gather(comm, L.g_seg, L.g_all, L.seg, kI32, st));
        {
          size_t mark = scratch.off;
          uint32_t* gflags = scratch.take<uint32_t>(G + 1);
          uint32_t* gscan = scratch.take<uint32_t>(G + 1);
          const int ggrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(G, 256), kNumSMs * 8));
          k_flags_nonneg<<<ggrid, 256, 0, st>>>(L.g_all, G, gflags);
          WFPG_CHECK_LAUNCH("k_flags_nonneg");
          WFPG_TRY(scan_u32(gflags, gscan, G, nullptr, L.total, scratch, st));
          LevelOffsets lo{};
          lo.depth = svo->depth;
          for (int l = 0; l <= svo->depth + 1 && l < 33; ++l) lo.off[l] = svo->level_off[l];
          k_global_items<<<ggrid, 256, 0, st>>>(L.g_all, G, gscan, L.seg, L.rank, lo, L.g_start,
                                                L.g_lev, L.g_item_path, L.g_item_g, L.total,
                                                L.g_n_items);
          WFPG_CHECK_LAUNCH("k_global_items");
          scratch.off = mark;
        }
        po.item_path = L.g_item_path;
        po.start_in = L.g_start;
        po.lev_in = L.g_lev;
        po.need = L.need;
        WFPG_CUDA(cudaMemsetAsync(L.need, 0, sizeof(int32_t) * L.cap, st));
        WFPG_CUDA(cudaMemsetAsync(L.origin_bits, 0, sizeof(uint64_t) * 3 * L.cap, st));
        size_t mark = scratch.off;
        WFPG_TRY(partition_spatial(vv, svo->counter, svo->parent, nullptr, nullptr, G,
                                   L.g_n_items, cfg->l_min, cfg->c_ray, (int)svo->n_nodes, po,
                                   scratch, st));
        k_bin_setup_global<<<bgrid, 128, 0, st>>>(
            L.n_bins, L.bin_node, L.bin_start, L.bin_count, po.sorted_items, L.g_item_path,
            paths->ray_o, paths->ray_d, L.hit_t, cfg->seed, L.sample, depth, cfg->jitter,
            L.origin_bits, L.jitters, &L.stats->bins[depth]);
        WFPG_CHECK_LAUNCH("k_bin_setup_global");
        scratch.off = mark;
        WFPG_TRY(comm_all_reduce_sum(comm, L.origin_bits, L.origins, 3 * L.cap, kU64, st));
        {
          size_t mk = scratch.off;
          uint32_t* nflags = scratch.take<uint32_t>(L.cap + 1);
          uint32_t* nscan = scratch.take<uint32_t>(L.cap + 1);
          const int64_t S = L.own_seg[depth];
          k_work_flags<<<bgrid, 128, 0, st>>>(L.need, L.n_bins, L.cap, L.rank * S,
                                              (L.rank + 1) * S, S * L.world, L.own_ok, nflags);
          WFPG_CHECK_LAUNCH("k_work_flags");
          WFPG_TRY(scan_u32(nflags, nscan, L.cap, nullptr, L.total, scratch, st));
          k_need_list<<<bgrid, 128, 0, st>>>(nflags, nscan, L.n_bins, L.need_list, L.total,
                                             L.n_need);
          WFPG_CHECK_LAUNCH("k_need_list");
          scratch.off = mk;
        }
      } else {
        size_t mark = scratch.off;
        WFPG_TRY(partition_spatial(vv, svo->counter, svo->parent, L.lam_pos, nullptr, P, L.n_lam,
                                   cfg->l_min, cfg->c_ray, (int)svo->n_nodes, po, scratch, st));
        k_bin_setup<<<bgrid, 128, 0, st>>>(L.n_bins, L.bin_node, L.bin_start, L.bin_count,
                                           po.sorted_items, L.lam, L.lam_pos, cfg->seed,
                                           L.sample, depth, cfg->jitter, L.origins, L.jitters,
                                           &L.stats->bins[depth]);
        WFPG_CHECK_LAUNCH("k_bin_setup");
        scratch.off = mark;
      }
      if (depth == last_bin_depth) WFPG_TRY(rec_ev(cfg->ev_rec_counters));
      if (want_image) {
        int igrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.n_pix, 256), kNumSMs * 8));
        k_bin_image<<<igrid, 256, 0, st>>>(L.bin_slot, L.bin_node, L.n_pix, P / L.n_pix,
                                           cfg->bin_image);
        WFPG_CHECK_LAUNCH("k_bin_image");
      }
      if (guided_depth) {
        const int n = std::max(8, cfg->field_res >> (depth - 1));
        FieldOut fo{L.vals, L.row_sum, L.marg, L.tot, cfg->product ? L.block_sums : nullptr,
                    cfg->epsilon, L.cum, L.bin_ctr};
        // multi-GPU: only the bins holding this rank's paths
        fo.block_rows = cfg->product ? L.block_rows : nullptr;
        const int32_t* work_n = global ? L.n_need : L.n_bins;
        fo.bin_list = global ? L.need_list : nullptr;
        WFPG_CUDA(cudaMemsetAsync(L.bin_ctr, 0, sizeof(int32_t), st));
        if (!svo_waited) {  // the previous pass's exitance update is complete
          WFPG_TRY(wait_ev(cfg->ev_wait_svo));
          svo_waited = true;
        }
        // stamped after the wait, so the field timing is the kernel's alone
        if (prof) {
          k_stamp_begin<<<1, 1, 0, st>>>(prof, depth);
          WFPG_CHECK_LAUNCH("k_stamp_begin");
        }
        WFPG_TRY(launch_fields(sv, vv, L.origins, L.jitters, L.cap, work_n, n, bp, fo, st));
        if (prof) {
          k_stamp_end<<<1, 1, 0, st>>>(prof, depth, n, work_n);
          WFPG_CHECK_LAUNCH("k_stamp_end");
        }
        if (global && L.own_seg[depth] > 0) {
          // bin ownership: everyone's floored values, then the other ranks'
          // bins' tables derived locally (bitwise the owners')
          const int64_t S = L.own_seg[depth], nn = (int64_t)n * n;
          WFPG_TRY(comm_all_gather(comm, L.vals + L.rank * S * nn, L.own_recv, S * nn, kF64, st));
          WFPG_TRY(launch_own_fill(L.own_recv, n, L.n_bins, L.own_ok, L.rank * S,
                                   (L.rank + 1) * S, L.cap, fo, st));
        }
        gv.mode = cfg->product ? 2 : 1;
        gv.n = n;
        gv.m = n / 8;
        gv.eps = cfg->epsilon;
        gv.pdf_scale = (double)(n * n) / (4.0 * WFPG_PI);
        gv.vals = L.vals;
        gv.row_sum = L.row_sum;
        gv.marg = L.marg;
        gv.total = L.tot;
        gv.block_sums = L.block_sums;
        gv.block_rows = cfg->product ? L.block_rows : nullptr;
        gv.cum = L.cum;
        gv.upper_dirs = cfg->upper_dirs;
        slots = L.bin_slot;
      }
    }
    WFPG_TRY(launch_shade(sv, gv, pv, depth, act, P, n_act, L.hit_t, L.hit_tri, slots,
                          cfg->russian_roulette != 0, cfg->rr_depth, st));
  }

  if (svo && !svo_waited) WFPG_TRY(wait_ev(cfg->ev_wait_svo));
  if (multi) {
    // Eq. 5 deposits of every rank, splatted in global path order (bands are
    // rank-ordered), so each rank's SVO update equals the 1-GPU update
    DepositSink sink{L.dep_leaf, L.dep_dir, L.dep_rad, L.dep_count,
                     P * (int64_t)std::max(1, cfg->max_depth)};
    WFPG_TRY(update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, rec_layout(paths), P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 0, nullptr, &sink));
    const int wgrid =
        (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.wire_cap, 256), kNumSMs * 4));
    k_wire_pack<<<wgrid, 256, 0, st>>>(L.dep_leaf, L.dep_dir, L.dep_rad, L.dep_count, L.wire_cap,
                                       L.wire_send);
    WFPG_CHECK_LAUNCH("k_wire_pack");
    WFPG_TRY(comm_all_gather(comm, L.wire_send, L.wire_recv, 1 + 7 * L.wire_cap, kU64, st));
    const int64_t wm = L.wire_cap * L.world;
    const int ugrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(wm, 256), kNumSMs * 4));
    k_wire_unpack<<<ugrid, 256, 0, st>>>(L.wire_recv, L.world, L.wire_cap, L.wdep_leaf,
                                         L.wdep_dir, L.wdep_rad, L.wdep_n, L.status);
    WFPG_CHECK_LAUNCH("k_wire_unpack");
    {
      size_t mark = scratch.off;
      WFPG_TRY(svo_accumulate(svo, L.wdep_leaf, L.wdep_dir, L.wdep_rad, wm, L.wdep_n,
                              cfg->deterministic, scratch, st));
      scratch.off = mark;
    }
    WFPG_CUDA(cudaMemsetAsync(L.dirty, 0, (size_t)svo->n_nodes, st));
    WFPG_TRY(svo_propagate_dirty(svo, L.wdep_leaf, wm, L.wdep_n, L.dirty, st));
    WFPG_CUDA(cudaMemcpyAsync(comm_status_host(comm), L.status, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, st));
  } else if (svo && cfg->dep_leaf) {
    // multi-GPU: export this rank's deposits; the caller gathers every rank's
    // lists and splats them in global path order (wfpg_svo_accumulate +
    // wfpg_svo_refresh_leaves), so all ranks end with the same SVO
    DepositSink sink{cfg->dep_leaf, cfg->dep_dir, cfg->dep_rad, cfg->dep_count,
                     cfg->dep_capacity};
    WFPG_TRY(update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, rec_layout(paths), P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 0, nullptr, &sink));
  } else if (svo && cfg->leaf_acc) {
    int64_t nleaf = svo->level_off[svo->depth + 1] - svo->level_off[svo->depth];
    WFPG_CUDA(cudaMemsetAsync(cfg->leaf_acc, 0, sizeof(double) * 8 * nleaf, st));
    wfpg_svo acc_view = leaf_acc_view(svo, cfg->leaf_acc);
    WFPG_TRY(update_exitance(&acc_view, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, rec_layout(paths), P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 0));
  } else if (svo) {
    // the SVO means are consistent at pass start, so only the deposited
    // subtrees need refreshing (bitwise equal to the full recompute)
    WFPG_CUDA(cudaMemsetAsync(L.dirty, 0, (size_t)svo->n_nodes, st));
    WFPG_TRY(update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, rec_layout(paths), P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 2, L.dirty));
  }
  if (svo) WFPG_TRY(rec_ev(cfg->ev_rec_svo));
  if (cfg->n_samples == 1) {
    // one sample: the mean (0 + r) / 1 is r itself (radiance sums are never
    // -0), so the frame is a plain device copy of the radiance
    WFPG_CUDA(cudaMemcpyAsync(frame, paths->radiance, sizeof(double) * 3 * (size_t)L.n_pix,
                              cudaMemcpyDeviceToDevice, st));
  } else {
    k_frame<<<(int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.n_pix, 256), kNumSMs * 8)),
              256, 0, st>>>(paths->radiance, L.n_pix, cfg->n_samples, frame);
    WFPG_CHECK_LAUNCH("k_frame");
  }

  return WFPG_OK;
}

// Eq. 7 running sum (accumulation.py:50-60): acc += hw * frame with the
// product rounded first, as numpy's `weighted_sum += hw * frame`; flags
// non-finite frame values (the reference raises on them).
__global__ void k_frame_accumulate(double* __restrict__ acc, const double* __restrict__ frame,
                                   int64_t n, double hw, int32_t* __restrict__ nonfinite) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double f = frame[i];
    if (!isfinite(f)) {
      if (nonfinite) atomicOr(nonfinite, 1);
      continue;
    }
    acc[i] = __dadd_rn(acc[i], __dmul_rn(hw, f));
  }
}

struct GraphEntry {
  const void* ws;
  uint64_t key;
  cudaGraphExec_t exec;
  uint64_t kernels;
};
// Graph cache: at most one captured graph and one "seen once" key per
// workspace (a new configuration on the same workspace replaces them);
// wfpg_graph_release drops a workspace's entries when its owner frees it.
static std::vector<GraphEntry> g_graphs;
static std::vector<std::pair<const void*, uint64_t>> g_seen;
static std::mutex g_graph_mu;

static uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// Everything that shapes the captured launch sequence: the config (minus the
// sample index, which the graph reads from device memory), all device
// pointers, sizes and the profiling switch.
static uint64_t pass_key(const wfpg_scene* sc, const wfpg_svo* svo, const wfpg_camera* cam,
                         const wfpg_pass_config* cfg, const wfpg_paths* paths, const double* frame,
                         size_t ws_bytes, const ProfDev* prof) {
  wfpg_pass_config c = *cfg;
  c.sample_index = 0;
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, &c, sizeof(c));
  h = fnv(h, sc, sizeof(*sc));
  if (svo) h = fnv(h, svo, sizeof(*svo));
  h = fnv(h, cam, sizeof(*cam));
  h = fnv(h, paths, sizeof(*paths));
  h = fnv(h, &frame, sizeof(frame));
  h = fnv(h, &ws_bytes, sizeof(ws_bytes));
  h = fnv(h, &prof, sizeof(prof));
  return h;
}

extern "C" int wfpg_render_pass(const wfpg_scene* scene, wfpg_svo* svo, const wfpg_camera* cam,
                                const wfpg_pass_config* cfg, wfpg_paths* paths, double* frame,
                                wfpg_pass_stats* stats, void* workspace, size_t ws_bytes,
                                void* stream) {
  NvtxRange nvtx_("wfpg_render_pass");
  if (!scene || !cam || !cfg || !paths || !frame || !cfg_ok(cfg)) {
    set_error("wfpg_render_pass: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (svo && cfg->l_min >= svo->depth) {
    set_error("l_min must be below the SVO depth");
    return WFPG_ERR_ARG;
  }
  if (svo && cfg->product && cfg->guided_depths > 0 && !cfg->upper_dirs) {
    set_error("wfpg_render_pass: product mode needs upper_dirs");
    return WFPG_ERR_ARG;
  }
  if (paths->max_depth != cfg->max_depth) {
    set_error("wfpg_render_pass: path state depth %d != config depth %d", paths->max_depth,
              cfg->max_depth);
    return WFPG_ERR_ARG;
  }
  Comm* comm = reinterpret_cast<Comm*>(cfg->comm);
  const bool multi = comm && svo;
  if (cfg->dep_leaf && cfg->n_samples != 1) {
    // band order is global path order only for one sample per pixel
    set_error("wfpg_render_pass: deposit export (dep_leaf) needs n_samples == 1");
    return WFPG_ERR_ARG;
  }
  if (multi && cfg->n_samples != 1) {
    set_error("wfpg_render_pass: a multi-GPU pass (comm) renders one sample per pixel");
    return WFPG_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  // the previous pass on this communicator must have applied its deposits
  if (multi) WFPG_TRY(comm_settle(comm));
  Arena a(workspace, ws_bytes);
  PassLayout L;
  carve_pass(a, svo, cam, cfg, L);
  if (!a.ok()) {
    set_error("wfpg_render_pass: workspace too small (%zu < %zu)", ws_bytes, a.off);
    return WFPG_ERR_WORKSPACE;
  }
  if (paths->n != L.P) {
    set_error("wfpg_render_pass: path state holds %lld paths, pass needs %lld",
              (long long)paths->n, (long long)L.P);
    return WFPG_ERR_ARG;
  }
  const int64_t n_img = (int64_t)cam->width * cam->height;
  if (cfg->pixel_offset < 0 || cfg->pixel_offset + L.n_pix > n_img) {
    set_error("wfpg_render_pass: pixel range outside the image");
    return WFPG_ERR_ARG;
  }
  ProfDev* prof = g_prof_on ? g_prof_dev : nullptr;
  if (multi) {
    const int64_t lo = (int64_t)L.rank * n_img / L.world, hi = (int64_t)(L.rank + 1) * n_img / L.world;
    if (cfg->pixel_offset != lo || L.n_pix != hi - lo) {
      set_error("wfpg_render_pass: rank %d must render pixels [%lld, %lld)", L.rank,
                (long long)lo, (long long)hi);
      return WFPG_ERR_ARG;
    }
  }
  k_set_i64<<<1, 1, 0, st>>>(L.sample, cfg->sample_index);
  WFPG_CHECK_LAUNCH("k_set_i64");
  if (!cfg->use_graph || (comm && !comm_capturable(comm))) {
    WFPG_TRY(enqueue_pass(scene, svo, cam, cfg, paths, frame, workspace, ws_bytes, L, prof, st));
  } else {
    const uint64_t key = pass_key(scene, svo, cam, cfg, paths, frame, ws_bytes, prof);
    std::lock_guard<std::mutex> lock(g_graph_mu);
    GraphEntry* ge = nullptr;
    for (auto& e : g_graphs)
      if (e.ws == workspace && e.key == key) ge = &e;
    bool seen = false;
    for (auto& e : g_seen)
      if (e.first == workspace && e.second == key) seen = true;
    // graphs are captured / replayed on a private non-blocking stream joined to
    // the caller's stream with events (the legacy default stream cannot be
    // captured)
    static cudaStream_t gs0 = nullptr;
    static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (!gs0) {
      WFPG_CUDA(cudaStreamCreateWithFlags(&gs0, cudaStreamNonBlocking));
      WFPG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      WFPG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    // a caller's own stream is captured / replayed on directly (so passes on
    // different streams can overlap); the legacy default stream cannot be
    // captured, so its passes go through a private stream joined by events
    const bool own_stream = st != nullptr && st != cudaStreamLegacy && st != cudaStreamPerThread;
    cudaStream_t gs = own_stream ? st : gs0;
    if ((ge || seen) && !own_stream) {
      WFPG_CUDA(cudaEventRecord(ev_fork, st));
      WFPG_CUDA(cudaStreamWaitEvent(gs, ev_fork, 0));
    }
    if (ge) {
      WFPG_CUDA(cudaGraphLaunch(ge->exec, gs));
      count_launch(ge->kernels);
      if (!own_stream) {
        WFPG_CUDA(cudaEventRecord(ev_join, gs));
        WFPG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
      }
    } else if (!seen) {
      // first pass of this configuration runs eagerly (one-time kernel attribute
      // setup happens outside any capture); the next one is captured
      for (size_t i = 0; i < g_seen.size(); ++i)
        if (g_seen[i].first == workspace) {
          g_seen.erase(g_seen.begin() + i);
          break;
        }
      g_seen.push_back({workspace, key});
      WFPG_TRY(enqueue_pass(scene, svo, cam, cfg, paths, frame, workspace, ws_bytes, L, prof, st));
    } else {
      for (size_t i = 0; i < g_graphs.size(); ++i)
        if (g_graphs[i].ws == workspace) {  // replaced configuration for this workspace
          cudaGraphExecDestroy(g_graphs[i].exec);
          g_graphs.erase(g_graphs.begin() + i);
          break;
        }
      const uint64_t before = wfpg_launch_count();
      WFPG_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_pass(scene, svo, cam, cfg, paths, frame, workspace, ws_bytes, L, prof, gs);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(gs, &graph);
      if (rc != WFPG_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamEndCapture");
      const uint64_t kernels = wfpg_launch_count() - before;
      count_launch(0 - kernels);  // captured, not executed
      cudaGraphExec_t exec;
      ce = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) return cuda_status(ce, "cudaGraphInstantiate");
      g_graphs.push_back({workspace, key, exec, kernels});
      WFPG_CUDA(cudaGraphLaunch(exec, gs));
      count_launch(kernels);
      if (!own_stream) {
        WFPG_CUDA(cudaEventRecord(ev_join, gs));
        WFPG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
      }
    }
  }

  if (multi) {
    DepositPending& pd = comm_pending(comm);
    pd.svo = *svo;
    pd.leaf = L.dep_leaf;
    pd.dir = L.dep_dir;
    pd.rad = L.dep_rad;
    pd.count = L.dep_count;
    pd.dirty = L.dirty;
    pd.stream = st;
    WFPG_CUDA(cudaEventRecord(comm_done_event(comm), st));
    pd.active = true;
  }
  if (stats) {
    StatsDev h;
    WFPG_CUDA(cudaMemcpyAsync(&h, L.stats, sizeof(StatsDev), cudaMemcpyDeviceToHost, st));
    WFPG_CUDA(cudaStreamSynchronize(st));
    if (h.overflow) {
      set_error("wfpg_render_pass: bin capacity %lld exceeded", (long long)L.cap);
      return WFPG_ERR_CAPACITY;
    }
    std::memset(stats, 0, sizeof(*stats));
    int run = 0;
    for (int d = 1; d <= cfg->max_depth; ++d) {
      if (h.live[d] == 0) break;  // the reference stops at the first empty depth
      stats->live_per_depth[run] = h.live[d];
      stats->rays_per_depth[run] = h.lam[d];
      stats->bins_per_depth[run] = h.bins[d];
      for (int m = 0; m < kMatStats; ++m) stats->mat_groups[run][m] = h.mats[d][m];
      ++run;
    }
    stats->depths_run = run;
    stats->deposits = h.deposits;
  }
  return WFPG_OK;
}

extern "C" int wfpg_profile_enable(int32_t on) {
  using namespace wfpg;
  if (!g_prof_dev) WFPG_CUDA(cudaMalloc(&g_prof_dev, sizeof(ProfDev)));
  WFPG_CUDA(cudaDeviceSynchronize());
  WFPG_CUDA(cudaMemset(g_prof_dev, 0, sizeof(ProfDev)));
  WFPG_CUDA(cudaDeviceSynchronize());
  g_prof_on = on != 0;
  return WFPG_OK;
}

// Synchronises the device and returns per-depth totals since enable.
extern "C" int wfpg_profile_read(double* field_ms, double* cones, int64_t* launches,
                                 int32_t max_depth) {
  using namespace wfpg;
  ProfDev h{};
  if (g_prof_dev) {
    WFPG_CUDA(cudaDeviceSynchronize());
    WFPG_CUDA(cudaMemcpy(&h, g_prof_dev, sizeof(ProfDev), cudaMemcpyDeviceToHost));
  }
  for (int d = 0; d <= max_depth && d <= kMaxDepth; ++d) {
    field_ms[d] = h.ms[d];
    cones[d] = h.cones[d];
    launches[d] = h.launches[d];
  }
  return WFPG_OK;
}

extern "C" int wfpg_frame_accumulate(double* acc, const double* frame, int64_t n, double hw,
                                     int32_t* nonfinite_flag, void* stream) {
  if (n < 0 || (n > 0 && (!acc || !frame))) {
    wfpg::set_error("wfpg_frame_accumulate: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(wfpg::ceil_div(n, 256),
                                                         (int64_t)wfpg::kNumSMs * 8));
  k_frame_accumulate<<<grid, 256, 0, (cudaStream_t)stream>>>(acc, frame, n, hw,
                                                                   nonfinite_flag);
  WFPG_CHECK_LAUNCH("k_frame_accumulate");
  return WFPG_OK;
}

extern "C" int wfpg_graph_release(const void* workspace) {
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (size_t i = 0; i < g_graphs.size();) {
    if (!workspace || g_graphs[i].ws == workspace) {
      cudaGraphExecDestroy(g_graphs[i].exec);
      g_graphs.erase(g_graphs.begin() + i);
    } else {
      ++i;
    }
  }
  for (size_t i = 0; i < g_seen.size();) {
    if (!workspace || g_seen[i].first == workspace)
      g_seen.erase(g_seen.begin() + i);
    else
      ++i;
  }
  return WFPG_OK;
}

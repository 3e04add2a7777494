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

#include "exitance.cuh"
#include "fields.cuh"
#include "partition.cuh"
#include "prims.cuh"
#include "svo_query.cuh"
#include "wavefront.cuh"

namespace wfpg {

constexpr int kMaxDepth = 31;
constexpr int kMatStats = 16;

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

__global__ void k_flags_alive(const uint8_t* __restrict__ alive, int64_t n,
                              uint32_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = alive[i] ? 1u : 0u;
}

__global__ void k_scatter_alive(const uint32_t* __restrict__ flags,
                                const uint32_t* __restrict__ scan, int64_t n,
                                int32_t* __restrict__ active, const uint32_t* __restrict__ total,
                                int32_t* __restrict__ n_out, int32_t* __restrict__ stat) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) active[scan[i]] = (int32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_out = (int32_t)*total;
    *stat = (int32_t)*total;
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

struct PassLayout {
  int64_t P, n_pix, cap;
  int n0;
  // buffers
  int32_t* active;
  uint32_t* flags;
  uint32_t* scan;
  uint32_t* total;
  int32_t* n_active;
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
  double* cum;
  int32_t* bin_ctr;  // dynamic bin scheduling of the field kernels
  uint8_t* dirty;
  double* upper_dirs;
  StatsDev* stats;
  int64_t* sample;  // device copy of cfg->sample_index (graph replays read it)
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
  L.cap = bin_capacity(svo, cfg, L.P);
  L.n0 = std::max(8, cfg->field_res);
  const int64_t P = L.P;
  L.active = a.take<int32_t>(P);
  L.flags = a.take<uint32_t>(P + 1);
  L.scan = a.take<uint32_t>(P + 1);
  L.total = a.take<uint32_t>(4);
  L.n_active = a.take<int32_t>(4);
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
      L.cum = a.take<double>(L.cap * (int64_t)L.n0 * L.n0);
      L.bin_ctr = a.take<int32_t>(4);
    }
  }
  L.scratch_off = a.off;
  size_t scratch = std::max(scan_ws_bytes(P + 1), partition_ws_bytes(P));
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
  const SceneView sv = make_scene_view(scene);
  const CameraView cv = make_camera_view(cam);
  const PathsView pv = make_paths_view(paths);
  SvoView vv{};
  if (svo) vv = make_view(svo);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(P, 256), kNumSMs * 8));

  WFPG_CUDA(cudaMemsetAsync(L.stats, 0, sizeof(StatsDev), st));
  const int64_t n_img = (int64_t)cam->width * cam->height;
  WFPG_TRY(launch_camera_init(cv, pv, P, L.n_pix, n_img, cfg->pixel_offset, L.sample,
                              cfg->seed, st));

  BlurParams bp{};
  bp.radius = cfg->blur_radius;
  for (int k = 0; k <= 2 * bp.radius && bp.radius > 0; ++k) bp.w[k] = cfg->blur_w[k];

  for (int depth = 1; depth <= cfg->max_depth; ++depth) {
    // live queue (np.nonzero(state.alive), wavefront.py:227)
    k_flags_alive<<<grid, 256, 0, st>>>(paths->alive, P, L.flags);
    WFPG_CHECK_LAUNCH("k_flags_alive");
    {
      size_t mark = scratch.off;
      WFPG_TRY(scan_u32(L.flags, L.scan, P, nullptr, L.total, scratch, st));
      scratch.off = mark;
    }
    k_scatter_alive<<<grid, 256, 0, st>>>(L.flags, L.scan, P, L.active, L.total, L.n_active,
                                          &L.stats->live[depth]);
    WFPG_CHECK_LAUNCH("k_scatter_alive");
    if (depth == 1 && sv.brute) {  // primary rays share the camera position
      WFPG_TRY(launch_intersect_origin(sv, cam->position, paths->ray_d, L.active, P, L.n_active,
                                       scene->ray_eps, L.hit_t, L.hit_tri, st));
    } else {
      WFPG_TRY(launch_intersect(sv, paths->ray_o, paths->ray_d, L.active, P, L.n_active,
                                scene->ray_eps, L.hit_t, L.hit_tri, false, st));
    }

    GuideView gv{};
    gv.mode = 0;
    const int32_t* slots = nullptr;
    if (svo) {
      k_flags_lambert<<<grid, 256, 0, st>>>(sv, L.active, L.n_active, L.hit_tri, P, L.flags,
                                            L.stats->mats[depth]);
      WFPG_CHECK_LAUNCH("k_flags_lambert");
      {
        size_t mark = scratch.off;
        WFPG_TRY(scan_u32(L.flags, L.scan, P, L.n_active, L.total, scratch, st));
        scratch.off = mark;
      }
      k_scatter_lambert<<<grid, 256, 0, st>>>(L.active, L.n_active, L.flags, L.scan, P,
                                              paths->ray_o, paths->ray_d, L.hit_t, L.lam,
                                              L.lam_pos, L.total, L.n_lam, &L.stats->lam[depth]);
      WFPG_CHECK_LAUNCH("k_scatter_lambert");
      const bool guided_depth = depth <= cfg->guided_depths;
      const bool want_image = depth == 1 && cfg->bin_image;
      if (guided_depth || want_image) {
        WFPG_CUDA(cudaMemsetAsync(L.bin_slot, 0xFF, sizeof(int32_t) * P, st));
      }
      // bin slots of guided depths are written by the partition itself
      PartitionOut po{L.bin_node, L.bin_start, L.bin_count, nullptr, L.n_bins,
                      &L.stats->overflow, L.cap, nullptr,
                      (guided_depth || want_image) ? L.bin_slot : nullptr, L.lam};
      po.clear_from = svo->level_off[cfg->l_min + 1];
      size_t mark = scratch.off;
      WFPG_TRY(partition_spatial(vv, svo->counter, svo->parent, L.lam_pos, nullptr, P, L.n_lam,
                                 cfg->l_min, cfg->c_ray, (int)svo->n_nodes, po, scratch, st));
      int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.cap, 128), kNumSMs * 8));
      k_bin_setup<<<bgrid, 128, 0, st>>>(L.n_bins, L.bin_node, L.bin_start, L.bin_count,
                                         po.sorted_items, L.lam, L.lam_pos, cfg->seed,
                                         L.sample, depth, cfg->jitter, L.origins, L.jitters,
                                         &L.stats->bins[depth]);
      WFPG_CHECK_LAUNCH("k_bin_setup");
      scratch.off = mark;
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
        WFPG_CUDA(cudaMemsetAsync(L.bin_ctr, 0, sizeof(int32_t), st));
        if (prof) {
          k_stamp_begin<<<1, 1, 0, st>>>(prof, depth);
          WFPG_CHECK_LAUNCH("k_stamp_begin");
        }
        WFPG_TRY(launch_fields(sv, vv, L.origins, L.jitters, L.cap, L.n_bins, n, bp, fo, st));
        if (prof) {
          k_stamp_end<<<1, 1, 0, st>>>(prof, depth, n, L.n_bins);
          WFPG_CHECK_LAUNCH("k_stamp_end");
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
        gv.cum = L.cum;
        gv.upper_dirs = cfg->upper_dirs;
        slots = L.bin_slot;
      }
    }
    WFPG_TRY(launch_shade(sv, gv, pv, depth, L.active, P, L.n_active, L.hit_t, L.hit_tri, slots,
                          cfg->russian_roulette != 0, cfg->rr_depth, st));
  }

  if (svo && cfg->dep_leaf) {
    // multi-GPU: export this rank's deposits; the caller gathers every rank's
    // lists and splats them in global path order (wfpg_svo_accumulate +
    // wfpg_svo_refresh_leaves), so all ranks end with the same SVO
    DepositSink sink{cfg->dep_leaf, cfg->dep_dir, cfg->dep_rad, cfg->dep_count,
                     cfg->dep_capacity};
    WFPG_TRY(update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, cfg->max_depth + 1, P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 0, nullptr, &sink));
  } else if (svo && cfg->leaf_acc) {
    int64_t nleaf = svo->level_off[svo->depth + 1] - svo->level_off[svo->depth];
    WFPG_CUDA(cudaMemsetAsync(cfg->leaf_acc, 0, sizeof(double) * 8 * nleaf, st));
    wfpg_svo acc_view = leaf_acc_view(svo, cfg->leaf_acc);
    WFPG_TRY(update_exitance(&acc_view, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, cfg->max_depth + 1, P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 0));
  } else if (svo) {
    // the SVO means are consistent at pass start, so only the deposited
    // subtrees need refreshing (bitwise equal to the full recompute)
    WFPG_CUDA(cudaMemsetAsync(L.dirty, 0, (size_t)svo->n_nodes, st));
    WFPG_TRY(update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T,
                             paths->rec_pos, cfg->max_depth + 1, P, cfg->deterministic,
                             &L.stats->deposits, scratch, st, 2, L.dirty));
  }
  k_frame<<<(int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L.n_pix, 256), kNumSMs * 8)), 256,
            0, st>>>(paths->radiance, L.n_pix, cfg->n_samples, frame);
  WFPG_CHECK_LAUNCH("k_frame");

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
  cudaStream_t st = as_stream(stream);
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
  k_set_i64<<<1, 1, 0, st>>>(L.sample, cfg->sample_index);
  WFPG_CHECK_LAUNCH("k_set_i64");
  if (!cfg->use_graph) {
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
    static cudaStream_t gs = nullptr;
    static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (!gs) {
      WFPG_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
      WFPG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      WFPG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    if (ge || seen) {
      WFPG_CUDA(cudaEventRecord(ev_fork, st));
      WFPG_CUDA(cudaStreamWaitEvent(gs, ev_fork, 0));
    }
    if (ge) {
      WFPG_CUDA(cudaGraphLaunch(ge->exec, gs));
      count_launch(ge->kernels);
      WFPG_CUDA(cudaEventRecord(ev_join, gs));
      WFPG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
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
      WFPG_CUDA(cudaEventRecord(ev_join, gs));
      WFPG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
    }
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

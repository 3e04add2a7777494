// Items 2 + 3 — SVO descents (_kernels.pyx:591-658), the exitance splat
// (svo.py:241-263), the bottom-up reduction (svo.py:265-313) and the
// approximate cone tracer (_kernels.pyx:661-757).
#include "geometry.cuh"
#include "prims.cuh"
#include "svo_query.cuh"

namespace wfpg {

__global__ void k_descend(SvoView v, const double* __restrict__ pts, int64_t n,
                          int32_t* __restrict__ out_node, uint8_t* __restrict__ out_present,
                          int32_t* __restrict__ out_deepest) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t qx = quantise(pts[3 * i], v.lox, v.scale, v.resolution);
    int32_t qy = quantise(pts[3 * i + 1], v.loy, v.scale, v.resolution);
    int32_t qz = quantise(pts[3 * i + 2], v.loz, v.scale, v.resolution);
    bool pres;
    int32_t lvl;
    int32_t node = descend_view(v, qx, qy, qz, v.depth, &pres, &lvl);
    if (out_node) out_node[i] = node;
    if (out_present) out_present[i] = pres ? 1 : 0;
    if (out_deepest) out_deepest[i] = node;  // compiled kernel: node == deepest
  }
}

// Quantise points to leaf coordinates with the compiled kernel's formula
// (_kernels.pyx:593-606): (long)((p - lo) * (R / size)), clamped to [0, R-1].
__global__ void k_quantise(double lox, double loy, double loz, double scale, int32_t res,
                           const double* __restrict__ pts, int64_t n,
                           int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[3 * i] = quantise(pts[3 * i], lox, scale, res);
    out[3 * i + 1] = quantise(pts[3 * i + 1], loy, scale, res);
    out[3 * i + 2] = quantise(pts[3 * i + 2], loz, scale, res);
  }
}

// ---------------------------------------------------------------------------
// exitance splat
// ---------------------------------------------------------------------------
// side a iff einsum(dir, normal) >= 0 (svo.py:256)
__device__ __forceinline__ bool splat_side_a(const double* normal, int32_t leaf, const double* d) {
  const double* nn = normal + 3 * (int64_t)leaf;
  return dot_einsum(d[0], d[1], d[2], nn[0], nn[1], nn[2]) >= 0.0;
}

__global__ void k_splat_atomic(int32_t* __restrict__ leaf, const double* __restrict__ dirs,
                               const double* __restrict__ rad, int64_t n_max,
                               const int32_t* __restrict__ n_dev, const double* __restrict__ normal,
                               double* sum_a, double* sum_b, double* w_a, double* w_b) {
  int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = leaf[i];
    if (l < 0) continue;
    bool a = splat_side_a(normal, l, dirs + 3 * i);
    double* s = (a ? sum_a : sum_b) + 3 * (int64_t)l;
    atomicAdd(s, rad[3 * i]);
    atomicAdd(s + 1, rad[3 * i + 1]);
    atomicAdd(s + 2, rad[3 * i + 2]);
    atomicAdd((a ? w_a : w_b) + l, 1.0);
  }
}

__global__ void k_splat_keys(const int32_t* __restrict__ leaf, int64_t n_max,
                             const int32_t* __restrict__ n_dev, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ idx, uint64_t sentinel) {
  int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = leaf[i];
    keys[i] = l < 0 ? sentinel : (uint64_t)l;  // misses sort last
    idx[i] = (uint32_t)i;
  }
}

// one thread per run of equal leaves: sequential adds in input order (np.add.at)
__global__ void k_splat_segments(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                 int64_t n_max, const int32_t* __restrict__ n_dev,
                                 const double* __restrict__ dirs, const double* __restrict__ rad,
                                 const double* __restrict__ normal, double* sum_a, double* sum_b,
                                 double* w_a, double* w_b, uint64_t sentinel) {
  int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    if (k == sentinel) continue;
    if (i > 0 && keys[i - 1] == k) continue;
    int32_t l = (int32_t)k;
    double a0 = sum_a[3 * (int64_t)l], a1 = sum_a[3 * (int64_t)l + 1], a2 = sum_a[3 * (int64_t)l + 2];
    double b0 = sum_b[3 * (int64_t)l], b1 = sum_b[3 * (int64_t)l + 1], b2 = sum_b[3 * (int64_t)l + 2];
    double wa = w_a[l], wb = w_b[l];
    for (int64_t j = i; j < n && keys[j] == k; ++j) {
      uint32_t s = idx[j];
      const double* r = rad + 3 * (int64_t)s;
      if (splat_side_a(normal, l, dirs + 3 * (int64_t)s)) {
        a0 = __dadd_rn(a0, r[0]);
        a1 = __dadd_rn(a1, r[1]);
        a2 = __dadd_rn(a2, r[2]);
        wa = __dadd_rn(wa, 1.0);
      } else {
        b0 = __dadd_rn(b0, r[0]);
        b1 = __dadd_rn(b1, r[1]);
        b2 = __dadd_rn(b2, r[2]);
        wb = __dadd_rn(wb, 1.0);
      }
    }
    sum_a[3 * (int64_t)l] = a0;
    sum_a[3 * (int64_t)l + 1] = a1;
    sum_a[3 * (int64_t)l + 2] = a2;
    sum_b[3 * (int64_t)l] = b0;
    sum_b[3 * (int64_t)l + 1] = b1;
    sum_b[3 * (int64_t)l + 2] = b2;
    w_a[l] = wa;
    w_b[l] = wb;
  }
}

size_t accumulate_ws_bytes(int64_t n) {
  return align_up(8 * (size_t)(n + 1)) + align_up(4 * (size_t)(n + 1)) + sort_ws_bytes(n) + 1024;
}

int svo_accumulate(wfpg_svo* svo, const int32_t* leaf, const double* dirs, const double* rad,
                   int64_t n, const int32_t* n_dev, int deterministic, Arena& ws,
                   cudaStream_t st) {
  if (n <= 0) return WFPG_OK;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8));
  if (!deterministic) {
    k_splat_atomic<<<grid, 256, 0, st>>>(const_cast<int32_t*>(leaf), dirs, rad, n, n_dev,
                                         svo->normal, svo->sum_a, svo->sum_b, svo->weight_a,
                                         svo->weight_b);
    WFPG_CHECK_LAUNCH("k_splat_atomic");
    return WFPG_OK;
  }
  uint64_t* keys = ws.take<uint64_t>(n);
  uint32_t* idx = ws.take<uint32_t>(n);
  if (!ws.ok()) {
    set_error("accumulate: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  const uint64_t sentinel = (uint64_t)svo->n_nodes;
  k_splat_keys<<<grid, 256, 0, st>>>(leaf, n, n_dev, keys, idx, sentinel);
  WFPG_CHECK_LAUNCH("k_splat_keys");
  WFPG_TRY(sort_pairs(keys, idx, n, n_dev, bits_for(sentinel), ws, st));
  k_splat_segments<<<grid, 256, 0, st>>>(keys, idx, n, n_dev, dirs, rad, svo->normal, svo->sum_a,
                                         svo->sum_b, svo->weight_a, svo->weight_b, sentinel);
  WFPG_CHECK_LAUNCH("k_splat_segments");
  return WFPG_OK;
}

// ---------------------------------------------------------------------------
// bottom-up reduction
// ---------------------------------------------------------------------------
__global__ void k_leaf_means(int64_t off, int64_t n, const double* __restrict__ sum_a,
                             const double* __restrict__ sum_b, const double* __restrict__ w_a,
                             const double* __restrict__ w_b, double* __restrict__ mean_a,
                             double* __restrict__ mean_b) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = off + k;
    double wa = w_a[i], wb = w_b[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      mean_a[3 * i + c] = wa > 0.0 ? __ddiv_rn(sum_a[3 * i + c], wa) : 0.0;
      mean_b[3 * i + c] = wb > 0.0 ? __ddiv_rn(sum_b[3 * i + c], wb) : 0.0;
    }
  }
}

// _average_children (svo.py:297-313)
__global__ void k_average_children(int64_t off, int64_t n, const int32_t* __restrict__ child_base,
                                   const uint8_t* __restrict__ child_mask,
                                   const double* __restrict__ normal, double* mean_a,
                                   double* mean_b) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = off + k;
    int64_t base = child_base[node];
    int cnt = __popc((uint32_t)child_mask[node]);
    const double* pn = normal + 3 * node;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
    for (int j = 0; j < cnt; ++j) {
      int64_t c = base + j;
      const double* cn = normal + 3 * c;
      bool aligned = dot_einsum(cn[0], cn[1], cn[2], pn[0], pn[1], pn[2]) >= 0.0;
      const double* ca = (aligned ? mean_a : mean_b) + 3 * c;
      const double* cb = (aligned ? mean_b : mean_a) + 3 * c;
      a0 = __dadd_rn(a0, ca[0]);
      a1 = __dadd_rn(a1, ca[1]);
      a2 = __dadd_rn(a2, ca[2]);
      b0 = __dadd_rn(b0, cb[0]);
      b1 = __dadd_rn(b1, cb[1]);
      b2 = __dadd_rn(b2, cb[2]);
    }
    double dc = (double)cnt;
    mean_a[3 * node] = __ddiv_rn(a0, dc);
    mean_a[3 * node + 1] = __ddiv_rn(a1, dc);
    mean_a[3 * node + 2] = __ddiv_rn(a2, dc);
    mean_b[3 * node] = __ddiv_rn(b0, dc);
    mean_b[3 * node + 1] = __ddiv_rn(b1, dc);
    mean_b[3 * node + 2] = __ddiv_rn(b2, dc);
  }
}

// Dirty-only refresh after a splat (the reference's propagate_up(dirty),
// svo.py:265-295): recompute the deposited leaves' means, flag their
// ancestors, then average flagged nodes level by level.  Internal means are
// pure functions of the leaf means, so this equals the full recompute bit for
// bit while touching only the deposited subtrees.  `dirty` (n_nodes bytes)
// must be zero on entry and is zero again on exit.
__global__ void k_dirty_leaves(const int32_t* __restrict__ leaf, int64_t n_max,
                               const int32_t* __restrict__ n_dev, const int32_t* __restrict__ parent,
                               const double* __restrict__ sum_a, const double* __restrict__ sum_b,
                               const double* __restrict__ w_a, const double* __restrict__ w_b,
                               double* __restrict__ mean_a, double* __restrict__ mean_b,
                               uint8_t* __restrict__ dirty) {
  int64_t n = dev_count(n_max, n_dev);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = leaf[k];
    if (i < 0) continue;
    const double wa = w_a[i], wb = w_b[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // identical values if several deposits share a leaf
      mean_a[3 * i + c] = wa > 0.0 ? __ddiv_rn(sum_a[3 * i + c], wa) : 0.0;
      mean_b[3 * i + c] = wb > 0.0 ? __ddiv_rn(sum_b[3 * i + c], wb) : 0.0;
    }
    for (int32_t p = parent[i]; p >= 0; p = parent[p]) dirty[p] = 1;
  }
}

__global__ void k_average_dirty(int64_t off, int64_t n, const int32_t* __restrict__ child_base,
                                const uint8_t* __restrict__ child_mask,
                                const double* __restrict__ normal, double* mean_a, double* mean_b,
                                uint8_t* __restrict__ dirty) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = off + k;
    if (!dirty[node]) continue;
    dirty[node] = 0;
    const int64_t base = child_base[node];
    const int cnt = __popc((uint32_t)child_mask[node]);
    const double* pn = normal + 3 * node;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
    for (int j = 0; j < cnt; ++j) {
      const int64_t c = base + j;
      const double* cn = normal + 3 * c;
      const bool aligned = dot_einsum(cn[0], cn[1], cn[2], pn[0], pn[1], pn[2]) >= 0.0;
      const double* ca = (aligned ? mean_a : mean_b) + 3 * c;
      const double* cb = (aligned ? mean_b : mean_a) + 3 * c;
      a0 = __dadd_rn(a0, ca[0]);
      a1 = __dadd_rn(a1, ca[1]);
      a2 = __dadd_rn(a2, ca[2]);
      b0 = __dadd_rn(b0, cb[0]);
      b1 = __dadd_rn(b1, cb[1]);
      b2 = __dadd_rn(b2, cb[2]);
    }
    const double dc = (double)cnt;
    mean_a[3 * node] = __ddiv_rn(a0, dc);
    mean_a[3 * node + 1] = __ddiv_rn(a1, dc);
    mean_a[3 * node + 2] = __ddiv_rn(a2, dc);
    mean_b[3 * node] = __ddiv_rn(b0, dc);
    mean_b[3 * node + 1] = __ddiv_rn(b1, dc);
    mean_b[3 * node + 2] = __ddiv_rn(b2, dc);
  }
}

int svo_propagate_dirty(wfpg_svo* svo, const int32_t* leaf, int64_t n_max, const int32_t* n_dev,
                        uint8_t* dirty, cudaStream_t st) {
  auto grid_for = [](int64_t m) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), (int64_t)kNumSMs * 8));
  };
  if (n_max > 0) {
    k_dirty_leaves<<<grid_for(n_max), 256, 0, st>>>(leaf, n_max, n_dev, svo->parent, svo->sum_a,
                                                    svo->sum_b, svo->weight_a, svo->weight_b,
                                                    svo->mean_a, svo->mean_b, dirty);
    WFPG_CHECK_LAUNCH("k_dirty_leaves");
  }
  for (int l = svo->depth - 1; l >= 0; --l) {
    int64_t o = svo->level_off[l], m = svo->level_off[l + 1] - o;
    k_average_dirty<<<grid_for(m), 256, 0, st>>>(o, m, svo->child_base, svo->child_mask,
                                                 svo->normal, svo->mean_a, svo->mean_b, dirty);
    WFPG_CHECK_LAUNCH("k_average_dirty");
  }
  return WFPG_OK;
}

int svo_propagate(wfpg_svo* svo, cudaStream_t st) {
  const int depth = svo->depth;
  auto grid_for = [](int64_t m) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), (int64_t)kNumSMs * 8));
  };
  int64_t lo = svo->level_off[depth], L = svo->level_off[depth + 1] - lo;
  k_leaf_means<<<grid_for(L), 256, 0, st>>>(lo, L, svo->sum_a, svo->sum_b, svo->weight_a,
                                            svo->weight_b, svo->mean_a, svo->mean_b);
  WFPG_CHECK_LAUNCH("k_leaf_means");
  for (int l = depth - 1; l >= 0; --l) {
    int64_t o = svo->level_off[l], m = svo->level_off[l + 1] - o;
    k_average_children<<<grid_for(m), 256, 0, st>>>(o, m, svo->child_base, svo->child_mask,
                                                    svo->normal, svo->mean_a, svo->mean_b);
    WFPG_CHECK_LAUNCH("k_average_children");
  }
  return WFPG_OK;
}

__global__ void k_apply_leaf_acc(int64_t off, int64_t L, const double* __restrict__ acc,
                                 double* sum_a, double* sum_b, double* w_a, double* w_b) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = off + k;
    for (int c = 0; c < 3; ++c) {
      sum_a[3 * i + c] = __dadd_rn(sum_a[3 * i + c], acc[3 * k + c]);
      sum_b[3 * i + c] = __dadd_rn(sum_b[3 * i + c], acc[3 * L + 3 * k + c]);
    }
    w_a[i] = __dadd_rn(w_a[i], acc[6 * L + k]);
    w_b[i] = __dadd_rn(w_b[i], acc[7 * L + k]);
  }
}

int svo_apply_leaf_acc(wfpg_svo* svo, const double* acc, cudaStream_t st) {
  int64_t off = svo->level_off[svo->depth], L = svo->level_off[svo->depth + 1] - off;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(L, 256), (int64_t)kNumSMs * 8));
  k_apply_leaf_acc<<<grid, 256, 0, st>>>(off, L, acc, svo->sum_a, svo->sum_b, svo->weight_a,
                                         svo->weight_b);
  WFPG_CHECK_LAUNCH("k_apply_leaf_acc");
  return svo_propagate(svo, st);
}

// A view of the SVO whose leaf accumulators are redirected into a zeroed
// per-pass leaf buffer (4 planes: sum_a, sum_b, weight_a, weight_b).
wfpg_svo leaf_acc_view(const wfpg_svo* svo, double* acc) {
  wfpg_svo v = *svo;
  int64_t off = svo->level_off[svo->depth], L = svo->level_off[svo->depth + 1] - off;
  v.sum_a = acc - 3 * off;
  v.sum_b = acc + 3 * L - 3 * off;
  v.weight_a = acc + 6 * L - off;
  v.weight_b = acc + 7 * L - off;
  return v;
}

// ---------------------------------------------------------------------------
// cone tracer (standalone batch API; the field generator inlines cone_query)
// ---------------------------------------------------------------------------
__global__ void k_trace_cones(SceneView s, SvoView v, const double* __restrict__ origins,
                              int32_t ostride, const double* __restrict__ dirs, int64_t n,
                              double omega, double* __restrict__ out) {
  extern __shared__ TriRec smt[];
  if (s.brute) load_tris_smem(s, smt);
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* o = origins + (int64_t)ostride * i;
    double rgb[3];
    cone_query(s, smt, v, o[0], o[1], o[2], dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], omega,
               rgb);
    out[3 * i] = rgb[0];
    out[3 * i + 1] = rgb[1];
    out[3 * i + 2] = rgb[2];
  }
}

}  // namespace wfpg

using namespace wfpg;

static bool svo_ok(const wfpg_svo* s) {
  return s && s->node_desc && s->depth >= 1 && s->depth <= 21 && s->resolution == (1 << s->depth);
}

extern "C" int wfpg_descend(const wfpg_svo* svo, const double* points, int64_t n,
                            int32_t* out_node, uint8_t* out_present, int32_t* out_deepest,
                            void* stream) {
  if (!svo_ok(svo) || n < 0 || (n > 0 && !points)) {
    set_error("wfpg_descend: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  SvoView v = make_view(svo);
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8);
  k_descend<<<grid, 256, 0, as_stream(stream)>>>(v, points, n, out_node, out_present, out_deepest);
  WFPG_CHECK_LAUNCH("k_descend");
  return WFPG_OK;
}

extern "C" int wfpg_svo_refresh_leaves(wfpg_svo* svo, const int32_t* leaf, int64_t n,
                                       uint8_t* dirty, void* stream) {
  if (!svo_ok(svo) || n < 0 || (n > 0 && !leaf) || !dirty) {
    set_error("wfpg_svo_refresh_leaves: bad arguments");
    return WFPG_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  WFPG_CUDA(cudaMemsetAsync(dirty, 0, (size_t)svo->n_nodes, st));
  return svo_propagate_dirty(svo, leaf, n, nullptr, dirty, st);
}

extern "C" int wfpg_quantise_points(const double* cube_lo, double cube_size, int32_t resolution,
                                    const double* points, int64_t n, int32_t* out_coords,
                                    void* stream) {
  if (!cube_lo || !(cube_size > 0.0) || resolution < 1 || n < 0 ||
      (n > 0 && (!points || !out_coords))) {
    set_error("wfpg_quantise_points: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  double scale = (double)resolution / cube_size;
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8);
  k_quantise<<<grid, 256, 0, as_stream(stream)>>>(cube_lo[0], cube_lo[1], cube_lo[2], scale,
                                                  resolution, points, n, out_coords);
  WFPG_CHECK_LAUNCH("k_quantise");
  return WFPG_OK;
}

extern "C" size_t wfpg_accumulate_workspace_bytes(int64_t n) { return accumulate_ws_bytes(n); }

extern "C" int wfpg_svo_accumulate(wfpg_svo* svo, const int32_t* leaf, const double* dirs,
                                   const double* rad, int64_t n, const int32_t* n_dev,
                                   int32_t deterministic, void* workspace, size_t ws_bytes,
                                   void* stream) {
  if (!svo_ok(svo) || n < 0 || (n > 0 && (!leaf || !dirs || !rad))) {
    set_error("wfpg_svo_accumulate: bad arguments");
    return WFPG_ERR_ARG;
  }
  Arena ws(workspace, ws_bytes);
  return svo_accumulate(svo, leaf, dirs, rad, n, n_dev, deterministic, ws, as_stream(stream));
}

extern "C" int wfpg_svo_propagate(wfpg_svo* svo, void* stream) {
  if (!svo_ok(svo)) {
    set_error("wfpg_svo_propagate: bad arguments");
    return WFPG_ERR_ARG;
  }
  return svo_propagate(svo, as_stream(stream));
}

extern "C" int wfpg_svo_apply_leaf_acc(wfpg_svo* svo, const double* leaf_acc, void* stream) {
  if (!svo_ok(svo) || !leaf_acc) {
    set_error("wfpg_svo_apply_leaf_acc: bad arguments");
    return WFPG_ERR_ARG;
  }
  return svo_apply_leaf_acc(svo, leaf_acc, as_stream(stream));
}

extern "C" int wfpg_trace_cones(const wfpg_scene* scene, const wfpg_svo* svo,
                                const double* origins, int32_t origin_stride, const double* dirs,
                                int64_t n, double omega, double* out, void* stream) {
  if (!scene || !svo_ok(svo) || n < 0 || (n > 0 && (!origins || !dirs || !out))) {
    set_error("wfpg_trace_cones: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  SceneView s = make_scene_view(scene);
  SvoView v = make_view(svo);
  size_t smem = s.brute ? sizeof(TriRec) * s.n_tris : 0;
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8);
  k_trace_cones<<<grid, 256, smem, as_stream(stream)>>>(s, v, origins, origin_stride, dirs, n,
                                                        omega, out);
  WFPG_CHECK_LAUNCH("k_trace_cones");
  return WFPG_OK;
}

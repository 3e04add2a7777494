// BVH construction on the device for large scenes, a
// linear BVH (Karras 2012, "Maximizing parallelism in the construction of
// BVHs, octrees, and k-d trees") on the SVO builder's Morton / radix-sort
// machinery.  It replaces the host build (bvh.py:33-119, binned SAH, ~20 s
// per 100 K triangles in numpy) where that is too slow; the traversals
// (bvh_nearest / bvh_occluded, _kernels.pyx:398-478) are unchanged.  The
// nearest hit is the minimum t over the triangles a ray meets, so results
// equal the host-BVH ones except for exact ties (a ray through a shared
// edge), which take the tree's visiting order as in the reference.
//
// Output layout = the host BVH's flattened arrays: node 0 is the root,
// internal nodes 0 .. n-2 (count 0, left / right children), leaves
// n-1 .. 2n-2 with one triangle each (count 1, left = slot in `order`);
// internal nodes over at most 4 triangles are then turned into leaves
// (count = size, left = first slot), leaving their subtrees unreachable.
#include "prims.cuh"

namespace wfpg {

// Karras' prefix metric on sorted keys: common leading bits, with the index
// as a tie-breaker for equal keys; -1 outside [0, n).
__device__ __forceinline__ int lbvh_delta(const uint64_t* __restrict__ k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  const uint64_t a = k[i], b = k[j];
  if (a == b) return 64 + __clz((uint32_t)i ^ (uint32_t)j);
  return __clzll(a ^ b);
}

__global__ void k_lbvh_codes(const double* __restrict__ v0, const double* __restrict__ v1,
                             const double* __restrict__ v2, int n, double lox, double loy,
                             double loz, double inv_x, double inv_y, double inv_z,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    // centroid of the triangle's box (bvh.py's split key), 21 bits per axis
    double c[3];
    for (int a = 0; a < 3; ++a) {
      const double x0 = v0[3 * t + a], x1 = v1[3 * t + a], x2 = v2[3 * t + a];
      c[a] = 0.5 * (fmin(x0, fmin(x1, x2)) + fmax(x0, fmax(x1, x2)));
    }
    auto q = [](double u) {
      const double s = u * 2097152.0;
      return (uint64_t)(s < 0.0 ? 0.0 : (s > 2097151.0 ? 2097151.0 : s));
    };
    keys[t] = morton3(q((c[0] - lox) * inv_x), q((c[1] - loy) * inv_y), q((c[2] - loz) * inv_z));
    idx[t] = (uint32_t)t;
  }
}

__global__ void k_lbvh_hierarchy(const uint64_t* __restrict__ k, int n,
                                 int32_t* __restrict__ left, int32_t* __restrict__ right,
                                 int32_t* __restrict__ count, int32_t* __restrict__ parent,
                                 int32_t* __restrict__ span) {
  const int leaf0 = n - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // leaf i
    left[leaf0 + i] = i;
    right[leaf0 + i] = -1;
    count[leaf0 + i] = 1;
    if (i >= n - 1) continue;
    // internal node i
    const int d = lbvh_delta(k, n, i, i + 1) - lbvh_delta(k, n, i, i - 1) >= 0 ? 1 : -1;
    const int dmin = lbvh_delta(k, n, i, i - d);
    int lmax = 2;
    while (lbvh_delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
      if (lbvh_delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = lbvh_delta(k, n, i, j);
    int s = 0, t = l;
    do {
      t = (t + 1) >> 1;
      if (lbvh_delta(k, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    const int gamma = i + s * d + (d < 0 ? d : 0);
    const int cl = (min(i, j) == gamma) ? leaf0 + gamma : gamma;
    const int cr = (max(i, j) == gamma + 1) ? leaf0 + gamma + 1 : gamma + 1;
    left[i] = cl;
    right[i] = cr;
    count[i] = 0;
    parent[cl] = i;
    parent[cr] = i;
    span[2 * i] = min(i, j);  // the node covers sorted primitives [first, last]
    span[2 * i + 1] = max(i, j);
  }
}

// Subtrees of at most kLeafTris triangles become one leaf over their
// contiguous slice of `order` (the host build's leaf size, bvh.py:14); the
// nodes below stay in the arrays but are no longer reachable.
constexpr int kLeafTris = 4;
__global__ void k_lbvh_collapse(int n, const int32_t* __restrict__ span,
                                int32_t* __restrict__ left, int32_t* __restrict__ count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    const int first = span[2 * i], size = span[2 * i + 1] - first + 1;
    if (size <= kLeafTris) {
      left[i] = first;
      count[i] = size;
    }
  }
}

// padded fp32 copy of a node box (scene.py _bvh_boxes_f32)
__device__ __forceinline__ void lbvh_store_box(double* lo, double* hi, float* box, int node,
                                               const double* l, const double* h, double pad0) {
  for (int a = 0; a < 3; ++a) {
    lo[3 * node + a] = l[a];
    hi[3 * node + a] = h[a];
    box[8 * node + a] = __double2float_rd(l[a] - (pad0 + 4e-7 * fabs(l[a])));
    box[8 * node + 4 + a] = __double2float_ru(h[a] + (pad0 + 4e-7 * fabs(h[a])));
  }
  box[8 * node + 3] = 0.0f;
  box[8 * node + 7] = 0.0f;
}

// Bottom-up boxes: each leaf walks toward the root; the second child to
// arrive at a node (atomic ticket) merges both boxes and continues.
__global__ void k_lbvh_boxes(const double* __restrict__ v0, const double* __restrict__ v1,
                             const double* __restrict__ v2, const uint32_t* __restrict__ sorted,
                             int n, const int32_t* __restrict__ left,
                             const int32_t* __restrict__ right, const int32_t* __restrict__ parent,
                             uint32_t* __restrict__ ticket, double* lo, double* hi, float* box,
                             int32_t* __restrict__ order, double pad0) {
  const int leaf0 = n - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int t = (int)sorted[i];
    order[i] = t;
    double l[3], h[3];
    for (int a = 0; a < 3; ++a) {
      const double x0 = v0[3 * t + a], x1 = v1[3 * t + a], x2 = v2[3 * t + a];
      l[a] = fmin(fmin(x0, x1), x2);
      h[a] = fmax(fmax(x0, x1), x2);
    }
    int node = leaf0 + i;
    lbvh_store_box(lo, hi, box, node, l, h, pad0);
    while (node != 0) {
      const int p = parent[node];
      __threadfence();
      if (atomicAdd(&ticket[p], 1u) == 0u) break;  // the sibling finishes this node
      __threadfence();
      const int c0 = left[p], c1 = right[p];
      const volatile double* vlo = lo;
      const volatile double* vhi = hi;
      for (int a = 0; a < 3; ++a) {
        l[a] = fmin(vlo[3 * c0 + a], vlo[3 * c1 + a]);
        h[a] = fmax(vhi[3 * c0 + a], vhi[3 * c1 + a]);
      }
      lbvh_store_box(lo, hi, box, p, l, h, pad0);
      node = p;
    }
  }
}

// tree depth (longest leaf-to-root walk): the traversals keep 64-entry stacks
__global__ void k_lbvh_depth(const int32_t* __restrict__ parent, int n, int32_t* __restrict__ out) {
  int deepest = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int node = n - 1 + i, d = 0;
    while (node != 0) {
      node = parent[node];
      ++d;
    }
    deepest = max(deepest, d);
  }
  atomicMax(out, deepest);
}

}  // namespace wfpg

using namespace wfpg;

extern "C" size_t wfpg_bvh_build_workspace_bytes(int64_t n_tris) {
  Arena a(nullptr, 0);
  const int64_t n = n_tris > 0 ? n_tris : 1;
  a.take<uint64_t>(n);
  a.take<uint32_t>(n);
  a.take<int32_t>(2 * n);
  a.take<uint32_t>(n);
  a.take<int32_t>(1);
  a.take<int32_t>(2 * n);
  return a.off + sort_ws_bytes(n) + 1024;
}

extern "C" int wfpg_bvh_build_device(const wfpg_scene* scene, double* lo, double* hi,
                                     int32_t* left, int32_t* right, int32_t* count,
                                     int32_t* order, float* box_f32, void* workspace,
                                     size_t ws_bytes, void* stream) {
  if (!scene || scene->n_tris <= 0 || !scene->v0 || !scene->v1 || !scene->v2 || !lo || !hi ||
      !left || !right || !count || !order || !box_f32) {
    set_error("wfpg_bvh_build_device: bad arguments");
    return WFPG_ERR_ARG;
  }
  const int n = scene->n_tris;
  cudaStream_t st = as_stream(stream);
  Arena a(workspace, ws_bytes);
  uint64_t* keys = a.take<uint64_t>(n);
  uint32_t* idx = a.take<uint32_t>(n);
  int32_t* parent = a.take<int32_t>(2 * (int64_t)n);
  uint32_t* ticket = a.take<uint32_t>(n);
  int32_t* depth_dev = a.take<int32_t>(1);
  int32_t* span = a.take<int32_t>(2 * (int64_t)n);
  if (!a.ok()) {
    set_error("bvh build: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  double ext[3], inv[3];
  double diag2 = 0.0;
  for (int k = 0; k < 3; ++k) {
    ext[k] = scene->bbox_hi[k] - scene->bbox_lo[k];
    inv[k] = ext[k] > 0.0 ? 1.0 / ext[k] : 0.0;
    diag2 += ext[k] * ext[k];
  }
  const double pad0 = 1e-5 * sqrt(diag2);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8));
  k_lbvh_codes<<<grid, 256, 0, st>>>(scene->v0, scene->v1, scene->v2, n, scene->bbox_lo[0],
                                     scene->bbox_lo[1], scene->bbox_lo[2], inv[0], inv[1], inv[2],
                                     keys, idx);
  WFPG_CHECK_LAUNCH("k_lbvh_codes");
  WFPG_TRY(sort_pairs(keys, idx, n, nullptr, 63, a, st));
  WFPG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(uint32_t) * (size_t)n, st));
  WFPG_CUDA(cudaMemsetAsync(parent, 0xff, sizeof(int32_t) * 2 * (size_t)n, st));
  k_lbvh_hierarchy<<<grid, 256, 0, st>>>(keys, n, left, right, count, parent, span);
  WFPG_CHECK_LAUNCH("k_lbvh_hierarchy");
  k_lbvh_boxes<<<grid, 256, 0, st>>>(scene->v0, scene->v1, scene->v2, idx, n, left, right, parent,
                                     ticket, lo, hi, box_f32, order, pad0);
  WFPG_CHECK_LAUNCH("k_lbvh_boxes");
  WFPG_CUDA(cudaMemsetAsync(depth_dev, 0, sizeof(int32_t), st));
  k_lbvh_depth<<<grid, 256, 0, st>>>(parent, n, depth_dev);
  WFPG_CHECK_LAUNCH("k_lbvh_depth");
  k_lbvh_collapse<<<grid, 256, 0, st>>>(n, span, left, count);
  WFPG_CHECK_LAUNCH("k_lbvh_collapse");
  int32_t depth = 0;
  WFPG_CUDA(cudaMemcpyAsync(&depth, depth_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  if (depth > 62) {  // a DFS stack holds at most depth + 1 entries
    set_error("device BVH depth %d exceeds the 64-entry traversal stacks", depth);
    return WFPG_ERR_ARG;
  }
  return WFPG_OK;
}

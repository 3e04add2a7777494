// Item 1 — SVO builder: conservative voxelisation (svo.py:49-136), Morton
// encoding + stable device radix sort + run-length unique (svo.py:424-433),
// level-by-level node allocation (svo.py:435-470) and the dual-normal k-means
// (svo.py:139-173, 472-499).  Every integer array and the normals are
// bit-exact with the reference; the fp64 steps use explicitly rounded
// intrinsics in numpy/OpenBLAS operation order (oracle/NUMERICS.md).
#include <vector>

#include "prims.cuh"

namespace wfpg {

// ---------------------------------------------------------------------------
// voxelisation
// ---------------------------------------------------------------------------
struct VoxRange {
  int32_t lo[3];
  int32_t n[3];
};

// svo.py:111-115: floor((tlo - cube_lo) / h) clipped to [0, r-1]
__device__ __forceinline__ int32_t vox_floor_clip(double x, double lo, double h, int32_t r) {
  double q = floor(__ddiv_rn(__dsub_rn(x, lo), h));
  long long qi = (long long)q;
  if (qi < 0) qi = 0;
  if (qi > r - 1) qi = r - 1;
  return (int32_t)qi;
}

__global__ void k_vox_ranges(const double* __restrict__ v0, const double* __restrict__ v1,
                             const double* __restrict__ v2, int32_t T, double lx, double ly,
                             double lz, double h, int32_t r, VoxRange* __restrict__ out,
                             int64_t* __restrict__ counts) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double lo3[3] = {lx, ly, lz};
  VoxRange vr;
  int64_t cnt = 1;
  for (int a = 0; a < 3; ++a) {
    double x0 = v0[3 * t + a], x1 = v1[3 * t + a], x2 = v2[3 * t + a];
    double tlo = fmin(fmin(x0, x1), x2);
    double thi = fmax(fmax(x0, x1), x2);
    int32_t ilo = vox_floor_clip(tlo, lo3[a], h, r);
    int32_t ihi = vox_floor_clip(thi, lo3[a], h, r);
    vr.lo[a] = ilo;
    vr.n[a] = ihi >= ilo ? ihi - ilo + 1 : 0;
    cnt *= vr.n[a];
  }
  out[t] = vr;
  counts[t] = cnt;
}

struct TriSat {
  double v0[3], v1[3], v2[3];
  double e[3][3];   // edges v1-v0, v2-v1, v0-v2
  double nrm[3];    // np.cross(e0, e1)
};

// K rows in the reference's batched matmul decide the BLAS kernel:
// (1,3)@(3,) takes the ddot order, K>=2 the dgemv order.
__device__ __forceinline__ double sat_dot(bool single, double x0, double x1, double x2, double m0,
                                          double m1, double m2) {
  return single ? dot_ddot(x0, x1, x2, m0, m1, m2) : dot_gemv(x0, x1, x2, m0, m1, m2);
}

// One axis of _tri_box_overlap (svo.py:71-82).  Returns false when separated.
__device__ __forceinline__ bool sat_axis(bool single, const double* a, const double* b,
                                         const double* d, const double* hh, double x, double y,
                                         double z) {
  // np.linalg.norm(axis) < 1e-30 -> test skipped
  double nrm = __dsqrt_rn(dot_ddot(x, y, z, x, y, z));
  if (nrm < 1e-30) return true;
  double pa = sat_dot(single, a[0], a[1], a[2], x, y, z);
  double pb = sat_dot(single, b[0], b[1], b[2], x, y, z);
  double pd = sat_dot(single, d[0], d[1], d[2], x, y, z);
  double r = sat_dot(single, hh[0], hh[1], hh[2], fabs(x), fabs(y), fabs(z));
  double lo = fmin(fmin(pa, pb), pd);
  double hi = fmax(fmax(pa, pb), pd);
  return (lo <= r) && (hi >= -r);
}

__device__ bool tri_box_overlap(const TriSat& T, bool single, const double* box_lo,
                                const double* box_hi) {
  double c[3], hh[3], a[3], b[3], d[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = __dmul_rn(0.5, __dadd_rn(box_lo[k], box_hi[k]));
    hh[k] = __dmul_rn(0.5, __dsub_rn(box_hi[k], box_lo[k]));
    a[k] = __dsub_rn(T.v0[k], c[k]);
    b[k] = __dsub_rn(T.v1[k], c[k]);
    d[k] = __dsub_rn(T.v2[k], c[k]);
  }
  // box face normals (svo.py:64-67)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double lo = fmin(fmin(a[k], b[k]), d[k]);
    double hi = fmax(fmax(a[k], b[k]), d[k]);
    if (!((lo <= hh[k]) && (hi >= -hh[k]))) return false;
  }
  // triangle normal (svo.py:85)
  if (!sat_axis(single, a, b, d, hh, T.nrm[0], T.nrm[1], T.nrm[2])) return false;
  // nine edge cross products (svo.py:87-90)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double* e = T.e[k];
    if (!sat_axis(single, a, b, d, hh, 0.0, -e[2], e[1])) return false;
    if (!sat_axis(single, a, b, d, hh, e[2], 0.0, -e[0])) return false;
    if (!sat_axis(single, a, b, d, hh, -e[1], e[0], 0.0)) return false;
  }
  return true;
}

__device__ __forceinline__ void load_tri_sat(const double* v0, const double* v1, const double* v2,
                                             int t, TriSat& T) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T.v0[k] = v0[3 * t + k];
    T.v1[k] = v1[3 * t + k];
    T.v2[k] = v2[3 * t + k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T.e[0][k] = __dsub_rn(T.v1[k], T.v0[k]);
    T.e[1][k] = __dsub_rn(T.v2[k], T.v1[k]);
    T.e[2][k] = __dsub_rn(T.v0[k], T.v2[k]);
  }
  // np.cross: (a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0)
  const double* p = T.e[0];
  const double* q = T.e[1];
  T.nrm[0] = __dsub_rn(__dmul_rn(p[1], q[2]), __dmul_rn(p[2], q[1]));
  T.nrm[1] = __dsub_rn(__dmul_rn(p[2], q[0]), __dmul_rn(p[0], q[2]));
  T.nrm[2] = __dsub_rn(__dmul_rn(p[0], q[1]), __dmul_rn(p[1], q[0]));
}

__device__ __forceinline__ int find_tri(const int64_t* __restrict__ off, int T, int64_t c) {
  // largest t with off[t] <= c
  int lo = 0, hi = T - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(&off[mid]) <= c)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void cand_coords(const VoxRange& vr, int64_t l, int32_t* x, int32_t* y,
                                            int32_t* z) {
  // meshgrid(indexing="ij").ravel(): x slowest, z fastest (svo.py:116-122)
  int64_t nyz = (int64_t)vr.n[1] * vr.n[2];
  *x = vr.lo[0] + (int32_t)(l / nyz);
  int64_t rem = l % nyz;
  *y = vr.lo[1] + (int32_t)(rem / vr.n[2]);
  *z = vr.lo[2] + (int32_t)(rem % vr.n[2]);
}

__global__ void k_vox_test(const double* __restrict__ v0, const double* __restrict__ v1,
                           const double* __restrict__ v2, int32_t T,
                           const VoxRange* __restrict__ ranges, const int64_t* __restrict__ off,
                           int64_t C, double lx, double ly, double lz, double h,
                           uint32_t* __restrict__ flags) {
  const double lo3[3] = {lx, ly, lz};
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    int t = find_tri(off, T, c);
    VoxRange vr = ranges[t];
    int64_t k = c - off[t];
    int64_t K = off[t + 1] - off[t];
    int32_t q[3];
    cand_coords(vr, k, &q[0], &q[1], &q[2]);
    TriSat S;
    load_tri_sat(v0, v1, v2, t, S);
    double blo[3], bhi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      blo[a] = __dadd_rn(lo3[a], __dmul_rn((double)q[a], h));  // cube_lo + cand * h
      bhi[a] = __dadd_rn(blo[a], h);
    }
    flags[c] = tri_box_overlap(S, K == 1, blo, bhi) ? 1u : 0u;
  }
}

__global__ void k_vox_emit(const VoxRange* __restrict__ ranges, const int64_t* __restrict__ off,
                           int32_t T, int64_t C, const uint32_t* __restrict__ flag_src,
                           const uint32_t* __restrict__ pos, int32_t* __restrict__ coords,
                           int32_t* __restrict__ tris) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (!flag_src[c]) continue;
    int t = find_tri(off, T, c);
    int32_t x, y, z;
    cand_coords(ranges[t], c - off[t], &x, &y, &z);
    uint32_t p = pos[c];
    coords[3 * (int64_t)p] = x;
    coords[3 * (int64_t)p + 1] = y;
    coords[3 * (int64_t)p + 2] = z;
    tris[p] = t;
  }
}

static int vox_common(const wfpg_scene* sc, const double* cube_lo, double side, int32_t r,
                      Arena& ws, cudaStream_t st, VoxRange** ranges_out, int64_t** off_out,
                      std::vector<int64_t>& off_host) {
  int32_t T = sc->n_tris;
  VoxRange* ranges = ws.take<VoxRange>(T);
  int64_t* counts = ws.take<int64_t>(T + 1);
  int64_t* off = ws.take<int64_t>(T + 1);
  if (!ws.ok()) {
    set_error("voxelize: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  double h = side / r;  // svo.py:106
  k_vox_ranges<<<(unsigned)ceil_div(T, 128), 128, 0, st>>>(sc->v0, sc->v1, sc->v2, T, cube_lo[0],
                                                          cube_lo[1], cube_lo[2], h, r, ranges,
                                                          counts);
  WFPG_CHECK_LAUNCH("k_vox_ranges");
  std::vector<int64_t> ch(T);
  WFPG_CUDA(cudaMemcpyAsync(ch.data(), counts, sizeof(int64_t) * T, cudaMemcpyDeviceToHost, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  off_host.assign(T + 1, 0);
  for (int t = 0; t < T; ++t) off_host[t + 1] = off_host[t] + ch[t];
  WFPG_CUDA(cudaMemcpyAsync(off, off_host.data(), sizeof(int64_t) * (T + 1),
                            cudaMemcpyHostToDevice, st));
  *ranges_out = ranges;
  *off_out = off;
  return WFPG_OK;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" size_t wfpg_voxelize_workspace_bytes(int32_t n_tris, int64_t n_candidates) {
  size_t b = align_up(sizeof(VoxRange) * (n_tris + 1)) + 2 * align_up(8 * (n_tris + 2));
  if (n_candidates > 0)
    b += 2 * align_up(sizeof(uint32_t) * n_candidates) + scan_ws_bytes(n_candidates) + 256;
  return b + 1024;
}

extern "C" int wfpg_voxelize_count(const wfpg_scene* sc, const double* cube_lo, double side,
                                   int32_t resolution, int64_t* n_candidates, void* workspace,
                                   size_t ws_bytes, void* stream) {
  if (!sc || !cube_lo || !n_candidates || resolution <= 0 || (resolution & (resolution - 1))) {
    set_error("resolution must be a positive power of two");
    return WFPG_ERR_ARG;
  }
  Arena ws(workspace, ws_bytes);
  VoxRange* ranges;
  int64_t* off;
  std::vector<int64_t> oh;
  WFPG_TRY(vox_common(sc, cube_lo, side, resolution, ws, as_stream(stream), &ranges, &off, oh));
  *n_candidates = oh.back();
  return WFPG_OK;
}

extern "C" int wfpg_voxelize_emit(const wfpg_scene* sc, const double* cube_lo, double side,
                                  int32_t resolution, int64_t n_candidates, int32_t* out_coords,
                                  int32_t* out_tris, int64_t capacity, int64_t* n_fragments,
                                  void* workspace, size_t ws_bytes, void* stream) {
  if (!sc || !cube_lo || !n_fragments || resolution <= 0 || (resolution & (resolution - 1))) {
    set_error("resolution must be a positive power of two");
    return WFPG_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  Arena ws(workspace, ws_bytes);
  VoxRange* ranges;
  int64_t* off;
  std::vector<int64_t> oh;
  WFPG_TRY(vox_common(sc, cube_lo, side, resolution, ws, st, &ranges, &off, oh));
  int64_t C = oh.back();
  if (C != n_candidates) {
    set_error("voxelize: candidate count changed between passes");
    return WFPG_ERR_ARG;
  }
  if (C >= (int64_t)UINT32_MAX) {
    set_error("voxelize: too many candidate voxels (%lld)", (long long)C);
    return WFPG_ERR_CAPACITY;
  }
  if (C == 0) {
    *n_fragments = 0;
    return WFPG_OK;
  }
  uint32_t* flags = ws.take<uint32_t>(C);
  uint32_t* pos = ws.take<uint32_t>(C);
  uint32_t* total = ws.take<uint32_t>(1);
  if (!ws.ok()) {
    set_error("voxelize: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  double h = side / resolution;
  int grid = (int)std::min<int64_t>(ceil_div(C, 256), (int64_t)kNumSMs * 16);
  k_vox_test<<<grid, 256, 0, st>>>(sc->v0, sc->v1, sc->v2, sc->n_tris, ranges, off, C, cube_lo[0],
                                   cube_lo[1], cube_lo[2], h, flags);
  WFPG_CHECK_LAUNCH("k_vox_test");
  WFPG_TRY(scan_u32(flags, pos, C, nullptr, total, ws, st));
  uint32_t th = 0;
  WFPG_CUDA(cudaMemcpyAsync(&th, total, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  *n_fragments = th;
  if ((int64_t)th > capacity) {
    set_error("voxelize: %u fragments exceed capacity %lld", th, (long long)capacity);
    return WFPG_ERR_CAPACITY;
  }
  k_vox_emit<<<grid, 256, 0, st>>>(ranges, off, sc->n_tris, C, flags, pos, out_coords, out_tris);
  WFPG_CHECK_LAUNCH("k_vox_emit");
  return WFPG_OK;
}

// ---------------------------------------------------------------------------
// octree structure
// ---------------------------------------------------------------------------
namespace wfpg {

// Levels from the sorted fragment codes in two streaming passes (svo.py:
// 416-500: np.unique per level, parents by searchsorted, children wired).
// A node of level l is a distinct value of code >> 3 (depth - l); sorted
// fragment i starts a new node at every level l >= lv(i), the coarsest
// level at which its code differs from fragment i-1's (from the highest
// differing bit; depth + 1 for a repeated code, 0 for i = 0).  So the node
// index of fragment i at level l is (#{j <= i : lv(j) <= l}) - 1: pass 1
// counts lv <= l per tile and level, a scan gives every tile's level
// offsets, and pass 2 recomputes the in-tile ranks (ballots) and writes
// every node once from the fragment that starts it — code, parent, first
// child and a bit in the parent's child mask.  Same arrays as the level-by-
// level build (levels in code order, root first).
constexpr int kLvBlock = 256;
constexpr int kLvWarps = kLvBlock / 32;
constexpr int kLvChunks = 16;                       // 32-fragment chunks per warp
constexpr int kLvTile = kLvBlock * kLvChunks;       // 4096 fragments per tile
constexpr int kLvMaxLevels = 22;                    // depth <= 21

struct BuildWs {
  uint64_t* codes;       // (F,) sorted fragment codes
  uint32_t* perm;        // (F,) stable sort permutation
  uint32_t* tile_cnt;    // (depth+1, tiles) level-major counts, then offsets
  uint32_t* counts;      // (depth+1,) level sizes
  uint32_t* leaf_start;  // (L+1,) first sorted fragment of each leaf
  double* sorted_n;      // (F,3) fragment normals in sorted-fragment order (phase B)
  int64_t tiles;
};

static void carve(Arena& a, int64_t F, int depth, BuildWs& w) {
  w.codes = a.take<uint64_t>(F);
  w.perm = a.take<uint32_t>(F);
  w.tiles = ceil_div(F > 0 ? F : 1, kLvTile);
  w.tile_cnt = a.take<uint32_t>((int64_t)(depth + 1) * w.tiles);
  w.counts = a.take<uint32_t>(depth + 2);
  w.leaf_start = a.take<uint32_t>(F + 1);
  w.sorted_n = a.take<double>(3 * F);
}

__global__ void k_frag_codes(const int32_t* __restrict__ coords, int64_t F,
                             uint64_t* __restrict__ codes, uint32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < F;
       i += (int64_t)gridDim.x * blockDim.x) {
    codes[i] = morton3((uint32_t)coords[3 * i], (uint32_t)coords[3 * i + 1],
                       (uint32_t)coords[3 * i + 2]);
    perm[i] = (uint32_t)i;
  }
}

// Morton codes straight from fp64 points (the compiled quantisation,
// _kernels.pyx:593-606, then morton3): no int32 coordinate array
__global__ void k_point_codes(const double* __restrict__ pts, int64_t n, double lox, double loy,
                              double loz, double scale, int32_t res, uint64_t* __restrict__ codes,
                              uint32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)quantise(pts[3 * i], lox, scale, res);
    const uint32_t y = (uint32_t)quantise(pts[3 * i + 1], loy, scale, res);
    const uint32_t z = (uint32_t)quantise(pts[3 * i + 2], loz, scale, res);
    codes[i] = morton3(x, y, z);
    perm[i] = (uint32_t)i;
  }
}

// coarsest level at which fragment i starts a node
__device__ __forceinline__ int start_level(const uint64_t* __restrict__ codes, int64_t i,
                                           int depth) {
  if (i == 0) return 0;
  const uint64_t x = codes[i] ^ codes[i - 1];
  if (x == 0) return depth + 1;
  const int hb = 63 - __clzll((long long)x);
  const int l = depth - hb / 3;
  return l < 1 ? 1 : l;
}

// pass 1: per tile and level, the number of fragments with lv <= level
__global__ void __launch_bounds__(kLvBlock) k_lv_count(const uint64_t* __restrict__ codes,
                                                       int64_t F, int depth, int64_t tiles,
                                                       uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t wc[kLvWarps][kLvMaxLevels];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kLvTile;
  uint32_t mine = 0;  // lane l: this warp's count for level l
  for (int c = 0; c < kLvChunks; ++c) {
    const int64_t i = t0 + ((int64_t)warp * kLvChunks + c) * 32 + lane;
    const int lv = i < F ? start_level(codes, i, depth) : depth + 1;
    for (int l = 0; l <= depth; ++l) {
      const uint32_t b = __ballot_sync(0xffffffffu, lv <= l);
      if (lane == l) mine += __popc(b);
    }
  }
  if (lane <= depth) wc[warp][lane] = mine;
  __syncthreads();
  if (threadIdx.x <= depth) {
    uint32_t s = 0;
    for (int w = 0; w < kLvWarps; ++w) s += wc[w][threadIdx.x];
    tile_cnt[(int64_t)threadIdx.x * tiles + blockIdx.x] = s;
  }
}

// one block per level: exclusive scan of the level's tile counts in place,
// level size to counts[level]
__global__ void __launch_bounds__(1024) k_lv_offsets(uint32_t* __restrict__ tile_cnt,
                                                     int64_t tiles,
                                                     uint32_t* __restrict__ counts) {
  __shared__ uint32_t sw[1024 / 32 + 1];
  uint32_t* c = tile_cnt + (int64_t)blockIdx.x * tiles;
  const int64_t per = (tiles + 1023) / 1024;
  const int64_t b0 = (int64_t)threadIdx.x * per, b1 = b0 + per < tiles ? b0 + per : tiles;
  uint32_t s = 0;
  for (int64_t b = b0; b < b1; ++b) s += c[b];
  uint32_t total;
  uint32_t run = block_exclusive_scan<1024>(s, sw, &total);
  for (int64_t b = b0; b < b1; ++b) {
    const uint32_t v = c[b];
    c[b] = run;
    run += v;
  }
  if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }

// pass 2: write every node from the fragment that starts it; each node sets
// its octant bit in its parent's child mask with a 32-bit atomicOr on the
// word holding the parent's byte (child_mask zeroed, 4-byte aligned, padded
// to whole words).
struct LevelOffs {
  int64_t off[kLvMaxLevels + 1];
};

__global__ void __launch_bounds__(kLvBlock) k_lv_emit(
    const uint64_t* __restrict__ codes, int64_t F, int depth, int64_t tiles,
    const uint32_t* __restrict__ tile_off, LevelOffs lo, uint64_t* __restrict__ ncodes,
    int32_t* __restrict__ parent, int32_t* __restrict__ child_base,
    uint8_t* __restrict__ child_mask, uint32_t* __restrict__ leaf_start) {
  __shared__ uint32_t wc[kLvWarps][kLvMaxLevels];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kLvTile;
  // warp counts per level, then each warp's exclusive offset within the tile
  uint32_t mine = 0;
  for (int c = 0; c < kLvChunks; ++c) {
    const int64_t i = t0 + ((int64_t)warp * kLvChunks + c) * 32 + lane;
    const int lv = i < F ? start_level(codes, i, depth) : depth + 1;
    for (int l = 0; l <= depth; ++l) {
      const uint32_t b = __ballot_sync(0xffffffffu, lv <= l);
      if (lane == l) mine += __popc(b);
    }
  }
  if (lane <= depth) wc[warp][lane] = mine;
  __syncthreads();
  // lane l: running count (fragments before this chunk with lv <= l), i.e.
  // tile offset + earlier warps of the tile
  uint32_t run = 0;
  if (lane <= depth) {
    run = tile_off[(int64_t)lane * tiles + blockIdx.x];
    for (int w = 0; w < warp; ++w) run += wc[w][lane];
  }
  const uint32_t le = lanemask_lt() | (1u << lane);
  for (int c = 0; c < kLvChunks; ++c) {
    const int64_t i = t0 + ((int64_t)warp * kLvChunks + c) * 32 + lane;
    const bool valid = i < F;
    const int lv = valid ? start_level(codes, i, depth) : depth + 1;
    const uint64_t code = valid ? codes[i] : 0;
    // inclusive rank of fragment i at level l: run_l + popc(ballot_l & le)
    uint32_t prev_rank = 0;  // rank at level l - 1
    for (int l = 0; l <= depth; ++l) {
      const uint32_t b = __ballot_sync(0xffffffffu, lv <= l);
      const uint32_t rank = __shfl_sync(0xffffffffu, run, l) + __popc(b & le);
      if (lane == l) run += __popc(b);
      if (valid && lv <= l) {
        const int64_t node = lo.off[l] + rank - 1;
        const uint64_t key = code >> (3 * (depth - l));
        ncodes[node] = key;
        parent[node] = l == 0 ? -1 : (int32_t)(lo.off[l - 1] + prev_rank - 1);
        if (l == depth) {
          child_base[node] = -1;
          leaf_start[rank - 1] = (uint32_t)i;
        }
        if (l > 0) {
          const int64_t p = lo.off[l - 1] + prev_rank - 1;
          atomicOr(reinterpret_cast<unsigned int*>(child_mask) + (p >> 2),
                   1u << (8 * (int)(p & 3) + (int)(key & 7u)));
          // a node's first child is started by the same fragment
          if (lv <= l - 1) child_base[p] = (int32_t)node;
        }
      }
      prev_rank = rank;
    }
  }
}

}  // namespace wfpg

extern "C" size_t wfpg_svo_build_workspace_bytes(int64_t n_fragments, int32_t depth) {
  Arena a(nullptr, 0);
  BuildWs w;
  carve(a, n_fragments, depth, w);
  return a.off + sort_ws_bytes(n_fragments) + 4096;
}

extern "C" int wfpg_svo_build_sorted(const void* workspace, int64_t n_fragments,
                                     const uint64_t** sorted_codes, const uint32_t** sort_perm) {
  Arena a(const_cast<void*>(workspace), SIZE_MAX);
  BuildWs w;
  carve(a, n_fragments, 1, w);
  *sorted_codes = w.codes;
  *sort_perm = w.perm;
  return WFPG_OK;
}

// codes (F,) in w.codes, identity in w.perm -> sorted codes, levels, level
// sizes (the one host read-back)
static int structure_from_codes(wfpg_svo* svo, int64_t F, BuildWs& w, Arena& a, cudaStream_t st) {
  const int depth = svo->depth;
  {
    size_t mark = a.off;
    WFPG_TRY(sort_pairs(w.codes, w.perm, F, nullptr, std::max(1, 3 * depth), a, st));
    a.off = mark;
  }
  k_lv_count<<<(unsigned)w.tiles, kLvBlock, 0, st>>>(w.codes, F, depth, w.tiles, w.tile_cnt);
  WFPG_CHECK_LAUNCH("k_lv_count");
  k_lv_offsets<<<depth + 1, 1024, 0, st>>>(w.tile_cnt, w.tiles, w.counts);
  WFPG_CHECK_LAUNCH("k_lv_offsets");
  std::vector<uint32_t> lvl_count(depth + 1);
  WFPG_CUDA(cudaMemcpyAsync(lvl_count.data(), w.counts, sizeof(uint32_t) * (depth + 1),
                            cudaMemcpyDeviceToHost, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  int64_t off = 0;
  for (int l = 0; l <= depth; ++l) {
    svo->level_off[l] = off;
    off += lvl_count[l];
  }
  svo->level_off[depth + 1] = off;
  svo->n_nodes = off;
  return WFPG_OK;
}

static int structure_args(const wfpg_svo* svo, int64_t n_fragments) {
  if (!svo || n_fragments <= 0) {
    set_error("cannot build an octree from an empty fragment list");
    return WFPG_ERR_ARG;
  }
  if (n_fragments >= (int64_t)INT32_MAX) {
    set_error("too many fragments");
    return WFPG_ERR_CAPACITY;
  }
  if (svo->depth < 0 || svo->depth >= kLvMaxLevels) {
    set_error("svo build: depth %d outside [0, %d]", svo->depth, kLvMaxLevels - 1);
    return WFPG_ERR_ARG;
  }
  return WFPG_OK;
}

extern "C" int wfpg_svo_build_structure(wfpg_svo* svo, const int32_t* frag_coords,
                                        int64_t n_fragments, void* workspace, size_t ws_bytes,
                                        void* stream) {
  NvtxRange nvtx_("wfpg_svo_build_structure");
  WFPG_TRY(structure_args(svo, n_fragments));
  cudaStream_t st = as_stream(stream);
  Arena a(workspace, ws_bytes);
  BuildWs w;
  carve(a, n_fragments, svo->depth, w);
  if (!a.ok()) {
    set_error("svo build: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  const int64_t F = n_fragments;
  const int grid = (int)std::min<int64_t>(ceil_div(F, 256), (int64_t)kNumSMs * 8);
  k_frag_codes<<<grid, 256, 0, st>>>(frag_coords, F, w.codes, w.perm);
  WFPG_CHECK_LAUNCH("k_frag_codes");
  return structure_from_codes(svo, F, w, a, st);
}

extern "C" int wfpg_svo_build_structure_points(wfpg_svo* svo, const double* points, int64_t n,
                                               void* workspace, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("wfpg_svo_build_structure_points");
  WFPG_TRY(structure_args(svo, n));
  if (!points || svo->resolution != (1 << svo->depth) || !(svo->size > 0.0)) {
    set_error("wfpg_svo_build_structure_points: bad arguments");
    return WFPG_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  Arena a(workspace, ws_bytes);
  BuildWs w;
  carve(a, n, svo->depth, w);
  if (!a.ok()) {
    set_error("svo build: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  const double scale = (double)svo->resolution / svo->size;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8);
  k_point_codes<<<grid, 256, 0, st>>>(points, n, svo->lo[0], svo->lo[1], svo->lo[2], scale,
                                      svo->resolution, w.codes, w.perm);
  WFPG_CHECK_LAUNCH("k_point_codes");
  return structure_from_codes(svo, n, w, a, st);
}

namespace wfpg {

// ---------------------------------------------------------------------------
// dual-normal k-means, svo.py:139-173, exact op order
// ---------------------------------------------------------------------------
struct LeafNormals {  // fragment normals of one leaf, sorted-fragment order
  const double* sorted_n;  // gathered once by k_gather_normals: the k-means
  int64_t start;           // passes re-read a leaf's rows from L1, not HBM
  __device__ __forceinline__ void get(int i, double* n) const {
    const double* p = sorted_n + 3 * (start + i);
    n[0] = p[0];
    n[1] = p[1];
    n[2] = p[2];
  }
};

// sorted_n[i] = normal of sorted fragment i: tri_n[frag_tris[perm[i]]], or
// tri_n[perm[i]] for per-fragment normals (frag_tris NULL: surface points).
// One random gather per fragment instead of one per k-means read.
__global__ void k_gather_normals(const uint32_t* __restrict__ perm,
                                 const int32_t* __restrict__ frag_tris,
                                 const double* __restrict__ tri_n, int64_t F,
                                 double* __restrict__ sorted_n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < F;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = perm[i];
    const int64_t t = frag_tris ? (int64_t)frag_tris[f] : f;
    const double* q = tri_n + 3 * t;
    const double x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
    double* o = sorted_n + 3 * i;
    o[0] = x;
    o[1] = y;
    o[2] = z;
  }
}

struct KidNormals {  // [kid_n; -kid_n]
  const double* normal;
  int64_t base;
  int cnt;
  __device__ __forceinline__ void get(int i, double* n) const {
    int k = i < cnt ? i : i - cnt;
    const double* p = normal + 3 * (base + k);
    if (i < cnt) {
      n[0] = p[0];
      n[1] = p[1];
      n[2] = p[2];
    } else {
      n[0] = -p[0];
      n[1] = -p[1];
      n[2] = -p[2];
    }
  }
};

template <class Src>
__device__ __forceinline__ bool kmeans_side(const Src& s, int i, const double* ma,
                                            const double* mb) {
  double n[3];
  s.get(i, n);
  double da = dot_gemv(n[0], n[1], n[2], ma[0], ma[1], ma[2]);
  double db = dot_gemv(n[0], n[1], n[2], mb[0], mb[1], mb[2]);
  return da >= db;  // ties toward side a
}

template <class Src>
__device__ void cluster_normals(const Src& s, int K, uint64_t key, double* out) {
  // pick = min(int(rng.next() * K), K - 1)  (svo.py:152)
  double u = u01(key, 0);
  long long pk = (long long)__dmul_rn(u, (double)K);
  int pick = (int)(pk < K - 1 ? pk : K - 1);
  double ma[3], mb[3], pa[3], pb[3];
  s.get(pick, ma);
  mb[0] = -ma[0];
  mb[1] = -ma[1];
  mb[2] = -ma[2];
  bool have_prev = false;
  for (int it = 0; it < 32; ++it) {
    if (have_prev) {
      bool same = true;
      for (int i = 0; i < K && same; ++i)
        same = kmeans_side(s, i, ma, mb) == kmeans_side(s, i, pa, pb);
      if (same) break;
    }
    double sa[3] = {0.0, 0.0, 0.0}, sb[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < K; ++i) {
      double n[3];
      s.get(i, n);
      bool side = dot_gemv(n[0], n[1], n[2], ma[0], ma[1], ma[2]) >=
                  dot_gemv(n[0], n[1], n[2], mb[0], mb[1], mb[2]);
      double* acc = side ? sa : sb;
      acc[0] = __dadd_rn(acc[0], n[0]);
      acc[1] = __dadd_rn(acc[1], n[1]);
      acc[2] = __dadd_rn(acc[2], n[2]);
    }
    for (int k = 0; k < 3; ++k) {
      pa[k] = ma[k];
      pb[k] = mb[k];
    }
    have_prev = true;
    double na = __dsqrt_rn(dot_ddot(sa[0], sa[1], sa[2], sa[0], sa[1], sa[2]));
    double nb = __dsqrt_rn(dot_ddot(sb[0], sb[1], sb[2], sb[0], sb[1], sb[2]));
    if (na > 1e-12)
      for (int k = 0; k < 3; ++k) ma[k] = __ddiv_rn(sa[k], na);
    if (nb > 1e-12) {
      for (int k = 0; k < 3; ++k) mb[k] = __ddiv_rn(sb[k], nb);
    } else {
      for (int k = 0; k < 3; ++k) mb[k] = -ma[k];
    }
  }
  out[0] = ma[0];
  out[1] = ma[1];
  out[2] = ma[2];
}

__global__ void k_leaf_normals(const uint64_t* __restrict__ codes, int64_t leaf_off, int64_t L,
                               const uint32_t* __restrict__ leaf_start,
                               const double* __restrict__ sorted_n, uint64_t seed,
                               double* __restrict__ normal) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x) {
    LeafNormals s{sorted_n, (int64_t)leaf_start[i]};
    int K = (int)(leaf_start[i + 1] - leaf_start[i]);
    double n0[3];
    s.get(0, n0);
    bool same = true;
    for (int j = 1; j < K && same; ++j) {
      double nj[3];
      s.get(j, nj);
      same = nj[0] == n0[0] && nj[1] == n0[1] && nj[2] == n0[2];
    }
    double out[3] = {n0[0], n0[1], n0[2]};
    if (!same) {
      uint64_t code = codes[leaf_off + i];
      cluster_normals(s, K, stream_key(seed, code * 4 + 2), out);
    }
    double* o = normal + 3 * (leaf_off + i);
    o[0] = out[0];
    o[1] = out[1];
    o[2] = out[2];
  }
}

__global__ void k_internal_normals(const uint64_t* __restrict__ codes, int64_t off, int64_t n,
                                   int level, const int32_t* __restrict__ child_base,
                                   const uint8_t* __restrict__ child_mask, uint64_t seed,
                                   double* __restrict__ normal) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t node = off + k;
    int64_t base = child_base[node];
    const int cnt = __popc((uint32_t)child_mask[node]);
    const double* kid = normal + 3 * base;
    double a0 = fabs(kid[0]), a1 = fabs(kid[1]), a2 = fabs(kid[2]);
    bool same = true;
    for (int j = 1; j < cnt && same; ++j)
      same = fabs(kid[3 * j]) == a0 && fabs(kid[3 * j + 1]) == a1 && fabs(kid[3 * j + 2]) == a2;
    double out[3] = {kid[0], kid[1], kid[2]};
    if (!same) {
      KidNormals s{normal, base, cnt};
      uint64_t stream = codes[node] * 4 + 3 + ((uint64_t)level << 48);
      cluster_normals(s, 2 * cnt, stream_key(seed, stream), out);
    }
    double* o = normal + 3 * node;
    o[0] = out[0];
    o[1] = out[1];
    o[2] = out[2];
  }
}

__global__ void k_node_desc(const int32_t* __restrict__ child_base,
                            const uint8_t* __restrict__ child_mask, int64_t n,
                            uint2* __restrict__ desc) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    desc[k] = make_uint2((uint32_t)child_base[k], (uint32_t)child_mask[k]);
}

__global__ void k_top_index(const uint2* __restrict__ desc, int32_t depth, int32_t T,
                            uint2* __restrict__ top) {
  const int64_t cells = (int64_t)1 << (3 * T);
  const uint32_t m = (1u << T) - 1u;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int sh = depth - T;
    const int32_t x = (int32_t)((c >> (2 * T)) & m) << sh;
    const int32_t y = (int32_t)((c >> T) & m) << sh;
    const int32_t z = (int32_t)(c & m) << sh;
    bool pres;
    int32_t lvl;
    int32_t node = descend_coords(desc, depth, x, y, z, T, &pres, &lvl);
    top[c] = make_uint2((uint32_t)node, (uint32_t)lvl | (pres ? 0x80000000u : 0u));
  }
}

int build_top_index(wfpg_svo* svo, cudaStream_t st) {
  const int T = svo->top_level;
  if (!svo->top_index || T <= 0) return WFPG_OK;
  if (T > svo->depth || T > 7) {
    set_error("top index level %d outside [1, min(depth, 7)]", T);
    return WFPG_ERR_ARG;
  }
  const int64_t cells = (int64_t)1 << (3 * T);
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cells, 256), (int64_t)kNumSMs * 8));
  k_top_index<<<grid, 256, 0, st>>>(reinterpret_cast<const uint2*>(svo->node_desc), svo->depth, T,
                                     reinterpret_cast<uint2*>(svo->top_index));
  WFPG_CHECK_LAUNCH("k_top_index");
  return WFPG_OK;
}

}  // namespace wfpg

extern "C" size_t wfpg_svo_top_index_bytes(int32_t top_level) {
  return top_level > 0 && top_level <= 7 ? (size_t)8 << (3 * top_level) : 0;
}

extern "C" int wfpg_svo_build_top_index(wfpg_svo* svo, void* stream) {
  if (!svo || !svo->node_desc || !svo->top_index || svo->top_level <= 0) {
    set_error("wfpg_svo_build_top_index: bad arguments");
    return WFPG_ERR_ARG;
  }
  return build_top_index(svo, (cudaStream_t)stream);
}

extern "C" int wfpg_svo_build_fill(wfpg_svo* svo, const int32_t* frag_tris,
                                   const double* tri_normals, int64_t n_fragments, uint64_t seed,
                                   void* workspace, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("wfpg_svo_build_fill");
  if (!svo || !svo->codes || !svo->parent || !svo->child_base || !svo->child_mask ||
      !svo->normal || !svo->node_desc) {
    set_error("svo build fill: missing node arrays");
    return WFPG_ERR_ARG;
  }
  const int depth = svo->depth;
  cudaStream_t st = as_stream(stream);
  Arena a(workspace, ws_bytes);
  BuildWs w;
  carve(a, n_fragments, depth, w);
  if (!a.ok()) {
    set_error("svo build: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  const int64_t n = svo->n_nodes;
  auto grid_for = [](int64_t m) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), (int64_t)kNumSMs * 8));
  };
  std::vector<int64_t> cnt(depth + 1);
  for (int l = 0; l <= depth; ++l) cnt[l] = svo->level_off[l + 1] - svo->level_off[l];
  LevelOffs lo;
  for (int l = 0; l <= depth + 1 && l <= kLvMaxLevels; ++l) lo.off[l] = svo->level_off[l];
  // structure: every node written once by the fragment that starts it
  WFPG_CUDA(cudaMemsetAsync(svo->child_mask, 0, (size_t)((n + 3) & ~(int64_t)3), st));
  k_lv_emit<<<(unsigned)w.tiles, kLvBlock, 0, st>>>(w.codes, n_fragments, depth, w.tiles,
                                                    w.tile_cnt, lo, svo->codes, svo->parent,
                                                    svo->child_base, svo->child_mask,
                                                    w.leaf_start);
  WFPG_CHECK_LAUNCH("k_lv_emit");
  k_set_u32<<<1, 1, 0, st>>>(w.leaf_start + cnt[depth], (uint32_t)n_fragments);
  WFPG_CHECK_LAUNCH("k_set_u32");
  // zeroed accumulators / means / counters (svo.py:448-455): 116 B per node,
  // written on a side stream while the normals are fitted (the gather and
  // k-means are latency-bound), joined before returning
  static cudaStream_t side = nullptr;
  static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (!side) {
    WFPG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    WFPG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    WFPG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }
  WFPG_CUDA(cudaEventRecord(ev_fork, st));
  WFPG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
  if (svo->sum_a) WFPG_CUDA(cudaMemsetAsync(svo->sum_a, 0, 24 * n, side));
  if (svo->sum_b) WFPG_CUDA(cudaMemsetAsync(svo->sum_b, 0, 24 * n, side));
  if (svo->weight_a) WFPG_CUDA(cudaMemsetAsync(svo->weight_a, 0, 8 * n, side));
  if (svo->weight_b) WFPG_CUDA(cudaMemsetAsync(svo->weight_b, 0, 8 * n, side));
  if (svo->mean_a) WFPG_CUDA(cudaMemsetAsync(svo->mean_a, 0, 24 * n, side));
  if (svo->mean_b) WFPG_CUDA(cudaMemsetAsync(svo->mean_b, 0, 24 * n, side));
  if (svo->counter) WFPG_CUDA(cudaMemsetAsync(svo->counter, 0, 4 * n, side));
  WFPG_CUDA(cudaEventRecord(ev_join, side));
  // normals: leaves, then internal levels bottom-up
  int64_t L = cnt[depth];
  k_gather_normals<<<grid_for(n_fragments), 256, 0, st>>>(w.perm, frag_tris, tri_normals,
                                                          n_fragments, w.sorted_n);
  WFPG_CHECK_LAUNCH("k_gather_normals");
  k_leaf_normals<<<grid_for(L), 128, 0, st>>>(svo->codes, svo->level_off[depth], L, w.leaf_start,
                                              w.sorted_n, seed, svo->normal);
  WFPG_CHECK_LAUNCH("k_leaf_normals");
  for (int l = depth - 1; l >= 0; --l) {
    k_internal_normals<<<grid_for(cnt[l]), 128, 0, st>>>(svo->codes, svo->level_off[l], cnt[l], l,
                                                         svo->child_base, svo->child_mask, seed,
                                                         svo->normal);
    WFPG_CHECK_LAUNCH("k_internal_normals");
  }
  k_node_desc<<<grid_for(n), 256, 0, st>>>(svo->child_base, svo->child_mask, n,
                                           reinterpret_cast<uint2*>(svo->node_desc));
  WFPG_CHECK_LAUNCH("k_node_desc");
  WFPG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  return build_top_index(svo, st);
}

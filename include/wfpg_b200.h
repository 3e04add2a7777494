/*
 * wfpg_b200.h — C ABI of the B200-native guided wavefront render path.
 *
 * Drop-in boundary for the reference package `wfpg` (arXiv 2405.06997 CPU
 * reference, /root/reference/pkg).  The reference crosses Python -> native
 * code at the Cython `def *_kernel` functions of src/wfpg/_kernels.pyx and
 * at the numpy-level SVO / guiding / wavefront functions; every entry point
 * below names the reference interface it replaces (file:line, paths relative
 * to /root/reference/pkg/src/wfpg/).
 *
 * Conventions
 *  - Plain C types only.  Every pointer inside a struct or argument is a
 *    DEVICE pointer unless the field comment says "host".
 *  - The caller owns every buffer.  Functions never allocate device memory;
 *    entry points that need scratch take a caller-provided workspace whose
 *    size is returned by the matching *_workspace_bytes() query.
 *  - All work is enqueued on `stream` (a cudaStream_t passed as void*).
 *    Functions that must report a device-side count to the host say so.
 *  - Return value: WFPG_OK (0) or a WFPG_ERR_* code; wfpg_last_error()
 *    returns a human-readable message for the last failure on this thread.
 *  - Index width: triangle ids, node ids and path ids are int32 on the
 *    device (the reference uses int64; the Python layer widens on export).
 *  - Floating point: fp64 throughout, like the reference.
 */
#ifndef WFPG_B200_H
#define WFPG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WFPG_ABI_VERSION 1

enum wfpg_status {
  WFPG_OK = 0,
  WFPG_ERR_ARG = 1,        /* invalid argument (reference: ValueError) */
  WFPG_ERR_CUDA = 2,       /* CUDA runtime error */
  WFPG_ERR_WORKSPACE = 3,  /* workspace too small */
  WFPG_ERR_CAPACITY = 4    /* a device-side count exceeded the caller's capacity */
};

/* ------------------------------------------------------------------------ */
/* Data contracts                                                            */
/* ------------------------------------------------------------------------ */

/* Scene arrays: scene.py:85-131 (Scene.__init__) + bvh.py:33-119 (Bvh). */
typedef struct wfpg_scene {
  int32_t n_tris;
  const double* v0;          /* (T,3) */
  const double* v1;          /* (T,3) original vertices (voxelize uses them, svo.py:110) */
  const double* v2;          /* (T,3) */
  const double* e1;          /* (T,3) v1 - v0 */
  const double* e2;          /* (T,3) v2 - v0 */
  const double* normals;     /* (T,3) unit geometric normals, bit-exact host copy */
  const int32_t* tri_mat;    /* (T,)  material id */
  const int32_t* mat_kind;   /* (M,)  0 lambert, 1 mirror, 2 emitter (scene.py:18) */
  const double* mat_rgb;     /* (M,3) */
  int32_t n_mats;
  int32_t n_emit;
  const double* emitter_cdf; /* (E,) area CDF */
  const int32_t* emitter_tris; /* (E,) */
  double emitter_area;
  double ray_eps;            /* 1e-4 * scene diagonal (scene.py:22,108) */
  double bbox_lo[3];         /* host values */
  double bbox_hi[3];
  int32_t bvh_nodes;
  const double* bvh_lo;      /* (N,3) */
  const double* bvh_hi;      /* (N,3) */
  const int32_t* bvh_left;   /* (N,) */
  const int32_t* bvh_right;  /* (N,) */
  const int32_t* bvh_count;  /* (N,) 0 = inner node */
  const int32_t* bvh_order;  /* (T,) */
  int32_t brute;             /* 1 when T <= 512: nearest-hit queries use the brute
                                force path (_kernelshim.py:13-21) */
  /* Optional (N,8) float BVH node boxes {lo.xyz, 0, hi.xyz, 0} widened by
   * 1e-5 of the scene diagonal + 4e-7 of the coordinate and rounded outward:
   * the traversals then run their slab tests in fp32 (triangle tests stay
   * fp64; the padding dwarfs every fp32 rounding, so no hit is culled).
   * NULL: fp64 boxes. */
  const float* bvh_box_f32;
} wfpg_scene;

/* Pinhole camera: scene.py:29-61 (Camera). Host values. */
typedef struct wfpg_camera {
  double position[3];
  double forward[3];
  double right[3];
  double up[3];              /* Camera.up_ortho */
  double tan_half;
  int32_t width;
  int32_t height;
} wfpg_camera;

/* Sparse voxel octree: svo.py:176-224 (SvoCache).  Level-grouped flat node
 * arrays, level 0 = root, node id = flat index. */
typedef struct wfpg_svo {
  int32_t depth;
  int32_t resolution;
  int64_t n_nodes;
  double lo[3];              /* host: cube_lo */
  double size;               /* host: cube_size */
  int64_t level_off[32];     /* host: depth+2 entries used */
  uint64_t* codes;           /* (n,) morton code at the node's level */
  int32_t* child_base;       /* (n,) first child, -1 for leaves */
  uint8_t* child_mask;       /* (n,); wfpg_svo_build_fill needs it 4-byte aligned
                                and padded to whole 32-bit words (word atomics) */
  int32_t* parent;           /* (n,) -1 for the root */
  uint32_t* node_desc;       /* (n,2) packed {child_base, child_mask} for descents */
  double* normal;            /* (n,3) normal_a (normal_b = -normal_a) */
  double* sum_a;             /* (n,3) */
  double* sum_b;             /* (n,3) */
  double* weight_a;          /* (n,)  */
  double* weight_b;          /* (n,)  */
  double* mean_a;            /* (n,3) */
  double* mean_b;            /* (n,3) */
  int32_t* counter;          /* (n,)  Alg. 2 ray counters, zero between calls */
  /* Optional dense index of the top `top_level` levels: 8^top_level entries
   * of 2 uint32 {node, reached level | present << 31}, indexed by the cell's
   * row-major coordinates at that level.  Built by wfpg_svo_build_top_index
   * (wfpg_svo_build_fill builds it too when set); every descent then starts
   * at level top_level with one load instead of top_level dependent ones.
   * NULL / top_level 0: plain root-to-leaf descents.  Same results either way. */
  uint32_t* top_index;
  int32_t top_level;
} wfpg_svo;

/* Wavefront path state: wavefront.py:53-71 (PathState), SoA. */
typedef struct wfpg_paths {
  int64_t n;
  int32_t max_depth;         /* rec arrays have max_depth+1 slots per path */
  double* ray_o;             /* (P,3) */
  double* ray_d;             /* (P,3) */
  double* beta;              /* (P,3) */
  double* radiance;          /* (P,3) */
  uint64_t* key;             /* (P,) */
  uint64_t* ctr;             /* (P,) */
  uint8_t* alive;            /* (P,) */
  double* prev_pdf;          /* (P,) */
  double* rec_pos;           /* (P,D+1,3), or (D+1,P,3): rec_depth_major */
  double* rec_T;             /* (P,D+1,3), or (D+1,P,3): rec_depth_major */
  double* emit_le;           /* (P,3) */
  int32_t* emit_depth;       /* (P,) */
  /* Optional (P,) deepest record slot written (0 = camera only).  When set,
   * the pass does not zero rec_pos / rec_T (2 x 24 (D+1) bytes per path):
   * slots above n_rec hold stale values, which readers mask (the exitance
   * update only reads slots <= emit_depth <= n_rec).  NULL: zeroed slots. */
  uint8_t* n_rec;
  /* Record layout: 0 = (P, D+1, 3), the reference's PathState layout;
   * 1 = (D+1, P, 3) depth-major — one depth's records of consecutive paths
   * are contiguous, so the shade kernel's record stores fill whole sectors
   * (the package's own PathState uses it). */
  int32_t rec_depth_major;
} wfpg_paths;

/* Per-depth guide tables: guiding.py:254-309 (GuideTables).  The B200 layout
 * keeps the floored field values plus their row sums, marginal CDF and
 * totals; conditional CDFs, pdf tables and product block CDFs are evaluated
 * on the fly by the samplers with the same arithmetic as fill_batch. */
typedef struct wfpg_guide {
  int32_t mode;              /* 0 off, 1 plain, 2 product */
  int32_t n;                 /* field resolution */
  int32_t capacity;          /* bin slots allocated */
  double eps;                /* guiding.EPSILON_FLOOR */
  double* vals;              /* (B,n,n) */
  double* row_sum;           /* (B,n)   values.sum(axis=2) */
  double* marg;              /* (B,n)   cumsum(row_sums)/totals */
  double* total;             /* (B,)    */
  double* block_sums;        /* (B,8,8) product mode (else may be NULL) */
  const int32_t* n_bins;     /* device count of valid slots */
  const double* upper_dirs;  /* (8,8,3) product-layer cell centres (guiding.UPPER_DIRS) */
  double* cum;               /* optional (B,n,n) unnormalised row prefix sums
                                (np.cumsum order); lets the plain sampler invert the
                                conditional CDF with a binary search */
  double* block_rows;        /* optional (B,8,8,n/8) product mode: row sums of every
                                block row (guiding.py:304 `rows`); the product sampler's
                                block marginal then reads them instead of re-summing */
} wfpg_guide;

/* Knobs of one render pass: wavefront.py:21-50 (GuidingConfig). */
typedef struct wfpg_pass_config {
  int32_t l_min;
  int32_t c_ray;
  int32_t field_res;
  int32_t guided_depths;
  int32_t max_depth;
  int32_t product;
  int32_t jitter;
  double blur_sigma;
  double epsilon;
  int32_t russian_roulette;
  int32_t rr_depth;
  uint64_t seed;
  int64_t sample_index;      /* first sample index of the pass */
  int32_t n_samples;         /* samples per pixel in this pass */
  int32_t deterministic;     /* 1: exitance splat in path order (np.add.at) */
  int32_t blur_radius;       /* core._blur_kernel radius (0: no blur) */
  double blur_w[33];         /* normalised blur taps, computed by numpy on the host */
  const double* upper_dirs;  /* device (8,8,3) guiding.UPPER_DIRS, product mode only */
  /* Image tiling (multi-GPU): this pass renders pixels [pixel_offset,
   * pixel_offset + n_pixels) of the camera image; RNG streams use the global
   * pixel index, so every path draws what it would draw on one GPU.
   * n_pixels = 0 renders the whole image. */
  int64_t pixel_offset;
  int64_t n_pixels;
  /* When non-NULL the Eq. 5 deposits of this pass go to this zeroed leaf
   * buffer (8 doubles per leaf: sum_a[3], sum_b[3], weight_a, weight_b as
   * four planes) instead of the SVO, and the bottom-up refresh is skipped;
   * the caller all-reduces it and applies it with wfpg_svo_apply_leaf_acc. */
  double* leaf_acc;
  /* 1: replay the pass as a CUDA graph.  The first call with a given
   * (workspace, configuration, buffers) runs eagerly, the second captures,
   * later calls replay; only sample_index may change between them. */
  int32_t use_graph;
  /* Optional (n_pixels,) int32 device buffer: the depth-1 bin node of every
   * pixel, -1 where its depth-1 vertex is not binned (collect_bin_image,
   * wavefront.py:221,254-256).  With several samples per pass the bin with
   * the largest node id wins, as the reference's in-order assignment over
   * node-sorted bins does. */
  int32_t* bin_image;
  /* Optional deposit export for multi-GPU runs (the sparse
   * alternative to a per-leaf all-reduce).  When dep_leaf is non-NULL the
   * pass writes its Eq. 5 deposits (leaf id or -1, unit direction, radiance)
   * in path-major / vertex-ascending order into these device buffers, the
   * count into *dep_count, and leaves the SVO untouched; dep_capacity must be
   * >= n_pixels * n_samples * max_depth.  Concatenating the ranks' lists in
   * band order gives the global path order, so splatting the concatenation
   * deterministically (wfpg_svo_accumulate) and refreshing
   * (wfpg_svo_refresh_leaves) reproduces a 1-GPU update of the same paths
   * bit for bit.  Takes precedence over leaf_acc. */
  int32_t* dep_leaf;
  double* dep_dir;
  double* dep_rad;
  int32_t* dep_count;
  int64_t dep_capacity;
  /* Optional multi-GPU communicator (wfpg_comm_init_*).  With
   * comm set (n_samples must be 1; pixel_offset / n_pixels give this rank's
   * band, band r = [r*n_img/W, (r+1)*n_img/W)) the pass is the 1-GPU pass of
   * the whole image restricted to this band, path for path:
   *  - guided depths bin GLOBALLY (Alg. 2 over every rank's lambert hits): the
   *    per-path start nodes are all-gathered, every rank runs the same
   *    partition, the bin origins (the k-th member in global path order) are
   *    contributed by the rank that owns that path (one all-reduce of bit
   *    patterns), and each rank generates the fields only of the bins its own
   *    paths belong to;
   *  - the Eq. 5 deposits of all ranks are all-gathered (fixed wire capacity
   *    per rank, dep_wire_capacity records; 0 = n_pixels / 4) and splatted in
   *    global path order, so every rank's SVO equals the 1-GPU SVO bit for
   *    bit.  A rank that exports more deposits than the wire holds makes
   *    every rank skip the in-pass splat; the exact variable-size exchange of
   *    that pass then runs before the next pass on this communicator (or in
   *    wfpg_comm_settle).
   * NCCL communicators are captured into the pass's CUDA graph; host-exchange
   * communicators run the pass eagerly.  Non-guided depths bin locally
   * (their bins only feed PassStats). */
  struct wfpg_comm* comm;
  int64_t dep_wire_capacity;
  /* Optional (n_samples,) int64 device array: the sample index of each
   * sample slot of the pass (any list, wavefront.py:207-215: path stream
   * (sample_list[s] * n_img + pixel) * 4).  NULL: sample_index + s.  The
   * bins' streams use sample_index, the list's first entry, as the
   * reference does (samples[0], wavefront.py:264). */
  const int64_t* sample_list;
  /* Multi-GPU bin ownership, per depth (index = depth, 0 unused): an upper
   * estimate of that depth's global bin count (e.g. 1.05x the previous
   * pass's), or 0.  With an estimate E > 0 and comm set, rank r generates
   * the fields of the bins [r*S, (r+1)*S), S = ceil(E / W), and the floored
   * values of all bins are all-gathered (S * n * n doubles per rank); every
   * rank then derives the other bins' tables from those values (bitwise the
   * owners' tables).  When the depth's actual bin count exceeds W * S, every
   * rank falls back to generating the bins its own paths use (exact either
   * way).  0: that fallback policy always (right for depth 1, whose bins
   * split with the image). */
  int32_t own_bins[32];
  /* Inter-pass overlap on one GPU (optional cudaEvent_t handles, NULL = none;
   * ignored with comm): passes on different streams may overlap where they
   * touch disjoint state.  The pass waits for ev_wait_counters before its
   * first Alg. 2 partition (the SVO's ray counters are shared) and for
   * ev_wait_svo before it first reads or writes the SVO exitance (fields or
   * the exitance update); it records ev_rec_counters after its last
   * partition and ev_rec_svo after its exitance update.  Chaining pass i+1's
   * waits on pass i's records keeps the reference's pass order for every
   * SVO access (wavefront.FramePipeline), while pass i+1's ray generation,
   * intersection and first binning overlap pass i's last depth and update.
   * Captured graphs contain them as external event nodes. */
  void* ev_wait_counters;
  void* ev_wait_svo;
  void* ev_rec_counters;
  void* ev_rec_svo;
  /* 1: bin only the guided depths (and depth 1 for bin_image).  The
   * reference bins every depth (wavefront.py:240-256), but the bins of
   * non-guided depths only feed PassStats (bins / rays / material groups of
   * those depths then read 0); frames and the SVO are identical either way.
   * 0 (default): the reference's behaviour. */
  int32_t skip_unguided_bins;
} wfpg_pass_config;

/* Per-pass statistics returned to the host: wavefront.py:81-85 (PassStats). */
typedef struct wfpg_pass_stats {
  int32_t depths_run;
  int32_t bins_per_depth[32];
  int32_t rays_per_depth[32];
  int32_t live_per_depth[32];
  int32_t deposits;
  int32_t mat_groups[32][64]; /* per depth, per material id (first 64 ids): paths of the
                                  depth's live queue that hit a triangle of that material
                                  (partition_material, wavefront.py:88-95,250-253) */
} wfpg_pass_stats;

/* ------------------------------------------------------------------------ */
/* Library                                                                   */
/* ------------------------------------------------------------------------ */

int wfpg_abi_version(void);
/* Struct layout of this build, for binding checks (ctypes / cgo mirrors):
 * struct_id 0 scene, 1 camera, 2 svo, 3 paths, 4 guide, 5 pass_config,
 * 6 pass_stats.  sizeof, or the byte offset of the named field; -1 when
 * unknown. */
int64_t wfpg_abi_sizeof(int32_t struct_id);
int64_t wfpg_abi_offsetof(int32_t struct_id, const char* field);

/* ------------------------------------------------------------------------ */
/* Multi-GPU communicator: the exchange steps of a banded     */
/* render pass (wfpg_pass_config.comm).                                      */
/* ------------------------------------------------------------------------ */

typedef struct wfpg_comm wfpg_comm;
/* A cudaEvent_t (timing disabled) for wfpg_pass_config's overlap events. */
int wfpg_event_create(void** event);
int wfpg_event_destroy(void* event);
/* cudaMemcpyAsync(cudaMemcpyDefault) on `stream` + synchronise: lets a host
 * exchange callback stage device buffers without a CUDA binding of its own. */
int wfpg_memcpy(void* dst, const void* src, size_t bytes, void* stream);
/* Host exchange callback: perform the collective `op` (0 all-gather: recv =
 * every rank's `count` elements in rank order; 1 all-reduce sum) on DEVICE
 * buffers of `dtype` (0 int32, 1 uint64, 2 float64); the stream has been
 * synchronised.  Return 0 on success. */
typedef int32_t (*wfpg_exchange_fn)(void* user, int32_t op, const void* send, void* recv,
                                    int64_t count, int32_t dtype, void* stream);
/* 1 when libnccl.so.2 can be loaded (dlopen; the process's NCCL is reused). */
int wfpg_comm_nccl_available(void);
/* 128-byte ncclUniqueId (rank 0), to be broadcast to every rank. */
int wfpg_comm_nccl_unique_id(uint8_t* out128);
/* NCCL communicator on the current device (collective over all ranks). */
int wfpg_comm_init_nccl(int32_t world, int32_t rank, const uint8_t* unique_id, wfpg_comm** out);
/* Host-exchange communicator (tests, gloo runs). */
int wfpg_comm_init_host(int32_t world, int32_t rank, wfpg_exchange_fn fn, void* user,
                        wfpg_comm** out);
/* Complete the deposit exchange of the last pass on this communicator
 * (synchronises with it; runs the exact exchange if the wire overflowed). */
int wfpg_comm_settle(wfpg_comm* comm);
int wfpg_comm_destroy(wfpg_comm* comm);
const char* wfpg_last_error(void);
/* Number of kernel launches issued by this library since load (process-wide). */
uint64_t wfpg_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Device primitives (scan, stable radix sort)                               */
/* ------------------------------------------------------------------------ */

size_t wfpg_scan_workspace_bytes(int64_t n);
/* Exclusive prefix sum of n uint32 values; writes the total to *total (device). */
int wfpg_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                  void* workspace, size_t ws_bytes, void* stream);

size_t wfpg_sort_workspace_bytes(int64_t n);
/* Stable LSD radix sort of (key, value) pairs on the low `key_bits` bits.
 * n_dev (optional, device int32) overrides n with a device-side count <= n. */
int wfpg_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, const int32_t* n_dev,
                        int32_t key_bits, void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Item 1 — SVO builder                                                      */
/* ------------------------------------------------------------------------ */

/* svo.py:94-136 (voxelize).  Pass 1: candidate counts -> upper bound of the
 * fragment count (host, synchronous). */
size_t wfpg_voxelize_workspace_bytes(int32_t n_tris, int64_t n_candidates);
/* Pass 1: number of candidate voxels (sum of triangle bbox voxel ranges),
 * host value, synchronous.  Workspace: wfpg_voxelize_workspace_bytes(T, 0). */
int wfpg_voxelize_count(const wfpg_scene* scene, const double* cube_lo, double side,
                        int32_t resolution, int64_t* n_candidates,
                        void* workspace, size_t ws_bytes, void* stream);
/* Pass 2: SAT-test every candidate and emit fragments in (tri, x, y, z)
 * order: coords (F,3) int32, tris (F,) int32.  *n_fragments (host) is set
 * even when capacity is too small (then WFPG_ERR_CAPACITY and nothing is
 * written).  Workspace: wfpg_voxelize_workspace_bytes(T, n_candidates). */
int wfpg_voxelize_emit(const wfpg_scene* scene, const double* cube_lo, double side,
                       int32_t resolution, int64_t n_candidates, int32_t* out_coords,
                       int32_t* out_tris, int64_t capacity, int64_t* n_fragments,
                       void* workspace, size_t ws_bytes, void* stream);

/* svo.py:416-500 (build_octree).  Phase A sorts/uniques fragments and sizes
 * the tree (host, synchronous: returns node count and level offsets in
 * svo->level_off).  Phase B fills the caller-allocated node arrays and fits
 * the dual normals (svo.py:139-173 cluster_normals, bit-exact). */
size_t wfpg_svo_build_workspace_bytes(int64_t n_fragments, int32_t depth);
int wfpg_svo_build_structure(wfpg_svo* svo, const int32_t* frag_coords, int64_t n_fragments,
                             void* workspace, size_t ws_bytes, void* stream);
/* frag_tris NULL: one normal per fragment (tri_normals is (F,3), fragment i's
 * normal at row i — SVOs over surface points / path vertices). */
int wfpg_svo_build_fill(wfpg_svo* svo, const int32_t* frag_tris, const double* tri_normals,
                        int64_t n_fragments, uint64_t seed,
                        void* workspace, size_t ws_bytes, void* stream);
/* Phase A from fp64 points (n,3) (surface points / path vertices): leaf
 * coordinates by the compiled quantisation against svo->lo / size /
 * resolution (_kernels.pyx:593-606), identical to wfpg_quantise_points +
 * wfpg_svo_build_structure without the coordinate array.  Phase B is
 * wfpg_svo_build_fill with frag_tris NULL (normals (n,3) per point). */
int wfpg_svo_build_structure_points(wfpg_svo* svo, const double* points, int64_t n,
                                    void* workspace, size_t ws_bytes, void* stream);
/* Debug/golden access to phase-A intermediates kept in the workspace. */
int wfpg_svo_build_sorted(const void* workspace, int64_t n_fragments,
                          const uint64_t** sorted_codes, const uint32_t** sort_perm);

/* ------------------------------------------------------------------------ */
/* Item 2 — exitance accumulation                                            */
/* ------------------------------------------------------------------------ */

/* _kernels.pyx:591-658 (descend_point/descend_kernel) -> node, present, deepest. */
int wfpg_descend(const wfpg_svo* svo, const double* points, int64_t n,
                 int32_t* out_node, uint8_t* out_present, int32_t* out_deepest, void* stream);

/* Bottom-up refresh of the leaves in leaf[0..n) and their ancestors only
 * (svo.py:265-313 with dirty leaves): leaf means from sum / weight, then the
 * dirty ancestors level by level; bitwise equal to wfpg_svo_propagate when
 * the means were consistent before the deposits.  leaf < 0 entries are
 * ignored.  dirty: n_nodes bytes of device scratch (zeroed here). */
int wfpg_svo_refresh_leaves(wfpg_svo* svo, const int32_t* leaf, int64_t n, uint8_t* dirty,
                            void* stream);

/* Fill svo->top_index (see wfpg_svo) from the node arrays; top_level in
 * [1, min(depth, 7)]; bytes = wfpg_svo_top_index_bytes(top_level). */
/* Host BVH build with the reference's decisions (bvh.py:33-119): the C++
 * port of paper_2405_06997_b200/bvh.py (binned SAH, 16 bins, <= 4 triangles
 * per leaf, stable partitions, depth-first numbering), bitwise the same
 * arrays.  Host pointers; node arrays of capacity 2T-1; *n_nodes = count. */
int wfpg_bvh_build_host(const double* v0, const double* v1, const double* v2, int64_t n,
                        double* lo, double* hi, int32_t* left, int32_t* right, int32_t* count,
                        int32_t* order, int64_t* n_nodes);

/* Device BVH build for scenes too large for the host
 * build (bvh.py:33-119): linear BVH over 63-bit Morton codes of the triangle
 * box centres (Karras 2012), subtrees of <= 4 triangles collapsed into
 * leaves (unreachable nodes stay in the arrays), written in the host
 * BVH's flattened layout (2T-1 nodes, root 0; lo / hi (N,3), left / right /
 * count (N,), order (T,), padded fp32 boxes (N,8) as wfpg_scene.bvh_box_f32).
 * Reads scene->v0/v1/v2, n_tris and the host bbox.  Nearest hits equal the
 * host BVH's except for exact ties.  Synchronises the stream; fails with
 * WFPG_ERR_ARG when the tree is deeper than the traversal stacks allow (62). */
size_t wfpg_bvh_build_workspace_bytes(int64_t n_tris);
int wfpg_bvh_build_device(const wfpg_scene* scene, double* lo, double* hi, int32_t* left,
                          int32_t* right, int32_t* count, int32_t* order, float* box_f32,
                          void* workspace, size_t ws_bytes, void* stream);

size_t wfpg_svo_top_index_bytes(int32_t top_level);
int wfpg_svo_build_top_index(wfpg_svo* svo, void* stream);

/* _kernels.pyx:593-606: points -> int32 leaf coords (F,3) with the compiled
 * quantisation (truncate (p - lo) * (R / size), clamp to [0, R-1]); cube_lo is
 * a HOST pointer to 3 doubles.  Feeds wfpg_svo_build_structure for SVOs built
 * from path vertices / synthetic points. */
int wfpg_quantise_points(const double* cube_lo, double cube_size, int32_t resolution,
                         const double* points, int64_t n, int32_t* out_coords, void* stream);

/* svo.py:254-263 (accumulate_batch): deposits applied in input order.
 * deterministic=1 reproduces np.add.at's sequential order (sort + segmented
 * sum); 0 uses fp64 atomics. */
size_t wfpg_accumulate_workspace_bytes(int64_t n);
int wfpg_svo_accumulate(wfpg_svo* svo, const int32_t* leaf, const double* dirs,
                        const double* rad, int64_t n, const int32_t* n_dev, int32_t deterministic,
                        void* workspace, size_t ws_bytes, void* stream);

/* svo.py:265-313 (propagate_up): full bottom-up recompute of mean_a/mean_b,
 * bitwise equal to the reference's dirty-only update. */
int wfpg_svo_propagate(wfpg_svo* svo, void* stream);

/* Adds an (all-reduced) leaf accumulator buffer into the SVO leaf sums and
 * refreshes every mean bottom-up (multi-GPU exitance exchange). */
int wfpg_svo_apply_leaf_acc(wfpg_svo* svo, const double* leaf_acc, void* stream);

/* wavefront.py:286-332 (update_exitance) over a finished pass. */
size_t wfpg_update_exitance_workspace_bytes(int64_t n_paths, int32_t max_depth);
int wfpg_update_exitance(wfpg_svo* svo, const wfpg_paths* paths, int32_t deterministic,
                         int32_t* n_deposits_dev, void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Item 3 — cone tracer                                                      */
/* ------------------------------------------------------------------------ */

/* _kernels.pyx:661-757 (trace_one/trace_kernel), _kernelshim.py:79-98.
 * origin_stride = 0 broadcasts a single origin. out (n,3) RGB. */
int wfpg_trace_cones(const wfpg_scene* scene, const wfpg_svo* svo, const double* origins,
                     int32_t origin_stride, const double* dirs, int64_t n, double omega,
                     double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Item 4 — field / PDF generation, guided + product sampling, MIS           */
/* ------------------------------------------------------------------------ */

/* guiding.py:231-251 (generate_fields_batch) fused with guiding.py:293-309
 * (GuideTables.fill_batch): one CTA per bin cone-traces the n x n octahedral
 * grid, takes luminance, blurs (core.py:170-195), floors at epsilon and
 * writes vals/row_sum/marg/total (+ block_sums in product mode).
 * origins (B,3), jitters (B,2). n_bins_dev optional device count <= n_bins.
 * blur_w: 2*blur_radius+1 taps (host), core._blur_kernel(sigma). */
int wfpg_generate_fields(const wfpg_scene* scene, const wfpg_svo* svo, const double* origins,
                         const double* jitters, int64_t n_bins, const int32_t* n_bins_dev,
                         int32_t n, int32_t blur_radius, const double* blur_w /* host */,
                         wfpg_guide* guide, void* stream);

/* guiding.py:293-309 (GuideTables.fill_batch) for caller-provided floored
 * values already stored in guide->vals: row sums, marginal CDF, totals and
 * (product) block sums. */
int wfpg_guide_fill(wfpg_guide* guide, int64_t n_bins, void* stream);

/* Materialise the reference's full GuideTables arrays (cond, pdftab and the
 * product block CDFs) from a B200 guide, for parity checks. */
int wfpg_guide_expand(const wfpg_guide* guide, int64_t n_bins, double* cond, double* pdftab,
                      double* blk_marg, double* blk_cond, void* stream);

/* ------------------------------------------------------------------------ */
/* Item 5 — wavefront stages                                                 */
/* ------------------------------------------------------------------------ */

/* _kernels.pyx:764-795 (camera_kernel). */
int wfpg_camera_rays(const wfpg_camera* cam, const uint64_t* keys, const int64_t* pixels,
                     int64_t n, double* out_o, double* out_d, void* stream);

/* _kernels.pyx:502-527 (intersect_kernel); misses: t = +inf, tri = -1. */
int wfpg_intersect(const wfpg_scene* scene, const double* origins, const double* dirs,
                   int64_t n, double t_min, double* out_t, int32_t* out_tri, void* stream);

/* _kernels.pyx:530-555 (occluded_kernel). */
int wfpg_occluded(const wfpg_scene* scene, const double* origins, const double* dirs,
                  int64_t n, double t_min, const double* t_max, uint8_t* out, void* stream);

/* _kernels.pyx:905-1253 (shade_one/shade_kernel), _kernelshim.py:113-151.
 * active (n_active,) path ids; bin_slot (P,) or NULL; guide may be NULL. */
int wfpg_shade_depth(const wfpg_scene* scene, wfpg_paths* paths, int32_t depth,
                     const int32_t* active, int64_t n_active, const int32_t* n_active_dev,
                     const double* hit_t, const int32_t* hit_tri, const wfpg_guide* guide,
                     const int32_t* bin_slot, int32_t rr_enabled, int32_t rr_depth, void* stream);

/* wavefront.py:98-157 (partition_spatial, Alg. 2).  positions (n,3) of the
 * lambert hits, path_idx (n,) ascending.  Outputs bins ordered by node id:
 * bin_node (B,), bin_start (B,), bin_count (B,), members (n,) path ids
 * grouped by bin, ascending within a bin; *n_bins_dev (device). */
size_t wfpg_partition_workspace_bytes(int64_t n, int64_t n_nodes);
int wfpg_partition_spatial(wfpg_svo* svo, const double* positions, const int32_t* path_idx,
                           int64_t n, const int32_t* n_dev, int32_t l_min, int32_t c_ray,
                           int32_t* bin_node, int32_t* bin_start, int32_t* bin_count,
                           int32_t* members, int32_t* n_bins_dev, int64_t bin_capacity,
                           void* workspace, size_t ws_bytes, void* stream);

/* wavefront.py:198-277 (render_pass): the whole pass on the device.
 * frame (H*W,3) receives the mean radiance of the pass; stats (host) is
 * filled after the pass (one synchronisation). */
size_t wfpg_render_workspace_bytes(const wfpg_scene* scene, const wfpg_svo* svo,
                                   const wfpg_camera* cam, const wfpg_pass_config* cfg);
int wfpg_render_pass(const wfpg_scene* scene, wfpg_svo* svo, const wfpg_camera* cam,
                     const wfpg_pass_config* cfg, wfpg_paths* paths, double* frame,
                     wfpg_pass_stats* stats, void* workspace, size_t ws_bytes, void* stream);

/* Drop the captured CUDA graph (and the seen-once key) of passes that ran
 * on `workspace` (NULL: all); call before freeing a workspace that was used
 * with use_graph = 1.  The render entry points serialise on an internal lock
 * for the graph cache. */
int wfpg_graph_release(const void* workspace);

/* Eq. 7 running sum on the device (accumulation.py:50-60): acc[i] += hw *
 * frame[i] (product rounded first, as numpy).  Non-finite frame values are
 * skipped and set *nonfinite_flag (device int32, optional) so the host can
 * raise like the reference. */
int wfpg_frame_accumulate(double* acc, const double* frame, int64_t n, double hw,
                          int32_t* nonfinite_flag, void* stream);

/* Live timing of the per-depth field kernels inside wfpg_render_pass (CUDA
 * events on the pass stream; collected when a pass returns stats).
 * field_ms / cones / launches have max_depth+1 entries indexed by depth. */
int wfpg_profile_enable(int32_t on);
int wfpg_profile_read(double* field_ms, double* cones, int64_t* launches, int32_t max_depth);

#ifdef __cplusplus
}
#endif

#endif /* WFPG_B200_H */

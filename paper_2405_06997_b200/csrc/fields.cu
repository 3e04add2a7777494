// Item 4 — per-bin radiance fields and their sampling tables, one CTA per
// bin (guiding.py:231-251 generate_fields_batch fused with guiding.py:293-309
// GuideTables.fill_batch).  The CTA cone-traces the n x n equal-area
// octahedral grid straight into shared memory, takes the luminance, applies
// the fold-aware separable Gaussian (core.py:156-195) in place, floors at
// epsilon, and writes the floored values plus row sums, marginal CDF, total
// and (product mode) 8x8 block sums.  The blur, sums and CDFs use the
// reference's numpy operation order, so given identical cone values the
// tables are bit-identical.
#include "fields.cuh"
#include "prims.cuh"
#include "shade.cuh"
#include "svo_query.cuh"

namespace wfpg {

// fold (core.py:156-167): reflect until inside, toggling the mirror flag
__device__ __forceinline__ int fold_index(int raw, int n, bool* flip) {
  bool f = false;
  while (raw < 0 || raw >= n) {
    raw = raw < 0 ? -1 - raw : 2 * n - 1 - raw;
    f = !f;
  }
  *flip = f;
  return raw;
}

// one reflection suffices when the blur radius is below n (the fixed-radius
// kernels): branch-free form of fold_index
__device__ __forceinline__ int fold_once(int raw, int n, bool* flip) {
  const bool lo = raw < 0, hi = raw >= n;
  *flip = lo | hi;
  return lo ? -1 - raw : (hi ? 2 * n - 1 - raw : raw);
}

#ifndef WFPG_SUBCONE_MAX_N
#define WFPG_SUBCONE_MAX_N 32  // quarter-tile cones in the warp cull (geometry.cuh)
#endif
#ifndef WFPG_LANE_TEST_MAX_N
#define WFPG_LANE_TEST_MAX_N 64
#endif

template <int N>
struct FieldCfg {
  static constexpr int kStride = N + 1;  // padded rows: conflict-free column walks
  // one warp per 8x4-cell tile at most: N=8 has 2 tiles, N=16 8, N=32 32.
  // Smaller CTAs for N <= 64 (measured: 256 / 128 / 64 threads beat 512 /
  // 256 / 128 and 128 / 64 / 32) keep more bins in flight per SM.
  // kThreads * kMinBlocks = 1024 -> a 64-register budget and 32+ warps per SM;
  // several CTAs (bins) per SM overlap one bin's barrier phases with
  // another's cone tracing
  static constexpr int kThreads = N >= 128 ? 1024 : (N == 64 ? 256 : (N == 32 ? 128 : 64));
  static constexpr int kMinBlocks = 1024 / kThreads;
  static constexpr int kPerLane = (N + 31) / 32;
};

template <int N>
__device__ void blur_rows(double* F, const BlurParams& bp) {
  constexpr int S = FieldCfg<N>::kStride;
  constexpr int PL = FieldCfg<N>::kPerLane;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = bp.radius;
  for (int j = warp; j < N / 2; j += nw) {
    const int jp = N - 1 - j;
    double oa[PL], ob[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      int i = lane + 32 * q;
      double a = 0.0, b = 0.0;
      if (i < N) {
        for (int k = 0; k <= 2 * r; ++k) {
          bool f;
          int c = fold_index(i + k - r, N, &f);
          double w = bp.w[k];
          double sa = f ? F[jp * S + c] : F[j * S + c];
          double sb = f ? F[j * S + c] : F[jp * S + c];
          a = __dadd_rn(a, __dmul_rn(w, sa));
          b = __dadd_rn(b, __dmul_rn(w, sb));
        }
      }
      oa[q] = a;
      ob[q] = b;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      int i = lane + 32 * q;
      if (i < N) {
        F[j * S + i] = oa[q];
        F[jp * S + i] = ob[q];
      }
    }
    __syncwarp();
  }
}

template <int N>
__device__ void blur_cols(double* F, const BlurParams& bp) {
  constexpr int S = FieldCfg<N>::kStride;
  constexpr int PL = FieldCfg<N>::kPerLane;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = bp.radius;
  for (int i = warp; i < N / 2; i += nw) {
    const int ip = N - 1 - i;
    double oa[PL], ob[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      int j = lane + 32 * q;
      double a = 0.0, b = 0.0;
      if (j < N) {
        for (int k = 0; k <= 2 * r; ++k) {
          bool f;
          int rr = fold_index(j + k - r, N, &f);
          double w = bp.w[k];
          double sa = f ? F[rr * S + ip] : F[rr * S + i];
          double sb = f ? F[rr * S + i] : F[rr * S + ip];
          a = __dadd_rn(a, __dmul_rn(w, sa));
          b = __dadd_rn(b, __dmul_rn(w, sb));
        }
      }
      oa[q] = a;
      ob[q] = b;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      int j = lane + 32 * q;
      if (j < N) {
        F[j * S + i] = oa[q];
        F[j * S + ip] = ob[q];
      }
    }
    __syncwarp();
  }
}

// Fixed-radius variants (sigma = 1 gives radius 3): interior outputs use an
// unrolled tap loop with compile-time offsets; only the r outputs at each
// edge take the fold path.  Same taps, same order, same rounding.
template <int N, int R>
__device__ void blur_rows_r(double* F, const BlurParams& bp) {
  static_assert(R < N, "fold_once needs the radius below the grid size");
  constexpr int S = FieldCfg<N>::kStride;
  constexpr int PL = FieldCfg<N>::kPerLane;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double w[2 * R + 1];
#pragma unroll
  for (int k = 0; k <= 2 * R; ++k) w[k] = bp.w[k];
  for (int j = warp; j < N / 2; j += nw) {
    const int jp = N - 1 - j;
    const double* A = F + j * S;
    const double* B = F + jp * S;
    double oa[PL], ob[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int i = lane + 32 * q;
      double a = 0.0, b = 0.0;
      if (i >= R && i < N - R) {
#pragma unroll
        for (int k = 0; k <= 2 * R; ++k) {
          a = __dadd_rn(a, __dmul_rn(w[k], A[i + k - R]));
          b = __dadd_rn(b, __dmul_rn(w[k], B[i + k - R]));
        }
      } else if (i < N) {
#pragma unroll
        for (int k = 0; k <= 2 * R; ++k) {
          bool f;
          const int c = fold_once(i + k - R, N, &f);
          a = __dadd_rn(a, __dmul_rn(w[k], f ? B[c] : A[c]));
          b = __dadd_rn(b, __dmul_rn(w[k], f ? A[c] : B[c]));
        }
      }
      oa[q] = a;
      ob[q] = b;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int i = lane + 32 * q;
      if (i < N) {
        F[j * S + i] = oa[q];
        F[jp * S + i] = ob[q];
      }
    }
    __syncwarp();
  }
}

template <int N, int R>
__device__ void blur_cols_r(double* F, const BlurParams& bp) {
  static_assert(R < N, "fold_once needs the radius below the grid size");
  constexpr int S = FieldCfg<N>::kStride;
  constexpr int PL = FieldCfg<N>::kPerLane;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double w[2 * R + 1];
#pragma unroll
  for (int k = 0; k <= 2 * R; ++k) w[k] = bp.w[k];
  for (int i = warp; i < N / 2; i += nw) {
    const int ip = N - 1 - i;
    double oa[PL], ob[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int j = lane + 32 * q;
      double a = 0.0, b = 0.0;
      if (j >= R && j < N - R) {
#pragma unroll
        for (int k = 0; k <= 2 * R; ++k) {
          const double* row = F + (j + k - R) * S;
          a = __dadd_rn(a, __dmul_rn(w[k], row[i]));
          b = __dadd_rn(b, __dmul_rn(w[k], row[ip]));
        }
      } else if (j < N) {
#pragma unroll
        for (int k = 0; k <= 2 * R; ++k) {
          bool f;
          const int rr = fold_once(j + k - R, N, &f);
          const double* row = F + rr * S;
          a = __dadd_rn(a, __dmul_rn(w[k], f ? row[ip] : row[i]));
          b = __dadd_rn(b, __dmul_rn(w[k], f ? row[i] : row[ip]));
        }
      }
      oa[q] = a;
      ob[q] = b;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int j = lane + 32 * q;
      if (j < N) {
        F[j * S + i] = oa[q];
        F[j * S + ip] = ob[q];
      }
    }
    __syncwarp();
  }
}

// Sliding-window variants (radius 3, N >= 16): one thread per (mirror pair,
// segment of N^2 / (2 threads) outputs: 8 at N = 64, 128), so a segment's 14 inputs per line are loaded once
// instead of 7 loads per output (the shared-memory pipe was the blur's
// limiter).  Every thread first reads its window head and right halo (the
// only positions other threads write), a barrier, then slides in place over
// its own segment.  Lanes map to consecutive lines (row pass) or columns
// (column pass), so the padded-row layout keeps every access conflict free.
// Same taps, same order, same rounding as blur_rows_r / blur_cols_r.
template <int N>
__device__ __forceinline__ void blur_rows_sw(double* F, const BlurParams& bp) {
  constexpr int S = FieldCfg<N>::kStride, NP = N / 2;
  constexpr int L = N * NP / FieldCfg<N>::kThreads;  // outputs per thread and line
  static_assert(NP * (N / L) == FieldCfg<N>::kThreads && L >= 2, "one thread per (pair, segment)");
  const int t = threadIdx.x;
  const int j = t % NP, c0 = (t / NP) * L;
  double* A = F + j * S;
  double* B = F + (N - 1 - j) * S;
  double xa[L + 6], xb[L + 6];  // virtual positions c0 - 3 + k
#pragma unroll
  for (int k = 0; k < L + 6; ++k) {
    if (k >= 7 && k <= L + 2) continue;  // inside the segment: read after the barrier
    bool f;
    const int c = fold_once(c0 - 3 + k, N, &f);
    xa[k] = f ? B[c] : A[c];
    xb[k] = f ? A[c] : B[c];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < L; ++q) {
    if (q >= 1 && q <= L - 4) {
      xa[6 + q] = A[c0 + 3 + q];
      xb[6 + q] = B[c0 + 3 + q];
    }
    // numpy's 0 + w0 x0 + ... : the leading 0 + p is p itself (p >= +0:
    // luminances and Gaussian taps are non-negative, so no -0 to normalise)
    double a = __dmul_rn(bp.w[0], xa[q]), b = __dmul_rn(bp.w[0], xb[q]);
#pragma unroll
    for (int k = 1; k < 7; ++k) {
      a = __dadd_rn(a, __dmul_rn(bp.w[k], xa[q + k]));
      b = __dadd_rn(b, __dmul_rn(bp.w[k], xb[q + k]));
    }
    A[c0 + q] = a;
    B[c0 + q] = b;
  }
}

// The column pass is the blur's last step: it applies the epsilon floor
// (guiding.py:249) as it writes each output and stores the floored value to
// the bin's global table row (lanes on consecutive columns: coalesced).
template <int N>
__device__ __forceinline__ void blur_cols_sw(double* F, const BlurParams& bp, double eps,
                                             double* __restrict__ gvals) {
  constexpr int S = FieldCfg<N>::kStride, NP = N / 2;
  constexpr int L = N * NP / FieldCfg<N>::kThreads;
  static_assert(NP * (N / L) == FieldCfg<N>::kThreads && L >= 2, "one thread per (pair, segment)");
  const int t = threadIdx.x;
  const int i = t % NP, ip = N - 1 - i, r0 = (t / NP) * L;
  double xa[L + 6], xb[L + 6];  // virtual rows r0 - 3 + k
#pragma unroll
  for (int k = 0; k < L + 6; ++k) {
    if (k >= 7 && k <= L + 2) continue;
    bool f;
    const int rr = fold_once(r0 - 3 + k, N, &f);
    const double* row = F + rr * S;
    xa[k] = f ? row[ip] : row[i];
    xb[k] = f ? row[i] : row[ip];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < L; ++q) {
    if (q >= 1 && q <= L - 4) {
      const double* row = F + (r0 + 3 + q) * S;
      xa[6 + q] = row[i];
      xb[6 + q] = row[ip];
    }
    // numpy's 0 + w0 x0 + ... : the leading 0 + p is p itself (p >= +0:
    // luminances and Gaussian taps are non-negative, so no -0 to normalise)
    double a = __dmul_rn(bp.w[0], xa[q]), b = __dmul_rn(bp.w[0], xb[q]);
#pragma unroll
    for (int k = 1; k < 7; ++k) {
      a = __dadd_rn(a, __dmul_rn(bp.w[k], xa[q + k]));
      b = __dadd_rn(b, __dmul_rn(bp.w[k], xb[q + k]));
    }
    a = a < eps ? eps : a;
    b = b < eps ? eps : b;
    F[(r0 + q) * S + i] = a;
    F[(r0 + q) * S + ip] = b;
    gvals[(r0 + q) * N + i] = a;
    gvals[(r0 + q) * N + ip] = b;
  }
}

#ifdef WFPG_FIELD_PHASES
// phase profiling build: cycles between the phase boundaries of thread 0,
// summed over bins and CTAs (phase 0 = setup, 1 trace, 2 blur, 3 floor +
// values, 4 row sums + marginal, 5 prefix sums + stores)
__device__ unsigned long long g_field_phase[40];  // [log2(N) - 3][phase]
template <int N>
__device__ __forceinline__ void ph_mark(int k) {
  static __shared__ long long last;
  constexpr int row = N == 8 ? 0 : (N == 16 ? 1 : (N == 32 ? 2 : (N == 64 ? 3 : 4)));
  long long now = clock64();
  if (k > 0) atomicAdd(&g_field_phase[row * 8 + k - 1], (unsigned long long)(now - last));
  last = now;
}
#endif

// PRODUCT: block sums (+ block row sums) for the product sampler; a separate
// instantiation so the plain kernel carries none of its registers.
// TRACE: the scene's nearest-hit path — kTraceBrute (triangle records in
// shared memory, warp-culled), kTracePacket (warp-cooperative BVH walk over
// the padded fp32 node boxes), kTraceLane (per-lane fp64 BVH walk, scenes
// without fp32 boxes) — one instantiation each so every path keeps its
// register budget.
enum { kTraceBrute = 0, kTracePacket = 1, kTraceLane = 2 };

template <int N, bool PRODUCT, int TRACE>
__global__ void __launch_bounds__(FieldCfg<N>::kThreads, FieldCfg<N>::kMinBlocks)
    k_fields(SceneView s, SvoView v, const double* __restrict__ origins,
             const double* __restrict__ jitters, int64_t nb_max, const int32_t* __restrict__ nb_dev,
             BlurParams bp, FieldOut out) {
  constexpr int S = FieldCfg<N>::kStride;
  static_assert(N > WFPG_SUBCONE_MAX_N || FieldCfg<N>::kThreads / 32 <= kSubWarps,
                "quarter-tile cones: one shared slot per warp");
  // warp tiles of 8 (u) x 4 (v) cells: the 32 cones of a warp are angularly
  // coherent, so whole-warp triangle culling is effective
  constexpr int TU = 8, TV = 4, TILES_U = N / TU, TILES = (N / TU) * (N / TV);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int tile_ctr;
  double* F = reinterpret_cast<double*>(smem_raw);
  double* rs = F + N * S;  // row sums (N)
  double* uv = rs + N;     // u of column i, then v of row j (2N)
  TriBin* tb = reinterpret_cast<TriBin*>(uv + 2 * N);
  const int64_t nb = dev_count(nb_max, nb_dev);
  const double omega = 4.0 * WFPG_PI / (double)(N * N);  // guiding.py:246
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ int64_t next_bin;
  __shared__ double tot_sh;
  // per-bin tables: u = i/n + ju/n, v = j/n + jv/n (guiding.py:239-244) and
  // the triangle records for the bin's origin (three threads per triangle).
  // The next bin's tables are built during this bin's blur (they are free
  // once the cone tracing is done), off the critical path.
  auto setup = [&](int64_t bb) {
    const double sx = origins[3 * bb], sy = origins[3 * bb + 1], sz = origins[3 * bb + 2];
    const int n_tb = TRACE == kTraceBrute ? 3 * s.n_tris : 0;
    for (int k = threadIdx.x; k < 2 * N + n_tb; k += blockDim.x) {
      if (k < 2 * N) {
        const int i = k < N ? k : k - N;
        const double jit = __ddiv_rn(jitters[2 * bb + (k < N ? 0 : 1)], (double)N);
        uv[k] = __dadd_rn(__ddiv_rn((double)i, (double)N), jit);
      } else {
        const int q = k - 2 * N;
        make_tri_bin_part(s, q / 3, q % 3, sx, sy, sz, tb[q / 3]);
      }
    }
  };
  // work item w -> bin (identity, or the multi-GPU work list); thread 0 owns
  // the work index, the loop carries only the bin
  auto bin_of = [&](int64_t w) -> int64_t { return out.bin_list ? (int64_t)out.bin_list[w] : w; };
  __shared__ int64_t cur_w;
  int64_t b = (int64_t)blockIdx.x < nb ? bin_of(blockIdx.x) : -1;
  if (threadIdx.x == 0) cur_w = blockIdx.x;
  if (b >= 0) setup(b);
  for (; b >= 0;) {
    const double ox = origins[3 * b], oy = origins[3 * b + 1], oz = origins[3 * b + 2];
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(0);
#endif
    if (threadIdx.x == 0) tile_ctr = nwarps;
    __syncthreads();
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(1);
#endif
    // 1. cone-trace every cell; tiles are handed out dynamically (cull
    // candidates and hit depths vary per tile, static striping left warps
    // idling at the barrier)
    for (int tile = warp; tile < TILES;) {
      const int i = (tile % TILES_U) * TU + (lane % TU);
      const int j = (tile / TILES_U) * TV + (lane / TU);
      double dx, dy, dz;
      octa_uv_to_dir_cell(uv[i], uv[N + j], &dx, &dy, &dz);
      double rgb[3] = {0.0, 0.0, 0.0};
      double bt;
      int32_t bid;
      if (TRACE == kTraceBrute)
        warp_nearest_bin<(N <= WFPG_LANE_TEST_MAX_N), (N <= WFPG_SUBCONE_MAX_N)>(
            tb, s.n_tris, dx, dy, dz, s.ray_eps, &bt, &bid);
      else if (TRACE == kTracePacket)
        warp_bvh_nearest(s, reinterpret_cast<int2*>(tb) + warp * kWarpBvhStack, ox, oy, oz, dx,
                         dy, dz, s.ray_eps, &bt, &bid,
                         reinterpret_cast<double*>(reinterpret_cast<int2*>(tb) +
                                                   nwarps * kWarpBvhStack) +
                             warp * kLeafStage * kLeafRec);
      else
        bvh_nearest(s, ox, oy, oz, dx, dy, dz, s.ray_eps, &bt, &bid);
      if (bid >= 0) {
        // the origin re-read here (L1) rather than held in registers
        // through the cull and the triangle tests
        const double* o3 = origins + 3 * b;
        cone_shade_hit(v, __ldg(o3), __ldg(o3 + 1), __ldg(o3 + 2), dx, dy, dz, bt, omega, rgb);
      }
      F[j * S + i] = luminance_rows(rgb[0], rgb[1], rgb[2]);
      int next = 0;
      if (lane == 0) next = atomicAdd(&tile_ctr, 1);
      tile = __shfl_sync(0xffffffffu, next, 0);
    }
    if (threadIdx.x == 0) {
      const int64_t wn =
          out.bin_ctr ? (int64_t)atomicAdd(out.bin_ctr, 1) + gridDim.x : cur_w + gridDim.x;
      cur_w = wn;
      next_bin = wn < nb ? bin_of(wn) : -1;
    }
    __syncthreads();
    const int64_t b_next = next_bin;
    if (b_next >= 0) setup(b_next);  // overlaps the blur below
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(2);
#endif
    // 2. fold-aware separable blur, horizontal then vertical (core.py:185-195)
    bool blurred = false;
    if constexpr (N >= 16) {
      if (bp.radius == 3) {
        blur_rows_sw<N>(F, bp);
        __syncthreads();
        blur_cols_sw<N>(F, bp, out.eps, out.vals + b * (int64_t)N * N);
        __syncthreads();
        blurred = true;
      }
    }
    if (blurred) {
    } else if (bp.radius == 3 && N > 8) {
      blur_rows_r<N, 3>(F, bp);
      __syncthreads();
      blur_cols_r<N, 3>(F, bp);
      __syncthreads();
    } else if (bp.radius > 0) {
      blur_rows<N>(F, bp);
      __syncthreads();
      blur_cols<N>(F, bp);
      __syncthreads();
    }
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(3);
#endif
    // 3. epsilon floor + store values (the sliding blur did both already);
    // one element per lane: conflict-free on the padded rows
    if (!blurred) {
      double* gv = out.vals + b * (int64_t)N * N;
      for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
        const int j = e / N, i = e % N;
        double x = F[j * S + i];
        x = x < out.eps ? out.eps : x;
        F[j * S + i] = x;
        gv[e] = x;
      }
      __syncthreads();
    }
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(4);
#endif
    // 4. row sums (0 + numpy pairwise: 8 strided accumulators combined as
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), exact for N in 8..128), 8 lanes
    // per row, then total / marginal CDF (guiding.py:296-298)
    for (int t = threadIdx.x; t < 8 * N; t += blockDim.x) {
      // 8 lanes per row; the two rows of a 16-lane shared-memory phase are 8
      // apart (16 banks on the padded rows), so the loads never conflict
      const int slot = t >> 3, k = t & 7;
      const int j = N >= 32 ? (slot & ~31) + ((slot & 31) >> 2) + 8 * (slot & 3) : slot;
      const double* row = F + j * S;
      double r = row[k];
      for (int i = k + 8; i < N; i += 8) r = __dadd_rn(r, row[i]);
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
      if (k == 0) {
        r = __dadd_rn(0.0, r);
        rs[j] = r;
        out.row_sum[b * N + j] = r;
      }
    }
    if (PRODUCT && out.block_sums && out.block_rows) {
      // every (block, row) pair in parallel, then the sequential sum of each
      // block's rows (guiding.py:302-304 order)
      constexpr int M = N / 8;
      double* br = out.block_rows + b * 64 * M;
      for (int t = threadIdx.x; t < 64 * M; t += blockDim.x) {
        const int q = t / M, r = t % M, bj = q / 8, bi = q % 8;
        br[t] = __dadd_rn(0.0, pairwise_row(F + (bj * M + r) * S + bi * M, M));
      }
      __syncthreads();
      for (int q = threadIdx.x; q < 64; q += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < M; ++r) acc = __dadd_rn(acc, br[q * M + r]);
        out.block_sums[b * 64 + q] = acc;
      }
    } else if (PRODUCT && out.block_sums) {
      constexpr int M = N / 8;
      for (int q = threadIdx.x; q < 64; q += blockDim.x) {
        const int bj = q / 8, bi = q % 8;
        double acc = 0.0;
        for (int r = 0; r < M; ++r)
          acc = __dadd_rn(acc, __dadd_rn(0.0, pairwise_row(F + (bj * M + r) * S + bi * M, M)));
        out.block_sums[b * 64 + q] = acc;
      }
    }
    __syncthreads();
    // total and the sequential running sum of the row sums (np.cumsum order,
    // in place) by thread 0, while the other warps turn each row of F into
    // its unnormalised prefix sums (np.cumsum order) for the samplers:
    // cond[j, i] = cum[j, i] / row_sum[j] is then one division at the picked
    // cell instead of a division per scanned cell
    if (threadIdx.x == 0) {
      const double tot = __dadd_rn(0.0, pairwise_row(rs, N));
      out.total[b] = tot;
      tot_sh = tot;
      double run = rs[0];
#pragma unroll 8
      for (int j = 1; j < N; ++j) {
        run = __dadd_rn(run, rs[j]);
        rs[j] = run;
      }
    } else if (out.cum && threadIdx.x >= 32) {
      for (int j = threadIdx.x - 32; j < N; j += blockDim.x - 32) {
        double run = F[j * S];
        for (int i = 1; i < N; ++i) {
          run = __dadd_rn(run, F[j * S + i]);
          F[j * S + i] = run;
        }
      }
    }
    __syncthreads();
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(5);
#endif
    // 5. marginal CDF divisions and the prefix-sum table stores, in parallel
    for (int j = threadIdx.x; j < N; j += blockDim.x) out.marg[b * N + j] = __ddiv_rn(rs[j], tot_sh);
    if (out.cum) {
      double* gc = out.cum + b * (int64_t)N * N;
      for (int e = threadIdx.x; e < N * N; e += blockDim.x) gc[e] = F[(e / N) * S + e % N];
    }
#ifdef WFPG_FIELD_PHASES
    if (threadIdx.x == 0) ph_mark<N>(6);
#endif
    __syncthreads();
    b = b_next;
  }
}

template <int N, bool PRODUCT, int TRACE>
static int launch_fields_n_(const SceneView& s, const SvoView& v, const double* origins,
                           const double* jitters, int64_t nb_max, const int32_t* nb_dev,
                           const BlurParams& bp, const FieldOut& out, cudaStream_t st) {
  constexpr int T = FieldCfg<N>::kThreads;
  size_t smem = sizeof(double) * (N * FieldCfg<N>::kStride + 3 * N) +
                (TRACE == kTraceBrute ? sizeof(TriBin) * s.n_tris
                 : TRACE == kTracePacket ? (sizeof(int2) * kWarpBvhStack +  // warp stacks,
                                            sizeof(double) * kLeafStage * kLeafRec) * (T / 32)  // leaf records
                                         : 0);
  static size_t configured = 0;
  if (smem > configured) {
    WFPG_CUDA(cudaFuncSetAttribute(k_fields<N, PRODUCT, TRACE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured = smem;
  }
  int per_sm = 0;
  WFPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fields<N, PRODUCT, TRACE>, T, smem));
  if (per_sm < 1) {
    set_error("fields: kernel does not fit (smem %zu)", smem);
    return WFPG_ERR_ARG;
  }
  int64_t grid = std::min<int64_t>(nb_max, (int64_t)kNumSMs * per_sm);
  if (grid < 1) return WFPG_OK;
  k_fields<N, PRODUCT, TRACE><<<(unsigned)grid, T, smem, st>>>(s, v, origins, jitters, nb_max, nb_dev, bp, out);
  WFPG_CHECK_LAUNCH("k_fields");
  return WFPG_OK;
}

template <int N>
static int launch_fields_n(const SceneView& s, const SvoView& v, const double* origins,
                           const double* jitters, int64_t nb_max, const int32_t* nb_dev,
                           const BlurParams& bp, const FieldOut& out, cudaStream_t st) {
#define WFPG_FIELDS_(P, T) launch_fields_n_<N, P, T>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st)
  const bool prod = out.block_sums != nullptr;
  if (s.brute) return prod ? WFPG_FIELDS_(true, kTraceBrute) : WFPG_FIELDS_(false, kTraceBrute);
  if (s.bbox32) return prod ? WFPG_FIELDS_(true, kTracePacket) : WFPG_FIELDS_(false, kTracePacket);
  return prod ? WFPG_FIELDS_(true, kTraceLane) : WFPG_FIELDS_(false, kTraceLane);
#undef WFPG_FIELDS_
}

int launch_fields(const SceneView& s, const SvoView& v, const double* origins,
                  const double* jitters, int64_t nb_max, const int32_t* nb_dev, int n,
                  const BlurParams& bp, const FieldOut& out, cudaStream_t st) {
  if (nb_max <= 0) return WFPG_OK;
  switch (n) {
    case 8: return launch_fields_n<8>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st);
    case 16: return launch_fields_n<16>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st);
    case 32: return launch_fields_n<32>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st);
    case 64: return launch_fields_n<64>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st);
    case 128: return launch_fields_n<128>(s, v, origins, jitters, nb_max, nb_dev, bp, out, st);
    default:
      set_error("field resolution must be one of 8, 16, 32, 64, 128 (got %d)", n);
      return WFPG_ERR_ARG;
  }
}

// ---------------------------------------------------------------------------
// reference-layout tables (GuideTables.fill_batch) for parity checks
// ---------------------------------------------------------------------------
__global__ void k_guide_expand(GuideView g, int64_t nb, double* cond, double* pdftab,
                               double* blk_marg, double* blk_cond) {
  const int n = g.n, m = g.m;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nb * n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = r / n;
    const double* row = g.vals + r * n;
    double rsum = g.row_sum[r];
    double run = 0.0;
    for (int i = 0; i < n; ++i) {
      run = i == 0 ? row[0] : __dadd_rn(run, row[i]);
      if (cond) cond[r * n + i] = __ddiv_rn(run, rsum);
      if (pdftab) pdftab[r * n + i] = __ddiv_rn(__dmul_rn(row[i], g.pdf_scale), g.total[b]);
    }
    if (g.mode == 2 && m > 0) {
      // r indexes (b, j); block row jin = j % m of block (bj = j / m, bi)
      int j = (int)(r % n);
      int bj = j / m, jin = j % m;
      for (int bi = 0; bi < 8; ++bi) {
        const double* brow = row + bi * m;
        double rw = __dadd_rn(0.0, pairwise_row(brow, m));
        double run2 = 0.0;
        int64_t cbase = ((((b * 8 + bj) * 8 + bi) * m) + jin) * m;
        for (int i = 0; i < m; ++i) {
          run2 = i == 0 ? brow[0] : __dadd_rn(run2, brow[i]);
          if (blk_cond) blk_cond[cbase + i] = __ddiv_rn(run2, rw);
        }
        if (blk_marg && jin == m - 1) {
          // the whole block is known here: cumsum of its row sums / block sum
          const double* blk0 = g.vals + (b * n + bj * m) * n + bi * m;
          double bsum = g.block_sums[(b * 8 + bj) * 8 + bi];
          double run3 = 0.0;
          for (int q = 0; q < m; ++q) {
            double rq = __dadd_rn(0.0, pairwise_row(blk0 + (int64_t)q * n, m));
            run3 = q == 0 ? rq : __dadd_rn(run3, rq);
            blk_marg[(((b * 8 + bj) * 8 + bi) * m) + q] = __ddiv_rn(run3, bsum);
          }
        }
      }
    }
  }
}

// GuideTables.fill_batch on caller-provided floored values (guiding.py:293-309)
__global__ void k_guide_fill(const double* __restrict__ vals, int n, int64_t nb,
                             double* __restrict__ row_sum, double* __restrict__ marg,
                             double* __restrict__ total, double* __restrict__ block_sums,
                             double* __restrict__ block_rows) {
  extern __shared__ double rs[];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const double* v = vals + b * (int64_t)n * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double r = __dadd_rn(0.0, pairwise_row(v + (int64_t)j * n, n));
      rs[j] = r;
      row_sum[b * n + j] = r;
    }
    if (block_sums) {
      const int M = n / 8;
      for (int q = threadIdx.x; q < 64; q += blockDim.x) {
        const int bj = q / 8, bi = q % 8;
        double acc = 0.0;
        for (int r = 0; r < M; ++r) {
          const double rr = __dadd_rn(0.0, pairwise_row(v + (int64_t)(bj * M + r) * n + bi * M, M));
          if (block_rows) block_rows[(b * 64 + q) * M + r] = rr;
          acc = __dadd_rn(acc, rr);
        }
        block_sums[b * 64 + q] = acc;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = __dadd_rn(0.0, pairwise_row(rs, n));
      total[b] = tot;
      double run = 0.0;
      for (int j = 0; j < n; ++j) {
        run = j == 0 ? rs[0] : __dadd_rn(run, rs[j]);
        marg[b * n + j] = __ddiv_rn(run, tot);
      }
    }
    __syncthreads();
  }
}

// Multi-GPU bin ownership (render.cu): every rank generated the fields of
// its own contiguous bin range [own_lo, own_hi) and the values of all bins
// were all-gathered into `src` (standard bin order).  This fills every other
// bin's tables from those values — values, row sums, marginal, total, row
// prefix sums and (product) block row sums / block sums — with the field
// kernel's arithmetic (numpy pairwise row sums, sequential cumsums), so the
// tables equal the ones the owning rank computed, bit for bit.  Runs only when
// *own_ok (the bin count fitted the ownership ranges).
__global__ void k_own_fill(const double* __restrict__ src, int n, const int32_t* __restrict__ n_bins,
                           const int32_t* __restrict__ own_ok, int64_t own_lo, int64_t own_hi,
                           double* __restrict__ vals, double* __restrict__ cum,
                           double* __restrict__ row_sum, double* __restrict__ marg,
                           double* __restrict__ total, double* __restrict__ block_sums,
                           double* __restrict__ block_rows) {
  extern __shared__ double rs[];
  if (!*own_ok) return;
  const int64_t nb = *n_bins;
  const int64_t nn = (int64_t)n * n;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    if (b >= own_lo && b < own_hi) continue;  // generated here
    const double* v = src + b * nn;
    double* dv = vals + b * nn;
    for (int64_t c = threadIdx.x; c < nn; c += blockDim.x) dv[c] = v[c];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double* row = v + (int64_t)j * n;
      double r = __dadd_rn(0.0, pairwise_row(row, n));
      rs[j] = r;
      row_sum[b * n + j] = r;
      if (cum) {
        double run = row[0];
        double* cr = cum + b * nn + (int64_t)j * n;
        cr[0] = run;
        for (int i = 1; i < n; ++i) {
          run = __dadd_rn(run, row[i]);
          cr[i] = run;
        }
      }
    }
    if (block_sums) {
      const int M = n / 8;
      for (int q = threadIdx.x; q < 64; q += blockDim.x) {
        const int bj = q / 8, bi = q % 8;
        double acc = 0.0;
        for (int r = 0; r < M; ++r) {
          const double rr = __dadd_rn(0.0, pairwise_row(v + (int64_t)(bj * M + r) * n + bi * M, M));
          if (block_rows) block_rows[(b * 64 + q) * M + r] = rr;
          acc = __dadd_rn(acc, rr);
        }
        block_sums[b * 64 + q] = acc;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double tot = __dadd_rn(0.0, pairwise_row(rs, n));
      total[b] = tot;
      double run = 0.0;
      for (int j = 0; j < n; ++j) {
        run = j == 0 ? rs[0] : __dadd_rn(run, rs[j]);
        rs[j] = run;
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) marg[b * n + j] = __ddiv_rn(rs[j], total[b]);
    __syncthreads();
  }
}

int launch_own_fill(const double* src, int n, const int32_t* n_bins, const int32_t* own_ok,
                    int64_t own_lo, int64_t own_hi, int64_t cap, const FieldOut& out,
                    cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cap, (int64_t)kNumSMs * 8));
  k_own_fill<<<grid, 128, sizeof(double) * n, st>>>(src, n, n_bins, own_ok, own_lo, own_hi,
                                                   out.vals, out.cum, out.row_sum, out.marg,
                                                   out.total, out.block_sums, out.block_rows);
  WFPG_CHECK_LAUNCH("k_own_fill");
  return WFPG_OK;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" int wfpg_guide_fill(wfpg_guide* guide, int64_t n_bins, void* stream) {
  if (!guide || n_bins < 0 || guide->n < 1 || guide->n > 128 || !guide->vals || !guide->row_sum ||
      !guide->marg || !guide->total || (guide->mode == 2 && (!guide->block_sums || guide->n % 8))) {
    set_error("wfpg_guide_fill: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n_bins == 0) return WFPG_OK;
  int grid = (int)std::min<int64_t>(n_bins, kNumSMs * 8);
  k_guide_fill<<<grid, 128, sizeof(double) * guide->n, as_stream(stream)>>>(
      guide->vals, guide->n, n_bins, guide->row_sum, guide->marg, guide->total,
      guide->mode == 2 ? guide->block_sums : nullptr,
      guide->mode == 2 ? guide->block_rows : nullptr);
  WFPG_CHECK_LAUNCH("k_guide_fill");
  return WFPG_OK;
}

extern "C" int wfpg_generate_fields(const wfpg_scene* scene, const wfpg_svo* svo,
                                    const double* origins, const double* jitters, int64_t n_bins,
                                    const int32_t* n_bins_dev, int32_t n, int32_t blur_radius,
                                    const double* blur_w, wfpg_guide* guide, void* stream) {
  if (!scene || !svo || !guide || n_bins < 0 || blur_radius < 0 || blur_radius > 16 ||
      (blur_radius > 0 && !blur_w) || (n_bins > 0 && (!origins || !jitters)) ||
      !guide->vals || !guide->row_sum || !guide->marg || !guide->total) {
    set_error("wfpg_generate_fields: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (guide->capacity < n_bins) {
    set_error("wfpg_generate_fields: guide capacity %d < %lld bins", guide->capacity,
              (long long)n_bins);
    return WFPG_ERR_CAPACITY;
  }
  BlurParams bp{};
  bp.radius = blur_radius;
  for (int k = 0; k <= 2 * blur_radius && blur_radius > 0; ++k) bp.w[k] = blur_w[k];
  FieldOut out{guide->vals, guide->row_sum, guide->marg, guide->total,
               guide->mode == 2 ? guide->block_sums : nullptr, guide->eps, guide->cum};
  out.block_rows = guide->mode == 2 ? guide->block_rows : nullptr;
  guide->n = n;
  return launch_fields(make_scene_view(scene), make_view(svo), origins, jitters, n_bins,
                       n_bins_dev, n, bp, out, as_stream(stream));
}

extern "C" int wfpg_guide_expand(const wfpg_guide* guide, int64_t n_bins, double* cond,
                                 double* pdftab, double* blk_marg, double* blk_cond,
                                 void* stream) {
  if (!guide || n_bins < 0 || (guide->mode == 2 && !guide->block_sums)) {
    set_error("wfpg_guide_expand: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n_bins == 0) return WFPG_OK;
  GuideView g{};
  g.mode = guide->mode;
  g.n = guide->n;
  g.m = guide->n / 8;
  g.pdf_scale = (double)(guide->n * guide->n) / (4.0 * WFPG_PI);
  g.vals = guide->vals;
  g.row_sum = guide->row_sum;
  g.total = guide->total;
  g.block_sums = guide->block_sums;
  int64_t rows = n_bins * guide->n;
  int grid = (int)std::min<int64_t>(ceil_div(rows, 128), kNumSMs * 8);
  k_guide_expand<<<grid, 128, 0, as_stream(stream)>>>(g, n_bins, cond, pdftab, blk_marg, blk_cond);
  WFPG_CHECK_LAUNCH("k_guide_expand");
  return WFPG_OK;
}

#ifdef WFPG_FIELD_PHASES
extern "C" int wfpg_field_phases(unsigned long long* out, int reset) {
  WFPG_CUDA(cudaDeviceSynchronize());
  WFPG_CUDA(cudaMemcpyFromSymbol(out, wfpg::g_field_phase, sizeof(unsigned long long) * 40));
  if (reset) {
    unsigned long long z[40] = {0};
    WFPG_CUDA(cudaMemcpyToSymbol(wfpg::g_field_phase, z, sizeof(z)));
  }
  return 0;
}
#endif

// Shared device helpers for the B200 guided wavefront path.
//
// Numerics follow the reference exactly where a bit-exact result is claimed
// (SVO build, Morton/sort, descents, blur, CDF tables); those helpers use the
// explicitly rounded intrinsics (__dmul_rn, __dadd_rn, __fma_rn, ...) so
// nvcc cannot contract them.  Everything else is plain fp64 device code.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/wfpg_b200.h"

#define WFPG_PI 3.141592653589793238462643383279502884
#define WFPG_INV_2_53 (1.0 / 9007199254740992.0)

namespace wfpg {

// ---------------------------------------------------------------------------
// error plumbing (implemented in runtime.cu)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
void count_launch(uint64_t k = 1);

#define WFPG_CHECK_LAUNCH(what)                                  \
  do {                                                           \
    ::wfpg::count_launch();                                      \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::wfpg::cuda_status(_e, what); \
  } while (0)

#define WFPG_CUDA(call)                                          \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::wfpg::cuda_status(_e, #call); \
  } while (0)

#define WFPG_TRY(call)                 \
  do {                                 \
    int _s = (call);                   \
    if (_s != WFPG_OK) return _s;      \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// NVTX ranges around the host entry points (header-only NVTX v3: inert
// unless a tool such as Nsight Systems injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
  char* base;
  size_t cap;
  size_t off;
  bool measure;  // size query only
  Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c), off(0), measure(b == nullptr) {}
  template <class T>
  T* take(int64_t count) {
    size_t bytes = align_up(sizeof(T) * (size_t)(count > 0 ? count : 1));
    T* p = measure ? nullptr : reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
  bool ok() const { return measure || off <= cap; }
};

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// counter-based RNG: core.py:204-228, _kernels.pyx:212-223 (splitmix64)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;

// core.py:213-216
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ (mix64(stream) * kPhi));
}
// core.py:226-228
__host__ __device__ __forceinline__ double u01(uint64_t key, uint64_t c) {
  uint64_t v = mix64(key + (c + 1) * kPhi);
  return (double)(v >> 11) * WFPG_INV_2_53;
}

// ---------------------------------------------------------------------------
// Morton: core.py:91-138, _kernels.pyx:562-573
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t spread21(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ __forceinline__ uint64_t morton3(uint64_t x, uint64_t y, uint64_t z) {
  return spread21(x) | (spread21(y) << 1) | (spread21(z) << 2);
}

// ---------------------------------------------------------------------------
// Exact numpy/OpenBLAS dot recipes (measured, see oracle/NUMERICS.md)
//   dgemv rows (K >= 2):   fma(x2,m2, fma(x0,m0, x1*m1))
//   ddot / (1,3)@(3,):    fma(x2,m2, fma(x1,m1, x0*m0))
//   np.linalg.norm(1-D):  sqrt(ddot(x,x))
//   einsum("ij,ij->i"):   (x0*y0 + x2*y2) + x1*y1
//   np.linalg.norm(axis=-1) of (...,3): sqrt((x0*x0 + x1*x1) + x2*x2)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dot_gemv(double x0, double x1, double x2, double m0, double m1,
                                           double m2) {
  return __fma_rn(x2, m2, __fma_rn(x0, m0, __dmul_rn(x1, m1)));
}
__device__ __forceinline__ double dot_ddot(double x0, double x1, double x2, double m0, double m1,
                                           double m2) {
  return __fma_rn(x2, m2, __fma_rn(x1, m1, __dmul_rn(x0, m0)));
}
__device__ __forceinline__ double dot_einsum(double x0, double x1, double x2, double y0, double y1,
                                             double y2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(x0, y0), __dmul_rn(x2, y2)), __dmul_rn(x1, y1));
}
__device__ __forceinline__ double norm_axis(double x, double y, double z) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// fp64 constants of the hot device functions in constant memory: an fp64
// literal costs two register moves per use (no 64-bit immediates), a
// constant-bank operand costs nothing (DFMA R, R, c[bank][off], R)
static __constant__ double c_k[24] = {
    0.2126, 0.7152, 0.0722,                                           // 0-2 LUMA_WEIGHTS
    1.0 / 355687428096000.0, 1.0 / 1307674368000.0, 1.0 / 6227020800.0,  // 3-5 sin
    1.0 / 39916800.0, 1.0 / 362880.0, 1.0 / 5040.0, 1.0 / 120.0, 1.0 / 6.0,  // 6-10
    1.0 / 6402373705728000.0, 1.0 / 20922789888000.0, 1.0 / 87178291200.0,  // 11-13 cos
    1.0 / 479001600.0, 1.0 / 3628800.0, 1.0 / 40320.0, 1.0 / 720.0, 1.0 / 24.0,  // 14-18
    0.5, WFPG_PI / 4.0, 0.70710678118654752440, 0.0, 0.0};             // 19-21

// luminance of an (M,3) RGB array: core.py:18-19 (rgb @ LUMA_WEIGHTS, dgemv)
__device__ __forceinline__ double luminance_rows(double r, double g, double b) {
  return dot_gemv(r, g, b, c_k[0], c_k[1], c_k[2]);
}

// ---------------------------------------------------------------------------
// Equal-area octahedral map
// ---------------------------------------------------------------------------
// numpy flavour (core.py:32-55): used for field cell directions and the
// product layer's upper directions.  Normalises by *division* by the norm.
__device__ __forceinline__ void octa_uv_to_dir_np(double u, double v, double* ox, double* oy,
                                                  double* oz) {
  double a = __dsub_rn(__dmul_rn(2.0, u), 1.0);
  double b = __dsub_rn(__dmul_rn(2.0, v), 1.0);
  double ap = fabs(a), bp = fabs(b);
  double sd = __dsub_rn(1.0, __dadd_rn(ap, bp));
  double d = fabs(sd);
  double r = __dsub_rn(1.0, d);
  double phi = (r == 0.0) ? 1.0 : __dadd_rn(__ddiv_rn(__dsub_rn(bp, ap), r), 1.0);
  phi = __dmul_rn(phi, WFPG_PI / 4.0);
  double rr = __dmul_rn(r, r);
  double z = copysign(__dsub_rn(1.0, rr), sd);
  double rho = __dmul_rn(r, __dsqrt_rn(fmax(__dsub_rn(2.0, rr), 0.0)));
  double s, c;
  sincos(phi, &s, &c);
  double x = __dmul_rn(copysign(c, a), rho);
  double y = __dmul_rn(copysign(s, b), rho);
  double nrm = norm_axis(x, y, z);
  *ox = __ddiv_rn(x, nrm);
  *oy = __ddiv_rn(y, nrm);
  *oz = __ddiv_rn(z, nrm);
}

// Division / square root without the IEEE slow-path checks, for values that
// only need to be within a few ulp (the field-cell map and hit distances,
// compared to the reference with a 1e-9 tolerance): hardware approximation
// refined by Newton steps.  Arguments must be normal, positive where noted.
__device__ __forceinline__ double fast_div(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  double q = a * r;
  return fma(fma(-b, q, a), r, q);
}
__device__ __forceinline__ double fast_sqrt(double x) {  // x > 0
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * y;
  double g = x * y;
  double e = fma(-g, h, 0.5);  // Goldschmidt / Newton on (g, h) -> (sqrt x, 1/(2 sqrt x))
  g = fma(g, e, g);
  h = fma(h, e, h);
  e = fma(-g, h, 0.5);
  g = fma(g, e, g);
  h = fma(h, e, h);
  return fma(fma(-g, g, x), h, g);
}

// sin / cos of t * pi / 4 for t in [0, 2]: x = (t - 1) * pi / 4 lies in
// [-pi/4, pi/4], where Taylor series to x^17 / x^18 are below 1e-18; then
// sin(pi/4 + x) = (sin x + cos x) / sqrt 2, cos(pi/4 + x) = (cos x - sin x) / sqrt 2.
// About 25 fp64 operations against ~60 instructions for sincospi, within
// 2 ulp of the exact values.
__device__ __forceinline__ void sincos_quarter_turn(double t, double* so, double* co) {
  const double x = (t - 1.0) * c_k[20];  // pi / 4
  const double x2 = x * x;
  double sp = c_k[3];                  // 1/17!
  sp = fma(sp, -x2, c_k[4]);           // 1/15!
  sp = fma(sp, -x2, c_k[5]);           // 1/13!
  sp = fma(sp, -x2, c_k[6]);           // 1/11!
  sp = fma(sp, -x2, c_k[7]);           // 1/9!
  sp = fma(sp, -x2, c_k[8]);           // 1/7!
  sp = fma(sp, -x2, c_k[9]);           // 1/5!
  sp = fma(sp, -x2, c_k[10]);          // 1/3!
  const double sx = fma(-x * x2, sp, x);
  double cp = c_k[11];                 // 1/18!
  cp = fma(cp, -x2, c_k[12]);          // 1/16!
  cp = fma(cp, -x2, c_k[13]);          // 1/14!
  cp = fma(cp, -x2, c_k[14]);          // 1/12!
  cp = fma(cp, -x2, c_k[15]);          // 1/10!
  cp = fma(cp, -x2, c_k[16]);          // 1/8!
  cp = fma(cp, -x2, c_k[17]);          // 1/6!
  cp = fma(cp, -x2, c_k[18]);          // 1/4!
  cp = fma(cp, -x2, c_k[19]);          // 1/2
  const double cx = fma(-x2, cp, 1.0);
  const double r2 = c_k[21];           // sqrt(1/2)
  *so = (sx + cx) * r2;
  *co = (cx - sx) * r2;
}

// Field-cell flavour of the numpy map: the same a, b, r and phi, with
// sin/cos from sincos_quarter_turn and without the final renormalisation (the vector is
// unit length analytically: rho^2 + z^2 = r^2 (2 - r^2) + (1 - r^2)^2 = 1;
// the numpy division changes it by an ulp or two).  Directions agree with
// octa_uv_to_dir_np to a few ulp — within the fields' 1e-9 tolerance — at
// one division instead of four and no general-argument sincos.
__device__ __forceinline__ void octa_uv_to_dir_cell(double u, double v, double* ox, double* oy,
                                                    double* oz) {
  // 2u is exact, so fma(2, u, -1) is the numpy 2u - 1 to the bit
  double a = __fma_rn(2.0, u, -1.0);
  double b = __fma_rn(2.0, v, -1.0);
  double ap = fabs(a), bp = fabs(b);
  double sd = __dsub_rn(1.0, __dadd_rn(ap, bp));
  double r = __dsub_rn(1.0, fabs(sd));
  double t = (r == 0.0) ? 1.0 : fast_div(bp - ap, r) + 1.0;  // phi / (pi/4)
  double rr = __dmul_rn(r, r);
  // r = 1 - |1 - (|a| + |b|)| is in [0, 1] for u, v in [0, 1], so
  // 2 - r^2 is in [1, 2] (no clamp needed)
  double rho = r * fast_sqrt(2.0 - rr);
  double s, c;
  sincos_quarter_turn(t, &s, &c);
  *ox = __dmul_rn(copysign(c, a), rho);
  *oy = __dmul_rn(copysign(s, b), rho);
  *oz = copysign(__dsub_rn(1.0, rr), sd);
}

// compiled flavour (_kernels.pyx:240-262): used by the guided sampler.
__device__ __forceinline__ void octa_uv_to_dir_k(double u, double v, double* ox, double* oy,
                                                 double* oz) {
  double a = 2.0 * u - 1.0;
  double b = 2.0 * v - 1.0;
  double ap = fabs(a), bp = fabs(b);
  double sd = 1.0 - (ap + bp);
  double d = fabs(sd);
  double r = 1.0 - d;
  double phi = (r == 0.0) ? 1.0 : (bp - ap) / r + 1.0;
  phi *= WFPG_PI / 4.0;
  double z = copysign(1.0 - r * r, sd);
  double rho = r * sqrt(fmax(2.0 - r * r, 0.0));
  double s, c;
  sincos(phi, &s, &c);
  double x = copysign(c, a) * rho;
  double y = copysign(s, b) * rho;
  double inv = 1.0 / sqrt(x * x + y * y + z * z);
  *ox = x * inv;
  *oy = y * inv;
  *oz = z * inv;
}

// _kernels.pyx:265-298
__device__ __forceinline__ void octa_dir_to_uv_k(double dx, double dy, double dz, double* ou,
                                                 double* ov) {
  double x = fabs(dx), y = fabs(dy);
  double r = sqrt(fmax(1.0 - fabs(dz), 0.0));
  double hi = fmax(x, y), lo = fmin(x, y);
  double ratio = hi > 0.0 ? lo / hi : 0.0;
  double phi = atan(ratio) * (2.0 / WFPG_PI);
  if (x < y) phi = 1.0 - phi;
  double vq = phi * r;
  double uq = r - vq;
  if (dz < 0.0) {
    double t = uq;
    uq = 1.0 - vq;
    vq = 1.0 - t;
  }
  uq = copysign(uq, dx);
  vq = copysign(vq, dy);
  double u = 0.5 * (uq + 1.0), v = 0.5 * (vq + 1.0);
  u = fmin(fmax(u, 0.0), 1.0 - 1e-12);
  v = fmin(fmax(v, 0.0), 1.0 - 1e-12);
  *ou = u;
  *ov = v;
}

// ---------------------------------------------------------------------------
// SVO descent: _kernels.pyx:591-621 (compiled quantisation formula)
// ---------------------------------------------------------------------------
struct SvoView {
  const uint2* desc;   // {child_base, child_mask}
  const uint2* top;    // dense top-level index (optional), see wfpg_svo.top_index
  int32_t top_level;
  const int32_t* parent;
  const double* normal;
  const double* mean_a;
  const double* mean_b;
  double lox, loy, loz, size;
  double scale;        // resolution / size
  double nudge;        // (size / resolution) * 1e-3 (_kernels.pyx:676)
  float half_log2_s0;     // 0.5 log2(size^2): best_cone_level's estimate (fp32)
  int32_t resolution, depth;
};

__host__ inline SvoView make_view(const wfpg_svo* s) {
  SvoView v;
  v.desc = reinterpret_cast<const uint2*>(s->node_desc);
  v.top = s->top_level > 0 && s->top_level <= s->depth ? reinterpret_cast<const uint2*>(s->top_index)
                                                       : nullptr;
  v.top_level = v.top ? s->top_level : 0;
  v.parent = s->parent;
  v.normal = s->normal;
  v.mean_a = s->mean_a;
  v.mean_b = s->mean_b;
  v.lox = s->lo[0];
  v.loy = s->lo[1];
  v.loz = s->lo[2];
  v.size = s->size;
  v.scale = (double)s->resolution / s->size;
  v.nudge = (s->size / s->resolution) * 1e-3;
  v.half_log2_s0 = 0.5f * log2f((float)(s->size * s->size));
  v.resolution = s->resolution;
  v.depth = s->depth;
  return v;
}

__device__ __forceinline__ int32_t quantise(double p, double lo, double scale, int32_t res) {
  double q = __dmul_rn(__dsub_rn(p, lo), scale);
  // (long) truncation toward zero, then clamp to [0, res - 1]
  // (_kernels.pyx:594-606).  The saturating 32-bit conversion gives the same
  // clamped cell for every q: out-of-range values saturate to the side they
  // clamp to anyway, NaN converts to 0 as the 64-bit path did.
  return min(max(__double2int_rz(q), 0), res - 1);
}

// Descend toward leaf coords (qx,qy,qz) through at most `max_level` levels.
// Returns the deepest materialised node; *present = reached max_level.
__device__ __forceinline__ int32_t descend_coords(const uint2* __restrict__ desc, int32_t depth,
                                                  int32_t qx, int32_t qy, int32_t qz,
                                                  int32_t max_level, bool* present,
                                                  int32_t* reached_level, int32_t start_node = 0,
                                                  int32_t start_level = 0) {
  int32_t node = start_node;
  int32_t lvl = start_level;
  bool pres = true;
  for (int32_t level = start_level + 1; level <= max_level; ++level) {
    int sh = depth - level;
    int oct = ((qx >> sh) & 1) | (((qy >> sh) & 1) << 1) | (((qz >> sh) & 1) << 2);
    uint2 d = __ldg(&desc[node]);
    uint32_t mask = d.y;
    if (!((mask >> oct) & 1u)) {
      pres = false;
      break;
    }
    node = (int32_t)d.x + __popc(mask & ((1u << oct) - 1u));
    lvl = level;
  }
  *present = pres;
  *reached_level = lvl;
  return node;
}

// Descent through an SvoView: with a top index, the first top_level levels
// are one load (row-major cell at that level); identical results.
__device__ __forceinline__ int32_t descend_view(const SvoView& v, int32_t qx, int32_t qy,
                                                int32_t qz, int32_t max_level, bool* present,
                                                int32_t* reached_level) {
  if (v.top && max_level >= v.top_level - 2) {
    const int T = v.top_level, sh = v.depth - T;
    const uint32_t cell = ((uint32_t)(qx >> sh) << (2 * T)) | ((uint32_t)(qy >> sh) << T) |
                          (uint32_t)(qz >> sh);
    const uint2 e = __ldg(&v.top[cell]);
    const int32_t lv = (int32_t)(e.y & 0xFFu);  // deepest materialised level <= T
    if (max_level <= lv) {
      // shallower target: its node is an ancestor of the indexed one (one
      // or two parent links instead of a descent from the root)
      int32_t node = (int32_t)e.x;
      for (int l = lv; l > max_level; --l) node = __ldg(&v.parent[node]);
      *present = true;
      *reached_level = max_level;
      return node;
    }
    if (!(e.y >> 31)) {
      *present = false;
      *reached_level = lv;
      return (int32_t)e.x;
    }
    return descend_coords(v.desc, v.depth, qx, qy, qz, max_level, present, reached_level,
                          (int32_t)e.x, T);
  }
  return descend_coords(v.desc, v.depth, qx, qy, qz, max_level, present, reached_level);
}

// ---------------------------------------------------------------------------
// Warp / block helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int BLOCK>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem_warp,
                                                         uint32_t* total) {
  // smem_warp: BLOCK/32 + 1 entries
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = BLOCK / 32;
    uint32_t w = lane < NW ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) smem_warp[lane] = w;  // inclusive
    if (lane == NW - 1) smem_warp[NW] = w;
  }
  __syncthreads();
  uint32_t base = warp > 0 ? smem_warp[warp - 1] : 0;
  uint32_t res = base + x - v;
  if (total) *total = smem_warp[BLOCK / 32];
  __syncthreads();
  return res;
}

}  // namespace wfpg

// Cone query device function + internal SVO entry points.
#pragma once
#include "geometry.cuh"

namespace wfpg {

// Footprint-matched level (trace_one, _kernels.pyx:685-702): the level lv in
// [0, depth] minimising |side_lv^2 - area| with deeper levels winning ties.
// Because side_lv^2 is an exact power-of-4 scaling of side_0^2, the error is
// unimodal in lv, so the level chosen over the materialised chain [0, L] of
// the reference equals min(L, best) with best taken over [0, depth]; the
// descent can therefore stop at `best` instead of walking to the leaf.
// (size / 2^lv)^2 == round(size * size) * 4^-lv exactly (power-of-two scaling
// commutes with rounding), so the per-level squares come from one product and
// exact multiplications by 4 — same bits as the reference's divisions.
__device__ __forceinline__ int best_cone_level(double size, int depth, double area,
                                               float half_log2_s0) {
  // The error |s0 * 4^-lv - area| falls while s0 * 4^-lv >= area and rises
  // after, so the integer optimum is floor or ceil of x = log4(s0 / area).
  // An fp32 estimate of x (error far below 1) brackets it; the candidates
  // are then compared exactly, deepest first with strict '<' (deeper wins
  // ties), which is what the level-by-level scan from the leaf level returns.
  const double s0 = size * size;
  // 0.5 log2(s0) comes with the view; log2(area) by the flush-to-zero MUFU
  // (area = t^2 omega with t > tmin is never subnormal; if it were, the
  // estimate would clamp to the deepest level, which is then the answer)
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"((float)area));
  const float x = half_log2_s0 - 0.5f * lg;
  const float xc = fminf(fmaxf(x, -4.0f), 64.0f);
  const int c = (int)floorf(xc);
  // the integer optimum is floor or ceil of the exact x; the estimate is
  // within ~1e-5 of it (fp32 conversions + __log2f), so away from integers
  // floor(estimate) = floor(x) and two candidates suffice
  const float fr = xc - (float)c;
  const bool safe = fr > 1e-4f && fr < 1.0f - 1e-4f;
  const int lo = min(max(safe ? c : c - 1, 0), depth), hi = min(max(safe ? c + 1 : c + 2, 0), depth);
  // exact power-of-two scaling: s0 * 2^(-2 lv)
  auto err = [&](int lv) {
    return fabs(__dmul_rn(s0, __longlong_as_double((long long)(1023 - 2 * lv) << 52)) - area);
  };
  int best = hi;
  double bd = err(hi);
  if (safe) {  // hi - lo <= 1: one more candidate, no loop
    if (lo < hi && err(lo) < bd) best = lo;
    return best;
  }
  for (int lv = hi - 1; lv >= lo; --lv) {
    const double diff = err(lv);
    if (diff < bd) {
      bd = diff;
      best = lv;
    }
  }
  return best;
}

// Shade a hit point for a cone of solid angle omega: nudge toward the apex,
// clamp into the cube, descend to the footprint level, return the exitance of
// the side facing the cone scaled by |d.n| (_kernels.pyx:673-713).
__device__ __forceinline__ void cone_shade_hit(const SvoView& v, double ox, double oy, double oz,
                                               double dx, double dy, double dz, double r,
                                               double omega, double* rgb) {
  const double nudge = v.nudge;  // (size / resolution) * 1e-3, precomputed on the host
  double qx = ox + r * dx - dx * nudge;
  double qy = oy + r * dy - dy * nudge;
  double qz = oz + r * dz - dz * nudge;
  // The reference clamps q into [lo + tiny, lo + size - tiny] and truncates
  // (q - lo) * scale, which lands in [0, R - 1] (tiny * scale = R 1e-12).
  // Truncation is monotone, so clamping the cell index instead is the same
  // cell for every q: below lo + tiny the index is <= 0, above
  // lo + size - tiny it is >= R - 1 (saturating conversion; NaN -> 0, as the
  // clamp's fmax(NaN, lo + tiny) gives cell 0).  Integer min / max instead
  // of six fp64 min / max (no DMNMX: compare + two selects each).
  const int32_t rm = v.resolution - 1;
  int32_t ix = min(max(__double2int_rz(__dmul_rn(__dsub_rn(qx, v.lox), v.scale)), 0), rm);
  int32_t iy = min(max(__double2int_rz(__dmul_rn(__dsub_rn(qy, v.loy), v.scale)), 0), rm);
  int32_t iz = min(max(__double2int_rz(__dmul_rn(__dsub_rn(qz, v.loz), v.scale)), 0), rm);
  int target = best_cone_level(v.size, v.depth, r * r * omega, v.half_log2_s0);
  bool pres;
  int32_t lvl;
  int32_t node = descend_view(v, ix, iy, iz, target, &pres, &lvl);
  const double* nn = v.normal + 3 * (int64_t)node;
  double da = dx * __ldg(nn) + dy * __ldg(nn + 1) + dz * __ldg(nn + 2);
  double w = fabs(da);
  const double* m = (da <= 0.0 ? v.mean_a : v.mean_b) + 3 * (int64_t)node;
  rgb[0] = __ldg(m) * w;
  rgb[1] = __ldg(m + 1) * w;
  rgb[2] = __ldg(m + 2) * w;
}

__device__ __forceinline__ void cone_query(const SceneView& s, const TriRec* smt, const SvoView& v,
                                           double ox, double oy, double oz, double dx, double dy,
                                           double dz, double omega, double* rgb) {
  rgb[0] = rgb[1] = rgb[2] = 0.0;
  double bt;
  int32_t btri;
  ray_nearest(s, smt, ox, oy, oz, dx, dy, dz, s.ray_eps, &bt, &btri);
  if (btri < 0) return;
  cone_shade_hit(v, ox, oy, oz, dx, dy, dz, bt, omega, rgb);
}

size_t accumulate_ws_bytes(int64_t n);
int svo_accumulate(wfpg_svo* svo, const int32_t* leaf, const double* dirs, const double* rad,
                   int64_t n, const int32_t* n_dev, int deterministic, Arena& ws,
                   cudaStream_t st);
int svo_propagate(wfpg_svo* svo, cudaStream_t st);
int svo_propagate_dirty(wfpg_svo* svo, const int32_t* leaf, int64_t n_max, const int32_t* n_dev,
                        uint8_t* dirty, cudaStream_t st);
int svo_apply_leaf_acc(wfpg_svo* svo, const double* acc, cudaStream_t st);
wfpg_svo leaf_acc_view(const wfpg_svo* svo, double* acc);

}  // namespace wfpg

// Ray casting device functions: brute-force nearest hit over a shared-memory
// triangle pack (wfpg_brute_nearest, _kernels.pyx:40-97) and the BVH
// traversals (bvh_nearest / bvh_occluded / tri_hit / box_near / box_hit,
// _kernels.pyx:319-478).  Same acceptance tests and tie rules as the
// reference: brute force keeps the minimum t with the lowest triangle id on
// ties; BVH traversal visits children nearest-first with the same stacks.
// Box tests run in fp32 on padded boxes (triangle boxes for the brute-force
// prefilter, bvh_box_f32 node boxes when present) — the padding dwarfs fp32
// rounding, so they only skip work; every accepted hit is the fp64 test's.
#pragma once
#include "common.cuh"

namespace wfpg {

struct SceneView {
  const double* v0;
  const double* e1;
  const double* e2;
  const double* normals;
  const int32_t* tri_mat;
  const int32_t* mat_kind;
  const double* mat_rgb;
  const double* em_cdf;
  const int32_t* em_tris;
  int32_t n_emit;
  double em_area;
  double ray_eps;
  int32_t n_tris;
  int32_t brute;
  const double* blo;
  const double* bhi;
  const int32_t* bleft;
  const int32_t* bright;
  const int32_t* bcount;
  const int32_t* border;
  const float4* bbox32;  // optional (N,2) padded fp32 node boxes
};

inline SceneView make_scene_view(const wfpg_scene* s) {
  SceneView v;
  v.v0 = s->v0;
  v.e1 = s->e1;
  v.e2 = s->e2;
  v.normals = s->normals;
  v.tri_mat = s->tri_mat;
  v.mat_kind = s->mat_kind;
  v.mat_rgb = s->mat_rgb;
  v.em_cdf = s->emitter_cdf;
  v.em_tris = s->emitter_tris;
  v.n_emit = s->n_emit;
  v.em_area = s->emitter_area;
  v.ray_eps = s->ray_eps;
  v.n_tris = s->n_tris;
  v.brute = s->brute;
  v.blo = s->bvh_lo;
  v.bhi = s->bvh_hi;
  v.bleft = s->bvh_left;
  v.bright = s->bvh_right;
  v.bcount = s->bvh_count;
  v.border = s->bvh_order;
  v.bbox32 = reinterpret_cast<const float4*>(s->bvh_box_f32);
  return v;
}

// Triangle record in shared memory: the fp64 vertex / edges plus an fp32
// bounding box padded by 1e-5 of the scene diagonal and 4e-7 of the largest
// coordinate (far above the fp32 rounding of ray origins, directions and slab
// distances), used to skip the exact test for rays that miss the box within
// the current [tmin, best] range.  Skipped triangles provably cannot be hit
// there, so results equal brute force over all triangles.
struct TriRec {
  double v0x, v0y, v0z, e1x, e1y, e1z, e2x, e2y, e2z;
  float blo[3], bhi[3];
};

// Per-ray fp32 slab setup for the box prefilter: reciprocal direction and
// origin * reciprocal, so a slab distance (b - o) / d is one FFMA,
// b * (1/d) - o * (1/d).  Its rounding (a few ulp of o / d) stays far inside
// the box padding (4e-7 of the largest coordinate), as the subtract-multiply
// form's did.
struct RaySlab {
  float ix, iy, iz, oix, oiy, oiz;
};

__device__ __forceinline__ RaySlab make_ray_slab(double ox, double oy, double oz, double dx,
                                                 double dy, double dz) {
  auto inv = [](double d) {
    float f = (float)d;
    if (fabsf(f) < 1e-30f) f = copysignf(1e-30f, f);
    return 1.0f / f;
  };
  const float ix = inv(dx), iy = inv(dy), iz = inv(dz);
  return RaySlab{ix, iy, iz, (float)ox * ix, (float)oy * iy, (float)oz * iz};
}

// may the ray meet the (padded) box at a parameter in [lo, hi]?
__device__ __forceinline__ bool slab_maybe(const RaySlab& r, const float* blo, const float* bhi,
                                           float lo, float hi) {
  float t0 = fmaf(blo[0], r.ix, -r.oix), t1 = fmaf(bhi[0], r.ix, -r.oix);
  float tn = fminf(t0, t1), tf = fmaxf(t0, t1);
  t0 = fmaf(blo[1], r.iy, -r.oiy);
  t1 = fmaf(bhi[1], r.iy, -r.oiy);
  tn = fmaxf(tn, fminf(t0, t1));
  tf = fminf(tf, fmaxf(t0, t1));
  t0 = fmaf(blo[2], r.iz, -r.oiz);
  t1 = fmaf(bhi[2], r.iz, -r.oiz);
  tn = fmaxf(tn, fminf(t0, t1));
  tf = fminf(tf, fmaxf(t0, t1));
  return (tn <= tf) & (tn <= hi) & (tf >= lo);
}

constexpr int kMaxBruteTris = 512;
constexpr int kBoxPrefilterMinTris = 48;

// Cooperative load of the triangle pack into shared memory.
__device__ __forceinline__ void load_tris_smem(const SceneView& s, TriRec* sm) {
  for (int t = threadIdx.x; t < s.n_tris; t += blockDim.x) {
    TriRec r;
    r.v0x = s.v0[3 * t];
    r.v0y = s.v0[3 * t + 1];
    r.v0z = s.v0[3 * t + 2];
    r.e1x = s.e1[3 * t];
    r.e1y = s.e1[3 * t + 1];
    r.e1z = s.e1[3 * t + 2];
    r.e2x = s.e2[3 * t];
    r.e2y = s.e2[3 * t + 1];
    r.e2z = s.e2[3 * t + 2];
    const double v[3] = {r.v0x, r.v0y, r.v0z}, a[3] = {r.e1x, r.e1y, r.e1z},
                 b[3] = {r.e2x, r.e2y, r.e2z};
    for (int c = 0; c < 3; ++c) {
      const double lo = fmin(v[c], fmin(v[c] + a[c], v[c] + b[c]));
      const double hi = fmax(v[c], fmax(v[c] + a[c], v[c] + b[c]));
      const double pad = 0.1 * s.ray_eps + 4e-7 * fmax(fabs(lo), fabs(hi));
      r.blo[c] = __double2float_rd(lo - pad);
      r.bhi[c] = __double2float_ru(hi + pad);
    }
    sm[t] = r;
  }
}

// _kernels.pyx:63-81 for one triangle.  Returns t (>0) when accepted, else -1.
__device__ __forceinline__ double mt_brute(const TriRec& T, double ox, double oy, double oz,
                                           double dx, double dy, double dz, double tmin) {
  double px = dy * T.e2z - dz * T.e2y;
  double py = dz * T.e2x - dx * T.e2z;
  double pz = dx * T.e2y - dy * T.e2x;
  double det = T.e1x * px + T.e1y * py + T.e1z * pz;
  double s = det > 0.0 ? 1.0 : -1.0;
  double ad = det * s;
  double tx = ox - T.v0x, ty = oy - T.v0y, tz = oz - T.v0z;
  double us = (tx * px + ty * py + tz * pz) * s;
  double qx = ty * T.e1z - tz * T.e1y;
  double qy = tz * T.e1x - tx * T.e1z;
  double qz = tx * T.e1y - ty * T.e1x;
  double vs = (dx * qx + dy * qy + dz * qz) * s;
  double ts = (T.e2x * qx + T.e2y * qy + T.e2z * qz) * s;
  bool ok = (ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) & (ts > tmin * ad);
  return ok ? ts / ad : -1.0;
}

__device__ __forceinline__ void brute_nearest(const TriRec* __restrict__ tris, int n, double ox,
                                              double oy, double oz, double dx, double dy,
                                              double dz, double tmin, double* bt, int32_t* bid) {
  double best = 1e300;
  int32_t id = -1;
  const RaySlab rs = make_ray_slab(ox, oy, oz, dx, dy, dz);
  const float lo = (float)tmin * 0.99999f;
  float hi = 3.0e38f;
  for (int t = 0; t < n; ++t) {
    const TriRec& T = tris[t];
    // the box prefilter pays off from a few dozen triangles on (measured:
    // 68-triangle C3 +3.5 % with it, 36-triangle Cornell +0.4 % and random
    // C5 cones +8 % without); same hits either way
    if (n > kBoxPrefilterMinTris && !slab_maybe(rs, T.blo, T.bhi, lo, hi)) continue;
    // mt_brute's test; the division only on accepting lanes (it used to be
    // evaluated for every candidate and selected away)
    double px = dy * T.e2z - dz * T.e2y;
    double py = dz * T.e2x - dx * T.e2z;
    double pz = dx * T.e2y - dy * T.e2x;
    double det = T.e1x * px + T.e1y * py + T.e1z * pz;
    double sg = det > 0.0 ? 1.0 : -1.0;
    double ad = det * sg;
    double tx = ox - T.v0x, ty = oy - T.v0y, tz = oz - T.v0z;
    double us = (tx * px + ty * py + tz * pz) * sg;
    double qx = ty * T.e1z - tz * T.e1y;
    double qy = tz * T.e1x - tx * T.e1z;
    double qz = tx * T.e1y - ty * T.e1x;
    double vs = (dx * qx + dy * qy + dz * qz) * sg;
    double ts = (T.e2x * qx + T.e2y * qy + T.e2z * qz) * sg;
    if ((ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) & (ts > tmin * ad)) {
      const double h = ts / ad;  // > tmin > 0
      if (h < best) {
        best = h;
        id = t;
        hi = __double2float_ru(h) * 1.00001f;
      }
    }
  }
  *bt = best;
  *bid = id;
}

// _kernels.pyx:339-372
__device__ __forceinline__ double tri_hit(const double* v0, const double* e1, const double* e2,
                                          double ox, double oy, double oz, double dx, double dy,
                                          double dz, double tmin, double tmax) {
  double px = dy * e2[2] - dz * e2[1];
  double py = dz * e2[0] - dx * e2[2];
  double pz = dx * e2[1] - dy * e2[0];
  double det = e1[0] * px + e1[1] * py + e1[2] * pz;
  double ad = fabs(det);
  if (ad <= 1e-300) return -1.0;
  double s = det > 0.0 ? 1.0 : -1.0;
  double tx = ox - v0[0], ty = oy - v0[1], tz = oz - v0[2];
  double us = (tx * px + ty * py + tz * pz) * s;
  if (us < 0.0 || us > ad) return -1.0;
  double qx = ty * e1[2] - tz * e1[1];
  double qy = tz * e1[0] - tx * e1[2];
  double qz = tx * e1[1] - ty * e1[0];
  double vs = (dx * qx + dy * qy + dz * qz) * s;
  if (vs < 0.0 || us + vs > ad) return -1.0;
  double ts = (e2[0] * qx + e2[1] * qy + e2[2] * qz) * s;
  if (ts > tmin * ad && ts < tmax * ad) return ts / ad;
  return -1.0;
}

// tri_hit with every early return folded into one acceptance test (the
// same conditions on the same values: us <= ad follows from us + vs <= ad
// with vs >= 0 under monotone rounding), so the lanes of a packet stay
// converged; the division runs on accepting lanes only.
__device__ __forceinline__ double tri_hit_nb(const double* v0, const double* e1,
                                             const double* e2, double ox, double oy, double oz,
                                             double dx, double dy, double dz, double tmin,
                                             double tmax) {
  const double e2x = __ldg(e2), e2y = __ldg(e2 + 1), e2z = __ldg(e2 + 2);
  const double e1x = __ldg(e1), e1y = __ldg(e1 + 1), e1z = __ldg(e1 + 2);
  const double tx = ox - __ldg(v0), ty = oy - __ldg(v0 + 1), tz = oz - __ldg(v0 + 2);
  double px = dy * e2z - dz * e2y;
  double py = dz * e2x - dx * e2z;
  double pz = dx * e2y - dy * e2x;
  double det = e1x * px + e1y * py + e1z * pz;
  double ad = fabs(det);
  double s = det > 0.0 ? 1.0 : -1.0;
  double us = (tx * px + ty * py + tz * pz) * s;
  double qx = ty * e1z - tz * e1y;
  double qy = tz * e1x - tx * e1z;
  double qz = tx * e1y - ty * e1x;
  double vs = (dx * qx + dy * qy + dz * qz) * s;
  double ts = (e2x * qx + e2y * qy + e2z * qz) * s;
  const bool ok = (ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) &
                  (ts > tmin * ad) & (ts < tmax * ad);
  return ok ? ts / ad : -1.0;
}

__device__ __forceinline__ void slab(const double* lo, const double* hi, double ox, double oy,
                                     double oz, double ix, double iy, double iz, double* tn,
                                     double* tf) {
  double t0 = (lo[0] - ox) * ix, t1 = (hi[0] - ox) * ix;
  double n = fmin(t0, t1), f = fmax(t0, t1);
  t0 = (lo[1] - oy) * iy;
  t1 = (hi[1] - oy) * iy;
  n = fmax(n, fmin(t0, t1));
  f = fmin(f, fmax(t0, t1));
  t0 = (lo[2] - oz) * iz;
  t1 = (hi[2] - oz) * iz;
  n = fmax(n, fmin(t0, t1));
  f = fmin(f, fmax(t0, t1));
  *tn = n;
  *tf = f;
}

// fp32 slab against a padded node box: (near, far) with the far side
// rounded up by 1e-6 so it stays conservative
__device__ __forceinline__ void slab32(const float4* box, const RaySlab& r, float* tn,
                                       float* tf) {
  const float4 lo = __ldg(box), hi = __ldg(box + 1);
  float t0 = fmaf(lo.x, r.ix, -r.oix), t1 = fmaf(hi.x, r.ix, -r.oix);
  float n = fminf(t0, t1), f = fmaxf(t0, t1);
  t0 = fmaf(lo.y, r.iy, -r.oiy);
  t1 = fmaf(hi.y, r.iy, -r.oiy);
  n = fmaxf(n, fminf(t0, t1));
  f = fminf(f, fmaxf(t0, t1));
  t0 = fmaf(lo.z, r.iz, -r.oiz);
  t1 = fmaf(hi.z, r.iz, -r.oiz);
  n = fmaxf(n, fminf(t0, t1));
  f = fminf(f, fmaxf(t0, t1));
  *tn = n;
  *tf = f;
}

// _kernels.pyx:398-445
__device__ __forceinline__ void bvh_nearest(const SceneView& b, double ox, double oy, double oz,
                                            double dx, double dy, double dz, double tmin,
                                            double* best_t, int32_t* best_tri) {
  int32_t stack[64];
  float dstack[64];  // entry distances rounded down: the skip test stays conservative
  double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
  const RaySlab rs = make_ray_slab(ox, oy, oz, dx, dy, dz);
  double bt = 1e300;
  int32_t bid = -1;
  stack[0] = 0;
  dstack[0] = 0.0f;
  int sp = 1;
  while (sp > 0) {
    --sp;
    if ((double)dstack[sp] >= bt) continue;
    int32_t node = stack[sp];
    int32_t cnt = b.bcount[node];
    if (cnt > 0) {
      int32_t first = b.bleft[node];
      for (int32_t k = first; k < first + cnt; ++k) {
        int32_t tri = b.border[k];
        double t = tri_hit(b.v0 + 3 * tri, b.e1 + 3 * tri, b.e2 + 3 * tri, ox, oy, oz, dx, dy, dz,
                           tmin, bt);
        if (t > 0.0) {
          bt = t;
          bid = tri;
        }
      }
    } else {
      int32_t c0 = b.bleft[node], c1 = b.bright[node];
      double n0, f0, n1, f1;
      if (b.bbox32) {  // padded fp32 boxes: conservative entry / exit distances
        float a0, a1, e0, e1;
        slab32(b.bbox32 + 2 * c0, rs, &a0, &e0);
        slab32(b.bbox32 + 2 * c1, rs, &a1, &e1);
        n0 = a0;
        n1 = a1;
        f0 = (double)e0 * (1.0 + 1e-6);
        f1 = (double)e1 * (1.0 + 1e-6);
      } else {
        slab(b.blo + 3 * c0, b.bhi + 3 * c0, ox, oy, oz, ix, iy, iz, &n0, &f0);
        slab(b.blo + 3 * c1, b.bhi + 3 * c1, ox, oy, oz, ix, iy, iz, &n1, &f1);
      }
      double d0 = (f0 >= n0 && n0 <= bt && f0 >= tmin) ? n0 : 1e301;
      double d1 = (f1 >= n1 && n1 <= bt && f1 >= tmin) ? n1 : 1e301;
      if (d0 > d1) {
        int32_t tn = c0;
        c0 = c1;
        c1 = tn;
        double td = d0;
        d0 = d1;
        d1 = td;
      }
      if (d1 < 1e301 && sp < 64) {
        stack[sp] = c1;
        dstack[sp] = __double2float_rd(d1);
        ++sp;
      }
      if (d0 < 1e301 && sp < 64) {
        stack[sp] = c0;
        dstack[sp] = __double2float_rd(d0);
        ++sp;
      }
    }
  }
  *best_t = bt;
  *best_tri = bid;
}

// _kernels.pyx:448-478
__device__ __forceinline__ bool bvh_occluded(const SceneView& b, double ox, double oy, double oz,
                                             double dx, double dy, double dz, double tmin,
                                             double tmax) {
  int32_t stack[64];
  double ix = 1.0 / dx, iy = 1.0 / dy, iz = 1.0 / dz;
  const RaySlab rs = make_ray_slab(ox, oy, oz, dx, dy, dz);
  const float tmax32 = (float)tmax * (1.0f + 1e-6f), tmin32 = (float)tmin * (1.0f - 1e-6f);
  stack[0] = 0;
  int sp = 1;
  while (sp > 0) {
    --sp;
    int32_t node = stack[sp];
    if (b.bbox32) {
      float n, f;
      slab32(b.bbox32 + 2 * node, rs, &n, &f);
      if (!(f * (1.0f + 1e-6f) >= n && n <= tmax32 && f * (1.0f + 1e-6f) >= tmin32)) continue;
    } else {
      double n, f;
      slab(b.blo + 3 * node, b.bhi + 3 * node, ox, oy, oz, ix, iy, iz, &n, &f);
      if (!(f >= n && n <= tmax && f >= tmin)) continue;
    }
    int32_t cnt = b.bcount[node];
    if (cnt > 0) {
      int32_t first = b.bleft[node];
      for (int32_t k = first; k < first + cnt; ++k) {
        int32_t tri = b.border[k];
        if (tri_hit(b.v0 + 3 * tri, b.e1 + 3 * tri, b.e2 + 3 * tri, ox, oy, oz, dx, dy, dz, tmin,
                    tmax) > 0.0)
          return true;
      }
    } else if (sp + 2 <= 64) {
      stack[sp] = b.bleft[node];
      stack[sp + 1] = b.bright[node];
      sp += 2;
    }
  }
  return false;
}

// Per-(origin, triangle) record for rays that share one origin (all cones of a
// field bin).  With tvec = o - v0 fixed, the Moeller-Trumbore quantities of
// _kernels.pyx:63-81 are linear in the ray direction d:
//   det   = e1 . (d x e2) = d . (e2 x e1)      -> d . n
//   u det = tvec . (d x e2) = d . (e2 x tvec)  -> d . w
//   v det = d . (tvec x e1)                    -> d . q
//   t det = e2 . (tvec x e1)                   -> ts0 (constant)
// so each candidate costs three 3-term dot products.  The reassociation moves
// det / u / v by a few ulp against the reference's operand order, which only
// matters for rays within ~1e-16 of a triangle edge (field tolerance 1e-9).
struct __align__(16) TriBin {
  double nx, ny, nz, wx, wy, wz, qx, qy, qz, ts0;
  // unit normals of the three planes through o and an edge, oriented toward
  // the opposite vertex: the triangle's solid angle seen from o is the
  // intersection of their positive half-spaces, so each plane on its own
  // bounds it.  A degenerate plane (o on or near the triangle's plane / an
  // edge line) is stored as the zero vector, which every test passes.
  // (fp32: the cull carries a 1e-5 slack, far above their rounding)
  float n0x, n0y, n0z, n1x, n1y, n1z, n2x, n2y, n2z;
  // unit normal of the triangle's own plane; `flat` when o lies within
  // 1e-5 * tmin of that plane (bin origins are hit points on surfaces): a
  // ray can then only hit the triangle beyond tmin if it is within 1e-5 of
  // parallel to the plane, so tiles that stay away from that band skip it
  float pnx, pny, pnz;
  // 0 when `flat`, +inf otherwise: the grazing-band test is
  // |a.pn| <= graze + unflat
  float unflat;
};

// One third of a triangle's record: part e computes the edge plane through o
// and edge e (and, for e = 0, the Moeller-Trumbore terms), so three threads
// build a record.  Degenerate edge planes are left as zero vectors.
__device__ __forceinline__ void make_tri_bin_part(const SceneView& s, int t, int e, double ox,
                                                  double oy, double oz, TriBin& B) {
  const double* v0 = s.v0 + 3 * t;
  const double* e1 = s.e1 + 3 * t;
  const double* e2 = s.e2 + 3 * t;
  if (e == 0) {
    const double tx = ox - v0[0], ty = oy - v0[1], tz = oz - v0[2];
    B.nx = e2[1] * e1[2] - e2[2] * e1[1];
    B.ny = e2[2] * e1[0] - e2[0] * e1[2];
    B.nz = e2[0] * e1[1] - e2[1] * e1[0];
    B.wx = e2[1] * tz - e2[2] * ty;
    B.wy = e2[2] * tx - e2[0] * tz;
    B.wz = e2[0] * ty - e2[1] * tx;
    B.qx = ty * e1[2] - tz * e1[1];
    B.qy = tz * e1[0] - tx * e1[2];
    B.qz = tx * e1[1] - ty * e1[0];
    B.ts0 = e2[0] * B.qx + e2[1] * B.qy + e2[2] * B.qz;
    // |ts0| = |tvec . (e1 x e2)| = plane distance * |n|
    const double n2 = B.nx * B.nx + B.ny * B.ny + B.nz * B.nz;
    const double inl = rsqrt(n2);
    B.pnx = (float)(B.nx * inl);
    B.pny = (float)(B.ny * inl);
    B.pnz = (float)(B.nz * inl);
    const double fl = 1e-5 * s.ray_eps;
    B.unflat = B.ts0 * B.ts0 < fl * fl * n2 ? 0.0f : INFINITY;
  }
  // directions from o to the three vertices (unnormalised: the thresholds
  // below are the unit-vector tests |a^ x b^| > 1e-9 and |n^ . c^| >= 1e-9
  // restated on squared lengths, so no square roots or divisions)
  double w[3][3], l2[3];
  bool degenerate = false;
  const double dl = 1e-9 * s.ray_eps;
  for (int k = 0; k < 3; ++k) {
    w[k][0] = v0[0] + (k == 1 ? e1[0] : (k == 2 ? e2[0] : 0.0)) - ox;
    w[k][1] = v0[1] + (k == 1 ? e1[1] : (k == 2 ? e2[1] : 0.0)) - oy;
    w[k][2] = v0[2] + (k == 1 ? e1[2] : (k == 2 ? e2[2] : 0.0)) - oz;
    l2[k] = w[k][0] * w[k][0] + w[k][1] * w[k][1] + w[k][2] * w[k][2];
    if (!(l2[k] > dl * dl)) degenerate = true;
  }
  float* nb = &B.n0x + 3 * e;
  nb[0] = nb[1] = nb[2] = 0.0f;
  if (degenerate) return;
  // the plane through o and edge e, oriented toward the opposite vertex
  const int e1i = (e + 1) % 3, e2i = (e + 2) % 3;
  const double* a = w[e];
  const double* b = w[e1i];
  const double* c = w[e2i];
  double nx = a[1] * b[2] - a[2] * b[1];
  double ny = a[2] * b[0] - a[0] * b[2];
  double nz = a[0] * b[1] - a[1] * b[0];
  const double m2 = nx * nx + ny * ny + nz * nz;
  if (!(m2 > 1e-18 * l2[e] * l2[e1i])) return;
  const double side = nx * c[0] + ny * c[1] + nz * c[2];
  if (!(side * side >= 1e-18 * m2 * l2[e2i])) return;  // o (nearly) in the triangle's plane
  const double inv = side < 0.0 ? -rsqrt(m2) : rsqrt(m2);
  nx *= inv;
  ny *= inv;
  nz *= inv;
  nb[0] = (float)nx;
  nb[1] = (float)ny;
  nb[2] = (float)nz;
}

// Whole record by one thread.
__device__ __forceinline__ void make_tri_bin(const SceneView& s, int t, double ox, double oy,
                                             double oz, TriBin& B) {
  for (int e = 0; e < 3; ++e) make_tri_bin_part(s, t, e, ox, oy, oz, B);
}

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_min_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Nearest hit for the 32 rays of a warp that share one origin.  The warp
// bounds its own 32 directions by a cone (axis = the tile's centre lane,
// cos of the half-angle = smallest dot with the axis).  A cone of half-angle
// th around a reaches the positive side of a plane with unit normal n only
// if a.n >= -sin(th); a triangle one of whose three edge planes (TriBin) the
// whole cone misses cannot be hit by any lane.  Lanes vote on 32 triangles at
// a time and the warp then tests only the surviving candidates, in ascending
// triangle order with the strict '<' of the brute-force kernel, so the result
// (minimum t, lowest id on ties) is brute force over all triangles (the 1e-6
// slack dwarfs the rounding of both the cull and the hit test).
//
// SUB (small fields, where an 8x4-cell tile spans up to an eighth of the
// sphere and one bounding cone culls almost nothing): the same test against
// the four 4x2-cell quarter tiles' cones, a triangle being a candidate when
// any quarter's cone can reach it (a quarter cone's radius is half the whole
// tile's).  The quarter cones live in the warp's slot of a small shared
// table (at most kSubWarps warps per CTA).
constexpr int kSubWarps = 8;
// MUFU reciprocal square root without the subnormal-input fixup rsqrtf
// carries (four extra instructions): every argument below is a normal float
// (squared lengths of unit vectors, or clamped to >= 1e-30)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
template <bool LANE_TEST = false, bool SUB = false>
__device__ __forceinline__ void warp_nearest_bin(const TriBin* __restrict__ tb, int n, double dx,
                                                 double dy, double dz, double tmin, double* bt,
                                                 int32_t* bid) {
  const int lane = threadIdx.x & 31;
  // quarter tile of a lane (i = lane % 8, j = lane / 8): (i >= 4) + 2 (j >= 2)
  __shared__ float4 sub_cone[SUB ? kSubWarps : 1][4];  // axis, reach
  __shared__ float sub_graze[SUB ? kSubWarps : 1][4];
  if constexpr (SUB) {
    const int w = threadIdx.x >> 5;
    const int c = 10 | (lane & 0x14);  // (i, j) = (2, 1) of the lane's quarter
    const float sx = __shfl_sync(0xffffffffu, (float)dx, c);
    const float sy = __shfl_sync(0xffffffffu, (float)dy, c);
    const float sz = __shfl_sync(0xffffffffu, (float)dz, c);
    const float l2 = sx * sx + sy * sy + sz * sz;
    const float il = rsqrt_ftz(l2);
    const float fl = l2 * il;
    float cq = ((float)dx * sx + (float)dy * sy + (float)dz * sz) * il - 4e-6f;
    cq = fminf(cq, __shfl_xor_sync(0xffffffffu, cq, 1));
    cq = fminf(cq, __shfl_xor_sync(0xffffffffu, cq, 2));
    cq = fminf(cq, __shfl_xor_sync(0xffffffffu, cq, 8));
    const float s2 = fmaxf(1.0f - cq * cq, 1e-30f);
    const float g2 = fmaxf(2.0f - 2.0f * cq, 1e-30f);
    // a quarter that does not fit in a half-space reaches everything
    const float rch = cq > 0.0f ? -(s2 * rsqrt_ftz(s2) + 1e-5f) * fl : -INFINITY;
    const float grz = cq > 0.0f ? (g2 * rsqrt_ftz(g2) + 3e-5f) * fl : INFINITY;
    __syncwarp();
    if (lane == c) {
      const int q = ((lane >> 2) & 1) | ((lane >> 3) & 2);
      sub_cone[w][q] = make_float4(sx, sy, sz, rch);
      sub_graze[w][q] = grz;
    }
    __syncwarp();
  }
  // axis: the centre lane's direction, broadcast as floats (any common axis is
  // valid).  The tile bound and the plane tests are evaluated in fp32 and
  // widened by 4e-6 (cos) and 1e-5 (sin) — far above fp32 rounding (~1e-7)
  // — so the cull stays conservative.
  const float fax = __shfl_sync(0xffffffffu, (float)dx, 12);
  const float fay = __shfl_sync(0xffffffffu, (float)dy, 12);
  const float faz = __shfl_sync(0xffffffffu, (float)dz, 12);
  // (MUFU reciprocal square roots: their ~1e-7 relative error sits far
  // inside the slacks)
  const float fal2 = fax * fax + fay * fay + faz * faz;
  const float inv_fal = rsqrt_ftz(fal2);
  const float fal = fal2 * inv_fal;
  float cm = ((float)dx * fax + (float)dy * fay + (float)dz * faz) * inv_fal - 4e-6f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cm = fminf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
  const bool cull = cm > 0.0f;
  // -|a| (sin(th) + slack): a ray within th of the axis cannot reach the
  // inner side of a plane whose normal n has a.n below this
  const float s2 = fmaxf(1.0f - cm * cm, 1e-30f);
  const float reach = -(s2 * rsqrt_ftz(s2) + 1e-5f) * fal;
  // every ray of the tile is within 2 sin(th/2) = sqrt(2 - 2 cos th) of the
  // unit axis, so |d.n| >= |a.n| - that: tiles clear of a flat triangle's
  // grazing band (|d.n| <= 1e-5, plus fp32 slack) cannot hit it past tmin
  const float g2 = fmaxf(2.0f - 2.0f * cm, 1e-30f);
  const float graze = (g2 * rsqrt_ftz(g2) + 3e-5f) * fal;
  double best = 1e300;
  int32_t id = -1;
  for (int g = 0; g < n; g += 32) {
    const int t = g + lane;
    bool cand = t < n;
    if (SUB && cand) {
      const TriBin& B = tb[t];
      const int w = threadIdx.x >> 5;
      bool any = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 A = sub_cone[w][q];
        const float d0 = A.x * B.n0x + A.y * B.n0y + A.z * B.n0z;
        const float d1 = A.x * B.n1x + A.y * B.n1y + A.z * B.n1z;
        const float d2 = A.x * B.n2x + A.y * B.n2y + A.z * B.n2z;
        const float dp = fabsf(A.x * B.pnx + A.y * B.pny + A.z * B.pnz);
        const bool inside = (d0 >= A.w) & (d1 >= A.w) & (d2 >= A.w);
        any |= inside & (dp <= sub_graze[w][q] + B.unflat);
      }
      cand = any;
    } else if (cand && cull) {
      // branch-free per lane (each lane holds a different triangle)
      const TriBin& B = tb[t];
      const float d0 = fax * B.n0x + fay * B.n0y + faz * B.n0z;
      const float d1 = fax * B.n1x + fay * B.n1y + faz * B.n1z;
      const float d2 = fax * B.n2x + fay * B.n2y + faz * B.n2z;
      const float dp = fabsf(fax * B.pnx + fay * B.pny + faz * B.pnz);
      const bool inside = (d0 >= reach) & (d1 >= reach) & (d2 >= reach);
      cand = inside & (dp <= graze + B.unflat);
    }
    unsigned m = __ballot_sync(0xffffffffu, cand);
    while (m) {
      const int k = g + __ffs(m) - 1;
      m &= m - 1;
      const TriBin& B = tb[k];
      if (LANE_TEST) {
        // each lane's own direction against the three edge planes (fp32,
        // 1e-5 slack): a ray outside the triangle's solid angle cannot hit
        // it, so the warp skips the exact test when no lane is inside
        const float fx = (float)dx, fy = (float)dy, fz = (float)dz;
        const bool in = (fx * B.n0x + fy * B.n0y + fz * B.n0z >= -1e-5f) &
                        (fx * B.n1x + fy * B.n1y + fz * B.n1z >= -1e-5f) &
                        (fx * B.n2x + fy * B.n2y + fz * B.n2z >= -1e-5f);
        if (!__any_sync(0xffffffffu, in)) continue;
      }
      double det = dx * B.nx + dy * B.ny + dz * B.nz;
      double sg = det > 0.0 ? 1.0 : -1.0;
      double ad = det * sg;
      double us = (dx * B.wx + dy * B.wy + dz * B.wz) * sg;
      double vs = (dx * B.qx + dy * B.qy + dz * B.qz) * sg;
      double ts = B.ts0 * sg;
      bool ok = (ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) & (ts > tmin * ad);
      if (__any_sync(0xffffffffu, ok)) {  // the division only when some lane hits
        double h = fast_div(ts, ad);  // ad > 1e-300 on the lanes that use it
        if (ok && h < best) {
          best = h;
          id = k;
        }
      }
    }
  }
  *bt = best;
  *bid = id;
}

// Brute-force any-hit (wfpg_brute_occluded, _kernels.pyx:99-138).
__device__ __forceinline__ bool brute_occluded(const TriRec* __restrict__ tris, int n, double ox,
                                               double oy, double oz, double dx, double dy,
                                               double dz, double tmin, double tmax) {
  const RaySlab rs = make_ray_slab(ox, oy, oz, dx, dy, dz);
  const float lo = (float)tmin * 0.99999f, hi = __double2float_ru(tmax) * 1.00001f;
  for (int t = 0; t < n; ++t) {
    const TriRec& T = tris[t];
    if (!slab_maybe(rs, T.blo, T.bhi, lo, hi)) continue;
    double px = dy * T.e2z - dz * T.e2y;
    double py = dz * T.e2x - dx * T.e2z;
    double pz = dx * T.e2y - dy * T.e2x;
    double det = T.e1x * px + T.e1y * py + T.e1z * pz;
    double s = det > 0.0 ? 1.0 : -1.0;
    double ad = det * s;
    double tx = ox - T.v0x, ty = oy - T.v0y, tz = oz - T.v0z;
    double us = (tx * px + ty * py + tz * pz) * s;
    double qx = ty * T.e1z - tz * T.e1y;
    double qy = tz * T.e1x - tx * T.e1z;
    double qz = tx * T.e1y - ty * T.e1x;
    double vs = (dx * qx + dy * qy + dz * qz) * s;
    double ts = (T.e2x * qx + T.e2y * qy + T.e2z * qz) * s;
    if ((ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) & (ts > tmin * ad) &
        (ts < tmax * ad))
      return true;
  }
  return false;
}

// Warp-cooperative nearest hit over the BVH for the 32 rays of a warp that
// share one origin (a field tile, `bvh_nearest` of _kernels.pyx:398-445 for
// each lane).  The warp walks the tree as one packet: node ids, child order
// and the stack are warp-uniform, the stack (node, lane mask) lives in this
// warp's slice of shared memory, each lane slab-tests its own ray against the
// padded fp32 child boxes and the warp descends into a child when any lane
// reaches it before that lane's current best t.  A lane mask travels with
// every stack entry (lanes outside a node's padded box cannot hit anything
// below it) and is re-tested against the updated best t when the entry is
// popped.  Leaves run the reference's fp64 `tri_hit` per lane.  Every lane
// ends with the minimum accepted t over all triangles — the value the
// per-lane walk returns; only which of two triangles at a bit-identical t is
// reported can differ, and the field tracer uses the hit distance alone.
// Rays of a field tile span a few degrees, so the packet visits about the
// nodes one ray visits, without the per-lane divergence of 32 separate walks.
constexpr int kWarpBvhStack = 64;
// per-warp staging of a leaf's per-(origin, triangle) Moeller-Trumbore terms
// (the TriBin terms: n = e2 x e1, w = e2 x tvec, q = tvec x e1, ts0 = e2.q,
// plus the triangle id): kLeafStage records of kLeafRec doubles
constexpr int kLeafStage = 8, kLeafRec = 12;

__device__ __forceinline__ bool slab32_reach(const float4* box, const RaySlab& r, float lo,
                                             float hi) {
  float n, f;
  slab32(box, r, &n, &f);
  f *= 1.0f + 1e-6f;
  return (f >= n) & (n <= hi) & (f >= lo);
}

__device__ __forceinline__ void warp_bvh_nearest(const SceneView& b, int2* __restrict__ wstack,
                                                 double ox, double oy, double oz, double dx,
                                                 double dy, double dz, double tmin,
                                                 double* best_t, int32_t* best_tri,
                                                 double* __restrict__ wrec = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned me = 1u << lane;
  const RaySlab rs = make_ray_slab(ox, oy, oz, dx, dy, dz);
  const float lo = (float)tmin * (1.0f - 1e-6f);
  double bt = 1e300;
  float hi = __int_as_float(0x7f800000);  // fp32 bound of bt, rounded up
  int32_t bid = -1;
  int sp = 0;
  int32_t node = 0;
  unsigned mask = __ballot_sync(0xffffffffu, slab32_reach(b.bbox32, rs, lo, hi));
  while (mask) {
    const int32_t cnt = __ldg(&b.bcount[node]);
    const int32_t c0 = __ldg(&b.bleft[node]);
    if (cnt > 0 && wrec) {
      // the warp's rays share one origin (a field bin): lanes build the
      // leaf's direction-linear triangle terms once, then every lane in the
      // mask tests its own direction with three dot products per triangle
      for (int32_t k0 = 0; k0 < cnt; k0 += kLeafStage) {
        const int kn = cnt - k0 < kLeafStage ? cnt - k0 : kLeafStage;
        __syncwarp();
        if (lane < kn) {
          const int32_t tri = __ldg(&b.border[c0 + k0 + lane]);
          const double* v0 = b.v0 + 3 * tri;
          const double* e1 = b.e1 + 3 * tri;
          const double* e2 = b.e2 + 3 * tri;
          const double e1x = __ldg(e1), e1y = __ldg(e1 + 1), e1z = __ldg(e1 + 2);
          const double e2x = __ldg(e2), e2y = __ldg(e2 + 1), e2z = __ldg(e2 + 2);
          const double tx = ox - __ldg(v0), ty = oy - __ldg(v0 + 1), tz = oz - __ldg(v0 + 2);
          double* r = wrec + lane * kLeafRec;
          const double qx = ty * e1z - tz * e1y, qy = tz * e1x - tx * e1z, qz = tx * e1y - ty * e1x;
          r[0] = e2y * e1z - e2z * e1y;
          r[1] = e2z * e1x - e2x * e1z;
          r[2] = e2x * e1y - e2y * e1x;
          r[3] = e2y * tz - e2z * ty;
          r[4] = e2z * tx - e2x * tz;
          r[5] = e2x * ty - e2y * tx;
          r[6] = qx;
          r[7] = qy;
          r[8] = qz;
          r[9] = e2x * qx + e2y * qy + e2z * qz;
          r[10] = __longlong_as_double((long long)tri);
        }
        __syncwarp();
        if (mask & me) {
          for (int k = 0; k < kn; ++k) {
            const double* r = wrec + k * kLeafRec;
            const double det = dx * r[0] + dy * r[1] + dz * r[2];
            const double sg = det > 0.0 ? 1.0 : -1.0;
            const double ad = det * sg;
            const double us = (dx * r[3] + dy * r[4] + dz * r[5]) * sg;
            const double vs = (dx * r[6] + dy * r[7] + dz * r[8]) * sg;
            const double ts = r[9] * sg;
            if ((ad > 1e-300) & (us >= 0.0) & (vs >= 0.0) & (us + vs <= ad) &
                (ts > tmin * ad) & (ts < bt * ad)) {
              const double h = ts / ad;
              if (h < bt) {
                bt = h;
                bid = (int32_t)__double_as_longlong(r[10]);
              }
            }
          }
          hi = bt < 1e300 ? __double2float_ru(bt) * (1.0f + 1e-6f) : hi;
        }
      }
      mask = 0;
    } else if (cnt > 0) {
      if (mask & me) {
        for (int32_t k = c0; k < c0 + cnt; ++k) {
          const int32_t tri = __ldg(&b.border[k]);
          const double t = tri_hit_nb(b.v0 + 3 * tri, b.e1 + 3 * tri, b.e2 + 3 * tri, ox, oy, oz,
                                      dx, dy, dz, tmin, bt);
          if (t > 0.0) {
            bt = t;
            bid = tri;
          }
        }
        hi = bt < 1e300 ? __double2float_ru(bt) * (1.0f + 1e-6f) : hi;
      }
      mask = 0;
    } else {
      const int32_t c1 = __ldg(&b.bright[node]);
      float n0, f0, n1, f1;
      slab32(b.bbox32 + 2 * c0, rs, &n0, &f0);
      slab32(b.bbox32 + 2 * c1, rs, &n1, &f1);
      f0 *= 1.0f + 1e-6f;
      f1 *= 1.0f + 1e-6f;
      const bool in = (mask & me) != 0;
      const bool h0 = in & (f0 >= n0) & (n0 <= hi) & (f0 >= lo);
      const bool h1 = in & (f1 >= n1) & (n1 <= hi) & (f1 >= lo);
      const unsigned m0 = __ballot_sync(0xffffffffu, h0);
      const unsigned m1 = __ballot_sync(0xffffffffu, h1);
      if (m0 && m1) {
        // nearer child first: the majority vote of the lanes reaching both
        const unsigned both = m0 & m1;
        const unsigned pref1 = __ballot_sync(0xffffffffu, h0 & h1 & (n1 < n0));
        const bool first1 = 2 * __popc(pref1) > __popc(both);
        if (sp < kWarpBvhStack) {
          if (lane == 0) wstack[sp] = first1 ? make_int2(c0, (int)m0) : make_int2(c1, (int)m1);
          ++sp;
        }
        node = first1 ? c1 : c0;
        mask = first1 ? m1 : m0;
      } else {
        node = m0 ? c0 : c1;
        mask = m0 ? m0 : m1;
      }
    }
    while (!mask && sp > 0) {
      __syncwarp();
      --sp;
      const int2 e = wstack[sp];
      node = e.x;
      const bool again =
          ((unsigned)e.y & me) && slab32_reach(b.bbox32 + 2 * node, rs, lo, hi);
      mask = __ballot_sync(0xffffffffu, again);
    }
  }
  __syncwarp();
  *best_t = bt;
  *best_tri = bid;
}

// ray_nearest (_kernels.pyx:481-489): brute force for small scenes (tris in
// shared memory), BVH otherwise.
__device__ __forceinline__ void ray_nearest(const SceneView& s, const TriRec* smt, double ox,
                                            double oy, double oz, double dx, double dy, double dz,
                                            double tmin, double* bt, int32_t* bid) {
  if (s.brute)
    brute_nearest(smt, s.n_tris, ox, oy, oz, dx, dy, dz, tmin, bt, bid);
  else
    bvh_nearest(s, ox, oy, oz, dx, dy, dz, tmin, bt, bid);
}

}  // namespace wfpg

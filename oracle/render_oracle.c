/*
 * render_oracle.c — CPU restatement of the reference's compiled render
 * kernels (_kernels.pyx) and of the numpy field pipeline (guiding.py:231-251).
 *
 * TEST INFRASTRUCTURE ONLY (see wfpg_oracle.c header).  Scalar fp64 C with
 * -ffp-contract=off; field generation is OpenMP-parallel over bins so that
 * the CPU baseline uses every host core.  Citations: paths relative to
 * /root/reference/pkg/src/wfpg/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.141592653589793238462643383279502884

uint64_t ov_stream_key(uint64_t seed, uint64_t stream);
double ov_u01(uint64_t key, uint64_t c);

typedef struct {
  int n_tris;
  const double *v0, *e1, *e2, *normals;
  const int32_t *tri_mat, *mat_kind;
  const double* mat_rgb;
  int n_emit;
  const double* em_cdf;
  const int64_t* em_tris;
  double em_area, ray_eps;
  const double *blo, *bhi;
  const int64_t *bleft, *bright, *bcount, *border;
  int brute;
} ov_scene;

typedef struct {
  int depth, resolution;
  double lo[3], size;
  const int64_t* child_base;
  const uint8_t* child_mask;
  const int64_t* parent;
  const double *normal, *mean_a, *mean_b;
} ov_svo;

/* ------------------------------------------------------------ ray casting */
/* wfpg_brute_nearest (_kernels.pyx:40-97): minimum t, lowest id on ties */
static void brute_nearest(const ov_scene* s, const double* o, const double* d, double tmin,
                          double* bt, int64_t* bid) {
  double best = 1e300;
  int64_t id = -1;
  for (int t = 0; t < s->n_tris; ++t) {
    const double *v0 = s->v0 + 3 * t, *e1 = s->e1 + 3 * t, *e2 = s->e2 + 3 * t;
    double px = d[1] * e2[2] - d[2] * e2[1];
    double py = d[2] * e2[0] - d[0] * e2[2];
    double pz = d[0] * e2[1] - d[1] * e2[0];
    double det = e1[0] * px + e1[1] * py + e1[2] * pz;
    double sg = det > 0.0 ? 1.0 : -1.0;
    double ad = det * sg;
    double tx = o[0] - v0[0], ty = o[1] - v0[1], tz = o[2] - v0[2];
    double us = (tx * px + ty * py + tz * pz) * sg;
    double qx = ty * e1[2] - tz * e1[1];
    double qy = tz * e1[0] - tx * e1[2];
    double qz = tx * e1[1] - ty * e1[0];
    double vs = (d[0] * qx + d[1] * qy + d[2] * qz) * sg;
    double ts = (e2[0] * qx + e2[1] * qy + e2[2] * qz) * sg;
    if (ad > 1e-300 && us >= 0.0 && vs >= 0.0 && us + vs <= ad && ts > tmin * ad) {
      double h = ts / ad;
      if (h < best) {
        best = h;
        id = t;
      }
    }
  }
  *bt = best;
  *bid = id;
}

/* tri_hit (_kernels.pyx:339-372) */
static double tri_hit(const double* v0, const double* e1, const double* e2, const double* o,
                      const double* d, double tmin, double tmax) {
  double px = d[1] * e2[2] - d[2] * e2[1];
  double py = d[2] * e2[0] - d[0] * e2[2];
  double pz = d[0] * e2[1] - d[1] * e2[0];
  double det = e1[0] * px + e1[1] * py + e1[2] * pz;
  double ad = fabs(det);
  if (ad <= 1e-300) return -1.0;
  double sg = det > 0.0 ? 1.0 : -1.0;
  double tx = o[0] - v0[0], ty = o[1] - v0[1], tz = o[2] - v0[2];
  double us = (tx * px + ty * py + tz * pz) * sg;
  if (us < 0.0 || us > ad) return -1.0;
  double qx = ty * e1[2] - tz * e1[1];
  double qy = tz * e1[0] - tx * e1[2];
  double qz = tx * e1[1] - ty * e1[0];
  double vs = (d[0] * qx + d[1] * qy + d[2] * qz) * sg;
  if (vs < 0.0 || us + vs > ad) return -1.0;
  double ts = (e2[0] * qx + e2[1] * qy + e2[2] * qz) * sg;
  if (ts > tmin * ad && ts < tmax * ad) return ts / ad;
  return -1.0;
}

static void slab(const double* lo, const double* hi, const double* o, const double* inv, double* tn,
                 double* tf) {
  double n = -INFINITY, f = INFINITY;
  for (int a = 0; a < 3; ++a) {
    double t0 = (lo[a] - o[a]) * inv[a], t1 = (hi[a] - o[a]) * inv[a];
    if (a == 0) {
      n = fmin(t0, t1);
      f = fmax(t0, t1);
    } else {
      n = fmax(n, fmin(t0, t1));
      f = fmin(f, fmax(t0, t1));
    }
  }
  *tn = n;
  *tf = f;
}

/* bvh_nearest (_kernels.pyx:398-445) */
static void bvh_nearest(const ov_scene* s, const double* o, const double* d, double tmin,
                        double* bt, int64_t* bid) {
  int64_t stack[64];
  double dstack[64];
  double inv[3] = {1.0 / d[0], 1.0 / d[1], 1.0 / d[2]};
  double best = 1e300;
  int64_t id = -1;
  int sp = 1;
  stack[0] = 0;
  dstack[0] = 0.0;
  while (sp > 0) {
    --sp;
    if (dstack[sp] >= best) continue;
    int64_t node = stack[sp];
    if (s->bcount[node] > 0) {
      for (int64_t k = s->bleft[node]; k < s->bleft[node] + s->bcount[node]; ++k) {
        int64_t t = s->border[k];
        double h = tri_hit(s->v0 + 3 * t, s->e1 + 3 * t, s->e2 + 3 * t, o, d, tmin, best);
        if (h > 0.0) {
          best = h;
          id = t;
        }
      }
    } else {
      int64_t c0 = s->bleft[node], c1 = s->bright[node];
      double n0, f0, n1, f1;
      slab(s->blo + 3 * c0, s->bhi + 3 * c0, o, inv, &n0, &f0);
      slab(s->blo + 3 * c1, s->bhi + 3 * c1, o, inv, &n1, &f1);
      double d0 = (f0 >= n0 && n0 <= best && f0 >= tmin) ? n0 : 1e301;
      double d1 = (f1 >= n1 && n1 <= best && f1 >= tmin) ? n1 : 1e301;
      if (d0 > d1) {
        int64_t tn = c0;
        c0 = c1;
        c1 = tn;
        double td = d0;
        d0 = d1;
        d1 = td;
      }
      if (d1 < 1e301 && sp < 64) {
        stack[sp] = c1;
        dstack[sp++] = d1;
      }
      if (d0 < 1e301 && sp < 64) {
        stack[sp] = c0;
        dstack[sp++] = d0;
      }
    }
  }
  *bt = best;
  *bid = id;
}

/* bvh_occluded (_kernels.pyx:448-478) */
static int bvh_occluded(const ov_scene* s, const double* o, const double* d, double tmin,
                        double tmax) {
  int64_t stack[64];
  double inv[3] = {1.0 / d[0], 1.0 / d[1], 1.0 / d[2]};
  int sp = 1;
  stack[0] = 0;
  while (sp > 0) {
    int64_t node = stack[--sp];
    double n, f;
    slab(s->blo + 3 * node, s->bhi + 3 * node, o, inv, &n, &f);
    if (!(f >= n && n <= tmax && f >= tmin)) continue;
    if (s->bcount[node] > 0) {
      for (int64_t k = s->bleft[node]; k < s->bleft[node] + s->bcount[node]; ++k) {
        int64_t t = s->border[k];
        if (tri_hit(s->v0 + 3 * t, s->e1 + 3 * t, s->e2 + 3 * t, o, d, tmin, tmax) > 0.0)
          return 1;
      }
    } else if (sp + 2 <= 64) {
      stack[sp] = s->bleft[node];
      stack[sp + 1] = s->bright[node];
      sp += 2;
    }
  }
  return 0;
}

static void ray_nearest(const ov_scene* s, const double* o, const double* d, double tmin,
                        double* bt, int64_t* bid) {
  if (s->brute)
    brute_nearest(s, o, d, tmin, bt, bid);
  else
    bvh_nearest(s, o, d, tmin, bt, bid);
}

void ov_intersect(const ov_scene* s, const double* o, const double* d, int64_t n, double tmin,
                  double* out_t, int64_t* out_tri) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    ray_nearest(s, o + 3 * i, d + 3 * i, tmin, out_t + i, out_tri + i);
    if (out_tri[i] < 0) out_t[i] = INFINITY;
  }
}

/* -------------------------------------------------------------- SVO walks */
/* descend_point (_kernels.pyx:591-621) */
static int64_t descend(const ov_svo* v, const double* p, int* present) {
  double scale = v->resolution / v->size;
  long q[3];
  for (int a = 0; a < 3; ++a) {
    q[a] = (long)((p[a] - v->lo[a]) * scale);
    if (q[a] < 0) q[a] = 0;
    if (q[a] > v->resolution - 1) q[a] = v->resolution - 1;
  }
  int64_t node = 0;
  *present = 1;
  for (int level = 1; level <= v->depth; ++level) {
    int sh = v->depth - level;
    int oct = (int)(((q[0] >> sh) & 1) | (((q[1] >> sh) & 1) << 1) | (((q[2] >> sh) & 1) << 2));
    unsigned mask = v->child_mask[node];
    if (!((mask >> oct) & 1u)) {
      *present = 0;
      return node;
    }
    node = v->child_base[node] + __builtin_popcount(mask & ((1u << oct) - 1u));
  }
  return node;
}

void ov_descend(const ov_svo* v, const double* p, int64_t n, int64_t* node, uint8_t* present) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int pr;
    node[i] = descend(v, p + 3 * i, &pr);
    present[i] = (uint8_t)pr;
  }
}

/* trace_one (_kernels.pyx:661-713), literal level walk */
static void trace_one(const ov_scene* s, const ov_svo* v, const double* o, const double* d,
                      double omega, double* out) {
  out[0] = out[1] = out[2] = 0.0;
  double bt;
  int64_t btri;
  ray_nearest(s, o, d, s->ray_eps, &bt, &btri);
  if (btri < 0) return;
  double nudge = (v->size / v->resolution) * 1e-3, tiny = v->size * 1e-12;
  double q[3];
  for (int a = 0; a < 3; ++a) {
    q[a] = o[a] + bt * d[a] - d[a] * nudge;
    q[a] = fmin(fmax(q[a], v->lo[a] + tiny), v->lo[a] + v->size - tiny);
  }
  int pres;
  int64_t deep = descend(v, q, &pres);
  double area = bt * bt * omega;
  int lv = 0;
  for (int64_t cur = deep; cur > 0; cur = v->parent[cur]) ++lv;
  double side = v->size / (double)(1 << lv);
  int64_t best = deep;
  double best_diff = fabs(side * side - area);
  for (int64_t cur = v->parent[deep]; cur >= 0; cur = v->parent[cur]) {
    --lv;
    side = v->size / (double)(1 << lv);
    double diff = fabs(side * side - area);
    if (diff < best_diff) {
      best_diff = diff;
      best = cur;
    }
  }
  const double* nn = v->normal + 3 * best;
  double da = d[0] * nn[0] + d[1] * nn[1] + d[2] * nn[2];
  double w = fabs(da);
  const double* m = (da <= 0.0 ? v->mean_a : v->mean_b) + 3 * best;
  out[0] = m[0] * w;
  out[1] = m[1] * w;
  out[2] = m[2] * w;
}

void ov_trace_cones(const ov_scene* s, const ov_svo* v, const double* origins, int ostride,
                    const double* dirs, int64_t n, double omega, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) trace_one(s, v, origins + ostride * i, dirs + 3 * i, omega, out + 3 * i);
}

/* ------------------------------------------------- octahedral map (numpy) */
/* core.py:32-55; normalisation by division by sqrt((x^2+y^2)+z^2) */
static void octa_np(double u, double v, double* out) {
  double a = 2.0 * u - 1.0, b = 2.0 * v - 1.0;
  double ap = fabs(a), bp = fabs(b);
  double sd = 1.0 - (ap + bp);
  double r = 1.0 - fabs(sd);
  double phi = (r == 0.0 ? 1.0 : (bp - ap) / r + 1.0) * (PI / 4.0);
  double z = copysign(1.0 - r * r, sd);
  double rho = r * sqrt(fmax(2.0 - r * r, 0.0));
  double x = copysign(cos(phi), a) * rho;
  double y = copysign(sin(phi), b) * rho;
  double nrm = sqrt((x * x + y * y) + z * z);
  out[0] = x / nrm;
  out[1] = y / nrm;
  out[2] = z / nrm;
}

/* ------------------------------------------------------- fields (numpy) */
static int fold_index(int raw, int n, int* flip) {
  int f = 0;
  while (raw < 0 || raw >= n) {
    raw = raw < 0 ? -1 - raw : 2 * n - 1 - raw;
    f = !f;
  }
  *flip = f;
  return raw;
}

/* core.gaussian_blur (core.py:170-195) on one n x n grid, in tap order */
static void blur(double* g, double* tmp, int n, const double* w, int r) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k <= 2 * r; ++k) {
        int f, c = fold_index(i + k - r, n, &f);
        acc = acc + w[k] * (f ? g[(n - 1 - j) * n + c] : g[j * n + c]);
      }
      tmp[j * n + i] = acc;
    }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k <= 2 * r; ++k) {
        int f, rr = fold_index(j + k - r, n, &f);
        acc = acc + w[k] * (f ? tmp[rr * n + (n - 1 - i)] : tmp[rr * n + i]);
      }
      g[j * n + i] = acc;
    }
}

/* guiding.generate_fields_batch (guiding.py:231-251) for B bins */
void ov_fields(const ov_scene* s, const ov_svo* v, const double* origins, const double* jitters,
               int64_t B, int n, const double* blur_w, int radius, double eps, double* out) {
  const double omega = 4.0 * PI / (n * n);
#pragma omp parallel
  {
    double* tmp = (double*)malloc(sizeof(double) * n * n);
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
      double* g = out + b * n * n;
      double ju = jitters[2 * b] / n, jv = jitters[2 * b + 1] / n;
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          double dir[3], rgb[3];
          octa_np((double)i / n + ju, (double)j / n + jv, dir);
          trace_one(s, v, origins + 3 * b, dir, omega, rgb);
          g[j * n + i] = fma(rgb[2], 0.0722, fma(rgb[0], 0.2126, rgb[1] * 0.7152));
        }
      if (radius > 0) blur(g, tmp, n, blur_w, radius);
      for (int c = 0; c < n * n; ++c) g[c] = g[c] < eps ? eps : g[c];
    }
    free(tmp);
  }
}

/* -------------------------------------------------------------- camera */
void ov_camera(const uint64_t* keys, const int64_t* pixels, int64_t n, int width, int height,
               const double* pos, const double* fwd, const double* right, const double* up,
               double tan_half, double* oo, double* od) {
  double aspect = (double)width / (double)height;
  for (int64_t i = 0; i < n; ++i) {
    double jx = ov_u01(keys[i], 0), jy = ov_u01(keys[i], 1);
    double sx = (2.0 * ((double)(pixels[i] % width) + jx) / width - 1.0) * tan_half * aspect;
    double sy = (1.0 - 2.0 * ((double)(pixels[i] / width) + jy) / height) * tan_half;
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = fwd[a] + sx * right[a] + sy * up[a];
    double inv = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int a = 0; a < 3; ++a) {
      oo[3 * i + a] = pos[a];
      od[3 * i + a] = d[a] * inv;
    }
  }
}

/* ----------------------------------------------------------- shading */
typedef struct {
  int mode, n, m;
  double eps;
  const double *marg, *cond, *pdftab, *vals, *block_sums, *blk_marg, *blk_cond, *upper_dirs;
} ov_guide;

static int upper_bound(const double* cdf, int n, double u) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cdf[mid] <= u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo > n - 1 ? n - 1 : lo;
}

static int invert_cdf(const double* cdf, int n, double u, double* frac) {
  int i = upper_bound(cdf, n, u);
  double lo = i > 0 ? cdf[i - 1] : 0.0, span = cdf[i] - lo, f = 0.0;
  if (span > 0.0) f = (u - lo) / span;
  if (f > 1.0 - 1e-12) f = 1.0 - 1e-12;
  if (f < 0.0) f = 0.0;
  *frac = f;
  return i;
}

/* uv_to_dir (_kernels.pyx:240-262) */
static void uv_to_dir(double u, double v, double* o) {
  double a = 2.0 * u - 1.0, b = 2.0 * v - 1.0, ap = fabs(a), bp = fabs(b);
  double sd = 1.0 - (ap + bp), r = 1.0 - fabs(sd);
  double phi = (r == 0.0 ? 1.0 : (bp - ap) / r + 1.0) * (PI / 4.0);
  double z = copysign(1.0 - r * r, sd), rho = r * sqrt(fmax(2.0 - r * r, 0.0));
  double x = copysign(cos(phi), a) * rho, y = copysign(sin(phi), b) * rho;
  double inv = 1.0 / sqrt(x * x + y * y + z * z);
  o[0] = x * inv;
  o[1] = y * inv;
  o[2] = z * inv;
}

/* dir_to_uv (_kernels.pyx:265-298) */
static void dir_to_uv(const double* d, double* ou, double* ov) {
  double x = fabs(d[0]), y = fabs(d[1]), r = sqrt(fmax(1.0 - fabs(d[2]), 0.0));
  double hi = fmax(x, y), lo = fmin(x, y), ratio = hi > 0.0 ? lo / hi : 0.0;
  double phi = atan(ratio) * (2.0 / PI);
  if (x < y) phi = 1.0 - phi;
  double vq = phi * r, uq = r - vq;
  if (d[2] < 0.0) {
    double t = uq;
    uq = 1.0 - vq;
    vq = 1.0 - t;
  }
  uq = copysign(uq, d[0]);
  vq = copysign(vq, d[1]);
  double u = 0.5 * (uq + 1.0), v = 0.5 * (vq + 1.0);
  *ou = fmin(fmax(u, 0.0), 1.0 - 1e-12);
  *ov = fmin(fmax(v, 0.0), 1.0 - 1e-12);
}

static void cell(int n, const double* d, int* i, int* j) {
  double u, v;
  dir_to_uv(d, &u, &v);
  *i = (int)(u * n);
  *j = (int)(v * n);
  if (*i > n - 1) *i = n - 1;
  if (*j > n - 1) *j = n - 1;
}

static double pdf_plain(const ov_guide* g, int slot, const double* d) {
  int i, j;
  cell(g->n, d, &i, &j);
  return g->pdftab[((int64_t)slot * g->n + j) * g->n + i];
}

static double pdf_product(const ov_guide* g, int slot, const double* upper, double upsum,
                          const double* d) {
  int i, j, n = g->n;
  cell(n, d, &i, &j);
  int bi = i / g->m, bj = j / g->m;
  return (upper[bj * 8 + bi] / upsum) *
         (g->vals[((int64_t)slot * n + j) * n + i] / g->block_sums[((int64_t)slot * 8 + bj) * 8 + bi]) *
         (double)(n * n) / (4.0 * PI);
}

static void cosine_dir(const double* ns, double u1, double u2, double* o) {
  double r = sqrt(u1), phi = 2.0 * PI * u2;
  double x = r * cos(phi), y = r * sin(phi), z = sqrt(fmax(1.0 - u1, 0.0));
  double s = copysign(1.0, ns[2]), a = -1.0 / (s + ns[2]), b = ns[0] * ns[1] * a;
  o[0] = x * (1.0 + s * ns[0] * ns[0] * a) + y * b + z * ns[0];
  o[1] = x * (s * b) + y * (s + ns[1] * ns[1] * a) + z * ns[1];
  o[2] = x * (-s * ns[0]) + y * (-ns[1]) + z * ns[2];
}

typedef struct {
  double *ray_o, *ray_d, *beta, *radiance;
  const uint64_t* key;
  uint64_t* ctr;
  uint8_t* alive;
  double *prev_pdf, *rec_pos, *rec_T, *emit_le;
  int32_t* emit_depth;
  int rec_depths;
} ov_paths;

/* shade_one (_kernels.pyx:905-1161) */
static void shade_one(int64_t p, int depth, const ov_scene* sa, const ov_guide* g,
                      const ov_paths* P, const double* hit_t, const int64_t* hit_tri,
                      const int32_t* bin_slot, int rr_enabled, int rr_depth) {
  int64_t tri = hit_tri[p];
  if (tri < 0) {
    P->alive[p] = 0;
    return;
  }
  double* ro = P->ray_o + 3 * p;
  double* rd = P->ray_d + 3 * p;
  double* beta = P->beta + 3 * p;
  double* rad = P->radiance + 3 * p;
  double t = hit_t[p], d[3] = {rd[0], rd[1], rd[2]};
  double pos[3] = {ro[0] + t * d[0], ro[1] + t * d[1], ro[2] + t * d[2]};
  int64_t rb = (p * P->rec_depths + depth) * 3;
  for (int a = 0; a < 3; ++a) {
    P->rec_pos[rb + a] = pos[a];
    P->rec_T[rb + a] = beta[a];
  }
  int mid = sa->tri_mat[tri], kind = sa->mat_kind[mid];
  const double* ng = sa->normals + 3 * tri;
  const double* mrgb = sa->mat_rgb + 3 * mid;
  double cos_in = -(ng[0] * d[0] + ng[1] * d[1] + ng[2] * d[2]);
  if (kind == 2) {
    double le[3] = {0.0, 0.0, 0.0};
    if (cos_in > 0.0)
      for (int a = 0; a < 3; ++a) le[a] = mrgb[a];
    double w = 1.0;
    if (P->prev_pdf[p] >= 0.0 && cos_in > 1e-9) {
      double pl = t * t / (sa->em_area * cos_in);
      w = P->prev_pdf[p] / (P->prev_pdf[p] + pl);
    }
    for (int a = 0; a < 3; ++a) {
      rad[a] += beta[a] * w * le[a];
      P->emit_le[3 * p + a] = le[a];
    }
    P->emit_depth[p] = depth;
    P->alive[p] = 0;
    return;
  }
  if (kind == 1) {
    if (cos_in == 0.0) {
      P->alive[p] = 0;
      return;
    }
    double flip = cos_in > 0.0 ? 1.0 : -1.0, ns[3] = {ng[0] * flip, ng[1] * flip, ng[2] * flip};
    double w = -d[0] * ns[0] + -d[1] * ns[1] + -d[2] * ns[2];
    for (int a = 0; a < 3; ++a) {
      beta[a] *= mrgb[a];
      ro[a] = pos[a];
      rd[a] = 2.0 * w * ns[a] + d[a];
    }
    P->prev_pdf[p] = -1.0;
    return;
  }
  int n = g->n, m = g->m, grazing = cos_in == 0.0;
  double flip = cos_in >= 0.0 ? 1.0 : -1.0, ns[3] = {ng[0] * flip, ng[1] * flip, ng[2] * flip};
  double al[3] = {mrgb[0], mrgb[1], mrgb[2]};
  uint64_t kk = P->key[p], c = P->ctr[p];
  int slot = g->mode > 0 ? bin_slot[p] : -1, guided = slot >= 0;
  double upper[64], upsum = 1.0;
  if (guided && g->mode == 2) {
    double alb = 0.2126 * al[0] + 0.7152 * al[1] + 0.0722 * al[2];
    upsum = 0.0;
    for (int q = 0; q < 64; ++q) {
      double mean = g->block_sums[(int64_t)slot * 64 + q] / (double)(m * m);
      const double* ud = g->upper_dirs + 3 * q;
      double cosf = ud[0] * ns[0] + ud[1] * ns[1] + ud[2] * ns[2];
      if (cosf < 0.0) cosf = 0.0;
      double val = mean * (alb / PI) * cosf;
      if (val < g->eps) val = g->eps;
      upper[q] = val;
      upsum += val;
    }
  }
  /* next-event estimation */
  double u1 = ov_u01(kk, c), u2 = ov_u01(kk, c + 1);
  c += 2;
  int li = upper_bound(sa->em_cdf, sa->n_emit, u1);
  int64_t lt = sa->em_tris[li];
  double b0 = li > 0 ? sa->em_cdf[li - 1] : 0.0, su = sa->em_cdf[li] - b0;
  double b1 = su > 0.0 ? (u1 - b0) / su : 0.0;
  if (b1 > 1.0 - 1e-12) b1 = 1.0 - 1e-12;
  if (b1 < 0.0) b1 = 0.0;
  su = sqrt(b1);
  double aa = 1.0 - su, bb = u2 * su, lp[3], del[3];
  for (int a = 0; a < 3; ++a) {
    lp[a] = sa->v0[3 * lt + a] + aa * sa->e1[3 * lt + a] + bb * sa->e2[3 * lt + a];
    del[a] = lp[a] - pos[a];
  }
  const double* ln = sa->normals + 3 * lt;
  const double* le = sa->mat_rgb + 3 * sa->tri_mat[lt];
  double dist = sqrt(del[0] * del[0] + del[1] * del[1] + del[2] * del[2]);
  if (dist > 2.0 * sa->ray_eps) {
    double dl[3] = {del[0] / dist, del[1] / dist, del[2] / dist};
    double cos_l = -(ln[0] * dl[0] + ln[1] * dl[1] + ln[2] * dl[2]);
    double cos_s = ns[0] * dl[0] + ns[1] * dl[1] + ns[2] * dl[2];
    if (cos_l > 1e-9 && cos_s > 0.0 && !grazing && le[0] + le[1] + le[2] > 0.0) {
      double pl = dist * dist / (sa->em_area * cos_l);
      if (!bvh_occluded(sa, pos, dl, sa->ray_eps, dist - sa->ray_eps)) {
        double p_cont;
        if (guided) {
          double pg = g->mode == 1 ? pdf_plain(g, slot, dl) : pdf_product(g, slot, upper, upsum, dl);
          p_cont = 0.5 * pg + 0.5 * (cos_s / PI);
        } else {
          p_cont = cos_s / PI;
        }
        double w = pl / (pl + p_cont), scale = (cos_s * w / pl) / PI;
        for (int a = 0; a < 3; ++a) rad[a] += beta[a] * al[a] * scale * le[a];
      }
    }
  }
  int rr_alive = 1;
  if (rr_enabled && depth >= rr_depth) {
    double u_rr = ov_u01(kk, c);
    c += 1;
    double q = fmax(fmax(beta[0], beta[1]), beta[2]);
    if (q > 1.0) q = 1.0;
    if (q < 0.05) q = 0.05;
    if (u_rr < q)
      for (int a = 0; a < 3; ++a) beta[a] /= q;
    else
      rr_alive = 0;
  }
  double wi[3] = {0.0, 0.0, 1.0}, cos_rel, pdf_mix;
  if (guided) {
    double coin = ov_u01(kk, c);
    c += 1;
    if (coin < 0.5) {
      double fv, fu;
      if (g->mode == 1) {
        double s1 = ov_u01(kk, c), s2 = ov_u01(kk, c + 1);
        c += 2;
        int gj = invert_cdf(g->marg + (int64_t)slot * n, n, s1, &fv);
        int gi = invert_cdf(g->cond + ((int64_t)slot * n + gj) * n, n, s2, &fu);
        uv_to_dir((gi + fu) / n, (gj + fv) / n, wi);
      } else {
        double s1 = ov_u01(kk, c), s2 = ov_u01(kk, c + 1), s3 = ov_u01(kk, c + 2),
               s4 = ov_u01(kk, c + 3);
        c += 4;
        double urow[8], ucdf[8];
        for (int bj = 0; bj < 8; ++bj) {
          urow[bj] = 0.0;
          for (int bi = 0; bi < 8; ++bi) urow[bj] += upper[bj * 8 + bi];
        }
        ucdf[0] = urow[0] / upsum;
        for (int bj = 1; bj < 8; ++bj) ucdf[bj] = ucdf[bj - 1] + urow[bj] / upsum;
        int bj = invert_cdf(ucdf, 8, s1, &fv);
        ucdf[0] = upper[bj * 8] / urow[bj];
        for (int bi = 1; bi < 8; ++bi) ucdf[bi] = ucdf[bi - 1] + upper[bj * 8 + bi] / urow[bj];
        int bi = invert_cdf(ucdf, 8, s2, &fu);
        int64_t blk = ((int64_t)slot * 8 + bj) * 8 + bi;
        int jin = invert_cdf(g->blk_marg + blk * m, m, s3, &fv);
        int iin = invert_cdf(g->blk_cond + (blk * m + jin) * m, m, s4, &fu);
        uv_to_dir((bi * m + iin + fu) / n, (bj * m + jin + fv) / n, wi);
      }
    } else {
      double s1 = ov_u01(kk, c), s2 = ov_u01(kk, c + 1);
      c += 2;
      cosine_dir(ns, s1, s2, wi);
    }
    cos_rel = wi[0] * ns[0] + wi[1] * ns[1] + wi[2] * ns[2];
    double pg = g->mode == 1 ? pdf_plain(g, slot, wi) : pdf_product(g, slot, upper, upsum, wi);
    pdf_mix = 0.5 * pg + 0.5 * (fmax(cos_rel, 0.0) / PI);
  } else {
    double s1 = ov_u01(kk, c), s2 = ov_u01(kk, c + 1);
    c += 2;
    cosine_dir(ns, s1, s2, wi);
    cos_rel = wi[0] * ns[0] + wi[1] * ns[1] + wi[2] * ns[2];
    pdf_mix = fmax(cos_rel, 0.0) / PI;
  }
  if (rr_alive && cos_rel > 0.0 && pdf_mix > 0.0 && !grazing) {
    double factor = (cos_rel / pdf_mix) / PI;
    for (int a = 0; a < 3; ++a) beta[a] *= al[a] * factor;
    P->alive[p] = (beta[0] > 0.0 || beta[1] > 0.0 || beta[2] > 0.0) ? 1 : 0;
  } else {
    beta[0] = beta[1] = beta[2] = 0.0;
    P->alive[p] = 0;
  }
  for (int a = 0; a < 3; ++a) {
    ro[a] = pos[a];
    rd[a] = wi[a];
  }
  P->prev_pdf[p] = pdf_mix;
  P->ctr[p] = c;
}

void ov_shade(const ov_scene* sa, const ov_guide* g, const ov_paths* P, int depth,
              const int64_t* active, int64_t n_active, const double* hit_t,
              const int64_t* hit_tri, const int32_t* bin_slot, int rr_enabled, int rr_depth) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_active; ++i)
    shade_one(active[i], depth, sa, g, P, hit_t, hit_tri, bin_slot, rr_enabled, rr_depth);
}

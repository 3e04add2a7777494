/*
 * wfpg_oracle.c — CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker / CPU baseline.  The product (paper_2405_06997_b200)
 * never links or calls it.
 *
 * Plain scalar C, compiled with -ffp-contract=off so that every fma() below
 * is explicit and every other expression rounds per operation; the operation
 * orders follow oracle/NUMERICS.md.  Each function cites the reference
 * (paths relative to /root/reference/pkg/src/wfpg/).  Parity is pinned by
 * tests/test_oracle.py against tests/golden/*.npz, which were produced by the
 * real reference (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.141592653589793238462643383279502884

/* ------------------------------------------------------------------ RNG */
/* core.py:204-228 */
static uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
static const uint64_t PHI = 0x9E3779B97F4A7C15ull;
uint64_t ov_stream_key(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ (mix64(stream) * PHI));
}
double ov_u01(uint64_t key, uint64_t c) {
  return (double)(mix64(key + (c + 1) * PHI) >> 11) * (1.0 / 9007199254740992.0);
}

/* --------------------------------------------------------- dot recipes */
static double dgemv3(const double* x, const double* m) {
  return fma(x[2], m[2], fma(x[0], m[0], x[1] * m[1]));
}
static double ddot3(const double* x, const double* m) {
  return fma(x[2], m[2], fma(x[1], m[1], x[0] * m[0]));
}
static double einsum3(const double* x, const double* y) {
  return (x[0] * y[0] + x[2] * y[2]) + x[1] * y[1];
}

/* ------------------------------------------------------ voxelisation SAT */
/* svo.py:49-91: one candidate box against one triangle.  `single` selects
 * the BLAS kernel numpy used for the batch (1 row -> ddot, >= 2 -> dgemv). */
static int sat_axis(int single, const double* a, const double* b, const double* d,
                    const double* hh, const double* ax) {
  if (sqrt(ddot3(ax, ax)) < 1e-30) return 1;
  double aa[3] = {fabs(ax[0]), fabs(ax[1]), fabs(ax[2])};
  double pa = single ? ddot3(a, ax) : dgemv3(a, ax);
  double pb = single ? ddot3(b, ax) : dgemv3(b, ax);
  double pd = single ? ddot3(d, ax) : dgemv3(d, ax);
  double r = single ? ddot3(hh, aa) : dgemv3(hh, aa);
  double lo = fmin(fmin(pa, pb), pd), hi = fmax(fmax(pa, pb), pd);
  return lo <= r && hi >= -r;
}

static int tri_box(const double* v0, const double* v1, const double* v2, const double* blo,
                   const double* bhi, int single) {
  double c[3], hh[3], a[3], b[3], d[3], e[3][3], n[3];
  for (int k = 0; k < 3; ++k) {
    c[k] = 0.5 * (blo[k] + bhi[k]);
    hh[k] = 0.5 * (bhi[k] - blo[k]);
    a[k] = v0[k] - c[k];
    b[k] = v1[k] - c[k];
    d[k] = v2[k] - c[k];
  }
  for (int k = 0; k < 3; ++k) {
    double lo = fmin(fmin(a[k], b[k]), d[k]), hi = fmax(fmax(a[k], b[k]), d[k]);
    if (!(lo <= hh[k] && hi >= -hh[k])) return 0;
  }
  for (int k = 0; k < 3; ++k) {
    e[0][k] = v1[k] - v0[k];
    e[1][k] = v2[k] - v1[k];
    e[2][k] = v0[k] - v2[k];
  }
  n[0] = e[0][1] * e[1][2] - e[0][2] * e[1][1];
  n[1] = e[0][2] * e[1][0] - e[0][0] * e[1][2];
  n[2] = e[0][0] * e[1][1] - e[0][1] * e[1][0];
  if (!sat_axis(single, a, b, d, hh, n)) return 0;
  for (int k = 0; k < 3; ++k) {
    double x[3] = {0.0, -e[k][2], e[k][1]};
    double y[3] = {e[k][2], 0.0, -e[k][0]};
    double z[3] = {-e[k][1], e[k][0], 0.0};
    if (!sat_axis(single, a, b, d, hh, x)) return 0;
    if (!sat_axis(single, a, b, d, hh, y)) return 0;
    if (!sat_axis(single, a, b, d, hh, z)) return 0;
  }
  return 1;
}

static long long floor_clip(double x, double lo, double h, int r) {
  long long q = (long long)floor((x - lo) / h);
  if (q < 0) q = 0;
  if (q > r - 1) q = r - 1;
  return q;
}

/* svo.py:94-136.  Writes up to `cap` fragments (coords (F,3) int64, tris (F,));
 * returns the total count. */
int64_t ov_voxelize(int T, const double* v0, const double* v1, const double* v2,
                    const double* cube_lo, double side, int r, int64_t* coords, int64_t* tris,
                    int64_t cap) {
  double h = side / r;
  int64_t nf = 0;
  for (int t = 0; t < T; ++t) {
    const double *p0 = v0 + 3 * t, *p1 = v1 + 3 * t, *p2 = v2 + 3 * t;
    long long lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      double tl = fmin(fmin(p0[k], p1[k]), p2[k]), th = fmax(fmax(p0[k], p1[k]), p2[k]);
      lo[k] = floor_clip(tl, cube_lo[k], h, r);
      hi[k] = floor_clip(th, cube_lo[k], h, r);
    }
    int64_t K = (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
    for (long long x = lo[0]; x <= hi[0]; ++x)
      for (long long y = lo[1]; y <= hi[1]; ++y)
        for (long long z = lo[2]; z <= hi[2]; ++z) {
          double blo[3] = {cube_lo[0] + (double)x * h, cube_lo[1] + (double)y * h,
                           cube_lo[2] + (double)z * h};
          double bhi[3] = {blo[0] + h, blo[1] + h, blo[2] + h};
          if (tri_box(p0, p1, p2, blo, bhi, K == 1)) {
            if (nf < cap) {
              coords[3 * nf] = x;
              coords[3 * nf + 1] = y;
              coords[3 * nf + 2] = z;
              tris[nf] = t;
            }
            ++nf;
          }
        }
  }
  return nf;
}

/* ------------------------------------------------------- dual-normal k-means */
/* svo.py:139-173 over rows[0..K) */
void ov_cluster_normals(const double* rows, int K, uint64_t key, double* out) {
  long long pk = (long long)(ov_u01(key, 0) * (double)K);
  int pick = (int)(pk < K - 1 ? pk : K - 1);
  double ma[3] = {rows[3 * pick], rows[3 * pick + 1], rows[3 * pick + 2]};
  double mb[3] = {-ma[0], -ma[1], -ma[2]};
  unsigned char* prev = (unsigned char*)malloc(K);
  unsigned char* cur = (unsigned char*)malloc(K);
  int have_prev = 0;
  for (int it = 0; it < 32; ++it) {
    for (int i = 0; i < K; ++i) cur[i] = dgemv3(rows + 3 * i, ma) >= dgemv3(rows + 3 * i, mb);
    if (have_prev && memcmp(prev, cur, K) == 0) break;
    memcpy(prev, cur, K);
    have_prev = 1;
    double sa[3] = {0.0, 0.0, 0.0}, sb[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < K; ++i) {
      double* s = cur[i] ? sa : sb;
      for (int k = 0; k < 3; ++k) s[k] = s[k] + rows[3 * i + k];
    }
    double na = sqrt(ddot3(sa, sa)), nb = sqrt(ddot3(sb, sb));
    if (na > 1e-12)
      for (int k = 0; k < 3; ++k) ma[k] = sa[k] / na;
    if (nb > 1e-12) {
      for (int k = 0; k < 3; ++k) mb[k] = sb[k] / nb;
    } else {
      for (int k = 0; k < 3; ++k) mb[k] = -ma[k];
    }
  }
  free(prev);
  free(cur);
  out[0] = ma[0];
  out[1] = ma[1];
  out[2] = ma[2];
}

/* svo.py:472-499: leaf normals over the sorted fragment normals, then the
 * internal levels bottom-up.  level_off (depth+2), codes, child_base,
 * child_mask as built; frag_n (F,3) sorted fragment normals, leaf_start (L+1). */
void ov_svo_normals(int depth, const int64_t* level_off, const uint64_t* codes,
                    const int64_t* child_base, const uint8_t* child_mask, const double* frag_n,
                    const int64_t* leaf_start, uint64_t seed, double* normal) {
  int64_t lb = level_off[depth], L = level_off[depth + 1] - lb;
  for (int64_t i = 0; i < L; ++i) {
    const double* seg = frag_n + 3 * leaf_start[i];
    int K = (int)(leaf_start[i + 1] - leaf_start[i]);
    int same = 1;
    for (int j = 1; j < K && same; ++j)
      same = seg[3 * j] == seg[0] && seg[3 * j + 1] == seg[1] && seg[3 * j + 2] == seg[2];
    double* o = normal + 3 * (lb + i);
    if (same) {
      o[0] = seg[0];
      o[1] = seg[1];
      o[2] = seg[2];
    } else {
      ov_cluster_normals(seg, K, ov_stream_key(seed, codes[lb + i] * 4 + 2), o);
    }
  }
  double* both = (double*)malloc(sizeof(double) * 3 * 16);
  for (int l = depth - 1; l >= 0; --l) {
    for (int64_t node = level_off[l]; node < level_off[l + 1]; ++node) {
      int64_t base = child_base[node];
      int cnt = __builtin_popcount(child_mask[node]);
      const double* kid = normal + 3 * base;
      int same = 1;
      for (int j = 1; j < cnt && same; ++j)
        same = fabs(kid[3 * j]) == fabs(kid[0]) && fabs(kid[3 * j + 1]) == fabs(kid[1]) &&
               fabs(kid[3 * j + 2]) == fabs(kid[2]);
      double* o = normal + 3 * node;
      if (same) {
        o[0] = kid[0];
        o[1] = kid[1];
        o[2] = kid[2];
        continue;
      }
      for (int j = 0; j < cnt; ++j)
        for (int k = 0; k < 3; ++k) {
          both[3 * j + k] = kid[3 * j + k];
          both[3 * (cnt + j) + k] = -kid[3 * j + k];
        }
      uint64_t stream = codes[node] * 4 + 3 + ((uint64_t)l << 48);
      ov_cluster_normals(both, 2 * cnt, ov_stream_key(seed, stream), o);
    }
  }
  free(both);
}

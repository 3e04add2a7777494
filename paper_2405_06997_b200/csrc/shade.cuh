// Guided sampling helpers + the per-path shading step (_kernels.pyx:800-1161).
#pragma once
#include "geometry.cuh"

namespace wfpg {

struct GuideView {
  int mode;  // 0 off, 1 plain, 2 product
  int n;
  int m;     // n / 8
  double eps;
  double pdf_scale;  // n*n / (4 pi) as computed by the reference (guiding.py:300)
  const double* vals;
  const double* row_sum;
  const double* marg;
  const double* total;
  const double* block_sums;
  const double* upper_dirs;  // (8,8,3) host-numpy octahedral cell centres
  const double* cum;         // optional row prefix sums (plain sampler fast path)
  const double* block_rows;  // optional (B,8,8,m) block row sums (product sampler)
};

// upper_bound (_kernels.pyx:802-812)
__device__ __forceinline__ int upper_bound_d(const double* cdf, int n, double u) {
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

// Number of leading elements of the non-decreasing row a[0..n) that satisfy
// `a[i] <= x` (strict = false) or `a[i] < x` (strict = true) — the
// upper_bound / lower_bound index — in two dependent rounds of independent
// loads instead of log2(n) dependent ones: 8 probes at the ends of n/8
// blocks, then the block that holds the boundary (16-byte loads).  n must be
// a multiple of 8 and a 16-byte aligned.  Same index as the binary search.
template <bool strict>
__device__ __forceinline__ int count_leading(const double* __restrict__ a, int n, double x) {
  const int B = n >> 3;
  int k = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double v = __ldg(a + j * B + B - 1);
    k += strict ? (v < x) : (v <= x);
  }
  if (k == 8 || B == 1) return k * B;
  const double2* blk = reinterpret_cast<const double2*>(a + k * B);
  int c = 0;
#pragma unroll 4
  for (int i = 0; i < (B >> 1); ++i) {
    const double2 v = __ldg(blk + i);
    c += strict ? (v.x < x) + (v.y < x) : (v.x <= x) + (v.y <= x);
  }
  return k * B + c;
}

__device__ __forceinline__ double residual(double u, double lo, double hi) {
  double span = hi - lo;
  double f = span > 0.0 ? (u - lo) / span : 0.0;
  if (f > 1.0 - 1e-12) f = 1.0 - 1e-12;
  if (f < 0.0) f = 0.0;
  return f;
}

// invert_cdf over a stored CDF (_kernels.pyx:815-827)
__device__ __forceinline__ int invert_cdf(const double* cdf, int n, double u, double* frac) {
  int i = upper_bound_d(cdf, n, u);
  double lo = i > 0 ? cdf[i - 1] : 0.0;
  *frac = residual(u, lo, cdf[i]);
  return i;
}

// invert_cdf over a guide-table row in global memory (n a multiple of 8)
__device__ __forceinline__ int invert_cdf_row(const double* cdf, int n, double u, double* frac) {
  int i = count_leading<false>(cdf, n, u);
  i = i > n - 1 ? n - 1 : i;
  double lo = i > 0 ? cdf[i - 1] : 0.0;
  *frac = residual(u, lo, cdf[i]);
  return i;
}

// invert_cdf over cumsum(v[0..n)) / denom evaluated on the fly, with the
// reference's sequential cumsum (guiding.py:299,309).  A linear scan returns
// the same index as the binary search because the CDF is non-decreasing.
__device__ __forceinline__ int invert_cumsum(const double* v, int stride, int n, double denom,
                                             double u, double* frac) {
  double run = 0.0, prev = 0.0, cur = 0.0;
  int i = 0;
  for (; i < n; ++i) {
    run = i == 0 ? v[0] : __dadd_rn(run, v[(int64_t)i * stride]);
    cur = __ddiv_rn(run, denom);
    if (cur > u) break;
    if (i < n - 1) prev = cur;
  }
  if (i >= n) i = n - 1;  // clamp: cur is cdf[n-1], prev cdf[n-2]
  double lo = i > 0 ? prev : 0.0;
  *frac = residual(u, lo, cur);
  return i;
}

// Same result as invert_cumsum given the stored prefix sums cum[0..n):
// cdf_i = cum_i / denom is non-decreasing; every cum_i < u*denom*(1-1e-12)
// gives cdf_i < u (the bound covers the roundings of the product and of the
// division), so a binary search finds the first index that can exceed u and
// the exact divisions are only evaluated from there (usually once).
__device__ __forceinline__ int invert_prefix(const double* cum, int n, double denom, double u,
                                             double* frac) {
  const double thr = u * denom * (1.0 - 1e-12);
  const int lo = count_leading<true>(cum, n, thr);  // first index with cum >= thr
  int i = lo < n ? lo : n - 1;
  double cur = __ddiv_rn(cum[i], denom);
  while (!(cur > u) && i < n - 1) {
    ++i;
    cur = __ddiv_rn(cum[i], denom);
  }
  double prev = i > 0 ? __ddiv_rn(cum[i - 1], denom) : 0.0;
  *frac = residual(u, prev, cur);
  return i;
}

// numpy pairwise sum of a contiguous row of length n (8 <= n <= 128 or n < 8)
__device__ __forceinline__ double pairwise_row(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a[i]);
    r1 = __dadd_rn(r1, a[i + 1]);
    r2 = __dadd_rn(r2, a[i + 2]);
    r3 = __dadd_rn(r3, a[i + 3]);
    r4 = __dadd_rn(r4, a[i + 4]);
    r5 = __dadd_rn(r5, a[i + 5]);
    r6 = __dadd_rn(r6, a[i + 6]);
    r7 = __dadd_rn(r7, a[i + 7]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ __forceinline__ void cell_of(int n, double dx, double dy, double dz, int* ci, int* cj) {
  double u, v;
  octa_dir_to_uv_k(dx, dy, dz, &u, &v);
  int i = (int)(u * n), j = (int)(v * n);
  *ci = i > n - 1 ? n - 1 : i;
  *cj = j > n - 1 ? n - 1 : j;
}

// pdf_plain_dir (_kernels.pyx:876-885): pdftab = vals * (n^2/4pi) / total
__device__ __forceinline__ double pdf_plain_cell(const GuideView& g, int slot, int i, int j) {
  double v = g.vals[((int64_t)slot * g.n + j) * g.n + i];
  return __ddiv_rn(__dmul_rn(v, g.pdf_scale), g.total[slot]);
}
__device__ __forceinline__ double pdf_plain(const GuideView& g, int slot, double dx, double dy,
                                            double dz) {
  int i, j;
  cell_of(g.n, dx, dy, dz, &i, &j);
  return pdf_plain_cell(g, slot, i, j);
}

// L2 prefetch of a guide-table entry a later lookup will read
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Per-path product layer (_kernels.pyx:1003-1019), register resident: cell
// k = bj * 8 + bi is block_mean * (lum(albedo) / pi) * max(0, upper_dir . n_s)
// floored at eps, a pure function of (slot, k, n_s, albedo), so the 64 cells
// are never stored: one pass accumulates upsum (sequential over k, the
// reference's order) and the 8 row sums (sequential over bi), and the
// samplers / pdfs re-evaluate the few cells they need.
struct ProductLayer {
  const double* bs;  // block sums of the path's bin (8, 8)
  double nsx, nsy, nsz;
  double lum_pi;     // lum(albedo) / pi
  double mm;         // m * m
  double inv_mm;     // 1 / (m * m), exact: m = n / 8 is a power of two
  double upsum;
  double urow[8];
};

// guiding.UPPER_DIRS (8,8,3), copied into constant memory by the shade
// launcher: every lane reads cell k of its own layer at the same k, so the
// reads are constant-cache broadcasts
static __constant__ double c_upper_dirs[192];

__device__ __forceinline__ double product_cell(const GuideView& g, const ProductLayer& L, int k) {
  // block_sums / (m m) (K:1008): m m is a power of two, so the product with
  // its exact reciprocal is the same rounding of the same real number
  const double mean = __dmul_rn(__ldg(L.bs + k), L.inv_mm);
  const double* ud = c_upper_dirs + 3 * k;
  double cosf = ud[0] * L.nsx + ud[1] * L.nsy + ud[2] * L.nsz;
  if (cosf < 0.0) cosf = 0.0;
  double val = mean * L.lum_pi * cosf;
  if (val < g.eps) val = g.eps;
  return val;
}

__device__ __forceinline__ void product_layer(const GuideView& g, int slot, double nsx,
                                              double nsy, double nsz, double alx, double aly,
                                              double alz, ProductLayer* L) {
  L->bs = g.block_sums + (int64_t)slot * 64;
  L->nsx = nsx;
  L->nsy = nsy;
  L->nsz = nsz;
  L->lum_pi = (0.2126 * alx + 0.7152 * aly + 0.0722 * alz) / WFPG_PI;
  L->mm = (double)(g.m * g.m);
  L->inv_mm = 1.0 / L->mm;
  double upsum = 0.0;
#pragma unroll
  for (int bj = 0; bj < 8; ++bj) {
    double row = 0.0;
#pragma unroll
    for (int bi = 0; bi < 8; ++bi) {
      const double v = product_cell(g, *L, bj * 8 + bi);
      upsum += v;
      row += v;
    }
    L->urow[bj] = row;
  }
  L->upsum = upsum;
}

// pdf_product_dir (_kernels.pyx:888-902)
__device__ __forceinline__ double pdf_product(const GuideView& g, int slot, const ProductLayer& L,
                                              double dx, double dy, double dz) {
  int i, j;
  cell_of(g.n, dx, dy, dz, &i, &j);
  int bi = i / g.m, bj = j / g.m;
  double v = g.vals[((int64_t)slot * g.n + j) * g.n + i];
  double bs = g.block_sums[((int64_t)slot * 8 + bj) * 8 + bi];
  return (product_cell(g, L, bj * 8 + bi) / L.upsum) * (v / bs) * (double)(g.n * g.n) /
         (4.0 * WFPG_PI);
}

// plain guided sample (_kernels.pyx:1093-1100): marginal then on-the-fly conditional
__device__ __forceinline__ void sample_plain(const GuideView& g, int slot, double s1, double s2,
                                             double* wx, double* wy, double* wz) {
  const int n = g.n;
  double fv, fu;
  int gj = invert_cdf_row(g.marg + (int64_t)slot * n, n, s1, &fv);
  const double denom = g.row_sum[(int64_t)slot * n + gj];
  int gi = g.cum ? invert_prefix(g.cum + ((int64_t)slot * n + gj) * n, n, denom, s2, &fu)
                 : invert_cumsum(g.vals + ((int64_t)slot * n + gj) * n, 1, n, denom, s2, &fu);
  octa_uv_to_dir_k((gi + fu) / n, (gj + fv) / n, wx, wy, wz);
}

// product guided sample (_kernels.pyx:1101-1127)
__device__ __forceinline__ void sample_product(const GuideView& g, int slot, const ProductLayer& L,
                                               double s1, double s2, double s3, double s4,
                                               double* wx, double* wy, double* wz) {
  const int n = g.n, m = g.m;
  double fv, fu;
  // upper row: running CDF of urow / upsum (sequential, as the reference)
  int bj = 7;
  {
    double prev = 0.0, cur = 0.0;
    for (int r = 0; r < 8; ++r) {
      cur = r == 0 ? L.urow[0] / L.upsum : prev + L.urow[r] / L.upsum;
      if (cur > s1 || r == 7) {
        bj = r;
        break;
      }
      prev = cur;
    }
    fv = residual(s1, bj > 0 ? prev : 0.0, cur);
  }
  int bi = 7;
  {
    const double rs = L.urow[bj];
    double prev = 0.0, cur = 0.0;
    for (int c = 0; c < 8; ++c) {
      const double v = product_cell(g, L, bj * 8 + c);
      cur = c == 0 ? v / rs : prev + v / rs;
      if (cur > s2 || c == 7) {
        bi = c;
        break;
      }
      prev = cur;
    }
    fu = residual(s2, bi > 0 ? prev : 0.0, cur);
  }
  // block rows of the selected block: rows[r] = 0 + pairwise(row r), the block
  // marginal is cumsum(rows) / block_sum (guiding.py:304-309)
  const double* blk = g.vals + ((int64_t)slot * n + bj * m) * n + bi * m;
  const double bsum = g.block_sums[((int64_t)slot * 8 + bj) * 8 + bi];
  const double* brows =
      g.block_rows ? g.block_rows + (((int64_t)slot * 8 + bj) * 8 + bi) * m : nullptr;
  int jin = m - 1;
  double rowj = 0.0;
  {
    double run = 0.0, prev = 0.0, cur = 0.0;
    for (int r = 0; r < m; ++r) {
      const double rr =
          brows ? __ldg(brows + r) : __dadd_rn(0.0, pairwise_row(blk + (int64_t)r * n, m));
      run = r == 0 ? rr : __dadd_rn(run, rr);
      cur = __ddiv_rn(run, bsum);
      if (cur > s3 || r == m - 1) {
        jin = r;
        rowj = rr;
        break;
      }
      prev = cur;
    }
    fv = residual(s3, jin > 0 ? prev : 0.0, cur);
  }
  int iin = invert_cumsum(blk + (int64_t)jin * n, 1, m, rowj, s4, &fu);
  int gj = bj * m + jin, gi = bi * m + iin;
  octa_uv_to_dir_k((gi + fu) / n, (gj + fv) / n, wx, wy, wz);
}

// cosine_dir (_kernels.pyx:830-843)
__device__ __forceinline__ void cosine_dir(double nx, double ny, double nz, double u1, double u2,
                                           double* ox, double* oy, double* oz) {
  double r = sqrt(u1);
  double phi = 2.0 * WFPG_PI * u2;
  double sp, cp;
  sincos(phi, &sp, &cp);
  double x = r * cp, y = r * sp;
  double z = sqrt(fmax(1.0 - u1, 0.0));
  double s = copysign(1.0, nz);
  double a = -1.0 / (s + nz);
  double b = nx * ny * a;
  *ox = x * (1.0 + s * nx * nx * a) + y * b + z * nx;
  *oy = x * (s * b) + y * (s + ny * ny * a) + z * ny;
  *oz = x * (-s * nx) + y * (-ny) + z * nz;
}

struct PathsView {
  double* ray_o;
  double* ray_d;
  double* beta;
  double* radiance;
  const uint64_t* key;
  uint64_t* ctr;
  uint8_t* alive;
  double* prev_pdf;
  double* rec_pos;
  double* rec_T;
  double* emit_le;
  int32_t* emit_depth;
  uint8_t* n_rec;  // optional: deepest record slot written
  int32_t rec_depths;
  int64_t rec_sp, rec_sd;  // record strides (doubles) per path and per depth
};

// shade_one (_kernels.pyx:905-1161) for path p.
__device__ void shade_path(int64_t p, int depth, const SceneView& sa, const GuideView& g,
                           const PathsView& P, const double* hit_t, const int32_t* hit_tri,
                           const int32_t* bin_slot, bool rr_enabled, int rr_depth);

}  // namespace wfpg

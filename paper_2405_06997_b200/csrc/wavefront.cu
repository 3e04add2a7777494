// Item 5 — wavefront stages: ray generation (_kernels.pyx:764-795), nearest /
// any-hit queue kernels (:502-555) and the per-depth shading step with NEE,
// one-sample MIS and guided / product sampling (:905-1253).
#include "prims.cuh"
#include "shade.cuh"
#include "wavefront.cuh"

namespace wfpg {

// ---------------------------------------------------------------------------
// camera rays
// ---------------------------------------------------------------------------
__device__ __forceinline__ void camera_ray(const CameraView& c, uint64_t key, int64_t pix,
                                           double* o, double* d) {
  double jx = u01(key, 0), jy = u01(key, 1);
  double aspect = (double)c.width / (double)c.height;
  double sx = (2.0 * ((double)(pix % c.width) + jx) / c.width - 1.0) * c.tan_half * aspect;
  double sy = (1.0 - 2.0 * ((double)(pix / c.width) + jy) / c.height) * c.tan_half;
  double dx = c.fwd[0] + sx * c.right[0] + sy * c.up[0];
  double dy = c.fwd[1] + sx * c.right[1] + sy * c.up[1];
  double dz = c.fwd[2] + sx * c.right[2] + sy * c.up[2];
  double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  o[0] = c.pos[0];
  o[1] = c.pos[1];
  o[2] = c.pos[2];
  d[0] = dx * inv;
  d[1] = dy * inv;
  d[2] = dz * inv;
}

__global__ void k_camera(CameraView c, const uint64_t* __restrict__ keys,
                         const int64_t* __restrict__ pixels, int64_t n, double* __restrict__ oo,
                         double* __restrict__ od) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    camera_ray(c, keys[i], pixels[i], oo + 3 * i, od + 3 * i);
}

// Pass initialisation (wavefront.py:211-219): keys, camera rays, ctr = 2,
// beta = 1, radiance = 0, alive, prev_pdf = -1, records, emitter slots.
// Tiles of 256 paths per block: the (P,3) arrays are written as contiguous
// runs of 768 doubles (directions staged in shared memory) instead of
// 24-byte-strided per-thread stores.
constexpr int kInitTile = 256;
__global__ void __launch_bounds__(kInitTile) k_init_paths(CameraView c, PathsView P,
                                                          int64_t n_paths, int64_t n_pix,
                                                          int64_t n_img, int64_t pix0,
                                                          const int64_t* __restrict__ sample_dev,
                                                          const int64_t* __restrict__ sample_list,
                                                          uint64_t seed) {
  __shared__ double sdir[3 * kInitTile];
  const int64_t sample0 = *sample_dev;
  for (int64_t base = (int64_t)blockIdx.x * kInitTile; base < n_paths;
       base += (int64_t)gridDim.x * kInitTile) {
    const int64_t p = base + threadIdx.x;
    const int m = (int)(n_paths - base < kInitTile ? n_paths - base : kInitTile);
    if (p < n_paths) {
      int64_t pix = pix0 + p % n_pix;  // global pixel index
      int64_t sample = sample_list ? sample_list[p / n_pix] : sample0 + p / n_pix;
      uint64_t key = stream_key(seed, (uint64_t)(sample * n_img + pix) * 4u);
      const_cast<uint64_t*>(P.key)[p] = key;
      double o[3];
      camera_ray(c, key, pix, o, sdir + 3 * threadIdx.x);
      P.ctr[p] = 2;
      P.alive[p] = 1;
      P.prev_pdf[p] = -1.0;
      P.emit_depth[p] = 0;
      if (P.n_rec) P.n_rec[p] = 0;
      double* rp = P.rec_pos + p * P.rec_sp;  // slot 0; zeroed by the launcher unless n_rec
      rp[0] = c.pos[0];
      rp[1] = c.pos[1];
      rp[2] = c.pos[2];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * m; e += kInitTile) {
      const int64_t g = 3 * base + e;
      P.ray_d[g] = sdir[e];
      P.ray_o[g] = c.pos[e % 3];
      P.beta[g] = 1.0;
      P.radiance[g] = 0.0;
      P.emit_le[g] = 0.0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// intersection queues
// ---------------------------------------------------------------------------
// Nearest hit for rays i < n (or for the active queue when `active` != NULL).
__global__ void k_intersect(SceneView s, const double* __restrict__ orig,
                            const double* __restrict__ dirs, const int32_t* __restrict__ active,
                            int64_t n_max, const int32_t* __restrict__ n_dev, double tmin,
                            double* __restrict__ out_t, int32_t* __restrict__ out_tri,
                            int inf_on_miss) {
  extern __shared__ TriRec smt[];
  if (s.brute) load_tris_smem(s, smt);
  __syncthreads();
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = active ? active[i] : i;
    double bt;
    int32_t id;
    ray_nearest(s, smt, orig[3 * r], orig[3 * r + 1], orig[3 * r + 2], dirs[3 * r],
                dirs[3 * r + 1], dirs[3 * r + 2], tmin, &bt, &id);
    out_t[r] = (id < 0 && inf_on_miss) ? __longlong_as_double(0x7ff0000000000000ll) : bt;
    out_tri[r] = id;
  }
}

__global__ void k_occluded(SceneView s, const double* __restrict__ orig,
                           const double* __restrict__ dirs, int64_t n, double tmin,
                           const double* __restrict__ tmax, uint8_t* __restrict__ out) {
  extern __shared__ TriRec smt[];
  if (s.brute) load_tris_smem(s, smt);
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool occ = s.brute ? brute_occluded(smt, s.n_tris, orig[3 * i], orig[3 * i + 1],
                                        orig[3 * i + 2], dirs[3 * i], dirs[3 * i + 1],
                                        dirs[3 * i + 2], tmin, tmax[i])
                       : bvh_occluded(s, orig[3 * i], orig[3 * i + 1], orig[3 * i + 2],
                                      dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], tmin,
                                      tmax[i]);
    out[i] = occ ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// shading
// ---------------------------------------------------------------------------
// BRUTE: shadow rays by brute force over the shared-memory triangles (small
// scenes), else BVH traversal; separate instantiations keep the BVH
// traversal's registers and stack out of the small-scene kernel
template <bool BRUTE, int MODE>
__device__ __forceinline__ void shade_path(int64_t p, int depth, const SceneView& sa,
                                           const GuideView& g, const PathsView& P,
                                           const double* hit_t, const int32_t* hit_tri,
                                           const int32_t* bin_slot, bool rr_enabled, int rr_depth,
                                           const TriRec* smt) {
  int32_t tri = hit_tri[p];
  if (tri < 0) {
    P.alive[p] = 0;
    return;
  }
  double* ro = P.ray_o + 3 * p;
  double* rd = P.ray_d + 3 * p;
  double* beta = P.beta + 3 * p;
  double* rad = P.radiance + 3 * p;
  const double t = hit_t[p];
  const double dx = rd[0], dy = rd[1], dz = rd[2];
  const double px = ro[0] + t * dx, py = ro[1] + t * dy, pz = ro[2] + t * dz;
  {
    int64_t rb = p * P.rec_sp + depth * P.rec_sd;
    P.rec_pos[rb] = px;
    P.rec_pos[rb + 1] = py;
    P.rec_pos[rb + 2] = pz;
    P.rec_T[rb] = beta[0];
    P.rec_T[rb + 1] = beta[1];
    P.rec_T[rb + 2] = beta[2];
    if (P.n_rec && P.n_rec[p] < depth) P.n_rec[p] = (uint8_t)depth;
  }
  const int mid = sa.tri_mat[tri];
  const int kind = sa.mat_kind[mid];
  const double ngx = sa.normals[3 * tri], ngy = sa.normals[3 * tri + 1],
               ngz = sa.normals[3 * tri + 2];
  const double cos_in = -(ngx * dx + ngy * dy + ngz * dz);
  const double* mrgb = sa.mat_rgb + 3 * mid;

  if (kind == 2) {  // emitter: terminal, MIS against NEE
    double lx = 0.0, ly = 0.0, lz = 0.0;
    if (cos_in > 0.0) {
      lx = mrgb[0];
      ly = mrgb[1];
      lz = mrgb[2];
    }
    double w = 1.0;
    double pp = P.prev_pdf[p];
    if (pp >= 0.0 && cos_in > 1e-9) {
      double pl = t * t / (sa.em_area * cos_in);
      w = pp / (pp + pl);
    }
    rad[0] += beta[0] * w * lx;
    rad[1] += beta[1] * w * ly;
    rad[2] += beta[2] * w * lz;
    P.emit_le[3 * p] = lx;
    P.emit_le[3 * p + 1] = ly;
    P.emit_le[3 * p + 2] = lz;
    P.emit_depth[p] = depth;
    P.alive[p] = 0;
    return;
  }
  if (kind == 1) {  // ideal mirror
    if (cos_in == 0.0) {
      P.alive[p] = 0;
      return;
    }
    double flip = cos_in > 0.0 ? 1.0 : -1.0;
    double nx = ngx * flip, ny = ngy * flip, nz = ngz * flip;
    double w = -dx * nx + -dy * ny + -dz * nz;
    beta[0] *= mrgb[0];
    beta[1] *= mrgb[1];
    beta[2] *= mrgb[2];
    ro[0] = px;
    ro[1] = py;
    ro[2] = pz;
    rd[0] = 2.0 * w * nx + dx;
    rd[1] = 2.0 * w * ny + dy;
    rd[2] = 2.0 * w * nz + dz;
    P.prev_pdf[p] = -1.0;
    return;
  }

  // lambert
  const bool grazing = cos_in == 0.0;
  const double flip = cos_in >= 0.0 ? 1.0 : -1.0;
  const double nsx = ngx * flip, nsy = ngy * flip, nsz = ngz * flip;
  const double alx = mrgb[0], aly = mrgb[1], alz = mrgb[2];
  const uint64_t kk = P.key[p];
  uint64_t c = P.ctr[p];
  const int slot = (MODE > 0 && bin_slot) ? bin_slot[p] : -1;
  const bool guided = slot >= 0;

  // product layer (_kernels.pyx:1003-1019): built after the shadow ray (a
  // pure function of the path's bin, n_s and albedo) so its registers are
  // not live across the occlusion loop
  ProductLayer layer;
  bool have_layer = false;

  // ---- next-event estimation (2 draws) ----
  {
    double u1 = u01(kk, c), u2 = u01(kk, c + 1);
    c += 2;
    int li = upper_bound_d(sa.em_cdf, sa.n_emit, u1);
    int ltri = sa.em_tris[li];
    double b0 = li > 0 ? sa.em_cdf[li - 1] : 0.0;
    double su = sa.em_cdf[li] - b0;
    double b1 = su > 0.0 ? (u1 - b0) / su : 0.0;
    if (b1 > 1.0 - 1e-12) b1 = 1.0 - 1e-12;
    if (b1 < 0.0) b1 = 0.0;
    su = sqrt(b1);
    double aa = 1.0 - su, bb = u2 * su;
    const double* lv0 = sa.v0 + 3 * ltri;
    const double* le1 = sa.e1 + 3 * ltri;
    const double* le2 = sa.e2 + 3 * ltri;
    double lpx = lv0[0] + aa * le1[0] + bb * le2[0];
    double lpy = lv0[1] + aa * le1[1] + bb * le2[1];
    double lpz = lv0[2] + aa * le1[2] + bb * le2[2];
    const double* ln = sa.normals + 3 * ltri;
    const double* le = sa.mat_rgb + 3 * sa.tri_mat[ltri];
    double ex = lpx - px, ey = lpy - py, ez = lpz - pz;
    double dist = sqrt(ex * ex + ey * ey + ez * ez);
    if (dist > 2.0 * sa.ray_eps) {
      double lx = ex / dist, ly = ey / dist, lz = ez / dist;
      double cos_l = -(ln[0] * lx + ln[1] * ly + ln[2] * lz);
      double cos_s = nsx * lx + nsy * ly + nsz * lz;
      if (cos_l > 1e-9 && cos_s > 0.0 && !grazing && le[0] + le[1] + le[2] > 0.0) {
        double pl = dist * dist / (sa.em_area * cos_l);
        // the guide-table entry of the light direction (plain guiding) is
        // requested before the shadow ray so its DRAM latency overlaps it
        int nci = 0, ncj = 0;
        if (MODE == 1 && guided) {
          cell_of(g.n, lx, ly, lz, &nci, &ncj);
          prefetch_l2(g.vals + ((int64_t)slot * g.n + ncj) * g.n + nci);
        }
        // any-hit: brute force over the triangles in shared memory for small
        // scenes (the hit / no-hit answer does not depend on the traversal)
        bool blocked = BRUTE ? brute_occluded(smt, sa.n_tris, px, py, pz, lx, ly, lz,
                                              sa.ray_eps, dist - sa.ray_eps)
                             : bvh_occluded(sa, px, py, pz, lx, ly, lz, sa.ray_eps,
                                            dist - sa.ray_eps);
        if (!blocked) {
          double p_cont;
          if (guided) {
            if (MODE == 2) {
              product_layer(g, slot, nsx, nsy, nsz, alx, aly, alz, &layer);
              have_layer = true;
            }
            double pg = MODE == 1 ? pdf_plain_cell(g, slot, nci, ncj)
                                    : pdf_product(g, slot, layer, lx, ly, lz);
            p_cont = 0.5 * pg + 0.5 * (cos_s / WFPG_PI);
          } else {
            p_cont = cos_s / WFPG_PI;
          }
          double w = pl / (pl + p_cont);
          double scale = (cos_s * w / pl) / WFPG_PI;
          rad[0] += beta[0] * alx * scale * le[0];
          rad[1] += beta[1] * aly * scale * le[1];
          rad[2] += beta[2] * alz * scale * le[2];
        }
      }
    }
  }

  // ---- optional russian roulette ----
  bool rr_alive = true;
  if (rr_enabled && depth >= rr_depth) {
    double u_rr = u01(kk, c);
    c += 1;
    double q = fmax(fmax(beta[0], beta[1]), beta[2]);
    if (q > 1.0) q = 1.0;
    if (q < 0.05) q = 0.05;
    if (u_rr < q) {
      beta[0] /= q;
      beta[1] /= q;
      beta[2] /= q;
    } else {
      rr_alive = false;
    }
  }

  // ---- continuation ----
  double wx = 0.0, wy = 0.0, wz = 1.0, cos_rel, pdf_mix;
  if (MODE == 2 && guided && !have_layer)
    product_layer(g, slot, nsx, nsy, nsz, alx, aly, alz, &layer);
  if (guided) {
    double coin = u01(kk, c);
    c += 1;
    if (coin < 0.5) {
      if (MODE == 1) {
        double s1 = u01(kk, c), s2 = u01(kk, c + 1);
        c += 2;
        sample_plain(g, slot, s1, s2, &wx, &wy, &wz);
      } else {
        double s1 = u01(kk, c), s2 = u01(kk, c + 1), s3 = u01(kk, c + 2), s4 = u01(kk, c + 3);
        c += 4;
        sample_product(g, slot, layer, s1, s2, s3, s4, &wx, &wy, &wz);
      }
    } else {
      double s1 = u01(kk, c), s2 = u01(kk, c + 1);
      c += 2;
      cosine_dir(nsx, nsy, nsz, s1, s2, &wx, &wy, &wz);
    }
    cos_rel = wx * nsx + wy * nsy + wz * nsz;
    double pg = MODE == 1 ? pdf_plain(g, slot, wx, wy, wz)
                            : pdf_product(g, slot, layer, wx, wy, wz);
    double pb = fmax(cos_rel, 0.0) / WFPG_PI;
    pdf_mix = 0.5 * pg + 0.5 * pb;
  } else {
    double s1 = u01(kk, c), s2 = u01(kk, c + 1);
    c += 2;
    cosine_dir(nsx, nsy, nsz, s1, s2, &wx, &wy, &wz);
    cos_rel = wx * nsx + wy * nsy + wz * nsz;
    pdf_mix = fmax(cos_rel, 0.0) / WFPG_PI;
  }

  if (rr_alive && cos_rel > 0.0 && pdf_mix > 0.0 && !grazing) {
    double factor = (cos_rel / pdf_mix) / WFPG_PI;
    beta[0] *= alx * factor;
    beta[1] *= aly * factor;
    beta[2] *= alz * factor;
    P.alive[p] = (beta[0] > 0.0 || beta[1] > 0.0 || beta[2] > 0.0) ? 1 : 0;
  } else {
    beta[0] = beta[1] = beta[2] = 0.0;
    P.alive[p] = 0;
  }
  ro[0] = px;
  ro[1] = py;
  ro[2] = pz;
  rd[0] = wx;
  rd[1] = wy;
  rd[2] = wz;
  P.prev_pdf[p] = pdf_mix;
  P.ctr[p] = c;
}

// MODE: 0 unguided, 1 plain guiding, 2 product guiding (GuideView.mode) — one
// instantiation each, so the plain kernel carries no product-layer registers
template <bool BRUTE, int MODE>
__global__ void __launch_bounds__(256, 3) k_shade(SceneView s, GuideView g, PathsView P, int depth,
                                               const int32_t* __restrict__ active, int64_t n_max,
                                               const int32_t* __restrict__ n_dev,
                                               const double* __restrict__ hit_t,
                                               const int32_t* __restrict__ hit_tri,
                                               const int32_t* __restrict__ bin_slot, int rr,
                                               int rr_depth) {
  extern __shared__ TriRec smt_shade[];
  if (BRUTE) load_tris_smem(s, smt_shade);
  __syncthreads();
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = active ? active[i] : i;
    shade_path<BRUTE, MODE>(p, depth, s, g, P, hit_t, hit_tri, bin_slot, rr != 0, rr_depth,
                            smt_shade);
  }
}

// Nearest hit of rays that all start at one point (the pinhole camera's
// primary rays): the per-(origin, triangle) records are built once per block
// and each warp culls triangles against the bounding cone of its 32 rays
// (warp_nearest_bin, the field kernel's tracer).  Consecutive pixels share a
// warp, so most triangles are rejected without a ray test.  Small scenes only
// (records in shared memory).
__global__ void __launch_bounds__(256) k_intersect_origin(SceneView s, double ox, double oy,
                                                          double oz,
                                                          const double* __restrict__ dirs,
                                                          const int32_t* __restrict__ active,
                                                          int64_t n_max,
                                                          const int32_t* __restrict__ n_dev,
                                                          double tmin, double* __restrict__ out_t,
                                                          int32_t* __restrict__ out_tri) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TriBin* tb = reinterpret_cast<TriBin*>(smem_raw);
  for (int t = threadIdx.x; t < s.n_tris; t += blockDim.x) make_tri_bin(s, t, ox, oy, oz, tb[t]);
  __syncthreads();
  const int64_t n = dev_count(n_max, n_dev);
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  // whole warps iterate together (warp_nearest_bin shuffles over all lanes);
  // lanes past the end borrow lane 0's ray and write nothing
  for (int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane; w0 < n;
       w0 += wstride) {
    const int64_t i = w0 + lane;
    const bool valid = i < n;
    const int64_t r = valid ? (active ? active[i] : i) : 0;
    double dx = valid ? dirs[3 * r] : 0.0, dy = valid ? dirs[3 * r + 1] : 0.0,
           dz = valid ? dirs[3 * r + 2] : 0.0;
    dx = __shfl_sync(0xffffffffu, dx, valid ? lane : 0);
    dy = __shfl_sync(0xffffffffu, dy, valid ? lane : 0);
    dz = __shfl_sync(0xffffffffu, dz, valid ? lane : 0);
    double bt;
    int32_t id;
    warp_nearest_bin(tb, s.n_tris, dx, dy, dz, tmin, &bt, &id);
    if (valid) {
      out_t[r] = bt;
      out_tri[r] = id;
    }
  }
}

// ---------------------------------------------------------------------------
// internal launchers
// ---------------------------------------------------------------------------
int launch_camera_init(const CameraView& c, const PathsView& P, int64_t n_paths, int64_t n_pix,
                       int64_t n_img, int64_t pix0, const int64_t* sample0,
                       const int64_t* sample_list, uint64_t seed, cudaStream_t st) {
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_paths, 256), kNumSMs * 8));
  // depth-major records span the whole (D+1, P, 3) array
  size_t rec_bytes = P.rec_sp == 3 && P.rec_depths > 1
                         ? sizeof(double) * (size_t)P.rec_depths * (size_t)P.rec_sd
                         : sizeof(double) * 3 * (size_t)P.rec_depths * (size_t)n_paths;
  if (!P.n_rec) {  // with n_rec, slots above it are masked by the readers
    WFPG_CUDA(cudaMemsetAsync(P.rec_pos, 0, rec_bytes, st));
    WFPG_CUDA(cudaMemsetAsync(P.rec_T, 0, rec_bytes, st));
  }
  const int igrid =
      (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_paths, kInitTile), kNumSMs * 8));
  k_init_paths<<<igrid, kInitTile, 0, st>>>(c, P, n_paths, n_pix, n_img, pix0, sample0,
                                            sample_list, seed);
  WFPG_CHECK_LAUNCH("k_init_paths");
  return WFPG_OK;
}

int launch_intersect(const SceneView& s, const double* orig, const double* dirs,
                     const int32_t* active, int64_t n_max, const int32_t* n_dev, double tmin,
                     double* out_t, int32_t* out_tri, bool inf_on_miss, cudaStream_t st) {
  if (n_max <= 0) return WFPG_OK;
  size_t smem = s.brute ? sizeof(TriRec) * s.n_tris : 0;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
  k_intersect<<<grid, 256, smem, st>>>(s, orig, dirs, active, n_max, n_dev, tmin, out_t, out_tri,
                                       inf_on_miss ? 1 : 0);
  WFPG_CHECK_LAUNCH("k_intersect");
  return WFPG_OK;
}

int launch_intersect_origin(const SceneView& s, const double* origin, const double* dirs,
                            const int32_t* active, int64_t n_max, const int32_t* n_dev,
                            double tmin, double* out_t, int32_t* out_tri, cudaStream_t st) {
  if (n_max <= 0) return WFPG_OK;
  if (!s.brute)
    return launch_intersect(s, nullptr, dirs, active, n_max, n_dev, tmin, out_t, out_tri, false,
                            st);
  size_t smem = sizeof(TriBin) * s.n_tris;
  // up to kMaxBruteTris records (72 KB) exceed the 48 KB default window
  static bool smem_opt_in = false;
  if (!smem_opt_in) {
    WFPG_CUDA(cudaFuncSetAttribute(k_intersect_origin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(TriBin) * kMaxBruteTris)));
    smem_opt_in = true;
  }
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
  k_intersect_origin<<<grid, 256, smem, st>>>(s, origin[0], origin[1], origin[2], dirs, active,
                                              n_max, n_dev, tmin, out_t, out_tri);
  WFPG_CHECK_LAUNCH("k_intersect_origin");
  return WFPG_OK;
}

int launch_shade(const SceneView& s, const GuideView& g, const PathsView& P, int depth,
                 const int32_t* active, int64_t n_max, const int32_t* n_dev, const double* hit_t,
                 const int32_t* hit_tri, const int32_t* bin_slot, bool rr, int rr_depth,
                 cudaStream_t st) {
  if (n_max <= 0) return WFPG_OK;
  if (g.mode == 2) {
    // power-of-two block area (exact reciprocal) and the upper-layer
    // directions in constant memory (product_cell)
    if (g.m < 1 || (g.m & (g.m - 1))) {
      set_error("shade: product mode needs n / 8 to be a power of two (n = %d)", g.n);
      return WFPG_ERR_ARG;
    }
    WFPG_CUDA(cudaMemcpyToSymbolAsync(c_upper_dirs, g.upper_dirs, sizeof(double) * 192, 0,
                                      cudaMemcpyDeviceToDevice, st));
  }
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
  const size_t smem = s.brute ? sizeof(TriRec) * s.n_tris : 0;
#define WFPG_SHADE_(B, M)                                                                   \
  k_shade<B, M><<<grid, 256, smem, st>>>(s, g, P, depth, active, n_max, n_dev, hit_t, hit_tri, \
                                         bin_slot, rr ? 1 : 0, rr_depth)
  const int mode = g.mode == 1 ? 1 : (g.mode == 2 ? 2 : 0);
  if (s.brute) {
    if (mode == 1) WFPG_SHADE_(true, 1);
    else if (mode == 2) WFPG_SHADE_(true, 2);
    else WFPG_SHADE_(true, 0);
  } else {
    if (mode == 1) WFPG_SHADE_(false, 1);
    else if (mode == 2) WFPG_SHADE_(false, 2);
    else WFPG_SHADE_(false, 0);
  }
#undef WFPG_SHADE_
  WFPG_CHECK_LAUNCH("k_shade");
  return WFPG_OK;
}

PathsView make_paths_view(const wfpg_paths* p) {
  PathsView v;
  v.ray_o = p->ray_o;
  v.ray_d = p->ray_d;
  v.beta = p->beta;
  v.radiance = p->radiance;
  v.key = p->key;
  v.ctr = p->ctr;
  v.alive = p->alive;
  v.prev_pdf = p->prev_pdf;
  v.rec_pos = p->rec_pos;
  v.n_rec = p->n_rec;
  v.rec_T = p->rec_T;
  v.emit_le = p->emit_le;
  v.emit_depth = p->emit_depth;
  v.rec_depths = p->max_depth + 1;
  v.rec_sp = p->rec_depth_major ? 3 : 3 * (int64_t)v.rec_depths;
  v.rec_sd = p->rec_depth_major ? 3 * p->n : 3;
  return v;
}

CameraView make_camera_view(const wfpg_camera* c) {
  CameraView v;
  for (int k = 0; k < 3; ++k) {
    v.pos[k] = c->position[k];
    v.fwd[k] = c->forward[k];
    v.right[k] = c->right[k];
    v.up[k] = c->up[k];
  }
  v.tan_half = c->tan_half;
  v.width = c->width;
  v.height = c->height;
  return v;
}

GuideView make_guide_view(const wfpg_guide* g) {
  GuideView v{};
  if (!g) return v;
  v.mode = g->mode;
  v.n = g->n;
  v.m = g->n / 8;
  v.eps = g->eps;
  v.pdf_scale = (double)(g->n * g->n) / (4.0 * WFPG_PI);
  v.vals = g->vals;
  v.row_sum = g->row_sum;
  v.marg = g->marg;
  v.total = g->total;
  v.block_sums = g->block_sums;
  v.upper_dirs = g->upper_dirs;
  v.cum = g->cum;
  v.block_rows = g->mode == 2 ? g->block_rows : nullptr;
  return v;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" int wfpg_camera_rays(const wfpg_camera* cam, const uint64_t* keys,
                                const int64_t* pixels, int64_t n, double* out_o, double* out_d,
                                void* stream) {
  if (!cam || n < 0 || (n > 0 && (!keys || !pixels || !out_o || !out_d))) {
    set_error("wfpg_camera_rays: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  CameraView c = make_camera_view(cam);
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8);
  k_camera<<<grid, 256, 0, as_stream(stream)>>>(c, keys, pixels, n, out_o, out_d);
  WFPG_CHECK_LAUNCH("k_camera");
  return WFPG_OK;
}

extern "C" int wfpg_intersect(const wfpg_scene* scene, const double* origins, const double* dirs,
                              int64_t n, double t_min, double* out_t, int32_t* out_tri,
                              void* stream) {
  if (!scene || n < 0 || (n > 0 && (!origins || !dirs || !out_t || !out_tri))) {
    set_error("wfpg_intersect: bad arguments");
    return WFPG_ERR_ARG;
  }
  return launch_intersect(make_scene_view(scene), origins, dirs, nullptr, n, nullptr, t_min,
                          out_t, out_tri, true, as_stream(stream));
}

extern "C" int wfpg_occluded(const wfpg_scene* scene, const double* origins, const double* dirs,
                             int64_t n, double t_min, const double* t_max, uint8_t* out,
                             void* stream) {
  if (!scene || n < 0 || (n > 0 && (!origins || !dirs || !t_max || !out))) {
    set_error("wfpg_occluded: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (n == 0) return WFPG_OK;
  SceneView s = make_scene_view(scene);
  size_t smem = s.brute ? sizeof(TriRec) * s.n_tris : 0;
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8);
  k_occluded<<<grid, 256, smem, as_stream(stream)>>>(s, origins, dirs, n, t_min, t_max, out);
  WFPG_CHECK_LAUNCH("k_occluded");
  return WFPG_OK;
}

extern "C" int wfpg_shade_depth(const wfpg_scene* scene, wfpg_paths* paths, int32_t depth,
                                const int32_t* active, int64_t n_active,
                                const int32_t* n_active_dev, const double* hit_t,
                                const int32_t* hit_tri, const wfpg_guide* guide,
                                const int32_t* bin_slot, int32_t rr_enabled, int32_t rr_depth,
                                void* stream) {
  if (!scene || !paths || depth < 1 || depth > paths->max_depth || !hit_t || !hit_tri) {
    set_error("wfpg_shade_depth: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (guide && guide->mode == 2 && (!guide->upper_dirs || !guide->block_sums)) {
    set_error("wfpg_shade_depth: product mode needs block sums and upper-layer directions");
    return WFPG_ERR_ARG;
  }
  GuideView g = make_guide_view(guide);
  return launch_shade(make_scene_view(scene), g, make_paths_view(paths), depth, active, n_active,
                      n_active_dev, hit_t, hit_tri, bin_slot, rr_enabled != 0, rr_depth,
                      as_stream(stream));
}

// Internal wavefront launchers shared by the ABI entry points and the pass driver.
#pragma once
#include "shade.cuh"

namespace wfpg {

struct CameraView {
  double pos[3], fwd[3], right[3], up[3];
  double tan_half;
  int32_t width, height;
};

PathsView make_paths_view(const wfpg_paths* p);
CameraView make_camera_view(const wfpg_camera* c);
GuideView make_guide_view(const wfpg_guide* g);

int launch_camera_init(const CameraView& c, const PathsView& P, int64_t n_paths, int64_t n_pix,
                       int64_t n_img, int64_t pix0, const int64_t* sample0,
                       const int64_t* sample_list, uint64_t seed,
                       cudaStream_t st);
// primary rays from one origin (host pointer to 3 doubles); brute-force scenes
// use the warp-culled tracer, others fall back to launch_intersect (which
// then needs per-ray origins: only call it with brute scenes)
int launch_intersect_origin(const SceneView& s, const double* origin, const double* dirs,
                            const int32_t* active, int64_t n_max, const int32_t* n_dev,
                            double tmin, double* out_t, int32_t* out_tri, cudaStream_t st);
int launch_intersect(const SceneView& s, const double* orig, const double* dirs,
                     const int32_t* active, int64_t n_max, const int32_t* n_dev, double tmin,
                     double* out_t, int32_t* out_tri, bool inf_on_miss, cudaStream_t st);
int launch_shade(const SceneView& s, const GuideView& g, const PathsView& P, int depth,
                 const int32_t* active, int64_t n_max, const int32_t* n_dev, const double* hit_t,
                 const int32_t* hit_tri, const int32_t* bin_slot, bool rr, int rr_depth,
                 cudaStream_t st);

}  // namespace wfpg

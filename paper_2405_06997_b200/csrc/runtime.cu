// Library runtime: error reporting, launch accounting, ABI version.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace wfpg {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return WFPG_ERR_CUDA;
}

void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace wfpg

extern "C" int wfpg_abi_version(void) { return WFPG_ABI_VERSION; }

extern "C" int wfpg_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return WFPG_OK;
  if (!dst || !src) {
    wfpg::set_error("wfpg_memcpy: bad arguments");
    return WFPG_ERR_ARG;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? WFPG_OK : wfpg::cuda_status(e, "wfpg_memcpy");
}
extern "C" const char* wfpg_last_error(void) { return wfpg::g_err; }
extern "C" uint64_t wfpg_launch_count(void) {
  return wfpg::g_launches.load(std::memory_order_relaxed);
}

// struct layout table (generated from include/wfpg_b200.h field lists)
#include <cstddef>
#include <cstring>

namespace {
struct FieldOff { const char* name; int64_t off; };
const FieldOff k_wfpg_scene[] = {
    {"n_tris", (int64_t)offsetof(wfpg_scene, n_tris)},
    {"v0", (int64_t)offsetof(wfpg_scene, v0)},
    {"v1", (int64_t)offsetof(wfpg_scene, v1)},
    {"v2", (int64_t)offsetof(wfpg_scene, v2)},
    {"e1", (int64_t)offsetof(wfpg_scene, e1)},
    {"e2", (int64_t)offsetof(wfpg_scene, e2)},
    {"normals", (int64_t)offsetof(wfpg_scene, normals)},
    {"tri_mat", (int64_t)offsetof(wfpg_scene, tri_mat)},
    {"mat_kind", (int64_t)offsetof(wfpg_scene, mat_kind)},
    {"mat_rgb", (int64_t)offsetof(wfpg_scene, mat_rgb)},
    {"n_mats", (int64_t)offsetof(wfpg_scene, n_mats)},
    {"n_emit", (int64_t)offsetof(wfpg_scene, n_emit)},
    {"emitter_cdf", (int64_t)offsetof(wfpg_scene, emitter_cdf)},
    {"emitter_tris", (int64_t)offsetof(wfpg_scene, emitter_tris)},
    {"emitter_area", (int64_t)offsetof(wfpg_scene, emitter_area)},
    {"ray_eps", (int64_t)offsetof(wfpg_scene, ray_eps)},
    {"bbox_lo", (int64_t)offsetof(wfpg_scene, bbox_lo)},
    {"bbox_hi", (int64_t)offsetof(wfpg_scene, bbox_hi)},
    {"bvh_nodes", (int64_t)offsetof(wfpg_scene, bvh_nodes)},
    {"bvh_lo", (int64_t)offsetof(wfpg_scene, bvh_lo)},
    {"bvh_hi", (int64_t)offsetof(wfpg_scene, bvh_hi)},
    {"bvh_left", (int64_t)offsetof(wfpg_scene, bvh_left)},
    {"bvh_right", (int64_t)offsetof(wfpg_scene, bvh_right)},
    {"bvh_count", (int64_t)offsetof(wfpg_scene, bvh_count)},
    {"bvh_order", (int64_t)offsetof(wfpg_scene, bvh_order)},
    {"brute", (int64_t)offsetof(wfpg_scene, brute)},
    {"bvh_box_f32", (int64_t)offsetof(wfpg_scene, bvh_box_f32)},
    {nullptr, 0}};
const FieldOff k_wfpg_camera[] = {
    {"position", (int64_t)offsetof(wfpg_camera, position)},
    {"forward", (int64_t)offsetof(wfpg_camera, forward)},
    {"right", (int64_t)offsetof(wfpg_camera, right)},
    {"up", (int64_t)offsetof(wfpg_camera, up)},
    {"tan_half", (int64_t)offsetof(wfpg_camera, tan_half)},
    {"width", (int64_t)offsetof(wfpg_camera, width)},
    {"height", (int64_t)offsetof(wfpg_camera, height)},
    {nullptr, 0}};
const FieldOff k_wfpg_svo[] = {
    {"depth", (int64_t)offsetof(wfpg_svo, depth)},
    {"resolution", (int64_t)offsetof(wfpg_svo, resolution)},
    {"n_nodes", (int64_t)offsetof(wfpg_svo, n_nodes)},
    {"lo", (int64_t)offsetof(wfpg_svo, lo)},
    {"size", (int64_t)offsetof(wfpg_svo, size)},
    {"level_off", (int64_t)offsetof(wfpg_svo, level_off)},
    {"codes", (int64_t)offsetof(wfpg_svo, codes)},
    {"child_base", (int64_t)offsetof(wfpg_svo, child_base)},
    {"child_mask", (int64_t)offsetof(wfpg_svo, child_mask)},
    {"parent", (int64_t)offsetof(wfpg_svo, parent)},
    {"node_desc", (int64_t)offsetof(wfpg_svo, node_desc)},
    {"normal", (int64_t)offsetof(wfpg_svo, normal)},
    {"sum_a", (int64_t)offsetof(wfpg_svo, sum_a)},
    {"sum_b", (int64_t)offsetof(wfpg_svo, sum_b)},
    {"weight_a", (int64_t)offsetof(wfpg_svo, weight_a)},
    {"weight_b", (int64_t)offsetof(wfpg_svo, weight_b)},
    {"mean_a", (int64_t)offsetof(wfpg_svo, mean_a)},
    {"mean_b", (int64_t)offsetof(wfpg_svo, mean_b)},
    {"counter", (int64_t)offsetof(wfpg_svo, counter)},
    {"top_index", (int64_t)offsetof(wfpg_svo, top_index)},
    {"top_level", (int64_t)offsetof(wfpg_svo, top_level)},
    {nullptr, 0}};
const FieldOff k_wfpg_paths[] = {
    {"n", (int64_t)offsetof(wfpg_paths, n)},
    {"max_depth", (int64_t)offsetof(wfpg_paths, max_depth)},
    {"ray_o", (int64_t)offsetof(wfpg_paths, ray_o)},
    {"ray_d", (int64_t)offsetof(wfpg_paths, ray_d)},
    {"beta", (int64_t)offsetof(wfpg_paths, beta)},
    {"radiance", (int64_t)offsetof(wfpg_paths, radiance)},
    {"key", (int64_t)offsetof(wfpg_paths, key)},
    {"ctr", (int64_t)offsetof(wfpg_paths, ctr)},
    {"alive", (int64_t)offsetof(wfpg_paths, alive)},
    {"prev_pdf", (int64_t)offsetof(wfpg_paths, prev_pdf)},
    {"rec_pos", (int64_t)offsetof(wfpg_paths, rec_pos)},
    {"rec_T", (int64_t)offsetof(wfpg_paths, rec_T)},
    {"emit_le", (int64_t)offsetof(wfpg_paths, emit_le)},
    {"emit_depth", (int64_t)offsetof(wfpg_paths, emit_depth)},
    {"n_rec", (int64_t)offsetof(wfpg_paths, n_rec)},
    {nullptr, 0}};
const FieldOff k_wfpg_guide[] = {
    {"mode", (int64_t)offsetof(wfpg_guide, mode)},
    {"n", (int64_t)offsetof(wfpg_guide, n)},
    {"capacity", (int64_t)offsetof(wfpg_guide, capacity)},
    {"eps", (int64_t)offsetof(wfpg_guide, eps)},
    {"vals", (int64_t)offsetof(wfpg_guide, vals)},
    {"row_sum", (int64_t)offsetof(wfpg_guide, row_sum)},
    {"marg", (int64_t)offsetof(wfpg_guide, marg)},
    {"total", (int64_t)offsetof(wfpg_guide, total)},
    {"block_sums", (int64_t)offsetof(wfpg_guide, block_sums)},
    {"n_bins", (int64_t)offsetof(wfpg_guide, n_bins)},
    {"upper_dirs", (int64_t)offsetof(wfpg_guide, upper_dirs)},
    {"cum", (int64_t)offsetof(wfpg_guide, cum)},
    {nullptr, 0}};
const FieldOff k_wfpg_pass_config[] = {
    {"l_min", (int64_t)offsetof(wfpg_pass_config, l_min)},
    {"c_ray", (int64_t)offsetof(wfpg_pass_config, c_ray)},
    {"field_res", (int64_t)offsetof(wfpg_pass_config, field_res)},
    {"guided_depths", (int64_t)offsetof(wfpg_pass_config, guided_depths)},
    {"max_depth", (int64_t)offsetof(wfpg_pass_config, max_depth)},
    {"product", (int64_t)offsetof(wfpg_pass_config, product)},
    {"jitter", (int64_t)offsetof(wfpg_pass_config, jitter)},
    {"blur_sigma", (int64_t)offsetof(wfpg_pass_config, blur_sigma)},
    {"epsilon", (int64_t)offsetof(wfpg_pass_config, epsilon)},
    {"russian_roulette", (int64_t)offsetof(wfpg_pass_config, russian_roulette)},
    {"rr_depth", (int64_t)offsetof(wfpg_pass_config, rr_depth)},
    {"seed", (int64_t)offsetof(wfpg_pass_config, seed)},
    {"sample_index", (int64_t)offsetof(wfpg_pass_config, sample_index)},
    {"n_samples", (int64_t)offsetof(wfpg_pass_config, n_samples)},
    {"deterministic", (int64_t)offsetof(wfpg_pass_config, deterministic)},
    {"blur_radius", (int64_t)offsetof(wfpg_pass_config, blur_radius)},
    {"blur_w", (int64_t)offsetof(wfpg_pass_config, blur_w)},
    {"upper_dirs", (int64_t)offsetof(wfpg_pass_config, upper_dirs)},
    {"pixel_offset", (int64_t)offsetof(wfpg_pass_config, pixel_offset)},
    {"n_pixels", (int64_t)offsetof(wfpg_pass_config, n_pixels)},
    {"leaf_acc", (int64_t)offsetof(wfpg_pass_config, leaf_acc)},
    {"use_graph", (int64_t)offsetof(wfpg_pass_config, use_graph)},
    {"bin_image", (int64_t)offsetof(wfpg_pass_config, bin_image)},
    {"dep_leaf", (int64_t)offsetof(wfpg_pass_config, dep_leaf)},
    {"dep_dir", (int64_t)offsetof(wfpg_pass_config, dep_dir)},
    {"dep_rad", (int64_t)offsetof(wfpg_pass_config, dep_rad)},
    {"dep_count", (int64_t)offsetof(wfpg_pass_config, dep_count)},
    {"dep_capacity", (int64_t)offsetof(wfpg_pass_config, dep_capacity)},
    {"comm", (int64_t)offsetof(wfpg_pass_config, comm)},
    {"dep_wire_capacity", (int64_t)offsetof(wfpg_pass_config, dep_wire_capacity)},
    {nullptr, 0}};
const FieldOff k_wfpg_pass_stats[] = {
    {"depths_run", (int64_t)offsetof(wfpg_pass_stats, depths_run)},
    {"bins_per_depth", (int64_t)offsetof(wfpg_pass_stats, bins_per_depth)},
    {"rays_per_depth", (int64_t)offsetof(wfpg_pass_stats, rays_per_depth)},
    {"live_per_depth", (int64_t)offsetof(wfpg_pass_stats, live_per_depth)},
    {"deposits", (int64_t)offsetof(wfpg_pass_stats, deposits)},
    {"mat_groups", (int64_t)offsetof(wfpg_pass_stats, mat_groups)},
    {nullptr, 0}};
struct StructInfo { int64_t size; const FieldOff* fields; };
const StructInfo k_structs[] = {
    {(int64_t)sizeof(wfpg_scene), k_wfpg_scene},
    {(int64_t)sizeof(wfpg_camera), k_wfpg_camera},
    {(int64_t)sizeof(wfpg_svo), k_wfpg_svo},
    {(int64_t)sizeof(wfpg_paths), k_wfpg_paths},
    {(int64_t)sizeof(wfpg_guide), k_wfpg_guide},
    {(int64_t)sizeof(wfpg_pass_config), k_wfpg_pass_config},
    {(int64_t)sizeof(wfpg_pass_stats), k_wfpg_pass_stats},
};
}  // namespace

extern "C" int64_t wfpg_abi_sizeof(int32_t struct_id) {
  if (struct_id < 0 || struct_id >= (int32_t)(sizeof(k_structs) / sizeof(k_structs[0]))) return -1;
  return k_structs[struct_id].size;
}

extern "C" int64_t wfpg_abi_offsetof(int32_t struct_id, const char* field) {
  if (!field || struct_id < 0 ||
      struct_id >= (int32_t)(sizeof(k_structs) / sizeof(k_structs[0])))
    return -1;
  for (const FieldOff* f = k_structs[struct_id].fields; f->name; ++f)
    if (std::strcmp(f->name, field) == 0) return f->off;
  return -1;
}

// Item 2 — Eq. 5 exitance update after a pass (wavefront.py:286-332):
// deposits (T_n / T_k) * L_e at every recorded vertex k of emitter-terminated
// paths, in path-major / k-ascending order, then splats them into the SVO
// leaves (deterministic or atomic) and refreshes the means bottom-up.
#include "exitance.cuh"
#include "prims.cuh"
#include "svo_query.cuh"

namespace wfpg {

__device__ __forceinline__ bool deposit_ok(const double* rt, int k, int64_t sd) {
  return rt[k * sd] > 0.0 && rt[k * sd + 1] > 0.0 && rt[k * sd + 2] > 0.0;
}

__global__ void k_dep_count(const int32_t* __restrict__ emit_depth,
                            const double* __restrict__ emit_le, const double* __restrict__ rec_T,
                            RecLayout rl, int64_t n, uint32_t* __restrict__ counts) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int nd = emit_depth[p];
    const double* le = emit_le + 3 * p;
    uint32_t c = 0;
    if (nd >= 2 && (le[0] + le[1] + le[2]) > 0.0) {
      const double* rt = rec_T + p * rl.sp;
      for (int k = 1; k < nd; ++k) c += deposit_ok(rt, k, rl.sd) ? 1u : 0u;
    }
    counts[p] = c;
  }
}

__global__ void k_dep_emit(SvoView v, const int32_t* __restrict__ emit_depth,
                           const double* __restrict__ emit_le, const double* __restrict__ rec_T,
                           const double* __restrict__ rec_pos, RecLayout rl, int64_t n,
                           const uint32_t* __restrict__ counts, const uint32_t* __restrict__ offs,
                           int32_t* __restrict__ leaf, double* __restrict__ dirs,
                           double* __restrict__ rad) {
  const double nudge = (v.size / v.resolution) * 1e-3;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (counts[p] == 0) continue;
    int nd = emit_depth[p];
    const double* rt = rec_T + p * rl.sp;
    const double* rp = rec_pos + p * rl.sp;
    const double* le = emit_le + 3 * p;
    const double* tn = rt + nd * rl.sd;
    uint32_t o = offs[p];
    for (int k = 1; k < nd; ++k) {
      if (!deposit_ok(rt, k, rl.sd)) continue;
      const double* tk = rt + k * rl.sd;
      double* r = rad + 3 * (int64_t)o;
      for (int c = 0; c < 3; ++c) r[c] = __dmul_rn(__ddiv_rn(tn[c], tk[c]), le[c]);
      const double* pos = rp + k * rl.sd;
      const double* prev = rp + (k - 1) * rl.sd;
      double d[3];
      for (int c = 0; c < 3; ++c) d[c] = __dsub_rn(prev[c], pos[c]);
      double nrm = norm_axis(d[0], d[1], d[2]);
      // the reference clamps the nudged point into [lo + tiny, lo + size -
      // tiny] before quantising; quantise's clamp of the cell index gives the
      // same cell for every point (truncation is monotone), so the point
      // clamp is not repeated here
      double q[3];
      for (int c = 0; c < 3; ++c) {
        d[c] = __ddiv_rn(d[c], nrm);
        q[c] = __dadd_rn(pos[c], __dmul_rn(d[c], nudge));
        dirs[3 * (int64_t)o + c] = d[c];
      }
      int32_t qx = quantise(q[0], v.lox, v.scale, v.resolution);
      int32_t qy = quantise(q[1], v.loy, v.scale, v.resolution);
      int32_t qz = quantise(q[2], v.loz, v.scale, v.resolution);
      bool pres;
      int32_t lvl;
      int32_t node = descend_view(v, qx, qy, qz, v.depth, &pres, &lvl);
      leaf[o] = pres ? node : -1;
      ++o;
    }
  }
}

size_t update_exitance_ws_bytes(int64_t n_paths, int max_depth) {
  int64_t n = n_paths > 0 ? n_paths : 1;
  int64_t m = n * (max_depth > 0 ? max_depth : 1);
  return align_up(4 * (n + 1)) * 2 + align_up(4 * m) + 2 * align_up(24 * m) + align_up(8) +
         std::max(scan_ws_bytes(n + 1), accumulate_ws_bytes(m)) + 4096;
}

int update_exitance(wfpg_svo* svo, const int32_t* emit_depth, const double* emit_le,
                    const double* rec_T, const double* rec_pos, RecLayout rl, int64_t n_paths,
                    int deterministic, int32_t* n_dep_out, Arena& ws, cudaStream_t st,
                    int propagate, uint8_t* dirty, const DepositSink* sink) {
  if (n_paths <= 0) return WFPG_OK;
  const int64_t m = n_paths * (int64_t)(rl.depths - 1 > 0 ? rl.depths - 1 : 1);
  if (sink && (sink->capacity < m || !sink->leaf || !sink->dir || !sink->rad || !sink->count)) {
    set_error("update_exitance: deposit sink needs capacity >= n_paths * max_depth (%lld)",
              (long long)m);
    return WFPG_ERR_ARG;
  }
  uint32_t* counts = ws.take<uint32_t>(n_paths + 1);
  uint32_t* offs = ws.take<uint32_t>(n_paths + 1);
  int32_t* leaf = sink ? sink->leaf : ws.take<int32_t>(m);
  double* dirs = sink ? sink->dir : ws.take<double>(3 * m);
  double* rad = sink ? sink->rad : ws.take<double>(3 * m);
  uint32_t* total = ws.take<uint32_t>(2);
  if (!ws.ok()) {
    set_error("update_exitance: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  SvoView v = make_view(svo);
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_paths, 256), kNumSMs * 8));
  k_dep_count<<<grid, 256, 0, st>>>(emit_depth, emit_le, rec_T, rl, n_paths, counts);
  WFPG_CHECK_LAUNCH("k_dep_count");
  {
    size_t mark = ws.off;
    WFPG_TRY(scan_u32(counts, offs, n_paths, nullptr, total, ws, st));
    ws.off = mark;
  }
  k_dep_emit<<<grid, 256, 0, st>>>(v, emit_depth, emit_le, rec_T, rec_pos, rl, n_paths,
                                   counts, offs, leaf, dirs, rad);
  WFPG_CHECK_LAUNCH("k_dep_emit");
  const int32_t* n_dev = reinterpret_cast<const int32_t*>(total);
  if (n_dep_out)
    WFPG_CUDA(cudaMemcpyAsync(n_dep_out, total, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  if (sink) {
    WFPG_CUDA(cudaMemcpyAsync(sink->count, total, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    return WFPG_OK;
  }
  {
    size_t mark = ws.off;
    WFPG_TRY(svo_accumulate(svo, leaf, dirs, rad, m, n_dev, deterministic, ws, st));
    ws.off = mark;
  }
  if (propagate == 2 && dirty) return svo_propagate_dirty(svo, leaf, m, n_dev, dirty, st);
  return propagate ? svo_propagate(svo, st) : WFPG_OK;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" size_t wfpg_update_exitance_workspace_bytes(int64_t n_paths, int32_t max_depth) {
  return update_exitance_ws_bytes(n_paths, max_depth) + 256;
}

extern "C" int wfpg_update_exitance(wfpg_svo* svo, const wfpg_paths* paths, int32_t deterministic,
                                    int32_t* n_deposits_dev, void* workspace, size_t ws_bytes,
                                    void* stream) {
  if (!svo || !paths || !paths->emit_depth || !paths->rec_T || !paths->rec_pos) {
    set_error("wfpg_update_exitance: bad arguments");
    return WFPG_ERR_ARG;
  }
  Arena ws(workspace, ws_bytes);
  return update_exitance(svo, paths->emit_depth, paths->emit_le, paths->rec_T, paths->rec_pos,
                         rec_layout(paths), paths->n, deterministic, n_deposits_dev, ws,
                         as_stream(stream), 1, nullptr);
}

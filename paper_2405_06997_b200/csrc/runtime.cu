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

extern "C" int wfpg_event_create(void** event) {
  if (!event) {
    wfpg::set_error("wfpg_event_create: bad arguments");
    return WFPG_ERR_ARG;
  }
  cudaEvent_t e;
  cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (err != cudaSuccess) return wfpg::cuda_status(err, "cudaEventCreateWithFlags");
  *event = (void*)e;
  return WFPG_OK;
}

extern "C" int wfpg_event_destroy(void* event) {
  if (event) cudaEventDestroy((cudaEvent_t)event);
  return WFPG_OK;
}

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

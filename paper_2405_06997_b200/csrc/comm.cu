// Multi-GPU exchange layer: the render pass's collectives
// go through a wfpg_comm, either NCCL (loaded with dlopen, so the library has
// no link-time NCCL dependency and shares the copy torch already mapped;
// its calls are enqueued on the pass stream and captured into the pass's
// CUDA graph) or a host exchange callback (tests and gloo runs: the stream is
// synchronised and the caller performs the collective on device buffers).
#include <dlfcn.h>
#include <nccl.h>

#include <vector>

#include "comm.cuh"
#include "svo_query.cuh"

namespace wfpg {

namespace {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*);
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*comm_destroy)(ncclComm_t);
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t);
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t);
  const char* (*error_string)(ncclResult_t);
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    // RTLD_NOLOAD first: reuse the NCCL the process already mapped (torch's)
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
      api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
      api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
      api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
      api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
      api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
      api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather &&
               api.all_reduce && api.error_string;
    }
  }
  return api;
}

int nccl_status(ncclResult_t r, const char* what) {
  set_error("NCCL error in %s: %s", what, nccl().error_string ? nccl().error_string(r) : "?");
  return WFPG_ERR_CUDA;
}

ncclDataType_t nccl_type(CommDtype dt) {
  switch (dt) {
    case kI32: return ncclInt32;
    case kU64: return ncclUint64;
    default: return ncclFloat64;
  }
}

size_t dtype_bytes(CommDtype dt) { return dt == kI32 ? 4 : 8; }

}  // namespace

struct Comm {
  int world = 1, rank = 0;
  int kind = 0;  // 0 NCCL, 1 host callback
  ncclComm_t nc = nullptr;
  wfpg_exchange_fn fn = nullptr;
  void* user = nullptr;
  int* status_host = nullptr;  // pinned
  cudaEvent_t done = nullptr;
  DepositPending pending;
  // scratch of the exact (overflow) exchange, grown on demand
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

int comm_world(const Comm* c) { return c ? c->world : 1; }
int comm_rank(const Comm* c) { return c ? c->rank : 0; }
bool comm_capturable(const Comm* c) { return c && c->kind == 0; }
int* comm_status_host(Comm* c) { return c->status_host; }
cudaEvent_t comm_done_event(Comm* c) { return c->done; }
DepositPending& comm_pending(Comm* c) { return c->pending; }

static int host_exchange(const Comm* c, int op, const void* send, void* recv, int64_t count,
                         CommDtype dt, cudaStream_t st) {
  WFPG_CUDA(cudaStreamSynchronize(st));
  int rc = c->fn(c->user, op, send, recv, count, (int32_t)dt, (void*)st);
  if (rc != 0) {
    set_error("host exchange callback failed (op %d, rc %d)", op, rc);
    return WFPG_ERR_CUDA;
  }
  return WFPG_OK;
}

int comm_all_gather(const Comm* c, const void* send, void* recv, int64_t count, CommDtype dt,
                    cudaStream_t st) {
  if (c->world == 1) {
    if (recv != send)
      WFPG_CUDA(cudaMemcpyAsync(recv, send, dtype_bytes(dt) * (size_t)count,
                                cudaMemcpyDeviceToDevice, st));
    return WFPG_OK;
  }
  if (c->kind == 1) return host_exchange(c, 0, send, recv, count, dt, st);
  ncclResult_t r = nccl().all_gather(send, recv, (size_t)count, nccl_type(dt), c->nc, st);
  return r == ncclSuccess ? WFPG_OK : nccl_status(r, "ncclAllGather");
}

int comm_all_reduce_sum(const Comm* c, const void* send, void* recv, int64_t count, CommDtype dt,
                        cudaStream_t st) {
  if (c->world == 1) {
    if (recv != send)
      WFPG_CUDA(cudaMemcpyAsync(recv, send, dtype_bytes(dt) * (size_t)count,
                                cudaMemcpyDeviceToDevice, st));
    return WFPG_OK;
  }
  if (c->kind == 1) return host_exchange(c, 1, send, recv, count, dt, st);
  ncclResult_t r =
      nccl().all_reduce(send, recv, (size_t)count, nccl_type(dt), ncclSum, c->nc, st);
  return r == ncclSuccess ? WFPG_OK : nccl_status(r, "ncclAllReduce");
}

// --- exact exchange of one pass's deposits (overflow of the wire capacity) ---

__global__ void k_dep_pack_all(const int32_t* __restrict__ leaf, const double* __restrict__ dir,
                               const double* __restrict__ rad, const int32_t* __restrict__ count,
                               int64_t cap, uint64_t* __restrict__ out) {
  const int64_t n = *count;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t* r = out + 7 * i;
    if (i < n) {
      r[0] = (uint64_t)(int64_t)leaf[i];
      for (int c = 0; c < 3; ++c) {
        r[1 + c] = (uint64_t)__double_as_longlong(dir[3 * i + c]);
        r[4 + c] = (uint64_t)__double_as_longlong(rad[3 * i + c]);
      }
    } else {
      r[0] = (uint64_t)(int64_t)-1;
      for (int c = 1; c < 7; ++c) r[c] = 0;
    }
  }
}

__global__ void k_dep_unpack_all(const uint64_t* __restrict__ in, const int64_t* __restrict__ cnt,
                                 int world, int64_t cap, int32_t* __restrict__ leaf,
                                 double* __restrict__ dir, double* __restrict__ rad) {
  // rank r's first cnt[r] records land at the prefix of the counts
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)world * cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cap);
    const int64_t k = i % cap;
    if (k >= cnt[r]) continue;
    int64_t o = k;
    for (int q = 0; q < r; ++q) o += cnt[q];
    const uint64_t* s = in + 7 * i;
    leaf[o] = (int32_t)(int64_t)s[0];
    for (int c = 0; c < 3; ++c) {
      dir[3 * o + c] = __longlong_as_double((long long)s[1 + c]);
      rad[3 * o + c] = __longlong_as_double((long long)s[4 + c]);
    }
  }
}

__global__ void k_count_to_i64(const int32_t* __restrict__ c, int64_t* __restrict__ out) {
  *out = (int64_t)*c;
}

int comm_settle(Comm* c) {
  NvtxRange nvtx_("wfpg_comm_settle");
  if (!c || !c->pending.active) return WFPG_OK;
  DepositPending& p = c->pending;
  p.active = false;
  WFPG_CUDA(cudaEventSynchronize(c->done));
  if (*c->status_host == 0) return WFPG_OK;  // the in-pass exchange applied everything
  // Some rank exported more deposits than the wire capacity: no rank applied
  // any of that pass's deposits (the decision is on the gathered counts, the
  // same on every rank).  Exchange the full lists now, in rank order.
  cudaStream_t st = p.stream;
  const int W = c->world;
  std::vector<int64_t> counts(W);
  int64_t* dcnt;
  int64_t* dcnt_all;
  WFPG_CUDA(cudaMallocAsync(&dcnt, sizeof(int64_t), st));
  WFPG_CUDA(cudaMallocAsync(&dcnt_all, sizeof(int64_t) * W, st));
  k_count_to_i64<<<1, 1, 0, st>>>(p.count, dcnt);
  WFPG_CHECK_LAUNCH("k_count_to_i64");
  WFPG_TRY(comm_all_gather(c, dcnt, dcnt_all, 1, kU64, st));
  WFPG_CUDA(cudaMemcpyAsync(counts.data(), dcnt_all, sizeof(int64_t) * W, cudaMemcpyDeviceToHost,
                            st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  int64_t cap = 1, total = 0;
  for (int64_t x : counts) {
    cap = std::max(cap, x);
    total += x;
  }
  const size_t pack = sizeof(uint64_t) * 7 * (size_t)cap;
  const size_t need = pack * (size_t)(W + 1) + (sizeof(int32_t) + 48) * (size_t)total +
                      accumulate_ws_bytes(total) + 8192;
  if (need > c->scratch_bytes) {
    if (c->scratch) WFPG_CUDA(cudaFree(c->scratch));
    WFPG_CUDA(cudaMalloc(&c->scratch, need));
    c->scratch_bytes = need;
  }
  Arena a(c->scratch, c->scratch_bytes);
  uint64_t* send = a.take<uint64_t>(7 * cap);
  uint64_t* recv = a.take<uint64_t>(7 * cap * W);
  int32_t* leaf = a.take<int32_t>(total);
  double* dir = a.take<double>(3 * total);
  double* rad = a.take<double>(3 * total);
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, 256), kNumSMs * 4));
  k_dep_pack_all<<<grid, 256, 0, st>>>(p.leaf, p.dir, p.rad, p.count, cap, send);
  WFPG_CHECK_LAUNCH("k_dep_pack_all");
  WFPG_TRY(comm_all_gather(c, send, recv, 7 * cap, kU64, st));
  grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap * W, 256), kNumSMs * 4));
  k_dep_unpack_all<<<grid, 256, 0, st>>>(recv, dcnt_all, W, cap, leaf, dir, rad);
  WFPG_CHECK_LAUNCH("k_dep_unpack_all");
  if (total > 0) {
    WFPG_TRY(svo_accumulate(&p.svo, leaf, dir, rad, total, nullptr, 1, a, st));
    WFPG_CUDA(cudaMemsetAsync(p.dirty, 0, (size_t)p.svo.n_nodes, st));
    WFPG_TRY(svo_propagate_dirty(&p.svo, leaf, total, nullptr, p.dirty, st));
  }
  WFPG_CUDA(cudaFreeAsync(dcnt, st));
  WFPG_CUDA(cudaFreeAsync(dcnt_all, st));
  WFPG_CUDA(cudaStreamSynchronize(st));
  *c->status_host = 0;
  return WFPG_OK;
}

static int comm_alloc_common(Comm* c) {
  WFPG_CUDA(cudaMallocHost(&c->status_host, sizeof(int)));
  *c->status_host = 0;
  WFPG_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  return WFPG_OK;
}

}  // namespace wfpg

using namespace wfpg;

extern "C" int wfpg_comm_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int wfpg_comm_nccl_unique_id(uint8_t* out) {
  if (!out) {
    set_error("wfpg_comm_nccl_unique_id: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (!nccl().ok) {
    set_error("NCCL (libnccl.so.2) is not loadable");
    return WFPG_ERR_CUDA;
  }
  ncclUniqueId id;
  ncclResult_t r = nccl().get_unique_id(&id);
  if (r != ncclSuccess) return nccl_status(r, "ncclGetUniqueId");
  memcpy(out, id.internal, sizeof(id.internal));
  return WFPG_OK;
}

extern "C" int wfpg_comm_init_nccl(int32_t world, int32_t rank, const uint8_t* unique_id,
                                   wfpg_comm** out) {
  if (world < 1 || rank < 0 || rank >= world || !unique_id || !out) {
    set_error("wfpg_comm_init_nccl: bad arguments");
    return WFPG_ERR_ARG;
  }
  if (!nccl().ok) {
    set_error("NCCL (libnccl.so.2) is not loadable");
    return WFPG_ERR_CUDA;
  }
  Comm* c = new Comm();
  c->world = world;
  c->rank = rank;
  c->kind = 0;
  ncclUniqueId id;
  memcpy(id.internal, unique_id, sizeof(id.internal));
  ncclResult_t r = nccl().comm_init_rank(&c->nc, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommInitRank");
  }
  int rc = comm_alloc_common(c);
  if (rc != WFPG_OK) {
    delete c;
    return rc;
  }
  *out = reinterpret_cast<wfpg_comm*>(c);
  return WFPG_OK;
}

extern "C" int wfpg_comm_init_host(int32_t world, int32_t rank, wfpg_exchange_fn fn, void* user,
                                   wfpg_comm** out) {
  if (world < 1 || rank < 0 || rank >= world || !fn || !out) {
    set_error("wfpg_comm_init_host: bad arguments");
    return WFPG_ERR_ARG;
  }
  Comm* c = new Comm();
  c->world = world;
  c->rank = rank;
  c->kind = 1;
  c->fn = fn;
  c->user = user;
  int rc = comm_alloc_common(c);
  if (rc != WFPG_OK) {
    delete c;
    return rc;
  }
  *out = reinterpret_cast<wfpg_comm*>(c);
  return WFPG_OK;
}

extern "C" int wfpg_comm_settle(wfpg_comm* comm) {
  return comm_settle(reinterpret_cast<Comm*>(comm));
}

extern "C" int wfpg_comm_destroy(wfpg_comm* comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return WFPG_OK;
  int rc = comm_settle(c);
  if (c->nc) nccl().comm_destroy(c->nc);
  if (c->status_host) cudaFreeHost(c->status_host);
  if (c->done) cudaEventDestroy(c->done);
  if (c->scratch) cudaFree(c->scratch);
  delete c;
  return rc;
}

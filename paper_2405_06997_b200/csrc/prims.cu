// Exclusive scan (reduce-then-scan) and stable LSD radix sort with warp-level
// multisplit ranking.  Both accept a device-side element count so they can run
// inside a pass without a host round trip.
#include "prims.cuh"

namespace wfpg {

// ---------------------------------------------------------------------------
// scan
// ---------------------------------------------------------------------------
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanBlock * kScanItems;

__global__ void __launch_bounds__(kScanBlock) k_scan_reduce(const uint32_t* __restrict__ in,
                                                            int64_t n_max,
                                                            const int32_t* __restrict__ n_dev,
                                                            uint32_t* __restrict__ partial) {
  __shared__ uint32_t sw[kScanBlock / 32 + 1];
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + (int64_t)k * kScanBlock + threadIdx.x;
    if (i < n) s += in[i];
  }
  uint32_t tot;
  block_exclusive_scan<kScanBlock>(s, sw, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanBlock) k_scan_partials(uint32_t* __restrict__ partial,
                                                              int64_t nb,
                                                              uint32_t* __restrict__ total) {
  __shared__ uint32_t sw[kScanBlock / 32 + 1];
  uint32_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScanBlock) {
    int64_t i = base + threadIdx.x;
    uint32_t v = i < nb ? partial[i] : 0;
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<kScanBlock>(v, sw, &tot);
    if (i < nb) partial[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(const uint32_t* in, uint32_t* out,
                                                           int64_t n_max,
                                                           const int32_t* __restrict__ n_dev,
                                                           const uint32_t* __restrict__ partial) {
  __shared__ uint32_t sw[kScanBlock / 32 + 1];
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  // blocked arrangement: thread t owns items base + t*ITEMS .. +ITEMS-1
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + (int64_t)threadIdx.x * kScanItems + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  uint32_t ex = block_exclusive_scan<kScanBlock>(s, sw, nullptr) + partial[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + (int64_t)threadIdx.x * kScanItems + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
}

size_t scan_ws_bytes(int64_t n_max) {
  return align_up(sizeof(uint32_t) * (size_t)(ceil_div(n_max > 0 ? n_max : 1, kScanTile) + 1));
}

int scan_u32(const uint32_t* in, uint32_t* out, int64_t n_max, const int32_t* n_dev,
             uint32_t* total, Arena& ws, cudaStream_t st) {
  if (n_max <= 0) {
    if (total) WFPG_CUDA(cudaMemsetAsync(total, 0, sizeof(uint32_t), st));
    return WFPG_OK;
  }
  int64_t nb = ceil_div(n_max, kScanTile);
  uint32_t* partial = ws.take<uint32_t>(nb + 1);
  if (!ws.ok()) {
    set_error("scan: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  k_scan_reduce<<<(unsigned)nb, kScanBlock, 0, st>>>(in, n_max, n_dev, partial);
  WFPG_CHECK_LAUNCH("k_scan_reduce");
  k_scan_partials<<<1, kScanBlock, 0, st>>>(partial, nb, total);
  WFPG_CHECK_LAUNCH("k_scan_partials");
  k_scan_tiles<<<(unsigned)nb, kScanBlock, 0, st>>>(in, out, n_max, n_dev, partial);
  WFPG_CHECK_LAUNCH("k_scan_tiles");
  return WFPG_OK;
}

// ---------------------------------------------------------------------------
// stable LSD radix sort, 8-bit digits
// ---------------------------------------------------------------------------
constexpr int kSortWarps = 8;
constexpr int kSortBlock = kSortWarps * 32;
constexpr int kSortIpt = 8;  // 32-item chunks per warp
constexpr int kSortTile = kSortBlock * kSortIpt;

template <typename KT>
__global__ void __launch_bounds__(kSortBlock) k_sort_hist(const KT* __restrict__ keys,
                                                          int64_t n_max,
                                                          const int32_t* __restrict__ n_dev,
                                                          int shift, int64_t nblocks,
                                                          uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[256];
  const int64_t n = dev_count(n_max, n_dev);
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int k = 0; k < kSortIpt; ++k) {
    int64_t i = base + (int64_t)k * kSortBlock + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  // digit-major (stride = worst-case tile count): each digit's tile counts
  // are contiguous for the per-digit scan
  if (base < n) hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// Digit offsets: one block per digit scans that digit's counts over the
// active tiles (ceil(n / tile), n from the device) in place and writes the
// digit total; the scatter blocks turn the 256 totals into digit bases.
constexpr int kOffThreads = 256;
__global__ void __launch_bounds__(kOffThreads) k_sort_offsets(uint32_t* __restrict__ hist,
                                                              int64_t n_max,
                                                              const int32_t* __restrict__ n_dev,
                                                              int64_t nblocks,
                                                              uint32_t* __restrict__ dtot) {
  __shared__ uint32_t sw[kOffThreads / 32 + 1];
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t nb = (n + kSortTile - 1) / kSortTile;
  uint32_t* h = hist + (int64_t)blockIdx.x * nblocks;
  const int64_t per = (nb + kOffThreads - 1) / kOffThreads;
  const int64_t b0 = (int64_t)threadIdx.x * per, b1 = b0 + per < nb ? b0 + per : nb;
  uint32_t s = 0;
  for (int64_t b = b0; b < b1; ++b) s += h[b];
  uint32_t total;
  uint32_t run = block_exclusive_scan<kOffThreads>(s, sw, &total);
  for (int64_t b = b0; b < b1; ++b) {
    const uint32_t c = h[b];
    h[b] = run;
    run += c;
  }
  if (threadIdx.x == 0) dtot[blockIdx.x] = total;
}

template <typename KT>
__global__ void __launch_bounds__(kSortBlock) k_sort_scatter(
    const KT* __restrict__ kin, const uint32_t* __restrict__ vin, KT* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n_max, const int32_t* __restrict__ n_dev, int shift,
    int64_t nblocks, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ dbase) {
  __shared__ uint32_t whist[kSortWarps][256];
  __shared__ uint32_t goff[256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t sw[kSortBlock / 32 + 1];
  __shared__ KT sk[kSortTile];
  __shared__ uint32_t sv[kSortTile];
  const int64_t n = dev_count(n_max, n_dev);
  if ((int64_t)blockIdx.x * kSortTile >= n) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortBlock) (&whist[0][0])[i] = 0;
  // digit base = exclusive prefix of the digit totals (thread t = digit t)
  const uint32_t base_t = block_exclusive_scan<kSortBlock>(dbase[threadIdx.x], sw, nullptr);
  goff[threadIdx.x] = base_t + offs[(int64_t)threadIdx.x * nblocks + blockIdx.x];
  __syncthreads();

  const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * 32 * kSortIpt;
  KT k[kSortIpt];
  uint32_t v[kSortIpt];
  uint32_t r[kSortIpt];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int c = 0; c < kSortIpt; ++c) {
    int64_t i = wbase + c * 32 + lane;
    bool valid = i < n;
    k[c] = valid ? kin[i] : 0;
    v[c] = valid ? vin[i] : 0;
    uint32_t dig = valid ? (uint32_t)((k[c] >> shift) & 255u) : 256u + lane;
    uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    uint32_t peers = __match_any_sync(0xffffffffu, dig) & vmask;
    uint32_t pre = valid ? whist[warp][dig & 255u] : 0;
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[warp][dig] = pre + __popc(peers);
    __syncwarp();
    r[c] = pre + __popc(peers & lt);
  }
  __syncthreads();
  // per digit (thread t = digit t): warp-exclusive offsets within the digit,
  // then the block-local start of each digit
  uint32_t run = 0;
  for (int w = 0; w < kSortWarps; ++w) {
    uint32_t t = whist[w][threadIdx.x];
    whist[w][threadIdx.x] = run;
    run += t;
  }
  __syncthreads();  // sw is reused by the scan below
  const uint32_t lstart = block_exclusive_scan<kSortBlock>(run, sw, nullptr);
  dstart[threadIdx.x] = lstart;
  goff[threadIdx.x] -= lstart;  // global position = goff[d] + block-local position
  __syncthreads();
  // reorder the tile in shared memory by digit (stable), then write each
  // digit's run with consecutive threads: coalesced stores instead of 256-way
  // scattered ones
#pragma unroll
  for (int c = 0; c < kSortIpt; ++c) {
    int64_t i = wbase + c * 32 + lane;
    if (i < n) {
      uint32_t dig = (uint32_t)((k[c] >> shift) & 255u);
      uint32_t lp = dstart[dig] + whist[warp][dig] + r[c];
      sk[lp] = k[c];
      sv[lp] = v[c];
    }
  }
  __syncthreads();
  const int64_t tbase = (int64_t)blockIdx.x * kSortTile;
  const int valid = (int)(n - tbase < kSortTile ? n - tbase : kSortTile);
  for (int e = threadIdx.x; e < valid; e += kSortBlock) {
    const KT key = sk[e];
    const uint32_t pos = goff[(uint32_t)((key >> shift) & 255u)] + (uint32_t)e;
    kout[pos] = key;
    vout[pos] = sv[e];
  }
}

template <typename KT>
__global__ void k_copy_pairs(const KT* __restrict__ ks, const uint32_t* __restrict__ vs,
                             KT* __restrict__ kd, uint32_t* __restrict__ vd, int64_t n_max,
                             const int32_t* __restrict__ n_dev) {
  const int64_t n = dev_count(n_max, n_dev);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    kd[i] = ks[i];
    vd[i] = vs[i];
  }
}

size_t sort_ws_bytes(int64_t n_max) {
  int64_t n = n_max > 0 ? n_max : 1;
  int64_t nb = ceil_div(n, kSortTile);
  return align_up(sizeof(uint64_t) * n) + align_up(sizeof(uint32_t) * n) +
         align_up(sizeof(uint32_t) * 256 * nb) + align_up(sizeof(uint32_t) * 256) + 1024;
}

template <typename KT>
static int sort_pairs_t(KT* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev, int key_bits,
                        Arena& ws, cudaStream_t st) {
  if (n_max <= 1) return WFPG_OK;
  int64_t nb = ceil_div(n_max, kSortTile);
  KT* k2 = ws.take<KT>(n_max);
  uint32_t* v2 = ws.take<uint32_t>(n_max);
  uint32_t* hist = ws.take<uint32_t>(256 * nb);
  uint32_t* dbase = ws.take<uint32_t>(256);
  if (!ws.ok()) {
    set_error("sort: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  int passes = (key_bits + 7) / 8;
  KT* ka = keys;
  uint32_t* va = vals;
  KT* kb = k2;
  uint32_t* vb = v2;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    k_sort_hist<KT><<<(unsigned)nb, kSortBlock, 0, st>>>(ka, n_max, n_dev, shift, nb, hist);
    WFPG_CHECK_LAUNCH("k_sort_hist");
    k_sort_offsets<<<256, kOffThreads, 0, st>>>(hist, n_max, n_dev, nb, dbase);
    WFPG_CHECK_LAUNCH("k_sort_offsets");
    k_sort_scatter<KT><<<(unsigned)nb, kSortBlock, 0, st>>>(ka, va, kb, vb, n_max, n_dev, shift, nb,
                                                         hist, dbase);
    WFPG_CHECK_LAUNCH("k_sort_scatter");
    KT* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  if (ka != keys) {
    // odd number of passes: copy the live prefix back
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
    k_copy_pairs<KT><<<grid, 256, 0, st>>>(ka, va, keys, vals, n_max, n_dev);
    WFPG_CHECK_LAUNCH("k_copy_pairs");
  }
  return WFPG_OK;
}


int sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev, int key_bits,
               Arena& ws, cudaStream_t st) {
  return sort_pairs_t(keys, vals, n_max, n_dev, key_bits, ws, st);
}
int sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev, int key_bits,
               Arena& ws, cudaStream_t st) {
  return sort_pairs_t(keys, vals, n_max, n_dev, key_bits < 32 ? key_bits : 32, ws, st);
}

}  // namespace wfpg

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" size_t wfpg_scan_workspace_bytes(int64_t n) { return wfpg::scan_ws_bytes(n); }

extern "C" int wfpg_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                             void* workspace, size_t ws_bytes, void* stream) {
  if (n < 0 || (n > 0 && (!in || !out))) {
    wfpg::set_error("wfpg_scan_u32: bad arguments");
    return WFPG_ERR_ARG;
  }
  wfpg::Arena ws(workspace, ws_bytes);
  return wfpg::scan_u32(in, out, n, nullptr, total, ws, wfpg::as_stream(stream));
}

extern "C" size_t wfpg_sort_workspace_bytes(int64_t n) { return wfpg::sort_ws_bytes(n); }

extern "C" int wfpg_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, const int32_t* n_dev,
                                   int32_t key_bits, void* workspace, size_t ws_bytes,
                                   void* stream) {
  if (n < 0 || key_bits < 1 || key_bits > 64 || (n > 0 && (!keys || !vals))) {
    wfpg::set_error("wfpg_sort_pairs_u64: bad arguments");
    return WFPG_ERR_ARG;
  }
  wfpg::Arena ws(workspace, ws_bytes);
  return wfpg::sort_pairs(keys, vals, n, n_dev, key_bits, ws, wfpg::as_stream(stream));
}

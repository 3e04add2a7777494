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
  if (base >= n) {  // past the live count (grids are sized for n_max): uniform exit
    if (threadIdx.x == 0) partial[blockIdx.x] = 0;
    return;
  }
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
  if (base >= n) return;  // uniform: nothing live in this tile
  // blocked arrangement: thread t owns items base + t*ITEMS .. +ITEMS-1,
  // loaded / stored as one 16-byte vector when all four are live and the
  // arrays are 16-byte aligned (a warp then moves 512 contiguous bytes)
  static_assert(kScanItems == 4, "uint4 vectors");
  const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
  const bool vec = i0 + kScanItems <= n &&
                   ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  uint32_t v[kScanItems];
  if (vec) {
    const uint4 q = *reinterpret_cast<const uint4*>(in + i0);
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < n ? in[i0 + k] : 0;
  }
  const uint32_t s = v[0] + v[1] + v[2] + v[3];
  const uint32_t ex = block_exclusive_scan<kScanBlock>(s, sw, nullptr) + partial[blockIdx.x];
  uint32_t o[kScanItems];
  o[0] = ex;
  o[1] = o[0] + v[0];
  o[2] = o[1] + v[1];
  o[3] = o[2] + v[2];
  if (vec) {
    *reinterpret_cast<uint4*>(out + i0) = make_uint4(o[0], o[1], o[2], o[3]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (i0 + k < n) out[i0 + k] = o[k];
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
// stable LSD radix sort over a few large chunks: per pass, a histogram kernel
// counts each chunk's digits (one block per chunk), one block per digit scans
// that digit's chunk counts, and the scatter kernel walks its chunk tile by
// tile with running digit offsets in shared memory — no look-back and a
// chunk-count table of radix x chunks entries.  Digits are up to 9 bits
// (passes = ceil(bits / 9), equal widths), so 36-bit Morton codes sort in 4
// passes.  Within a tile every warp ranks its 32-item chunks by match_any
// (stable), the tile is reordered by digit in shared memory and each digit's
// run is stored by consecutive threads.
// ---------------------------------------------------------------------------
constexpr int kCsWarps = 16;
constexpr int kCsBlock = kCsWarps * 32;
constexpr int kCsIpt = 8;                    // 32-item chunks per warp
constexpr int kCsTile = kCsBlock * kCsIpt;   // 4096 items per tile
constexpr int kCsMaxBits = 9;
constexpr int kCsMaxRadix = 1 << kCsMaxBits;
constexpr int kCsChunks = kNumSMs * 2;       // scatter blocks resident at once

struct CsPlan {
  int passes, bits;
};
static CsPlan cs_plan(int key_bits) {
  CsPlan p;
  p.passes = (key_bits + kCsMaxBits - 1) / kCsMaxBits;
  if (p.passes < 1) p.passes = 1;
  p.bits = (key_bits + p.passes - 1) / p.passes;
  return p;
}

// chunk c covers [c * len, (c + 1) * len) of the live count, len a tile multiple
__device__ __forceinline__ int64_t cs_chunk_len(int64_t n) {
  const int64_t tiles = (n + kCsTile - 1) / kCsTile;
  return ((tiles + kCsChunks - 1) / kCsChunks) * kCsTile;
}

template <typename KT>
__global__ void __launch_bounds__(256) k_cs_hist(const KT* __restrict__ keys, int64_t n_max,
                                                 const int32_t* __restrict__ n_dev, int shift,
                                                 int bits, uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[kCsMaxRadix];
  const int radix = 1 << bits;
  const uint32_t dm = (uint32_t)radix - 1u;
  for (int i = threadIdx.x; i < radix; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t len = cs_chunk_len(n);
  const int64_t b0 = (int64_t)blockIdx.x * len;
  const int64_t b1 = b0 + len < n ? b0 + len : n;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
    atomicAdd(&h[(uint32_t)((keys[i] >> shift) & dm)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < radix; d += blockDim.x)
    counts[(int64_t)d * kCsChunks + blockIdx.x] = h[d];
}

// one block per digit: exclusive scan of the digit's chunk counts in place,
// digit total to dtot
constexpr int kCsOffThreads = ((kCsChunks + 31) / 32) * 32;
__global__ void __launch_bounds__(kCsOffThreads) k_cs_offsets(uint32_t* __restrict__ counts,
                                                              uint32_t* __restrict__ dtot) {
  __shared__ uint32_t sw[kCsOffThreads / 32 + 1];
  uint32_t* c = counts + (int64_t)blockIdx.x * kCsChunks;
  const bool in = threadIdx.x < kCsChunks;
  const uint32_t v = in ? c[threadIdx.x] : 0u;
  uint32_t total;
  const uint32_t ex = block_exclusive_scan<kCsOffThreads>(v, sw, &total);
  if (in) c[threadIdx.x] = ex;
  if (threadIdx.x == 0) dtot[blockIdx.x] = total;
}

template <typename KT>
__global__ void __launch_bounds__(kCsBlock) k_cs_scatter(
    const KT* __restrict__ kin, const uint32_t* __restrict__ vin, KT* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n_max, const int32_t* __restrict__ n_dev, int shift,
    int bits, const uint32_t* __restrict__ counts, const uint32_t* __restrict__ dtot) {
  extern __shared__ __align__(16) unsigned char cs_smem[];
  const int radix = 1 << bits;
  const uint32_t dm = (uint32_t)radix - 1u;
  KT* sk = reinterpret_cast<KT*>(cs_smem);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kCsTile);
  uint32_t* whist = sv + kCsTile;              // [kCsWarps][radix]
  uint32_t* run = whist + kCsWarps * radix;    // [radix] running global offsets
  uint32_t* goff = run + radix;                // [radix]
  uint32_t* dstart = goff + radix;             // [radix]
  __shared__ uint32_t sw[kCsBlock / 32 + 1];
  const int64_t n = dev_count(n_max, n_dev);
  const int64_t len = cs_chunk_len(n);
  const int64_t c0 = (int64_t)blockIdx.x * len;
  if (c0 >= n) return;
  const int64_t c1 = c0 + len < n ? c0 + len : n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = threadIdx.x;
  {
    // digit bases (exclusive scan of the digit totals) + this chunk's offset
    const uint32_t t = d < radix ? dtot[d] : 0u;
    const uint32_t base = block_exclusive_scan<kCsBlock>(t, sw, nullptr);
    if (d < radix) run[d] = base + counts[(int64_t)d * kCsChunks + blockIdx.x];
  }
  const uint32_t lt = lanemask_lt();
  uint32_t* wh = whist + warp * radix;
  for (int64_t tbase = c0; tbase < c1; tbase += kCsTile) {
    for (int i = threadIdx.x; i < kCsWarps * radix; i += kCsBlock) whist[i] = 0;
    __syncthreads();
    const int64_t wbase = tbase + (int64_t)warp * 32 * kCsIpt;
    KT k[kCsIpt];
    uint32_t v[kCsIpt];
    uint32_t r[kCsIpt];
    // all of the tile's loads in flight before the first ranking step
#pragma unroll
    for (int c = 0; c < kCsIpt; ++c) {
      const int64_t i = wbase + c * 32 + lane;
      const bool valid = i < c1;
      k[c] = valid ? kin[i] : (KT)0;
      v[c] = valid ? vin[i] : 0u;
    }
#pragma unroll
    for (int c = 0; c < kCsIpt; ++c) {
      const int64_t i = wbase + c * 32 + lane;
      const bool valid = i < c1;
      const uint32_t dig = valid ? (uint32_t)((k[c] >> shift) & dm) : (uint32_t)radix + lane;
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      const uint32_t peers = __match_any_sync(0xffffffffu, dig) & vmask;
      const uint32_t pre = valid ? wh[dig] : 0u;
      __syncwarp();
      if (valid && (peers & lt) == 0) wh[dig] = pre + __popc(peers);
      __syncwarp();
      r[c] = pre + __popc(peers & lt);
    }
    __syncthreads();
    // thread d = digit d: warp-exclusive offsets within the digit, the tile's
    // digit count, the tile-local digit starts
    uint32_t cnt = 0;
    if (d < radix) {
      for (int w = 0; w < kCsWarps; ++w) {
        const uint32_t t = whist[w * radix + d];
        whist[w * radix + d] = cnt;
        cnt += t;
      }
    }
    const uint32_t lstart = block_exclusive_scan<kCsBlock>(cnt, sw, nullptr);
    if (d < radix) {
      dstart[d] = lstart;
      goff[d] = run[d] - lstart;  // global position = goff + tile position
      run[d] += cnt;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kCsIpt; ++c) {
      const int64_t i = wbase + c * 32 + lane;
      if (i < c1) {
        const uint32_t dig = (uint32_t)((k[c] >> shift) & dm);
        const uint32_t lp = dstart[dig] + wh[dig] + r[c];
        sk[lp] = k[c];
        sv[lp] = v[c];
      }
    }
    __syncthreads();
    const int valid = (int)(c1 - tbase < kCsTile ? c1 - tbase : kCsTile);
    for (int e = threadIdx.x; e < valid; e += kCsBlock) {
      const KT key = sk[e];
      const uint32_t pos = goff[(uint32_t)((key >> shift) & dm)] + (uint32_t)e;
      kout[pos] = key;
      vout[pos] = sv[e];
    }
    __syncthreads();  // sk / sv / whist are reused by the next tile
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

template <typename KT>
static size_t cs_smem_bytes(int bits) {
  const int radix = 1 << bits;
  return sizeof(KT) * kCsTile + sizeof(uint32_t) * kCsTile +
         sizeof(uint32_t) * (size_t)(kCsWarps + 3) * radix;
}

size_t sort_ws_bytes(int64_t n_max) {
  int64_t n = n_max > 0 ? n_max : 1;
  return align_up(sizeof(uint64_t) * n) + align_up(sizeof(uint32_t) * n) +
         align_up(sizeof(uint32_t) * (size_t)kCsMaxRadix * kCsChunks) +
         align_up(sizeof(uint32_t) * kCsMaxRadix) + 1024;
}

// kres / vres (optional): report the buffers that hold the result instead of
// copying it back into keys / vals after an odd number of passes (the
// caller then keeps the workspace taken here alive while it reads them)
template <typename KT>
static int sort_pairs_t(KT* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev, int key_bits,
                        Arena& ws, cudaStream_t st, KT** kres = nullptr,
                        uint32_t** vres = nullptr) {
  if (kres) *kres = keys;
  if (vres) *vres = vals;
  if (n_max <= 1) return WFPG_OK;
  if (n_max >= (int64_t)UINT32_MAX) {
    set_error("sort: %lld items exceed the 32-bit index range", (long long)n_max);
    return WFPG_ERR_CAPACITY;
  }
  const CsPlan plan = cs_plan(key_bits);
  const int radix = 1 << plan.bits;
  KT* k2 = ws.take<KT>(n_max);
  uint32_t* v2 = ws.take<uint32_t>(n_max);
  uint32_t* counts = ws.take<uint32_t>((int64_t)kCsMaxRadix * kCsChunks);
  uint32_t* dtot = ws.take<uint32_t>(kCsMaxRadix);
  if (!ws.ok()) {
    set_error("sort: workspace too small");
    return WFPG_ERR_WORKSPACE;
  }
  const size_t smem = cs_smem_bytes<KT>(plan.bits);
  static bool configured = false;
  if (!configured) {
    WFPG_CUDA(cudaFuncSetAttribute(k_cs_scatter<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)cs_smem_bytes<KT>(kCsMaxBits)));
    configured = true;
  }
  // fewer chunks than kCsChunks are live when n is small; the others return
  const unsigned grid = (unsigned)std::min<int64_t>(kCsChunks, ceil_div(n_max, kCsTile));
  KT* ka = keys;
  uint32_t* va = vals;
  KT* kb = k2;
  uint32_t* vb = v2;
  for (int p = 0; p < plan.passes; ++p) {
    const int shift = p * plan.bits;
    // chunks past the live count must read as zero counts
    if (grid < (unsigned)kCsChunks || n_dev)
      WFPG_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t)radix * kCsChunks, st));
    k_cs_hist<KT><<<grid, 256, 0, st>>>(ka, n_max, n_dev, shift, plan.bits, counts);
    WFPG_CHECK_LAUNCH("k_cs_hist");
    k_cs_offsets<<<radix, kCsOffThreads, 0, st>>>(counts, dtot);
    WFPG_CHECK_LAUNCH("k_cs_offsets");
    k_cs_scatter<KT><<<grid, kCsBlock, smem, st>>>(ka, va, kb, vb, n_max, n_dev, shift,
                                                   plan.bits, counts, dtot);
    WFPG_CHECK_LAUNCH("k_cs_scatter");
    KT* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  if (kres && vres) {
    *kres = ka;
    *vres = va;
  } else if (ka != keys) {
    // odd number of passes: copy the live prefix back
    int cgrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256), kNumSMs * 8));
    k_copy_pairs<KT><<<cgrid, 256, 0, st>>>(ka, va, keys, vals, n_max, n_dev);
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
int sort_pairs_nocopy(uint32_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev,
                      int key_bits, Arena& ws, cudaStream_t st, uint32_t** kres,
                      uint32_t** vres) {
  return sort_pairs_t(keys, vals, n_max, n_dev, key_bits < 32 ? key_bits : 32, ws, st, kres,
                      vres);
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

// Device-wide primitives (internal C++ API): exclusive scan, stable radix sort.
#pragma once
#include "common.cuh"

namespace wfpg {

size_t scan_ws_bytes(int64_t n_max);
// Exclusive scan of n uint32 values.  n = n_dev ? min(*n_dev, n_max) : n_max.
// total (device, optional) receives the sum.  in and out may alias.
int scan_u32(const uint32_t* in, uint32_t* out, int64_t n_max, const int32_t* n_dev,
             uint32_t* total, Arena& ws, cudaStream_t st);

size_t sort_ws_bytes(int64_t n_max);
// Stable LSD radix sort of (key, value) pairs on the low key_bits bits, in place.
int sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev,
               int key_bits, Arena& ws, cudaStream_t st);
int sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev,
               int key_bits, Arena& ws, cudaStream_t st);
// Same sort without the copy-back after an odd pass count: *kres / *vres
// name the buffers holding the result (keys / vals or workspace taken from
// ws, which the caller must not release while it reads them).
int sort_pairs_nocopy(uint32_t* keys, uint32_t* vals, int64_t n_max, const int32_t* n_dev,
                      int key_bits, Arena& ws, cudaStream_t st, uint32_t** kres,
                      uint32_t** vres);

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

__device__ __forceinline__ int64_t dev_count(int64_t n_max, const int32_t* n_dev) {
  if (!n_dev) return n_max;
  int64_t v = *n_dev;
  return v < n_max ? v : n_max;
}

}  // namespace wfpg

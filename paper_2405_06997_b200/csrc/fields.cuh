#pragma once
#include "geometry.cuh"

namespace wfpg {

struct BlurParams {
  int radius;
  double w[33];
};

struct FieldOut {
  double* vals;
  double* row_sum;
  double* marg;
  double* total;
  double* block_sums;  // NULL unless product mode
  double eps;
  double* cum = nullptr;  // optional (B,n,n) row prefix sums
  // optional zeroed device counter: bins after each CTA's first are handed
  // out dynamically (bin costs vary; static striding left SMs idle at the end)
  int32_t* bin_ctr = nullptr;
  // optional work list: work item w generates bin bin_list[w] (the outputs
  // stay indexed by bin); nb_max / nb_dev then count work items.  Multi-GPU
  // ranks generate only the bins their own paths belong to.
  const int32_t* bin_list = nullptr;
  // optional (B, 8, 8, n/8) product-mode block row sums (0 + pairwise row
  // sum of each row of each 8x8 block, guiding.py:304): the product sampler
  // reads its block marginal from here instead of re-summing the rows
  double* block_rows = nullptr;
};

int launch_fields(const SceneView& s, const SvoView& v, const double* origins,
                  const double* jitters, int64_t nb_max, const int32_t* nb_dev, int n,
                  const BlurParams& bp, const FieldOut& out, cudaStream_t st);

// multi-GPU bin ownership: tables of the bins other ranks generated, from the
// all-gathered values (bitwise the owners' tables)
int launch_own_fill(const double* src, int n, const int32_t* n_bins, const int32_t* own_ok,
                    int64_t own_lo, int64_t own_hi, int64_t cap, const FieldOut& out,
                    cudaStream_t st);

}  // namespace wfpg

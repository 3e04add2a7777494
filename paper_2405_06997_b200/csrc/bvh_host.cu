// Host BVH build in C++ with the reference's decisions (bvh.py:33-119 as
// restated in paper_2405_06997_b200/bvh.py): 16 centroid bins on the widest
// centroid axis (first maximum), at most 4 triangles per leaf, surface-area
// cost with strict improvement, stable left/right partition, median
// fallback, depth-first numbering with both children allocated before the
// left one is processed.  Same fp64 operations in the same order as the
// numpy code (no FMA contraction on the host: x86-64 without -mfma), so the
// arrays are bitwise those of the Python build — which matches the
// reference's — at ~1000x its speed.  Host-only code (scene preprocessing,
// like the reference's own load-time build); traversal is on the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kMaxLeafTris = 4;
constexpr int kBins = 16;

struct Box3 {
  double lo[3], hi[3];
};

inline double box_area(const double* lo, const double* hi) {
  double e[3];
  for (int a = 0; a < 3; ++a) {
    const double d = hi[a] - lo[a];
    e[a] = d > 0.0 ? d : 0.0;  // np.maximum(hi - lo, 0.0)
  }
  const double s = (e[0] * e[1] + e[1] * e[2]) + e[2] * e[0];
  return 2.0 * s;
}

struct Builder {
  const double *tlo, *thi, *cen;  // (n,3) each
  std::vector<int64_t> order;
  std::vector<double> lo, hi;
  std::vector<int32_t> left, right, count;
  std::vector<int64_t> scratch;
  std::vector<int32_t> bin;

  int64_t add_node() {
    lo.insert(lo.end(), 3, 0.0);
    hi.insert(hi.end(), 3, 0.0);
    left.push_back(-1);
    right.push_back(-1);
    count.push_back(0);
    return (int64_t)count.size() - 1;
  }

  // _choose_split: returns the left count after partitioning order[start,end)
  // in place, or -1 for "no split" (median fallback, order unchanged)
  int64_t choose_split(int64_t start, int64_t end) {
    double clo[3], chi[3];
    for (int a = 0; a < 3; ++a) {
      clo[a] = std::numeric_limits<double>::infinity();
      chi[a] = -std::numeric_limits<double>::infinity();
    }
    for (int64_t k = start; k < end; ++k) {
      const double* c = cen + 3 * order[k];
      for (int a = 0; a < 3; ++a) {
        clo[a] = std::min(clo[a], c[a]);
        chi[a] = std::max(chi[a], c[a]);
      }
    }
    int axis = 0;
    double best_ext = chi[0] - clo[0];
    for (int a = 1; a < 3; ++a)
      if (chi[a] - clo[a] > best_ext) {
        best_ext = chi[a] - clo[a];
        axis = a;
      }
    const double extent = chi[axis] - clo[axis];
    if (extent <= 0.0) return -1;
    const double scale = (double)kBins / extent;
    Box3 bb[kBins];
    int64_t cnt[kBins];
    for (int k = 0; k < kBins; ++k) {
      cnt[k] = 0;
      for (int a = 0; a < 3; ++a) {
        bb[k].lo[a] = std::numeric_limits<double>::infinity();
        bb[k].hi[a] = -std::numeric_limits<double>::infinity();
      }
    }
    const int64_t m = end - start;
    bin.resize((size_t)m);
    for (int64_t k = start; k < end; ++k) {
      const int64_t t = order[k];
      double q = (cen[3 * t + axis] - clo[axis]) * scale;
      q = std::min(q, (double)(kBins - 1));  // np.minimum then astype(int64)
      const int b = (int)(int64_t)q;
      bin[(size_t)(k - start)] = b;
      ++cnt[b];
      for (int a = 0; a < 3; ++a) {
        bb[b].lo[a] = std::min(bb[b].lo[a], tlo[3 * t + a]);
        bb[b].hi[a] = std::max(bb[b].hi[a], thi[3 * t + a]);
      }
    }
    double best = std::numeric_limits<double>::infinity();
    int split = -1;
    for (int s = 1; s < kBins; ++s) {
      int64_t nl = 0, nr = 0;
      double llo[3], lhi[3], rlo[3], rhi[3];
      for (int a = 0; a < 3; ++a) {
        llo[a] = rlo[a] = std::numeric_limits<double>::infinity();
        lhi[a] = rhi[a] = -std::numeric_limits<double>::infinity();
      }
      for (int k = 0; k < kBins; ++k) {
        const bool l = k < s;
        (l ? nl : nr) += cnt[k];
        for (int a = 0; a < 3; ++a) {
          double& mn = l ? llo[a] : rlo[a];
          double& mx = l ? lhi[a] : rhi[a];
          mn = std::min(mn, bb[k].lo[a]);
          mx = std::max(mx, bb[k].hi[a]);
        }
      }
      if (nl == 0 || nr == 0) continue;
      const double cost = box_area(llo, lhi) * (double)nl + box_area(rlo, rhi) * (double)nr;
      if (cost < best) {
        best = cost;
        split = s;
      }
    }
    if (split < 0) return -1;
    // stable partition: concatenate([ids[go_left], ids[~go_left]])
    scratch.resize((size_t)m);
    int64_t nleft = 0;
    for (int64_t k = 0; k < m; ++k)
      if (bin[(size_t)k] < split) scratch[(size_t)nleft++] = order[start + k];
    int64_t w = nleft;
    for (int64_t k = 0; k < m; ++k)
      if (bin[(size_t)k] >= split) scratch[(size_t)w++] = order[start + k];
    std::copy(scratch.begin(), scratch.begin() + m, order.begin() + start);
    return nleft;
  }

  void build(int64_t n) {
    order.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
    add_node();
    struct Job {
      int64_t node, start, end;
    };
    std::vector<Job> todo{{0, 0, n}};
    while (!todo.empty()) {
      const Job j = todo.back();
      todo.pop_back();
      double* nlo = &lo[3 * j.node];
      double* nhi = &hi[3 * j.node];
      for (int a = 0; a < 3; ++a) {
        nlo[a] = std::numeric_limits<double>::infinity();
        nhi[a] = -std::numeric_limits<double>::infinity();
      }
      for (int64_t k = j.start; k < j.end; ++k) {
        const int64_t t = order[(size_t)k];
        for (int a = 0; a < 3; ++a) {
          nlo[a] = std::min(nlo[a], tlo[3 * t + a]);
          nhi[a] = std::max(nhi[a], thi[3 * t + a]);
        }
      }
      const int64_t m = j.end - j.start;
      if (m <= kMaxLeafTris) {
        left[(size_t)j.node] = (int32_t)j.start;
        count[(size_t)j.node] = (int32_t)m;
        continue;
      }
      int64_t mid = j.start + m / 2;
      const int64_t nl = choose_split(j.start, j.end);
      if (nl > 0 && nl < m) mid = j.start + nl;
      const int64_t k0 = add_node();
      const int64_t k1 = add_node();
      left[(size_t)j.node] = (int32_t)k0;
      right[(size_t)j.node] = (int32_t)k1;
      todo.push_back({k1, mid, j.end});
      todo.push_back({k0, j.start, mid});
    }
  }
};

}  // namespace

using namespace wfpg;

// Builds into caller arrays of capacity 2n-1 nodes (the tree never needs
// more); *n_nodes receives the node count.
extern "C" int wfpg_bvh_build_host(const double* v0, const double* v1, const double* v2,
                                   int64_t n, double* lo, double* hi, int32_t* left,
                                   int32_t* right, int32_t* count, int32_t* order,
                                   int64_t* n_nodes) {
  if (n <= 0 || n >= INT32_MAX || !v0 || !v1 || !v2 || !lo || !hi || !left || !right || !count ||
      !order || !n_nodes) {
    set_error("wfpg_bvh_build_host: bad arguments");
    return WFPG_ERR_ARG;
  }
  std::vector<double> tlo((size_t)(3 * n)), thi((size_t)(3 * n)), cen((size_t)(3 * n));
  for (int64_t i = 0; i < 3 * n; ++i) {
    const double a = v0[i], b = v1[i], c = v2[i];
    tlo[(size_t)i] = std::min(std::min(a, b), c);
    thi[(size_t)i] = std::max(std::max(a, b), c);
    cen[(size_t)i] = (tlo[(size_t)i] + thi[(size_t)i]) * 0.5;
  }
  Builder bld;
  bld.tlo = tlo.data();
  bld.thi = thi.data();
  bld.cen = cen.data();
  bld.build(n);
  const int64_t nn = (int64_t)bld.count.size();
  if (nn > 2 * n - 1) {
    set_error("wfpg_bvh_build_host: node count %lld exceeds the capacity", (long long)nn);
    return WFPG_ERR_ARG;
  }
  std::copy(bld.lo.begin(), bld.lo.end(), lo);
  std::copy(bld.hi.begin(), bld.hi.end(), hi);
  std::copy(bld.left.begin(), bld.left.end(), left);
  std::copy(bld.right.begin(), bld.right.end(), right);
  std::copy(bld.count.begin(), bld.count.end(), count);
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)bld.order[(size_t)i];
  *n_nodes = nn;
  return WFPG_OK;
}

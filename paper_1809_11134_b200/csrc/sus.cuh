// Stochastic universal sampling at any population size (sus_select,
// ga.py:95-116) with the reference's exact rounding.
//
// The reference's walk is
//   total = np.sum(f); spacing = total / count; pointer = uniform(0, spacing)
//   for k < count: while index < P-1 and cumulative + f[index] <= pointer:
//                      cumulative += f[index]; index += 1
//                  picks[k] = index; pointer += spacing
// Both running sums are sequentially rounded recurrences,
//   C[j+1] = fl(C[j] + f[j])        (C[0] = 0)
//   p[k+1] = fl(p[k] + spacing)     (p[0] = pointer)
// and both are nondecreasing (f >= 0), so the walk stops pointer k at the
// first j <= P-2 with C[j+1] > p[k] (else P-1).  Here:
//   * np.sum's pairwise tree (numpy's pairwise_sum: 8 accumulators below 128
//     elements, halving at a multiple of 8 above) is evaluated by a block:
//     the recursion's top levels are expanded into up to 2^8 subtrees, one
//     per thread (np_pairwise_sum, iterative), then combined level by level
//     in the recursion's own order -- bit-identical to the sequential sum;
//   * the two recurrences run on two threads of different warps (the only
//     sequential part left: one dependent add per element) over
//     shared-memory tiles the other warps load and store, double-buffered;
//   * the picks are a grid-wide binary search over C (sus_search_kernel).
#pragma once

#include <cstdint>

#include "np_random.cuh"

namespace isq {

constexpr int kSusThreads = 512;  // block of sus_chains_block / np_pairwise_sum_block
constexpr int kSusTile = 1024;    // elements per staged tile (2 buffers x (f/C + p) = 32 KB)

// Node `i` (d path bits, most significant first: 0 = left) of numpy's
// pairwise recursion over n elements: its offset and length.
__device__ __forceinline__ void pairwise_node(int64_t n, int d, int i, int64_t& off, int64_t& m) {
  off = 0;
  m = n;
  for (int l = d - 1; l >= 0; --l) {
    int64_t h = m / 2;
    h -= h % 8;
    if ((i >> l) & 1) {
      off += h;
      m -= h;
    } else {
      m = h;
    }
  }
}

// np.sum(a[0..n)) on a whole block of kThreads (>= 256) threads; `sm` holds
// kThreads doubles.  Every thread returns the total.
template <int kThreads>
__device__ double np_pairwise_sum_block(const double* a, int64_t n, double* sm) {
  static_assert(kThreads >= 256, "the expansion uses up to 256 subtrees");
  // depth d: 2^d subtrees, every node above them internal (> 128 elements);
  // node lengths at depth d are >= n / 2^d - 8 d
  int d = 0;
  while (d < 8 && (n >> (d + 1)) >= 256) ++d;
  const int nodes = 1 << d;
  if ((int)threadIdx.x < nodes) {
    int64_t off, m;
    pairwise_node(n, d, (int)threadIdx.x, off, m);
    sm[threadIdx.x] = np_pairwise_sum(a + off, m);
  }
  __syncthreads();
  for (int w = nodes >> 1; w >= 1; w >>= 1) {  // parent j = left 2j + right 2j+1
    double v = 0.0;
    if ((int)threadIdx.x < w) v = __dadd_rn(sm[2 * threadIdx.x], sm[2 * threadIdx.x + 1]);
    __syncthreads();
    if ((int)threadIdx.x < w) sm[threadIdx.x] = v;
    __syncthreads();
  }
  const double total = sm[0];
  __syncthreads();
  return total;
}

// Cg[j] = C[j+1] for j < nf and Pg[k] = p[k] for k < np, in the walk's own
// rounding, on a block of kSusThreads: thread 0 runs the C chain, thread 32
// the pointer chain, warps 2.. stage the tiles (load f of tile t+1, store
// tile t-1) while the chains run on tile t.
__device__ inline void sus_chains_block(const double* f, int64_t nf, double pointer, double spacing, int64_t np,
                                 double* Cg, double* Pg) {
  __shared__ double X[2][kSusTile];  // f of a tile, overwritten in place by C
  __shared__ double Y[2][kSusTile];  // pointers of a tile
  const int tid = threadIdx.x;
  const int64_t len = nf > np ? nf : np;
  const int64_t ntiles = (len + kSusTile - 1) / kSusTile;
  constexpr int kStagers = kSusThreads - 64;
  const int sid = tid - 64;
  auto load = [&](int64_t t, int b) {
    const int64_t base = t * kSusTile;
    for (int i = sid; i < kSusTile; i += kStagers)
      if (base + i < nf) X[b][i] = f[base + i];
  };
  auto store = [&](int64_t t, int b) {
    const int64_t base = t * kSusTile;
    for (int i = sid; i < kSusTile; i += kStagers) {
      if (base + i < nf) Cg[base + i] = X[b][i];
      if (base + i < np) Pg[base + i] = Y[b][i];
    }
  };
  if (tid >= 64 && ntiles > 0) load(0, 0);
  __syncthreads();
  double c = 0.0, p = pointer;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int b = (int)(t & 1);
    const int64_t base = t * kSusTile;
    if (tid == 0) {
      const int m = (int)(nf - base < kSusTile ? (nf - base > 0 ? nf - base : 0) : kSusTile);
      int i = 0;
      for (; i + 8 <= m; i += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = X[b][i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          c = __dadd_rn(c, x[u]);
          X[b][i + u] = c;
        }
      }
      for (; i < m; ++i) {
        c = __dadd_rn(c, X[b][i]);
        X[b][i] = c;
      }
    } else if (tid == 32) {
      const int m = (int)(np - base < kSusTile ? (np - base > 0 ? np - base : 0) : kSusTile);
      for (int i = 0; i < m; ++i) {
        Y[b][i] = p;
        p = __dadd_rn(p, spacing);
      }
    } else if (tid >= 64) {
      if (t >= 1) store(t - 1, b ^ 1);
      if (t + 1 < ntiles) load(t + 1, b ^ 1);
    }
    __syncthreads();
  }
  if (tid >= 64 && ntiles > 0) store(ntiles - 1, (int)((ntiles - 1) & 1));
  __syncthreads();
}

// picks[k] = first j in [0, nC) with C[j] > p[k], else nC (nC = P - 1): where
// the sequential walk stops pointer k.  `flag` (optional): skip unless *flag.
template <class Pick>
__global__ void sus_search_kernel(const double* __restrict__ C, int64_t nC, const double* __restrict__ Pt, int64_t np,
                                  Pick* __restrict__ picks, const int* flag, const int32_t* stop) {
  if (stop != nullptr && *stop) return;
  if (flag != nullptr && !*flag) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < np; k += (int64_t)gridDim.x * blockDim.x) {
    const double pk = Pt[k];
    int64_t lo = 0, hi = nC;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (C[mid] <= pk)
        lo = mid + 1;
      else
        hi = mid;
    }
    picks[k] = (Pick)lo;
  }
}

}  // namespace isq

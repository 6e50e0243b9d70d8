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
//     the recursion's top levels are expanded into up to 2^10 subtrees, one
//     per thread (np_pairwise_sum, iterative), then combined level by level
//     in the recursion's own order -- bit-identical to the sequential sum;
//   * the two recurrences are evaluated exactly in parallel, one block each:
//     the cumulative sum by exact_chain_block (a block-wide scan of the
//     mantissa maps of each binade's grid, plain adds only where the grid
//     form does not hold), the pointers by exact_const_chain_block (a
//     constant increment: closed form inside each binade);
//   * the picks are a grid-wide binary search over C (sus_search_kernel).
#pragma once

#include <climits>
#include <cstdint>

#include "np_random.cuh"

namespace isq {

constexpr int kSusThreads = 1024;  // block of exact_chain_block / np_pairwise_sum_block

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

// np.sum(a[0..n)) on a whole block of kThreads (a power of two >= 256) threads; `sm` holds
// kThreads doubles.  Every thread returns the total.
template <int kThreads>
__device__ double np_pairwise_sum_block(const double* a, int64_t n, double* sm) {
  static_assert(kThreads >= 256 && (kThreads & (kThreads - 1)) == 0, "a power of two >= 256");
  constexpr int kMaxD = __builtin_ctz(kThreads);  // up to one subtree per thread
  // depth d: 2^d subtrees, every node above them internal (> 128 elements);
  // node lengths at depth d are >= n / 2^d - 8 d
  int d = 0;
  while (d < kMaxD && (n >> (d + 1)) >= 256) ++d;
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

// The same total over the GPU (large n): the 2^d subtree sums by
// pairwise_parts_kernel (one thread each), then their tree on one block.
constexpr int kPwMaxDepth = 13;  // up to 8192 subtrees
__host__ __device__ inline int pairwise_grid_depth(int64_t n) {
  int d = 0;
  while (d < kPwMaxDepth && (n >> (d + 1)) >= 256) ++d;
  return d;
}
static __global__ void __launch_bounds__(256) pairwise_parts_kernel(const double* a, int64_t n, int d, double* parts) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < (1 << d)) {
    int64_t off, m;
    pairwise_node(n, d, i, off, m);
    parts[i] = np_pairwise_sum(a + off, m);
  }
}
// `sm`: 2^d doubles.  Every thread returns the total.
template <int kThreads>
__device__ double np_pairwise_combine_block(const double* parts, int d, double* sm) {
  constexpr int kPer = (1 << kPwMaxDepth) / 2 / kThreads > 0 ? (1 << kPwMaxDepth) / 2 / kThreads : 1;
  const int nodes = 1 << d;
  for (int i = threadIdx.x; i < nodes; i += kThreads) sm[i] = parts[i];
  __syncthreads();
  for (int w = nodes >> 1; w >= 1; w >>= 1) {  // parent j = left 2j + right 2j+1
    double v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int j = k * kThreads + threadIdx.x;
      v[k] = j < w ? __dadd_rn(sm[2 * j], sm[2 * j + 1]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int j = k * kThreads + threadIdx.x;
      if (j < w) sm[j] = v[k];
    }
    __syncthreads();
  }
  const double total = sm[0];
  __syncthreads();
  return total;
}

// ------------------------------------------------------------------------
// A sequentially rounded running sum, evaluated in parallel and exactly:
//   x[i+1] = RN(x[i] + f[i])          out[i] = x[i+1],  i < n
// (f[i] >= 0; f == nullptr: every f[i] = fconst).  Write x = (2^52 + K) u +
// 0 with K its mantissa field and u = 2^(E-1075) its ulp (E the biased
// exponent).  While x stays in one binade, RN(x + f) only moves K along that
// grid: with f/u = g + r (g integer, 0 <= r < 1)
//   r != 1/2:  K -> K + G,  G = g + (r > 1/2)
//   r == 1/2:  K -> even(K + g)   (round half to even: the even of K+g, K+g+1)
// as long as x + f < 2^(E-1022) - u/2.  Both maps are of the form
// K -> even(K + a) + b or K -> K + a, a family closed under composition
// (even(even(y) + k) = even(y) + even(k)), so a tile is one block-wide scan of
// these maps applied to the tile's starting K -- up to the first element that
// leaves the binade or meets a subnormal-range x.  That element (and, while
// the parallel form keeps stopping early -- the first doublings of x -- a
// growing run after it) is added by one thread with the plain RN add.  Every
// accepted value is the double with exponent E and mantissa K, so the result
// is bit-identical to the sequential loop.  Tiles of 8192 elements are
// staged in shared memory (coalesced loads and stores; each thread owns 8
// contiguous elements).
constexpr int kChainE = 8;                         // elements per thread per tile
constexpr int kChainTile = kSusThreads * kChainE;  // 8192
constexpr uint64_t kChainSat = 1ull << 60;         // saturation (any K >= 2^52 is out of the binade)
constexpr int kChainGoodRun = 64;                  // a parallel run this long resets the scalar budget
constexpr int kChainWarm = 1024;                   // plain adds at least this far (an attempt costs ~14k cycles)
constexpr int kChainMaxBudget = 1 << 16;

// Dynamic shared memory of a kernel calling exact_chain_block: one padded tile.
constexpr size_t kChainSmem = (size_t)(kChainTile + kChainTile / 8) * sizeof(double);
__device__ __forceinline__ int chain_pad(int i) { return i + (i >> 3); }  // rows of 8, stride 9: conflict-free

__device__ __forceinline__ uint64_t chain_sat(uint64_t v) { return v > kChainSat ? kChainSat : v; }
__device__ __forceinline__ uint64_t chain_even(uint64_t v) { return v + (v & 1); }

// K -> e ? even(K + a) + b : K + a
struct ChainMap {
  uint64_t a, b;
  bool e;
};
__device__ __forceinline__ ChainMap chain_then(const ChainMap& f1, const ChainMap& f2) {  // f1, then f2
  if (!f2.e) return f1.e ? ChainMap{f1.a, chain_sat(f1.b + f2.a), true} : ChainMap{chain_sat(f1.a + f2.a), 0, false};
  if (!f1.e) return ChainMap{chain_sat(f1.a + f2.a), f2.b, true};
  return ChainMap{f1.a, chain_sat(chain_even(f1.b + f2.a) + f2.b), true};
}
__device__ __forceinline__ uint64_t chain_apply(const ChainMap& f, uint64_t K) {
  return f.e ? chain_sat(chain_even(chain_sat(K + f.a)) + f.b) : chain_sat(K + f.a);
}
__device__ __forceinline__ ChainMap chain_shfl_up(const ChainMap& m, int o) {
  ChainMap r;
  r.a = __shfl_up_sync(0xffffffffu, m.a, o);
  r.b = __shfl_up_sync(0xffffffffu, m.b, o);
  r.e = __shfl_up_sync(0xffffffffu, (int)m.e, o) != 0;
  return r;
}

#ifdef ISQ_SUS_PROFILE
// per block: parallel attempts, scalar elements, parallel cycles, scalar cycles
__device__ unsigned long long g_sus_prof[2][4];
#define SUS_PROF(k, v) \
  if (threadIdx.x == 0) atomicAdd(&g_sus_prof[blockIdx.x & 1][k], (unsigned long long)(v))
#else
#define SUS_PROF(k, v)
#endif

// One staged tile [0, len) of the chain (global offset j, values in sbuf,
// or the constant fconst when has_f is false), from x; the outputs replace
// the values in sbuf.  The scalar-run state (budget, grow, warm) carries
// over from tile to tile.
struct ChainState {
  double x;
  int budget;  // elements still to add on one thread before the next parallel attempt
  int grow;    // the budget after a short parallel run (doubles while they stay short)
  bool warm;   // the first doublings of x: plain adds (see the scalar branch)
};
__device__ inline void chain_tile_exact(bool has_f, double fconst, int64_t j, int len, ChainState& cs,
                                        double* sbuf) {
  __shared__ ChainMap s_warp[kSusThreads / 32];
  __shared__ int s_stop, s_pos, s_budget;
  __shared__ bool s_warm;
  __shared__ double s_x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* f = has_f ? sbuf : nullptr;  // only tested against null below
  double x = cs.x;
  int budget = cs.budget, grow = cs.grow;
  bool warm = cs.warm, warm_done = false;
  int pos = 0;
  while (pos < len) {
    if (budget > 0) {  // plain adds on thread 0, in shared memory
#ifdef ISQ_SUS_PROFILE
      const long long t0 = clock64();
#endif
      if (tid == 0) {
        int end = pos + budget < len ? pos + budget : len;
        int i = pos;
        if (warm) {  // warm-up: to the first binade change after kChainWarm elements (a parallel
                     // attempt then starts near a binade's start and covers about as many
                     // elements as came before)
          bool more = true;
          while (more && i + 8 <= len) {  // groups of 8: the loads ahead of the dependent adds
            const int eb = (int)((uint64_t)__double_as_longlong(x) >> 52);
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = f ? sbuf[chain_pad(i + k)] : fconst;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              x = __dadd_rn(x, v[k]);
              sbuf[chain_pad(i + k)] = x;
            }
            i += 8;
            more = j + i < kChainWarm || (int)((uint64_t)__double_as_longlong(x) >> 52) == eb;
          }
          while (more && i < len) {
            const int eb = (int)((uint64_t)__double_as_longlong(x) >> 52);
            x = __dadd_rn(x, f ? sbuf[chain_pad(i)] : fconst);
            sbuf[chain_pad(i)] = x;
            ++i;
            more = j + i < kChainWarm || (int)((uint64_t)__double_as_longlong(x) >> 52) == eb;
          }
          end = i;
          warm_done = !more;
        }
        for (; i + 8 <= end; i += 8) {
          double v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = f ? sbuf[chain_pad(i + k)] : fconst;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            x = __dadd_rn(x, v[k]);
            sbuf[chain_pad(i + k)] = x;
          }
        }
        for (; i < end; ++i) {
          x = __dadd_rn(x, f ? sbuf[chain_pad(i)] : fconst);
          sbuf[chain_pad(i)] = x;
        }
        s_x = x;
        s_pos = end;
        s_budget = warm ? (warm_done ? 0 : 1) : budget - (end - pos);
        s_warm = warm && !warm_done;
      }
      __syncthreads();
      SUS_PROF(1, s_pos - pos);
      SUS_PROF(3, clock64() - t0);
      x = s_x;
      pos = s_pos;
      budget = s_budget;
      warm = s_warm;
      __syncthreads();
      continue;
    }
    // parallel attempt on [pos, len)
#ifdef ISQ_SUS_PROFILE
    const long long t1 = clock64();
#endif
    const bool par = x >= 0x1p-900;  // block-uniform
    const uint64_t xb = (uint64_t)__double_as_longlong(x);
    const int E = (int)((xb >> 52) & 0x7ff);
    const int ue = E - 1075;                          // u = 2^ue
    const uint64_t K0 = xb & ((1ull << 52) - 1);
    if (tid == 0) s_stop = par ? len : pos;
    const int i0 = tid * kChainE;
    ChainMap op[kChainE];
    uint64_t F2[kChainE];  // floor(2 f/u)
    ChainMap mine{0, 0, false};
    int my_stop = INT32_MAX;
#pragma unroll
    for (int e = 0; e < kChainE; ++e) {
      const int i = i0 + e;
      op[e] = ChainMap{0, 0, false};
      F2[e] = 0;
      if (par && i >= pos && i < len) {
        const uint64_t fb = (uint64_t)__double_as_longlong(f ? sbuf[chain_pad(i)] : fconst);
        const int ex = (int)((fb >> 52) & 0x7ff);
        const uint64_t m = (fb & ((1ull << 52) - 1)) | (ex ? (1ull << 52) : 0ull);  // f = m 2^(ex-1075)
        const int shift = ue - (ex ? ex - 1075 : -1074);
        if (ex == 0x7ff || (m != 0 && shift <= 0)) {
          my_stop = min(my_stop, i);  // inf / nan, or f >= 2^52 u: leaves the binade
        } else if (m != 0 && shift < 64) {
          const uint64_t g0 = m >> shift, rem = m & ((1ull << shift) - 1), half = 1ull << (shift - 1);
          if (g0 >= (1ull << 52)) my_stop = min(my_stop, i);
          op[e] = rem == half ? ChainMap{g0, 0, true} : ChainMap{g0 + (rem > half ? 1u : 0u), 0, false};
          F2[e] = m >> (shift - 1);
        }  // shift >= 64: f < u / 2^10, the identity map
        mine = chain_then(mine, op[e]);
      }
    }
    // exclusive block scan of the per-thread maps
    ChainMap incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const ChainMap v = chain_shfl_up(incl, o);
      if (lane >= o) incl = chain_then(v, incl);
    }
    if (lane == 31) s_warp[wid] = incl;
    ChainMap excl = chain_shfl_up(incl, 1);
    if (lane == 0) excl = ChainMap{0, 0, false};
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the warp totals
      ChainMap w = lane < kSusThreads / 32 ? s_warp[lane] : ChainMap{0, 0, false};
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const ChainMap v = chain_shfl_up(w, o);
        if (lane >= o) w = chain_then(v, w);
      }
      ChainMap ex = chain_shfl_up(w, 1);
      if (lane == 0) ex = ChainMap{0, 0, false};
      if (lane < kSusThreads / 32) s_warp[lane] = ex;
    }
    __syncthreads();
    const ChainMap pre = chain_then(s_warp[wid], excl);
    // binade check on each element's starting K: x[i] + f[i] < 2^(E-1022) - u/2
    //   <=>  floor(2 f/u) < 2^53 - 1 - 2 K[i]
    uint64_t Kst = chain_apply(pre, K0);
    if (par) {
      uint64_t k = Kst;
#pragma unroll
      for (int e = 0; e < kChainE; ++e) {
        const int i = i0 + e;
        if (i >= pos && i < len && i < my_stop) {
          if (k >= (1ull << 52) || F2[e] >= (1ull << 53) - 1 - 2 * k) my_stop = min(my_stop, i);
          k = chain_apply(op[e], k);
          F2[e] = k;  // K[i+1], for the accept pass
        }
      }
      if (my_stop < len) atomicMin(&s_stop, my_stop);
    }
    __syncthreads();
    const int stop = s_stop;
    if (par) {  // accepted [pos, stop) (all checked above: stop <= every my_stop): exponent E, mantissa K[i+1]
#pragma unroll
      for (int e = 0; e < kChainE; ++e) {
        const int i = i0 + e;
        if (i >= pos && i < stop) {
          const double v = __longlong_as_double((long long)(((uint64_t)E << 52) | F2[e]));
          sbuf[chain_pad(i)] = v;
          if (i == stop - 1) s_x = v;
        }
      }
    }
    __syncthreads();
    if (stop > pos) x = s_x;
    // a stop: its element on thread 0 next, with a run after it that grows
    // while the parallel form keeps stopping early
    if (stop < len) {
      if (stop - pos >= kChainGoodRun) {
        grow = 16;
        budget = 1;
      } else {
        grow = min(2 * grow, kChainMaxBudget);
        budget = grow;
      }
    }
    pos = stop;
    __syncthreads();
    SUS_PROF(0, 1);
    SUS_PROF(2, clock64() - t1);
  }
  cs.x = x;
  cs.budget = budget;
  cs.grow = grow;
  cs.warm = warm;
}

// `sbuf`: kChainSmem bytes of shared memory.
__device__ inline void exact_chain_block(const double* f, double fconst, int64_t n, double x0, double* out,
                                         double* sbuf) {
  const int tid = threadIdx.x;
  ChainState cs{x0, 1, 16, true};
  for (int64_t j = 0; j < n; j += kChainTile) {
    const int len = (int)(n - j < kChainTile ? n - j : kChainTile);
#pragma unroll
    for (int k = 0; k < kChainE; ++k) {  // coalesced tile load (the constant chain stages nothing)
      const int i = k * kSusThreads + tid;
      if (f != nullptr && i < len) sbuf[chain_pad(i)] = f[j + i];
    }
    __syncthreads();
    chain_tile_exact(f != nullptr, fconst, j, len, cs, sbuf);
#pragma unroll
    for (int k = 0; k < kChainE; ++k) {  // coalesced store of the tile
      const int i = k * kSusThreads + tid;
      if (i < len) out[j + i] = sbuf[chain_pad(i)];
    }
    __syncthreads();
  }
#ifdef ISQ_SUS_PROFILE
  if (tid == 0)
    printf("exact_chain_block n=%lld const=%d: attempts %llu scalar %llu par_cycles %llu scalar_cycles %llu\n",
           (long long)n, f == nullptr, g_sus_prof[blockIdx.x & 1][0], g_sus_prof[blockIdx.x & 1][1],
           g_sus_prof[blockIdx.x & 1][2], g_sus_prof[blockIdx.x & 1][3]);
#endif
}

// The same recurrence with a constant increment (the SUS pointers,
// x[k+1] = RN(x[k] + spacing)): inside a binade every step applies the same
// map, so K after i steps is closed-form -- K[1] = map(K[0]), then + d per
// step (d = G, or even(g) for an exact tie: K[1] is even then) -- and the
// steps that stay in the binade are a prefix counted directly.  One round per
// binade (plus one plain add for the step that leaves it), the values written
// by the whole block.
__device__ inline void exact_const_chain_block(double inc, int64_t n, double x0, double* out) {
  __shared__ double s_x;
  __shared__ int64_t s_m;
  __shared__ uint64_t s_K1, s_d;
  __shared__ int s_E;
  const int tid = threadIdx.x;
  double x = x0;
  int64_t j = 0;
  while (j < n) {
    if (tid == 0) {
      int64_t m = 0;
      uint64_t K1 = 0, d = 0;
      const uint64_t xb = (uint64_t)__double_as_longlong(x);
      const int E = (int)((xb >> 52) & 0x7ff);
      const uint64_t fb = (uint64_t)__double_as_longlong(inc);
      const int ex = (int)((fb >> 52) & 0x7ff);
      if (x >= 0x1p-900 && ex != 0x7ff) {
        const uint64_t K0 = xb & ((1ull << 52) - 1);
        const uint64_t mm = (fb & ((1ull << 52) - 1)) | (ex ? (1ull << 52) : 0ull);
        const int shift = (E - 1075) - (ex ? ex - 1075 : -1074);
        uint64_t F2 = 0;
        bool ok = true;
        ChainMap op{0, 0, false};
        if (mm != 0 && shift <= 0) {
          ok = false;
        } else if (mm != 0 && shift < 64) {
          const uint64_t g0 = mm >> shift, rem = mm & ((1ull << shift) - 1), half = 1ull << (shift - 1);
          ok = g0 < (1ull << 52);
          op = rem == half ? ChainMap{g0, 0, true} : ChainMap{g0 + (rem > half ? 1u : 0u), 0, false};
          F2 = mm >> (shift - 1);
        }
        if (ok && F2 < (1ull << 53) - 1) {
          const uint64_t Kmax = ((1ull << 53) - 2 - F2) / 2;  // a step from K stays inside iff K <= Kmax
          if (K0 <= Kmax && K0 < (1ull << 52)) {
            K1 = chain_apply(op, K0);
            d = op.e ? chain_even(op.a) : op.a;
            const int64_t rest = n - j;
            if (K1 > Kmax) {
              m = 1;
            } else if (d == 0) {
              m = rest;
            } else {
              const uint64_t more = (Kmax - K1) / d + 1;  // steps 1 .. more start at or below Kmax
              m = more + 1 >= (uint64_t)rest ? rest : (int64_t)(more + 1);
            }
            if (m > rest) m = rest;
          }
        }
        s_E = E;
      }
      s_m = m;
      s_K1 = K1;
      s_d = d;
      if (m == 0) {  // the step leaves the binade (or x is in the subnormal range): the plain add
        x = __dadd_rn(x, inc);
        out[j] = x;
        s_x = x;
      } else {
        s_x = __longlong_as_double((long long)(((uint64_t)s_E << 52) | (K1 + (uint64_t)(m - 1) * d)));
      }
    }
    __syncthreads();
    const int64_t m = s_m;
    if (m > 0) {
      const uint64_t K1 = s_K1, d = s_d, Eb = (uint64_t)s_E << 52;
      for (int64_t i = tid; i < m; i += kSusThreads)
        out[j + i] = __longlong_as_double((long long)(Eb | (K1 + (uint64_t)i * d)));
    }
    x = s_x;
    j += m > 0 ? m : 1;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------
// The cumulative sum over many tiles (P - 1 >= kChainGridMinTiles tiles): the
// tiles' maps are computed in parallel over the GPU, only the carry between
// them is serial.
//   sums     tile sums (any order) -> apx[t], an approximate prefix: x at tile
//            t's start to within ~1e-12 relative, so its binade E[t] is the
//            exact one unless x sits at a binade edge;
//   analyze  per tile, under E[t]: the composite map of the whole tile, its
//            headroom H[t] = max_i 2 (a_i + b_i) + 2 + floor(2 f_i/u) over the
//            prefix maps (K[i] <= K[0] + a_i + b_i + 1, so 2 K[0] + H[t] <
//            2^53 - 1 keeps every element of the tile inside the binade), and
//            whether any element leaves the grid form outright;
//   serial   one block walks the tiles: a tile whose start x has exponent
//            E[t] and passes the headroom test advances x by its map (O(1));
//            any other tile (the first doublings of x, the ~20 binade
//            crossings) runs chain_tile_exact from x and writes its outputs;
//   apply    the other tiles' outputs from their exact start values.
// Exact as exact_chain_block (same maps, same plain adds), far fewer serial
// steps.
constexpr int64_t kChainGridMinTiles = 16;

struct ChainGridScratch {
  double* apx;      // approximate prefix at each tile's start
  double* xs;       // exact x at each tile's start (serial)
  uint64_t* map_a;  // composite map of each tile under E[t]
  uint64_t* map_b;
  uint64_t* head;   // headroom H[t]; UINT64_MAX: the grid form does not hold
  int* E;           // binade exponent assumed for tile t
  int* slow;        // tile t was processed exactly by the serial kernel
  uint8_t* map_e;
  double* parts;    // pairwise_parts_kernel's subtree sums (2^kPwMaxDepth)
};
constexpr size_t kChainGridTileBytes = 5 * 8 + 4 + 4 + 1;  // per tile: apx xs map_a map_b head, E slow, map_e
__host__ __device__ inline size_t chain_grid_scratch_bytes(int64_t n) {
  const int64_t T = (n + kChainTile - 1) / kChainTile;
  return (((size_t)T * kChainGridTileBytes + 63) & ~(size_t)63) + ((size_t)8 << kPwMaxDepth);
}
__host__ __device__ inline ChainGridScratch chain_grid_scratch(void* base, int64_t n) {
  const int64_t T = (n + kChainTile - 1) / kChainTile;
  ChainGridScratch g;
  char* p = static_cast<char*>(base);
  g.apx = reinterpret_cast<double*>(p);
  g.xs = g.apx + T;
  g.map_a = reinterpret_cast<uint64_t*>(g.xs + T);
  g.map_b = g.map_a + T;
  g.head = g.map_b + T;
  g.E = reinterpret_cast<int*>(g.head + T);
  g.slow = g.E + T;
  g.map_e = reinterpret_cast<uint8_t*>(g.slow + T);
  g.parts = reinterpret_cast<double*>(p + (((size_t)T * kChainGridTileBytes + 63) & ~(size_t)63));
  return g;
}

// Per-thread maps of a staged tile under exponent E (the attempt's first
// pass): op / F2 for the thread's kChainE elements, the exclusive prefix map
// `pre` of its first element, the tile's composite `total`, `bad` if an
// element leaves the grid form outright.  Block-wide (syncs).
__device__ inline void chain_tile_maps(const double* sbuf, int len, int E, ChainMap (&op)[kChainE],
                                       uint64_t (&F2)[kChainE], ChainMap& pre, ChainMap& total, bool& bad) {
  __shared__ ChainMap s_warp[kSusThreads / 32];
  __shared__ ChainMap s_total;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ue = E - 1075;
  const int i0 = tid * kChainE;
  ChainMap mine{0, 0, false};
  bad = false;
#pragma unroll
  for (int e = 0; e < kChainE; ++e) {
    const int i = i0 + e;
    op[e] = ChainMap{0, 0, false};
    F2[e] = 0;
    if (i < len) {
      const uint64_t fb = (uint64_t)__double_as_longlong(sbuf[chain_pad(i)]);
      const int ex = (int)((fb >> 52) & 0x7ff);
      const uint64_t m = (fb & ((1ull << 52) - 1)) | (ex ? (1ull << 52) : 0ull);
      const int shift = ue - (ex ? ex - 1075 : -1074);
      if (ex == 0x7ff || (fb >> 63) || (m != 0 && shift <= 0)) {
        bad = true;
      } else if (m != 0 && shift < 64) {
        const uint64_t g0 = m >> shift, rem = m & ((1ull << shift) - 1), half = 1ull << (shift - 1);
        if (g0 >= (1ull << 52)) bad = true;
        op[e] = rem == half ? ChainMap{g0, 0, true} : ChainMap{g0 + (rem > half ? 1u : 0u), 0, false};
        F2[e] = m >> (shift - 1);
      }
      mine = chain_then(mine, op[e]);
    }
  }
  ChainMap incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const ChainMap v = chain_shfl_up(incl, o);
    if (lane >= o) incl = chain_then(v, incl);
  }
  if (lane == 31) s_warp[wid] = incl;
  ChainMap excl = chain_shfl_up(incl, 1);
  if (lane == 0) excl = ChainMap{0, 0, false};
  __syncthreads();
  if (wid == 0) {
    ChainMap w = lane < kSusThreads / 32 ? s_warp[lane] : ChainMap{0, 0, false};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const ChainMap v = chain_shfl_up(w, o);
      if (lane >= o) w = chain_then(v, w);
    }
    if (lane == kSusThreads / 32 - 1) s_total = w;
    ChainMap ex = chain_shfl_up(w, 1);
    if (lane == 0) ex = ChainMap{0, 0, false};
    if (lane < kSusThreads / 32) s_warp[lane] = ex;
  }
  __syncthreads();
  pre = chain_then(s_warp[wid], excl);
  total = s_total;
  __syncthreads();
}

__device__ __forceinline__ void chain_load_tile(const double* f, int64_t j, int len, double* sbuf) {
#pragma unroll
  for (int k = 0; k < kChainE; ++k) {
    const int i = k * kSusThreads + threadIdx.x;
    if (i < len) sbuf[chain_pad(i)] = f[j + i];
  }
  __syncthreads();
}

// Tile sums, then (block 0 of a second launch) their exclusive prefix.
static __global__ void __launch_bounds__(kSusThreads) chain_tile_sums_kernel(const double* f, int64_t n, double* apx) {
  __shared__ double s_part[kSusThreads / 32];
  const int64_t j = (int64_t)blockIdx.x * kChainTile;
  double v = 0.0;
  for (int64_t i = j + threadIdx.x; i < n && i < j + kChainTile; i += kSusThreads) v += f[i];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSusThreads / 32; ++w) t += s_part[w];
    apx[blockIdx.x] = t;
  }
}
static __global__ void chain_prefix_kernel(double* apx, int64_t T, double x0) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double run = x0;
    for (int64_t t = 0; t < T; ++t) {
      const double v = apx[t];
      apx[t] = run;
      run += v;
    }
  }
}

static __global__ void __launch_bounds__(kSusThreads) chain_analyze_kernel(const double* f, int64_t n, ChainGridScratch g) {
  extern __shared__ double sbuf[];
  __shared__ int s_bad;
  __shared__ unsigned long long s_head;
  const int64_t t = blockIdx.x;
  const int64_t j = t * kChainTile;
  const int len = (int)(n - j < kChainTile ? n - j : kChainTile);
  const double ax = g.apx[t];
  const int E = (int)(((uint64_t)__double_as_longlong(ax) >> 52) & 0x7ff);
  if (!(ax >= 0x1p-900) || E == 0x7ff) {  // subnormal-range (or non-finite) start: exact path
    if (threadIdx.x == 0) {
      g.head[t] = UINT64_MAX;
      g.E[t] = E;
    }
    return;
  }
  if (threadIdx.x == 0) {
    s_bad = 0;
    s_head = 0;
  }
  chain_load_tile(f, j, len, sbuf);
  ChainMap op[kChainE], pre, total;
  uint64_t F2[kChainE];
  bool bad;
  chain_tile_maps(sbuf, len, E, op, F2, pre, total, bad);
  uint64_t h = 0;
  ChainMap p = pre;
#pragma unroll
  for (int e = 0; e < kChainE; ++e) {
    const int i = threadIdx.x * kChainE + e;
    if (i < len) {
      const uint64_t hi = chain_sat(chain_sat(2 * chain_sat(p.a + p.b)) + 2 + F2[e]);
      h = hi > h ? hi : h;
      p = chain_then(p, op[e]);
    }
  }
  if (bad) s_bad = 1;
  atomicMax(&s_head, (unsigned long long)h);
  __syncthreads();
  if (threadIdx.x == 0) {
    g.head[t] = s_bad ? UINT64_MAX : (uint64_t)s_head;
    g.map_a[t] = total.a;
    g.map_b[t] = total.b;
    g.map_e[t] = total.e ? 1 : 0;
    g.E[t] = E;
  }
}

// One block: the carry through the tiles (see above).
static __global__ void __launch_bounds__(kSusThreads) chain_serial_kernel(const double* f, int64_t n, double x0,
                                                                   double* out, ChainGridScratch g) {
  extern __shared__ double sbuf[];
  __shared__ int s_fast;
  __shared__ double s_x;
  const int64_t T = (n + kChainTile - 1) / kChainTile;
  ChainState cs{x0, 1, 16, true};
  for (int64_t t = 0; t < T; ++t) {
    const int64_t j = t * kChainTile;
    const int len = (int)(n - j < kChainTile ? n - j : kChainTile);
    if (threadIdx.x == 0) {
      const uint64_t xb = (uint64_t)__double_as_longlong(cs.x);
      const int E = (int)((xb >> 52) & 0x7ff);
      const uint64_t K = xb & ((1ull << 52) - 1);
      const uint64_t H = g.head[t];
      const bool fast = !cs.warm && cs.x >= 0x1p-900 && E == g.E[t] && H != UINT64_MAX &&
                        H < (1ull << 53) - 1 && 2 * K < (1ull << 53) - 1 - H;
      g.xs[t] = cs.x;
      g.slow[t] = fast ? 0 : 1;
      s_fast = fast;
      if (fast) {
        const ChainMap m{g.map_a[t], g.map_b[t], g.map_e[t] != 0};
        s_x = __longlong_as_double((long long)(((uint64_t)E << 52) | chain_apply(m, K)));
      }
    }
    __syncthreads();
    if (s_fast) {
      cs.x = s_x;  // the next tile starts a fresh parallel attempt
      cs.budget = 0;
      cs.grow = 16;
    } else {
      chain_load_tile(f, j, len, sbuf);
      chain_tile_exact(true, 0.0, j, len, cs, sbuf);
#pragma unroll
      for (int k = 0; k < kChainE; ++k) {
        const int i = k * kSusThreads + threadIdx.x;
        if (i < len) out[j + i] = sbuf[chain_pad(i)];
      }
    }
    __syncthreads();
  }
}

static __global__ void __launch_bounds__(kSusThreads) chain_apply_kernel(const double* f, int64_t n, double* out,
                                                                  ChainGridScratch g) {
  extern __shared__ double sbuf[];
  const int64_t t = blockIdx.x;
  if (g.slow[t]) return;
  const int64_t j = t * kChainTile;
  const int len = (int)(n - j < kChainTile ? n - j : kChainTile);
  const int E = g.E[t];
  chain_load_tile(f, j, len, sbuf);
  ChainMap op[kChainE], pre, total;
  uint64_t F2[kChainE];
  bool bad;
  chain_tile_maps(sbuf, len, E, op, F2, pre, total, bad);
  const uint64_t K0 = (uint64_t)__double_as_longlong(g.xs[t]) & ((1ull << 52) - 1);
  uint64_t k = chain_apply(pre, K0);
#pragma unroll
  for (int e = 0; e < kChainE; ++e) {
    const int i = threadIdx.x * kChainE + e;
    if (i < len) {
      k = chain_apply(op[e], k);
      out[j + i] = __longlong_as_double((long long)(((uint64_t)E << 52) | k));
    }
  }
}

inline bool chain_grid_worth(int64_t n) { return n >= kChainGridMinTiles * kChainTile; }

// The kernels' dynamic shared memory attribute, on the current device (call
// outside stream capture, before the first launch).
static inline cudaError_t prepare_exact_chain_grid() {
  const void* ks[] = {(const void*)chain_analyze_kernel, (const void*)chain_serial_kernel,
                      (const void*)chain_apply_kernel};
  for (const void* k : ks) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// (The kernels and both host functions have internal linkage: each translation
// unit sets the attribute on, and launches, its own copies.)
// Host launcher: the cumulative sums out[i] = x[i+1] of f[0..n) from x0 with
// the grid scheme (scratch: chain_grid_scratch_bytes(n) bytes; after
// prepare_exact_chain_grid).
static inline cudaError_t launch_exact_chain_grid(const double* f, int64_t n, double x0, double* out, void* scratch,
                                           cudaStream_t s) {
  const int64_t T = (n + kChainTile - 1) / kChainTile;
  const ChainGridScratch g = chain_grid_scratch(scratch, n);
  cudaError_t e;
  chain_tile_sums_kernel<<<(unsigned)T, kSusThreads, 0, s>>>(f, n, g.apx);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  chain_prefix_kernel<<<1, 32, 0, s>>>(g.apx, T, x0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  chain_analyze_kernel<<<(unsigned)T, kSusThreads, kChainSmem, s>>>(f, n, g);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  chain_serial_kernel<<<1, kSusThreads, kChainSmem, s>>>(f, n, x0, out, g);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  chain_apply_kernel<<<(unsigned)T, kSusThreads, kChainSmem, s>>>(f, n, out, g);
  return cudaGetLastError();
}

// np.sum(a[0..n)) stage 1 (pairwise_parts_kernel) into scratch's parts; stage
// 2 is np_pairwise_combine_block(parts, pairwise_grid_depth(n), ...).
static inline cudaError_t launch_pairwise_parts(const double* a, int64_t n, void* scratch, int64_t chain_n,
                                                cudaStream_t s) {
  const int d = pairwise_grid_depth(n);
  pairwise_parts_kernel<<<((1 << d) + 255) / 256, 256, 0, s>>>(a, n, d, chain_grid_scratch(scratch, chain_n).parts);
  return cudaGetLastError();
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

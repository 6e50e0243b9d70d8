// GPUGA baseline generation loop (GaEngine.step, ga.py:165-194).
//
// Genomes live on the device as two (double-buffered by generation parity)
// SoA banks: codes[P*L] u8 (gate_choices index, ga.py:47-59) and thetas[P*L]
// f64.  One generation g:
//   eval    fitness of this rank's genome shard            (fitness_rows)
//   (multi-GPU: all-gather of the fitness vector)
//   reduce  max / first argmax (elite) / mean, best-so-far + genome capture
//   sus     stochastic universal sampling, exact sequential replica of
//           sus_select (ga.py:95-116) incl. numpy's pairwise np.sum
//   breed   thread per (child, gene): two-point crossover of the pair
//           (ga.py:81-92, 177-187) + per-gene mutation (ga.py:119-138); elite
//           copied unmutated to slot 0
//   advance generation += 1, stop reason (ga.py:189-193)
// Draws: per-pair crossover stream (DOM_GA_PAIR, g, pair), per-(child, gene)
// mutation stream (DOM_GA_MUT, g, child, gene), SUS stream (DOM_GA_SUS, g).
#include <cstring>
#include <string>

#include <cooperative_groups.h>

#include "engine_common.cuh"
#include "fitness_multi.cuh"
#include "fitness_warp.cuh"
#include "isq_internal.h"
#include "sus.cuh"

namespace isq {

struct GaDevState {
  uint64_t generation;
  uint64_t rec_base;
  double best_fitness;
  int64_t elite;
  int32_t stop;
  int32_t improved;
};

struct GaArgs {
  int n, L, ncodes;
  int64_t P;
  double rate, mrange, structural, target_fitness;
  uint64_t max_generations, seed;
  uint8_t* codes[2];
  double* thetas[2];
  double* fitness;
  double* fitness_alt;  // cooperative single-barrier launch: odd generations' fitness
  int32_t* parents;
  GaDevState* st;
  GenRecord* records;
  int rec_cap;
  uint8_t* best_codes;
  double* best_thetas;
  const double2* target;
  double* part_max;
  double* part_sum;
  int64_t* part_arg;
  int n_parts;
  double* sus_C;  // P > kSusCache: the walk's running sums (sus.cuh)
  double* sus_P;
  int* sus_flag;
  void* sus_grid;  // P - 1 >= chain_grid_worth: scratch of the grid-wide chain (else null)
  int precision;  // fitness arithmetic: ISQ_PRECISION_FP64 / _FP32
  FastDiv div_L, div_P;  // gene index -> genome; pair index mod P (P * L < 2^32)
};

__device__ __forceinline__ int ga_cur(const GaArgs& a) { return (int)(a.st->generation & 1); }

// ------------------------------------------------------------------ eval ---
template <int NQ, int MINB, class R>
__global__ void __launch_bounds__(kFitThreads, MINB) ga_eval_kernel(GaArgs a, int64_t c0, int64_t c1) {
  using G = Geo<NQ>;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ FitScratch<NQ, R> sh[kFitWarps];
  if (a.st->stop) return;
  const int cur = ga_cur(a);
  for (int i = threadIdx.x; i < G::D * G::D; i += blockDim.x) Ts[i] = a.target[i];
  __syncthreads();
  fitness_rows_fast<NQ, R>(c1 - c0, a.L, a.codes[cur] + c0 * a.L, a.thetas[cur] + c0 * a.L, Ts, sh,
                      a.fitness + c0, kFitWarps);
}

// ---------------------------------------------------------------- reduce ---
constexpr int kGaRed = 256;

__device__ __forceinline__ void ga_reduce_partial_body(const GaArgs& a, int part, double* smax, double* ssum,
                                                       int64_t* sarg) {
  const int64_t per = (a.P + a.n_parts - 1) / a.n_parts;
  const int64_t lo = (int64_t)part * per;
  const int64_t hi = min(a.P, lo + per);
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kGaRed) {
    const double f = a.fitness[i];
    sum += f;
    if (f > m) {
      m = f;
      arg = i;
    }
  }
  smax[threadIdx.x] = m;
  ssum[threadIdx.x] = sum;
  sarg[threadIdx.x] = arg;
  __syncthreads();
  for (int off = kGaRed / 2; off >= 1; off >>= 1) {
    if (threadIdx.x < off) {
      const double m2 = smax[threadIdx.x + off];
      const int64_t a2 = sarg[threadIdx.x + off];
      if (m2 > smax[threadIdx.x] || (m2 == smax[threadIdx.x] && a2 < sarg[threadIdx.x])) {
        smax[threadIdx.x] = m2;
        sarg[threadIdx.x] = a2;
      }
      ssum[threadIdx.x] += ssum[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.part_max[part] = smax[0];
    a.part_sum[part] = ssum[0];
    a.part_arg[part] = sarg[0];
  }
}

__global__ void __launch_bounds__(kGaRed) ga_reduce_partials(GaArgs a) {
  if (a.st->stop) return;
  __shared__ double smax[kGaRed], ssum[kGaRed];
  __shared__ int64_t sarg[kGaRed];
  ga_reduce_partial_body(a, blockIdx.x, smax, ssum, sarg);
}

// Final reduction + best-so-far update (ga.py:171-174) + SUS (ga.py:95-116).
// SUS is a sequential walk (cumulative sums compared against pointer +=
// spacing): thread 0 replays its two running sums exactly, the picks are
// then searched in parallel (below); warp 0 copies the elite genome.
constexpr int kSusCache = 512;   // fitness values staged in shared memory for the sequential walk

struct NoIdleWork {
  __device__ __forceinline__ void operator()() const {}
};

// `idle` runs on threads 1.. of the block while thread 0 walks the SUS.
// With `scratch` (>= P doubles of shared memory, P <= kSusCache) the walk is
// replaced by its exact parallel form: thread 0 writes the walk's running
// sums C[i+1] = C[i] + f[i] (in place over the staged fitness) and its
// pointer sequence p[k+1] = p[k] + spacing, both in the walk's own
// sequential rounding, and every thread k finds parents[k] = the first
// i <= P-2 with C[i+1] > p[k] (else P-1) by binary search: both sequences are
// nondecreasing (fitness >= 0), so that is where the walk stops.
// Thread 0: combine the partial reductions, best-so-far update (ga.py:171-174),
// generation record.
__device__ __forceinline__ void ga_reduce_final(const GaArgs& a, int& s_improved, int64_t& s_elite) {
  GaDevState* st = a.st;
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  for (int i = 0; i < a.n_parts; ++i) {
    const double pm = a.part_max[i];
    if (pm > m || (pm == m && a.part_arg[i] < arg)) {
      m = pm;
      arg = a.part_arg[i];
    }
    sum += a.part_sum[i];
  }
  const int improved = m > st->best_fitness;
  if (improved) st->best_fitness = m;
  st->elite = arg;
  st->improved = improved;
  GenRecord r;
  r.gen_best = m;
  r.gen_mean = sum / (double)a.P;
  r.best_fitness = st->best_fitness;
  r.pad = 0.0;
  const uint64_t ri = st->generation - st->rec_base;
  if (ri < (uint64_t)a.rec_cap) a.records[ri] = r;
  s_improved = improved;
  s_elite = arg;
}

template <class Idle = NoIdleWork>
__device__ __forceinline__ void ga_reduce_sus_body(const GaArgs& a, int* s_improved_p, int64_t* s_elite_p,
                                                   Idle idle = Idle(), double* scratch = nullptr,
                                                   int scratch_n = 0) {
  __shared__ double sfit[kSusCache];
  __shared__ int s_search;
  int& s_improved = *s_improved_p;
  int64_t& s_elite = *s_elite_p;
  GaDevState* st = a.st;
  const int cur = ga_cur(a);
  // the walk below is one thread's dependent loads: serve them from shared memory
  const bool cached = a.P <= kSusCache;
  if (cached)
    for (int64_t i = threadIdx.x; i < a.P; i += blockDim.x) sfit[i] = a.fitness[i];
  __syncthreads();
  const double* fit = cached ? sfit : a.fitness;
  if (threadIdx.x == 0) {
    ga_reduce_final(a, s_improved, s_elite);

    // ---- sus_select(fitnesses, P, stream) ----
    NpStream rs;
    rs.init(a.seed, DOM_GA_SUS, st->generation, 0, 0);
    const double total = np_pairwise_sum(fit, a.P);
    int search = 0;
    if (total <= 0.0) {
      for (int64_t k = 0; k < a.P; ++k) a.parents[k] = (int32_t)rs.integers(a.P);
    } else if (cached && scratch != nullptr && a.P <= scratch_n) {
      const double spacing = __ddiv_rn(total, (double)a.P);
      double pointer = rs.uniform(0.0, spacing);
      double cumulative = 0.0;
      for (int k = 0; k < (int)a.P; ++k) {
        cumulative = __dadd_rn(cumulative, sfit[k]);
        sfit[k] = cumulative;  // C[k + 1]
        scratch[k] = pointer;
        pointer = __dadd_rn(pointer, spacing);
      }
      search = 1;
    } else {
      const double spacing = __ddiv_rn(total, (double)a.P);
      double pointer = rs.uniform(0.0, spacing);
      double cumulative = 0.0;
      int64_t index = 0;
      for (int64_t k = 0; k < a.P; ++k) {
        while (index < a.P - 1 && __dadd_rn(cumulative, fit[index]) <= pointer) {
          cumulative = __dadd_rn(cumulative, fit[index]);
          ++index;
        }
        a.parents[k] = (int32_t)index;
        pointer = __dadd_rn(pointer, spacing);
      }
    }
    s_search = search;
  } else {
    idle();
  }
  __syncthreads();
  if (s_search) {
    for (int k = threadIdx.x; k < (int)a.P; k += blockDim.x) {
      const double pk = scratch[k];
      int lo = 0, hi = (int)a.P - 1;  // first j in [0, P-2] with C[j + 1] > pk, else P - 1
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sfit[mid] <= pk)
          lo = mid + 1;
        else
          hi = mid;
      }
      a.parents[k] = lo;
    }
    __syncthreads();
  }
  if (s_improved && threadIdx.x < 32) {
    for (int j = threadIdx.x; j < a.L; j += 32) {
      a.best_codes[j] = a.codes[cur][s_elite * a.L + j];
      a.best_thetas[j] = a.thetas[cur][s_elite * a.L + j];
    }
  }
}

__global__ void __launch_bounds__(kGaRed) ga_reduce_sus_kernel(GaArgs a) {
  __shared__ int s_improved;
  __shared__ int64_t s_elite;
  __shared__ double pointers[kSusCache];
  if (a.st->stop) return;
  ga_reduce_sus_body(a, &s_improved, &s_elite, NoIdleWork(), pointers, kSusCache);
}

// P > kSusCache: the same selection on two blocks (sus.cuh).  Block 0: the
// final reduction and record, then the cumulative sums C[1..P-1] and the
// elite copy; block 1: numpy's pairwise total, then the pointer sequence (or,
// when every fitness is zero, the uniform draws, with the flag telling
// sus_search_kernel to skip).  The running sums are exact-parallel
// (exact_chain_block), bit-identical to the sequential walk.
__global__ void __launch_bounds__(kSusThreads) ga_reduce_sus_large_kernel(GaArgs a) {
  __shared__ int s_improved;
  __shared__ int64_t s_elite;
  __shared__ double sm[kSusThreads];
  extern __shared__ double chain_smem[];
  if (a.st->stop) return;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) ga_reduce_final(a, s_improved, s_elite);
    if (a.sus_grid == nullptr) exact_chain_block(a.fitness, 0.0, a.P - 1, 0.0, a.sus_C, chain_smem);
    __syncthreads();  // s_improved / s_elite
    if (s_improved && threadIdx.x < 32) {
      const int cur = ga_cur(a);
      for (int j = threadIdx.x; j < a.L; j += 32) {
        a.best_codes[j] = a.codes[cur][s_elite * a.L + j];
        a.best_thetas[j] = a.thetas[cur][s_elite * a.L + j];
      }
    }
    return;
  }
  const double total =
      a.sus_grid != nullptr
          ? np_pairwise_combine_block<kSusThreads>(chain_grid_scratch(a.sus_grid, a.P - 1).parts,
                                                   pairwise_grid_depth(a.P), chain_smem)
          : np_pairwise_sum_block<kSusThreads>(a.fitness, a.P, sm);
  NpStream rs;
  rs.init(a.seed, DOM_GA_SUS, a.st->generation, 0, 0);
  if (total <= 0.0) {
    if (threadIdx.x == 0) {
      for (int64_t k = 0; k < a.P; ++k) a.parents[k] = (int32_t)rs.integers(a.P);
      *a.sus_flag = 0;
    }
    return;
  }
  const double spacing = __ddiv_rn(total, (double)a.P);
  const double pointer = rs.uniform(0.0, spacing);
  if (threadIdx.x == 0) {
    a.sus_P[0] = pointer;
    *a.sus_flag = 1;
  }
  exact_const_chain_block(spacing, a.P - 1, pointer, a.sus_P + 1);
}

// ----------------------------------------------------------------- breed ---
// Child i >= 1 is the (i-1)%2-th child of pair k = (i-1)/2 of parents
// (parents[2k % P], parents[(2k+1) % P]) (ga.py:177-187); slot 0 is the elite.
// The random draws of gene t (its pair's crossover cuts, its own mutation)
// depend only on (generation, pair / child, gene), so the cooperative kernel
// draws them while block 0 runs the sequential SUS (ga_breed_draw), and
// ga_breed_apply only gathers the parents' genes.
struct GeneDraw {
  int p, q;     // crossover cuts [p, q)
  int mut;      // 0 none, 1 structural (code), 2 angle (delta)
  int code;
  double delta;
};
// two_point_crossover cuts of pair k: p, q = sorted(integers(0, L + 1, size=2)); none for L < 2
__device__ __forceinline__ void ga_pair_cuts(const GaArgs& a, int64_t k, uint64_t g, int& p, int& q) {
  p = q = 0;
  if (a.L >= 2) {
    NpStream cs;
    cs.init(a.seed, DOM_GA_PAIR, g, (uint64_t)k, 0);
    const int x = (int)cs.integers(a.L + 1), y = (int)cs.integers(a.L + 1);
    p = x < y ? x : y;
    q = x < y ? y : x;
  }
}
// ga_mutate for gene j of child i (ga.py:126-137)
__device__ __forceinline__ void ga_gene_mutation(const GaArgs& a, int64_t i, int j, uint64_t g, GeneDraw& d) {
  NpStream ms;
  ms.init(a.seed, DOM_GA_MUT, g, (uint64_t)i, (uint64_t)j);
  if (ms.random() < a.rate) {
    if (ms.random() < a.structural) {
      d.mut = 1;
      d.code = (int)ms.integers(a.ncodes);
    } else {
      d.mut = 2;
      d.delta = ms.uniform(-a.mrange, a.mrange);
    }
  }
}
__device__ __forceinline__ GeneDraw ga_breed_draw(const GaArgs& a, int64_t t, uint64_t g) {
  GeneDraw d;
  d.p = d.q = d.mut = d.code = 0;
  d.delta = 0.0;
  const int64_t i = a.div_L.div((uint32_t)t);
  const int j = (int)(t - i * a.L);
  if (i == 0) return d;
  ga_pair_cuts(a, (i - 1) >> 1, g, d.p, d.q);
  ga_gene_mutation(a, i, j, g, d);
  return d;
}
__device__ __forceinline__ void ga_breed_apply(const GaArgs& a, int64_t t, int cur, int64_t elite,
                                               const GeneDraw& d, const int32_t* parents = nullptr) {
  if (parents == nullptr) parents = a.parents;
  const int nxt = cur ^ 1;
  const int64_t i = a.div_L.div((uint32_t)t);
  const int j = (int)(t - i * a.L);
  if (i == 0) {
    a.codes[nxt][j] = a.codes[cur][elite * a.L + j];
    a.thetas[nxt][j] = a.thetas[cur][elite * a.L + j];
    return;
  }
  const int64_t k = (i - 1) >> 1;
  const bool first = ((i - 1) & 1) == 0;
  const uint32_t k0 = (uint32_t)(2 * k), k1 = k0 + 1u;
  const int64_t pa = parents[k0 - a.div_P.div(k0) * (uint32_t)a.P],
                pb = parents[k1 - a.div_P.div(k1) * (uint32_t)a.P];
  const bool inside = j >= d.p && j < d.q;
  const int64_t src = (first != inside) ? pa : pb;  // child a: a outside, b inside
  int code = a.codes[cur][src * a.L + j];
  double theta = a.thetas[cur][src * a.L + j];
  if (d.mut == 1) code = d.code;
  else if (d.mut == 2) theta = py_mod(__dadd_rn(theta, d.delta), kTwoPiD);
  a.codes[nxt][i * a.L + j] = (uint8_t)code;
  a.thetas[nxt][i * a.L + j] = theta;
}
__device__ __forceinline__ void ga_breed_gene(const GaArgs& a, int64_t t, uint64_t g, int cur, int64_t elite) {
  ga_breed_apply(a, t, cur, elite, ga_breed_draw(a, t, g));
}

// Large populations: chunks of 256 genes; the crossover cuts of the chunk's
// pairs are drawn once per pair into shared memory (not once per gene: the
// pair stream was half of this kernel's Philox work).
constexpr int kBreedThreads = 256;
__global__ void __launch_bounds__(kBreedThreads) ga_breed_kernel(GaArgs a) {
  __shared__ int2 s_cut[kBreedThreads / 2 + 2];
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int cur = ga_cur(a);
  const int64_t total = a.P * a.L;
  const int64_t elite = a.st->elite;
  for (int64_t t0 = (int64_t)blockIdx.x * kBreedThreads; t0 < total; t0 += (int64_t)gridDim.x * kBreedThreads) {
    const int64_t i_lo = a.div_L.div((uint32_t)t0);
    const int64_t i_hi = a.div_L.div((uint32_t)min(total - 1, t0 + kBreedThreads - 1));
    const int64_t k_lo = i_lo >= 1 ? (i_lo - 1) >> 1 : 0;
    const int npairs = i_hi >= 1 ? (int)(((i_hi - 1) >> 1) - k_lo + 1) : 0;
    __syncthreads();  // the previous chunk's readers
    for (int r = threadIdx.x; r < npairs; r += kBreedThreads) {
      int p, q;
      ga_pair_cuts(a, k_lo + r, g, p, q);
      s_cut[r] = make_int2(p, q);
    }
    __syncthreads();
    const int64_t t = t0 + threadIdx.x;
    if (t < total) {
      GeneDraw d;
      d.p = d.q = d.mut = d.code = 0;
      d.delta = 0.0;
      const int64_t i = a.div_L.div((uint32_t)t);
      if (i > 0) {
        const int2 c = s_cut[((i - 1) >> 1) - k_lo];
        d.p = c.x;
        d.q = c.y;
        ga_gene_mutation(a, i, (int)(t - i * a.L), g, d);
      }
      ga_breed_apply(a, t, cur, elite, d);
    }
  }
}

__device__ __forceinline__ void ga_advance_body(const GaArgs& a) {
  GaDevState* st = a.st;
  st->generation += 1;
  if (st->best_fitness >= a.target_fitness)
    st->stop = 1;
  else if (st->generation >= a.max_generations)
    st->stop = 2;
}

__global__ void ga_advance_kernel(GaArgs a) {
  if (a.st->stop) return;
  ga_advance_body(a);
}

// Launch-bound populations (C2): n whole generations in one single-block
// launch over the same device bodies as the multi-kernel generation.
template <int NQ>
__global__ void __launch_bounds__(kGaRed, 1) ga_small_kernel(GaArgs a, int n_gens) {
  using G = Geo<NQ>;
  constexpr int kWarps = kGaRed / 32;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ FitScratch<NQ, double, kSmallNR> sh[kWarps];
  __shared__ double smax[kGaRed], ssum[kGaRed];
  __shared__ int64_t sarg[kGaRed];
  __shared__ int s_improved;
  __shared__ int64_t s_elite;
  for (int i = threadIdx.x; i < G::D * G::D; i += kGaRed) Ts[i] = a.target[i];
  const int64_t genes = a.P * a.L;
  for (int it = 0; it < n_gens; ++it) {
    __syncthreads();
    if (a.st->stop) return;  // uniform: written by thread 0 before the barrier
    const uint64_t g = a.st->generation;
    const int cur = ga_cur(a);
    fitness_rows_fast<NQ, double, kSmallNR, true>(a.P, a.L, a.codes[cur], a.thetas[cur], Ts, sh, a.fitness, kWarps,
                                            nullptr, nullptr, small_cpw<NQ>(a.P, kWarps));
    __syncthreads();
    for (int part = 0; part < a.n_parts; ++part) {
      ga_reduce_partial_body(a, part, smax, ssum, sarg);
      __syncthreads();
    }
    ga_reduce_sus_body(a, &s_improved, &s_elite, NoIdleWork(), ssum, kGaRed);
    __syncthreads();
    const int64_t elite = a.st->elite;
    for (int64_t t = threadIdx.x; t < genes; t += kGaRed) ga_breed_gene(a, t, g, cur, elite);
    __syncthreads();
    if (threadIdx.x == 0) ga_advance_body(a);
  }
}

// random_genome (ga.py:68-73), one stream per (genome, gene).
__global__ void ga_init_kernel(GaArgs a) {
  const int64_t total = a.P * a.L;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / a.L;
    const int j = (int)(t - i * a.L);
    NpStream s;
    s.init(a.seed, DOM_GA_INIT, 0, (uint64_t)i, (uint64_t)j);
    a.codes[0][t] = (uint8_t)s.integers(a.ncodes);
    a.thetas[0][t] = s.uniform(0.0, kTwoPiD);
  }
}

// --------------------------------------------------------------- handle ---
struct GaHandle {
  GaArgs a;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  int64_t shard = 0;
  int max_batch = 0;
  GenGraph graph;  // isq_ga_step on small populations
  int launch_mode = ISQ_LAUNCH_AUTO;
};

static void ga_free(GaHandle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->graph.reset();
  GaArgs& a = h->a;
  for (int b = 0; b < 2; ++b) {
    cudaFree(a.codes[b]);
    cudaFree(a.thetas[b]);
  }
  cudaFree(a.fitness);
  cudaFree(a.fitness_alt);
  cudaFree(a.parents);
  cudaFree(a.st);
  cudaFree(a.records);
  cudaFree(a.best_codes);
  cudaFree(a.best_thetas);
  cudaFree((void*)a.target);
  cudaFree(a.part_max);
  cudaFree(a.part_sum);
  cudaFree(a.part_arg);
  cudaFree(a.sus_C);
  cudaFree(a.sus_P);
  cudaFree(a.sus_flag);
  cudaFree(a.sus_grid);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

static int ga_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

template <int NQ, int MINB, class R>
static isq_status ga_launch_eval_nq(const GaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  const void* k = (const void*)ga_eval_kernel<NQ, MINB, R>;
  const int64_t warps = (c1 - c0 + kFitCPW<NQ> - 1) / kFitCPW<NQ>;
  const int grid = persistent_grid(k, 0, warps, kFitWarps);
  ga_eval_kernel<NQ, MINB, R><<<grid, kFitThreads, 0, s>>>(a, c0, c1);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

template <int NQ>
static isq_status ga_launch_eval_prec(const GaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  if (a.precision == ISQ_PRECISION_FP32) return ga_launch_eval_nq<NQ, fit_min_blocks<NQ, float>(), float>(a, c0, c1, s);
  return ga_launch_eval_nq<NQ, fit_min_blocks<NQ, double>(), double>(a, c0, c1, s);
}

static isq_status ga_launch_eval(const GaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  if (c1 <= c0) return ISQ_OK;
  switch (a.n) {
    case 2: return ga_launch_eval_prec<2>(a, c0, c1, s);
    case 3: return ga_launch_eval_prec<3>(a, c0, c1, s);
    case 4: return ga_launch_eval_prec<4>(a, c0, c1, s);
    case 5: return ga_launch_eval_prec<5>(a, c0, c1, s);
    default:
      if (a.n > ISQ_MAX_FAST_WIRES && a.n <= ISQ_MAX_WIRES)  // the current genomes by generation parity
        return launch_fitness_generic(a.n, a.L, c1 - c0, a.codes[0] + c0 * a.L, a.thetas[0] + c0 * a.L,
                                      reinterpret_cast<const double*>(a.target), a.fitness + c0, nullptr,
                                      &a.st->stop, s, nullptr, a.codes[1] + c0 * a.L, a.thetas[1] + c0 * a.L,
                                      &a.st->generation);
      set_error("numberOfWires outside the supported range 2..13");
      return ISQ_ERR_UNSUPPORTED;
  }
}

// Single-block path: one fitness round (P <= 8 warps) and few genes; larger
// launch-bound populations (C2, P = 50) run faster as a CUDA graph of the
// multi-kernel generation, whose fitness kernel spreads the circuits over SMs.
// Launch-bound populations beyond one block's fitness round (C2: 50
// genomes): n generations in one cooperative launch of up to one block per
// SM, the phases separated by grid-wide barriers — fitness (all blocks),
// reductions + SUS (block 0), breeding (all blocks), advance (block 0).
// Single-barrier generation of the cooperative launch (one round, P <= kGaRed,
// one rank): after the fitness barrier EVERY block reduces the generation's
// fitness and runs the SUS itself — identical inputs and arithmetic, so
// identical picks — keeps its own copy of the engine state (generation, best,
// stop) and breeds its own warps' children from its shared-memory parents.
// Block 0 alone writes the device state, the record and the best genome.
// `fit` is this generation's fitness buffer (generations alternate between
// two, so a block that runs ahead into the next scoring never overwrites
// values another block is still reading).  Returns the stop reason.
template <class Idle>
__device__ __forceinline__ int ga_select_local(const GaArgs& a, uint64_t g, int cur, const double* fit,
                                               uint64_t rec_base, double& best, double* smax, double* ssum,
                                               int64_t* sarg, int32_t* spar, int64_t* s_elite, Idle idle) {
  __shared__ double sfit[kGaRed];
  __shared__ int s_search, s_stop, s_improved;
  // the SUS stream's first block depends only on (seed, g): thread 0 computes
  // it now, under the reduction's barriers, not on the walk's critical path
  NpStream rs;
  if (threadIdx.x == 0) {
    rs.init(a.seed, DOM_GA_SUS, g, 0, 0);
    rs.prime();
  }
  // generation best / first argmax / sum (ga_reduce_partial_body + the combine of ga_reduce_sus_body)
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  {
    double lm = -1.0, ls = 0.0;
    int64_t la = INT64_MAX;
    for (int64_t i = threadIdx.x; i < a.P; i += kGaRed) {
      const double f = fit[i];
      sfit[i] = f;
      ls += f;
      if (f > lm) {
        lm = f;
        la = i;
      }
    }
    smax[threadIdx.x] = lm;
    ssum[threadIdx.x] = ls;
    sarg[threadIdx.x] = la;
    __syncthreads();
    for (int off = kGaRed / 2; off >= 1; off >>= 1) {
      if (threadIdx.x < off) {
        const double m2 = smax[threadIdx.x + off];
        const int64_t a2 = sarg[threadIdx.x + off];
        if (m2 > smax[threadIdx.x] || (m2 == smax[threadIdx.x] && a2 < sarg[threadIdx.x])) {
          smax[threadIdx.x] = m2;
          sarg[threadIdx.x] = a2;
        }
        ssum[threadIdx.x] += ssum[threadIdx.x + off];
      }
      __syncthreads();
    }
    m = smax[0];
    arg = sarg[0];
    sum = 0.0 + ssum[0];
  }
  __syncthreads();  // ssum is reused for the pointers below
  if (threadIdx.x == 0) {
    const int improved = m > best;
    if (improved) best = m;
    const uint64_t gn = g + 1;
    const int stop = best >= a.target_fitness ? 1 : (gn >= a.max_generations ? 2 : 0);
    if (blockIdx.x == 0) {
      GaDevState* st = a.st;
      st->best_fitness = best;
      st->elite = arg;
      st->improved = improved;
      GenRecord r;
      r.gen_best = m;
      r.gen_mean = sum / (double)a.P;
      r.best_fitness = best;
      r.pad = 0.0;
      const uint64_t ri = g - rec_base;
      if (ri < (uint64_t)a.rec_cap) a.records[ri] = r;
      st->generation = gn;
      st->stop = stop;
    }
    *s_elite = arg;
    s_improved = improved;
    s_stop = stop;
    // sus_select (ga.py:95-116), the parallel-search form of ga_reduce_sus_body
    const double total = np_pairwise_sum(sfit, a.P);
    int search = 0;
    if (total <= 0.0) {
      for (int64_t k = 0; k < a.P; ++k) {
        spar[k] = (int32_t)rs.integers(a.P);
        if (blockIdx.x == 0) a.parents[k] = spar[k];  // isq_ga_parents
      }
    } else {
      const double spacing = __ddiv_rn(total, (double)a.P);
      double pointer = rs.uniform(0.0, spacing);
      double cumulative = 0.0;
      int k = 0;
      for (; k + 8 <= (int)a.P; k += 8) {  // the loads ahead of the two dependent chains
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = sfit[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          cumulative = __dadd_rn(cumulative, v[u]);
          sfit[k + u] = cumulative;  // C[k + 1]
          ssum[k + u] = pointer;
          pointer = __dadd_rn(pointer, spacing);
        }
      }
      for (; k < (int)a.P; ++k) {
        cumulative = __dadd_rn(cumulative, sfit[k]);
        sfit[k] = cumulative;
        ssum[k] = pointer;
        pointer = __dadd_rn(pointer, spacing);
      }
      search = 1;
    }
    s_search = search;
  } else {
    idle();
  }
  __syncthreads();
  if (s_search) {
    for (int k = threadIdx.x; k < (int)a.P; k += kGaRed) {
      const double pk = ssum[k];
      int lo = 0, hi = (int)a.P - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sfit[mid] <= pk)
          lo = mid + 1;
        else
          hi = mid;
      }
      spar[k] = lo;
      if (blockIdx.x == 0) a.parents[k] = lo;  // isq_ga_parents
    }
  }
  if (blockIdx.x == 0 && s_improved && threadIdx.x < 32) {
    for (int j = threadIdx.x; j < a.L; j += 32) {
      a.best_codes[j] = a.codes[cur][*s_elite * a.L + j];
      a.best_thetas[j] = a.thetas[cur][*s_elite * a.L + j];
    }
  }
  __syncthreads();
  return s_stop;
}

template <int NQ>
__global__ void __launch_bounds__(kGaRed, 1) ga_coop_kernel(GaArgs a, int n_gens, int local_select) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using G = Geo<NQ>;
  constexpr int kWarps = kGaRed / 32;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ FitScratch<NQ, double, kSmallNR> sh[kWarps];
  __shared__ double smax[kGaRed], ssum[kGaRed];
  __shared__ int64_t sarg[kGaRed];
  __shared__ int s_improved;
  __shared__ int64_t s_elite;
  for (int i = threadIdx.x; i < G::D * G::D; i += kGaRed) Ts[i] = a.target[i];
  __syncthreads();
  const int64_t genes = a.P * a.L;
  // One round (P <= circuits of one pass of the grid, always true at the
  // sizes this launch is chosen for): warp w scores circuits [w CPW, (w+1) CPW)
  // (fitness_rows_fast: CPW = 1 at n = 5, 32 / 2^n below) and breeds the same
  // children, so what it scores next is its own writes and breeding needs no
  // grid barrier after it.  Otherwise genes are bred grid-stride behind a
  // third barrier.
  const int CPW = small_cpw<NQ>(a.P, (int64_t)gridDim.x * kWarps);  // uniform over the grid
  const bool one_round = a.P <= (int64_t)gridDim.x * kWarps * CPW;
  const int lane = threadIdx.x & 31;
  const int64_t wc = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);  // this warp's batch
  const int64_t wt0 = wc * CPW * a.L;          // first gene of the warp's children
  const int wgenes = CPW * a.L;                // genes of the warp's children
  auto wgene = [&](int u) -> int64_t {         // u-th gene of the warp's children (or `genes`)
    const int64_t t = wt0 + u;
    return u < wgenes && t < genes ? t : genes;
  };
  if (local_select && one_round && a.P <= kGaRed) {
    __shared__ int32_t spar[kGaRed];
    uint64_t g = a.st->generation;
    const uint64_t rec_base = a.st->rec_base;
    double best = a.st->best_fitness;
    if (a.st->stop) return;
    // gene u of the warp's children on lane 31 - u (mod 32): lane 0 (thread 0
    // of the block runs the SUS chains) has no gene when they hold < 32
    const int jl = 31 - lane;
    for (int it = 0; it < n_gens; ++it) {
      const int cur = (int)(g & 1);
      double* fit = (g & 1) ? a.fitness_alt : a.fitness;
      fitness_rows_fast<NQ, double, kSmallNR, true>(a.P, a.L, a.codes[cur], a.thetas[cur], Ts, sh, fit, kWarps,
                                              nullptr, nullptr, CPW);
      grid.sync();
      const int64_t t0 = wgene(jl);
      GeneDraw d0;
      const int stop = ga_select_local(a, g, cur, fit, rec_base, best, smax, ssum, sarg, spar, &s_elite, [&] {
        if (t0 < genes) d0 = ga_breed_draw(a, t0, g);
      });
      if (threadIdx.x == 0 && t0 < genes) d0 = ga_breed_draw(a, t0, g);
      const int64_t elite = s_elite;
      if (t0 < genes) ga_breed_apply(a, t0, cur, elite, d0, spar);
      for (int u = jl + 32; u < wgenes; u += 32) {
        const int64_t t = wgene(u);
        if (t < genes) ga_breed_apply(a, t, cur, elite, ga_breed_draw(a, t, g), spar);
      }
      __threadfence_block();  // the warp's children, read back by its own next scoring
      __syncwarp();
      ++g;
      if (stop) break;
    }
    // the last scored generation's fitness belongs in a.fitness (isq_ga_fitness)
    if ((g - 1) & 1) {
      for (int i = lane; i < CPW; i += 32)
        if (wc * CPW + i < a.P) a.fitness[wc * CPW + i] = a.fitness_alt[wc * CPW + i];
    }
    return;
  }
  for (int it = 0; it < n_gens; ++it) {
    if (a.st->stop) return;  // uniform across the grid: written before the last grid barrier
    const uint64_t g = a.st->generation;
    const int cur = ga_cur(a);
    fitness_rows_fast<NQ, double, kSmallNR, true>(a.P, a.L, a.codes[cur], a.thetas[cur], Ts, sh, a.fitness, kWarps,
                                            nullptr, nullptr, CPW);
    grid.sync();
    // this thread's first gene: its draws while block 0 reduces and selects
    const int64_t t0 = one_round ? wgene(lane) : (int64_t)blockIdx.x * kGaRed + threadIdx.x;
    GeneDraw d0;
    if (blockIdx.x != 0 && t0 < genes) d0 = ga_breed_draw(a, t0, g);
    if (blockIdx.x == 0) {
      for (int part = 0; part < a.n_parts; ++part) {
        ga_reduce_partial_body(a, part, smax, ssum, sarg);
        __syncthreads();
      }
      ga_reduce_sus_body(
          a, &s_improved, &s_elite,
          [&] {
            if (t0 < genes) d0 = ga_breed_draw(a, t0, g);
          },
          ssum, kGaRed);
      if (threadIdx.x == 0) {
        if (t0 < genes) d0 = ga_breed_draw(a, t0, g);
        // advance here (breeding reads g and cur from registers): the stop
        // check at the top of the next iteration sees it after the barrier
        // that ends breeding
        ga_advance_body(a);
      }
    }
    grid.sync();
    const int64_t elite = a.st->elite;
    if (one_round) {
      if (t0 < genes) ga_breed_apply(a, t0, cur, elite, d0);
      for (int u = lane + 32; u < wgenes; u += 32) {
        const int64_t t = wgene(u);
        if (t < genes) ga_breed_gene(a, t, g, cur, elite);
      }
      __threadfence_block();  // the warp's children, read back by its own next scoring
      __syncwarp();
    } else {
      if (t0 < genes) ga_breed_apply(a, t0, cur, elite, d0);
      for (int64_t t = t0 + (int64_t)gridDim.x * kGaRed; t < genes; t += (int64_t)gridDim.x * kGaRed)
        ga_breed_gene(a, t, g, cur, elite);
      grid.sync();
    }
  }
}

#ifndef ISQ_GA_LOCAL_SELECT
#define ISQ_GA_LOCAL_SELECT 1
#endif
template <int NQ>
static isq_status ga_launch_coop_nq(const GaArgs& a, int n_gens, cudaStream_t s) {
  int per_sm = 0;
  ISQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ga_coop_kernel<NQ>, kGaRed, 0));
  constexpr int64_t per_block = kGaRed / 32;  // one circuit per warp if the grid allows (small_cpw)
  const int64_t want = (a.P + per_block - 1) / per_block;
  int64_t grid = (int64_t)num_sms() * (per_sm > 0 ? 1 : 0);
  if (grid > want) grid = want;
  if (grid < 1) {
    set_error("cooperative GA kernel does not fit on an SM");
    return ISQ_ERR_CUDA;
  }
  GaArgs args = a;
  int local_select = ISQ_GA_LOCAL_SELECT;
  void* params[] = {(void*)&args, (void*)&n_gens, (void*)&local_select};
  ISQ_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)ga_coop_kernel<NQ>, dim3((unsigned)grid), dim3(kGaRed),
                                           params, 0, s));
  return ISQ_OK;
}

static isq_status ga_launch_coop(const GaArgs& a, int n_gens, cudaStream_t s) {
  switch (a.n) {
    case 2: return ga_launch_coop_nq<2>(a, n_gens, s);
    case 3: return ga_launch_coop_nq<3>(a, n_gens, s);
    case 4: return ga_launch_coop_nq<4>(a, n_gens, s);
    case 5: return ga_launch_coop_nq<5>(a, n_gens, s);
    default:
      set_error("numberOfWires outside the supported range 2..13");
      return ISQ_ERR_UNSUPPORTED;
  }
}

constexpr int64_t kGaSmallGenes = 1 << 12;
constexpr int64_t kGaSmallPop = kGaRed / 32;

static isq_status ga_launch_small(const GaArgs& a, int n_gens, cudaStream_t s) {
  switch (a.n) {
    case 2: ga_small_kernel<2><<<1, kGaRed, 0, s>>>(a, n_gens); break;
    case 3: ga_small_kernel<3><<<1, kGaRed, 0, s>>>(a, n_gens); break;
    case 4: ga_small_kernel<4><<<1, kGaRed, 0, s>>>(a, n_gens); break;
    case 5: ga_small_kernel<5><<<1, kGaRed, 0, s>>>(a, n_gens); break;
    default:
      set_error("numberOfWires outside the supported range 2..13");
      return ISQ_ERR_UNSUPPORTED;
  }
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

// Small populations: reductions, SUS, breeding and advance of one generation
// in a single block (same device bodies as the four-kernel finish).
constexpr int64_t kGaTailGenes = 1 << 14;

__global__ void __launch_bounds__(kGaRed) ga_tail_kernel(GaArgs a) {
  __shared__ double smax[kGaRed], ssum[kGaRed];
  __shared__ int64_t sarg[kGaRed];
  __shared__ int s_improved;
  __shared__ int64_t s_elite;
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int cur = ga_cur(a);
  for (int part = 0; part < a.n_parts; ++part) {
    ga_reduce_partial_body(a, part, smax, ssum, sarg);
    __syncthreads();
  }
  ga_reduce_sus_body(a, &s_improved, &s_elite, NoIdleWork(), ssum, kGaRed);
  __syncthreads();
  const int64_t elite = a.st->elite;
  for (int64_t t = threadIdx.x; t < a.P * a.L; t += kGaRed) ga_breed_gene(a, t, g, cur, elite);
  __syncthreads();
  if (threadIdx.x == 0) ga_advance_body(a);
}

static isq_status ga_launch_finish(const GaArgs& a, cudaStream_t s) {
  if (a.P * a.L <= kGaTailGenes) {
    ga_tail_kernel<<<1, kGaRed, 0, s>>>(a);
    ISQ_CUDA_TRY(cudaGetLastError());
    return ISQ_OK;
  }
  ga_reduce_partials<<<a.n_parts, kGaRed, 0, s>>>(a);
  if (a.P > kSusCache) {
    if (a.sus_grid != nullptr) {  // the running sums and numpy's total over the whole GPU (sus.cuh)
      ISQ_CUDA_TRY(launch_pairwise_parts(a.fitness, a.P, a.sus_grid, a.P - 1, s));
      ISQ_CUDA_TRY(launch_exact_chain_grid(a.fitness, a.P - 1, 0.0, a.sus_C, a.sus_grid, s));
    }
    ga_reduce_sus_large_kernel<<<2, kSusThreads, kChainSmem, s>>>(a);
    sus_search_kernel<int32_t><<<ga_blocks(a.P), 256, 0, s>>>(a.sus_C, a.P - 1, a.sus_P, a.P, a.parents,
                                                              a.sus_flag, &a.st->stop);
  } else {
    ga_reduce_sus_kernel<<<1, kGaRed, 0, s>>>(a);
  }
  ga_breed_kernel<<<ga_blocks(a.P * a.L), kBreedThreads, 0, s>>>(a);
  ga_advance_kernel<<<1, 1, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

}  // namespace isq

using namespace isq;

#define GA_TRY(expr)                                                 \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) {                                         \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      ga_free(h);                                                    \
      return ISQ_ERR_CUDA;                                           \
    }                                                                \
  } while (0)

static isq_status ga_null_handle() {
  set_error("null engine handle");
  return ISQ_ERR_CONFIG;
}

extern "C" {

isq_status isq_ga_create(const isq_ga_config* cfg, const double* target, int32_t device,
                         int32_t max_batch, void** out) {
  *out = nullptr;
  auto bad = [](const std::string& m, isq_status code = ISQ_ERR_CONFIG) {
    set_error(m);
    return code;
  };
  if (cfg->number_of_wires < 2) return bad("numberOfWires must be ≥ 2");
  if (cfg->size_of_individual < 1) return bad("sizeOfIndividual must be ≥ 1");
  if (cfg->population < 2) return bad("GA population must be ≥ 2");
  if (!(cfg->mutation_rate >= 0.0 && cfg->mutation_rate <= 1.0))
    return bad("mutation rate must be in [0, 1]");
  if (!(cfg->structural_rate >= 0.0 && cfg->structural_rate <= 1.0))
    return bad("structural rate must be in [0, 1]");
  if (!(cfg->target_fitness > 0.0 && cfg->target_fitness <= 1.0))
    return bad("targetFitness must be in (0, 1]");
  if (cfg->max_generations < 1) return bad("maxGenerations must be ≥ 1");
  if (cfg->number_of_wires > ISQ_MAX_WIRES)
    return bad("numberOfWires exceeds the device kernels (2..13 wires, the reference's default 4^n <= 2^26 cap)",
               ISQ_ERR_UNSUPPORTED);
  if (cfg->population >= (1LL << 31)) return bad("population must be < 2^31", ISQ_ERR_UNSUPPORTED);
  if ((int64_t)cfg->population * cfg->size_of_individual >= (1LL << 32))
    return bad("population * sizeOfIndividual must be < 2^32", ISQ_ERR_UNSUPPORTED);
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return bad("invalid rank/world");
  if (cfg->precision != ISQ_PRECISION_FP64 && cfg->precision != ISQ_PRECISION_FP32)
    return bad("precision must be ISQ_PRECISION_FP64 or ISQ_PRECISION_FP32");
  GaHandle* h = new GaHandle();
  h->device = device;
  h->rank = cfg->rank;
  h->world = cfg->world;
  h->max_batch = max_batch < 1 ? 1 : max_batch;
  GaArgs& a = h->a;
  std::memset(&a, 0, sizeof(a));
  a.n = cfg->number_of_wires;
  a.L = cfg->size_of_individual;
  a.P = cfg->population;
  a.div_L.init((uint32_t)a.L);
  a.div_P.init((uint32_t)a.P);
  a.ncodes = 3 * a.n + a.n * (a.n - 1) / 2;
  a.rate = cfg->mutation_rate;
  a.mrange = cfg->mutation_range;
  a.structural = cfg->structural_rate;
  a.target_fitness = cfg->target_fitness;
  a.max_generations = (uint64_t)cfg->max_generations;
  a.seed = cfg->seed;
  a.precision = cfg->precision;
  a.rec_cap = h->max_batch;
  h->shard = (a.P + h->world - 1) / h->world;
  const int64_t D = 1LL << a.n;
  GA_TRY(cudaSetDevice(device));
  GA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  for (int b = 0; b < 2; ++b) {
    GA_TRY(cudaMalloc((void**)&a.codes[b], a.P * a.L));
    GA_TRY(cudaMalloc((void**)&a.thetas[b], a.P * a.L * 8));
  }
  GA_TRY(cudaMalloc((void**)&a.fitness, h->shard * h->world * 8));
  GA_TRY(cudaMalloc((void**)&a.fitness_alt, h->shard * h->world * 8));
  GA_TRY(cudaMalloc((void**)&a.parents, a.P * 4));
  GA_TRY(cudaMalloc((void**)&a.st, sizeof(GaDevState)));
  GA_TRY(cudaMalloc((void**)&a.records, sizeof(GenRecord) * h->max_batch));
  GA_TRY(cudaMalloc((void**)&a.best_codes, a.L));
  GA_TRY(cudaMalloc((void**)&a.best_thetas, a.L * 8));
  GA_TRY(cudaMalloc((void**)&a.target, D * D * 16));
  a.n_parts = (int)((a.P + 4095) / 4096);
  if (a.n_parts > 1024) a.n_parts = 1024;
  if (a.n_parts < 1) a.n_parts = 1;
  GA_TRY(cudaMalloc((void**)&a.part_max, a.n_parts * 8));
  GA_TRY(cudaMalloc((void**)&a.part_sum, a.n_parts * 8));
  GA_TRY(cudaMalloc((void**)&a.part_arg, a.n_parts * 8));
  if (a.P > kSusCache) {
    GA_TRY(cudaFuncSetAttribute((const void*)ga_reduce_sus_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kChainSmem));
    GA_TRY(cudaMalloc((void**)&a.sus_C, a.P * 8));
    GA_TRY(cudaMalloc((void**)&a.sus_P, a.P * 8));
    GA_TRY(cudaMalloc((void**)&a.sus_flag, sizeof(int)));
    if (chain_grid_worth(a.P - 1)) {  // the running sums over the whole GPU (sus.cuh)
      GA_TRY(prepare_exact_chain_grid());
      GA_TRY(cudaMalloc(&a.sus_grid, chain_grid_scratch_bytes(a.P - 1)));
    }
  }
  GA_TRY(cudaMemcpy((void*)a.target, target, D * D * 16, cudaMemcpyHostToDevice));
  GaDevState s0;
  std::memset(&s0, 0, sizeof(s0));
  GA_TRY(cudaMemcpy(a.st, &s0, sizeof(s0), cudaMemcpyHostToDevice));
  GA_TRY(cudaMemset(a.best_codes, 0, a.L));
  GA_TRY(cudaMemset(a.best_thetas, 0, a.L * 8));
  GA_TRY(cudaMemset(a.fitness, 0, h->shard * h->world * 8));
  ga_init_kernel<<<ga_blocks(a.P * a.L), 256, 0, h->stream>>>(a);
  GA_TRY(cudaGetLastError());
  GA_TRY(cudaStreamSynchronize(h->stream));
  *out = h;
  return ISQ_OK;
}

isq_status isq_ga_destroy(void* handle) {
  ga_free(static_cast<GaHandle*>(handle));
  return ISQ_OK;
}

isq_status isq_ga_set_stream(void* handle, void* stream) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (h->own_stream) cudaStreamDestroy(h->stream);
  h->own_stream = false;
  h->stream = (cudaStream_t)stream;
  return ISQ_OK;
}

isq_status isq_ga_begin_batch(void* handle) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaMemcpyAsync(&h->a.st->rec_base, &h->a.st->generation, 8,
                               cudaMemcpyDeviceToDevice, h->stream));
  return ISQ_OK;
}

isq_status isq_ga_eval(void* handle) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  const int64_t c0 = h->rank * h->shard;
  const int64_t c1 = c0 + h->shard < h->a.P ? c0 + h->shard : h->a.P;
  return ga_launch_eval(h->a, c0, c1, h->stream);
}

isq_status isq_ga_finish(void* handle) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return ga_launch_finish(h->a, h->stream);
}

isq_status isq_ga_read_batch(void* handle, isq_generation_record* records, int32_t* n_done,
                             int32_t* stop_reason, uint64_t* generation, double* best_fitness) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  GaDevState s;
  ISQ_CUDA_TRY(cudaMemcpy(&s, h->a.st, sizeof(s), cudaMemcpyDeviceToHost));
  int64_t done = (int64_t)(s.generation - s.rec_base);
  if (done > h->max_batch) done = h->max_batch;
  if (done > 0 && records)
    ISQ_CUDA_TRY(cudaMemcpy(records, h->a.records, sizeof(GenRecord) * done, cudaMemcpyDeviceToHost));
  if (n_done) *n_done = (int32_t)done;
  if (stop_reason) *stop_reason = s.stop;
  if (generation) *generation = s.generation;
  if (best_fitness) *best_fitness = s.best_fitness;
  return ISQ_OK;
}

isq_status isq_ga_step(void* handle, int32_t n, isq_generation_record* records, int32_t* n_done,
                       int32_t* stop_reason) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  if (h->world != 1) {
    set_error("isq_ga_step drives a single rank; use eval / all-gather / finish for world > 1");
    return ISQ_ERR_CONFIG;
  }
  if (n > h->max_batch) {
    set_error("n exceeds the handle's record capacity (max_batch)");
    return ISQ_ERR_CONFIG;
  }
  isq_status st = isq_ga_begin_batch(handle);
  if (st != ISQ_OK) return st;
  const GaArgs& a = h->a;
  const int mode = h->launch_mode;
  if (mode == ISQ_LAUNCH_FUSED && a.precision != ISQ_PRECISION_FP64) {
    set_error("the fused single-block generation is fp64 only");
    return ISQ_ERR_CONFIG;
  }
  const bool fp64 = a.precision == ISQ_PRECISION_FP64;
  if (mode == ISQ_LAUNCH_FUSED && a.n > ISQ_MAX_FAST_WIRES) {
    set_error("the fused GA launch supports numberOfWires <= 5");
    return ISQ_ERR_CONFIG;
  }
  if (mode == ISQ_LAUNCH_FUSED ||
      (mode == ISQ_LAUNCH_AUTO && fp64 && a.n <= ISQ_MAX_FAST_WIRES && a.P * a.L <= kGaTailGenes)) {
    // one launch for n generations: one block when the population is one
    // fitness round, a cooperative grid otherwise
    const bool one_block = a.P <= kGaSmallPop && a.P * a.L <= kGaSmallGenes;
    st = n <= 0 ? ISQ_OK : one_block ? ga_launch_small(a, n, h->stream) : ga_launch_coop(a, n, h->stream);
    if (st != ISQ_OK) return st;
    return isq_ga_read_batch(handle, records, n_done, stop_reason, nullptr, nullptr);
  }
  // n > 5 runs the generic fitness kernel, whose scratch is allocated on
  // first use: plain launches only (a capture would record the allocation)
  const int per_graph = (mode == ISQ_LAUNCH_KERNELS || a.n > ISQ_MAX_FAST_WIRES) ? 0
                        : mode == ISQ_LAUNCH_GRAPH                              ? 16
                                                                                : graph_generations(a.P * a.L);
  st = run_generations(h->graph, h->stream, n, per_graph, [&a](cudaStream_t s) {
    isq_status r = ga_launch_eval(a, 0, a.P, s);
    return r != ISQ_OK ? r : ga_launch_finish(a, s);
  });
  if (st != ISQ_OK) return st;
  return isq_ga_read_batch(handle, records, n_done, stop_reason, nullptr, nullptr);
}

isq_status isq_ga_set_launch_mode(void* handle, int32_t mode) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  if (mode < ISQ_LAUNCH_AUTO || mode > ISQ_LAUNCH_FUSED) {
    set_error("unknown launch mode");
    return ISQ_ERR_CONFIG;
  }
  h->launch_mode = mode;
  return ISQ_OK;
}

isq_status isq_ga_buffers(void* handle, void** fitness_dev, int64_t* shard_len, void** stream) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  if (fitness_dev) *fitness_dev = h->a.fitness;
  if (shard_len) *shard_len = h->shard;
  if (stream) *stream = h->stream;
  return ISQ_OK;
}

isq_status isq_ga_best(void* handle, uint8_t* codes, double* thetas, double* fitness) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  ISQ_CUDA_TRY(cudaMemcpy(codes, h->a.best_codes, h->a.L, cudaMemcpyDeviceToHost));
  ISQ_CUDA_TRY(cudaMemcpy(thetas, h->a.best_thetas, h->a.L * 8, cudaMemcpyDeviceToHost));
  GaDevState s;
  ISQ_CUDA_TRY(cudaMemcpy(&s, h->a.st, sizeof(s), cudaMemcpyDeviceToHost));
  *fitness = s.best_fitness;
  return ISQ_OK;
}

isq_status isq_ga_get_state(void* handle, uint8_t* codes, double* thetas, uint64_t* generation,
                            double* best_fitness, int32_t* stop) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  const GaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  GaDevState s;
  ISQ_CUDA_TRY(cudaMemcpy(&s, a.st, sizeof(s), cudaMemcpyDeviceToHost));
  const int cur = (int)(s.generation & 1);
  if (codes) ISQ_CUDA_TRY(cudaMemcpy(codes, a.codes[cur], a.P * a.L, cudaMemcpyDeviceToHost));
  if (thetas) ISQ_CUDA_TRY(cudaMemcpy(thetas, a.thetas[cur], a.P * a.L * 8, cudaMemcpyDeviceToHost));
  if (generation) *generation = s.generation;
  if (best_fitness) *best_fitness = s.best_fitness;
  if (stop) *stop = s.stop;
  return ISQ_OK;
}

isq_status isq_ga_set_state(void* handle, const uint8_t* codes, const double* thetas,
                            uint64_t generation, double best_fitness, int32_t stop,
                            const uint8_t* best_codes, const double* best_thetas) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  const GaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int64_t i = 0; codes && i < a.P * a.L; ++i)
    if (codes[i] >= a.ncodes) {
      set_error("gate code out of range for numberOfWires");
      return ISQ_ERR_CONFIG;
    }
  const int cur = (int)(generation & 1);
  if (codes) ISQ_CUDA_TRY(cudaMemcpy(a.codes[cur], codes, a.P * a.L, cudaMemcpyHostToDevice));
  if (thetas) ISQ_CUDA_TRY(cudaMemcpy(a.thetas[cur], thetas, a.P * a.L * 8, cudaMemcpyHostToDevice));
  if (best_codes) ISQ_CUDA_TRY(cudaMemcpy(a.best_codes, best_codes, a.L, cudaMemcpyHostToDevice));
  if (best_thetas)
    ISQ_CUDA_TRY(cudaMemcpy(a.best_thetas, best_thetas, a.L * 8, cudaMemcpyHostToDevice));
  GaDevState s;
  std::memset(&s, 0, sizeof(s));
  s.generation = generation;
  s.rec_base = generation;
  s.best_fitness = best_fitness;
  s.stop = stop;
  ISQ_CUDA_TRY(cudaMemcpy(a.st, &s, sizeof(s), cudaMemcpyHostToDevice));
  return ISQ_OK;
}

isq_status isq_ga_set_limits(void* handle, int64_t max_generations, double target_fitness,
                             int32_t stop) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  if (max_generations < 1) {
    set_error("maxGenerations must be ≥ 1");
    return ISQ_ERR_CONFIG;
  }
  if (!(target_fitness > 0.0 && target_fitness <= 1.0)) {
    set_error("targetFitness must be in (0, 1]");
    return ISQ_ERR_CONFIG;
  }
  if (stop < 0 || stop > 2) {
    set_error("stop must be 0 (running), 1 (target-reached) or 2 (generation-limit)");
    return ISQ_ERR_CONFIG;
  }
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->a.max_generations = (uint64_t)max_generations;
  h->a.target_fitness = target_fitness;
  h->graph.reset();
  ISQ_CUDA_TRY(cudaMemcpy(&h->a.st->stop, &stop, sizeof(stop), cudaMemcpyHostToDevice));
  return ISQ_OK;
}

isq_status isq_ga_fitness(void* handle, double* out) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  ISQ_CUDA_TRY(cudaMemcpy(out, h->a.fitness, h->a.P * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_ga_parents(void* handle, int32_t* out) {
  GaHandle* h = static_cast<GaHandle*>(handle);
  if (!h) return ga_null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  ISQ_CUDA_TRY(cudaMemcpy(out, h->a.parents, h->a.P * 4, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

}  // extern "C"

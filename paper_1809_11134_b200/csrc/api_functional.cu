// The reference's functional API (engine.py:105-263, ga.py:62-138) on the
// device, with the per-unit counter streams of the engines in place of the
// reference's sequential numpy Generators (csrc/np_random.cuh; DESIGN.md
// §5.1): a call names the stream position (seed, generation, index) and
// computes exactly what the engine computes for that unit, so these entry
// points are the engine's own operators, callable one at a time.
//
//   init_population      per-slot stream (seed, DOM_INIT, 0, slot)
//   construct_segments   per-slot stream (seed, DOM_MEASURE, gen, slot)
//   sample_circuit       per-circuit stream (seed, DOM_SAMPLE, gen, circuit)
//   mutate_population    per-slot stream (seed, DOM_MUTATE, gen, slot)
//   SegmentFitnessTable  device hash of the (flat, position) entries + slot_max
//   random_genome        per-gene stream (seed, DOM_GA_INIT, 0, genome, gene)
//   sus_select           stream (seed, DOM_GA_SUS, gen)
//   two_point_crossover  stream (seed, DOM_GA_PAIR, gen, pair)
//   ga_mutate            per-gene stream (seed, DOM_GA_MUT, gen, child, gene)
#include <cstring>
#include <string>
#include <vector>

#include "engine_common.cuh"
#include "isq_internal.h"
#include "sus.cuh"

namespace isq {

namespace {

isq_status bad_config(const std::string& m) {
  set_error(m);
  return ISQ_ERR_CONFIG;
}

isq_status check_layout(int n, int L, int64_t P) {
  if (n < ISQ_MIN_WIRES || n > ISQ_MAX_WIRES) {
    set_error("numberOfWires=" + std::to_string(n) + " is outside the supported range 2..13");
    return ISQ_ERR_UNSUPPORTED;
  }
  if (L < 1 || P < 1) return bad_config("sizeOfIndividual and sizeOfPopulation must be ≥ 1");
  const int64_t K = n + (int64_t)n * (n - 1) / 2;
  if (K * P * L >= (1LL << 32) - 1) {
    set_error("qubit_count = K*P*L must stay below 2^32 for the device engine");
    return ISQ_ERR_UNSUPPORTED;
  }
  return ISQ_OK;
}

// A one-rank QeqeaArgs carrying only the layout and stream parameters the
// per-slot / per-circuit device functions read.
QeqeaArgs functional_args(int n, int L, int64_t P, uint64_t seed) {
  QeqeaArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = n;
  a.L = L;
  a.P = P;
  a.K = n + (int64_t)n * (n - 1) / 2;
  a.Q = a.K * P * L;
  a.Qt = (int64_t)n * P * L;
  a.seed = seed;
  a.world = 1;
  a.S = P;
  a.Lr = L;
  a.p_bounds[1] = L;
  a.div_L.init((uint32_t)L);
  a.div_LP.init((uint32_t)(L * P));
  a.div_Lr.init((uint32_t)L);
  a.div_S.init((uint32_t)P);
  a.Qloc = a.Q;
  a.Qtloc = a.Qt;
  return a;
}

int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}

// RAII device buffer.
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes < 16 ? 16 : bytes); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

#define TRYF(expr)                                                          \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));        \
      return ISQ_ERR_CUDA;                                                  \
    }                                                                       \
  } while (0)

}  // namespace

// ------------------------------------------------------------------ QEQEA ---

__global__ void fn_init_population_kernel(QeqeaArgs a, double* theta, double2* q) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q; s += (int64_t)gridDim.x * blockDim.x) {
    double t;
    double2 qq[3];
    init_slot_value(a.seed, s, s < a.Qt, t, qq);
    theta[s] = t;
    if (s < a.Qt) {
#pragma unroll
      for (int k = 0; k < 3; ++k) q[3 * s + k] = qq[k];
    }
  }
}

__global__ void fn_construct_segments_kernel(QeqeaArgs a, uint64_t g, const double2* q, int8_t* axes) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Qt; s += (int64_t)gridDim.x * blockDim.x) {
    double re[3] = {q[3 * s].x, q[3 * s + 1].x, q[3 * s + 2].x};
    double im[3] = {q[3 * s].y, q[3 * s + 1].y, q[3 * s + 2].y};
    NpStream st;
    st.init(a.seed, DOM_MEASURE, g, (uint64_t)s, 0);
    bool ok = true;
    axes[s] = (int8_t)measure_axis(re, im, a.n_meas, st, &ok);
  }
}

__global__ void __launch_bounds__(128) fn_sample_kernel(QeqeaArgs a, uint64_t g, int64_t c0, int64_t count,
                                                        uint32_t* flats) {
  __shared__ uint64_t blk[4][36];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * 4 + wib; c < count; c += (int64_t)gridDim.x * 4)
    sample_circuit_warp(a, g, c0 + c, flats + c * a.L, blk[wib], lane);
}

__global__ void fn_widen_kernel(const uint32_t* in, int64_t* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void fn_mutate_population_kernel(QeqeaArgs a, uint64_t g, double* theta, double2* q,
                                            const double* slot_max, uint8_t* mutated) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q; s += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    v.theta = theta[s];
    const bool has_q = s < a.Qt;
    if (has_q) {
#pragma unroll
      for (int k = 0; k < 3; ++k) v.q[k] = q[3 * s + k];
    }
    bool qpath = false;
    const bool m = mutate_slot(a, s, g, slot_max[s], v, &qpath);
    mutated[s] = m ? (qpath ? 2 : 1) : 0;
    if (m) {
      theta[s] = v.theta;
      if (qpath) {
#pragma unroll
        for (int k = 0; k < 3; ++k) q[3 * s + k] = v.q[k];
      }
    }
  }
}

// ------------------------------------------------- SegmentFitnessTable ---
// entries: open-addressing hash of key = flat * L + position + 1 (0 = empty)
// -> fitness bits (u64 atomicMax: fitness >= 0); slot_max: u64 atomicMax.
struct TableHandle {
  int64_t Q = 0;
  int L = 0;
  int device = 0;
  int64_t cap = 0;
  unsigned long long* keys = nullptr;
  unsigned long long* vals = nullptr;
  unsigned long long* count = nullptr;  // occupied entries
  double* smax = nullptr;
};

__device__ __forceinline__ uint64_t table_hash(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ int64_t table_slot(unsigned long long* keys, unsigned long long* count, int64_t cap,
                                              unsigned long long key) {
  int64_t h = (int64_t)(table_hash(key) & (uint64_t)(cap - 1));
  while (true) {
    const unsigned long long k = atomicCAS(&keys[h], 0ULL, key);
    if (k == 0ULL) {
      atomicAdd(count, 1ULL);
      return h;
    }
    if (k == key) return h;
    h = (h + 1) & (cap - 1);
  }
}

// SegmentFitnessTable.update (engine.py:211-222) for a batch of blueprints in
// order: touch (circuit c, position p) improves iff its fitness beats the
// running entry; the union of improved slots is order-independent (a slot is
// in it iff the batch's best touch of one of its keys beats the entry).
__global__ void fn_table_update_kernel(TableHandle t, int64_t touches, const int64_t* flats, const double* fits,
                                       uint8_t* improved) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < touches;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / t.L;
    const int p = (int)(i - c * t.L);
    const int64_t flat = flats[i];
    const double fit = fits[c];
    if (!(fit > 0.0)) {  // entries.get(key, 0.0): a zero fitness creates no entry
      improved[i] = 0;
      continue;
    }
    const unsigned long long bits = (unsigned long long)__double_as_longlong(fit);
    const int64_t h = table_slot(t.keys, t.count, t.cap, (unsigned long long)(flat * t.L + p + 1));
    const unsigned long long old = atomicMax(&t.vals[h], bits);
    improved[i] = fit > __longlong_as_double((long long)old) ? 1 : 0;
    atomicMax(reinterpret_cast<unsigned long long*>(t.smax + flat), bits);
  }
}

__global__ void fn_table_rehash_kernel(TableHandle dst, const unsigned long long* keys,
                                       const unsigned long long* vals, int64_t cap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
    if (keys[i] == 0ULL) continue;
    const int64_t h = table_slot(dst.keys, dst.count, dst.cap, keys[i]);
    dst.vals[h] = vals[i];
  }
}

static void table_free(TableHandle* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  cudaFree(t->keys);
  cudaFree(t->vals);
  cudaFree(t->count);
  cudaFree(t->smax);
  delete t;
}

// Capacity for `want` entries at load <= 1/2.
static isq_status table_reserve(TableHandle* t, int64_t want) {
  int64_t cap = t->cap;
  while (cap < 2 * want) cap *= 2;
  if (cap == t->cap) return ISQ_OK;
  TableHandle nt = *t;
  nt.cap = cap;
  nt.keys = nullptr;
  nt.vals = nullptr;
  nt.count = nullptr;
  TRYF(cudaMalloc((void**)&nt.keys, cap * 8));
  TRYF(cudaMalloc((void**)&nt.vals, cap * 8));
  TRYF(cudaMalloc((void**)&nt.count, 8));
  TRYF(cudaMemset(nt.keys, 0, cap * 8));
  TRYF(cudaMemset(nt.vals, 0, cap * 8));
  TRYF(cudaMemset(nt.count, 0, 8));
  fn_table_rehash_kernel<<<grid_for(t->cap), 256>>>(nt, t->keys, t->vals, t->cap);
  TRYF(cudaGetLastError());
  TRYF(cudaDeviceSynchronize());
  cudaFree(t->keys);
  cudaFree(t->vals);
  cudaFree(t->count);
  t->keys = nt.keys;
  t->vals = nt.vals;
  t->count = nt.count;
  t->cap = cap;
  return ISQ_OK;
}

// -------------------------------------------------------------------- GA ---

__global__ void fn_ga_random_genomes_kernel(int L, int ncodes, uint64_t seed, int64_t first, int64_t count,
                                            uint8_t* codes, double* thetas) {
  const int64_t total = count * L;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / L;
    const int j = (int)(t - i * L);
    NpStream s;
    s.init(seed, DOM_GA_INIT, 0, (uint64_t)(first + i), (uint64_t)j);
    codes[t] = (uint8_t)s.integers(ncodes);
    thetas[t] = s.uniform(0.0, kTwoPiD);
  }
}

// sus_select (ga.py:95-116) on two blocks (sus.cuh): block 0 the cumulative
// sums C[1..P-1], block 1 numpy's pairwise total and the pointers (or the
// uniform draws when every fitness is zero: *flag = 0 skips the search).
__global__ void __launch_bounds__(kSusThreads)
    fn_ga_sus_kernel(const double* f, int64_t P, int64_t count, uint64_t seed, uint64_t g, int64_t* picks,
                     double* C, double* Pt, int* flag, void* grid) {
  __shared__ double sm[kSusThreads];
  extern __shared__ double chain_smem[];
  if (blockIdx.x == 0) {
    if (grid == nullptr) exact_chain_block(f, 0.0, P - 1, 0.0, C, chain_smem);
    return;
  }
  __shared__ int s_neg;
  if (threadIdx.x == 0) s_neg = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x)
    if (!(f[i] >= 0.0)) s_neg = 1;  // negative or NaN: the sums are not monotone
  const double total = grid != nullptr  // syncs first
                           ? np_pairwise_combine_block<kSusThreads>(chain_grid_scratch(grid, P - 1).parts,
                                                                    pairwise_grid_depth(P), chain_smem)
                           : np_pairwise_sum_block<kSusThreads>(f, P, sm);
  NpStream rs;
  rs.init(seed, DOM_GA_SUS, g, 0, 0);
  if (total <= 0.0) {
    if (threadIdx.x == 0) {
      for (int64_t k = 0; k < count; ++k) picks[k] = rs.integers(P);
      *flag = 0;
    }
    return;
  }
  const double spacing = __ddiv_rn(total, (double)count);
  const double pointer = rs.uniform(0.0, spacing);
  if (s_neg) {  // the reference's walk itself, on one thread (engine fitness is never negative)
    if (threadIdx.x == 0) {
      double p = pointer, cumulative = 0.0;
      int64_t index = 0;
      for (int64_t k = 0; k < count; ++k) {
        while (index < P - 1 && __dadd_rn(cumulative, f[index]) <= p) {
          cumulative = __dadd_rn(cumulative, f[index]);
          ++index;
        }
        picks[k] = index;
        p = __dadd_rn(p, spacing);
      }
      *flag = 0;
    }
    return;
  }
  if (threadIdx.x == 0) {
    Pt[0] = pointer;
    *flag = 1;
  }
  exact_const_chain_block(spacing, count - 1, pointer, Pt + 1);
}

// two_point_crossover cuts (ga.py:81-92): sorted(integers(0, L + 1, size=2)), no draw for L < 2.
__global__ void fn_ga_cuts_kernel(int L, uint64_t seed, uint64_t g, int64_t first, int64_t count, int32_t* pq) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    int p = 0, q = 0;
    if (L >= 2) {
      NpStream cs;
      cs.init(seed, DOM_GA_PAIR, g, (uint64_t)(first + k), 0);
      const int x = (int)cs.integers(L + 1), y = (int)cs.integers(L + 1);
      p = x < y ? x : y;
      q = x < y ? y : x;
    }
    pq[2 * k] = p;
    pq[2 * k + 1] = q;
  }
}

// ga_mutate (ga.py:119-138), gene j of child `first + i`.
__global__ void fn_ga_mutate_kernel(int L, int ncodes, double rate, double mrange, double structural, uint64_t seed,
                                    uint64_t g, int64_t first, int64_t count, uint8_t* codes, double* thetas) {
  const int64_t total = count * L;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / L;
    const int j = (int)(t - i * L);
    NpStream ms;
    ms.init(seed, DOM_GA_MUT, g, (uint64_t)(first + i), (uint64_t)j);
    if (ms.random() >= rate) continue;
    if (ms.random() < structural)
      codes[t] = (uint8_t)ms.integers(ncodes);
    else
      thetas[t] = py_mod(__dadd_rn(thetas[t], ms.uniform(-mrange, mrange)), kTwoPiD);
  }
}

}  // namespace isq

using namespace isq;

extern "C" {

isq_status isq_init_population(int32_t n, int32_t L, int64_t P, uint64_t seed, double* thetas, double* qutrits,
                               int32_t device) {
  isq_status st = check_layout(n, L, P);
  if (st != ISQ_OK) return st;
  TRYF(cudaSetDevice(device));
  const QeqeaArgs a = functional_args(n, L, P, seed);
  DevBuf dt, dq;
  TRYF(dt.alloc(a.Q * 8));
  TRYF(dq.alloc(a.Qt * 48));
  fn_init_population_kernel<<<grid_for(a.Q), 256>>>(a, dt.as<double>(), dq.as<double2>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(thetas, dt.p, a.Q * 8, cudaMemcpyDeviceToHost));
  TRYF(cudaMemcpy(qutrits, dq.p, a.Qt * 48, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_construct_segments(int32_t n, int32_t L, int64_t P, int32_t n_meas, uint64_t seed,
                                  uint64_t generation, const double* qutrits, int8_t* axes, int32_t device) {
  isq_status st = check_layout(n, L, P);
  if (st != ISQ_OK) return st;
  if (n_meas < 1) return bad_config("nMeas must be ≥ 1");
  TRYF(cudaSetDevice(device));
  QeqeaArgs a = functional_args(n, L, P, seed);
  a.n_meas = n_meas;
  DevBuf dq, dx;
  TRYF(dq.alloc(a.Qt * 48));
  TRYF(dx.alloc(a.Qt));
  TRYF(cudaMemcpy(dq.p, qutrits, a.Qt * 48, cudaMemcpyHostToDevice));
  fn_construct_segments_kernel<<<grid_for(a.Qt), 256>>>(a, generation, dq.as<double2>(), dx.as<int8_t>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(axes, dx.p, a.Qt, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_sample_circuits(int32_t n, int32_t L, int64_t P, uint64_t seed, uint64_t generation, int64_t c0,
                               int64_t count, int64_t* flats, int32_t device) {
  isq_status st = check_layout(n, L, P);
  if (st != ISQ_OK) return st;
  if (c0 < 0 || count < 0) return bad_config("circuit range out of bounds");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  const QeqeaArgs a = functional_args(n, L, P, seed);
  DevBuf d32, d64;
  TRYF(d32.alloc(count * L * 4));
  TRYF(d64.alloc(count * L * 8));
  fn_sample_kernel<<<grid_for(count, 4), 128>>>(a, generation, c0, count, d32.as<uint32_t>());
  fn_widen_kernel<<<grid_for(count * L), 256>>>(d32.as<uint32_t>(), d64.as<int64_t>(), count * L);
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(flats, d64.p, count * L * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_mutate_population(const isq_qeqea_config* cfg, uint64_t generation, double* thetas, double* qutrits,
                                 const double* slot_max, uint8_t* mutated, int32_t device) {
  isq_status st = check_layout(cfg->number_of_wires, cfg->size_of_individual, cfg->size_of_population);
  if (st != ISQ_OK) return st;
  if (!(cfg->probability_of_mutation >= 0.0 && cfg->probability_of_mutation <= 1.0))
    return bad_config("probabilityOfMutation must be in [0, 1]");
  if (!(cfg->mutation_range > 0.0)) return bad_config("mutationRange must be > 0");
  TRYF(cudaSetDevice(device));
  QeqeaArgs a = functional_args(cfg->number_of_wires, cfg->size_of_individual, cfg->size_of_population, cfg->seed);
  a.p_mut = cfg->probability_of_mutation;
  a.mutation_range = cfg->mutation_range;
  DevBuf dt, dq, ds, dm;
  TRYF(dt.alloc(a.Q * 8));
  TRYF(dq.alloc(a.Qt * 48));
  TRYF(ds.alloc(a.Q * 8));
  TRYF(dm.alloc(a.Q));
  TRYF(cudaMemcpy(dt.p, thetas, a.Q * 8, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(dq.p, qutrits, a.Qt * 48, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(ds.p, slot_max, a.Q * 8, cudaMemcpyHostToDevice));
  fn_mutate_population_kernel<<<grid_for(a.Q), 256>>>(a, generation, dt.as<double>(), dq.as<double2>(),
                                                      ds.as<double>(), dm.as<uint8_t>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(thetas, dt.p, a.Q * 8, cudaMemcpyDeviceToHost));
  TRYF(cudaMemcpy(qutrits, dq.p, a.Qt * 48, cudaMemcpyDeviceToHost));
  TRYF(cudaMemcpy(mutated, dm.p, a.Q, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_table_create(int64_t qubit_count, int32_t length, int32_t device, void** handle) {
  *handle = nullptr;
  if (qubit_count < 1 || length < 1) return bad_config("qubit_count and sizeOfIndividual must be ≥ 1");
  TRYF(cudaSetDevice(device));
  TableHandle* t = new TableHandle();
  t->Q = qubit_count;
  t->L = length;
  t->device = device;
  t->cap = 1024;
  cudaError_t e = cudaMalloc((void**)&t->keys, t->cap * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&t->vals, t->cap * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&t->count, 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&t->smax, qubit_count * 8);
  if (e == cudaSuccess) e = cudaMemset(t->keys, 0, t->cap * 8);
  if (e == cudaSuccess) e = cudaMemset(t->vals, 0, t->cap * 8);
  if (e == cudaSuccess) e = cudaMemset(t->count, 0, 8);
  if (e == cudaSuccess) e = cudaMemset(t->smax, 0, qubit_count * 8);
  if (e != cudaSuccess) {
    table_free(t);
    set_error(std::string("table allocation: ") + cudaGetErrorString(e));
    return ISQ_ERR_CUDA;
  }
  *handle = t;
  return ISQ_OK;
}

isq_status isq_table_destroy(void* handle) {
  table_free(static_cast<TableHandle*>(handle));
  return ISQ_OK;
}

isq_status isq_table_update(void* handle, int64_t count, const int64_t* blueprints, const double* fitness,
                            uint8_t* improved) {
  TableHandle* t = static_cast<TableHandle*>(handle);
  if (!t) return bad_config("null table handle");
  if (count <= 0) return ISQ_OK;
  const int64_t touches = count * t->L;
  for (int64_t i = 0; i < touches; ++i)
    if (blueprints[i] < 0 || blueprints[i] >= t->Q) return bad_config("blueprint slot out of range");
  for (int64_t c = 0; c < count; ++c)
    if (!(fitness[c] >= 0.0)) return bad_config("fitness must be a number >= 0");
  TRYF(cudaSetDevice(t->device));
  unsigned long long have = 0;
  TRYF(cudaMemcpy(&have, t->count, 8, cudaMemcpyDeviceToHost));
  isq_status st = table_reserve(t, (int64_t)have + touches);
  if (st != ISQ_OK) return st;
  DevBuf df, dv, di;
  TRYF(df.alloc(touches * 8));
  TRYF(dv.alloc(count * 8));
  TRYF(di.alloc(touches));
  TRYF(cudaMemcpy(df.p, blueprints, touches * 8, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(dv.p, fitness, count * 8, cudaMemcpyHostToDevice));
  fn_table_update_kernel<<<grid_for(touches), 256>>>(*t, touches, df.as<int64_t>(), dv.as<double>(),
                                                    di.as<uint8_t>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(improved, di.p, touches, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_table_read(void* handle, double* slot_max, int64_t* n_entries, int64_t* keys, double* values) {
  TableHandle* t = static_cast<TableHandle*>(handle);
  if (!t) return bad_config("null table handle");
  TRYF(cudaSetDevice(t->device));
  if (slot_max) TRYF(cudaMemcpy(slot_max, t->smax, t->Q * 8, cudaMemcpyDeviceToHost));
  unsigned long long have = 0;
  TRYF(cudaMemcpy(&have, t->count, 8, cudaMemcpyDeviceToHost));
  if (n_entries) *n_entries = (int64_t)have;
  if (keys || values) {
    std::vector<unsigned long long> k(t->cap), v(t->cap);
    TRYF(cudaMemcpy(k.data(), t->keys, t->cap * 8, cudaMemcpyDeviceToHost));
    TRYF(cudaMemcpy(v.data(), t->vals, t->cap * 8, cudaMemcpyDeviceToHost));
    int64_t o = 0;
    for (int64_t i = 0; i < t->cap; ++i) {
      if (k[i] == 0ULL) continue;
      if (keys) keys[o] = (int64_t)(k[i] - 1);  // flat * L + position
      if (values) std::memcpy(&values[o], &v[i], 8);
      ++o;
    }
  }
  return ISQ_OK;
}

isq_status isq_table_set_slot_max(void* handle, const double* slot_max) {
  TableHandle* t = static_cast<TableHandle*>(handle);
  if (!t) return bad_config("null table handle");
  TRYF(cudaSetDevice(t->device));
  TRYF(cudaMemcpy(t->smax, slot_max, t->Q * 8, cudaMemcpyHostToDevice));
  return ISQ_OK;
}

isq_status isq_apply_gates(int32_t n, int32_t length, int64_t count, const uint8_t* codes, const double* thetas,
                           const double* acc_in, double* acc_out, int32_t device) {
  if (n < ISQ_MIN_WIRES || n > ISQ_MAX_WIRES) {
    set_error("numberOfWires=" + std::to_string(n) + " is outside the supported range 2..13");
    return n < 2 ? ISQ_ERR_CONFIG : ISQ_ERR_UNSUPPORTED;
  }
  if (length < 0 || count < 0) return bad_config("negative circuit length or count");
  const int ncodes = 3 * n + n * (n - 1) / 2;
  for (int64_t i = 0; i < count * (int64_t)length; ++i)
    if (codes[i] >= ncodes) return bad_config("gate code out of range for numberOfWires");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  const int64_t DD = (int64_t)1 << (2 * n);
  DevBuf dc, dt, di, dout, df, dT;
  TRYF(dc.alloc(count * length + 1));
  TRYF(dt.alloc((count * length + 1) * 8));
  TRYF(di.alloc(count * DD * 16));
  TRYF(dout.alloc(count * DD * 16));
  TRYF(df.alloc(count * 8));
  TRYF(dT.alloc(DD * 16));
  TRYF(cudaMemset(dT.p, 0, DD * 16));
  if (length > 0) {
    TRYF(cudaMemcpy(dc.p, codes, count * length, cudaMemcpyHostToDevice));
    TRYF(cudaMemcpy(dt.p, thetas, count * length * 8, cudaMemcpyHostToDevice));
  }
  TRYF(cudaMemcpy(di.p, acc_in, count * DD * 16, cudaMemcpyHostToDevice));
  isq_status st = launch_fitness_generic(n, length, count, dc.as<uint8_t>(), dt.as<double>(), dT.as<double>(),
                                         df.as<double>(), dout.as<double>(), nullptr, nullptr, nullptr,
                                         nullptr, nullptr, nullptr, di.as<double>());
  if (st != ISQ_OK) return st;
  TRYF(cudaMemcpy(acc_out, dout.p, count * DD * 16, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_ga_random_genomes(int32_t n, int32_t L, uint64_t seed, int64_t first, int64_t count, uint8_t* codes,
                                 double* thetas, int32_t device) {
  isq_status st = check_layout(n, L, 1);
  if (st != ISQ_OK) return st;
  if (first < 0 || count < 0) return bad_config("genome range out of bounds");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  DevBuf dc, dt;
  TRYF(dc.alloc(count * L));
  TRYF(dt.alloc(count * L * 8));
  fn_ga_random_genomes_kernel<<<grid_for(count * L), 256>>>(L, 3 * n + n * (n - 1) / 2, seed, first, count,
                                                            dc.as<uint8_t>(), dt.as<double>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(codes, dc.p, count * L, cudaMemcpyDeviceToHost));
  TRYF(cudaMemcpy(thetas, dt.p, count * L * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_ga_sus_select(int64_t P, const double* fitness, int64_t count, uint64_t seed, uint64_t generation,
                             int64_t* picks, int32_t device) {
  if (P < 1 || count < 0) return bad_config("sus_select needs at least one fitness value");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  DevBuf df, dp;
  TRYF(df.alloc(P * 8));
  TRYF(dp.alloc(count * 8));
  TRYF(cudaMemcpy(df.p, fitness, P * 8, cudaMemcpyHostToDevice));
  DevBuf dC, dP, dflag;
  TRYF(dC.alloc(P * 8));
  TRYF(dP.alloc(count * 8));
  TRYF(dflag.alloc(sizeof(int)));
  TRYF(cudaFuncSetAttribute((const void*)fn_ga_sus_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kChainSmem));
  const bool grid = chain_grid_worth(P - 1);  // the running sums over the whole GPU (sus.cuh)
  DevBuf dg;
  if (grid) {
    TRYF(prepare_exact_chain_grid());
    TRYF(dg.alloc(chain_grid_scratch_bytes(P - 1)));
    TRYF(launch_pairwise_parts(df.as<double>(), P, dg.p, P - 1, nullptr));
    TRYF(launch_exact_chain_grid(df.as<double>(), P - 1, 0.0, dC.as<double>(), dg.p, nullptr));
  }
  fn_ga_sus_kernel<<<2, kSusThreads, kChainSmem>>>(df.as<double>(), P, count, seed, generation, dp.as<int64_t>(),
                                       dC.as<double>(), dP.as<double>(), dflag.as<int>(), grid ? dg.p : nullptr);
  TRYF(cudaGetLastError());
  sus_search_kernel<int64_t><<<grid_for(count), 256>>>(dC.as<double>(), P - 1, dP.as<double>(), count,
                                                       dp.as<int64_t>(), dflag.as<int>(), nullptr);
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(picks, dp.p, count * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_ga_crossover_cuts(int32_t L, uint64_t seed, uint64_t generation, int64_t first, int64_t count,
                                 int32_t* cuts, int32_t device) {
  if (L < 0 || first < 0 || count < 0) return bad_config("crossover range out of bounds");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  DevBuf dc;
  TRYF(dc.alloc(count * 8));
  fn_ga_cuts_kernel<<<grid_for(count), 256>>>(L, seed, generation, first, count, dc.as<int32_t>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(cuts, dc.p, count * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_ga_mutate_genomes(const isq_ga_config* cfg, uint64_t generation, int64_t first, int64_t count,
                                 uint8_t* codes, double* thetas, int32_t device) {
  const int n = cfg->number_of_wires, L = cfg->size_of_individual;
  isq_status st = check_layout(n, L, 1);
  if (st != ISQ_OK) return st;
  if (first < 0 || count < 0) return bad_config("genome range out of bounds");
  if (count == 0) return ISQ_OK;
  TRYF(cudaSetDevice(device));
  DevBuf dc, dt;
  TRYF(dc.alloc(count * L));
  TRYF(dt.alloc(count * L * 8));
  TRYF(cudaMemcpy(dc.p, codes, count * L, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(dt.p, thetas, count * L * 8, cudaMemcpyHostToDevice));
  fn_ga_mutate_kernel<<<grid_for(count * L), 256>>>(L, 3 * n + n * (n - 1) / 2, cfg->mutation_rate,
                                                    cfg->mutation_range, cfg->structural_rate, cfg->seed, generation,
                                                    first, count, dc.as<uint8_t>(), dt.as<double>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(codes, dc.p, count * L, cudaMemcpyDeviceToHost));
  TRYF(cudaMemcpy(thetas, dt.p, count * L * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

}  // extern "C"

// ===================================================================
// encoding.py's per-unit operators (encoding.py:40-132), batched: element i
// is unit `first + i` of the counter streams the engines use --
//   mutate_angle / mutate_qutrit: the slot's mutation stream (seed, MUTATE,
//     generation, slot) after the engine's mask and coin draws (engine.py:
//     241-242), i.e. exactly the step mutate_population gives that slot;
//   estimate_axis: the slot's measurement stream (seed, MEASURE, generation,
//     slot), as construct_segments;
//   measure_qutrit (not drawn by the engines): (seed, MEASURE, generation,
//     slot, sub = 1);
//   random_angle / random_qutrit: the slot's init stream (init_population).
// ===================================================================
namespace isq_enc {  // (named: a second anonymous namespace confuses the kernel stubs)

__global__ void enc_mutate_angles_kernel(int64_t count, const double* th, const double* f, double range,
                                         uint64_t seed, uint64_t g, int64_t first, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    stream_block(seed, DOM_MUTATE, g, (uint64_t)(first + i), 0, 1, w);
    const double sign = u64_to_double(w[2]) < 0.5 ? 1.0 : -1.0;  // encoding.py:51
    const double step = __dmul_rn(__dmul_rn(sign, __dsub_rn(1.0, f[i])), range);
    out[i] = py_mod(__dadd_rn(th[i], step), kTwoPiD);
  }
}

__global__ void enc_mutate_qutrits_kernel(int64_t count, const double2* q, const double* f, uint64_t seed, uint64_t g,
                                          int64_t first, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    stream_block(seed, DOM_MUTATE, g, (uint64_t)(first + i), 0, 1, w);
    const int which = (int)((uint32_t)(w[2] & 0xffffffffULL) >> 29);  // integers(8): Lemire, bound 8
    const double range = which < 3 ? kHalfPiD : kTwoPiD;               // SU3_RANGES (encoding.py:23)
    const double value = __dadd_rn(0.0, __dmul_rn(__dmul_rn(range, __dsub_rn(1.0, f[i])), u64_to_double(w[3])));
    double2 v[3] = {q[3 * i], q[3 * i + 1], q[3 * i + 2]};
    su3_one_param(which, value, v);
#pragma unroll
    for (int k = 0; k < 3; ++k) out[3 * i + k] = v[k];
  }
}

// born_probabilities (encoding.py:66-71): numpy |q|^2, the left-to-right sum,
// the 1e-6 norm invariant, the division.
__device__ __forceinline__ bool enc_born(const double2* q, double pr[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = np_cabs(q[k].x, q[k].y);
    pr[k] = __dmul_rn(a, a);
  }
  const double norm = __dadd_rn(__dadd_rn(pr[0], pr[1]), pr[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) pr[k] = __ddiv_rn(pr[k], norm);
  return !(fabs(__dsub_rn(norm, 1.0)) > 1e-6);
}

__global__ void enc_born_kernel(int64_t count, const double2* q, double* probs, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double pr[3];
    if (!enc_born(q + 3 * i, pr)) atomicOr(bad, 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) probs[3 * i + k] = pr[k];
  }
}

__global__ void enc_estimate_axes_kernel(int64_t count, const double2* q, int n_meas, uint64_t seed, uint64_t g,
                                         int64_t first, int8_t* axes, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double pr[3];
    if (!enc_born(q + 3 * i, pr)) atomicOr(bad, 1);
    const double re[3] = {q[3 * i].x, q[3 * i + 1].x, q[3 * i + 2].x};
    const double im[3] = {q[3 * i].y, q[3 * i + 1].y, q[3 * i + 2].y};
    NpStream st;
    st.init(seed, DOM_MEASURE, g, (uint64_t)(first + i), 0);
    bool ok = true;
    axes[i] = (int8_t)measure_axis(re, im, n_meas, st, &ok);
  }
}

// measure_qutrit (encoding.py:74-77): Generator.choice(3, p=probs) -- cdf =
// cumsum(p), cdf /= cdf[-1], one random(), searchsorted(side='right').
__global__ void enc_measure_qutrits_kernel(int64_t count, const double2* q, uint64_t seed, uint64_t g, int64_t first,
                                           int8_t* axes, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double pr[3];
    if (!enc_born(q + 3 * i, pr)) atomicOr(bad, 1);
    const double c0 = pr[0], c1 = __dadd_rn(c0, pr[1]), c2 = __dadd_rn(c1, pr[2]);
    const double d0 = __ddiv_rn(c0, c2), d1 = __ddiv_rn(c1, c2), d2 = __ddiv_rn(c2, c2);
    uint64_t w[4];
    stream_block(seed, DOM_MEASURE, g, (uint64_t)(first + i), 1, 1, w);
    const double u = u64_to_double(w[0]);
    axes[i] = (int8_t)((d0 <= u) + (d1 <= u) + (d2 <= u));
  }
}

// su3_operator (encoding.py:87-116) for general parameters (theta1..3,
// phi1..5): the engines only ever need one nonzero parameter
// (su3_one_param); this is the full template, entry by entry.
__device__ __forceinline__ double2 enc_cis(double a) {  // e^{i a}
  double s, c;
  sincos(a, &s, &c);
  return make_double2(c, s);
}
__device__ __forceinline__ double2 enc_scale(double2 z, double r) { return make_double2(z.x * r, z.y * r); }
__device__ __forceinline__ double2 enc_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

__global__ void enc_su3_kernel(int64_t count, const double* prm, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double* p = prm + 8 * i;
    double s1, c1, s2, c2, s3, c3;
    sincos(p[0], &s1, &c1);
    sincos(p[1], &s2, &c2);
    sincos(p[2], &s3, &c3);
    const double f1 = p[3], f2 = p[4], f3 = p[5], f4 = p[6], f5 = p[7];
    double2* u = out + 9 * i;
    u[0] = enc_scale(enc_scale(enc_cis(f1), c1), c2);
    u[1] = enc_scale(enc_cis(f3), s1);
    u[2] = enc_scale(enc_scale(enc_cis(f4), c1), s2);
    u[3] = enc_sub(enc_scale(enc_scale(enc_cis(-f4 - f5), s2), s3), enc_scale(enc_scale(enc_scale(enc_cis(f1 + f2 - f3), s1), c2), c3));
    u[4] = enc_scale(enc_scale(enc_cis(f2), c1), c3);
    u[5] = enc_sub(enc_scale(enc_scale(enc_cis(-f1 - f5), -c2), s3), enc_scale(enc_scale(enc_scale(enc_cis(f2 - f3 + f4), s1), s2), c3));
    u[6] = enc_sub(enc_scale(enc_scale(enc_cis(-f2 - f4), -s2), c3), enc_scale(enc_scale(enc_scale(enc_cis(f1 - f3 + f5), s1), c2), s3));
    u[7] = enc_scale(enc_scale(enc_cis(f5), c1), s3);
    u[8] = enc_sub(enc_scale(enc_scale(enc_cis(-f1 - f2), c2), c3), enc_scale(enc_scale(enc_scale(enc_cis(-f3 + f4 + f5), s1), s2), s3));
  }
}

__global__ void enc_init_slots_kernel(int64_t count, uint64_t seed, int64_t first, int with_qutrit, double* th,
                                      double2* q) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double t;
    double2 v[3];
    init_slot_value(seed, first + i, with_qutrit != 0, t, v);
    th[i] = t;
    if (with_qutrit) {
#pragma unroll
      for (int k = 0; k < 3; ++k) q[3 * i + k] = v[k];
    }
  }
}

isq_status enc_range(int64_t count, int64_t first) {
  if (count < 0 || first < 0) return bad_config("unit range out of bounds");
  return ISQ_OK;
}

// Shared host side of the three Born-rule entries: `kind` 0 born, 1 estimate, 2 measure.
isq_status enc_born_call(int kind, int64_t count, const double* qutrits, int32_t n_meas, uint64_t seed,
                         uint64_t generation, int64_t first, void* out, int32_t device) {
  isq_status st = enc_range(count, first);
  if (st != ISQ_OK || count == 0) return st;
  if (kind == 1 && n_meas < 1) return bad_config("nMeas must be ≥ 1");
  TRYF(cudaSetDevice(device));
  DevBuf dq, dout, dbad;
  const size_t ob = kind == 0 ? (size_t)count * 24 : (size_t)count;
  TRYF(dq.alloc(count * 48));
  TRYF(dout.alloc(ob));
  TRYF(dbad.alloc(sizeof(int)));
  TRYF(cudaMemset(dbad.p, 0, sizeof(int)));
  TRYF(cudaMemcpy(dq.p, qutrits, count * 48, cudaMemcpyHostToDevice));
  if (kind == 0)
    enc_born_kernel<<<grid_for(count), 256>>>(count, dq.as<double2>(), dout.as<double>(), dbad.as<int>());
  else if (kind == 1)
    enc_estimate_axes_kernel<<<grid_for(count), 256>>>(count, dq.as<double2>(), n_meas, seed, generation, first,
                                                       dout.as<int8_t>(), dbad.as<int>());
  else
    enc_measure_qutrits_kernel<<<grid_for(count), 256>>>(count, dq.as<double2>(), seed, generation, first,
                                                         dout.as<int8_t>(), dbad.as<int>());
  TRYF(cudaGetLastError());
  int bad = 0;
  TRYF(cudaMemcpy(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) {
    set_error("qutrit norm² deviates from 1 by more than 1e-6");
    return ISQ_ERR_INVARIANT;
  }
  TRYF(cudaMemcpy(out, dout.p, ob, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}
}  // namespace isq_enc

using namespace isq_enc;

extern "C" {

isq_status isq_mutate_angles(int64_t count, const double* thetas, const double* segment_fitness,
                             double mutation_range, uint64_t seed, uint64_t generation, int64_t first, double* out,
                             int32_t device) {
  isq_status st = enc_range(count, first);
  if (st != ISQ_OK || count == 0) return st;
  TRYF(cudaSetDevice(device));
  DevBuf dt, df, dout;
  TRYF(dt.alloc(count * 8));
  TRYF(df.alloc(count * 8));
  TRYF(dout.alloc(count * 8));
  TRYF(cudaMemcpy(dt.p, thetas, count * 8, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(df.p, segment_fitness, count * 8, cudaMemcpyHostToDevice));
  enc_mutate_angles_kernel<<<grid_for(count), 256>>>(count, dt.as<double>(), df.as<double>(), mutation_range, seed,
                                                     generation, first, dout.as<double>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(out, dout.p, count * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_mutate_qutrits(int64_t count, const double* qutrits, const double* segment_fitness, uint64_t seed,
                              uint64_t generation, int64_t first, double* out, int32_t device) {
  isq_status st = enc_range(count, first);
  if (st != ISQ_OK || count == 0) return st;
  TRYF(cudaSetDevice(device));
  DevBuf dq, df, dout;
  TRYF(dq.alloc(count * 48));
  TRYF(df.alloc(count * 8));
  TRYF(dout.alloc(count * 48));
  TRYF(cudaMemcpy(dq.p, qutrits, count * 48, cudaMemcpyHostToDevice));
  TRYF(cudaMemcpy(df.p, segment_fitness, count * 8, cudaMemcpyHostToDevice));
  enc_mutate_qutrits_kernel<<<grid_for(count), 256>>>(count, dq.as<double2>(), df.as<double>(), seed, generation,
                                                      first, dout.as<double2>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(out, dout.p, count * 48, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}


isq_status isq_born_probabilities(int64_t count, const double* qutrits, double* probs, int32_t device) {
  return enc_born_call(0, count, qutrits, 1, 0, 0, 0, probs, device);
}

isq_status isq_estimate_axes(int64_t count, const double* qutrits, int32_t n_meas, uint64_t seed, uint64_t generation,
                             int64_t first, int8_t* axes, int32_t device) {
  return enc_born_call(1, count, qutrits, n_meas, seed, generation, first, axes, device);
}

isq_status isq_measure_qutrits(int64_t count, const double* qutrits, uint64_t seed, uint64_t generation,
                               int64_t first, int8_t* axes, int32_t device) {
  return enc_born_call(2, count, qutrits, 1, seed, generation, first, axes, device);
}

isq_status isq_su3_operators(int64_t count, const double* params, double* out, int32_t device) {
  isq_status st = enc_range(count, 0);
  if (st != ISQ_OK || count == 0) return st;
  TRYF(cudaSetDevice(device));
  DevBuf dp, dout;
  TRYF(dp.alloc(count * 64));
  TRYF(dout.alloc(count * 144));
  TRYF(cudaMemcpy(dp.p, params, count * 64, cudaMemcpyHostToDevice));
  enc_su3_kernel<<<grid_for(count), 256>>>(count, dp.as<double>(), dout.as<double2>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(out, dout.p, count * 144, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

isq_status isq_init_slots(int64_t count, uint64_t seed, int64_t first, int32_t with_qutrit, double* thetas,
                          double* qutrits, int32_t device) {
  isq_status st = enc_range(count, first);
  if (st != ISQ_OK || count == 0) return st;
  if (with_qutrit && qutrits == nullptr) return bad_config("qutrits output missing");
  TRYF(cudaSetDevice(device));
  DevBuf dt, dq;
  TRYF(dt.alloc(count * 8));
  TRYF(dq.alloc(with_qutrit ? count * 48 : 16));
  enc_init_slots_kernel<<<grid_for(count), 256>>>(count, seed, first, with_qutrit, dt.as<double>(),
                                                  dq.as<double2>());
  TRYF(cudaGetLastError());
  TRYF(cudaMemcpy(thetas, dt.p, count * 8, cudaMemcpyDeviceToHost));
  if (with_qutrit) TRYF(cudaMemcpy(qutrits, dq.p, count * 48, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

}  // extern "C"

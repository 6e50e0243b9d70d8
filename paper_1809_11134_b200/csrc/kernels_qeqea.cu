// QEQEA generation loop kernels (QeqeaEngine.step, engine.py:318-361).
//
// One generation g is the launch sequence
//   sample   this rank's circuits: blueprints (flat slots)                     (K2)
//   route    world > 1: touches grouped by the rank owning their position
//            (caller: all-to-all of the flats)
//   values   owned touches: live slot (lazy mutation) + measured gate code    (K1, K5)
//            (caller, world > 1: all-to-all of codes / angles back)
//   unroute  world > 1: codes / angles back into circuit order
//   fitness  compose + score this rank's circuits                             (K3)
//   elite    world > 1: shard best + its gates (caller: all-gather of fitness + elites)
//   reduce   gen max / first argmax / mean, best-so-far, record, best gates   (K4)
//   commit   owned touches: improved & mutated -> committed bank, slot_max    (K4, K5)
//   advance  generation += 1, stop reason (engine.py:354-358)
// Every kernel reads the generation from device state and returns
// immediately once a stop reason is set, so batches of generations are
// enqueued without host round trips.
#include "engine_common.cuh"
#include "fitness_multi.cuh"
#include "fitness_warp.cuh"
#include "isq_internal.h"
#include "qeqea_internal.h"

namespace isq {

// ---------------------------------------------------------------- eval ---
// sample (all circuits, flats -> HBM) | values (shard touches -> gate code +
// live angle) | fitness_fast_kernel (kernels_fitness.cu).  Separate kernels
// keep each one's hot code inside the instruction cache and give the random
// bank gathers thread-level memory parallelism.

#ifndef ISQ_SAMPLE_RUN
#define ISQ_SAMPLE_RUN 16
#endif
constexpr int kSampleRun = ISQ_SAMPLE_RUN;  // circuits per warp task of the batched sampler (64: a partial last wave)
#ifndef ISQ_FIT_DYNAMIC
#define ISQ_FIT_DYNAMIC 1
#endif
#ifndef ISQ_SAMPLE_FULL_GRID
#define ISQ_SAMPLE_FULL_GRID 1
#endif

__global__ void __launch_bounds__(kThreadsPerBlock) qeqea_sample_flats_kernel(QeqeaArgs a) {
  __shared__ uint64_t blk[kWarpsPerBlock][128 * kSampleIlp];
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  const int64_t c1 = min(a.P, a.c0 + a.S);
  if (sample_blocks_per_circuit(a) <= 32) {
    // short circuits (L <= 128): runs of kSampleRun circuits per warp, all lanes on Philox
    for (int64_t r = a.c0 + ((int64_t)blockIdx.x * kWarpsPerBlock + wib) * kSampleRun; r < c1;
         r += nwarps * kSampleRun)
      sample_circuits_batched(a, g, r, min(c1, r + kSampleRun), a.flats + (r - a.c0) * a.L, blk[wib], lane);
    return;
  }
  for (int64_t c = a.c0 + (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < c1; c += nwarps)
    sample_circuit_warp(a, g, c, a.flats + (c - a.c0) * a.L, blk[wib], lane);
}

// Position p -> owning rank, and the offset of (circuit c_loc, position p) in
// the owner-grouped exchange layout: block o holds S x Lr(o) entries, row =
// circuit, starting at S * p_bounds[o].
__device__ __forceinline__ int64_t routed_index(const QeqeaArgs& a, int64_t c_loc, int p) {
  int o = 0;
  while (p >= a.p_bounds[o + 1]) ++o;
  const int lo = a.p_bounds[o], lr = a.p_bounds[o + 1] - lo;
  return a.S * lo + c_loc * lr + (p - lo);
}

// world > 1: this rank's touches grouped by owner (padding circuits send
// kNoSlot).  Peer transport: stored straight into the owner's receive buffer
// at the place the all-to-all would put them (block of source rank r at
// r * S * Lr(o), row = circuit, column = owned position).
__global__ void qeqea_route_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  const int64_t n = a.S * a.L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c_loc = a.div_L.div((uint32_t)i);
    const int p = (int)(i - c_loc * a.L);
    const uint32_t f = a.c0 + c_loc < a.P ? a.flats[i] : kNoSlot;
    if (a.peers) {
      int o = 0;
      while (p >= a.p_bounds[o + 1]) ++o;
      const int lo = a.p_bounds[o], lr = a.p_bounds[o + 1] - lo;
      a.peers->recv_flats[o][(a.rank * a.S + c_loc) * lr + (p - lo)] = f;
    } else {
      a.send_flats[routed_index(a, c_loc, p)] = f;
    }
  }
  if (a.peers) __threadfence_system();
}

// world > 1: the owners' gate codes / live angles back into circuit order.
__global__ void qeqea_unroute_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  const int64_t n = a.S * a.L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c_loc = a.div_L.div((uint32_t)i);
    const int64_t src = routed_index(a, c_loc, (int)(i - c_loc * a.L));
    a.gate_codes[i] = a.recv_codes[src];
    a.gate_thetas[i] = a.recv_thetas[src];
  }
}

// One thread per owned touch t (row = global circuit, column = owned
// position): committed record -> live value (pending mutation of g-1).
// Rotation touches (1/3 at C5) additionally need the Born measurement; those
// are compacted into a shared-memory queue so the costly measurement runs on
// full warps instead of on the 1/3 of lanes that need it.  Also records, per
// touch, the slot_max the generation started from and whether the slot
// carries a pending mutation (the commit consumes both).
#ifndef ISQ_VAL_GRID_CAP
#define ISQ_VAL_GRID_CAP (1 << 30)
#endif
#ifndef ISQ_VAL_GRID_TILES
#define ISQ_VAL_GRID_TILES 1
#endif
#ifndef ISQ_VAL_PREDRAW
#define ISQ_VAL_PREDRAW 1
#endif
#ifndef ISQ_VAL_THREADS
#define ISQ_VAL_THREADS 256
#endif
constexpr int kValThreads = ISQ_VAL_THREADS;
#ifndef ISQ_VAL_PER_THREAD
#define ISQ_VAL_PER_THREAD 2
#endif
// touches per thread per tile (measured, C4 / C5 generations: 256 x 2 2.88k gen/s / 15.15 ms, 256 x 3 2.73k /
// 15.39, 256 x 1 2.74k / 15.86, 256 x 4 2.56k / 15.94, 128 x 2 2.86k / 15.17, 512 x 1 2.66k / 16.09)
constexpr int kValPerThread = ISQ_VAL_PER_THREAD;
constexpr int kValTile = kValThreads * kValPerThread;

// Per tile: the touches' committed records, staged by cp.async (no registers
// held while the random gathers are in flight), then updated in place.
struct ValuesShared {
  RotRec rec[kValTile];     // committed record (an IntRec in the first 16 B); qutrit updated in place
  uint32_t s[kValTile];     // slot of each touch
  double value[kValTile];   // pending SU(3) parameter (qutrit mutation)
  int8_t which[kValTile];   // its parameter index
  uint16_t task[kValTile];  // rotation touches to measure
  uint16_t qq[kValTile];    // of which with a pending qutrit mutation
  int ntask, nq;
};

// Gate code / live angle of owned touch t, to the owner-side arrays and, with
// the peer transport, straight into the receive buffers of the circuit's rank
// (block of this owner at S * p_lo, row = circuit - j * S, column = q).
__device__ __forceinline__ int64_t peer_recv_index(const QeqeaArgs& a, int64_t t, int64_t& j) {
  const int64_t c = a.div_Lr.div((uint32_t)t);
  j = a.div_S.div((uint32_t)c);
  return a.S * a.p_lo + (c - j * a.S) * a.Lr + (t - c * a.Lr);
}
__device__ __forceinline__ void emit_code(const QeqeaArgs& a, int64_t t, uint8_t code) {
  if (a.peers) {
    int64_t j;
    const int64_t idx = peer_recv_index(a, t, j);
    a.peers->recv_codes[j][idx] = code;
  } else {
    a.owner_codes[t] = code;
  }
}
__device__ __forceinline__ void emit_theta(const QeqeaArgs& a, int64_t t, double theta) {
  a.owner_thetas[t] = theta;  // the commit reads it back
  if (a.peers) {
    int64_t j;
    const int64_t idx = peer_recv_index(a, t, j);
    a.peers->recv_thetas[j][idx] = theta;
  }
}

// Values phase of owned touch t up to the Born measurement: the live value
// goes to v (angle mutations applied; a qutrit mutation is returned in
// which / value), the angle / starting slot_max / mutation flags to the touch
// arrays, and interaction slots get their gate code.  Returns true when the
// touch is a rotation slot still to be measured (measure_code).
__device__ __forceinline__ bool value_touch_from(const QeqeaArgs& a, int64_t t, uint64_t g, uint32_t s,
                                                 LiveSlot& v, int& which, double& value) {
  which = -1;
  if (s == kNoSlot) {  // padding circuit: never commits (fitness <= 1 < 2)
    emit_code(a, t, 0);
    emit_theta(a, t, 0.0);
    a.touch_fbefore[t] = 2.0;
    a.touch_mutated[t] = 0;
    return false;
  }
  const double f = load_committed(a, slot_local(a, s), v);
  const int m = g > 0 ? mutate_decide(a, s, g - 1, f, v, which, value) : MUT_NONE;
  if (m != MUT_QUTRIT) which = -1;
  emit_theta(a, t, v.theta);
  a.touch_fbefore[t] = f;
  a.touch_mutated[t] = (uint8_t)((m != MUT_NONE ? 1 : 0) | (m == MUT_QUTRIT ? 2 : 0));
  const int64_t kind = slot_kind(a, s);
  if (kind < a.n) return true;
  emit_code(a, t, (uint8_t)(3 * a.n + (kind - a.n)));
  return false;
}

__device__ __forceinline__ bool value_touch_head(const QeqeaArgs& a, int64_t t, uint64_t g, uint32_t& s,
                                                 LiveSlot& v, int& which, double& value) {
  s = a.owner_flats[t];
  return value_touch_from(a, t, g, s, v, which, value);
}

// construct_segments for one rotation slot (engine.py:167-170): Born
// measurement on the slot's (generation, slot) stream -> gate code.
template <bool kBTPE = true>
__device__ __forceinline__ uint8_t measure_code_on(const QeqeaArgs& a, uint32_t s, NpStream& st, double re[3],
                                                   double im[3]) {
  bool ok = true;
  const int axis = measure_axis<kBTPE>(re, im, a.n_meas, st, &ok);
  return (uint8_t)(3 * (slot_kind(a, s)) + axis);
}
template <bool kBTPE = true>
__device__ __forceinline__ uint8_t measure_code(const QeqeaArgs& a, uint32_t s, uint64_t g, double re[3],
                                                double im[3]) {
  NpStream st;
  st.init(a.seed, DOM_MEASURE, g, (uint64_t)s, 0);
  return measure_code_on<kBTPE>(a, s, st, re, im);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// Per tile of kValTile owned touches: (0) the records of all the tile's
// touches gathered into shared memory with cp.async; (1) lazy angle
// mutations, rotation touches queued; (2) the queued qutrit mutations (5 % of
// touches) on full warps; (3) the Born measurements of the queued rotation
// touches on full warps.
// BIG: n_meas > kInversionMaxMeas (the BTPE binomial branch compiled in).
template <bool BIG>
__global__ void __launch_bounds__(kValThreads) qeqea_values_kernel(QeqeaArgs a, int64_t t1) {
  extern __shared__ __align__(64) unsigned char val_smem[];
  ValuesShared& sm = *reinterpret_cast<ValuesShared*>(val_smem);
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  for (int64_t base = (int64_t)blockIdx.x * kValTile; base < t1; base += (int64_t)gridDim.x * kValTile) {
    if (threadIdx.x == 0) sm.ntask = sm.nq = 0;
#pragma unroll
    for (int u = 0; u < kValPerThread; ++u) {
      const int i = u * kValThreads + threadIdx.x;
      if (base + i >= t1) break;
      const uint32_t s = a.owner_flats[base + i];
      sm.s[i] = s;
      if (s == kNoSlot) continue;
      const int64_t loc = slot_local(a, s);
      if (loc < a.Qtloc) {
        const char* src = reinterpret_cast<const char*>(a.rot + loc);
#pragma unroll
        for (int k = 0; k < 4; ++k) cp_async16(reinterpret_cast<char*>(&sm.rec[i]) + 16 * k, src + 16 * k);
      } else {
        cp_async16(&sm.rec[i], a.inter + (loc - a.Qtloc));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
#if ISQ_VAL_PREDRAW
    // the mutation draws need only the stream key: computed while the
    // records are in flight
    MutDraw md[kValPerThread];
#pragma unroll
    for (int u = 0; u < kValPerThread; ++u) {
      const int i = u * kValThreads + threadIdx.x;
      md[u].bits = 0;
      md[u].d3 = 0.0;
      if (g > 0 && base + i < t1) {
        const uint32_t s = sm.s[i];
        if (s != kNoSlot) md[u] = mutate_draw(a, s, g - 1);
      }
    }
#endif
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kValPerThread; ++u) {
      const int i = u * kValThreads + threadIdx.x;
      const int64_t t = base + i;
      if (t >= t1) break;
      const uint32_t s = sm.s[i];
      if (s == kNoSlot) {  // padding circuit: never commits (fitness <= 1 < 2)
        emit_code(a, t, 0);
        emit_theta(a, t, 0.0);
        a.touch_fbefore[t] = 2.0;
        a.touch_mutated[t] = 0;
        continue;
      }
      const int64_t kind = slot_kind(a, s);
      const double2 ts = reinterpret_cast<const double2*>(&sm.rec[i])[kind < a.n ? 3 : 0];
      LiveSlot v;
      v.theta = ts.x;
      const double f = ts.y;
      int which = -1;
      double value = 0.0;
      // the qutrit stays in shared memory: a qutrit mutation only needs which / value here
#if ISQ_VAL_PREDRAW
      const int m = g > 0 ? mutate_apply(a, s, md[u], f, v, which, value) : MUT_NONE;
#else
      const int m = g > 0 ? mutate_decide(a, s, g - 1, f, v, which, value) : MUT_NONE;
#endif
      emit_theta(a, t, v.theta);
      a.touch_fbefore[t] = f;
      a.touch_mutated[t] = (uint8_t)((m != MUT_NONE ? 1 : 0) | (m == MUT_QUTRIT ? 2 : 0));
      if (kind < a.n) {
        sm.task[atomicAdd(&sm.ntask, 1)] = (uint16_t)i;
        if (m == MUT_QUTRIT) {
          sm.which[i] = (int8_t)which;
          sm.value[i] = value;
          sm.qq[atomicAdd(&sm.nq, 1)] = (uint16_t)i;
        }
      } else {
        emit_code(a, t, (uint8_t)(3 * a.n + (kind - a.n)));
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < sm.nq; j += kValThreads) {
      const int i = sm.qq[j];
      su3_one_param(sm.which[i], sm.value[i], sm.rec[i].q);
      // the live qutrit for the commit (every touch of the slot holds the same value)
#pragma unroll
      for (int k = 0; k < 3; ++k) a.qlive[3 * (base + i) + k] = sm.rec[i].q[k];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < sm.ntask; k += kValThreads) {
      const int i = sm.task[k];
      const double2* q = sm.rec[i].q;
      double re[3] = {q[0].x, q[1].x, q[2].x};
      double im[3] = {q[0].y, q[1].y, q[2].y};
      emit_code(a, base + i, measure_code<BIG>(a, sm.s[i], g, re, im));
    }
    __syncthreads();
  }
  if (a.peers) __threadfence_system();
}

// world > 1: best circuit of this rank's shard (first index on ties) and its
// gates, packed for the all-gather as [fitness, circuit, L angles, L code bytes].
__global__ void __launch_bounds__(256) qeqea_elite_kernel(QeqeaArgs a) {
  __shared__ double smax[256];
  __shared__ int64_t sarg[256];
  if (a.st->stop) return;
  const int64_t c1 = min(a.P, a.c0 + a.S);
  double m = -1.0;
  int64_t arg = INT64_MAX;
  for (int64_t c = a.c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const double f = a.fitness[c];
    if (f > m) {
      m = f;
      arg = c;
    }
  }
  smax[threadIdx.x] = m;
  sarg[threadIdx.x] = arg;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if (threadIdx.x < off) {
      const double m2 = smax[threadIdx.x + off];
      const int64_t a2 = sarg[threadIdx.x + off];
      if (m2 > smax[threadIdx.x] || (m2 == smax[threadIdx.x] && a2 < sarg[threadIdx.x])) {
        smax[threadIdx.x] = m2;
        sarg[threadIdx.x] = a2;
      }
    }
    __syncthreads();
  }
  const int64_t best = sarg[0];
  // own slot of the elite buffer; peer transport: every rank's copy
  for (int dst = a.peers ? 0 : a.rank; dst < (a.peers ? a.world : a.rank + 1); ++dst) {
    double* e = (a.peers ? a.peers->elite[dst] : a.elite) + (int64_t)a.rank * a.elite_len;
    if (threadIdx.x == 0) {
      e[0] = smax[0];
      e[1] = (double)(best == INT64_MAX ? -1 : best);
    }
    if (best == INT64_MAX) continue;
    uint8_t* codes = reinterpret_cast<uint8_t*>(e + 2 + a.L);
    for (int p = threadIdx.x; p < a.L; p += blockDim.x) {
      e[2 + p] = a.gate_thetas[(best - a.c0) * a.L + p];
      codes[p] = a.gate_codes[(best - a.c0) * a.L + p];
    }
  }
  if (a.peers) __threadfence_system();
}

// Peer transport: this rank's fitness shard into every other rank's fitness
// vector (the all-gather, as direct NVLink stores).
__global__ void qeqea_fitness_broadcast_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  const int64_t n = a.S * (a.world - 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / a.S, c = a.c0 + (i - k * a.S);
    const int dst = (int)(k < a.rank ? k : k + 1);
    a.peers->fitness[dst][c] = a.fitness[c];
  }
  __threadfence_system();
}

// -------------------------------------------------------------- reduce ---

constexpr int kRedThreads = 256;

// Deterministic block partial `part` of (max with first argmax, sum) over
// fitness[0, P); kRedThreads threads, shared scratch of kRedThreads each.
__device__ __forceinline__ void reduce_partial_body(const QeqeaArgs& a, int part, double* smax,
                                                    double* ssum, int64_t* sarg) {
  const int64_t per = (a.P + a.n_parts - 1) / a.n_parts;
  const int64_t lo = (int64_t)part * per;
  const int64_t hi = min(a.P, lo + per);
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  int64_t i = lo + threadIdx.x;
  constexpr int kBatch = 8;  // loads issued together, then folded in index order (same sums)
  for (; i + (kBatch - 1) * kRedThreads < hi; i += kBatch * kRedThreads) {
    double f[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) f[k] = a.fitness[i + k * kRedThreads];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      sum += f[k];
      if (f[k] > m) {
        m = f[k];
        arg = i + k * kRedThreads;
      }
    }
  }
  for (; i < hi; i += kRedThreads) {
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
  for (int off = kRedThreads / 2; off >= 1; off >>= 1) {
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

__global__ void __launch_bounds__(kRedThreads) qeqea_reduce_partials(QeqeaArgs a) {
  if (a.st->stop) return;
  __shared__ double smax[kRedThreads], ssum[kRedThreads];
  __shared__ int64_t sarg[kRedThreads];
  reduce_partial_body(a, blockIdx.x, smax, ssum, sarg);
}

// Final reduction, best-so-far update (strict >, first circuit on ties,
// engine.py:341-343), the generation record, and capture of the new best
// circuit's gates by warp 0.  All threads of the block call it.
// Thread 0: the generation's (max, first argmax, sum) -> best-so-far,
// record; every thread then syncs and warp 0 captures an improved best's
// gates from (codes, thetas) (the circuit-side arrays, or the single-block
// kernel's shared-memory copies).
__device__ __forceinline__ void reduce_final_core(const QeqeaArgs& a, double m, double sum, int64_t arg,
                                                  int* s_improved, int64_t* s_best, const uint8_t* codes,
                                                  const double* thetas) {
  QeqeaDevState* st = a.st;
  if (threadIdx.x == 0) {
    const double mean = sum / (double)a.P;
    st->gen_best = m;
    st->gen_mean = mean;
    const int improved = m > st->best_fitness;
    if (improved) {
      st->best_fitness = m;
      st->best_circuit = arg;
    }
    st->improved = improved;
    GenRecord r;
    r.gen_best = m;
    r.gen_mean = mean;
    r.best_fitness = st->best_fitness;
    r.pad = 0.0;
    const uint64_t ri = st->generation - st->rec_base;
    if (ri < (uint64_t)a.rec_cap) a.records[ri] = r;
    *s_improved = improved;
    *s_best = arg;
  }
  __syncthreads();
  if (*s_improved && threadIdx.x < 32) {
    const int64_t best = *s_best;
    for (int p = threadIdx.x; p < a.L; p += 32) {
      if (a.world == 1) {
        // the generation's gate codes / live angles of every circuit are still
        // in place (do not recompute them from the bank: the commit rewrites it)
        a.best_codes[p] = codes[best * a.L + p];
        a.best_thetas[p] = thetas[best * a.L + p];
      } else {
        // gathered elite record of the rank that scored the best circuit
        const double* e = a.elite + (best / a.S) * a.elite_len;
        a.best_codes[p] = reinterpret_cast<const uint8_t*>(e + 2 + a.L)[p];
        a.best_thetas[p] = e[2 + p];
      }
    }
  }
}

__device__ __forceinline__ void reduce_final_body(const QeqeaArgs& a, int* s_improved, int64_t* s_best) {
  // the partials staged by the whole block (one round trip), then folded by
  // thread 0 in part order (the same result as a serial walk over them)
  __shared__ double s_pm[1024], s_ps[1024];
  __shared__ int64_t s_pa[1024];
  for (int i = threadIdx.x; i < a.n_parts; i += blockDim.x) {
    s_pm[i] = a.part_max[i];
    s_ps[i] = a.part_sum[i];
    s_pa[i] = a.part_arg[i];
  }
  __syncthreads();
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.n_parts; ++i) {
      const double pm = s_pm[i];
      if (pm > m || (pm == m && s_pa[i] < arg)) {
        m = pm;
        arg = s_pa[i];
      }
      sum += s_ps[i];
    }
  }
  reduce_final_core(a, m, sum, arg, s_improved, s_best, a.gate_codes, a.gate_thetas);
}

__global__ void __launch_bounds__(kRedThreads) qeqea_reduce_final(QeqeaArgs a) {
  __shared__ int s_improved;
  __shared__ int64_t s_best;
  if (a.st->stop) return;
  reduce_final_body(a, &s_improved, &s_best);
}

// -------------------------------------------------------------- commit ---

#ifndef ISQ_COMMIT_THREADS
#define ISQ_COMMIT_THREADS 256
#endif
constexpr int kCommitThreads = ISQ_COMMIT_THREADS;
#ifndef ISQ_COMMIT_FULL_GRID
#define ISQ_COMMIT_FULL_GRID 1
#endif

// Elitist accept + table update over the owned touches (engine.py:345-351 +
// 202-222): a slot mutated at g-1 keeps its mutation iff some circuit of
// generation g that touched it beat its slot_max, and slot_max becomes the
// max over its touches (u64 atomicMax; fitness >= 0, so integer order ==
// double order).  The values kernel recorded each touch's starting slot_max
// and pending-mutation flag, so only improving touches do random bank traffic.
// The commit of touch t from its values: `fit` its circuit's fitness, `fb`
// the slot_max it started from, `s` its slot, `mf` its mutation flags,
// `theta` its live angle.
__device__ __forceinline__ void commit_touch_core(const QeqeaArgs& a, int64_t t, double fit, double fb, uint32_t s,
                                                  uint8_t mf, double theta) {
  if (!(fit > fb)) return;
  const int64_t loc = slot_local(a, s);
  if (mf & 2) {
    // qutrit mutation: the live qutrit the values kernel derived (the same
    // value in every touch of the slot, so concurrent stores agree); theta
    // is unchanged by a qutrit mutation (encoding.py:119-132)
    const double2* q = a.qlive + 3 * t;
    double2* r = a.rot[loc].q;
    const double2 q0 = q[0], q1 = q[1], q2 = q[2];
    r[0] = q0;
    r[1] = q1;
    r[2] = q2;
  } else if (mf & 1) {
    // angle mutation: every improving touch holds the same live angle
    // (values kernel), so the idempotent store needs no arbitration
    if (loc < a.Qtloc)
      a.rot[loc].theta = theta;
    else
      a.inter[loc - a.Qtloc].theta = theta;
  }
  atomicMax(reinterpret_cast<unsigned long long*>(smax_ptr(a, loc)),
            (unsigned long long)__double_as_longlong(fit));
}
__device__ __forceinline__ void commit_touch(const QeqeaArgs& a, int64_t t, uint64_t g) {
  const double fit = a.fitness[a.div_Lr.div((uint32_t)t)];
  const double fb = a.touch_fbefore[t];
  if (!(fit > fb)) return;
  commit_touch_core(a, t, fit, fb, a.owner_flats[t], a.touch_mutated[t], a.owner_thetas[t]);
}

__global__ void __launch_bounds__(kCommitThreads) qeqea_commit_table_kernel(QeqeaArgs a, int64_t t1) {
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < t1;
       t += (int64_t)gridDim.x * blockDim.x)
    commit_touch(a, t, g);
}

__device__ __forceinline__ void advance_body(const QeqeaArgs& a) {
  QeqeaDevState* st = a.st;
  st->generation += 1;
  if (st->best_fitness >= a.target_fitness)
    st->stop = 1;
  else if (st->generation >= a.max_generations)
    st->stop = 2;
}

__global__ void qeqea_advance_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  advance_body(a);
}

// ---------------------------------------------------------- population ---

// Per-slot initial bank (init_population, engine.py:105-112; oracle/streams.py
// init_slot): theta = uniform(0, 2pi) and a Box-Muller complex Gaussian qutrit.
__global__ void qeqea_init_kernel(QeqeaArgs a) {
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < a.Qloc;
       loc += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = slot_global(a, loc);
    double theta;
    double2 q[3];
    init_slot_value(a.seed, s, loc < a.Qtloc, theta, q);
    if (loc >= a.Qtloc) {
      a.inter[loc - a.Qtloc].theta = theta;
      a.inter[loc - a.Qtloc].smax = 0.0;
    } else {
      a.rot[loc].theta = theta;
      a.rot[loc].smax = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) a.rot[loc].q[k] = q[k];
    }
  }
}

// Live bank at the current generation (the reference's engine.pop after the
// last step, i.e. committed values with the pending mutation applied), over
// the owned slots in local order (world 1: the reference's flat order).
__global__ void qeqea_live_kernel(QeqeaArgs a, double* theta_out, double2* q_out) {
  const uint64_t g = a.st->generation;
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < a.Qloc;
       loc += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    live_slot(a, slot_global(a, loc), g, v);
    theta_out[loc] = v.theta;
    if (loc < a.Qtloc) {
#pragma unroll
      for (int k = 0; k < 3; ++k) q_out[loc * 3 + k] = v.q[k];
    }
  }
}

// Records <-> the reference's arrays (owned slots, local order): theta[Qloc],
// qamp[3][Qtloc] (axis-major), slot_max[Qloc].
__global__ void qeqea_pack_kernel(QeqeaArgs a, double* theta, double2* qamp, double* smax) {
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < a.Qloc;
       loc += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    const double f = load_committed(a, loc, v);
    theta[loc] = v.theta;
    smax[loc] = f;
    if (loc < a.Qtloc) {
#pragma unroll
      for (int k = 0; k < 3; ++k) qamp[k * a.Qtloc + loc] = v.q[k];
    }
  }
}

__global__ void qeqea_unpack_kernel(QeqeaArgs a, const double* theta, const double2* qamp,
                                    const double* smax) {
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < a.Qloc;
       loc += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    v.theta = theta[loc];
    if (loc < a.Qtloc) {
#pragma unroll
      for (int k = 0; k < 3; ++k) v.q[k] = qamp[k * a.Qtloc + loc];
    }
    store_committed(a, loc, v);
    *smax_ptr(a, loc) = smax ? smax[loc] : 0.0;
  }
}

// Blueprints and gate codes of circuits [c0, c1) at the current generation
// (parity / introspection, world 1; same device functions as the generation).
__global__ void __launch_bounds__(kThreadsPerBlock)
    qeqea_sample_kernel(QeqeaArgs a, int64_t c0, int64_t c1, int64_t* flats_out, uint8_t* codes_out,
                        double* thetas_out) {
  extern __shared__ uint32_t dyn_flats[];
  __shared__ uint64_t blk[kWarpsPerBlock][36];
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* flats = dyn_flats + wib * a.L;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = c0 + (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < c1; c += nwarps) {
    sample_circuit_warp(a, g, c, flats, blk[wib], lane);
    for (int p = lane; p < a.L; p += 32) {
      const int64_t s = flats[p];
      LiveSlot v;
      live_slot(a, s, g, v);
      const int64_t o = (c - c0) * a.L + p;
      flats_out[o] = s;
      codes_out[o] = (uint8_t)slot_gate_code(a, s, g, v);
      thetas_out[o] = v.theta;
    }
  }
}

// --------------------------------------------------- small populations ---

// Launch-bound populations (C1-C3: P*L of a few hundred touches): n whole
// generations in one single-block launch, every phase a block-wide loop over
// the same device bodies the multi-kernel generation uses (identical
// results), separated by __syncthreads.  The generation's intermediates --
// blueprints, gate codes / live angles, starting slot_max and mutation flags
// per touch, fitness -- stay in (dynamic) shared memory: at these sizes a
// phase is a few hundred cycles of work, and reading the previous phase's
// output back through L2 cost about as much again per phase (ncu: ~half the
// warp stall samples of a C1 generation sat on those loads).
struct SmallMirror {
  double* th;       // live angle per touch
  double* fb;       // slot_max the touch started from
  double* fit;      // fitness per circuit
  uint32_t* flats;  // blueprint per touch
  uint8_t* code;    // gate code per touch
  uint8_t* mut;     // mutation flags per touch
};
__host__ __device__ inline size_t small_mirror_bytes(int64_t touches, int64_t P) {
  return (size_t)touches * (8 + 8 + 4 + 1 + 1) + (size_t)P * 8 + 16;
}
__device__ __forceinline__ SmallMirror small_mirror(unsigned char* base, int64_t touches, int64_t P) {
  SmallMirror m;
  m.th = reinterpret_cast<double*>(base);
  m.fb = m.th + touches;
  m.fit = m.fb + touches;
  m.flats = reinterpret_cast<uint32_t*>(m.fit + P);
  m.code = reinterpret_cast<uint8_t*>(m.flats + touches);
  m.mut = m.code + touches;
  return m;
}

// BIG: nMeas > kInversionMaxMeas (numpy's BTPE branch compiled in; without
// it the kernel is 8.5k instead of 19k instructions)
template <int NQ, bool BIG>
__global__ void __launch_bounds__(kRedThreads, 1) qeqea_small_kernel(QeqeaArgs a, int n_gens) {
  using G = Geo<NQ>;
  constexpr int kWarps = kRedThreads / 32;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ FitScratch<NQ, double, kSmallNR> sh[kWarps];
  __shared__ uint64_t blk[kWarps][36];
  __shared__ int s_improved;
  __shared__ int64_t s_best;
  __shared__ double s_m, s_sum;
  __shared__ int64_t s_arg;
  extern __shared__ __align__(16) unsigned char small_dyn[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < G::D * G::D; i += kRedThreads) Ts[i] = a.target[i];
  const int64_t touches = a.P * a.L;
  const SmallMirror mi = small_mirror(small_dyn, touches, a.P);
  for (int it = 0; it < n_gens; ++it) {
    __syncthreads();
    if (a.st->stop) return;  // uniform: written by thread 0 before the barrier
    const uint64_t g = a.st->generation;
    for (int64_t c = wib; c < a.P; c += kWarps) sample_circuit_warp(a, g, c, mi.flats + c * a.L, blk[wib], lane);
    __syncthreads();
    for (int64_t t = threadIdx.x; t < touches; t += kRedThreads) {
      // values (value_touch_from + the measurement), into shared memory
      const uint32_t s = mi.flats[t];
      // the measurement stream's first block depends only on (g, s): start it
      // before the record load and the mutation
      NpStream ms;
      ms.init(a.seed, DOM_MEASURE, g, (uint64_t)s, 0);
      const int64_t kind = slot_kind(a, s);
      if (kind < a.n) ms.prime();
      LiveSlot v;
      const double f = load_committed(a, slot_local(a, s), v);
      int which = -1;
      double value = 0.0;
      const int m = g > 0 ? mutate_decide(a, s, g - 1, f, v, which, value) : MUT_NONE;
      mi.th[t] = v.theta;
      if constexpr (!kFitMulti<NQ>) a.gate_thetas[t] = v.theta;  // FastEval stages gates with cp.async (global)
      mi.fb[t] = f;
      mi.mut[t] = (uint8_t)((m != MUT_NONE ? 1 : 0) | (m == MUT_QUTRIT ? 2 : 0));
      if (kind < a.n) {
        if (m == MUT_QUTRIT) {
          su3_one_param(which, value, v.q);
#pragma unroll
          for (int k = 0; k < 3; ++k) a.qlive[3 * t + k] = v.q[k];
        }
        double re[3] = {v.q[0].x, v.q[1].x, v.q[2].x};
        double im[3] = {v.q[0].y, v.q[1].y, v.q[2].y};
        mi.code[t] = measure_code_on<BIG>(a, s, ms, re, im);
      } else {
        mi.code[t] = (uint8_t)(3 * a.n + (kind - a.n));
      }
      if constexpr (!kFitMulti<NQ>) a.gate_codes[t] = mi.code[t];
    }
    __syncthreads();
    if constexpr (kFitMulti<NQ>)  // n <= 3: plain loads of the gates, from shared memory
      fitness_rows_fast<NQ, double, kSmallNR, true>(a.P, a.L, mi.code, mi.th, Ts, sh, mi.fit, kWarps, nullptr,
                                                    nullptr, small_cpw<NQ>(a.P, kWarps));
    else
      fitness_rows_fast<NQ, double, kSmallNR, true>(a.P, a.L, a.gate_codes, a.gate_thetas, Ts, sh, mi.fit, kWarps,
                                                    nullptr, nullptr, small_cpw<NQ>(a.P, kWarps));
    __syncthreads();
    // reductions: the same pairwise tree as reduce_partial_body (P <= 32: its
    // upper levels only add zeros), as shuffles
    if (wib == 0) {
      double m = -1.0, sum = 0.0;
      int64_t arg = INT64_MAX;
      if (lane < a.P) {
        m = sum = mi.fit[lane];
        arg = lane;
        a.fitness[lane] = m;  // host readback (isq_qeqea_fitness)
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double m2 = __shfl_down_sync(0xffffffffu, m, off);
        const int64_t a2 = __shfl_down_sync(0xffffffffu, arg, off);
        const double s2 = __shfl_down_sync(0xffffffffu, sum, off);
        if (m2 > m || (m2 == m && a2 < arg)) {
          m = m2;
          arg = a2;
        }
        sum += s2;
      }
      if (lane == 0) {
        s_m = m;
        s_sum = sum;
        s_arg = arg;
      }
    }
    __syncthreads();
    reduce_final_core(a, s_m, s_sum, s_arg, &s_improved, &s_best, mi.code, mi.th);
    __syncthreads();
    for (int64_t t = threadIdx.x; t < touches; t += kRedThreads)
      commit_touch_core(a, t, mi.fit[a.div_Lr.div((uint32_t)t)], mi.fb[t], mi.flats[t], mi.mut[t], mi.th[t]);
    __syncthreads();
    if (threadIdx.x == 0) advance_body(a);
  }
}

// Single-rank populations of at most one fitness round (P <= 8 warps) and this
// many touches run qeqea_small_kernel; larger launch-bound ones run as a CUDA
// graph of the multi-kernel generation (its fitness kernel spreads over SMs).
constexpr int64_t kSmallTouches = 1 << 12;
constexpr int64_t kSmallPop = kRedThreads / 32;

// ------------------------------------------------------------ launchers ---

static int blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}



isq_status qeqea_configure_device() {
  // > 48 KB of dynamic shared memory needs the opt-in (per device)
  ISQ_CUDA_TRY(cudaFuncSetAttribute((const void*)qeqea_values_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ValuesShared)));
  ISQ_CUDA_TRY(cudaFuncSetAttribute((const void*)qeqea_values_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(ValuesShared)));
  return ISQ_OK;
}

static cudaError_t launch_values(const QeqeaArgs& a, int64_t t1, cudaStream_t s) {
#if ISQ_VAL_GRID_TILES
  // one block per tile: the hardware scheduler balances the tiles over the
  // SMs (a grid-stride loop over 16 blocks per SM left a partial last wave:
  // 3.49 -> 3.35 ms at C5)
  int64_t nb = (t1 + kValTile - 1) / kValTile;
  if (nb > ISQ_VAL_GRID_CAP) nb = ISQ_VAL_GRID_CAP;
  if (nb < 1) nb = 1;
  if (a.n_meas > kInversionMaxMeas)
    qeqea_values_kernel<true><<<(unsigned)nb, kValThreads, sizeof(ValuesShared), s>>>(a, t1);
  else
    qeqea_values_kernel<false><<<(unsigned)nb, kValThreads, sizeof(ValuesShared), s>>>(a, t1);
#else
  if (a.n_meas > kInversionMaxMeas)
    qeqea_values_kernel<true><<<blocks_for(t1, kValThreads), kValThreads, sizeof(ValuesShared), s>>>(a, t1);
  else
    qeqea_values_kernel<false><<<blocks_for(t1, kValThreads), kValThreads, sizeof(ValuesShared), s>>>(a, t1);
#endif
  return cudaGetLastError();
}

isq_status qeqea_launch_prepare(const QeqeaArgs& a, cudaStream_t s) {
  if (a.c0 < a.P) {
#if ISQ_SAMPLE_FULL_GRID
    // one warp task per warp (the hardware balances them; a persistent grid
    // left ~8 % of the warps a fourth task)
    const int64_t tasks = (a.S + kSampleRun - 1) / kSampleRun;
    const int grid_s = (int)((tasks + kWarpsPerBlock - 1) / kWarpsPerBlock);
#else
    const int grid_s = persistent_grid((const void*)qeqea_sample_flats_kernel, 0, (a.S + kSampleRun - 1) / kSampleRun);
#endif
    qeqea_sample_flats_kernel<<<grid_s, kThreadsPerBlock, 0, s>>>(a);
  }
  if (a.world > 1) {
    qeqea_route_kernel<<<blocks_for(a.S * a.L, 256), 256, 0, s>>>(a);
  } else {
    ISQ_CUDA_TRY(launch_values(a, a.P * a.L, s));
  }
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_values(const QeqeaArgs& a, cudaStream_t s) {
  if (a.world > 1) {
    ISQ_CUDA_TRY(launch_values(a, a.world * a.S * a.Lr, s));
  }
  return ISQ_OK;
}

isq_status qeqea_launch_score(const QeqeaArgs& a, cudaStream_t s) {
  if (a.world > 1) qeqea_unroute_kernel<<<blocks_for(a.S * a.L, 256), 256, 0, s>>>(a);
  const int64_t count = a.P - a.c0 < a.S ? a.P - a.c0 : a.S;
  if (count > 0) {
    isq_status st = launch_fitness_batch_stoppable(a.n, a.L, count, a.gate_codes, a.gate_thetas,
                                                   reinterpret_cast<const double*>(a.target),
                                                   a.fitness + a.c0, &a.st->stop, s, 0, a.precision, nullptr,
                                                   ISQ_FIT_DYNAMIC ? &a.st->fit_next : nullptr);
    if (st != ISQ_OK) return st;
  }
  if (a.world > 1) {
    if (a.peers) qeqea_fitness_broadcast_kernel<<<blocks_for(a.S * (a.world - 1), 256), 256, 0, s>>>(a);
    qeqea_elite_kernel<<<1, 256, 0, s>>>(a);
  }
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_eval(const QeqeaArgs& a, cudaStream_t s) {
  isq_status st = qeqea_launch_prepare(a, s);
  if (st != ISQ_OK) return st;
  return qeqea_launch_score(a, s);
}

isq_status qeqea_launch_finish(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_reduce_partials<<<a.n_parts, kRedThreads, 0, s>>>(a);
  qeqea_reduce_final<<<1, kRedThreads, 0, s>>>(a);
  const int64_t t1 = a.world * a.S * a.Lr;
#if ISQ_COMMIT_FULL_GRID
  {
    // one touch per thread (no grid-stride loop): no partial last wave
    int64_t nb = (t1 + kCommitThreads - 1) / kCommitThreads;
    if (nb < 1) nb = 1;
    qeqea_commit_table_kernel<<<(unsigned)nb, kCommitThreads, 0, s>>>(a, t1);
  }
#else
  qeqea_commit_table_kernel<<<blocks_for(t1, kCommitThreads), kCommitThreads, 0, s>>>(a, t1);
#endif
  qeqea_advance_kernel<<<1, 1, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

bool qeqea_small(const QeqeaArgs& a) {
  return a.world == 1 && a.precision == ISQ_PRECISION_FP64 && a.n <= ISQ_MAX_FAST_WIRES && a.P <= kSmallPop &&
         a.P * a.L <= kSmallTouches;
}

isq_status qeqea_launch_small(const QeqeaArgs& a, int n_gens, cudaStream_t s) {
  if (a.world != 1 || a.precision != ISQ_PRECISION_FP64) {
    set_error("the fused single-block generation is single-rank fp64 only");
    return ISQ_ERR_CONFIG;
  }
  if (a.P > 32 || a.P * a.L > kSmallTouches) {
    set_error("the fused single-block generation needs sizeOfPopulation <= 32 and P * L <= 4096");
    return ISQ_ERR_UNSUPPORTED;
  }
  const size_t dyn = small_mirror_bytes(a.P * a.L, a.P);
  const bool big = a.n_meas > kInversionMaxMeas;
  auto go = [&](auto kernel) -> isq_status {
    static bool sized[6][2] = {};
    if (!sized[a.n][big]) {  // the shared-memory copies of the generation exceed the 48 KB default
      ISQ_CUDA_TRY(cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)small_mirror_bytes(kSmallTouches, 32)));
      sized[a.n][big] = true;
    }
    kernel<<<1, kRedThreads, dyn, s>>>(a, n_gens);
    ISQ_CUDA_TRY(cudaGetLastError());
    return ISQ_OK;
  };
  switch (a.n) {
    case 2: return big ? go(qeqea_small_kernel<2, true>) : go(qeqea_small_kernel<2, false>);
    case 3: return big ? go(qeqea_small_kernel<3, true>) : go(qeqea_small_kernel<3, false>);
    case 4: return big ? go(qeqea_small_kernel<4, true>) : go(qeqea_small_kernel<4, false>);
    case 5: return big ? go(qeqea_small_kernel<5, true>) : go(qeqea_small_kernel<5, false>);
    default:
      set_error("the fused single-block generation supports numberOfWires <= 5");
      return ISQ_ERR_UNSUPPORTED;
  }
}

isq_status qeqea_launch_init(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_init_kernel<<<blocks_for(a.Qloc, 256), 256, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_pack(const QeqeaArgs& a, double* theta, double* qamp, double* smax,
                             cudaStream_t s) {
  qeqea_pack_kernel<<<blocks_for(a.Qloc, 256), 256, 0, s>>>(a, theta, reinterpret_cast<double2*>(qamp), smax);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_unpack(const QeqeaArgs& a, const double* theta, const double* qamp,
                               const double* smax, cudaStream_t s) {
  qeqea_unpack_kernel<<<blocks_for(a.Qloc, 256), 256, 0, s>>>(
      a, theta, reinterpret_cast<const double2*>(qamp), smax);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_live(const QeqeaArgs& a, double* theta_out, double* q_out, cudaStream_t s) {
  qeqea_live_kernel<<<blocks_for(a.Qloc, 256), 256, 0, s>>>(a, theta_out, reinterpret_cast<double2*>(q_out));
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_sample(const QeqeaArgs& a, int64_t c0, int64_t c1, int64_t* flats,
                               uint8_t* codes, double* thetas, cudaStream_t s) {
  if (c1 <= c0) return ISQ_OK;
  const size_t dyn = (size_t)kWarpsPerBlock * a.L * sizeof(uint32_t);
  const int grid = persistent_grid((const void*)qeqea_sample_kernel, dyn, c1 - c0);
  qeqea_sample_kernel<<<grid, kThreadsPerBlock, dyn, s>>>(a, c0, c1, flats, codes, thetas);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

}  // namespace isq

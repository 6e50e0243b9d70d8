// Device state and per-slot helpers of the QEQEA generation loop.
//
// Reference: QeqeaEngine.step (engine.py:318-361).  The bank lives in HBM
// indexed by the flat slot index of Eq. 9 (engine.py:82-87), as arrays of
// aligned per-slot records - every generation touches O(P*L) slots at random,
// so one record per slot is one DRAM transaction instead of one per field:
//
//   rot[Qt]     64 B  {q0, q1, q2 (complex), theta, slot_max}   rotation region
//   inter[Q-Qt] 16 B  {theta, slot_max}                          interaction region
//
// slot_max is SegmentFitnessTable.slot_max (engine.py:202-222), updated with a
// 64-bit atomicMax (fitness >= 0, so integer order == double order).  The host
// sees the reference's arrays (thetas[Q], qutrits[Qt,3], slot_max[Q]) through
// pack/unpack kernels.
//
// Lazy mutation.  The reference mutates ~p_mut of all Q slots
// at the end of every generation and reverts the un-improved ones at the next
// (engine.py:345-352).  Because every draw comes from a per-(generation, slot)
// counter stream, the live value of slot s at generation g is a pure function
//     live_g(s) = mutate_{g-1}(committed(s), slot_max(s), Philox(g-1, s))
// so generation g computes it on the fly for the O(P*L) slots its circuits
// touch, and commits it only for touched, improved, mutated slots.  No pass
// over the Q-slot bank is ever made (C5: Q = 1.0e9).
#pragma once
#include <cstdint>

#include "np_random.cuh"

namespace isq {

struct QeqeaDevState {
  uint64_t generation;   // generations completed (engine.generation)
  uint64_t rec_base;     // generation at the start of the current host batch
  double best_fitness;   // engine.best_fitness
  int64_t best_circuit;  // circuit index whose gates are being captured this generation (-1 none)
  int32_t stop;          // 0 running, 1 target-reached, 2 generation-limit
  int32_t improved;      // best improved in the generation being finished
  double gen_best, gen_mean;
  unsigned long long fit_next;  // next circuit batch of the fitness launch (dynamic scheduling)
};

struct GenRecord {
  double gen_best;
  double gen_mean;
  double best_fitness;
  double pad;
};

struct alignas(64) RotRec {
  double2 q[3];
  double theta;
  double smax;
};
struct alignas(16) IntRec {
  double theta;
  double smax;
};

constexpr int kMaxWorld = 64;
constexpr uint32_t kNoSlot = 0xffffffffu;  // padding touch of a padding circuit

// NVLink peer-memory transport (world > 1, isq_qeqea_set_peers): the
// exchange buffers of every rank, mapped into this process (own rank: local).
struct PeerTable {
  uint32_t* recv_flats[kMaxWorld];  // owner o: touches of its positions, from every circuit rank
  uint8_t* recv_codes[kMaxWorld];   // circuit rank j: gate codes of its circuits, from every owner
  double* recv_thetas[kMaxWorld];
  double* fitness[kMaxWorld];       // every rank: the whole fitness vector
  double* elite[kMaxWorld];         // every rank: all shard elites
};

// Device view of one engine handle.  Multi-GPU layout (population sharding,
// DESIGN.md §8): rank r scores circuits [c0, c0 + S) and owns the bank slots
// of positions [p_lo, p_lo + Lr) (every slot kind and individual); a slot's
// position is fixed by Eq. 9, so the touches of position p always go to the
// same owner.  World 1: c0 = 0, S = P, p_lo = 0, Lr = L, and the owner-side
// touch arrays alias the circuit-side ones.
// Division of 32-bit unsigned values by a runtime-invariant divisor d >= 1:
// q = (mulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1
// (Granlund & Montgomery), exact for every n < 2^32.  Slot, touch and
// circuit indices are all below 2^32 (slots are uint32).
struct FastDiv {
  uint32_t d, m;
  int l;
  __host__ void init(uint32_t dd) {
    d = dd;
    l = 0;
    while ((1ull << l) < dd) ++l;
    m = (uint32_t)((((1ull << l) - dd) << 32) / dd + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, m) + n) >> l);
  }
};

struct QeqeaArgs {
  // configuration (engine.py:33-43)
  int n, L;
  int64_t P, K, Q, Qt;
  double p_mut, mutation_range, target_fitness;
  int n_meas;
  uint64_t max_generations;
  uint64_t seed;
  int precision;   // fitness arithmetic: ISQ_PRECISION_FP64 / _FP32
  // sharding
  int world, rank;
  int64_t S;       // circuits per rank (padded: world * S >= P)
  int64_t c0;      // first circuit of this rank
  int p_lo, Lr;    // owned positions
  int p_bounds[kMaxWorld + 1];  // owner o holds positions [p_bounds[o], p_bounds[o + 1])
  FastDiv div_L, div_LP, div_Lr, div_S;  // by L, L * P (slot -> kind), Lr, S
  int64_t Qloc, Qtloc;  // owned slots / owned rotation-region slots
  // bank (owned slots, local index, see slot_local)
  RotRec* rot;     // Qtloc records
  IntRec* inter;   // Qloc - Qtloc records
  // circuit side (this rank's S circuits x L positions)
  double* fitness;       // world * S: the whole (gathered) fitness vector
  uint32_t* flats;       // S * L sampled slots
  uint8_t* gate_codes;   // S * L gate codes (fitness input)
  double* gate_thetas;   // S * L live angles
  // owner side (world * S circuits x Lr owned positions, row = global circuit)
  uint32_t* owner_flats;    // touches of the owned slots
  uint8_t* owner_codes;     // their gate codes / live angles (sent back to the circuit ranks)
  double* owner_thetas;
  double* touch_fbefore;    // slot_max each touch started the generation from
  uint8_t* touch_mutated;   // bit 0 pending mutation, bit 1 it is a qutrit mutation
  double2* qlive;           // 3 per owned touch: the live qutrit of a qutrit-mutated touch (values
                            // kernel), so the commit stores it without re-deriving it
  // world > 1 exchange buffers (send side of flats, receive side of codes / angles)
  uint32_t* send_flats;     // S * L, grouped by owner
  uint8_t* recv_codes;      // S * L, grouped by owner
  double* recv_thetas;
  double* elite;            // world * elite_len: per-rank shard best (fitness, circuit, L angles, L codes)
  int elite_len;
  const PeerTable* peers;   // device table; non-null: the producing kernels store into the
                            // consuming ranks' buffers directly (no all-to-all / all-gather)
  QeqeaDevState* st;
  GenRecord* records;
  uint8_t* best_codes;   // L
  double* best_thetas;   // L
  const double2* target; // D * D
  // reduction scratch
  double* part_max;
  double* part_sum;
  int64_t* part_arg;
  int n_parts;
  int rec_cap;  // capacity of `records`
};

// Eq. 9 flat index s = (kind P + i) L + p  <->  owned local index (kind P + i) Lr + (p - p_lo).
__host__ __device__ __forceinline__ int64_t slot_local(const QeqeaArgs& a, int64_t s) {
#ifdef __CUDA_ARCH__
  const int64_t ki = a.div_L.div((uint32_t)s);
#else
  const int64_t ki = s / a.L;
#endif
  return ki * a.Lr + (s - ki * a.L - a.p_lo);
}
// Slot kind (rotation wire k < n, else interaction pair k - n) of slot s.
__device__ __forceinline__ int64_t slot_kind(const QeqeaArgs& a, uint32_t s) { return a.div_LP.div(s); }
__host__ __device__ __forceinline__ int64_t slot_global(const QeqeaArgs& a, int64_t loc) {
  const int64_t ki = loc / a.Lr;
  return ki * a.L + a.p_lo + (loc - ki * a.Lr);
}

constexpr double kTwoPiD = 6.283185307179586;   // encoding.py:13 TWO_PI = 2.0 * math.pi
constexpr double kHalfPiD = 1.5707963267948966;  // math.pi / 2

// Python / numpy float remainder with the sign of the divisor (x % m, m > 0).
__device__ __forceinline__ double py_mod(double x, double m) {
  // |x| < 2m (an angle in [0, m) plus one bounded step): fmod is x, or x - m,
  // which is exact there (Sterbenz); anything else takes the general path
  if (x > 0.0 && x < m) return x;
  if (x >= m && x < 2.0 * m) return __dsub_rn(x, m);
  double r = fmod(x, m);
  if (r != 0.0) {
    if (r < 0.0) r = __dadd_rn(r, m);
  } else {
    r = 0.0;
  }
  return r;
}

struct LiveSlot {
  double theta;
  double2 q[3];
};

__device__ __forceinline__ double* smax_ptr(const QeqeaArgs& a, int64_t loc) {
  return loc < a.Qtloc ? &a.rot[loc].smax : &a.inter[loc - a.Qtloc].smax;
}

// Committed value of the owned slot `loc` (one 64 B or 16 B record load); returns slot_max.
__device__ __forceinline__ double load_committed(const QeqeaArgs& a, int64_t loc, LiveSlot& v) {
  if (loc < a.Qtloc) {
    const double2* r = reinterpret_cast<const double2*>(a.rot + loc);
    v.q[0] = r[0];
    v.q[1] = r[1];
    v.q[2] = r[2];
    const double2 ts = r[3];
    v.theta = ts.x;
    return ts.y;
  }
  const double2 ts = *reinterpret_cast<const double2*>(a.inter + (loc - a.Qtloc));
  v.theta = ts.x;
  return ts.y;
}

__device__ __forceinline__ void store_committed(const QeqeaArgs& a, int64_t loc, const LiveSlot& v) {
  if (loc < a.Qtloc) {
    double2* r = reinterpret_cast<double2*>(a.rot + loc);
    r[0] = v.q[0];
    r[1] = v.q[1];
    r[2] = v.q[2];
    a.rot[loc].theta = v.theta;
  } else {
    a.inter[loc - a.Qtloc].theta = v.theta;
  }
}

// encoding.py:119-132 with exactly one non-zero SU(3) parameter (encoding.py:87-116):
// theta1/2/3 are real Givens rotations on axes (0,1)/(0,2)/(1,2), phi1/phi2 are
// diagonal phases, phi3..phi5 leave the state unchanged; then renormalise.
__device__ __forceinline__ void su3_one_param(int which, double v, double2 q[3]) {
  double2 o0 = q[0], o1 = q[1], o2 = q[2];
  if (which < 3) {
    double s, c;
    sincos(v, &s, &c);
    if (which == 0) {  // [[c, s, 0], [-s, c, 0], [0, 0, 1]]
      o0 = make_double2(c * q[0].x + s * q[1].x, c * q[0].y + s * q[1].y);
      o1 = make_double2(c * q[1].x - s * q[0].x, c * q[1].y - s * q[0].y);
    } else if (which == 1) {  // [[c, 0, s], [0, 1, 0], [-s, 0, c]]
      o0 = make_double2(c * q[0].x + s * q[2].x, c * q[0].y + s * q[2].y);
      o2 = make_double2(c * q[2].x - s * q[0].x, c * q[2].y - s * q[0].y);
    } else {  // [[1, 0, 0], [0, c, -s], [0, s, c]]
      o1 = make_double2(c * q[1].x - s * q[2].x, c * q[1].y - s * q[2].y);
      o2 = make_double2(s * q[1].x + c * q[2].x, s * q[1].y + c * q[2].y);
    }
  } else if (which < 5) {
    double s, c;
    sincos(v, &s, &c);
    // phi1: diag(e^{iv}, 1, e^{-iv});  phi2: diag(1, e^{iv}, e^{-iv})
    double2& up = (which == 3) ? o0 : o1;
    const double2 x = (which == 3) ? q[0] : q[1];
    up = make_double2(c * x.x - s * x.y, c * x.y + s * x.x);
    o2 = make_double2(c * q[2].x + s * q[2].y, c * q[2].y - s * q[2].x);
  }
  const double nrm = sqrt((o0.x * o0.x + o1.x * o1.x + o2.x * o2.x) +
                          (o0.y * o0.y + o1.y * o1.y + o2.y * o2.y));
  q[0] = make_double2(o0.x / nrm, o0.y / nrm);
  q[1] = make_double2(o1.x / nrm, o1.y / nrm);
  q[2] = make_double2(o2.x / nrm, o2.y / nrm);
}

// mutate_population's per-slot body (engine.py:244-262) for generation `mg`
// on stream (seed, DOM_MUTATE, mg, s): returns true when the slot was
// mutated (masked and slot_max < 1) and applies the mutation to v.
// Draw layout of the first block: w0 mask, w1 coin, w2 integers(8) (low
// u32) or the angle sign, w3 the SU(3) parameter value.
enum : int { MUT_NONE = 0, MUT_ANGLE = 1, MUT_QUTRIT = 2 };

// The draw-dependent part of the per-slot mutation: the angle step is applied
// to v.theta; a qutrit mutation is returned as (which, value) for
// su3_one_param, so a caller can run those (5 % of slots, costly and
// divergent) compacted.
// The draws of slot s's mutation stream (generation mg), which depend on
// nothing but the stream key, so a caller can compute them while the slot's
// record is still in flight: bit 0 masked (random() < p_mut), bit 1 coin,
// bit 2 angle sign (random() < 0.5), bits 8..10 integers(8); d3 the uniform's
// double.
struct MutDraw {
  uint32_t bits;
  double d3;
};
__device__ __forceinline__ MutDraw mutate_draw(const QeqeaArgs& a, int64_t s, uint64_t mg) {
  uint64_t w[4];
  stream_block(a.seed, DOM_MUTATE, mg, (uint64_t)s, 0, 1, w);
  MutDraw d;
  d.bits = (u64_to_double(w[0]) < a.p_mut ? 1u : 0u) | (u64_to_double(w[1]) < 0.5 ? 2u : 0u) |
           (u64_to_double(w[2]) < 0.5 ? 4u : 0u) | (((uint32_t)(w[2] & 0xffffffffULL) >> 29) << 8);
  d.d3 = u64_to_double(w[3]);
  return d;
}
__device__ __forceinline__ int mutate_apply(const QeqeaArgs& a, int64_t s, const MutDraw& d, double f,
                                            LiveSlot& v, int& which, double& value) {
  if (!(d.bits & 1u)) return MUT_NONE;  // random() >= p_mut
  if (!(f < 1.0)) return MUT_NONE;
  const bool coin = (d.bits & 2u) != 0;
  const double omf = __dsub_rn(1.0, f);
  if (coin && s < a.Qt) {
    which = (int)((d.bits >> 8) & 7u);                     // Lemire, bound 8
    const double range = which < 3 ? kHalfPiD : kTwoPiD;  // encoding.py:23
    value = __dadd_rn(0.0, __dmul_rn(__dmul_rn(range, omf), d.d3));
    return MUT_QUTRIT;
  }
  const double sign = (d.bits & 4u) ? 1.0 : -1.0;  // encoding.py:51
  const double step = __dmul_rn(__dmul_rn(sign, omf), a.mutation_range);
  v.theta = py_mod(__dadd_rn(v.theta, step), kTwoPiD);
  return MUT_ANGLE;
}
__device__ __forceinline__ int mutate_decide(const QeqeaArgs& a, int64_t s, uint64_t mg, double f,
                                             LiveSlot& v, int& which, double& value) {
  return mutate_apply(a, s, mutate_draw(a, s, mg), f, v, which, value);
}

__device__ __forceinline__ bool mutate_slot(const QeqeaArgs& a, int64_t s, uint64_t mg, double f,
                                            LiveSlot& v, bool* qutrit_path = nullptr) {
  int which = 0;
  double value = 0.0;
  const int m = mutate_decide(a, s, mg, f, v, which, value);
  if (qutrit_path) *qutrit_path = m == MUT_QUTRIT;
  if (m == MUT_QUTRIT) su3_one_param(which, value, v.q);
  return m != MUT_NONE;
}

// Initial value of slot s (init_population, engine.py:105-112; oracle/streams.py
// init_slot): theta = uniform(0, 2pi) from block 1 of stream (seed, DOM_INIT, 0,
// s), and for rotation-region slots a normalised complex Gaussian qutrit by
// Box-Muller from the next six uniforms.
__device__ __forceinline__ void init_slot_value(uint64_t seed, int64_t s, bool with_qutrit, double& theta,
                                                double2 q[3]) {
  uint64_t w0[4], w1[4];
  stream_block(seed, DOM_INIT, 0, (uint64_t)s, 0, 1, w0);
  theta = __dadd_rn(0.0, __dmul_rn(kTwoPiD, u64_to_double(w0[0])));
  if (!with_qutrit) return;
  stream_block(seed, DOM_INIT, 0, (uint64_t)s, 0, 2, w1);
  const uint64_t u[6] = {w0[1], w0[2], w0[3], w1[0], w1[1], w1[2]};
  double re[3], im[3], nn = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double u1 = u64_to_double(u[2 * k]), u2 = u64_to_double(u[2 * k + 1]);
    const double r = sqrt(-2.0 * log(1.0 - u1));
    double sn, cs;
    sincos(kTwoPiD * u2, &sn, &cs);
    re[k] = r * cs;
    im[k] = r * sn;
    nn += re[k] * re[k] + im[k] * im[k];
  }
  const double nrm = sqrt(nn);
#pragma unroll
  for (int k = 0; k < 3; ++k) q[k] = make_double2(re[k] / nrm, im[k] / nrm);
}

// Live value of the (owned) slot s during generation g (committed value plus
// the pending mutation drawn at the end of generation g-1).
__device__ __forceinline__ void live_slot(const QeqeaArgs& a, int64_t s, uint64_t g, LiveSlot& v,
                                          bool* mutated = nullptr) {
  const double f = load_committed(a, slot_local(a, s), v);
  bool m = false;
  if (g > 0) m = mutate_slot(a, s, g - 1, f, v);
  if (mutated) *mutated = m;
}

// Gate code of slot s with its measured axis (SegmentBank.descriptor, engine.py:134-146;
// construct_segments, engine.py:167-170).
__device__ __forceinline__ int slot_gate_code(const QeqeaArgs& a, int64_t s, uint64_t g,
                                              const LiveSlot& v) {
  const int64_t kind = slot_kind(a, (uint32_t)s);
  if (kind < a.n) {
    NpStream st;
    st.init(a.seed, DOM_MEASURE, g, (uint64_t)s, 0);
    double re[3] = {v.q[0].x, v.q[1].x, v.q[2].x};
    double im[3] = {v.q[0].y, v.q[1].y, v.q[2].y};
    bool ok = true;
    const int axis = measure_axis(re, im, a.n_meas, st, &ok);
    return 3 * (int)kind + axis;
  }
  return 3 * a.n + (int)(kind - a.n);
}

// sample_circuit (engine.py:174-184) for circuit c at generation g on stream
// (seed, DOM_SAMPLE, g, c): integers(P, size=L) then integers(K, size=L),
// flat = kind*L*P + individual*L + position.  Warp-cooperative: per chunk of
// 32 positions the (at most 9) distinct Philox blocks holding their u32 draws
// are computed once by lanes 0..8 into `blk` (shared, 9*4 words) and every
// lane takes its two draws from there (numpy consumes u32 halves low-first).
// If any draw would be rejected by numpy's Lemire sampler, lane 0 replays the
// whole circuit sequentially.  Writes flats[0..L).
__device__ __forceinline__ void sample_circuit_warp(const QeqeaArgs& a, uint64_t g, int64_t c,
                                                    uint32_t* flats, uint64_t* blk, int lane) {
  const int L = a.L;
  const uint32_t rngP = (uint32_t)(a.P - 1), rngK = (uint32_t)(a.K - 1);
  const int offk = (a.P == 1) ? 0 : L;  // integers(1, ...) consumes no draws
  bool reject = false;
  for (int base = 0; base < L; base += 32) {
    const int ib0 = base >> 3;            // first block (0-based) of the individual draws
    const int kb0 = (offk + base) >> 3;   // first block of the kind draws
    if (lane < 9) {
      const int b = lane < 4 ? ib0 + lane : kb0 + (lane - 4);
      uint64_t w[4];
      stream_block(a.seed, DOM_SAMPLE, g, (uint64_t)c, 0, (uint64_t)b + 1, w);
#pragma unroll
      for (int k = 0; k < 4; ++k) blk[lane * 4 + k] = w[k];
    }
    __syncwarp();
    const int p = base + lane;
    if (p < L) {
      uint32_t ind = 0;
      if (a.P > 1) {
        const uint64_t word = blk[((p >> 3) - ib0) * 4 + ((p & 7) >> 1)];
        const uint32_t u = (p & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
        reject |= lemire_rejects(u, rngP);
        ind = lemire_value(u, rngP);
      }
      const int uk = offk + p;
      const uint64_t word = blk[(4 + (uk >> 3) - kb0) * 4 + ((uk & 7) >> 1)];
      const uint32_t u = (uk & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
      reject |= lemire_rejects(u, rngK);
      const uint32_t kind = lemire_value(u, rngK);
      flats[p] = (uint32_t)((int64_t)kind * L * a.P + (int64_t)ind * L + p);
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, reject)) {
    if (lane == 0) {
      NpStream st;
      st.init(a.seed, DOM_SAMPLE, g, (uint64_t)c, 0);
      for (int p = 0; p < L; ++p) flats[p] = (uint32_t)(st.integers(a.P) * L + p);
      for (int p = 0; p < L; ++p) flats[p] += (uint32_t)(st.integers(a.K) * L * a.P);
    }
    __syncwarp();
  }
}

// Lane-parallel sampling of several short circuits at once (2L u32 draws in
// B = ceil(2L / 8) Philox blocks, B <= 32, i.e. L <= 128): every lane computes
// one (circuit, block) pair, so 32 / B circuits share one round and all lanes
// run Philox (sample_circuit_warp keeps 9 of 32 lanes busy).  Same draws, same
// Lemire rejection replay, same flats as sample_circuit_warp.
// blk: 32 x 4 words of shared memory per warp.
__device__ __forceinline__ int sample_blocks_per_circuit(const QeqeaArgs& a) {
  const int draws = (a.P > 1 ? a.L : 0) + a.L;
  return (draws + 7) >> 3;
}

// `blk`: kSampleIlp * 128 u64 per warp.  Each lane computes kSampleIlp
// independent Philox blocks per round (interleaved: the rounds' dependent
// multiply chains overlap).  Measured with 16-circuit warp tasks, C4 / C5
// generations: 1 -> 2.97k gen/s / 15.13 ms (1 with 64-circuit tasks: 2.89k /
// 15.16), 3 -> 2.98k / 15.09, 4 -> 2.98k / 15.09.
#ifndef ISQ_SAMPLE_ILP
#define ISQ_SAMPLE_ILP 3
#endif
constexpr int kSampleIlp = ISQ_SAMPLE_ILP;
__device__ __forceinline__ void sample_circuits_batched(const QeqeaArgs& a, uint64_t g, int64_t c0, int64_t c1,
                                                        uint32_t* flats, uint64_t* blk, int lane) {
  const int L = a.L;
  const int B = sample_blocks_per_circuit(a);
  const int cpr = 32 / B * kSampleIlp;  // circuits per round
  const uint32_t rngP = (uint32_t)(a.P - 1), rngK = (uint32_t)(a.K - 1);
  const int offk = (a.P == 1) ? 0 : L;
  for (int64_t cb = c0; cb < c1; cb += cpr) {
    {
      uint64_t w[kSampleIlp][4];
#pragma unroll
      for (int h = 0; h < kSampleIlp; ++h) {  // block slot lane + 32 h (always computed: straight-line code)
        const int ci = (lane / B) + h * (32 / B), b = lane - (lane / B) * B;
        stream_block(a.seed, DOM_SAMPLE, g, (uint64_t)(cb + ci), 0, (uint64_t)b + 1, w[h]);
      }
#pragma unroll
      for (int h = 0; h < kSampleIlp; ++h) {
        const int ci = (lane / B) + h * (32 / B), b = lane - (lane / B) * B;
        if (lane / B < 32 / B && cb + ci < c1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) blk[(ci * B + b) * 4 + k] = w[h][k];
        }
      }
    }
    __syncwarp();
    const int nc = (int)min((int64_t)cpr, c1 - cb);
    for (int ci = 0; ci < nc; ++ci) {
      const uint64_t* cb_blk = blk + ci * B * 4;
      bool reject = false;
      for (int p = lane; p < L; p += 32) {
        uint32_t ind = 0;
        if (a.P > 1) {
          const uint64_t word = cb_blk[(p >> 3) * 4 + ((p & 7) >> 1)];
          const uint32_t u = (p & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
          reject |= lemire_rejects(u, rngP);
          ind = lemire_value(u, rngP);
        }
        const int uk = offk + p;
        const uint64_t word = cb_blk[(uk >> 3) * 4 + ((uk & 7) >> 1)];
        const uint32_t u = (uk & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
        reject |= lemire_rejects(u, rngK);
        const uint32_t kind = lemire_value(u, rngK);
        flats[(cb + ci - c0) * L + p] = (uint32_t)((int64_t)kind * L * a.P + (int64_t)ind * L + p);
      }
      if (__any_sync(0xffffffffu, reject)) {  // numpy's Lemire rejected a draw: replay the stream
        __syncwarp();
        if (lane == 0) {
          uint32_t* f = flats + (cb + ci - c0) * L;
          NpStream st;
          st.init(a.seed, DOM_SAMPLE, g, (uint64_t)(cb + ci), 0);
          for (int p = 0; p < L; ++p) f[p] = (uint32_t)(st.integers(a.P) * L + p);
          for (int p = 0; p < L; ++p) f[p] += (uint32_t)(st.integers(a.K) * L * a.P);
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace isq

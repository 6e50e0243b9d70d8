// Device state and per-slot helpers of the QEQEA generation loop.
//
// Reference: QeqeaEngine.step (engine.py:318-361).  The bank lives in HBM as
// structure-of-arrays over the flat slot index of Eq. 9 (engine.py:82-87):
//
//   theta[Q]            committed angles                  f64
//   qamp[3][Qt]         committed qutrit amplitudes       double2 (re, im) per axis
//   slot_max[Q]         SegmentFitnessTable.slot_max      f64 (u64 atomicMax; fitness >= 0)
//   claim[Q]            commit arbitration stamp          u32 (generation + 1)
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
};

struct GenRecord {
  double gen_best;
  double gen_mean;
  double best_fitness;
  double pad;
};

struct QeqeaArgs {
  // configuration (engine.py:33-43)
  int n, L;
  int64_t P, K, Q, Qt;
  double p_mut, mutation_range, target_fitness;
  int n_meas;
  uint64_t max_generations;
  uint64_t seed;
  // bank
  double* theta;
  double2* qamp;  // 3 * Qt, axis-major
  double* slot_max;
  uint32_t* claim;
  // per generation
  double* fitness;   // P (padded to world * shard)
  uint32_t* flats;   // P * L scratch between commit and table kernels
  uint8_t* gate_codes;   // shard * L gate codes of the generation (params -> fitness)
  double* gate_thetas;   // shard * L live angles
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

constexpr double kTwoPiD = 6.283185307179586;   // encoding.py:13 TWO_PI = 2.0 * math.pi
constexpr double kHalfPiD = 1.5707963267948966;  // math.pi / 2

// Python / numpy float remainder with the sign of the divisor (x % m, m > 0).
__device__ __forceinline__ double py_mod(double x, double m) {
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

__device__ __forceinline__ void load_committed(const QeqeaArgs& a, int64_t s, LiveSlot& v) {
  v.theta = a.theta[s];
  if (s < a.Qt) {
#pragma unroll
    for (int k = 0; k < 3; ++k) v.q[k] = a.qamp[k * a.Qt + s];
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
__device__ __forceinline__ bool mutate_slot(const QeqeaArgs& a, int64_t s, uint64_t mg, double f,
                                            LiveSlot& v) {
  uint64_t w[4];
  stream_block(a.seed, DOM_MUTATE, mg, (uint64_t)s, 0, 1, w);
  if (!(u64_to_double(w[0]) < a.p_mut)) return false;
  if (!(f < 1.0)) return false;
  const bool coin = u64_to_double(w[1]) < 0.5;
  const double omf = __dsub_rn(1.0, f);
  if (coin && s < a.Qt) {
    const int which = (int)((uint32_t)(w[2] & 0xffffffffULL) >> 29);  // Lemire, bound 8
    const double range = which < 3 ? kHalfPiD : kTwoPiD;             // encoding.py:23
    const double value = __dadd_rn(0.0, __dmul_rn(__dmul_rn(range, omf), u64_to_double(w[3])));
    su3_one_param(which, value, v.q);
  } else {
    const double sign = u64_to_double(w[2]) < 0.5 ? 1.0 : -1.0;  // encoding.py:51
    const double step = __dmul_rn(__dmul_rn(sign, omf), a.mutation_range);
    v.theta = py_mod(__dadd_rn(v.theta, step), kTwoPiD);
  }
  return true;
}

// Live value of slot s during generation g (committed value plus the pending
// mutation drawn at the end of generation g-1).
__device__ __forceinline__ void live_slot(const QeqeaArgs& a, int64_t s, uint64_t g, LiveSlot& v,
                                          bool* mutated = nullptr) {
  load_committed(a, s, v);
  bool m = false;
  if (g > 0) m = mutate_slot(a, s, g - 1, a.slot_max[s], v);
  if (mutated) *mutated = m;
}

// Gate code of slot s with its measured axis (SegmentBank.descriptor, engine.py:134-146;
// construct_segments, engine.py:167-170).
__device__ __forceinline__ int slot_gate_code(const QeqeaArgs& a, int64_t s, uint64_t g,
                                              const LiveSlot& v) {
  const int64_t kind = s / (a.L * a.P);
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
// flat = kind*L*P + individual*L + position.  Warp-cooperative: every lane
// computes the u32 draws of its positions directly from the counter (fast
// path); if any draw would be rejected by numpy's Lemire sampler, lane 0
// replays the stream sequentially.  Writes flats[0..L).
__device__ __forceinline__ void sample_circuit_warp(const QeqeaArgs& a, uint64_t g, int64_t c,
                                                    uint32_t* flats, int lane) {
  const int L = a.L;
  const uint32_t rngP = (uint32_t)(a.P - 1), rngK = (uint32_t)(a.K - 1);
  const int offk = (a.P == 1) ? 0 : L;  // integers(1, ...) consumes no draws
  bool reject = false;
  for (int p = lane; p < L; p += 32) {
    uint32_t ind = 0;
    if (a.P > 1) {
      uint64_t w[4];
      stream_block(a.seed, DOM_SAMPLE, g, (uint64_t)c, 0, (uint64_t)(p >> 3) + 1, w);
      const uint64_t word = w[(p & 7) >> 1];
      const uint32_t u = (p & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
      reject |= lemire_rejects(u, rngP);
      ind = lemire_value(u, rngP);
    }
    const int uk = offk + p;
    uint64_t w[4];
    stream_block(a.seed, DOM_SAMPLE, g, (uint64_t)c, 0, (uint64_t)(uk >> 3) + 1, w);
    const uint64_t word = w[(uk & 7) >> 1];
    const uint32_t u = (uk & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
    reject |= lemire_rejects(u, rngK);
    const uint32_t kind = lemire_value(u, rngK);
    flats[p] = (uint32_t)((int64_t)kind * L * a.P + (int64_t)ind * L + p);
  }
  if (__any_sync(0xffffffffu, reject)) {
    __syncwarp();
    if (lane == 0) {
      NpStream st;
      st.init(a.seed, DOM_SAMPLE, g, (uint64_t)c, 0);
      for (int p = 0; p < L; ++p) flats[p] = (uint32_t)(st.integers(a.P) * L + p);
      for (int p = 0; p < L; ++p) flats[p] += (uint32_t)(st.integers(a.K) * L * a.P);
    }
  }
  __syncwarp();
}

}  // namespace isq

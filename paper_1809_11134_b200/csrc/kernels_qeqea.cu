// QEQEA generation loop kernels (QeqeaEngine.step, engine.py:318-361).
//
// One generation g is the launch sequence
//   eval     circuits [c0, c1): sample + live slots + measure + compose + score  (K1-K3)
//   (multi-GPU: all-gather of the fitness vector)
//   reduce   gen max / first argmax / mean, best-so-far, record               (K4)
//   capture  gates of the new best circuit (engine.py:341-343)
//   commit   improved & mutated touched slots -> committed bank              (K5, lazy revert)
//   table    slot_max scatter-max (SegmentFitnessTable.update)               (K4)
//   advance  generation += 1, stop reason (engine.py:354-358)
// Every kernel reads the generation from device state and returns
// immediately once a stop reason is set, so batches of generations are
// enqueued without host round trips.
#include "engine_common.cuh"
#include "fitness_warp.cuh"
#include "isq_internal.h"
#include "qeqea_internal.h"

namespace isq {

// ---------------------------------------------------------------- eval ---
// sample (all circuits, flats -> HBM) | values (shard touches -> gate code +
// live angle) | fitness_fast_kernel (kernels_fitness.cu).  Separate kernels
// keep each one's hot code inside the instruction cache and give the random
// bank gathers thread-level memory parallelism.

__global__ void __launch_bounds__(kThreadsPerBlock)
    qeqea_sample_flats_kernel(QeqeaArgs a, int64_t c0, int64_t c1) {
  __shared__ uint64_t blk[kWarpsPerBlock][36];
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = c0 + (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < c1; c += nwarps)
    sample_circuit_warp(a, g, c, a.flats + c * a.L, blk[wib], lane);
}

// One thread per touch of the shard: committed record -> live value (pending
// mutation of g-1).  Rotation touches (1/3 at C5) additionally need the Born
// measurement; those are compacted into a shared-memory queue so the costly
// measurement runs on full warps instead of on the 1/3 of lanes that need it.
// Also records, per touch, the slot_max the generation started from and
// whether the slot carries a pending mutation (the fused single-rank commit
// consumes both).
constexpr int kValThreads = 256;
constexpr int kValPerThread = 3;  // touches per thread per tile: ~1 measurement task per thread

struct MeasureTask {  // 56 B: 768 tasks fit the 48 KB static shared limit
  double re[3], im[3];
  uint32_t s;
  uint32_t out;
};

__global__ void __launch_bounds__(kValThreads) qeqea_values_kernel(QeqeaArgs a, int64_t t0, int64_t t1) {
  __shared__ MeasureTask tasks[kValThreads * kValPerThread];
  __shared__ int ntask;
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  constexpr int kTile = kValThreads * kValPerThread;
  for (int64_t base = t0 + (int64_t)blockIdx.x * kTile; base < t1; base += (int64_t)gridDim.x * kTile) {
    if (threadIdx.x == 0) ntask = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kValPerThread; ++u) {
      const int64_t i = base + u * kValThreads + threadIdx.x;
      if (i >= t1) break;
      const uint32_t s = a.flats[i];
      LiveSlot v;
      const double f = load_committed(a, s, v);
      bool qpath = false;
      const bool mutated = g > 0 && mutate_slot(a, s, g - 1, f, v, &qpath);
      const int64_t o = i - t0;
      a.gate_thetas[o] = v.theta;
      a.touch_fbefore[o] = f;
      a.touch_mutated[o] = (uint8_t)((mutated ? 1 : 0) | (mutated && qpath ? 2 : 0));
      const int64_t kind = (int64_t)s / (a.L * a.P);
      if (kind < a.n) {
        const int k = atomicAdd(&ntask, 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          tasks[k].re[c] = v.q[c].x;
          tasks[k].im[c] = v.q[c].y;
        }
        tasks[k].s = s;
        tasks[k].out = (uint32_t)o;
      } else {
        a.gate_codes[o] = (uint8_t)(3 * a.n + (kind - a.n));
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < ntask; k += kValThreads) {
      const MeasureTask& t = tasks[k];
      NpStream st;
      st.init(a.seed, DOM_MEASURE, g, (uint64_t)t.s, 0);
      double re[3] = {t.re[0], t.re[1], t.re[2]};
      double im[3] = {t.im[0], t.im[1], t.im[2]};
      bool ok = true;
      const int axis = measure_axis(re, im, a.n_meas, st, &ok);
      const int64_t kind = (int64_t)t.s / (a.L * a.P);
      a.gate_codes[t.out] = (uint8_t)(3 * kind + axis);
    }
    __syncthreads();
  }
}

// -------------------------------------------------------------- reduce ---

constexpr int kRedThreads = 256;

// Deterministic block partials of (max with first argmax, sum) over fitness[0, P).
__global__ void __launch_bounds__(kRedThreads) qeqea_reduce_partials(QeqeaArgs a) {
  if (a.st->stop) return;
  __shared__ double smax[kRedThreads], ssum[kRedThreads];
  __shared__ int64_t sarg[kRedThreads];
  const int64_t per = (a.P + a.n_parts - 1) / a.n_parts;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = min(a.P, lo + per);
  double m = -1.0, sum = 0.0;
  int64_t arg = INT64_MAX;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
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
    a.part_max[blockIdx.x] = smax[0];
    a.part_sum[blockIdx.x] = ssum[0];
    a.part_arg[blockIdx.x] = sarg[0];
  }
}

// Final reduction, best-so-far update (strict >, first circuit on ties,
// engine.py:341-343), the generation record, and capture of the new best
// circuit's gates by warp 0.
__global__ void __launch_bounds__(kRedThreads) qeqea_reduce_final(QeqeaArgs a) {
  __shared__ int s_improved;
  __shared__ int64_t s_best;
  QeqeaDevState* st = a.st;
  if (st->stop) return;
  if (threadIdx.x == 0) {
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
    s_improved = improved;
    s_best = arg;
  }
  __syncthreads();
  if (!s_improved || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint64_t g = st->generation;
  for (int p = lane; p < a.L; p += 32) {
    if (a.fused_commit) {
      // single rank: the generation's gate codes / live angles of every
      // circuit are still in place (and the commit may already be rewriting
      // the bank, so do not recompute them from it)
      a.best_codes[p] = a.gate_codes[s_best * a.L + p];
      a.best_thetas[p] = a.gate_thetas[s_best * a.L + p];
    } else {
      const int64_t s = a.flats[s_best * a.L + p];
      LiveSlot v;
      live_slot(a, s, g, v);
      a.best_codes[p] = (uint8_t)slot_gate_code(a, s, g, v);
      a.best_thetas[p] = v.theta;
    }
  }
}

// -------------------------------------------------------------- commit ---

// Elitist accept (engine.py:345-351 + 211-222): a slot mutated at g-1 keeps
// its mutation iff some circuit of generation g that touched it beat its
// slot_max.  Only touched slots can be improved, so walk the touches (thread
// per touch); one improving touch per slot wins the claim stamp and writes
// the live value into the committed bank.
__global__ void __launch_bounds__(256) qeqea_commit_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  if (g == 0) return;
  const int64_t total = a.P * a.L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = a.flats[i];
    const double fit = a.fitness[i / a.L];
    if (!(fit > *smax_ptr(a, s))) continue;
    LiveSlot v;
    const double f = load_committed(a, s, v);
    if (!mutate_slot(a, s, g - 1, f, v)) continue;
    if (atomicMax(&a.claim[s], (uint32_t)(g + 1)) >= (uint32_t)(g + 1)) continue;
    store_committed(a, s, v);
  }
}

constexpr int kCommitThreads = 256;

// Single-rank fused commit + table (every touch of the generation went through
// qeqea_values_kernel, which recorded the slot_max it started from and the
// pending-mutation flag): only improving touches do random bank traffic.
__global__ void __launch_bounds__(kCommitThreads)
    qeqea_commit_table_kernel(QeqeaArgs a, int64_t t0, int64_t t1) {
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  for (int64_t i = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double fit = a.fitness[i / a.L];
    const double fb = a.touch_fbefore[i];
    if (!(fit > fb)) continue;
    const uint32_t s = a.flats[i];
    const uint8_t mf = a.touch_mutated[i];
    if (mf & 2) {
      // qutrit mutation: one improving touch per slot recomputes and writes it
      if (atomicMax(&a.claim[s], (uint32_t)(g + 1)) < (uint32_t)(g + 1)) {
        LiveSlot v;
        load_committed(a, s, v);  // commit writes only theta / qutrit, never slot_max
        mutate_slot(a, s, g - 1, fb, v);
        store_committed(a, s, v);
      }
    } else if (mf & 1) {
      // angle mutation: every improving touch holds the same live angle
      // (values kernel), so the idempotent store needs no arbitration
      if (s < a.Qt)
        a.rot[s].theta = a.gate_thetas[i];
      else
        a.inter[s - a.Qt].theta = a.gate_thetas[i];
    }
    atomicMax(reinterpret_cast<unsigned long long*>(smax_ptr(a, s)),
              (unsigned long long)__double_as_longlong(fit));
  }
}

// SegmentFitnessTable.update slot_max part: scatter-max of the circuit fitness
// over its touched slots (fitness >= 0, so u64 order == double order).
__global__ void qeqea_table_kernel(QeqeaArgs a) {
  if (a.st->stop) return;
  const int64_t total = a.P * a.L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = a.flats[i];
    const double fit = a.fitness[i / a.L];
    double* sm = smax_ptr(a, s);
    if (fit > *sm)
      atomicMax(reinterpret_cast<unsigned long long*>(sm), (unsigned long long)__double_as_longlong(fit));
  }
}

__global__ void qeqea_advance_kernel(QeqeaArgs a) {
  QeqeaDevState* st = a.st;
  if (st->stop) return;
  st->generation += 1;
  if (st->best_fitness >= a.target_fitness)
    st->stop = 1;
  else if (st->generation >= a.max_generations)
    st->stop = 2;
}

// ---------------------------------------------------------- population ---

// Per-slot initial bank (init_population, engine.py:105-112; oracle/streams.py
// init_slot): theta = uniform(0, 2pi) and a Box-Muller complex Gaussian qutrit.
__global__ void qeqea_init_kernel(QeqeaArgs a) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q;
       s += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w0[4], w1[4];
    stream_block(a.seed, DOM_INIT, 0, (uint64_t)s, 0, 1, w0);
    const double theta = __dadd_rn(0.0, __dmul_rn(kTwoPiD, u64_to_double(w0[0])));
    a.claim[s] = 0;
    if (s >= a.Qt) {
      a.inter[s - a.Qt].theta = theta;
      a.inter[s - a.Qt].smax = 0.0;
    } else {
      a.rot[s].theta = theta;
      a.rot[s].smax = 0.0;
      stream_block(a.seed, DOM_INIT, 0, (uint64_t)s, 0, 2, w1);
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
      for (int k = 0; k < 3; ++k) a.rot[s].q[k] = make_double2(re[k] / nrm, im[k] / nrm);
    }
  }
}

// Live bank at the current generation (the reference's engine.pop after the
// last step, i.e. committed values with the pending mutation applied).
__global__ void qeqea_live_kernel(QeqeaArgs a, double* theta_out, double2* q_out) {
  const uint64_t g = a.st->generation;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q;
       s += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    live_slot(a, s, g, v);
    theta_out[s] = v.theta;
    if (s < a.Qt) {
#pragma unroll
      for (int k = 0; k < 3; ++k) q_out[s * 3 + k] = v.q[k];
    }
  }
}

// Records <-> the reference's arrays: theta[Q], qamp[3][Qt] (axis-major), slot_max[Q].
__global__ void qeqea_pack_kernel(QeqeaArgs a, double* theta, double2* qamp, double* smax) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q;
       s += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    const double f = load_committed(a, s, v);
    theta[s] = v.theta;
    smax[s] = f;
    if (s < a.Qt) {
#pragma unroll
      for (int k = 0; k < 3; ++k) qamp[k * a.Qt + s] = v.q[k];
    }
  }
}

__global__ void qeqea_unpack_kernel(QeqeaArgs a, const double* theta, const double2* qamp,
                                    const double* smax) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.Q;
       s += (int64_t)gridDim.x * blockDim.x) {
    LiveSlot v;
    v.theta = theta[s];
    if (s < a.Qt) {
#pragma unroll
      for (int k = 0; k < 3; ++k) v.q[k] = qamp[k * a.Qt + s];
    }
    store_committed(a, s, v);
    *smax_ptr(a, s) = smax ? smax[s] : 0.0;
    a.claim[s] = 0;
  }
}

// Blueprints and gate codes of circuits [c0, c1) at the current generation
// (parity / introspection; same device functions as the eval kernel).
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

// ------------------------------------------------------------ launchers ---

static int blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}



isq_status qeqea_launch_prepare(const QeqeaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  const int grid_s = persistent_grid((const void*)qeqea_sample_flats_kernel, 0, a.P);
  qeqea_sample_flats_kernel<<<grid_s, kThreadsPerBlock, 0, s>>>(a, 0, a.P);
  if (c1 > c0)
    qeqea_values_kernel<<<blocks_for((c1 - c0) * a.L, kValThreads), kValThreads, 0, s>>>(a, c0 * a.L, c1 * a.L);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_score(const QeqeaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  if (c1 <= c0) return ISQ_OK;
  return launch_fitness_batch_stoppable(a.n, a.L, c1 - c0, a.gate_codes, a.gate_thetas,
                                        reinterpret_cast<const double*>(a.target), a.fitness + c0,
                                        &a.st->stop, s);
}

isq_status qeqea_launch_eval(const QeqeaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  isq_status st = qeqea_launch_prepare(a, c0, c1, s);
  if (st != ISQ_OK) return st;
  return qeqea_launch_score(a, c0, c1, s);
}

static void launch_reduce(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_reduce_partials<<<a.n_parts, kRedThreads, 0, s>>>(a);
  qeqea_reduce_final<<<1, kRedThreads, 0, s>>>(a);
}

isq_status qeqea_launch_finish(const QeqeaArgs& a, cudaStream_t s) {
  launch_reduce(a, s);
  if (a.fused_commit) {
    qeqea_commit_table_kernel<<<blocks_for(a.P * a.L, kCommitThreads), kCommitThreads, 0, s>>>(a, 0, a.P * a.L);
  } else {
    qeqea_commit_kernel<<<blocks_for(a.P * a.L, 256), 256, 0, s>>>(a);
    qeqea_table_kernel<<<blocks_for(a.P * a.L, 256), 256, 0, s>>>(a);
  }
  qeqea_advance_kernel<<<1, 1, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_init(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_init_kernel<<<blocks_for(a.Q, 256), 256, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_pack(const QeqeaArgs& a, double* theta, double* qamp, double* smax,
                             cudaStream_t s) {
  qeqea_pack_kernel<<<blocks_for(a.Q, 256), 256, 0, s>>>(a, theta, reinterpret_cast<double2*>(qamp), smax);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_unpack(const QeqeaArgs& a, const double* theta, const double* qamp,
                               const double* smax, cudaStream_t s) {
  qeqea_unpack_kernel<<<blocks_for(a.Q, 256), 256, 0, s>>>(
      a, theta, reinterpret_cast<const double2*>(qamp), smax);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_live(const QeqeaArgs& a, double* theta_out, double* q_out, cudaStream_t s) {
  qeqea_live_kernel<<<blocks_for(a.Q, 256), 256, 0, s>>>(a, theta_out, reinterpret_cast<double2*>(q_out));
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

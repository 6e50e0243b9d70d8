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
// Two kernels: `params` turns every (circuit, position) of the shard into a
// gate (code, live angle) - sampling, lazy mutation, Born measurement - and
// `fitness_fast_kernel` (kernels_fitness.cu) composes and scores them.
// Splitting keeps each kernel's hot code inside the instruction cache.

__global__ void __launch_bounds__(kThreadsPerBlock)
    qeqea_params_kernel(QeqeaArgs a, int64_t c0, int64_t c1) {
  extern __shared__ uint32_t dyn_flats[];
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* flats = dyn_flats + wib * a.L;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = c0 + (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < c1; c += nwarps) {
    sample_circuit_warp(a, g, c, flats, lane);
    for (int p = lane; p < a.L; p += 32) {
      const int64_t s = flats[p];
      LiveSlot v;
      live_slot(a, s, g, v);
      const int64_t o = (c - c0) * a.L + p;
      a.gate_codes[o] = (uint8_t)slot_gate_code(a, s, g, v);
      a.gate_thetas[o] = v.theta;
    }
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
  extern __shared__ uint32_t cap_flats[];
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
  sample_circuit_warp(a, g, s_best, cap_flats, lane);
  for (int p = lane; p < a.L; p += 32) {
    const int64_t s = cap_flats[p];
    LiveSlot v;
    live_slot(a, s, g, v);
    a.best_codes[p] = (uint8_t)slot_gate_code(a, s, g, v);
    a.best_thetas[p] = v.theta;
  }
}

// -------------------------------------------------------------- commit ---

// Elitist accept (engine.py:345-351 + 211-222): a slot mutated at g-1 keeps
// its mutation iff some circuit of generation g that touched it beat its
// slot_max.  Only touched slots can be improved, so walk the touches; one
// touch per slot wins the claim stamp and writes the live value into the
// committed bank.  Also writes the flats for the table kernel.
__global__ void __launch_bounds__(kThreadsPerBlock) qeqea_commit_kernel(QeqeaArgs a) {
  extern __shared__ uint32_t dyn_flats[];
  if (a.st->stop) return;
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* flats = dyn_flats + wib * a.L;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < a.P; c += nwarps) {
    sample_circuit_warp(a, g, c, flats, lane);
    const double fit = a.fitness[c];
    for (int p = lane; p < a.L; p += 32) {
      const uint32_t s = flats[p];
      a.flats[c * a.L + p] = s;
      if (g == 0) continue;
      const double f = a.slot_max[s];
      if (!(fit > f)) continue;
      LiveSlot v;
      load_committed(a, s, v);
      if (!mutate_slot(a, s, g - 1, f, v)) continue;
      if (atomicMax(&a.claim[s], (uint32_t)(g + 1)) >= (uint32_t)(g + 1)) continue;
      a.theta[s] = v.theta;
      if (s < a.Qt) {
#pragma unroll
        for (int k = 0; k < 3; ++k) a.qamp[k * a.Qt + s] = v.q[k];
      }
    }
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
    if (fit > a.slot_max[s])
      atomicMax(reinterpret_cast<unsigned long long*>(a.slot_max) + s,
                (unsigned long long)__double_as_longlong(fit));
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
    a.theta[s] = __dadd_rn(0.0, __dmul_rn(kTwoPiD, u64_to_double(w0[0])));
    a.slot_max[s] = 0.0;
    a.claim[s] = 0;
    if (s < a.Qt) {
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
      for (int k = 0; k < 3; ++k) a.qamp[k * a.Qt + s] = make_double2(re[k] / nrm, im[k] / nrm);
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

// Blueprints and gate codes of circuits [c0, c1) at the current generation
// (parity / introspection; same device functions as the eval kernel).
__global__ void __launch_bounds__(kThreadsPerBlock)
    qeqea_sample_kernel(QeqeaArgs a, int64_t c0, int64_t c1, int64_t* flats_out, uint8_t* codes_out,
                        double* thetas_out) {
  extern __shared__ uint32_t dyn_flats[];
  const uint64_t g = a.st->generation;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* flats = dyn_flats + wib * a.L;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = c0 + (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < c1; c += nwarps) {
    sample_circuit_warp(a, g, c, flats, lane);
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

isq_status qeqea_launch_eval(const QeqeaArgs& a, int64_t c0, int64_t c1, cudaStream_t s) {
  if (c1 <= c0) return ISQ_OK;
  const size_t dyn = (size_t)kWarpsPerBlock * a.L * sizeof(uint32_t);
  const void* k = (const void*)qeqea_params_kernel;
  if (dyn > 48 * 1024) ISQ_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  const int grid = persistent_grid(k, dyn, c1 - c0);
  qeqea_params_kernel<<<grid, kThreadsPerBlock, dyn, s>>>(a, c0, c1);
  ISQ_CUDA_TRY(cudaGetLastError());
  return launch_fitness_batch_stoppable(a.n, a.L, c1 - c0, a.gate_codes, a.gate_thetas,
                                        reinterpret_cast<const double*>(a.target), a.fitness + c0,
                                        &a.st->stop, s);
}

isq_status qeqea_launch_finish(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_reduce_partials<<<a.n_parts, kRedThreads, 0, s>>>(a);
  const size_t cap = (size_t)a.L * sizeof(uint32_t);
  qeqea_reduce_final<<<1, kRedThreads, cap, s>>>(a);
  const size_t dyn = (size_t)kWarpsPerBlock * a.L * sizeof(uint32_t);
  const int grid_c = persistent_grid((const void*)qeqea_commit_kernel, dyn, a.P);
  qeqea_commit_kernel<<<grid_c, kThreadsPerBlock, dyn, s>>>(a);
  qeqea_table_kernel<<<blocks_for(a.P * a.L, 256), 256, 0, s>>>(a);
  qeqea_advance_kernel<<<1, 1, 0, s>>>(a);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

isq_status qeqea_launch_init(const QeqeaArgs& a, cudaStream_t s) {
  qeqea_init_kernel<<<blocks_for(a.Q, 256), 256, 0, s>>>(a);
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

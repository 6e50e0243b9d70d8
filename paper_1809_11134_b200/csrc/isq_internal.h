// Internal declarations shared by the CUDA translation units of libisq.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

#include "../../include/isq.h"

namespace isq {

// Thread-local last error (isq_last_error).
void set_error(const std::string& msg);

#define ISQ_CUDA_TRY(expr)                                                                 \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      ::isq::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                \
      return ISQ_ERR_CUDA;                                                                 \
    }                                                                                      \
  } while (0)

constexpr int kWarpsPerBlock = 4;
constexpr int kThreadsPerBlock = 32 * kWarpsPerBlock;
// Fitness kernels: 2 warps per block keeps the per-warp chunk scratch
// (FastChunk, ~9.6 KB) plus the target inside the 48 KB static shared limit.
constexpr int kFitWarps = 2;
constexpr int kFitThreads = 32 * kFitWarps;

int num_sms();
// Number of resident blocks for a persistent grid of `kernel`.
int persistent_grid(const void* kernel, size_t dyn_smem, int64_t work_warps,
                    int warps_per_block = kWarpsPerBlock);

// fitness / compose over explicit gate lists (device pointers); precision:
// ISQ_PRECISION_FP64 / _FP32 (the fitness-only kernel; composition is fp64).
isq_status launch_fitness_batch(int n, int L, int64_t count, const uint8_t* codes,
                                const double* thetas, const double* target_dev,
                                double* fitness_dev, double* unitary_dev, cudaStream_t stream,
                                int precision = ISQ_PRECISION_FP64, int* bad_code = nullptr);

// fitness-only batch that skips all work once *stop != 0 (engine generations).
isq_status launch_fitness_batch_stoppable(int n, int L, int64_t count, const uint8_t* codes,
                                          const double* thetas, const double* target_dev,
                                          double* fitness_dev, const int32_t* stop,
                                          cudaStream_t stream, int blocks_per_sm = 0,
                                          int precision = ISQ_PRECISION_FP64,
                                          int* bad_code = nullptr,
                                          unsigned long long* dyn = nullptr);
// Circuits holding a code that is not a gate of the wire count get a NaN
// fitness, and *bad_code (device int, nullable) is set to 1.

// Launch-bound small populations: `per_graph` generations captured once into
// a CUDA graph (on a private capture stream, so the caller's stream may be the
// legacy default stream) and replayed on the handle's stream.  Valid because
// every generation kernel reads the generation / stop flag from device state
// and takes only handle-constant arguments.
struct GenGraph {
  cudaGraphExec_t exec = nullptr;
  int gens = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    gens = 0;
  }
};

template <class EnqueueOne>
isq_status run_generations(GenGraph& g, cudaStream_t stream, int n, int per_graph, EnqueueOne enqueue_one) {
  int done = 0;
  if (per_graph > 1 && n >= per_graph) {
    if (g.exec == nullptr || g.gens != per_graph) {
      g.reset();
      cudaStream_t cap = nullptr;
      ISQ_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
      isq_status st = ISQ_OK;
      for (int i = 0; e == cudaSuccess && st == ISQ_OK && i < per_graph; ++i) st = enqueue_one(cap);
      cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
      if (e == cudaSuccess) e = e2;
      if (e == cudaSuccess && st == ISQ_OK) e = cudaGraphInstantiate(&g.exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      cudaStreamDestroy(cap);
      if (st != ISQ_OK) return st;
      ISQ_CUDA_TRY(e);
      g.gens = per_graph;
    }
    for (; done + per_graph <= n; done += per_graph) ISQ_CUDA_TRY(cudaGraphLaunch(g.exec, stream));
  }
  for (; done < n; ++done) {
    isq_status st = enqueue_one(stream);
    if (st != ISQ_OK) return st;
  }
  return ISQ_OK;
}

// Generations per graph for a population of `touches` = P * L gate slots
// (0: plain launches; large populations are not launch-bound).
// CUDA graphs pay off while launch gaps are a visible share of a generation
// (measured: C4, 2^21 gate slots, 2468 -> 2551 gen/s; 2^23 slots +0.8 %).
inline int graph_generations(int64_t touches) { return touches <= (1LL << 22) ? 16 : 0; }

// n = ISQ_MAX_FAST_WIRES+1 .. ISQ_MAX_WIRES: block-per-circuit fitness (unitary
// != nullptr: composition from I with the exact global phase, as compose_kernel).
// codes_alt / thetas_alt / parity: the GA's double-buffered genomes (odd
// generation counter -> the alternate buffers).
isq_status launch_fitness_generic(int n, int L, int64_t count, const uint8_t* codes, const double* thetas,
                                  const double* target, double* fitness, double* unitary, const int32_t* stop,
                                  cudaStream_t stream, int* bad_code, const uint8_t* codes_alt = nullptr,
                                  const double* thetas_alt = nullptr, const uint64_t* parity = nullptr,
                                  const double* init = nullptr);

isq_status launch_overlap_fitness(int64_t D, int64_t count, const double* S, const double* T,
                                  double* out, cudaStream_t stream);

}  // namespace isq

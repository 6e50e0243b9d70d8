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

// fitness / compose over explicit gate lists (device pointers).
isq_status launch_fitness_batch(int n, int L, int64_t count, const uint8_t* codes,
                                const double* thetas, const double* target_dev,
                                double* fitness_dev, double* unitary_dev, cudaStream_t stream);

// fitness-only batch that skips all work once *stop != 0 (engine generations).
isq_status launch_fitness_batch_stoppable(int n, int L, int64_t count, const uint8_t* codes,
                                          const double* thetas, const double* target_dev,
                                          double* fitness_dev, const int32_t* stop,
                                          cudaStream_t stream, int blocks_per_sm = 0);

isq_status launch_overlap_fitness(int64_t D, int64_t count, const double* S, const double* T,
                                  double* out, cudaStream_t stream);

}  // namespace isq

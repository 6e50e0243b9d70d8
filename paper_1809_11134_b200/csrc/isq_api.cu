// C ABI of libisq: argument validation, host<->device staging, error state.
#include <string>
#include <vector>

#include "isq_internal.h"
#include "np_random.cuh"

namespace isq {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

static isq_status check_shape(int32_t n, int32_t length, int64_t count) {
  if (n < ISQ_MIN_WIRES || n > ISQ_MAX_WIRES) {
    set_error("numberOfWires=" + std::to_string(n) + " outside the compiled range " +
              std::to_string(ISQ_MIN_WIRES) + ".." + std::to_string(ISQ_MAX_WIRES));
    return n < 2 ? ISQ_ERR_CONFIG : ISQ_ERR_UNSUPPORTED;
  }
  if (length < 0 || count < 0) {
    set_error("negative circuit length or count");
    return ISQ_ERR_CONFIG;
  }
  return ISQ_OK;
}

static isq_status check_codes(int32_t n, const uint8_t* codes, int64_t total) {
  const int ncodes = 3 * n + n * (n - 1) / 2;
  uint8_t mx = 0;
  for (int64_t i = 0; i < total; ++i) mx = codes[i] > mx ? codes[i] : mx;  // vectorised max
  if (mx < ncodes) return ISQ_OK;
  for (int64_t i = 0; i < total; ++i) {
    if (codes[i] >= ncodes) {
      set_error("gate code " + std::to_string((int)codes[i]) + " at index " + std::to_string(i) +
                " is not a valid gate for numberOfWires=" + std::to_string(n));
      return ISQ_ERR_CONFIG;
    }
  }
  return ISQ_OK;
}

}  // namespace isq

using namespace isq;

extern "C" {

const char* isq_last_error(void) { return g_last_error.c_str(); }

int32_t isq_abi_version(void) { return 1; }

void isq_philox_block(uint64_t seed, uint64_t domain, uint64_t gen, uint64_t index, uint64_t sub,
                      uint64_t block, uint64_t* out) {
  stream_block(seed, domain, gen, index, sub, block, out);
}

isq_status isq_fitness_batch_device(int32_t n, int32_t length, int64_t count,
                                    const uint8_t* codes_dev, const double* thetas_dev,
                                    const double* target_dev, double* fitness_dev,
                                    double* unitary_dev, void* stream) {
  isq_status st = check_shape(n, length, count);
  if (st != ISQ_OK) return st;
  return launch_fitness_batch(n, length, count, codes_dev, thetas_dev, target_dev, fitness_dev,
                              unitary_dev, (cudaStream_t)stream);
}

isq_status isq_fitness_batch(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                             const double* thetas, const double* target, double* fitness_out,
                             double* unitary_out, int32_t device) {
  isq_status st = check_shape(n, length, count);
  if (st != ISQ_OK) return st;
  const int64_t total = count * (int64_t)length;
  st = check_codes(n, codes, total);
  if (st != ISQ_OK) return st;
  if (count == 0) return ISQ_OK;
  ISQ_CUDA_TRY(cudaSetDevice(device));
  const int64_t D = 1LL << n;
  uint8_t* d_codes = nullptr;
  double *d_thetas = nullptr, *d_target = nullptr, *d_fit = nullptr, *d_u = nullptr;
  cudaStream_t s = nullptr;
  isq_status rc = ISQ_OK;
  auto fail = [&](cudaError_t e, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    rc = ISQ_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) {
    fail(e, "cudaStreamCreate");
    return rc;
  }
  do {
    if ((e = cudaMallocAsync((void**)&d_codes, total > 0 ? total : 1, s))) { fail(e, "cudaMalloc"); break; }
    if ((e = cudaMallocAsync((void**)&d_thetas, (total > 0 ? total : 1) * 8, s))) { fail(e, "cudaMalloc"); break; }
    if ((e = cudaMallocAsync((void**)&d_target, 2 * D * D * 8, s))) { fail(e, "cudaMalloc"); break; }
    if ((e = cudaMallocAsync((void**)&d_fit, count * 8, s))) { fail(e, "cudaMalloc"); break; }
    if (unitary_out && (e = cudaMallocAsync((void**)&d_u, count * 2 * D * D * 8, s))) { fail(e, "cudaMalloc"); break; }
    if (total > 0) {
      if ((e = cudaMemcpyAsync(d_codes, codes, total, cudaMemcpyHostToDevice, s))) { fail(e, "H2D codes"); break; }
      if ((e = cudaMemcpyAsync(d_thetas, thetas, total * 8, cudaMemcpyHostToDevice, s))) { fail(e, "H2D thetas"); break; }
    }
    if ((e = cudaMemcpyAsync(d_target, target, 2 * D * D * 8, cudaMemcpyHostToDevice, s))) { fail(e, "H2D target"); break; }
    rc = launch_fitness_batch(n, length, count, d_codes, d_thetas, d_target, d_fit, d_u, s);
    if (rc != ISQ_OK) break;
    if ((e = cudaMemcpyAsync(fitness_out, d_fit, count * 8, cudaMemcpyDeviceToHost, s))) { fail(e, "D2H fitness"); break; }
    if (unitary_out && (e = cudaMemcpyAsync(unitary_out, d_u, count * 2 * D * D * 8, cudaMemcpyDeviceToHost, s))) { fail(e, "D2H unitary"); break; }
    if ((e = cudaStreamSynchronize(s))) { fail(e, "cudaStreamSynchronize"); break; }
  } while (0);
  cudaFreeAsync(d_codes, s);
  cudaFreeAsync(d_thetas, s);
  cudaFreeAsync(d_target, s);
  cudaFreeAsync(d_fit, s);
  if (d_u) cudaFreeAsync(d_u, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return rc;
}

isq_status isq_fitness_of_unitaries(int64_t dim, int64_t count, const double* unitaries,
                                    const double* target, double* fitness_out, int32_t device) {
  if (dim < 1 || count < 0) {
    set_error("fitness dimension mismatch");
    return ISQ_ERR_CONFIG;
  }
  if (count == 0) return ISQ_OK;
  ISQ_CUDA_TRY(cudaSetDevice(device));
  const size_t mb = (size_t)dim * dim * 16;
  double *d_s = nullptr, *d_t = nullptr, *d_o = nullptr;
  isq_status rc = ISQ_OK;
  cudaError_t e = cudaSuccess;
  do {
    if ((e = cudaMalloc((void**)&d_s, mb * count))) break;
    if ((e = cudaMalloc((void**)&d_t, mb))) break;
    if ((e = cudaMalloc((void**)&d_o, 8 * count))) break;
    if ((e = cudaMemcpy(d_s, unitaries, mb * count, cudaMemcpyHostToDevice))) break;
    if ((e = cudaMemcpy(d_t, target, mb, cudaMemcpyHostToDevice))) break;
    rc = launch_overlap_fitness(dim, count, d_s, d_t, d_o, nullptr);
    if (rc != ISQ_OK) break;
    if ((e = cudaMemcpy(fitness_out, d_o, 8 * count, cudaMemcpyDeviceToHost))) break;
  } while (0);
  if (e != cudaSuccess) {
    set_error(std::string("isq_fitness_of_unitaries: ") + cudaGetErrorString(e));
    rc = ISQ_ERR_CUDA;
  }
  cudaFree(d_s);
  cudaFree(d_t);
  cudaFree(d_o);
  return rc;
}

}  // extern "C"

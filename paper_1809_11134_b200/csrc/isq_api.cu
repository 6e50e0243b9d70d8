// C ABI of libisq: argument validation, host<->device staging, error state.
#include <map>
#include <mutex>
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

int32_t isq_abi_version(void) { return 2; }

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

// Host-buffer fitness: a per-device staging context (grow-only device buffers,
// two streams) pipelines the batch in chunks so the host->device copy of chunk
// i+1 overlaps the fitness kernel of chunk i and the fitness read-back.
// Pinned host buffers give full-bandwidth DMA; pageable ones still work.
struct BatchContext {
  int device = -1;
  cudaStream_t copy = nullptr, comp = nullptr;
  uint8_t* codes[2] = {nullptr, nullptr};
  double* thetas[2] = {nullptr, nullptr};
  double* fit[2] = {nullptr, nullptr};
  double* target = nullptr;
  int* bad = nullptr;             // device flag: an invalid gate code was seen
  unsigned char* unit = nullptr;  // compose output (not pipelined)
  size_t cap_rows = 0, cap_len = 0, cap_unit = 0, cap_target = 0;
  cudaEvent_t loaded[2], done[2];
  std::mutex mu;
};

static BatchContext* batch_context(int device) {
  static std::mutex g;
  static BatchContext* ctx[64] = {nullptr};
  std::lock_guard<std::mutex> lk(g);
  if (device < 0 || device >= 64) return nullptr;
  if (!ctx[device]) {
    BatchContext* c = new BatchContext();
    c->device = device;
    cudaSetDevice(device);
    cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&c->comp, cudaStreamNonBlocking);
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&c->loaded[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->done[b], cudaEventDisableTiming);
    }
    ctx[device] = c;
  }
  return ctx[device];
}

static isq_status fitness_batch_host(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                                     const double* thetas, const double* target, double* fitness_out,
                                     double* unitary_out, int32_t device, int32_t precision) {
  isq_status st = check_shape(n, length, count);
  if (st != ISQ_OK) return st;
  const int64_t total = count * (int64_t)length;
  if (unitary_out) {  // readout path: codes checked on the host
    st = check_codes(n, codes, total);
    if (st != ISQ_OK) return st;
  }
  if (count == 0) return ISQ_OK;
  ISQ_CUDA_TRY(cudaSetDevice(device));
  BatchContext* c = batch_context(device);
  if (!c) {
    set_error("invalid device ordinal");
    return ISQ_ERR_CONFIG;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  const int64_t D = 1LL << n;
  // circuits per pipeline stage: ~1/32 of the batch (2^14..2^17), so the
  // last stage's score, which nothing overlaps, stays short
  int64_t chunk = count / 32;
  chunk = chunk < (1 << 14) ? (1 << 14) : (chunk > (1 << 17) ? (1 << 17) : chunk);
  if (chunk > count) chunk = count;
  const size_t len = (size_t)(length > 0 ? length : 1);
  if ((size_t)chunk > c->cap_rows || len > c->cap_len) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(c->codes[b]);
      cudaFree(c->thetas[b]);
      cudaFree(c->fit[b]);
    }
    c->cap_rows = (size_t)chunk;
    c->cap_len = len;
    for (int b = 0; b < 2; ++b) {
      ISQ_CUDA_TRY(cudaMalloc((void**)&c->codes[b], c->cap_rows * c->cap_len));
      ISQ_CUDA_TRY(cudaMalloc((void**)&c->thetas[b], c->cap_rows * c->cap_len * 8));
      ISQ_CUDA_TRY(cudaMalloc((void**)&c->fit[b], c->cap_rows * 8));
    }
  }
  if ((size_t)(D * D * 16) > c->cap_target) {  // n > 5 targets are up to 1024 x 1024
    ISQ_CUDA_TRY(cudaStreamSynchronize(c->comp));
    cudaFree(c->target);
    c->target = nullptr;
    c->cap_target = 0;
    ISQ_CUDA_TRY(cudaMalloc((void**)&c->target, D * D * 16));
    c->cap_target = (size_t)(D * D * 16);
  }
  ISQ_CUDA_TRY(cudaMemcpyAsync(c->target, target, D * D * 16, cudaMemcpyHostToDevice, c->copy));
  if (unitary_out) {
    // composition output (readout path): chunk by chunk, not pipelined; at
    // most 256 MB of unitaries per chunk
    const int64_t per_chunk = ((int64_t)256 << 20) / (D * D * 16);
    if (chunk > per_chunk) chunk = per_chunk < 1 ? 1 : per_chunk;
    const size_t ub = (size_t)chunk * D * D * 16;
    if (ub > c->cap_unit) {
      cudaFree(c->unit);
      c->cap_unit = ub;
      ISQ_CUDA_TRY(cudaMalloc((void**)&c->unit, ub));
    }
    for (int64_t off = 0; off < count; off += chunk) {
      const int64_t m = (count - off) < chunk ? (count - off) : chunk;
      if (length > 0) {
        ISQ_CUDA_TRY(cudaMemcpyAsync(c->codes[0], codes + off * length, m * length,
                                     cudaMemcpyHostToDevice, c->copy));
        ISQ_CUDA_TRY(cudaMemcpyAsync(c->thetas[0], thetas + off * length, m * length * 8,
                                     cudaMemcpyHostToDevice, c->copy));
      }
      ISQ_CUDA_TRY(cudaStreamSynchronize(c->copy));
      st = launch_fitness_batch(n, length, m, c->codes[0], c->thetas[0], c->target, c->fit[0],
                                reinterpret_cast<double*>(c->unit), c->comp);
      if (st != ISQ_OK) return st;
      ISQ_CUDA_TRY(cudaMemcpyAsync(fitness_out + off, c->fit[0], m * 8, cudaMemcpyDeviceToHost, c->comp));
      ISQ_CUDA_TRY(cudaMemcpyAsync(unitary_out + off * D * D * 2, c->unit, (size_t)m * D * D * 16,
                                   cudaMemcpyDeviceToHost, c->comp));
      ISQ_CUDA_TRY(cudaStreamSynchronize(c->comp));
    }
    return ISQ_OK;
  }
  // pipelined: copy stream loads chunk i into buffer i%2 while comp scores chunk i-1;
  // gate codes are validated by the fitness kernel itself (device flag)
  if (!c->bad) ISQ_CUDA_TRY(cudaMalloc((void**)&c->bad, sizeof(int)));
  ISQ_CUDA_TRY(cudaMemsetAsync(c->bad, 0, sizeof(int), c->comp));
  int64_t i = 0;
  for (int64_t off = 0; off < count; off += chunk, ++i) {
    const int b = (int)(i & 1);
    const int64_t m = (count - off) < chunk ? (count - off) : chunk;
    ISQ_CUDA_TRY(cudaStreamWaitEvent(c->copy, c->done[b], 0));  // buffer b free again
    if (length > 0) {
      ISQ_CUDA_TRY(cudaMemcpyAsync(c->codes[b], codes + off * length, m * length,
                                   cudaMemcpyHostToDevice, c->copy));
      ISQ_CUDA_TRY(cudaMemcpyAsync(c->thetas[b], thetas + off * length, m * length * 8,
                                   cudaMemcpyHostToDevice, c->copy));
    }
    ISQ_CUDA_TRY(cudaEventRecord(c->loaded[b], c->copy));
    ISQ_CUDA_TRY(cudaStreamWaitEvent(c->comp, c->loaded[b], 0));
    st = launch_fitness_batch(n, length, m, c->codes[b], c->thetas[b], c->target, c->fit[b],
                              nullptr, c->comp, precision, c->bad);
    if (st != ISQ_OK) return st;
    ISQ_CUDA_TRY(cudaMemcpyAsync(fitness_out + off, c->fit[b], m * 8, cudaMemcpyDeviceToHost, c->comp));
    ISQ_CUDA_TRY(cudaEventRecord(c->done[b], c->comp));
  }
  int bad = 0;
  ISQ_CUDA_TRY(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->comp));
  ISQ_CUDA_TRY(cudaStreamSynchronize(c->comp));
  if (bad) return check_codes(n, codes, total);  // locate it for the message
  return ISQ_OK;
}

// Persistent per-(device, stream) device counters for the dynamically
// scheduled fitness launches of isq_fitness_batch_device_ex (8 bytes each,
// kept for the life of the process); nullptr when allocation fails.
static unsigned long long* stream_counter(cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned long long*> counters;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, stream);
  auto it = counters.find(key);
  if (it != counters.end()) return it->second;
  unsigned long long* c = nullptr;
  if (cudaMalloc((void**)&c, sizeof(*c)) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free allocation error
    return nullptr;
  }
  counters[key] = c;
  return c;
}

static isq_status check_precision(int32_t precision) {
  if (precision == ISQ_PRECISION_FP64 || precision == ISQ_PRECISION_FP32) return ISQ_OK;
  set_error("precision must be ISQ_PRECISION_FP64 or ISQ_PRECISION_FP32");
  return ISQ_ERR_CONFIG;
}

isq_status isq_fitness_batch(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                             const double* thetas, const double* target, double* fitness_out,
                             double* unitary_out, int32_t device) {
  return fitness_batch_host(n, length, count, codes, thetas, target, fitness_out, unitary_out, device,
                            ISQ_PRECISION_FP64);
}

isq_status isq_fitness_batch_ex(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                                const double* thetas, const double* target, double* fitness_out,
                                int32_t device, int32_t precision) {
  isq_status st = check_precision(precision);
  if (st != ISQ_OK) return st;
  return fitness_batch_host(n, length, count, codes, thetas, target, fitness_out, nullptr, device,
                            precision);
}

isq_status isq_fitness_batch_device_ex(int32_t n, int32_t length, int64_t count,
                                       const uint8_t* codes_dev, const double* thetas_dev,
                                       const double* target_dev, double* fitness_dev,
                                       int32_t precision, void* stream) {
  isq_status st = check_shape(n, length, count);
  if (st == ISQ_OK) st = check_precision(precision);
  if (st != ISQ_OK) return st;
  if (count <= 0) return ISQ_OK;
  // the dynamic-scheduling counter of this launch: one persistent counter per
  // (device, stream), reset in stream order by the launch itself, so
  // launches on one stream reuse it and concurrent streams never share one;
  // without it the kernel falls back to a static grid stride
  const cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* ctr = stream_counter(s);
  return launch_fitness_batch_stoppable(n, length, count, codes_dev, thetas_dev, target_dev, fitness_dev, nullptr,
                                        s, 0, precision, nullptr, ctr);
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

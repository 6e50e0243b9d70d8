// Diagnostics: FP64 / FP32 CUDA-core FMA peak microbenchmark (roofline
// denominator for the fitness kernel; MEASURED_PEAKS.json carries only HBM and
// bf16 tensor figures).  Each thread runs 8 independent FMA chains.
#include "isq_internal.h"

namespace isq {

template <typename T>
__global__ void __launch_bounds__(256) fma_peak_kernel(int iters, T seed, T* sink) {
  T a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
    a6 = a0 + 6, a7 = a0 + 7;
  const T b = (T)0.999999, c = (T)1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == (T)-1.2345) sink[0] = s;  // never true; keeps the chains live
}

}  // namespace isq

using namespace isq;

extern "C" isq_status isq_fma_peak(int32_t fp64, int32_t device, double* flops_per_s) {
  ISQ_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  ISQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int blocks = sms * 8, threads = 256, iters = fp64 ? 2048 : 8192;
  void* sink = nullptr;
  ISQ_CUDA_TRY(cudaMalloc(&sink, 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    if (fp64)
      fma_peak_kernel<double><<<blocks, threads>>>(iters, 1.0, (double*)sink);
    else
      fma_peak_kernel<float><<<blocks, threads>>>(iters, 1.0f, (float*)sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  ISQ_CUDA_TRY(cudaGetLastError());
  *flops_per_s = 2.0 * 64.0 * (double)iters * threads * blocks / (best * 1e-3);
  return ISQ_OK;
}

// Timing of the exact-parallel SUS running sums (csrc/sus.cuh) on one block,
// against the plain sequential chain on one thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1809_11134_b200/csrc tools/susbench.cu -o /tmp/susbench
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "sus.cuh"

using namespace isq;

__global__ void __launch_bounds__(kSusThreads) chain_kernel(const double* f, int64_t n, double* out) {
  extern __shared__ double sb[];
  exact_chain_block(f, 0.0, n, 0.0, out, sb);
}
__global__ void __launch_bounds__(kSusThreads) chain_const_kernel(double s, double p0, int64_t n, double* out) {
  exact_const_chain_block(s, n, p0, out);
}
__global__ void seq_kernel(const double* f, int64_t n, double* out) {
  double x = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    x = __dadd_rn(x, f[i]);
    out[i] = x;
  }
}
__global__ void __launch_bounds__(kSusThreads) total_kernel(const double* f, int64_t n, double* out) {
  __shared__ double sm[kSusThreads];
  const double t = np_pairwise_sum_block<kSusThreads>(f, n, sm);
  if (threadIdx.x == 0) out[0] = t;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
  std::vector<double> h(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(0.0, 0.05);
  for (auto& v : h) v = U(g);
  double *f, *o1, *o2, *t;
  cudaMalloc(&f, n * 8);
  cudaMalloc(&o1, n * 8);
  cudaMalloc(&o2, n * 8);
  cudaMalloc(&t, 8);
  cudaMemcpy(f, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute((const void*)chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmem);
  cudaFuncSetAttribute((const void*)chain_const_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    chain_kernel<<<1, kSusThreads, kChainSmem>>>(f, n, o1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("exact_chain_block  n=%lld  %.3f ms\n", (long long)n, ms);
    cudaEventRecord(a);
    chain_const_kernel<<<1, kSusThreads, kChainSmem>>>(0.0123456789, 0.00321, n, o2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("exact_chain const  n=%lld  %.3f ms\n", (long long)n, ms);
    {
      std::vector<double> c(n);
      cudaMemcpy(c.data(), o2, n * 8, cudaMemcpyDeviceToHost);
      double p = 0.00321;
      int64_t bad = 0;
      for (int64_t i = 0; i < n; ++i) {
        p = p + 0.0123456789;
        bad += c[i] != p;
      }
      printf("const chain mismatches vs host: %lld\n", (long long)bad);
    }
    cudaEventRecord(a);
    total_kernel<<<1, kSusThreads>>>(f, n, t);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("pairwise total     n=%lld  %.3f ms\n", (long long)n, ms);
    cudaEventRecord(a);
    seq_kernel<<<1, 1>>>(f, n, o2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("sequential chain   n=%lld  %.3f ms\n", (long long)n, ms);
  }
  std::vector<double> r1(n), r2(n);
  cudaMemcpy(r1.data(), o1, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), o2, n * 8, cudaMemcpyDeviceToHost);
#ifdef ISQ_SUS_PROFILE
  unsigned long long prof[4];
  cudaMemcpyFromSymbol(prof, g_sus_prof, sizeof(prof));  // block 0
  printf("profile (all runs): attempts %llu scalar elements %llu parallel cycles %llu scalar cycles %llu\n", prof[0],
         prof[1], prof[2], prof[3]);
#endif
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) bad += r1[i] != r2[i];
  printf("mismatches vs sequential: %lld  (%s)\n", (long long)bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

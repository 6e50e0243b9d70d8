// Timing of the exact-parallel SUS running sums (csrc/sus.cuh) on one block,
// against the plain sequential chain on one thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1809_11134_b200/csrc tools/susbench.cu -o /tmp/susbench
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
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

__global__ void __launch_bounds__(kSusThreads) combine_kernel(const double* parts, int d, double* out) {
  extern __shared__ double sm[];
  const double t = np_pairwise_combine_block<kSusThreads>(parts, d, sm);
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
  // the grid-wide chain (launch_exact_chain_grid) on several value kinds, vs the host walk
  if (prepare_exact_chain_grid() != cudaSuccess) return 1;
  const int64_t sizes[] = {n, kChainGridMinTiles * kChainTile + 5, 3 * n + 77};
  for (int64_t m : sizes) {
    std::vector<double> hv(m), ho(m), want(m);
    double *df, *dout;
    void* scratch;
    cudaMalloc(&df, m * 8);
    cudaMalloc(&dout, m * 8);
    cudaMalloc(&scratch, chain_grid_scratch_bytes(m));
    for (int kind = 0; kind < 6; ++kind) {
      std::mt19937_64 r(100 + kind);
      std::uniform_real_distribution<double> u01(0.0, 1.0);
      for (int64_t i = 0; i < m; ++i) {
        const double v = u01(r);
        switch (kind) {
          case 0: hv[i] = 0.05 * v; break;                                   // engine-like
          case 1: hv[i] = std::floor(v * 64) / 64.0; break;                  // dyadic: exact ties
          case 2: hv[i] = v < 0.3 ? 0.0 : (v > 0.9999 ? 1e6 * v : v); break;  // zeros and spikes
          case 3: hv[i] = 1e-310 * v; break;                                 // subnormal start
          case 4: hv[i] = i < m / 2 ? 0.0 : v; break;                        // zero prefix
          default: hv[i] = std::ldexp(v, (int)(i % 40) - 20); break;         // wide exponent range
        }
      }
      double x = 0.0;
      for (int64_t i = 0; i < m; ++i) want[i] = x = x + hv[i];
      cudaMemcpy(df, hv.data(), m * 8, cudaMemcpyHostToDevice);
      cudaMemset(dout, 0xff, m * 8);
      launch_exact_chain_grid(df, m, 0.0, dout, scratch, 0);  // warm
      cudaEventRecord(a);
      launch_exact_chain_grid(df, m, 0.0, dout, scratch, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(ho.data(), dout, m * 8, cudaMemcpyDeviceToHost);
      int64_t nb = 0;
      for (int64_t i = 0; i < m; ++i) nb += std::memcmp(&ho[i], &want[i], 8) != 0;
      std::vector<int> slow((m + kChainTile - 1) / kChainTile);
      const ChainGridScratch g = chain_grid_scratch(scratch, m);
      cudaMemcpy(slow.data(), g.slow, slow.size() * 4, cudaMemcpyDeviceToHost);
      int ns = 0;
      for (int v : slow) ns += v;
      {  // numpy's total over the grid vs the one-block form
        double *t1, *t2;
        cudaMalloc(&t1, 8);
        cudaMalloc(&t2, 8);
        cudaFuncSetAttribute((const void*)combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 << kPwMaxDepth);
        cudaEventRecord(a);
        launch_pairwise_parts(df, m, scratch, m, 0);
        combine_kernel<<<1, kSusThreads, 8 << kPwMaxDepth>>>(g.parts, pairwise_grid_depth(m), t1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms2;
        cudaEventElapsedTime(&ms2, a, b);
        total_kernel<<<1, kSusThreads>>>(df, m, t2);
        double h1, h2;
        cudaMemcpy(&h1, t1, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&h2, t2, 8, cudaMemcpyDeviceToHost);
        printf("  pairwise grid total %.3f ms  %s\n", ms2, std::memcmp(&h1, &h2, 8) == 0 ? "equal" : "DIFFERENT");
        bad += std::memcmp(&h1, &h2, 8) != 0;
        cudaFree(t1);
        cudaFree(t2);
      }
      printf("grid chain n=%lld kind %d  %.3f ms  slow tiles %d/%zu  mismatches %lld  (%s)\n", (long long)m, kind, ms,
             ns, slow.size(), (long long)nb, cudaGetErrorString(cudaGetLastError()));
      bad += nb;
    }
    cudaFree(df);
    cudaFree(dout);
    cudaFree(scratch);
  }
  return bad != 0;
}

// Random-gather microbenchmark: DRAM cost of one random access of W bytes
// (8..128) into a 16 GB table, plus random 8 B atomicMax RMW.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

template <int W>
__global__ void gather(const uint4* __restrict__ tab, uint64_t nrec, int64_t n, double* out) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    if constexpr (W == 8) {
      acc += reinterpret_cast<const double*>(tab)[r * 16];
    } else if constexpr (W == 16) {
      const uint4 v = tab[r * 8];
      acc += __longlong_as_double(((uint64_t)v.y << 32) | v.x);
    } else {
      const uint4* p = tab + r * 8;
#pragma unroll
      for (int k = 0; k < W / 16; ++k) {
        const uint4 v = p[k];
        acc += __longlong_as_double(((uint64_t)v.y << 32) | v.x) + (double)v.z;
      }
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

// 64 B records read with two 256-bit loads (sm_100 LDG.256) instead of four 128-bit ones
__global__ void gather64_v256(const double* __restrict__ tab, uint64_t nrec, int64_t n, double* out) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    const double* p = tab + r * 16;
    double a, b, c, d, e, f, g, h;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(e), "=d"(f), "=d"(g), "=d"(h) : "l"(p + 4));
    acc += a + b + c + d + e + f + g + h;
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void rmw(unsigned long long* tab, uint64_t nrec, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    atomicMax(tab + r * 16, (unsigned long long)i);
  }
}

__global__ void scatter_store(unsigned long long* tab, uint64_t nrec, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    tab[r * 16] = (unsigned long long)i;
  }
}

// load, compare, RED only when larger (most touches of a converged bank do not improve)
__global__ void rmw_cond(unsigned long long* tab, uint64_t nrec, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    if (tab[r * 16] < (unsigned long long)i) atomicMax(tab + r * 16, (unsigned long long)i);
  }
}

int main() {
  const size_t bytes = 16ULL << 30;  // 16 GB table of 128 B records
  const uint64_t nrec = bytes / 128;
  uint4* tab;
  double* out;
  cudaMalloc(&tab, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(tab, 0, bytes);
  const int64_t n = 64LL << 20;  // 67M random accesses
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int k = 0; k < 5; ++k) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-12s %8.3f ms  %6.2f Gacc/s\n", name, ms, n / (ms * 1e6));
  };
  const int grid = 148 * 8, blk = 256;
  for (int gran : {-1}) {
  if (gran > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
  printf("-- L2 fetch granularity %zu B%s\n", cur, gran < 0 ? " (default)" : "");
  run("gather8", [&] { gather<8><<<grid, blk>>>(tab, nrec, n, out); });
  run("gather16", [&] { gather<16><<<grid, blk>>>(tab, nrec, n, out); });
  run("gather32", [&] { gather<32><<<grid, blk>>>(tab, nrec, n, out); });
  run("gather64", [&] { gather<64><<<grid, blk>>>(tab, nrec, n, out); });
  run("gather128", [&] { gather<128><<<grid, blk>>>(tab, nrec, n, out); });
  run("gather64v256", [&] { gather64_v256<<<grid, blk>>>((const double*)tab, nrec, n, out); });
  run("atomicmax8", [&] { rmw<<<grid, blk>>>((unsigned long long*)tab, nrec, n); });
  run("store8", [&] { scatter_store<<<grid, blk>>>((unsigned long long*)tab, nrec, n); });
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

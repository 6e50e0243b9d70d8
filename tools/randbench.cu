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

// random stores of W bytes (16: one 128-bit store; 32 / 64: 256-bit stores): a
// full 32 B sector written needs no DRAM read for the merge
template <int W>
__global__ void scatter_wide(double* tab, uint64_t nrec, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(i * 0x9E3779B97F4A7C15ULL) % nrec;
    double* p = tab + r * 16;
    const double v = (double)i;
    if constexpr (W == 16) {
      asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v), "d"(v));
    } else {
#pragma unroll
      for (int k = 0; k < W / 32; ++k)
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * k), "d"(v), "d"(v), "d"(v), "d"(v));
    }
  }
}

// duplicate detection in an L2-resident bitmap (seen / dup bit per key):
// `n` random keys below `nkeys`, one ATOM (OR, old value used) per key and a
// RED into the dup bitmap for repeats
__global__ void dedup_bits(uint32_t* seen, uint32_t* dup, uint64_t nkeys, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = mix(i * 0x9E3779B97F4A7C15ULL) % nkeys;
    const uint32_t bit = 1u << (k & 31);
    if (atomicOr(seen + (k >> 5), bit) & bit) atomicOr(dup + (k >> 5), bit);
  }
}
__global__ void dedup_read(const uint32_t* dup, uint64_t nkeys, int64_t n, uint8_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = mix(i * 0x9E3779B97F4A7C15ULL) % nkeys;
    flag[i] = (dup[k >> 5] >> (k & 31)) & 1;
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
  run("store16", [&] { scatter_wide<16><<<grid, blk>>>((double*)tab, nrec, n); });
  run("store32", [&] { scatter_wide<32><<<grid, blk>>>((double*)tab, nrec, n); });
  run("store64", [&] { scatter_wide<64><<<grid, blk>>>((double*)tab, nrec, n); });
  {
    // one position group: 16 positions x P = 2^20 touches into 16 x 15 x 2^20 keys
    const int64_t ng = 16LL << 20;
    const uint64_t nkeys = 16ULL * 15 * (1 << 20);
    uint32_t* seen = reinterpret_cast<uint32_t*>(tab);
    uint32_t* dup = seen + nkeys / 32 + 1024;
    uint8_t* flag = reinterpret_cast<uint8_t*>(dup + nkeys / 32 + 1024);
    const size_t bm = nkeys / 8 + 4096;
    printf("-- dedup group: %lld keys-touches, bitmaps 2 x %.1f MB\n", (long long)ng, bm / 1e6);
    run("dedup_memset", [&] { cudaMemsetAsync(seen, 0, 2 * bm); });
    run("dedup_bits", [&] { dedup_bits<<<grid, blk>>>(seen, dup, nkeys, ng); });
    run("dedup_read", [&] { dedup_read<<<grid, blk>>>(dup, nkeys, ng, flag); });
  }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// DFMA latency / per-warp issue micro-benchmark (B200): W warps per SMSP,
// C independent dependency chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0) / (iters * 8.0 * C);
}

template <int C>
void run(int warps_per_smsp, double* d) {
  const int iters = 4096;
  chains<C><<<148, 128 * warps_per_smsp>>>(d, iters, 0.999, 0.001);
  cudaDeviceSynchronize();
  double h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("chains=%2d warps/SMSP=%d : %.2f cycles per DFMA per warp (SMSP: %.2f cycles/DFMA)\n", C,
         warps_per_smsp, h[1], h[1] / warps_per_smsp);
}

int main() {
  double* d;
  cudaMalloc(&d, 16);
  for (int w : {1, 2, 3, 4}) {
    run<1>(w, d);
    run<2>(w, d);
    run<4>(w, d);
    run<8>(w, d);
    run<16>(w, d);
  }
  return 0;
}

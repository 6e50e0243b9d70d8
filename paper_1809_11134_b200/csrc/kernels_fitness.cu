// Fitness / composition of explicit gate lists (GA genomes, best-circuit
// readout, the functional API).  Replaces compose_gates + fitness_value
// (gates.py:187-195, fitness.py:36-49) for a batch of circuits.
#include <map>
#include <mutex>

#include "isq_internal.h"
#include "fitness_multi.cuh"
#include "fitness_warp.cuh"
#include "unitary_warp.cuh"

namespace isq {

struct ChunkShared {
  int op[32];
  double a[32];
  double b[32];
};

// Fitness only (the hot path).  MINB = 6 resident 2-warp blocks per SM
// (<= 168 registers) gives 3 warps per scheduler for the n = 5
// register-resident state (measured: 2 warps per scheduler at 244 registers
// is 11 % slower).
#ifdef ISQ_FIT_MAXNREG  // register-cap experiments (tools/): replaces the min-blocks bound
#define ISQ_FIT_BOUNDS __maxnreg__(ISQ_FIT_MAXNREG)
#else
#define ISQ_FIT_BOUNDS __launch_bounds__(kFitThreads, MINB)
#endif
template <int NQ, int MINB, class R>
__global__ void ISQ_FIT_BOUNDS
    fitness_fast_kernel(int64_t count, int L, const uint8_t* __restrict__ codes,
                        const double* __restrict__ thetas, const double2* __restrict__ target,
                        double* __restrict__ fitness, const int32_t* __restrict__ stop, int* bad_code,
                        unsigned long long* dyn) {
  using G = Geo<NQ>;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ FitScratch<NQ, R> sh[kFitWarps];
  if (stop != nullptr && *stop) return;
  for (int i = threadIdx.x; i < G::D * G::D; i += blockDim.x) Ts[i] = target[i];
  __syncthreads();
  fitness_rows_fast<NQ, R>(count, L, codes, thetas, Ts, sh, fitness, kFitWarps, bad_code, dyn);
}

// fp32 variant: the column of S in 64 float registers: 8 resident 2-warp
// blocks per SM (<= 128 registers, 4 warps per scheduler).

// Composition with the exact global phase (compose_gates readout) + fitness.
template <int NQ>
__global__ void __launch_bounds__(kThreadsPerBlock)
    compose_kernel(int64_t count, int L, const uint8_t* __restrict__ codes,
                         const double* __restrict__ thetas, const double2* __restrict__ target,
                         double* __restrict__ fitness, double2* __restrict__ unitary) {
  using G = Geo<NQ>;
  __shared__ double2 Ts[G::D * G::D];
  __shared__ ChunkShared sh[kWarpsPerBlock];
  for (int i = threadIdx.x; i < G::D * G::D; i += blockDim.x) Ts[i] = target[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  ChunkShared& cs = sh[wib];
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t c = (int64_t)blockIdx.x * kWarpsPerBlock + wib; c < count; c += nwarps) {
    WarpUnitary<NQ> st;
    st.set_identity(lane);
    double mant = 1.0, phase = 0.0;
    const uint8_t* cc = codes + c * (int64_t)L;
    const double* ct = thetas + c * (int64_t)L;
    for (int base = 0; base < L; base += 32) {
      const int p = base + lane;
      GateParam g;
      if (p < L) {
        g = gate_param<NQ>((int)cc[p], ct[p]);
      } else {
        g.op = -1;
        g.a = g.b = 0.0;
        g.scale = 1.0;
        g.phase = 0.0;
      }
      int ex;
      mant = frexp(mant * warp_prod(g.scale), &ex);
      st.scale_all(ldexp(1.0, ex));
      if (unitary) phase += warp_sum(g.phase);
      cs.op[lane] = g.op;
      cs.a[lane] = g.a;
      cs.b[lane] = g.b;
      __syncwarp();
      const int nq = min(32, L - base);
#pragma unroll 1
      for (int q = 0; q < nq; ++q) st.apply(cs.op[q], cs.a[q], cs.b[q], lane);
      __syncwarp();
    }
    double ore, oim;
    st.overlap(Ts, lane, ore, oim);
    const double ov = fabs(mant) * hypot(ore, oim);
    if (lane == 0) fitness[c] = fitness_from_overlap(ov, G::D);
    if (unitary != nullptr && lane < G::ACTIVE) {
      double ps, pc;
      sincos(phase, &ps, &pc);
      const double fr = mant * pc, fi = mant * ps;
      const int j = lane & (G::D - 1);
      const int h = (lane >> NQ) & (G::LPC - 1);
      double2* U = unitary + c * (int64_t)(G::D * G::D);
#pragma unroll
      for (int r = 0; r < G::E; ++r) {
        const double xr = st.re[r], xi = st.im[r];
        U[(h * G::E + r) * G::D + j] = make_double2(fr * xr - fi * xi, fr * xi + fi * xr);
      }
    }
  }
}

// fitness_value on explicit matrices (fitness.py:36-49): one block per pair
// (S_c, T); block reduction of conj(S) * T in a fixed order.
__global__ void __launch_bounds__(256)
    overlap_fitness_kernel(int64_t D, int64_t count, const double2* __restrict__ S,
                           const double2* __restrict__ T, double* __restrict__ out) {
  __shared__ double red_r[256], red_i[256];
  const int64_t DD = D * D;
  for (int64_t c = blockIdx.x; c < count; c += gridDim.x) {
    const double2* s = S + c * DD;
    double ar = 0.0, ai = 0.0;
    for (int64_t i = threadIdx.x; i < DD; i += blockDim.x) {
      const double2 x = s[i], t = T[i];
      ar = fma(x.x, t.x, ar);
      ar = fma(x.y, t.y, ar);
      ai = fma(x.x, t.y, ai);
      ai = fma(-x.y, t.x, ai);
    }
    red_r[threadIdx.x] = ar;
    red_i[threadIdx.x] = ai;
    __syncthreads();
    for (int off = 128; off >= 1; off >>= 1) {
      if (threadIdx.x < off) {
        red_r[threadIdx.x] += red_r[threadIdx.x + off];
        red_i[threadIdx.x] += red_i[threadIdx.x + off];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = fitness_from_overlap(hypot(red_r[0], red_i[0]), (int)D);
    __syncthreads();
  }
}

isq_status launch_overlap_fitness(int64_t D, int64_t count, const double* S, const double* T,
                                  double* out, cudaStream_t stream) {
  if (count <= 0) return ISQ_OK;
  const int grid = (int)(count < 65535 ? count : 65535);
  overlap_fitness_kernel<<<grid, 256, 0, stream>>>(D, count, reinterpret_cast<const double2*>(S),
                                                   reinterpret_cast<const double2*>(T), out);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

// ------------------------------------------------------ n = 6 .. 13 ---
// numberOfWires above the register-resident kernels (the reference allows up
// to its 4^n <= 2^26 cap, engine.py:43,60-63): one block per circuit with
// the 2^n x 2^n state in global scratch (L1 / L2 resident per block), every
// gate applied as what it is on all columns at once -- a rotation as D/2
// row-pair butterflies per column, Rz / ZZ as row phases -- with the exact
// gate matrices (gates.py:60-116: cos(th/2) I - i sin(th/2) sigma,
// exp(-i th/2 signs)).  kCompose: S from I, gates in order, the unitary and
// its overlap with T out (compose_gates + fitness_value); otherwise
// M = S^dagger T from T with the adjoints in reverse order and the fitness
// from the trace (the same adjoint evaluation as the fast kernels).
constexpr int kGenericThreads = 256;

__device__ __forceinline__ void generic_apply(double2* M, int n, int code, double th) {
  const int D = 1 << n;
  const int64_t DD = (int64_t)D * D;
  double s, c;
  sincos(0.5 * th, &s, &c);
  if (code < 3 * n && code % 3 != 2) {  // Rx / Ry on wire w: row bit n - w
    const int b = n - 1 - code / 3;
    const bool rx = code % 3 == 0;
    const int m = 1 << b;
    for (int64_t idx = threadIdx.x; idx < DD / 2; idx += blockDim.x) {
      const int64_t i = idx / D;                                // row pair
      const int col = (int)(idx - i * D);
      const int64_t r0 = ((i >> b) << (b + 1)) | (i & (m - 1));  // bit b cleared
      double2* pa = M + r0 * D + col;
      double2* pb = pa + (int64_t)m * D;
      const double2 a = *pa, bb = *pb;
      if (rx) {  // [[c, -is], [-is, c]]
        *pa = make_double2(c * a.x + s * bb.y, c * a.y - s * bb.x);
        *pb = make_double2(c * bb.x + s * a.y, c * bb.y - s * a.x);
      } else {  // [[c, -s], [s, c]]
        *pa = make_double2(c * a.x - s * bb.x, c * a.y - s * bb.y);
        *pb = make_double2(s * a.x + c * bb.x, s * a.y + c * bb.y);
      }
    }
    return;
  }
  int mask;
  if (code < 3 * n) {
    mask = 1 << (n - 1 - code / 3);  // Rz: e^{-i th/2} on bit 0, e^{+i th/2} on bit 1
  } else {
    int i = 1, t = code - 3 * n;
    while (t >= n - i) {
      t -= n - i;
      ++i;
    }
    mask = (1 << (n - i)) | (1 << (n - (i + 1 + t)));  // ZZ: e^{-i th/2} when the bits agree
  }
  for (int64_t idx = threadIdx.x; idx < DD; idx += blockDim.x) {
    const int r = (int)(idx / D);
    const int par = __popc(r & mask) & 1;
    const double sg = par ? 1.0 : -1.0;  // phase e^{i sg th/2}
    const double2 x = M[idx];
    const double ps = sg * s;
    M[idx] = make_double2(c * x.x - ps * x.y, c * x.y + ps * x.x);
  }
}

// GenericInput: the circuits' codes / angles; with `parity` set (the GA's
// generation counter) the odd generations read the alternate buffers.
struct GenericInput {
  const uint8_t* codes;
  const double* thetas;
  const uint8_t* codes_alt;
  const double* thetas_alt;
  const uint64_t* parity;
  const double2* init;  // kCompose: starting matrices (count x D x D) instead of I (apply_gate)
};

template <bool kCompose>
__global__ void __launch_bounds__(kGenericThreads)
    fitness_generic_kernel(int n, int L, int64_t count, GenericInput in, const double2* __restrict__ target,
                           double* __restrict__ fitness, double2* __restrict__ unitary, double2* scratch,
                           const int32_t* __restrict__ stop, int* bad_code) {
  __shared__ double red_r[kGenericThreads], red_i[kGenericThreads];
  if (stop != nullptr && *stop) return;
  const bool alt = in.parity != nullptr && (*in.parity & 1);
  const uint8_t* __restrict__ codes = alt ? in.codes_alt : in.codes;
  const double* __restrict__ thetas = alt ? in.thetas_alt : in.thetas;
  const int D = 1 << n;
  const int64_t DD = (int64_t)D * D;
  const int ncodes = 3 * n + n * (n - 1) / 2;
  double2* M = scratch + (int64_t)blockIdx.x * DD;
  for (int64_t cc = blockIdx.x; cc < count; cc += gridDim.x) {
    for (int64_t i = threadIdx.x; i < DD; i += blockDim.x) {
      if (kCompose) {
        const int64_t r = i / D;
        M[i] = in.init ? in.init[cc * DD + i] : make_double2(r == i - r * D ? 1.0 : 0.0, 0.0);
      } else {
        M[i] = target[i];
      }
    }
    bool bad = false;
    __syncthreads();
    for (int q = 0; q < L; ++q) {
      const int p = kCompose ? q : L - 1 - q;  // adjoints in reverse order
      const int code = codes[cc * L + p];
      const double th = thetas[cc * L + p];
      if (code >= ncodes) {
        bad = true;
      } else {
        generic_apply(M, n, code, kCompose ? th : -th);
      }
      __syncthreads();
    }
    double ar = 0.0, ai = 0.0;
    if (kCompose) {  // fitness_value(S, T): |sum conj(S) * T|
      for (int64_t i = threadIdx.x; i < DD; i += blockDim.x) {
        const double2 x = M[i], t = target[i];
        ar = fma(x.x, t.x, ar);
        ar = fma(x.y, t.y, ar);
        ai = fma(x.x, t.y, ai);
        ai = fma(-x.y, t.x, ai);
        unitary[cc * DD + i] = x;
      }
    } else {  // |tr(S^dagger T)|
      for (int j = threadIdx.x; j < D; j += blockDim.x) {
        const double2 x = M[(int64_t)j * D + j];
        ar += x.x;
        ai += x.y;
      }
    }
    red_r[threadIdx.x] = ar;
    red_i[threadIdx.x] = ai;
    __syncthreads();
    for (int off = kGenericThreads / 2; off >= 1; off >>= 1) {
      if (threadIdx.x < off) {
        red_r[threadIdx.x] += red_r[threadIdx.x + off];
        red_i[threadIdx.x] += red_i[threadIdx.x + off];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      fitness[cc] = bad ? __longlong_as_double(0x7ff8000000000000LL)
                        : fitness_from_overlap(hypot(red_r[0], red_i[0]), D);
      if (bad && bad_code) atomicOr(bad_code, 1);
    }
    __syncthreads();
  }
}

// Scratch of the generic kernel per (device, stream): launches on one stream
// are ordered, so they may share it; concurrent streams never do.  Grow-only,
// kept for the process lifetime (n = 10: 16 MB per resident circuit).
static double2* generic_scratch(size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<double2*, size_t>> pool;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto& e = pool[std::make_pair(dev, stream)];
  if (e.second < bytes) {
    if (e.first) {
      cudaStreamSynchronize(stream);  // earlier launches on this stream still read it
      cudaFree(e.first);
    }
    e.first = nullptr;
    e.second = 0;
    if (cudaMalloc((void**)&e.first, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    e.second = bytes;
  }
  return e.first;
}

isq_status launch_fitness_generic(int n, int L, int64_t count, const uint8_t* codes, const double* thetas,
                                  const double* target, double* fitness, double* unitary, const int32_t* stop,
                                  cudaStream_t stream, int* bad_code, const uint8_t* codes_alt,
                                  const double* thetas_alt, const uint64_t* parity, const double* init) {
  if (count <= 0) return ISQ_OK;
  const GenericInput in{codes, thetas, codes_alt, thetas_alt, parity, reinterpret_cast<const double2*>(init)};
  const int64_t DD = (int64_t)1 << (2 * n);
  int64_t grid = (int64_t)num_sms() * (n <= 8 ? 2 : 1);
  if (grid > count) grid = count;
  // n >= 11: one resident matrix is 64 MB .. 1 GB (n = 13); bound the
  // scratch by a quarter of the free memory (at least one circuit)
  size_t free_b = 0, total_b = 0;
  if (n >= 11 && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
    const int64_t fit = (int64_t)(free_b / 4 / (size_t)(DD * sizeof(double2)));
    if (grid > fit) grid = fit < 1 ? 1 : fit;
  }
  double2* scratch = generic_scratch((size_t)grid * DD * sizeof(double2), stream);
  if (!scratch) {
    set_error("cannot allocate the n >= 6 fitness scratch");
    return ISQ_ERR_CUDA;
  }
  const double2* T = reinterpret_cast<const double2*>(target);
  if (unitary)
    fitness_generic_kernel<true><<<(unsigned)grid, kGenericThreads, 0, stream>>>(
        n, L, count, in, T, fitness, reinterpret_cast<double2*>(unitary), scratch, stop, bad_code);
  else
    fitness_generic_kernel<false><<<(unsigned)grid, kGenericThreads, 0, stream>>>(
        n, L, count, in, T, fitness, nullptr, scratch, stop, bad_code);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int persistent_grid(const void* kernel, size_t dyn_smem, int64_t work_warps, int warps_per_block) {
  const int num_sms = isq::num_sms();
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 32 * warps_per_block, dyn_smem);
  if (per_sm <= 0) per_sm = 1;
  const int64_t need = (work_warps + warps_per_block - 1) / warps_per_block;
  const int64_t full = (int64_t)num_sms * per_sm;
  int64_t g = need < full ? need : full;
  return (int)(g < 1 ? 1 : g);
}

template <int NQ>
static isq_status launch_nq(int L, int64_t count, const uint8_t* codes, const double* thetas,
                            const double* target, double* fitness, double* unitary,
                            cudaStream_t stream) {
  const void* k = (const void*)compose_kernel<NQ>;
  const int grid = persistent_grid(k, 0, count);
  compose_kernel<NQ><<<grid, kThreadsPerBlock, 0, stream>>>(
      count, L, codes, thetas, reinterpret_cast<const double2*>(target), fitness,
      reinterpret_cast<double2*>(unitary));
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

template <int NQ, int MINB, class R>
static isq_status launch_fast(int L, int64_t count, const uint8_t* codes, const double* thetas,
                              const double* target, double* fitness, const int32_t* stop,
                              int blocks_per_sm, cudaStream_t stream, int* bad_code,
                              unsigned long long* dyn) {
  const void* k = (const void*)fitness_fast_kernel<NQ, MINB, R>;
  const int64_t warps = (count + kFitCPW<NQ> - 1) / kFitCPW<NQ>;
  int grid = persistent_grid(k, 0, warps, kFitWarps);
  if (blocks_per_sm > 0 && grid > num_sms() * blocks_per_sm) grid = num_sms() * blocks_per_sm;
  fitness_fast_kernel<NQ, MINB, R><<<grid, kFitThreads, 0, stream>>>(
      count, L, codes, thetas, reinterpret_cast<const double2*>(target), fitness, stop, bad_code, dyn);
  ISQ_CUDA_TRY(cudaGetLastError());
  return ISQ_OK;
}

template <int NQ>
static isq_status launch_fast_prec(int L, int64_t count, const uint8_t* codes, const double* thetas,
                                   const double* target, double* fitness, const int32_t* stop,
                                   int blocks_per_sm, int precision, cudaStream_t stream, int* bad,
                                   unsigned long long* dyn) {
  if (precision == ISQ_PRECISION_FP32)
    return launch_fast<NQ, fit_min_blocks<NQ, float>(), float>(L, count, codes, thetas, target, fitness, stop,
                                                    blocks_per_sm, stream, bad, dyn);
  return launch_fast<NQ, fit_min_blocks<NQ, double>(), double>(L, count, codes, thetas, target, fitness, stop,
                                                  blocks_per_sm, stream, bad, dyn);
}

isq_status launch_fitness_batch_stoppable(int n, int L, int64_t count, const uint8_t* codes,
                                          const double* thetas, const double* target,
                                          double* fitness, const int32_t* stop,
                                          cudaStream_t stream, int blocks_per_sm, int precision,
                                          int* bad_code, unsigned long long* dyn) {
  if (count <= 0) return ISQ_OK;
  const int b = blocks_per_sm, p = precision;
  int* bc = bad_code;
  if (dyn != nullptr) ISQ_CUDA_TRY(cudaMemsetAsync(dyn, 0, sizeof(*dyn), stream));
  switch (n) {
    case 2: return launch_fast_prec<2>(L, count, codes, thetas, target, fitness, stop, b, p, stream, bc, dyn);
    case 3: return launch_fast_prec<3>(L, count, codes, thetas, target, fitness, stop, b, p, stream, bc, dyn);
    case 4: return launch_fast_prec<4>(L, count, codes, thetas, target, fitness, stop, b, p, stream, bc, dyn);
    case 5: return launch_fast_prec<5>(L, count, codes, thetas, target, fitness, stop, b, p, stream, bc, dyn);
    default:
      if (n > ISQ_MAX_FAST_WIRES && n <= ISQ_MAX_WIRES)  // fp64 only (the fp32 variant is a fast-kernel option)
        return launch_fitness_generic(n, L, count, codes, thetas, target, fitness, nullptr, stop, stream, bc);
      set_error("numberOfWires outside the supported range 2..13");
      return ISQ_ERR_UNSUPPORTED;
  }
}

isq_status launch_fitness_batch(int n, int L, int64_t count, const uint8_t* codes,
                                const double* thetas, const double* target, double* fitness,
                                double* unitary, cudaStream_t stream, int precision, int* bad_code) {
  if (count <= 0) return ISQ_OK;
  if (unitary == nullptr)
    return launch_fitness_batch_stoppable(n, L, count, codes, thetas, target, fitness, nullptr, stream,
                                          0, precision, bad_code);
  switch (n) {  // composition readout: always fp64
    case 2: return launch_nq<2>(L, count, codes, thetas, target, fitness, unitary, stream);
    case 3: return launch_nq<3>(L, count, codes, thetas, target, fitness, unitary, stream);
    case 4: return launch_nq<4>(L, count, codes, thetas, target, fitness, unitary, stream);
    case 5: return launch_nq<5>(L, count, codes, thetas, target, fitness, unitary, stream);
    default:
      if (n > ISQ_MAX_FAST_WIRES && n <= ISQ_MAX_WIRES)
        return launch_fitness_generic(n, L, count, codes, thetas, target, fitness, unitary, nullptr, stream,
                                      bad_code);
      set_error("numberOfWires=" + std::to_string(n) + " is outside the supported range 2..13");
      return ISQ_ERR_UNSUPPORTED;
  }
}

}  // namespace isq

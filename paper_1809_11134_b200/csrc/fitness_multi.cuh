// Fitness of small circuits (n <= 4): several circuits per warp, one column
// per lane, every row in registers.
//
// Replaces evaluate_circuit / fitness_value (engine.py:187-199,
// fitness.py:36-49) and GA decode + score (ga.py:76-78,167-170) for
// n = 2..4 in the throughput kernels.  The n = 5 evaluator (fitness_warp.cuh)
// gives one circuit a whole warp, lane = column; at n <= 4 that layout
// spreads each D = 2^n row column over 32 / D lanes, pays a shuffle per
// register row for every rotation on a lane-held row bit, and pays the
// per-gate setup for one circuit per warp.  Here a warp holds CPW = 32 / D
// circuits side by side: lane l = g D + j is column j of circuit g of the
// warp's batch, with all D rows of that column in registers, so every
// rotation is register-local (the 3-shear lifting of fitness_warp.cuh) and
// the per-gate bookkeeping is shared by CPW circuits.
//
// The circuits of a warp run different gate sequences.  Each position is one
// step for the whole warp: the diagonal gates (Rz, ZZ) only multiply the
// pending row phase lane j carries for row j (see fitness_warp.cuh), the
// rotations of the step compute their flush factors with per-lane shuffles
// inside their group, and the register lifting runs in a switch on the
// rotation's row bit, so groups rotating on different bits serialise.  At
// the QEQEA and GA gate mixes a step holds ~1.1 distinct rotation cases
// (n = 3, 4 circuits) or ~0.5 (n = 4, 2 circuits), about what one circuit
// per warp would execute, while every other cost is divided by CPW.
#pragma once
#include <type_traits>

#include "fitness_warp.cuh"

namespace isq {

template <int NQ>
struct MGeo {
  static constexpr int D = 1 << NQ;
  static constexpr int CPW = 32 / D;        // circuits per warp
  static constexpr int CHUNK = 64 / CPW;    // positions per circuit per chunk (64 gates per warp)
  static constexpr int GATES = CPW * CHUNK; // = 64: two per lane
};

// Per-warp shared scratch of one chunk: gate k = g * CHUNK + q (circuit g of
// the batch, step q).
template <int NQ, class R>
struct MultiChunk {
  using R2 = typename Cplx<R>::T;
  R2 e1[MGeo<NQ>::GATES];       // rotation: (p, q) of the lifting; diagonal: e^{-i r/2}
  uint32_t rpar[MGeo<NQ>::GATES];  // diagonal: bit r = parity of row r under the gate mask
  int info[MGeo<NQ>::GATES];       // GT_* | row bit << 8
  R2 fac[32];                      // flush factors, lane g D + r = row r of circuit g
};

template <int NQ, class R>
struct MultiEval {
  using MG = MGeo<NQ>;
  using R2 = typename Cplx<R>::T;
  static constexpr int D = MG::D;
  R re[D], im[D];  // column j of circuit g
  R wr, wi;        // pending phase of row j of circuit g

  __device__ __forceinline__ void begin(const double2* __restrict__ T, int j) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double tx, ty;  // volatile: keeps the column out of the loop-invariant registers
      asm volatile("ld.v2.f64 {%0, %1}, [%2];" : "=d"(tx), "=d"(ty) : "l"(T + r * D + j));
      re[r] = R(tx);
      im[r] = R(ty);
    }
    wr = R(1);
    wi = R(0);
  }

  __device__ __forceinline__ void cmul(int r, R fc, R fs) {
    const R t1 = fs * im[r];
    const R t2 = fs * re[r];
    re[r] = fma(fc, re[r], -t1);
    im[r] = fma(fc, im[r], t2);
  }

  // Flush of row bit B fused with the Rx lifting on it (fitness_warp.cuh
  // flush_lift, all rows in registers).
  template <int B>
  __device__ __forceinline__ void flush_lift(const R2* fac, R p, R q) {
    constexpr int m = 1 << B;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      if (r & m) continue;
      const int r1 = r | m;
      const R2 f = fac[r1];
      cmul(r1, f.x, f.y);
      re[r] = fma(p, im[r1], re[r]);
      im[r1] = fma(q, re[r], im[r1]);
      re[r] = fma(p, im[r1], re[r]);
      re[r1] = fma(p, im[r], re[r1]);
      im[r] = fma(q, re[r1], im[r]);
      re[r1] = fma(p, im[r], re[r1]);
    }
  }

  __device__ __forceinline__ void flush_rotate(int b, const R2* fac, R p, R q) {
    switch (b) {
      case 0: flush_lift<0>(fac, p, q); break;
      case 1: if constexpr (NQ > 1) flush_lift<1>(fac, p, q); break;
      case 2: if constexpr (NQ > 2) flush_lift<2>(fac, p, q); break;
      case 3: if constexpr (NQ > 3) flush_lift<3>(fac, p, q); break;
      default: break;
    }
  }

  // Lockstep alternative to run_chunk (the latency-bound single-block kernels,
  // one circuit per warp, where run_chunk's bit alignment is pure overhead):
  // one step of every circuit of the warp, gate k = g CHUNK + q of the chunk,
  // the rotation case chosen per group.  Same arithmetic per circuit.
  __device__ __forceinline__ void step(const MultiChunk<NQ, R>& sm, R2* fac, int k, int lane, int j) {
    const int inf = sm.info[k];
    R2 e = sm.e1[k];
    const bool rot = inf != GT_DIAG;
    if (!__any_sync(0xffffffffu, rot)) {  // every circuit diagonal at this step
      e.y = flip_sign_bit(e.y, sm.rpar[k] << (31 - j));
      const R t = wr * e.y;
      wr = fma(wr, e.x, -wi * e.y);
      wi = fma(wi, e.x, t);
      return;
    }
    const int b = inf >> 8;
    const int m = rot ? 1 << b : 0;
    const bool ry = (inf & 3) == GT_RY;
    // rotation: rows with bit b set take the flush factor w_r conj(w_{r^m})
    // (times -i for Ry: S^dagger) and carry their partner's phase (times i)
    const R orr = __shfl_sync(0xffffffffu, ry ? -wi : wr, lane ^ m);
    const R ori = __shfl_sync(0xffffffffu, ry ? wr : wi, lane ^ m);
    if (rot) {
      fac[lane] = Cplx<R>::make(fma(wr, orr, wi * ori), fma(wi, orr, -wr * ori));
      if (j & m) {
        wr = orr;
        wi = ori;
      }
    } else {
      e.y = flip_sign_bit(e.y, sm.rpar[k] << (31 - j));
      const R t = wr * e.y;
      wr = fma(wr, e.x, -wi * e.y);
      wi = fma(wi, e.x, t);
    }
    __syncwarp();
    if (rot) flush_rotate(b, fac + (lane & ~(D - 1)), e.x, e.y);
    __syncwarp();
  }

  // Physical register bit of logical row bit lb (pmap: 4 bits per logical bit).
  static __device__ __forceinline__ int phys_bit(int pmap, int lb) { return (pmap >> (4 * lb)) & 15; }

  // Exchange physical row bits 0 and B of this lane's column where `doit`:
  // rows r with bit 0 set and bit B clear trade places with r ^ (1 | 2^B).
  template <int B>
  __device__ __forceinline__ void swap_bits(bool doit) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
      if (!(r & 1) || (r & (1 << B))) continue;
      const int r2 = r ^ 1 ^ (1 << B);
      const R a = re[r], b = re[r2], c = im[r], d = im[r2];
      re[r] = doit ? b : a;
      re[r2] = doit ? a : b;
      im[r] = doit ? d : c;
      im[r2] = doit ? c : d;
    }
  }

  // One chunk of every circuit of the warp (gate k = g CHUNK + q, q < nq).
  // The circuits advance independently, each through its own gate list:
  // a group first runs its diagonal gates up to its next rotation (they only
  // touch the pending phase), then every group standing at a rotation
  // applies it in the same pass.  To make that pass the same code for every
  // group, each group first moves the rotation's row bit to physical bit 0
  // (an exchange of register halves, under a per-lane predicate), keeping
  // the logical -> physical bit map in `pmap`, the logical index of the row
  // whose phase the lane carries in `lrow`, and moving the phases with the
  // rows.  A warp then makes max over its circuits of their rotation counts
  // lifting passes (n = 3, L = 16, 4 circuits: ~7.6) instead of one divergent
  // case per distinct rotation bit per position (~18), and every pass does the
  // same arithmetic per row pair as before, so the fitness is bit-identical.
  __device__ __forceinline__ void run_chunk(const MultiChunk<NQ, R>& sm, R2* fac, int kb, int nq, int lane, int j,
                                            int& pmap, int& lrow) {
    const int gbase = lane & ~(D - 1);
    int qg = 0;  // this circuit's next step (uniform within the group)
    while (true) {
      int inf = qg < nq ? sm.info[kb + qg] : GT_DIAG;
      while (qg < nq && inf == GT_DIAG) {  // diagonal run: the pending phase only
        R2 e = sm.e1[kb + qg];
        e.y = flip_sign_bit(e.y, sm.rpar[kb + qg] << (31 - lrow));
        const R t = wr * e.y;
        wr = fma(wr, e.x, -wi * e.y);
        wi = fma(wi, e.x, t);
        ++qg;
        inf = qg < nq ? sm.info[kb + qg] : GT_DIAG;
      }
      const bool pending = qg < nq;
      if (!__any_sync(0xffffffffu, pending)) break;
      // align: the rotation's row bit to physical bit 0
      const int lb = inf >> 8;
      const int pb = pending ? phys_bit(pmap, lb) : 0;
#pragma unroll
      for (int b = 1; b < NQ; ++b) {
        const bool doit = pb == b;
        if (!__any_sync(0xffffffffu, doit)) continue;
        switch (b) {
          case 1: swap_bits<1>(doit); break;
          case 2: if constexpr (NQ > 2) swap_bits<2>(doit); break;
          case 3: if constexpr (NQ > 3) swap_bits<3>(doit); break;
          default: break;
        }
        // the phases and logical labels move with their rows
        const bool moved = doit && (((j ^ (j >> b)) & 1) != 0);  // bits 0 and b of row j differ
        const int src = gbase + (moved ? j ^ 1 ^ (1 << b) : j);
        wr = __shfl_sync(0xffffffffu, wr, src);
        wi = __shfl_sync(0xffffffffu, wi, src);
        lrow = __shfl_sync(0xffffffffu, lrow, src);
        if (doit) {  // logical bit at physical 0 <-> logical bit lb (at physical b)
          int l0 = 0;
#pragma unroll
          for (int x = 0; x < NQ; ++x)
            if (phys_bit(pmap, x) == 0) l0 = x;
          pmap = (pmap & ~(15 << (4 * l0)) & ~(15 << (4 * lb))) | (b << (4 * l0));
        }
      }
      // rotation on physical bit 0: rows with it set take w_r conj(w_{r^1})
      // (times -i for Ry: S^dagger) and carry their partner's phase (times i)
      const bool ry = (inf & 3) == GT_RY;
      const R orr = __shfl_xor_sync(0xffffffffu, ry ? -wi : wr, 1);
      const R ori = __shfl_xor_sync(0xffffffffu, ry ? wr : wi, 1);
      R2 e = Cplx<R>::make(R(0), R(0));
      if (pending) {
        fac[lane] = Cplx<R>::make(fma(wr, orr, wi * ori), fma(wi, orr, -wr * ori));
        if (j & 1) {
          wr = orr;
          wi = ori;
        }
        e = sm.e1[kb + qg];
        ++qg;
      }
      __syncwarp();
      if (pending) flush_lift<0>(fac + gbase, e.x, e.y);
      __syncwarp();
    }
  }

  // |tr(S^dagger T)| of circuit g: sum over its lanes (columns j) of
  // e^{i phi} M[j][j], the diagonal entry sitting in physical row pj.
  __device__ __forceinline__ double finish(int lane, int j, int pmap) {
    int pj = 0;
#pragma unroll
    for (int lb = 0; lb < NQ; ++lb) pj |= ((j >> lb) & 1) << phys_bit(pmap, lb);
    R xr = re[0], xi = im[0];
#pragma unroll
    for (int r = 1; r < D; ++r) {
      xr = sel(pj == r, re[r], xr);
      xi = sel(pj == r, im[r], xi);
    }
    const int src = (lane & ~(D - 1)) + pj;  // the lane carrying physical row pj's phase
    const double wx = __shfl_sync(0xffffffffu, wr, src), wy = __shfl_sync(0xffffffffu, wi, src);
    const double dr = xr, di = xi;
    double ar = fma(wx, dr, -wy * di), ai = fma(wx, di, wy * dr);
#pragma unroll
    for (int off = D / 2; off >= 1; off >>= 1) {
      ar += __shfl_xor_sync(0xffffffffu, ar, off);
      ai += __shfl_xor_sync(0xffffffffu, ai, off);
    }
    return fitness_from_overlap(hypot(ar, ai), D);
  }
};

// Bits [lo, hi) of a warp mask (clipped to [0, 32)).
__device__ __forceinline__ unsigned range_mask(int lo, int hi) {
  lo = lo < 0 ? 0 : lo;
  hi = hi > 32 ? 32 : hi;
  if (hi <= lo) return 0u;
  const unsigned w = (unsigned)(hi - lo);
  return (w == 32 ? 0xffffffffu : ((1u << w) - 1u)) << lo;
}

// Grid-stride (or counter-scheduled, `dyn`) body of the fitness kernels for
// n <= ISQ_MULTI_MAXNQ: warp batches of `cpw` (<= CPW) consecutive circuits,
// groups g >= cpw idle.  A circuit's arithmetic does not depend on cpw, so the
// latency-bound single-block kernels run fewer circuits per warp (more warps,
// fewer serialised rotation cases per step) with bit-identical results.
template <int NQ, class R = double, bool kLockstep = false>
__device__ __forceinline__ void fitness_rows_multi(int64_t count, int L, const uint8_t* __restrict__ codes,
                                                   const double* __restrict__ thetas,
                                                   const double2* __restrict__ Ts, MultiChunk<NQ, R>* sh,
                                                   double* __restrict__ fitness, int warps_per_block,
                                                   int* bad_code = nullptr, unsigned long long* dyn = nullptr,
                                                   int cpw = MGeo<NQ>::CPW) {
  using MG = MGeo<NQ>;
  using E = FastEval<NQ, R>;  // gate preparation (E::prepare) is shared with n = 5
  using R2 = typename Cplx<R>::T;
  constexpr int D = MG::D, CHUNK = MG::CHUNK;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int g = lane / D, j = lane & (D - 1);
  MultiChunk<NQ, R>& cs = sh[wib];
  const int64_t nwarps = (int64_t)gridDim.x * warps_per_block;
  auto grab = [&]() -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(dyn, (unsigned long long)cpw);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  int64_t c0 = dyn ? grab() : ((int64_t)blockIdx.x * warps_per_block + wib) * cpw;
  // the two gates this lane prepares per chunk: k0 = lane, k1 = lane + 32
  // (circuit k / CHUNK of the batch, step k % CHUNK); loaded one chunk ahead
  auto load = [&](int64_t cb, int nb, int k, int& code, double& th) {
    const int gg = k / CHUNK, q = k % CHUNK;
    const int nq = min(CHUNK, L - nb);
    code = -2;  // neutral (past the end of the circuit or the batch)
    th = 0.0;
    const int64_t c = cb + gg;
    if (q < nq && gg < cpw && c < count) {
      const int64_t at = c * (int64_t)L + (L - 1 - nb - q);  // adjoint order: last position first
      code = codes[at];
      th = -thetas[at];
    }
  };
  int code0, code1;
  double th0, th1;
  // lanes whose gate k = lane + 32 h belongs to circuit g of the batch
  const unsigned own0 = range_mask(g * CHUNK, (g + 1) * CHUNK);
  const unsigned own1 = range_mask(g * CHUNK - 32, (g + 1) * CHUNK - 32);
  load(c0, 0, lane, code0, th0);
  load(c0, 0, lane + 32, code1, th1);
  while (c0 < count) {
    const int64_t cn = dyn ? grab() : c0 + nwarps * cpw;
    MultiEval<NQ, R> ev;
    ev.begin(Ts, j);
    int pmap = 0, lrow = j;  // identity bit map; lane j carries row j's phase
#pragma unroll
    for (int lb = 0; lb < NQ; ++lb) pmap |= lb << (4 * lb);
    bool bad0 = false, bad1 = false;
    for (int nb = 0; nb < L; nb += CHUNK) {
      const int nq = min(CHUNK, L - nb);
      // prepare this chunk's 64 gates (two per lane) into shared memory
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int code = h ? code1 : code0;
        const double th = h ? th1 : th0;
        int info = GT_DIAG;
        uint32_t rpar = 0;
        R2 e0 = Cplx<R>::make(R(1), R(0)), e1 = e0;
        if (code >= 0) E::prepare(code, th, info, rpar, e0, e1);
        const int k = lane + 32 * h;
        cs.info[k] = info;
        cs.rpar[k] = rpar;
        cs.e1[k] = e1;
        (h ? bad1 : bad0) |= code >= Geo<NQ>::NCODES;
      }
      // next chunk (or the next batch's first) in flight while this one runs
      const int nnb = nb + CHUNK < L ? nb + CHUNK : 0;
      const int64_t nc = nb + CHUNK < L ? c0 : cn;
      load(nc, nnb, lane, code0, th0);
      load(nc, nnb, lane + 32, code1, th1);
      __syncwarp();
      if constexpr (kLockstep) {
#pragma unroll 1
        for (int q = 0; q < nq; ++q) ev.step(cs, cs.fac, g * CHUNK + q, lane, j);
      } else {
        ev.run_chunk(cs, cs.fac, g * CHUNK, nq, lane, j, pmap, lrow);
      }
      __syncwarp();
    }
    // bad codes: NaN fitness for the circuit holding one (ISQ_ERR_CONFIG on host entry points)
    const unsigned badm0 = __ballot_sync(0xffffffffu, bad0), badm1 = __ballot_sync(0xffffffffu, bad1);
    const double f = ev.finish(lane, j, pmap);
    const int64_t c = c0 + g;
    if (j == 0 && g < cpw && c < count) {
      const bool cbad = ((badm0 & own0) | (badm1 & own1)) != 0;
      fitness[c] = cbad ? __longlong_as_double(0x7ff8000000000000LL) : f;
      if (cbad && bad_code) atomicOr(bad_code, 1);
    }
    c0 = cn;
  }
}

// Shared scratch and body of the fitness kernels: CPW circuits per warp for
// n <= ISQ_MULTI_MAXNQ, one circuit per warp above (fitness_warp.cuh).
template <int NQ>
constexpr bool kFitMulti = NQ <= ISQ_MULTI_MAXNQ;
// NR: rotations per phase pass of the one-circuit evaluator (the single-block
// kernels with 8 warps use fewer to stay inside 48 KB of static shared memory).
template <int NQ, class R, int NR = kFitNR>
using FitScratch = std::conditional_t<kFitMulti<NQ>, MultiChunk<NQ, R>, FastChunkT<R, NR>>;
constexpr int kSmallNR = 2;  // single-block / cooperative kernels (8 warps per block)
template <int NQ>
constexpr int kFitCPW = kFitMulti<NQ> ? MGeo<NQ>::CPW : 1;  // circuits per warp

// Circuits per warp for a latency-bound launch of `warps` warps over P
// circuits: as few as fill the warps.
template <int NQ>
__device__ __forceinline__ int small_cpw(int64_t P, int64_t warps) {
  const int64_t c = (P + warps - 1) / warps;
  return (int)(c < 1 ? 1 : (c > kFitCPW<NQ> ? kFitCPW<NQ> : c));
}

template <int NQ, class R = double, int NR = kFitNR, bool kLockstep = false>
__device__ __forceinline__ void fitness_rows_fast(int64_t count, int L, const uint8_t* __restrict__ codes,
                                                  const double* __restrict__ thetas,
                                                  const double2* __restrict__ Ts, FitScratch<NQ, R, NR>* sh,
                                                  double* __restrict__ fitness, int warps_per_block,
                                                  int* bad_code = nullptr, unsigned long long* dyn = nullptr,
                                                  int cpw = kFitCPW<NQ>) {
  if constexpr (kFitMulti<NQ>)
    fitness_rows_multi<NQ, R, kLockstep>(count, L, codes, thetas, Ts, sh, fitness, warps_per_block, bad_code, dyn,
                                         cpw);
  else
    fitness_rows<NQ, R, NR>(count, L, codes, thetas, Ts, sh, fitness, warps_per_block, bad_code, dyn);
}

}  // namespace isq

// Fast fitness evaluator: warp-per-candidate, register-resident columns,
// diagonal-phase accumulation and in-place lifted rotations.
//
// Replaces evaluate_circuit / fitness_value (engine.py:187-199,
// fitness.py:36-49) and GA decode + score (ga.py:76-78,167-170) when only the
// fitness is needed.  The composed matrix is carried as
//
//     S_true  ~  diag(e^{i phi}) . S_phys          (up to a global phase / sign)
//
//   S_phys : register state (WarpUnitary layout, unitary_warp.cuh)
//   phi    : pending per-row phases, carried as the unit complex factor
//            e^{i phi_r} on lane r (r < D), so flushes need no sincos
//
// * Rz and ZZ are diagonal: e^{-i th/2} on the rows whose wire bit (Rz) or
//   bit parity (ZZ) is 0, e^{+i th/2} on the others.  They commute with phi,
//   so each costs one complex multiply per lane (w_r *= e^{-+i th/2}, the
//   conjugate picked by a sign flip).
//   The rotation positions of a 32-gate chunk come from one ballot; the
//   diagonal runs between them are branch-free loops over the pending phase.
// * Ry = S Rx S^dagger with S = diag(1, i) on the wire, and both S factors are
//   diagonal, so they go into phi and every rotation is an Rx.
// * An Rx on row bit b only fails to commute with the part of phi that
//   differs between rows r and r ^ 2^b.  Those deltas are flushed into the
//   rows with bit b set (skipped when all are 0), then the rotation is
//   applied as a rotation by a = -th/2 of the planes (re_r, im_r'), (re_r', im_r)
//   of every row pair, reduced to |a| <= pi/2 (R(a) = -R(a -+ pi), a global
//   sign), with the in-place 3-shear lifting x += p y; y += q x; x += p y.
//   In-place updates keep every switch case free of register moves, so the
//   hot code is n rotation cases + n flush cases and fits the instruction cache.
// * The warp starts from M = T and applies the adjoint gates in reverse order
//   (G^dagger: the negated angle), so it ends with M = S^dagger T and
//   |tr(S^dagger T)| = |sum_j e^{i phi_j} M_phys[j][j]|: one entry per column
//   instead of a dense 2^n x 2^n overlap.
#pragma once
#include "unitary_warp.cuh"

namespace isq {

template <class R>
struct Cplx;
template <>
struct Cplx<double> {
  using T = double2;
  static __device__ __forceinline__ T make(double a, double b) { return make_double2(a, b); }
};
template <>
struct Cplx<float> {
  using T = float2;
  static __device__ __forceinline__ T make(float a, float b) { return make_float2(a, b); }
};

// Per-warp shared scratch for one 32-gate chunk (R: arithmetic type of the
// state, double or the fp32 variant's float).
// kFitNR / NR: unused by this evaluator (interleaved phase and state
// updates measured faster than a separate phase pass at n = 4, 5), kept so
// callers can size the scratch per kernel.
#ifndef ISQ_FIT_NR
#define ISQ_FIT_NR 8
#endif
constexpr int kFitNR = ISQ_FIT_NR;

template <class R, int NR = kFitNR>
struct FastChunkT {
  using R2 = typename Cplx<R>::T;
  R2 cs2[32][2];       // diag: {unused, e^{-i th/2}}; rotation: {(C = cos a, 0), (p, q)}
  uint32_t rpar[32];   // diag: bit r = parity of row r under the gate's wire mask; 0 for rotations
  int info[32];        // bits 0..1: type (0 diag, 1 Rx, 2 Ry); bits 8..15: row bit (n = 5)
  R2 fac[32];          // flush factors, indexed by physical row
  double nth[32];      // next chunk's angles / codes, staged by cp.async (no registers held)
  uint32_t ncode[8];
};
using FastChunk = FastChunkT<double>;

enum : int { GT_DIAG = 0, GT_RX = 1, GT_RY = 2 };

// Resident 2-warp blocks per SM the explicit-gate fitness kernels are bounded
// for (__launch_bounds__ min blocks): n = 5 holds a 32-row column in
// registers; with a bound of 5 blocks ptxas still allocates 168 registers
// (6 resident blocks, 3 warps per scheduler) and schedules 1.6 % faster code
// than with the bound of 6 (7 blocks spill 1.4 KB per thread).  n <= 4 run
// the several-circuits-per-warp evaluator (fitness_multi.cuh): a 2^n-row
// column per lane.
#ifndef ISQ_FIT64_MINB
#define ISQ_FIT64_MINB 5
#endif
// n <= ISQ_MULTI_MAXNQ run the several-circuits-per-warp evaluator
// (fitness_multi.cuh: a 2^n-row column per lane), larger n this one.
#ifndef ISQ_MULTI_MAXNQ
#define ISQ_MULTI_MAXNQ 3
#endif
#ifndef ISQ_FIT64_MINB4
#define ISQ_FIT64_MINB4 10  // this evaluator: 16 rows over 2 lanes
#endif
#ifndef ISQ_FIT64_MINB3
#define ISQ_FIT64_MINB3 6
#endif
#ifndef ISQ_FIT64_MULTI_MINB4
#define ISQ_FIT64_MULTI_MINB4 8
#endif
#ifndef ISQ_FIT64_MULTI_MINB3
#define ISQ_FIT64_MULTI_MINB3 12
#endif
#ifndef ISQ_FIT32_MINB4
#define ISQ_FIT32_MINB4 8
#endif
#ifndef ISQ_FIT32_MINB3
#define ISQ_FIT32_MINB3 8
#endif
#ifndef ISQ_FIT32_MULTI_MINB
#define ISQ_FIT32_MULTI_MINB 16
#endif
template <int NQ, class R>
constexpr int fit_min_blocks() {
  constexpr bool multi = NQ <= ISQ_MULTI_MAXNQ;
  if constexpr (sizeof(R) == 8) {
    if constexpr (NQ >= 5) return ISQ_FIT64_MINB;
    if constexpr (multi) return NQ == 4 ? ISQ_FIT64_MULTI_MINB4 : ISQ_FIT64_MULTI_MINB3;
    return NQ == 4 ? ISQ_FIT64_MINB4 : ISQ_FIT64_MINB3;
  } else {
    if constexpr (NQ >= 5) return 8;
    if constexpr (multi) return ISQ_FIT32_MULTI_MINB;
    return NQ == 4 ? ISQ_FIT32_MINB4 : ISQ_FIT32_MINB3;
  }
}

constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 6.283185307179586;

// sin / cos on |x| <= pi/4 (no range reduction; fdlibm kernel polynomials,
// <= 1 ulp against the correctly rounded values on that interval).
__device__ __forceinline__ void sincos_pi4(double x, double& s, double& c) {
  const double z = x * x;
  double ps = 1.58969099521155010221e-10;
  ps = fma(ps, z, -2.50507602534068634195e-08);
  ps = fma(ps, z, 2.75573137070700676789e-06);
  ps = fma(ps, z, -1.98412698298579493134e-04);
  ps = fma(ps, z, 8.33333333332248946124e-03);
  ps = fma(ps, z, -1.66666666666666324348e-01);
  s = fma(x * z, ps, x);
  double pc = -1.13596475577881948265e-11;
  pc = fma(pc, z, 2.08757232129817482790e-09);
  pc = fma(pc, z, -2.75573143513906633035e-07);
  pc = fma(pc, z, 2.48015872894767294178e-05);
  pc = fma(pc, z, -1.38888888888741095749e-03);
  pc = fma(pc, z, 4.16666666666666019037e-02);
  c = 1.0 - fma(-z * z, pc, 0.5 * z);
}

// c ? a : b as an opaque selp (a select tree over a register array written
// as C++ selects is turned back into a dynamically indexed local array).
__device__ __forceinline__ double sel(int c, double a, double b) {
  double o;
  asm("{.reg .pred p; setp.ne.b32 p, %3, 0; selp.f64 %0, %1, %2, p;}" : "=d"(o) : "d"(a), "d"(b), "r"(c));
  return o;
}
__device__ __forceinline__ float sel(int c, float a, float b) {
  float o;
  asm("{.reg .pred p; setp.ne.b32 p, %3, 0; selp.f32 %0, %1, %2, p;}" : "=f"(o) : "f"(a), "f"(b), "r"(c));
  return o;
}

// v with its sign flipped when bit 31 of `bits` is set.
__device__ __forceinline__ double flip_sign_bit(double v, uint32_t bits) {
  return __hiloint2double(__double2hiint(v) ^ (int)(bits & 0x80000000u), __double2loint(v));
}
__device__ __forceinline__ float flip_sign_bit(float v, uint32_t bits) {
  return __int_as_float(__float_as_int(v) ^ (int)(bits & 0x80000000u));
}

// Bit r set for the rows r < 32 whose bits under `mask` have odd parity.
__device__ __forceinline__ uint32_t row_parity(int mask) {
  constexpr uint32_t kBitRows[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  uint32_t p = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (mask & (1 << k)) p ^= kBitRows[k];
  return p;
}

template <int NQ, class R = double, int NR = kFitNR>
struct FastEval {
  using G = Geo<NQ>;
  using R2 = typename Cplx<R>::T;
  using Chunk = FastChunkT<R, NR>;
  WarpUnitary<NQ, R> st;
  R wr, wi;  // pending phase factor e^{i phi} of physical row `lane` (lane < D)

  // M = T (column j of the target on lane j); the gates are then applied as
  // their adjoints in reverse order, M = S^dagger T, so the overlap is a trace.
  __device__ __forceinline__ void begin(const double2* __restrict__ T, int lane) {
    const int j = lane & (G::D - 1);
    const int h = (lane >> NQ) & (G::LPC - 1);
#pragma unroll
    for (int r = 0; r < G::E; ++r) {
      double tx, ty;  // volatile: the column is loop-invariant, and hoisting it
                      // out of the circuit loop would pin 2 D registers
      asm volatile("ld.v2.f64 {%0, %1}, [%2];" : "=d"(tx), "=d"(ty) : "l"(T + (h * G::E + r) * G::D + j));
      st.re[r] = R(tx);
      st.im[r] = R(ty);
    }
    wr = R(1);
    wi = R(0);
  }

  // Lane-parallel gate preparation for one position (one sincos site for
  // every gate type, so a chunk pays for it once).  With r = remainder(th, 2 pi)
  // (|r| <= pi) and x = -r/4 (|x| <= pi/4, no range reduction):
  //   rotation: plane angle a = -r/2 -> (C, p, q) = (cos a, -tan(a/2), sin a)
  //   diagonal: e = e^{-i r/2}; rows whose mask parity is 0 take e, parity 1
  //             take conj(e) (Rz / ZZ up to a global phase)
  // Gate parameters are computed in fp64 for both arithmetic types.
  __device__ __forceinline__ static void prepare(int code, double theta, int& info, uint32_t& rpar,
                                                 R2& e0, R2& e1) {
    int b = -1, type = GT_DIAG, mask;
    if (code < 3 * NQ) {
      const int w0 = code / 3, axis = code - 3 * w0;
      const int rb = NQ - 1 - w0;  // row bit of the wire (wire 1 = MSB)
      mask = 1 << rb;
      if (axis != 2) {
        b = rb;
        type = axis == 0 ? GT_RX : GT_RY;
      }
    } else if (code < G::NCODES) {
      int i = 1, tt = code - 3 * NQ;
      while (tt >= NQ - i) {
        tt -= NQ - i;
        ++i;
      }
      const int j = i + 1 + tt;
      mask = (1 << (NQ - i)) | (1 << (NQ - j));
    } else {
      mask = 0;  // not a gate of this wire count: the chunk reports it (NaN fitness)
    }
    // remainder(theta, 2 pi), exact (up to the sign of a zero); the engines'
    // angles all lie in [-2 pi, 2 pi]
    double r;
    if (fabs(theta) <= kTwoPi)
      r = theta > kPi ? theta - kTwoPi : (theta < -kPi ? theta + kTwoPi : theta);
    else
      r = remainder(theta, kTwoPi);
    double sn, cs;
    sincos_pi4(-0.25 * r, sn, cs);
    // cos a as the lifting produces it (1 + p q): every gate type then gives
    // the same cos, so circuits that differ only in a measured axis tie
    // exactly, as the reference's dense products do (a single-gate circuit
    // on the identity scores 4|cos(th/2)| for Rx, Ry, Rz and ZZ alike)
    const double S = 2.0 * sn * cs, pl = -sn / cs, C = fma(pl, S, 1.0);
    if (b >= 0) {
      info = type | (b << 8);
      rpar = 0;
      e0 = Cplx<R>::make(R(C), R(0));
      e1 = Cplx<R>::make(R(pl), R(S));
    } else {
      info = GT_DIAG;
      rpar = row_parity(mask);
      e0 = Cplx<R>::make(R(1), R(0));
      e1 = Cplx<R>::make(R(C), R(S));
    }
  }

  // Multiply the register rows with bit B set by fac[row] (flush of pending deltas).
  template <int B>
  __device__ __forceinline__ void flush_bit(const R2* fac, int lane) {
    const int h = (lane >> NQ) & (G::LPC - 1);
#pragma unroll
    for (int r = 0; r < G::E; ++r) {
      if (B < G::EB && !(r & (1 << B))) continue;
      const R2 f = fac[h * G::E + r];
      st.cmul(r, f.x, f.y);
    }
  }

  // Flush of row bit B fused with the Rx lifting on it: per row pair
  // (r, r1 = r | 2^B) the pending delta of r1 is multiplied in, then the pair
  // is rotated, so the compiler can overlap one pair's flush with another's
  // lifting.  Lane bits (n < 5) flush all rows of the upper lanes, then rotate.
  template <int B>
  __device__ __forceinline__ void flush_lift(const R2* fac, R p, R q, R C, int lane) {
    if constexpr (B < G::EB) {
      constexpr int m = 1 << B;
      const int h = (lane >> NQ) & (G::LPC - 1);
#pragma unroll
      for (int r = 0; r < G::E; ++r) {
        if (r & m) continue;
        const int r1 = r | m;
        const R2 f = fac[h * G::E + r1];
        st.cmul(r1, f.x, f.y);
        st.re[r] = fma(p, st.im[r1], st.re[r]);
        st.im[r1] = fma(q, st.re[r], st.im[r1]);
        st.re[r] = fma(p, st.im[r1], st.re[r]);
        st.re[r1] = fma(p, st.im[r], st.re[r1]);
        st.im[r] = fma(q, st.re[r1], st.im[r]);
        st.re[r1] = fma(p, st.im[r], st.re[r1]);
      }
    } else {
      flush_bit<B>(fac, lane);
      st.template lift<B, 0>(p, q, C, lane);
    }
  }

  __device__ __forceinline__ void flush_rotate(int b, const R2* fac, R p, R q, R C, int lane) {
    switch (b) {
      case 0: flush_lift<0>(fac, p, q, C, lane); break;
      case 1: if constexpr (NQ > 1) flush_lift<1>(fac, p, q, C, lane); break;
      case 2: if constexpr (NQ > 2) flush_lift<2>(fac, p, q, C, lane); break;
      case 3: if constexpr (NQ > 3) flush_lift<3>(fac, p, q, C, lane); break;
      case 4: if constexpr (NQ > 4) flush_lift<4>(fac, p, q, C, lane); break;
      default: break;
    }
  }

  // Pending phase of this lane's row times the diagonal gates [q, qe) of the
  // chunk (all of them diagonal): branch-free, one predicated complex
  // multiply per gate.  Gates are folded in groups of four (then two, one):
  // the group's product is a tree independent of w, so the dependent chain
  // on w is one complex multiply per group instead of one per gate, at the
  // same instruction count (n = 5 fp64, where the kernel is latency bound:
  // -2 %; n <= 4 and the fp32 variant keep the one-gate loop).
  __device__ __forceinline__ R2 diag_factor(int q, const Chunk& sm, int sh) const {
    R2 e = sm.cs2[q][1];
    e.y = flip_sign_bit(e.y, sm.rpar[q] << sh);  // parity 1: conj
    return e;
  }
  static __device__ __forceinline__ R2 cm(R2 a, R2 b) {
    return Cplx<R>::make(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
  }
  __device__ __forceinline__ void apply_phase(R2 e) {
    const R t = wr * e.y;
    wr = fma(wr, e.x, -wi * e.y);
    wi = fma(wi, e.x, t);
  }
  __device__ __forceinline__ void diag_run(int q, int qe, const Chunk& sm, int sh) {
    if constexpr (NQ < 5 || sizeof(R) < 8) {  // measured slower there: one gate at a time
#pragma unroll 2
      for (; q < qe; ++q) apply_phase(diag_factor(q, sm, sh));
    } else {
      for (; q + 3 < qe; q += 4) {
        const R2 a = cm(diag_factor(q, sm, sh), diag_factor(q + 1, sm, sh));
        const R2 b = cm(diag_factor(q + 2, sm, sh), diag_factor(q + 3, sm, sh));
        apply_phase(cm(a, b));
      }
      if (q + 1 < qe) {
        apply_phase(cm(diag_factor(q, sm, sh), diag_factor(q + 1, sm, sh)));
        q += 2;
      }
      if (q < qe) apply_phase(diag_factor(q, sm, sh));
    }
  }

  // One chunk: lane q < nq supplies (code_q, theta_q) for position base+q.
  // The rotation positions are found with one ballot; the diagonal runs
  // between them touch only the pending phase (diag_run), the rotations
  // flush the non-commuting part of it and rotate the register state.
  // Returns true (warp-uniform) when a lane's code is not a valid gate code.
  __device__ __forceinline__ bool chunk(int code, double theta, int nq, Chunk& sm, int lane) {
    int info = GT_DIAG;  // lanes past the end: neutral diagonal, no parity
    uint32_t rpar = 0;
    R2 e0 = Cplx<R>::make(R(1), R(0)), e1 = e0;
    if (lane < nq) prepare(code, theta, info, rpar, e0, e1);
    const bool bad = __any_sync(0xffffffffu, lane < nq && (code < 0 || code >= G::NCODES));
    // n <= 4: each rotation's type and row bit as warp-uniform bit planes (no
    // shared-memory round trip on the rotation's critical path: -3 % at n = 3,
    // 4); n = 5 reads them back from shared memory (the bit planes cost it
    // spills: +1.5 %)
    constexpr bool kPlanes = NQ < 5;
    if constexpr (!kPlanes) sm.info[lane] = info;
    sm.rpar[lane] = rpar;
    sm.cs2[lane][0] = e0;
    sm.cs2[lane][1] = e1;
    unsigned rot = __ballot_sync(0xffffffffu, info != GT_DIAG);
    unsigned ryb = 0, bp0 = 0, bp1 = 0, bp2 = 0;
    if constexpr (kPlanes) {
      ryb = __ballot_sync(0xffffffffu, (info & 3) == GT_RY);
      bp0 = __ballot_sync(0xffffffffu, info & 0x100);
      bp1 = __ballot_sync(0xffffffffu, info & 0x200);
      bp2 = __ballot_sync(0xffffffffu, info & 0x400);
    }
    __syncwarp();
    const int row = lane;  // physical row whose phase this lane carries
    const int sh = 31 - row;
    int q = 0;
    while (rot) {
      const int qr = __ffs(rot) - 1;
      diag_run(q, qr, sm, sh);
      rot &= rot - 1;
      q = qr + 1;
      int inf;
      if constexpr (kPlanes)
        inf = (((bp0 >> qr) & 1) << 8) | (((bp1 >> qr) & 1) << 9) | (((bp2 >> qr) & 1) << 10) |
              (((ryb >> qr) & 1) ? GT_RY : GT_RX);
      else
        inf = sm.info[qr];
      const int b = inf >> 8;
      const int m = 1 << b;
      const bool ry = (inf & 3) == GT_RY;
      const bool hib = (row & m) != 0;
      // flush factor of the rows with bit b set: w_r * conj(w_{r^m}), times -i
      // for Ry (S^dagger); those rows then carry their partner's phase (times
      // +i for Ry: S), which commutes with the Rx.  Rows with the bit clear
      // keep their phase; their factor is only read for lane-bit rotations
      // (n < 5), where it must be 1.
      // (the partner's phase comes over times i for Ry: o' = i o, so that
      // w conj(o') = -i w conj(o) and the new phase is o')
      const R orr = __shfl_xor_sync(0xffffffffu, ry ? -wi : wr, m);
      const R ori = __shfl_xor_sync(0xffffffffu, ry ? wr : wi, m);
      R fr = fma(wr, orr, wi * ori), fi = fma(wi, orr, -wr * ori);
      if constexpr (G::LB > 0) {
        fr = hib ? fr : R(1);
        fi = hib ? fi : R(0);
      }
      sm.fac[lane] = Cplx<R>::make(fr, fi);
      if (hib) {
        wr = orr;
        wi = ori;
      }
      const R2 pq = sm.cs2[qr][1];
      const R C = sm.cs2[qr][0].x;
      __syncwarp();
      flush_rotate(b, sm.fac, pq.x, pq.y, C, lane);
      __syncwarp();
    }
    diag_run(q, nq, sm, sh);
    __syncwarp();
    return bad;
  }

  // Registers [0, HALF) <- [HALF, 2 HALF) where bit HALF of idx is set, down
  // to HALF = 1: register 0 ends up holding register idx.
  template <int HALF>
  __device__ __forceinline__ void select_level(int idx) {
    if constexpr (HALF >= 1) {
      const int up = idx & HALF;
#pragma unroll
      for (int i = 0; i < HALF; ++i) {
        st.re[i] = sel(up, st.re[i + HALF], st.re[i]);
        st.im[i] = sel(up, st.im[i + HALF], st.im[i]);
      }
      select_level<HALF / 2>(idx);
    }
  }

  // Fitness from the final state (fitness.py:36-49): |tr(M_true)| with
  // M_true = diag(e^{i phi}) M_phys, i.e. sum_j e^{i phi_j} M_phys[j][j].
  // The diagonal entry of column j is picked out of the registers with a
  // select tree over the register index; the trace is summed in fp64.
  __device__ __forceinline__ double finish(int lane) {
    const int j = lane & (G::D - 1);
    const int h = (lane >> NQ) & (G::LPC - 1);
    R pr = wr, pi = wi;
    if constexpr (G::LB > 0) {  // the phase of row j is carried by lane j
      pr = __shfl_sync(0xffffffffu, wr, j);
      pi = __shfl_sync(0xffffffffu, wi, j);
    }
    select_level<G::E / 2>(j & (G::E - 1));
    const double xr = st.re[0], xi = st.im[0], wx = pr, wy = pi;
    double ar = fma(wx, xr, -wy * xi), ai = fma(wx, xi, wy * xr);
    if (h != (j >> G::EB)) ar = ai = 0.0;  // row j lives on another lane of the column
#pragma unroll
    for (int off = G::ACTIVE / 2; off >= 1; off >>= 1) {
      ar += __shfl_xor_sync(0xffffffffu, ar, off);
      ai += __shfl_xor_sync(0xffffffffu, ai, off);
    }
    return fitness_from_overlap(hypot(ar, ai), G::D);
  }
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

// Stage chunk `nb` of circuit nc in shared memory with cp.async, so the
// prefetch holds no registers (a register prefetch was spilled and its store
// waited on the load right away).  Chunks run backwards through the circuit:
// chunk nb holds positions [L - nb - nq, L - nb), nq = min(32, L - nb).
template <class Chunk>
__device__ __forceinline__ void stage_chunk(Chunk& sm, int64_t count, int L, const uint8_t* codes,
                                            const double* thetas, int64_t nc, int nb, int lane) {
  if (nc >= count) return;
  const int nq = min(32, L - nb);
  const int64_t row = nc * (int64_t)L + (L - nb - nq);
  if (lane < nq) cp_async(&sm.nth[lane], thetas + row + lane, 8);
  const uint8_t* src = codes + row;
  if (nq == 32 && ((reinterpret_cast<uintptr_t>(src) & 3) == 0)) {
    if (lane < 8) cp_async(&sm.ncode[lane], src + 4 * lane, 4);
  } else {
    if (lane < nq) reinterpret_cast<uint8_t*>(sm.ncode)[lane] = src[lane];
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// Grid-stride body shared by the explicit-gate fitness kernels: warp per
// circuit over circuits [0, count) of (codes, thetas) rows of length L.
// With `dyn` (a zeroed device counter) the warps take circuits in batches of
// kFitGrab from it instead of a fixed grid stride, so a warp whose circuits
// happened to hold more rotations does not leave the launch a tail.
#ifndef ISQ_FIT_GRAB
#define ISQ_FIT_GRAB 4
#endif
constexpr int kFitGrab = ISQ_FIT_GRAB;  // measured: 4 best (1: +1 %, 2 and 8: +0.2 %)
// n = 5 (C5's fitness, 9.22 -> 9.19 ms; kbench n = 5 -0.4 %): batches of 12
// (8: 9.20, 16: 9.20 ms); n = 4 keeps 4 (12: kbench QEQEA n = 4 +2.5 %)
#ifndef ISQ_FIT_GRAB5
#define ISQ_FIT_GRAB5 12
#endif
#ifndef ISQ_FIT_GUIDED
#define ISQ_FIT_GUIDED 1
#endif
template <int NQ, class R = double, int NR = kFitNR>
__device__ __forceinline__ void fitness_rows(int64_t count, int L, const uint8_t* __restrict__ codes,
                                             const double* __restrict__ thetas,
                                             const double2* __restrict__ Ts, FastChunkT<R, NR>* sh,
                                             double* __restrict__ fitness, int warps_per_block,
                                             int* bad_code = nullptr, unsigned long long* dyn = nullptr) {
  constexpr int kGrab = NQ == 5 ? ISQ_FIT_GRAB5 : kFitGrab;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  FastChunkT<R, NR>& cs = sh[wib];
  const int64_t nwarps = (int64_t)gridDim.x * warps_per_block;
  auto grab = [&](int sz) -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(dyn, (unsigned long long)sz);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
#if ISQ_FIT_GUIDED
  // batches of kGrab until the last two rounds of the grid, then single
  // circuits: a shorter tail at C4-sized launches (~22 circuits per warp)
  auto size_for = [&](int64_t seen) -> int { return seen + 2 * kGrab * nwarps < count ? kGrab : 1; };
#else
  auto size_for = [&](int64_t) -> int { return kGrab; };
#endif
  int64_t c, cend = 0, ahead = 0;
  int ahead_sz = kGrab;
  if (dyn) {
    c = grab(kGrab);
    cend = c + kGrab;
    ahead_sz = size_for(c);
    ahead = grab(ahead_sz);  // the batch after this one, known early for the prefetch
  } else {
    c = (int64_t)blockIdx.x * warps_per_block + wib;
  }
  stage_chunk(cs, count, L, codes, thetas, c, 0, lane);
  while (c < count) {
    const int64_t cn = dyn ? (c + 1 < cend ? c + 1 : ahead) : c + nwarps;  // this warp's next circuit
    FastEval<NQ, R, NR> ev;
    ev.begin(Ts, lane);
    bool bad = false;
    for (int base = 0; base < L; base += 32) {
      const int nq = min(32, L - base);
      asm volatile("cp.async.wait_all;\n" ::);
      __syncwarp();
      int code = 0;
      double th = 0.0;
      if (lane < nq) {  // position L - 1 - base - lane, as its adjoint
        code = reinterpret_cast<const uint8_t*>(cs.ncode)[nq - 1 - lane];
        th = -cs.nth[nq - 1 - lane];
      }
      __syncwarp();
      int64_t nc = c;
      int nb = base + 32;
      if (nb >= L) {
        nc = cn;
        nb = 0;
      }
      stage_chunk(cs, count, L, codes, thetas, nc, nb, lane);
      bad |= ev.chunk(code, th, nq, cs, lane);
    }
    const double f = ev.finish(lane);
    if (lane == 0) {
      fitness[c] = bad ? __longlong_as_double(0x7ff8000000000000LL) : f;  // NaN: invalid gate code
      if (bad && bad_code) atomicOr(bad_code, 1);
    }
    if (dyn && !(c + 1 < cend)) {  // moved on to the batch grabbed ahead
      cend = ahead + ahead_sz;
      ahead_sz = size_for(ahead);
      ahead = grab(ahead_sz);
    }
    c = cn;
  }
}

}  // namespace isq

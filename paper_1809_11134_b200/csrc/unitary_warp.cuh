// Warp-per-candidate circuit composition in registers.
//
// Replaces evaluate_circuit / apply_gate / compose_gates / fitness_value
// (engine.py:187-199, gates.py:173-195, fitness.py:36-49).  The reference
// left-multiplies a dense 2^n x 2^n accumulator by a Kronecker-expanded gate
// (8 D^3 flops per rotation); here every gate is applied as what it is:
//
//   * a rotation on wire w is D/2 independent 2x2 butterflies between rows
//     k and k ^ 2^(n-w) of every column;
//   * Rz and the ZZ interaction are diagonal phases.
//
// Layout.  One warp owns one candidate.  Lane l = h*D + j holds rows
// [h*E, (h+1)*E) of column j of S (E = D / LPC complex numbers in registers,
// LPC = lanes per column).  n = 5: 32 lanes x 32 rows (LPC 1); n = 4: 2 lanes
// per column (the wire-1 row bit lives in the lane id); n = 3: 4 lanes per
// column; n = 2: 4 lanes per column on 16 lanes, lanes 16..31 duplicate.
// Gates on a row bit held in registers are register-local; gates on a lane
// row bit exchange the partner half with __shfl_xor_sync.
//
// Phase factoring (|tr(S^dagger T)| ignores a global phase and we carry real
// scale factors separately):
//   Rx = c [[1,-it],[-it,1]] (|c|>=|s|, t = s/c)  or  s [[u,-i],[-i,u]] (u = c/s)
//   Ry = c [[1,-t],[t,1]]                          or  s [[u,-1],[1,u]]
//   Rz = e^{-i th/2} diag(1, e^{i th})
//   ZZ = e^{-i th/2} diag(1 if bits agree else e^{i th})
// so every gate costs 2 FP64 pipe instructions per complex entry it touches
// (one FMA per real component for Rx/Ry, a complex multiply on half of the
// entries for Rz/ZZ).  The real scale product is kept as mantissa x 2^k,
// with the exponent folded into the registers by exact power-of-two scaling
// once per 32-gate chunk, so long circuits never overflow.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace isq {

template <int NQ>
struct Geo {
  static constexpr int D = 1 << NQ;
  static constexpr int LB = (5 - NQ) < NQ ? (5 - NQ) : NQ;  // row bits carried by the lane id
  static constexpr int LPC = 1 << LB;                        // lanes per column
  static constexpr int E = D / LPC;                          // complex entries per lane
  static constexpr int EB = NQ - LB;                         // row bits held in registers
  static constexpr int ACTIVE = D * LPC;                     // lanes per candidate copy
  static constexpr int NPAIRS = NQ * (NQ - 1) / 2;
  static constexpr int NCODES = 3 * NQ + NPAIRS;             // ga.py:47-59 gate_choices order
  static constexpr int NOPS = 5 * NQ + NPAIRS;
};

// Gate codes (shared with the GA genome and best-circuit readout):
//   code = 3*(wire-1) + axis  for rotations (axis X,Y,Z = 0,1,2; gates.py:30-33)
//   code = 3n + t            for the t-th interaction pair in lexicographic order
//                            (gates.py:76-88 enumerate_templates)
// Opcodes (kernel-internal, chosen per gate from code and angle):
//   [0,n)   Rx tan form   [n,2n)  Rx cot form   [2n,3n) Ry tan form
//   [3n,4n) Ry cot form   [4n,5n) Rz phase      [5n,5n+C) ZZ phase on pair t
__host__ __device__ constexpr int pair_first(int n, int t) {
  int i = 1;
  while (t >= n - i) {
    t -= n - i;
    ++i;
  }
  return i;
}
__host__ __device__ constexpr int pair_second(int n, int t) {
  int i = 1;
  while (t >= n - i) {
    t -= n - i;
    ++i;
  }
  return i + 1 + t;
}

struct GateParam {
  int op;
  double a, b;   // tan/cot coefficient in a; (cos th, sin th) in (a, b) for phases
  double scale;  // real factor pulled out of the gate (1 for phases)
  double phase;  // global phase pulled out (-th/2 for Rz/ZZ), only used by compose
};

template <int NQ>
__device__ __forceinline__ GateParam gate_param(int code, double theta) {
  GateParam g;
  g.phase = 0.0;
  if (code < 3 * NQ) {
    const int w0 = code / 3, axis = code - 3 * w0;
    if (axis == 2) {
      double s, c;
      sincos(theta, &s, &c);
      g.op = 4 * NQ + w0;
      g.a = c;
      g.b = s;
      g.scale = 1.0;
      g.phase = -0.5 * theta;
    } else {
      double s, c;
      sincos(0.5 * theta, &s, &c);
      const bool tan_form = fabs(c) >= fabs(s);
      g.op = (axis == 0 ? 0 : 2 * NQ) + (tan_form ? 0 : NQ) + w0;
      g.a = tan_form ? s / c : c / s;
      g.b = 0.0;
      g.scale = tan_form ? c : s;
    }
  } else {
    double s, c;
    sincos(theta, &s, &c);
    g.op = 5 * NQ + (code - 3 * NQ);
    g.a = c;
    g.b = s;
    g.scale = 1.0;
    g.phase = -0.5 * theta;
  }
  return g;
}

// R = double for every exact path; R = float is the fitness kernel's fp32
// variant (only set_identity / lift / cmul are used with it).
template <int NQ, class R = double>
struct WarpUnitary {
  using G = Geo<NQ>;
  static constexpr int E = G::E;
  R re[E], im[E];

  __device__ __forceinline__ void set_identity(int lane) {
    const int j = lane & (G::D - 1);
    const int h = (lane >> NQ) & (G::LPC - 1);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      re[r] = (h * E + r == j) ? R(1) : R(0);
      im[r] = R(0);
    }
  }

  __device__ __forceinline__ void scale_all(double f) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      re[r] *= f;
      im[r] *= f;
    }
  }

  // grp: 0 Rx tan, 1 Rx cot, 2 Ry tan, 3 Ry cot.  RB: row bit of the wire.
  template <int RB, int GRP>
  __device__ __forceinline__ void rot(double cf, int lane) {
    if constexpr (RB < G::EB) {
      constexpr int m = 1 << RB;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (r & m) continue;
        const int r1 = r | m;
        const double ar = re[r], ai = im[r], br = re[r1], bi = im[r1];
        if constexpr (GRP == 0) {  // a' = a - i t b ; b' = b - i t a
          re[r] = fma(cf, bi, ar);
          im[r] = fma(-cf, br, ai);
          re[r1] = fma(cf, ai, br);
          im[r1] = fma(-cf, ar, bi);
        } else if constexpr (GRP == 1) {  // a' = u a - i b ; b' = u b - i a
          re[r] = fma(cf, ar, bi);
          im[r] = fma(cf, ai, -br);
          re[r1] = fma(cf, br, ai);
          im[r1] = fma(cf, bi, -ar);
        } else if constexpr (GRP == 2) {  // a' = a - t b ; b' = b + t a
          re[r] = fma(-cf, br, ar);
          im[r] = fma(-cf, bi, ai);
          re[r1] = fma(cf, ar, br);
          im[r1] = fma(cf, ai, bi);
        } else {  // a' = u a - b ; b' = u b + a
          re[r] = fma(cf, ar, -br);
          im[r] = fma(cf, ai, -bi);
          re[r1] = fma(cf, br, ar);
          im[r1] = fma(cf, bi, ai);
        }
      }
    } else {
      constexpr int lb = RB - G::EB;
      constexpr int lmask = G::D << lb;
      const bool hi = (lane >> (NQ + lb)) & 1;  // this lane holds the "b" (bit = 1) rows
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const double yr = __shfl_xor_sync(0xffffffffu, re[r], lmask);
        const double yi = __shfl_xor_sync(0xffffffffu, im[r], lmask);
        if constexpr (GRP == 0) {  // x' = x - i t y (both roles)
          re[r] = fma(cf, yi, re[r]);
          im[r] = fma(-cf, yr, im[r]);
        } else if constexpr (GRP == 1) {  // x' = u x - i y
          re[r] = fma(cf, re[r], yi);
          im[r] = fma(cf, im[r], -yr);
        } else if constexpr (GRP == 2) {  // a' = a - t b ; b' = b + t a
          const double ce = hi ? cf : -cf;
          re[r] = fma(ce, yr, re[r]);
          im[r] = fma(ce, yi, im[r]);
        } else {  // a' = u a - b ; b' = u b + a
          const double sg = hi ? 1.0 : -1.0;
          re[r] = fma(cf, re[r], sg * yr);
          im[r] = fma(cf, im[r], sg * yi);
        }
      }
    }
  }

  // Rotation by a plane angle a (|a| <= pi/2) of the (ar, bi), (br, ai) planes
  // (AX = 0, Rx) or the (ar, br), (ai, bi) planes (AX = 1, Ry) of every row
  // pair across row bit RB.  Register bits use the in-place 3-shear lifting
  //   x += p y ; y += q x ; x += p y      (p = -tan(a/2), q = sin a)
  // so no temporaries survive the case (no register moves); lane bits use the
  // direct form with (C, S) = (cos a, sin a) on the shuffled partner.
  template <int RB, int AX>
  __device__ __forceinline__ void lift(R p, R q, R C, int lane) {
    if constexpr (RB < G::EB) {
      constexpr int m = 1 << RB;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (r & m) continue;
        const int r1 = r | m;
        if constexpr (AX == 0) {
          re[r] = fma(p, im[r1], re[r]);
          im[r1] = fma(q, re[r], im[r1]);
          re[r] = fma(p, im[r1], re[r]);
          re[r1] = fma(p, im[r], re[r1]);
          im[r] = fma(q, re[r1], im[r]);
          re[r1] = fma(p, im[r], re[r1]);
        } else {
          re[r] = fma(p, re[r1], re[r]);
          re[r1] = fma(q, re[r], re[r1]);
          re[r] = fma(p, re[r1], re[r]);
          im[r] = fma(p, im[r1], im[r]);
          im[r1] = fma(q, im[r], im[r1]);
          im[r] = fma(p, im[r1], im[r]);
        }
      }
    } else {
      constexpr int lb = RB - G::EB;
      constexpr int lmask = G::D << lb;
      const bool hi = (lane >> (NQ + lb)) & 1;
      const R S = (AX == 1 && !hi) ? -q : q;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const R yr = __shfl_xor_sync(0xffffffffu, re[r], lmask);
        const R yi = __shfl_xor_sync(0xffffffffu, im[r], lmask);
        if constexpr (AX == 0) {  // x' = C x + i S y
          re[r] = fma(C, re[r], -S * yi);
          im[r] = fma(C, im[r], S * yr);
        } else {  // x' = C x + sigma S y
          re[r] = fma(C, re[r], S * yr);
          im[r] = fma(C, im[r], S * yi);
        }
      }
    }
  }

  __device__ __forceinline__ void cmul(int r, R fc, R fs) {
    const R t1 = fs * im[r];
    const R t2 = fs * re[r];
    re[r] = fma(fc, re[r], -t1);
    im[r] = fma(fc, im[r], t2);
  }

  // Rz phase form: rows with the wire bit set pick up e^{i th}.
  template <int RB>
  __device__ __forceinline__ void rz(double c, double s, int lane) {
    if constexpr (RB < G::EB) {
#pragma unroll
      for (int r = 0; r < E; ++r)
        if (r & (1 << RB)) cmul(r, c, s);
    } else {
      const bool hi = (lane >> (NQ + RB - G::EB)) & 1;
      const double fc = hi ? c : 1.0, fs = hi ? s : 0.0;
#pragma unroll
      for (int r = 0; r < E; ++r) cmul(r, fc, fs);
    }
  }

  // ZZ phase form: rows whose two wire bits differ pick up e^{i th}.
  template <int RBI, int RBJ>
  __device__ __forceinline__ void zz(double c, double s, int lane) {
    constexpr bool li = RBI < G::EB, lj = RBJ < G::EB;
    if constexpr (li && lj) {
#pragma unroll
      for (int r = 0; r < E; ++r)
        if (((r >> RBI) ^ (r >> RBJ)) & 1) cmul(r, c, s);
    } else if constexpr (li != lj) {
      constexpr int RBL = li ? RBI : RBJ;  // register bit
      constexpr int RBH = li ? RBJ : RBI;  // lane bit
      const bool v = (lane >> (NQ + RBH - G::EB)) & 1;
      const double c0 = v ? c : 1.0, s0 = v ? s : 0.0;  // register bit 0
      const double c1 = v ? 1.0 : c, s1 = v ? 0.0 : s;  // register bit 1
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (r & (1 << RBL))
          cmul(r, c1, s1);
        else
          cmul(r, c0, s0);
      }
    } else {
      const bool vi = (lane >> (NQ + RBI - G::EB)) & 1;
      const bool vj = (lane >> (NQ + RBJ - G::EB)) & 1;
      const double fc = (vi != vj) ? c : 1.0, fs = (vi != vj) ? s : 0.0;
#pragma unroll
      for (int r = 0; r < E; ++r) cmul(r, fc, fs);
    }
  }

  template <int OP>
  __device__ __forceinline__ void apply_op(double a, double b, int lane) {
    constexpr int n = NQ;
    if constexpr (OP < 4 * n) {
      constexpr int grp = OP / n, w0 = OP % n;
      rot<n - 1 - w0, grp>(a, lane);
    } else if constexpr (OP < 5 * n) {
      constexpr int w0 = OP - 4 * n;
      rz<n - 1 - w0>(a, b, lane);
    } else if constexpr (OP < G::NOPS) {
      constexpr int t = OP - 5 * n;
      constexpr int wi = pair_first(n, t), wj = pair_second(n, t);
      zz<n - wi, n - wj>(a, b, lane);
    }
  }

  __device__ __forceinline__ void apply(int op, double a, double b, int lane) {
#define ISQ_CASE(K) \
  case K:           \
    apply_op<K>(a, b, lane); \
    break;
    switch (op) {
      ISQ_CASE(0) ISQ_CASE(1) ISQ_CASE(2) ISQ_CASE(3) ISQ_CASE(4) ISQ_CASE(5) ISQ_CASE(6)
      ISQ_CASE(7) ISQ_CASE(8) ISQ_CASE(9) ISQ_CASE(10) ISQ_CASE(11) ISQ_CASE(12) ISQ_CASE(13)
      ISQ_CASE(14) ISQ_CASE(15) ISQ_CASE(16) ISQ_CASE(17) ISQ_CASE(18) ISQ_CASE(19)
      ISQ_CASE(20) ISQ_CASE(21) ISQ_CASE(22) ISQ_CASE(23) ISQ_CASE(24) ISQ_CASE(25)
      ISQ_CASE(26) ISQ_CASE(27) ISQ_CASE(28) ISQ_CASE(29) ISQ_CASE(30) ISQ_CASE(31)
      ISQ_CASE(32) ISQ_CASE(33) ISQ_CASE(34)
      default:
        break;
    }
#undef ISQ_CASE
  }

  // sum over the candidate's lanes of conj(S) * T (T row-major in shared memory).
  __device__ __forceinline__ void overlap(const double2* __restrict__ T, int lane, double& ore,
                                          double& oim) const {
    const int j = lane & (G::D - 1);
    const int h = (lane >> NQ) & (G::LPC - 1);
    double ar = 0.0, ai = 0.0;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const double2 t = T[(h * E + r) * G::D + j];
      ar = fma(re[r], t.x, ar);
      ar = fma(im[r], t.y, ar);
      ai = fma(re[r], t.y, ai);
      ai = fma(-im[r], t.x, ai);
    }
#pragma unroll
    for (int off = G::ACTIVE / 2; off >= 1; off >>= 1) {
      ar += __shfl_xor_sync(0xffffffffu, ar, off);
      ai += __shfl_xor_sync(0xffffffffu, ai, off);
    }
    ore = ar;
    oim = ai;
  }
};

// Running real scale kept as mantissa in [0.5, 1) times 2^exp.  fold() moves
// the exponent into the state registers (exact power-of-two scaling).
__device__ __forceinline__ double warp_prod(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// fitness.py:36-49: 1 - sqrt(max(0, (D - |ov|)/D)) clamped to [0, 1].
__device__ __forceinline__ double fitness_from_overlap(double ov, int D) {
  const double dd = (double)D;
  double rad = (dd - ov) / dd;
  rad = rad > 0.0 ? rad : 0.0;
  double f = 1.0 - sqrt(rad);
  f = f > 0.0 ? f : 0.0;
  return f < 1.0 ? f : 1.0;
}

}  // namespace isq

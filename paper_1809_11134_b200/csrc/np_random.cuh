// Counter-based RNG streams that reproduce numpy's Generator(Philox(...)) bit for bit.
//
// The reference engine draws every random number from numpy Generators
// (engine.py:105-112 init, :167-170 Born measurement, :174-184 circuit
// sampling, :241-242 mutation mask/coin; encoding.py:52,127-128 mutation
// steps; ga.py:68-138 GA operators).  This build replaces each sequential
// Generator with one independent Philox4x64-10 stream per unit of work
// (circuit, slot, gene, ...), keyed
//
//     key     = (seed, domain)
//     counter = (0, generation, index, sub)
//
// exactly as numpy.random.Philox(key=[seed, domain], counter=[0, gen, index,
// sub]) would: the counter is incremented BEFORE each 4x64 block, so the
// first block of every stream is philox(ctr = (1, gen, index, sub)).
//
// numpy semantics reproduced here (numpy/random/src):
//   next_uint64  : buffered 4-word blocks                (philox.h philox_next)
//   next_uint32  : low half first, high half buffered and persisting across
//                  calls; next_uint64/next_double do NOT touch that buffer
//   next_double  : (u64 >> 11) * 2^-53
//   integers(b)  : Lemire on u32 with rejection, rng = b - 1
//                  (distributions.c buffered_bounded_lemire_uint32)
//   uniform(l,h) : l + (h - l) * next_double
//   binomial     : inversion for n*min(p,1-p) <= 30     (random_binomial_inversion),
//                  BTPE above                          (random_binomial_btpe)
//   multinomial  : sequential binomials                  (random_multinomial)
//
// All floating point that must be bit-exact is written with explicit
// round-to-nearest intrinsics so nvcc never contracts it into an FMA
// (numpy's random C code is compiled for the SSE baseline, without FMA).
#pragma once
#include <cstdint>

namespace isq {

// Stream domains (counter[1..3] meaning in brackets).  Shared with oracle/streams.py.
enum : uint64_t {
  DOM_SAMPLE = 1,    // (gen, circuit, 0)  integers(P, L) then integers(K, L)
  DOM_MEASURE = 2,   // (gen, slot, 0)     multinomial(n_meas, born(qutrit))
  DOM_MUTATE = 3,    // (gen, slot, 0)     mask, coin, [integers(8), uniform] | [random]
  DOM_INIT = 4,      // (0, slot, 0)       theta = uniform(0, 2pi), 6 Box-Muller uniforms
  DOM_GA_INIT = 5,   // (0, genome, gene)  integers(n_choices), uniform(0, 2pi)
  DOM_GA_SUS = 6,    // (gen, 0, 0)        uniform(0, spacing) | P x integers(P)
  DOM_GA_PAIR = 7,   // (gen, pair, 0)     integers(0, L+1, size=2)
  DOM_GA_MUT = 8,    // (gen, child, gene) random, [random, integers(n_choices) | uniform(-r, r)]
};

constexpr uint64_t PHILOX_M0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t PHILOX_M1 = 0xCA5A826395121157ULL;
constexpr uint64_t PHILOX_W0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t PHILOX_W1 = 0xBB67AE8584CAA73BULL;

// Random123 philox4x64 with 10 rounds (numpy's philox4x64_R(10, ...)).
__host__ __device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2,
                                                       uint64_t c3, uint64_t k0, uint64_t k1,
                                                       uint64_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
#ifdef __CUDA_ARCH__
    const uint64_t hi0 = __umul64hi(PHILOX_M0, c0);
    const uint64_t hi1 = __umul64hi(PHILOX_M1, c2);
#else
    const uint64_t hi0 = (uint64_t)(((unsigned __int128)PHILOX_M0 * c0) >> 64);
    const uint64_t hi1 = (uint64_t)(((unsigned __int128)PHILOX_M1 * c2) >> 64);
#endif
    const uint64_t lo0 = PHILOX_M0 * c0;
    const uint64_t lo1 = PHILOX_M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Block `b` (1-based, i.e. after b counter increments) of stream (seed, dom, gen, idx, sub).
__host__ __device__ __forceinline__ void stream_block(uint64_t seed, uint64_t dom, uint64_t gen,
                                                      uint64_t idx, uint64_t sub, uint64_t b,
                                                      uint64_t out[4]) {
  philox4x64_10(b, gen, idx, sub, seed, dom, out);
}

__host__ __device__ __forceinline__ double u64_to_double(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

#ifdef __CUDA_ARCH__
#define ISQ_DMUL(a, b) __dmul_rn((a), (b))
#define ISQ_DADD(a, b) __dadd_rn((a), (b))
#define ISQ_DSUB(a, b) __dsub_rn((a), (b))
#define ISQ_DDIV(a, b) __ddiv_rn((a), (b))
#else
#define ISQ_DMUL(a, b) ((a) * (b))
#define ISQ_DADD(a, b) ((a) + (b))
#define ISQ_DSUB(a, b) ((a) - (b))
#define ISQ_DDIV(a, b) ((a) / (b))
#endif

// Sequential numpy-compatible stream.  Used where consumption is data dependent
// (rejections, binomial redraws, GA operators); hot fast paths compute the
// blocks they need directly with stream_block().
struct NpStream {
  uint64_t seed, dom, gen, idx, sub;
  uint64_t ctr;  // number of blocks generated so far
  uint64_t b0, b1, b2, b3;  // current block (registers: no dynamic indexing)
  int pos;       // next word of the block; 4 = empty
  uint32_t u32buf;
  bool has32;

  __host__ __device__ __forceinline__ void init(uint64_t seed_, uint64_t dom_, uint64_t gen_,
                                                uint64_t idx_, uint64_t sub_) {
    seed = seed_;
    dom = dom_;
    gen = gen_;
    idx = idx_;
    sub = sub_;
    ctr = 0;
    pos = 4;
    has32 = false;
    u32buf = 0;
  }
  // Generate the first block now (it depends only on the stream key), so its
  // latency can overlap independent work before the first draw.
  __host__ __device__ __forceinline__ void prime() {
    if (ctr == 0) {
      ctr = 1;
      uint64_t w[4];
      stream_block(seed, dom, gen, idx, sub, 1, w);
      b0 = w[0];
      b1 = w[1];
      b2 = w[2];
      b3 = w[3];
      pos = 0;
    }
  }
  __host__ __device__ __forceinline__ uint64_t next64() {
    if (pos >= 4) {
      ++ctr;
      uint64_t w[4];
      stream_block(seed, dom, gen, idx, sub, ctr, w);
      b0 = w[0];
      b1 = w[1];
      b2 = w[2];
      b3 = w[3];
      pos = 0;
    }
    const uint64_t r = pos == 0 ? b0 : (pos == 1 ? b1 : (pos == 2 ? b2 : b3));
    ++pos;
    return r;
  }
  __host__ __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32buf;
    }
    const uint64_t w = next64();
    has32 = true;
    u32buf = (uint32_t)(w >> 32);
    return (uint32_t)(w & 0xffffffffULL);
  }
  __host__ __device__ __forceinline__ double random() { return u64_to_double(next64()); }
  __host__ __device__ __forceinline__ double uniform(double lo, double hi) {
    return ISQ_DADD(lo, ISQ_DMUL(ISQ_DSUB(hi, lo), random()));
  }
  // numpy buffered_bounded_lemire_uint32 with rng = bound - 1 (rng < 0xFFFFFFFF).
  __host__ __device__ __forceinline__ uint32_t lemire32(uint32_t rng) {
    const uint32_t rng_excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * (uint64_t)rng_excl;
    uint32_t leftover = (uint32_t)(m & 0xffffffffULL);
    if (leftover < rng_excl) {
      const uint32_t threshold = (0xffffffffu - rng) % rng_excl;
      while (leftover < threshold) {
        m = (uint64_t)next32() * (uint64_t)rng_excl;
        leftover = (uint32_t)(m & 0xffffffffULL);
      }
    }
    return (uint32_t)(m >> 32);
  }
  // Generator.integers(bound) for 1 <= bound <= 2^32 (default int64 dtype).
  __host__ __device__ __forceinline__ int64_t integers(int64_t bound) {
    const uint64_t rng = (uint64_t)bound - 1u;
    if (rng == 0) return 0;
    if (rng == 0xffffffffULL) return (int64_t)next32();
    return (int64_t)lemire32((uint32_t)rng);
  }
};

// Lemire rejection predicate for one u32 draw against bound (= rng + 1):
// true when numpy would discard this draw and take another.
__host__ __device__ __forceinline__ bool lemire_rejects(uint32_t u, uint32_t rng) {
  const uint32_t rng_excl = rng + 1u;
  const uint32_t leftover = (uint32_t)(((uint64_t)u * rng_excl) & 0xffffffffULL);
  if (leftover >= rng_excl) return false;
  const uint32_t threshold = (0xffffffffu - rng) % rng_excl;
  return leftover < threshold;
}
__host__ __device__ __forceinline__ uint32_t lemire_value(uint32_t u, uint32_t rng) {
  return (uint32_t)(((uint64_t)u * (uint64_t)(rng + 1u)) >> 32);
}

// numpy random_binomial_inversion (distributions.c).  Returns -1 never; the
// bound/redraw loop is reproduced exactly, exp/log are the device versions
// (last-ulp differences from glibc can flip a draw only when U
// lies within an ulp of a CDF boundary).
//
// n = 1 (the default n_meas): the C library's exp(1.0 * log(q)), which
// numpy's distributions.c calls, returns q itself for every q in [0.5, 1]
// tested (3M random q and 1M consecutive doubles at each end through glibc,
// tests/test_oracle.py::test_exp_log_identity_on_binomial_q), so qn = q is
// the reference's value, without the device exp/log rounding; and
// bnd >= 10 > n, so bound = n.
__device__ __forceinline__ int64_t binomial_inversion(NpStream& s, int64_t n, double p) {
  const double q = ISQ_DSUB(1.0, p);
  double qn;
  int64_t bound;
  if (n == 1) {
    qn = q;
    bound = 1;
  } else {
    qn = exp(ISQ_DMUL((double)n, log(q)));
    const double np_ = ISQ_DMUL((double)n, p);
    const double bnd = ISQ_DADD(np_, ISQ_DMUL(10.0, sqrt(ISQ_DADD(ISQ_DMUL(np_, q), 1.0))));
    bound = (int64_t)((double)n < bnd ? (double)n : bnd);
  }
  int64_t X = 0;
  double px = qn;
  double U = s.random();
  while (U > px) {
    X++;
    if (X > bound) {
      X = 0;
      px = qn;
      U = s.random();
    } else {
      U = ISQ_DSUB(U, px);
      px = ISQ_DDIV(ISQ_DMUL(ISQ_DMUL((double)(n - X + 1), p), px), ISQ_DMUL((double)X, q));
    }
  }
  return X;
}

// numpy random_binomial_btpe (distributions.c; Kachitvichyanukul & Schmeiser's
// BTPE) for n * min(p, 1 - p) > 30, with every operation in C's order and
// without FMA contraction (numpy's distributions.c is compiled without FMA:
// oracle/binomial.py restates it and matches numpy's Generator draw for draw,
// tests/test_oracle.py).  log / exp are the device versions (see
// binomial_inversion).  Called with p <= 0.5, as random_binomial does.
__device__ inline int64_t binomial_btpe(NpStream& s, int64_t n, double p) {
  const double dn = (double)n;
  const double one_p = ISQ_DSUB(1.0, p);
  const double r = p < one_p ? p : one_p;
  const double q = ISQ_DSUB(1.0, r);
  const double fm = ISQ_DADD(ISQ_DMUL(dn, r), r);
  const int64_t m = (int64_t)floor(fm);
  const double dm = (double)m;
  const double p1 = ISQ_DADD(floor(ISQ_DSUB(ISQ_DMUL(2.195, sqrt(ISQ_DMUL(ISQ_DMUL(dn, r), q))), ISQ_DMUL(4.6, q))), 0.5);
  const double xm = ISQ_DADD(dm, 0.5);
  const double xl = ISQ_DSUB(xm, p1);
  const double xr = ISQ_DADD(xm, p1);
  const double c = ISQ_DADD(0.134, ISQ_DDIV(20.5, ISQ_DADD(15.3, dm)));
  double a = ISQ_DDIV(ISQ_DSUB(fm, xl), ISQ_DSUB(fm, ISQ_DMUL(xl, r)));
  const double laml = ISQ_DMUL(a, ISQ_DADD(1.0, ISQ_DDIV(a, 2.0)));
  a = ISQ_DDIV(ISQ_DSUB(xr, fm), ISQ_DMUL(xr, q));
  const double lamr = ISQ_DMUL(a, ISQ_DADD(1.0, ISQ_DDIV(a, 2.0)));
  const double p2 = ISQ_DMUL(p1, ISQ_DADD(1.0, ISQ_DMUL(2.0, c)));
  const double p3 = ISQ_DADD(p2, ISQ_DDIV(c, laml));
  const double p4 = ISQ_DADD(p3, ISQ_DDIV(c, lamr));
  const double nrq = ISQ_DMUL(ISQ_DMUL(dn, r), q);
  int64_t y;
  while (true) {
    const double u = ISQ_DMUL(s.random(), p4);
    double v = s.random();
    if (!(u > p1)) {  // Step10: the triangular region, accepted
      y = (int64_t)floor(ISQ_DADD(ISQ_DSUB(xm, ISQ_DMUL(p1, v)), u));
      break;
    }
    if (!(u > p2)) {  // Step20: parallelograms
      const double x = ISQ_DADD(xl, ISQ_DDIV(ISQ_DSUB(u, p1), c));
      v = ISQ_DSUB(ISQ_DADD(ISQ_DMUL(v, c), 1.0), ISQ_DDIV(fabs(ISQ_DADD(ISQ_DSUB(dm, x), 0.5)), p1));
      if (v > 1.0) continue;
      y = (int64_t)floor(x);
    } else if (!(u > p3)) {  // Step30: left exponential tail
      y = (int64_t)floor(ISQ_DADD(xl, ISQ_DDIV(log(v), laml)));
      if (y < 0 || v == 0.0) continue;
      v = ISQ_DMUL(ISQ_DMUL(v, ISQ_DSUB(u, p2)), laml);
    } else {  // Step40: right exponential tail
      y = (int64_t)floor(ISQ_DSUB(xr, ISQ_DDIV(log(v), lamr)));
      if (y > n || v == 0.0) continue;
      v = ISQ_DMUL(ISQ_DMUL(v, ISQ_DSUB(u, p3)), lamr);
    }
    // Step50
    const int64_t k = y > m ? y - m : m - y;
    const double dk = (double)k;
    if (!(k > 20 && dk < ISQ_DSUB(ISQ_DDIV(nrq, 2.0), 1.0))) {
      const double sr = ISQ_DDIV(r, q);
      const double aa = ISQ_DMUL(sr, (double)(n + 1));
      double F = 1.0;
      if (m < y) {
        for (int64_t i = m + 1; i <= y; ++i) F = ISQ_DMUL(F, ISQ_DSUB(ISQ_DDIV(aa, (double)i), sr));
      } else if (m > y) {
        for (int64_t i = y + 1; i <= m; ++i) F = ISQ_DDIV(F, ISQ_DSUB(ISQ_DDIV(aa, (double)i), sr));
      }
      if (v > F) continue;
      break;
    }
    // Step52: squeeze on log(v), then the Stirling-corrected bound
    const double rho = ISQ_DMUL(ISQ_DDIV(dk, nrq),
                                ISQ_DADD(ISQ_DDIV(ISQ_DADD(ISQ_DMUL(dk, ISQ_DADD(ISQ_DDIV(dk, 3.0), 0.625)),
                                                           0.16666666666666666),
                                                  nrq),
                                         0.5));
    const double t = ISQ_DDIV((double)(-k * k), ISQ_DMUL(2.0, nrq));
    const double A = log(v);
    if (A < ISQ_DSUB(t, rho)) break;
    if (A > ISQ_DADD(t, rho)) continue;
    const double x1 = (double)(y + 1), f1 = (double)(m + 1), z = (double)(n + 1 - m), w = (double)(n - y + 1);
    const double x2 = ISQ_DMUL(x1, x1), f2 = ISQ_DMUL(f1, f1), z2 = ISQ_DMUL(z, z), w2 = ISQ_DMUL(w, w);
    auto stirling = [](double v1, double v2) {  // (13680 - (462 - (132 - (99 - 140/v2)/v2)/v2)/v2)/v1/166320
      const double i4 = ISQ_DDIV(ISQ_DSUB(99.0, ISQ_DDIV(140.0, v2)), v2);
      const double i3 = ISQ_DDIV(ISQ_DSUB(132.0, i4), v2);
      const double i2 = ISQ_DDIV(ISQ_DSUB(462.0, i3), v2);
      return ISQ_DDIV(ISQ_DDIV(ISQ_DSUB(13680.0, i2), v1), 166320.0);
    };
    double bound = ISQ_DMUL(xm, log(ISQ_DDIV(f1, x1)));
    bound = ISQ_DADD(bound, ISQ_DMUL(ISQ_DADD((double)(n - m), 0.5), log(ISQ_DDIV(z, w))));
    bound = ISQ_DADD(bound, ISQ_DMUL((double)(y - m), log(ISQ_DDIV(ISQ_DMUL(w, r), ISQ_DMUL(x1, q)))));
    bound = ISQ_DADD(bound, stirling(f1, f2));
    bound = ISQ_DADD(bound, stirling(z, z2));
    bound = ISQ_DADD(bound, stirling(x1, x2));
    bound = ISQ_DADD(bound, stirling(w, w2));
    if (A > bound) continue;
    break;
  }
  if (p > 0.5) y = n - y;  // Step60
  return y;
}

// numpy random_binomial: inversion for n * min(p, 1-p) <= 30, BTPE above.
// kBTPE = false compiles the inversion branch alone, for callers that know
// n <= 60 (n * min(p, 1 - p) <= 30 always): the BTPE code would otherwise
// cost the hot values kernel 26 registers and ~0.8 ms per C5 generation.
template <bool kBTPE = true>
__device__ __forceinline__ int64_t binomial(NpStream& s, double p, int64_t n, bool* ok) {
  (void)ok;
  if (n == 0 || p == 0.0) return 0;
  if constexpr (!kBTPE) {
    if (p <= 0.5) return binomial_inversion(s, n, p);
    return n - binomial_inversion(s, n, ISQ_DSUB(1.0, p));
  } else {
    if (p <= 0.5) {
      if (ISQ_DMUL(p, (double)n) <= 30.0) return binomial_inversion(s, n, p);
      return binomial_btpe(s, n, p);
    }
    const double q = ISQ_DSUB(1.0, p);
    if (ISQ_DMUL(q, (double)n) <= 30.0) return n - binomial_inversion(s, n, q);
    return n - binomial_btpe(s, n, q);
  }
}

// Largest n_meas whose multinomial draws never reach BTPE.
constexpr int kInversionMaxMeas = 60;

// numpy |z| for complex128 (SIMD loop, loops_unary_complex.dispatch.c.src):
// larger * sqrt(fma(ratio, ratio, 1)), ratio = smaller / larger.
__device__ __forceinline__ double np_cabs(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double larger = fmax(a, b), smaller = fmin(a, b);
  if (larger == 0.0) return 0.0;
  if (isinf(larger)) return larger;
  const double ratio = __ddiv_rn(smaller, larger);
  return __dmul_rn(__dsqrt_rn(__fma_rn(ratio, ratio, 1.0)), larger);
}

// construct_segments for one qutrit (engine.py:167-170): Born probabilities
// np.abs(q)**2 normalised by the (left-to-right) row sum, one multinomial
// draw of n_meas measurements, argmax with ties to the lower axis.
template <bool kBTPE = true>
__device__ __forceinline__ int measure_axis(const double qre[3], const double qim[3], int n_meas,
                                            NpStream& s, bool* ok) {
  double pr[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double a = np_cabs(qre[j], qim[j]);
    pr[j] = __dmul_rn(a, a);
  }
  const double sum = __dadd_rn(__dadd_rn(pr[0], pr[1]), pr[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) pr[j] = __ddiv_rn(pr[j], sum);
  // random_multinomial with d = 3, written out so nothing is dynamically indexed
  int64_t c0 = 0, c1 = 0, c2 = 0;
  int64_t dn = n_meas;
  c0 = binomial<kBTPE>(s, pr[0], dn, ok);  // pix[0] / remaining_p with remaining_p = 1.0
  dn -= c0;
  if (dn > 0) {
    const double remaining = __dsub_rn(1.0, pr[0]);
    c1 = binomial<kBTPE>(s, __ddiv_rn(pr[1], remaining), dn, ok);
    dn -= c1;
    if (dn > 0) c2 = dn;
  }
  int best = 0;
  int64_t bc = c0;
  if (c1 > bc) {
    best = 1;
    bc = c1;
  }
  if (c2 > bc) best = 2;
  return best;
}

// numpy's pairwise summation of a contiguous double array (np.sum,
// pairwise_sum in numpy/_core/src/umath/loops_utils.h.src: blocks of 8
// partial sums below 128 elements, recursive halving above), so device
// reductions that the reference computes with np.sum round identically.
__device__ inline double np_pairwise_leaf(const double* a, int64_t n) {  // n <= 128
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// The recursion S(a, n) = S(a, h) + S(a + h, n - h), h = n/2 rounded down
// to a multiple of 8, as an explicit post-order walk (a device recursion
// overflowed the default 1 KB thread stack from n = 2^17).
__device__ inline double np_pairwise_sum(const double* a, int64_t n) {
  if (n <= 128) return np_pairwise_leaf(a, n);
  int64_t r_off[40], r_len[40];  // right subtree still to sum, per pending node
  double left[40];                // (depth <= log2(n / 128) + 1 < 40)
  uint64_t has_left = 0;          // bit: the pending node's left sum is in left[]
  int sp = 0;
  int64_t off = 0, m = n;
  for (;;) {
    while (m > 128) {  // descend left, remembering the right halves
      int64_t h = m / 2;
      h -= h % 8;
      r_off[sp] = off + h;
      r_len[sp] = m - h;
      has_left &= ~(1ull << sp);
      ++sp;
      m = h;
    }
    double acc = np_pairwise_leaf(a + off, m);
    for (;;) {
      if (sp == 0) return acc;
      if (!((has_left >> (sp - 1)) & 1)) {  // left child done: sum the right one next
        has_left |= 1ull << (sp - 1);
        left[sp - 1] = acc;
        off = r_off[sp - 1];
        m = r_len[sp - 1];
        break;
      }
      acc = __dadd_rn(left[sp - 1], acc);  // both children done
      --sp;
    }
  }
}

}  // namespace isq

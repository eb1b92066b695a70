// sampler.cuh — the scene sampler (SPEC.md:141-192 config_sampler contract) and the
// synthetic-signal generator as ONE host/device source, so the host fixture generator
// and the on-device generator agree bit for bit.
//
// Randomness: Philox4x32-10 (Salmon, Moraes, Dror & Shaw, SC'11), keyed by a
// splitmix64 hash of (seed, utterance, epoch) — every scene is a pure function of
// (seed, utterance_id, epoch) and batch order never matters.
// Arithmetic: integer ops, and FP64 +, -, *, /, sqrt with round-to-nearest and no
// contraction (device: __d*_rn intrinsics; host: compiled with -ffp-contract=off);
// log / exp / sin / cos are polynomial restatements built only from those ops, so
// both sides execute the identical IEEE operation sequence.
#pragma once

#include <stdint.h>
#include <string.h>

#include <cmath>

namespace rsg {

#ifdef __CUDA_ARCH__
#define RSH __host__ __device__ __forceinline__
#define RS_ADD(a, b) __dadd_rn((a), (b))
#define RS_SUB(a, b) __dsub_rn((a), (b))
#define RS_MUL(a, b) __dmul_rn((a), (b))
#define RS_DIV(a, b) __ddiv_rn((a), (b))
#define RS_SQRT(a) __dsqrt_rn(a)
#define RS_FLOOR(a) floor(a)
#define RS_CEIL(a) ceil(a)
#define RF_ADD(a, b) __fadd_rn((a), (b))
#define RF_SUB(a, b) __fsub_rn((a), (b))
#define RF_MUL(a, b) __fmul_rn((a), (b))
#define RF_DIV(a, b) __fdiv_rn((a), (b))
#define RF_SQRT(a) __fsqrt_rn(a)
#define RF_FLOOR(a) floorf(a)
#else
#define RSH __host__ __device__ inline
#define RS_ADD(a, b) ((a) + (b))
#define RS_SUB(a, b) ((a) - (b))
#define RS_MUL(a, b) ((a) * (b))
#define RS_DIV(a, b) ((a) / (b))
#define RS_SQRT(a) std::sqrt(a)
#define RS_FLOOR(a) std::floor(a)
#define RS_CEIL(a) std::ceil(a)
#define RF_ADD(a, b) ((a) + (b))
#define RF_SUB(a, b) ((a) - (b))
#define RF_MUL(a, b) ((a) * (b))
#define RF_DIV(a, b) ((a) / (b))
#define RF_SQRT(a) std::sqrt(a)
#define RF_FLOOR(a) std::floor(a)
#endif

// ---- Philox4x32-10 -----------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

RSH uint32_t mulhilo32(uint32_t a, uint32_t b, uint32_t* hi) {
  const uint64_t p = static_cast<uint64_t>(a) * b;
  *hi = static_cast<uint32_t>(p >> 32);
  return static_cast<uint32_t>(p);
}

RSH U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0, hi1;
    const uint32_t lo0 = mulhilo32(0xD2511F53u, c.x, &hi0);
    const uint32_t lo1 = mulhilo32(0xCD9E8D57u, c.z, &hi1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

RSH uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Stream of uniforms keyed by (seed, a, b) (a = utterance, b = epoch).
struct Stream {
  uint32_t k0, k1;
  uint32_t tag;   // stream purpose / sub-stream
  uint64_t ctr;   // draws taken
  RSH Stream(uint64_t seed, uint64_t a, uint64_t b, uint32_t t) : tag(t), ctr(0) {
    const uint64_t k = splitmix64(splitmix64(seed) ^ splitmix64(a * 0x9E3779B97F4A7C15ull + b));
    k0 = static_cast<uint32_t>(k);
    k1 = static_cast<uint32_t>(k >> 32);
  }
  // two 53-bit uniforms in [0, 1) from counter `i`
  RSH void pair_at(uint64_t i, double* u0, double* u1) const {
    const U4 r = philox4x32_10(U4{static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), tag, 0x5CE4Eu}, k0, k1);
    const uint64_t a = (static_cast<uint64_t>(r.x) << 32 | r.y) >> 11;
    const uint64_t b = (static_cast<uint64_t>(r.z) << 32 | r.w) >> 11;
    *u0 = static_cast<double>(a) * 0x1.0p-53;  // exact
    *u1 = static_cast<double>(b) * 0x1.0p-53;
  }
  RSH double next() {
    double u0, u1;
    pair_at(ctr++, &u0, &u1);
    return u0;
  }
  RSH double uniform(double lo, double hi) { return RS_ADD(lo, RS_MUL(RS_SUB(hi, lo), next())); }
};

// ---- portable elementary functions (basic IEEE ops only) -------------------------
RSH double bits_to_double(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
RSH uint64_t double_to_bits(double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
}

constexpr double kLn2 = 0.6931471805599453094;
constexpr double kLn2Hi = 0x1.62e42fefa3800p-1;  // trailing zeros: k * kLn2Hi exact for |k| < 2^11
constexpr double kLn2Lo = 0x1.ef35793c76730p-45;
constexpr double kPi = 3.141592653589793116;
constexpr double kPio2Hi = 0x1.921fb54400000p0;  // trailing zeros
constexpr double kPio2Lo = 0x1.0b4611a626331p-34;

// natural log, x > 0 normal: x = m 2^e, m in [sqrt(1/2), sqrt(2)), atanh series
RSH double plog(double x) {
  uint64_t b = double_to_bits(x);
  int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
  b = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  double m = bits_to_double(b);
  if (m > 1.4142135623730951) {
    m = RS_MUL(m, 0.5);
    e += 1;
  }
  const double s = RS_DIV(RS_SUB(m, 1.0), RS_ADD(m, 1.0));
  const double s2 = RS_MUL(s, s);
  double p = 1.0 / 23.0;
  p = RS_ADD(1.0 / 21.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 19.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 17.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 15.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 13.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 11.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 9.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 7.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 5.0, RS_MUL(s2, p));
  p = RS_ADD(1.0 / 3.0, RS_MUL(s2, p));
  p = RS_ADD(1.0, RS_MUL(s2, p));
  const double lm = RS_MUL(RS_MUL(2.0, s), p);
  const double ed = static_cast<double>(e);
  return RS_ADD(RS_MUL(ed, kLn2Hi), RS_ADD(RS_MUL(ed, kLn2Lo), lm));
}

// exp(x), |x| < 700: x = k ln2 + r, Taylor to degree 13, scale by 2^k via the exponent
RSH double pexp(double x) {
  const double k = RS_FLOOR(RS_ADD(RS_MUL(x, 1.0 / kLn2), 0.5));
  const double r = RS_SUB(RS_SUB(x, RS_MUL(k, kLn2Hi)), RS_MUL(k, kLn2Lo));
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = RS_ADD(1.0 / 479001600.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 39916800.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 3628800.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 362880.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 40320.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 5040.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 720.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 120.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 24.0, RS_MUL(r, p));
  p = RS_ADD(1.0 / 6.0, RS_MUL(r, p));
  p = RS_ADD(0.5, RS_MUL(r, p));
  p = RS_ADD(1.0, RS_MUL(r, p));
  p = RS_ADD(1.0, RS_MUL(r, p));
  const int ki = static_cast<int>(k);
  return bits_to_double(double_to_bits(p) + (static_cast<uint64_t>(static_cast<int64_t>(ki)) << 52));
}

// sin and cos of x, |x| < 64: quadrant reduction by pi/2 (Cody-Waite), Taylor polynomials
RSH void psincos(double x, double* sn, double* cs) {
  const double k = RS_FLOOR(RS_ADD(RS_MUL(x, 2.0 / kPi), 0.5));
  const double r = RS_SUB(RS_SUB(x, RS_MUL(k, kPio2Hi)), RS_MUL(k, kPio2Lo));
  const double r2 = RS_MUL(r, r);
  double s = -1.0 / 1307674368000.0;  // -1/15!
  s = RS_ADD(1.0 / 6227020800.0, RS_MUL(r2, s));
  s = RS_ADD(-1.0 / 39916800.0, RS_MUL(r2, s));
  s = RS_ADD(1.0 / 362880.0, RS_MUL(r2, s));
  s = RS_ADD(-1.0 / 5040.0, RS_MUL(r2, s));
  s = RS_ADD(1.0 / 120.0, RS_MUL(r2, s));
  s = RS_ADD(-1.0 / 6.0, RS_MUL(r2, s));
  s = RS_ADD(r, RS_MUL(RS_MUL(r, r2), s));
  double c = 1.0 / 20922789888000.0;  // 1/16!
  c = RS_ADD(-1.0 / 87178291200.0, RS_MUL(r2, c));
  c = RS_ADD(1.0 / 479001600.0, RS_MUL(r2, c));
  c = RS_ADD(-1.0 / 3628800.0, RS_MUL(r2, c));
  c = RS_ADD(1.0 / 40320.0, RS_MUL(r2, c));
  c = RS_ADD(-1.0 / 720.0, RS_MUL(r2, c));
  c = RS_ADD(1.0 / 24.0, RS_MUL(r2, c));
  c = RS_ADD(-0.5, RS_MUL(r2, c));
  c = RS_ADD(1.0, RS_MUL(r2, c));
  const int q = static_cast<int>(static_cast<int64_t>(k) & 3);
  const double sv = q == 0 ? s : (q == 1 ? c : (q == 2 ? -s : -c));
  const double cv = q == 0 ? c : (q == 1 ? -s : (q == 2 ? -c : s));
  *sn = sv;
  *cs = cv;
}

// ---- the sampler ------------------------------------------------------------------
struct SamplerSpecD {  // mirrors rs_sampler_spec (include/roomsim_gpu.h)
  double dim_lo[3], dim_hi[3];
  double refl_lo, refl_hi, t60_max;
  double t60_lo, t60_hi;
  double snr_lo, snr_hi;
  double mic_spacing, mic_radius, clearance;
  double sec_lo, sec_hi;
  double fs, c0, signal_std;
  int32_t num_noises, mic_count, n_weights, pad;
  double weights[8];
};

constexpr uint32_t kTagScene = 0x5CE7Eu, kTagSignal = 0x516Au;

// noise count for utterance `utt` (the first draws of its stream)
RSH int sampler_num_noises(const SamplerSpecD& sp, uint64_t seed, uint64_t utt, uint64_t epoch) {
  if (sp.n_weights <= 0) return sp.num_noises;
  Stream g(seed, utt, epoch, kTagScene + 1);
  double tot = 0.0;
  for (int i = 0; i < sp.n_weights; ++i) tot = RS_ADD(tot, sp.weights[i]);
  const double u = RS_MUL(g.next(), tot);
  double cum = 0.0;
  for (int i = 0; i < sp.n_weights; ++i) {
    cum = RS_ADD(cum, sp.weights[i]);
    if (u < cum) return i;
  }
  return sp.n_weights - 1;
}

struct SceneOut {
  double room[3], refl;
  int32_t order;
  int64_t horizon, n_samples;
};

// One utterance: room, reflection, T60 -> K and horizon, I sources (row 0 target),
// J mics, SNRs, N_x.  `src`/`mic`/`snr` have room for I / J / I entries.
RSH SceneOut sampler_scene(const SamplerSpecD& sp, uint64_t seed, uint64_t utt, uint64_t epoch, int n_src,
                           double* src, double* mic, double* snr) {
  Stream g(seed, utt, epoch, kTagScene);
  SceneOut o{};
  double t60 = 0.0;
  for (int attempt = 0;; ++attempt) {  // rejection: T60 inside the spec
    for (int a = 0; a < 3; ++a) o.room[a] = g.uniform(sp.dim_lo[a], sp.dim_hi[a]);
    const double V = RS_MUL(RS_MUL(o.room[0], o.room[1]), o.room[2]);
    const double S = RS_MUL(2.0, RS_ADD(RS_ADD(RS_MUL(o.room[0], o.room[1]), RS_MUL(o.room[0], o.room[2])),
                                        RS_MUL(o.room[1], o.room[2])));
    if (sp.t60_hi > 0.0) {  // sample T60, solve r from Eyring: r = exp(-0.0805 V / (S T60))
      t60 = g.uniform(sp.t60_lo, sp.t60_hi);
      o.refl = pexp(RS_DIV(RS_MUL(-0.0805, V), RS_MUL(S, t60)));
      if (o.refl > 0.0 && o.refl < 1.0) break;
    } else {  // sample r, Eyring T60 = 0.161 V / (-S ln r^2)
      o.refl = g.uniform(sp.refl_lo, sp.refl_hi);
      t60 = RS_DIV(RS_MUL(0.161, V), RS_MUL(-S, plog(RS_MUL(o.refl, o.refl))));
      if (t60 <= sp.t60_max) break;
    }
    if (attempt > 10000) break;  // spec error guard (ranges incompatible)
  }
  const double nrm = RS_SQRT(RS_ADD(RS_ADD(RS_MUL(o.room[0], o.room[0]), RS_MUL(o.room[1], o.room[1])),
                                    RS_MUL(o.room[2], o.room[2])));
  o.order = static_cast<int32_t>(RS_CEIL(RS_DIV(RS_MUL(sp.c0, t60), nrm)));
  o.horizon = static_cast<int64_t>(RS_CEIL(RS_MUL(t60, sp.fs)));
  const double c = sp.clearance;
  for (int i = 0; i < n_src; ++i)
    for (int a = 0; a < 3; ++a) src[3 * i + a] = g.uniform(c, RS_SUB(o.room[a], c));
  const double ext = sp.mic_radius > 0.0 ? sp.mic_radius : RS_MUL(sp.mic_spacing, 0.5);
  double centre[3];
  centre[0] = g.uniform(RS_ADD(c, ext), RS_SUB(RS_SUB(o.room[0], c), ext));
  centre[1] = g.uniform(RS_ADD(c, ext), RS_SUB(RS_SUB(o.room[1], c), ext));
  centre[2] = g.uniform(c, RS_SUB(o.room[2], c));
  const double phi = RS_MUL(RS_MUL(2.0, kPi), g.next());
  const int J = sp.mic_count;
  if (sp.mic_radius > 0.0) {
    for (int m = 0; m < J; ++m) {
      const double ang = RS_ADD(phi, RS_DIV(RS_MUL(RS_MUL(2.0, kPi), static_cast<double>(m)), static_cast<double>(J)));
      double sn, cs;
      psincos(ang, &sn, &cs);
      mic[3 * m + 0] = RS_ADD(centre[0], RS_MUL(sp.mic_radius, cs));
      mic[3 * m + 1] = RS_ADD(centre[1], RS_MUL(sp.mic_radius, sn));
      mic[3 * m + 2] = centre[2];
    }
  } else {
    double sn, cs;
    psincos(phi, &sn, &cs);
    const double h = RS_MUL(sp.mic_spacing, 0.5);
    for (int m = 0; m < J && m < 2; ++m) {
      const double sg = m == 0 ? -1.0 : 1.0;
      mic[3 * m + 0] = RS_ADD(centre[0], RS_MUL(sg, RS_MUL(cs, h)));
      mic[3 * m + 1] = RS_ADD(centre[1], RS_MUL(sg, RS_MUL(sn, h)));
      mic[3 * m + 2] = centre[2];
    }
  }
  snr[0] = 0.0;
  for (int i = 1; i < n_src; ++i) snr[i] = g.uniform(sp.snr_lo, sp.snr_hi);
  const double secs = g.uniform(sp.sec_lo, sp.sec_hi);
  o.n_samples = static_cast<int64_t>(RS_FLOOR(RS_ADD(RS_MUL(secs, sp.fs), 0.5)));
  return o;
}

// ---- FP32 restatements for the signal generator (same construction, fewer terms) ----
RSH float plogf_(float x) {  // x in (0, 1]
  uint32_t b;
  memcpy(&b, &x, 4);
  int e = static_cast<int>((b >> 23) & 0xff) - 127;
  b = (b & 0x007FFFFFu) | 0x3F800000u;
  float m;
  memcpy(&m, &b, 4);
  if (m > 1.41421356f) {
    m = RF_MUL(m, 0.5f);
    e += 1;
  }
  const float s = RF_DIV(RF_SUB(m, 1.0f), RF_ADD(m, 1.0f));
  const float s2 = RF_MUL(s, s);
  float p = 1.0f / 11.0f;
  p = RF_ADD(1.0f / 9.0f, RF_MUL(s2, p));
  p = RF_ADD(1.0f / 7.0f, RF_MUL(s2, p));
  p = RF_ADD(1.0f / 5.0f, RF_MUL(s2, p));
  p = RF_ADD(1.0f / 3.0f, RF_MUL(s2, p));
  p = RF_ADD(1.0f, RF_MUL(s2, p));
  const float ed = static_cast<float>(e);
  return RF_ADD(RF_MUL(ed, 0.693147182f), RF_MUL(RF_MUL(2.0f, s), p));
}

RSH void psincosf_(float x, float* sn, float* cs) {  // x in [0, 2 pi)
  const float k = RF_FLOOR(RF_ADD(RF_MUL(x, 0.636619772f), 0.5f));
  const float r = RF_SUB(RF_SUB(x, RF_MUL(k, 1.5703125f)), RF_MUL(k, 4.83826794e-4f));  // pi/2 = hi + lo
  const float r2 = RF_MUL(r, r);
  float s = 1.0f / 362880.0f;
  s = RF_ADD(-1.0f / 5040.0f, RF_MUL(r2, s));
  s = RF_ADD(1.0f / 120.0f, RF_MUL(r2, s));
  s = RF_ADD(-1.0f / 6.0f, RF_MUL(r2, s));
  s = RF_ADD(r, RF_MUL(RF_MUL(r, r2), s));
  float c = 1.0f / 3628800.0f;
  c = RF_ADD(-1.0f / 40320.0f, RF_MUL(r2, c));
  c = RF_ADD(1.0f / 720.0f, RF_MUL(r2, c));
  c = RF_ADD(-1.0f / 24.0f, RF_MUL(r2, c));
  c = RF_ADD(0.5f, RF_MUL(r2, c));  // 1/2 - r^2 (1/24 - ...)
  c = RF_SUB(1.0f, RF_MUL(r2, c));
  const int q = static_cast<int>(k) & 3;
  *sn = q == 0 ? s : (q == 1 ? c : (q == 2 ? -s : -c));
  *cs = q == 0 ? c : (q == 1 ? -s : (q == 2 ? -c : s));
}

// Two samples N(0, std) by Box-Muller in FP32 from two 24-bit uniforms.
RSH void box_muller(float sd, uint32_t a, uint32_t b, float* z0, float* z1) {
  const float u0 = static_cast<float>(a >> 8) * 0x1.0p-24f;  // exact, [0, 1)
  const float u1 = static_cast<float>(b >> 8) * 0x1.0p-24f;
  const float r = RF_SQRT(RF_MUL(-2.0f, plogf_(RF_SUB(1.0f, u0))));  // 1 - u0 in (0, 1]
  float sn, cs;
  psincosf_(RF_MUL(6.28318548f, u1), &sn, &cs);
  *z0 = RF_MUL(sd, RF_MUL(r, cs));
  *z1 = RF_MUL(sd, RF_MUL(r, sn));
}

#ifdef __CUDA_ARCH__
// ---- device: the two Box-Muller pairs of a quad in the two halves of packed FP32x2 ops ----
// Every half executes box_muller's exact IEEE operation sequence (round to nearest), so the
// samples equal the host's bit for bit.  Products go through fma.rn.f32x2(a, b, -0): that
// is round(a*b) exactly (also for signed zeros), and unlike mul.rn.f32x2 ptxas cannot fuse
// it with the following add into an FFMA2 (which would skip a rounding).
struct F2 {
  float x, y;
};
__device__ __forceinline__ unsigned long long f2b(F2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ F2 b2f(unsigned long long v) {
  F2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// The -0 addend must be a run-time value: with an immediate, ptxas rewrites the fma into a
// multiply and then contracts multiply + add into one FFMA2 after all.
__device__ __forceinline__ F2 pmul(F2 a, F2 b, unsigned long long nz) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2b(a)), "l"(f2b(b)), "l"(nz));
  return b2f(d);
}
__device__ __forceinline__ F2 padd(F2 a, F2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2b(a)), "l"(f2b(b)));
  return b2f(d);
}
__device__ __forceinline__ F2 psub(F2 a, F2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2b(a)), "l"(f2b(b)));
  return b2f(d);
}
__device__ __forceinline__ F2 bc(float v) { return F2{v, v}; }

// plogf_ on both halves (x in (0, 1])
__device__ __forceinline__ F2 plogf2(F2 x, unsigned long long nz) {
  float mv[2];
  float ev[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t b = __float_as_uint(h ? x.y : x.x);
    int e = static_cast<int>((b >> 23) & 0xff) - 127;
    b = (b & 0x007FFFFFu) | 0x3F800000u;
    float m = __uint_as_float(b);
    if (m > 1.41421356f) {
      m = __fmul_rn(m, 0.5f);
      e += 1;
    }
    mv[h] = m;
    ev[h] = static_cast<float>(e);
  }
  const F2 m{mv[0], mv[1]};
  const F2 num = psub(m, bc(1.0f)), den = padd(m, bc(1.0f));
  const F2 sv{__fdiv_rn(num.x, den.x), __fdiv_rn(num.y, den.y)};
  const F2 s2 = pmul(sv, sv, nz);
  F2 p = bc(1.0f / 11.0f);
  p = padd(bc(1.0f / 9.0f), pmul(s2, p, nz));
  p = padd(bc(1.0f / 7.0f), pmul(s2, p, nz));
  p = padd(bc(1.0f / 5.0f), pmul(s2, p, nz));
  p = padd(bc(1.0f / 3.0f), pmul(s2, p, nz));
  p = padd(bc(1.0f), pmul(s2, p, nz));
  return padd(pmul(F2{ev[0], ev[1]}, bc(0.693147182f), nz), pmul(pmul(bc(2.0f), sv, nz), p, nz));
}

// psincosf_ on both halves (x in [0, 2 pi))
__device__ __forceinline__ void psincosf2(F2 x, F2* sn, F2* cs, unsigned long long nz) {
  const F2 kk = padd(pmul(x, bc(0.636619772f), nz), bc(0.5f));
  const F2 k{floorf(kk.x), floorf(kk.y)};
  const F2 r = psub(psub(x, pmul(k, bc(1.5703125f), nz)), pmul(k, bc(4.83826794e-4f), nz));
  const F2 r2 = pmul(r, r, nz);
  F2 s = bc(1.0f / 362880.0f);
  s = padd(bc(-1.0f / 5040.0f), pmul(r2, s, nz));
  s = padd(bc(1.0f / 120.0f), pmul(r2, s, nz));
  s = padd(bc(-1.0f / 6.0f), pmul(r2, s, nz));
  s = padd(r, pmul(pmul(r, r2, nz), s, nz));
  F2 c = bc(1.0f / 3628800.0f);
  c = padd(bc(-1.0f / 40320.0f), pmul(r2, c, nz));
  c = padd(bc(1.0f / 720.0f), pmul(r2, c, nz));
  c = padd(bc(-1.0f / 24.0f), pmul(r2, c, nz));
  c = padd(bc(0.5f), pmul(r2, c, nz));
  c = psub(bc(1.0f), pmul(r2, c, nz));
  float so[2], co[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float sh = h ? s.y : s.x, ch = h ? c.y : c.x;
    const int q = static_cast<int>(h ? k.y : k.x) & 3;
    so[h] = q == 0 ? sh : (q == 1 ? ch : (q == 2 ? -sh : -ch));
    co[h] = q == 0 ? ch : (q == 1 ? -sh : (q == 2 ? -ch : sh));
  }
  *sn = F2{so[0], so[1]};
  *cs = F2{co[0], co[1]};
}

// box_muller(sd, a0, b0) -> z[0], z[1] and box_muller(sd, a1, b1) -> z[2], z[3]
__device__ __forceinline__ void box_muller2(float sd, uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1, float* z) {
  // -0 in both halves, from the run-time standard deviation (ptxas cannot fold it)
  const float nzf = __fmul_rn(-0.0f, fabsf(sd));
  const unsigned long long nz = f2b(F2{nzf, nzf});
  const F2 u0{static_cast<float>(a0 >> 8) * 0x1.0p-24f, static_cast<float>(a1 >> 8) * 0x1.0p-24f};  // exact
  const F2 u1{static_cast<float>(b0 >> 8) * 0x1.0p-24f, static_cast<float>(b1 >> 8) * 0x1.0p-24f};
  const F2 lg = plogf2(psub(bc(1.0f), u0), nz);
  const F2 t = pmul(bc(-2.0f), lg, nz);
  const F2 r{__fsqrt_rn(t.x), __fsqrt_rn(t.y)};
  F2 sn, cs;
  psincosf2(pmul(bc(6.28318548f), u1, nz), &sn, &cs, nz);
  const F2 zc = pmul(bc(sd), pmul(r, cs, nz), nz), zs = pmul(bc(sd), pmul(r, sn, nz), nz);
  z[0] = zc.x;
  z[1] = zs.x;
  z[2] = zc.y;
  z[3] = zs.y;
}
#endif

// Samples 4q .. 4q+3 of a source stream: counter q of the stream's Philox sequence gives
// four 32-bit words, two Box-Muller pairs.
RSH void signal_quad(const SamplerSpecD& sp, const Stream& g, uint64_t q, float* z) {
  const U4 w = philox4x32_10(U4{static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), g.tag, 0x51A1u},
                             g.k0, g.k1);
  const float sd = static_cast<float>(sp.signal_std);
#ifdef __CUDA_ARCH__
  box_muller2(sd, w.x, w.y, w.z, w.w, z);
#else
  box_muller(sd, w.x, w.y, z, z + 1);
  box_muller(sd, w.z, w.w, z + 2, z + 3);
#endif
}

}  // namespace rsg

// fft.cuh — FP32 complex FFT building blocks for sm_100a.
//
// Replaces the reference's RadixTwoRealFft (roomsim/fft.hpp:57-169) on the
// device.  Design:
//   * a real transform of size N is a complex transform of size M = N/2 of
//     the packed signal z[k] = x[2k] + i x[2k+1] (the reference's packing,
//     fft.hpp:51-56, :92), plus a pairing pass over (k, M-k);
//   * the complex transform is a Stockham autosort FFT: every pass reads R
//     strided elements per butterfly from shared memory into registers,
//     applies twiddles, runs an in-register radix-R DFT (R <= 16) and writes
//     the autosorted result back, so input and output are both in natural
//     order and no bit-reversal pass exists;
//   * shared-memory index i is stored at PAD(i) = i + i/16 so the stride-R
//     writes of the first passes are bank-conflict free;
//   * twiddles come from FP64-accurate tables (rounded once to FP32).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rsg {

// ---- complex helpers ---------------------------------------------------------
// sm_100a has packed FP32x2 instructions (FADD2 / FMUL2 / FFMA2): one issue slot
// for both halves of a complex value, with per-half swizzle / negate / scalar
// broadcast operand modifiers, so a complex add is one instruction and a complex
// multiply two.  The FFT kernels are issue-bound, so this roughly halves their FP32
// instruction count (IEEE round-to-nearest per half, same as the scalar forms).
// RSG_NO_F32X2 selects the scalar forms (A/B measurement).
#ifndef RSG_NO_F32X2
__device__ __forceinline__ unsigned long long f2_u(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 u_f2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(d);
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(d);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
  return u_f2(d);
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)), "l"(f2_u(c)));
  return u_f2(d);
}
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return f2_add(a, b); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return f2_sub(a, b); }
// Half-negated swizzles (i b, conj b) as one FMUL2 by a (+-1, +-1) pair: ptxas folds
// the swap and the one-half negate into operand modifiers (MOV + FADD otherwise).
__device__ __forceinline__ float2 f2_ib(float2 b) { return f2_mul(make_float2(b.y, b.x), make_float2(-1.f, 1.f)); }
__device__ __forceinline__ float2 f2_conj(float2 b) { return f2_mul(b, make_float2(1.f, -1.f)); }
// (a.x b.x - a.y b.y, a.x b.y + a.y b.x) = a.x (b.x, b.y) + a.y (-b.y, b.x): the
// a.x / a.y factors are scalar-broadcast operands
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return f2_fma(make_float2(a.y, a.y), f2_ib(b), f2_mul(make_float2(a.x, a.x), b));
}
// a * conj(b) = a.x (b.x, -b.y) + a.y (b.y, b.x)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return f2_fma(make_float2(a.y, a.y), make_float2(b.y, b.x), f2_mul(make_float2(a.x, a.x), f2_conj(b)));
}
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return f2_mul(a, make_float2(s, s)); }
#else
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
#endif
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 c_rot(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
// multiply by exp(-+ i pi/4) (forward -, inverse +)
template <bool INV>
__device__ __forceinline__ float2 c_w8(float2 a) {
  const float c = 0.70710678118654752f;
#ifndef RSG_NO_F32X2
  // c (a + (a.y, -a.x)) forward, c (a + (-a.y, a.x)) inverse
  return c_scale(c_add(a, c_rot<INV>(a)), c);
#else
  return INV ? make_float2(c * (a.x - a.y), c * (a.x + a.y)) : make_float2(c * (a.x + a.y), c * (a.y - a.x));
#endif
}
// multiply by exp(-+ 3 i pi/4)
template <bool INV>
__device__ __forceinline__ float2 c_w83(float2 a) {
  const float c = 0.70710678118654752f;
#ifndef RSG_NO_F32X2
  // forward c ((a.y, -a.x) - a), inverse c ((-a.y, a.x) - a)
  return c_scale(c_sub(c_rot<INV>(a), a), c);
#else
  return INV ? make_float2(-c * (a.x + a.y), c * (a.x - a.y)) : make_float2(c * (a.y - a.x), -c * (a.x + a.y));
#endif
}

// ---- in-register DFTs, natural order in and out -----------------------------
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  __device__ __forceinline__ static void run(float2*) {}
};

template <bool INV>
struct Dft<2, INV> {
  __device__ __forceinline__ static void run(float2* v) {
    const float2 a = v[0], b = v[1];
    v[0] = c_add(a, b);
    v[1] = c_sub(a, b);
  }
};

template <bool INV>
struct Dft<4, INV> {
  __device__ __forceinline__ static void run(float2* v) {
    const float2 t0 = c_add(v[0], v[2]), t1 = c_sub(v[0], v[2]);
    const float2 t2 = c_add(v[1], v[3]), t3 = c_rot<INV>(c_sub(v[1], v[3]));
    v[0] = c_add(t0, t2);
    v[2] = c_sub(t0, t2);
    v[1] = c_add(t1, t3);
    v[3] = c_sub(t1, t3);
  }
};

template <bool INV>
struct Dft<8, INV> {
  // 8 = 4 (inner, over n1 with n = 2 n1 + n2) x 2 (outer).
  __device__ __forceinline__ static void run(float2* v) {
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, INV>::run(e);
    Dft<4, INV>::run(o);
    o[1] = c_w8<INV>(o[1]);
    o[2] = c_rot<INV>(o[2]);
    o[3] = c_w83<INV>(o[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = c_add(e[k], o[k]);
      v[k + 4] = c_sub(e[k], o[k]);
    }
  }
};

template <bool INV>
struct Dft<16, INV> {
  // 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2.
  __device__ __forceinline__ static void run(float2* v) {
    float2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
      for (int n1 = 0; n1 < 4; ++n1) y[n2][n1] = v[4 * n1 + n2];
      Dft<4, INV>::run(y[n2]);
    }
    // twiddles W16^(n2 k1)
    const float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f;
    const float2 w1 = make_float2(c1, INV ? s1 : -s1);
    const float2 w3 = make_float2(s1, INV ? c1 : -c1);
    y[1][1] = c_mul(y[1][1], w1);
    y[1][2] = c_w8<INV>(y[1][2]);
    y[1][3] = c_mul(y[1][3], w3);
    y[2][1] = c_w8<INV>(y[2][1]);
    y[2][2] = c_rot<INV>(y[2][2]);
    y[2][3] = c_w83<INV>(y[2][3]);
    y[3][1] = c_mul(y[3][1], w3);
    y[3][2] = c_w83<INV>(y[3][2]);
    // W16^9 = -W16^1
    y[3][3] = c_mul(y[3][3], make_float2(-w1.x, -w1.y));
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      float2 z[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
      Dft<4, INV>::run(z);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = z[k2];
    }
  }
};

template <bool INV>
struct Dft<32, INV> {
  // 32 = 16 (inner, over n1 with n = 2 n1 + n2) x 2 (outer): X[k] = E[k] + W32^k O[k],
  // X[k + 16] = E[k] - W32^k O[k].
  __device__ __forceinline__ static void run(float2* v) {
    float2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    Dft<16, INV>::run(e);
    Dft<16, INV>::run(o);
    // W32^k = exp(-+ 2 pi i k / 32), k = 1..15 (k = 4, 8, 12 by the special forms)
    constexpr float C[8] = {1.f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                            0.70710678118654752f, 0.55557023301960218f, 0.38268343236508978f,
                            0.19509032201612825f};
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      if (k == 4) o[k] = c_w8<INV>(o[k]);
      else if (k == 8) o[k] = c_rot<INV>(o[k]);
      else if (k == 12) o[k] = c_w83<INV>(o[k]);
      else {
        // cos(2 pi k/32), sin(2 pi k/32) from the first-octant table
        const float c = k <= 8 ? C[k] : -C[16 - k];
        const float sn = k <= 8 ? C[8 - k] : C[k - 8];
        o[k] = c_mul(o[k], make_float2(c, INV ? sn : -sn));
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = c_add(e[k], o[k]);
      v[k + 16] = c_sub(e[k], o[k]);
    }
  }
};

// ---- compile-time plan of an M-point complex FFT ----------------------------
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

template <int M>
struct Plan {
  static constexpr int LOG = ilog2(M);
  // complex elements per thread: whole transform for M < 16, else 16 (32 for
  // the two largest sizes so that T <= 512 threads keeps 128 registers).
#ifndef RSG_E
#define RSG_E 16  // complex elements (max radix) per thread for M >= 1024
#endif
#ifndef RSG_E_SMALL
#define RSG_E_SMALL 8  // ... for M <= 512
#endif
  // complex elements (= max radix) per thread, per size (measured on B200):
  // 8 up to M = 512, 16 above, 32 for the two largest (T <= 512 threads)
  static constexpr int E = M < RSG_E_SMALL ? M : (M >= 8192 ? 32 : (M <= 512 ? RSG_E_SMALL : RSG_E));
  static constexpr int T = M / E;                          // threads per transform
  static constexpr int LE = ilog2(E < 16 ? E : (E >= 32 ? 32 : 16));  // log2 of the max radix
  static constexpr int NP = LOG == 0 ? 1 : (LOG + LE - 1) / LE;  // Stockham passes
  // Layout of the array between passes: PAD(i) = i + i/16 by default.  The output
  // of a radix-8 pass with NS = 8 (E = 8 sizes, M >= 128) is written in the
  // Q layout i + 8*(i/64) instead: its butterfly outputs land at 64a + k + 8r,
  // which PAD maps onto the same banks for the two 8-thread groups a, a+1 of a
  // half-warp (2-way conflicts on every 64-bit store); Q moves them 8 banks apart
  // and still reads conflict-free in the next pass.
  __host__ __device__ static constexpr bool q_out(int p) {
    return E == 8 && p >= 1 && p < NP - 1 && ns(p) == 8;
  }
  __host__ __device__ static constexpr bool q_in(int p) { return p >= 1 && q_out(p - 1); }
  static constexpr int PADDED = (E == 8 && NP >= 3) ? M + M / 8 : M + M / 16;  // smem float2 slots
  __host__ __device__ static constexpr int radix(int p) {
    return p < NP - 1 ? (1 << LE) : (1 << (LOG - LE * (NP - 1)));
  }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : ns(p - 1) * radix(p - 1); }
  // offset (in float2) of pass p's twiddle-base table w_k = exp(-2 pi i k / (NS R)),
  // k < NS: the tables of passes 1..p-1 precede it
  __host__ __device__ static constexpr int tw_off(int p) {
    return p <= 1 ? 0 : tw_off(p - 1) + ns(p - 1);
  }
  // total pass-twiddle table size, then the pairing table W^k, k in [0, M/2]
  static constexpr int TW_PASS = NP >= 2 ? tw_off(NP) : 0;
  static constexpr int TW_TOTAL = TW_PASS + M / 2 + 1;
};

__host__ __device__ __forceinline__ constexpr int PAD(int i) { return i + (i >> 4); }

// Q-layout slot of element t + c (t < T <= 64, c a compile-time offset whose
// low six bits plus T stay within 64, so no carry reaches bit 6): one base
// register plus a compile-time offset.
template <int T>
__device__ __forceinline__ int q_slot(int t, int c) {
  return t + c + 8 * (c >> 6);
}

// smem slot of element base + r*STEP.  When STEP is a multiple of 16 the
// padding distributes over the sum, so every r is a compile-time offset from
// one base register (no per-element address arithmetic).
template <int STEP>
__device__ __forceinline__ float2& slot(float2* s, int base, int r) {
  if constexpr (STEP % 16 == 0)
    return s[PAD(base) + r * PAD(STEP)];
  else
    return s[PAD(base + r * STEP)];
}

// Twiddle load that the compiler may not hoist out of the round loop (keeps
// register pressure bounded for the large transforms).
__device__ __forceinline__ float2 ld_tw(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// Twiddle-table load: from shared memory (TWS) or through the non-hoistable
// global path.
template <bool TWS>
__device__ __forceinline__ float2 tw_load(const float2* p) {
  if constexpr (TWS) return *p;
  else return ld_tw(p);
}

// One Stockham pass (p > 0) of a transform stored in smem `s`, executed by the
// T threads of a group (t = thread index within the group).  The caller
// synchronises before the pass; the pass synchronises between its reads and
// writes (in-place) and after its writes.
//
// Thread t runs butterflies j = t + q*T (q < NB).  All smem and twiddle
// addresses are one base register per pass plus compile-time offsets:
//   read   slot(j + r*STRIDE)            = PAD(t) + q*PAD(T) + r*PAD(STRIDE)
//   write  slot((j-k)*R + k + r*NS), k = j mod NS, which is either the same k
//          for every q (NS | T) or k = j (NS >= M/R, the last pass).
// Multiply v[r] by w^r (forward) or conj(w)^r (inverse), r = 1..R-1, with the
// powers generated from the single loaded base w by a shallow product tree
// (at most 5 roundings deep): one coalesced load per butterfly instead of R-1.
template <int R, bool INV>
__device__ __forceinline__ void apply_twiddles(float2* v, float2 w1) {
  auto mul = [](float2 a, float2 b) { return INV ? c_mulc(a, b) : c_mul(a, b); };
  if constexpr (R == 2) {
    v[1] = mul(v[1], w1);
  } else if constexpr (R == 4) {
    const float2 w2 = c_mul(w1, w1), w3 = c_mul(w2, w1);
    v[1] = mul(v[1], w1); v[2] = mul(v[2], w2); v[3] = mul(v[3], w3);
  } else if constexpr (R == 8) {
    const float2 w2 = c_mul(w1, w1), w3 = c_mul(w2, w1), w4 = c_mul(w2, w2);
    v[1] = mul(v[1], w1); v[2] = mul(v[2], w2); v[3] = mul(v[3], w3); v[4] = mul(v[4], w4);
    v[5] = mul(v[5], c_mul(w4, w1)); v[6] = mul(v[6], c_mul(w4, w2)); v[7] = mul(v[7], c_mul(w4, w3));
  } else if constexpr (R == 16) {
    const float2 w2 = c_mul(w1, w1), w3 = c_mul(w2, w1), w4 = c_mul(w2, w2);
    v[1] = mul(v[1], w1); v[2] = mul(v[2], w2); v[3] = mul(v[3], w3); v[4] = mul(v[4], w4);
    v[5] = mul(v[5], c_mul(w4, w1)); v[6] = mul(v[6], c_mul(w4, w2)); v[7] = mul(v[7], c_mul(w4, w3));
    const float2 w8 = c_mul(w4, w4);
    v[8] = mul(v[8], w8);
    v[9] = mul(v[9], c_mul(w8, w1)); v[10] = mul(v[10], c_mul(w8, w2)); v[11] = mul(v[11], c_mul(w8, w3));
    const float2 w12 = c_mul(w8, w4);
    v[12] = mul(v[12], w12);
    v[13] = mul(v[13], c_mul(w12, w1)); v[14] = mul(v[14], c_mul(w12, w2)); v[15] = mul(v[15], c_mul(w12, w3));
  } else if constexpr (R == 32) {
    // w^r = w^(r & 3) w^(r & 12) w^(r & 16): three table levels, at most 6 roundings deep
    float2 lo[4], mid[4];
    lo[0] = make_float2(1.f, 0.f);
    lo[1] = w1;
    lo[2] = c_mul(w1, w1);
    lo[3] = c_mul(lo[2], w1);
    mid[0] = make_float2(1.f, 0.f);
    mid[1] = c_mul(lo[2], lo[2]);      // w^4
    mid[2] = c_mul(mid[1], mid[1]);    // w^8
    mid[3] = c_mul(mid[2], mid[1]);    // w^12
    const float2 w16 = c_mul(mid[2], mid[2]);
#pragma unroll
    for (int r = 1; r < 32; ++r) {
      float2 p = (r & 3) == 0 ? mid[(r >> 2) & 3] : ((r & 12) == 0 ? lo[r & 3] : c_mul(mid[(r >> 2) & 3], lo[r & 3]));
      if (r & 16) p = (r & 15) == 0 ? w16 : c_mul(w16, p);
      v[r] = mul(v[r], p);
    }
  }
}

struct CtaBar {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// L2 layout: PAD(i) + 8*(i/128), the output layout of the fused pairing pass
// (fused_pair_512) — conflict-free for its butterfly -> thread map.
__host__ __device__ __forceinline__ constexpr int L2S(int i) { return i + (i >> 4) + 8 * (i >> 7); }

template <int M, int P, bool INV, class Bar = CtaBar, bool TWS = false, bool L2IN = false>
__device__ __forceinline__ void stockham_pass(float2* s, int t, const float2* __restrict__ tw,
                                              bool active, Bar bar = Bar()) {
  using PL = Plan<M>;
  constexpr int R = PL::radix(P), NS = PL::ns(P), T = PL::T, NB = PL::E / R, STRIDE = M / R;
  static_assert(NB == 1 || T % NS == 0 || NS >= STRIDE, "unsupported pass shape");
  constexpr bool LIN = (NB == 1) || (T % 16 == 0);  // padding distributes over q*T
  constexpr bool SAME_K = (NB == 1) || (T % NS == 0);
  float2 v[NB][R];
  const int kt = t % NS;  // k of butterfly q = 0
  if (active) {
    const float2* sr = s + PAD(t);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (L2IN) {
          static_assert(NB == 1 && STRIDE == 64 && T == 64, "L2 input: the pass after fused_pair_512");
          v[q][r] = s[PAD(t) + 68 * r + 8 * (r >> 1)];  // L2S(t + 64 r), t < 64
        } else if constexpr (PL::q_in(P))
          v[q][r] = s[q_slot<T>(t, q * T + r * STRIDE)];
        else if constexpr (STRIDE % 16 == 0 && LIN)
          v[q][r] = sr[q * PAD(T) + r * PAD(STRIDE)];
        else
          v[q][r] = s[PAD(t + q * T + r * STRIDE)];
      }
      if constexpr (NS > 1) {
        const float2 w1 = tw_load<TWS>(tw + PL::tw_off(P) + (SAME_K ? kt : t + q * T));
        apply_twiddles<R, INV>(v[q], w1);
      }
      Dft<R, INV>::run(v[q]);
    }
  }
  bar();
  if (active) {
    if constexpr (NS == 1 && R == 16 && NB == 1) {
      float2* sw = s + 17 * t;  // PAD(16 t + r) = 17 t + r
#pragma unroll
      for (int r = 0; r < R; ++r) sw[r] = v[0][r];
    } else if constexpr (PL::q_out(P)) {
      // i = 64a + k + 8r + q*T*R with t = 8a + k: Q(i) = i + 8a + q*T*R/8
      static_assert(R == 8 && NS == 8 && T % 8 == 0 && (T * R) % 64 == 0, "Q-layout pass shape");
      float2* sw = s + (t - kt) * R + kt + (t >> 3) * 8;
#pragma unroll
      for (int q = 0; q < NB; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) sw[q * (T * R + T) + r * NS] = v[q][r];
    } else {
      // base of q = 0; for q > 0 the base moves by q*T*R (same k) or q*T (k = j)
      const int base0 = SAME_K ? (t - kt) * R + kt : t;
      constexpr int QSTEP = SAME_K ? T * R : T;
#pragma unroll
      for (int q = 0; q < NB; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (NS % 16 == 0 && QSTEP % 16 == 0 && LIN)
            s[PAD(base0) + q * PAD(QSTEP) + r * PAD(NS)] = v[q][r];
          else
            s[PAD(base0 + q * QSTEP + r * NS)] = v[q][r];
        }
      }
    }
  }
  bar();
}

// Pass 0 of a forward transform whose packed input z[c] = (x[2c], x[2c+1])
// comes straight from global memory: x points at the block start, elements
// at or beyond `take` are the zero padding.  Writes smem, then syncs.
template <int M, class Src, class Bar = CtaBar, bool NOCHK = false>
__device__ __forceinline__ void first_pass(float2* s, int t, bool active, const Src* x, int take,
                                           Bar bar = Bar()) {
  using PL = Plan<M>;
  constexpr int R = PL::radix(0), T = PL::T, NB = PL::E / R, STRIDE = M / R;
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * T;
      const Src* xb = x + 2 * j;
      const int lim = take - 2 * j;
      float2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int off = 2 * r * STRIDE;
        if constexpr (NOCHK) {  // zero padding already in the source buffer
          v[r].x = static_cast<float>(xb[off]);
          v[r].y = static_cast<float>(xb[off + 1]);
        } else {
          v[r].x = off < lim ? static_cast<float>(xb[off]) : 0.f;
          v[r].y = off + 1 < lim ? static_cast<float>(xb[off + 1]) : 0.f;
        }
      }
      Dft<R, false>::run(v);
      if constexpr (R == 16) {
#pragma unroll
        for (int r = 0; r < R; ++r) s[17 * j + r] = v[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) s[PAD(j * R + r)] = v[r];
      }
    }
  }
  bar();
}

// Remaining forward passes 1..NP-1.
template <int M, int P = 1, class Bar = CtaBar, bool TWS = false>
__device__ __forceinline__ void forward_rest(float2* s, int t, const float2* tw, bool active,
                                             Bar bar = Bar()) {
  if constexpr (P < Plan<M>::NP) {
    stockham_pass<M, P, false, Bar, TWS>(s, t, tw, active, bar);
    forward_rest<M, P + 1, Bar, TWS>(s, t, tw, active, bar);
  }
}

// All inverse passes 0..NP-1 from smem to smem (unnormalised, conj twiddles).
template <int M, int P = 0, class Bar = CtaBar>
__device__ __forceinline__ void inverse_all(float2* s, int t, const float2* tw, bool active,
                                            Bar bar = Bar()) {
  if constexpr (P < Plan<M>::NP) {
    stockham_pass<M, P, true>(s, t, tw, active, bar);
    inverse_all<M, P + 1>(s, t, tw, active, bar);
  }
}

// Inverse passes 0..NP-2 (smem -> smem); the last pass is stockham_emit_pass.
template <int M, int P = 0, class Bar = CtaBar, bool TWS = false>
__device__ __forceinline__ void inverse_but_last(float2* s, int t, const float2* tw, bool active,
                                                 Bar bar = Bar()) {
  if constexpr (P + 1 < Plan<M>::NP) {
    stockham_pass<M, P, true, Bar, TWS>(s, t, tw, active, bar);
    inverse_but_last<M, P + 1, Bar, TWS>(s, t, tw, active, bar);
  }
}

// Last inverse pass: reads smem, twiddles, DFT, then a barrier (smem may be
// reused) and hands every output element to `emit(q, r, c, v)` in registers,
// c = complex index in natural order (c = j + r*M/R).
#ifndef EMIT_BATCH
#define EMIT_BATCH 4
#endif
template <int M, class Bar, class Emit, bool TWS = false, bool SYNC = true>
__device__ __forceinline__ void stockham_emit_pass(float2* s, int t, const float2* __restrict__ tw,
                                                   bool active, Bar bar, Emit emit) {
  using PL = Plan<M>;
  constexpr int P = PL::NP - 1;
  constexpr int R = PL::radix(P), NS = PL::ns(P), T = PL::T, NB = PL::E / R, STRIDE = M / R;
  static_assert(NS == STRIDE, "last pass writes natural order");
  constexpr bool LIN = (NB == 1) || (T % 16 == 0);
  float2 v[NB][R];
  if (active) {
    const float2* sr = s + PAD(t);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (PL::q_in(P))
          v[q][r] = s[q_slot<T>(t, q * T + r * STRIDE)];
        else if constexpr (STRIDE % 16 == 0 && LIN)
          v[q][r] = sr[q * PAD(T) + r * PAD(STRIDE)];
        else
          v[q][r] = s[PAD(t + q * T + r * STRIDE)];
      }
      if constexpr (NS > 1) {
        const float2 w1 = tw_load<TWS>(tw + PL::tw_off(P) + t + q * T);  // k = j in the last pass
        apply_twiddles<R, true>(v[q], w1);
      }
      Dft<R, true>::run(v[q]);
    }
  }
  if constexpr (SYNC) bar();
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        emit(q, r, t + q * T + r * STRIDE, v[q][r]);
        // keep the emit's loads from being hoisted all at once (register pressure)
        if ((r & (EMIT_BATCH - 1)) == EMIT_BATCH - 1) asm volatile("" ::: "memory");
      }
  }
}

// OLA spectral step for one transform held in smem (natural order Z = FFT(z)):
// untangle the packed real spectrum (fft.hpp:152-161), multiply by the
// pre-scaled RIR spectrum G = H / (4M) (bins 0..M), and repack for the inverse
// (fft.hpp:104-110).  Per pair (k, M-k), with a = Z[k], b = conj(Z[M-k]):
//   S = a + b, D = -i (a - b), X2 = S + W^k D = 2 X[k], X2m = S - W^k D = 2 conj(X[M-k])
//   P = X2 G[k], Q = X2m conj(G[M-k]), U = P + Q, V = (P - Q) conj(W^k)
//   Z'[k] = U + i V,  Z'[M-k] = conj(U) + i conj(V).
// W^k = exp(-2 pi i k / N) comes from the plan's pairing table.
template <int M, class Bar = CtaBar, bool G_SMEM = false, bool TWS = false>
__device__ __forceinline__ void spectral_multiply(float2* s, int t, const float2* __restrict__ G,
                                                  const float2* __restrict__ W, bool active,
                                                  Bar bar = Bar()) {
  auto ldg = [](const float2* p) { return G_SMEM ? *p : ld_tw(p); };
  auto ldw = [](const float2* p) { return tw_load<TWS>(p); };
  constexpr int T = Plan<M>::T;
  if (active) {
#pragma unroll 2
    for (int k = t; k < (M + 1) / 2; k += T) {  // k in [0, M/2) (k = 0 for M = 1); bin 0 pairs with itself
      const int km = (M - k) & (M - 1);
      const float2 a = s[PAD(k)];
      const float2 b = c_conj(s[PAD(km)]);
      const float2 w = ldw(W + k);
      const float2 S = c_add(a, b);
      const float2 D = c_rot<false>(c_sub(a, b));
      const float2 wD = c_mul(w, D);
      const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
      const float2 P = c_mul(X2, ldg(G + k));
      const float2 Q = c_mulc(X2m, ldg(G + (M - k)));
      const float2 U = c_add(P, Q);
      const float2 V = c_mulc(c_sub(P, Q), w);
      s[PAD(k)] = make_float2(U.x - V.y, U.y + V.x);
      if (k != 0) s[PAD(km)] = make_float2(U.x + V.y, V.x - U.y);
    }
    if (t == 0) {
      if (M >= 2) {  // k = M/2, its own partner
        const int k = M / 2;
        const float2 a = s[PAD(k)];
        const float2 b = c_conj(a);
        const float2 w = ldw(W + k);
        const float2 S = c_add(a, b);
        const float2 D = c_rot<false>(c_sub(a, b));
        const float2 wD = c_mul(w, D);
        const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
        const float2 g = ldg(G + k);
        const float2 P = c_mul(X2, g);
        const float2 Q = c_mulc(X2m, g);
        const float2 U = c_add(P, Q);
        const float2 V = c_mulc(c_sub(P, Q), w);
        s[PAD(k)] = make_float2(U.x - V.y, U.y + V.x);
      }
    }
  }
  bar();
}

// ---- M = 512: last forward pass + untangle x G x repack + first inverse pass in
// registers.  Thread t runs butterfly j = sigma(t) of both passes, chosen so that j and
// its partner 64 - j (which holds Z[M - k] for every k = j + 64 r of j) sit in lanes
// l and l ^ 16 of one warp:  warp 0: lanes 0-15 -> j = 0-15, lane 16 -> 32,
// lanes 17-31 -> 80 - l;  warp 1: lanes 0-15 -> 16-31, lanes 16-31 -> 64 - l.
// Each lane computes the pairs (k, M-k) for its r = 0..3 from the partner's raw
// Z[j' + 64 r'], r' = 4..7 (shuffled in) and returns the partner's outputs (shuffled
// back); j = 0 and j = 32 pair with themselves.  Formulas as spectral_multiply.
// Reads the Q layout (output of the NS = 8 pass), writes the L2 layout.
template <class Bar>
__device__ __forceinline__ void fused_pair_512(float2* s, int t, const float2* tws, const float2* G,
                                               const float2* W, bool active, Bar bar) {
  using PL = Plan<512>;
  constexpr int M = 512;
  static_assert(PL::T == 64 && PL::NP == 3 && PL::radix(2) == 8 && PL::ns(2) == 64, "plan shape");
  const int w = t >> 5, l = t & 31;
  const int j = w == 0 ? (l < 16 ? l : (l == 16 ? 32 : 80 - l)) : (l < 16 ? 16 + l : 64 - l);
  float2 v[8];
  if (active) {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = s[j + 72 * r];  // q_slot(j + 64 r), j < 64
    apply_twiddles<8, false>(v, tws[PL::tw_off(2) + j]);
    Dft<8, false>::run(v);  // v[r] = Z[j + 64 r]
  }
  // partner's raw Z[j' + 64 r'], r' = 4..7 (all lanes shuffle; inactive lanes carry junk)
  float2 pv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    pv[r].x = __shfl_xor_sync(0xffffffffu, v[4 + r].x, 16);
    pv[r].y = __shfl_xor_sync(0xffffffffu, v[4 + r].y, 16);
  }
  // one pair (k, M - k): a = Z[k], b = conj(Z[M - k]) -> (Z'[k], Z'[M - k])
  auto pair = [&](int k, float2 a, float2 b, float2& zk, float2& zm) {
    const float2 wk = W[k];
    const float2 S = c_add(a, b);
    const float2 D = c_rot<false>(c_sub(a, b));
    const float2 wD = c_mul(wk, D);
    const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
    const float2 P = c_mul(X2, G[k]);
    const float2 Q = c_mulc(X2m, G[M - k]);
    const float2 U = c_add(P, Q);
    const float2 V = c_mulc(c_sub(P, Q), wk);
    zk = make_float2(U.x - V.y, U.y + V.x);
    zm = make_float2(U.x + V.y, V.x - U.y);
  };
  float2 out[8];   // Z' of this butterfly
  float2 back[4];  // Z' of the partner's r' = 4..7 (sent back)
  // One code path for all lanes (no divergence): the partner element of r is
  //   j = 0: r' = 8 - r in this lane (r = 0: Z[0] itself, G[M - 0] = G[M]);
  //   j = 32: r' = 7 - r in this lane;  otherwise r' = 7 - r in the partner (pv[3 - r]).
  const bool self0 = j == 0, self32 = j == 32;
  if (active) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2 bsrc = self0 ? v[(8 - r) & 7] : (self32 ? v[7 - r] : pv[3 - r]);
      float2 zk, zm;
      pair(j + 64 * r, v[r], c_conj(bsrc), zk, zm);
      out[r] = zk;
      back[3 - r] = zm;
      if (self32) out[7 - r] = zm;
      if (self0 && r > 0) out[8 - r] = zm;
    }
    if (self0) {  // k = M/2 pairs with itself (one lane)
      float2 zm;
      pair(M / 2, v[4], c_conj(v[4]), out[4], zm);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    float2 got;
    got.x = __shfl_xor_sync(0xffffffffu, back[r].x, 16);
    got.y = __shfl_xor_sync(0xffffffffu, back[r].y, 16);
    if (!self0 && !self32) out[4 + r] = got;
  }
  if (active) Dft<8, true>::run(out);  // inverse pass 0 (NS = 1)
  bar();                               // every thread's reads of s are done
  if (active) {
    float2* sw = s + L2S(8 * j);       // L2S(8 j + r) = L2S(8 j) + r
#pragma unroll
    for (int r = 0; r < 8; ++r) sw[r] = out[r];
  }
  bar();
}

// ---- M = 256: the same fusion for the 8 x 8 x 4 plan (one warp per transform).  The last
// forward pass (radix 4, NS = 64) gives thread t butterflies j = t and t + 32, i.e.
// Z[t + 64 r] (b1) and Z[t + 32 + 64 r] (b2), r < 4; the inverse pass 0 (radix 8, NS = 1)
// needs Z'[t + 32 r], r < 8 — the same eight bins.  The partner of k = t + 64 r is
// M - k = (32 - t) + 32 + 64 (3 - r): lane 32 - t's b2[3 - r] (lanes l and 32 - l; lane
// 16 is its own partner, lane 0 pairs within b1 and within b2).  Each lane computes the
// pairs of its b1 from the partner's raw b2 (shuffled in) and returns the partner's new b2
// (shuffled back).  Reads the Q layout (output of the NS = 8 pass), writes the PAD layout
// inverse pass 1 reads.  Formulas as spectral_multiply.
template <class Bar>
__device__ __forceinline__ void fused_pair_256(float2* s, int t, const float2* tws, const float2* G,
                                               const float2* W, bool active, Bar bar) {
  using PL = Plan<256>;
  constexpr int M = 256;
  static_assert(PL::T == 32 && PL::NP == 3 && PL::radix(2) == 4 && PL::ns(2) == 64 && PL::q_in(2),
                "plan shape");
  float2 b1[4], b2[4];
  if (active) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      b1[r] = s[q_slot<32>(t, 64 * r)];       // element t + 64 r
      b2[r] = s[q_slot<32>(t, 32 + 64 * r)];  // element t + 32 + 64 r
    }
    apply_twiddles<4, false>(b1, tws[PL::tw_off(2) + t]);
    Dft<4, false>::run(b1);  // b1[r] = Z[t + 64 r]
    apply_twiddles<4, false>(b2, tws[PL::tw_off(2) + t + 32]);
    Dft<4, false>::run(b2);  // b2[r] = Z[t + 32 + 64 r]
  }
  const int partner = (32 - t) & 31;
  float2 pv[4];  // partner's raw b2 (all lanes shuffle; inactive lanes carry junk)
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    pv[r].x = __shfl_sync(0xffffffffu, b2[r].x, partner);
    pv[r].y = __shfl_sync(0xffffffffu, b2[r].y, partner);
  }
  auto wk_of = [&](int k) {  // W^k = exp(-2 pi i k / 2M), k in [0, M]: table holds k <= M/2
    if (k <= M / 2) return W[k];
    const float2 w = W[M - k];
    return make_float2(-w.x, w.y);
  };
  auto pair = [&](int k, float2 a, float2 b, float2& zk, float2& zm) {
    const float2 wk = wk_of(k);
    const float2 S = c_add(a, b);
    const float2 D = c_rot<false>(c_sub(a, b));
    const float2 wD = c_mul(wk, D);
    const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
    const float2 P = c_mul(X2, G[k]);
    const float2 Q = c_mulc(X2m, G[M - k]);
    const float2 U = c_add(P, Q);
    const float2 V = c_mulc(c_sub(P, Q), wk);
    zk = make_float2(U.x - V.y, U.y + V.x);
    zm = make_float2(U.x + V.y, V.x - U.y);
  };
  float2 o1[4], o2[4], back[4];
  const bool self0 = t == 0;
  if (active) {
    if (!self0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float2 zk, zm;
        pair(t + 64 * r, b1[r], c_conj(pv[3 - r]), zk, zm);
        o1[r] = zk;
        back[3 - r] = zm;  // the partner's new b2[3 - r] (Z'[M - k])
      }
    } else {  // bins 64 r (b1) and 32 + 64 r (b2) pair within themselves
      float2 zm;
      pair(0, b1[0], c_conj(b1[0]), o1[0], zm);
      pair(64, b1[1], c_conj(b1[3]), o1[1], o1[3]);
      pair(M / 2, b1[2], c_conj(b1[2]), o1[2], zm);
      pair(32, b2[0], c_conj(b2[3]), o2[0], o2[3]);
      pair(96, b2[1], c_conj(b2[2]), o2[1], o2[2]);
#pragma unroll
      for (int r = 0; r < 4; ++r) back[r] = make_float2(0.f, 0.f);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    float2 got;
    got.x = __shfl_sync(0xffffffffu, back[r].x, partner);
    got.y = __shfl_sync(0xffffffffu, back[r].y, partner);
    if (!self0) o2[r] = got;
  }
  float2 v[8];  // Z'[t + 32 r], r < 8
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    v[2 * r] = o1[r];
    v[2 * r + 1] = o2[r];
  }
  if (active) Dft<8, true>::run(v);  // inverse pass 0 (NS = 1)
  bar();                             // every lane's reads of s are done
  if (active) {
#pragma unroll
    for (int r = 0; r < 8; ++r) s[PAD(8 * t + r)] = v[r];
  }
  bar();
}

}  // namespace rsg

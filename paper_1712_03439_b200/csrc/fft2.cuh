// fft2.cuh — complex N-point Stockham transforms for the two-stream OLA filter
// (ola2.cu).  Two real OLA blocks ride in one complex transform (z = x_a + i x_b);
// since h is real, IFFT(FFT(z) H) = (x_a (*) h) + i (x_b (*) h), so the filter
// needs no untangle/repack pass.  The inverse runs its radices in reverse order
// (PlanC<N, true>): its first pass then has the forward last pass's radix and
// butterfly -> element map, so the last forward pass, the multiply by H and the
// first inverse pass run in registers with no shared-memory round trip between
// them (fused_mid).
#pragma once

#include "fft.cuh"

namespace rsg {

// N = 2^LOG complex points, E elements (= max radix) per thread, T = N/E threads.
// Forward: radices (E, ..., E, REM); reversed: (REM, E, ..., E).
#ifndef RSG_OLA2_E
#define RSG_OLA2_E 16
#endif
template <int N_, bool REV, int EMAX = RSG_OLA2_E>
struct PlanC {
  static constexpr int N = N_;
  static constexpr int LOG = ilog2(N);
  static constexpr int E = N < EMAX ? N : EMAX;
  static constexpr int T = N / E;
  static constexpr int LE = ilog2(E);
  static constexpr int NP = LOG == 0 ? 1 : (LOG + LE - 1) / LE;
  static constexpr int REM = 1 << (LOG - LE * (NP - 1));
  __host__ __device__ static constexpr int radix(int p) {
    return REV ? (p == 0 ? REM : E) : (p < NP - 1 ? E : REM);
  }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : ns(p - 1) * radix(p - 1); }
  __host__ __device__ static constexpr int tw_off(int p) { return p <= 1 ? 0 : tw_off(p - 1) + ns(p - 1); }
  static constexpr int TW_PASS = NP >= 2 ? tw_off(NP) : 0;  // pass-base tables (k < NS per pass)
  static constexpr int PADDED = N + N / 16;
};

// Pass P (P >= 1) of plan PL from smem to smem, in place (bar between reads and writes).
template <class PL, int P, bool INV, class Bar>
__device__ __forceinline__ void pass_c(float2* s, int t, const float2* tw, bool active, Bar bar) {
  constexpr int R = PL::radix(P), NS = PL::ns(P), T = PL::T, NB = PL::E / R, STRIDE = PL::N / R;
  static_assert(NB == 1 || T % NS == 0 || NS >= STRIDE, "unsupported pass shape");
  constexpr bool LIN = (NB == 1) || (T % 16 == 0);
  constexpr bool SAME_K = (NB == 1) || (T % NS == 0);
  float2 v[NB][R];
  const int kt = t % NS;
  if (active) {
    const float2* sr = s + PAD(t);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (STRIDE % 16 == 0 && LIN)
          v[q][r] = sr[q * PAD(T) + r * PAD(STRIDE)];
        else
          v[q][r] = s[PAD(t + q * T + r * STRIDE)];
      }
      if constexpr (NS > 1) {
        const float2 w1 = tw[PL::tw_off(P) + (SAME_K ? kt : t + q * T)];
        apply_twiddles<R, INV>(v[q], w1);
      }
      Dft<R, INV>::run(v[q]);
    }
  }
  bar();
  if (active) {
    const int base0 = SAME_K ? (t - kt) * R + kt : t;
    constexpr int QSTEP = SAME_K ? T * R : T;
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (NS % 16 == 0 && QSTEP % 16 == 0 && LIN)
          s[PAD(base0) + q * PAD(QSTEP) + r * PAD(NS)] = v[q][r];
        else
          s[PAD(base0 + q * QSTEP + r * NS)] = v[q][r];
      }
  }
  bar();
}

// Write the outputs of a P = 0 pass (NS = 1: element j*R + r) and sync.
template <class PL, int R, int NB, class Bar>
__device__ __forceinline__ void write_p0(float2* s, int t, float2 (&v)[NB][R], bool active, Bar bar) {
  constexpr int T = PL::T;
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * T;
      if constexpr (R == 16) {
#pragma unroll
        for (int r = 0; r < R; ++r) s[17 * j + r] = v[q][r];  // PAD(16 j + r) = 17 j + r
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) s[PAD(j * R + r)] = v[q][r];
      }
    }
  }
  bar();
}

// Forward pass 0 of two real streams: z[n] = (xa[n], xb[n]), zero at n >= ta / tb.
template <class PL, class Bar>
__device__ __forceinline__ void first_pass_c(float2* s, int t, bool active, const float* xa, int ta,
                                             const float* xb, int tb, Bar bar) {
  constexpr int R = PL::radix(0), T = PL::T, NB = PL::E / R, STRIDE = PL::N / R;
  float2 v[NB][R];
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * T;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = j + r * STRIDE;
        v[q][r] = make_float2(n < ta ? xa[n] : 0.f, n < tb ? xb[n] : 0.f);
      }
      Dft<R, false>::run(v[q]);
    }
  }
  write_p0<PL, R, NB>(s, t, v, active, bar);
}

// Last forward pass of PF, times H, first inverse pass of PI, in registers.
// H[k] = hs[k] for k <= N/2, conj(hs[N - k]) above (h real).
template <class PF, class PI, class Bar>
__device__ __forceinline__ void fused_mid(float2* s, int t, const float2* twf, const float2* hs, bool active,
                                          Bar bar) {
  constexpr int P = PF::NP - 1;
  constexpr int N = PF::N, R = PF::radix(P), NS = PF::ns(P), T = PF::T, NB = PF::E / R, STRIDE = N / R;
  static_assert(PI::radix(0) == R && NS == STRIDE, "fused pass shape");
  float2 v[NB][R];
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * T;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = s[PAD(j + r * STRIDE)];
      if constexpr (NS > 1) apply_twiddles<R, false>(v[q], twf[PF::tw_off(P) + j]);
      Dft<R, false>::run(v[q]);  // v[q][r] = Z[j + r*STRIDE]
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = j + r * STRIDE;
        const float2 h = k <= N / 2 ? hs[k] : c_conj(hs[N - k]);
        v[q][r] = c_mul(v[q][r], h);
      }
      Dft<R, true>::run(v[q]);  // inverse pass 0 (NS = 1: no twiddles)
    }
  }
  bar();
  write_p0<PI, R, NB>(s, t, v, active, bar);
}

// Last inverse pass of PI: reads smem, then hands each output (natural index c)
// to emit(c, v) in registers (after a barrier: smem may be reused).
template <class PI, class Bar, class Emit>
__device__ __forceinline__ void emit_pass_c(float2* s, int t, const float2* twi, bool active, Bar bar,
                                            Emit emit) {
  constexpr int P = PI::NP - 1;
  constexpr int R = PI::radix(P), NS = PI::ns(P), T = PI::T, NB = PI::E / R, STRIDE = PI::N / R;
  static_assert(NS == STRIDE, "last pass writes natural order");
  constexpr bool LIN = (NB == 1) || (T % 16 == 0);
  float2 v[NB][R];
  if (active) {
    const float2* sr = s + PAD(t);
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (STRIDE % 16 == 0 && LIN)
          v[q][r] = sr[q * PAD(T) + r * PAD(STRIDE)];
        else
          v[q][r] = s[PAD(t + q * T + r * STRIDE)];
      }
      if constexpr (NS > 1) apply_twiddles<R, true>(v[q], twi[PI::tw_off(P) + t + q * T]);
      Dft<R, true>::run(v[q]);
    }
  }
  bar();
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        emit(t + q * T + r * STRIDE, v[q][r]);
        if ((r & 3) == 3) asm volatile("" ::: "memory");
      }
  }
}

// Forward passes 1..NP-2 / inverse passes 1..NP-2.
template <class PL, int P, bool INV, class Bar>
__device__ __forceinline__ void middle_passes(float2* s, int t, const float2* tw, bool active, Bar bar) {
  if constexpr (P < PL::NP - 1) {
    pass_c<PL, P, INV>(s, t, tw, active, bar);
    middle_passes<PL, P + 1, INV>(s, t, tw, active, bar);
  }
}

}  // namespace rsg

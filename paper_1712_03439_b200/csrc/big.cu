// big.cu — K4 in place: a mixed-radix FFT that rewrites every butterfly's own slots, one
// work item (a run of OLA blocks of one pair) per CTA, for M = N/2 = 1024 … 16384 (the
// planner's default; M = 512 is supported and opt-in: RSG_IP="9,14" — measured slower than
// ola_small_kernel<512>).
//
// Reference: convolve_ola (convolution.hpp:219-255) with RadixTwoRealFft
// (fft.hpp:57-169): per block, the real N-point transform of the zero-padded
// L-sample block, times H, inverse, overlap-added at b*L; mean_power's Σy²
// (audio_buffer.hpp:66-75) of the final samples.
//
// Why a separate kernel: the Stockham passes of ola_small_kernel<M> hold a thread's whole
// E = 32-element share across the barrier between a pass's reads and writes; at one
// 512-thread CTA per SM (the transform alone is 136 KB of smem) that leaves 128
// registers and the kernel spills ~1 KB per thread (53 GB of local-memory traffic per
// config-5 launch).  Here every pass is in place: a butterfly reads its R elements,
// transforms them and writes them back to the same slots, so no value lives across a
// barrier and a thread holds one butterfly (R <= 32 complex) at a time.
//
//   forward: decimation in frequency (natural order in, digit-reversed out), radices
//            R_0 .. R_{P-1}, twiddles after each butterfly's DFT; pass 0 loads the
//            packed block z[n] = x[2n] + i x[2n+1] straight from the signal;
//   pairing: untangle x G x repack (the formulas of spectral_multiply, fft.cuh) on
//            (k, M - k), both read from their digit-reversed slots, in place;
//   inverse: decimation in time with the passes in reverse order (digit-reversed in,
//            natural out), conj twiddles before each DFT; the last pass hands the
//            outputs c = t + S_0 r to the emit in registers;
//   emit:    overlap carry in smem (N_h - 1 floats, single buffer: all carry reads,
//            barrier, carry writes), every owned output written once, FP32 per-block
//            power partials folded into FP64 in a fixed order (deterministic).
//
// Slot of element i: i + i/16 + i/2^LS0 with 2^LS0 = max(256, S_0).  With the radix orders
// below every access of every pass (strides S_p, the S = 1 blocks, and the pairing's
// k -> digit-reversed slot, which moves by S_0 per k) is bank-conflict free on 64-bit
// accesses.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fft.cuh"
#include "kernels.cuh"
#include "mixfin.cuh"
#include "power.cuh"

namespace rsg {
namespace {

// Per-size tuning (CTAs per SM the register budget is set for; G and the pairing
// table staged in smem or read through L1): measured on B200, config-4 render.
#ifndef RSG_IP_MINB_1024
#define RSG_IP_MINB_1024 8
#endif
#ifndef RSG_IP_GS_1024
#define RSG_IP_GS_1024 true
#endif
#ifndef RSG_IP_MINB_2048
#define RSG_IP_MINB_2048 6
#endif
#ifndef RSG_IP_GS_2048
#define RSG_IP_GS_2048 false
#endif
#ifndef RSG_IP_MINB_4096
#define RSG_IP_MINB_4096 3
#endif
#ifndef RSG_IP_GS_4096
#define RSG_IP_GS_4096 false
#endif

template <int M>
struct IpPlan;
template <>
struct IpPlan<16384> {
  static constexpr int NP = 3, T = 512, MINB = 1, LS0 = 9;
  static constexpr bool GS = false;
  __host__ __device__ static constexpr int radix(int p) { return p == 2 ? 16 : 32; }
};
template <>
struct IpPlan<8192> {
  static constexpr int NP = 3, T = 256, MINB = 2, LS0 = 8;
  static constexpr bool GS = false;
  __host__ __device__ static constexpr int radix(int p) { return p == 0 ? 32 : 16; }
};
template <>
struct IpPlan<512> {
  static constexpr int NP = 3, T = 32, MINB = 16, LS0 = 8;
  static constexpr bool GS = true;
  __host__ __device__ static constexpr int radix(int p) { return p == 1 ? 2 : 16; }
};
template <>
struct IpPlan<1024> {
  static constexpr int NP = 3, T = 64, MINB = RSG_IP_MINB_1024, LS0 = 8;
  static constexpr bool GS = RSG_IP_GS_1024;
  __host__ __device__ static constexpr int radix(int p) { return p == 1 ? 4 : 16; }
};
template <>
struct IpPlan<2048> {
  static constexpr int NP = 3, T = 128, MINB = RSG_IP_MINB_2048, LS0 = 8;
  static constexpr bool GS = RSG_IP_GS_2048;
  __host__ __device__ static constexpr int radix(int p) { return p == 1 ? 8 : 16; }
};
template <>
struct IpPlan<4096> {
  static constexpr int NP = 3, T = 256, MINB = RSG_IP_MINB_4096, LS0 = 8;
  static constexpr bool GS = RSG_IP_GS_4096;
  __host__ __device__ static constexpr int radix(int p) { return 16; }
};
template <class PL, int M>
struct IpShape {
  // S_p = M / (R_0 ... R_p): the stride of pass p; W_p = R_0 ... R_{p-1}: the weight of
  // digit p in the frequency index k = sum m_p W_p (its slot is sum m_p S_p)
  __host__ __device__ static constexpr int stride(int p) { return p < 0 ? M : stride(p - 1) / PL::radix(p); }
  __host__ __device__ static constexpr int weight(int p) { return p == 0 ? 1 : weight(p - 1) * PL::radix(p - 1); }
  // twiddle-base table: pass p (p < NP - 1) holds S_p bases exp(-2 pi i j / (R_p S_p))
  __host__ __device__ static constexpr int tw_off(int p) { return p == 0 ? 0 : tw_off(p - 1) + stride(p - 1); }
  static constexpr int TWN = tw_off(PL::NP - 1);
  // smem-staged filter G (M + 1 bins) and pairing table W (M/2 + 1), float2, even counts
  static constexpr bool GS = PL::GS;
  static constexpr int GSN = (M + 2) & ~1, WSN = (M / 2 + 2) & ~1;
  static constexpr int SLOTS = M + M / 16 + (M >> PL::LS0);
  static_assert(stride(0) == PL::T && stride(PL::NP - 1) == 1, "plan shape");
};

template <class PL>
__device__ __forceinline__ int ipad(int i) { return i + (i >> 4) + (i >> PL::LS0); }

// digit-reversed slot of frequency index k (compile-time powers of two: every digit is
// a shift and a mask)
template <class PL, int M, int P = 0>
__device__ __forceinline__ int ip_pos(unsigned k) {
  using SH = IpShape<PL, M>;
  if constexpr (P == PL::NP) {
    return 0;
  } else {
    constexpr unsigned W = SH::weight(P), R = PL::radix(P), S = SH::stride(P);
    return static_cast<int>(((k / W) % R) * S) + ip_pos<PL, M, P + 1>(k);
  }
}

// Slot offset of element base + r*S from the slot of base, for a butterfly base
// b*R*S + j (j < S): each padding term i/D (D = 16, S_0) either distributes over r*S
// (D <= S) or is constant over the butterfly (D >= R*S, powers of two), so the
// offsets are compile-time constants and a pass needs one slot computation per
// butterfly.
template <int D, int R, int S, int M>
__host__ __device__ constexpr int ip_off_d(int r) {
  // D <= S: distributes; D >= R S: constant over the butterfly; otherwise only a pass with
  // a single block (R S = M, j < S, S | D) adds no carry into bit log2(D)
  return D <= S ? r * S / D : (D >= R * S ? 0 : r * S / D);
}
template <class PL, int R, int S, int M>
__host__ __device__ constexpr int ip_off(int r) {
  return r * S + ip_off_d<16, R, S, M>(r) + ip_off_d<(1 << PL::LS0), R, S, M>(r);
}
template <int D, int R, int S, int M>
__host__ __device__ constexpr bool ip_off_ok() { return D <= S || D >= R * S || (R * S == M && D % S == 0); }

// In-place pass p of the forward (DIF) or inverse (DIT) transform.
template <class PL, int M, int P, bool INV>
__device__ __forceinline__ void ip_pass(float2* s, const float2* tws, int t) {
  using SH = IpShape<PL, M>;
  constexpr int R = PL::radix(P), S = SH::stride(P), NB = M / (R * PL::T);
  static_assert(NB >= 1 && M % (R * PL::T) == 0, "pass shape");
  static_assert(ip_off_ok<16, R, S, M>() && ip_off_ok<(1 << PL::LS0), R, S, M>(),
                "padding terms distribute over the butterfly");
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const unsigned u = static_cast<unsigned>(t + q * PL::T);
    const unsigned j = u % unsigned(S);
    const int pb = ipad<PL>(static_cast<int>((u / unsigned(S)) * unsigned(R * S) + j));
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[pb + ip_off<PL, R, S, M>(r)];
    if constexpr (!INV) {
      Dft<R, false>::run(v);
      if constexpr (S > 1) apply_twiddles<R, false>(v, tws[SH::tw_off(P) + j]);
    } else {
      if constexpr (S > 1) apply_twiddles<R, true>(v, tws[SH::tw_off(P) + j]);
      Dft<R, true>::run(v);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) s[pb + ip_off<PL, R, S, M>(r)] = v[r];
  }
}

template <class PL, int M, int P>
__device__ __forceinline__ void ip_forward_rest(float2* s, const float2* tws, int t) {
  if constexpr (P < PL::NP) {
    ip_pass<PL, M, P, false>(s, tws, t);
    __syncthreads();
    ip_forward_rest<PL, M, P + 1>(s, tws, t);
  }
}
// inverse passes NP-1 .. 1 (pass 0 is the emit pass)
template <class PL, int M, int P>
__device__ __forceinline__ void ip_inverse_rest(float2* s, const float2* tws, int t) {
  if constexpr (P >= 1) {
    ip_pass<PL, M, P, true>(s, tws, t);
    __syncthreads();
    ip_inverse_rest<PL, M, P - 1>(s, tws, t);
  }
}

// One pair (k, M - k) of the spectral step (spectral_multiply, fft.cuh); k = M - k
// pairs only with itself (k = 0: partner slot 0 and G[M]; k = M/2).
template <class PL, int M, bool GS>
__device__ __forceinline__ void ip_pair(float2* s, int k, const float2* __restrict__ G,
                                        const float2* __restrict__ W) {
  auto ld = [](const float2* p) { return GS ? *p : ld_tw(p); };  // smem-staged or global
  const int km = (M - k) & (M - 1);
  const int pa = ipad<PL>(ip_pos<PL, M>(static_cast<unsigned>(k)));
  const int pb = ipad<PL>(ip_pos<PL, M>(static_cast<unsigned>(km)));
  const float2 a = s[pa];
  const float2 b = c_conj(s[pb]);
  const float2 w = ld(W + k);
  const float2 S = c_add(a, b);
  const float2 D = c_rot<false>(c_sub(a, b));
  const float2 wD = c_mul(w, D);
  const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
  const float2 P = c_mul(X2, ld(G + k));
  const float2 Q = c_mulc(X2m, ld(G + (M - k)));
  const float2 U = c_add(P, Q);
  const float2 V = c_mulc(c_sub(P, Q), w);
  s[pa] = make_float2(U.x - V.y, U.y + V.x);
  if (k != 0 && km != k) s[pb] = make_float2(U.x + V.y, V.x - U.y);
}

// One thread: pull [p, p + bytes) into L2 ahead of use (1-D bulk prefetch; the window
// is widened to 16-byte alignment).
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(bytes) + 15) & ~uintptr_t(15);
  for (uintptr_t a = a0; a < a1; a += (1u << 20)) {
    const unsigned n = static_cast<unsigned>(a1 - a < (1u << 20) ? a1 - a : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
  }
}

// Quads per thread per trip of the K4 epilogue's mix (mixfin.cuh).  The mix loop waits on its
// loads (long-scoreboard stalls are 2/3 of its samples), so bytes in flight are its speed: two
// quads of every source per thread, also at 80 registers (12-16 bytes of spills in the epilogue
// only; config 4 measured 26.9-27.1 ms vs 27.3-27.8 ms with one).
#ifndef RSG_FIN_UN_BIG
#define RSG_FIN_UN_BIG 2
#endif
#ifndef RSG_FIN_UN_SMALL
#define RSG_FIN_UN_SMALL 2
#endif
__host__ __device__ constexpr int fin_un(int threads, int minb) {
  return threads * minb <= 512 ? RSG_FIN_UN_BIG : RSG_FIN_UN_SMALL;
}

template <int M>
__global__ void __launch_bounds__(IpPlan<M>::T, IpPlan<M>::MINB) ola_ip_kernel(OlaArgs a, int ccap) {
  using PL = IpPlan<M>;
  using SH = IpShape<PL, M>;
  constexpr int T = PL::T, N = 2 * M;
  constexpr int R0 = PL::radix(0), S0 = SH::stride(0);
  static_assert(S0 == T, "passes 0 (forward) and 0 (inverse): one butterfly per thread");
  extern __shared__ __align__(128) float2 smem[];
  float2* s = smem;
  float2* tws = smem + SH::SLOTS;
  // sizes up to M = 4096 also stage the pair's G and the pairing table W in smem
  constexpr bool GS = SH::GS;
  float2* gs = tws + ((SH::TWN + 1) & ~1);
  float2* ws = gs + (GS ? SH::GSN : 0);
  float* carry = reinterpret_cast<float*>(ws + (GS ? SH::WSN : 0));
  const int t = threadIdx.x;
  const OlaItem it = a.items[blockIdx.x];
  const PairPlan& pl = a.plan[it.pair];
  const PairMeta& pm = a.pair[it.pair];
  const float* __restrict__ x = a.signals + pm.sig_off;
  const long long nx = pm.nx;
  const float2* __restrict__ Gg = a.spec + pl.spec_off;
  const float2* __restrict__ Wg = a.tw + Plan<M>::TW_PASS;  // pairing table W^k, k <= M/2
  const float2* G = GS ? gs : Gg;
  const float2* W = GS ? ws : Wg;
  float* __restrict__ y = a.y + pl.y_off;
  const int L = static_cast<int>(pl.L);
  const int B = static_cast<int>(pl.B);
  const int ovl = N - L;  // N_h - 1 <= ccap
  const long long own_lo = static_cast<long long>(it.b_own) * L;
  const long long own_hi = it.b_end == B ? pl.out_len : static_cast<long long>(it.b_end) * L;
  // twiddle bases, FP64 sincospi rounded once
  for (int i = t; i < SH::TWN; i += T) {
    int p = 0;
#pragma unroll
    for (int q = 1; q < PL::NP - 1; ++q)
      if (i >= SH::tw_off(q)) p = q;
    const int j = i - SH::tw_off(p);
    const int span = PL::radix(p) * SH::stride(p);
    double sn, cs;
    sincospi(-2.0 * j / span, &sn, &cs);
    tws[i] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
  for (int i = t; i < ovl; i += T) carry[i] = 0.f;
  if constexpr (GS) {
    for (int i = t; i <= M; i += T) gs[i] = ld_tw(Gg + i);
    for (int i = t; i <= M / 2; i += T) ws[i] = ld_tw(Wg + i);
  }
  if (t == 0) {  // the pair's filter and the run's first block
    if (!GS) prefetch_l2(Gg, (M + 1) * sizeof(float2));
    const long long s0 = static_cast<long long>(it.b_begin) * L;
    prefetch_l2(x + s0, 4 * (nx - s0 < L ? nx - s0 : L));
  }
  __syncthreads();
  double pw = 0.0;  // this lane's Σ y² of the current power segment
#pragma unroll 1
  for (int b = it.b_begin; b < it.b_end; ++b) {
    const long long start = static_cast<long long>(b) * L;
    const int take = static_cast<int>(nx - start < L ? nx - start : L);
    const float* xb = x + start;
    if (t == 0 && b + 1 < it.b_end) {  // next block's samples land in L2 during this one
      const long long s1 = start + L;
      prefetch_l2(x + s1, 4 * (nx - s1 < L ? nx - s1 : L));
    }
    // forward pass 0 (S_0 = T): z[t + S_0 r] from the signal, zero past `take`
    {
      float2 v[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int n2 = 2 * (t + S0 * r), w0 = 2 * ((t & ~31) + S0 * r);
        if (w0 + 64 <= take) {  // the warp's 64 samples are all in the block (uniform)
          v[r].x = __ldg(xb + n2);
          v[r].y = __ldg(xb + n2 + 1);
        } else {
          v[r].x = n2 < take ? __ldg(xb + n2) : 0.f;
          v[r].y = n2 + 1 < take ? __ldg(xb + n2 + 1) : 0.f;
        }
      }
      Dft<R0, false>::run(v);
      apply_twiddles<R0, false>(v, tws[t]);
#pragma unroll
      for (int r = 0; r < R0; ++r) s[ipad<PL>(t) + ip_off<PL, R0, S0, M>(r)] = v[r];
    }
    __syncthreads();
    ip_forward_rest<PL, M, 1>(s, tws, t);
    // pairs (k, M - k), k in [0, M/2]: consecutive k on consecutive threads
#pragma unroll 2
    for (int k = t; k < M / 2; k += T) ip_pair<PL, M, GS>(s, k, G, W);
    if (t == 0) ip_pair<PL, M, GS>(s, M / 2, G, W);
    __syncthreads();
    ip_inverse_rest<PL, M, PL::NP - 1>(s, tws, t);
    // inverse pass 0: outputs c = t + S_0 r in registers
    float2 v[R0];
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = s[ipad<PL>(t) + ip_off<PL, R0, S0, M>(r)];
    apply_twiddles<R0, true>(v, tws[t]);
    Dft<R0, true>::run(v);
    // Warp-uniform classification per r: the warp's 64 samples e in [w0, w0 + 64)
    // are contiguous, so all but the few r that straddle ovl, L, lo or hi take a
    // branch-free path (float2 carry loads, plain stores).
    const int wt = t & ~31;
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int e = 2 * (t + S0 * r), w0 = 2 * (wt + S0 * r);
      if (w0 + 64 <= ovl) {
        v[r] = c_add(v[r], *reinterpret_cast<const float2*>(carry + e));
      } else if (w0 < ovl) {
        if (e < ovl) v[r].x += carry[e];
        if (e + 1 < ovl) v[r].y += carry[e + 1];
      }
    }
    __syncthreads();  // carry reads and this block's smem reads are done
    const int lo = static_cast<int>(max(own_lo - start, -1ll));
    const int hi = static_cast<int>(min(own_hi - start, static_cast<long long>(N)));
    const int fe = b == B - 1 ? N : L;  // e < fe: final after this block
    float* yb = y + start;
    // 8-byte stores where the block start allows (measured: pays at M >= 8192 only)
    const bool y_al = M >= 8192 && (reinterpret_cast<uintptr_t>(yb) & 7) == 0;  // block-uniform
    const bool c_al = M >= 8192 && (L & 1) == 0;
    float pb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int e = 2 * (t + S0 * r), w0 = 2 * (wt + S0 * r), w1 = w0 + 64;
      if (w1 <= fe && w0 >= lo && w1 <= hi) {  // final and owned
        if (y_al) {
          *reinterpret_cast<float2*>(yb + e) = v[r];
        } else {
          yb[e] = v[r].x;
          yb[e + 1] = v[r].y;
        }
        pb[(r & 1) * 2] = fmaf(v[r].x, v[r].x, pb[(r & 1) * 2]);
        pb[(r & 1) * 2 + 1] = fmaf(v[r].y, v[r].y, pb[(r & 1) * 2 + 1]);
      } else if (w0 >= fe) {  // carried into the next block
        if (c_al) {
          *reinterpret_cast<float2*>(carry + e - L) = v[r];
        } else {
          carry[e - L] = v[r].x;
          carry[e + 1 - L] = v[r].y;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int eh = e + h;
          const float val = h ? v[r].y : v[r].x;
          if (eh < fe) {
            if (eh >= lo && eh < hi) {
              yb[eh] = val;
              pb[(r & 1) * 2 + h] = fmaf(val, val, pb[(r & 1) * 2 + h]);
            }
          } else {
            carry[eh - L] = val;
          }
        }
      }
    }
    // power: per-lane FP64 sum over the segment, stored at its end (power.cuh)
    pw += static_cast<double>((pb[0] + pb[1]) + (pb[2] + pb[3]));
    if (closes_segment(b, it.b_end, a.seg)) {
      const long long part0 = __ldg(&a.plan[it.pair].part0);  // reloaded: nothing 64-bit lives across blocks
      store_segment_power<T>(a.part + part0 + static_cast<long long>(b / a.seg) * parts_per_block_of(T), pw, t,
                             b >= it.b_own);
      pw = 0.0;
    }
  }
  // the channel's last work item mixes it (mixfin.cuh); the transform buffer is free by now
  finish_item<T, fin_un(T, PL::MINB)>(a.fin, it.pair, t, reinterpret_cast<unsigned char*>(smem));
}

template <int M>
size_t ip_smem(int ccap) {
  using SH = IpShape<IpPlan<M>, M>;
  return (static_cast<size_t>(SH::SLOTS) + ((SH::TWN + 1) & ~1) + (SH::GS ? SH::GSN + SH::WSN : 0)) *
             sizeof(float2) +
         static_cast<size_t>(ccap) * sizeof(float);
}

template <int M>
cudaError_t ip_t(const OlaArgs& a, int ccap, cudaStream_t st) {
  const size_t smem = ip_smem<M>(ccap);
  cudaError_t e = ensure_dynamic_smem(ola_ip_kernel<M>, smem);
  if (e != cudaSuccess) return e;
  ola_ip_kernel<M><<<a.count, IpPlan<M>::T, smem, st>>>(a, ccap);
  return cudaGetLastError();
}


// ============================================================================
// K4 "two blocks per transform" (ola_ipc_kernel<C>): consecutive OLA blocks 2j and 2j + 1
// of one pair ride one C = N point COMPLEX transform, z = x_a + i x_b.  h is real, so
// IFFT(FFT(z) H) = (x_a * h) + i (x_b * h): no untangle / repack step, and the product
// with H is pointwise — it runs in registers between the last forward pass (stride 1)
// and the first inverse pass, which share one butterfly's slots.  Per block that is 4
// reads + 4 writes of N/2 complex in shared memory against 6 + 6 (plus the filter and
// the pairing table through L1) in ola_ip_kernel<N/2>, which is shared-memory bound.
// The filter is read from Gp, K3's copy of H / N over all N bins in the order the
// butterflies want it: Gp[r * (C / R) + u] is the bin of element r of the last pass's
// butterfly u (IpcPerm), so a warp's loads are contiguous.  Block 2j always pairs with
// block 2j + 1 (zero past the pair's last block): which blocks share a transform
// depends on the pair only, whatever the run split (render invariance).
// Reference: convolve_ola, convolution.hpp:219-255; mean_power, audio_buffer.hpp:66-75.
// ============================================================================
// The product step reads the pair's H through L1 (the CTA re-reads the same 32-64 KB every
// transform; written by this CTA before its first block, or by K3 in an earlier launch): K4
// alone 19.7-20.1 -> 19.4-19.5 ms per config-4 render against L2-only loads.
#ifndef RSG_IPC_H_L1
#define RSG_IPC_H_L1 1
#endif
#ifndef RSG_IPC_MINB_4096
#define RSG_IPC_MINB_4096 3
#endif
#ifndef RSG_IPC_MINB_8192
#define RSG_IPC_MINB_8192 2
#endif
template <int C>
struct IpcPlan;
template <>
struct IpcPlan<4096> {
  static constexpr int NP = 3, T = 256, MINB = RSG_IPC_MINB_4096, LS0 = 8;
  static constexpr bool GS = false, DB = true;
  __host__ __device__ static constexpr int radix(int) { return 16; }
};
template <>
struct IpcPlan<8192> {
  static constexpr int NP = 3, T = 256, MINB = RSG_IPC_MINB_8192, LS0 = 8;
  static constexpr bool GS = false, DB = false;
  __host__ __device__ static constexpr int radix(int p) { return p == 0 ? 32 : 16; }
};

template <class PL, int C, int P>
__device__ __forceinline__ void ipc_forward_mid(float2* s, const float2* tws, int t) {
  if constexpr (P < PL::NP - 1) {
    ip_pass<PL, C, P, false>(s, tws, t);
    __syncthreads();
    ipc_forward_mid<PL, C, P + 1>(s, tws, t);
  }
}
template <class PL, int C, int P>
__device__ __forceinline__ void ipc_inverse_mid(float2* s, const float2* tws, int t) {
  if constexpr (P >= 1) {
    ip_pass<PL, C, P, true>(s, tws, t);
    __syncthreads();
    ipc_inverse_mid<PL, C, P - 1>(s, tws, t);
  }
}

template <int C>
__global__ void __launch_bounds__(IpcPlan<C>::T, IpcPlan<C>::MINB) ola_ipc_kernel(OlaArgs a, int ccap) {
  using PL = IpcPlan<C>;
  using SH = IpShape<PL, C>;
  constexpr int T = PL::T;
  constexpr int R0 = PL::radix(0), S0 = SH::stride(0);
  constexpr int RL = PL::radix(PL::NP - 1), NBL = C / (RL * T);  // last pass: stride 1
  static_assert(S0 == T, "passes 0 (forward) and 0 (inverse): one butterfly per thread");
  static_assert(SH::stride(PL::NP - 1) == 1 && RL == 16 && NBL >= 1, "last pass shape");
  constexpr bool DB = PL::DB;  // double-buffered carry
  extern __shared__ __align__(128) float2 smem[];
  float2* s = smem;
  float2* tws = smem + SH::SLOTS;
  float* carry = reinterpret_cast<float*>(tws + ((SH::TWN + 1) & ~1));
  const int t = threadIdx.x;
  const OlaItem it = a.items[blockIdx.x];
  const PairPlan& pl = a.plan[it.pair];
  const PairMeta& pm = a.pair[it.pair];
  const float* __restrict__ x = a.signals + pm.sig_off;
  const long long nx = pm.nx;
  // (not __restrict__ / no read-only path: the item may write the filter itself, below)
  float2* Gp = const_cast<float2*>(a.spec) + pl.spec_off;
  float* __restrict__ y = a.y + pl.y_off;
  const int L = static_cast<int>(pl.L);
  const int B = static_cast<int>(pl.B);
  const int ovl = C - L;  // N_h - 1 <= ccap
  const long long own_lo = static_cast<long long>(it.b_own) * L;
  const long long own_hi = it.b_end == B ? pl.out_len : static_cast<long long>(it.b_end) * L;
  for (int i = t; i < SH::TWN; i += T) {  // twiddle bases, FP64 sincospi rounded once
    int p = 0;
#pragma unroll
    for (int q = 1; q < PL::NP - 1; ++q)
      if (i >= SH::tw_off(q)) p = q;
    const int j = i - SH::tw_off(p);
    const int span = PL::radix(p) * SH::stride(p);
    double sn, cs;
    sincospi(-2.0 * j / span, &sn, &cs);
    tws[i] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
  for (int i = t; i < ovl; i += T) carry[i] = 0.f;
  if (t == 0) {  // the run's first two blocks (and the pair's filter when K3 wrote it)
    if (!a.rir) prefetch_l2(Gp, C * sizeof(float2));
    const long long s0 = static_cast<long long>(it.b_begin) * L;
    prefetch_l2(x + s0, 4 * (nx - s0 < 2 * L ? nx - s0 : 2 * L));
  }
  __syncthreads();
  if (a.rir) {
    // The filter, by the item itself (K3's work, convolution.hpp:238-239): the forward transform
    // of the truncated RIR (FP64 taps rounded to FP32, zero-padded to N, imaginary part 0) leaves
    // H(k) in the digit-reversed slots the product step reads, so after the last pass element r
    // of butterfly u IS Gp[r (C / RL) + u]: scaled by 1 / N and stored from registers, coalesced.
    // One forward transform per item (a whole pair's blocks in a batched render: ~3% of its work)
    // instead of a K3 launch that wrote the same 32 KB per pair through scattered smem reads.
    const double* __restrict__ h = a.rir + pm.rir_off;
    const int nh = ovl + 1;
    {
      float2 v[R0];
      const int rh = nh - t;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        v[r].x = S0 * r < rh ? static_cast<float>(h[t + S0 * r]) : 0.f;
        v[r].y = 0.f;
      }
      Dft<R0, false>::run(v);
      apply_twiddles<R0, false>(v, tws[t]);
#pragma unroll
      for (int r = 0; r < R0; ++r) s[ipad<PL>(t) + ip_off<PL, R0, S0, C>(r)] = v[r];
    }
    __syncthreads();
    ipc_forward_mid<PL, C, 1>(s, tws, t);
    const float inv_n = 1.0f / static_cast<float>(C);
#pragma unroll
    for (int q = 0; q < NBL; ++q) {
      const int u = t + q * T;
      const int pb = ipad<PL>(u * RL);
      float2 v[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) v[r] = s[pb + ip_off<PL, RL, 1, C>(r)];
      Dft<RL, false>::run(v);
#pragma unroll
      for (int r = 0; r < RL; ++r) Gp[r * (C / RL) + u] = c_scale(v[r], inv_n);
    }
    __syncthreads();  // the filter (global, this CTA's own writes) and the transform buffer are settled
  }
  double pw = 0.0;  // this lane's Σ y² of the current power segment
#pragma unroll 1
  for (int b = it.b_begin; b < it.b_end; b += 2) {  // b even: blocks b (real part) and b + 1 (imaginary)
    const long long start = static_cast<long long>(b) * L;
    const int take_a = static_cast<int>(nx - start < L ? nx - start : L);
    const bool has_b = b + 1 < it.b_end;  // false only past the pair's last block
    const long long rem_b = nx - start - L;
    const int take_b = has_b ? static_cast<int>(rem_b < 0 ? 0 : (rem_b < L ? rem_b : L)) : 0;
    const float* xa = x + start;
    const float* xb = xa + L;
    if (t == 0 && b + 2 < it.b_end) {  // the next two blocks land in L2 during this transform
      const long long s1 = start + 2 * static_cast<long long>(L);
      if (s1 < nx) prefetch_l2(x + s1, 4 * (nx - s1 < 2 * L ? nx - s1 : 2 * L));
    }
    {  // forward pass 0 (S_0 = T): z[t + S_0 r] = x_a + i x_b from the signal, zero past the blocks
      float2 v[R0];
      const int ra = take_a - t, rb = take_b - t;
#pragma unroll
      for (int r = 0; r < R0; ++r) {  // predicated loads: S_0 r < take - t
        v[r].x = S0 * r < ra ? __ldg(xa + t + S0 * r) : 0.f;
        v[r].y = S0 * r < rb ? __ldg(xb + t + S0 * r) : 0.f;
      }
      Dft<R0, false>::run(v);
      apply_twiddles<R0, false>(v, tws[t]);
#pragma unroll
      for (int r = 0; r < R0; ++r) s[ipad<PL>(t) + ip_off<PL, R0, S0, C>(r)] = v[r];
    }
    __syncthreads();
    ipc_forward_mid<PL, C, 1>(s, tws, t);
    // last forward pass, x H / N, first inverse pass: one butterfly's slots, in registers
#pragma unroll
    for (int q = 0; q < NBL; ++q) {
      const int u = t + q * T;
      const int pb = ipad<PL>(u * RL);
      float2 v[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) v[r] = s[pb + ip_off<PL, RL, 1, C>(r)];
      Dft<RL, false>::run(v);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
#if RSG_IPC_H_L1
        v[r] = c_mul(v[r], Gp[r * (C / RL) + u]);  // through L1: the CTA re-reads its pair's H every trip
#else
        v[r] = c_mul(v[r], __ldcg(Gp + r * (C / RL) + u));
#endif
      }
      Dft<RL, true>::run(v);
#pragma unroll
      for (int r = 0; r < RL; ++r) s[pb + ip_off<PL, RL, 1, C>(r)] = v[r];
    }
    __syncthreads();
    ipc_inverse_mid<PL, C, PL::NP - 2>(s, tws, t);
    // inverse pass 0: outputs e = t + S_0 r in registers (.x: block b, .y: block b + 1)
    float2 v[R0];
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = s[ipad<PL>(t) + ip_off<PL, R0, S0, C>(r)];
    apply_twiddles<R0, true>(v, tws[t]);
    Dft<R0, true>::run(v);
    // emit block b, then block b + 1 (its head overlaps block b's tail through the carry).  With two
    // carry buffers (DB; N = 4096: 14.9 vs 15.2 ms; N = 8192 measured 3% slower with them and keeps
    // one): block b reads buffer 0 (the previous transform's tail) and writes its tail to
    // buffer 1, block b + 1 reads buffer 1 and writes buffer 0 — every buffer is rewritten in full
    // (e - L covers [0, ovl)), reads and writes of one buffer are always a barrier apart, and the
    // emit needs one barrier instead of three.
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1) {
        if (!has_b) break;
        __syncthreads();  // block b's tail is in the carry; this transform's smem reads are done
      }
      const int bb = b + h;
      const long long st = start + static_cast<long long>(h) * L;
      const float* cin = carry + (DB ? h * ccap : 0);
      const int ovl_t = ovl - t;
#pragma unroll
      for (int r = 0; r < R0; ++r)
        if (S0 * r < ovl_t) (h ? v[r].y : v[r].x) += cin[t + S0 * r];
      if constexpr (!DB) __syncthreads();  // one buffer: its reads end before its writes begin
      const int lo = static_cast<int>(max(own_lo - st, -1ll));
      const int hi = static_cast<int>(min(own_hi - st, static_cast<long long>(C)));
      const int fe = bb == B - 1 ? C : L;  // e < fe: final after this block
      float* yb = y + st + t;
      float* cb = carry + (DB ? (1 - h) * ccap : 0) + t - L;
      float p0 = 0.f, p1 = 0.f;
      const int fe_t = fe - t, lo_t = lo - t, hi_t = hi - t;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const float val = h ? v[r].y : v[r].x;
        if (S0 * r < fe_t) {
          if (S0 * r >= lo_t && S0 * r < hi_t) {
            yb[S0 * r] = val;
            if (r & 1) p1 = fmaf(val, val, p1); else p0 = fmaf(val, val, p0);
          }
        } else {
          cb[S0 * r] = val;
        }
      }
      pw += static_cast<double>(p0 + p1);
      if (closes_segment(bb, it.b_end, a.seg)) {
        const long long part0 = __ldg(&a.plan[it.pair].part0);
        store_segment_power<T>(a.part + part0 + static_cast<long long>(bb / a.seg) * parts_per_block_of(T), pw, t,
                               bb >= it.b_own);
        pw = 0.0;
      }
    }
    // (the next transform's passes put barriers between these carry / smem accesses and its own)
  }
  // the channel's last work item mixes it (mixfin.cuh); the transform buffer is free by now
  finish_item<T, fin_un(T, PL::MINB)>(a.fin, it.pair, t, reinterpret_cast<unsigned char*>(smem));
}

template <int C>
size_t ipc_smem(int ccap) {
  using SH = IpShape<IpcPlan<C>, C>;
  return (static_cast<size_t>(SH::SLOTS) + ((SH::TWN + 1) & ~1)) * sizeof(float2) +
         (IpcPlan<C>::DB ? 2 : 1) * static_cast<size_t>(ccap) * sizeof(float);  // carry buffer(s)
}

template <int C>
cudaError_t ipc_t(const OlaArgs& a, int ccap, cudaStream_t st) {
  const size_t smem = ipc_smem<C>(ccap);
  cudaError_t e = ensure_dynamic_smem(ola_ipc_kernel<C>, smem);
  if (e != cudaSuccess) return e;
  ola_ipc_kernel<C><<<a.count, IpcPlan<C>::T, smem, st>>>(a, ccap);
  return cudaGetLastError();
}

}  // namespace

#define RSG_IP_DISPATCH(L, CALL)                     \
  switch (L) {                                       \
    case 9: { constexpr int M = 512; return CALL; }    \
    case 10: { constexpr int M = 1024; return CALL; }  \
    case 11: { constexpr int M = 2048; return CALL; }  \
    case 12: { constexpr int M = 4096; return CALL; }  \
    case 13: { constexpr int M = 8192; return CALL; }  \
    case 14: { constexpr int M = 16384; return CALL; } \
  }

namespace {
int ccap_of(int64_t max_nh) { return static_cast<int>((std::max<int64_t>(max_nh - 1, 1) + 3) & ~int64_t(3)); }
size_t ip_smem_of(int log2m, int ccap) {
  RSG_IP_DISPATCH(log2m, ip_smem<M>(ccap))
  return 0;
}
int ip_threads_of(int log2m) {
  RSG_IP_DISPATCH(log2m, IpPlan<M>::T)
  return 0;
}
int ip_minb_of(int log2m) {  // CTAs per SM the register budget is set for
  RSG_IP_DISPATCH(log2m, IpPlan<M>::MINB)
  return 1;
}
}  // namespace

// Sizes (log2 M) with an in-place K4 and the largest N_h - 1 its carry can hold.
bool ip_supported(int log2m, int64_t max_nh) {
  if (ip_threads_of(log2m) == 0) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return ip_smem_of(log2m, ccap_of(max_nh)) + 1024 <= static_cast<size_t>(optin);
}

int ip_resident(int log2m, int64_t max_nh) {
  const size_t need = ip_smem_of(log2m, ccap_of(max_nh)) + 1024;
  const int by_smem = static_cast<int>((228 * 1024) / need);
  const int by_threads = 2048 / ip_threads_of(log2m);
  return std::max(1, std::min(std::min(by_smem, by_threads), ip_minb_of(log2m)));
}

int ip_parts_per_block(int log2m) {
  RSG_IP_DISPATCH(log2m, parts_per_block_of(IpPlan<M>::T))
  return 0;
}

cudaError_t launch_ola_ip(int log2m, const OlaArgs& a, int64_t max_nh, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  RSG_IP_DISPATCH(log2m, ip_t<M>(a, ccap_of(max_nh), s))
  return cudaErrorInvalidValue;
}


// ---- two blocks per transform (ola_ipc_kernel<C>, C = N) --------------------------------
#define RSG_IPC_DISPATCH(LN, CALL)                   \
  switch (LN) {                                      \
    case 12: { constexpr int C = 4096; return CALL; } \
    case 13: { constexpr int C = 8192; return CALL; } \
  }
namespace {
size_t ipc_smem_of(int log2n, int ccap) {
  RSG_IPC_DISPATCH(log2n, ipc_smem<C>(ccap))
  return 0;
}
int ipc_minb_of(int log2n) {
  RSG_IPC_DISPATCH(log2n, IpcPlan<C>::MINB)
  return 1;
}
int ipc_threads_of(int log2n) {
  RSG_IPC_DISPATCH(log2n, IpcPlan<C>::T)
  return 0;
}
template <int C>
IpcPerm ipc_perm_t() {
  using PL = IpcPlan<C>;
  auto lg = [](int v) { int l = 0; while ((1 << l) < v) ++l; return l; };
  return IpcPerm{1, lg(PL::radix(0)), lg(PL::radix(1)), lg(PL::radix(2)), lg(C)};
}
}  // namespace

bool ipc_supported(int log2n, int64_t max_nh) {
  if (ipc_threads_of(log2n) == 0) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return ipc_smem_of(log2n, ccap_of(max_nh)) + 1024 <= static_cast<size_t>(optin);
}
int ipc_resident(int log2n, int64_t max_nh) {
  const size_t need = ipc_smem_of(log2n, ccap_of(max_nh)) + 1024;
  const int by_smem = static_cast<int>((228 * 1024) / need);
  const int by_threads = 2048 / ipc_threads_of(log2n);
  return std::max(1, std::min(std::min(by_smem, by_threads), ipc_minb_of(log2n)));
}
int ipc_parts_per_block(int log2n) {
  RSG_IPC_DISPATCH(log2n, parts_per_block_of(IpcPlan<C>::T))
  return 0;
}
IpcPerm ipc_perm(int log2n) {
  RSG_IPC_DISPATCH(log2n, ipc_perm_t<C>())
  return IpcPerm{};
}
cudaError_t launch_ola_ipc(int log2n, const OlaArgs& a, int64_t max_nh, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  RSG_IPC_DISPATCH(log2n, ipc_t<C>(a, ccap_of(max_nh), s))
  return cudaErrorInvalidValue;
}

}  // namespace rsg

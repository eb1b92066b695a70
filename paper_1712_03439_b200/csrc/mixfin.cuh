// mixfin.cuh — the SNR-scaled mix as device functions shared by K5 / K6
// (kernels.cu) and the K4 epilogue (big.cu): "the last K4 work item of an output channel
// mixes it".
//
// A channel (utterance u, mic j) is the sum over the utterance's sources i of alpha_ij y_ij.
// alpha_ij needs the mean power of the WHOLE y_ij and of the target's y_0j (SPEC.md:341,
// :365), so no sample of the channel can be mixed before every K4 work item of its I pairs
// has finished.  K4 is FP32-bound and leaves most of the HBM bandwidth idle; a separate mix
// kernel afterwards is HBM-bound and leaves the FP32 pipe idle.  So every work item, after
// its last block, makes its stores visible (__threadfence) and decrements its channel's
// counter; the item that brings it to zero computes the channel's powers and gains and mixes
// the channel — inside the K4 launch, on an SM whose other resident CTAs keep transforming.
// The arithmetic is the same code K5 / K6 run (pair_power_warp, pair_gain, MixQuadAcc), so the
// bytes do not depend on which item finished last, nor on whether a channel was mixed here or
// by mix_kernel (render invariance).
#pragma once
#include "kernels.cuh"

namespace rsg {

constexpr int kMixMaxI = 8;  // sources whose metadata is cached per CTA (more: read per use)

// mean_power (audio_buffer.hpp:66-75) of a pair from its K4 partials (power.cuh): lane l sums
// partials l, l + 32, ... then a fixed butterfly — one order per pair.  All 32 lanes call it.
template <bool CG>
__device__ __forceinline__ double pair_power_warp(const double* part, int npart, long long out_len, int lane) {
  double s = 0.0;
  for (int k = lane; k < npart; k += 32) s += CG ? __ldcg(part + k) : part[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s / static_cast<double>(out_len);
}

// alpha_ij = sqrt(P_0j / (P_ij 10^(snr_i/10))), alpha_0j = 1.
// *degenerate: a power that is not positive (the render fails with DegenerateInput).
__device__ __forceinline__ double pair_gain(bool target, double P, double Pt, double snr_lin, bool* degenerate) {
  if (target) {
    *degenerate = !(P > 0.0);
    return 1.0;
  }
  if (!(P > 0.0) || !(Pt > 0.0)) {
    *degenerate = true;
    return 0.0;
  }
  *degenerate = false;
  return sqrt(Pt / (P * snr_lin));
}

// One source row's quad at n (zero past the row's end).  CG: L2-coherent loads (rows written
// by other SMs during this launch); else streaming loads.
template <bool CG>
__device__ __forceinline__ float4 mix_quad(const float* row, long long ol, long long n) {
  if (n + 3 < ol) {
    const float4* q = reinterpret_cast<const float4*>(row + n);
    return CG ? __ldcg(q) : __ldcs(q);
  }
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (CG) {
    if (n < ol) v.x = __ldcg(row + n);
    if (n + 1 < ol) v.y = __ldcg(row + n + 1);
    if (n + 2 < ol) v.z = __ldcg(row + n + 2);
  } else {
    if (n < ol) v.x = row[n];
    if (n + 1 < ol) v.y = row[n + 1];
    if (n + 2 < ol) v.z = row[n + 2];
  }
  return v;
}

// A quad's running sums, in source order (SPEC.md:351 fixes the order, not the width).  FP32 FMAs
// with the gain rounded to FP32: at most one rounding of 2^-24 of the partial sum per source —
// < 4e-7 of the peak for 6 sources, against the 1e-5 bar.  (FP64 sums cost a conversion and a
// DFMA per sample and source; the FP64 pipe issues a warp instruction every ~4 cycles per SM,
// which bound mix_kernel — not HBM — and made a one-CTA channel mix 3x slower than its loads.)
#ifndef RSG_FIN_AHEAD
#define RSG_FIN_AHEAD 2  // 32-KB tiles of every row the K4 epilogue's mix keeps ahead in L2
#endif
#ifndef RSG_MIX_FP64
#define RSG_MIX_FP64 0
#endif
#if RSG_MIX_FP64
using mix_gain_t = double;
struct MixQuadAcc {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  __device__ __forceinline__ void add(double g, float4 v) {
    a0 = fma(g, static_cast<double>(v.x), a0);
    a1 = fma(g, static_cast<double>(v.y), a1);
    a2 = fma(g, static_cast<double>(v.z), a2);
    a3 = fma(g, static_cast<double>(v.w), a3);
  }
};
#else
using mix_gain_t = float;
struct MixQuadAcc {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  __device__ __forceinline__ void add(float g, float4 v) {
    a0 = __fmaf_rn(g, v.x, a0);
    a1 = __fmaf_rn(g, v.y, a1);
    a2 = __fmaf_rn(g, v.z, a2);
    a3 = __fmaf_rn(g, v.w, a3);
  }
};
#endif

// out[n] for n in [n, n + 4) ∩ [.., n1): the sums in source order; samples in [len, stride) are
// the zero-filled tail.
__device__ __forceinline__ void mix_store(float* out, bool out16, long long n, long long n1, long long len,
                                          const MixQuadAcc& c) {
  const float4 o = make_float4(static_cast<float>(c.a0), n + 1 < len ? static_cast<float>(c.a1) : 0.f,
                               n + 2 < len ? static_cast<float>(c.a2) : 0.f,
                               n + 3 < len ? static_cast<float>(c.a3) : 0.f);
  if (out16 && n + 3 < n1) {
    __stcs(reinterpret_cast<float4*>(out + n), o);
  } else {
    out[n] = o.x;
    if (n + 1 < n1) out[n + 1] = o.y;
    if (n + 2 < n1) out[n + 2] = o.z;
    if (n + 3 < n1) out[n + 3] = o.w;
  }
}

// The channel's metadata, in shared memory.
struct MixChan {
  const float* row[kMixMaxI];
  long long len[kMixMaxI];
  double gain[kMixMaxI];
};

// The K4 epilogue's state in device memory (OlaArgs::fin; null: every channel is mixed by
// mix_kernel).
struct MixFin {
  int32_t* left;             // per channel of the chunk: K4 work items still running
  const int32_t* pair_chan;  // per pair: its channel, or -1 (the channel is mixed by mix_kernel)
  const double* snr_lin;     // per global source, as GainArgs::snr_lin
  const double* part;        // K4 power partials
  const PairMeta* pair;
  MixArgs mix;               // chan_* arrays over ALL channels of the chunk
};

// [p, p + bytes) into L2 (asynchronous; the range is widened to 16-byte alignment).
__device__ __forceinline__ void mix_prefetch_l2(const void* p, long long bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(bytes) + 15) & ~uintptr_t(15);
  if (a1 > a0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(static_cast<unsigned>(a1 - a0)) : "memory");
}

// Trips [0, trips) of a channel with exactly NI sources: trip `it` covers samples
// [it UN 4T, (it + 1) UN 4T), UN quads per thread, all NI x UN loads in flight before the sums.
// Rows are addressed as 32-bit quad indices from `ybase` (one IMAD.WIDE per load, half the
// registers of pointers); nothing in the loop but the loads, the FMAs and the stores — the CTA
// shares its SM with K4 CTAs that want every issue slot.
template <bool CG, int T, int NI, int UN>
__device__ __forceinline__ void mix_trips(const MixChan& mc, const float* ybase, float* out, bool out16, int trips,
                                          int tid) {
  constexpr int QT = 8 / UN;  // trips per prefetch tile (8 x 4T samples)
  unsigned ri[NI];            // row i's quad index of this thread's first quad
  mix_gain_t g[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    ri[i] = static_cast<unsigned>((mc.row[i] - ybase) >> 2) + tid;
    g[i] = static_cast<mix_gain_t>(mc.gain[i]);
  }
  const float4* yq = reinterpret_cast<const float4*>(ybase);
  float4* op = reinterpret_cast<float4*>(out) + tid;
  auto prefetch_tile = [&](int k) {  // samples [k 32T, (k + 1) 32T) of row tid
    if (tid < NI) {
      const long long lo = k * (32ll * T), ol = mc.len[tid];
      if (lo < ol) mix_prefetch_l2(mc.row[tid] + lo, 4 * (ol - lo < 32ll * T ? ol - lo : 32ll * T));
    }
  };
#pragma unroll
  for (int k = 0; k < RSG_FIN_AHEAD; ++k) prefetch_tile(k);
#pragma unroll 1
  for (int it = 0; it < trips; ++it) {
    if ((it & (QT - 1)) == 0) prefetch_tile(it / QT + RSG_FIN_AHEAD);
    const unsigned base = static_cast<unsigned>(it) * (UN * T);
    float4 v[UN][NI];
#pragma unroll
    for (int q = 0; q < UN; ++q)
#pragma unroll
      for (int i = 0; i < NI; ++i)
        v[q][i] = CG ? __ldcg(yq + (ri[i] + base + q * T)) : __ldcs(yq + (ri[i] + base + q * T));
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      MixQuadAcc acc;
#pragma unroll
      for (int i = 0; i < NI; ++i) acc.add(g[i], v[q][i]);
      const float4 o = make_float4(static_cast<float>(acc.a0), static_cast<float>(acc.a1),
                                   static_cast<float>(acc.a2), static_cast<float>(acc.a3));
      if (out16) {
        __stcs(op + (base + q * T), o);
      } else {  // a channel that does not start on a 16-byte boundary
        float* os = out + 4ll * (base + q * T + tid);
        os[0] = o.x;
        os[1] = o.y;
        os[2] = o.z;
        os[3] = o.w;
      }
    }
  }
}

// One whole channel, samples [0, stride), by the T threads of a CTA.  Trips whose quads lie
// inside every row take mix_trips; the channel's tail takes the checked path.  Sums in source
// order, as mix_kernel.  `ybase`: a 16-byte aligned address at or below every row, within 64 GB.
template <bool CG, int T, int UN>
__device__ __forceinline__ void mix_channel(const MixChan& mc, int I, const float* ybase, float* out, long long len,
                                            long long stride, int tid) {
  constexpr long long TRIP = 4ll * T * UN;  // samples per trip
  const bool out16 = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  const int Ic = I < kMixMaxI ? I : kMixMaxI;
  long long full = len < stride ? len : stride;  // samples inside every row
  for (int i = 0; i < Ic; ++i) full = mc.len[i] < full ? mc.len[i] : full;
  const int trips = static_cast<int>(full / TRIP);
  switch (Ic) {
    case 1: mix_trips<CG, T, 1, UN>(mc, ybase, out, out16, trips, tid); break;
    case 2: mix_trips<CG, T, 2, UN>(mc, ybase, out, out16, trips, tid); break;
    case 3: mix_trips<CG, T, 3, UN>(mc, ybase, out, out16, trips, tid); break;
    case 4: mix_trips<CG, T, 4, UN>(mc, ybase, out, out16, trips, tid); break;
    case 5: mix_trips<CG, T, 5, UN>(mc, ybase, out, out16, trips, tid); break;
    case 6: mix_trips<CG, T, 6, UN>(mc, ybase, out, out16, trips, tid); break;
    case 7: mix_trips<CG, T, 7, UN>(mc, ybase, out, out16, trips, tid); break;
    default: mix_trips<CG, T, 8, UN>(mc, ybase, out, out16, trips, tid); break;
  }
  for (long long n = trips * TRIP + 4ll * tid; n < stride; n += 4ll * T) {  // the tail, checked
    MixQuadAcc acc;
    if (n < len) {
#pragma unroll 1
      for (int i = 0; i < Ic; ++i) acc.add(static_cast<mix_gain_t>(mc.gain[i]), mix_quad<CG>(mc.row[i], mc.len[i], n));
    }
    mix_store(out, out16, n, stride, len, acc);
  }
}

// The channel `ch` by the T threads of the CTA whose work item finished it last.  Not inlined:
// its registers are allocated apart from the K4 block loop's.  `smem`: the CTA's dynamic shared
// memory (free after the block loop).
template <int T, int UN>
__device__ __noinline__ void mix_finished_channel(const MixFin* __restrict__ finp, int ch, int t,
                                                  unsigned char* smem) {
  MixChan* mc = reinterpret_cast<MixChan*>(smem);
  const MixFin& f = *finp;
  const MixArgs& a = f.mix;
  const long long u = a.chan_utt[ch];
  const int j = a.chan_mic[ch];
  const int I = a.utt_I[u], J = a.utt_J[u];  // I <= kMixMaxI (the host fuses no wider channel)
  const long long pair0 = a.utt_pair0[u];
  {  // powers: a warp per source, the order of power_kernel
    const int w = t >> 5, lane = t & 31;
    for (int i = w; i < I; i += T / 32) {
      const long long p = pair0 + static_cast<long long>(i) * J + j;
      const PairPlan& pl = a.plan[p];
      const double P = pair_power_warp<true>(f.part + pl.part0, pl.npart, pl.out_len, lane);
      if (lane == 0) {
        mc->gain[i] = P;
        mc->row[i] = a.y + pl.y_off;
        mc->len[i] = pl.out_len;
      }
    }
  }
  __syncthreads();
  double g = 0.0;
  if (t < I) {  // gains: gain_kernel's arithmetic
    const long long p = pair0 + static_cast<long long>(t) * J + j;
    bool deg;
    g = pair_gain(t == 0, mc->gain[t], mc->gain[0], f.snr_lin[f.pair[p].src_idx], &deg);
  }
  __syncthreads();
  if (t < I) mc->gain[t] = g;
  __syncthreads();
  mix_channel<true, T, UN>(*mc, I, a.y, a.out + a.chan_out[ch], a.utt_len[u], a.utt_stride[u], t);
}

// K4 epilogue, called by all T threads of a work item's CTA after its last store.
// `smem`: the CTA's dynamic shared memory, 128-byte aligned (free after the block loop).
template <int T, int UN>
__device__ __forceinline__ void finish_item(const MixFin* __restrict__ finp, int pair, int t, unsigned char* smem) {
  if (!finp) return;  // uniform over the launch
  int* flag = reinterpret_cast<int*>(smem + sizeof(MixChan));
  __threadfence();    // this thread's y and power-partial stores, device-wide
  __syncthreads();
  if (t == 0) {
    const int ch = __ldg(finp->pair_chan + pair);
    int last = -1;
    if (ch >= 0 && atomicSub(finp->left + ch, 1) == 1) {
      last = ch;
      __threadfence();  // the other items' stores, seen before the reads below
    }
    *flag = last;
  }
  __syncthreads();
  const int ch = *flag;
  if (ch >= 0) mix_finished_channel<T, UN>(finp, ch, t, smem);  // uniform over the CTA
}

}  // namespace rsg

// warp.cu — K4 two-stream, warp-per-transform variant for N = 512 and 1024.
//
// Reference: convolve_ola (convolution.hpp:219-255) with RadixTwoRealFft
// (fft.hpp:57-169); mean_power's Σy² (audio_buffer.hpp:66-75).
//
// As in ola2.cu, two OLA runs of one pair share each complex N-point transform
// (z = x_a + i x_b; h is real, so IFFT(FFT(z) H) = (x_a * h) + i (x_b * h)).  Here
// the transform is N = 32 T points held by T = N/32 lanes (half a warp or one
// warp), 32 complex values per lane, in three in-place steps with only
// __syncwarp between them:
//   A  forward DIF pass, radix 32, stride T: lane j loads z[j + T r] straight from
//      the two signal windows (coalesced), DFT32, twiddles W_N^(j r), writes its
//      32 slots back;
//   F  fused: radix-T butterflies over 32 contiguous slots (the forward DIF pass
//      with stride 1, whose output sits at slot T m0 + m1 for frequency
//      k = m0 + 32 m1), times H[k], the inverse DIT pass with stride 1, in
//      registers, written back in place;
//   E  inverse DIT pass, radix 32, stride T: conj twiddles, inverse DFT32; lane j
//      holds output samples j + T r of both runs -> overlap carry (smem, one buffer
//      per run: all reads, __syncwarp, all writes), owned outputs, power.
// Per real block that is two shared-memory round trips of the transform (K4 needs
// seven) and no CTA barrier; lanes of different transforms never wait on each
// other.  Slot of element i: i + i/T (stride-T and stride-1 accesses both
// conflict-free on 64-bit accesses).
#include <cmath>

#include "fft.cuh"
#include "kernels.cuh"

namespace rsg {
namespace {

template <int N>
struct WPlan {
  static constexpr int T = N / 32;          // lanes per transform (16 or 32)
  static constexpr int LT = ilog2(T);
  static constexpr int R1 = T;              // radix of the fused pass
  static constexpr int NB1 = 32 / T;        // fused butterflies per lane (32 in all)
  static constexpr int G = 128 / T;         // transforms per 128-thread CTA
  static constexpr int SLOTS = N + N / T;   // float2 slots of one transform
  // 128-thread CTAs per SM: 16 warps at N = 512; 12 at N = 1024, whose 168 registers
  // keep the 32-point passes out of local memory
  static constexpr int MINB = N == 512 ? 4 : 3;
  static_assert(T == 16 || T == 32, "N = 512 or 1024");
};

template <int N>
__device__ __forceinline__ int wpad(int i) { return i + (i >> WPlan<N>::LT); }

__device__ __forceinline__ void prefetch_l2w(const void* p, long long bytes) {
  if (bytes <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(bytes) + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(static_cast<unsigned>(a1 - a0)) : "memory");
}

// smem per group: the transform, the two runs' carries (ccap floats each), then the
// block parameters of both runs (WPAR ints; kept in smem, not registers, so the
// 32-point passes have the register file to themselves)
constexpr int WPAR = 12;
template <int N>
__host__ __device__ constexpr int w_hs_floats() { return 2 * ((N / 2 + 1 + 1) & ~1); }  // H / N, k <= N/2
template <int N>
__host__ __device__ constexpr int w_group_floats(int ccap) {
  return 2 * WPlan<N>::SLOTS + w_hs_floats<N>() + 2 * ccap + WPAR;
}

template <int N>
__global__ void __launch_bounds__(128, WPlan<N>::MINB) ola_w_kernel(Ola2Args a) {
  using PL = WPlan<N>;
  constexpr int T = PL::T, R1 = PL::R1;
  extern __shared__ __align__(16) float2 smem[];
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int item = blockIdx.x * PL::G + g;
  const bool has = item < a.count;
  const OlaItem2 it = a.items[has ? item : 0];
  const PairPlan& pl = a.plan[it.pair];
  const PairMeta& pm = a.pair[it.pair];
  const float* __restrict__ x = a.signals + pm.sig_off;
  const long long nx = pm.nx;
  const float2* __restrict__ G = a.spec + pl.spec_off;  // H / (2N), k in [0, N/2]
  float* __restrict__ y = a.y + pl.y_off;
  const int L = static_cast<int>(pl.L);
  const int B = static_cast<int>(pl.B);
  const int ovl = N - L;  // N_h - 1 <= ccap
  const int ccap = a.ccap;
  float2* s = smem + g * (w_group_floats<N>(ccap) / 2);
  float2* hs = s + PL::SLOTS;  // the pair's H / N, staged once per item
  float* carry0 = reinterpret_cast<float*>(hs + w_hs_floats<N>() / 2);
  // twiddle base of lane t for passes A / E: exp(-2 pi i t / N)
  float2 w;
  {
    double sn, cs;
    sincospi(-2.0 * t / N, &sn, &cs);
    w = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
  const int rb[2] = {it.a_begin, it.b_begin}, ro[2] = {it.a_own, it.b_own}, re[2] = {it.a_end, it.b_end};
  int trips = has ? max(re[0] - rb[0], re[1] - rb[1]) : 0;
  trips = __reduce_max_sync(0xffffffffu, trips);
  if (has) {
    for (int i = t; i < 2 * ccap; i += T) carry0[i] = 0.f;
    for (int i = t; i <= N / 2; i += T) hs[i] = c_scale(__ldg(G + i), 2.0f);  // H / N (exact x2)
  }
  if (has && t == 0)
    for (int r = 0; r < 2; ++r)
      if (rb[r] < re[r]) {
        const long long s0 = static_cast<long long>(rb[r]) * L;
        prefetch_l2w(x + s0, 4 * (nx - s0 < L ? nx - s0 : L));
      }
  __syncwarp();
  int* par = reinterpret_cast<int*>(carry0 + 2 * ccap);  // [start, take, lo, hi, fe] x 2
  double pw = 0.0;
#pragma unroll 1
  for (int k = 0; k < trips; ++k) {
    if (t < 2) {
      const int r = t;
      const int b = rb[r] + k;
      const bool act = has && b < re[r];
      const int start = act ? b * L : 0;
      const int own_lo = ro[r] * L;
      const long long own_hi = re[r] == B ? pl.out_len : static_cast<long long>(re[r]) * L;
      par[5 * r + 0] = start;
      par[5 * r + 1] = act ? static_cast<int>(nx - start < L ? nx - start : L) : 0;
      par[5 * r + 2] = act ? own_lo - start : N;  // inactive run: owns nothing, carries nothing
      par[5 * r + 3] = act ? static_cast<int>(min(own_hi - start, static_cast<long long>(N))) : N;
      par[5 * r + 4] = !act || b == B - 1 ? N : L;
      if (act && b + 1 < re[r]) {
        const long long s1 = static_cast<long long>(start) + L;
        prefetch_l2w(x + s1, 4 * (nx - s1 < L ? nx - s1 : L));
      }
    }
    __syncwarp();
    // ---- A: forward DIF pass, radix 32, stride T ----
    {
      const float* xa = x + par[0];
      const float* xb = x + par[5];
      const int ta = par[1], tb = par[6];
      float2 v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int n = t + T * r;
        v[r].x = n < ta ? __ldg(xa + n) : 0.f;
        v[r].y = n < tb ? __ldg(xb + n) : 0.f;
      }
      Dft<32, false>::run(v);
      apply_twiddles<32, false>(v, w);
#pragma unroll
      for (int r = 0; r < 32; ++r) s[t + (T + 1) * r] = v[r];  // wpad(t + T r)
    }
    __syncwarp();
    // ---- F: forward DIF stride-1 pass x H, inverse DIT stride-1 pass ----
#pragma unroll
    for (int q = 0; q < PL::NB1; ++q) {
      const int b = t + T * q;  // butterfly (= m0): slots R1 b + m1, frequency b + 32 m1
      const float2* Gb = hs + b;
      const float2* Gm = hs + (N - b);
      float2 v[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) v[r] = s[(R1 + 1) * b + r];
      Dft<R1, false>::run(v);
      asm volatile("" ::: "memory");  // keep the H loads below the DFT (registers)
#pragma unroll
      for (int r = 0; r < R1; ++r) {
        // frequency k = b + 32 r; H[k] = conj(H[N - k]) above N/2 (h real).  k <= N/2
        // exactly for r < R1/2 (and r = R1/2, b = 0, the real Nyquist bin, where the
        // conj below is exact), so each half is one base pointer plus constant offsets.
        const float2 h = r < R1 / 2 ? Gb[32 * r] : c_conj(Gm[-32 * r]);
        v[r] = c_mul(v[r], h);
      }
      Dft<R1, true>::run(v);
#pragma unroll
      for (int r = 0; r < R1; ++r) s[(R1 + 1) * b + r] = v[r];
    }
    __syncwarp();
    // ---- E: inverse DIT pass, radix 32, stride T, back in place ----
    {
      float2 v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = s[t + (T + 1) * r];
      apply_twiddles<32, true>(v, w);
      Dft<32, true>::run(v);
#pragma unroll
      for (int r = 0; r < 32; ++r) s[t + (T + 1) * r] = v[r];
    }
    __syncwarp();
    // ---- overlap-add and emit from smem (compact loop: small code, few registers) ----
    // samples n = t + T r, r = 0..31; the group's T samples of one r are contiguous,
    // so the classification below is uniform over the group except where a range
    // straddles ovl, L, lo or hi.  All carry reads precede all carry writes.
    // carry add, in place in the transform slots (slot of sample n = t + T r: n + r);
    // r < rc covers every sample below ovl
    const int rc = min(32, (ovl + T - 1) / T);
#pragma unroll 4
    for (int r = 0; r < rc; ++r) {
      const int n = t + T * r;
      if (n < ovl) {
        float2 z = s[n + r];
        z.x += carry0[n];
        z.y += carry0[ccap + n];
        s[n + r] = z;
      }
    }
    __syncwarp();  // all carry reads are done
    float pb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* sq = reinterpret_cast<const float*>(s) + q;
      float* yq = y + par[5 * q];
      const int lo = par[5 * q + 2], hi = par[5 * q + 3], fe = par[5 * q + 4];
      float* cq = carry0 + q * ccap - L;
      // the group's samples of r are [T r, T r + T): r in [ra, rb) are all final and
      // owned, r >= rcar all carried; the few r in between take the per-sample path
      const int ra = min(32, max(0, (lo + T - 1) / T));
      const int rb = max(ra, min(fe, hi) / T);
      const int rcar = min(32, max(rb, (fe + T - 1) / T));
      auto general = [&](int r) {
        const int n = t + T * r;
        const float val = sq[2 * (n + r)];
        if (n < fe) {
          if (n >= lo && n < hi) {
            yq[n] = val;
            pb[2 * q] = fmaf(val, val, pb[2 * q]);
          }
        } else {
          cq[n] = val;
        }
      };
#pragma unroll 1
      for (int r = 0; r < ra; ++r) general(r);
#pragma unroll 4
      for (int r = ra; r < rb; ++r) {
        const int n = t + T * r;
        const float val = sq[2 * (n + r)];
        yq[n] = val;
        pb[2 * q + (r & 1)] = fmaf(val, val, pb[2 * q + (r & 1)]);
      }
#pragma unroll 1
      for (int r = rb; r < rcar; ++r) general(r);
#pragma unroll 4
      for (int r = rcar; r < 32; ++r) {
        const int n = t + T * r;
        cq[n] = sq[2 * (n + r)];
      }
    }
    pw += static_cast<double>((pb[0] + pb[1]) + (pb[2] + pb[3]));
    __syncwarp();  // carry writes visible before the next block's reads; smem reuse
  }
  // Σ y² of both runs' owned samples (fixed order) -> part[item]
  for (int o = T / 2; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
  if (t == 0 && has) a.part[item] = pw;
}

template <int N>
size_t w_smem(int ccap) {
  return static_cast<size_t>(WPlan<N>::G) * w_group_floats<N>(ccap) * sizeof(float);
}

template <int N>
cudaError_t w_t(const Ola2Args& a, cudaStream_t st) {
  const size_t smem = w_smem<N>(a.ccap);
  cudaError_t e = cudaFuncSetAttribute(ola_w_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ola_w_kernel<N>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  ola_w_kernel<N><<<(a.count + WPlan<N>::G - 1) / WPlan<N>::G, 128, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool w_supported(int log2n, int64_t max_nh) {
  if (log2n != 9 && log2n != 10) return false;
  const int ccap = static_cast<int>((std::max<int64_t>(max_nh - 1, 1) + 3) & ~int64_t(3));
  return (log2n == 9 ? w_smem<512>(ccap) : w_smem<1024>(ccap)) <= 227 * 1024;
}

int w_resident_items(int log2n, int64_t max_nh) {
  const int ccap = static_cast<int>((std::max<int64_t>(max_nh - 1, 1) + 3) & ~int64_t(3));
  const size_t cta = (log2n == 9 ? w_smem<512>(ccap) : w_smem<1024>(ccap)) + 1024;
  const int minb = log2n == 9 ? WPlan<512>::MINB : WPlan<1024>::MINB;
  const int ctas = std::max(1, std::min(minb, static_cast<int>((228 * 1024) / cta)));
  return ctas * (log2n == 9 ? WPlan<512>::G : WPlan<1024>::G);
}

cudaError_t launch_ola_w(int log2n, const Ola2Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  switch (log2n) {
    case 9: return w_t<512>(a, s);
    case 10: return w_t<1024>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsg

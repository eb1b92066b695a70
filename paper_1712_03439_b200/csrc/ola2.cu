// ola2.cu — K4 two-stream variant: two OLA runs of one pair share each complex
// N-point transform (N = the real FFT size of the plan).  Run A rides in the real
// part, run B in the imaginary part; the RIR is real, so one forward transform,
// one multiply by H and one inverse transform filter one block of each run
// (convolution.hpp:242-253: same blocks, same per-block arithmetic as K4 up to
// FP32 rounding).  Versus K4 (half-size real transforms with the untangle/repack
// pass, ola_small_kernel) per block: no pairing pass, the last forward pass, the
// multiply and the first inverse pass run in registers (fft2.cuh fused_mid), and
// the input is read stride-1 from the TMA stage.
//
// Each run keeps its own overlap carry and writes only the outputs it owns, so
// the result is the same deterministic, seam-free OLA as K4.
#include <cmath>

#include "async.cuh"
#include "fft2.cuh"
#include "kernels.cuh"
#include "power.cuh"

namespace rsg {
namespace {

template <int T>
struct Bar2 {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (T == 1) {
    } else if constexpr (T <= 32) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
    }
  }
};

// elements per thread by size (measured): 8 up to N = 64 (registers), 16 above
__host__ __device__ constexpr int ola2_e_of(int log2n) { return log2n <= 6 ? 8 : 16; }
template <int N>
using PlanF = PlanC<N, false, ola2_e_of(ilog2(N))>;
template <int N>
using PlanI = PlanC<N, true, ola2_e_of(ilog2(N))>;
__host__ __device__ constexpr int ola2_t_of(int log2n) {  // threads per transform (PlanC::T)
  return (1 << log2n) / ((1 << log2n) < ola2_e_of(log2n) ? (1 << log2n) : ola2_e_of(log2n));
}
__host__ __device__ constexpr int ola2_cta(int log2n) {  // one group per CTA from 32 threads up, groups of a warp below
  return ola2_t_of(log2n) >= 32 ? ola2_t_of(log2n) : 32;
}
#ifndef RSG_OLA2_WARPS
#define RSG_OLA2_WARPS 8
#endif
__host__ __device__ constexpr int ola2_warps(int log2n) {  // resident-warp target per SM
  return log2n <= 8 ? 16 : RSG_OLA2_WARPS;
}
__host__ __device__ constexpr int ola2_minb(int log2n) {
  return ola2_warps(log2n) / (ola2_cta(log2n) / 32) > 0 ? ola2_warps(log2n) / (ola2_cta(log2n) / 32) : 1;
}

// One group's shared-memory region, in float2 (all offsets even: 16-byte aligned).
// The overlap carries and input windows are sized for the launch's largest N_h and
// L (Ola2Args::ccap / scap, floats, multiples of 4), not for the worst case N.
struct Layout2 {
  int hs, carry, stage, mbar, total;
  __host__ __device__ static constexpr int ev(int v) { return (v + 1) & ~1; }
  __host__ __device__ Layout2(int padded, int n, int ccap, int scap) {
    hs = ev(padded);
    carry = ev(hs + n / 2 + 1);    // [stream][buffer] carries of ccap floats
    stage = carry + 2 * ccap;      // [stream] input windows of scap floats
    mbar = stage + scap;           // one mbarrier per stream
    total = ev(mbar + 2);
  }
};

template <int N>
__global__ void __launch_bounds__(ola2_cta(ilog2(N)), ola2_minb(ilog2(N))) ola2_kernel(Ola2Args a) {
  using PF = PlanF<N>;
  using PI = PlanI<N>;
  extern __shared__ __align__(16) float2 smem[];
  constexpr int T = PF::T;
  constexpr int CTA = ola2_cta(ilog2(N));
  constexpr int G = CTA / T;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int item = blockIdx.x * G + g;
  const bool has = item < a.count;
  const OlaItem2 it = a.items[has ? item : 0];
  const PairPlan& pl = a.plan[it.pair];
  const PairMeta& pm = a.pair[it.pair];
  const float* __restrict__ x = a.signals + pm.sig_off;
  const int nx = static_cast<int>(pm.nx);
  float* __restrict__ y = a.y + pl.y_off;
  const int L = static_cast<int>(pl.L);
  const int B = static_cast<int>(pl.B);
  const int out_len = static_cast<int>(pl.out_len);
  constexpr int TWF = (PF::TW_PASS + 1) & ~1, TWI = (PI::TW_PASS + 1) & ~1;
  float2* twf = smem;
  float2* twi = smem + TWF;
  const Layout2 ly(PF::PADDED, N, a.ccap, a.scap);
  float2* base = smem + TWF + TWI + g * ly.total;
  float2* s = base;
  float2* hs = base + ly.hs;
  float* carry0 = reinterpret_cast<float*>(base + ly.carry);
  float* stage0 = reinterpret_cast<float*>(base + ly.stage);
  unsigned long long* mbar0 = reinterpret_cast<unsigned long long*>(base + ly.mbar);
  const int ccap = a.ccap;
  const Bar2<T> bar{1 + g};
  // the two runs: r = 0 (real part), 1 (imaginary part)
  const int rb[2] = {it.a_begin, it.b_begin}, ro[2] = {it.a_own, it.b_own}, re_[2] = {it.a_end, it.b_end};
  int trips = 0;
  if (has) trips = max(re_[0] - rb[0], re_[1] - rb[1]);
  if constexpr (T < 32) trips = __reduce_max_sync(0xffffffffu, trips);
  auto window = [&](int b, int& d, int& take, bool& bulk) {
    const int st = b * L;
    take = nx - st < L ? nx - st : L;
    d = static_cast<int>((reinterpret_cast<uintptr_t>(x + st) & 15u) >> 2);
    bulk = st + take + 4 <= nx;
  };
  // one input window per run, refilled one block ahead (after the pass that consumed it)
  auto stage_of = [&](int r) { return stage0 + r * a.scap; };
  auto prefetch = [&](int r, int k) {
    const int b = rb[r] + k;
    if (b >= re_[r]) return;
    int d, take;
    bool bulk;
    window(b, d, take, bulk);
    if (bulk && t == 0 && take > 0)
      bulk_g2s(stage_of(r), x + b * L - d, static_cast<unsigned>(((d + take) * 4 + 15) & ~15), mbar0 + r);
  };
  for (int i = threadIdx.x; i < PF::TW_PASS; i += CTA) cp_async8(twf + i, a.twf + i);
  for (int i = threadIdx.x; i < PI::TW_PASS; i += CTA) cp_async8(twi + i, a.twi + i);
  if (has) {
    const float2* Gsrc = a.spec + pl.spec_off;  // G = H / (2N) for k in [0, N/2]
    for (int k = t; k <= N / 2; k += T) cp_async8(hs + k, Gsrc + k);
    for (int i = t; i < 4 * ccap; i += T) carry0[i] = 0.f;
    if (t == 0) {
      for (int i = 0; i < 2; ++i) mbar_init(mbar0 + i, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  cp_async_wait_all();
  if (has)
    for (int k = t; k <= N / 2; k += T) hs[k] = c_scale(hs[k], 2.0f);  // H / N (exact x2)
  __syncthreads();
  if (has) {
    prefetch(0, 0);
    prefetch(1, 0);
  }
  double pw[2] = {0.0, 0.0};  // per run: this lane's Σ y² of the current power segment
#pragma unroll 1
  for (int k = 0; k < trips; ++k) {
    int b[2], d[2] = {0, 0}, take[2] = {0, 0};
    bool act[2];
    const float* src[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      b[r] = rb[r] + k;
      act[r] = has && b[r] < re_[r];
      float* stg = stage_of(r);
      if (act[r]) {
        bool bulk;
        window(b[r], d[r], take[r], bulk);
        if (bulk) {
          if (take[r] > 0) mbar_wait(mbar0 + r, k & 1);
        } else {
          const float* xs = x + b[r] * L;
          for (int i = t; i < take[r]; i += T) cp_async4(stg + d[r] + i, xs + i);
          cp_async_wait_all();
        }
      }
      src[r] = stg + d[r];
      if (!act[r]) take[r] = 0;
    }
    const bool active = act[0] || act[1];
    bar();
    first_pass_c<PF>(s, t, active, src[0], take[0], src[1], take[1], bar);
    if (has) {  // this iteration's windows are consumed: load the next blocks
      prefetch(0, k + 1);
      prefetch(1, k + 1);
    }
    middle_passes<PF, 1, false>(s, t, twf, active, bar);
    fused_mid<PF, PI>(s, t, twf, hs, active, bar);
    middle_passes<PI, 1, true>(s, t, twi, active, bar);
    // emit: element e of run r's block: e < L (or its last block) final, else carry
    float pb[2] = {0.f, 0.f};  // one chain per run
    const float* cin[2];
    float* cout[2];
    int lo[2], hi[2], start[2];
    bool last[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      cin[r] = carry0 + (2 * r + (k & 1)) * ccap;
      cout[r] = carry0 + (2 * r + ((k + 1) & 1)) * ccap;
      start[r] = b[r] * L;
      const int own_lo = ro[r] * L;
      const int own_hi = re_[r] == B ? out_len : re_[r] * L;
      lo[r] = act[r] ? own_lo - start[r] : N;  // inactive run: nothing owned
      hi[r] = act[r] ? own_hi - start[r] : N;
      last[r] = b[r] == B - 1;
    }
    emit_pass_c<PI>(s, t, twi, active, bar, [&](int e, float2 v) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float val = (e < ccap ? cin[r][e] : 0.f) + (r ? v.y : v.x);
        if (e < L || last[r]) {
          if (e >= lo[r] && e < hi[r]) {
            y[start[r] + e] = val;
            pb[r] = fmaf(val, val, pb[r]);
          }
        } else {
          cout[r][e - L] = val;
        }
      }
    });
    // power: per-lane FP64 sums over each run's segment, stored at its end (power.cuh)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      pw[r] += static_cast<double>(pb[r]);
      const bool seg_end = act[r] && closes_segment(b[r], re_[r]);
      if (__any_sync(0xffffffffu, seg_end)) {
        store_segment_power<T>(a.part + pl.part0 + static_cast<long long>(b[r] / kPowerSeg) * parts_per_block_of(T),
                               pw[r], t, seg_end && b[r] >= ro[r]);
        if (seg_end) pw[r] = 0.0;
      }
    }
  }
}

template <int N>
size_t ola2_smem(int ccap, int scap) {
  using PF = PlanF<N>;
  using PI = PlanI<N>;
  constexpr int G = ola2_cta(ilog2(N)) / PF::T;
  const Layout2 ly(PF::PADDED, N, ccap, scap);
  return (static_cast<size_t>(G) * ly.total + ((PF::TW_PASS + 1) & ~1) + ((PI::TW_PASS + 1) & ~1)) *
         sizeof(float2);
}

template <int N>
cudaError_t ola2_t(const Ola2Args& a, cudaStream_t s) {
  constexpr int CTA = ola2_cta(ilog2(N)), G = CTA / PlanF<N>::T;
  const size_t smem = ola2_smem<N>(a.ccap, a.scap);
  cudaError_t e = ensure_dynamic_smem(ola2_kernel<N>, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ola2_kernel<N>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  ola2_kernel<N><<<(a.count + G - 1) / G, CTA, smem, s>>>(a);
  return cudaGetLastError();
}

template <class PL>
void fill_c(float2* h) {
  const double pi = 3.14159265358979323846;
  for (int p = 1; p < PL::NP; ++p) {
    const int R = PL::radix(p), NS = PL::ns(p);
    for (int k = 0; k < NS; ++k) {
      const double ang = -2.0 * pi * k / (static_cast<double>(NS) * R);
      h[PL::tw_off(p) + k] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
  }
}

}  // namespace

bool ola2_supported(int log2n) { return log2n >= kOla2MinLog2N && log2n <= kOla2MaxLog2N; }

int ola2_parts_per_block(int log2n) { return parts_per_block_of(ola2_t_of(log2n)); }

int ola2_resident_items(int log2n) {
  const int cta = ola2_cta(log2n), t = ola2_t_of(log2n);
  return ola2_minb(log2n) * (cta / t);
}

// [forward table | reversed table] sizes for the context's twiddle buffer
int ola2_tw_total(int log2n, bool rev) {
  switch (log2n) {
#define RSG_CASE(L) case L: return rev ? PlanI<(1 << L)>::TW_PASS : PlanF<(1 << L)>::TW_PASS;
    RSG_CASE(5) RSG_CASE(6) RSG_CASE(7) RSG_CASE(8) RSG_CASE(9) RSG_CASE(10) RSG_CASE(11) RSG_CASE(12)
#undef RSG_CASE
  }
  return 0;
}

void ola2_fill_twiddles(int log2n, bool rev, float2* h) {
  switch (log2n) {
#define RSG_CASE(L) \
  case L: if (rev) fill_c<PlanI<(1 << L)>>(h); else fill_c<PlanF<(1 << L)>>(h); break;
    RSG_CASE(5) RSG_CASE(6) RSG_CASE(7) RSG_CASE(8) RSG_CASE(9) RSG_CASE(10) RSG_CASE(11) RSG_CASE(12)
#undef RSG_CASE
  }
}

cudaError_t launch_ola2(int log2n, const Ola2Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  switch (log2n) {
    case 5: return ola2_t<32>(a, s);
    case 6: return ola2_t<64>(a, s);
    case 7: return ola2_t<128>(a, s);
    case 8: return ola2_t<256>(a, s);
    case 9: return ola2_t<512>(a, s);
    case 10: return ola2_t<1024>(a, s);
    case 11: return ola2_t<2048>(a, s);
    case 12: return ola2_t<4096>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsg

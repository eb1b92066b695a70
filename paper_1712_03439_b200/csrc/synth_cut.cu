// synth_cut.cu — K1 for truncated renders (eta > 0): synthesize only the part of each RIR
// that truncate_rir can keep, bit-exact.
//
// Reference: synthesize_rir (roomsim/room_model.hpp:141-174) then truncate_rir (:203-213)
// keeping taps [0, n_c + 2), n_c = last n with h[n]^2 >= p_th, p_th = max h^2 10^(-eta/10)
// (:177-197).  The reference builds the whole RIR (every image of the (2K+1)^3 lattice,
// accumulated per delay bin in enumeration order), but with a -20 dB cut only the first
// few hundred to few thousand of up to 14,400 bins survive, and the images landing in the
// discarded tail are the vast majority (their count grows with the cube of the delay).
//
// One CTA per pair:
//  1. Pass 1 (approximate, FP32, any order): every image's bin D' = ceil(fl32(d) fs/c0) and
//     amplitude r^g / d accumulated with shared-memory atomics into FP32 bins b'.
//     |fl32(d) fs/c0 - d fs/c0| is below 0.01 bins, so the exact bin D of an image is D' - 1,
//     D' or D' + 1, and with the FP32 rounding of the amplitudes and of the sums (relative
//     error < 1e-3 for < 16,000 terms per bin)
//        h[n] <= UB[n] = (b'[n-1] + b'[n] + b'[n+1]) (1 + 2e-3).
//  2. Every amplitude is positive, so max_n h[n] >= h[D_0] >= 1/d_0 (the direct path,
//     computed exactly): p_th >= p_lo = (1/d_0)^2 10^(-eta/10).  Any n with UB[n]^2 < p_lo
//     has h[n]^2 < p_th: it is neither the cut index nor kept.  So with n_ub = last n with
//     UB[n]^2 >= p_lo, the kept taps lie in [0, n_exact), n_exact = min(len, n_ub + 2), and
//     the maximum of h lies there too.
//  3. Pass 2 (exact): the bins [0, n_exact) in FP64, in windows of `win` bins: the images
//     whose D' falls in [w0 - 1, w1] are compacted in enumeration order into a candidate
//     list, and that list is folded into the window exactly like K1 (rir_synth_kernel): same
//     _rn arithmetic, every bin receives its contributions sequentially in enumeration
//     order — so bins [0, n_exact) equal the reference bit for bit.
// K2 (rir_cut_kernel) then cuts within [0, n_exact) (PairRir::exact_len); the RIR length
// (rir_len), max_delay and the geometry flag are exact as in K1.
#include <cmath>

#include "kernels.cuh"

namespace rsg {

namespace {

__device__ __forceinline__ unsigned lanemask_lt_() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void shared_add_rn_(unsigned a, double v) {
  double cur;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cur) : "r"(a) : "memory");
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(__dadd_rn(cur, v)) : "memory");
}

constexpr int kCutNT = 512;   // threads per CTA (16 warps)
constexpr int kCutIPT = 4;    // candidate entries per thread per fold chunk
constexpr int kCutNW = kCutNT / 32;
constexpr int kCutCH = kCutIPT * kCutNT;  // entries per fold chunk
constexpr int kCutNV = kCutIPT * kCutNW;  // virtual warps per fold chunk
constexpr int kCutOB = 4;                 // log2(kCutNW)
constexpr int kCutNQ = (kCutNV + 3) / 4;
constexpr int kCutRS = 16 * ((((4 * kCutNQ + 15) / 16) % 2 == 0) ? (4 * kCutNQ + 15) / 16 + 1 : (4 * kCutNQ + 15) / 16);

struct CutLayout {  // byte offsets of the dynamic shared memory
  int bins, ax, axf, rg, rgf, cand, ent_a, ent_d, cnt, wcnt, total;
  __host__ __device__ CutLayout(int cap, int win, int K, int cand_cap) {
    const int W = 2 * K + 1;
    auto up = [](int v) { return (v + 15) & ~15; };
    bins = 0;
    const int region = 4 * cap > 8 * win ? 4 * cap : 8 * win;  // FP32 pass-1 bins / FP64 window
    ax = up(region);
    axf = up(ax + 8 * 3 * W);
    rg = up(axf + 4 * 3 * W);
    rgf = up(rg + 8 * (3 * K + 1));
    cand = up(rgf + 4 * (3 * K + 1));
    ent_a = up(cand + 4 * cand_cap);
    ent_d = up(ent_a + 8 * kCutCH);
    cnt = up(ent_d + 4 * kCutCH);
    wcnt = up(cnt + kCutNW * kCutRS);
    total = up(wcnt + 4 * (kCutNW + 1));
  }
};

// Image index i -> (ix, iy, iz), lattice width W.
__device__ __forceinline__ void decode(int i, int W, int& ix, int& iy, int& iz) {
  ix = i / (W * W);
  const int r = i - ix * W * W;
  iy = r / W;
  iz = r - iy * W;
}

}  // namespace

__global__ void __launch_bounds__(kCutNT) rir_synth_cut_kernel(SynthCutArgs a, int cap, int win, int cand_cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int p = a.pairs[blockIdx.x];
  const PairMeta& pm = a.pair[p];
  const UttMeta& um = a.utt[pm.utt];
  const int K = um.order, W = 2 * K + 1;
  const CutLayout ly(cap, win, K, cand_cap);
  float* b32 = reinterpret_cast<float*>(sm + ly.bins);
  double* bins = reinterpret_cast<double*>(sm + ly.bins);
  double* ax = reinterpret_cast<double*>(sm + ly.ax);
  float* axf = reinterpret_cast<float*>(sm + ly.axf);
  double* rg = reinterpret_cast<double*>(sm + ly.rg);
  float* rgf = reinterpret_cast<float*>(sm + ly.rgf);
  int* cand = reinterpret_cast<int*>(sm + ly.cand);
  double* ent_a = reinterpret_cast<double*>(sm + ly.ent_a);
  int* ent_d = reinterpret_cast<int*>(sm + ly.ent_d);
  unsigned char* cnt8 = sm + ly.cnt;
  int* wcnt = reinterpret_cast<int*>(sm + ly.wcnt);
  __shared__ double s_amp0;
  __shared__ int s_geo, s_nub;
  __shared__ unsigned long long s_dmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double spm = um.spm;
  const int len = static_cast<int>(pm.rir_cap);  // min(exact lattice max delay + 1, horizon)
  const unsigned lt = lanemask_lt_();
  unsigned bins_s;
  asm volatile("mov.b32 %0, %1;" : "=r"(bins_s) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(bins))));
  // ---- tables (room_model.hpp:126-127, :37, :43), exact FP64 and their FP32 roundings ----
  for (int idx = tid; idx < 3 * W; idx += kCutNT) {
    const int axis = idx / W, n = idx - axis * W - K;
    const double L = um.dims[axis], s = pm.src[axis];
    const double mirrored = (n % 2 == 0) ? s : __dsub_rn(L, s);
    const double pos = __dadd_rn(__dmul_rn(static_cast<double>(n), L), mirrored);
    const double diff = __dsub_rn(pos, pm.mic[axis]);
    ax[idx] = __dmul_rn(diff, diff);
    axf[idx] = static_cast<float>(ax[idx]);
  }
  for (int g = tid; g <= 3 * K; g += kCutNT) {
    rg[g] = a.rg[um.rg_off + g];
    rgf[g] = static_cast<float>(rg[g]);
  }
  for (int n = tid; n < len; n += kCutNT) b32[n] = 0.f;
  __syncthreads();
  if (tid == 0) {
    // geometry (room_model.hpp:157-158): some image at distance 0 <=> a zero term on every axis
    bool z[3] = {false, false, false};
    double mx[3] = {0.0, 0.0, 0.0};
    for (int axis = 0; axis < 3; ++axis)
      for (int n = 0; n < W; ++n) {
        const double v = ax[axis * W + n];
        z[axis] |= v == 0.0;
        mx[axis] = v > mx[axis] ? v : mx[axis];
      }
    s_geo = z[0] && z[1] && z[2];
    // exact max delay over the lattice (host lattice_max_delay, api.cu)
    s_dmax = static_cast<unsigned long long>(ceil(__dmul_rn(__dsqrt_rn(__dadd_rn(__dadd_rn(mx[0], mx[1]), mx[2])), spm)));
    // direct path: n = (0, 0, 0), g = 0
    const double d0 = __dsqrt_rn(__dadd_rn(__dadd_rn(ax[K], ax[W + K]), ax[2 * W + K]));
    s_amp0 = __ddiv_rn(rg[0], d0);
    s_nub = -1;
  }
  __syncthreads();
  PairRir& out = a.out[p];
  if (s_geo) {
    if (tid == 0) {
      out.max_delay = s_dmax;
      out.flags |= 1;
    }
    return;
  }
  const long long V = static_cast<long long>(W) * W * W;
  const float spmf = static_cast<float>(spm);
  const int step_z = kCutNT % W, step_q = kCutNT / W;
  const int step_y = step_q % W, step_x = step_q / W;
  // ---- pass 1: approximate FP32 bins, any order ----
  {
    int iz = tid % W, iy, ix;
    {
      const int q = tid / W;
      iy = q % W;
      ix = q / W;
    }
    for (long long i = tid; i < V; i += kCutNT) {
      const float d2 = (axf[ix] + axf[W + iy]) + axf[2 * W + iz];
      const float d = sqrtf(d2);
      const int D = static_cast<int>(ceilf(d * spmf));
      if (D < len) {
        const int g = abs(ix - K) + abs(iy - K) + abs(iz - K);
        atomicAdd(&b32[D], rgf[g] / d);
      }
      iz += step_z;
      int cy = step_y;
      if (iz >= W) { iz -= W; ++cy; }
      iy += cy;
      int cx = step_x;
      while (iy >= W) { iy -= W; ++cx; }
      ix += cx;
    }
  }
  __syncthreads();
  // ---- exact range: n_exact = min(len, n_ub + 2) ----
  {
    const double p_lo = __dmul_rn(__dmul_rn(s_amp0, s_amp0), a.eta_factor) * (1.0 - 1e-6);
    int last = -1;
    for (int n = tid; n < len; n += kCutNT) {
      const double s = static_cast<double>(n > 0 ? b32[n - 1] : 0.f) + static_cast<double>(b32[n]) +
                       static_cast<double>(n + 1 < len ? b32[n + 1] : 0.f);
      const double ub = s * (1.0 + 2e-3);
      if (ub * ub >= p_lo) last = n;
    }
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0 && last >= 0) atomicMax(&s_nub, last);
  }
  __syncthreads();
  const int n_exact = min(len, s_nub + 2);
  // ---- pass 2: exact bins [0, n_exact) in windows of `win` bins ----
  for (int w0 = 0; w0 < n_exact; w0 += win) {
    const int w1 = min(n_exact, w0 + win), wl = w1 - w0;
    __syncthreads();  // pass-1 bins / the previous window are no longer read
    for (int n = tid; n < wl; n += kCutNT) bins[n] = 0.0;
    int ncand = 0;
    // fold the candidate list [0, ncand) into the window: K1's ordered scatter
    auto flush = [&]() {
      __syncthreads();  // candidates and zeroed bins visible
      for (int base = 0; base < ncand; base += kCutCH) {
        int rel_bin[kCutIPT];
        double amp[kCutIPT];
#pragma unroll
        for (int h = 0; h < kCutIPT; ++h) {
          const int e = base + h * kCutNT + tid;
          rel_bin[h] = -1;
          amp[h] = 0.0;
          if (e < ncand) {
            int ix, iy, iz;
            decode(cand[e], W, ix, iy, iz);
            const double d2 = __dadd_rn(__dadd_rn(ax[ix], ax[W + iy]), ax[2 * W + iz]);
            const double d = __dsqrt_rn(d2);
            const long long D = static_cast<long long>(ceil(__dmul_rn(d, spm)));
            const long long rel = D - w0;
            if (rel >= 0 && rel < wl) {
              const int g = abs(ix - K) + abs(iy - K) + abs(iz - K);
              amp[h] = __ddiv_rn(rg[g], d);
              rel_bin[h] = static_cast<int>(rel);
            }
          }
        }
        // publish: per entry slot, lane masks per owner (as rir_synth_kernel)
        int owner[kCutIPT];
        unsigned mine[kCutIPT];
#pragma unroll
        for (int h = 0; h < kCutIPT; ++h) {
          owner[h] = (rel_bin[h] ^ (rel_bin[h] >> 4)) & (kCutNW - 1);
          mine[h] = __ballot_sync(0xffffffffu, rel_bin[h] >= 0);
          unsigned row = mine[h];
#pragma unroll
          for (int k = 0; k < kCutOB; ++k) {
            const unsigned bk = __ballot_sync(0xffffffffu, (owner[h] >> k) & 1);
            mine[h] &= ((owner[h] >> k) & 1) ? bk : ~bk;
            row &= ((lane >> k) & 1) ? bk : ~bk;
          }
          if (lane < kCutNW) cnt8[lane * kCutRS + h * kCutNW + warp] = static_cast<unsigned char>(__popc(row));
        }
        __syncthreads();
        unsigned ub[kCutIPT], utotal = 0u;
#pragma unroll
        for (int h = 0; h < kCutIPT; ++h) ub[h] = 0u;
        if (lane < kCutNW) {
          const unsigned* rowp = reinterpret_cast<const unsigned*>(cnt8 + lane * kCutRS);
#pragma unroll
          for (int q = 0; q < kCutNQ; ++q) {
            const unsigned wq = 4 * q + 4 <= kCutNV ? rowp[q] : (rowp[q] & ((1u << (8 * (kCutNV - 4 * q))) - 1u));
            utotal = __dp4a(wq, 0x01010101u, utotal);
#pragma unroll
            for (int h = 0; h < kCutIPT; ++h) {
              const int nb = h * kCutNW + warp - 4 * q;
              const unsigned m = nb <= 0 ? 0u : nb >= 4 ? 0xffffffffu : (1u << (8 * nb)) - 1u;
              ub[h] = __dp4a(wq & m, 0x01010101u, ub[h]);
            }
          }
        }
        const int total = static_cast<int>(utotal);
        int incl = total;
#pragma unroll
        for (int o = 1; o < kCutNW; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int obase = incl - total;
#pragma unroll
        for (int h = 0; h < kCutIPT; ++h) {
          const int seg = __shfl_sync(0xffffffffu, obase + static_cast<int>(ub[h]), rel_bin[h] >= 0 ? owner[h] : 0);
          if (rel_bin[h] >= 0) {
            const int pos = seg + __popc(mine[h] & lt);
            ent_d[pos] = rel_bin[h];
            ent_a[pos] = amp[h];
          }
        }
        const int my_base = __shfl_sync(0xffffffffu, obase, warp);
        const int my_total = __shfl_sync(0xffffffffu, total, warp);
        __syncthreads();
        for (int r0 = 0; r0 < my_total; r0 += 32) {
          const int l = r0 + lane;
          const bool valid = l < my_total;
          const int bn = valid ? ent_d[my_base + l] : -1 - lane;
          const double av = valid ? ent_a[my_base + l] : 0.0;
          const unsigned grp = __match_any_sync(0xffffffffu, bn);
          const int rank = __popc(grp & lt);
          const int rounds = __reduce_max_sync(0xffffffffu, valid ? __popc(grp) : 0);
          const unsigned ba = bins_s + 8u * static_cast<unsigned>(bn);
          if (valid && rank == 0) shared_add_rn_(ba, av);
          for (int r = 1; r < rounds; ++r) {
            __syncwarp();
            if (valid && rank == r) shared_add_rn_(ba, av);
          }
          __syncwarp();
        }
        __syncthreads();  // entries / counts reused by the next chunk
      }
      ncand = 0;
    };
    // candidates in enumeration order: FP32 bin D' in [w0 - 1, w1]
    int iz = tid % W, iy, ix;
    {
      const int q = tid / W;
      iy = q % W;
      ix = q / W;
    }
    for (long long i0 = 0; i0 < V; i0 += kCutNT) {
      const long long i = i0 + tid;
      bool flag = false;
      if (i < V) {
        const float d2 = (axf[ix] + axf[W + iy]) + axf[2 * W + iz];
        const int D = static_cast<int>(ceilf(sqrtf(d2) * spmf));
        flag = D >= w0 - 1 && D <= w1;
      }
      const unsigned m = __ballot_sync(0xffffffffu, flag);
      if (lane == 0) wcnt[warp] = __popc(m);
      __syncthreads();
      int off = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kCutNW; ++w) {
        const int c = wcnt[w];
        off += w < warp ? c : 0;
        tot += c;
      }
      if (flag) cand[ncand + off + __popc(m & lt)] = static_cast<int>(i);
      ncand += tot;
      __syncthreads();  // wcnt reused
      if (ncand > cand_cap - kCutNT) flush();
      iz += step_z;
      int cy = step_y;
      if (iz >= W) { iz -= W; ++cy; }
      iy += cy;
      int cx = step_x;
      while (iy >= W) { iy -= W; ++cx; }
      ix += cx;
    }
    if (ncand > 0) flush();
    __syncthreads();
    double* dst = a.rir + pm.rir_off + w0;
    for (int n = tid; n < wl; n += kCutNT) dst[n] = bins[n];
  }
  if (tid == 0) {
    out.max_delay = s_dmax;
    out.exact_len = n_exact;
  }
}

size_t synth_cut_smem_bytes(int cap, int win, int max_order, int cand_cap) {
  return static_cast<size_t>(CutLayout(cap, win, max_order, cand_cap).total);
}

cudaError_t launch_synth_cut(const SynthCutArgs& a, int n_pairs, int cap, int win, int max_order, int cand_cap,
                             cudaStream_t s) {
  if (n_pairs == 0) return cudaSuccess;
  const size_t smem = synth_cut_smem_bytes(cap, win, max_order, cand_cap);
  cudaError_t e = cudaFuncSetAttribute(rir_synth_cut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  rir_synth_cut_kernel<<<n_pairs, kCutNT, smem, s>>>(a, cap, win, cand_cap);
  return cudaGetLastError();
}

}  // namespace rsg

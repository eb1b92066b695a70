// synth_bound.cu — K1a: which bins of a RIR can survive the -eta dB cut.
//
// Reference: synthesize_rir (roomsim/room_model.hpp:141-174) builds the whole RIR — every
// image of the (2K+1)^3 lattice, accumulated per delay bin in enumeration order — and
// truncate_rir (:203-213) then keeps taps [0, n_c + 2), n_c = last n with h[n]^2 >= p_th,
// p_th = max h^2 10^(-eta/10) (:177-197).  With a -20 dB cut a few hundred to a few thousand
// of up to 14,400 bins survive, and the images that land in the discarded tail are the vast
// majority (their count grows with the cube of the delay).  This kernel finds, per pair, a
// prefix [0, n_exact) that provably contains every kept tap and the maximum, so that K1
// (rir_synth_kernel) runs its exact, ordered FP64 accumulation only over the images that can
// land there (the sub-lattice inside the sphere of delay n_exact) — bit-exact results at a
// fraction of the ordered-scatter work.
//
//  1. Bound pass (FP32, any order): every image's approximate bin D' = ceil(fl32(d) fs/c0) and
//     an UPPER bound of its amplitude r^g / d in fixed point, q = floor(2^20 (r^g/d) / a_0 (1 + e)) + 1
//     with a_0 = 1/d_0 the direct path's amplitude, added to a 32-bit integer bin by a native
//     shared-memory atomic (sm_100a has no shared-memory float atomic: atomicAdd(float*) on
//     shared memory is a compare-and-swap loop; ATOMS.ADD on u32 is one instruction).  Integer
//     sums are exact and order independent.  Each add returns the old value, so a bin reaching
//     2^31 is always seen by the thread whose add crosses it (every q < 2^22): overflow cannot
//     go unnoticed, and such a pair falls back to the full synthesis.
//  2. |fl32(d) fs/c0 - d fs/c0| < 0.02 bins for RIRs up to 32768 bins, so an image's exact bin
//     D is D' - 1, D' or D' + 1, and with the FP32 roundings (< 1e-6 relative, covered by a
//     1e-3 margin)      h[n] <= UB[n] = (b[n-1] + b[n] + b[n+1]) (a_0 / 2^20) (1 + 1e-3).
//  3. Every amplitude is positive (0 < r < 1, room_model.hpp:57-65), and FP64 addition of
//     non-negative terms is monotone, so max_n h[n] >= h[D_0] >= a_0 (computed exactly as K1
//     does): p_th >= p_lo = a_0^2 10^(-eta/10) (1 - 1e-6).  Any n with UB[n]^2 < p_lo has
//     h[n]^2 < p_th: it is neither the cut index nor the maximum.  With n_ub the last n with
//     UB[n]^2 >= p_lo, all kept taps lie in [0, n_exact), n_exact = min(len, n_ub + 2).
// K2 (rir_cut_kernel) then scans [0, n_exact) only.  max_delay and the geometry flag are the
// exact values K1 would produce (per-axis maxima / zeros of the squared offsets).
#include <cmath>

#include "kernels.cuh"

namespace rsg {

namespace {
constexpr float kBoundScale = 1048576.f;  // 2^20 fixed-point units per a_0
}  // namespace

// kBoundNT = 512 threads per pair, or 128 for the small lattices (K <= 12: a few thousand
// images; the CTA's fixed costs dominate and four times as many CTAs fit an SM)
template <int kBoundNT>
__global__ void __launch_bounds__(kBoundNT) rir_bound_kernel(SynthBoundArgs a, int cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int p = a.pairs[blockIdx.x];
  const PairMeta& pm = a.pair[p];
  const UttMeta& um = a.utt[pm.utt];
  const int K = um.order, W = 2 * K + 1;
  unsigned* bins = reinterpret_cast<unsigned*>(sm);                      // [cap]
  double* ax = reinterpret_cast<double*>(sm + ((4 * static_cast<size_t>(cap) + 15) & ~size_t(15)));  // [3W] exact
  float* axf = reinterpret_cast<float*>(ax + 3 * W);                      // [3W]
  float* rgs = axf + 3 * W;                                               // [3K+1]: r^g 2^20 / a_0, rounded up
  __shared__ double s_a0;
  __shared__ int s_state, s_last, s_d0;  // state: 0 cut, 1 geometry error, 2 no cut (direct path outside)
  __shared__ unsigned long long s_dmax;
  const int tid = threadIdx.x, lane = tid & 31;
  const double spm = um.spm;
  const int len = static_cast<int>(pm.rir_cap);  // min(exact lattice max delay + 1, horizon) <= cap
  PairRir& out = a.out[p];
  // squared per-axis offsets exactly as K1 (room_model.hpp:126-127, :37, :43)
  for (int idx = tid; idx < 3 * W; idx += kBoundNT) {
    const int axis = idx / W, n = idx - axis * W - K;
    const double L = um.dims[axis], s = pm.src[axis];
    const double mirrored = (n % 2 == 0) ? s : __dsub_rn(L, s);
    const double pos = __dadd_rn(__dmul_rn(static_cast<double>(n), L), mirrored);
    const double diff = __dsub_rn(pos, pm.mic[axis]);
    ax[idx] = __dmul_rn(diff, diff);
    axf[idx] = static_cast<float>(ax[idx]);
  }
  for (int n = tid; n < len; n += kBoundNT) bins[n] = 0u;
  if (tid == 0) s_last = -1;
  __syncthreads();
  if (tid == 0) {
    // geometry (room_model.hpp:157-158): an image at distance 0 <=> a zero term on every axis;
    // exact max delay (api.cu lattice_max_delay): the per-axis maxima, every step monotone
    bool z[3] = {false, false, false};
    double mx[3] = {0.0, 0.0, 0.0};
    for (int axis = 0; axis < 3; ++axis)
      for (int n = 0; n < W; ++n) {
        const double v = ax[axis * W + n];
        z[axis] |= v == 0.0;
        mx[axis] = v > mx[axis] ? v : mx[axis];
      }
    s_dmax = static_cast<unsigned long long>(ceil(__dmul_rn(__dsqrt_rn(__dadd_rn(__dadd_rn(mx[0], mx[1]), mx[2])), spm)));
    // direct path: image (0, 0, 0), g = 0 (room_model.hpp:159-162)
    const double d0 = __dsqrt_rn(__dadd_rn(__dadd_rn(ax[K], ax[W + K]), ax[2 * W + K]));
    const double dl0 = ceil(__dmul_rn(d0, spm));
    s_a0 = d0 > 0.0 ? __ddiv_rn(a.rg[um.rg_off], d0) : 0.0;
    s_d0 = dl0 < 2.0e9 ? static_cast<int>(dl0) : 2000000000;
    s_state = (z[0] && z[1] && z[2]) ? 1 : ((s_d0 >= len || !(s_a0 > 0.0)) ? 2 : 0);
  }
  __syncthreads();
  if (s_state != 0) {
    if (tid == 0) {
      out.max_delay = s_dmax;
      if (s_state == 1) out.flags |= 1;
      out.exact_len = 0;  // K1 runs in full (and reports the geometry error itself)
    }
    return;
  }
  {  // r^g in fixed point, rounded up
    const double sc = static_cast<double>(kBoundScale) / s_a0;
    for (int g = tid; g <= 3 * K; g += kBoundNT) {
      const double v = a.rg[um.rg_off + g] * sc * (1.0 + 2e-6);  // + the FP32 roundings of q
      float f = static_cast<float>(v);
      if (static_cast<double>(f) < v) f = nextafterf(f, INFINITY);
      rgs[g] = f;
    }
  }
  __syncthreads();
  const float spmf = static_cast<float>(spm);
  int ovf = 0;
  // Row-wise walk: a thread takes whole (ix, iy) rows, so the x/y part of the squared distance
  // and of the reflection count is computed once per row and the inner loop over iz is ~20
  // instructions per image (the image-major walk of K1 spent ~80 on index arithmetic).
  {
    const float* axz = axf + 2 * W;
    const unsigned ulen = static_cast<unsigned>(len);
    for (int row = tid; row < W * W; row += kBoundNT) {
      const int ix = row / W, iy = row - ix * W;
      const float d2xy = axf[ix] + axf[W + iy];
      const int gxy = abs(ix - K) + abs(iy - K);
#pragma unroll 4
      for (int iz = 0; iz < W; ++iz) {
        const float d2 = d2xy + axz[iz];
        const float rs = rsqrtf(d2);
        const unsigned D = static_cast<unsigned>(__float2int_ru((d2 * rs) * spmf));  // negative / NaN -> huge
        if (D <= ulen) {  // D = len: the exact bin may be len - 1
          const float qf = rgs[gxy + abs(iz - K)] * rs;
          if (!(qf < 4.0e6f)) ovf = 1;  // an amplitude above the direct path's (cannot happen) or NaN
          const unsigned q = static_cast<unsigned>(__float2int_rz(fminf(qf, 4.0e6f))) + 1u;
          const unsigned old = atomicAdd(&bins[D < ulen ? D : ulen - 1u], q);
          ovf |= static_cast<int>((old + q) >> 31);
        }
      }
    }
  }
  if (__syncthreads_or(ovf)) {
    if (tid == 0) {
      out.max_delay = s_dmax;
      out.exact_len = 0;
    }
    return;
  }
  {
    const double unit = s_a0 / static_cast<double>(kBoundScale) * (1.0 + 1e-3);
    const double p_lo = __dmul_rn(__dmul_rn(s_a0, s_a0), a.eta_factor) * (1.0 - 1e-6);
    int last = -1;
    for (int n = tid; n < len; n += kBoundNT) {
      const unsigned long long s = static_cast<unsigned long long>(n > 0 ? bins[n - 1] : 0u) + bins[n] +
                                   (n + 1 < len ? bins[n + 1] : 0u);
      const double ub = static_cast<double>(s) * unit;
      if (ub * ub >= p_lo) last = n;
    }
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0 && last >= 0) atomicMax(&s_last, last);
  }
  __syncthreads();
  if (tid == 0) {
    out.max_delay = s_dmax;
    const int n_exact = min(len, max(s_last, s_d0) + 2);
    out.exact_len = n_exact >= len ? 0 : n_exact;
  }
}

cudaError_t launch_synth_bound(const SynthBoundArgs& a, int n_pairs, int cap, int max_order, cudaStream_t s, int nt) {
  if (n_pairs == 0) return cudaSuccess;
  const int W = 2 * max_order + 1;
  const size_t smem = ((4 * static_cast<size_t>(cap) + 15) & ~size_t(15)) + sizeof(double) * 3 * W + sizeof(float) * 3 * W +
                      sizeof(float) * (3 * max_order + 1) + 16;
  auto go = [&](auto kern, int threads) {
    cudaError_t e = ensure_dynamic_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<n_pairs, threads, smem, s>>>(a, cap);
    return cudaGetLastError();
  };
  return nt == 128 ? go(rir_bound_kernel<128>, 128) : go(rir_bound_kernel<512>, 512);
}

}  // namespace rsg

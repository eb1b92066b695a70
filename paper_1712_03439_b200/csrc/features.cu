// features.cu — log-Mel front end on the rendered channels (the
// paper's consumer of the simulator): 128 log-Mel energies per
// 32 ms frame (512 samples at 16 kHz, periodic Hann window) every 10 ms (160 samples),
// triangular HTK-mel filters between 125 and 7500 Hz on the power spectrum, natural
// log with a floor; four consecutive frames stacked into a 512-element vector and the
// stacked sequence down-sampled by three (stacked vector t = frames 3t .. 3t+3).
//
// One warp per frame (tiles of 8 consecutive frames per CTA): each warp windows its
// frame (read straight from global memory, L1 serves the overlaps) and runs the
// 512-point real FFT as the 256-point complex Stockham transform of the packed frame
// (fft.cuh, the same building blocks as K3/K4), untangles the power spectrum, applies
// the sparse filterbank and writes each log energy into every stacked vector that
// contains its frame.
#include <cmath>

#include "fft.cuh"
#include "kernels.cuh"

namespace rsg {
namespace {

constexpr int kFrame = 512, kHop = 160, kMels = 128, kFramesPerCta = 8;
using PLM = Plan<256>;

__device__ __forceinline__ float2 pair_tw256(const float2* W, int k) {  // exp(-2 pi i k / 512), k in [0, 256]
  if (k <= 128) return W[k];
  const float2 w = W[256 - k];
  return make_float2(-w.x, w.y);
}

constexpr int kMaxNnz = 2 * (kFrame / 2 + 1);  // each bin feeds at most two triangles

struct WarpBar {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

// One warp per frame (the 256-point transform needs exactly 32 threads), persistent
// over the tiles; warps never wait for each other.  The window and the filterbank are
// staged in shared memory once per CTA.
__global__ void __launch_bounds__(kFramesPerCta * PLM::T) logmel_kernel(LogMelArgs a) {
  constexpr int T = PLM::T;  // 32
  static_assert(T == 32, "one warp per transform");
  __shared__ float win[kFrame];
  __shared__ int mptr[kMels + 1];
  __shared__ short mbin[kMaxNnz];
  __shared__ float mw[kMaxNnz];
  __shared__ __align__(16) float2 fft[kFramesPerCta][PLM::PADDED];
  __shared__ __align__(16) float xw[kFramesPerCta][kFrame];  // windowed frame, then its power spectrum
  for (int i = threadIdx.x; i < kFrame; i += blockDim.x) win[i] = a.window[i];
  for (int i = threadIdx.x; i <= kMels; i += blockDim.x) mptr[i] = a.mel_ptr[i];
  const int nnz = a.mel_ptr[kMels];
  for (int i = threadIdx.x; i < nnz; i += blockDim.x) {
    mbin[i] = static_cast<short>(a.mel_bin[i]);
    mw[i] = a.mel_w[i];
  }
  __syncthreads();
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const float2* W = a.tw + PLM::TW_PASS;
  float* x = xw[g];
  float2* s = fft[g];
  const WarpBar bar{};
  for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const LogMelTile tl = a.tiles[tile];
    if (g >= tl.nfr) continue;  // warp-uniform
    const int f = tl.f0 + g;
    const float* src = a.wave + tl.wave_off + static_cast<long long>(f) * kHop;
    if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
#pragma unroll
      for (int i = 0; i < kFrame / 128; ++i) {
        const int n = 4 * (t + 32 * i);
        const float4 v = __ldg(reinterpret_cast<const float4*>(src + n));
        *reinterpret_cast<float4*>(x + n) =
            make_float4(win[n] * v.x, win[n + 1] * v.y, win[n + 2] * v.z, win[n + 3] * v.w);
      }
    } else {
      for (int n = t; n < kFrame; n += T) x[n] = win[n] * __ldg(src + n);
    }
    __syncwarp();
    first_pass<256, float, WarpBar, true>(s, t, true, x, kFrame, bar);
    forward_rest<256, 1, WarpBar>(s, t, a.tw, true, bar);
    for (int k = t; k <= 256; k += T) {  // X[k] = (Z[k] + conj Z[M-k] + W^k (-i)(Z[k] - conj Z[M-k])) / 2
      const float2 za = s[PAD(k & 255)];
      const float2 zb = c_conj(s[PAD((256 - k) & 255)]);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      const float2 X = c_scale(c_add(S, c_mul(pair_tw256(W, k), D)), 0.5f);
      x[k] = X.x * X.x + X.y * X.y;  // power spectrum over the (consumed) windowed frame
    }
    __syncwarp();
    for (int m = t; m < kMels; m += T) {
      float e = 0.f;
      for (int i = mptr[m]; i < mptr[m + 1]; ++i) e = fmaf(mw[i], x[mbin[i]], e);
      const float lm = __logf(fmaxf(e, a.log_floor));
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // stacked vector t_out holds frames 3 t_out .. 3 t_out + 3
        const int q = f - c;
        if (q >= 0 && q % 3 == 0 && q / 3 < tl.nstack)
          a.feat[tl.feat_off + static_cast<long long>(q / 3) * (4 * kMels) + c * kMels + m] = lm;
      }
    }
    __syncwarp();  // x and s are reused by this warp's next frame
  }
}

}  // namespace

cudaError_t launch_logmel(const LogMelArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return cudaSuccess;
  const int grid = a.n_tiles < 148 * 8 ? a.n_tiles : 148 * 8;
  logmel_kernel<<<grid, kFramesPerCta * PLM::T, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rsg

// features.cu — log-Mel front end on the rendered channels (the
// paper's consumer of the simulator): 128 log-Mel energies per
// 32 ms frame (512 samples at 16 kHz, periodic Hann window) every 10 ms (160 samples),
// triangular HTK-mel filters between 125 and 7500 Hz on the power spectrum, natural
// log with a floor; four consecutive frames stacked into a 512-element vector and the
// stacked sequence down-sampled by three (stacked vector t = frames 3t .. 3t+3).
//
// One CTA = 8 consecutive frames of one channel: the 1632 samples they span are read
// once into shared memory; each 32-thread group windows its frame and runs the
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

__global__ void __launch_bounds__(kFramesPerCta * PLM::T) logmel_kernel(LogMelArgs a) {
  constexpr int T = PLM::T;  // 32 threads per transform
  __shared__ float smp[(kFramesPerCta - 1) * kHop + kFrame];
  __shared__ __align__(16) float2 fft[kFramesPerCta][PLM::PADDED];
  __shared__ __align__(16) float xw[kFramesPerCta][kFrame];  // windowed frame, then its power spectrum
  float(*pw)[kFrame] = xw;
  const LogMelTile tl = a.tiles[blockIdx.x];
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const bool active = g < tl.nfr;
  const float* src = a.wave + tl.wave_off + static_cast<long long>(tl.f0) * kHop;
  const int span = (tl.nfr - 1) * kHop + kFrame;
  for (int i = threadIdx.x; i < span; i += blockDim.x) smp[i] = src[i];
  __syncthreads();
  if (active)
    for (int n = t; n < kFrame; n += T) xw[g][n] = a.window[n] * smp[g * kHop + n];
  __syncthreads();
  first_pass<256, float, CtaBar, true>(fft[g], t, active, xw[g], kFrame);
  forward_rest<256>(fft[g], t, a.tw, active);
  if (active) {
    const float2* W = a.tw + PLM::TW_PASS;
    const float2* s = fft[g];
    for (int k = t; k <= 256; k += T) {  // X[k] = (Z[k] + conj Z[M-k] + W^k (-i)(Z[k] - conj Z[M-k])) / 2
      const float2 za = s[PAD(k & 255)];
      const float2 zb = c_conj(s[PAD((256 - k) & 255)]);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      const float2 X = c_scale(c_add(S, c_mul(pair_tw256(W, k), D)), 0.5f);
      pw[g][k] = X.x * X.x + X.y * X.y;
    }
  }
  __syncthreads();
  if (active) {
    const int f = tl.f0 + g;
    for (int m = t; m < kMels; m += T) {
      float e = 0.f;
      for (int i = a.mel_ptr[m]; i < a.mel_ptr[m + 1]; ++i) e = fmaf(a.mel_w[i], pw[g][a.mel_bin[i]], e);
      const float lm = logf(fmaxf(e, a.log_floor));
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // stacked vector t_out holds frames 3 t_out .. 3 t_out + 3
        const int q = f - c;
        if (q >= 0 && q % 3 == 0 && q / 3 < tl.nstack)
          a.feat[tl.feat_off + static_cast<long long>(q / 3) * (4 * kMels) + c * kMels + m] = lm;
      }
    }
  }
}

}  // namespace

cudaError_t launch_logmel(const LogMelArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return cudaSuccess;
  logmel_kernel<<<a.n_tiles, kFramesPerCta * PLM::T, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rsg

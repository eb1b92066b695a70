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
#include "mixfin.cuh"

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

// One frame on one warp: window src[0, 512) into x, the 512-point real FFT as the
// 256-point complex transform of the packed frame, the power spectrum, the sparse
// filterbank and the log; each log energy goes into every stacked vector that holds
// frame f.  src may be global (16-byte aligned: float4 loads) or shared memory.
__device__ __forceinline__ void frame_logmel(const float* src, bool al16, int f, long long feat_off, int nstack,
                                             const float* win, const int* mptr, const short* mbin,
                                             const float* mw, const float2* tw, float log_floor, float* x,
                                             float2* s, float* feat, int t) {
  constexpr int T = PLM::T;
  const float2* W = tw + PLM::TW_PASS;
  const WarpBar bar{};
  if (al16) {
#pragma unroll
    for (int i = 0; i < kFrame / 128; ++i) {
      const int n = 4 * (t + 32 * i);
      const float4 v = *reinterpret_cast<const float4*>(src + n);
      *reinterpret_cast<float4*>(x + n) =
          make_float4(win[n] * v.x, win[n + 1] * v.y, win[n + 2] * v.z, win[n + 3] * v.w);
    }
  } else {
    for (int n = t; n < kFrame; n += T) x[n] = win[n] * src[n];
  }
  __syncwarp();
  first_pass<256, float, WarpBar, true>(s, t, true, x, kFrame, bar);
  forward_rest<256, 1, WarpBar>(s, t, tw, true, bar);
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
    const float lm = __logf(fmaxf(e, log_floor));
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // stacked vector t_out holds frames 3 t_out .. 3 t_out + 3
      const int q = f - c;
      if (q >= 0 && q % 3 == 0 && q / 3 < nstack)
        feat[feat_off + static_cast<long long>(q / 3) * (4 * kMels) + c * kMels + m] = lm;
    }
  }
  __syncwarp();  // x and s are reused by this warp's next frame
}

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
  // a contiguous range of tiles per CTA: the first tile's channel by a 32-ary search of the warp
  // (the largest ch with tile_begin[ch] <= tile), the following ones by stepping forward
  const int tile_lo = static_cast<int>(static_cast<long long>(a.n_tiles) * blockIdx.x / gridDim.x);
  const int tile_hi = static_cast<int>(static_cast<long long>(a.n_tiles) * (blockIdx.x + 1) / gridDim.x);
  int lo = 0;
  {
    int n = a.n_chan;  // tile_begin[lo] <= tile_lo < tile_begin[lo + n]
    while (n > 1) {
      const int step = (n + 31) / 32;
      const int idx = lo + t * step;
      const bool le = idx < lo + n && __ldg(&a.chans[idx].tile_begin) <= tile_lo;
      const int k = 31 - __clz(__ballot_sync(0xffffffffu, le));  // lane 0 always holds
      const int hi = lo + n;
      lo += k * step;
      n = min(step, hi - lo);
    }
  }
  for (int tile = tile_lo; tile < tile_hi; ++tile) {
    while (__ldg(&a.chans[lo + 1].tile_begin) <= tile) ++lo;  // (chans[n_chan].tile_begin = n_tiles > tile)
    const LogMelChan chn = a.chans[lo];
    const int f0 = 8 * (tile - chn.tile_begin);
    const int used = chn.nstack > 0 ? 3 * (chn.nstack - 1) + 4 : 0;  // frames that reach a stacked vector
    if (f0 + g >= used) continue;  // warp-uniform
    const int f = f0 + g;
    const float* src = a.wave + chn.wave_off + static_cast<long long>(f) * kHop;
    frame_logmel(src, (reinterpret_cast<uintptr_t>(src) & 15u) == 0, f, chn.feat_off, chn.nstack, win, mptr, mbin,
                 mw, a.tw, a.log_floor, xw[g], fft[g], a.feat, t);
  }
}

// ---- mix + log-Mel in one kernel (the render's features mode) --------------------------
// One CTA per (channel, tile of kMixTile output samples): it mixes the tile plus the
// kFrame - 1 samples its last frames reach into (the arithmetic of mix_kernel, MixQuadAcc:
// FP32 FMAs in source order), writes the tile to the output
// channel when one is given, and computes from shared memory the log-Mel of every
// stacked-vector frame that starts in the tile.  The waveform never has to be re-read
// from HBM, and with no output channel it is never written at all.
constexpr int kMixTile = 4096;
constexpr int kTileBuf = kMixTile + kFrame;  // + the frames' reach (kFrame - 1), rounded to quads

__device__ __forceinline__ float4 mix_quad_f(const float* row, long long ol, long long n) {
  if (n + 3 < ol) return __ldcs(reinterpret_cast<const float4*>(row + n));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (n < ol) v.x = row[n];
  if (n + 1 < ol) v.y = row[n + 1];
  if (n + 2 < ol) v.z = row[n + 2];
  return v;
}

constexpr int kFuseMaxI = 8;

__global__ void __launch_bounds__(kFramesPerCta * PLM::T) mix_logmel_kernel(MixArgs a, MixFeatArgs lf) {
  constexpr int NT = kFramesPerCta * PLM::T;  // 256
  extern __shared__ __align__(16) unsigned char fsm[];
  float* tile = reinterpret_cast<float*>(fsm);                                  // [kTileBuf]
  float* xw = tile + kTileBuf;                                                   // [8][kFrame]
  float2* fft = reinterpret_cast<float2*>(xw + kFramesPerCta * kFrame);         // [8][PADDED]
  float* win = reinterpret_cast<float*>(fft + kFramesPerCta * PLM::PADDED);      // [kFrame]
  float* mw = win + kFrame;                                                      // [kMaxNnz]
  int* mptr = reinterpret_cast<int*>(mw + kMaxNnz);                              // [kMels + 1]
  short* mbin = reinterpret_cast<short*>(mptr + kMels + 1);                      // [kMaxNnz]
  __shared__ const float* s_row[kFuseMaxI];
  __shared__ long long s_len[kFuseMaxI];
  __shared__ double s_gain[kFuseMaxI];
  const long long ch = blockIdx.y;
  const long long u = a.chan_utt[ch];
  const long long stride = a.utt_stride[u];
  const long long n0 = static_cast<long long>(blockIdx.x) * kMixTile;
  if (n0 >= stride) return;
  const int j = a.chan_mic[ch];
  const long long len = a.utt_len[u];
  const int I = a.utt_I[u], J = a.utt_J[u];
  const long long pair0 = a.utt_pair0[u];
  if (threadIdx.x < kFuseMaxI && threadIdx.x < I) {
    const long long p = pair0 + static_cast<long long>(threadIdx.x) * J + j;
    s_row[threadIdx.x] = a.y + a.plan[p].y_off;
    s_len[threadIdx.x] = a.plan[p].out_len;
    s_gain[threadIdx.x] = a.gain[p];
  }
  for (int i = threadIdx.x; i < kFrame; i += NT) win[i] = lf.window[i];
  for (int i = threadIdx.x; i <= kMels; i += NT) mptr[i] = lf.mel_ptr[i];
  const int nnz = lf.mel_ptr[kMels];
  for (int i = threadIdx.x; i < nnz; i += NT) {
    mbin[i] = static_cast<short>(lf.mel_bin[i]);
    mw[i] = lf.mel_w[i];
  }
  __syncthreads();
  const int Ic = I < kFuseMaxI ? I : kFuseMaxI;
  float* out = a.out ? a.out + a.chan_out[ch] : nullptr;
  const long long n_out = n0 + kMixTile < stride ? n0 + kMixTile : stride;  // samples written by this CTA
  // mix [n0, n0 + kTileBuf) into smem (mix_kernel's arithmetic), write [n0, n_out)
  for (int q = threadIdx.x; q < kTileBuf / 4; q += NT) {
    const long long n = n0 + 4 * q;
    MixQuadAcc acc;
    if (n < len) {
      int i = 0;
      for (; i + 1 < Ic; i += 2) {
        const float4 va = mix_quad_f(s_row[i], s_len[i], n);
        const float4 vb = mix_quad_f(s_row[i + 1], s_len[i + 1], n);
        acc.add(s_gain[i], va);
        acc.add(s_gain[i + 1], vb);
      }
      if (i < Ic) acc.add(s_gain[i], mix_quad_f(s_row[i], s_len[i], n));
      for (i = kFuseMaxI; i < I; ++i) {
        const long long p = pair0 + static_cast<long long>(i) * J + j;
        acc.add(a.gain[p], mix_quad_f(a.y + a.plan[p].y_off, a.plan[p].out_len, n));
      }
    }
    const float4 o = make_float4(static_cast<float>(acc.a0), n + 1 < len ? static_cast<float>(acc.a1) : 0.f,
                                 n + 2 < len ? static_cast<float>(acc.a2) : 0.f,
                                 n + 3 < len ? static_cast<float>(acc.a3) : 0.f);
    *reinterpret_cast<float4*>(tile + 4 * q) = o;
    if (out && n < n_out) {
      if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0 && n + 3 < n_out) {
        __stcs(reinterpret_cast<float4*>(out + n), o);
      } else {
        out[n] = o.x;
        if (n + 1 < n_out) out[n + 1] = o.y;
        if (n + 2 < n_out) out[n + 2] = o.z;
        if (n + 3 < n_out) out[n + 3] = o.w;
      }
    }
  }
  __syncthreads();
  // frames of the stacked vectors that start in [n0, n0 + kMixTile)
  const long long F = len >= kFrame ? 1 + (len - kFrame) / kHop : 0;
  const int S = F >= 4 ? static_cast<int>((F - 4) / 3 + 1) : 0;
  const long long used = S > 0 ? 3LL * (S - 1) + 4 : 0;
  const long long f_lo = (n0 + kHop - 1) / kHop;
  long long f_hi = (n0 + kMixTile + kHop - 1) / kHop;  // exclusive
  if (f_hi > used) f_hi = used;
  const int g = threadIdx.x / PLM::T, t = threadIdx.x % PLM::T;
  for (long long f = f_lo + g; f < f_hi; f += kFramesPerCta) {
    const float* src = tile + (f * kHop - n0);
    frame_logmel(src, ((f * kHop - n0) & 3) == 0, static_cast<int>(f), lf.feat_off[ch], S, win, mptr, mbin, mw,
                 lf.tw, lf.log_floor, xw + g * kFrame, fft + g * PLM::PADDED, lf.feat, t);
  }
}

size_t mix_logmel_smem() {
  return sizeof(float) * (kTileBuf + kFramesPerCta * kFrame) + sizeof(float2) * kFramesPerCta * PLM::PADDED +
         sizeof(float) * (kFrame + kMaxNnz) + sizeof(int) * (kMels + 1) + sizeof(short) * kMaxNnz + 16;
}

}  // namespace

cudaError_t launch_mix_logmel(const MixArgs& a, const MixFeatArgs& lf, int64_t n_chan, int64_t max_len,
                              cudaStream_t s) {
  if (n_chan == 0 || max_len == 0) return cudaSuccess;
  const size_t smem = mix_logmel_smem();
  cudaError_t e = cudaFuncSetAttribute(mix_logmel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((max_len + kMixTile - 1) / kMixTile), static_cast<unsigned>(n_chan));
  mix_logmel_kernel<<<grid, kFramesPerCta * PLM::T, smem, s>>>(a, lf);
  return cudaGetLastError();
}

cudaError_t launch_logmel(const LogMelArgs& a, cudaStream_t s) {
  if (a.n_tiles == 0) return cudaSuccess;
  const int grid = a.n_tiles < 148 * 8 ? a.n_tiles : 148 * 8;
  logmel_kernel<<<grid, kFramesPerCta * PLM::T, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rsg

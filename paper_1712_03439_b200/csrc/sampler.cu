// sampler.cu — the scene sampler and signal generator (sampler.cuh) on the host (the
// fixture generator) and on the device, behind the C-ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/roomsim_gpu.h"
#include "sampler.cuh"

namespace rsg {
int report_error(int code, const std::string& msg);  // api.cu: sets rs_last_error()
static_assert(sizeof(SamplerSpecD) == sizeof(rs_sampler_spec), "rs_sampler_spec layout");

namespace {

const SamplerSpecD& spec_of(const rs_sampler_spec* s) { return *reinterpret_cast<const SamplerSpecD*>(s); }

__global__ void counts_kernel(SamplerSpecD sp, uint64_t seed, int64_t first, int64_t n, int64_t epoch,
                              int32_t* n_src) {
  const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (u < n) n_src[u] = 1 + sampler_num_noises(sp, seed, static_cast<uint64_t>(first + u), epoch);
}

__global__ void scenes_kernel(SamplerSpecD sp, uint64_t seed, int64_t first, int64_t n, int64_t epoch,
                              const int64_t* src_begin, double* room, double* refl, int32_t* order,
                              int64_t* horizon, double* src_pos, double* mic_pos, double* snr, int64_t* nsamp) {
  const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (u >= n) return;
  const int64_t s0 = src_begin[u];
  const int I = static_cast<int>(src_begin[u + 1] - s0);
  const SceneOut o = sampler_scene(sp, seed, static_cast<uint64_t>(first + u), epoch, I, src_pos + 3 * s0,
                                   mic_pos + 3 * u * sp.mic_count, snr + s0);
  for (int a = 0; a < 3; ++a) room[3 * u + a] = o.room[a];
  refl[u] = o.refl;
  order[u] = o.order;
  horizon[u] = o.horizon;
  nsamp[u] = o.n_samples;
}

struct SrcInfo {
  int64_t utt, off, len;
  int32_t local, pad;
};

// Persistent grid over (source, tile) work units: unit u of the flat list belongs to the
// source whose tile prefix `first_tile` brackets it (binary search, one thread per CTA); a
// tile is kSigQuads quads per thread.  (A 2-D grid sized by the longest source launched
// millions of empty CTAs for the short ones.)
constexpr int kSigThreads = 256, kSigQuads = 8;
constexpr int kSigTile = kSigQuads * kSigThreads;  // quads per tile
__global__ void __launch_bounds__(kSigThreads) signals_kernel(SamplerSpecD sp, uint64_t seed, int64_t epoch,
                                                              const SrcInfo* src, const int64_t* first_tile,
                                                              int64_t n_src, int64_t n_tiles, float* out) {
  __shared__ int64_t s_src;
  for (int64_t u = blockIdx.x; u < n_tiles; u += gridDim.x) {
    __syncthreads();  // the previous tile's s_src is consumed
    if (threadIdx.x == 0) {
      int64_t lo = 0, hi = n_src - 1;  // last source with first_tile <= u
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (first_tile[mid] <= u) lo = mid; else hi = mid - 1;
      }
      s_src = lo;
    }
    __syncthreads();
    const int64_t lo = s_src;
    const SrcInfo si = src[lo];
    const Stream g(seed ^ 0x5EED5EED5EEDull, static_cast<uint64_t>(si.utt), static_cast<uint64_t>(epoch),
                   kTagSignal + static_cast<uint32_t>(si.local));
    const int64_t nquads = (si.len + 3) / 4;
    float* o = out + si.off;
    const bool al16 = (reinterpret_cast<uintptr_t>(o) & 15u) == 0;
    const int64_t tile = u - first_tile[lo];
#pragma unroll 1
    for (int k = 0; k < kSigQuads; ++k) {
      const int64_t q = (tile * kSigQuads + k) * kSigThreads + threadIdx.x;
      if (q >= nquads) break;
      float z[4];
      signal_quad(sp, g, static_cast<uint64_t>(q), z);
      if (al16 && 4 * q + 3 < si.len) {
        *reinterpret_cast<float4*>(o + 4 * q) = make_float4(z[0], z[1], z[2], z[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * q + i < si.len) o[4 * q + i] = z[i];
      }
    }
  }
}

int sfail(int code, const std::string& m) { return report_error(code, m); }

int check_spec(const rs_sampler_spec* s) {
  if (!s) return sfail(RS_ERR_CONFIG, "null sampler spec");
  for (int a = 0; a < 3; ++a)
    if (!(s->dim_lo[a] > 0.0) || s->dim_hi[a] < s->dim_lo[a] ||
        s->dim_lo[a] - 2.0 * s->clearance <= 0.0)
      return sfail(RS_ERR_CONFIG, "room ranges incompatible with the wall clearance");
  if (s->n_weights < 0 || s->n_weights > 8) return sfail(RS_ERR_CONFIG, "at most 8 noise-count weights");
  double tot = 0.0;
  for (int i = 0; i < s->n_weights; ++i) {
    if (s->weights[i] < 0.0) return sfail(RS_ERR_CONFIG, "noise-count weights must be non-negative");
    tot += s->weights[i];
  }
  if (s->n_weights > 0 && !(tot > 0.0)) return sfail(RS_ERR_CONFIG, "noise-count weights all zero");
  if (s->mic_count < 1 || (s->mic_radius <= 0.0 && s->mic_count > 2))
    return sfail(RS_ERR_CONFIG, "line arrays hold 1 or 2 mics; use mic_radius > 0 for more");
  if (!(s->fs > 0.0) || !(s->c0 > 0.0)) return sfail(RS_ERR_CONFIG, "sample rate and speed of sound must be positive");
  return RS_OK;
}

}  // namespace
}  // namespace rsg

using namespace rsg;

extern "C" {

int rs_sampler_counts(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt,
                      int64_t epoch, int32_t* n_src) {
  if (int st = check_spec(spec)) return st;
  for (int64_t u = 0; u < n_utt; ++u)
    n_src[u] = 1 + sampler_num_noises(spec_of(spec), seed, static_cast<uint64_t>(first_utt + u), epoch);
  return RS_OK;
}

int rs_sample_scenes(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt, int64_t epoch,
                     const int64_t* src_begin, double* room_dims, double* reflection, int32_t* image_order,
                     int64_t* max_taps, double* src_pos, double* mic_pos, double* snr_db, int64_t* n_samples) {
  if (int st = check_spec(spec)) return st;
  const SamplerSpecD& sp = spec_of(spec);
  for (int64_t u = 0; u < n_utt; ++u) {
    const int64_t s0 = src_begin[u];
    const SceneOut o = sampler_scene(sp, seed, static_cast<uint64_t>(first_utt + u), epoch,
                                     static_cast<int>(src_begin[u + 1] - s0), src_pos + 3 * s0,
                                     mic_pos + 3 * u * sp.mic_count, snr_db + s0);
    for (int a = 0; a < 3; ++a) room_dims[3 * u + a] = o.room[a];
    reflection[u] = o.refl;
    image_order[u] = o.order;
    max_taps[u] = o.horizon;
    n_samples[u] = o.n_samples;
  }
  return RS_OK;
}

int rs_sampler_counts_device(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt,
                             int64_t epoch, int32_t* n_src_dev, void* stream) {
  if (int st = check_spec(spec)) return st;
  if (n_utt <= 0) return RS_OK;
  counts_kernel<<<static_cast<unsigned>((n_utt + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      spec_of(spec), seed, first_utt, n_utt, epoch, n_src_dev);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RS_OK : sfail(RS_ERR_CUDA, cudaGetErrorString(e));
}

int rs_sample_scenes_device(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt,
                            int64_t epoch, const int64_t* src_begin_dev, double* room_dims, double* reflection,
                            int32_t* image_order, int64_t* max_taps, double* src_pos, double* mic_pos,
                            double* snr_db, int64_t* n_samples, void* stream) {
  if (int st = check_spec(spec)) return st;
  if (n_utt <= 0) return RS_OK;
  scenes_kernel<<<static_cast<unsigned>((n_utt + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      spec_of(spec), seed, first_utt, n_utt, epoch, src_begin_dev, room_dims, reflection, image_order, max_taps,
      src_pos, mic_pos, snr_db, n_samples);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RS_OK : sfail(RS_ERR_CUDA, cudaGetErrorString(e));
}

int rs_generate_signals_host(const rs_sampler_spec* spec, uint64_t seed, int64_t epoch, int64_t n_src,
                             const int64_t* utt_of_src, const int32_t* src_local, const int64_t* sig_off,
                             const int64_t* sig_len, float* out) {
  if (int st = check_spec(spec)) return st;
  const SamplerSpecD& sp = spec_of(spec);
  for (int64_t s = 0; s < n_src; ++s) {
    const Stream g(seed ^ 0x5EED5EED5EEDull, static_cast<uint64_t>(utt_of_src[s]), static_cast<uint64_t>(epoch),
                   kTagSignal + static_cast<uint32_t>(src_local[s]));
    float* o = out + sig_off[s];
    const int64_t len = sig_len[s];
    for (int64_t q = 0; 4 * q < len; ++q) {
      float z[4];
      signal_quad(sp, g, static_cast<uint64_t>(q), z);
      for (int i = 0; i < 4; ++i)
        if (4 * q + i < len) o[4 * q + i] = z[i];
    }
  }
  return RS_OK;
}

}  // extern "C"

// A batch's per-source generator table, on the device once: every epoch's signals are then
// one kernel launch with no host work, no allocation and no synchronisation.
struct rs_signal_plan {
  SamplerSpecD spec;
  uint64_t seed = 0;
  int64_t n_src = 0, n_tiles = 0, grid = 0;
  unsigned char* d = nullptr;  // n_src SrcInfo, then the n_src tile prefixes
  size_t info_bytes = 0;
};

extern "C" {

int rs_signal_plan_create(const rs_sampler_spec* spec, uint64_t seed, int64_t n_src, const int64_t* utt_of_src,
                          const int32_t* src_local, const int64_t* sig_off, const int64_t* sig_len,
                          rs_signal_plan** out) {
  if (!out) return sfail(RS_ERR_CONFIG, "null output pointer");
  if (int st = check_spec(spec)) return st;
  auto* p = new rs_signal_plan();
  p->spec = spec_of(spec);
  p->seed = seed;
  p->n_src = n_src < 0 ? 0 : n_src;
  p->info_bytes = static_cast<size_t>(p->n_src) * sizeof(SrcInfo);
  std::vector<unsigned char> table(p->info_bytes + static_cast<size_t>(p->n_src) * sizeof(int64_t));
  SrcInfo* info = reinterpret_cast<SrcInfo*>(table.data());
  int64_t* first = reinterpret_cast<int64_t*>(table.data() + p->info_bytes);
  for (int64_t s = 0; s < p->n_src; ++s) {
    info[s] = SrcInfo{utt_of_src[s], sig_off[s], sig_len[s], src_local[s], 0};
    first[s] = p->n_tiles;
    p->n_tiles += ((sig_len[s] + 3) / 4 + kSigTile - 1) / kSigTile;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p->grid = std::min<int64_t>(p->n_tiles, static_cast<int64_t>(sms) * 8);
  cudaError_t e = cudaSuccess;
  if (!table.empty()) {
    e = cudaMalloc(reinterpret_cast<void**>(&p->d), table.size());
    if (e == cudaSuccess) e = cudaMemcpy(p->d, table.data(), table.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    if (p->d) cudaFree(p->d);
    delete p;
    return sfail(e == cudaErrorMemoryAllocation ? RS_ERR_OOM : RS_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = p;
  return RS_OK;
}

int rs_signal_plan_generate(rs_signal_plan* p, int64_t epoch, float* out_dev, void* stream) {
  if (!p) return sfail(RS_ERR_CONFIG, "null signal plan");
  if (p->n_tiles == 0) return RS_OK;
  signals_kernel<<<static_cast<unsigned>(p->grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p->spec, p->seed, epoch, reinterpret_cast<const SrcInfo*>(p->d),
      reinterpret_cast<const int64_t*>(p->d + p->info_bytes), p->n_src, p->n_tiles, out_dev);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RS_OK : sfail(RS_ERR_CUDA, cudaGetErrorString(e));
}

int rs_signal_plan_destroy(rs_signal_plan* p) {
  if (!p) return RS_OK;
  if (p->d) cudaFree(p->d);
  delete p;
  return RS_OK;
}

int rs_generate_signals(const rs_sampler_spec* spec, uint64_t seed, int64_t epoch, int64_t n_src,
                        const int64_t* utt_of_src, const int32_t* src_local, const int64_t* sig_off,
                        const int64_t* sig_len, float* out_dev, void* stream) {
  if (int st = check_spec(spec)) return st;
  if (n_src <= 0) return RS_OK;
  rs_signal_plan* p = nullptr;
  if (int st = rs_signal_plan_create(spec, seed, n_src, utt_of_src, src_local, sig_off, sig_len, &p)) return st;
  int st = rs_signal_plan_generate(p, epoch, out_dev, stream);
  const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));  // before the table is freed
  rs_signal_plan_destroy(p);
  if (st) return st;
  return e == cudaSuccess ? RS_OK : sfail(RS_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"

// api.cu — the C-ABI (include/roomsim_gpu.h) and the host-side orchestration
// of the hot path: validation with the reference's error taxonomy, the
// host-computed constants that must match glibc (r^g, 10^(-eta/10),
// 10^(snr/10)), the FFT-size planner (an exact mirror of
// roomsim/convolution.hpp:72-161), bucketing of pairs by transform size, and
// the kernel sequence K1a -> K1 -> K2 -> plan -> K3 -> K4 (with the mix in its epilogue,
// mixfin.cuh) -> K5 -> K6 (the channels the epilogue does not cover).
#include <algorithm>
#include <array>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/roomsim_gpu.h"
#include "kernels.cuh"
#include "mixfin.cuh"
#include "power.cuh"

using namespace rsg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

// error reporting shared with the other translation units (sampler.cu)
namespace rsg {
int report_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace rsg

namespace {

#define RS_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? RS_ERR_OOM : RS_ERR_CUDA,          \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

#define RS_TRY(call)              \
  do {                            \
    int st_ = (call);             \
    if (st_ != RS_OK) return st_; \
  } while (0)

// NVTX range over a host phase of the render (nsys / ncu timelines; header-only NVTX3, a no-op
// without a profiler attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Device buffer that only grows (the ctx's arena).
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return RS_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    want = want + want / 8;  // headroom so slowly growing batches do not thrash
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      e = cudaMalloc(&p, bytes);
      want = bytes;
    }
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(RS_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    cap = want;
    return RS_OK;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Page-locked host staging (bump allocator) so H2D/D2H copies are truly async.
struct PinnedArena {
  char* p = nullptr;
  char* dp = nullptr;
  size_t cap = 0, used = 0;
  int reserve(size_t bytes) {  // only call while no copy from this arena is pending
    if (bytes <= cap) return RS_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = bytes + bytes / 4 + 4096;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), want, cudaHostAllocMapped);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(RS_ERR_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    cap = want;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), p, 0);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, std::string("cudaHostGetDevicePointer: ") + cudaGetErrorString(e));
    return RS_OK;
  }
  void reset() { used = 0; }
  // device-side alias of a pointer into this arena (mapped pinned memory)
  template <class T>
  T* dev(T* h) const { return reinterpret_cast<T*>(dp + (reinterpret_cast<char*>(h) - p)); }
  template <class T>
  T* alloc(size_t n) {
    used = (used + 63) & ~size_t(63);
    T* r = reinterpret_cast<T*>(p + used);
    used += std::max<size_t>(n, 1) * sizeof(T);
    return used <= cap ? r : nullptr;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

template <class T>
size_t staged_bytes(const std::vector<T>& v) { return ((std::max<size_t>(v.size(), 1) * sizeof(T) + 63) & ~size_t(63)) + 64; }

size_t bit_ceil_sz(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
bool has_single_bit(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
int log2_exact(size_t n) {
  int l = 0;
  while ((static_cast<size_t>(1) << l) < n) ++l;
  return l;
}

// ---- planner: exact mirror of roomsim/convolution.hpp:72-161 ----------------
int cost_validate(double I, double J, size_t nx, size_t nh) {
  if (I <= 0.0 || J <= 0.0) return fail(RS_ERR_CONFIG, "source and mic counts must be positive");
  if (nx == 0 || nh == 0) return fail(RS_ERR_CONFIG, "signal and RIR lengths must be positive");
  return RS_OK;
}
int checked_fft_size(size_t n, size_t min_legal, const char* what) {
  if (n < 2 || !has_single_bit(n))
    return fail(RS_ERR_PLAN, std::string(what) + ": FFT size must be a power of two >= 2");
  if (n < min_legal) return fail(RS_ERR_PLAN, std::string(what) + ": FFT size too small for this workload");
  return RS_OK;
}
size_t fft_size_for(size_t n) { return bit_ceil_sz(std::max<size_t>(n, 2)); }  // :82-84
size_t block_count(size_t nx, size_t nh, size_t n) {                           // :108-112
  const size_t L = n - nh + 1;
  return (nx + L - 1) / L;
}
double cost_ola_raw(double I, double J, size_t nx, size_t nh, size_t n) {  // :119-127
  const double nd = static_cast<double>(n);
  const double blocks = static_cast<double>(block_count(nx, nh, n));
  return I * J * (blocks * (4.0 * nd * std::log2(nd) + 2.0 * nd) + 2.0 * nd * std::log2(nd));
}
double cost_full_raw(double I, double J, size_t n) {  // :100-105
  const double nd = static_cast<double>(n);
  return I * J * (6.0 * nd * std::log2(nd) + 2.0 * nd);
}
int plan_for_impl(double I, double J, size_t nx, size_t nh, int strategy, int* s, size_t* n,
                  double* c) {
  RS_TRY(cost_validate(I, J, nx, nh));
  switch (strategy) {
    case RS_DIRECT:
      *s = RS_DIRECT;
      *n = 0;
      *c = I * J * static_cast<double>(nx) * static_cast<double>(nh);
      return RS_OK;
    case RS_FULL_FFT: {
      const size_t nn = fft_size_for(nx + nh - 1);
      *s = RS_FULL_FFT;
      *n = nn;
      *c = cost_full_raw(I, J, nn);
      return RS_OK;
    }
    case RS_OVERLAP_ADD: {
      const size_t n_max = fft_size_for(nx + nh - 1);
      double best = std::numeric_limits<double>::infinity();
      size_t best_n = 0;
      for (size_t nn = fft_size_for(nh); nn <= n_max; nn <<= 1) {
        const double cc = cost_ola_raw(I, J, nx, nh, nn);
        if (cc < best) {
          best = cc;
          best_n = nn;
        }
      }
      *s = RS_OVERLAP_ADD;
      *n = best_n;
      *c = best;
      return RS_OK;
    }
  }
  return fail(RS_ERR_PLAN, "unknown strategy");
}
int choose_plan_impl(double I, double J, size_t nx, size_t nh, int* s, size_t* n, double* c) {
  int s1, s2;
  size_t n1, n2;
  double c1, c2;
  RS_TRY(plan_for_impl(I, J, nx, nh, RS_OVERLAP_ADD, &s1, &n1, &c1));
  RS_TRY(plan_for_impl(I, J, nx, nh, RS_FULL_FFT, &s2, &n2, &c2));
  if (c2 < c1) {
    *s = s2; *n = n2; *c = c2;
  } else {
    *s = s1; *n = n1; *c = c1;
  }
  return RS_OK;
}

// Host loops over utterances / pairs on a few threads (OpenMP; the planner's glibc pow and
// exact lattice maxima would otherwise keep the first chunk's kernels waiting).  Every
// iteration writes only its own slots, so the result does not depend on the thread count.
template <class F>
void host_parallel_for(int64_t n, F&& f, int64_t min_n = 64) {
  static const int nthr = [] {
    const char* e = std::getenv("RSG_HOST_THREADS");
    int v = e ? std::atoi(e) : 8;
    return std::max(1, v);
  }();
  if (n < min_n || nthr == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
#pragma omp parallel for num_threads(nthr) schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) f(i);
}

// Exact max over the image lattice of ceil(|image - mic| * fs/c0): the squared
// distance is a sum of per-axis terms and every rounded operation on the way
// (fl(x*x), fl(a+b), sqrt, fl(d*spm), ceil) is monotone, so the maximum is the
// one of the per-axis maxima (room_model.hpp:126-127, :42-44, :159-160).
uint64_t lattice_max_delay(const double* L, const double* s, const double* m, int K, double spm) {
  double mx[3];
  for (int a = 0; a < 3; ++a) {
    double best = 0.0;
    for (int n = -K; n <= K; ++n) {
      const double mirrored = (n % 2 == 0) ? s[a] : L[a] - s[a];
      const double pos = static_cast<double>(n) * L[a] + mirrored;
      const double diff = pos - m[a];
      const double sq = diff * diff;
      best = sq > best ? sq : best;
    }
    mx[a] = best;
  }
  return static_cast<uint64_t>(std::ceil(std::sqrt(mx[0] + mx[1] + mx[2]) * spm));
}

// RoomConfig::validate, room_model.hpp:57-65
int room_validate(const double* L, double r, double fs, double c0, int order) {
  if (L[0] <= 0.0 || L[1] <= 0.0 || L[2] <= 0.0) return fail(RS_ERR_CONFIG, "room dimensions must be positive");
  if (r <= 0.0 || r >= 1.0) return fail(RS_ERR_CONFIG, "reflection coefficient must lie in (0, 1)");
  if (fs <= 0.0) return fail(RS_ERR_CONFIG, "sample rate must be positive");
  if (c0 <= 0.0) return fail(RS_ERR_CONFIG, "speed of sound must be positive");
  if (order < 0) return fail(RS_ERR_CONFIG, "image order must be non-negative");
  return RS_OK;
}
bool strictly_inside(const double* L, const double* p) {  // room_model.hpp:79-84
  for (int a = 0; a < 3; ++a)
    if (!(p[a] > 0.0 && p[a] < L[a])) return false;
  return true;
}

}  // namespace

// ============================================================================
// Context
// ============================================================================
struct rs_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // stage boundaries of the last render: begin, synth, cut, plan, spectrum, ola, end
  static constexpr int kStages = 7;
  cudaEvent_t st[kStages] = {};
  bool st_valid = false;
  double host_plan_ms = 0;
  double stage_ms[6] = {};
  bool stage_valid = false;
  float2* tw[kMaxLog2M + 1] = {};
  float2* tw2f[kOla2MaxLog2N + 1] = {};  // two-stream K4: forward / reversed pass tables
  float2* tw2i[kOla2MaxLog2N + 1] = {};
  DevBuf tw_all;
  // arena
  DevBuf utt, pair, rg, items, olaitems, rir, rirout, plan, lists, spec, y, sumsq, gain, power, flags,
      snr, chan_utt, chan_mic, chan_out, utt_len, utt_stride, utt_pair0, utt_I, utt_J, sig, out,
      scratch_a, scratch_b;
  struct rs_render_state* rs = nullptr;
  // last render (debug fetch)
  std::vector<PairPlan> h_plan;
  std::vector<PairMeta> h_pair;
  std::vector<PairRir> h_rir;
  int64_t last_pairs = 0;
  // timing of the last render
  double ola_ms = 0, ola_flops = 0, alg_bytes = 0;
  int64_t launches = 0;
  int fused_mix = -1;  // rs_ctx_set_fused_mix: 1 / 0, -1 = the process default (RSG_FUSED_MIX)
  int64_t fused_channels = 0, mixed_channels = 0;  // last render: channels mixed by the K4 epilogue / all
  // side streams: the per-size K4 launches of a chunk run concurrently (fills each
  // launch's tail with another size's CTAs)
  // K4 side streams: two lanes of kSide (consecutive render chunks alternate lanes, so a chunk's
  // K4 launches do not queue behind the previous chunk's and fill its tail)
  static constexpr int kSide = 4, kLanes = 2;
  cudaStream_t side[kLanes * kSide] = {};
  cudaEvent_t side_fork[kLanes] = {}, side_join[kLanes * kSide] = {};
  // log-Mel front end tables (built on first use)
  DevBuf lm_window, lm_ptr, lm_bin, lm_w, lm_tiles;
  bool lm_ready = false;
  // profiling level 2: K4 launches serialized on the filter stream, one event pair per
  // (size, variant) span; rows of the last render, merged by (log2 N, variant)
  int prof_level = 0;
  struct K4Span { int log2n, var; int64_t pairs; double flops, exec_flops; cudaEvent_t a, b; };
  std::vector<K4Span> k4_spans;      // this render's spans (events pending)
  std::vector<cudaEvent_t> ev_pool;  // reusable events
  size_t ev_used = 0;
  struct K4Row { int log2n, var; int64_t pairs; double flops, ms, exec_flops; };
  std::vector<K4Row> k4_rows;
  cudaEvent_t pool_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
};

namespace {

int ctx_init(rs_ctx* c) {
  RS_CUDA(cudaSetDevice(c->device));
  RS_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  RS_CUDA(cudaEventCreate(&c->ev0));
  RS_CUDA(cudaEventCreate(&c->ev1));
  for (auto& e : c->st) RS_CUDA(cudaEventCreate(&e));
  for (int i = 0; i < rs_ctx::kLanes * rs_ctx::kSide; ++i) {
    RS_CUDA(cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking));
    RS_CUDA(cudaEventCreateWithFlags(&c->side_join[i], cudaEventDisableTiming));
  }
  for (auto& e : c->side_fork) RS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RS_CUDA(kernels_init());
  size_t total = 0;
  size_t off[kMaxLog2M + 1], off2[kOla2MaxLog2N + 1][2] = {};
  for (int l = 0; l <= kMaxLog2M; ++l) {
    off[l] = total;
    total += (static_cast<size_t>(tw_total(l)) + 1) & ~size_t(1);
  }
  for (int l = kOla2MinLog2N; l <= kOla2MaxLog2N; ++l)
    for (int r = 0; r < 2; ++r) {
      off2[l][r] = total;
      total += (static_cast<size_t>(ola2_tw_total(l, r == 1)) + 1) & ~size_t(1);
    }
  std::vector<float2> h(total);
  for (int l = 0; l <= kMaxLog2M; ++l) fill_twiddles(l, h.data() + off[l]);
  for (int l = kOla2MinLog2N; l <= kOla2MaxLog2N; ++l)
    for (int r = 0; r < 2; ++r) ola2_fill_twiddles(l, r == 1, h.data() + off2[l][r]);
  RS_TRY(c->tw_all.ensure(total * sizeof(float2)));
  RS_CUDA(cudaMemcpy(c->tw_all.p, h.data(), total * sizeof(float2), cudaMemcpyHostToDevice));
  for (int l = 0; l <= kMaxLog2M; ++l) c->tw[l] = c->tw_all.as<float2>() + off[l];
  for (int l = kOla2MinLog2N; l <= kOla2MaxLog2N; ++l) {
    c->tw2f[l] = c->tw_all.as<float2>() + off2[l][0];
    c->tw2i[l] = c->tw_all.as<float2>() + off2[l][1];
  }
  return RS_OK;
}

template <class T>
int upload(rs_ctx* c, DevBuf& b, const std::vector<T>& v) {
  RS_TRY(b.ensure(std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (!v.empty())
    RS_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return RS_OK;
}

// Work of one pair in the metric's units: (2B+1) 5 N log2 N.
double pair_flops(const PairPlan& p) {
  const double n = std::ldexp(1.0, p.log2n);
  return (2.0 * static_cast<double>(p.B) + 1.0) * 5.0 * n * p.log2n;
}

// ---- stage B: spectrum + OLA over planned pairs --------------------------------
// Every pair's K4 variant is a function of its own (N, N_h) only (so are its power
// partials, power.cuh): a pair renders to the same bytes whatever else shares its chunk.
// Pairs are bucketed by (transform size, variant); buckets run largest work first.
// Each pair's blocks are split into runs (K4 work items) long enough that the
// recomputed overlap blocks cost <= ~6%, short enough to fill the GPU.
enum K4Variant { kVarSmall = 0, kVarIp = 1, kVarOla2 = 2, kVarLarge = 3, kVarIpc = 4, kVarCount = 5 };

struct Span {
  int l;
  int var;
  int64_t list_off, list_n, item_off, item_n;
  int64_t max_nh = 1;  // largest N_h of the span (in-place / two-stream carry size)
  int64_t max_l = 1;   // largest L of the span (two-stream input window)
  int seg = kPowerSeg; // OLA blocks per power segment
};

// A batch of one large span (four-step path): pairs [pair_lo, pair_hi) of the
// span's list, their (pair, block) units [unit_lo, unit_hi) and stage-D items
// [item_lo, item_hi) (global indices); the batch's units share one scratch.
struct LargeBatch { int span; int64_t pair_lo, pair_hi, unit_lo, unit_hi, item_lo, item_hi; };

struct FilterPlan {
  std::vector<int32_t> lists;
  std::vector<OlaItem> items;
  std::vector<Span> spans;
  std::vector<OlaItem2> items2;     // two-stream spans
  std::vector<int2> units;          // large spans: (pair, block)
  std::vector<LargeBatch> batches;
  int64_t max_scratch = 0;          // complex elements of the largest batch's scratch
  int64_t spec_total = 0, y_total = 0, part_total = 0;
  double flops = 0;
  // per pair: the metric's flops, (2B+1) 5 N log2 N of the REFERENCE plan (filled by the caller
  // when the executed block size differs from it; otherwise by plan_filter from the plans)
  std::vector<double> alg;
};

// Sizes that take the four-step path: every M > 16384 (and M = 8192 / 16384 pairs whose
// overlap carry does not fit next to the in-place transform).  Tuning override
// RSG_LARGE_MIN = smallest log2 M.
bool use_large(int l) {
  static const int v = [] {
    const char* e = std::getenv("RSG_LARGE_MIN");
    return e ? std::atoi(e) : -1;
  }();
  static const bool ip_force = std::getenv("RSG_IP_FORCE") != nullptr;
  static_cast<void>(ip_force);
  if (l > kMaxLog2M) return true;
  if (v >= 0) return l >= v;
  return false;
}
// Largest N_h whose overlap carry fits next to the in-place K4's transform (0: none).
int64_t ip_max_nh(int l) {
  // (a function-local static's initializer runs once, thread-safe: renders may run in several
  // host threads, one context each)
  static const std::array<int64_t, kMaxLog2M + 1> cache = [] {
    std::array<int64_t, kMaxLog2M + 1> c{};
    for (int k = 0; k <= kMaxLog2M; ++k) {
      int64_t lo = 0, hi = int64_t(2) << k;  // N_h <= N
      while (lo < hi) {  // largest nh with ip_supported(k, nh)
        const int64_t mid = (lo + hi + 1) / 2;
        if (ip_supported(k, mid)) lo = mid; else hi = mid - 1;
      }
      c[k] = lo;
    }
    return c;
  }();
  return l >= 0 && l <= kMaxLog2M ? cache[l] : 0;
}
// Sizes (log2 M) that take the in-place one-CTA K4 (big.cu) when the pair's carry fits in
// shared memory (tuning override RSG_IP="lo,hi"; "0,0" disables it).
bool use_ip(int l, int64_t nh) {
  static const std::pair<int, int> r = [] {
    const char* e = std::getenv("RSG_IP");
    int lo = 10, hi = 14;
    if (e) std::sscanf(e, "%d,%d", &lo, &hi);
    return std::make_pair(lo, hi);
  }();
  return l >= r.first && l <= r.second && nh <= ip_max_nh(l);
}
// Real FFT sizes (log2 N) that run the two-stream K4 (tuning override RSG_OLA2="lo,hi";
// "0,0" disables it).
bool use_ola2(int log2n) {
  static const std::pair<int, int> r = [] {
    const char* e = std::getenv("RSG_OLA2");
    int lo = -1, hi = -1;
    if (e) std::sscanf(e, "%d,%d", &lo, &hi);
    return std::make_pair(lo, hi);
  }();
  if (!ola2_supported(log2n)) return false;
  if (r.first >= 0) return log2n >= r.first && log2n <= r.second;
  // default: the size where it measured faster than K4 inside the config-4 render
  // (ncu launch list, B200); elsewhere K4 is as fast or faster
  return log2n == 8;
}
// Real FFT sizes (log2 N) that run two blocks per complex transform (ola_ipc_kernel, big.cu)
// when the pair's carry fits next to the transform (tuning override RSG_IPC="lo,hi"; "0,0"
// disables it).
bool use_ipc(int log2n, int64_t nh) {
  static const std::pair<int, int> r = [] {
    const char* e = std::getenv("RSG_IPC");
    int lo = 12, hi = 13;
    if (e) std::sscanf(e, "%d,%d", &lo, &hi);
    return std::make_pair(lo, hi);
  }();
  if (log2n < r.first || log2n > r.second) return false;
  static const std::array<int64_t, kLargeMaxLog2M + 2> cache = [] {
    std::array<int64_t, kLargeMaxLog2M + 2> c{};
    for (int k = 0; k <= kLargeMaxLog2M + 1; ++k) {
      int64_t lo = 0, hi = int64_t(1) << k;  // largest nh with ipc_supported(k, nh)
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (ipc_supported(k, mid)) lo = mid; else hi = mid - 1;
      }
      c[k] = lo;
    }
    return c;
  }();
  return nh <= cache[log2n];
}
constexpr int kSmallMaxLog2MHost = 12;  // ola_small_kernel<M> sizes (kernels.cu)
int k4_variant(int l, int64_t nh) {
  if (use_large(l)) return kVarLarge;
  if (use_ola2(l + 1)) return kVarOla2;
  if (use_ipc(l + 1, nh)) return kVarIpc;
  if (use_ip(l, nh)) return kVarIp;
  if (l <= kSmallMaxLog2MHost) return kVarSmall;
  return kVarLarge;  // M >= 8192 whose overlap carry does not fit in shared memory
}

// ---- executed block size ("re-blocking") ------------------------------------------
// A pair's output is the linear convolution x * h whatever block size the overlap-add runs
// at; the reference's plan (N, L, B) is what the API reports (bit-exact), the block size
// the device EXECUTES is chosen per pair to minimise its modelled K4 time:
//   (2 B(N') + 1) N' log2 N' / eff(N'),   B(N') = ceil(N_x / (N' - N_h + 1)),
// eff(N') the measured fraction of the FP32 roofline of the kernel that runs size N'
// (B200, config-4 render, bench.py by_size).  With the reference's N = bit_ceil(2 N_h) a
// block yields L in (N/2, 3N/4] new samples per N-point transform pair; at N' = 4096 /
// 8192 the short filters yield ~0.9 N' and run on the kernels with the best fractions.
// The choice depends on the pair's (N_x, N_h) only (render invariance).
// Forced plans (RS_PLAN_FORCED: the caller names the FFT size) execute as given.
// RSG_REBLOCK=0 executes the reference's plan everywhere; RSG_REBLOCK_EFF="l=e,l=e" overrides eff.
struct ReblockCfg {
  bool on = true;
  double eff[kLargeMaxLog2M + 2];
};
const ReblockCfg& reblock_cfg() {
  static const ReblockCfg cfg = [] {
    ReblockCfg c;
    for (double& e : c.eff) e = 0.12;  // four-step sizes
    //            N =   2     4     8     16    32     64     128    256   512   1024  2048   4096   8192  16384 32768
    const double m[] = {0.01, 0.01, 0.01, 0.02, 0.075, 0.117, 0.194, 0.24, 0.40, 0.46, 0.50, 0.66, 0.63, 0.50, 0.56};
    for (int l = 1; l <= 15; ++l) c.eff[l] = m[l - 1];
    if (const char* e = std::getenv("RSG_REBLOCK")) c.on = std::atoi(e) != 0;
    if (const char* e = std::getenv("RSG_REBLOCK_EFF")) {
      int l = 0, used = 0;
      double v = 0;
      while (std::sscanf(e, "%d=%lf%n", &l, &v, &used) == 2) {
        if (l >= 1 && l <= kLargeMaxLog2M + 1 && v > 0) c.eff[l] = v;
        e += used;
        if (*e == ',') ++e;
      }
    }
    return c;
  }();
  return cfg;
}
// log2 of the executed FFT size of a pair whose reference plan is 2^ref_log2n.
int exec_log2n(size_t nx, size_t nh, int ref_log2n) {
  const ReblockCfg& c = reblock_cfg();
  if (!c.on) return ref_log2n;
  int lmin = 1;
  while ((size_t(1) << lmin) < nh) ++lmin;  // N' >= N_h: L >= 1
  const int lmax = std::max(13, std::min(ref_log2n, kLargeMaxLog2M + 1));
  int best = ref_log2n;
  double best_cost = -1;
  for (int l = lmin; l <= lmax; ++l) {
    const size_t n = size_t(1) << l;
    const double blocks = static_cast<double>(block_count(nx, nh, n));
    const double eff = k4_variant(l - 1, static_cast<int64_t>(nh)) == kVarLarge ? c.eff[kLargeMaxLog2M + 1] : c.eff[l];
    const double cost = (2.0 * blocks + 1.0) * static_cast<double>(n) * l / eff;
    if (best_cost < 0 || cost < best_cost) {
      best = l;
      best_cost = cost;
    }
  }
  return best;
}

constexpr int64_t kLargeScratchBytes = int64_t(1) << 31;  // per batch (16 M bytes per unit)

// float2 entries of a pair's filter region: M + 1 bins, or all N in ola_ipc_kernel's order.
int64_t spec_len(int log2n, int64_t nh) {
  const int64_t n = int64_t(1) << log2n;
  return k4_variant(log2n - 1, nh) == kVarIpc ? n : n / 2 + 1;
}

// Blocks before a run start whose tails overlap it: ceil((N_h - 1) / L).
int64_t pre_blocks(const PairPlan& p) {
  const int64_t n = int64_t(1) << p.log2n;
  return (n - p.L + p.L - 1) / p.L;
}

int plan_filter(std::vector<PairPlan>& plans, FilterPlan& fp) {
  const int64_t n_pairs = static_cast<int64_t>(plans.size());
  constexpr int NB = (kLargeMaxLog2M + 1) * kVarCount;
  std::vector<std::vector<int32_t>> bucket(NB);
  std::vector<double> work(n_pairs);
  fp.flops = 0;
  const bool have_alg = static_cast<int64_t>(fp.alg.size()) == n_pairs;
  if (!have_alg) fp.alg.assign(n_pairs, 0.0);
  for (int64_t p = 0; p < n_pairs; ++p) {
    const int l = plans[p].log2n - 1;
    if (l < 0 || l > kLargeMaxLog2M) return fail(RS_ERR_UNSUPPORTED, "FFT size outside the supported range");
    bucket[l * kVarCount + k4_variant(l, plans[p].nh)].push_back(static_cast<int32_t>(p));
    work[p] = pair_flops(plans[p]);  // executed plan: scheduling weight
    if (!have_alg) fp.alg[p] = work[p];
    fp.flops += fp.alg[p];
  }
  // largest pairs first (LPT) within every one-CTA bucket so each launch's tail is short; the
  // order is scheduling only (a pair's bytes do not depend on it), sorted on host threads
  host_parallel_for(NB, [&](int64_t key) {
    if (key % kVarCount != kVarLarge && bucket[key].size() > 1)
      std::stable_sort(bucket[key].begin(), bucket[key].end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
  }, 1);
  std::vector<int> order(NB);
  std::iota(order.begin(), order.end(), 0);
  std::vector<double> bucket_work(NB, 0.0);
  for (int k = 0; k < NB; ++k)
    for (int32_t p : bucket[k]) bucket_work[k] += work[p];
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return bucket_work[a] > bucket_work[b]; });
  fp.lists.clear();
  fp.items.clear();
  fp.spans.clear();
  fp.units.clear();
  fp.items2.clear();
  fp.batches.clear();
  fp.max_scratch = 0;
  int64_t part_acc = 0;
  for (int key : order) {
    auto& v = bucket[key];
    if (v.empty()) continue;
    const int l = key / kVarCount, var = key % kVarCount;
    Span sp{l, var, static_cast<int64_t>(fp.lists.size()), static_cast<int64_t>(v.size()), 0, 0};
    int64_t total_blocks = 0, max_pre = 1;
    for (int32_t p : v) {
      sp.max_nh = std::max<int64_t>(sp.max_nh, plans[p].nh);
      sp.max_l = std::max<int64_t>(sp.max_l, plans[p].L);
      total_blocks += plans[p].B;
      max_pre = std::max<int64_t>(max_pre, pre_blocks(plans[p]));
    }
    if (var == kVarLarge) {  // four-step path, batched by scratch size
      sp.item_off = static_cast<int64_t>(fp.items.size());
      const int64_t m = int64_t(1) << l;
      const int64_t per_batch = std::max<int64_t>(1, kLargeScratchBytes / (16 * m));
      LargeBatch bt{static_cast<int>(fp.spans.size()), 0, 0, static_cast<int64_t>(fp.units.size()), 0,
                    static_cast<int64_t>(fp.items.size()), 0};
      auto close = [&](int64_t i) {
        bt.pair_hi = i;
        bt.unit_hi = static_cast<int64_t>(fp.units.size());
        bt.item_hi = static_cast<int64_t>(fp.items.size());
        if (bt.pair_hi > bt.pair_lo) {
          fp.batches.push_back(bt);
          fp.max_scratch = std::max(fp.max_scratch, (bt.unit_hi - bt.unit_lo) * m);
        }
        bt.pair_lo = i;
        bt.unit_lo = bt.unit_hi;
        bt.item_lo = bt.item_hi;
      };
      for (int64_t i = 0; i < static_cast<int64_t>(v.size()); ++i) {
        PairPlan& pl = plans[v[i]];
        if (static_cast<int64_t>(fp.units.size()) - bt.unit_lo + pl.B > per_batch) close(i);
        const int64_t unit0 = static_cast<int64_t>(fp.units.size()) - bt.unit_lo;
        for (int64_t b = 0; b < pl.B; ++b) fp.units.push_back(make_int2(v[i], static_cast<int>(b)));
        const int64_t tiles = (pl.out_len + large_tile() - 1) / large_tile();
        pl.part0 = part_acc;
        pl.npart = static_cast<int32_t>(tiles);
        part_acc += tiles;
        for (int64_t tl = 0; tl < tiles; ++tl)
          fp.items.push_back(OlaItem{v[i], static_cast<int32_t>(tl), static_cast<int32_t>(unit0), 0});
      }
      close(static_cast<int64_t>(v.size()));
      sp.item_n = static_cast<int64_t>(fp.items.size()) - sp.item_off;
      fp.spans.push_back(sp);
      fp.lists.insert(fp.lists.end(), v.begin(), v.end());
      continue;
    }
    if (var == kVarOla2) {  // two-stream K4: an item is a pair of runs of one pair
      // Runs of a fixed length per pair (16 overlap blocks' worth, whole power segments): the
      // two runs sharing a complex transform round into each other, so which blocks pair
      // up must not depend on the rest of the chunk.
      sp.item_off = static_cast<int64_t>(fp.items2.size());
      const int ppb = ola2_parts_per_block(l + 1);
      for (int32_t p : v) {
        PairPlan& pl = plans[p];
        const int64_t pre = pre_blocks(pl);
        const int64_t len = kPowerSeg * std::max<int64_t>(pre, 1);  // 16 overlap blocks' worth, whole segments
        int64_t nr = (pl.B + len - 1) / len;
        if (nr > 1 && (nr & 1)) ++nr;  // an even number of runs: two per item (the last may be empty)
        pl.part0 = part_acc;
        pl.npart = static_cast<int32_t>(power_segments(pl.B) * ppb);
        part_acc += pl.npart;
        for (int64_t r = 0; r < nr; r += 2) {
          OlaItem2 it{p, 0, 0, 0, static_cast<int32_t>(pl.B), static_cast<int32_t>(pl.B),
                      static_cast<int32_t>(pl.B), 0};
          for (int h = 0; h < 2 && r + h < nr; ++h) {
            const int64_t r0 = std::min<int64_t>(pl.B, (r + h) * len), r1 = std::min<int64_t>(pl.B, r0 + len);
            if (r0 >= r1) continue;  // empty run: stays (B, B, B), no trips, owns nothing
            const int32_t b0 = static_cast<int32_t>(r0 == 0 ? 0 : std::max<int64_t>(0, r0 - pre));
            if (h == 0) {
              it.a_begin = b0; it.a_own = static_cast<int32_t>(r0); it.a_end = static_cast<int32_t>(r1);
            } else {
              it.b_begin = b0; it.b_own = static_cast<int32_t>(r0); it.b_end = static_cast<int32_t>(r1);
            }
          }
          fp.items2.push_back(it);
        }
      }
      sp.item_n = static_cast<int64_t>(fp.items2.size()) - sp.item_off;
      fp.spans.push_back(sp);
      fp.lists.insert(fp.lists.end(), v.begin(), v.end());
      continue;
    }
    const bool ipc = var == kVarIpc;
    const bool ip = var == kVarIp || ipc;
    const int64_t slots = 148LL * (ipc ? ipc_resident(l + 1, sp.max_nh)
                                       : (ip ? ip_resident(l, sp.max_nh) : ola_resident_groups(l)));
    // work items per resident slot (measured, config 4): the in-place K4 prefers long runs
    // (each item stages its filter and twiddles), ola_small<512> too, the M <= 256 sizes
    // more items (shorter tails)
    static const int64_t run_div_env = [] {
      const char* e = std::getenv("RSG_RUN_DIV");  // tuning override
      return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(0);
    }();
    const int64_t run_div = run_div_env ? run_div_env : (ip ? 2 : (l <= 8 ? 12 : 3));
    // the in-place K4 at M >= 8192: a few long blocks per pair — 2-block power segments and
    // runs down to 2 (pre-)blocks, so even a small bucket fills the SMs (each run recomputes
    // its overlap blocks: up to half the work of a 2-block run, paid only where it buys CTAs)
    const int seg = (ip && !ipc && l >= 13) ? kPowerSegLarge : kPowerSeg;
    const int64_t min_run = (ip && !ipc && l >= 13) ? 2 * max_pre : 16 * max_pre;
    int64_t run = std::max<int64_t>((total_blocks + run_div * slots - 1) / (run_div * slots), min_run);
    run = (run + seg - 1) / seg * seg;  // runs start on power-segment boundaries
    sp.seg = seg;
    const int ppb = ipc ? ipc_parts_per_block(l + 1) : (ip ? ip_parts_per_block(l) : small_parts_per_block(l));
    sp.item_off = static_cast<int64_t>(fp.items.size());
    for (int32_t p : v) {
      PairPlan& pl = plans[p];
      const int64_t pre = pre_blocks(pl);
      pl.part0 = part_acc;
      pl.npart = static_cast<int32_t>(power_segments(pl.B, seg) * ppb);
      part_acc += pl.npart;
      for (int64_t r0 = 0; r0 < pl.B; r0 += run) {
        const int64_t r1 = std::min<int64_t>(pl.B, r0 + run);
        int64_t b0 = r0 == 0 ? 0 : std::max<int64_t>(0, r0 - pre);
        if (ipc) b0 &= ~int64_t(1);  // blocks 2j and 2j + 1 always share a transform
        fp.items.push_back(OlaItem{p, static_cast<int32_t>(b0), static_cast<int32_t>(r0), static_cast<int32_t>(r1)});
      }
    }
    sp.item_n = static_cast<int64_t>(fp.items.size()) - sp.item_off;
    fp.spans.push_back(sp);
    fp.lists.insert(fp.lists.end(), v.begin(), v.end());
  }
  fp.part_total = part_acc;
  fp.spec_total = fp.y_total = 0;
  for (const auto& q : plans) {
    fp.spec_total = std::max<int64_t>(fp.spec_total, q.spec_off + spec_len(q.log2n, q.nh));
    fp.y_total = std::max<int64_t>(fp.y_total, q.y_off + ((q.out_len + 3) & ~int64_t(3)));  // rows padded to whole quads
  }
  return RS_OK;
}

// Device buffers of one filter stage (K3 + K4 + K5 + K6 of a chunk).
struct FilterBufs {
  DevBuf plan, lists, olaitems, spec, y, part, units, scratch, yblk, olaitems2;
};

thread_local int64_t g_copy_launches = 0;  // pcie_copy_kernel launches of the current render
// Host-buffer renders move metadata with pcie_copy_kernel (the copy engines are busy
// with signal/output transfers and serve copies in FIFO order); device-buffer renders
// keep the copy engines, which are otherwise idle.
thread_local bool g_kernel_copies = false;

// Small pinned-host <-> device copy on `st` by the path chosen above.
int small_copy(void* dst, void* dst_mapped, const void* src, const void* src_mapped, size_t bytes,
               cudaMemcpyKind kind, cudaStream_t st) {
  if (bytes == 0) return RS_OK;
  if (g_kernel_copies) {
    RS_CUDA(launch_pcie_copy(dst_mapped, src_mapped, bytes, st));
    ++g_copy_launches;
  } else {
    RS_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, st));
  }
  return RS_OK;
}

// Async H2D of a host vector through a pinned arena (or synchronously staged
// pageable memory when `arena` is null).
template <class T>
int upload_on(DevBuf& b, const std::vector<T>& v, cudaStream_t st, PinnedArena* arena) {
  RS_TRY(b.ensure(std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (v.empty()) return RS_OK;
  const void* src = v.data();
  if (arena) {
    T* h = arena->alloc<T>(v.size());
    if (!h) return fail(RS_ERR_OOM, "pinned staging arena exhausted");
    std::memcpy(h, v.data(), v.size() * sizeof(T));
    return small_copy(b.p, b.p, h, arena->dev(h), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
  }
  RS_CUDA(cudaMemcpyAsync(b.p, src, v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return RS_OK;
}

// K4 variants whose work items run the mix epilogue (mixfin.cuh): the one-CTA-per-item kernels
// of big.cu.  A channel with a pair on another variant is mixed by mix_kernel.
// RSG_FUSED_MIX=0: mix_kernel mixes every channel.
bool fin_variant(int var) { return var == kVarIp || var == kVarIpc; }
bool fused_mix_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RSG_FUSED_MIX");
    return !(e && e[0] == '0');
  }();
  return on;
}

int launch_filter(rs_ctx* c, FilterBufs& fb, FilterPlan& fp, const std::vector<PairPlan>& plans,
                  const PairMeta* d_pair, const double* d_rir, const float* d_signals, cudaStream_t st,
                  PinnedArena* arena, cudaEvent_t ev_k4a, cudaEvent_t ev_k4b, const MixFin* d_fin = nullptr,
                  int lane = 0);

template <class T>
int upload(rs_ctx* c, DevBuf& b, const std::vector<T>& v);

// K3 + K4 of a planned set of pairs on stream `st`.
int launch_filter(rs_ctx* c, FilterBufs& fb, FilterPlan& fp, const std::vector<PairPlan>& plans,
                  const PairMeta* d_pair, const double* d_rir, const float* d_signals, cudaStream_t st,
                  PinnedArena* arena, cudaEvent_t ev_k4a, cudaEvent_t ev_k4b, const MixFin* d_fin, int lane) {
  RS_TRY(upload_on(fb.lists, fp.lists, st, arena));
  RS_TRY(upload_on(fb.plan, plans, st, arena));
  RS_TRY(upload_on(fb.olaitems, fp.items, st, arena));
  RS_TRY(fb.spec.ensure(std::max<int64_t>(fp.spec_total, 1) * sizeof(float2)));
  RS_TRY(fb.y.ensure(std::max<int64_t>(fp.y_total, 1) * sizeof(float)));
  RS_TRY(fb.part.ensure(std::max<int64_t>(fp.part_total, 1) * sizeof(double)));
  if (!fp.items2.empty()) RS_TRY(upload_on(fb.olaitems2, fp.items2, st, arena));
  if (!fp.batches.empty()) {
    RS_TRY(upload_on(fb.units, fp.units, st, arena));
    RS_TRY(fb.scratch.ensure(fp.max_scratch * sizeof(float2)));
    RS_TRY(fb.yblk.ensure(fp.max_scratch * 2 * sizeof(float)));
  }
  const int32_t* d_lists = fb.lists.as<int32_t>();
  double* d_part = fb.part.as<double>();
  // ola_ipc_kernel items transform their pair's RIR themselves (RSG_IPC_K3=1: a K3 launch instead)
  static const bool ipc_k3 = std::getenv("RSG_IPC_K3") != nullptr;
  for (const Span& sp : fp.spans) {
    if (sp.var == kVarLarge) continue;  // spectrum inside the four-step batches
    if (sp.var == kVarIpc && !ipc_k3) continue;
    SpecArgs a{d_lists + sp.list_off, static_cast<int32_t>(sp.list_n), d_pair, fb.plan.as<PairPlan>(),
               d_rir, fb.spec.as<float2>(), c->tw[sp.l], sp.var == kVarIpc ? ipc_perm(sp.l + 1) : IpcPerm{}};
    RS_CUDA(launch_spectrum(sp.l, a, st));
    ++c->launches;
  }
  if (ev_k4a) RS_CUDA(cudaEventRecord(ev_k4a, st));
  // fork: each size's K4 launch on its own side stream (the four-step batches share one
  // scratch, so they stay in order on one stream), joined back into `st` below
  cudaStream_t* side = c->side + lane * rs_ctx::kSide;
  cudaEvent_t* side_join = c->side_join + lane * rs_ctx::kSide;
  RS_CUDA(cudaEventRecord(c->side_fork[lane], st));
  bool used[rs_ctx::kSide] = {};
  int next_side = 0;
  std::function<cudaStream_t()> side_for = [&]() -> cudaStream_t {
    const int i = next_side++ % rs_ctx::kSide;
    if (!used[i]) {
      cudaStreamWaitEvent(side[i], c->side_fork[lane], 0);
      used[i] = true;
    }
    return side[i];
  };
  const bool serial = c->prof_level >= 2;  // diagnostic: one stream, one event pair per span
  auto span_flops = [&](const Span& sp) {
    double f = 0;
    for (int64_t i = 0; i < sp.list_n; ++i) f += fp.alg[fp.lists[sp.list_off + i]];
    return f;
  };
  auto span_begin = [&](const Span& sp) {
    if (!serial) return;
    double ef = 0;  // flops of the executed plans
    for (int64_t i = 0; i < sp.list_n; ++i) ef += pair_flops(plans[fp.lists[sp.list_off + i]]);
    rs_ctx::K4Span k{sp.l + 1, sp.var, sp.list_n, span_flops(sp), ef, c->pool_event(), c->pool_event()};
    cudaEventRecord(k.a, st);
    c->k4_spans.push_back(k);
  };
  auto span_end = [&]() {
    if (serial) cudaEventRecord(c->k4_spans.back().b, st);
  };
  if (serial) side_for = [&]() -> cudaStream_t { return st; };
  cudaStream_t large_st = fp.batches.empty() ? st : side_for();
  int open_span = -1;
  for (const LargeBatch& bt : fp.batches) {
    const Span& sp = fp.spans[bt.span];
    if (bt.span != open_span) {
      if (open_span >= 0) span_end();
      span_begin(sp);
      open_span = bt.span;
    }
    int l1, l2;
    large_split(sp.l, &l1, &l2);
    LargeArgs a{fb.units.as<int2>() + bt.unit_lo, d_lists + sp.list_off + bt.pair_lo,
                static_cast<int32_t>(bt.unit_hi - bt.unit_lo), static_cast<int32_t>(bt.pair_hi - bt.pair_lo),
                d_pair, fb.plan.as<PairPlan>(), d_signals, d_rir, fb.spec.as<float2>(), fb.scratch.as<float2>(),
                fb.yblk.as<float>(), fb.y.as<float>(), d_part,
                fb.olaitems.as<OlaItem>() + bt.item_lo, static_cast<int32_t>(bt.item_hi - bt.item_lo),
                c->tw[l1], c->tw[l2]};
    for (int stage = 0; stage < 6; ++stage) {
      RS_CUDA(launch_large(sp.l, a, stage, large_st));
      ++c->launches;
    }
  }
  if (open_span >= 0) span_end();
  for (const Span& sp : fp.spans) {
    if (sp.var != kVarLarge) span_begin(sp);
    if (sp.var == kVarOla2) {
      Ola2Args a{fb.olaitems2.as<OlaItem2>() + sp.item_off, static_cast<int32_t>(sp.item_n), d_pair,
                 fb.plan.as<PairPlan>(), d_signals, fb.spec.as<float2>(), fb.y.as<float>(), d_part,
                 c->tw2f[sp.l + 1], c->tw2i[sp.l + 1],
                 static_cast<int32_t>((std::max<int64_t>(sp.max_nh - 1, 1) + 3) & ~int64_t(3)),
                 static_cast<int32_t>((sp.max_l + 8 + 3) & ~int64_t(3))};
      RS_CUDA(launch_ola2(sp.l + 1, a, side_for()));
      ++c->launches;
    } else if (sp.var == kVarSmall || sp.var == kVarIp || sp.var == kVarIpc) {
      OlaArgs a{fb.olaitems.as<OlaItem>() + sp.item_off, static_cast<int32_t>(sp.item_n), d_pair,
                fb.plan.as<PairPlan>(), d_signals, fb.spec.as<float2>(), fb.y.as<float>(), d_part, c->tw[sp.l],
                sp.seg, (sp.var == kVarIpc && !ipc_k3) ? d_rir : nullptr,
                fin_variant(sp.var) ? d_fin : nullptr};
      if (sp.var == kVarIpc)
        RS_CUDA(launch_ola_ipc(sp.l + 1, a, sp.max_nh, side_for()));
      else if (sp.var == kVarIp)
        RS_CUDA(launch_ola_ip(sp.l, a, sp.max_nh, side_for()));
      else
        RS_CUDA(launch_ola(sp.l, a, side_for()));
      ++c->launches;
    }
    if (sp.var != kVarLarge) span_end();
  }
  for (int i = 0; i < rs_ctx::kSide; ++i)  // join
    if (used[i]) {
      RS_CUDA(cudaEventRecord(side_join[i], side[i]));
      RS_CUDA(cudaStreamWaitEvent(st, side_join[i], 0));
    }
  if (ev_k4b) RS_CUDA(cudaEventRecord(ev_k4b, st));
  return RS_OK;
}

// Profiling level 2: turn the render's per-span events into rows merged by (N, variant).
void collect_k4_rows(rs_ctx* c) {
  c->k4_rows.clear();
  for (const auto& k : c->k4_spans) {
    float ms = 0;
    cudaEventElapsedTime(&ms, k.a, k.b);
    bool merged = false;
    for (auto& r : c->k4_rows)
      if (r.log2n == k.log2n && r.var == k.var) {
        r.pairs += k.pairs;
        r.flops += k.flops;
        r.exec_flops += k.exec_flops;
        r.ms += ms;
        merged = true;
      }
    if (!merged) c->k4_rows.push_back(rs_ctx::K4Row{k.log2n, k.var, k.pairs, k.flops, ms, k.exec_flops});
  }
  c->k4_spans.clear();
  c->ev_used = 0;
}

int finish_timing(rs_ctx* c) {
  if (!c->profiling) return RS_OK;
  float ms = 0;
  RS_CUDA(cudaEventSynchronize(c->ev1));
  RS_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->ola_ms = ms;
  return RS_OK;
}

// ---- the batched render: a chunked two-stream pipeline -----------------------
// Utterances are processed in chunks.  Stream A runs chunk k's input upload,
// K1 (synth) and K2 (cut) and returns the per-pair RIR summary to pinned host
// memory; the host plans chunk k (reference planner) while the GPU is busy
// with chunk k-1's filter on a filter stream, which then runs K3, K4 (the last
// work item of an output channel mixes it), K5, K6 for the channels K4 left,
// and the output download of chunk k.  Chunks are independent (utterances
// share nothing), so results do not depend on the chunking.
struct RenderIO {
  const float* d_signals;  // device signals (sig_off indexes them)
  float* d_out;            // device output base (out_off indexes it); null: features only
  const float* h_signals;  // host path: upload per chunk into d_signals
  float* h_out;            // host path: download per chunk from d_out
  float* d_feat = nullptr;            // features mode: stacked log-Mel vectors (mix_logmel_kernel)
  const int64_t* feat_off = nullptr;  // per output channel (utterance-major, then mic), host
};

// The reference planner's layout of a pair (convolution.hpp:72-161), as reported.
struct RefLayout { int32_t log2n = 0; int64_t L = 0, B = 0; };

struct Chunk {
  int64_t u0 = 0, u1 = 0, p0 = 0, P = 0;
  std::vector<UttMeta> utt;
  std::vector<double> rg;
  std::vector<PairMeta> pair;
  std::vector<SynthItem> items;
  std::vector<std::tuple<int64_t, int64_t, int, int>> synth_class;  // (offset, count, slice cap, threads)
  std::vector<int32_t> bound_pairs;                                  // truncated renders: synth_bound.cu
  std::vector<std::tuple<int64_t, int64_t, int, int>> bound_class;   // (offset, count, cap, threads)
  std::vector<int> place_err;            // per pair: config / placement error (K1 skips the pair)
  std::vector<std::string> place_msg;
  std::vector<uint8_t> empty_sig;        // per pair: N_x == 0 (reported after the RIR's own errors)
  std::vector<int> utt_err;              // per utterance: no target or no mic
  std::vector<std::string> utt_msg;
  std::vector<PairPlan> plans;   // executed plans (device)
  std::vector<RefLayout> ref;    // the reference's plans (reported)
  std::vector<int32_t> strategy;
  std::vector<int64_t> ulen;
  FilterPlan fp;
  int max_order = 0, slice = 1;
  int64_t rir_total = 0;
  DevBuf d_chan_feat, d_fin, d_chan_left, d_pair_chan, d_chan_utt2, d_chan_mic2, d_chan_out2;
  DevBuf d_utt, d_pair, d_rg, d_items, d_bound, d_rir, d_rirout, d_gain, d_power, d_flags, d_snr, d_chan_utt,
      d_chan_mic, d_chan_out, d_utt_len, d_utt_stride, d_utt_pair0, d_utt_I, d_utt_J;
  FilterBufs fb;
  PinnedArena hA, hB;
  PairRir* h_rir = nullptr;
  int32_t* h_flags = nullptr;
  double* h_gain = nullptr;
  double* h_power = nullptr;
  cudaEvent_t ev_rir = nullptr, ev_syn0 = nullptr, ev_syn1 = nullptr, ev_k4a = nullptr, ev_k4b = nullptr,
              ev_mix0 = nullptr, ev_mix1 = nullptr, ev_sig = nullptr, ev_out = nullptr;
  int init_events() {
    cudaEvent_t* evs[] = {&ev_rir, &ev_syn0, &ev_syn1, &ev_k4a, &ev_k4b, &ev_mix0, &ev_mix1};
    for (auto* e : evs)
      if (!*e) RS_CUDA(cudaEventCreate(e));
    cudaEvent_t* sync_only[] = {&ev_sig, &ev_out};
    for (auto* e : sync_only)
      if (!*e) RS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return RS_OK;
  }
  void release() {
    DevBuf* bufs[] = {&d_chan_feat, &d_fin, &d_chan_left, &d_pair_chan, &d_chan_utt2, &d_chan_mic2, &d_chan_out2, &d_utt, &d_pair, &d_rg, &d_items, &d_bound, &d_rir, &d_rirout, &d_gain, &d_power, &d_flags,
                      &d_snr, &d_chan_utt, &d_chan_mic, &d_chan_out, &d_utt_len, &d_utt_stride,
                      &d_utt_pair0, &d_utt_I, &d_utt_J, &fb.plan, &fb.lists, &fb.olaitems, &fb.spec,
                      &fb.y, &fb.part, &fb.units, &fb.scratch, &fb.yblk, &fb.olaitems2};
    for (DevBuf* b : bufs) b->release();
    hA.release();
    hB.release();
    cudaEvent_t evs[] = {ev_rir, ev_syn0, ev_syn1, ev_k4a, ev_k4b, ev_mix0, ev_mix1, ev_sig, ev_out};
    for (auto e : evs)
      if (e) cudaEventDestroy(e);
  }
};

}  // namespace

struct rs_render_state {
  FilterBufs conv;                  // single-pair convolve path
  std::vector<Chunk> chunks;
  std::vector<int64_t> pair_chunk;  // global pair -> chunk
  // sA: K1/K2 and RIR summaries; sB / sB2: K3-K6 (the filter streams); sH/sD: host<->device copies of the
  // signals and outputs, so the PCIe transfers run back to back under the kernels.
  cudaStream_t sA = nullptr, sB = nullptr, sB2 = nullptr, sH = nullptr, sD = nullptr;
  cudaEvent_t ev_start = nullptr, ev_endA = nullptr, ev_endB = nullptr, ev_endB2 = nullptr, ev_endH = nullptr,
              ev_endD = nullptr;
  // RSG_TRACE=1: per-chunk timeline of the pipeline (device events + host marks) on stderr
  bool tracing = false;
  cudaEvent_t tr0 = nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> trace_ev;
  std::vector<std::pair<std::string, double>> trace_host;
  std::chrono::steady_clock::time_point trace_t0;
  void mark(cudaStream_t st, const std::string& label) {
    if (!tracing) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    trace_ev.emplace_back(label, e);
  }
  void hmark(const std::string& label) {
    if (tracing)
      trace_host.emplace_back(
          label, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - trace_t0).count());
  }
  void dump() {
    if (!tracing) return;
    for (auto& [l, e] : trace_ev) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tr0, e);
      std::fprintf(stderr, "[trace] dev %8.2f %s\n", ms, l.c_str());
      cudaEventDestroy(e);
    }
    for (auto& [l, t] : trace_host) std::fprintf(stderr, "[trace] host %8.2f %s\n", t, l.c_str());
    trace_ev.clear();
    trace_host.clear();
  }
};

namespace {

int state_init(rs_ctx* c);

// Host metadata of chunk k (validation with the reference's messages).
int prep_chunk(const rs_scene_batch* b, Chunk& ch) {
  NvtxRange nv("roomsim: prep chunk (host metadata, K1 classes)");
  ch.items.clear();
  ch.max_order = 0; ch.slice = 1; ch.rir_total = 0;
  const int64_t U = ch.u1 - ch.u0;
  // serial: per-utterance pair and r^g-table extents (prefix sums)
  std::vector<int64_t> pair_start(U + 1, 0), rg_start(U + 1, 0);
  for (int64_t lu = 0; lu < U; ++lu) {
    const int64_t u = ch.u0 + lu;
    const int64_t I = b->src_begin[u + 1] - b->src_begin[u], J = b->mic_begin[u + 1] - b->mic_begin[u];
    const int K = b->image_order[u];
    const bool bad = room_validate(b->room_dims + 3 * u, b->reflection[u], b->sample_rate[u], b->speed_of_sound[u], K);
    pair_start[lu + 1] = pair_start[lu] + std::max<int64_t>(I, 0) * std::max<int64_t>(J, 0);
    rg_start[lu + 1] = rg_start[lu] + 3 * (bad ? 0 : K) + 1;
    if (!bad) ch.max_order = std::max(ch.max_order, K);
  }
  const int64_t P = pair_start[U];
  ch.utt.assign(U, UttMeta{});
  ch.rg.assign(rg_start[U], 0.0);
  ch.pair.assign(P, PairMeta{});
  ch.place_err.assign(P, RS_OK);
  ch.place_msg.assign(P, std::string());
  ch.empty_sig.assign(P, 0);
  ch.utt_err.assign(U, RS_OK);
  ch.utt_msg.assign(U, std::string());
  // parallel over utterances: tables, pair metadata, exact RIR lengths, recorded errors
  // (glibc pow for r^g and the exact lattice maxima dominate the host's share of a render)
  host_parallel_for(U, [&](int64_t lu) {
    const int64_t u = ch.u0 + lu;
    const double* L = b->room_dims + 3 * u;
    const int64_t s0 = b->src_begin[u], I = b->src_begin[u + 1] - s0;
    const int64_t m0 = b->mic_begin[u], J = b->mic_begin[u + 1] - m0;
    // Errors are recorded, not returned: plan_chunk reports the first one in the order the
    // reference meets them (utterance, then pair; per pair: RoomConfig::validate and the
    // placements inside synthesize_rir, geometry, truncation, then the convolution).
    if (I < 1 || J < 1) {
      ch.utt_err[lu] = RS_ERR_CONFIG;
      ch.utt_msg[lu] = "scene needs a target and a microphone";
    }
    int K = b->image_order[u];
    const int cfg_err = room_validate(L, b->reflection[u], b->sample_rate[u], b->speed_of_sound[u], K);
    const std::string cfg_msg = cfg_err ? g_err : std::string();  // g_err is thread-local
    if (cfg_err) K = 0;  // no lattice for an invalid room: its pairs carry the config error
    UttMeta& um = ch.utt[lu];
    for (int a = 0; a < 3; ++a) um.dims[a] = L[a];
    um.spm = b->sample_rate[u] / b->speed_of_sound[u];  // room_model.hpp:150
    um.order = K;
    um.rg_off = static_cast<int32_t>(rg_start[lu]);
    um.max_taps = b->max_taps ? b->max_taps[u] : 0;
    for (int g = 0; g <= 3 * K; ++g) ch.rg[rg_start[lu] + g] = std::pow(b->reflection[u], static_cast<double>(g));
    int64_t cap = um.max_taps;
    if (cap <= 0) {  // bound on the farthest lattice image
      double d2 = 0;
      for (int a = 0; a < 3; ++a) {
        const double e = (K + 2.0) * L[a];
        d2 += e * e;
      }
      cap = static_cast<int64_t>(std::ceil(std::sqrt(d2) * um.spm)) + 2;
    }
    int64_t p = pair_start[lu];
    for (int64_t i = 0; i < I; ++i)
      for (int64_t j = 0; j < J; ++j, ++p) {
        PairMeta& pm = ch.pair[p];
        const double* sp = b->src_pos + 3 * (s0 + i);
        const double* mp = b->mic_pos + 3 * (m0 + j);
        for (int a = 0; a < 3; ++a) {
          pm.src[a] = sp[a];
          pm.mic[a] = mp[a];
        }
        pm.utt = static_cast<int32_t>(lu);
        pm.src_idx = static_cast<int32_t>(s0 + i);
        pm.mic_local = static_cast<int32_t>(j);
        pm.src_local = static_cast<int32_t>(i);
        pm.sig_off = b->sig_off[s0 + i];
        pm.nx = b->sig_len[s0 + i];
        // RIR length = min(max_delay + 1, horizon), known exactly before the synth
        int64_t pcap = cfg_err ? 1 : cap;
        if (!cfg_err && strictly_inside(L, sp) && strictly_inside(L, mp)) {
          const int64_t md = static_cast<int64_t>(lattice_max_delay(L, sp, mp, K, um.spm)) + 1;
          pcap = um.max_taps > 0 ? std::min<int64_t>(md, um.max_taps) : md;
        }
        pm.rir_cap = pcap;
        if (cfg_err) {  // room_model.hpp:143 (validate first)
          ch.place_err[p] = cfg_err;
          ch.place_msg[p] = cfg_msg;
        } else if (!strictly_inside(L, sp)) {  // room_model.hpp:144-145
          ch.place_err[p] = RS_ERR_PLACEMENT;
          ch.place_msg[p] = "source must lie strictly inside the room";
        } else if (!strictly_inside(L, mp)) {  // :146-147
          ch.place_err[p] = RS_ERR_PLACEMENT;
          ch.place_msg[p] = "microphone must lie strictly inside the room";
        }
        ch.empty_sig[p] = pm.nx <= 0 ? 1 : 0;
      }
  });
  for (int64_t p = 0; p < P; ++p) {  // RIR regions (serial prefix)
    ch.pair[p].rir_off = ch.rir_total;
    ch.rir_total += ch.pair[p].rir_cap;
  }
  ch.P = static_cast<int64_t>(ch.pair.size());
  // K1 launch classes: (threads, slice size).  Small lattices (K <= 12) use
  // 128-thread CTAs; slices are grouped so the dynamic smem fits the class.
  // A RIR of (14400, kSynthBig] bins (> 0.9 s at 16 kHz) is synthesized by one CTA (one per SM): every slice
  // CTA enumerates the whole image lattice, so two near-equal slices cost twice the image
  // work (config 5: K1 -18%).  Shorter RIRs keep two slices at two CTAs per SM, which
  // measured faster (config 4).  Tuning override RSG_SYNTH_BIG = "lo,hi" bins.
  static const std::pair<int64_t, int64_t> big = [] {
    const char* e = std::getenv("RSG_SYNTH_BIG");
    long long lo = 14400, hi = kSynthBig;
    if (e) std::sscanf(e, "%lld,%lld", &lo, &hi);
    return std::make_pair(static_cast<int64_t>(lo), static_cast<int64_t>(hi));
  }();
  static const int kClass[4] = {2048, 6144, kSynthSlice, kSynthBig};
  std::vector<SynthItem> cls[2][4];
  // Truncated renders: the bound pass (synth_bound.cu) finds the prefix of each RIR the cut can
  // keep, and K1 synthesizes only that — in short slices, since the prefix is typically a few
  // hundred to a few thousand bins (a slice beyond it exits at once).  RSG_SYNTH_CUT=0: the
  // whole RIR as for eta = 0.
  static const bool cut_off = [] {
    const char* e = std::getenv("RSG_SYNTH_CUT");
    return e && e[0] == '0';
  }();
  static const int kBoundCap[4] = {4096, 8192, 16384, kBoundMaxCap};
  std::vector<int32_t> bound_cls[2][4];
  ch.bound_pairs.clear();
  ch.bound_class.clear();
  for (int64_t p = 0; p < ch.P; ++p) {
    if (ch.place_err[p]) continue;
    const int64_t cap = ch.pair[p].rir_cap;
    const int K = ch.utt[ch.pair[p].utt].order;
    int small = K <= 12 ? 1 : 0;  // measured crossover of the 128- and 512-thread K1
    if (b->eta_db > 0.0 && !cut_off && cap <= kBoundMaxCap) {
      static const int cut_slice = [] { const char* e = std::getenv("RSG_CUT_SLICE"); return e ? std::atoi(e) : kSynthCutSlice; }();
      // largest K on the 128-thread exact kernel: 40 in a full chunk (the best K1 + K1a throughput);
      // 12 in a small chunk, whose K1 launches do not fill the GPU — the launch then lasts as long
      // as its longest CTA, and 512 threads shorten that (512 utterances: K1 windows 2.2 -> 1.7 ms)
      static const int cut_small_k_env = [] { const char* e = std::getenv("RSG_CUT_SMALL_K"); return e ? std::atoi(e) : -1; }();
      const int cut_small_k = cut_small_k_env >= 0 ? cut_small_k_env : (ch.P < 8192 ? 12 : 40);
      static const int bound_small_k = [] { const char* e = std::getenv("RSG_BOUND_SMALL_K"); return e ? std::atoi(e) : 6; }();
      int bc = 0;
      while (cap > kBoundCap[bc]) ++bc;
      bound_cls[K <= bound_small_k ? 1 : 0][bc].push_back(static_cast<int32_t>(p));
      small = K <= cut_small_k ? 1 : 0;
      for (int64_t lo = 0; lo < cap; lo += cut_slice) {
        const int64_t len = std::min<int64_t>(cut_slice, cap - lo);
        cls[small][len <= kClass[0] ? 0 : (len <= kClass[1] ? 1 : 2)].push_back(
            SynthItem{static_cast<int32_t>(p), static_cast<int32_t>(lo), static_cast<int32_t>(len), 0});
      }
      continue;
    }
    if (cap > std::max<int64_t>(kSynthSlice, big.first) && cap <= big.second) {
      cls[small][3].push_back(SynthItem{static_cast<int32_t>(p), 0, static_cast<int32_t>(cap), 0});
      continue;
    }
    for (int64_t lo = 0; lo < cap; lo += kSynthSlice) {
      const int64_t len = std::min<int64_t>(kSynthSlice, cap - lo);
      const int k = len <= kClass[0] ? 0 : (len <= kClass[1] ? 1 : 2);
      cls[small][k].push_back(SynthItem{static_cast<int32_t>(p), static_cast<int32_t>(lo), static_cast<int32_t>(len), 0});
    }
  }
  for (int small = 0; small < 2; ++small)
    for (int k = 3; k >= 0; --k) {  // large lattices and longest RIRs first
      if (bound_cls[small][k].empty()) continue;
      ch.bound_class.emplace_back(static_cast<int64_t>(ch.bound_pairs.size()),
                                  static_cast<int64_t>(bound_cls[small][k].size()), kBoundCap[k], small ? 128 : 512);
      ch.bound_pairs.insert(ch.bound_pairs.end(), bound_cls[small][k].begin(), bound_cls[small][k].end());
    }
  ch.synth_class.clear();
  for (int small = 0; small < 2; ++small)
    for (int k = 3; k >= 0; --k) {  // large lattices and slices first
      int cap = 1;
      for (const auto& itm : cls[small][k]) cap = std::max(cap, itm.slice_len);
      ch.synth_class.emplace_back(static_cast<int64_t>(ch.items.size()), static_cast<int64_t>(cls[small][k].size()),
                                  cap, small ? 128 : 512);
      ch.items.insert(ch.items.end(), cls[small][k].begin(), cls[small][k].end());
      ch.slice = std::max(ch.slice, cap);
    }
  return RS_OK;
}

// Stream A: inputs, K1, K2, RIR summary -> pinned host.
int enqueue_synth(rs_ctx* c, const rs_scene_batch* b, Chunk& ch, cudaStream_t sA) {
  NvtxRange nv("roomsim: enqueue K1a / K1 / K2");
  RS_TRY(ch.init_events());
  size_t need = staged_bytes(ch.utt) + staged_bytes(ch.pair) + staged_bytes(ch.rg) + staged_bytes(ch.items) +
                staged_bytes(ch.bound_pairs) +
                ((std::max<int64_t>(ch.P, 1) * sizeof(PairRir) + 63) & ~size_t(63)) + 64;
  RS_TRY(ch.hA.reserve(need));
  ch.hA.reset();
  if (c->profiling) RS_CUDA(cudaEventRecord(ch.ev_syn0, sA));
  RS_TRY(upload_on(ch.d_utt, ch.utt, sA, &ch.hA));
  RS_TRY(upload_on(ch.d_pair, ch.pair, sA, &ch.hA));
  RS_TRY(upload_on(ch.d_rg, ch.rg, sA, &ch.hA));
  RS_TRY(upload_on(ch.d_items, ch.items, sA, &ch.hA));
  RS_TRY(ch.d_rir.ensure(std::max<int64_t>(ch.rir_total, 1) * sizeof(double)));
  RS_TRY(ch.d_rirout.ensure(std::max<int64_t>(ch.P, 1) * sizeof(PairRir)));
  RS_CUDA(cudaMemsetAsync(ch.d_rirout.p, 0, std::max<int64_t>(ch.P, 1) * sizeof(PairRir), sA));
  const double eta_factor = b->eta_db > 0.0 ? std::pow(10.0, -b->eta_db / 10.0) : 0.0;
  if (!ch.bound_pairs.empty()) {  // K1a: the prefix of each RIR the cut can keep
    RS_TRY(upload_on(ch.d_bound, ch.bound_pairs, sA, &ch.hA));
    for (const auto& [off, n, cap, nt] : ch.bound_class) {
      SynthBoundArgs sb{ch.d_utt.as<UttMeta>(), ch.d_pair.as<PairMeta>(), ch.d_rg.as<double>(),
                        ch.d_bound.as<int32_t>() + off, ch.d_rirout.as<PairRir>(), eta_factor};
      RS_CUDA(launch_synth_bound(sb, static_cast<int>(n), cap, ch.max_order, sA, nt));
      ++c->launches;
    }
  }
  // one K1 launch per slice-size class, so short RIRs get more CTAs per SM
  for (size_t k = 0; k < ch.synth_class.size(); ++k) {
    const auto& [off, n, cap, nt] = ch.synth_class[k];
    if (n == 0) continue;
    SynthArgs sa{ch.d_utt.as<UttMeta>(), ch.d_pair.as<PairMeta>(), ch.d_rg.as<double>(),
                 ch.d_items.as<SynthItem>() + off, ch.d_rir.as<double>(), ch.d_rirout.as<PairRir>()};
    RS_CUDA(launch_synth(sa, static_cast<int>(n), ch.max_order, cap, sA, nt));
    ++c->launches;
  }
  CutArgs ca{ch.d_pair.as<PairMeta>(), ch.d_utt.as<UttMeta>(), ch.d_rir.as<double>(), ch.d_rirout.as<PairRir>(),
             eta_factor};
  RS_CUDA(launch_cut(ca, static_cast<int>(ch.P), sA));
  ++c->launches;
  if (c->profiling) RS_CUDA(cudaEventRecord(ch.ev_syn1, sA));
  ch.h_rir = ch.hA.alloc<PairRir>(ch.P);
  RS_TRY(small_copy(ch.h_rir, ch.hA.dev(ch.h_rir), ch.d_rirout.p, ch.d_rirout.p, ch.P * sizeof(PairRir),
                    cudaMemcpyDeviceToHost, sA));
  RS_CUDA(cudaEventRecord(ch.ev_rir, sA));
  return RS_OK;
}

// Host: errors in reference order and the planner (after chunk k's RIR summary).
int plan_chunk(const rs_scene_batch* b, Chunk& ch, const int64_t* out_stride) {
  NvtxRange nv("roomsim: plan chunk (wait for the RIR summary, reference planner)");
  const auto t_wait0 = std::chrono::steady_clock::now();
  RS_CUDA(cudaEventSynchronize(ch.ev_rir));
  if (std::getenv("RSG_TRACE"))
    std::fprintf(stderr, "[trace] chunk of %lld pairs waited %.3f ms for its RIR summary\n", static_cast<long long>(ch.P),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wait0).count());
  ch.plans.assign(ch.P, PairPlan{});
  ch.ref.assign(ch.P, RefLayout{});
  ch.fp.alg.assign(ch.P, 0.0);
  ch.strategy.assign(ch.P, RS_OVERLAP_ADD);
  ch.ulen.assign(ch.u1 - ch.u0, 0);
  int64_t spec_off = 0, y_off = 0;
  // utterance-level errors (no target / mic) of utterances [next_utt, upto), in order
  int64_t next_utt = 0;
  auto utt_check = [&](int64_t upto) -> int {
    for (; next_utt < upto; ++next_utt)
      if (ch.utt_err[next_utt]) return fail(ch.utt_err[next_utt], ch.utt_msg[next_utt]);
    return RS_OK;
  };
  // Per pair, on the host threads (a small render's first plan is on its critical path: ~160 ns
  // per pair serially): the pair's own checks in the reference's order and its plans, everything
  // but the offsets.  A failing pair records its status and message (fail() writes the worker
  // thread's g_err); the serial pass below reports the first error in utterance / pair order.
  std::vector<int> pair_err(ch.P, RS_OK);
  std::vector<std::string> pair_msg(ch.P);
  auto plan_pair = [&](int64_t p) -> int {
    const PairRir& r = ch.h_rir[p];
    if (r.flags & 1) return fail(RS_ERR_GEOMETRY, "microphone coincides with an image source");
    if (r.flags & 8) return fail(RS_ERR_CUDA, "internal: device RIR length exceeds the host bound");
    if (r.flags & 2) return fail(RS_ERR_DEGENERATE, "all-zero impulse response has no power");
    const size_t nh = static_cast<size_t>(r.keep);
    const size_t nx = static_cast<size_t>(ch.pair[p].nx);
    if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
    size_t n = 0;
    int s = RS_OVERLAP_ADD;
    double cost;
    if (b->plan_rule == RS_PLAN_CHOOSE) {
      // choose_plan validates the lengths before convolve sees the signal (convolution.hpp:94-98)
      RS_TRY(choose_plan_impl(1.0, 1.0, nx, nh, &s, &n, &cost));
      if (s == RS_FULL_FFT) n = fft_size_for(nx + nh - 1);
    } else if (b->plan_rule == RS_PLAN_FORCED) {
      n = static_cast<size_t>(b->forced_fft_size);
      // convolve_ola checks its input before the FFT size (convolution.hpp:221-227)
      if (ch.empty_sig[p]) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
      RS_TRY(checked_fft_size(n, nh, "overlap-add"));
    } else if (b->plan_rule == RS_PLAN_POW2_TWICE) {
      n = bit_ceil_sz(2 * nh);
    } else {
      return fail(RS_ERR_CONFIG, "unknown plan rule");
    }
    if (ch.empty_sig[p]) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
    if (n < 2 || n > (static_cast<size_t>(2) << kLargeMaxLog2M))
      return fail(RS_ERR_UNSUPPORTED, "FFT size " + std::to_string(n) + " not supported by the device kernels");
    ch.strategy[p] = s;
    PairPlan& pl = ch.plans[p];
    // the reference's plan: reported, and the metric's flops
    RefLayout& rl = ch.ref[p];
    rl.log2n = log2_exact(n);
    rl.L = static_cast<int64_t>(n - nh + 1);
    rl.B = static_cast<int64_t>(block_count(nx, nh, n));
    ch.fp.alg[p] = (2.0 * static_cast<double>(rl.B) + 1.0) * 5.0 * static_cast<double>(n) * rl.log2n;
    // the executed plan (exec_log2n above)
    if (b->plan_rule != RS_PLAN_FORCED) n = size_t(1) << exec_log2n(nx, nh, rl.log2n);
    pl.log2n = log2_exact(n);
    pl.nh = static_cast<int64_t>(nh);
    pl.L = static_cast<int64_t>(n - nh + 1);
    pl.B = static_cast<int64_t>(block_count(nx, nh, n));
    pl.out_len = static_cast<int64_t>(nx + nh - 1);
    return RS_OK;
  };
  constexpr int64_t kPlanBlock = 256;  // pairs per parallel iteration
  host_parallel_for((ch.P + kPlanBlock - 1) / kPlanBlock, [&](int64_t blk) {
    const int64_t hi = std::min<int64_t>(ch.P, (blk + 1) * kPlanBlock);
    for (int64_t p = blk * kPlanBlock; p < hi; ++p) {
      if (ch.place_err[p]) continue;  // reported below; its RIR summary is not meaningful
      pair_err[p] = plan_pair(p);
      if (pair_err[p]) pair_msg[p] = g_err;  // g_err is thread-local
    }
  }, 2);
  for (int64_t p = 0; p < ch.P; ++p) {  // serial: errors in order, offsets
    RS_TRY(utt_check(ch.pair[p].utt + 1));
    if (ch.place_err[p]) return fail(ch.place_err[p], ch.place_msg[p]);
    if (pair_err[p]) return fail(pair_err[p], pair_msg[p]);
    PairPlan& pl = ch.plans[p];
    pl.spec_off = spec_off;
    pl.y_off = y_off;
    spec_off += spec_len(pl.log2n, pl.nh);
    y_off += (pl.out_len + 3) & ~int64_t(3);  // 16-byte aligned rows: the mix reads float4
    int64_t& ul = ch.ulen[ch.pair[p].utt];
    ul = std::max(ul, pl.out_len);
  }
  if (std::getenv("RSG_TRACE")) {  // truncated-synthesis statistics of the chunk
    double sl = 0, se = 0, sk = 0, full = 0, vol = 0, volx = 0;
    for (int64_t p = 0; p < ch.P; ++p) {
      const PairRir& r = ch.h_rir[p];
      const double e = r.exact_len > 0 ? r.exact_len : r.len;
      sl += r.len; se += e; sk += r.keep; full += r.exact_len > 0 ? 0 : 1;
      const double W = 2.0 * ch.utt[ch.pair[p].utt].order + 1.0;
      vol += W * W * W;
      volx += W * W * W * std::min(1.0, std::pow(e / std::max<double>(r.len, 1), 3.0));
    }
    std::fprintf(stderr, "[trace] chunk of %lld pairs: mean len %.0f, exact_len %.0f, keep %.0f; %.0f pairs in full; images %.3g, ~in exact sphere %.3g\n",
                 static_cast<long long>(ch.P), sl / ch.P, se / ch.P, sk / ch.P, full, vol, volx);
  }
  RS_TRY(utt_check(static_cast<int64_t>(ch.utt_err.size())));  // trailing utterances without pairs
  for (int64_t u = ch.u0; u < ch.u1; ++u)
    if (out_stride[u] < ch.ulen[u - ch.u0]) return fail(RS_ERR_CONFIG, "output stride too small");
  return plan_filter(ch.plans, ch.fp);
}

// Filter stream: K3, K4 + mix epilogue, K5, K6 (+ output download on the host path).
int enqueue_filter(rs_ctx* c, const rs_scene_batch* b, Chunk& ch, const RenderIO& io, const int64_t* out_off,
                   const int64_t* out_stride, cudaStream_t sB, cudaStream_t sD, int lane) {
  NvtxRange nv("roomsim: enqueue K3 / K4 + mix epilogue / K5 / K6");
  const int64_t U = ch.u1 - ch.u0;
  std::vector<double> snr_lin(b->src_begin[ch.u1] - b->src_begin[ch.u0]);
  const int64_t s_first = b->src_begin[ch.u0];
  for (size_t s = 0; s < snr_lin.size(); ++s) snr_lin[s] = std::pow(10.0, b->snr_db[s_first + s] / 10.0);
  std::vector<int64_t> pair0(U), ustride(U);
  std::vector<int32_t> uI(U), uJ(U);
  std::vector<int64_t> ch_utt, ch_out;
  std::vector<int32_t> ch_mic;
  int64_t max_stride = 0, acc = 0;
  for (int64_t lu = 0; lu < U; ++lu) {
    const int64_t u = ch.u0 + lu;
    uI[lu] = static_cast<int32_t>(b->src_begin[u + 1] - b->src_begin[u]);
    uJ[lu] = static_cast<int32_t>(b->mic_begin[u + 1] - b->mic_begin[u]);
    pair0[lu] = acc;
    acc += static_cast<int64_t>(uI[lu]) * uJ[lu];
    ustride[lu] = out_stride[u];
    max_stride = std::max(max_stride, out_stride[u]);
    for (int32_t j = 0; j < uJ[lu]; ++j) {
      ch_utt.push_back(lu);
      ch_mic.push_back(j);
      ch_out.push_back(out_off[u] + j * out_stride[u]);
    }
  }
  // ---- fused mix (mixfin.cuh): a channel whose pairs all run on the one-CTA-per-item K4 kernels
  // is mixed by its last work item inside the K4 launch; the other channels by mix_kernel.
  const int64_t n_chan = static_cast<int64_t>(ch_utt.size());
  const bool fuse = (c->fused_mix < 0 ? fused_mix_enabled() : c->fused_mix != 0) && !io.d_feat && io.d_out;
  std::vector<int32_t> pair_chan(std::max<int64_t>(ch.P, 1), -1), left(std::max<int64_t>(n_chan, 1), 0);
  std::vector<int64_t> ch_utt2, ch_out2;  // the channels left to mix_kernel
  std::vector<int32_t> ch_mic2;
  {
    std::vector<int32_t> items_of(ch.P, 0);
    std::vector<uint8_t> ok(ch.P, 0);
    if (fuse)
      for (const Span& sp : ch.fp.spans)
        if (fin_variant(sp.var))
          for (int64_t i = sp.item_off; i < sp.item_off + sp.item_n; ++i) {
            ++items_of[ch.fp.items[i].pair];
            ok[ch.fp.items[i].pair] = 1;
          }
    int64_t cidx = 0;
    for (int64_t lu = 0; lu < U; ++lu)
      for (int32_t j = 0; j < uJ[lu]; ++j, ++cidx) {
        bool all = fuse && uI[lu] >= 1 && uI[lu] <= kMixMaxI;
        int32_t cnt = 0;
        for (int32_t i = 0; i < uI[lu] && all; ++i) {
          const int64_t p = pair0[lu] + static_cast<int64_t>(i) * uJ[lu] + j;
          all = ok[p] != 0;
          cnt += items_of[p];
        }
        if (all) {
          left[cidx] = cnt;
          for (int32_t i = 0; i < uI[lu]; ++i) pair_chan[pair0[lu] + static_cast<int64_t>(i) * uJ[lu] + j] = static_cast<int32_t>(cidx);
        } else {
          ch_utt2.push_back(ch_utt[cidx]);
          ch_mic2.push_back(ch_mic[cidx]);
          ch_out2.push_back(ch_out[cidx]);
        }
      }
  }
  const int64_t n_chan2 = static_cast<int64_t>(ch_utt2.size());
  const bool any_fused = n_chan2 < n_chan;
  c->fused_channels += n_chan - n_chan2;
  c->mixed_channels += n_chan;
  std::vector<MixFin> finv(1);
  size_t need = staged_bytes(ch.fp.lists) + staged_bytes(ch.plans) + staged_bytes(ch.fp.items) +
                staged_bytes(ch.fp.items2) + staged_bytes(ch.fp.units) +
                staged_bytes(snr_lin) + staged_bytes(pair0) + staged_bytes(uI) + staged_bytes(uJ) +
                staged_bytes(ch_utt) + staged_bytes(ch_mic) + staged_bytes(ch_out) + staged_bytes(ch.ulen) +
                staged_bytes(ustride) + 3 * (((std::max<int64_t>(ch.P, 1) * 8) + 63) & ~size_t(63)) + 256 +
                (io.d_feat ? staged_bytes(ch_out) : 0) + staged_bytes(pair_chan) + staged_bytes(left) +
                staged_bytes(ch_utt2) + staged_bytes(ch_mic2) + staged_bytes(ch_out2) + staged_bytes(finv);
  RS_TRY(ch.hB.reserve(need));
  ch.hB.reset();
  // the mix's metadata goes up before K4: the epilogue reads it
  RS_TRY(upload_on(ch.d_snr, snr_lin, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_utt_pair0, pair0, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_utt_I, uI, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_utt_J, uJ, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_chan_utt, ch_utt, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_chan_mic, ch_mic, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_chan_out, ch_out, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_utt_len, ch.ulen, sB, &ch.hB));
  RS_TRY(upload_on(ch.d_utt_stride, ustride, sB, &ch.hB));
  RS_TRY(ch.d_gain.ensure(std::max<int64_t>(ch.P, 1) * sizeof(double)));
  RS_TRY(ch.d_power.ensure(std::max<int64_t>(ch.P, 1) * sizeof(double)));
  RS_TRY(ch.d_flags.ensure(std::max<int64_t>(ch.P, 1) * sizeof(int32_t)));
  // (launch_filter sizes these three the same way: the pointers below stay valid)
  RS_TRY(ch.fb.plan.ensure(std::max<size_t>(ch.plans.size(), 1) * sizeof(PairPlan)));
  RS_TRY(ch.fb.y.ensure(std::max<int64_t>(ch.fp.y_total, 1) * sizeof(float)));
  RS_TRY(ch.fb.part.ensure(std::max<int64_t>(ch.fp.part_total, 1) * sizeof(double)));
  MixArgs ma{ch.d_chan_utt.as<int64_t>(), ch.d_chan_mic.as<int32_t>(), ch.d_chan_out.as<int64_t>(),
             ch.d_utt_len.as<int64_t>(), ch.d_utt_stride.as<int64_t>(), ch.d_utt_pair0.as<int64_t>(),
             ch.d_utt_I.as<int32_t>(), ch.d_utt_J.as<int32_t>(), ch.fb.plan.as<PairPlan>(), ch.fb.y.as<float>(),
             ch.d_gain.as<double>(), io.d_out, 4096};
  const MixFin* d_fin = nullptr;
  if (any_fused) {
    RS_TRY(upload_on(ch.d_pair_chan, pair_chan, sB, &ch.hB));
    RS_TRY(upload_on(ch.d_chan_left, left, sB, &ch.hB));
    finv[0] = MixFin{ch.d_chan_left.as<int32_t>(), ch.d_pair_chan.as<int32_t>(), ch.d_snr.as<double>() - s_first,
                     ch.fb.part.as<double>(), ch.d_pair.as<PairMeta>(), ma};
    RS_TRY(upload_on(ch.d_fin, finv, sB, &ch.hB));
    d_fin = ch.d_fin.as<MixFin>();
  }
  if (io.h_signals) RS_CUDA(cudaStreamWaitEvent(sB, ch.ev_sig, 0));
  RS_TRY(launch_filter(c, ch.fb, ch.fp, ch.plans, ch.d_pair.as<PairMeta>(), ch.d_rir.as<double>(), io.d_signals,
                       sB, &ch.hB, ch.ev_k4a, ch.ev_k4b, d_fin, lane));
  if (c->profiling) RS_CUDA(cudaEventRecord(ch.ev_mix0, sB));
  RS_CUDA(cudaMemsetAsync(ch.d_flags.p, 0, std::max<int64_t>(ch.P, 1) * sizeof(int32_t), sB));
  GainArgs ga{ch.d_pair.as<PairMeta>(), ch.fb.plan.as<PairPlan>(), ch.d_utt_pair0.as<int64_t>(),
              ch.d_utt_J.as<int32_t>(), ch.fb.part.as<double>(), ch.d_snr.as<double>() - s_first,
              ch.d_gain.as<double>(), ch.d_power.as<double>(), ch.d_flags.as<int32_t>(), ch.P};
  RS_CUDA(launch_gain(ga, sB));
  c->launches += 2;
  if (any_fused) {  // mix_kernel: the channels no K4 epilogue mixed
    RS_TRY(upload_on(ch.d_chan_utt2, ch_utt2, sB, &ch.hB));
    RS_TRY(upload_on(ch.d_chan_mic2, ch_mic2, sB, &ch.hB));
    RS_TRY(upload_on(ch.d_chan_out2, ch_out2, sB, &ch.hB));
    ma.chan_utt = ch.d_chan_utt2.as<int64_t>();
    ma.chan_mic = ch.d_chan_mic2.as<int32_t>();
    ma.chan_out = ch.d_chan_out2.as<int64_t>();
  }
  if (io.d_feat) {  // features mode: mix + log-Mel in one kernel (features.cu)
    std::vector<int64_t> ch_feat(ch_utt.size());
    const int64_t c0 = b->mic_begin[ch.u0];  // global index of the chunk's first channel
    for (size_t k = 0; k < ch_feat.size(); ++k) ch_feat[k] = io.feat_off[c0 + static_cast<int64_t>(k)];
    RS_TRY(upload_on(ch.d_chan_feat, ch_feat, sB, &ch.hB));
    const MixFeatArgs lf{io.d_feat, ch.d_chan_feat.as<int64_t>(), c->lm_window.as<float>(), c->lm_ptr.as<int32_t>(),
                         c->lm_bin.as<int32_t>(), c->lm_w.as<float>(), c->tw[8], 1e-10f};
    RS_CUDA(launch_mix_logmel(ma, lf, static_cast<int64_t>(ch_utt.size()), max_stride, sB));
    ++c->launches;
  } else if (n_chan2 > 0) {
    RS_CUDA(launch_mix(ma, n_chan2, max_stride, sB));
    ++c->launches;
  }
  if (c->profiling) RS_CUDA(cudaEventRecord(ch.ev_mix1, sB));
  ch.h_flags = ch.hB.alloc<int32_t>(ch.P);
  ch.h_gain = ch.hB.alloc<double>(ch.P);
  ch.h_power = ch.hB.alloc<double>(ch.P);
  if (ch.P) {
    RS_TRY(small_copy(ch.h_flags, ch.hB.dev(ch.h_flags), ch.d_flags.p, ch.d_flags.p, ch.P * sizeof(int32_t),
                      cudaMemcpyDeviceToHost, sB));
    RS_TRY(small_copy(ch.h_gain, ch.hB.dev(ch.h_gain), ch.d_gain.p, ch.d_gain.p, ch.P * sizeof(double),
                      cudaMemcpyDeviceToHost, sB));
    RS_TRY(small_copy(ch.h_power, ch.hB.dev(ch.h_power), ch.d_power.p, ch.d_power.p, ch.P * sizeof(double),
                      cudaMemcpyDeviceToHost, sB));
  }
  if (io.h_out) {  // host path: this chunk's output span, on the download stream
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t u = ch.u0; u < ch.u1; ++u) {
      lo = std::min(lo, out_off[u]);
      hi = std::max(hi, out_off[u] + (b->mic_begin[u + 1] - b->mic_begin[u]) * out_stride[u]);
    }
    if (hi > lo) {
      RS_CUDA(cudaEventRecord(ch.ev_out, sB));
      RS_CUDA(cudaStreamWaitEvent(sD, ch.ev_out, 0));
      RS_CUDA(cudaMemcpyAsync(io.h_out + lo, io.d_out + lo, (hi - lo) * sizeof(float), cudaMemcpyDeviceToHost, sD));
    }
  }
  return RS_OK;
}

int render_impl(rs_ctx* c, const rs_scene_batch* b, const RenderIO& io, const int64_t* out_off,
                const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout, double* gains,
                double* power);

int state_init(rs_ctx* c) {
  if (c->rs) return RS_OK;
  c->rs = new rs_render_state();
  // Stream A (K1, K2) runs above stream B's priority: chunk k+1's synthesis is enqueued while
  // chunk k-1's K4 grids still have CTAs waiting; at equal priority it would only start
  // once those grids had been dispatched, and the host could not plan chunk k+1 in time.
  {
    int prio_lo = 0, prio_hi = 0;
    RS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    static const bool flat = std::getenv("RSG_FLAT_PRIORITY") != nullptr;  // diagnostic
    RS_CUDA(cudaStreamCreateWithPriority(&c->rs->sA, cudaStreamNonBlocking, flat ? prio_lo : prio_hi));
  }
  // The filter streams carry a chunk's uploads, K5 and the K6 tail (K4 itself runs on the ctx's
  // side streams, at the default priority): above the K4 launches of the other lane, so a chunk's
  // gains and summary do not wait for SMs under the next chunk's K4.
  {
    int prio_lo = 0, prio_hi = 0;
    RS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    RS_CUDA(cudaStreamCreateWithPriority(&c->rs->sB, cudaStreamNonBlocking, prio_hi));
    RS_CUDA(cudaStreamCreateWithPriority(&c->rs->sB2, cudaStreamNonBlocking, prio_hi));
  }
  RS_CUDA(cudaStreamCreateWithFlags(&c->rs->sH, cudaStreamNonBlocking));
  RS_CUDA(cudaStreamCreateWithFlags(&c->rs->sD, cudaStreamNonBlocking));
  cudaEvent_t* evs[] = {&c->rs->ev_start, &c->rs->ev_endA, &c->rs->ev_endB, &c->rs->ev_endB2, &c->rs->ev_endH,
                        &c->rs->ev_endD};
  for (auto* e : evs) RS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return RS_OK;
}

void destroy_state(rs_ctx* c) {
  if (!c->rs) return;
  rs_render_state* r = c->rs;
  cudaStream_t ss[] = {r->sA, r->sB, r->sB2, r->sH, r->sD};
  for (auto st : ss)
    if (st) cudaStreamSynchronize(st);
  for (auto& ch : r->chunks) ch.release();
  FilterBufs& f = r->conv;
  DevBuf* bufs[] = {&f.plan, &f.lists, &f.olaitems, &f.spec, &f.y, &f.part, &f.units, &f.scratch, &f.yblk,
                    &f.olaitems2};
  for (DevBuf* b : bufs) b->release();
  for (auto st : ss)
    if (st) cudaStreamDestroy(st);
  cudaEvent_t evs[] = {r->ev_start, r->ev_endA, r->ev_endB, r->ev_endB2, r->ev_endH, r->ev_endD};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  delete r;
  c->rs = nullptr;
}

// Pairs per chunk: large enough to fill the GPU with one chunk's K4, small enough that
// host planning and K1/K2 of the next chunk hide behind it.  Device-buffer renders:
// 16384 (config 4: 3 chunks; measured 2.5% faster than 6144 and K4 +0.03 of its
// roofline — fewer, fuller K4 launches); host-buffer renders keep 6144 so the first
// chunk's upload and the last chunk's download stay short (PCIe-bound).
constexpr int64_t kChunkPairsDevice = 16384;
constexpr int64_t kChunkPairsHost = 6144;
constexpr int64_t kFirstChunkPairs = 4096;
// Renders of fewer than 2 full chunks open with a quarter of their pairs and split the rest in
// two (measured, 512 utterances = 6144 pairs, chunks alternating between the two filter streams:
// opening chunks of 768 / 1024 / 1536 / 2048 pairs 4.38 / 4.40 / 4.16 / 4.20 ms vs 4.24 ms for two
// equal chunks — a shorter K4 launch underfills the GPU).
constexpr int64_t kFirstChunkDivSmall = 4;

int render_impl(rs_ctx* c, const rs_scene_batch* b, const RenderIO& io, const int64_t* out_off,
                const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout, double* gains,
                double* power) {
  if (!b || b->n_utt < 0) return fail(RS_ERR_CONFIG, "invalid scene batch");
  NvtxRange nv_render("roomsim: render_batch");
  const auto t_enter = std::chrono::steady_clock::now();
  static thread_local std::chrono::steady_clock::time_point t_last_return = t_enter;
  RS_TRY(state_init(c));
  rs_render_state& R = *c->rs;
  const int64_t U = b->n_utt;
  c->launches = 0;
  c->fused_channels = c->mixed_channels = 0;
  g_copy_launches = 0;
  const bool host_io = io.h_signals || io.h_out;
  g_kernel_copies = host_io;
  // ---- chunking by pair count ----------------------------------------------------
  static const int64_t chunk_env = [] {
    const char* e = std::getenv("RSG_CHUNK_PAIRS");  // tuning override
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(0);
  }();
  int64_t total_pairs = 0;
  for (int64_t u = 0; u < U; ++u)
    total_pairs += (b->src_begin[u + 1] - b->src_begin[u]) * (b->mic_begin[u + 1] - b->mic_begin[u]);
  // Device renders open with a short chunk, so the first filter starts soon after the call (its
  // K1 and host planning are the pipeline's fill time).  Renders of fewer than 2 full chunks
  // (e.g. one rank's share under strong scaling) open with a quarter of their pairs and split the
  // rest in two, so the host planner of one chunk overlaps the others' kernels.
  static const int64_t first_env = [] {
    const char* e = std::getenv("RSG_FIRST_CHUNK");  // tuning override (pairs; 0: none)
    return e ? std::atoll(e) : int64_t(-1);
  }();
  const bool small_total = total_pairs <= 2 * kChunkPairsDevice;
  const int64_t first_pairs =
      first_env >= 0 ? first_env
                     : (small_total ? (total_pairs / kFirstChunkDivSmall >= 1024 ? total_pairs / kFirstChunkDivSmall : 0)
                                    : kFirstChunkPairs);
  const bool open_short = !host_io && !chunk_env && first_pairs > 0 && total_pairs > 3 * first_pairs;
  const int64_t dev_chunk = small_total
                                ? std::max<int64_t>(2048, (total_pairs - (open_short ? first_pairs : 0) + 1) / 2)
                                : kChunkPairsDevice;
  const int64_t chunk_pairs = chunk_env ? chunk_env : (host_io ? kChunkPairsHost : dev_chunk);
  // Host path: the last chunk_pairs are split C/2, C/4, C/4 so the pipeline drains
  // quickly (only the final chunk's filter and download follow the last upload).
  std::vector<std::pair<int64_t, int64_t>> ranges;
  {
    int64_t total = 0;
    for (int64_t u = 0; u < U; ++u)
      total += (b->src_begin[u + 1] - b->src_begin[u]) * (b->mic_begin[u + 1] - b->mic_begin[u]);
    int64_t u0 = 0, pairs = 0, done = 0;
    auto target = [&] {
      const int64_t rem = total - done;
      if (!host_io) return done == 0 && open_short ? std::min(first_pairs, chunk_pairs) : chunk_pairs;
      if (rem > chunk_pairs) return std::min(chunk_pairs, rem - chunk_pairs);
      return rem > chunk_pairs / 4 ? std::max<int64_t>(rem / 2, chunk_pairs / 4) : rem;
    };
    int64_t want = target();
    for (int64_t u = 0; u < U; ++u) {
      pairs += (b->src_begin[u + 1] - b->src_begin[u]) * (b->mic_begin[u + 1] - b->mic_begin[u]);
      if (pairs >= want || u + 1 == U) {
        ranges.emplace_back(u0, u + 1);
        u0 = u + 1;
        done += pairs;
        pairs = 0;
        want = target();
      }
    }
  }
  const int nch = static_cast<int>(ranges.size());
  if (static_cast<int>(R.chunks.size()) < nch) R.chunks.resize(nch);
  int64_t p_acc = 0;
  for (int k = 0; k < nch; ++k) {
    Chunk& ch = R.chunks[k];
    ch.u0 = ranges[k].first;
    ch.u1 = ranges[k].second;
    ch.p0 = p_acc;
    for (int64_t u = ch.u0; u < ch.u1; ++u)
      p_acc += (b->src_begin[u + 1] - b->src_begin[u]) * (b->mic_begin[u + 1] - b->mic_begin[u]);
  }
  const int64_t Ptot = p_acc;
  c->last_pairs = Ptot;
  // ---- fork from the caller's stream ---------------------------------------------------
  RS_CUDA(cudaEventRecord(R.ev_start, c->stream));
  R.tracing = std::getenv("RSG_TRACE") != nullptr;
  if (R.tracing) {
    if (!R.tr0) cudaEventCreate(&R.tr0);
    cudaEventRecord(R.tr0, c->stream);
    R.trace_t0 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[trace] host gap since the last render returned %.2f ms, entry to fork %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t_enter - t_last_return).count(),
                 std::chrono::duration<double, std::milli>(R.trace_t0 - t_enter).count());
  }
  RS_CUDA(cudaStreamWaitEvent(R.sA, R.ev_start, 0));
  RS_CUDA(cudaStreamWaitEvent(R.sB, R.ev_start, 0));
  RS_CUDA(cudaStreamWaitEvent(R.sB2, R.ev_start, 0));
  RS_CUDA(cudaStreamWaitEvent(R.sH, R.ev_start, 0));
  RS_CUDA(cudaStreamWaitEvent(R.sD, R.ev_start, 0));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[0], c->stream));
  // Host path: chunk k's signal span goes up on sH, kSigAhead chunks ahead of the
  // filter.  Not all at once: the copy engine serves H2D copies in FIFO order, so the
  // small per-chunk metadata uploads on sA/sB would otherwise queue behind every
  // chunk's signals.
  constexpr int kSigAhead = 2;
  auto enqueue_sig = [&](int k) -> int {
    if (!io.h_signals || k >= nch) return RS_OK;
    Chunk& ch = R.chunks[k];
    RS_TRY(ch.init_events());
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t s = b->src_begin[ch.u0]; s < b->src_begin[ch.u1]; ++s) {
      lo = std::min(lo, b->sig_off[s]);
      hi = std::max(hi, b->sig_off[s] + b->sig_len[s]);
    }
    if (hi > lo)
      RS_CUDA(cudaMemcpyAsync(const_cast<float*>(io.d_signals) + lo, io.h_signals + lo, (hi - lo) * sizeof(float),
                              cudaMemcpyHostToDevice, R.sH));
    RS_CUDA(cudaEventRecord(ch.ev_sig, R.sH));
    R.mark(R.sH, "sig done " + std::to_string(k));
    return RS_OK;
  };
  int status = RS_OK;
  auto t_plan = 0.0;
  // A chunk's layouts, output lengths and algorithmic bytes come from its plan alone: filled
  // while its kernels run, so only the gains and powers are left after the final sync.
  double alg_bytes = 0;
  R.pair_chunk.assign(Ptot, 0);
  auto fill_layouts = [&](Chunk& ch) {
    const int k = static_cast<int>(&ch - R.chunks.data());
    for (int64_t p = 0; p < ch.P; ++p) {
      const int64_t gp = ch.p0 + p;
      R.pair_chunk[gp] = k;
      if (layout) {
        rs_pair_layout& L = layout[gp];
        const PairRir& r = ch.h_rir[p];
        L.rir_len = r.len;
        L.rir_keep = r.keep;
        L.cutoff = b->eta_db > 0.0 ? r.cutoff : -1;
        L.fft_size = int64_t(1) << ch.ref[p].log2n;
        L.block_len = ch.ref[p].L;
        L.n_blocks = ch.ref[p].B;
        L.out_len = ch.plans[p].out_len;
        L.strategy = ch.strategy[p];
        L.flags = r.flags;
      }
      alg_bytes += 4.0 * ch.plans[p].nh;
    }
    for (int64_t u = ch.u0; u < ch.u1; ++u) {
      if (out_len) out_len[u] = ch.ulen[u - ch.u0];
      for (int64_t s = b->src_begin[u]; s < b->src_begin[u + 1]; ++s) alg_bytes += 4.0 * b->sig_len[s];
      alg_bytes += 4.0 * (b->mic_begin[u + 1] - b->mic_begin[u]) * ch.ulen[u - ch.u0];
    }
  };
  // ---- the pipeline: synth(k+1) is enqueued before the host plans chunk k -----------
  // Device renders synthesize every chunk's RIRs before the first filter (every chunk owns its
  // buffers): the K1 launches cover the host's planning of chunk 0, and no K1 runs beside the
  // K4 launches of earlier chunks.  Host renders (PCIe-bound) keep one chunk of look-ahead.
  static const int ahead_env = [] {
    const char* e = std::getenv("RSG_SYNTH_AHEAD");  // tuning override (chunks)
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int ahead = ahead_env ? ahead_env : (host_io ? 1 : std::max(1, nch));
  const bool serial = c->prof_level >= 2;
  for (int j = 0; j < nch && j < (serial ? 1 : ahead) && !status; ++j) {
    status = prep_chunk(b, R.chunks[j]);
    if (!status) status = enqueue_synth(c, b, R.chunks[j], R.sA);
  }
  for (int k = 0; k < kSigAhead && !status; ++k) status = enqueue_sig(k);
  // Profiling level 2 (the per-size K4 breakdown) serializes the whole render: chunk k+1's
  // synth waits for chunk k's filter, so no K1 runs beside the K4 launches being timed.
  for (int k = 0; k < nch && !status; ++k) {
    if (k + ahead < nch && !serial) {
      status = prep_chunk(b, R.chunks[k + ahead]);
      if (!status) status = enqueue_synth(c, b, R.chunks[k + ahead], R.sA);
      if (status) break;
    }
    R.hmark("plan wait " + std::to_string(k));
    const auto t0 = std::chrono::steady_clock::now();
    status = plan_chunk(b, R.chunks[k], out_stride);
    R.hmark("plan done " + std::to_string(k));
    t_plan += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (status) break;
    // Renders of fewer than two full chunks alternate their chunks between two filter streams (and
    // two lanes of K4 side streams): chunks share nothing, so chunk k + 1's K4 CTAs fill the tail
    // of chunk k's launches instead of waiting behind them (512 utterances: 4.36 -> 4.22 ms).  Full
    // renders measured the same either way (26.9 ms) and keep their launches in chunk order on one
    // stream.  RSG_LANES=1 / 2 forces the choice.
    static const int lanes_env = [] {
      const char* e = std::getenv("RSG_LANES");
      return e ? std::atoi(e) : 0;
    }();
    const bool two_lanes = lanes_env ? lanes_env >= 2 : small_total;
    const int lane = two_lanes ? (k & 1) : 0;
    cudaStream_t sBk = lane ? R.sB2 : R.sB;
    status = enqueue_filter(c, b, R.chunks[k], io, out_off, out_stride, sBk, R.sD, lane);
    if (!status) fill_layouts(R.chunks[k]);  // host work under the chunk's kernels
    if (serial && !status && k + 1 < nch) {
      RS_CUDA(cudaEventRecord(R.chunks[k].ev_out, sBk));
      RS_CUDA(cudaStreamWaitEvent(R.sA, R.chunks[k].ev_out, 0));
      status = prep_chunk(b, R.chunks[k + 1]);
      if (!status) status = enqueue_synth(c, b, R.chunks[k + 1], R.sA);
    }
    R.mark(sBk, "filter+mix enq-end " + std::to_string(k));
    R.mark(R.sD, "d2h done " + std::to_string(k));
    R.mark(R.sA, "sA at " + std::to_string(k));
    if (!status) status = enqueue_sig(k + kSigAhead);
  }
  // ---- join back into the caller's stream -------------------------------------------
  cudaEventRecord(R.ev_endA, R.sA);
  cudaEventRecord(R.ev_endB, R.sB);
  cudaEventRecord(R.ev_endB2, R.sB2);
  cudaEventRecord(R.ev_endH, R.sH);
  cudaEventRecord(R.ev_endD, R.sD);
  cudaStreamWaitEvent(c->stream, R.ev_endA, 0);
  cudaStreamWaitEvent(c->stream, R.ev_endB, 0);
  cudaStreamWaitEvent(c->stream, R.ev_endB2, 0);
  cudaStreamWaitEvent(c->stream, R.ev_endH, 0);
  cudaStreamWaitEvent(c->stream, R.ev_endD, 0);
  if (c->profiling) cudaEventRecord(c->st[6], c->stream);
  RS_CUDA(cudaStreamSynchronize(c->stream));
  R.hmark("sync done");
  if (c->prof_level >= 2) collect_k4_rows(c);
  c->launches += g_copy_launches;
  g_kernel_copies = false;
  R.dump();
  if (status) return status;
  c->host_plan_ms = t_plan;
  // ---- results, degenerate-power check, timing --------------------------------------
  c->h_plan.clear();
  c->h_pair.clear();
  double flops = 0, ola_ms = 0, syn_ms = 0, mix_ms = 0;
  // K4 device time: consecutive chunks run their K4 launches on alternating streams, so their
  // event windows may overlap — the union of the windows, not their sum.
  if (c->profiling && nch > 0) {
    std::vector<std::pair<float, float>> win(nch);
    for (int k = 0; k < nch; ++k) {
      RS_CUDA(cudaEventElapsedTime(&win[k].first, R.chunks[0].ev_k4a, R.chunks[k].ev_k4a));
      RS_CUDA(cudaEventElapsedTime(&win[k].second, R.chunks[0].ev_k4a, R.chunks[k].ev_k4b));
    }
    std::sort(win.begin(), win.end());
    float hi = win[0].first;
    for (const auto& w : win) {
      if (w.second > hi) ola_ms += w.second - std::max(w.first, hi);
      hi = std::max(hi, w.second);
    }
  }
  for (int k = 0; k < nch; ++k) {
    Chunk& ch = R.chunks[k];
    flops += ch.fp.flops;
    if (c->profiling) {
      float f;
      RS_CUDA(cudaEventElapsedTime(&f, ch.ev_syn0, ch.ev_syn1));
      syn_ms += f;
      RS_CUDA(cudaEventElapsedTime(&f, ch.ev_mix0, ch.ev_mix1));
      mix_ms += f;
    }
    for (int64_t p = 0; p < ch.P; ++p)
      if (ch.h_flags[p] & 4) return fail(RS_ERR_DEGENERATE, "signal has no energy: SNR gain undefined");
    if (gains) std::memcpy(gains + ch.p0, ch.h_gain, ch.P * sizeof(double));
    if (power) std::memcpy(power + ch.p0, ch.h_power, ch.P * sizeof(double));
  }
  const double bytes = alg_bytes;
  c->ola_flops = flops;
  c->alg_bytes = bytes;
  c->ola_ms = ola_ms;
  c->st_valid = false;
  c->stage_ms[0] = syn_ms;
  c->stage_ms[1] = 0;
  c->stage_ms[2] = 0;
  c->stage_ms[3] = 0;
  c->stage_ms[4] = ola_ms;
  c->stage_ms[5] = mix_ms;
  c->stage_valid = c->profiling;
  t_last_return = std::chrono::steady_clock::now();
  if (R.tracing)
    std::fprintf(stderr, "[trace] %lld of %lld channels mixed by the K4 epilogue\n",
                 static_cast<long long>(c->fused_channels), static_cast<long long>(c->mixed_channels));
  if (R.tracing)
    std::fprintf(stderr, "[trace] host return at %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t_last_return - R.trace_t0).count());
  return RS_OK;
}

int check_ctx(rs_ctx* c) {
  if (!c) return fail(RS_ERR_CONFIG, "null context");
  RS_CUDA(cudaSetDevice(c->device));
  return RS_OK;
}

// Convolution of one host pair through stage B at FFT size n (OLA).
int convolve_host(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh, size_t n,
                  double* out) {
  if (nx == 0) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
  if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  RS_TRY(checked_fft_size(n, nh, "overlap-add"));
  if (n > (static_cast<size_t>(2) << kLargeMaxLog2M))
    return fail(RS_ERR_UNSUPPORTED, "FFT size " + std::to_string(n) + " not supported by the device kernels");
  c->launches = 0;
  RS_TRY(c->scratch_a.ensure(std::max(nx, nh) * sizeof(double)));
  RS_TRY(c->sig.ensure(nx * sizeof(float)));
  RS_TRY(c->rir.ensure(nh * sizeof(double)));
  RS_CUDA(cudaMemcpyAsync(c->scratch_a.p, x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  RS_CUDA(launch_convert_d2f(c->scratch_a.as<double>(), c->sig.as<float>(), static_cast<int64_t>(nx), c->stream));
  RS_CUDA(cudaMemcpyAsync(c->rir.p, h, nh * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  PairMeta pm{};
  pm.sig_off = 0;
  pm.nx = static_cast<int64_t>(nx);
  pm.rir_off = 0;
  pm.rir_cap = static_cast<int64_t>(nh);
  std::vector<PairMeta> pv{pm};
  RS_TRY(upload(c, c->pair, pv));
  std::vector<PairPlan> plv(1);
  PairPlan& pl = plv[0];
  pl.log2n = log2_exact(n);
  pl.nh = static_cast<int64_t>(nh);
  pl.L = static_cast<int64_t>(n - nh + 1);
  pl.B = static_cast<int64_t>(block_count(nx, nh, n));
  pl.out_len = static_cast<int64_t>(nx + nh - 1);
  RS_TRY(state_init(c));
  FilterPlan fp;
  RS_TRY(plan_filter(plv, fp));
  FilterBufs& fb = c->rs->conv;
  RS_TRY(launch_filter(c, fb, fp, plv, c->pair.as<PairMeta>(), c->rir.as<double>(), c->sig.as<float>(), c->stream,
                       nullptr, c->profiling ? c->ev0 : nullptr, c->profiling ? c->ev1 : nullptr));
  const double flops = fp.flops;
  const size_t ol = nx + nh - 1;
  RS_TRY(c->scratch_b.ensure(ol * sizeof(double)));
  RS_CUDA(launch_convert_f2d(fb.y.as<float>(), c->scratch_b.as<double>(), static_cast<int64_t>(ol), c->stream));
  RS_CUDA(cudaMemcpyAsync(out, c->scratch_b.p, ol * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  if (c->prof_level >= 2) collect_k4_rows(c);
  RS_TRY(finish_timing(c));
  c->ola_flops = flops;
  c->alg_bytes = 4.0 * (nx + nh + ol);
  return RS_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }
const char* rs_version(void) { return "roomsim-b200 0.1 (sm_100a)"; }

int rs_ctx_create(int device, rs_ctx** out) {
  if (!out) return fail(RS_ERR_CONFIG, "null output pointer");
  auto* c = new rs_ctx();
  c->device = device;
  const int st = ctx_init(c);
  if (st != RS_OK) {
    delete c;
    return st;
  }
  *out = c;
  return RS_OK;
}

int rs_ctx_destroy(rs_ctx* c) {
  if (!c) return RS_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->tw_all, &c->utt, &c->pair, &c->rg, &c->items, &c->olaitems, &c->rir, &c->rirout,
                    &c->plan, &c->lists, &c->spec, &c->y, &c->sumsq, &c->gain, &c->power,
                    &c->flags, &c->snr, &c->chan_utt, &c->chan_mic, &c->chan_out, &c->utt_len,
                    &c->utt_stride, &c->utt_pair0, &c->utt_I, &c->utt_J, &c->sig, &c->out,
                    &c->scratch_a, &c->scratch_b};
  for (DevBuf* b : bufs) b->release();
  destroy_state(c);
  for (int i = 0; i < rs_ctx::kLanes * rs_ctx::kSide; ++i) {
    if (c->side[i]) cudaStreamDestroy(c->side[i]);
    if (c->side_join[i]) cudaEventDestroy(c->side_join[i]);
  }
  for (auto e : c->side_fork)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto& e : c->st)
    if (e) cudaEventDestroy(e);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return RS_OK;
}

int rs_ctx_set_stream(rs_ctx* c, void* stream) {
  RS_TRY(check_ctx(c));
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
  return RS_OK;
}

int rs_ctx_synchronize(rs_ctx* c) {
  RS_TRY(check_ctx(c));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  return RS_OK;
}

int rs_ctx_stage_times(rs_ctx* c, double* ms, int n, double* host_plan_ms) {
  RS_TRY(check_ctx(c));
  if (host_plan_ms) *host_plan_ms = c->host_plan_ms;
  for (int i = 0; i < n; ++i) ms[i] = (c->stage_valid && i < 6) ? c->stage_ms[i] : -1.0;
  return RS_OK;
}

int rs_ctx_set_profiling(rs_ctx* c, int enabled) {
  RS_TRY(check_ctx(c));
  c->profiling = enabled != 0;
  c->prof_level = enabled;
  return RS_OK;
}

int rs_ctx_k4_breakdown(rs_ctx* c, int cap, int32_t* log2n, int32_t* variant, int64_t* pairs, double* flops,
                        double* ms, double* exec_flops) {
  if (!c) return -fail(RS_ERR_CONFIG, "null context");
  const int n = static_cast<int>(c->k4_rows.size());
  for (int i = 0; i < n && i < cap; ++i) {
    const auto& r = c->k4_rows[i];
    if (log2n) log2n[i] = r.log2n;
    if (variant) variant[i] = r.var;
    if (pairs) pairs[i] = r.pairs;
    if (flops) flops[i] = r.flops;
    if (ms) ms[i] = r.ms;
    if (exec_flops) exec_flops[i] = r.exec_flops;
  }
  return n;
}

int rs_ctx_set_fused_mix(rs_ctx* c, int on) {
  if (!c) return fail(RS_ERR_CONFIG, "null context");
  c->fused_mix = on < 0 ? -1 : (on != 0);
  return RS_OK;
}

int rs_ctx_mix_counts(rs_ctx* c, int64_t* fused_channels, int64_t* channels) {
  if (!c) return fail(RS_ERR_CONFIG, "null context");
  if (fused_channels) *fused_channels = c->fused_channels;
  if (channels) *channels = c->mixed_channels;
  return RS_OK;
}

int rs_ctx_last_timing(rs_ctx* c, double* ola_ms, double* ola_flops, double* alg_bytes,
                       int64_t* launches) {
  RS_TRY(check_ctx(c));
  if (ola_ms) *ola_ms = c->ola_ms;
  if (ola_flops) *ola_flops = c->ola_flops;
  if (alg_bytes) *alg_bytes = c->alg_bytes;
  if (launches) *launches = c->launches;
  return RS_OK;
}

double rs_cost_direct(double I, double J, size_t nx, size_t nh) {
  if (cost_validate(I, J, nx, nh)) return NAN;
  return I * J * static_cast<double>(nx) * static_cast<double>(nh);
}
double rs_cost_full_fft(double I, double J, size_t nx, size_t nh, size_t n) {
  if (cost_validate(I, J, nx, nh) || checked_fft_size(n, nx + nh - 1, "full FFT")) return NAN;
  return cost_full_raw(I, J, n);
}
double rs_cost_ola(double I, double J, size_t nx, size_t nh, size_t n) {
  if (cost_validate(I, J, nx, nh) || checked_fft_size(n, nh, "overlap-add")) return NAN;
  return cost_ola_raw(I, J, nx, nh, n);
}
size_t rs_ola_block_count(size_t nx, size_t nh, size_t n) { return block_count(nx, nh, n); }
int rs_plan_for(double I, double J, size_t nx, size_t nh, int strategy, int* s, size_t* n, double* c) {
  return plan_for_impl(I, J, nx, nh, strategy, s, n, c);
}
int rs_choose_plan(double I, double J, size_t nx, size_t nh, int* s, size_t* n, double* c) {
  return choose_plan_impl(I, J, nx, nh, s, n, c);
}

static int rfft_common(rs_ctx* c, size_t n, size_t count, const double* in, double* out, bool inverse) {
  RS_TRY(check_ctx(c));
  if (n < 2 || !has_single_bit(n)) return fail(RS_ERR_PLAN, "FFT size must be a power of two >= 2");
  if (n > (static_cast<size_t>(2) << kLargeMaxLog2M))
    return fail(RS_ERR_UNSUPPORTED, "FFT size " + std::to_string(n) + " not supported by the device kernels");
  if (count == 0) return RS_OK;
  const int l = log2_exact(n) - 1;
  const bool large = l > kMaxLog2M;  // four-step stages (large.cu)
  const size_t M = n / 2;
  const size_t nin = count * (inverse ? 2 * (M + 1) : n);
  const size_t nout = count * (inverse ? n : 2 * (M + 1));
  RS_TRY(c->scratch_a.ensure(std::max(nin, nout) * sizeof(double)));
  RS_TRY(c->scratch_b.ensure(nin * sizeof(float)));
  RS_TRY(c->sig.ensure(nout * sizeof(float)));
  RS_CUDA(cudaMemcpyAsync(c->scratch_a.p, in, nin * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  RS_CUDA(launch_convert_d2f(c->scratch_a.as<double>(), c->scratch_b.as<float>(), static_cast<int64_t>(nin), c->stream));
  if (large) {
    int l1, l2;
    large_split(l, &l1, &l2);
    RS_TRY(state_init(c));
    FilterBufs& fb = c->rs->conv;
    RS_TRY(fb.scratch.ensure(count * M * sizeof(float2)));
    RS_CUDA(launch_large_rfft(l, inverse, c->scratch_b.as<float>(), reinterpret_cast<const float2*>(c->scratch_b.p),
                              c->sig.as<float>(), reinterpret_cast<float2*>(c->sig.p), static_cast<int>(count),
                              fb.scratch.as<float2>(), c->tw[l1], c->tw[l2], c->stream));
  } else if (inverse)
    RS_CUDA(launch_rfft(l, true, nullptr, reinterpret_cast<const float2*>(c->scratch_b.p), c->sig.as<float>(),
                        nullptr, static_cast<int>(count), c->tw[l], c->stream));
  else
    RS_CUDA(launch_rfft(l, false, c->scratch_b.as<float>(), nullptr, nullptr,
                        reinterpret_cast<float2*>(c->sig.p), static_cast<int>(count), c->tw[l], c->stream));
  RS_CUDA(launch_convert_f2d(c->sig.as<float>(), c->scratch_a.as<double>(), static_cast<int64_t>(nout), c->stream));
  RS_CUDA(cudaMemcpyAsync(out, c->scratch_a.p, nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  return RS_OK;
}

int rs_rfft_forward(rs_ctx* c, size_t n, size_t count, const double* in, double* out) {
  return rfft_common(c, n, count, in, out, false);
}
int rs_rfft_inverse(rs_ctx* c, size_t n, size_t count, const double* in, double* out) {
  return rfft_common(c, n, count, in, out, true);
}

int rs_synthesize_rir(rs_ctx* c, const double room_dims[3], double reflection, double sample_rate,
                      double speed_of_sound, int image_order, const double src[3], const double mic[3],
                      int64_t max_taps, double* out, size_t cap, size_t* len) {
  RS_TRY(check_ctx(c));
  // A one-utterance, one-pair batch through K1 + K2 (no truncation).
  const double fs = sample_rate, c0 = speed_of_sound, r = reflection;
  const int32_t K = image_order;
  const int64_t mt = max_taps;
  RS_TRY(room_validate(room_dims, r, fs, c0, K));
  if (!strictly_inside(room_dims, src)) return fail(RS_ERR_PLACEMENT, "source must lie strictly inside the room");
  if (!strictly_inside(room_dims, mic)) return fail(RS_ERR_PLACEMENT, "microphone must lie strictly inside the room");
  UttMeta um{};
  for (int a = 0; a < 3; ++a) um.dims[a] = room_dims[a];
  um.spm = fs / c0;
  um.order = K;
  um.rg_off = 0;
  um.max_taps = mt;
  std::vector<double> rg;
  for (int g = 0; g <= 3 * K; ++g) rg.push_back(std::pow(r, static_cast<double>(g)));
  const int64_t md = static_cast<int64_t>(lattice_max_delay(room_dims, src, mic, K, um.spm)) + 1;
  const int64_t capd = mt > 0 ? std::min<int64_t>(md, mt) : md;
  PairMeta pm{};
  for (int a = 0; a < 3; ++a) {
    pm.src[a] = src[a];
    pm.mic[a] = mic[a];
  }
  pm.rir_cap = capd;
  std::vector<SynthItem> items;
  int slice = 1;
  for (int64_t lo = 0; lo < capd; lo += kSynthSlice) {
    const int64_t l = std::min<int64_t>(kSynthSlice, capd - lo);
    items.push_back(SynthItem{0, static_cast<int32_t>(lo), static_cast<int32_t>(l), 0});
    slice = std::max<int>(slice, static_cast<int>(l));
  }
  RS_TRY(upload(c, c->utt, std::vector<UttMeta>{um}));
  RS_TRY(upload(c, c->pair, std::vector<PairMeta>{pm}));
  RS_TRY(upload(c, c->rg, rg));
  RS_TRY(upload(c, c->items, items));
  RS_TRY(c->rir.ensure(capd * sizeof(double)));
  RS_TRY(c->rirout.ensure(sizeof(PairRir)));
  RS_CUDA(cudaMemsetAsync(c->rirout.p, 0, sizeof(PairRir), c->stream));
  SynthArgs sa{c->utt.as<UttMeta>(), c->pair.as<PairMeta>(), c->rg.as<double>(), c->items.as<SynthItem>(),
               c->rir.as<double>(), c->rirout.as<PairRir>()};
  RS_CUDA(launch_synth(sa, static_cast<int>(items.size()), K, slice, c->stream));
  CutArgs ca{c->pair.as<PairMeta>(), c->utt.as<UttMeta>(), c->rir.as<double>(), c->rirout.as<PairRir>(), 0.0};
  RS_CUDA(launch_cut(ca, 1, c->stream));
  PairRir hr{};
  RS_CUDA(cudaMemcpyAsync(&hr, c->rirout.p, sizeof(PairRir), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  if (hr.flags & 1) return fail(RS_ERR_GEOMETRY, "microphone coincides with an image source");
  if (static_cast<size_t>(hr.len) > cap) return fail(RS_ERR_UNSUPPORTED, "RIR longer than output capacity");
  RS_CUDA(cudaMemcpy(out, c->rir.p, hr.len * sizeof(double), cudaMemcpyDeviceToHost));
  *len = static_cast<size_t>(hr.len);
  return RS_OK;
}

int rs_truncate_rir(rs_ctx* c, const double* h, size_t n, double eta_db, size_t* keep,
                    size_t* cutoff_index, double* threshold) {
  RS_TRY(check_ctx(c));
  if (n == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  if (eta_db <= 0.0) return fail(RS_ERR_CONFIG, "cut-off threshold must be positive dB");
  UttMeta um{};
  PairMeta pm{};
  pm.rir_cap = static_cast<int64_t>(n);
  RS_TRY(upload(c, c->utt, std::vector<UttMeta>{um}));
  RS_TRY(upload(c, c->pair, std::vector<PairMeta>{pm}));
  RS_TRY(c->rir.ensure(n * sizeof(double)));
  RS_TRY(c->rirout.ensure(sizeof(PairRir)));
  RS_CUDA(cudaMemcpyAsync(c->rir.p, h, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  PairRir init{};
  init.max_delay = n - 1;
  RS_CUDA(cudaMemcpyAsync(c->rirout.p, &init, sizeof(PairRir), cudaMemcpyHostToDevice, c->stream));
  CutArgs ca{c->pair.as<PairMeta>(), c->utt.as<UttMeta>(), c->rir.as<double>(), c->rirout.as<PairRir>(),
             std::pow(10.0, -eta_db / 10.0)};
  RS_CUDA(launch_cut(ca, 1, c->stream));
  PairRir hr{};
  RS_CUDA(cudaMemcpyAsync(&hr, c->rirout.p, sizeof(PairRir), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  if (hr.flags & 8) return fail(RS_ERR_CUDA, "internal: device RIR length exceeds the host bound");
  if (hr.flags & 2) return fail(RS_ERR_DEGENERATE, "all-zero impulse response has no power");
  if (keep) *keep = static_cast<size_t>(hr.keep);
  if (cutoff_index) *cutoff_index = static_cast<size_t>(hr.cutoff);
  if (threshold) *threshold = hr.threshold;
  return RS_OK;
}

int rs_convolve_ola(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh,
                    size_t fft_size, double* out) {
  RS_TRY(check_ctx(c));
  return convolve_host(c, x, nx, h, nh, fft_size, out);
}

int rs_convolve_full_fft(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh,
                         double* out) {
  RS_TRY(check_ctx(c));
  if (nx == 0) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
  if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  // One transform covering the whole output == a single OLA block (convolution.hpp:182-212).
  return convolve_host(c, x, nx, h, nh, fft_size_for(nx + nh - 1), out);
}

int rs_convolve_direct(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh, double* out) {
  RS_TRY(check_ctx(c));
  if (nx == 0) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
  if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  const size_t ol = nx + nh - 1;
  RS_TRY(c->scratch_a.ensure((nx + nh) * sizeof(double)));
  RS_TRY(c->scratch_b.ensure(ol * sizeof(double)));
  double* dx = c->scratch_a.as<double>();
  double* dh = dx + nx;
  RS_CUDA(cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  RS_CUDA(cudaMemcpyAsync(dh, h, nh * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev0, c->stream));
  RS_CUDA(launch_direct_conv(dx, static_cast<int64_t>(nx), dh, static_cast<int64_t>(nh), c->scratch_b.as<double>(),
                             c->stream));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev1, c->stream));
  RS_CUDA(cudaMemcpyAsync(out, c->scratch_b.p, ol * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_TRY(finish_timing(c));
  c->launches = 1;
  c->ola_flops = 2.0 * static_cast<double>(nx) * static_cast<double>(nh);
  c->alg_bytes = 8.0 * (nx + nh + ol);
  return RS_OK;
}

int rs_convolve(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh, int strategy,
                size_t fft_size, double* out) {
  RS_TRY(check_ctx(c));
  switch (strategy) {
    case RS_DIRECT:
      return rs_convolve_direct(c, x, nx, h, nh, out);
    case RS_FULL_FFT:
      return rs_convolve_full_fft(c, x, nx, h, nh, out);
    case RS_OVERLAP_ADD:
      if (fft_size == 0) return fail(RS_ERR_PLAN, "overlap-add plan is missing an FFT size");
      return convolve_host(c, x, nx, h, nh, fft_size, out);
  }
  return fail(RS_ERR_PLAN, "unknown strategy");
}

int64_t rs_batch_num_pairs(const rs_scene_batch* b) {
  if (!b) return 0;
  int64_t n = 0;
  for (int64_t u = 0; u < b->n_utt; ++u)
    n += (b->src_begin[u + 1] - b->src_begin[u]) * (b->mic_begin[u + 1] - b->mic_begin[u]);
  return n;
}

int rs_render_batch_device(rs_ctx* c, const rs_scene_batch* b, float* out_dev, const int64_t* out_off,
                           const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                           double* gains, double* power) {
  RS_TRY(check_ctx(c));
  if (!b) return fail(RS_ERR_CONFIG, "invalid scene batch");
  RenderIO io{b->signals, out_dev, nullptr, nullptr};
  return render_impl(c, b, io, out_off, out_stride, out_len, layout, gains, power);
}

int rs_render_batch(rs_ctx* c, const rs_scene_batch* b, float* out, const int64_t* out_off,
                    const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                    double* gains, double* power) {
  RS_TRY(check_ctx(c));
  if (!b) return fail(RS_ERR_CONFIG, "invalid scene batch");
  // Per-chunk H2D of the signal span (stream A) and D2H of the output span
  // (stream B) overlap the other chunks' kernels; pass page-locked buffers
  // for the copies to be asynchronous.
  int64_t sig_end = 0, out_end = 0;
  for (int64_t s = 0; s < (b->n_utt ? b->src_begin[b->n_utt] : 0); ++s)
    sig_end = std::max(sig_end, b->sig_off[s] + b->sig_len[s]);
  for (int64_t u = 0; u < b->n_utt; ++u)
    out_end = std::max(out_end, out_off[u] + (b->mic_begin[u + 1] - b->mic_begin[u]) * out_stride[u]);
  RS_TRY(c->sig.ensure(std::max<int64_t>(sig_end, 1) * sizeof(float)));
  RS_TRY(c->out.ensure(std::max<int64_t>(out_end, 1) * sizeof(float)));
  RenderIO io{c->sig.as<float>(), c->out.as<float>(), b->signals, out};
  return render_impl(c, b, io, out_off, out_stride, out_len, layout, gains, power);
}

static int locate_pair(rs_ctx* c, int64_t pair, Chunk** ch, int64_t* local) {
  if (!c->rs || pair < 0 || pair >= static_cast<int64_t>(c->rs->pair_chunk.size()))
    return fail(RS_ERR_CONFIG, "pair index out of range");
  *ch = &c->rs->chunks[c->rs->pair_chunk[pair]];
  *local = pair - (*ch)->p0;
  return RS_OK;
}

int rs_last_pair_signal(rs_ctx* c, int64_t pair, float* out, size_t cap, size_t* len) {
  RS_TRY(check_ctx(c));
  Chunk* ch;
  int64_t lp;
  RS_TRY(locate_pair(c, pair, &ch, &lp));
  const PairPlan& p = ch->plans[lp];
  if (static_cast<size_t>(p.out_len) > cap) return fail(RS_ERR_UNSUPPORTED, "capacity too small");
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_CUDA(cudaMemcpy(out, ch->fb.y.as<float>() + p.y_off, p.out_len * sizeof(float), cudaMemcpyDeviceToHost));
  *len = static_cast<size_t>(p.out_len);
  return RS_OK;
}

int rs_last_pair_rir(rs_ctx* c, int64_t pair, double* out, size_t cap, size_t* len) {
  RS_TRY(check_ctx(c));
  Chunk* ch;
  int64_t lp;
  RS_TRY(locate_pair(c, pair, &ch, &lp));
  const size_t n = static_cast<size_t>(ch->plans[lp].nh);
  if (n > cap) return fail(RS_ERR_UNSUPPORTED, "capacity too small");
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_CUDA(cudaMemcpy(out, ch->d_rir.as<double>() + ch->pair[lp].rir_off, n * sizeof(double), cudaMemcpyDeviceToHost));
  *len = n;
  return RS_OK;
}

}  // extern "C"

namespace {
// Periodic Hann window and the HTK-mel filterbank (FP64 on the host, once per context).
int logmel_tables(rs_ctx* c) {
  if (!c->lm_ready) {  // periodic Hann window and the HTK-mel filterbank, FP64 on the host
    const double pi = 3.14159265358979323846;
    std::vector<float> win(512);
    for (int n = 0; n < 512; ++n) win[n] = static_cast<float>(0.5 - 0.5 * std::cos(2.0 * pi * n / 512.0));
    auto mel = [](double f) { return 2595.0 * std::log10(1.0 + f / 700.0); };
    auto hz = [](double m) { return 700.0 * (std::pow(10.0, m / 2595.0) - 1.0); };
    const double m_lo = mel(125.0), m_hi = mel(7500.0);
    std::vector<double> edge(130);
    for (int i = 0; i < 130; ++i) edge[i] = hz(m_lo + (m_hi - m_lo) * i / 129.0);
    std::vector<int32_t> ptr(129, 0), bin;
    std::vector<float> w;
    for (int m = 0; m < 128; ++m) {
      for (int k = 0; k <= 256; ++k) {
        const double f = k * 16000.0 / 512.0;
        double v = 0.0;
        if (f > edge[m] && f <= edge[m + 1]) v = (f - edge[m]) / (edge[m + 1] - edge[m]);
        else if (f > edge[m + 1] && f < edge[m + 2]) v = (edge[m + 2] - f) / (edge[m + 2] - edge[m + 1]);
        if (v > 0.0) {
          bin.push_back(k);
          w.push_back(static_cast<float>(v));
        }
      }
      ptr[m + 1] = static_cast<int32_t>(bin.size());
    }
    RS_TRY(upload(c, c->lm_window, win));
    RS_TRY(upload(c, c->lm_ptr, ptr));
    RS_TRY(upload(c, c->lm_bin, bin));
    RS_TRY(upload(c, c->lm_w, w));
    c->lm_ready = true;
  }
  return RS_OK;
}
}  // namespace

extern "C" {

// ---- log-Mel front end ----------------------
int rs_logmel_shape(int64_t n_samples, int64_t* n_frames, int64_t* n_stacked) {
  const int64_t F = n_samples >= 512 ? 1 + (n_samples - 512) / 160 : 0;
  if (n_frames) *n_frames = F;
  if (n_stacked) *n_stacked = F >= 4 ? (F - 4) / 3 + 1 : 0;
  return RS_OK;
}

int rs_logmel_device(rs_ctx* c, const float* wave_dev, int64_t n_chan, const int64_t* chan_off,
                     const int64_t* chan_len, float* feat_dev, const int64_t* feat_off) {
  RS_TRY(check_ctx(c));
  RS_TRY(logmel_tables(c));
  // per-channel table only: the kernel derives a tile (8 frames) from its index
  std::vector<LogMelChan> chans(static_cast<size_t>(std::max<int64_t>(n_chan, 0)) + 1);
  int64_t n_tiles = 0;
  for (int64_t ch = 0; ch < n_chan; ++ch) {
    int64_t F, S;
    rs_logmel_shape(chan_len[ch], &F, &S);
    const int64_t used = S > 0 ? 3 * (S - 1) + 4 : 0;  // frames that reach a stacked vector
    chans[ch] = LogMelChan{chan_off[ch], feat_off[ch], static_cast<int32_t>(n_tiles), static_cast<int32_t>(S)};
    n_tiles += (used + 7) / 8;
  }
  if (n_tiles > INT32_MAX) return fail(RS_ERR_UNSUPPORTED, "too many log-Mel frames in one call");
  chans[n_chan] = LogMelChan{0, 0, static_cast<int32_t>(n_tiles), 0};
  c->launches = 0;
  if (n_tiles == 0) return RS_OK;
  RS_TRY(upload(c, c->lm_tiles, chans));
  LogMelArgs a{wave_dev, feat_dev, c->lm_tiles.as<LogMelChan>(), static_cast<int32_t>(n_chan),
               static_cast<int32_t>(n_tiles),
               c->lm_window.as<float>(), c->lm_ptr.as<int32_t>(), c->lm_bin.as<int32_t>(), c->lm_w.as<float>(),
               c->tw[8], 1e-10f};
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev0, c->stream));
  RS_CUDA(launch_logmel(a, c->stream));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev1, c->stream));
  c->launches = 1;
  RS_CUDA(cudaStreamSynchronize(c->stream));
  if (c->profiling) {
    float ms = 0;
    RS_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->ola_ms = ms;
  }
  return RS_OK;
}

int rs_render_features_device(rs_ctx* c, const rs_scene_batch* b, float* out_dev, const int64_t* out_off,
                              const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout, double* gains,
                              double* power, float* feat_dev, const int64_t* feat_off) {
  RS_TRY(check_ctx(c));
  if (!b) return fail(RS_ERR_CONFIG, "invalid scene batch");
  if (!feat_dev || !feat_off) return fail(RS_ERR_CONFIG, "features mode needs a feature buffer and offsets");
  RS_TRY(logmel_tables(c));
  if (out_dev) {
    // The waveforms are wanted too: they are mixed in the K4 launches' epilogue (mixfin.cuh) and
    // the log-Mel reads them back — measured faster than the mix + log-Mel kernel, which keeps the
    // whole mix out of the K4 launches (config 4: 26.9 + 10.9 ms vs 42.2 ms); same bytes
    // (test_fused_mix_logmel_matches_separate).  Without an output buffer the fused kernel runs
    // and no waveform is written.
    RenderIO io{b->signals, out_dev, nullptr, nullptr};
    std::vector<int64_t> len_tmp(static_cast<size_t>(std::max<int64_t>(b->n_utt, 1)));
    int64_t* ol = out_len ? out_len : len_tmp.data();
    RS_TRY(render_impl(c, b, io, out_off, out_stride, ol, layout, gains, power));
    const int64_t launches = c->launches;
    const double ola_ms = c->ola_ms;
    std::vector<int64_t> ch_off, ch_len;
    for (int64_t u = 0; u < b->n_utt; ++u)
      for (int64_t j = 0; j < b->mic_begin[u + 1] - b->mic_begin[u]; ++j) {
        ch_off.push_back(out_off[u] + j * out_stride[u]);
        ch_len.push_back(ol[u]);
      }
    RS_TRY(rs_logmel_device(c, out_dev, static_cast<int64_t>(ch_off.size()), ch_off.data(), ch_len.data(), feat_dev,
                            feat_off));
    c->launches += launches;
    c->ola_ms = ola_ms;
    return RS_OK;
  }
  RenderIO io{b->signals, out_dev, nullptr, nullptr};
  io.d_feat = feat_dev;
  io.feat_off = feat_off;
  return render_impl(c, b, io, out_off, out_stride, out_len, layout, gains, power);
}

}  // extern "C"

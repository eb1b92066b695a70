// api.cu — the C-ABI (include/roomsim_gpu.h) and the host-side orchestration
// of the hot path: validation with the reference's error taxonomy, the
// host-computed constants that must match glibc (r^g, 10^(-eta/10),
// 10^(snr/10)), the FFT-size planner (an exact mirror of
// roomsim/convolution.hpp:72-161), bucketing of pairs by transform size, and
// the kernel sequence K1 -> K2 -> plan -> K3 -> K4 -> K5 -> K6.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/roomsim_gpu.h"
#include "kernels.cuh"

using namespace rsg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

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
  float2* tw[kMaxLog2M + 1] = {};
  DevBuf tw_all;
  // arena
  DevBuf utt, pair, rg, items, olaitems, rir, rirout, plan, lists, spec, y, sumsq, gain, power, flags,
      snr, chan_utt, chan_mic, chan_out, utt_len, utt_stride, utt_pair0, utt_I, utt_J, sig, out,
      scratch_a, scratch_b;
  // last render (debug fetch)
  std::vector<PairPlan> h_plan;
  std::vector<PairMeta> h_pair;
  std::vector<PairRir> h_rir;
  int64_t last_pairs = 0;
  // timing of the last render
  double ola_ms = 0, ola_flops = 0, alg_bytes = 0;
  int64_t launches = 0;
};

namespace {

int ctx_init(rs_ctx* c) {
  RS_CUDA(cudaSetDevice(c->device));
  RS_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  RS_CUDA(cudaEventCreate(&c->ev0));
  RS_CUDA(cudaEventCreate(&c->ev1));
  for (auto& e : c->st) RS_CUDA(cudaEventCreate(&e));
  RS_CUDA(kernels_init());
  size_t total = 0;
  size_t off[kMaxLog2M + 1];
  for (int l = 0; l <= kMaxLog2M; ++l) {
    off[l] = total;
    total += static_cast<size_t>(tw_total(l));
  }
  std::vector<float2> h(total);
  for (int l = 0; l <= kMaxLog2M; ++l) fill_twiddles(l, h.data() + off[l]);
  RS_TRY(c->tw_all.ensure(total * sizeof(float2)));
  RS_CUDA(cudaMemcpy(c->tw_all.p, h.data(), total * sizeof(float2), cudaMemcpyHostToDevice));
  for (int l = 0; l <= kMaxLog2M; ++l) c->tw[l] = c->tw_all.as<float2>() + off[l];
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

// ---- stage B: spectrum + OLA over planned pairs (shared by render/convolve) ----
// Pairs are bucketed by transform size; buckets run largest work first.  Each
// pair's blocks are split into runs (K4 work items) long enough that the
// recomputed overlap blocks cost <= ~6%, short enough to fill the GPU.
int run_filter(rs_ctx* c, std::vector<PairPlan>& plans, const float* d_signals,
               const double* d_rir, double* flops_out) {
  const int64_t n_pairs = static_cast<int64_t>(plans.size());
  std::vector<std::vector<int32_t>> bucket(kMaxLog2M + 1);
  std::vector<double> work(n_pairs);
  double flops = 0;
  for (int64_t p = 0; p < n_pairs; ++p) {
    const int l = plans[p].log2n - 1;
    if (l < 0 || l > kMaxLog2M) return fail(RS_ERR_UNSUPPORTED, "FFT size outside the supported range");
    bucket[l].push_back(static_cast<int32_t>(p));
    work[p] = pair_flops(plans[p]);
    flops += work[p];
  }
  std::vector<int32_t> lists;
  std::vector<OlaItem> items;
  struct Span { int l; int64_t list_off, list_n, item_off, item_n; };
  std::vector<Span> spans;
  std::vector<int> order(kMaxLog2M + 1);
  std::iota(order.begin(), order.end(), 0);
  std::vector<double> bucket_work(kMaxLog2M + 1, 0.0);
  for (int l = 0; l <= kMaxLog2M; ++l)
    for (int32_t p : bucket[l]) bucket_work[l] += work[p];
  std::sort(order.begin(), order.end(), [&](int a, int b) { return bucket_work[a] > bucket_work[b]; });
  for (int l : order) {
    auto& v = bucket[l];
    if (v.empty()) continue;
    // largest pairs first (LPT) so the tail of the launch is short
    std::stable_sort(v.begin(), v.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
    int64_t total_blocks = 0;
    int64_t max_pre = 1;
    for (int32_t p : v) {
      total_blocks += plans[p].B;
      const int64_t n = int64_t(1) << plans[p].log2n;
      max_pre = std::max<int64_t>(max_pre, (n - plans[p].L + plans[p].L - 1) / plans[p].L);
    }
    const int64_t slots = 148LL * 2 * ola_groups(l);
    int64_t run = std::max<int64_t>((total_blocks + 4 * slots - 1) / (4 * slots), 16 * max_pre);
    Span sp{l, static_cast<int64_t>(lists.size()), static_cast<int64_t>(v.size()),
            static_cast<int64_t>(items.size()), 0};
    for (int32_t p : v) {
      PairPlan& pl = plans[p];
      const int64_t n = int64_t(1) << pl.log2n;
      const int64_t pre = (n - pl.L + pl.L - 1) / pl.L;  // ceil((N_h - 1) / L)
      pl.item0 = static_cast<int64_t>(items.size());
      pl.nitems = 0;
      for (int64_t r0 = 0; r0 < pl.B; r0 += run) {
        const int64_t r1 = std::min<int64_t>(pl.B, r0 + run);
        const int64_t b0 = r0 == 0 ? 0 : std::max<int64_t>(0, r0 - pre);
        items.push_back(OlaItem{p, static_cast<int32_t>(b0), static_cast<int32_t>(r0), static_cast<int32_t>(r1)});
        ++pl.nitems;
      }
    }
    sp.item_n = static_cast<int64_t>(items.size()) - sp.item_off;
    spans.push_back(sp);
    lists.insert(lists.end(), v.begin(), v.end());
  }
  RS_TRY(upload(c, c->lists, lists));
  RS_TRY(upload(c, c->plan, plans));
  RS_TRY(upload(c, c->olaitems, items));
  int64_t spec_total = 0, y_total = 0;
  for (const auto& p : plans) {
    spec_total = std::max<int64_t>(spec_total, p.spec_off + (int64_t(1) << (p.log2n - 1)) + 1);
    y_total = std::max<int64_t>(y_total, p.y_off + p.out_len);
  }
  RS_TRY(c->spec.ensure(std::max<int64_t>(spec_total, 1) * sizeof(float2)));
  RS_TRY(c->y.ensure(std::max<int64_t>(y_total, 1) * sizeof(float)));
  RS_TRY(c->sumsq.ensure(std::max<size_t>(items.size(), 1) * sizeof(double)));
  const int32_t* d_lists = c->lists.as<int32_t>();
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[3], c->stream));
  for (const Span& sp : spans) {
    SpecArgs a{d_lists + sp.list_off, static_cast<int32_t>(sp.list_n), c->pair.as<PairMeta>(),
               c->plan.as<PairPlan>(), d_rir, c->spec.as<float2>(), c->tw[sp.l]};
    RS_CUDA(launch_spectrum(sp.l, a, c->stream));
    ++c->launches;
  }
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev0, c->stream));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[4], c->stream));
  for (const Span& sp : spans) {
    OlaArgs a{c->olaitems.as<OlaItem>() + sp.item_off, static_cast<int32_t>(sp.item_n),
              c->pair.as<PairMeta>(), c->plan.as<PairPlan>(), d_signals, c->spec.as<float2>(),
              c->y.as<float>(), c->sumsq.as<double>() + sp.item_off, c->tw[sp.l]};
    RS_CUDA(launch_ola(sp.l, a, c->stream));
    ++c->launches;
  }
  if (c->profiling) RS_CUDA(cudaEventRecord(c->ev1, c->stream));
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[5], c->stream));
  if (flops_out) *flops_out = flops;
  return RS_OK;
}

int finish_timing(rs_ctx* c) {
  if (!c->profiling) return RS_OK;
  float ms = 0;
  RS_CUDA(cudaEventSynchronize(c->ev1));
  RS_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->ola_ms = ms;
  return RS_OK;
}

// ---- the batched render ------------------------------------------------------
struct RenderIO {
  const float* d_signals;  // device signals (already offset so sig_off indexes it)
  float* d_out;            // device output base
};

int render_impl(rs_ctx* c, const rs_scene_batch* b, const RenderIO& io, const int64_t* out_off,
                const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                double* gains, double* power) {
  if (!b || b->n_utt < 0) return fail(RS_ERR_CONFIG, "invalid scene batch");
  const int64_t U = b->n_utt;
  c->launches = 0;
  // ---- host validation + metadata -------------------------------------------
  std::vector<UttMeta> utt(U);
  std::vector<double> rg;
  std::vector<PairMeta> pairs;
  std::vector<int64_t> pair0(U + 1, 0);
  std::vector<int32_t> uI(U), uJ(U);
  std::vector<int> place_err;  // per pair: 0 ok, else status (in pair order)
  std::vector<std::string> place_msg;
  int max_order = 0;
  int64_t rir_total = 0;
  for (int64_t u = 0; u < U; ++u) {
    const double* L = b->room_dims + 3 * u;
    const int K = b->image_order[u];
    RS_TRY(room_validate(L, b->reflection[u], b->sample_rate[u], b->speed_of_sound[u], K));
    const int64_t s0 = b->src_begin[u], I = b->src_begin[u + 1] - s0;
    const int64_t m0 = b->mic_begin[u], J = b->mic_begin[u + 1] - m0;
    if (I < 1 || J < 1) return fail(RS_ERR_CONFIG, "scene needs a target and a microphone");
    uI[u] = static_cast<int32_t>(I);
    uJ[u] = static_cast<int32_t>(J);
    UttMeta& um = utt[u];
    for (int a = 0; a < 3; ++a) um.dims[a] = L[a];
    um.spm = b->sample_rate[u] / b->speed_of_sound[u];  // room_model.hpp:150
    um.order = K;
    um.rg_off = static_cast<int32_t>(rg.size());
    um.max_taps = b->max_taps ? b->max_taps[u] : 0;
    for (int g = 0; g <= 3 * K; ++g) rg.push_back(std::pow(b->reflection[u], static_cast<double>(g)));
    max_order = std::max(max_order, K);
    // RIR capacity: the horizon, or a bound on the farthest lattice image.
    int64_t cap = um.max_taps;
    if (cap <= 0) {
      double d2 = 0;
      for (int a = 0; a < 3; ++a) {
        const double e = (K + 2.0) * L[a];
        d2 += e * e;
      }
      cap = static_cast<int64_t>(std::ceil(std::sqrt(d2) * um.spm)) + 2;
    }
    pair0[u] = static_cast<int64_t>(pairs.size());
    for (int64_t i = 0; i < I; ++i)
      for (int64_t j = 0; j < J; ++j) {
        PairMeta pm{};
        const double* sp = b->src_pos + 3 * (s0 + i);
        const double* mp = b->mic_pos + 3 * (m0 + j);
        for (int a = 0; a < 3; ++a) {
          pm.src[a] = sp[a];
          pm.mic[a] = mp[a];
        }
        pm.utt = static_cast<int32_t>(u);
        pm.src_idx = static_cast<int32_t>(s0 + i);
        pm.mic_local = static_cast<int32_t>(j);
        pm.src_local = static_cast<int32_t>(i);
        pm.sig_off = b->sig_off[s0 + i];
        pm.nx = b->sig_len[s0 + i];
        pm.rir_off = rir_total;
        pm.rir_cap = cap;
        rir_total += cap;
        int err = RS_OK;
        std::string msg;
        if (!strictly_inside(L, sp)) {  // room_model.hpp:144-145
          err = RS_ERR_PLACEMENT;
          msg = "source must lie strictly inside the room";
        } else if (!strictly_inside(L, mp)) {  // :146-147
          err = RS_ERR_PLACEMENT;
          msg = "microphone must lie strictly inside the room";
        } else if (pm.nx <= 0) {
          err = RS_ERR_DEGENERATE;
          msg = "convolution input must be non-empty mono audio";
        }
        place_err.push_back(err);
        place_msg.push_back(msg);
        pairs.push_back(pm);
      }
  }
  pair0[U] = static_cast<int64_t>(pairs.size());
  const int64_t P = static_cast<int64_t>(pairs.size());
  c->last_pairs = P;
  // K1 work items: (pair, slice) for pairs with valid placements.
  std::vector<SynthItem> items;
  int slice = 1;
  for (int64_t p = 0; p < P; ++p) {
    if (place_err[p]) continue;
    const int64_t cap = pairs[p].rir_cap;
    for (int64_t lo = 0; lo < cap; lo += kSynthSlice) {
      const int64_t len = std::min<int64_t>(kSynthSlice, cap - lo);
      items.push_back(SynthItem{static_cast<int32_t>(p), static_cast<int32_t>(lo), static_cast<int32_t>(len), 0});
      slice = std::max<int>(slice, static_cast<int>(len));
    }
  }
  RS_TRY(upload(c, c->utt, utt));
  RS_TRY(upload(c, c->pair, pairs));
  RS_TRY(upload(c, c->rg, rg));
  RS_TRY(upload(c, c->items, items));
  RS_TRY(c->rir.ensure(std::max<int64_t>(rir_total, 1) * sizeof(double)));
  RS_TRY(c->rirout.ensure(std::max<int64_t>(P, 1) * sizeof(PairRir)));
  RS_CUDA(cudaMemsetAsync(c->rirout.p, 0, std::max<int64_t>(P, 1) * sizeof(PairRir), c->stream));
  // ---- K1 synth, K2 cut ---------------------------------------------------------
  c->st_valid = c->profiling;
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[0], c->stream));
  SynthArgs sa{c->utt.as<UttMeta>(), c->pair.as<PairMeta>(), c->rg.as<double>(),
               c->items.as<SynthItem>(), c->rir.as<double>(), c->rirout.as<PairRir>()};
  RS_CUDA(launch_synth(sa, static_cast<int>(items.size()), max_order, slice, c->stream));
  ++c->launches;
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[1], c->stream));
  const double eta_factor = b->eta_db > 0.0 ? std::pow(10.0, -b->eta_db / 10.0) : 0.0;
  CutArgs ca{c->pair.as<PairMeta>(), c->utt.as<UttMeta>(), c->rir.as<double>(),
             c->rirout.as<PairRir>(), eta_factor};
  RS_CUDA(launch_cut(ca, static_cast<int>(P), c->stream));
  ++c->launches;
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[2], c->stream));
  c->h_rir.resize(P);
  if (P)
    RS_CUDA(cudaMemcpyAsync(c->h_rir.data(), c->rirout.p, P * sizeof(PairRir), cudaMemcpyDeviceToHost,
                            c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  // ---- errors in reference order, then the planner --------------------------------
  const auto t_plan0 = std::chrono::steady_clock::now();
  std::vector<PairPlan> plans(P);
  std::vector<int64_t> ulen(U, 0);
  std::vector<int32_t> strategy(P, RS_OVERLAP_ADD);
  int64_t spec_off = 0, y_off = 0;
  for (int64_t p = 0; p < P; ++p) {
    if (place_err[p]) return fail(place_err[p], place_msg[p]);
    const PairRir& r = c->h_rir[p];
    if (r.flags & 1) return fail(RS_ERR_GEOMETRY, "microphone coincides with an image source");
    if (r.flags & 2) return fail(RS_ERR_DEGENERATE, "all-zero impulse response has no power");
    const size_t nh = static_cast<size_t>(r.keep);
    const size_t nx = static_cast<size_t>(pairs[p].nx);
    if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
    size_t n = 0;
    int s = RS_OVERLAP_ADD;
    double cost;
    if (b->plan_rule == RS_PLAN_CHOOSE) {
      RS_TRY(choose_plan_impl(1.0, 1.0, nx, nh, &s, &n, &cost));
      if (s == RS_FULL_FFT) n = fft_size_for(nx + nh - 1);
    } else if (b->plan_rule == RS_PLAN_FORCED) {
      n = static_cast<size_t>(b->forced_fft_size);
      RS_TRY(checked_fft_size(n, nh, "overlap-add"));
    } else if (b->plan_rule == RS_PLAN_POW2_TWICE) {
      n = bit_ceil_sz(2 * nh);
    } else {
      return fail(RS_ERR_CONFIG, "unknown plan rule");
    }
    if (n < 2 || n > (static_cast<size_t>(2) << kMaxLog2M))
      return fail(RS_ERR_UNSUPPORTED, "FFT size " + std::to_string(n) + " not supported by the device kernels");
    strategy[p] = s;
    PairPlan& pl = plans[p];
    pl.log2n = log2_exact(n);
    pl.nh = static_cast<int64_t>(nh);
    pl.L = static_cast<int64_t>(n - nh + 1);
    pl.B = static_cast<int64_t>(block_count(nx, nh, n));
    pl.out_len = static_cast<int64_t>(nx + nh - 1);
    pl.spec_off = spec_off;
    pl.y_off = y_off;
    spec_off += static_cast<int64_t>(n / 2 + 1);
    y_off += pl.out_len;
    ulen[pairs[p].utt] = std::max(ulen[pairs[p].utt], pl.out_len);
  }
  for (int64_t u = 0; u < U; ++u)
    if (out_stride[u] < ulen[u]) return fail(RS_ERR_CONFIG, "output stride too small");
  // ---- K3 + K4 -------------------------------------------------------------------
  c->host_plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_plan0).count();
  double flops = 0;
  RS_TRY(run_filter(c, plans, io.d_signals, c->rir.as<double>(), &flops));
  // ---- K5 gains + K6 mix ------------------------------------------------------------
  std::vector<double> snr_lin(b->src_begin[U]);
  for (int64_t s = 0; s < b->src_begin[U]; ++s) snr_lin[s] = std::pow(10.0, b->snr_db[s] / 10.0);
  RS_TRY(upload(c, c->snr, snr_lin));
  std::vector<int64_t> pair0v(pair0.begin(), pair0.end() - 1);
  RS_TRY(upload(c, c->utt_pair0, pair0v));
  RS_TRY(upload(c, c->utt_I, uI));
  RS_TRY(upload(c, c->utt_J, uJ));
  RS_TRY(c->gain.ensure(std::max<int64_t>(P, 1) * sizeof(double)));
  RS_TRY(c->power.ensure(std::max<int64_t>(P, 1) * sizeof(double)));
  RS_TRY(c->flags.ensure(std::max<int64_t>(P, 1) * sizeof(int32_t)));
  RS_CUDA(cudaMemsetAsync(c->flags.p, 0, std::max<int64_t>(P, 1) * sizeof(int32_t), c->stream));
  GainArgs ga{c->pair.as<PairMeta>(), c->plan.as<PairPlan>(), c->utt_pair0.as<int64_t>(),
              c->utt_J.as<int32_t>(), c->sumsq.as<double>(), c->snr.as<double>(), c->gain.as<double>(),
              c->power.as<double>(), c->flags.as<int32_t>(), P};
  RS_CUDA(launch_gain(ga, c->stream));
  ++c->launches;
  std::vector<int64_t> ch_utt, ch_out, ustride(out_stride, out_stride + U);
  std::vector<int32_t> ch_mic;
  int64_t max_stride = 0;
  for (int64_t u = 0; u < U; ++u) {
    max_stride = std::max(max_stride, out_stride[u]);
    for (int32_t j = 0; j < uJ[u]; ++j) {
      ch_utt.push_back(u);
      ch_mic.push_back(j);
      ch_out.push_back(out_off[u] + j * out_stride[u]);
    }
  }
  RS_TRY(upload(c, c->chan_utt, ch_utt));
  RS_TRY(upload(c, c->chan_mic, ch_mic));
  RS_TRY(upload(c, c->chan_out, ch_out));
  RS_TRY(upload(c, c->utt_len, ulen));
  RS_TRY(upload(c, c->utt_stride, ustride));
  MixArgs ma{c->chan_utt.as<int64_t>(), c->chan_mic.as<int32_t>(), c->chan_out.as<int64_t>(),
             c->utt_len.as<int64_t>(), c->utt_stride.as<int64_t>(), c->utt_pair0.as<int64_t>(),
             c->utt_I.as<int32_t>(), c->utt_J.as<int32_t>(), c->plan.as<PairPlan>(), c->y.as<float>(),
             c->gain.as<double>(), io.d_out, 4096};
  RS_CUDA(launch_mix(ma, static_cast<int64_t>(ch_utt.size()), max_stride, c->stream));
  ++c->launches;
  if (c->profiling) RS_CUDA(cudaEventRecord(c->st[6], c->stream));
  // ---- results, degenerate-power check --------------------------------------------
  std::vector<int32_t> hflags(P);
  std::vector<double> hgain(P), hpower(P);
  if (P) {
    RS_CUDA(cudaMemcpyAsync(hflags.data(), c->flags.p, P * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    RS_CUDA(cudaMemcpyAsync(hgain.data(), c->gain.p, P * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    RS_CUDA(cudaMemcpyAsync(hpower.data(), c->power.p, P * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_TRY(finish_timing(c));
  c->ola_flops = flops;
  // algorithmic bytes: sources once, RIR taps once, mic outputs once
  double bytes = 0;
  for (int64_t u = 0; u < U; ++u) {
    for (int64_t s = b->src_begin[u]; s < b->src_begin[u + 1]; ++s) bytes += 4.0 * b->sig_len[s];
    bytes += 4.0 * uJ[u] * ulen[u];
  }
  for (const auto& pl : plans) bytes += 4.0 * pl.nh;
  c->alg_bytes = bytes;
  for (int64_t p = 0; p < P; ++p)
    if (hflags[p] & 4) return fail(RS_ERR_DEGENERATE, "signal has no energy: SNR gain undefined");
  c->h_plan = plans;
  c->h_pair = pairs;
  if (out_len)
    for (int64_t u = 0; u < U; ++u) out_len[u] = ulen[u];
  for (int64_t p = 0; p < P; ++p) {
    if (layout) {
      rs_pair_layout& L = layout[p];
      L.rir_len = c->h_rir[p].len;
      L.rir_keep = c->h_rir[p].keep;
      L.cutoff = b->eta_db > 0.0 ? c->h_rir[p].cutoff : -1;
      L.fft_size = int64_t(1) << plans[p].log2n;
      L.block_len = plans[p].L;
      L.n_blocks = plans[p].B;
      L.out_len = plans[p].out_len;
      L.strategy = strategy[p];
      L.flags = c->h_rir[p].flags;
    }
    if (gains) gains[p] = hgain[p];
    if (power) power[p] = hpower[p];
  }
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
  if (n > (static_cast<size_t>(2) << kMaxLog2M))
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
  double flops = 0;
  RS_TRY(run_filter(c, plv, c->sig.as<float>(), c->rir.as<double>(), &flops));
  const size_t ol = nx + nh - 1;
  RS_TRY(c->scratch_b.ensure(ol * sizeof(double)));
  RS_CUDA(launch_convert_f2d(c->y.as<float>(), c->scratch_b.as<double>(), static_cast<int64_t>(ol), c->stream));
  RS_CUDA(cudaMemcpyAsync(out, c->scratch_b.p, ol * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
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
  for (int i = 0; i < n; ++i) ms[i] = -1.0;
  if (!c->st_valid) return RS_OK;
  RS_CUDA(cudaEventSynchronize(c->st[rs_ctx::kStages - 1]));
  for (int i = 0; i + 1 < rs_ctx::kStages && i < n; ++i) {
    float f = 0;
    RS_CUDA(cudaEventElapsedTime(&f, c->st[i], c->st[i + 1]));
    ms[i] = f;
  }
  return RS_OK;
}

int rs_ctx_set_profiling(rs_ctx* c, int enabled) {
  RS_TRY(check_ctx(c));
  c->profiling = enabled != 0;
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
  if (n > (static_cast<size_t>(2) << kMaxLog2M))
    return fail(RS_ERR_UNSUPPORTED, "FFT size " + std::to_string(n) + " not supported by the device kernels");
  if (count == 0) return RS_OK;
  const int l = log2_exact(n) - 1;
  const size_t M = n / 2;
  const size_t nin = count * (inverse ? 2 * (M + 1) : n);
  const size_t nout = count * (inverse ? n : 2 * (M + 1));
  RS_TRY(c->scratch_a.ensure(std::max(nin, nout) * sizeof(double)));
  RS_TRY(c->scratch_b.ensure(nin * sizeof(float)));
  RS_TRY(c->sig.ensure(nout * sizeof(float)));
  RS_CUDA(cudaMemcpyAsync(c->scratch_a.p, in, nin * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  RS_CUDA(launch_convert_d2f(c->scratch_a.as<double>(), c->scratch_b.as<float>(), static_cast<int64_t>(nin), c->stream));
  if (inverse)
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
  int64_t capd = mt;
  if (capd <= 0) {
    double d2 = 0;
    for (int a = 0; a < 3; ++a) {
      const double e = (K + 2.0) * room_dims[a];
      d2 += e * e;
    }
    capd = static_cast<int64_t>(std::ceil(std::sqrt(d2) * um.spm)) + 2;
  }
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

int rs_convolve(rs_ctx* c, const double* x, size_t nx, const double* h, size_t nh, int strategy,
                size_t fft_size, double* out) {
  RS_TRY(check_ctx(c));
  switch (strategy) {
    case RS_DIRECT:
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
  RenderIO io{b->signals, out_dev};
  return render_impl(c, b, io, out_off, out_stride, out_len, layout, gains, power);
}

int rs_render_batch(rs_ctx* c, const rs_scene_batch* b, float* out, const int64_t* out_off,
                    const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                    double* gains, double* power) {
  RS_TRY(check_ctx(c));
  if (!b) return fail(RS_ERR_CONFIG, "invalid scene batch");
  // H2D of the signal span, render on device, D2H of the output span.
  int64_t sig_end = 0, out_end = 0;
  for (int64_t s = 0; s < (b->n_utt ? b->src_begin[b->n_utt] : 0); ++s)
    sig_end = std::max(sig_end, b->sig_off[s] + b->sig_len[s]);
  for (int64_t u = 0; u < b->n_utt; ++u)
    out_end = std::max(out_end, out_off[u] + (b->mic_begin[u + 1] - b->mic_begin[u]) * out_stride[u]);
  RS_TRY(c->sig.ensure(std::max<int64_t>(sig_end, 1) * sizeof(float)));
  RS_TRY(c->out.ensure(std::max<int64_t>(out_end, 1) * sizeof(float)));
  if (sig_end)
    RS_CUDA(cudaMemcpyAsync(c->sig.p, b->signals, sig_end * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  RenderIO io{c->sig.as<float>(), c->out.as<float>()};
  RS_TRY(render_impl(c, b, io, out_off, out_stride, out_len, layout, gains, power));
  if (out_end)
    RS_CUDA(cudaMemcpyAsync(out, c->out.p, out_end * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  RS_CUDA(cudaStreamSynchronize(c->stream));
  return RS_OK;
}

int rs_last_pair_signal(rs_ctx* c, int64_t pair, float* out, size_t cap, size_t* len) {
  RS_TRY(check_ctx(c));
  if (pair < 0 || pair >= static_cast<int64_t>(c->h_plan.size())) return fail(RS_ERR_CONFIG, "pair index out of range");
  const PairPlan& p = c->h_plan[pair];
  if (static_cast<size_t>(p.out_len) > cap) return fail(RS_ERR_UNSUPPORTED, "capacity too small");
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_CUDA(cudaMemcpy(out, c->y.as<float>() + p.y_off, p.out_len * sizeof(float), cudaMemcpyDeviceToHost));
  *len = static_cast<size_t>(p.out_len);
  return RS_OK;
}

int rs_last_pair_rir(rs_ctx* c, int64_t pair, double* out, size_t cap, size_t* len) {
  RS_TRY(check_ctx(c));
  if (pair < 0 || pair >= static_cast<int64_t>(c->h_plan.size())) return fail(RS_ERR_CONFIG, "pair index out of range");
  const size_t n = static_cast<size_t>(c->h_plan[pair].nh);
  if (n > cap) return fail(RS_ERR_UNSUPPORTED, "capacity too small");
  RS_CUDA(cudaStreamSynchronize(c->stream));
  RS_CUDA(cudaMemcpy(out, c->rir.as<double>() + c->h_pair[pair].rir_off, n * sizeof(double), cudaMemcpyDeviceToHost));
  *len = n;
  return RS_OK;
}

}  // extern "C"

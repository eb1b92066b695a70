// roomsim_gpu.hpp — drop-in C++ adapter: the reference's API in the
// reference's own types (roomsim::RoomConfig, Placement, Rir, AudioBuffer,
// ConvolutionPlan; /root/reference/proj/include/roomsim/X.hpp), executed on
// the B200 through the C-ABI of roomsim_gpu.h.  Header-only; include it after
// (or instead of) the reference headers and link libroomsim_gpu.so.
//
//   roomsim::gpu::synthesize_rir    replaces roomsim::synthesize_rir   (room_model.hpp:141-174)
//   roomsim::gpu::truncate_rir      replaces roomsim::truncate_rir     (room_model.hpp:203-213)
//   roomsim::gpu::convolve_ola      replaces roomsim::convolve_ola     (convolution.hpp:219-255)
//   roomsim::gpu::convolve_full_fft replaces roomsim::convolve_full_fft(convolution.hpp:182-212)
//   roomsim::gpu::convolve_direct   replaces roomsim::convolve_direct  (convolution.hpp:164-179), FP64 bit-exact
//   roomsim::gpu::convolve          replaces roomsim::convolve         (convolution.hpp:258-271)
//   roomsim::gpu::CudaRealFft       a RealFftEngine (fft.hpp:38-49) for the templated reference
//                                   functions: roomsim::convolve_ola<roomsim::gpu::CudaRealFft>
//   roomsim::gpu::render_batch      SPEC.md:348-356 render over many scenes at once (the hot path)
//
// Errors: every non-zero C-ABI status is rethrown as the matching reference
// exception class (errors.hpp:22-68); device failures throw roomsim::Error.
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "roomsim/audio_buffer.hpp"
#include "roomsim/convolution.hpp"
#include "roomsim/errors.hpp"
#include "roomsim/fft.hpp"
#include "roomsim/room_model.hpp"
#include "roomsim_gpu.h"

namespace roomsim::gpu {

[[noreturn]] inline void throw_status(int st) {
  const std::string msg = rs_last_error();
  switch (st) {
    case RS_ERR_PLACEMENT: throw PlacementError(msg);
    case RS_ERR_GEOMETRY: throw GeometryError(msg);
    case RS_ERR_DEGENERATE: throw DegenerateInputError(msg);
    case RS_ERR_PLAN: throw PlanError(msg);
    case RS_ERR_CONFIG: throw ConfigError(msg);
    case RS_ERR_FORMAT: throw FormatError(msg);
    case RS_ERR_IO: throw IoError(msg);
    default: throw Error("roomsim_gpu: " + msg);
  }
}
inline void check(int st) {
  if (st != RS_OK) throw_status(st);
}

// One device, one stream, one arena.  Not shared between threads
// (the reference's engine rule, fft.hpp:36-37).
class Context {
 public:
  explicit Context(int device = 0) { check(rs_ctx_create(device, &ctx_)); }
  ~Context() { rs_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rs_ctx* get() const { return ctx_; }

 private:
  rs_ctx* ctx_ = nullptr;
};

// Per-thread default context (device 0).
inline Context& default_context() {
  thread_local Context ctx(0);
  return ctx;
}

// ---- room model -------------------------------------------------------------
inline Rir synthesize_rir(const RoomConfig& room, const Placement& source, const Placement& mic,
                          int64_t max_taps = 0, Context& ctx = default_context()) {
  const double dims[3] = {room.dimensions.x, room.dimensions.y, room.dimensions.z};
  const double s[3] = {source.position.x, source.position.y, source.position.z};
  const double m[3] = {mic.position.x, mic.position.y, mic.position.z};
  double ext2 = 0;
  for (double L : dims) ext2 += ((room.image_order + 2.0) * L) * ((room.image_order + 2.0) * L);
  size_t cap = static_cast<size_t>(std::ceil(std::sqrt(ext2) * room.sample_rate / room.speed_of_sound)) + 4;
  if (max_taps > 0 && static_cast<size_t>(max_taps) < cap) cap = static_cast<size_t>(max_taps);
  Rir rir;
  rir.sample_rate = room.sample_rate;
  rir.samples.resize(cap);
  size_t len = 0;
  check(rs_synthesize_rir(ctx.get(), dims, room.reflection_coefficient, room.sample_rate,
                          room.speed_of_sound, room.image_order, s, m, max_taps, rir.samples.data(),
                          cap, &len));
  rir.samples.resize(len);
  return rir;
}

inline Rir truncate_rir(const Rir& rir, double eta_db, Context& ctx = default_context()) {
  size_t keep = 0, nc = 0;
  double th = 0;
  check(rs_truncate_rir(ctx.get(), rir.samples.data(), rir.samples.size(), eta_db, &keep, &nc, &th));
  Rir out;
  out.sample_rate = rir.sample_rate;
  out.truncation_db = eta_db;
  out.samples.assign(rir.samples.begin(), rir.samples.begin() + static_cast<std::ptrdiff_t>(keep));
  return out;
}

// ---- planner (host, bit-identical to the reference) ------------------------------
inline ConvolutionPlan choose_plan(const CostInputs& c) {
  int s = 0;
  size_t n = 0;
  double cost = 0;
  check(rs_choose_plan(c.num_sources, c.num_mics, c.signal_len, c.rir_len, &s, &n, &cost));
  ConvolutionPlan p;
  p.strategy = s == RS_DIRECT ? Strategy::direct : (s == RS_FULL_FFT ? Strategy::full_fft : Strategy::overlap_add);
  if (s != RS_DIRECT) p.fft_size = n;
  p.predicted_cost = cost;
  return p;
}

// ---- convolution ------------------------------------------------------------------
namespace detail {
inline void check_io(const AudioBuffer& x, const Rir& h) {  // convolution.hpp:221-226
  x.validate();
  if (!x.is_mono() || x.num_frames() == 0)
    throw DegenerateInputError("convolution input must be non-empty mono audio");
  if (h.samples.empty()) throw DegenerateInputError("empty impulse response");
  if (x.sample_rate != h.sample_rate) throw ConfigError("signal and RIR sample rates differ");
}
}  // namespace detail

inline AudioBuffer convolve_ola(const AudioBuffer& x, const Rir& h, std::size_t fft_size,
                                Context& ctx = default_context()) {
  detail::check_io(x, h);
  std::vector<double> out(x.num_frames() + h.samples.size() - 1);
  check(rs_convolve_ola(ctx.get(), x.channel(0).data(), x.num_frames(), h.samples.data(),
                        h.samples.size(), fft_size, out.data()));
  return AudioBuffer::mono(std::move(out), x.sample_rate);
}

inline AudioBuffer convolve_full_fft(const AudioBuffer& x, const Rir& h, Context& ctx = default_context()) {
  detail::check_io(x, h);
  std::vector<double> out(x.num_frames() + h.samples.size() - 1);
  check(rs_convolve_full_fft(ctx.get(), x.channel(0).data(), x.num_frames(), h.samples.data(),
                             h.samples.size(), out.data()));
  return AudioBuffer::mono(std::move(out), x.sample_rate);
}

inline AudioBuffer convolve_direct(const AudioBuffer& x, const Rir& h, Context& ctx = default_context()) {
  detail::check_io(x, h);
  std::vector<double> out(x.num_frames() + h.samples.size() - 1);
  check(rs_convolve_direct(ctx.get(), x.channel(0).data(), x.num_frames(), h.samples.data(),
                           h.samples.size(), out.data()));
  return AudioBuffer::mono(std::move(out), x.sample_rate);
}

inline AudioBuffer convolve(const AudioBuffer& x, const Rir& h, const ConvolutionPlan& plan,
                            Context& ctx = default_context()) {
  switch (plan.strategy) {
    case Strategy::direct:
      return convolve_direct(x, h, ctx);
    case Strategy::full_fft:
      return convolve_full_fft(x, h, ctx);
    case Strategy::overlap_add:
      if (!plan.fft_size) throw PlanError("overlap-add plan is missing an FFT size");
      return convolve_ola(x, h, *plan.fft_size, ctx);
  }
  throw PlanError("unknown strategy");
}

// ---- RealFftEngine on the device (fft.hpp:38-49) ------------------------------------
// Satisfies roomsim::RealFftEngine, so the reference's own templated functions
// run their transforms on the B200: roomsim::convolve_ola<CudaRealFft>(x, h, N).
// (Per-transform round trips: correct, but the batched calls above are the
// fast path.)
class CudaRealFft {
 public:
  explicit CudaRealFft(std::size_t size) : size_(size) {
    if (size < 2 || (size & (size - 1)) != 0) throw PlanError("FFT size must be a power of two >= 2");
  }
  std::size_t size() const { return size_; }
  std::size_t spectrum_size() const { return size_ / 2 + 1; }
  void forward(std::span<const double> in, std::span<std::complex<double>> out) {
    if (in.size() != size_) throw PlanError("sample span does not match FFT size");
    if (out.size() != spectrum_size()) throw PlanError("spectrum span does not match FFT size");
    check(rs_rfft_forward(default_context().get(), size_, 1, in.data(), reinterpret_cast<double*>(out.data())));
  }
  void inverse(std::span<const std::complex<double>> in, std::span<double> out) {
    if (out.size() != size_) throw PlanError("sample span does not match FFT size");
    if (in.size() != spectrum_size()) throw PlanError("spectrum span does not match FFT size");
    check(rs_rfft_inverse(default_context().get(), size_, 1, reinterpret_cast<const double*>(in.data()),
                          out.data()));
  }

 private:
  std::size_t size_;
};
static_assert(RealFftEngine<CudaRealFft>);

// ---- SPEC render over a batch of scenes (the hot path) --------------------------------
struct Scene {  // one target + noises, per-mic RIRs synthesized on device
  RoomConfig room;
  std::vector<Placement> sources;  // [0] is the target
  std::vector<Placement> mics;
  std::vector<AudioBuffer> signals;  // one mono buffer per source
  std::vector<double> snr_db;        // per source ([0] unused)
  int64_t max_taps = 0;              // RIR horizon (0 = full lattice)
};

struct MixOutput {
  std::vector<AudioBuffer> channels;         // per scene: J channels of equal length
  std::vector<std::vector<double>> gains;    // per scene: alpha, [i * J + j]
};

// eta_db > 0 applies truncate_rir(h, eta_db); plan_rule is an rs_plan_rule.
inline MixOutput render_batch(const std::vector<Scene>& scenes, double eta_db = 0.0,
                              int plan_rule = RS_PLAN_CHOOSE, int64_t forced_fft_size = 0,
                              Context& ctx = default_context()) {
  const int64_t U = static_cast<int64_t>(scenes.size());
  std::vector<int64_t> sb{0}, mb{0}, max_taps, sig_off, sig_len, out_off, out_stride;
  std::vector<double> dims, refl, fs, c0, spos, mpos, snr;
  std::vector<int32_t> order;
  std::vector<float> sig;
  int64_t out_total = 0;
  for (const Scene& s : scenes) {
    s.room.validate();
    sb.push_back(sb.back() + static_cast<int64_t>(s.sources.size()));
    mb.push_back(mb.back() + static_cast<int64_t>(s.mics.size()));
    dims.insert(dims.end(), {s.room.dimensions.x, s.room.dimensions.y, s.room.dimensions.z});
    refl.push_back(s.room.reflection_coefficient);
    fs.push_back(s.room.sample_rate);
    c0.push_back(s.room.speed_of_sound);
    order.push_back(s.room.image_order);
    max_taps.push_back(s.max_taps);
    int64_t nx_max = 0;
    for (size_t i = 0; i < s.sources.size(); ++i) {
      const auto& p = s.sources[i].position;
      spos.insert(spos.end(), {p.x, p.y, p.z});
      snr.push_back(i < s.snr_db.size() ? s.snr_db[i] : 0.0);
      const auto& ch = s.signals.at(i).channel(0);
      sig_off.push_back(static_cast<int64_t>(sig.size()));
      sig_len.push_back(static_cast<int64_t>(ch.size()));
      nx_max = std::max<int64_t>(nx_max, static_cast<int64_t>(ch.size()));
      for (double v : ch) sig.push_back(static_cast<float>(v));
    }
    for (const auto& m : s.mics) mpos.insert(mpos.end(), {m.position.x, m.position.y, m.position.z});
    double ext2 = 0;
    for (double L : {s.room.dimensions.x, s.room.dimensions.y, s.room.dimensions.z})
      ext2 += ((s.room.image_order + 2.0) * L) * ((s.room.image_order + 2.0) * L);
    const int64_t lattice =
        static_cast<int64_t>(std::ceil(std::sqrt(ext2) * s.room.sample_rate / s.room.speed_of_sound)) + 4;
    const int64_t cap = s.max_taps > 0 ? s.max_taps : lattice;
    out_off.push_back(out_total);
    out_stride.push_back(nx_max + cap - 1);
    out_total += (nx_max + cap - 1) * static_cast<int64_t>(s.mics.size());
  }
  rs_scene_batch b{};
  b.n_utt = U;
  b.src_begin = sb.data();
  b.mic_begin = mb.data();
  b.room_dims = dims.data();
  b.reflection = refl.data();
  b.sample_rate = fs.data();
  b.speed_of_sound = c0.data();
  b.image_order = order.data();
  b.max_taps = max_taps.data();
  b.src_pos = spos.data();
  b.mic_pos = mpos.data();
  b.snr_db = snr.data();
  b.sig_off = sig_off.data();
  b.sig_len = sig_len.data();
  b.signals = sig.data();
  b.eta_db = eta_db;
  b.plan_rule = plan_rule;
  b.forced_fft_size = forced_fft_size;
  std::vector<float> out(static_cast<size_t>(out_total));
  std::vector<int64_t> out_len(static_cast<size_t>(U));
  std::vector<double> gains(static_cast<size_t>(rs_batch_num_pairs(&b)));
  check(rs_render_batch(ctx.get(), &b, out.data(), out_off.data(), out_stride.data(), out_len.data(),
                        nullptr, gains.data(), nullptr));
  MixOutput res;
  int64_t p0 = 0;
  for (int64_t u = 0; u < U; ++u) {
    const int64_t J = mb[u + 1] - mb[u], I = sb[u + 1] - sb[u];
    std::vector<std::vector<double>> chans;
    for (int64_t j = 0; j < J; ++j) {
      const float* y = out.data() + out_off[u] + j * out_stride[u];
      chans.emplace_back(y, y + out_len[u]);
    }
    res.channels.emplace_back(std::move(chans), scenes[u].room.sample_rate);
    res.gains.emplace_back(gains.begin() + p0, gains.begin() + p0 + I * J);
    p0 += I * J;
  }
  return res;
}

}  // namespace roomsim::gpu

// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include,
// passed with -I by oracle/Makefile; nothing is copied) into
// oracle/_ref/libroomsim_ref.so and exposes the reference's own functions
// through a C ABI with the same signatures as oracle/roomsim_oracle.h
// (prefix ref_ instead of orc_).  It is used
//   * to pin the plain-C restatement (tests/test_oracle_pin.py), and
//   * as the CPU baseline / `bench.py --impl reference` arm: the reference
//     pipeline synthesize_rir -> truncate_rir -> choose_plan -> convolve ->
//     SPEC render, run on the host's cores.
// The SPEC mixer has no reference code; ref_render_batch
// restates it on top of the reference's convolve() and mean_power().
#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <malloc.h>

#include "roomsim/audio_buffer.hpp"
#include "roomsim/convolution.hpp"
#include "roomsim/errors.hpp"
#include "roomsim/fft.hpp"
#include "roomsim/room_model.hpp"

#include "../include/roomsim_gpu.h"

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const roomsim::PlacementError*>(&e)) return RS_ERR_PLACEMENT;
  if (dynamic_cast<const roomsim::GeometryError*>(&e)) return RS_ERR_GEOMETRY;
  if (dynamic_cast<const roomsim::DegenerateInputError*>(&e)) return RS_ERR_DEGENERATE;
  if (dynamic_cast<const roomsim::PlanError*>(&e)) return RS_ERR_PLAN;
  if (dynamic_cast<const roomsim::ConfigError*>(&e)) return RS_ERR_CONFIG;
  if (dynamic_cast<const roomsim::FormatError*>(&e)) return RS_ERR_FORMAT;
  if (dynamic_cast<const roomsim::IoError*>(&e)) return RS_ERR_IO;
  return RS_ERR_UNSUPPORTED;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

roomsim::RoomConfig make_room(const double room[3], double refl, double fs, double c0,
                              int order) {
  roomsim::RoomConfig r;
  r.dimensions = {room[0], room[1], room[2]};
  r.reflection_coefficient = refl;
  r.sample_rate = fs;
  r.speed_of_sound = c0;
  r.image_order = order;
  return r;
}

roomsim::Placement place(const double p[3]) { return roomsim::Placement{{p[0], p[1], p[2]}}; }

roomsim::CostInputs cost_inputs(double I, double J, size_t nx, size_t nh) {
  roomsim::CostInputs c;
  c.num_sources = I;
  c.num_mics = J;
  c.signal_len = nx;
  c.rir_len = nh;
  return c;
}

roomsim::Rir make_rir(const double* h, size_t n, double fs = 16000.0) {
  roomsim::Rir r;
  r.samples.assign(h, h + n);
  r.sample_rate = fs;
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

size_t ref_virtual_source_count(int order) {
  roomsim::RoomConfig r;
  r.image_order = order;
  return r.virtual_source_count();
}

int ref_enumerate_images(const double room[3], double refl, double fs, double c0, int order,
                         const double src[3], double* pos, int* refl_count, size_t cap) {
  return guarded([&] {
    const auto imgs = roomsim::enumerate_images(make_room(room, refl, fs, c0, order), place(src));
    if (imgs.size() > cap) {
      g_err = "capacity";
      return (int)RS_ERR_UNSUPPORTED;
    }
    for (size_t v = 0; v < imgs.size(); ++v) {
      pos[3 * v] = imgs[v].position.x;
      pos[3 * v + 1] = imgs[v].position.y;
      pos[3 * v + 2] = imgs[v].position.z;
      refl_count[v] = imgs[v].reflection_count;
    }
    return (int)RS_OK;
  });
}

int ref_synthesize_rir(const double room[3], double refl, double fs, double c0, int order,
                       const double src[3], const double mic[3], int64_t max_taps,
                       double* out, size_t cap, size_t* len) {
  return guarded([&] {
    auto rir = roomsim::synthesize_rir(make_room(room, refl, fs, c0, order), place(src),
                                       place(mic));
    size_t n = rir.samples.size();
    if (max_taps > 0 && (size_t)max_taps < n) n = (size_t)max_taps;
    if (n > cap) {
      g_err = "RIR longer than output capacity";
      return (int)RS_ERR_UNSUPPORTED;
    }
    std::memcpy(out, rir.samples.data(), n * sizeof(double));
    *len = n;
    return (int)RS_OK;
  });
}

int ref_power_threshold(const double* h, size_t n, double eta_db, double* p_th) {
  return guarded([&] {
    *p_th = roomsim::power_threshold(make_rir(h, n), eta_db);
    return (int)RS_OK;
  });
}

int ref_cutoff_index(const double* h, size_t n, double threshold, size_t* n_c) {
  return guarded([&] {
    *n_c = roomsim::cutoff_index(make_rir(h, n), threshold);
    return (int)RS_OK;
  });
}

int ref_truncate_rir(const double* h, size_t n, double eta_db, size_t* keep, size_t* n_c,
                     double* p_th) {
  return guarded([&] {
    const auto rir = make_rir(h, n);
    const auto out = roomsim::truncate_rir(rir, eta_db);
    *keep = out.samples.size();
    const double th = roomsim::power_threshold(rir, eta_db);
    if (n_c) *n_c = roomsim::cutoff_index(rir, th);
    if (p_th) *p_th = th;
    return (int)RS_OK;
  });
}

double ref_cost_direct(double I, double J, size_t nx, size_t nh) {
  try { return roomsim::cost_direct(cost_inputs(I, J, nx, nh)); }
  catch (const std::exception& e) { g_err = e.what(); return NAN; }
}
double ref_cost_full_fft(double I, double J, size_t nx, size_t nh, size_t n) {
  try { return roomsim::cost_full_fft(cost_inputs(I, J, nx, nh), n); }
  catch (const std::exception& e) { g_err = e.what(); return NAN; }
}
double ref_cost_ola(double I, double J, size_t nx, size_t nh, size_t n) {
  try { return roomsim::cost_ola(cost_inputs(I, J, nx, nh), n); }
  catch (const std::exception& e) { g_err = e.what(); return NAN; }
}
size_t ref_ola_block_count(size_t nx, size_t nh, size_t n) {
  return roomsim::ola_block_count(nx, nh, n);
}

static void put_plan(const roomsim::ConvolutionPlan& p, int* s, size_t* n, double* c) {
  *s = p.strategy == roomsim::Strategy::direct     ? RS_DIRECT
       : p.strategy == roomsim::Strategy::full_fft ? RS_FULL_FFT
                                                   : RS_OVERLAP_ADD;
  *n = p.fft_size ? *p.fft_size : 0;
  *c = p.predicted_cost;
}

int ref_plan_for(double I, double J, size_t nx, size_t nh, int strategy, int* s_out,
                 size_t* n_out, double* cost_out) {
  return guarded([&] {
    const auto s = strategy == RS_DIRECT     ? roomsim::Strategy::direct
                   : strategy == RS_FULL_FFT ? roomsim::Strategy::full_fft
                                             : roomsim::Strategy::overlap_add;
    put_plan(roomsim::plan_for(cost_inputs(I, J, nx, nh), s), s_out, n_out, cost_out);
    return (int)RS_OK;
  });
}

int ref_choose_plan(double I, double J, size_t nx, size_t nh, int* s_out, size_t* n_out,
                    double* cost_out) {
  return guarded([&] {
    put_plan(roomsim::choose_plan(cost_inputs(I, J, nx, nh)), s_out, n_out, cost_out);
    return (int)RS_OK;
  });
}

int ref_rfft_forward(size_t n, const double* in, double* out) {
  return guarded([&] {
    roomsim::RadixTwoRealFft f(n);
    std::vector<std::complex<double>> spec(f.spectrum_size());
    f.forward(std::span<const double>(in, n), spec);
    std::memcpy(out, spec.data(), spec.size() * sizeof(std::complex<double>));
    return (int)RS_OK;
  });
}

int ref_rfft_inverse(size_t n, const double* in, double* out) {
  return guarded([&] {
    roomsim::RadixTwoRealFft f(n);
    std::vector<std::complex<double>> spec(f.spectrum_size());
    std::memcpy(spec.data(), in, spec.size() * sizeof(std::complex<double>));
    f.inverse(spec, std::span<double>(out, n));
    return (int)RS_OK;
  });
}

static int conv_common(const double* x, size_t nx, const double* h, size_t nh, double* out,
                       int strategy, size_t n) {
  return guarded([&] {
    auto xb = roomsim::AudioBuffer::mono(std::vector<double>(x, x + nx), 16000.0);
    auto hr = make_rir(h, nh);
    roomsim::AudioBuffer y;
    if (strategy == RS_DIRECT) y = roomsim::convolve_direct(xb, hr);
    else if (strategy == RS_FULL_FFT) y = roomsim::convolve_full_fft(xb, hr);
    else y = roomsim::convolve_ola(xb, hr, n);
    std::memcpy(out, y.channel(0).data(), y.num_frames() * sizeof(double));
    return (int)RS_OK;
  });
}

int ref_convolve_direct(const double* x, size_t nx, const double* h, size_t nh, double* out) {
  return conv_common(x, nx, h, nh, out, RS_DIRECT, 0);
}
int ref_convolve_full_fft(const double* x, size_t nx, const double* h, size_t nh, double* out) {
  return conv_common(x, nx, h, nh, out, RS_FULL_FFT, 0);
}
int ref_convolve_ola(const double* x, size_t nx, const double* h, size_t nh, size_t n,
                     double* out) {
  return conv_common(x, nx, h, nh, out, RS_OVERLAP_ADD, n);
}

int ref_mean_power(const double* v, size_t n, double* p) {
  return guarded([&] {
    *p = roomsim::mean_power(roomsim::AudioBuffer::mono(std::vector<double>(v, v + n), 16000.0));
    return (int)RS_OK;
  });
}

// SPEC.md:338-346 compute_gain (no reference code): same formula as the
// C restatement.
int ref_compute_gain(double p_target, double p_noise, double snr_db, double* alpha) {
  if (!(p_target > 0.0)) { g_err = "target has no energy"; return RS_ERR_DEGENERATE; }
  if (!(p_noise > 0.0)) { g_err = "noise has no energy"; return RS_ERR_DEGENERATE; }
  *alpha = std::sqrt(p_target / (p_noise * std::pow(10.0, snr_db / 10.0)));
  return RS_OK;
}

// One utterance of SPEC.md:348-356 render, through the reference functions.
static int render_one(const rs_scene_batch* b, int64_t u, int64_t pair0, double* out,
                      const int64_t* out_off, const int64_t* out_stride, int64_t* out_len,
                      rs_pair_layout* layout, double* gains, double* power) {
  return guarded([&] {
    const int64_t s0 = b->src_begin[u], I = b->src_begin[u + 1] - s0;
    const int64_t m0 = b->mic_begin[u], J = b->mic_begin[u + 1] - m0;
    const auto room = make_room(b->room_dims + 3 * u, b->reflection[u], b->sample_rate[u],
                                b->speed_of_sound[u], b->image_order[u]);
    const int64_t cap = b->max_taps ? b->max_taps[u] : 0;
    std::vector<roomsim::AudioBuffer> conv((size_t)(I * J));
    std::vector<double> pw((size_t)(I * J));
    for (int64_t i = 0; i < I; ++i) {
      const int64_t nx = b->sig_len[s0 + i];
      std::vector<double> xs((size_t)nx);
      for (int64_t k = 0; k < nx; ++k) xs[(size_t)k] = (double)b->signals[b->sig_off[s0 + i] + k];
      const auto x = roomsim::AudioBuffer::mono(std::move(xs), room.sample_rate);
      for (int64_t j = 0; j < J; ++j) {
        auto h = roomsim::synthesize_rir(room, place(b->src_pos + 3 * (s0 + i)),
                                         place(b->mic_pos + 3 * (m0 + j)));
        const size_t full = h.samples.size();
        if (cap > 0 && (size_t)cap < full) h.samples.resize((size_t)cap);  // T60 horizon
        const size_t rir_len = h.samples.size();
        int64_t n_c = -1;
        if (b->eta_db > 0.0) {
          n_c = (int64_t)roomsim::cutoff_index(h, roomsim::power_threshold(h, b->eta_db));
          h = roomsim::truncate_rir(h, b->eta_db);
        }
        roomsim::ConvolutionPlan plan;
        if (b->plan_rule == RS_PLAN_CHOOSE) {
          plan = roomsim::choose_plan(cost_inputs(1.0, 1.0, (size_t)nx, h.samples.size()));
        } else {
          plan.strategy = roomsim::Strategy::overlap_add;
          plan.fft_size = b->plan_rule == RS_PLAN_FORCED
                              ? (size_t)b->forced_fft_size
                              : std::bit_ceil(2 * h.samples.size());
        }
        auto y = roomsim::convolve(x, h, plan);
        const size_t k = (size_t)(i * J + j);
        pw[k] = roomsim::mean_power(y);
        if (layout) {
          rs_pair_layout& L = layout[pair0 + (int64_t)k];
          const size_t nh = h.samples.size();
          const size_t n = plan.fft_size ? *plan.fft_size : 0;
          L.rir_len = (int64_t)rir_len;
          L.rir_keep = (int64_t)nh;
          L.cutoff = n_c;
          L.fft_size = (int64_t)n;
          L.block_len = (int64_t)(n - nh + 1);
          L.n_blocks = (int64_t)roomsim::ola_block_count((size_t)nx, nh, n);
          L.out_len = (int64_t)y.num_frames();
          L.strategy = plan.strategy == roomsim::Strategy::direct     ? RS_DIRECT
                       : plan.strategy == roomsim::Strategy::full_fft ? RS_FULL_FFT
                                                                      : RS_OVERLAP_ADD;
          L.flags = 0;
        }
        conv[k] = std::move(y);
      }
    }
    std::vector<double> alpha((size_t)(I * J), 1.0);  // target gain 1
    for (int64_t j = 0; j < J; ++j)
      for (int64_t i = 1; i < I; ++i) {
        const int st = ref_compute_gain(pw[(size_t)j], pw[(size_t)(i * J + j)],
                                        b->snr_db[s0 + i], &alpha[(size_t)(i * J + j)]);
        if (st) throw roomsim::DegenerateInputError(g_err);
      }
    size_t maxlen = 0;
    for (const auto& c : conv) maxlen = std::max(maxlen, c.num_frames());
    if ((int64_t)maxlen > out_stride[u]) throw roomsim::ConfigError("output stride too small");
    for (int64_t j = 0; j < J; ++j) {
      double* yj = out + out_off[u] + j * out_stride[u];
      std::fill(yj, yj + maxlen, 0.0);
      for (int64_t i = 0; i < I; ++i) {  // source order
        const double a = alpha[(size_t)(i * J + j)];
        const auto& c = conv[(size_t)(i * J + j)].channel(0);
        for (size_t n = 0; n < c.size(); ++n) yj[n] += a * c[n];
      }
    }
    if (out_len) out_len[u] = (int64_t)maxlen;
    for (int64_t k = 0; k < I * J; ++k) {
      if (gains) gains[pair0 + k] = alpha[(size_t)k];
      if (power) power[pair0 + k] = pw[(size_t)k];
    }
    return (int)RS_OK;
  });
}

int ref_render_batch(const rs_scene_batch* b, double* out, const int64_t* out_off,
                     const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                     double* gains, double* power, int threads) {
  std::vector<int64_t> pair0((size_t)b->n_utt + 1, 0);
  for (int64_t u = 0; u < b->n_utt; ++u)
    pair0[(size_t)u + 1] = pair0[(size_t)u] + (b->src_begin[u + 1] - b->src_begin[u]) *
                                                  (b->mic_begin[u + 1] - b->mic_begin[u]);
  std::atomic<int64_t> next{0};
  std::atomic<int> status{0};
  std::mutex mu;
  std::string first_err;
  auto worker = [&] {
    for (;;) {
      const int64_t u = next.fetch_add(1);
      if (u >= b->n_utt || status.load()) break;
      const int st = render_one(b, u, pair0[(size_t)u], out, out_off, out_stride, out_len,
                                layout, gains, power);
      if (st) {
        std::lock_guard<std::mutex> lk(mu);
        if (!status.load()) {
          status = st;
          first_err = g_err;
        }
      }
    }
  };
  if (threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
  }
  if (status.load()) g_err = first_err;
  return status.load();
}

int ref_hardware_concurrency(void) { return (int)std::thread::hardware_concurrency(); }

// Equivalent of GLIBC_TUNABLES=glibc.malloc.mmap_threshold=67108864 (SURVEY.md
// §3: the reference allocates its FFT scratch per call, which serialises
// threads on mmap page faults with the default threshold).
int ref_set_malloc_tuning(int enabled) {
  if (!enabled) return 0;
  mallopt(M_MMAP_THRESHOLD, 64 << 20);
  mallopt(M_TRIM_THRESHOLD, 256 << 20);
  return 1;
}

}  // extern "C"

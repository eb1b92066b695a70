// Drop-in test: the reference's own API and templates, with the B200 path
// plugged in through include/roomsim_gpu.hpp.  Built by `make adapter` where
// the reference headers exist; run by tests/test_gpu_adapter.py on a GPU.
#include <cmath>
#include <cstdio>
#include <random>

#include "roomsim_gpu.hpp"

using namespace roomsim;

static int failures = 0;
#define EXPECT(cond, ...)                  \
  do {                                     \
    if (!(cond)) {                         \
      std::printf("FAIL: " __VA_ARGS__);   \
      std::printf("\n");                   \
      ++failures;                          \
    }                                      \
  } while (0)

static double rel_err(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0, e = 0;
  for (size_t i = 0; i < b.size(); ++i) {
    m = std::max(m, std::abs(b[i]));
    e = std::max(e, std::abs(a[i] - b[i]));
  }
  return e / std::max(m, 1e-300);
}

int main() {
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  // synthesize_rir / truncate_rir: bit-exact against the reference
  for (int t = 0; t < 20; ++t) {
    RoomConfig room;
    room.dimensions = {3 + 7 * U(g), 3 + 5 * U(g), 2.5 + 3.5 * U(g)};
    room.reflection_coefficient = 0.2 + 0.7 * U(g);
    room.image_order = t % 9;
    Placement s{{0.5 + (room.dimensions.x - 1) * U(g), 0.5 + (room.dimensions.y - 1) * U(g), 0.5 + (room.dimensions.z - 1) * U(g)}};
    Placement m{{0.5 + (room.dimensions.x - 1) * U(g), 0.5 + (room.dimensions.y - 1) * U(g), 0.5 + (room.dimensions.z - 1) * U(g)}};
    const Rir want = synthesize_rir(room, s, m);
    const Rir got = gpu::synthesize_rir(room, s, m);
    EXPECT(want.samples == got.samples, "synthesize_rir bits differ (case %d)", t);
    const Rir tw = truncate_rir(want, 20.0), tg = gpu::truncate_rir(got, 20.0);
    EXPECT(tw.samples.size() == tg.samples.size(), "truncate_rir length differs (case %d)", t);
  }
  // convolve_ola through the adapter and through the reference template with the device engine
  std::normal_distribution<double> Nd(0.0, 1.0);
  for (int t = 0; t < 10; ++t) {
    std::vector<double> x(1000 + 997 * t), hs(50 + 37 * t);
    for (auto& v : x) v = Nd(g);
    for (auto& v : hs) v = Nd(g);
    const auto xb = AudioBuffer::mono(x, 16000.0);
    Rir h;
    h.samples = hs;
    const std::size_t n = std::bit_ceil(2 * hs.size());
    const AudioBuffer want = convolve_ola(xb, h, n);
    const AudioBuffer got = gpu::convolve_ola(xb, h, n);
    EXPECT(rel_err(got.channel(0), want.channel(0)) <= 1e-5, "gpu::convolve_ola case %d", t);
    const AudioBuffer eng = convolve_ola<gpu::CudaRealFft>(xb, h, n);
    EXPECT(rel_err(eng.channel(0), want.channel(0)) <= 1e-5, "convolve_ola<CudaRealFft> case %d", t);
    const ConvolutionPlan p = choose_plan(CostInputs{1.0, 1.0, x.size(), hs.size()});
    const ConvolutionPlan q = gpu::choose_plan(CostInputs{1.0, 1.0, x.size(), hs.size()});
    EXPECT(p.fft_size == q.fft_size && p.predicted_cost == q.predicted_cost && p.strategy == q.strategy,
           "choose_plan differs case %d", t);
  }
  // convolve dispatch (convolution.hpp:258-271): direct is FP64 and bit-exact, the FFT
  // strategies FP32 within 1e-5 of the peak
  for (int t = 0; t < 6; ++t) {
    std::vector<double> x(300 + 611 * t), hs(20 + 131 * t);
    for (auto& v : x) v = Nd(g);
    for (auto& v : hs) v = Nd(g);
    const auto xb = AudioBuffer::mono(x, 16000.0);
    Rir h;
    h.samples = hs;
    const AudioBuffer dw = convolve_direct(xb, h), dg = gpu::convolve_direct(xb, h);
    EXPECT(dw.channel(0) == dg.channel(0), "gpu::convolve_direct bits differ case %d", t);
    const ConvolutionPlan plans[3] = {plan_for(CostInputs{1.0, 1.0, x.size(), hs.size()}, Strategy::direct),
                                      plan_for(CostInputs{1.0, 1.0, x.size(), hs.size()}, Strategy::full_fft),
                                      plan_for(CostInputs{1.0, 1.0, x.size(), hs.size()}, Strategy::overlap_add)};
    for (const ConvolutionPlan& p : plans) {
      const AudioBuffer want = convolve(xb, h, p), got = gpu::convolve(xb, h, p);
      EXPECT(got.channel(0).size() == want.channel(0).size(), "gpu::convolve length case %d", t);
      if (p.strategy == Strategy::direct)
        EXPECT(got.channel(0) == want.channel(0), "gpu::convolve(direct) bits case %d", t);
      else
        EXPECT(rel_err(got.channel(0), want.channel(0)) <= 1e-5, "gpu::convolve strategy %d case %d",
               static_cast<int>(p.strategy), t);
    }
  }
  // error taxonomy
  bool threw = false;
  try {
    RoomConfig room;
    room.dimensions = {5, 5, 5};
    room.reflection_coefficient = 0.5;
    gpu::synthesize_rir(room, Placement{{0, 1, 1}}, Placement{{2, 2, 2}});
  } catch (const PlacementError&) {
    threw = true;
  }
  EXPECT(threw, "PlacementError not rethrown");
  threw = false;
  try {
    gpu::convolve_ola(AudioBuffer::mono(std::vector<double>(10, 1.0), 16000.0), Rir{std::vector<double>(8, 1.0)}, 4);
  } catch (const PlanError&) {
    threw = true;
  }
  EXPECT(threw, "PlanError not rethrown");
  // SPEC render: single target, K = 0, d = 1 m -> y = x delayed by 47
  gpu::Scene sc;
  sc.room.dimensions = {5, 5, 5};
  sc.room.reflection_coefficient = 0.5;
  sc.room.image_order = 0;
  sc.sources = {Placement{{1, 1, 1}}, Placement{{1, 1, 1}}};
  sc.mics = {Placement{{2, 1, 1}}};
  std::vector<double> x(500);
  for (auto& v : x) v = Nd(g);
  sc.signals = {AudioBuffer::mono(x, 16000.0), AudioBuffer::mono(x, 16000.0)};
  sc.snr_db = {0.0, 0.0};
  const gpu::MixOutput mo = gpu::render_batch({sc});
  const auto& y = mo.channels[0].channel(0);
  double e = 0;
  for (size_t i = 0; i < x.size(); ++i) e = std::max(e, std::abs(y[47 + i] - 2.0 * x[i]));
  EXPECT(y.size() == 547 && e <= 1e-5 * 2 * 4.0, "render_batch coherent sum (err %g)", e);
  EXPECT(std::abs(mo.gains[0][1] - 1.0) < 1e-9, "render_batch alpha");
  if (failures == 0) std::printf("ADAPTER OK\n");
  return failures == 0 ? 0 : 1;
}

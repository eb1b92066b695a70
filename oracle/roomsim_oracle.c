/*
 * roomsim_oracle.c — TEST INFRASTRUCTURE ONLY (see roomsim_oracle.h).
 *
 * Plain-C restatement of the reference hot path, written from the reference
 * headers' documented algorithm.  Each function cites the reference lines it
 * restates (paths relative to /root/reference/proj/include/).  Arithmetic is
 * FP64 in the reference's operation order; build with -ffp-contract=off and
 * no -march=native (oracle/Makefile) so no FMA contraction changes a bit.
 */
#define _GNU_SOURCE
#include "roomsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------------ */
/* room_model.hpp                                                            */
/* ------------------------------------------------------------------------ */

/* RoomConfig::validate, roomsim/room_model.hpp:57-65 */
static int room_validate(const double L[3], double r, double fs, double c0, int order) {
  if (L[0] <= 0.0 || L[1] <= 0.0 || L[2] <= 0.0)
    return fail(RS_ERR_CONFIG, "room dimensions must be positive");
  if (r <= 0.0 || r >= 1.0) return fail(RS_ERR_CONFIG, "reflection coefficient must lie in (0, 1)");
  if (fs <= 0.0) return fail(RS_ERR_CONFIG, "sample rate must be positive");
  if (c0 <= 0.0) return fail(RS_ERR_CONFIG, "speed of sound must be positive");
  if (order < 0) return fail(RS_ERR_CONFIG, "image order must be non-negative");
  return RS_OK;
}

/* strictly_inside, roomsim/room_model.hpp:79-84 */
static int strictly_inside(const double L[3], const double p[3]) {
  for (int a = 0; a < 3; ++a)
    if (!(p[a] > 0.0 && p[a] < L[a])) return 0;
  return 1;
}

/* RoomConfig::virtual_source_count, roomsim/room_model.hpp:67-71 */
size_t orc_virtual_source_count(int order) {
  size_t per_axis = 2 * (size_t)order + 1;
  return per_axis * per_axis * per_axis;
}

/* Image coordinate along one axis, roomsim/room_model.hpp:123-128:
 * even n -> n*L + s, odd n -> n*L + (L - s). */
static double image_coord(int n, double length, double s) {
  const double mirrored = (n % 2 == 0) ? s : length - s;
  return (double)n * length + mirrored;
}

/* enumerate_images, roomsim/room_model.hpp:109-134 (order nx -> ny -> nz). */
int orc_enumerate_images(const double room[3], double refl, double fs, double c0, int order,
                         const double src[3], double* pos, int* refl_count, size_t cap) {
  int st = room_validate(room, refl, fs, c0, order);
  if (st) return st;
  if (!strictly_inside(room, src))
    return fail(RS_ERR_PLACEMENT, "source must lie strictly inside the room");
  if (cap < orc_virtual_source_count(order)) return fail(RS_ERR_UNSUPPORTED, "capacity");
  size_t v = 0;
  for (int nx = -order; nx <= order; ++nx)
    for (int ny = -order; ny <= order; ++ny)
      for (int nz = -order; nz <= order; ++nz, ++v) {
        pos[3 * v + 0] = image_coord(nx, room[0], src[0]);
        pos[3 * v + 1] = image_coord(ny, room[1], src[1]);
        pos[3 * v + 2] = image_coord(nz, room[2], src[2]);
        refl_count[v] = abs(nx) + abs(ny) + abs(nz);
      }
  return RS_OK;
}

/* norm(a - b), roomsim/room_model.hpp:36-46: sqrt(x*x + y*y + z*z), evaluated
 * left to right. */
static double distance3(const double a[3], const double b[3]) {
  const double x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
  return sqrt(x * x + y * y + z * z);
}

/* synthesize_rir, roomsim/room_model.hpp:141-174.  The image loop is run
 * twice (max delay + geometry check, then accumulation in enumeration order)
 * instead of buffering V taps; both passes evaluate identical expressions.
 * max_taps > 0 additionally keeps only the first max_taps taps (harness-side
 * T60 horizon). */
int orc_synthesize_rir(const double room[3], double refl, double fs, double c0, int order,
                       const double src[3], const double mic[3], int64_t max_taps,
                       double* out, size_t cap, size_t* len) {
  int st = room_validate(room, refl, fs, c0, order);
  if (st) return st;
  if (!strictly_inside(room, src))
    return fail(RS_ERR_PLACEMENT, "source must lie strictly inside the room");
  if (!strictly_inside(room, mic))
    return fail(RS_ERR_PLACEMENT, "microphone must lie strictly inside the room");
  const double spm = fs / c0; /* :150 */
  size_t max_delay = 0;
  for (int pass = 0; pass < 2; ++pass) {
    size_t n = 0;
    if (pass == 1) {
      n = max_delay + 1;
      if (max_taps > 0 && (size_t)max_taps < n) n = (size_t)max_taps;
      if (n > cap) return fail(RS_ERR_UNSUPPORTED, "RIR longer than output capacity");
      memset(out, 0, n * sizeof(double)); /* :169 */
      *len = n;
    }
    for (int nx = -order; nx <= order; ++nx) {
      const double px = image_coord(nx, room[0], src[0]);
      for (int ny = -order; ny <= order; ++ny) {
        const double py = image_coord(ny, room[1], src[1]);
        for (int nz = -order; nz <= order; ++nz) {
          const double p[3] = {px, py, image_coord(nz, room[2], src[2])};
          const double d = distance3(p, mic); /* :156 */
          if (d <= 0.0)                       /* :157-158 */
            return fail(RS_ERR_GEOMETRY, "microphone coincides with an image source");
          const size_t delay = (size_t)ceil(d * spm); /* :159-160 */
          if (pass == 0) {
            if (delay > max_delay) max_delay = delay; /* :164 */
          } else if (delay < n) {
            const int g = abs(nx) + abs(ny) + abs(nz);
            const double amp = pow(refl, (double)g) / d; /* :161-162 */
            out[delay] += amp;                           /* :170 */
          }
        }
      }
    }
  }
  return RS_OK;
}

/* power_threshold, roomsim/room_model.hpp:177-185 */
int orc_power_threshold(const double* h, size_t n, double eta_db, double* p_th) {
  if (n == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  if (eta_db <= 0.0) return fail(RS_ERR_CONFIG, "cut-off threshold must be positive dB");
  double max_power = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double p = h[i] * h[i];
    max_power = (max_power < p) ? p : max_power; /* std::max */
  }
  if (max_power == 0.0) return fail(RS_ERR_DEGENERATE, "all-zero impulse response has no power");
  *p_th = max_power * pow(10.0, -eta_db / 10.0);
  return RS_OK;
}

/* cutoff_index, roomsim/room_model.hpp:188-197 */
int orc_cutoff_index(const double* h, size_t n, double threshold, size_t* n_c) {
  if (n == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  if (threshold <= 0.0) return fail(RS_ERR_CONFIG, "power threshold must be positive");
  for (size_t i = n; i-- > 0;) {
    if (h[i] * h[i] >= threshold) {
      *n_c = i;
      return RS_OK;
    }
  }
  *n_c = 0;
  return RS_OK;
}

/* truncate_rir, roomsim/room_model.hpp:203-213: keep = min(n_c + 2, n). */
int orc_truncate_rir(const double* h, size_t n, double eta_db, size_t* keep, size_t* n_c,
                     double* p_th) {
  double th;
  size_t c;
  int st = orc_power_threshold(h, n, eta_db, &th);
  if (st) return st;
  st = orc_cutoff_index(h, n, th, &c);
  if (st) return st;
  *keep = (c + 2 < n) ? c + 2 : n;
  if (n_c) *n_c = c;
  if (p_th) *p_th = th;
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* convolution.hpp: cost models and planner                                  */
/* ------------------------------------------------------------------------ */

static int has_single_bit(size_t n) { return n != 0 && (n & (n - 1)) == 0; }
static size_t bit_ceil(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* CostInputs::validate, roomsim/convolution.hpp:55-60 */
static int cost_validate(double I, double J, size_t nx, size_t nh) {
  if (I <= 0.0 || J <= 0.0) return fail(RS_ERR_CONFIG, "source and mic counts must be positive");
  if (nx == 0 || nh == 0) return fail(RS_ERR_CONFIG, "signal and RIR lengths must be positive");
  return RS_OK;
}

/* detail::checked_fft_size, roomsim/convolution.hpp:72-79 */
static int checked_fft_size(size_t n, size_t min_legal, const char* what) {
  char msg[256];
  if (n < 2 || !has_single_bit(n)) {
    snprintf(msg, sizeof msg, "%s: FFT size must be a power of two >= 2", what);
    return fail(RS_ERR_PLAN, msg);
  }
  if (n < min_legal) {
    snprintf(msg, sizeof msg, "%s: FFT size too small for this workload", what);
    return fail(RS_ERR_PLAN, msg);
  }
  return RS_OK;
}

/* detail::fft_size_for, roomsim/convolution.hpp:82-84 */
static size_t fft_size_for(size_t n) { return bit_ceil(n < 2 ? 2 : n); }

/* cost_direct, roomsim/convolution.hpp:89-93 (NaN on invalid input) */
double orc_cost_direct(double I, double J, size_t nx, size_t nh) {
  if (cost_validate(I, J, nx, nh)) return NAN;
  return I * J * (double)nx * (double)nh;
}

/* cost_full_fft, roomsim/convolution.hpp:100-105 */
double orc_cost_full_fft(double I, double J, size_t nx, size_t nh, size_t n) {
  if (cost_validate(I, J, nx, nh)) return NAN;
  if (checked_fft_size(n, nx + nh - 1, "full FFT")) return NAN;
  const double nd = (double)n;
  return I * J * (6.0 * nd * log2(nd) + 2.0 * nd);
}

/* ola_block_count, roomsim/convolution.hpp:108-112 */
size_t orc_ola_block_count(size_t nx, size_t nh, size_t n) {
  const size_t L = n - nh + 1;
  return (nx + L - 1) / L;
}

/* cost_ola, roomsim/convolution.hpp:119-127 */
double orc_cost_ola(double I, double J, size_t nx, size_t nh, size_t n) {
  if (cost_validate(I, J, nx, nh)) return NAN;
  if (checked_fft_size(n, nh, "overlap-add")) return NAN;
  const double nd = (double)n;
  const double blocks = (double)orc_ola_block_count(nx, nh, n);
  return I * J * (blocks * (4.0 * nd * log2(nd) + 2.0 * nd) + 2.0 * nd * log2(nd));
}

/* plan_for, roomsim/convolution.hpp:130-152 */
int orc_plan_for(double I, double J, size_t nx, size_t nh, int strategy, int* s_out,
                 size_t* n_out, double* cost_out) {
  int st = cost_validate(I, J, nx, nh);
  if (st) return st;
  switch (strategy) {
    case RS_DIRECT:
      *s_out = RS_DIRECT;
      *n_out = 0;
      *cost_out = orc_cost_direct(I, J, nx, nh);
      return RS_OK;
    case RS_FULL_FFT: {
      const size_t n = fft_size_for(nx + nh - 1);
      *s_out = RS_FULL_FFT;
      *n_out = n;
      *cost_out = orc_cost_full_fft(I, J, nx, nh, n);
      return RS_OK;
    }
    case RS_OVERLAP_ADD: {
      const size_t n_max = fft_size_for(nx + nh - 1);
      double best = INFINITY;
      size_t best_n = 0;
      for (size_t n = fft_size_for(nh); n <= n_max; n <<= 1) {
        const double c = orc_cost_ola(I, J, nx, nh, n);
        if (c < best) {
          best = c;
          best_n = n;
        }
      }
      *s_out = RS_OVERLAP_ADD;
      *n_out = best_n;
      *cost_out = best;
      return RS_OK;
    }
  }
  return fail(RS_ERR_PLAN, "unknown strategy");
}

/* choose_plan, roomsim/convolution.hpp:157-161: ties go to overlap-add. */
int orc_choose_plan(double I, double J, size_t nx, size_t nh, int* s_out, size_t* n_out,
                    double* cost_out) {
  int s1, s2;
  size_t n1, n2;
  double c1, c2;
  int st = orc_plan_for(I, J, nx, nh, RS_OVERLAP_ADD, &s1, &n1, &c1);
  if (st) return st;
  st = orc_plan_for(I, J, nx, nh, RS_FULL_FFT, &s2, &n2, &c2);
  if (st) return st;
  if (c2 < c1) {
    *s_out = s2; *n_out = n2; *cost_out = c2;
  } else {
    *s_out = s1; *n_out = n1; *cost_out = c1;
  }
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* fft.hpp: RadixTwoRealFft                                                  */
/* ------------------------------------------------------------------------ */

typedef struct { double re, im; } cpx;

/* (a+bi)(c+di) = (ac - bd) + (ad + bc)i, the std::complex product. */
static inline cpx cmul(cpx a, cpx b) {
  cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cpx cadd(cpx a, cpx b) { cpx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cpx csub(cpx a, cpx b) { cpx r = {a.re - b.re, a.im - b.im}; return r; }
static inline cpx cconj(cpx a) { cpx r = {a.re, -a.im}; return r; }
static inline cpx cscale(double s, cpx a) { cpx r = {a.re * s, a.im * s}; return r; }

typedef struct {
  size_t size, half;
  cpx* ctw;   /* exp(-2 pi i k / half), k < half/2   (fft.hpp:62-68) */
  cpx* rtw;   /* exp(-2 pi i k / size), k <= half    (fft.hpp:69-75) */
  size_t* rev;/* bit reversal of log2(half) bits       (fft.hpp:76-82) */
  cpx* work;
} rfft;

static const double kPi = 3.141592653589793; /* std::numbers::pi */

/* RadixTwoRealFft::RadixTwoRealFft, roomsim/fft.hpp:59-84 */
static int rfft_init(rfft* f, size_t size) {
  memset(f, 0, sizeof *f);
  if (size < 2 || !has_single_bit(size))
    return fail(RS_ERR_PLAN, "FFT size must be a power of two >= 2");
  f->size = size;
  f->half = size / 2;
  const size_t nct = f->half / 2;
  f->ctw = (cpx*)malloc((nct ? nct : 1) * sizeof(cpx));
  f->rtw = (cpx*)malloc((f->half + 1) * sizeof(cpx));
  f->rev = (size_t*)malloc(f->half * sizeof(size_t));
  f->work = (cpx*)malloc(f->half * sizeof(cpx));
  for (size_t k = 0; k < nct; ++k) {
    const double phase = -2.0 * kPi * (double)k / (double)f->half;
    f->ctw[k].re = cos(phase);
    f->ctw[k].im = sin(phase);
  }
  for (size_t k = 0; k <= f->half; ++k) {
    const double phase = -2.0 * kPi * (double)k / (double)size;
    f->rtw[k].re = cos(phase);
    f->rtw[k].im = sin(phase);
  }
  int bits = 0;
  while (((size_t)1 << bits) < f->half) ++bits;
  for (size_t i = 0; i < f->half; ++i) {
    size_t r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1u) << (bits - 1 - b);
    f->rev[i] = r;
  }
  return RS_OK;
}

static void rfft_free(rfft* f) {
  free(f->ctw); free(f->rtw); free(f->rev); free(f->work);
}

/* RadixTwoRealFft::complex_fft, roomsim/fft.hpp:126-147 */
static void complex_fft(const rfft* f, cpx* a, int inverse) {
  const size_t n = f->half;
  if (n <= 1) return;
  for (size_t i = 0; i < n; ++i) {
    const size_t j = f->rev[i];
    if (i < j) { cpx t = a[i]; a[i] = a[j]; a[j] = t; }
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half_len = len / 2, stride = n / len;
    for (size_t start = 0; start < n; start += len)
      for (size_t j = 0; j < half_len; ++j) {
        cpx w = f->ctw[j * stride];
        if (inverse) w = cconj(w);
        const cpx u = a[start + j];
        const cpx v = cmul(a[start + j + half_len], w);
        a[start + j] = cadd(u, v);
        a[start + j + half_len] = csub(u, v);
      }
  }
}

/* forward, roomsim/fft.hpp:90-95 + untangle, :152-161 */
static void rfft_forward(rfft* f, const double* in, cpx* out) {
  const size_t h = f->half;
  for (size_t k = 0; k < h; ++k) { f->work[k].re = in[2 * k]; f->work[k].im = in[2 * k + 1]; }
  complex_fft(f, f->work, 0);
  const cpx mhalf_i = {0.0, -0.5};
  for (size_t k = 0; k <= h; ++k) {
    const cpx a = f->work[k % h];
    const cpx b = cconj(f->work[(h - k) % h]);
    const cpx even = cscale(0.5, cadd(a, b));
    const cpx odd = cmul(mhalf_i, csub(a, b));
    out[k] = cadd(even, cmul(f->rtw[k], odd));
  }
}

/* inverse, roomsim/fft.hpp:98-117 */
static void rfft_inverse(rfft* f, const cpx* in, double* out) {
  const size_t h = f->half;
  const cpx unit_i = {0.0, 1.0};
  for (size_t k = 0; k < h; ++k) {
    const cpx a = in[k];
    const cpx b = cconj(in[h - k]);
    const cpx even = cscale(0.5, cadd(a, b));
    const cpx odd = cmul(cscale(0.5, csub(a, b)), cconj(f->rtw[k]));
    f->work[k] = cadd(even, cmul(unit_i, odd));
  }
  complex_fft(f, f->work, 1);
  const double scale = 1.0 / (double)h;
  for (size_t k = 0; k < h; ++k) {
    out[2 * k] = f->work[k].re * scale;
    out[2 * k + 1] = f->work[k].im * scale;
  }
}

int orc_rfft_forward(size_t n, const double* in, double* out) {
  rfft f;
  int st = rfft_init(&f, n);
  if (st) return st;
  rfft_forward(&f, in, (cpx*)out);
  rfft_free(&f);
  return RS_OK;
}

int orc_rfft_inverse(size_t n, const double* in, double* out) {
  rfft f;
  int st = rfft_init(&f, n);
  if (st) return st;
  rfft_inverse(&f, (const cpx*)in, out);
  rfft_free(&f);
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* convolution.hpp: convolve_direct / full_fft / ola                         */
/* ------------------------------------------------------------------------ */

/* Input checks shared by the three strategies, roomsim/convolution.hpp:165-170 */
static int conv_validate(size_t nx, size_t nh) {
  if (nx == 0) return fail(RS_ERR_DEGENERATE, "convolution input must be non-empty mono audio");
  if (nh == 0) return fail(RS_ERR_DEGENERATE, "empty impulse response");
  return RS_OK;
}

/* convolve_direct, roomsim/convolution.hpp:164-179 */
int orc_convolve_direct(const double* x, size_t nx, const double* h, size_t nh, double* out) {
  int st = conv_validate(nx, nh);
  if (st) return st;
  memset(out, 0, (nx + nh - 1) * sizeof(double));
  for (size_t i = 0; i < nx; ++i) {
    const double v = x[i];
    for (size_t j = 0; j < nh; ++j) out[i + j] += v * h[j];
  }
  return RS_OK;
}

/* convolve_full_fft, roomsim/convolution.hpp:182-212 */
int orc_convolve_full_fft(const double* x, size_t nx, const double* h, size_t nh, double* out) {
  int st = conv_validate(nx, nh);
  if (st) return st;
  const size_t out_len = nx + nh - 1;
  const size_t n = fft_size_for(out_len);
  rfft f;
  st = rfft_init(&f, n);
  if (st) return st;
  double* padded = (double*)calloc(n, sizeof(double));
  cpx* ss = (cpx*)malloc((f.half + 1) * sizeof(cpx));
  cpx* rs = (cpx*)malloc((f.half + 1) * sizeof(cpx));
  memcpy(padded, x, nx * sizeof(double));
  rfft_forward(&f, padded, ss);
  memset(padded, 0, n * sizeof(double));
  memcpy(padded, h, nh * sizeof(double));
  rfft_forward(&f, padded, rs);
  for (size_t k = 0; k <= f.half; ++k) ss[k] = cmul(ss[k], rs[k]);
  rfft_inverse(&f, ss, padded);
  memcpy(out, padded, out_len * sizeof(double));
  free(padded); free(ss); free(rs);
  rfft_free(&f);
  return RS_OK;
}

/* convolve_ola, roomsim/convolution.hpp:219-255 */
int orc_convolve_ola(const double* x, size_t nx, const double* h, size_t nh, size_t n,
                     double* out) {
  int st = conv_validate(nx, nh);
  if (st) return st;
  st = checked_fft_size(n, nh, "overlap-add");
  if (st) return st;
  const size_t L = n - nh + 1;         /* :230 */
  const size_t out_len = nx + nh - 1; /* :231 */
  rfft f;
  st = rfft_init(&f, n);
  if (st) return st;
  double* padded = (double*)calloc(n, sizeof(double));
  cpx* rs = (cpx*)malloc((f.half + 1) * sizeof(cpx));
  cpx* bs = (cpx*)malloc((f.half + 1) * sizeof(cpx));
  memcpy(padded, h, nh * sizeof(double));
  rfft_forward(&f, padded, rs); /* :238-239 */
  memset(out, 0, out_len * sizeof(double));
  for (size_t start = 0; start < nx; start += L) { /* :242-253 */
    const size_t take = (L < nx - start) ? L : nx - start;
    memset(padded, 0, n * sizeof(double));
    memcpy(padded, x + start, take * sizeof(double));
    rfft_forward(&f, padded, bs);
    for (size_t k = 0; k <= f.half; ++k) bs[k] = cmul(bs[k], rs[k]);
    rfft_inverse(&f, bs, padded);
    const size_t limit = (n < out_len - start) ? n : out_len - start;
    for (size_t i = 0; i < limit; ++i) out[start + i] += padded[i];
  }
  free(padded); free(rs); free(bs);
  rfft_free(&f);
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* audio_buffer.hpp + SPEC mixer                                             */
/* ------------------------------------------------------------------------ */

/* mean_power, roomsim/audio_buffer.hpp:66-75 */
int orc_mean_power(const double* v, size_t n, double* p) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += v[i] * v[i];
  if (n == 0) return fail(RS_ERR_DEGENERATE, "mean power of an empty buffer");
  *p = acc / (double)n;
  return RS_OK;
}

/* compute_gain: alpha with
 * 10 log10(P_t / (alpha^2 P_n)) = snr_db  ->  alpha = sqrt(P_t / (P_n 10^(snr/10))). */
int orc_compute_gain(double p_target, double p_noise, double snr_db, double* alpha) {
  if (!(p_target > 0.0)) return fail(RS_ERR_DEGENERATE, "target has no energy");
  if (!(p_noise > 0.0)) return fail(RS_ERR_DEGENERATE, "noise has no energy");
  *alpha = sqrt(p_target / (p_noise * pow(10.0, snr_db / 10.0)));
  return RS_OK;
}

/* One utterance of SPEC.md:348-356 render. */
typedef struct {
  const rs_scene_batch* b;
  double* out;
  const int64_t* out_off;
  const int64_t* out_stride;
  int64_t* out_len;
  rs_pair_layout* layout;
  double* gains;
  double* power;
  int64_t* pair_begin;
  volatile int64_t next;
  pthread_mutex_t mu;
  int status;
  char err[512];
} render_job;

static int render_one(render_job* job, int64_t u) {
  const rs_scene_batch* b = job->b;
  const int64_t s0 = b->src_begin[u], I = b->src_begin[u + 1] - s0;
  const int64_t m0 = b->mic_begin[u], J = b->mic_begin[u + 1] - m0;
  const double* room = b->room_dims + 3 * u;
  const int order = b->image_order[u];
  const int64_t cap_taps = b->max_taps ? b->max_taps[u] : 0;
  int st = room_validate(room, b->reflection[u], b->sample_rate[u], b->speed_of_sound[u], order);
  if (st) return st;
  if (I < 1 || J < 1) return fail(RS_ERR_CONFIG, "scene needs a target and a microphone");
  /* Upper bound on lattice delay for RIR buffers. */
  double* conv[I * J];
  size_t conv_len[I * J];
  double pw[I * J];
  memset(conv, 0, sizeof conv);
  int64_t maxlen = 0;
  st = RS_OK;
  for (int64_t i = 0; i < I && !st; ++i) {
    const size_t nx = (size_t)b->sig_len[s0 + i];
    double* x = (double*)malloc((nx ? nx : 1) * sizeof(double));
    for (size_t k = 0; k < nx; ++k) x[k] = (double)b->signals[b->sig_off[s0 + i] + (int64_t)k];
    for (int64_t j = 0; j < J && !st; ++j) {
      const int64_t p = job->pair_begin[u] + i * J + j;
      /* RIR: synthesize (+ horizon) then optional truncate. */
      size_t cap = cap_taps > 0 ? (size_t)cap_taps : 0;
      if (cap == 0) {
        /* bound: farthest lattice image */
        double d2 = 0;
        for (int a = 0; a < 3; ++a) {
          double e = (fabs((double)order) + 1.0) * room[a] + room[a];
          d2 += e * e;
        }
        cap = (size_t)ceil(sqrt(d2) * b->sample_rate[u] / b->speed_of_sound[u]) + 2;
      }
      double* h = (double*)malloc(cap * sizeof(double));
      size_t nh = 0;
      st = orc_synthesize_rir(room, b->reflection[u], b->sample_rate[u], b->speed_of_sound[u],
                              order, b->src_pos + 3 * (s0 + i), b->mic_pos + 3 * (m0 + j),
                              cap_taps, h, cap, &nh);
      size_t keep = nh, n_c = 0;
      if (!st && b->eta_db > 0.0) st = orc_truncate_rir(h, nh, b->eta_db, &keep, &n_c, NULL);
      int strat = RS_OVERLAP_ADD;
      size_t fft_n = 0;
      double cost;
      if (!st) {
        if (b->plan_rule == RS_PLAN_CHOOSE)
          st = orc_choose_plan(1.0, 1.0, nx, keep, &strat, &fft_n, &cost);
        else if (b->plan_rule == RS_PLAN_FORCED)
          fft_n = (size_t)b->forced_fft_size;
        else
          fft_n = bit_ceil(2 * keep);
      }
      const size_t out_len = nx + keep - 1;
      double* y = NULL;
      if (!st) {
        y = (double*)malloc(out_len * sizeof(double));
        if (strat == RS_FULL_FFT)
          st = orc_convolve_full_fft(x, nx, h, keep, y);
        else if (strat == RS_DIRECT)
          st = orc_convolve_direct(x, nx, h, keep, y);
        else
          st = orc_convolve_ola(x, nx, h, keep, fft_n, y);
      }
      if (!st) st = orc_mean_power(y, out_len, &pw[i * J + j]);
      conv[i * J + j] = y;
      conv_len[i * J + j] = out_len;
      if ((int64_t)out_len > maxlen) maxlen = (int64_t)out_len;
      if (job->layout && !st) {
        rs_pair_layout* L = &job->layout[p];
        L->rir_len = (int64_t)nh;
        L->rir_keep = (int64_t)keep;
        L->cutoff = b->eta_db > 0.0 ? (int64_t)n_c : -1;
        L->fft_size = (int64_t)fft_n;
        L->block_len = (int64_t)(fft_n - keep + 1);
        L->n_blocks = (int64_t)orc_ola_block_count(nx, keep, fft_n);
        L->out_len = (int64_t)out_len;
        L->strategy = strat;
        L->flags = 0;
      }
      free(h);
    }
    free(x);
  }
  if (!st) {
    double alpha[I * J];
    for (int64_t j = 0; j < J && !st; ++j) {
      alpha[j] = 1.0; /* target gain */
      for (int64_t i = 1; i < I && !st; ++i)
        st = orc_compute_gain(pw[j], pw[i * J + j], b->snr_db[s0 + i], &alpha[i * J + j]);
    }
    if (!st) {
      if (maxlen > job->out_stride[u]) st = fail(RS_ERR_UNSUPPORTED, "output stride too small");
    }
    if (!st) {
      for (int64_t j = 0; j < J; ++j) {
        double* yj = job->out + job->out_off[u] + j * job->out_stride[u];
        memset(yj, 0, (size_t)maxlen * sizeof(double));
        for (int64_t i = 0; i < I; ++i) { /* source order */
          const double a = alpha[i * J + j];
          const double* c = conv[i * J + j];
          for (size_t n = 0; n < conv_len[i * J + j]; ++n) yj[n] += a * c[n];
        }
      }
      if (job->out_len) job->out_len[u] = maxlen;
      for (int64_t k = 0; k < I * J; ++k) {
        const int64_t p = job->pair_begin[u] + k;
        if (job->gains) job->gains[p] = alpha[k];
        if (job->power) job->power[p] = pw[k];
      }
    }
  }
  for (int64_t k = 0; k < I * J; ++k) free(conv[k]);
  return st;
}

static void* render_worker(void* arg) {
  render_job* job = (render_job*)arg;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    const int64_t u = job->next++;
    const int stop = job->status != 0;
    pthread_mutex_unlock(&job->mu);
    if (stop || u >= job->b->n_utt) break;
    const int st = render_one(job, u);
    if (st) {
      pthread_mutex_lock(&job->mu);
      if (!job->status) {
        job->status = st;
        snprintf(job->err, sizeof job->err, "%s", g_err);
      }
      pthread_mutex_unlock(&job->mu);
    }
  }
  return NULL;
}

int orc_render_batch(const rs_scene_batch* b, double* out, const int64_t* out_off,
                     const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                     double* gains, double* power, int threads) {
  render_job job;
  memset(&job, 0, sizeof job);
  job.b = b; job.out = out; job.out_off = out_off; job.out_stride = out_stride;
  job.out_len = out_len; job.layout = layout; job.gains = gains; job.power = power;
  job.pair_begin = (int64_t*)malloc((size_t)(b->n_utt + 1) * sizeof(int64_t));
  job.pair_begin[0] = 0;
  for (int64_t u = 0; u < b->n_utt; ++u)
    job.pair_begin[u + 1] = job.pair_begin[u] + (b->src_begin[u + 1] - b->src_begin[u]) *
                                                    (b->mic_begin[u + 1] - b->mic_begin[u]);
  pthread_mutex_init(&job.mu, NULL);
  if (threads <= 1) {
    render_worker(&job);
  } else {
    pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, render_worker, &job);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&job.mu);
  free(job.pair_begin);
  if (job.status) snprintf(g_err, sizeof g_err, "%s", job.err);
  return job.status;
}

/*
 * roomsim_gpu.h — C-ABI of the B200 (sm_100a) room-simulation hot path.
 *
 * This is the drop-in boundary between the reference's C++ simulator API
 * (header-only library `roomsim`, /root/reference/proj/include/roomsim/X.hpp)
 * and the hand-written CUDA kernels in paper_1712_03439_b200/csrc/.  Every
 * entry point takes plain pointers and sizes; no CUDA or torch types appear
 * in the signatures (streams are passed as opaque `void*`).
 *
 * Each function names the reference interface it replaces.  Citation
 * convention: `roomsim/X.hpp:N` is /root/reference/proj/include/roomsim/X.hpp
 * line N; `SPEC.md:N` is /root/reference/SPEC.md line N.
 *
 * Status codes map 1:1 onto the reference exception taxonomy
 * (roomsim/errors.hpp:22-68).  On a non-zero status, rs_last_error() returns
 * the message the reference would have put in `Error::what()`.
 */
#ifndef ROOMSIM_GPU_H_
#define ROOMSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (roomsim/errors.hpp:22-68) ------------------------------ */
enum rs_status {
  RS_OK = 0,
  RS_ERR_PLACEMENT = 1,   /* PlacementError        errors.hpp:29-32 */
  RS_ERR_GEOMETRY = 2,    /* GeometryError         errors.hpp:35-38 */
  RS_ERR_DEGENERATE = 3,  /* DegenerateInputError  errors.hpp:41-44 */
  RS_ERR_PLAN = 4,        /* PlanError             errors.hpp:47-50 */
  RS_ERR_CONFIG = 5,      /* ConfigError           errors.hpp:53-56 */
  RS_ERR_FORMAT = 6,      /* FormatError           errors.hpp:59-62 */
  RS_ERR_IO = 7,          /* IoError               errors.hpp:65-68 */
  RS_ERR_CUDA = 16,       /* device / driver failure (no reference analogue) */
  RS_ERR_OOM = 17,        /* device allocation failure */
  RS_ERR_UNSUPPORTED = 18 /* size outside what the kernels implement */
};

/* ---- convolution strategies (roomsim/convolution.hpp:33) ------------------ */
enum rs_strategy { RS_DIRECT = 0, RS_FULL_FFT = 1, RS_OVERLAP_ADD = 2 };

/* ---- how render() picks the FFT size of each (source, mic) pair ----------- */
enum rs_plan_rule {
  RS_PLAN_CHOOSE = 0,     /* choose_plan() per pair (convolution.hpp:157-161) */
  RS_PLAN_FORCED = 1,     /* overlap_add at forced_fft_size (plan_hint) */
  RS_PLAN_POW2_TWICE = 2  /* overlap_add at bit_ceil(2*N_h) (BASELINE configs 3-4) */
};

/* Opaque per-device context: one device, one stream, one arena.  Not to be
 * shared by concurrent callers (the reference's engine rule, fft.hpp:36-37). */
typedef struct rs_ctx rs_ctx;

const char* rs_last_error(void);        /* thread-local Error::what() mirror */
const char* rs_version(void);

int rs_ctx_create(int device, rs_ctx** out);
int rs_ctx_destroy(rs_ctx* ctx);
/* Launch all work of `ctx` on `stream` (a cudaStream_t; NULL = the ctx's own). */
int rs_ctx_set_stream(rs_ctx* ctx, void* stream);
int rs_ctx_synchronize(rs_ctx* ctx);
/* Device time (ms) of the OLA filter kernels (K4) of the last render, measured
 * with CUDA events on the launching streams; also total algorithmic flops and
 * bytes of that render (SURVEY.md §8d formulas). */
int rs_ctx_last_timing(rs_ctx* ctx, double* ola_ms, double* ola_flops,
                       double* alg_bytes, int64_t* kernel_launches);
/* Output channels of the last render mixed inside the K4 launches (the SNR-scaled mix,
 * SPEC.md:338-356, fused into the overlap-add epilogue: the last work item of a channel
 * mixes it) and all output channels of that render; the rest went through the mix kernel. */
int rs_ctx_mix_counts(rs_ctx* ctx, int64_t* fused_channels, int64_t* channels);
/* on = 0: every channel of this ctx's renders goes through the mix kernel; 1: the K4 epilogue
 * mixes the channels it can (the default); -1: the process default (RSG_FUSED_MIX).  The
 * rendered bytes are the same either way. */
int rs_ctx_set_fused_mix(rs_ctx* ctx, int on);
/* Device time (ms) of the stages of the last render (profiling on), summed over
 * the render's chunks: [0] inputs + K1 synth + K2 cut (stream A), [4] K4 OLA
 * (with the mix of the channels its epilogue covers), [5] K5 gains + K6 mix of the remaining
 * channels (filter stream; with chunks alternating between two filter streams the window
 * also sees the wait for SMs under the next chunk's K4); [1..3] are 0 (the host planner and K3 run
 * overlapped with the other stream); host_plan_ms = host wall time of the
 * planner.  Entries are -1 when unavailable. */
int rs_ctx_stage_times(rs_ctx* ctx, double* ms, int n, double* host_plan_ms);
/* Enable event timing of the OLA kernels (adds events; off by default).  Level 2
 * (diagnostic) also serializes the K4 launches of each chunk on one stream and times
 * every (FFT size, kernel variant) span separately: rs_ctx_k4_breakdown. */
int rs_ctx_set_profiling(rs_ctx* ctx, int enabled);
/* Per-(executed log2 N, variant) rows of the last render at profiling level 2 (variant: 0
 * ola_small_kernel, 1 in-place ola_ip_kernel, 2 two-stream ola2_kernel, 3 four-step, 4 two
 * blocks per transform ola_ipc_kernel): pairs, algorithmic FFT flops ((2B+1) 5 N log2 N per
 * pair, N and B of the REFERENCE's plan), device ms, and the same formula on the plan the
 * device executed (batched renders re-block).  Returns the row count (rows
 * beyond `cap` are not written); negative on error. */
int rs_ctx_k4_breakdown(rs_ctx* ctx, int cap, int32_t* log2n, int32_t* variant, int64_t* pairs,
                        double* flops, double* ms, double* exec_flops);

/* ---- host-side planner (convolution.hpp:72-161), exact FP64 mirror -------- */
double rs_cost_direct(double num_sources, double num_mics, size_t nx, size_t nh);
double rs_cost_full_fft(double num_sources, double num_mics, size_t nx, size_t nh,
                        size_t fft_size);
double rs_cost_ola(double num_sources, double num_mics, size_t nx, size_t nh,
                   size_t fft_size);
size_t rs_ola_block_count(size_t nx, size_t nh, size_t fft_size);
/* plan_for (convolution.hpp:130-152) / choose_plan (:157-161). */
int rs_plan_for(double num_sources, double num_mics, size_t nx, size_t nh,
                int strategy, int* strategy_out, size_t* fft_size_out, double* cost_out);
int rs_choose_plan(double num_sources, double num_mics, size_t nx, size_t nh,
                   int* strategy_out, size_t* fft_size_out, double* cost_out);

/* ---- RealFftEngine seam (fft.hpp:38-49, RadixTwoRealFft fft.hpp:57-169) ---
 * Batch of `count` transforms of size n (power of two, 2 <= n <= 2^23; n > 32768 runs
 * through the four-step stages).
 * forward: in [count][n] reals -> out [count][n/2+1] complex (re,im
 * interleaved), unnormalized.  inverse: includes 1/N (fft.hpp:33-36).
 * Host pointers; FP32 arithmetic on the device.                             */
int rs_rfft_forward(rs_ctx* ctx, size_t n, size_t count, const double* in, double* out);
int rs_rfft_inverse(rs_ctx* ctx, size_t n, size_t count, const double* in, double* out);

/* ---- room model (room_model.hpp:104-213) ---------------------------------
 * synthesize_rir (room_model.hpp:141-174), FP64, bit-exact.  `max_taps` > 0
 * keeps only the first max_taps taps (the fixture's T60 horizon); 0 keeps the
 * full lattice length max_delay+1.  `out` must hold `cap` doubles; the
 * produced length is written to *len (RS_ERR_UNSUPPORTED if len > cap).    */
int rs_synthesize_rir(rs_ctx* ctx, const double room_dims[3], double reflection,
                      double sample_rate, double speed_of_sound, int image_order,
                      const double src[3], const double mic[3], int64_t max_taps,
                      double* out, size_t cap, size_t* len);
/* truncate_rir (room_model.hpp:203-213): keep = min(n_c+2, n). */
int rs_truncate_rir(rs_ctx* ctx, const double* h, size_t n, double eta_db,
                    size_t* keep, size_t* cutoff_index, double* threshold);

/* ---- convolution (convolution.hpp:164-271) -------------------------------
 * x: nx doubles (mono AudioBuffer), h: nh doubles (Rir.samples), out:
 * nx+nh-1 doubles.  The FFT strategies compute in FP32 on the device
 * (max |err| <= 1e-5 of the peak); convolve_direct in FP64, bit-exact.
 * rs_convolve dispatches on strategy like roomsim::convolve
 * (convolution.hpp:258-271): RS_DIRECT -> rs_convolve_direct, RS_FULL_FFT ->
 * rs_convolve_full_fft, RS_OVERLAP_ADD -> rs_convolve_ola (fft_size 0 is a
 * PlanError, "overlap-add plan is missing an FFT size").                    */
/* convolve_direct (convolution.hpp:164-179): the definition sum, FP64, with the
 * reference's accumulation order (bit-exact). */
int rs_convolve_direct(rs_ctx* ctx, const double* x, size_t nx, const double* h, size_t nh,
                       double* out);
int rs_convolve_ola(rs_ctx* ctx, const double* x, size_t nx, const double* h, size_t nh,
                    size_t fft_size, double* out);
int rs_convolve_full_fft(rs_ctx* ctx, const double* x, size_t nx, const double* h,
                         size_t nh, double* out);
int rs_convolve(rs_ctx* ctx, const double* x, size_t nx, const double* h, size_t nh,
                int strategy, size_t fft_size, double* out);

/* ---- batched scene render: synth -> cut -> plan -> OLA -> SNR mix --------
 * The hot path of BASELINE.json north_star.  One call renders n_utt scenes
 * (SPEC.md:348-356 `render`), each with I_u = src_begin[u+1]-src_begin[u]
 * sources (source 0 is the target, gain 1) and J_u mics.  Pairs are numbered
 * utterance-major, then source, then mic: pair = pair_begin(u) + i*J_u + j.
 * All metadata arrays are host pointers.                                    */
typedef struct rs_scene_batch {
  int64_t n_utt;
  const int64_t* src_begin;    /* [n_utt+1] CSR into sources */
  const int64_t* mic_begin;    /* [n_utt+1] CSR into mics */
  const double* room_dims;     /* [n_utt*3] RoomConfig.dimensions (room_model.hpp:50) */
  const double* reflection;    /* [n_utt]   RoomConfig.reflection_coefficient */
  const double* sample_rate;   /* [n_utt]   RoomConfig.sample_rate */
  const double* speed_of_sound;/* [n_utt]   RoomConfig.speed_of_sound */
  const int32_t* image_order;  /* [n_utt]   RoomConfig.image_order (K) */
  const int64_t* max_taps;     /* [n_utt]   RIR horizon cap (0 = none) */
  const double* src_pos;       /* [n_src*3] */
  const double* mic_pos;       /* [n_mic*3] */
  const double* snr_db;        /* [n_src]   (the target's entry is ignored) */
  const int64_t* sig_off;      /* [n_src]   sample offset of source signal in `signals` */
  const int64_t* sig_len;      /* [n_src]   N_x of each source */
  const float* signals;        /* packed FP32 samples (host or device, see below) */
  double eta_db;               /* > 0: truncate_rir(h, eta_db); <= 0: untruncated */
  int32_t plan_rule;           /* enum rs_plan_rule */
  int64_t forced_fft_size;     /* for RS_PLAN_FORCED */
} rs_scene_batch;

/* Per-pair layout report, for bit-exact checks against the reference. */
typedef struct rs_pair_layout {
  int64_t rir_len;     /* synthesized (horizon-cut) length */
  int64_t rir_keep;    /* length after truncate_rir (== rir_len if eta <= 0) */
  int64_t cutoff;      /* n_c (room_model.hpp:188-197), -1 if untruncated */
  int64_t fft_size;    /* N */
  int64_t block_len;   /* L = N - N_h + 1 (convolution.hpp:230) */
  int64_t n_blocks;    /* B = ceil(N_x / L) (convolution.hpp:108-112) */
  int64_t out_len;     /* N_x + N_h - 1 */
  int32_t strategy;    /* enum rs_strategy of the plan */
  int32_t flags;       /* nonzero: geometry error on device */
} rs_pair_layout;

/* Output: mic j of utterance u is written at out + out_off[u] + j*out_stride[u]
 * for n < out_len[u] (channel length = max_{i,j}(N_x,i + N_h,ij - 1),
 * SPEC.md:334).  out_stride[u] must be >= that length; an upper bound is
 * max_i N_x,i + max_taps[u] - 1 (or the untruncated lattice length).
 * `layout` [n_pairs], `gains` [n_pairs] (alpha_ij),
 * `power` [n_pairs] (mean_power of each reverberant pair signal) and
 * out_len [n_utt] are host arrays and may be NULL.
 *
 * rs_render_batch: `signals` and `out` are HOST pointers (pinned or pageable);
 *   H2D/D2H copies are part of the call (the e2e path).
 * rs_render_batch_device: `signals` and `out` are DEVICE pointers on the ctx's
 *   device (inputs resident in HBM; the throughput path).                    */
int64_t rs_batch_num_pairs(const rs_scene_batch* batch);
int rs_render_batch(rs_ctx* ctx, const rs_scene_batch* batch, float* out,
                    const int64_t* out_off, const int64_t* out_stride, int64_t* out_len,
                    rs_pair_layout* layout, double* gains, double* power);
int rs_render_batch_device(rs_ctx* ctx, const rs_scene_batch* batch, float* out_dev,
                           const int64_t* out_off, const int64_t* out_stride,
                           int64_t* out_len, rs_pair_layout* layout, double* gains,
                           double* power);
/* Copy the reverberant (pre-mix) signal h_ij * x_i of pair `pair` of the last
 * render to host memory (debug / SNR-fidelity checks). `cap` floats. */
int rs_last_pair_signal(rs_ctx* ctx, int64_t pair, float* out, size_t cap, size_t* len);
/* Copy the synthesized (and truncated) RIR of pair `pair` of the last render. */
int rs_last_pair_rir(rs_ctx* ctx, int64_t pair, double* out, size_t cap, size_t* len);

/* ---- scene sampler and signal generator (SPEC.md:141-192 config_sampler; SURVEY.md
 * §8f row 1).  The reference specifies the sampler contract but ships no code.  Every
 * scene is a pure function of (seed, utterance, epoch) (Philox4x32-10 counter streams
 * keyed by a hash of the three); the host functions are the fixture generator and
 * produce the same bits as the device functions (one shared source, IEEE basic ops
 * only).  Noise count: categorical over 0..n_weights-1 when n_weights > 0 (SPEC
 * default weights 0.15/0.35/0.30/0.20, mean 1.55), else num_noises.              */
typedef struct rs_sampler_spec {
  double dim_lo[3], dim_hi[3];   /* room dimension ranges, metres */
  double refl_lo, refl_hi;       /* reflection coefficient range (t60_hi <= 0) */
  double t60_max;                /* resample while Eyring T60 > t60_max (t60_hi <= 0) */
  double t60_lo, t60_hi;         /* t60_hi > 0: sample T60, r = exp(-0.0805 V / (S T60)) */
  double snr_lo, snr_hi;         /* SNR range, dB (noise sources) */
  double mic_spacing;            /* line array (mic_radius <= 0): 1 or 2 mics */
  double mic_radius;             /* > 0: circular array of mic_count mics */
  double clearance;              /* minimum distance of every placement to the walls */
  double sec_lo, sec_hi;         /* utterance duration range, seconds */
  double fs, c0;                 /* sample rate, speed of sound */
  double signal_std;             /* synthetic signals: N(0, signal_std^2) */
  int32_t num_noises;            /* fixed noise count when n_weights == 0 */
  int32_t mic_count;
  int32_t n_weights;             /* 0..8 */
  int32_t pad_;
  double weights[8];
} rs_sampler_spec;

/* Sources per utterance (1 + noise count) of utterances first_utt .. first_utt+n_utt-1. */
int rs_sampler_counts(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt,
                      int64_t epoch, int32_t* n_src);
/* Scenes into the rs_scene_batch arrays (host).  src_begin: CSR from rs_sampler_counts;
 * mic_pos holds n_utt * mic_count rows; max_taps = ceil(T60 fs) (the T60 horizon);
 * n_samples = N_x per utterance (shared by its sources). */
int rs_sample_scenes(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt, int64_t n_utt,
                     int64_t epoch, const int64_t* src_begin, double* room_dims, double* reflection,
                     int32_t* image_order, int64_t* max_taps, double* src_pos, double* mic_pos,
                     double* snr_db, int64_t* n_samples);
/* The same on the device (all pointers device memory; `stream` a cudaStream_t or NULL). */
int rs_sampler_counts_device(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt,
                             int64_t n_utt, int64_t epoch, int32_t* n_src_dev, void* stream);
int rs_sample_scenes_device(const rs_sampler_spec* spec, uint64_t seed, int64_t first_utt,
                            int64_t n_utt, int64_t epoch, const int64_t* src_begin_dev,
                            double* room_dims, double* reflection, int32_t* image_order,
                            int64_t* max_taps, double* src_pos, double* mic_pos, double* snr_db,
                            int64_t* n_samples, void* stream);
/* Synthetic source signals, N(0, signal_std^2) (Box-Muller on Philox), keyed by
 * (seed, utterance, epoch) and the source's index within its utterance; written at
 * out + sig_off[s] for sig_len[s] samples.  Metadata arrays are host arrays. */
int rs_generate_signals_host(const rs_sampler_spec* spec, uint64_t seed, int64_t epoch, int64_t n_src,
                             const int64_t* utt_of_src, const int32_t* src_local,
                             const int64_t* sig_off, const int64_t* sig_len, float* out);
int rs_generate_signals(const rs_sampler_spec* spec, uint64_t seed, int64_t epoch, int64_t n_src,
                        const int64_t* utt_of_src, const int32_t* src_local, const int64_t* sig_off,
                        const int64_t* sig_len, float* out_dev, void* stream);
/* The same generator for a fixed batch across epochs: the per-source table is built and
 * uploaded once (create); each epoch is then one kernel launch on `stream` with no host
 * work, allocation or synchronisation (generate).  Bit-exact with the calls above. */
typedef struct rs_signal_plan rs_signal_plan;
int rs_signal_plan_create(const rs_sampler_spec* spec, uint64_t seed, int64_t n_src,
                          const int64_t* utt_of_src, const int32_t* src_local,
                          const int64_t* sig_off, const int64_t* sig_len, rs_signal_plan** out);
int rs_signal_plan_generate(rs_signal_plan* plan, int64_t epoch, float* out_dev, void* stream);
int rs_signal_plan_destroy(rs_signal_plan* plan);

/* ---- log-Mel front end -------------------
 * 128 log-Mel energies per 32 ms frame (512 samples, periodic Hann) every 10 ms (160
 * samples), HTK-mel triangles 125-7500 Hz on |X|^2, ln(max(E, 1e-10)); 4 frames
 * stacked into 512-element vectors, down-sampled by 3 (vector t = frames 3t..3t+3).
 * For 16 kHz audio.  Channel ch: chan_len[ch] samples at wave_dev + chan_off[ch];
 * its n_stacked vectors are written at feat_dev + feat_off[ch] (device pointers,
 * host offset arrays). */
int rs_logmel_shape(int64_t n_samples, int64_t* n_frames, int64_t* n_stacked);
int rs_logmel_device(rs_ctx* ctx, const float* wave_dev, int64_t n_chan, const int64_t* chan_off,
                     const int64_t* chan_len, float* feat_dev, const int64_t* feat_off);
/* The render with the log-Mel front end fused into the mix (one kernel per chunk: each
 * output tile is mixed into shared memory and the frames starting in it are featurized
 * there): rs_render_batch_device's arguments plus feat_dev / feat_off (per output channel,
 * utterance-major then mic; capacity from rs_logmel_shape(out_stride[u])).  out_dev may be
 * NULL: the waveforms are then never written to HBM (the fused kernel).  With out_dev the
 * waveforms are mixed in the overlap-add launches' epilogue and the log-Mel reads them back
 * (measured faster than the fused kernel when the waveforms are wanted anyway).  Features are
 * bit-identical to rs_logmel_device on the rendered channels either way. */
int rs_render_features_device(rs_ctx* ctx, const rs_scene_batch* batch, float* out_dev,
                              const int64_t* out_off, const int64_t* out_stride, int64_t* out_len,
                              rs_pair_layout* layout, double* gains, double* power, float* feat_dev,
                              const int64_t* feat_off);

#ifdef __cplusplus
}
#endif
#endif /* ROOMSIM_GPU_H_ */

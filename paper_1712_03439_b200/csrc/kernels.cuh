// kernels.cuh — device-side data layout shared by the kernels and the host
// orchestration (api.cu).  See DESIGN.md §"Data layout in HBM".
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

namespace rsg {

// Raise — never lower — a kernel's dynamic shared-memory limit.  Launch sites whose size varies
// with the batch (carry / slice capacities) call this instead of cudaFuncSetAttribute: renders
// running in several host threads (one context each) launch the same kernels with different
// sizes, and a limit set to exactly one launch's size could be lowered by another thread between
// this call and the launch ("invalid argument").
template <class K>
inline cudaError_t ensure_dynamic_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = cur[std::make_pair(dev, reinterpret_cast<const void*>(kern))];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) have = bytes;
  return e;
}

// Per utterance (room) — RoomConfig (roomsim/room_model.hpp:49-72) plus the
// host-computed constants that must match glibc bit for bit.
struct UttMeta {
  double dims[3];
  double spm;        // samples_per_meter = fs / c0 (room_model.hpp:150), host FP64
  int32_t order;     // K
  int32_t rg_off;    // offset of the r^g table (g = 0..3K, std::pow on the host)
  int64_t max_taps;  // horizon cap (0 = none)
};

// Per (source, mic) pair.
struct PairMeta {
  double src[3];
  double mic[3];
  int32_t utt;
  int32_t src_idx;   // global source index (signal, snr)
  int32_t mic_local; // j
  int32_t src_local; // i
  int64_t sig_off;   // offset of x_i in the signal buffer
  int64_t nx;        // N_x
  int64_t rir_off;   // FP64 RIR region (synth output) [rir_cap]
  int64_t rir_cap;
};

// Per pair, produced on device by K1/K2, consumed by the planner.
struct PairRir {
  unsigned long long max_delay;  // K1 atomicMax over images
  int64_t len;                   // min(max_delay + 1, horizon)
  int64_t keep;                  // after truncate_rir
  int64_t cutoff;                // n_c
  double threshold;              // p_th (room_model.hpp:184)
  int32_t flags;                 // 1: geometry error (d <= 0), 2: degenerate (all-zero)
  int32_t exact_len;             // > 0: K1 synthesizes only bins [0, exact_len) (synth_bound.cu): every
                                 // later bin is provably below the cut threshold; 0: the whole RIR
};

// Per pair, written by the host planner (after K2) and consumed by K3/K4/mix.
struct PairPlan {
  int64_t spec_off;  // float2 offset of G (M+1 bins)
  int64_t y_off;     // float offset of the reverberant pair signal
  int64_t nh;        // N_h (truncated)
  int64_t L;         // block length N - N_h + 1
  int64_t B;         // block count
  int64_t out_len;   // N_x + N_h - 1
  int32_t log2n;     // N = 2^log2n
  int32_t npart;     // power partials of this pair (consecutive, see power.cuh)
  int64_t part0;     // index of the pair's first power partial
};

// K4 work item: a run of OLA blocks of one pair.  The item owns output
// positions [b_own*L, b_end*L) (to out_len for the pair's last run) and also
// recomputes blocks [b_begin, b_own) whose tails overlap that range, so runs
// are independent: no seams, no atomics, deterministic.
struct OlaItem {
  int32_t pair;
  int32_t b_begin;
  int32_t b_own;
  int32_t b_end;
};

// K1 work item: one (pair, bin-slice).
struct SynthItem {
  int32_t pair;
  int32_t slice_lo;  // first bin of the slice
  int32_t slice_len; // bins in the slice
  int32_t pad;
};

struct SynthArgs {
  const UttMeta* utt;
  const PairMeta* pair;
  const double* rg;
  const SynthItem* items;
  double* rir;
  PairRir* out;
};

// K1a (synth_bound.cu): for truncated renders, the prefix of each RIR that truncate_rir can keep.
struct SynthBoundArgs {
  const UttMeta* utt;
  const PairMeta* pair;
  const double* rg;
  const int32_t* pairs;  // pairs of this launch
  PairRir* out;          // exact_len, max_delay, geometry flag
  double eta_factor;     // pow(10, -eta/10), host std::pow; > 0
};
constexpr int kBoundMaxCap = 32768;  // longest RIR (bins) the bound pass takes
cudaError_t launch_synth_bound(const SynthBoundArgs& a, int n_pairs, int cap, int max_order, cudaStream_t s, int nt);

struct CutArgs {
  const PairMeta* pair;
  const UttMeta* utt;
  const double* rir;
  PairRir* out;
  double eta_factor;  // pow(10, -eta/10), host std::pow; <= 0: no truncation
};

// Filter layout of the two-blocks-per-transform K4 (big.cu, ola_ipc_kernel<C>): all C = N
// bins of H / N, bin k at r * (C / R2) + u with slot(k) = (k mod R0) S0 + ((k / R0) mod R1) S1 +
// k / (R0 R1) (the in-place transform's digit-reversed slot), u = slot / R2, r = slot mod R2.
struct IpcPerm {
  int32_t on = 0;
  int32_t lr0 = 0, lr1 = 0, lr2 = 0, lc = 0;  // log2 of the radices and of C
  __host__ __device__ int index(int k) const {
    const int slot = ((k & ((1 << lr0) - 1)) << (lr1 + lr2)) | (((k >> lr0) & ((1 << lr1) - 1)) << lr2) |
                     (k >> (lr0 + lr1));
    return ((slot & ((1 << lr2) - 1)) << (lc - lr2)) | (slot >> lr2);
  }
  __host__ __device__ int bin(int idx) const {  // inverse of index()
    const int slot = ((idx & ((1 << (lc - lr2)) - 1)) << lr2) | (idx >> (lc - lr2));
    return (slot >> (lr1 + lr2)) | (((slot >> lr2) & ((1 << lr1) - 1)) << lr0) |
           ((slot & ((1 << lr2) - 1)) << (lr0 + lr1));
  }
};

struct SpecArgs {
  const int32_t* list;  // pairs of this FFT size
  int32_t count;
  const PairMeta* pair;
  const PairPlan* plan;
  const double* rir;
  float2* spec;
  const float2* tw;     // twiddle tables of this M
  IpcPerm perm;         // on: write H / N over all N bins in ola_ipc_kernel's order
};

struct OlaArgs {
  const OlaItem* items;
  int32_t count;
  const PairMeta* pair;
  const PairPlan* plan;
  const float* signals;
  const float2* spec;
  float* y;             // reverberant pair signals
  double* part;         // power partials: segment s, warp w of a pair at plan.part0 + s * ppb + w
  const float2* tw;
  int32_t seg = 16;     // OLA blocks per power segment (power.cuh)
  // ola_ipc_kernel only: the FP64 RIRs (PairMeta::rir_off).  Non-null: every work item transforms
  // its pair's truncated RIR itself and writes H / N to `spec` in the butterflies' order before
  // its first block (no K3 launch for the span); null: `spec` was filled by K3.
  const double* rir = nullptr;
  // ola_ip_kernel / ola_ipc_kernel: the K4 epilogue's state (mixfin.cuh) — the last work item of
  // an output channel mixes it.  Null: mix_kernel mixes every channel.
  const struct MixFin* fin = nullptr;
};

struct MixArgs {
  const int64_t* chan_utt;    // per output channel: utterance
  const int32_t* chan_mic;    // j
  const int64_t* chan_out;    // float offset of the channel in `out`
  const int64_t* utt_len;     // output length per utterance
  const int64_t* utt_stride;  // channel stride per utterance (tail zero-filled)
  const int64_t* utt_pair0;   // first pair of the utterance
  const int32_t* utt_I;
  const int32_t* utt_J;
  const PairPlan* plan;
  const float* y;
  const double* gain;
  float* out;
  int64_t tile;               // samples per CTA
};

struct GainArgs {
  const PairMeta* pair;
  const PairPlan* plan;
  const int64_t* utt_pair0;
  const int32_t* utt_J;
  const double* part;         // power partials (PairPlan::part0 / npart), summed in a fixed order
  const double* snr_lin;      // per global source: pow(10, snr/10) (host std::pow)
  double* gain;
  double* power;
  int32_t* flags;
  int64_t n_pairs;
};

// K4 two-stream variant (ola2.cu): runs A and B of one pair share each complex
// transform.  Owned ranges as OlaItem.
struct OlaItem2 {
  int32_t pair;
  int32_t a_begin, a_own, a_end;
  int32_t b_begin, b_own, b_end;
  int32_t pad;
};

struct Ola2Args {
  const OlaItem2* items;
  int32_t count;
  const PairMeta* pair;
  const PairPlan* plan;
  const float* signals;
  const float2* spec;   // K3's G = H / (2N), k in [0, N/2]
  float* y;
  double* part;         // power partials (as OlaArgs::part, per run's block)
  const float2* twf;    // PlanC<N, false> pass tables
  const float2* twi;    // PlanC<N, true> pass tables
  int32_t ccap;         // floats per carry buffer: >= max N_h - 1 of the launch, multiple of 4
  int32_t scap;         // floats per input window: >= max L + 8 of the launch, multiple of 4
};
constexpr int kOla2MinLog2N = 5, kOla2MaxLog2N = 12;
bool ola2_supported(int log2n);
int ola2_resident_items(int log2n);
int ola2_tw_total(int log2n, bool rev);
void ola2_fill_twiddles(int log2n, bool rev, float2* host);
cudaError_t launch_ola2(int log2n, const Ola2Args& a, cudaStream_t s);

// log-Mel front end (features.cu).
// Per channel; a tile is 8 consecutive frames of one channel, tiles are numbered channel by
// channel (tile_begin) and the kernel finds a tile's channel by a warp-wide 32-ary search — the
// host never lists the ~10^6 tiles of a batch.
struct LogMelChan {
  int64_t wave_off;    // channel start in `wave`
  int64_t feat_off;    // channel start in `feat` (stacked vectors of 512 floats)
  int32_t tile_begin;  // first tile of the channel
  int32_t nstack;      // stacked vectors of the channel; frames that reach one: 3 (nstack - 1) + 4
};
struct LogMelArgs {
  const float* wave;
  float* feat;
  const LogMelChan* chans;  // n_chan + 1 entries: the last one's tile_begin = n_tiles
  int32_t n_chan;
  int32_t n_tiles;
  const float* window;    // [512] periodic Hann
  const int32_t* mel_ptr; // [129] CSR rows of the filterbank
  const int32_t* mel_bin;
  const float* mel_w;
  const float2* tw;       // Plan<256> tables
  float log_floor;
};
cudaError_t launch_logmel(const LogMelArgs& a, cudaStream_t s);
// Mix + log-Mel fused (features.cu): MixArgs::out may be null (waveforms not written).
struct MixFeatArgs {
  float* feat;
  const int64_t* feat_off;  // per output channel of the launch (device)
  const float* window;
  const int32_t* mel_ptr;
  const int32_t* mel_bin;
  const float* mel_w;
  const float2* tw;         // Plan<256> tables
  float log_floor;
};
cudaError_t launch_mix_logmel(const MixArgs& a, const MixFeatArgs& lf, int64_t n_chan, int64_t max_len,
                              cudaStream_t s);

// Large transforms (large.cu): four-step FFT through global scratch.
struct LargeArgs {
  const int2* units;         // (pair, block) per unit of this batch
  const int32_t* spec_pairs; // pairs of this batch (spectrum stages)
  int32_t n_units;
  int32_t n_spec;
  const PairMeta* pair;
  const PairPlan* plan;
  const float* signals;
  const double* rir;
  float2* spec;              // per pair: G(k1 + M1 k2) at [k1*M2 + k2], G(M) at [M]
  float2* scratch;           // per unit: M complex
  float* yblk;               // per unit: N = 2M block output samples
  float* y;
  double* part;              // power partials: one per stage-D tile at plan.part0 + tile
  const OlaItem* items;      // stage-D tiles: {pair, tile, unit of block 0, 0}
  int32_t n_items;
  const float2* tw1;         // Plan<M1> twiddle tables
  const float2* tw2;         // Plan<M2> twiddle tables
};
constexpr int kLargeMaxLog2M = 22;  // M <= 2^22 (N <= 2^23) through the four-step path
void large_split(int log2m, int* l1, int* l2);
int large_tile();
// stage: 0/1 spectrum (cols, rows), 2 cols fwd, 3 rows, 4 cols inv, 5 overlap-add
cudaError_t launch_large(int log2m, const LargeArgs& a, int stage, cudaStream_t s);
// RealFftEngine seam for M = N/2 >= 8192: natural-order spectra through the same four-step
// stages; `scratch` holds count * M complex
cudaError_t launch_large_rfft(int log2m, bool inverse, const float* in_real, const float2* in_spec,
                              float* out_real, float2* out_spec, int count, float2* scratch,
                              const float2* tw1, const float2* tw2, cudaStream_t s);

// Power partials per OLA block of each K4 variant (one per warp of the group that
// transforms the block; power.cuh).
int small_parts_per_block(int log2m);  // ola_small_kernel<M>
int ip_parts_per_block(int log2m);     // ola_ip_kernel<M>
int ola2_parts_per_block(int log2n);   // ola2_kernel<N> (per run's block)

// ---- launchers (kernels.cu) --------------------------------------------------
// In-place one-CTA K4 for M = 8192, 16384 (big.cu); the carry (N_h - 1 floats) must fit
// next to the transform in shared memory.
bool ip_supported(int log2m, int64_t max_nh);
int ip_resident(int log2m, int64_t max_nh);  // CTAs (work items) resident per SM
cudaError_t launch_ola_ip(int log2m, const OlaArgs& a, int64_t max_nh, cudaStream_t s);

// Two blocks per complex transform (big.cu), N = 4096, 8192; the filter region holds N bins.
bool ipc_supported(int log2n, int64_t max_nh);
int ipc_resident(int log2n, int64_t max_nh);
int ipc_parts_per_block(int log2n);
IpcPerm ipc_perm(int log2n);
cudaError_t launch_ola_ipc(int log2n, const OlaArgs& a, int64_t max_nh, cudaStream_t s);

constexpr int kMaxLog2M = 14;  // M <= 16384  (N <= 32768) in one CTA
int cta_threads(int log2m);
int ola_groups(int log2m);     // K4 work items per CTA
int ola_resident_groups(int log2m);  // K4 work items resident per SM
size_t ola_smem_bytes(int log2m);
int tw_total(int log2m);       // float2 entries of the twiddle table of 2^log2m
void fill_twiddles(int log2m, float2* host);  // host, FP64 -> FP32
cudaError_t kernels_init();    // smem attributes

constexpr int kSynthThreads = 512;
constexpr int kSynthSlice = 10240;  // FP64 bins per K1 CTA (80 KB: two 512-thread CTAs per SM with 4 images/thread)
constexpr int kSynthCutSlice = 4096;  // FP64 bins per K1 CTA of a truncated synthesis (synth_bound.cu)
constexpr int kSynthBig = 22528;    // FP64 bins of the one-slice class (one 512-thread CTA per SM; + bin tags)
size_t synth_smem_bytes(int max_order, int slice, int nt, int ipt, int fold = 0, int ht = 256);

// nt = 512 (16 warps) or 128 (4 warps, small lattices)
cudaError_t launch_synth(const SynthArgs& a, int n_items, int max_order, int slice,
                         cudaStream_t s, int nt = 512);
cudaError_t launch_cut(const CutArgs& a, int n_pairs, cudaStream_t s);
cudaError_t launch_spectrum(int log2m, const SpecArgs& a, cudaStream_t s);
cudaError_t launch_ola(int log2m, const OlaArgs& a, cudaStream_t s);
cudaError_t launch_gain(const GainArgs& a, cudaStream_t s);  // K5: power (warp per pair) + gains
cudaError_t launch_mix(const MixArgs& a, int64_t n_chan, int64_t max_len, cudaStream_t s);
// dst/src: device or mapped-pinned-host pointers, 16-byte aligned
cudaError_t launch_pcie_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);
// Seam kernels (RealFftEngine): count transforms of size 2^(log2m+1).
cudaError_t launch_rfft(int log2m, bool inverse, const float* in_real, const float2* in_spec,
                        float* out_real, float2* out_spec, int count, const float2* tw,
                        cudaStream_t s);
// convolve_direct (convolution.hpp:164-179): FP64, bit-exact, out has nx + nh - 1 doubles
cudaError_t launch_direct_conv(const double* x, int64_t nx, const double* h, int64_t nh, double* out,
                               cudaStream_t s);
cudaError_t launch_convert_d2f(const double* in, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_convert_f2d(const float* in, double* out, int64_t n, cudaStream_t s);

}  // namespace rsg

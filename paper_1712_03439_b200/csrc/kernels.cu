// kernels.cu — the sm_100a kernels of the room-simulation hot path.
//
//   K1 rir_synth_kernel     synthesize_rir        roomsim/room_model.hpp:141-174 (FP64, bit-exact)
//   K2 rir_cut_kernel       power_threshold/cutoff_index/truncate_rir  room_model.hpp:177-213
//   K3 rir_spectrum_kernel  the RIR transform of convolve_ola         convolution.hpp:238-239
//   K4 ola_small_kernel     the OLA block loop + Σy^2                 convolution.hpp:242-253,
//                                                                     audio_buffer.hpp:66-75
//   K5 gain_kernel          SPEC compute_gain
//   K6 mix_kernel           SPEC render sum (channels K4's epilogue leaves)
//   rfft_*_kernel           RealFftEngine seam                        fft.hpp:38-49
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "async.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "mixfin.cuh"
#include "power.cuh"

#ifndef RSG_E
#define RSG_E 16
#endif
#ifndef RSG_E_SMALL
#define RSG_E_SMALL 8
#endif


namespace rsg {

// ============================================================================
// K1: image-method RIR synthesis, bit-exact against the reference.
//
// One CTA per (pair, slice of delay bins).  The RIR slice lives in shared
// memory as FP64.  Images are processed in enumeration order (nx -> ny -> nz,
// room_model.hpp:118-120) in chunks of NT, one per thread; every bin must
// receive its contributions sequentially in that order (rir[delay] += amp,
// :170).  Each chunk is resolved by "owner" warps: warp o owns the bins with
// (bin mod NW) == o.  After the chunk's images are computed, each warp
// publishes one ballot-built lane mask per owner; the entries are then
// counting-sorted into owner-major lists (stable: compute-warp order, then
// lane order = enumeration order), and each owner folds its list into the bins
// in rounds — round r applies the r-th entry of every equal-delay group, so
// no two lanes touch one bin at once and each bin sees its entries in order.
// All arithmetic uses _rn intrinsics so no FMA contraction can change a bit;
// r^g comes from the host's std::pow.
// ============================================================================
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// FP64 load from a 32-bit shared address (tables written before a __syncthreads)
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// *(double*)shared[a] = *(double*)shared[a] + v, round to nearest (no contraction)
__device__ __forceinline__ void shared_add_rn(unsigned a, double v) {
  double cur;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cur) : "r"(a) : "memory");
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(__dadd_rn(cur, v)) : "memory");
}

// IPT = images per thread per chunk (4 measured best; 2 where 4 would cost occupancy)
// FOLD: how a round of an owner's list is ordered — 0: match_any groups (NT = 128: claims
// measured 6% slower there); 2: ordered claims, no match_any (the 512-thread classes: K1 -15%
// on the one-CTA class vs byte tags + match_any, -10% on the sliced one vs match_any)
// HT: claim words per owner warp (FOLD 2; a power of two)
template <int NT, int IPT, int FOLD, int HT = 256>
__global__ void __launch_bounds__(NT) rir_synth_kernel(SynthArgs a, int slice_cap) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int NW = NT / 32;  // warps = owner warps
  constexpr int CH = IPT * NT;  // images per chunk: IPT x NW "virtual warps" of 32, in order
  constexpr int NV = IPT * NW;  // virtual warps per chunk
  static_assert(NW >= 2 && NW <= 32 && (NW & (NW - 1)) == 0, "power-of-two warp count");
  constexpr int OB = NW == 2 ? 1 : NW == 4 ? 2 : NW == 8 ? 3 : NW == 16 ? 4 : 5;  // owner bits
  constexpr int NQ = (NV + 3) / 4;  // 4-byte words per owner's count row
  // row stride in bytes: 16-byte aligned (uint4 row loads) and an odd number of 16-byte
  // units, so the owners' rows start in different banks (8-way conflicts otherwise)
  constexpr int RS = 16 * ((((4 * NQ + 15) / 16) % 2 == 0) ? (4 * NQ + 15) / 16 + 1 : (4 * NQ + 15) / 16);
  const SynthItem it = a.items[blockIdx.x];
  const PairMeta& pm = a.pair[it.pair];
  const UttMeta& um = a.utt[pm.utt];
  const int K = um.order, W = 2 * K + 1;
  const double spm = um.spm;
  double* bins = reinterpret_cast<double*>(sm);
  double* ax = bins + slice_cap;                 // [3][W] squared per-axis offsets
  double* rg = ax + 3 * W;                       // [3K+1]
  double* ent_a = rg + (3 * K + 1);              // [CH] owner-major sorted amplitudes
  int* ent_d = reinterpret_cast<int*>(ent_a + CH);           // [CH] their bins
  // [NW owner][NV virtual warp] entry counts, one byte each (<= 32), 16-byte aligned rows
  // of RS bytes (offset arithmetic keeps the accesses in the shared window: STS/LDS)
  const uintptr_t cnt_off = (reinterpret_cast<uintptr_t>(ent_d + CH) - reinterpret_cast<uintptr_t>(sm) + 15) & ~uintptr_t(15);
  unsigned char* cnt8 = sm + cnt_off;
  // FOLD 2's claim words follow the count rows
  const unsigned tag_s = static_cast<unsigned>(__cvta_generic_to_shared(sm)) +
                         static_cast<unsigned>(cnt_off + ((NW * RS + 15) & ~15));
  // per owner warp, HT 32-bit claim words, all ones between rounds
  if constexpr (FOLD == 2) {
    unsigned* cl = reinterpret_cast<unsigned*>(sm + cnt_off + ((NW * RS + 15) & ~15));
    for (int i = threadIdx.x; i < NW * HT; i += NT) cl[i] = 0xffffffffu;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Truncated renders (synth_bound.cu): only bins [0, exact_len) are needed
  const int exact_len = a.out[it.pair].exact_len;
  const int lo = it.slice_lo;
  const int len = exact_len > 0 ? min(it.slice_len, exact_len - lo) : it.slice_len;
  if (len <= 0) return;  // the slice lies beyond the exact range (CTA-uniform)
  // 32-bit shared address of the bins, computed once (laundered through asm: otherwise the
  // compiler re-derives the CTA's shared window, S2UR SR_CgaCtaId, at every use)
  unsigned bins_s;
  asm volatile("mov.b32 %0, %1;" : "=r"(bins_s) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(bins))));
  const unsigned ax_s = bins_s + 8u * static_cast<unsigned>(slice_cap);
  const unsigned rg_s = ax_s + 8u * static_cast<unsigned>(3 * W);
  for (int l = tid; l < len; l += NT) bins[l] = 0.0;
  for (int idx = tid; idx < 3 * W; idx += NT) {
    const int axis = idx / W, n = idx - axis * W - K;
    const double L = um.dims[axis], s = pm.src[axis];
    // room_model.hpp:126-127: mirrored = n even ? s : L - s; pos = n*L + mirrored
    const double mirrored = (n % 2 == 0) ? s : __dsub_rn(L, s);
    const double pos = __dadd_rn(__dmul_rn(static_cast<double>(n), L), mirrored);
    const double diff = __dsub_rn(pos, pm.mic[axis]);  // room_model.hpp:37 (a - b)
    ax[idx] = __dmul_rn(diff, diff);                    // :43 v.x * v.x
  }
  for (int g = tid; g <= 3 * K; g += NT) rg[g] = a.rg[um.rg_off + g];
  // Sub-lattice [x0, x0 + bx) x [y0, y0 + by) x [z0, z0 + bz): the whole lattice, or — when only
  // bins [0, exact_len) are wanted — the box around the sphere of delay exact_len: an image
  // outside it has one squared axis offset above (exact_len / spm)^2 (1 + 1e-9), so its delay
  // is >= exact_len.  Enumeration order within the box is the reference's order restricted to
  // it (ix -> iy -> iz ascending), so the wanted bins receive the same terms in the same order.
  __shared__ int s_box[6];
  if (tid < 6) s_box[tid] = (tid & 1) ? -1 : W;
  __syncthreads();
  // squared distance beyond which an image's delay is >= exact_len for certain
  const double rr = static_cast<double>(exact_len) / spm;
  const double d2max = exact_len > 0 ? rr * rr * (1.0 + 1e-9) : 1.0e300;
  if (exact_len > 0) {
    for (int idx = tid; idx < 3 * W; idx += NT) {
      const int axis = idx / W, n = idx - axis * W;
      if (ax[idx] <= d2max) {
        atomicMin(&s_box[2 * axis], n);
        atomicMax(&s_box[2 * axis + 1], n);
      }
    }
  } else if (tid < 3) {
    s_box[2 * tid] = 0;
    s_box[2 * tid + 1] = W - 1;
  }
  __syncthreads();
  const int x0 = s_box[0], y0 = s_box[2], z0 = s_box[4];
  const int bx = s_box[1] - x0 + 1, by = s_box[3] - y0 + 1, bz = s_box[5] - z0 + 1;
  if (bx <= 0 || by <= 0 || bz <= 0) {  // no image can land in the range (cannot happen: the direct path does)
    double* out0 = a.rir + pm.rir_off + lo;
    for (int l = tid; l < len; l += NT) out0[l] = 0.0;
    return;
  }

  const long long V = static_cast<long long>(bx) * by * bz;
  // image index i = (jx by + jy) bz + jz within the box, advanced incrementally by NT per
  // image slot; (ix, iy, iz) = (x0 + jx, y0 + jy, z0 + jz)
  int iz = tid % bz, iy, ix;
  {
    const int q = tid / bz;
    iy = q % by;
    ix = q / by;
  }
  const int step_z = NT % bz, step_q = NT / bz;
  const int step_y = step_q % by, step_x = step_q / by;
  const unsigned axx_s = ax_s + 8u * static_cast<unsigned>(x0);
  const unsigned axy_s = ax_s + 8u * static_cast<unsigned>(W + y0);
  const unsigned axz_s = ax_s + 8u * static_cast<unsigned>(2 * W + z0);
  const int kx = K - x0, ky = K - y0, kz = K - z0;
  const unsigned lt = lanemask_lt();
  unsigned long long max_d = 0;
  int geo = 0;
  for (long long base = 0; base < V; base += CH) {
    int rel_bin[IPT];
    double amp[IPT];
#pragma unroll
    for (int h = 0; h < IPT; ++h) {  // image base + h NT + tid
      const long long i = base + h * NT + tid;
      rel_bin[h] = -1;
      amp[h] = 0.0;
      if (i < V) {
        // norm: sqrt((x*x + y*y) + z*z), room_model.hpp:43
        const double d2 = __dadd_rn(__dadd_rn(lds_f64(axx_s + 8u * ix), lds_f64(axy_s + 8u * iy)),
                                    lds_f64(axz_s + 8u * iz));
        if (d2 > d2max) {  // beyond the exact range (truncated synthesis): no sqrt, no entry
          // (index advance below)
        } else {
        const double d = __dsqrt_rn(d2);
        if (d <= 0.0) geo = 1;                     // :157-158
        const double dl = ceil(__dmul_rn(d, spm));  // :159-160
        const unsigned long long D = static_cast<unsigned long long>(dl);
        max_d = D > max_d ? D : max_d;
        const long long rel = static_cast<long long>(D) - lo;
        if (rel >= 0 && rel < len) {
          const int g = abs(ix - kx) + abs(iy - ky) + abs(iz - kz);
          amp[h] = __ddiv_rn(lds_f64(rg_s + 8u * g), d);  // :161-162 pow(r, g) / d
          rel_bin[h] = static_cast<int>(rel);
        }
        }
      }
      // advance (ix, iy, iz) by NT images
      iz += step_z;
      int cy = step_y;
      if (iz >= bz) { iz -= bz; ++cy; }
      iy += cy;
      int cx = step_x;
      while (iy >= by) { iy -= by; ++cx; }
      ix += cx;
    }
#ifndef RSG_X_NOSCATTER
    // ---- publish: per image slot, lane masks per owner from OB + 1 ballots ----
    // owner of a bin: any function of the bin keeps each bin's entries in order; mixing
    // in bin/16 spreads one owner's FP64 bins over all smem banks (bin mod NW alone
    // puts them all in one bank pair)
    int owner[IPT];
    unsigned mine[IPT];
#pragma unroll
    for (int h = 0; h < IPT; ++h) {
      owner[h] = (rel_bin[h] ^ (rel_bin[h] >> 4)) & (NW - 1);
      mine[h] = __ballot_sync(0xffffffffu, rel_bin[h] >= 0);  // lanes sharing my owner
      unsigned row = mine[h];                                   // lane o < NW: lanes owned by o
#pragma unroll
      for (int k = 0; k < OB; ++k) {
        const unsigned bk = __ballot_sync(0xffffffffu, (owner[h] >> k) & 1);
        mine[h] &= ((owner[h] >> k) & 1) ? bk : ~bk;
        row &= ((lane >> k) & 1) ? bk : ~bk;
      }
      if (lane < NW) cnt8[lane * RS + h * NW + warp] = static_cast<unsigned char>(__popc(row));
    }
    __syncthreads();
    // ---- stable counting sort into owner-major lists (order: slot, warp, lane) ----
    // lane o < NW: entries of owner o in virtual warps before slot h's (`before[h]`) and
    // in all (`total`): byte sums of the owner's count row by dp4a
    unsigned ub[IPT], utotal = 0u;
#pragma unroll
    for (int h = 0; h < IPT; ++h) ub[h] = 0u;
    if (lane < NW) {
      const unsigned* rowp = reinterpret_cast<const unsigned*>(cnt8 + lane * RS);
#pragma unroll
      for (int q4 = 0; q4 < NQ; q4 += 4) {  // 16-byte loads (a strided 4-byte loop is conflicted)
        unsigned rv[4];
        if (q4 + 4 <= NQ) {
          const uint4 r4 = *reinterpret_cast<const uint4*>(rowp + q4);
          rv[0] = r4.x; rv[1] = r4.y; rv[2] = r4.z; rv[3] = r4.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) rv[u] = q4 + u < NQ ? rowp[q4 + u] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q4 + u;
          if (q >= NQ) break;
          const unsigned wq = 4 * q + 4 <= NV ? rv[u] : (rv[u] & ((1u << (8 * (NV - 4 * q))) - 1u));
          utotal = __dp4a(wq, 0x01010101u, utotal);
#pragma unroll
          for (int h = 0; h < IPT; ++h) {
            const int nb = h * NW + warp - 4 * q;  // bytes of word q before this slot's virtual warp
            const unsigned m = nb <= 0 ? 0u : nb >= 4 ? 0xffffffffu : (1u << (8 * nb)) - 1u;
            ub[h] = __dp4a(wq & m, 0x01010101u, ub[h]);
          }
        }
      }
    }
    const int total = static_cast<int>(utotal);
    int incl = total;  // inclusive scan of the owner totals over lanes 0..NW-1
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int obase = incl - total;  // list start of owner `lane`
#pragma unroll
    for (int h = 0; h < IPT; ++h) {
      const int seg = __shfl_sync(0xffffffffu, obase + static_cast<int>(ub[h]), rel_bin[h] >= 0 ? owner[h] : 0);
      if (rel_bin[h] >= 0) {
        const int pos = seg + __popc(mine[h] & lt);
        ent_d[pos] = rel_bin[h];
        ent_a[pos] = amp[h];
      }
    }
    const int my_base = __shfl_sync(0xffffffffu, obase, warp);
    const int my_total = __shfl_sync(0xffffffffu, total, warp);
    __syncthreads();
    // ---- owner `warp` folds its list: round r applies the r-th entry of each
    // equal-delay group (lane order = enumeration order) ----
    for (int r0 = 0; r0 < my_total; r0 += 32) {
      const int l = r0 + lane;
      const bool valid = l < my_total;
      const int bn = valid ? ent_d[my_base + l] : -1 - lane;  // distinct dummy keys for idle lanes
      const double av = valid ? ent_a[my_base + l] : 0.0;
      // Fast path: every lane claims its bin in a byte tag; if each valid lane reads back its
      // own id the round's bins are distinct (the bins of one owner are touched by this warp
      // only), so all entries apply at once.  A shared bin leaves some lane with another id:
      // then match_any orders the round as below.  (MATCH.ANY's latency was the fold's
      // largest stall.)
      if constexpr (FOLD == 2) {
        // Ordered claims: every pending lane min-reduces its lane id into its bin's claim
        // word (a hash of the bin; the owner's bins map 1:1 to bin >> 4); the lowest lane of
        // each word wins, applies its entry and resets the word, the others retry.  Each bin
        // therefore sees its entries in lane order; bins sharing a word only serialize.
        // A round of distinct bins takes one pass; no match_any.
        const unsigned cw = tag_s + 4u * static_cast<unsigned>(warp * HT + (((bn >> 4) ^ (bn >> 12)) & (HT - 1)));
        const unsigned ba = bins_s + 8u * static_cast<unsigned>(bn);
        bool pending = valid;
        for (;;) {
          if (pending) asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(cw), "r"(lane) : "memory");
          __syncwarp();
          unsigned w = 0xffffffffu;
          if (pending) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(cw) : "memory");
          const bool win = pending && w == static_cast<unsigned>(lane);
          __syncwarp();  // every claim word read before a winner resets it
          if (win) {
            shared_add_rn(ba, av);
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(cw), "r"(0xffffffffu) : "memory");
          }
          pending = pending && !win;
          if (!__any_sync(0xffffffffu, pending)) break;
          __syncwarp();
        }
        __syncwarp();
        continue;
      }
      const unsigned grp = __match_any_sync(0xffffffffu, bn);
      const int rank = __popc(grp & lt);
      const int rounds = __reduce_max_sync(0xffffffffu, valid ? __popc(grp) : 0);
      // bins[bn] += av through a 32-bit shared address (a generic pointer re-derives the
      // CTA's shared window every iteration: S2UR on the critical path)
      const unsigned ba = bins_s + 8u * static_cast<unsigned>(bn);
      if (valid && rank == 0) shared_add_rn(ba, av);
      for (int r = 1; r < rounds; ++r) {
        __syncwarp();
        if (valid && rank == r) shared_add_rn(ba, av);
      }
      __syncwarp();
    }
#endif
  }
  __syncthreads();
  double* out = a.rir + pm.rir_off + lo;
  for (int l = tid; l < len; l += NT) out[l] = bins[l];
  // max delay / geometry flag over the CTA
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, max_d, o);
    max_d = other > max_d ? other : max_d;
    geo |= __shfl_xor_sync(0xffffffffu, geo, o);
  }
  if (lane == 0 && exact_len <= 0) {  // (the bound pass wrote both for a truncated synthesis)
    atomicMax(&a.out[it.pair].max_delay, max_d);
    if (geo) atomicOr(&a.out[it.pair].flags, 1);
  }
}

size_t synth_smem_bytes(int max_order, int slice, int nt, int ipt, int fold, int ht) {
  const int W = 2 * max_order + 1, nw = nt / 32, ch = ipt * nt, nv = ipt * nw;
  const int u16 = (4 * ((nv + 3) / 4) + 15) / 16;  // count-row stride (kernel's RS)
  const int rs = 16 * (u16 % 2 == 0 ? u16 + 1 : u16);
  return sizeof(double) * (static_cast<size_t>(slice) + 3 * W + 3 * max_order + 1 + ch) + sizeof(int) * ch +
         ((static_cast<size_t>(nw) * rs + 15) & ~size_t(15)) + (fold == 2 ? 4 * static_cast<size_t>(nw) * ht : 0) + 16 + 16;
}

cudaError_t launch_synth(const SynthArgs& a, int n_items, int max_order, int slice, cudaStream_t s,
                         int nt) {
  if (n_items == 0) return cudaSuccess;
  // 4 images per thread unless that would drop a 512-thread CTA below 2 per SM (when not
  // even 2 images per thread keep 2 per SM, 4)
  static const int fold_big = [] {
    const char* e = getenv("RSG_K1_FOLD");
    return e ? atoi(e) : 2;
  }();
  static const int fold_sliced = [] {
    const char* e = getenv("RSG_K1_FOLD_S");
    return e ? atoi(e) : 2;
  }();
  const bool big = nt == 512 && slice > kSynthSlice;  // the one-CTA class
  const int fold = big ? fold_big : fold_sliced;
  // claim words per warp: 64 keeps two sliced 512-thread CTAs per SM
  const int ht = nt == 512 && !big ? 64 : 256;
  const bool two4 = 2 * synth_smem_bytes(max_order, slice, nt, 4, fold, ht) <= 227 * 1024;
  const bool two2 = 2 * synth_smem_bytes(max_order, slice, nt, 2, fold, ht) <= 227 * 1024;
  const bool one4 = synth_smem_bytes(max_order, slice, nt, 4, fold, ht) <= 227 * 1024;
  const int ipt = (nt == 512 && ((!two4 && two2) || !one4)) ? 2 : 4;
  const size_t smem = synth_smem_bytes(max_order, slice, nt, ipt, fold, ht);
  auto go = [&](auto kern, int threads) -> cudaError_t {
    cudaError_t e = ensure_dynamic_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<n_items, threads, smem, s>>>(a, slice);
    return cudaGetLastError();
  };
  if (nt == 128) return go(rir_synth_kernel<128, 4, 0>, 128);  // claims measured 6% slower here
  if (fold == 2 && big) return ipt == 4 ? go(rir_synth_kernel<512, 4, 2>, 512) : go(rir_synth_kernel<512, 2, 2>, 512);
  if (fold == 2) return ipt == 4 ? go(rir_synth_kernel<512, 4, 2, 64>, 512) : go(rir_synth_kernel<512, 2, 2, 64>, 512);
  return ipt == 4 ? go(rir_synth_kernel<512, 4, 0>, 512) : go(rir_synth_kernel<512, 2, 0>, 512);
}

// ============================================================================
// K2: -eta dB tail cut.  One CTA per pair: exact FP64 max of h^2 and the last
// index with h^2 >= p_th (max reductions are order independent, so the result
// equals the reference's sequential scans bit for bit).
// ============================================================================
__global__ void __launch_bounds__(256) rir_cut_kernel(CutArgs a) {
  const int p = blockIdx.x;
  const PairMeta& pm = a.pair[p];
  const UttMeta& um = a.utt[pm.utt];
  PairRir& r = a.out[p];
  __shared__ double red_d[8];
  __shared__ long long red_i[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long len = static_cast<long long>(r.max_delay) + 1;
  if (um.max_taps > 0 && um.max_taps < len) len = um.max_taps;
  if (len > pm.rir_cap) {  // cannot happen: the host computes the same maximum exactly
    if (threadIdx.x == 0) r.flags |= 8;
    len = pm.rir_cap;
  }
  if (r.flags & 1) len = 0;
  const double* h = a.rir + pm.rir_off;
  if (a.eta_factor <= 0.0 || len == 0) {
    if (tid == 0) {
      r.len = len;
      r.keep = len;
      r.cutoff = -1;
    }
    return;
  }
  // bins at and beyond exact_len were not synthesized: all provably below the threshold
  const long long scan = (r.exact_len > 0 && r.exact_len < len) ? r.exact_len : len;
  double mx = 0.0;
  for (long long n = tid; n < scan; n += 256) mx = fmax(mx, __dmul_rn(h[n], h[n]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red_d[warp] = mx;
  __syncthreads();
  mx = red_d[0];
  for (int w = 1; w < 8; ++w) mx = fmax(mx, red_d[w]);
  const double th = __dmul_rn(mx, a.eta_factor);  // room_model.hpp:184
  long long last = -1;
  for (long long n = tid; n < scan; n += 256)
    if (__dmul_rn(h[n], h[n]) >= th) last = n;  // room_model.hpp:193-195
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(0xffffffffu, last, o);
    last = other > last ? other : last;
  }
  if (lane == 0) red_i[warp] = last;
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < 8; ++w) last = red_i[w] > last ? red_i[w] : last;
    const long long nc = last < 0 ? 0 : last;
    r.len = len;
    r.threshold = th;
    r.cutoff = nc;
    r.keep = nc + 2 < len ? nc + 2 : len;  // room_model.hpp:209
    if (mx == 0.0) r.flags |= 2;
  }
}

cudaError_t launch_cut(const CutArgs& a, int n_pairs, cudaStream_t s) {
  if (n_pairs == 0) return cudaSuccess;
  rir_cut_kernel<<<n_pairs, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// FFT sizing helpers
// ============================================================================
__host__ __device__ constexpr int e_of(int log2m) {  // == Plan<1 << log2m>::E
  return (1 << log2m) < RSG_E_SMALL ? (1 << log2m)
                                    : (log2m >= 13 ? 32 : ((1 << log2m) <= 512 ? RSG_E_SMALL : RSG_E));
}
// smem float2 slots of one transform (== Plan<1 << log2m>::PADDED)
__host__ __device__ constexpr int padded_of(int log2m) {
  return (e_of(log2m) == 8 && (log2m + 2) / 3 >= 3) ? (1 << log2m) + (1 << log2m) / 8
                                                    : (1 << log2m) + (1 << log2m) / 16;
}
__host__ __device__ constexpr int cta_threads_of(int log2m) {
  // T = M / E threads per transform (E = 16, or 32 for M >= 8192); >= 256 per CTA.
  return (1 << log2m) / e_of(log2m) > 256 ? (1 << log2m) / e_of(log2m) : 256;
}
int cta_threads(int log2m) { return cta_threads_of(log2m); }

static_assert(padded_of(3) == Plan<8>::PADDED && padded_of(6) == Plan<64>::PADDED &&
                  padded_of(7) == Plan<128>::PADDED && padded_of(9) == Plan<512>::PADDED &&
                  padded_of(10) == Plan<1024>::PADDED && padded_of(14) == Plan<16384>::PADDED,
              "host smem sizing matches the device plan");

template <int M>
__host__ __device__ constexpr int groups_of() {
  return cta_threads_of(Plan<M>::LOG) / Plan<M>::T;
}

size_t ola_smem_bytes(int log2m) {
  const int M = 1 << log2m;
  const int E = e_of(log2m);
  const int T = M / E;
  const int G = cta_threads_of(log2m) / T;
  return static_cast<size_t>(G) * padded_of(log2m) * sizeof(float2);
}

template <int M>
static int tw_total_t() { return Plan<M>::TW_TOTAL; }

int tw_total(int log2m) {
  switch (log2m) {
#define RSG_CASE(L) case L: return Plan<(1 << L)>::TW_TOTAL;
    RSG_CASE(0) RSG_CASE(1) RSG_CASE(2) RSG_CASE(3) RSG_CASE(4) RSG_CASE(5) RSG_CASE(6)
    RSG_CASE(7) RSG_CASE(8) RSG_CASE(9) RSG_CASE(10) RSG_CASE(11) RSG_CASE(12) RSG_CASE(13)
    RSG_CASE(14)
#undef RSG_CASE
  }
  return 0;
}

template <int M>
static void fill_twiddles_t(float2* h) {
  using PL = Plan<M>;
  const double pi = 3.14159265358979323846;
  for (int p = 1; p < PL::NP; ++p) {
    const int R = PL::radix(p), NS = PL::ns(p);
    const double span = static_cast<double>(NS) * R;
    for (int k = 0; k < NS; ++k) {  // base w_k; powers are generated in registers
      const double ang = -2.0 * pi * static_cast<double>(k) / span;
      h[PL::tw_off(p) + k] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
  }
  // pairing table W^k = exp(-2 pi i k / N), N = 2M, k in [0, M/2]
  for (int k = 0; k <= M / 2; ++k) {
    const double ang = -2.0 * pi * static_cast<double>(k) / (2.0 * M);
    h[PL::TW_PASS + k] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
  }
}

void fill_twiddles(int log2m, float2* host) {
  switch (log2m) {
#define RSG_CASE(L) case L: fill_twiddles_t<(1 << L)>(host); break;
    RSG_CASE(0) RSG_CASE(1) RSG_CASE(2) RSG_CASE(3) RSG_CASE(4) RSG_CASE(5) RSG_CASE(6)
    RSG_CASE(7) RSG_CASE(8) RSG_CASE(9) RSG_CASE(10) RSG_CASE(11) RSG_CASE(12) RSG_CASE(13)
    RSG_CASE(14)
#undef RSG_CASE
  }
}

// W^k for k in [0, M] from the pairing table (k <= M/2 stored; W^k = -conj(W^(M-k)) above).
template <int M>
__device__ __forceinline__ float2 pair_twiddle(const float2* W, int k) {
  if (k <= M / 2) return __ldg(W + k);
  const float2 w = __ldg(W + (M - k));
  return make_float2(-w.x, w.y);
}

// ============================================================================
// K3: RIR spectrum.  G[k] = H[k] / (4M) for k = 0..M, H the real FFT of the
// truncated RIR zero-padded to N (convolution.hpp:238-239; untangle as
// fft.hpp:152-161).  The 1/(4M) folds the inverse's 1/M and the two 1/2's of
// the untangle/repack into the filter, so K4 needs no scaling pass.
// ============================================================================
template <int M>
__global__ void __launch_bounds__(cta_threads_of(Plan<M>::LOG)) rir_spectrum_kernel(SpecArgs a) {
  using PL = Plan<M>;
  extern __shared__ __align__(16) float2 smem[];
  constexpr int G = groups_of<M>();
  const int g = threadIdx.x / PL::T, t = threadIdx.x % PL::T;
  const int item = blockIdx.x * G + g;
  const bool active = item < a.count;
  float2* s = smem + g * PL::PADDED;
  const int p = active ? a.list[item] : 0;
  const PairPlan& pl = a.plan[p];
  const double* h = a.rir + a.pair[p].rir_off;
  const long long nh = pl.nh;
  first_pass<M>(s, t, active, h, static_cast<int>(nh));
  forward_rest<M>(s, t, a.tw, active);
  if (active) {
    const float2* W = a.tw + PL::TW_PASS;
    const float scale = 1.0f / (8.0f * M);
    float2* out = a.spec + pl.spec_off;
    auto untangle = [&](int k) {  // 2 H(k) sqrt-free: S + W^k D of the packed transform
      const float2 za = s[PAD(k & (M - 1))];
      const float2 zb = c_conj(s[PAD((M - k) & (M - 1))]);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      return c_add(S, c_mul(pair_twiddle<M>(W, k), D));
    };
    if (a.perm.on) {
      // H / N over all N bins (H(N - k) = conj H(k)) in ola_ipc_kernel's order, walked in
      // OUTPUT order so the stores coalesce (bin order scatters 8-byte stores over 128-byte
      // lines: K3 was store-bound, 95% L1 throughput)
      for (int idx = t; idx < 2 * M; idx += PL::T) {
        const int k = a.perm.bin(idx);
        const float2 g = c_scale(untangle(k <= M ? k : 2 * M - k), 2.0f * scale);
        out[idx] = k <= M ? g : c_conj(g);
      }
    } else {
      for (int k = t; k <= M; k += PL::T) out[k] = c_scale(untangle(k), scale);
    }
  }
}

// ============================================================================
// K4: the OLA filter.  A CTA holds G independent groups of T threads; each
// group takes one work item (a run of OLA blocks of one pair) and, per block,
// runs the forward Stockham FFT of the packed block (loaded straight from the
// FP32 source signal), the spectral multiply with the pair's G, and the
// inverse FFT, whose last pass writes the block's N outputs from registers
// into the pair's output: plain stores where the block is the first writer,
// read-add-write (earlier blocks first, as convolution.hpp:251-252) on the
// N_h - 1 overlap.  Groups synchronise with their own barrier (__syncwarp or
// a named bar.sync), never with the whole CTA, and every sample's FP64 y^2 is
// accumulated once, when it is final.  Reference: convolve_ola,
// convolution.hpp:219-255; mean_power, audio_buffer.hpp:66-75.
// ============================================================================
template <int T>
struct GroupBar {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (T == 1) {
      // one thread per transform: no inter-thread exchange
    } else if constexpr (T <= 32) {
      __syncwarp();  // groups of a warp run convergent (uniform trip count)
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
    }
  }
};


// ---- small/medium transforms (M <= 4096): everything a block needs is in
// shared memory.  Per group: the transform buffer, the pair's filter spectrum
// G (staged once per work item), the N_h - 1 sample overlap carried from the
// previous block (so the output is written once, final, never re-read), and
// the next block's input, prefetched with cp.async while the current block is
// transformed.

constexpr int kSmallMaxLog2M = 12;

#ifndef RSG_K4_WARPS
#define RSG_K4_WARPS 8  // target resident warps / SM for the radix-16 K4 sizes
#endif
// K4 (small M) CTA: a single group when T >= 64, else 64 threads of groups.
__host__ __device__ constexpr int k4_cta_of(int log2m) {
  return (1 << log2m) / e_of(log2m) > 64 ? (1 << log2m) / e_of(log2m) : 64;
}
// resident-warp target per SM: 16 for the radix-8 sizes, 8 for radix-16 (measured)
__host__ __device__ constexpr int k4_warps_of(int log2m) { return (1 << log2m) <= 512 ? 16 : RSG_K4_WARPS; }
__host__ __device__ constexpr int k4_minb_of(int log2m) {
  return k4_warps_of(log2m) / (k4_cta_of(log2m) / 32) > 0 ? k4_warps_of(log2m) / (k4_cta_of(log2m) / 32) : 1;
}

int ola_groups(int log2m) {
  const int M = 1 << log2m;
  const int E = e_of(log2m);
  const int cta = log2m <= kSmallMaxLog2M ? k4_cta_of(log2m) : cta_threads_of(log2m);
  return cta / (M / E);
}

// K4 work-item groups resident per SM (for sizing work items).
int ola_resident_groups(int log2m) {
  if (log2m > kSmallMaxLog2M) return ola_groups(log2m);
  const int cta = k4_cta_of(log2m);
  return k4_minb_of(log2m) * ola_groups(log2m) > 0 ? k4_minb_of(log2m) * ola_groups(log2m) : 1;
  (void)cta;
}

template <int M>
struct SmallLayout {  // float2 offsets inside one group's region, all even (16-byte aligned)
  static constexpr int ev(int v) { return (v + 1) & ~1; }
  static constexpr int FFT = 0;
  static constexpr int GS = ev(Plan<M>::PADDED);
  static constexpr int CARRY = ev(GS + M + 1);     // 2 x N floats (double-buffered)
  static constexpr int STAGE = ev(CARRY + 2 * M);  // 2 x (N + 8) floats: two blocks in flight
  static constexpr int STAGE_STRIDE = ev(M + 4);   // float2 per stage buffer (even: 16-B aligned)
  static constexpr int MBAR = ev(STAGE + 2 * STAGE_STRIDE);  // two 8-byte mbarriers
  static constexpr int TOTAL = ev(MBAR + 2);
  static_assert(STAGE % 2 == 0 && STAGE_STRIDE % 2 == 0 && TOTAL % 2 == 0, "16-byte alignment of the bulk-copy windows");
};


template <int M>
__global__ void __launch_bounds__(k4_cta_of(Plan<M>::LOG), k4_minb_of(Plan<M>::LOG))
ola_small_kernel(OlaArgs a) {
  using PL = Plan<M>;
  using LY = SmallLayout<M>;
  extern __shared__ __align__(16) float2 smem[];
  constexpr int T = PL::T;
  constexpr int CTA = k4_cta_of(PL::LOG);
  constexpr int G = CTA / T;
  constexpr int N = 2 * M;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int item = blockIdx.x * G + g;
  const bool has = item < a.count;
  const OlaItem it = a.items[has ? item : 0];
  const PairPlan& pl = a.plan[it.pair];
  const PairMeta& pm = a.pair[it.pair];
  const float* __restrict__ x = a.signals + pm.sig_off;
  const int nx = static_cast<int>(pm.nx);
  float* __restrict__ y = a.y + pl.y_off;
  const int L = static_cast<int>(pl.L);
  const int B = static_cast<int>(pl.B);
  const int out_len = static_cast<int>(pl.out_len);
  constexpr int TWN = (PL::TW_TOTAL + 1) & ~1;  // per-CTA twiddle tables (pass bases + W)
  float2* tws = smem;
  float2* base = smem + TWN + g * LY::TOTAL;
  float2* s = base + LY::FFT;
  float2* gs = base + LY::GS;
  float* carry0 = reinterpret_cast<float*>(base + LY::CARRY);  // 2 x N floats, zero beyond N_h - 1
  float* stage0 = reinterpret_cast<float*>(base + LY::STAGE);  // 2 buffers of N + 8 floats
  const GroupBar<T> bar{1 + g};
  int trips = has ? it.b_end - it.b_begin : 0;
  if constexpr (T < 32) trips = __reduce_max_sync(0xffffffffu, trips);
  const int own_lo = it.b_own * L;
  const int own_hi = it.b_end == B ? out_len : it.b_end * L;
  // block b's samples -> stage[0, take) (4-byte cp.async: any alignment); fixed
  // trip count N/T = 2E, predicated
  unsigned long long* mbar0 = reinterpret_cast<unsigned long long*>(base + LY::MBAR);
  // Block b's samples land in stage(b)[d, d + take) with d = (address mod 16)/4:
  // one 1-D TMA bulk copy (cp.async.bulk, a 16-byte aligned window) issued by
  // one thread two blocks ahead (double-buffered), or — near the end of the
  // signal, where the window would read past it — per-thread 4-byte cp.async
  // at consumption time.
  auto window = [&](int b, int& d, int& take, bool& bulk) {
    const int st = b * L;
    take = nx - st < L ? nx - st : L;
    d = static_cast<int>((reinterpret_cast<uintptr_t>(x + st) & 15u) >> 2);
    bulk = st + take + 4 <= nx;
  };
  auto stage_of = [&](int k) { return stage0 + (k & 1) * (2 * LY::STAGE_STRIDE); };
  auto prefetch = [&](int k) {  // k: index of the block within this item
    const int b = it.b_begin + k;
    int d, take;
    bool bulk;
    window(b, d, take, bulk);
    if (bulk && t == 0)
      bulk_g2s(stage_of(k), x + b * L - d, static_cast<unsigned>(((d + take) * 4 + 15) & ~15), mbar0 + (k & 1));
  };
  for (int i = threadIdx.x; i < PL::TW_TOTAL; i += CTA) cp_async8(tws + i, a.tw + i);
  const float2* W = tws + PL::TW_PASS;
  if (has) {
    const float2* Gsrc = a.spec + pl.spec_off;
    for (int k = t; k <= M; k += T) cp_async8(gs + k, Gsrc + k);
    for (int i = t; i < 2 * N; i += T) carry0[i] = 0.f;
    if (t == 0) {
      mbar_init(mbar0, 1);
      mbar_init(mbar0 + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  cp_async_wait_all();
  __syncthreads();  // per-CTA twiddles, G, carry and barriers in place (all threads)
  double pw = 0.0;  // this lane's Σ y² of the current power segment
  // Up to M = RSG_K4_DIRECT_MAX pass 0 reads the block straight from the signal
  // (L2-prefetched two blocks ahead by one thread) instead of the TMA stage: measured
  // 2-27% faster at M <= 256, 5% slower at M = 512
#ifndef RSG_K4_DIRECT_MAX
#define RSG_K4_DIRECT_MAX 256
#endif
  constexpr bool kDirect = M <= RSG_K4_DIRECT_MAX;
  auto prefetch_l2_block = [&](int b) {
    if (b < it.b_end && t == 0) {
      const long long st = static_cast<long long>(b) * L;
      const long long n = nx - st < L ? nx - st : L;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(x + st) & ~uintptr_t(15);
      const uintptr_t a1 = (reinterpret_cast<uintptr_t>(x + st + n) + 15) & ~uintptr_t(15);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(static_cast<unsigned>(a1 - a0)) : "memory");
    }
  };
#ifndef RSG_X_NOLOAD
  if (has) {
    if constexpr (kDirect) {
      prefetch_l2_block(it.b_begin);
      prefetch_l2_block(it.b_begin + 1);
    } else {
      prefetch(0);
      if (it.b_begin + 1 < it.b_end) prefetch(1);
    }
  }
#endif
#pragma unroll 1
  for (int k = 0; k < trips; ++k) {
    const int b = it.b_begin + k;
    const bool active = has && b < it.b_end;
    const int start = b * L;
    int d = 0, take = 0;
    bool bulk = false;
    float* stage = stage_of(k);
    if (kDirect) {
      take = active ? (nx - start < L ? nx - start : L) : 0;
    } else if (active) {
      window(b, d, take, bulk);
#ifndef RSG_X_NOLOAD
      if (bulk) {
        mbar_wait(mbar0 + (k & 1), (k >> 1) & 1);
      } else {
        const float* src = x + start;
#pragma unroll
        for (int m = 0; m < N / T; ++m) {
          const int i = t + m * T;
          if (i < take) cp_async4(stage + d + i, src + i);
        }
        cp_async_wait_all();
      }
#endif
    }
    bar();
    first_pass<M, float, GroupBar<T>, false>(s, t, active, kDirect ? x + start : stage + d, take, bar);
#if !defined(RSG_NO_PREFETCH) && !defined(RSG_X_NOLOAD)
    if constexpr (kDirect) {
      if (active) prefetch_l2_block(b + 2);
    } else {
      if (active && b + 2 < it.b_end) prefetch(k + 2);  // lands while blocks b, b+1 are transformed
    }
#endif
#ifndef RSG_NO_FUSED_PAIR
    if constexpr (M == 512) {  // last forward pass + pairing + first inverse pass in registers
      stockham_pass<M, 1, false, GroupBar<T>, true>(s, t, tws, active, bar);
      fused_pair_512(s, t, tws, gs, W, active, bar);
      stockham_pass<M, 1, true, GroupBar<T>, true, true>(s, t, tws, active, bar);
    } else if constexpr (M == 256) {
      stockham_pass<M, 1, false, GroupBar<T>, true>(s, t, tws, active, bar);
      fused_pair_256(s, t, tws, gs, W, active, bar);
      stockham_pass<M, 1, true, GroupBar<T>, true>(s, t, tws, active, bar);
    } else
#endif
    {
      forward_rest<M, 1, GroupBar<T>, true>(s, t, tws, active, bar);
      spectral_multiply<M, GroupBar<T>, true, true>(s, t, gs, W, active, bar);
      inverse_but_last<M, 0, GroupBar<T>, true>(s, t, tws, active, bar);
    }
    // emit: e < L -> final output (carry + v), e >= L -> carry for block b+1
    float* yb = y + start;
    const int lo = own_lo - start;
    const int hi = own_hi - start;
    const bool last = b == B - 1;
    // carry of this block (read) and of the next (written): double-buffered, so
    // the emit needs no barrier and nothing stays live across one
    const float* cin = carry0 + (k & 1) * N;
    float* carry = carry0 + ((k + 1) & 1) * N;
    // this block's power partials (FP32, <= 2E terms over four independent chains so the
    // FMAs do not serialise), folded into FP64 below in a fixed order
    float pb[4] = {0.f, 0.f, 0.f, 0.f};
    auto emit_fn = [&](int q, int r, int c, float2 v) {
      const int e0 = 2 * c;
      const float2 ci = *reinterpret_cast<const float2*>(cin + e0);
      const float2 acc = make_float2(ci.x + v.x, ci.y + v.y);
#ifndef RSG_EMIT_NOFAST
      if constexpr (T >= 32 && PL::E == 8) {
        // A warp's elements of one r are 64 consecutive samples [w0, w0 + 64): classify them
        // once, warp-uniformly (the per-element tests below were a quarter of the kernel's
        // instructions: branches, predicates, divergence bookkeeping)
        const int w0 = 2 * (c & ~31);
        if (w0 >= lo && w0 + 64 <= hi && (w0 + 64 <= L || last)) {  // all final and owned
#ifndef RSG_X_NOSTORE
          yb[e0] = acc.x;
          yb[e0 + 1] = acc.y;
#endif
          pb[2 * (r & 1)] = fmaf(acc.x, acc.x, pb[2 * (r & 1)]);
          pb[2 * (r & 1) + 1] = fmaf(acc.y, acc.y, pb[2 * (r & 1) + 1]);
          return;
        }
        if (w0 >= L && !last) {  // all carried into the next block
          carry[e0 - L] = acc.x;
          carry[e0 + 1 - L] = acc.y;
          return;
        }
      }
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = e0 + h;
        const float val = h ? acc.y : acc.x;
        if (e < L || last) {  // final sample
          if (e >= lo && e < hi) {
#ifndef RSG_X_NOSTORE
            yb[e] = val;
#endif
#ifndef RSG_X_NOPOWER
            pb[2 * (r & 1) + h] = fmaf(val, val, pb[2 * (r & 1) + h]);
#endif
          }
        } else {
          carry[e - L] = val;  // partial sum for the next block
        }
      }
    };
    stockham_emit_pass<M, GroupBar<T>, decltype(emit_fn), true, false>(s, t, tws, active, bar, emit_fn);
    // power: per-lane FP64 sum over the segment, stored at its end (power.cuh)
    pw += static_cast<double>((pb[0] + pb[1]) + (pb[2] + pb[3]));
    const bool seg_end = active && closes_segment(b, it.b_end);
    if (__any_sync(0xffffffffu, seg_end)) {
      store_segment_power<T>(a.part + pl.part0 + static_cast<long long>(b / kPowerSeg) * parts_per_block_of(T), pw,
                             t, seg_end && b >= it.b_own);
      if (seg_end) pw = 0.0;
    }
    // (N_h - 1 > L, three or more overlapping blocks, needs no extra step: the
    // old carry at e in [L, N_h - 1) comes from the other buffer.)
  }
}

// ============================================================================
// Seam kernels: natural-order real FFTs (RadixTwoRealFft::forward/inverse).
// ============================================================================
template <int M>
__global__ void __launch_bounds__(cta_threads_of(Plan<M>::LOG))
rfft_forward_kernel(const float* in, float2* out, int count, const float2* tw) {
  using PL = Plan<M>;
  extern __shared__ __align__(16) float2 smem[];
  constexpr int G = groups_of<M>();
  const int g = threadIdx.x / PL::T, t = threadIdx.x % PL::T;
  const int item = blockIdx.x * G + g;
  const bool active = item < count;
  float2* s = smem + g * PL::PADDED;
  const float* x = in + static_cast<long long>(active ? item : 0) * (2 * M);
  first_pass<M>(s, t, active, x, 2 * M);
  forward_rest<M>(s, t, tw, active);
  if (active) {
    const float2* W = tw + PL::TW_PASS;
    float2* o = out + static_cast<long long>(item) * (M + 1);
    for (int k = t; k <= M; k += PL::T) {
      const float2 za = s[PAD(k & (M - 1))];
      const float2 zb = c_conj(s[PAD((M - k) & (M - 1))]);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      o[k] = c_scale(c_add(S, c_mul(pair_twiddle<M>(W, k), D)), 0.5f);
    }
  }
}

template <int M>
__global__ void __launch_bounds__(cta_threads_of(Plan<M>::LOG))
rfft_inverse_kernel(const float2* in, float* out, int count, const float2* tw) {
  using PL = Plan<M>;
  extern __shared__ __align__(16) float2 smem[];
  constexpr int G = groups_of<M>();
  const int g = threadIdx.x / PL::T, t = threadIdx.x % PL::T;
  const int item = blockIdx.x * G + g;
  const bool active = item < count;
  float2* s = smem + g * PL::PADDED;
  const float2* X = in + static_cast<long long>(active ? item : 0) * (M + 1);
  const float2* W = tw + PL::TW_PASS;
  if (active) {
    // fft.hpp:104-110: Z[k] = Ye + i Yo, Ye = (X[k] + conj(X[M-k]))/2,
    // Yo = (X[k] - conj(X[M-k]))/2 * conj(W^k)
    for (int k = t; k < M; k += PL::T) {
      const float2 xa = X[k], xb = c_conj(X[M - k]);
      const float2 e = c_scale(c_add(xa, xb), 0.5f);
      const float2 o = c_mulc(c_scale(c_sub(xa, xb), 0.5f), pair_twiddle<M>(W, k));
      s[PAD(k)] = make_float2(e.x - o.y, e.y + o.x);
    }
  }
  __syncthreads();
  inverse_all<M>(s, t, tw, active);
  if (active) {
    float* o = out + static_cast<long long>(item) * (2 * M);
    const float sc = 1.0f / M;
    for (int k = t; k < M; k += PL::T) {
      const float2 v = s[PAD(k)];
      o[2 * k] = v.x * sc;
      o[2 * k + 1] = v.y * sc;
    }
  }
}

// ---- dispatch over M ----------------------------------------------------------
size_t k4_smem_bytes(int log2m) {
  if (log2m > kSmallMaxLog2M) return ola_smem_bytes(log2m);
  const int M = 1 << log2m;
  auto ev = [](int v) { return (v + 1) & ~1; };
  const int per_group = ev(ev(ev(ev(ev(padded_of(log2m)) + M + 1) + 2 * M) + 2 * ev(M + 4)) + 2);  // SmallLayout<M>::TOTAL
  const int twn = (tw_total(log2m) + 1) & ~1;            // per-CTA twiddle tables
  return (static_cast<size_t>(ola_groups(log2m)) * per_group + twn) * sizeof(float2);
}

template <int M>
static cudaError_t set_attrs() {
  const int smem = static_cast<int>(ola_smem_bytes(Plan<M>::LOG));
  cudaError_t e;
  const int carve = cudaSharedmemCarveoutMaxShared;
  if constexpr (Plan<M>::LOG <= kSmallMaxLog2M) {
    if ((e = cudaFuncSetAttribute(ola_small_kernel<M>, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
    if ((e = cudaFuncSetAttribute(ola_small_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(k4_smem_bytes(Plan<M>::LOG))))) return e;
  }
  if ((e = cudaFuncSetAttribute(rir_spectrum_kernel<M>, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
  if ((e = cudaFuncSetAttribute(rir_spectrum_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(rfft_forward_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  if ((e = cudaFuncSetAttribute(rfft_inverse_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
  return cudaSuccess;
}

cudaError_t kernels_init() {
  cudaError_t e = cudaSuccess;
#define RSG_CASE(L) if (e == cudaSuccess) e = set_attrs<(1 << L)>();
  RSG_CASE(0) RSG_CASE(1) RSG_CASE(2) RSG_CASE(3) RSG_CASE(4) RSG_CASE(5) RSG_CASE(6)
  RSG_CASE(7) RSG_CASE(8) RSG_CASE(9) RSG_CASE(10) RSG_CASE(11) RSG_CASE(12) RSG_CASE(13)
  RSG_CASE(14)
#undef RSG_CASE
  return e;
}

template <int M>
static cudaError_t spectrum_t(const SpecArgs& a, cudaStream_t s) {
  constexpr int G = groups_of<M>();
  const int grid = (a.count + G - 1) / G;
  rir_spectrum_kernel<M><<<grid, cta_threads_of(Plan<M>::LOG), ola_smem_bytes(Plan<M>::LOG), s>>>(a);
  return cudaGetLastError();
}

template <int M>
static cudaError_t ola_t(const OlaArgs& a, cudaStream_t s) {
  if constexpr (Plan<M>::LOG <= kSmallMaxLog2M) {
    constexpr int CTA = k4_cta_of(Plan<M>::LOG), G = CTA / Plan<M>::T;
    ola_small_kernel<M><<<(a.count + G - 1) / G, CTA, k4_smem_bytes(Plan<M>::LOG), s>>>(a);
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;  // M > 4096: the in-place (big.cu) or four-step (large.cu) K4
}

int small_parts_per_block(int log2m) { return parts_per_block_of((1 << log2m) / e_of(log2m)); }

template <int M>
static cudaError_t rfft_t(bool inverse, const float* in_real, const float2* in_spec,
                          float* out_real, float2* out_spec, int count, const float2* tw,
                          cudaStream_t s) {
  constexpr int G = groups_of<M>();
  const int grid = (count + G - 1) / G;
  const size_t smem = ola_smem_bytes(Plan<M>::LOG);
  if (inverse)
    rfft_inverse_kernel<M><<<grid, cta_threads_of(Plan<M>::LOG), smem, s>>>(in_spec, out_real, count, tw);
  else
    rfft_forward_kernel<M><<<grid, cta_threads_of(Plan<M>::LOG), smem, s>>>(in_real, out_spec, count, tw);
  return cudaGetLastError();
}

#define RSG_DISPATCH(L, CALL)                                                             \
  switch (L) {                                                                            \
    case 0: { constexpr int M = 1; return CALL; }                                         \
    case 1: { constexpr int M = 2; return CALL; }                                         \
    case 2: { constexpr int M = 4; return CALL; }                                         \
    case 3: { constexpr int M = 8; return CALL; }                                         \
    case 4: { constexpr int M = 16; return CALL; }                                        \
    case 5: { constexpr int M = 32; return CALL; }                                        \
    case 6: { constexpr int M = 64; return CALL; }                                        \
    case 7: { constexpr int M = 128; return CALL; }                                       \
    case 8: { constexpr int M = 256; return CALL; }                                       \
    case 9: { constexpr int M = 512; return CALL; }                                       \
    case 10: { constexpr int M = 1024; return CALL; }                                     \
    case 11: { constexpr int M = 2048; return CALL; }                                     \
    case 12: { constexpr int M = 4096; return CALL; }                                     \
    case 13: { constexpr int M = 8192; return CALL; }                                     \
    case 14: { constexpr int M = 16384; return CALL; }                                    \
  }                                                                                       \
  return cudaErrorInvalidValue;

cudaError_t launch_spectrum(int log2m, const SpecArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  RSG_DISPATCH(log2m, spectrum_t<M>(a, s))
}

cudaError_t launch_ola(int log2m, const OlaArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  RSG_DISPATCH(log2m, ola_t<M>(a, s))
}

cudaError_t launch_rfft(int log2m, bool inverse, const float* in_real, const float2* in_spec,
                        float* out_real, float2* out_spec, int count, const float2* tw,
                        cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  RSG_DISPATCH(log2m, rfft_t<M>(inverse, in_real, in_spec, out_real, out_spec, count, tw, s))
}

// ============================================================================
// K5: SNR gains.  alpha_ij = sqrt(P_0j / (P_ij 10^(snr_i/10)))
// with P = mean_power (audio_buffer.hpp:66-75) = Σy^2 / len; alpha_0j = 1.
// ============================================================================
// K5a: mean power of every pair from its K4 partials (power.cuh): a warp per pair, lane l
// summing partials l, l + 32, ... then a fixed butterfly — one order per pair.
__global__ void __launch_bounds__(256) power_kernel(GainArgs a) {
  const long long p = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= a.n_pairs) return;  // warp-uniform
  const PairPlan& pl = a.plan[p];
  const double P = pair_power_warp<false>(a.part + pl.part0, pl.npart, pl.out_len, lane);
  if (lane == 0) a.power[p] = P;
}

// K5b: gains from the powers; alpha_0j = 1.
__global__ void gain_kernel(GainArgs a) {
  const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p >= a.n_pairs) return;
  const PairMeta& pm = a.pair[p];
  const long long p0 = a.utt_pair0[pm.utt] + pm.mic_local;  // target pair at mic j
  const bool target = pm.src_local == 0;
  bool deg;
  a.gain[p] = pair_gain(target, a.power[p], target ? 0.0 : a.power[p0], a.snr_lin[pm.src_idx], &deg);
  if (deg) a.flags[p] |= 4;
}

cudaError_t launch_gain(const GainArgs& a, cudaStream_t s) {
  if (a.n_pairs == 0) return cudaSuccess;
  power_kernel<<<static_cast<unsigned>((a.n_pairs + 7) / 8), 256, 0, s>>>(a);
  gain_kernel<<<static_cast<unsigned>((a.n_pairs + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ============================================================================
// K6: the mix y_j[n] = Σ_i alpha_ij (h_ij * x_i)[n], zero-padded, summed in
// source order by FP32 FMAs (MixQuadAcc, mixfin.cuh) — for the
// channels the K4 epilogue does not mix (a pair on a K4 variant without it, more than
// 8 sources, RSG_FUSED_MIX=0); the epilogue runs the same arithmetic.
// ============================================================================
__global__ void __launch_bounds__(256) mix_kernel(MixArgs a) {
  const long long ch = blockIdx.y;
  const long long u = a.chan_utt[ch];
  const long long stride = a.utt_stride[u];
  const long long n0 = blockIdx.x * a.tile;
  if (n0 >= stride) return;
  const int j = a.chan_mic[ch];
  const long long len = a.utt_len[u];
  const long long n1 = n0 + a.tile < stride ? n0 + a.tile : stride;
  const int I = a.utt_I[u], J = a.utt_J[u];
  const long long pair0 = a.utt_pair0[u];
  // the channel's per-source row / length / gain, read once per CTA (no dependent
  // metadata loads in the sample loop)
  __shared__ const float* s_row[kMixMaxI];
  __shared__ long long s_len[kMixMaxI];
  __shared__ double s_gain[kMixMaxI];
  if (threadIdx.x < kMixMaxI && threadIdx.x < I) {
    const long long p = pair0 + static_cast<long long>(threadIdx.x) * J + j;
    s_row[threadIdx.x] = a.y + a.plan[p].y_off;
    s_len[threadIdx.x] = a.plan[p].out_len;
    s_gain[threadIdx.x] = a.gain[p];
  }
  __syncthreads();
  const int Ic = I < kMixMaxI ? I : kMixMaxI;
  float* out = a.out + a.chan_out[ch];
  const bool out16 = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  // four consecutive samples per thread: float4 loads of every source's row (rows are
  // 16-byte aligned, y_off % 4 == 0), two sources' loads in flight at a time, FP64 sums in
  // source order, one float4 store
  for (long long n = n0 + 4 * threadIdx.x; n < n1; n += 4 * blockDim.x) {
    MixQuadAcc acc;
    if (n < len) {
      int i = 0;
      for (; i + 1 < Ic; i += 2) {
        const float4 va = mix_quad<false>(s_row[i], s_len[i], n);
        const float4 vb = mix_quad<false>(s_row[i + 1], s_len[i + 1], n);
        acc.add(s_gain[i], va);
        acc.add(s_gain[i + 1], vb);
      }
      if (i < Ic) acc.add(s_gain[i], mix_quad<false>(s_row[i], s_len[i], n));
      for (i = kMixMaxI; i < I; ++i) {  // beyond the cached sources
        const long long p = pair0 + static_cast<long long>(i) * J + j;
        acc.add(a.gain[p], mix_quad<false>(a.y + a.plan[p].y_off, a.plan[p].out_len, n));
      }
    }
    mix_store(out, out16, n, n1, len, acc);  // [len, stride): the zero-filled tail
  }
}

cudaError_t launch_mix(const MixArgs& a, int64_t n_chan, int64_t max_len, cudaStream_t s) {
  if (n_chan == 0 || max_len == 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((max_len + a.tile - 1) / a.tile), static_cast<unsigned>(n_chan));
  mix_kernel<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ---- small host<->device copies through the SMs ----------------------------------
// Per-chunk metadata and summaries move through mapped pinned memory with a kernel
// instead of the copy engines: the engines serve copies in FIFO order, and these
// small transfers must not queue behind a chunk's signal or output transfer.
__global__ void pcie_copy_kernel(char* __restrict__ dst, const char* __restrict__ src, size_t n) {
  const size_t n16 = n / 16;
  uint4* d16 = reinterpret_cast<uint4*>(dst);
  const uint4* s16 = reinterpret_cast<const uint4*>(src);
  const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = tid; i < n16; i += stride) d16[i] = s16[i];
  const size_t t = n16 * 16 + tid;
  if (t < n) dst[t] = src[t];
}

cudaError_t launch_pcie_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return cudaErrorMisalignedAddress;
  const size_t n16 = bytes / 16 + 1;
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n16 + 255) / 256, 148 * 4));
  pcie_copy_kernel<<<blocks, 256, 0, s>>>(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
  return cudaGetLastError();
}

// ---- convolve_direct (convolution.hpp:164-179), FP64, bit-exact ----------------------
// The reference accumulates out[i + j] += x[i] * h[j] with i outermost, so out[n] receives
// x[i] * h[n - i] for ascending i, starting from 0.0.  One thread per output sample adds
// the same products in the same order with round-to-nearest multiply and add (no FMA
// contraction): the result equals the reference bit for bit.  The h window of a CTA's 256
// outputs and the x samples it needs are staged through shared memory in 256-sample tiles.
__global__ void __launch_bounds__(256) direct_conv_kernel(const double* __restrict__ x, int64_t nx,
                                                          const double* __restrict__ h, int64_t nh,
                                                          double* __restrict__ out) {
  __shared__ double xs[256];
  __shared__ double hs[512];
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 256;
  const int64_t n = n0 + threadIdx.x;
  const int64_t out_len = nx + nh - 1;
  // i ranges over [max(0, n - nh + 1), min(n, nx - 1)]; the CTA's union:
  const int64_t i_lo = n0 - nh + 1 > 0 ? n0 - nh + 1 : 0;
  const int64_t i_hi = (n0 + 255 < nx - 1 ? n0 + 255 : nx - 1);
  double acc = 0.0;
  for (int64_t i0 = i_lo; i0 <= i_hi; i0 += 256) {
    __syncthreads();
    const int64_t i = i0 + threadIdx.x;
    xs[threadIdx.x] = i <= i_hi ? x[i] : 0.0;
    // h[n - i] for this tile: n - i in (n0 - i0 - 256, n0 + 255 - i0]; stage 512 taps
    // starting at j0 = n0 - i0 - 255
    const int64_t j0 = n0 - i0 - 255;
    for (int k = threadIdx.x; k < 512; k += 256) {
      const int64_t j = j0 + k;
      hs[k] = (j >= 0 && j < nh) ? h[j] : 0.0;
    }
    __syncthreads();
    if (n < out_len) {
      const int64_t a = n - nh + 1 > i0 ? n - nh + 1 : i0;        // first i of this tile for n
      const int64_t bnd = n < i0 + 255 ? n : i0 + 255;
      const int64_t b = bnd < i_hi ? bnd : i_hi;                  // last i
      for (int64_t ii = a; ii <= b; ++ii)
        acc = __dadd_rn(acc, __dmul_rn(xs[ii - i0], hs[(n - ii) - j0]));
    }
  }
  if (n < out_len) out[n] = acc;
}

cudaError_t launch_direct_conv(const double* x, int64_t nx, const double* h, int64_t nh, double* out,
                               cudaStream_t s) {
  const int64_t out_len = nx + nh - 1;
  if (out_len <= 0) return cudaSuccess;
  direct_conv_kernel<<<static_cast<unsigned>((out_len + 255) / 256), 256, 0, s>>>(x, nx, h, nh, out);
  return cudaGetLastError();
}

// ---- conversions -------------------------------------------------------------
__global__ void d2f_kernel(const double* in, float* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}
__global__ void f2d_kernel(const float* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}
cudaError_t launch_convert_d2f(const double* in, float* out, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = static_cast<int>((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  d2f_kernel<<<grid, 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}
cudaError_t launch_convert_f2d(const float* in, double* out, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = static_cast<int>((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  f2d_kernel<<<grid, 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace rsg

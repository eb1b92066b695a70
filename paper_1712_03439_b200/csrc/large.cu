// large.cu — the OLA filter for transforms too large for one CTA's shared memory
// (M = N/2 >= 2^kLargeMinLog2M complex points), as a four-step FFT through a
// global scratch buffer.  Same arithmetic contract as K3/K4 (FP32, the half-size
// complex transform of the packed real block, the untangle/multiply/repack of
// convolution.hpp:238-253 with fft.hpp:104-110/152-161), different data movement:
//
//   M = M1 * M2, input index n = n1*M2 + n2, output index k = k1 + M1*k2
//   stage A  (per block, tile of CT columns n2)  : z[n1*M2 + n2] -> FFT_M1 over n1,
//            times W_M^(n2 k1)                   -> scratch row k1, column n2
//   stage B  (per block, row pair k1, M1-k1)     : FFT_M2 over n2 -> X[k1 + M1 k2];
//            X[k] and X[M-k] sit in rows k1 and M1-k1 (k1 = 0, M1/2 pair with
//            themselves), so the untangle x G x repack runs here; then the inverse
//            FFT_M2 and conj(W_M^(n2 k1)) -> scratch row k1 (in place)
//   stage C  (per block, tile of CT columns)     : inverse FFT_M1 over k1 -> the
//            block's N output samples
//   stage D  (per pair, tile of output samples)  : overlap-add of the block
//            outputs in ascending block order + Σ y^2 of the tile (FP64)
//
// The RIR spectrum runs stages A and B on the packed RIR (stage B untangles
// into G = H / (4M), stored row-major by k1 for coalesced stage-B reads).
// Every sum has a fixed order: deterministic, no atomics.
#include <cmath>

#include "fft.cuh"
#include "kernels.cuh"

namespace rsg {
namespace {

// W_M^x = exp(-2 pi i x / M) (x reduced mod M: exact argument; sincospif is
// measured faster here than a table gather)
__device__ __forceinline__ float2 twiddle_m(int x, int log2M) {
  const int r = x & ((1 << log2M) - 1);
  float sn, cs;
  sincospif(-2.0f * ldexpf(static_cast<float>(r), -log2M), &sn, &cs);
  return make_float2(cs, sn);
}
// W^k = exp(-2 pi i k / N), N = 2M, k in [0, M]
__device__ __forceinline__ float2 twiddle_n(int k, int log2M) {
  float sn, cs;
  sincospif(-ldexpf(static_cast<float>(k), -log2M), &sn, &cs);
  return make_float2(cs, sn);
}

template <int M1, int M2>
constexpr int col_tile() {  // columns per stage-A/C CTA: <= 512 threads, <= 16 columns, <= M2
  return (512 / Plan<M1>::T) < 16 ? ((512 / Plan<M1>::T) < M2 ? 512 / Plan<M1>::T : M2) : (16 < M2 ? 16 : M2);
}

// ---- stage A: column FFTs of a tile (block input or RIR) ----------------------
template <int M1, int M2, bool SPEC>
__global__ void __launch_bounds__(col_tile<M1, M2>() * Plan<M1>::T) large_cols_fwd(LargeArgs a) {
  using P1 = Plan<M1>;
  constexpr int CT = col_tile<M1, M2>(), NT = CT * P1::T, TILES = M2 / CT;
  constexpr int LOGM = P1::LOG + Plan<M2>::LOG;
  extern __shared__ __align__(16) float2 smem[];
  const int unit = blockIdx.x / TILES, c0 = (blockIdx.x % TILES) * CT;
  const int2 un = SPEC ? make_int2(a.spec_pairs[unit], 0) : a.units[unit];
  const PairPlan& pl = a.plan[un.x];
  const PairMeta& pm = a.pair[un.x];
  long long take;
  const float* xs = nullptr;
  const double* hs = nullptr;
  if constexpr (SPEC) {
    hs = a.rir + pm.rir_off;
    take = pl.nh;
  } else {
    const long long st = static_cast<long long>(un.y) * pl.L;
    xs = a.signals + pm.sig_off + st;
    take = pm.nx - st < pl.L ? pm.nx - st : pl.L;
  }
  // gather: element n1 of column c is z[n1*M2 + c0 + c] = (src[2n], src[2n+1])
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int n1 = idx / CT, c = idx - n1 * CT;
    const long long n = static_cast<long long>(n1) * M2 + c0 + c;
    float2 v;
    if constexpr (SPEC) {
      v.x = 2 * n < take ? static_cast<float>(hs[2 * n]) : 0.f;
      v.y = 2 * n + 1 < take ? static_cast<float>(hs[2 * n + 1]) : 0.f;
    } else {
      v.x = 2 * n < take ? xs[2 * n] : 0.f;
      v.y = 2 * n + 1 < take ? xs[2 * n + 1] : 0.f;
    }
    smem[c * P1::PADDED + PAD(n1)] = v;
  }
  __syncthreads();
  const int c = threadIdx.x / P1::T, t = threadIdx.x % P1::T;
  forward_rest<M1, 0>(smem + c * P1::PADDED, t, a.tw1, true);
  float2* dst = a.scratch + static_cast<long long>(unit) * (M1 * M2);
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int k1 = idx / CT, cc = idx - k1 * CT;
    const float2 v = smem[cc * P1::PADDED + PAD(k1)];
    dst[static_cast<long long>(k1) * M2 + c0 + cc] = c_mul(v, twiddle_m((c0 + cc) * k1, LOGM));
  }
}

// ---- stage B: row FFTs, untangle (SPEC) or pairing + inverse row FFTs ----------
template <int M1, int M2, bool SPEC>
__global__ void __launch_bounds__(2 * Plan<M2>::T) large_rows(LargeArgs a) {
  using P2 = Plan<M2>;
  constexpr int T = P2::T, JOBS = M1 / 2 + 1;
  constexpr int LOGM = Plan<M1>::LOG + P2::LOG;
  constexpr int M = M1 * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int unit = blockIdx.x / JOBS, job = blockIdx.x % JOBS;
  const int pair = SPEC ? a.spec_pairs[unit] : a.units[unit].x;
  const PairPlan& pl = a.plan[pair];
  float2* G = a.spec + pl.spec_off;  // G[k1*M2 + k2] = G(k1 + M1 k2); G[M] = G(M)
  const bool self = job == 0 || job == M1 / 2;
  const int row0 = job, row1 = (M1 - job) & (M1 - 1);
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const bool active = g == 0 || !self;
  const int row = g ? row1 : row0;
  float2* s = smem + g * P2::PADDED;
  float2* src = a.scratch + static_cast<long long>(unit) * M + static_cast<long long>(row) * M2;
  if (active)
    for (int n2 = t; n2 < M2; n2 += T) s[PAD(n2)] = src[n2];
  __syncthreads();
  forward_rest<M2, 0>(s, t, a.tw2, active);  // s[PAD(k2)] = X[row + M1 k2]
  float2* s0 = smem;
  float2* s1 = self ? smem : smem + P2::PADDED;
  // element k2 of row0 pairs with element m(k2) of row1:
  //   row pair (k1, M1-k1): M2-1-k2;  row 0: (M2-k2) mod M2;  row M1/2: M2-1-k2
  auto partner = [&](int k2) { return job == 0 ? ((M2 - k2) & (M2 - 1)) : (M2 - 1 - k2); };
  if constexpr (SPEC) {
    // every element k of both rows: G(k) = (Z[k] + conj Z[M-k] + W^k (-i)(Z[k] - conj Z[M-k])) / (8M)
    const float scale = 1.0f / (8.0f * M);
    for (int e = threadIdx.x; e < 2 * M2; e += 2 * T) {
      const int gg = e / M2, k2 = e - gg * M2;
      if (gg == 1 && self) continue;
      const int rk = gg ? row1 : row0;
      const int k = rk + M1 * k2;
      const float2 za = (gg ? s1 : s0)[PAD(k2)];
      const float2 zb = c_conj((gg ? s0 : s1)[PAD(partner(k2))]);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      G[static_cast<long long>(rk) * M2 + k2] = c_scale(c_add(S, c_mul(twiddle_n(k, LOGM), D)), scale);
      if (k == 0) {  // G(M) = (S - D) / (8M): W^M = -1
        G[M] = c_scale(c_sub(S, D), scale);
      }
    }
  } else {
    // pairs (k, M-k) once each; the same formulas as spectral_multiply
    const int npairs = job == 0 ? M2 / 2 + 1 : (job == M1 / 2 ? M2 / 2 : M2);
    for (int e = threadIdx.x; e < npairs; e += 2 * T) {
      const int k2 = e, m2 = partner(k2);
      const int k = row0 + M1 * k2;
      const bool own = self && m2 == k2;  // k = 0 or k = M/2: its own partner
      const float2 za = s0[PAD(k2)];
      const float2 zb = c_conj(s1[PAD(m2)]);
      const float2 w = twiddle_n(k, LOGM);
      const float2 S = c_add(za, zb);
      const float2 D = c_rot<false>(c_sub(za, zb));
      const float2 wD = c_mul(w, D);
      const float2 X2 = c_add(S, wD), X2m = c_sub(S, wD);
      const float2 gk = G[static_cast<long long>(row0) * M2 + k2];
      const float2 gm = k == 0 ? G[M] : G[static_cast<long long>(row1) * M2 + m2];
      const float2 P = c_mul(X2, gk);
      const float2 Q = c_mulc(X2m, gm);
      const float2 U = c_add(P, Q);
      const float2 V = c_mulc(c_sub(P, Q), w);
      s0[PAD(k2)] = make_float2(U.x - V.y, U.y + V.x);
      if (!own) s1[PAD(m2)] = make_float2(U.x + V.y, V.x - U.y);
    }
    __syncthreads();
    inverse_all<M2>(s, t, a.tw2, active);  // natural n2
    if (active)
      for (int n2 = t; n2 < M2; n2 += T) src[n2] = c_mulc(s[PAD(n2)], twiddle_m(n2 * row, LOGM));
  }
}

// ---- stage C: inverse column FFTs -> block outputs ------------------------------
template <int M1, int M2>
__global__ void __launch_bounds__(col_tile<M1, M2>() * Plan<M1>::T) large_cols_inv(LargeArgs a) {
  using P1 = Plan<M1>;
  constexpr int CT = col_tile<M1, M2>(), NT = CT * P1::T, TILES = M2 / CT;
  constexpr long long M = static_cast<long long>(M1) * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int unit = blockIdx.x / TILES, c0 = (blockIdx.x % TILES) * CT;
  const float2* src = a.scratch + unit * M;
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int k1 = idx / CT, c = idx - k1 * CT;
    smem[c * P1::PADDED + PAD(k1)] = src[static_cast<long long>(k1) * M2 + c0 + c];
  }
  __syncthreads();
  const int c = threadIdx.x / P1::T, t = threadIdx.x % P1::T;
  inverse_all<M1>(smem + c * P1::PADDED, t, a.tw1, true);
  float2* out = reinterpret_cast<float2*>(a.yblk + unit * (2 * M));  // packed (y[2n], y[2n+1])
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int n1 = idx / CT, cc = idx - n1 * CT;
    out[static_cast<long long>(n1) * M2 + c0 + cc] = smem[cc * P1::PADDED + PAD(n1)];
  }
}

}  // namespace

// ---- stage D: overlap-add of block outputs + Σ y^2 per tile ----------------------
constexpr int kLargeTile = 2048;  // output samples per stage-D item

__global__ void __launch_bounds__(256) large_ola_sum(LargeArgs a, long long n_fft) {
  const int item = blockIdx.x;
  const OlaItem it = a.items[item];
  const PairPlan& pl = a.plan[it.pair];
  const long long L = pl.L, B = pl.B, out_len = pl.out_len;
  const float* yb = a.yblk + static_cast<long long>(it.b_own) * n_fft;  // block 0 of the pair
  float* y = a.y + pl.y_off;
  double pw = 0.0;
  const long long n0 = static_cast<long long>(it.b_begin) * kLargeTile;
  for (int i = 0; i < kLargeTile / 256; ++i) {
    const long long n = n0 + i * 256 + threadIdx.x;
    if (n >= out_len) break;
    long long b_lo = n >= n_fft ? (n - n_fft) / L + 1 : 0;
    const long long b_hi = n / L < B - 1 ? n / L : B - 1;
    float acc = 0.f;
    for (long long b = b_lo; b <= b_hi; ++b) acc += yb[b * n_fft + (n - b * L)];  // ascending blocks
    y[n] = acc;
    pw = fma(static_cast<double>(acc), static_cast<double>(acc), pw);
  }
  // the tile's partial (fixed order) -> the pair's slot of this tile (power.cuh)
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    a.part[pl.part0 + it.b_begin] = tot;
  }
}

namespace {

template <int M1, int M2>
cudaError_t large_launch(const LargeArgs& a, int stage, cudaStream_t s) {
  using P1 = Plan<M1>;
  using P2 = Plan<M2>;
  constexpr int CT = col_tile<M1, M2>(), TILES = M2 / CT;
  const size_t smem_cols = static_cast<size_t>(CT) * P1::PADDED * sizeof(float2);
  const size_t smem_rows = 2 * static_cast<size_t>(P2::PADDED) * sizeof(float2);
  cudaError_t e = cudaSuccess;
  switch (stage) {
    case 0:  // spectrum: A on the RIRs
      if (a.n_spec == 0) return cudaSuccess;
      e = cudaFuncSetAttribute(large_cols_fwd<M1, M2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cols);
      if (e != cudaSuccess) return e;
      large_cols_fwd<M1, M2, true><<<a.n_spec * TILES, CT * P1::T, smem_cols, s>>>(a);
      break;
    case 1:  // spectrum: B (untangle into G)
      if (a.n_spec == 0) return cudaSuccess;
      e = cudaFuncSetAttribute(large_rows<M1, M2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rows);
      if (e != cudaSuccess) return e;
      large_rows<M1, M2, true><<<a.n_spec * (M1 / 2 + 1), 2 * P2::T, smem_rows, s>>>(a);
      break;
    case 2:
      if (a.n_units == 0) return cudaSuccess;
      e = cudaFuncSetAttribute(large_cols_fwd<M1, M2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cols);
      if (e != cudaSuccess) return e;
      large_cols_fwd<M1, M2, false><<<a.n_units * TILES, CT * P1::T, smem_cols, s>>>(a);
      break;
    case 3:
      if (a.n_units == 0) return cudaSuccess;
      e = cudaFuncSetAttribute(large_rows<M1, M2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rows);
      if (e != cudaSuccess) return e;
      large_rows<M1, M2, false><<<a.n_units * (M1 / 2 + 1), 2 * P2::T, smem_rows, s>>>(a);
      break;
    case 4:
      if (a.n_units == 0) return cudaSuccess;
      e = cudaFuncSetAttribute(large_cols_inv<M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cols);
      if (e != cudaSuccess) return e;
      large_cols_inv<M1, M2><<<a.n_units * TILES, CT * P1::T, smem_cols, s>>>(a);
      break;
    case 5:
      if (a.n_items == 0) return cudaSuccess;
      large_ola_sum<<<a.n_items, 256, 0, s>>>(a, 2LL * M1 * M2);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

// ---- the RealFftEngine seam (fft.hpp:38-49) for large N: natural-order spectra ------
namespace {

// forward stage A: column FFTs of the packed real input (no zero padding)
template <int M1, int M2>
__global__ void __launch_bounds__(col_tile<M1, M2>() * Plan<M1>::T)
rfft_cols_fwd(const float* in, float2* scratch, const float2* tw1) {
  using P1 = Plan<M1>;
  constexpr int CT = col_tile<M1, M2>(), NT = CT * P1::T, TILES = M2 / CT;
  constexpr int LOGM = P1::LOG + Plan<M2>::LOG;
  constexpr long long M = static_cast<long long>(M1) * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int item = blockIdx.x / TILES, c0 = (blockIdx.x % TILES) * CT;
  const float2* z = reinterpret_cast<const float2*>(in + item * 2 * M);
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int n1 = idx / CT, c = idx - n1 * CT;
    smem[c * P1::PADDED + PAD(n1)] = z[static_cast<long long>(n1) * M2 + c0 + c];
  }
  __syncthreads();
  forward_rest<M1, 0>(smem + (threadIdx.x / P1::T) * P1::PADDED, threadIdx.x % P1::T, tw1, true);
  float2* dst = scratch + item * M;
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int k1 = idx / CT, cc = idx - k1 * CT;
    dst[static_cast<long long>(k1) * M2 + c0 + cc] = c_mul(smem[cc * P1::PADDED + PAD(k1)], twiddle_m((c0 + cc) * k1, LOGM));
  }
}

// forward stage B: row FFTs of rows k1, M1 - k1, untangle into X[k] (natural order, N/2 + 1)
template <int M1, int M2>
__global__ void __launch_bounds__(2 * Plan<M2>::T) rfft_rows_fwd(const float2* scratch, float2* out, const float2* tw2) {
  using P2 = Plan<M2>;
  constexpr int T = P2::T, JOBS = M1 / 2 + 1;
  constexpr int LOGM = Plan<M1>::LOG + P2::LOG;
  constexpr long long M = static_cast<long long>(M1) * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int item = blockIdx.x / JOBS, job = blockIdx.x % JOBS;
  const bool self = job == 0 || job == M1 / 2;
  const int row0 = job, row1 = (M1 - job) & (M1 - 1);
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const bool active = g == 0 || !self;
  float2* s = smem + g * P2::PADDED;
  const float2* src = scratch + item * M + static_cast<long long>(g ? row1 : row0) * M2;
  if (active)
    for (int n2 = t; n2 < M2; n2 += T) s[PAD(n2)] = src[n2];
  __syncthreads();
  forward_rest<M2, 0>(s, t, tw2, active);
  float2* s0 = smem;
  float2* s1 = self ? smem : smem + P2::PADDED;
  auto partner = [&](int k2) { return job == 0 ? ((M2 - k2) & (M2 - 1)) : (M2 - 1 - k2); };
  float2* o = out + item * (M + 1);
  for (int e = threadIdx.x; e < 2 * M2; e += 2 * T) {
    const int gg = e / M2, k2 = e - gg * M2;
    if (gg == 1 && self) continue;
    const int rk = gg ? row1 : row0;
    const int k = rk + M1 * k2;
    const float2 za = (gg ? s1 : s0)[PAD(k2)];
    const float2 zb = c_conj((gg ? s0 : s1)[PAD(partner(k2))]);
    const float2 S = c_add(za, zb);
    const float2 D = c_rot<false>(c_sub(za, zb));
    o[k] = c_scale(c_add(S, c_mul(twiddle_n(k, LOGM), D)), 0.5f);
    if (k == 0) o[M] = c_scale(c_sub(S, D), 0.5f);  // W^M = -1
  }
}

// inverse stage B: repack row k1 of the spectrum (fft.hpp:104-110), inverse row FFT,
// conj twiddles -> scratch
template <int M1, int M2>
__global__ void __launch_bounds__(Plan<M2>::T) rfft_rows_inv(const float2* in, float2* scratch, const float2* tw2) {
  using P2 = Plan<M2>;
  constexpr int T = P2::T;
  constexpr int LOGM = Plan<M1>::LOG + P2::LOG;
  constexpr long long M = static_cast<long long>(M1) * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int item = blockIdx.x / M1, row = blockIdx.x % M1;
  const int t = threadIdx.x;
  const float2* X = in + item * (M + 1);
  for (int k2 = t; k2 < M2; k2 += T) {
    const long long k = row + static_cast<long long>(M1) * k2;
    const float2 xa = X[k], xb = c_conj(X[M - k]);
    const float2 e = c_scale(c_add(xa, xb), 0.5f);
    const float2 o = c_mulc(c_scale(c_sub(xa, xb), 0.5f), twiddle_n(static_cast<int>(k), LOGM));
    smem[PAD(k2)] = make_float2(e.x - o.y, e.y + o.x);
  }
  __syncthreads();
  inverse_all<M2>(smem, t, tw2, true);
  float2* dst = scratch + item * M + static_cast<long long>(row) * M2;
  for (int n2 = t; n2 < M2; n2 += T) dst[n2] = c_mulc(smem[PAD(n2)], twiddle_m(n2 * row, LOGM));
}

// inverse stage C: inverse column FFTs -> N real samples, scaled by 1/M (fft.hpp:112-116)
template <int M1, int M2>
__global__ void __launch_bounds__(col_tile<M1, M2>() * Plan<M1>::T)
rfft_cols_inv(const float2* scratch, float* out, const float2* tw1) {
  using P1 = Plan<M1>;
  constexpr int CT = col_tile<M1, M2>(), NT = CT * P1::T, TILES = M2 / CT;
  constexpr long long M = static_cast<long long>(M1) * M2;
  extern __shared__ __align__(16) float2 smem[];
  const int item = blockIdx.x / TILES, c0 = (blockIdx.x % TILES) * CT;
  const float2* src = scratch + item * M;
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int k1 = idx / CT, c = idx - k1 * CT;
    smem[c * P1::PADDED + PAD(k1)] = src[static_cast<long long>(k1) * M2 + c0 + c];
  }
  __syncthreads();
  inverse_all<M1>(smem + (threadIdx.x / P1::T) * P1::PADDED, threadIdx.x % P1::T, tw1, true);
  float2* o = reinterpret_cast<float2*>(out + item * 2 * M);
  const float sc = 1.0f / static_cast<float>(M);
  for (int idx = threadIdx.x; idx < M1 * CT; idx += NT) {
    const int n1 = idx / CT, cc = idx - n1 * CT;
    o[static_cast<long long>(n1) * M2 + c0 + cc] = c_scale(smem[cc * P1::PADDED + PAD(n1)], sc);
  }
}

template <int M1, int M2>
cudaError_t rfft_large_t(bool inverse, const float* in_real, const float2* in_spec, float* out_real,
                         float2* out_spec, int count, float2* scratch, const float2* tw1, const float2* tw2,
                         cudaStream_t s) {
  using P1 = Plan<M1>;
  using P2 = Plan<M2>;
  constexpr int CT = col_tile<M1, M2>(), TILES = M2 / CT;
  const int smem_cols = CT * P1::PADDED * static_cast<int>(sizeof(float2));
  cudaError_t e;
  if (!inverse) {
    if ((e = cudaFuncSetAttribute(rfft_cols_fwd<M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cols)))
      return e;
    rfft_cols_fwd<M1, M2><<<count * TILES, CT * P1::T, smem_cols, s>>>(in_real, scratch, tw1);
    const int smem_rows = 2 * P2::PADDED * static_cast<int>(sizeof(float2));
    if ((e = cudaFuncSetAttribute(rfft_rows_fwd<M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_rows)))
      return e;
    rfft_rows_fwd<M1, M2><<<count * (M1 / 2 + 1), 2 * P2::T, smem_rows, s>>>(scratch, out_spec, tw2);
  } else {
    const int smem_row = P2::PADDED * static_cast<int>(sizeof(float2));
    if ((e = cudaFuncSetAttribute(rfft_rows_inv<M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_row)))
      return e;
    rfft_rows_inv<M1, M2><<<count * M1, P2::T, smem_row, s>>>(in_spec, scratch, tw2);
    if ((e = cudaFuncSetAttribute(rfft_cols_inv<M1, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cols)))
      return e;
    rfft_cols_inv<M1, M2><<<count * TILES, CT * P1::T, smem_cols, s>>>(scratch, out_real, tw1);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_large_rfft(int log2m, bool inverse, const float* in_real, const float2* in_spec,
                              float* out_real, float2* out_spec, int count, float2* scratch,
                              const float2* tw1, const float2* tw2, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  switch (log2m) {
#define RSG_RF(L, A, B) \
  case L: return rfft_large_t<A, B>(inverse, in_real, in_spec, out_real, out_spec, count, scratch, tw1, tw2, s);
    RSG_RF(13, 64, 128) RSG_RF(14, 128, 128) RSG_RF(15, 128, 256) RSG_RF(16, 256, 256) RSG_RF(17, 256, 512)
    RSG_RF(18, 512, 512) RSG_RF(19, 512, 1024) RSG_RF(20, 1024, 1024) RSG_RF(21, 1024, 2048)
    RSG_RF(22, 2048, 2048)
#undef RSG_RF
    default: return cudaErrorInvalidValue;
  }
}

// log2 M -> (log2 M1, log2 M2): M1 = 2^floor(l/2) columns of M2 = 2^ceil(l/2)
void large_split(int log2m, int* l1, int* l2) {
  *l1 = log2m / 2;
  *l2 = log2m - log2m / 2;
}

int large_tile() { return kLargeTile; }

cudaError_t launch_large(int log2m, const LargeArgs& a, int stage, cudaStream_t s) {
  switch (log2m) {
    case 6: return large_launch<8, 8>(a, stage, s);
    case 7: return large_launch<8, 16>(a, stage, s);
    case 8: return large_launch<16, 16>(a, stage, s);
    case 9: return large_launch<16, 32>(a, stage, s);
    case 10: return large_launch<32, 32>(a, stage, s);
    case 11: return large_launch<32, 64>(a, stage, s);
    case 12: return large_launch<64, 64>(a, stage, s);
    case 13: return large_launch<64, 128>(a, stage, s);
    case 14: return large_launch<128, 128>(a, stage, s);
    case 15: return large_launch<128, 256>(a, stage, s);
    case 16: return large_launch<256, 256>(a, stage, s);
    case 17: return large_launch<256, 512>(a, stage, s);
    case 18: return large_launch<512, 512>(a, stage, s);
    case 19: return large_launch<512, 1024>(a, stage, s);
    case 20: return large_launch<1024, 1024>(a, stage, s);
    case 21: return large_launch<1024, 2048>(a, stage, s);
    case 22: return large_launch<2048, 2048>(a, stage, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsg

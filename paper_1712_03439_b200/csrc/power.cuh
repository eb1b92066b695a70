// power.cuh — per-segment power partials of the K4 variants.
//
// mean_power (audio_buffer.hpp:66-75) of a reverberant pair signal is Σ y² / len.  A
// pair's OLA blocks are grouped in segments of kPowerSeg consecutive blocks (segment s =
// blocks [16 s, 16 s + 16)); the planner starts every K4 run on a segment boundary, so a
// segment is always filtered by one work item.  Each lane sums its FP32 per-block Σ y²
// over the segment in FP64 (block order); at the segment's end the group's lanes are
// reduced by a fixed butterfly and one FP64 partial per (segment, warp of the group) is
// stored.  The gain kernel sums a pair's partials in a fixed order.  The power therefore
// depends only on the pair and its kernel variant (chosen from the pair's N and N_h), not
// on how its blocks were split into work items, which render chunk it rode in or which
// other pairs shared the launch — so a render's bytes do not depend on the batch
// composition, the chunk size or the number of ranks.
#pragma once

namespace rsg {

constexpr int kPowerSeg = 16;  // OLA blocks per power segment (runs start on multiples)

// partials per segment: one per warp of the group (one for groups narrower than a warp)
__host__ __device__ constexpr int parts_per_block_of(int T) { return T < 32 ? 1 : T / 32; }
__host__ __device__ constexpr long long power_segments(long long B, int seg = kPowerSeg) { return (B + seg - 1) / seg; }
// The in-place K4 at M >= 8192 (few, long blocks per pair) uses 2-block segments, so its runs
// can be short enough to spread a small bucket over the SMs.
constexpr int kPowerSegLarge = 2;

// true when block b closes a segment (of seg blocks) of a run ending at b_end
__device__ __forceinline__ bool closes_segment(int b, int b_end, int seg = kPowerSeg) {
  return (b + 1) % seg == 0 || b + 1 == b_end;
}

// v: this lane's FP64 Σ y² over one segment.  The group's T lanes (T < 32: a T-aligned
// lane range of the warp; else whole warps) reduce theirs; lane 0 of each warp of the
// group stores at slot[warp of the group] when `write`.  All 32 lanes of the warp must
// call it.
template <int T>
__device__ __forceinline__ void store_segment_power(double* slot, double v, int t, bool write) {
  constexpr int W = T < 32 ? T : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (write && (t & (W - 1)) == 0) slot[t / 32] = v;
}

}  // namespace rsg

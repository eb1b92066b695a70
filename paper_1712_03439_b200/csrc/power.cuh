// power.cuh — per-block power partials of the K4 variants.
//
// mean_power (audio_buffer.hpp:66-75) of a reverberant pair signal is Σ y² / len.  Every
// K4 variant writes one FP64 partial per (OLA block, warp of the group that transformed
// the block): the warp's lanes' FP32 Σ y² over the block's final, owned samples, summed
// in FP64 by a fixed butterfly.  The gain kernel sums a pair's partials in a fixed order.
// The sum therefore depends only on the pair and the kernel variant (chosen from the
// pair's N and N_h), not on how its blocks were split into work items, which render
// chunk it rode in or which other pairs shared the launch — so a render's bytes do not
// depend on the batch composition, the chunk size or the number of ranks.
#pragma once

namespace rsg {

__host__ __device__ constexpr int parts_per_block_of(int T) { return T < 32 ? 1 : T / 32; }

// v: this lane's FP32 Σ y² of one block.  The group's T lanes (T < 32: a T-aligned lane
// range of the warp; else whole warps) reduce theirs; lane 0 of each warp of the group
// stores at slot[warp of the group] when `write`.  All 32 lanes of the warp must call it.
template <int T>
__device__ __forceinline__ void store_block_power(double* slot, float v, int t, bool write) {
  constexpr int W = T < 32 ? T : 32;
  double d = static_cast<double>(v);
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if (write && (t & (W - 1)) == 0) slot[t / 32] = d;
}

}  // namespace rsg

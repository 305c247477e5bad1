// topk.cuh -- exact warp-cooperative top-R selection on 64-bit composite keys.
//
// Steps 2 and 5 of PAPER.md §4.2 only require a partial order (PAPER.md:369-377,
// 416-424); readings R9/R10 totalise it with the list index / item id.  Packing
// (distance, index) into one uint64 makes a single unsigned compare implement that
// total order, so any correct selection network is bit-exact and order-independent:
//   Step 2 / build ranking: key = (uint64(d_i) << 32) | i                (d_i >= 0)
//   Step 5:                 key = (uint64(D)  << 32) | (uint32(id) ^ 0x80000000)
//                           (the XOR maps signed id order onto unsigned order, so the
//                           padding item -1 sorts before item 0 at equal D).
#pragma once
#include <stdint.h>

namespace v3db {

__device__ __forceinline__ uint64_t step2_key(int32_t dist, int32_t idx) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(dist)) << 32) | static_cast<uint32_t>(idx);
}
__device__ __forceinline__ uint64_t step5_key(int32_t dist, int32_t id) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(dist)) << 32) |
         (static_cast<uint32_t>(id) ^ 0x80000000u);
}
__device__ __forceinline__ int32_t step5_id(uint64_t key) {
  return static_cast<int32_t>(static_cast<uint32_t>(key) ^ 0x80000000u);
}

// Insert `key` (warp-uniform, key < T[R-1]) into the ascending shared-memory list
// T[0..R), dropping the largest entry.  All 32 lanes must call.  Returns T[R-1].
__device__ __forceinline__ uint64_t warp_insert(uint64_t* T, int R, uint64_t key) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int j = lane; j < R; j += 32) cnt += (T[j] < key) ? 1 : 0;
  const int pos = __reduce_add_sync(0xffffffffu, cnt);
  // shift T[pos..R-2] up by one, 32 entries at a time from the top down
  for (int c = ((R - 2) >> 5) << 5; c >= ((pos >> 5) << 5) && c >= 0; c -= 32) {
    const int j = c + lane;
    const bool mv = (j >= pos) && (j < R - 1);
    uint64_t v = 0;
    if (mv) v = T[j];
    __syncwarp();
    if (mv) T[j + 1] = v;
    __syncwarp();
  }
  if (lane == 0) T[pos] = key;
  __syncwarp();
  return T[R - 1];
}

// Offer one candidate per lane; inserts those below the current threshold `thr`
// (warp-uniform, == T[R-1]) in lane order.  Returns the updated threshold.
__device__ __forceinline__ uint64_t warp_offer(uint64_t* T, int R, uint64_t thr, uint64_t key) {
  unsigned mask = __ballot_sync(0xffffffffu, key < thr);
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
    if (kk < thr) thr = warp_insert(T, R, kk);
  }
  return thr;
}

}  // namespace v3db

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

namespace v3db {

// Register-resident exact warp top-k (k <= 32*KR): entry j of the ascending list lives in
// lane j % 32, register j / 32.  Insertion of a warp-uniform key: its rank from KR ballots,
// then a one-position shift of the tail through shuffles -- no shared memory, no
// __syncwarp.  `thr` caches entry k-1 (the admission threshold).
template <int KR>
struct WarpTopK {
  uint64_t v[KR];
  uint64_t thr;
  int k;

  __device__ __forceinline__ void init(int k_) {
#pragma unroll
    for (int r = 0; r < KR; ++r) v[r] = ~0ull;
    thr = ~0ull;
    k = k_;
  }
  __device__ __forceinline__ uint64_t entry(int j) const {  // warp-uniform j
    // select v[j >> 5] with explicit selp: a plain conditional chain is turned into a
    // dynamically indexed (local-memory) access by the compiler
    const uint32_t rj = static_cast<uint32_t>(j >> 5);
    uint64_t x = v[0];
#pragma unroll
    for (int r = 1; r < KR; ++r)
      asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, %3;\n\tselp.b64 %0, %1, %0, p;\n\t}" : "+l"(x) : "l"(v[r]), "r"(rj), "r"(static_cast<uint32_t>(r)));
    return __shfl_sync(0xffffffffu, x, j & 31);
  }
  __device__ __forceinline__ void insert(uint64_t key) {  // warp-uniform, key < thr
    const int lane = threadIdx.x & 31;
    int pos = 0;
#pragma unroll
    for (int r = 0; r < KR; ++r) pos += __popc(__ballot_sync(0xffffffffu, v[r] < key));
#pragma unroll
    for (int r = KR - 1; r >= 0; --r) {
      uint64_t up = __shfl_up_sync(0xffffffffu, v[r], 1);
      if (r > 0) {
        const uint64_t carry = __shfl_sync(0xffffffffu, v[r > 0 ? r - 1 : 0], 31);
        if (lane == 0) up = carry;
      }
      const int j = r * 32 + lane;
      v[r] = (j > pos) ? up : ((j == pos) ? key : v[r]);
    }
    thr = entry(k - 1);
  }
  // One candidate per lane; keys below the threshold are inserted in lane order.
  __device__ __forceinline__ void offer(uint64_t key) {
    unsigned mask = __ballot_sync(0xffffffffu, key < thr);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
      if (kk < thr) insert(kk);
    }
  }
  // Write entries [0, k) with f(j, key) (lane-strided).
  template <class F>
  __device__ __forceinline__ void store(F f) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < KR; ++r)
      if (r * 32 + lane < k) f(r * 32 + lane, v[r]);
  }
};

// Call f.template operator()<KR>() with KR = the smallest power of two, 32*KR >= k.
template <class F>
__host__ __forceinline__ void dispatch_kr(int k, F f) {
  if (k <= 32) f.template operator()<1>();
  else if (k <= 64) f.template operator()<2>();
  else if (k <= 128) f.template operator()<4>();
  else if (k <= 256) f.template operator()<8>();
  else if (k <= 512) f.template operator()<16>();
  else f.template operator()<32>();
}

}  // namespace v3db

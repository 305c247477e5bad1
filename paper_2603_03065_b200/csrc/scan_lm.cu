// scan_lm.cu -- Steps 3-5 of PAPER.md §4.2, list-major, on the 5th-gen tensor cores.
//
// Step 3 builds LUT_{i,m,c} = dist(C_{m,c}, (q - mu_i)^{(m)}) and Step 4 sums
// the entries a slot's codes select.  With xhat_{i,j} the slot's reconstruction
// (its codewords concatenated) that sum is the exact integer identity
//     d~_{i,j} = sum_m LUT_{i,m,code_m} = dist(q - mu_i, xhat) = d_i + P_{i,j} - 2 <q, xhat_{i,j}>
// with P_{i,j} = ||xhat||^2 + 2 <mu_i, xhat> (per slot, built once) -- every term an integer below
// 2^31, so the result equals the literal Steps 3-4 bit for bit.
// Grouped by list, the per-query terms <q, xhat> of all the queries probing list i form a dense
// int8 contraction  [128 slots x D] . [D x n_i queries] -> int32, issued as tcgen05.mma.kind::i8
// (M = 128 slots, N = the probing queries, K = 32) with the slots' xhat brought in by TMA and the
// gathered query rows by cp.async; the accumulators live in TMEM.  Each list tile is read once per
// batch for all the queries that probe it instead of once per query.
//
// Work item = (list i, up to NT of the (query, rank) pairs probing it).  Warp roles (persistent
// CTA, one per SM; a CTA draws its next item from a grid-wide counter when it is ready for one):
//   warp 0      one lane: draws the items and publishes them through a shared-memory ring every role
//               reads; TMA loads of the xhat tiles (128 slots x 128-byte K panel) into a ring;
//   warp 1      one lane: the MMAs (double-buffered B operand, NACC TMEM accumulators);
//   warps 2-3   gather the item's query rows into the 128B-swizzled K-major B operand (cp.async)
//               and the per-pair metadata (trace row, d_i, group-minimum row);
//   warps 4-19  epilogue: tcgen05.ld (lane = slot, column = pair), D = d_i + P - 2 acc, padding
//               slots d_max, the whole trace row segment with coalesced stores
//               (32 lanes = 32 consecutive slots), and the minimum D of every 32-slot group.
// Step 5, lm_select_fast_kernel, one CTA per query: tau = the k-th smallest group
// minimum (>= the k-th smallest D: k distinct candidates reach it), then an exact radix selection
// of the k smallest (D, item) keys among the slots of the groups whose minimum is <= tau (read
// back from the trace), ties at the k-th distance resolved by item id (R10).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "tc_common.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

constexpr int kTile = 128;                              // slots per tile (UMMA M) = TMEM lanes
constexpr int kPanel = 128;                             // bytes of K per swizzled panel
constexpr uint32_t kAStageBytes = kTile * kPanel;       // 16 KB
constexpr int kEpiWarps = 16;                           // 4 per TMEM lane quadrant
constexpr int kChunk = 16;                              // accumulator columns per tcgen05.ld
constexpr int kNB = 3;                                  // B operand (query rows) buffers
constexpr int kWarpTma = 0, kWarpMma = 1, kWarpGat = 2, kNGat = 2, kWarpEpi = 4;
#ifndef V3DB_LM_STAGES
#define V3DB_LM_STAGES 6  // xhat tile stages of lm_kernel (fewer where shared memory is short)
#endif
constexpr int kIR = 8;                                  // item ring entries (lm_kernel's work-item sequence)
constexpr int kPre = 4;                                 // items published ahead of the one being loaded
constexpr int kThreads = 32 * (kWarpEpi + kEpiWarps);  // 640
constexpr uint32_t kFull = 0xffffffffu;
// staging row of one column (32 slots): 36 words -- the 32 lanes' stores hit distinct banks and the
// 16-byte reads of the group-minimum pass (two lanes per column) are conflict-free
constexpr int kStageRow = 36;
constexpr uint32_t kStageBytes = kEpiWarps * kChunk * kStageRow * 4u;

struct LmArgs {
  int nprobe, L, Lp, dim, kp, NT, nacc, lg_nacc, S, nb, ngroups;
  const int8_t* queries;
  const int32_t* pairs;   // pair ids (q * nprobe + rho) grouped by list
  const int4* items;      // (list, first pair, pairs, valid slots of the list)
  const int* n_items;
  int* next_item;         // work counter (zeroed by the grouping), or NULL: static round-robin
  const int32_t* ldist;   // [nq * nprobe] d_i of each pair
  const int32_t* counts;  // [nlist]
  const int32_t* pterm;   // [nlist][L]
  int32_t* trace;         // [nq][nprobe][L]
  int32_t* gmin;          // [nq][nprobe][ngroups]
  uint32_t off_b, off_meta, off_sd, off_p, off_stage, off_bar, b_bytes;
  int p_stride;  // ints per P buffer (L rounded up to 4)
  int bulk;      // L % 4 == 0: the trace leaves through the staged 16-byte stores
};

struct PairMeta {     // 16 B, read by the epilogue as one broadcast LDS.128
  uint64_t row;       // address of the pair's trace row: trace + pair * L
  int d;              // d_i
  int goff;           // pair * ngroups
};

// Slots per group of the group minima (the unit Step 5 selects candidates by): 32 = a warp's
// slots of a tile (measured against 16: C4 select 0.447 vs 0.478 ms, C3 0.115 vs 0.099).
constexpr int kG = 32;
static_assert(kG == 32, "group = the 32 slots (TMEM lanes) of one warp");
__device__ __forceinline__ int mc_goff(const PairMeta* mt, int jc, int col) { return mt[jc * 16 + col].goff; }
__device__ __forceinline__ void bulk_g2s_lm(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// Minimum over each group of kG lanes (32: the warp; 16: each half) of each of 16 columns
// x[0..15] (x is consumed): a butterfly in which each exchange halves the columns a lane keeps;
// lane l returns the minimum of column colmin_col(l) over its group (for kG = 32, lanes l and l ^ 1
// hold the same column).
__device__ __forceinline__ int colmin16(int (&x)[16], int lane) {
  constexpr int top = kG == 32 ? 16 : 8;
#pragma unroll
  for (int st = 0; st < 4; ++st) {
    const int half = 8 >> st, bit = top >> st;
    const bool up = lane & bit;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const int snd = up ? x[i] : x[i + half];
      const int kp = up ? x[i + half] : x[i];
      x[i] = min(kp, __shfl_xor_sync(0xffffffffu, snd, bit));
    }
  }
  if constexpr (kG == 32) return min(x[0], __shfl_xor_sync(0xffffffffu, x[0], 1));
  return x[0];
}
__device__ __forceinline__ int colmin_col(int lane) {
  if constexpr (kG == 32) return lane >> 1 & 15;  // bits 4..1 of the lane
  return lane & 15;
}

// ----------------------------------------------------------------------------------------------
// The contraction + epilogue kernel.
// ----------------------------------------------------------------------------------------------
#ifdef LM_EXP_TIMES  // experiment build: per-CTA start / end times of lm_kernel (tools/lm_times.py)
__device__ unsigned long long g_lm_times[2 * 256];
__device__ __forceinline__ unsigned long long lm_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
__global__ void __launch_bounds__(kThreads, 1) lm_kernel(const __grid_constant__ CUtensorMap tmX, const LmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef LM_EXP_TIMES
  if (threadIdx.x == 0) g_lm_times[2 * blockIdx.x] = lm_now();
#endif
  // 1024-byte alignment by pointer arithmetic on the shared array (an integer round trip would
  // make every access through `smem` a generic-address LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                         // [S][128 x 128 B]
  uint8_t* sB = smem + a.off_b;                               // [nb][kp][NT x 128 B]
  PairMeta* meta = reinterpret_cast<PairMeta*>(smem + a.off_meta);  // [nb][NT]
  int* sd = reinterpret_cast<int*>(smem + a.off_sd);         // [nb][NT] d_i of each pair
  int* sP = reinterpret_cast<int*>(smem + a.off_p);          // [nb][p_stride] P terms of the item's list
  int* stage = reinterpret_cast<int*>(smem + a.off_stage);   // [kEpiWarps][2][kChunk][kStageRow]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* afull = bars;                  // [S]
  uint64_t* aempty = afull + a.S;          // [S]
  uint64_t* bfull = aempty + a.S;          // [kNB]
  uint64_t* bempty = bfull + kNB;          // [kNB]
  uint64_t* accf = bempty + kNB;           // [nacc]
  uint64_t* acce = accf + a.nacc;          // [nacc]
  uint64_t* ifull = acce + a.nacc;         // [kIR]
  uint64_t* iempty = ifull + kIR;          // [kIR]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iempty + kIR);
  // The CTA's work-item sequence.  The TMA thread draws the items -- from the grid-wide counter
  // next_item (a CTA takes its next item when it is ready for one: the static round-robin deal left
  // the last CTA 5-20 % behind the mean, tools/lm_times.py) or, without a counter, round-robin -- and
  // publishes each item (pairs < 0: no more items) through this ring, kPre items ahead of the one
  // it is loading (the gather works ahead of the loads); every other role reads the sequence from
  // here, so all roles of the CTA see the same items in the same order.
  int4* ring = reinterpret_cast<int4*>(
      smem + ((a.off_bar + 8u * (2 * a.S + 2 * kNB + 2 * a.nacc + 2 * kIR) + 16u + 15u) & ~15u));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = *a.n_items;
  const int NT = a.NT, L = a.L;

  if (tid == 0) {
    for (int s = 0; s < a.S; ++s) {
      tc::mbar_init(afull + s, 1);
      tc::mbar_init(aempty + s, 1);
    }
    for (int r = 0; r < kIR; ++r) {
      tc::mbar_init(ifull + r, 1);
      tc::mbar_init(iempty + r, 1 + kNGat + kEpiWarps);  // MMA thread, gather warps, epilogue warps
    }
    for (int b = 0; b < kNB; ++b) {
      tc::mbar_init(bfull + b, kNGat);
      tc::mbar_init(bempty + b, 1 + kEpiWarps);
    }
    for (int c = 0; c < a.nacc; ++c) {
      tc::mbar_init(accf + c, 1);
      tc::mbar_init(acce + c, kEpiWarps / 2);  // one epilogue group drains an accumulator
    }
    tc::mbar_fence_init();
  }
  if (warp == kWarpMma) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpTma) {
    // ------------------------------------------------------------ xhat tiles (TMA)
    if (lane == 0) {
      tc::tma_prefetch(&tmX);
      int s = 0, u = 0;
      // The first kPre items of a CTA are dealt round-robin (their loads in flight together), the
      // rest drawn from the counter; each draw's atomic is issued one draw early.
      const int G = static_cast<int>(gridDim.x);
      int4 pre[kPre];
#pragma unroll
      for (int d = 0; d < kPre; ++d) {
        const int j = static_cast<int>(blockIdx.x) + d * G;
        pre[d] = j < n_items ? __ldg(a.items + j) : make_int4(0, 0, -1, 0);
      }
      int jn = a.next_item ? kPre * G + atomicAdd(a.next_item, 1) : static_cast<int>(blockIdx.x) + kPre * G;
      int ip = 0;  // items published
      bool done = false;
#pragma unroll
      for (int d = 0; d < kPre; ++d) {
        if (!done) {
          ring[d] = pre[d];
          tc::mbar_arrive(ifull + d);  // release: the entry is written
          done = pre[d].z < 0;
          ++ip;
        }
      }
      for (int il = 0;; ++il) {
        while (!done && ip < il + kPre) {
          const int r = ip & (kIR - 1), j = jn;
          if (ip >= kIR) tc::mbar_wait_sleep(iempty + r, (ip / kIR - 1) & 1);  // every reader is past entry ip - kIR
          done = j >= n_items;
          ring[r] = done ? make_int4(0, 0, -1, 0) : __ldg(a.items + j);
          tc::mbar_arrive(ifull + r);
          ++ip;
          if (!done) jn = a.next_item ? kPre * G + atomicAdd(a.next_item, 1) : j + G;
        }
        const int4 it = ring[il & (kIR - 1)];  // (this thread's own entry: not reused before entry il + kIR)
        if (it.z < 0) break;
        const int nvt = (it.w + kTile - 1) / kTile;
        for (int t = 0; t < nvt; ++t) {
          for (int p = 0; p < a.kp; ++p) {
            if (u > 0) tc::mbar_wait_sleep(aempty + s, (u - 1) & 1);
            tc::mbar_expect_tx(afull + s, kAStageBytes);
            tc::tma_load_2d(sA + s * kAStageBytes, &tmX, afull + s, p * kPanel, it.x * a.Lp + t * kTile);
            if (++s == a.S) {
              s = 0;
              ++u;
            }
          }
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int s = 0, u = 0, b = 0, bph = 0, tcount = 0;
      for (int i = 0;; ++i) {
        const int r = i & (kIR - 1);
        tc::mbar_wait_sleep(ifull + r, (i / kIR) & 1);
        const int4 it = ring[r];
        const int nvt = (it.w + kTile - 1) / kTile;
        tc::mbar_arrive(iempty + r);
        if (it.z < 0) break;
        const int N = (it.z + 15) & ~15;  // UMMA N for M = 128: multiple of 16
        const uint32_t idesc = tc::idesc_s8(kTile, N);
        tc::mbar_wait_sleep(bfull + b, bph);
        tc::fence_after_sync();
        const uint32_t b_addr = tc::smem_u32(sB + b * a.b_bytes);
        for (int t = 0; t < nvt; ++t, ++tcount) {
          const int acc = tcount & (a.nacc - 1), ua = tcount >> a.lg_nacc;
          if (ua > 0) {
            tc::mbar_wait_sleep(acce + acc, (ua - 1) & 1);
            tc::fence_after_sync();
          }
          for (int p = 0; p < a.kp; ++p) {
            tc::mbar_wait_sleep(afull + s, u & 1);
            tc::fence_after_sync();
            const int nk = min(4, (a.dim - p * kPanel + 31) / 32);
            const uint32_t a_addr = tc::smem_u32(sA + s * kAStageBytes);
            const uint32_t bp = b_addr + p * NT * kPanel;
            for (int kk = 0; kk < nk; ++kk)
              tc::mma_s8(tmem + acc * NT, tc::desc_sw128(a_addr + kk * 32), tc::desc_sw128(bp + kk * 32), idesc,
                         (p | kk) != 0);
            tc::mma_commit(aempty + s);
            if (++s == a.S) {
              s = 0;
              ++u;
            }
          }
          tc::mma_commit(accf + acc);
        }
        tc::mma_commit(bempty + b);  // the B buffer is free once this item's MMAs completed
        if (++b == a.nb) {
          b = 0;
          bph ^= 1;
        }
      }
    }
  } else if (warp < kWarpEpi) {
    // ------------------------------------------------------------ gather: B operand + metadata
    const int gt = tid - kWarpGat * 32;  // 0 .. 63
    const int cpr = a.dim >> 4;          // 16-byte chunks per query row
    int b = 0, use = 0;  // buffer, times the ring wrapped
    for (int i = 0;; ++i) {
      const int ri = i & (kIR - 1);
      tc::mbar_wait_sleep(ifull + ri, (i / kIR) & 1);
      const int4 it = ring[ri];
      const int cnt = it.w;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(iempty + ri);
      if (it.z < 0) break;
      if (use > 0) tc::mbar_wait_sleep(bempty + b, (use - 1) & 1);
      uint8_t* dst = sB + b * a.b_bytes;
      PairMeta* mt = meta + b * NT;
      {  // the P terms of the list's valid slots: one bulk copy completing on the item's barrier
        if (gt == 0 && a.p_stride && cnt > 0) {
          const uint32_t pbytes = 16u * ((cnt + 3) / 4);
          tc::mbar_expect_tx_only(bfull + b, pbytes);
          bulk_g2s_lm(sP + b * a.p_stride, a.pterm + static_cast<int64_t>(it.x) * L, pbytes, bfull + b);
        }
      }
      // per pair: metadata, d_i, and the query row (cp.async into the swizzled B operand)
      for (int r = gt; r < it.z; r += 32 * kNGat) {
        const int pr = __ldg(a.pairs + it.y + r);
        const int dl = __ldg(a.ldist + pr);
        const int q = pr / a.nprobe;
        mt[r] = PairMeta{reinterpret_cast<uint64_t>(a.trace + static_cast<int64_t>(pr) * L), dl, pr * a.ngroups};
        sd[b * NT + r] = dl;
        const int8_t* qrow = a.queries + static_cast<int64_t>(q) * a.dim;
        for (int c = 0; c < cpr; ++c)
          tc::cp_async16(dst + (c >> 3) * NT * kPanel + tc::sw128_offset(r, c & 7), qrow + c * 16, 16);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bfull + b);
      if (++b == a.nb) {
        b = 0;
        ++use;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Two groups of 8 warps take alternate tiles (two tiles drain at once).  Within a group, warp:
    // TMEM lane quadrant qd (its 32 slots of the tile) and column group cg (chunks of 16 columns
    // cg, cg + 2, ...).  Thread = one slot; per column (pair) D = d_i + P - 2 acc (padding slots
    // d_max).  Staged path (L % 4 == 0): the warp writes its 32 x 16 block of D to shared memory,
    // two lanes per column take the 32-slot group minimum from there and eight lanes per column
    // store the column's 128 trace bytes with 16-byte stores.  Otherwise the lanes store the trace
    // directly and the minimum is a lane butterfly.
    const int e = warp - kWarpEpi, qd = warp & 3, grp = e >> 3, cg = (e >> 2) & 1;
    constexpr int NCG = 2;
    int* stg = stage + e * (kChunk * kStageRow);
    int b = 0, bph = 0, tcount = 0, tall = 0;
    for (int i = 0;; ++i) {
      const int ri = i & (kIR - 1);
      tc::mbar_wait_sleep(ifull + ri, (i / kIR) & 1);
      const int4 it = ring[ri];
      const int cnt = it.w;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(iempty + ri);
      if (it.z < 0) break;
      const int np = it.z;
      const int nvt = (cnt + kTile - 1) / kTile, ntl = (L + kTile - 1) / kTile;
      const PairMeta* mt = meta + b * NT;
      const int* dcol = sd + b * NT;
      const int* pP = sP + b * a.p_stride;
      tc::mbar_wait_sleep(bfull + b, bph);
      for (int t = 0; t < ntl; ++t, ++tall) {
        const bool mine = (tall & 1) == grp;
        const int sbase = t * kTile + qd * 32, slot = sbase + lane;
        const uint64_t toff = 4ull * static_cast<uint32_t>(slot);
        if (t < nvt) {
          // a valid tile goes to group (tile count) mod 2 and accumulator (tile count) mod nacc, nacc
          // even: each group owns its accumulators and waits on every phase of their barriers (a
          // group that skipped a phase would misread the parity -- assigning by the running count of
          // all tiles, padding-only ones included, did that)
          const int acc = tcount & (a.nacc - 1), ua = tcount >> a.lg_nacc;
          const bool own = (tcount & 1) == grp;
          ++tcount;
          if (!own) continue;
          const bool valid = slot < cnt;
          const int32_t P = !valid ? 0 : a.p_stride ? pP[slot] : __ldg(a.pterm + static_cast<int64_t>(it.x) * L + slot);
          const bool full = sbase + 32 <= cnt;                // warp-uniform: every slot valid (< L)
          const int nsl = min(32, L - sbase);                 // slots of this group inside the row
          tc::mbar_wait_sleep(accf + acc, ua & 1);
          tc::fence_after_sync();
          // D of one chunk of 16 columns into x[] (d_max for padding slots and absent columns)
          auto dvals = [&](const uint32_t(&v)[kChunk], int jc, int (&x)[kChunk], int ncol) {
            const int4* d4 = reinterpret_cast<const int4*>(dcol + jc * kChunk);
            int dv[kChunk];
#pragma unroll
            for (int c4 = 0; c4 < kChunk / 4; ++c4) {
              const int4 w = d4[c4];
              dv[4 * c4] = w.x, dv[4 * c4 + 1] = w.y, dv[4 * c4 + 2] = w.z, dv[4 * c4 + 3] = w.w;
            }
            if (full && ncol == kChunk) {
#pragma unroll
              for (int c = 0; c < kChunk; ++c) x[c] = dv[c] + P - 2 * static_cast<int32_t>(v[c]);
            } else {
#pragma unroll
              for (int c = 0; c < kChunk; ++c)
                x[c] = valid && c < ncol ? dv[c] + P - 2 * static_cast<int32_t>(v[c]) : kDMax;
            }
          };
          // staged path: the 32 x 16 block of D through shared memory -- two lanes per column take
          // the 32-slot group minimum, eight lanes per column store its 128 trace bytes (16 B each)
          auto chunk_stage = [&](const uint32_t(&v)[kChunk], int jc) {
            const int ncol = min(kChunk, np - jc * kChunk);
            int x[kChunk];
            dvals(v, jc, x, ncol);
            __syncwarp();  // the previous chunk's reads of the stage are done
#pragma unroll
            for (int c = 0; c < kChunk; ++c) stg[c * kStageRow + lane] = x[c];
            __syncwarp();
            const int col = lane >> 1;
            const int4* r4 = reinterpret_cast<const int4*>(stg + col * kStageRow + (lane & 1) * 16);
            int m = kDMax;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int4 w = r4[u];
              m = min(m, min(min(w.x, w.y), min(w.z, w.w)));
            }
            m = min(m, __shfl_xor_sync(kFull, m, 1));
            if (!(lane & 1) && col < ncol) a.gmin[mc_goff(mt, jc, col) + t * 4 + qd] = m;
            const int pp = lane & 7;
            if (4 * pp < nsl) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int c = (lane >> 3) + 4 * i;
                if (c < ncol) {
                  const int4 w = *reinterpret_cast<const int4*>(stg + c * kStageRow + 4 * pp);
                  __stcs(reinterpret_cast<int4*>(mt[jc * kChunk + c].row + 4ull * static_cast<uint32_t>(sbase + 4 * pp)), w);
                }
              }
            }
          };
          // direct path: lanes store the trace, butterfly minima
          auto chunk_direct = [&](const uint32_t(&v)[kChunk], int jc) {
            const PairMeta* mc = mt + jc * kChunk;
            const int ncol = min(kChunk, np - jc * kChunk);
            int x[kChunk];
            dvals(v, jc, x, ncol);
#pragma unroll
            for (int c = 0; c < kChunk; ++c)
              if (c < ncol && slot < L) __stcs(reinterpret_cast<int32_t*>(mc[c].row + toff), x[c]);
            const int gm = colmin16(x, lane), col = colmin_col(lane);
            if (!(lane & 1) && col < ncol) a.gmin[mc[col].goff + t * 4 + qd] = gm;
          };
          // two chunks per round: both TMEM loads in flight before the first is used
          const uint32_t tbase = tmem + (static_cast<uint32_t>(qd * 32) << 16) + acc * NT;
          // (a warp whose 32 slots lie past the row end -- L not a multiple of 128 -- has nothing)
          for (int jc = cg; sbase < L && jc * kChunk < np; jc += 2 * NCG) {
            const int jd = jc + NCG;
            const bool two = jd * kChunk < np;  // warp-uniform
            uint32_t v0[kChunk], v1[kChunk];
            tc::tmem_ld16(tbase + jc * kChunk, v0);
            if (two) tc::tmem_ld16(tbase + jd * kChunk, v1);
            tc::tmem_ld_wait();
            if (a.bulk) {
              chunk_stage(v0, jc);
              if (two) chunk_stage(v1, jd);
            } else {
              chunk_direct(v0, jc);
              if (two) chunk_direct(v1, jd);
            }
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(acce + acc);
        } else if (mine && slot < L) {
          // a tile of padding only: D = d_max, nothing read
          for (int c = cg; c < np; c += NCG) {
            __stcs(reinterpret_cast<int32_t*>(mt[c].row + toff), kDMax);
            if (lane == 0) a.gmin[mt[c].goff + t * 4 + qd] = kDMax;  // group sentinel
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bempty + b);
      if (++b == a.nb) {
        b = 0;
        bph ^= 1;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
#ifdef LM_EXP_TIMES
  if (threadIdx.x == 0) g_lm_times[2 * blockIdx.x + 1] = lm_now();
#endif
  if (warp == kWarpMma) tc::tmem_dealloc(tmem, 512);
}

// ----------------------------------------------------------------------------------------------
// Grouping: the (query, rank) pairs by probed list, and the work items.
// ----------------------------------------------------------------------------------------------
__global__ void pair_hist_kernel(const int32_t* __restrict__ lists, int64_t npairs, int* __restrict__ hist) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < npairs;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(hist + __ldg(lists + p), 1);
}

// cur[i] = exclusive prefix of hist (the list's first pair in list order, advanced by the pair
// scatter), the work items (list, first pair, pairs <= NT, valid slots of the list) of every list in
// list order, n_items[0] = their number and n_items[1] = 0 (the main kernel's work counter).  One CTA of 1024 threads per 1024 lists (a cooperative launch, <= 32 CTAs): a block scan,
// the CTA totals exchanged through agg[] across one grid barrier, then contiguous cur / item stores.
// (One CTA for every list spent ~31 us at C4 on its dependent scan chains at ~1 IPC.)
__device__ __forceinline__ int2 warp_incl_scan2(int2 v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v.x, o), z = __shfl_up_sync(0xffffffffu, v.y, o);
    if (lane >= o) {
      v.x += y;
      v.y += z;
    }
  }
  return v;
}
__global__ void __launch_bounds__(1024) lm_scan_items_kernel(const int* __restrict__ hist,
                                                             const int32_t* __restrict__ counts, int nlist, int NT,
                                                             int* __restrict__ cur, int4* __restrict__ items,
                                                             int* __restrict__ n_items, int2* __restrict__ agg) {
  __shared__ int2 wt[32];
  __shared__ int2 base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, i = (blockIdx.x << 10) + tid;
  const int h = i < nlist ? __ldg(hist + i) : 0, ni = (h + NT - 1) / NT;
  const int2 inc = warp_incl_scan2(make_int2(h, ni), lane);
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int2 v = wt[lane];
    const int2 wi = warp_incl_scan2(v, lane);
    wt[lane] = make_int2(wi.x - v.x, wi.y - v.y);
    if (lane == 31) agg[blockIdx.x] = wi;  // this CTA's totals
  }
  __threadfence();
  cooperative_groups::this_grid().sync();
  if (warp == 0) {  // the totals of the CTAs before this one
    int2 v = lane < static_cast<int>(blockIdx.x) ? agg[lane] : make_int2(0, 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    if (lane == 0) {
      base = v;
      if (blockIdx.x == gridDim.x - 1) {
        n_items[0] = v.y + agg[blockIdx.x].y;
        n_items[1] = 0;  // lm_kernel's work counter
      }
    }
  }
  __syncthreads();
  if (i < nlist) {
    const int run = base.x + wt[warp].x + inc.x - h;
    int irun = base.y + wt[warp].y + inc.y - ni;
    cur[i] = run;
    const int cnt = ni > 0 ? __ldg(counts + i) : 0;
    for (int q = 0; q < ni; ++q) items[irun++] = make_int4(i, run + q * NT, min(NT, h - q * NT), cnt);
  }
}
cudaError_t launch_scan_items(const int* hist, const int32_t* counts, int nlist, int NT, int* cur, int4* items,
                              int* n_items, int2* agg, cudaStream_t st) {
  const unsigned g = static_cast<unsigned>(std::max(1, (nlist + 1023) >> 10));  // <= 32 (nlist <= 32768)
  void* args[] = {&hist, &counts, &nlist, &NT, &cur, &items, &n_items, &agg};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lm_scan_items_kernel), dim3(g), dim3(1024), args, 0,
                                     st);
}

// The pair ids grouped by list: pairs[cur[list]++] = p (the order inside a list is free: every pair
// has its own trace row and group minima).  Each thread takes kScatPer pairs with all their atomics
// in flight at once (one latency per thread, not one per pair).
constexpr int kScatPer = 8;
__global__ void __launch_bounds__(256) pair_scatter_kernel(const int32_t* __restrict__ lists, int64_t npairs,
                                                           int* __restrict__ cur, int32_t* __restrict__ pairs) {
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 256 * kScatPer + threadIdx.x;
  int l[kScatPer], pos[kScatPer];
#pragma unroll
  for (int u = 0; u < kScatPer; ++u) {
    const int64_t p = p0 + 256 * u;
    l[u] = p < npairs ? __ldg(lists + p) : -1;
  }
#pragma unroll
  for (int u = 0; u < kScatPer; ++u) pos[u] = l[u] >= 0 ? atomicAdd(cur + l[u], 1) : 0;
#pragma unroll
  for (int u = 0; u < kScatPer; ++u)
    if (l[u] >= 0) pairs[pos[u]] = static_cast<int32_t>(p0 + 256 * u);
}
// The same for few lists (nlist <= kScatSmemLists), where many pairs share a list and the global
// atomics on one counter serialise (C1: 312 pairs per list): the CTA's kScatPer * 256 pairs are
// counted per list in shared memory, each list touched reserves its range with ONE global atomic,
// and the pairs are placed from there.
constexpr int kScatSmemLists = 8192;
__global__ void __launch_bounds__(256) pair_scatter_smem_kernel(const int32_t* __restrict__ lists, int64_t npairs,
                                                                int nlist, int* __restrict__ cur,
                                                                int32_t* __restrict__ pairs) {
  extern __shared__ int cnt[];  // [nlist]: counts, then each list's global base
  for (int i = threadIdx.x; i < nlist; i += 256) cnt[i] = 0;
  __syncthreads();
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 256 * kScatPer + threadIdx.x;
  int l[kScatPer], pos[kScatPer];
#pragma unroll
  for (int u = 0; u < kScatPer; ++u) {
    const int64_t p = p0 + 256 * u;
    l[u] = p < npairs ? __ldg(lists + p) : -1;
  }
#pragma unroll
  for (int u = 0; u < kScatPer; ++u) pos[u] = l[u] >= 0 ? atomicAdd(cnt + l[u], 1) : 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nlist; i += 256)
    if (cnt[i]) cnt[i] = atomicAdd(cur + i, cnt[i]);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kScatPer; ++u)
    if (l[u] >= 0) pairs[cnt[l[u]] + pos[u]] = static_cast<int32_t>(p0 + 256 * u);
}
cudaError_t launch_pair_scatter(const int32_t* lists, int64_t npairs, int nlist, int* cur, int32_t* pairs,
                                cudaStream_t st) {
  const unsigned g = static_cast<unsigned>((npairs + 256 * kScatPer - 1) / (256 * kScatPer));
  if (g == 0) return cudaSuccess;
  if (nlist <= kScatSmemLists) {
    const int sm = static_cast<int>(sizeof(int) * nlist);
    cudaError_t e = cudaFuncSetAttribute(pair_scatter_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    pair_scatter_smem_kernel<<<g, 256, sm, st>>>(lists, npairs, nlist, cur, pairs);
  } else {
    pair_scatter_kernel<<<g, 256, 0, st>>>(lists, npairs, cur, pairs);
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// Step 5: exact per-query selection from the group minima and the trace.
// ----------------------------------------------------------------------------------------------
constexpr int kSelThreads = 256;
constexpr int kWarpProbeCap = 128;  // largest nprobe of the cached selection path
constexpr int kSelGroups = 4096;  // selected-group list capacity (more: every valid group is scanned)

// Distance types of Step 5: int32 (BASELINE.json's int8 path) and int64 (the paper's 16-bit fixed
// point, NEXT-1).  U = the unsigned domain of the histograms / radix digits (every valid D >= 0);
// Key = the total (D, item) order of R10 (item as signed int32: key id ^ 0x80000000).
struct KeyFx {
  int64_t d;
  uint32_t id;  // item ^ 0x80000000
};
template <class T>
struct DistT;
template <>
struct DistT<int32_t> {
  using U = uint32_t;
  using Key = uint64_t;
  static constexpr int32_t kMax = 0x7fffffff;
  __device__ static Key key(int32_t d, int32_t id) { return step5_key(d, id); }
  __device__ static int32_t id(Key k) { return step5_id(k); }
  __device__ static int32_t dist(Key k) { return static_cast<int32_t>(k >> 32); }
  __device__ static bool less(Key a, Key b) { return a < b; }
  __device__ static int bitlen(U x) { return 32 - __clz(x | 1u); }
};
template <>
struct DistT<int64_t> {
  using U = uint64_t;
  using Key = KeyFx;
  static constexpr int64_t kMax = 0x7fffffffffffffffLL;
  __device__ static Key key(int64_t d, int32_t id) { return KeyFx{d, static_cast<uint32_t>(id) ^ 0x80000000u}; }
  __device__ static int32_t id(Key k) { return static_cast<int32_t>(k.id ^ 0x80000000u); }
  __device__ static int64_t dist(Key k) { return k.d; }
  __device__ static bool less(Key a, Key b) { return a.d < b.d || (a.d == b.d && a.id < b.id); }
  __device__ static int bitlen(U x) { return 64 - __clzll(static_cast<long long>(x | 1ull)); }
};

template <class T>
struct SelArgs {
  int nprobe, L, ngroups, k;
  const int32_t* lists;
  const int32_t* counts;
  const int32_t* ids;
  const T* trace;
  const T* gmin;
  int32_t* out_ids;
  T* out_dist;
};

// CTA-wide radix selection (8-bit digits) of the kk-th smallest (1-based) value among those
// `gen(i, &v)` yields for i in [0, n); every value is known to be <= bound, so the leading digits
// above bound's top bit are skipped.  Returns the value; *below = how many yielded values are smaller.
template <class U, class Gen>
__device__ U cta_radix_select(int n, int kk, U bound, Gen gen, int* hist, int* sc, int* below) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int ND = sizeof(U);
  const int top = sizeof(U) == 8 ? 64 - __clzll(static_cast<long long>(bound | 1)) : 32 - __clz(static_cast<uint32_t>(bound | 1));
  const int pass0 = ND - 1 - (top - 1) / 8;
  U prefix = 0;
  const int k0 = kk;
  for (int pass = pass0; pass < ND; ++pass) {
    const int shift = 8 * (ND - 1 - pass);
    for (int x = tid; x < 256; x += kSelThreads) hist[x] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kSelThreads) {
      U v;
      if (gen(i, v) && (pass == pass0 || (v >> (shift + 8)) == prefix)) atomicAdd(hist + static_cast<int>((v >> shift) & 255), 1);
    }
    __syncthreads();
    if (warp == 0) {
      int h[8], sum = 0;
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        h[x] = hist[lane * 8 + x];
        sum += h[x];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int w = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += w;
      }
      int cum = incl - sum;
      if (cum < kk && kk <= incl) {
        int bin = lane * 8;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          if (cum + h[x] >= kk) break;
          cum += h[x];
          ++bin;
        }
        sc[0] = bin;
        sc[1] = kk - cum;
      }
    }
    __syncthreads();
    prefix = (prefix << 8) | static_cast<U>(sc[0]);
    kk = sc[1];
    __syncthreads();
  }
  *below = k0 - kk;
  return prefix;
}

// Streaming selection (no per-query capacity limit): every pass re-reads the group minima and the
// candidates' distances from global memory.  Used for the queries the cached path cannot hold.
template <class T>
__device__ void select_streaming(const SelArgs<T>& a, int64_t q, uint8_t* sm) {
  using Tr = DistT<T>;
  using U = typename Tr::U;
  using Key = typename Tr::Key;
  int* pl = reinterpret_cast<int*>(sm);            // [nprobe] probed list
  int* pc = pl + a.nprobe;                         // [nprobe] its count
  int* hist = pc + a.nprobe;                       // [256]
  int* sc = hist + 256;                            // [16] scratch
  int* sel = sc + 16;                              // [kSelGroups] selected groups (rho << 16 | g)
  Key* keys = reinterpret_cast<Key*>(sel + kSelGroups);  // [k]
  const int tid = threadIdx.x;
  const int nprobe = a.nprobe, L = a.L, NG = a.ngroups, k = a.k;
  const U tau_all = static_cast<U>(Tr::kMax) - 1;  // every valid D (< d_max)
  __syncthreads();  // the caller may have used the same shared memory
  for (int r = tid; r < nprobe; r += kSelThreads) {
    const int li = a.lists[q * nprobe + r];
    pl[r] = li;
    pc[r] = __ldg(a.counts + li);
  }
  if (tid < 16) sc[tid] = 0;
  __syncthreads();
  const T* gq = a.gmin + q * nprobe * NG;
  const T* tq = a.trace + q * nprobe * static_cast<int64_t>(L);
  // valid groups: (rho, g) with kG g < count_rho
  auto gen_g = [&](int i, U& v) {
    const int rho = i / NG, g = i - rho * NG;
    if (kG * g >= pc[rho]) return false;
    v = static_cast<U>(gq[i]);
    return true;
  };
  {
    int nvalid_g = 0;
    for (int r = tid; r < nprobe; r += kSelThreads) nvalid_g += (pc[r] + kG - 1) / kG;
    if (nvalid_g) atomicAdd(sc + 2, nvalid_g);
  }
  __syncthreads();
  const int V = sc[2];
  int below = 0;
  // tau = the k-th smallest group minimum (each is a real candidate's D), or "everything" if fewer
  // than k valid groups exist
  const U tau = V >= k ? cta_radix_select<U>(nprobe * NG, k, tau_all, gen_g, hist, sc, &below) : tau_all;
  // the selected groups (minimum <= tau)
  if (tid == 0) {
    sc[3] = 0;
    sc[4] = 0;
  }
  __syncthreads();
  for (int i = tid; i < nprobe * NG; i += kSelThreads) {
    U v;
    if (gen_g(i, v) && v <= tau) {
      const int rho = i / NG, g = i - rho * NG;
      const int pos = atomicAdd(sc + 3, 1);
      if (pos < kSelGroups) sel[pos] = (rho << 16) | g;
    }
  }
  __syncthreads();
  const int nsel = sc[3];
  const bool all = nsel > kSelGroups || nprobe > 65535 || NG > 65535;  // fall back to every valid group
  const int total_slots = all ? nprobe * NG * kG : nsel * kG;
  // candidate i: slot i % kG of selected group i / kG (or of group i / kG of the query)
  auto slot_of = [&](int i, int& rho, int& j) {
    const int gi = i / kG;
    int g;
    if (all) {
      rho = gi / NG;
      g = gi - rho * NG;
    } else {
      const int sg = sel[gi];
      rho = sg >> 16;
      g = sg & 0xffff;
    }
    j = kG * g + i % kG;
    return j < pc[rho];
  };
  auto gen_d = [&](int i, U& v) {
    int rho, j;
    if (!slot_of(i, rho, j)) return false;
    v = static_cast<U>(tq[rho * static_cast<int64_t>(L) + j]);
    return v <= tau;
  };
  // how many candidates (valid, D <= tau) exist
  if (tid == 0) sc[5] = 0;
  __syncthreads();
  {
    int c = 0;
    for (int i = tid; i < total_slots; i += kSelThreads) {
      U v;
      c += gen_d(i, v) ? 1 : 0;
    }
    atomicAdd(sc + 5, c);
  }
  __syncthreads();
  const int ncand = sc[5];
  const int kk = min(k, ncand);
  U dk = ~U(0);
  uint32_t idk = 0xffffffffu;
  if (ncand > k) {
    // the k-th smallest D; then, if the ties at it do not all fit, the (k - below)-th smallest item
    // key among them (R10: (D, id) order, id as signed int32 -> key id ^ 0x80000000)
    dk = cta_radix_select<U>(total_slots, k, tau, gen_d, hist, sc, &below);
    const int need = k - below;
    if (tid == 0) sc[6] = 0;
    __syncthreads();
    {
      int c = 0;
      for (int i = tid; i < total_slots; i += kSelThreads) {
        U v;
        c += (gen_d(i, v) && v == dk) ? 1 : 0;
      }
      atomicAdd(sc + 6, c);
    }
    __syncthreads();
    if (sc[6] > need) {
      auto gen_id = [&](int i, uint32_t& v) {
        int rho, j;
        if (!slot_of(i, rho, j)) return false;
        if (static_cast<U>(tq[rho * static_cast<int64_t>(L) + j]) != dk) return false;
        v = static_cast<uint32_t>(__ldg(a.ids + static_cast<int64_t>(pl[rho]) * L + j)) ^ 0x80000000u;
        return true;
      };
      int b2 = 0;
      idk = cta_radix_select<uint32_t>(total_slots, need, 0xffffffffu, gen_id, hist, sc, &b2);
    }
  }
  // collect the min(k, ncand) winners as resolved (D, item) keys, then place them by rank
  if (tid == 0) sc[7] = 0;
  __syncthreads();
  for (int i = tid; i < total_slots; i += kSelThreads) {
    U v;
    if (!gen_d(i, v) || v > dk) continue;
    int rho, j;
    slot_of(i, rho, j);
    const int32_t id = __ldg(a.ids + static_cast<int64_t>(pl[rho]) * L + j);
    if (v == dk && (static_cast<uint32_t>(id) ^ 0x80000000u) > idk) continue;
    const int pos = atomicAdd(sc + 7, 1);
    V3DB_DCHECK(pos < kk);
    keys[pos] = Tr::key(static_cast<T>(v), id);
  }
  __syncthreads();
  const int m = sc[7];
  for (int e2 = tid; e2 < m; e2 += kSelThreads) {
    const Key key = keys[e2];
    int rank = 0;
    for (int f = 0; f < m; ++f) rank += Tr::less(keys[f], key) ? 1 : 0;
    a.out_ids[q * k + rank] = Tr::id(key);
    a.out_dist[q * k + rank] = Tr::dist(key);
  }
  for (int r = m + tid; r < k; r += kSelThreads) {  // fewer than k valid candidates (R11)
    a.out_ids[q * k + r] = -1;
    a.out_dist[q * k + r] = Tr::kMax;
  }
}

// ---------------------------------------------------------------------------------------------
// Step 5, one CTA per query, small shared footprint (8 CTAs per SM for int32 distances):
//  1. the valid group minima are cached in shared memory; tau = the upper edge of a histogram bin
//     holding the k-th smallest one (>= it, hence >= the k-th smallest D: k distinct candidates
//     reach it);
//  2. the candidates -- the valid slots with D <= tau of the groups whose minimum is <= tau -- are
//     read from the trace ONCE, a warp per group (lane = slot: one 128-byte load), and compacted
//     into shared memory as (D - dmin, rho, slot);
//  3. the k smallest (D, item) keys among them are exact: 256-bin histograms of D - dmin over a
//     shrinking window of the compacted candidates; candidates below the window's target bin win
//     outright, the target bin is refined until it holds <= kBinCap entries, which are ranked on
//     their full (D, item) keys (R10).
// Queries beyond the caches (kSelGcap valid groups, kCandCap candidates, or more than kBinCap
// candidates tied at one distance) take the streaming path.
// ---------------------------------------------------------------------------------------------
constexpr int kSelGcap = 2048;     // cached group minima per query
constexpr int kCandCap = 2048;     // compacted candidates per query
constexpr int kSelKmax = 256;      // largest k of the cached path
constexpr int kBinCap = 256;       // entries of the final histogram bin ranked pairwise
#ifndef V3DB_SW_H
#define V3DB_SW_H 4
#endif
#ifndef V3DB_FAST_MINB
#define V3DB_FAST_MINB 6
#endif
constexpr int kSwH = V3DB_SW_H;    // selected groups per lane octet and candidate step (loads in flight)
constexpr int kFastMinBlocks = V3DB_FAST_MINB;  // lm_select_fast_kernel CTAs per SM (40 registers)
static_assert(kG == 32, "the candidate gather maps a group's slots to the lanes of a warp");

template <class T>
struct SelSmem {
  using U = typename DistT<T>::U;
  using Key = typename DistT<T>::Key;
  U gv[kSelGcap];                  // valid group minima; then the candidates' D - dmin
  union {
    int gid[kSelGcap];             // rho << 16 | g, compacted to the selected groups
    struct {
      Key keys[kSelKmax];          // winners (after the gather: gid is dead)
      Key bin[kBinCap];            // final-bin entries
    } w;
  };
  int cf[kCandCap];                // candidate rho << 24 | slot
  int hist[256];
  int pl[kWarpProbeCap];           // probed lists
  int pc[kWarpProbeCap];           // their counts
  int pg[kWarpProbeCap + 1];       // valid-group prefix
  T mm[2];                         // the query's smallest / largest valid group minimum
  int sc[40];
};
static_assert(sizeof(int) * kSelGcap >= 2 * sizeof(DistT<int64_t>::Key) * kSelKmax, "winner arrays alias gid");

// Block-wide: the bin of hist[0, 256) holding rank kk (1-based); *before = entries below it,
// *inbin = its population.  256 threads; ends with a barrier.
__device__ __forceinline__ int cta_bin_of(int* hist, int* sc, int kk, int* before, int* inbin) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = hist[tid];
  int incl = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int w = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += w;
  }
  if (lane == 31) sc[24 + warp] = incl;
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) base += w < warp ? sc[24 + w] : 0;
  const int excl = base + incl - h;
  if (excl < kk && kk <= excl + h) {
    sc[0] = tid;
    sc[1] = excl;
    sc[2] = h;
  }
  __syncthreads();
  *before = sc[1];
  *inbin = sc[2];
  return sc[0];
}

// Hands query q to the streaming selection: flags[0] counts, flags[1..] lists.
__device__ __forceinline__ void flag_query(int* flags, int64_t q) { flags[1 + atomicAdd(flags, 1)] = static_cast<int>(q); }

template <class T>
__device__ __forceinline__ T warp_min(T v) {
  if constexpr (sizeof(T) == 4) {
    return __reduce_min_sync(kFull, v);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T w = __shfl_xor_sync(kFull, v, o);
      v = w < v ? w : v;
    }
    return v;
  }
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
  if constexpr (sizeof(T) == 4) {
    return __reduce_max_sync(kFull, v);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T w = __shfl_xor_sync(kFull, v, o);
      v = w > v ? w : v;
    }
    return v;
  }
}

template <class T>
__global__ void __launch_bounds__(kSelThreads, kFastMinBlocks) lm_select_fast_kernel(const SelArgs<T> a, int* __restrict__ flags) {
  using Tr = DistT<T>;
  using U = typename Tr::U;
  using Key = typename Tr::Key;
  __shared__ SelSmem<T> S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t q = blockIdx.x;
  const int nprobe = a.nprobe, L = a.L, NG = a.ngroups, k = a.k;
  const T* gq = a.gmin + q * nprobe * NG;
  const T* tq = a.trace + q * nprobe * static_cast<int64_t>(L);
  for (int r = tid; r < nprobe; r += kSelThreads) {
    const int li = a.lists[q * nprobe + r];
    S.pl[r] = li;
    S.pc[r] = __ldg(a.counts + li);
  }
  if (tid < 40) S.sc[tid] = 0;
  if (tid == 0) {
    S.mm[0] = Tr::kMax;
    S.mm[1] = 0;
  }
  __syncthreads();
  if (warp == 0) {  // prefix sums of the valid groups per probe
    int carry = 0;
    for (int r0 = 0; r0 < nprobe; r0 += 32) {
      const int r = r0 + lane;
      const int c = r < nprobe ? (S.pc[r] + kG - 1) / kG : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int w = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += w;
      }
      if (r < nprobe) S.pg[r] = carry + incl - c;
      carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) S.pg[nprobe] = carry;
  }
  __syncthreads();
  const int V = S.pg[nprobe];
  if (V > kSelGcap) {
    if (tid == 0) flag_query(flags, q);
    return;
  }
  // the valid group minima (8 loads in flight per thread), their minimum and maximum
  T mn = Tr::kMax, mx = 0;
  {
    const int tot = nprobe * NG;
    for (int i0 = tid; i0 < tot; i0 += 8 * kSelThreads) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kSelThreads;
        v[u] = i < tot ? gq[i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kSelThreads;
        if (i < tot) {
          const int r = i / NG, g = i - r * NG;
          if (kG * g < S.pc[r]) {
            const int pos = S.pg[r] + g;
            S.gv[pos] = static_cast<U>(v[u]);
            S.gid[pos] = (r << 16) | g;
            mn = v[u] < mn ? v[u] : mn;
            mx = v[u] > mx ? v[u] : mx;
          }
        }
      }
    }
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  if (lane == 0) {
    if constexpr (sizeof(T) == 4) {
      atomicMin(&S.mm[0], mn);
      atomicMax(&S.mm[1], mx);
    } else {
      atomicMin(reinterpret_cast<long long*>(&S.mm[0]), static_cast<long long>(mn));
      atomicMax(reinterpret_cast<long long*>(&S.mm[1]), static_cast<long long>(mx));
    }
  }
  __syncthreads();
  const U dmin = static_cast<U>(S.mm[0]);
  const U tmax = static_cast<U>(Tr::kMax) - 1 - dmin;  // relative bound of every valid D
  U tau = tmax;  // relative
  if (V >= k) {
    U w0 = 0, span = static_cast<U>(S.mm[1]) - dmin + 1;
    int need = k;
    for (;;) {
      const int bits = Tr::bitlen(span - 1);
      const int sh = bits > 8 ? bits - 8 : 0;
      S.hist[tid] = 0;
      __syncthreads();
      for (int i = tid; i < V; i += kSelThreads) {
        const U rel = S.gv[i] - dmin;
        if (rel >= w0 && rel - w0 < span) atomicAdd(S.hist + static_cast<int>((rel - w0) >> sh), 1);
      }
      __syncthreads();
      int before, inbin;
      const int b = cta_bin_of(S.hist, S.sc, need, &before, &inbin);
      w0 += static_cast<U>(b) << sh;
      span = U(1) << sh;
      need -= before;
      if (sh == 0 || inbin <= 8) break;  // a bin of <= 8 group minima: tight enough
    }
    tau = w0 + span - 1;
    if (tau > tmax) tau = tmax;
  }
  // compact the selected groups (minimum <= tau) into gid[0, nsel)
  if (tid == 0) S.sc[5] = 0;
  __syncthreads();
  int mine[8], nm = 0;  // a thread's selected groups (V <= 2048: at most 8 per thread)
  for (int i = tid; i < V; i += kSelThreads)
    if (S.gv[i] - dmin <= tau) mine[nm++] = S.gid[i];
  __syncthreads();
  {
    int base = nm ? atomicAdd(S.sc + 5, nm) : 0;
    for (int x = 0; x < nm; ++x) S.gid[base + x] = mine[x];
  }
  __syncthreads();
  const int nsel = S.sc[5];
  const U none = ~U(0);
  // the candidates, read once: 8 lanes per selected group, 4 consecutive slots per lane (16-byte
  // loads when L % 4 == 0), each warp 4 kSwH groups per step (kSwH loads in flight per lane); the
  // valid slots with D - dmin <= tau are appended to (gv, cf)
  U* cd = S.gv;  // the group minima are dead (every thread is past the compaction barrier)
  {
    const int sub = lane >> 3, part = lane & 7;
    const bool vec = (L & 3) == 0;
    constexpr int kStep = 4 * kSwH;
    for (int t0 = warp * kStep; t0 < nsel; t0 += kStep * (kSelThreads / 32)) {
      T v[kSwH][4];
      int tag[kSwH], lim[kSwH];
#pragma unroll
      for (int h = 0; h < kSwH; ++h) {
        const int t = t0 + 4 * h + sub;
        tag[h] = -1;
        lim[h] = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) v[h][w] = T(0);
        if (t < nsel) {
          const int id = S.gid[t], r = id >> 16, j0 = kG * (id & 0xffff) + 4 * part;
          lim[h] = S.pc[r] - j0;
          tag[h] = (r << 24) | j0;
          const T* src = tq + r * static_cast<int64_t>(L) + j0;
          if (vec) {
            if (j0 < L) {
              if constexpr (sizeof(T) == 4) {
                const int4 x = __ldcs(reinterpret_cast<const int4*>(src));
                v[h][0] = x.x, v[h][1] = x.y, v[h][2] = x.z, v[h][3] = x.w;
              } else {
                const longlong2 x0 = __ldcs(reinterpret_cast<const longlong2*>(src));
                const longlong2 x1 = __ldcs(reinterpret_cast<const longlong2*>(src) + 1);
                v[h][0] = x0.x, v[h][1] = x0.y, v[h][2] = x1.x, v[h][3] = x1.y;
              }
            }
          } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) v[h][w] = w < lim[h] ? src[w] : T(0);
          }
        }
      }
      U rel[kSwH][4];
      int c = 0;
#pragma unroll
      for (int h = 0; h < kSwH; ++h)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const U rl = static_cast<U>(v[h][w]) - dmin;
          rel[h][w] = w < lim[h] && rl <= tau ? rl : none;
          c += rel[h][w] != none ? 1 : 0;
        }
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(kFull, incl, 31);
      if (tot == 0) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(S.sc + 6, tot);
      int pos = __shfl_sync(kFull, base, 0) + incl - c;
#pragma unroll
      for (int h = 0; h < kSwH; ++h)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (rel[h][w] != none) {
            if (pos < kCandCap) {
              cd[pos] = rel[h][w];
              S.cf[pos] = tag[h] + w;
            }
            ++pos;
          }
    }
  }
  __syncthreads();
  const int C = S.sc[6];
  if (C > kCandCap) {
    if (tid == 0) flag_query(flags, q);
    return;
  }
  auto item_of = [&](int f) {
    const int t = S.cf[f];
    return __ldg(a.ids + static_cast<int64_t>(S.pl[t >> 24]) * L + (t & 0xffffff));
  };
  int m = k;
  if (C <= k) {  // every candidate wins (fewer than k valid: (-1, d_max) tail, R11)
    for (int f = tid; f < C; f += kSelThreads) S.w.keys[f] = Tr::key(static_cast<T>(cd[f] + dmin), item_of(f));
    m = C;
  } else {
    // window [w0, w0 + span) of D - dmin holding the k-th smallest candidate; `need` = its rank in it
    U w0 = 0, span = tau + 1;
    int need = k;
    for (;;) {
      const int bits = Tr::bitlen(span - 1);
      const int sh = bits > 8 ? bits - 8 : 0;
      S.hist[tid] = 0;
      __syncthreads();
      for (int f = tid; f < C; f += kSelThreads) {
        const U rel = cd[f];
        if (rel >= w0 && rel - w0 < span) atomicAdd(S.hist + static_cast<int>((rel - w0) >> sh), 1);
      }
      __syncthreads();
      int before, inbin;
      const int b = cta_bin_of(S.hist, S.sc, need, &before, &inbin);
      const U hi = w0 + (static_cast<U>(b) << sh);
      const bool last = sh == 0 || inbin <= kBinCap;
      if (last && inbin > kBinCap) {  // more than kBinCap candidates tied at one distance
        if (tid == 0) flag_query(flags, q);
        return;
      }
      // candidates below the target bin win; on the last pass the bin's entries are gathered too
      for (int f = tid; f < C; f += kSelThreads) {
        const U rel = cd[f];
        if (rel < w0) continue;
        if (rel < hi) {
          S.w.keys[atomicAdd(S.sc + 7, 1)] = Tr::key(static_cast<T>(rel + dmin), item_of(f));
        } else if (last && rel - hi < (U(1) << sh)) {
          S.w.bin[atomicAdd(S.sc + 8, 1)] = Tr::key(static_cast<T>(rel + dmin), item_of(f));
        }
      }
      w0 = hi;
      span = U(1) << sh;
      need -= before;
      __syncthreads();
      if (last) {
        const int nb = S.sc[8], nlo = S.sc[7];
        V3DB_DCHECK(nb == inbin && nlo + need == k);
        for (int e2 = tid; e2 < nb; e2 += kSelThreads) {  // the `need` smallest keys of the bin
          const Key key = S.w.bin[e2];
          int rank = 0;
          for (int f = 0; f < nb; ++f) rank += Tr::less(S.w.bin[f], key) ? 1 : 0;
          if (rank < need) S.w.keys[nlo + rank] = key;
        }
        break;
      }
    }
  }
  __syncthreads();
  for (int e2 = tid; e2 < m; e2 += kSelThreads) {
    const Key key = S.w.keys[e2];
    int rank = 0;
    for (int f = 0; f < m; ++f) rank += Tr::less(S.w.keys[f], key) ? 1 : 0;
    a.out_ids[q * k + rank] = Tr::id(key);
    a.out_dist[q * k + rank] = Tr::dist(key);
  }
  for (int r = m + tid; r < k; r += kSelThreads) {
    a.out_ids[q * k + r] = -1;
    a.out_dist[q * k + r] = Tr::kMax;
  }
}

// ---------------------------------------------------------------------------------------------
// Step 5, one WARP per query (the default where it applies): no block barriers, every pass
// warp-synchronous.  The group minima are read from L1/L2 in each pass (a group without a valid
// slot holds the sentinel d_max, written by lm_kernel); tau = the upper edge of a linear histogram
// bin holding the k-th smallest valid group minimum (>= the k-th smallest D); the candidates -- the
// valid slots with D <= tau of the groups whose minimum is <= tau -- are read once (lane = slot of
// the group) and compacted into shared memory; a linear-bin refinement over the candidates finds
// the window [0, w) holding the k smallest D with at most kSwBin entries in its last bin; those
// entries (at most k + kSwBin - 1) get their full (D, item) keys (R10) and are put in order by a
// counting sort over 256 bins plus a pairwise rank inside each bin; the first k are written.
// Queries beyond the caches (kSwCand candidates, more than kSwBin entries tied at one distance)
// are flagged for the streaming path.
// ---------------------------------------------------------------------------------------------
#ifndef V3DB_SW_WARPS
#define V3DB_SW_WARPS 4
#endif
constexpr int kSwWarps = V3DB_SW_WARPS;  // queries per CTA (6 CTAs per SM)
constexpr int kSwCand = 384;    // compacted candidates per query
constexpr int kSwSel = 256;     // selected groups per query
constexpr int kSwBin = 32;      // entries of the last window bin
constexpr int kSwKeys = kSelKmax + kSwBin;

template <class T>
struct SwSmem {  // per warp
  using U = typename DistT<T>::U;
  using Key = typename DistT<T>::Key;
  int hist[256];
  int pl[kWarpProbeCap];
  int pc[kWarpProbeCap];
  int sel[kSwSel];                // selected groups: rho << 16 | g
  U cd[kSwCand];                  // candidate D - dmin
  int cf[kSwCand];                // candidate rho << 24 | slot; then the window entries in bin order
  Key keys[kSwKeys];              // the window's entries
};

// Warp-wide: the bin of h[0, 256) holding rank kk (1-based); *before = entries below it,
// *inbin = its population.
__device__ __forceinline__ int warp_bin_of(const int* h, int kk, int* before, int* inbin) {
  const int lane = threadIdx.x & 31;
  int hb[8], sum = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    hb[b] = h[lane * 8 + b];
    sum += hb[b];
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  int cum = incl - sum, bin = -1, cb = 0;
  if (cum < kk && kk <= incl) {
    bin = lane * 8;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (cum + hb[b] >= kk) {
        cb = hb[b];
        break;
      }
      cum += hb[b];
      ++bin;
    }
  }
  const int src = __ffs(__ballot_sync(kFull, bin >= 0)) - 1;
  *before = __shfl_sync(kFull, cum, src);
  *inbin = __shfl_sync(kFull, cb, src);
  return __shfl_sync(kFull, bin, src);
}

// NPL: group minima per lane held in registers (tot = nprobe * ngroups <= 32 NPL).
template <class T, int NPL>
__global__ void __launch_bounds__(32 * kSwWarps) lm_select_warp_kernel(const SelArgs<T> a, int64_t nq,
                                                                       int* __restrict__ flags) {
  using Tr = DistT<T>;
  using U = typename Tr::U;
  using Key = typename Tr::Key;
  extern __shared__ __align__(16) uint8_t swm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * kSwWarps + warp;
  if (q >= nq) return;
  SwSmem<T>& S = reinterpret_cast<SwSmem<T>*>(swm)[warp];
  const int nprobe = a.nprobe, L = a.L, NG = a.ngroups, k = a.k, tot = nprobe * NG;
  const T* gq = a.gmin + q * tot;
  const T* tq = a.trace + q * nprobe * static_cast<int64_t>(L);
  const unsigned lt = (1u << lane) - 1u;
  const U none = ~U(0);
  // the probed lists first (their counts are a second dependent load), then the group minima
  // (element 32 u + lane in gv[u]; beyond tot: the sentinel), all in flight together
  int pli[kWarpProbeCap / 32];
#pragma unroll
  for (int x = 0; x < kWarpProbeCap / 32; ++x) {
    const int r = 32 * x + lane;
    pli[x] = r < nprobe ? a.lists[q * nprobe + r] : 0;
  }
  T gv[NPL];
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int i = 32 * u + lane;
    gv[u] = i < tot ? gq[i] : Tr::kMax;
  }
#pragma unroll
  for (int x = 0; x < kWarpProbeCap / 32; ++x) {
    const int r = 32 * x + lane;
    if (r < nprobe) {
      S.pl[r] = pli[x];
      S.pc[r] = __ldg(a.counts + pli[x]);
    }
  }
  T mn = Tr::kMax, mx = 0;
  int V = 0;
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    if (gv[u] != Tr::kMax) {
      mn = gv[u] < mn ? gv[u] : mn;
      mx = gv[u] > mx ? gv[u] : mx;
      ++V;
    }
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  V = __reduce_add_sync(kFull, V);
  const U dmin = static_cast<U>(mn);
  const U tmax = static_cast<U>(Tr::kMax) - 1 - dmin;  // relative bound of every valid D
  U tau = tmax;
  if (V >= k) {  // tau: refine a linear histogram of the group minima around rank k
    U w0 = 0, span = static_cast<U>(mx) - dmin + 1;
    int need = k;
    for (;;) {
      const int sh = max(0, Tr::bitlen(span - 1) - 8);
#pragma unroll
      for (int b = 0; b < 8; ++b) S.hist[lane * 8 + b] = 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < NPL; ++u) {
        const U rel = static_cast<U>(gv[u]) - dmin - w0;
        if (gv[u] != Tr::kMax && rel < span) atomicAdd(S.hist + static_cast<int>(rel >> sh), 1);
      }
      __syncwarp();
      int before, inbin;
      const int b = warp_bin_of(S.hist, need, &before, &inbin);
      __syncwarp();
      w0 += static_cast<U>(b) << sh;
      span = U(1) << sh;
      need -= before;
      if (sh == 0 || inbin <= 8) break;  // a bin of <= 8 group minima: tight enough
    }
    tau = w0 + span - 1;
    if (tau > tmax) tau = tmax;
  }
  // the selected groups (minimum <= tau), as rho << 16 | g; (rho, g) of i = 32 u + lane advance by
  // 32 = da NG + db per register
  int ns = 0;
  {
    int r = lane / NG, g = lane - r * NG;
    const int da = 32 / NG, db = 32 - da * NG;
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
      const bool sl = gv[u] != Tr::kMax && static_cast<U>(gv[u]) - dmin <= tau;
      const unsigned bal = __ballot_sync(kFull, sl);
      const int pos = ns + __popc(bal & lt);
      if (sl && pos < kSwSel) S.sel[pos] = (r << 16) | g;
      ns += __popc(bal);
      g += db;
      r += da;
      if (g >= NG) {
        g -= NG;
        ++r;
      }
    }
  }
  if (ns > kSwSel) {
    if (lane == 0) flag_query(flags, q);
    return;
  }
  __syncwarp();
  // the candidates: 8 lanes per selected group, 4 consecutive slots per lane (one 16-byte load per
  // 4 int32 values when L % 4 == 0), 4 kSwH groups per step (kSwH loads in flight per lane: the loop
  // is bound by their latency); kept if valid and D - dmin <= tau
  int C = 0;
  {
    const int sub = lane >> 3, part = lane & 7;
    const bool vec = (L & 3) == 0;
    for (int t0 = 0; t0 < ns; t0 += 4 * kSwH) {
      T v[kSwH][4];
      int tag[kSwH], lim[kSwH];
#pragma unroll
      for (int h = 0; h < kSwH; ++h) {
        const int t = t0 + 4 * h + sub;
        tag[h] = -1;
        lim[h] = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) v[h][w] = T(0);
        if (t < ns) {
          const int e = S.sel[t], r = e >> 16, j0 = kG * (e & 0xffff) + 4 * part;
          lim[h] = S.pc[r] - j0;  // valid slots from j0 on
          tag[h] = (r << 24) | j0;
          const T* src = tq + r * static_cast<int64_t>(L) + j0;
          if (vec) {
            if (j0 < L) {
              if constexpr (sizeof(T) == 4) {
                const int4 x = __ldcs(reinterpret_cast<const int4*>(src));
                v[h][0] = x.x, v[h][1] = x.y, v[h][2] = x.z, v[h][3] = x.w;
              } else {
                const longlong2 x0 = __ldcs(reinterpret_cast<const longlong2*>(src));
                const longlong2 x1 = __ldcs(reinterpret_cast<const longlong2*>(src) + 1);
                v[h][0] = x0.x, v[h][1] = x0.y, v[h][2] = x1.x, v[h][3] = x1.y;
              }
            }
          } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) v[h][w] = w < lim[h] ? src[w] : T(0);
          }
        }
      }
      U rel[kSwH][4];
      int c = 0;
#pragma unroll
      for (int h = 0; h < kSwH; ++h)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const U rl = static_cast<U>(v[h][w]) - dmin;
          rel[h][w] = w < lim[h] && rl <= tau ? rl : none;
          c += rel[h][w] != none ? 1 : 0;
        }
      // this lane's kept values, placed after the lower lanes' (one warp-wide scan per step)
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = C + incl - c;
#pragma unroll
      for (int h = 0; h < kSwH; ++h)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (rel[h][w] != none) {
            if (pos < kSwCand) {
              S.cd[pos] = rel[h][w];
              S.cf[pos] = tag[h] + w;
            }
            ++pos;
          }
      C += __shfl_sync(kFull, incl, 31);
    }
  }
  if (C > kSwCand) {
    if (lane == 0) flag_query(flags, q);
    return;
  }
  __syncwarp();
  // the window [0, w) of D - dmin holding the k smallest candidates, at most kSwBin in its last bin
  U w = tau + 1;
  if (C > k) {
    U w0 = 0, span = tau + 1;
    int need = k;
    for (;;) {
      const int sh = max(0, Tr::bitlen(span - 1) - 8);
#pragma unroll
      for (int b = 0; b < 8; ++b) S.hist[lane * 8 + b] = 0;
      __syncwarp();
      for (int f = lane; f < C; f += 32) {
        const U rel = S.cd[f] - w0;
        if (rel < span) atomicAdd(S.hist + static_cast<int>(rel >> sh), 1);
      }
      __syncwarp();
      int before, inbin;
      const int b = warp_bin_of(S.hist, need, &before, &inbin);
      __syncwarp();
      w0 += static_cast<U>(b) << sh;
      span = U(1) << sh;
      need -= before;
      if (inbin <= kSwBin) break;
      if (sh == 0) {  // more than kSwBin candidates tied at one distance
        if (lane == 0) flag_query(flags, q);
        return;
      }
    }
    w = w0 + span;
  }
  // the window's entries as full keys (four item-id loads in flight per lane)
  int M = 0;
  for (int f0 = 0; f0 < C; f0 += 128) {
    int32_t id[4];
    bool in[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = f0 + 32 * u + lane;
      in[u] = f < C && S.cd[f] < w;
      id[u] = 0;
      if (in[u]) {
        const int t = S.cf[f];
        id[u] = __ldg(a.ids + static_cast<int64_t>(S.pl[t >> 24]) * L + (t & 0xffffff));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = f0 + 32 * u + lane;
      const unsigned bt = __ballot_sync(kFull, in[u]);
      if (in[u]) S.keys[M + __popc(bt & lt)] = Tr::key(static_cast<T>(S.cd[f] + dmin), id[u]);
      M += __popc(bt);
    }
  }
  __syncwarp();
  V3DB_DCHECK(M <= kSwKeys);
  // counting sort of the M keys by D over 256 bins of [0, w), then the rank inside each bin
  {
    int* cf = S.cf;  // reused: the window entries' indices in bin order (M <= kSwKeys <= kSwCand)
    const int sh = max(0, Tr::bitlen(w - 1) - 8);
#pragma unroll
    for (int b = 0; b < 8; ++b) S.hist[lane * 8 + b] = 0;
    __syncwarp();
    for (int e2 = lane; e2 < M; e2 += 32)
      atomicAdd(S.hist + static_cast<int>((static_cast<U>(Tr::dist(S.keys[e2])) - dmin) >> sh), 1);
    __syncwarp();
    int hb[8], sum = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      hb[b] = S.hist[lane * 8 + b];
      sum += hb[b];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      S.hist[lane * 8 + b] = run;  // exclusive start; advanced to the bin's end by the scatter
      run += hb[b];
    }
    __syncwarp();
    for (int e2 = lane; e2 < M; e2 += 32) {
      const int b = static_cast<int>((static_cast<U>(Tr::dist(S.keys[e2])) - dmin) >> sh);
      cf[atomicAdd(S.hist + b, 1)] = e2 | (b << 16);
    }
    __syncwarp();
    for (int p = lane; p < M; p += 32) {
      const int e2 = cf[p] & 0xffff, b = cf[p] >> 16;
      const int s0 = b ? S.hist[b - 1] : 0, s1 = S.hist[b];
      const Key key = S.keys[e2];
      int rank = s0;
      for (int x = s0; x < s1; ++x) rank += Tr::less(S.keys[cf[x] & 0xffff], key) ? 1 : 0;
      if (rank < k) {
        a.out_ids[q * k + rank] = Tr::id(key);
        a.out_dist[q * k + rank] = Tr::dist(key);
      }
    }
  }
  for (int r = M + lane; r < k; r += 32) {  // fewer than k valid candidates (R11)
    a.out_ids[q * k + r] = -1;
    a.out_dist[q * k + r] = Tr::kMax;
  }
}

// The queries the cached path flagged (flags[0] of them, listed in flags[1..]), or every query when
// it does not apply (flags NULL): a grid-stride loop, one query per CTA at a time.
template <class T>
__global__ void __launch_bounds__(kSelThreads) lm_select_cta_kernel(const SelArgs<T> a, const int* __restrict__ flags,
                                                                     int64_t nq) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int64_t n = flags ? flags[0] : nq;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    select_streaming<T>(a, flags ? flags[1 + i] : i, sm);
    __syncthreads();  // the shared memory is reused by the next query
  }
}

// Step 5 launch (both distance types): the cached selection, then the streaming one for the queries
// it flagged; flags: scratch int [1 + nq] (a count, then the flagged query indices).
template <class T>
cudaError_t launch_select(const SelArgs<T>& sa, int64_t nq, int* flags, cudaStream_t st) {
  using Key = typename DistT<T>::Key;
  const size_t ssm = sizeof(int) * (2 * sa.nprobe + 256 + 16 + kSelGroups) + 16 + sizeof(Key) * sa.k;
  const bool fast = sa.k <= kSelKmax && sa.nprobe <= kWarpProbeCap && sa.ngroups <= 65535;
  // one warp per query where the group minima are many against k (tau from them is then tight and
  // the candidates few); the CTA kernel (a larger candidate cache) otherwise
  const int64_t sopt = opt(V3DB_OPT_SELECT_CTA);
  const int64_t tot_g = static_cast<int64_t>(sa.nprobe) * sa.ngroups;
  const bool warp = fast && tot_g <= 32 * 64 && (sopt == 2 || (sopt == 0 && tot_g >= 8 * static_cast<int64_t>(sa.k)));
  cudaError_t e = cudaSuccess;
  if (fast) {
    e = cudaMemsetAsync(flags, 0, sizeof(int), st);
    if (e == cudaSuccess && warp) {
      const size_t wsm = sizeof(SwSmem<T>) * kSwWarps;
      const unsigned g = static_cast<unsigned>((nq + kSwWarps - 1) / kSwWarps);
      auto run = [&](auto kern) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wsm));
        if (e == cudaSuccess) kern<<<g, 32 * kSwWarps, wsm, st>>>(sa, nq, flags);
      };
      const int tot = sa.nprobe * sa.ngroups;
      if (tot <= 32 * 8) run(lm_select_warp_kernel<T, 8>);
      else if (tot <= 32 * 16) run(lm_select_warp_kernel<T, 16>);
      else if (tot <= 32 * 32) run(lm_select_warp_kernel<T, 32>);
      else if (tot <= 32 * 48) run(lm_select_warp_kernel<T, 48>);
      else run(lm_select_warp_kernel<T, 64>);
      note_launch();
      if (e == cudaSuccess) e = cudaGetLastError();
    } else if (e == cudaSuccess) {
      lm_select_fast_kernel<T><<<static_cast<unsigned>(nq), kSelThreads, 0, st>>>(sa, flags);
      note_launch();
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lm_select_cta_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ssm));
  if (e == cudaSuccess) {
    // flagged queries are rare: a small grid that exits at once when there are none (an nq-CTA grid
    // cost 9-30 us of empty blocks per call)
    const int64_t grid = fast ? std::min<int64_t>(nq, 4 * 148) : nq;
    lm_select_cta_kernel<T><<<static_cast<unsigned>(grid), kSelThreads, ssm, st>>>(sa, fast ? flags : nullptr, nq);
    note_launch();
    e = cudaGetLastError();
  }
  return e;
}

size_t al(size_t x, size_t b) { return (x + b - 1) / b * b; }

// ----------------------------------------------------------------------------------------------
// NEXT-1 list-major (fixed point): the same identity in int64,
//     D_{i,j} = d_i + P_{i,j} - 2 <q, xhat_{i,j}>,
// with <q, xhat> = sum_{s,t} 256^(s+t) <xhat_s, q_t> over three balanced int8 limbs per coordinate
// (v = v_0 + 256 v_1 + 65536 v_2, fx_coarse_tc.cu): nine tcgen05 kind::i8 products into five exact
// int32 accumulators per (128 slots x NTF pairs) tile (|acc_u| <= 3 * 128^2 * dim < 2^31), combined
// in int64 by the epilogue.  Same warp roles and grouping as lm_kernel; D and the group minima are
// int64; Step 5 is the int64 instantiation of the same selection kernels.
// ----------------------------------------------------------------------------------------------
// Tile width: 32 pairs x 5 accumulators x 2 sets (320 TMEM columns), one set per epilogue group.  (96
// pairs in one set -- a third of the MMAs per pair, since a kind::i8 MMA costs ~160 cycles whatever N --
// measured slower at C4, 3.28 vs 3.10 ms: the kernel is bound by its DRAM traffic, not the MMA rate.)
constexpr int kNTF = 32;          // pairs per item
constexpr int kFSetsLm = 2;       // accumulator sets = epilogue groups (one each)
constexpr int kFGroups = kFSetsLm, kFColGroups = 4 / kFGroups, kFColsPerWarp = kNTF / kFColGroups;
constexpr int kFStageRow = 68;    // words per staged column (32 int64 + 4 words pad)
constexpr int kFSub = 8;          // columns per epilogue sub-chunk
constexpr int64_t kDMaxFxLm = 0x7fffffffffffffffLL;

struct LmFxArgs {
  int nprobe, L, Lp, dim, kp, S, nb, ngroups, p_stride;
  int64_t rows_x;            // rows per xhat limb plane (nlist * Lp)
  int64_t rows_q;            // rows per query limb plane (nq)
  const int8_t* ql;          // [3][nq][dim] query limbs
  const int32_t* pairs;
  const int4* items;
  const int* n_items;
  int* next_item;            // work counter (zeroed by the grouping), or NULL: static round-robin
  const int64_t* ldist;      // [nq * nprobe] d_i of each pair
  const int32_t* counts;
  const int64_t* pterm;      // [nlist][L]
  int64_t* trace;            // [nq][nprobe][L]
  int64_t* gmin;             // [nq][nprobe][ngroups]
  uint32_t off_b, off_meta, off_p, off_stage, off_bar, b_bytes;
};

__global__ void __launch_bounds__(kThreads, 1) lm_fx_kernel(const __grid_constant__ CUtensorMap tmX, const LmFxArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                                      // [S][128 x 128 B] (one limb each)
  uint8_t* sB = smem + a.off_b;                                            // [nb][3 limbs][kp][NTF x 128 B]
  uint64_t* mrow = reinterpret_cast<uint64_t*>(smem + a.off_meta);         // [nb][NTF] trace row address
  int64_t* md = reinterpret_cast<int64_t*>(mrow + a.nb * kNTF);            // [nb][NTF] d_i
  int* mgoff = reinterpret_cast<int*>(md + a.nb * kNTF);                   // [nb][NTF] group-minimum row
  int64_t* sP = reinterpret_cast<int64_t*>(smem + a.off_p);                // [nb][p_stride] P terms
  int64_t* stage = reinterpret_cast<int64_t*>(smem + a.off_stage);         // [kEpiWarps][kFSub][34]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* afull = bars;                  // [S]
  uint64_t* aempty = afull + a.S;          // [S]
  uint64_t* bfull = aempty + a.S;          // [kNB]
  uint64_t* bempty = bfull + kNB;          // [kNB]
  uint64_t* accf = bempty + kNB;           // [kFSetsLm]
  uint64_t* acce = accf + kFSetsLm;        // [kFSetsLm]
  uint64_t* ifull = acce + kFSetsLm;       // [kIR]
  uint64_t* iempty = ifull + kIR;          // [kIR]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iempty + kIR);
  // the CTA's work-item sequence, drawn and published by the TMA thread (see lm_kernel)
  int4* ring = reinterpret_cast<int4*>(
      smem + ((a.off_bar + 8u * (2 * a.S + 2 * kNB + 2 * kFSetsLm + 2 * kIR) + 16u + 15u) & ~15u));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = *a.n_items;
  const int L = a.L;

  if (tid == 0) {
    for (int s = 0; s < a.S; ++s) {
      tc::mbar_init(afull + s, 1);
      tc::mbar_init(aempty + s, 1);
    }
    for (int b = 0; b < kNB; ++b) {
      tc::mbar_init(bfull + b, kNGat);
      tc::mbar_init(bempty + b, 1 + kEpiWarps);
    }
    for (int c = 0; c < kFSetsLm; ++c) {
      tc::mbar_init(accf + c, 1);
      tc::mbar_init(acce + c, kEpiWarps / kFGroups);
    }
    for (int r = 0; r < kIR; ++r) {
      tc::mbar_init(ifull + r, 1);
      tc::mbar_init(iempty + r, 1 + kNGat + kEpiWarps);
    }
    tc::mbar_fence_init();
  }
  if (warp == kWarpMma) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpTma) {
    // ------------------------------------------------------------ xhat limb tiles (TMA)
    if (lane == 0) {
      tc::tma_prefetch(&tmX);
      int s = 0, u = 0;
      const int G = static_cast<int>(gridDim.x);
      int4 pre[kPre];
#pragma unroll
      for (int d = 0; d < kPre; ++d) {
        const int j = static_cast<int>(blockIdx.x) + d * G;
        pre[d] = j < n_items ? __ldg(a.items + j) : make_int4(0, 0, -1, 0);
      }
      int jn = a.next_item ? kPre * G + atomicAdd(a.next_item, 1) : static_cast<int>(blockIdx.x) + kPre * G;
      int ip = 0;
      bool done = false;
#pragma unroll
      for (int d = 0; d < kPre; ++d) {
        if (!done) {
          ring[d] = pre[d];
          tc::mbar_arrive(ifull + d);
          done = pre[d].z < 0;
          ++ip;
        }
      }
      for (int il = 0;; ++il) {
        while (!done && ip < il + kPre) {
          const int r = ip & (kIR - 1), j = jn;
          if (ip >= kIR) tc::mbar_wait_sleep(iempty + r, (ip / kIR - 1) & 1);
          done = j >= n_items;
          ring[r] = done ? make_int4(0, 0, -1, 0) : __ldg(a.items + j);
          tc::mbar_arrive(ifull + r);
          ++ip;
          if (!done) jn = a.next_item ? kPre * G + atomicAdd(a.next_item, 1) : j + G;
        }
        const int4 it = ring[il & (kIR - 1)];
        if (it.z < 0) break;
        const int nvt = (it.w + kTile - 1) / kTile;
        for (int t = 0; t < nvt; ++t)
          for (int p = 0; p < a.kp; ++p)
            for (int l = 0; l < 3; ++l) {
              if (u > 0) tc::mbar_wait_sleep(aempty + s, (u - 1) & 1);
              tc::mbar_expect_tx(afull + s, kAStageBytes);
              tc::tma_load_2d(sA + s * kAStageBytes, &tmX, afull + s, p * kPanel,
                              static_cast<int>(l * a.rows_x + static_cast<int64_t>(it.x) * a.Lp + t * kTile));
              if (++s == a.S) {
                s = 0;
                ++u;
              }
            }
      }
    }
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int s = 0, u = 0, b = 0, bph = 0, tcount = 0;
      for (int i = 0;; ++i) {
        const int r = i & (kIR - 1);
        tc::mbar_wait_sleep(ifull + r, (i / kIR) & 1);
        const int4 it = ring[r];
        const int nvt = (it.w + kTile - 1) / kTile;
        tc::mbar_arrive(iempty + r);
        if (it.z < 0) break;
        const int N = (it.z + 15) & ~15;
        const uint32_t idesc = tc::idesc_s8(kTile, N);
        tc::mbar_wait_sleep(bfull + b, bph);
        tc::fence_after_sync();
        const uint32_t b_addr = tc::smem_u32(sB + b * a.b_bytes);
        for (int t = 0; t < nvt; ++t, ++tcount) {
          const int set = tcount % kFSetsLm, use = tcount / kFSetsLm;
          if (use > 0) {
            tc::mbar_wait_sleep(acce + set, (use - 1) & 1);
            tc::fence_after_sync();
          }
          const uint32_t acc0 = tmem + set * (5 * kNTF);
          for (int p = 0; p < a.kp; ++p) {
            int st[3];
            for (int l = 0; l < 3; ++l) {
              st[l] = s;
              tc::mbar_wait_sleep(afull + s, u & 1);
              if (++s == a.S) {
                s = 0;
                ++u;
              }
            }
            tc::fence_after_sync();
            const int nk = min(4, (a.dim - p * kPanel + 31) / 32);
            uint64_t dA[3], dB[3];
#pragma unroll
            for (int l = 0; l < 3; ++l) {
              dA[l] = tc::desc_sw128(tc::smem_u32(sA + st[l] * kAStageBytes));
              dB[l] = tc::desc_sw128(b_addr + (l * a.kp + p) * kNTF * kPanel);
            }
            for (int k = 0; k < nk; ++k) {
              const uint32_t first = (p == 0 && k == 0) ? 1u : 0u;
              // u = sl + t: 2 1 3 2 0 4 2 1 3 (no accumulator updated back to back); accumulate
              // except on an accumulator's first product of the tile
#define LMF_MMA(SL, T, FIRSTPAIR) \
  tc::mma_s8(acc0 + ((SL) + (T)) * kNTF, dA[SL] + 2 * k, dB[T] + 2 * k, idesc, (FIRSTPAIR) ? (first ^ 1u) : 1u)
              LMF_MMA(2, 0, true);
              LMF_MMA(1, 0, true);
              LMF_MMA(2, 1, true);
              LMF_MMA(1, 1, false);
              LMF_MMA(0, 0, true);
              LMF_MMA(2, 2, true);
              LMF_MMA(0, 2, false);
              LMF_MMA(0, 1, false);
              LMF_MMA(1, 2, false);
#undef LMF_MMA
            }
            for (int l = 0; l < 3; ++l) tc::mma_commit(aempty + st[l]);
          }
          tc::mma_commit(accf + set);
        }
        tc::mma_commit(bempty + b);
        if (++b == a.nb) {
          b = 0;
          bph ^= 1;
        }
      }
    }
  } else if (warp < kWarpEpi) {
    // ------------------------------------------------------------ gather: query limbs + metadata
    const int gt = tid - kWarpGat * 32;  // 0 .. 63
    const int cpr = a.dim >> 4;
    int b = 0, use = 0;
    for (int i = 0;; ++i) {
      const int ri = i & (kIR - 1);
      tc::mbar_wait_sleep(ifull + ri, (i / kIR) & 1);
      const int4 it = ring[ri];
      const int cnt = it.w;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(iempty + ri);
      if (it.z < 0) break;
      if (use > 0) tc::mbar_wait_sleep(bempty + b, (use - 1) & 1);
      uint8_t* dst = sB + b * a.b_bytes;
      {
        if (gt == 0 && a.p_stride && cnt > 0) {
          const uint32_t pbytes = 16u * ((cnt + 1) / 2);
          tc::mbar_expect_tx_only(bfull + b, pbytes);
          bulk_g2s_lm(sP + b * a.p_stride, a.pterm + static_cast<int64_t>(it.x) * L, pbytes, bfull + b);
        }
      }
      for (int r = gt; r < it.z; r += 32 * kNGat) {
        const int pr = __ldg(a.pairs + it.y + r);
        const int q = pr / a.nprobe;
        mrow[b * kNTF + r] = reinterpret_cast<uint64_t>(a.trace + static_cast<int64_t>(pr) * L);
        md[b * kNTF + r] = __ldg(a.ldist + pr);
        mgoff[b * kNTF + r] = pr * a.ngroups;
        for (int l = 0; l < 3; ++l) {
          const int8_t* qrow = a.ql + (l * a.rows_q + q) * a.dim;
          for (int c = 0; c < cpr; ++c)
            tc::cp_async16(dst + ((l * a.kp) + (c >> 3)) * kNTF * kPanel + tc::sw128_offset(r, c & 7), qrow + c * 16, 16);
        }
      }
      tc::cp_async_commit();
      tc::cp_async_wait<0>();
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bfull + b);
      if (++b == a.nb) {
        b = 0;
        ++use;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Two groups of 8 warps take alternate tiles; warp = TMEM lane quadrant qd (32 slots) x column
    // half cg (16 pairs, two sub-chunks of 8).  Thread = slot: D (int64) of each column to the trace
    // (32 lanes = 256 consecutive bytes); the column's 32 staged D in shared memory give the group
    // minimum (four lanes per column, eight values each).
    const int e = warp - kWarpEpi, qd = warp & 3, cg = (e >> 2) % kFColGroups, grp = (e >> 2) / kFColGroups;
    int64_t* stg = stage + e * (kFSub * (kFStageRow / 2));
    int b = 0, bph = 0, tcount = 0, tall = 0;
    for (int i = 0;; ++i) {
      const int ri = i & (kIR - 1);
      tc::mbar_wait_sleep(ifull + ri, (i / kIR) & 1);
      const int4 it = ring[ri];
      const int cnt = it.w;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(iempty + ri);
      if (it.z < 0) break;
      const int np = it.z;
      const int nvt = (cnt + kTile - 1) / kTile, ntl = (L + kTile - 1) / kTile;
      const uint64_t* mr = mrow + b * kNTF;
      const int64_t* mdd = md + b * kNTF;
      const int* mg = mgoff + b * kNTF;
      const int64_t* pP = sP + b * a.p_stride;
      tc::mbar_wait_sleep(bfull + b, bph);
      for (int t = 0; t < ntl; ++t, ++tall) {
        const bool mine = (tall % kFGroups) == grp;
        const int sbase = t * kTile + qd * 32, slot = sbase + lane;
        const uint64_t toff = 8ull * static_cast<uint32_t>(slot);
        if (t < nvt) {
          // valid tile: group = set = (tile count) mod 2 (each group owns one accumulator set and waits
          // on every phase of its barriers)
          const int set = tcount % kFSetsLm, use = tcount / kFSetsLm;
          ++tcount;
          if (set != grp) continue;
          const bool valid = slot < cnt;
          const int64_t P = !valid ? 0 : a.p_stride ? pP[slot] : __ldg(a.pterm + static_cast<int64_t>(it.x) * L + slot);
          tc::mbar_wait_sleep(accf + set, use & 1);
          tc::fence_after_sync();
          const uint32_t tbase = tmem + (static_cast<uint32_t>(qd * 32) << 16) + set * (5 * kNTF);
          const int cend = sbase < L ? min(np, (cg + 1) * kFColsPerWarp) : 0;
          bool released = false;
          for (int c0 = cg * kFColsPerWarp; c0 < cend; c0 += kFSub) {
            uint32_t v0[8], v1[8], v2[8], v3[8], v4[8];
            tc::tmem_ld8(tbase + 0 * kNTF + c0, v0);
            tc::tmem_ld8(tbase + 1 * kNTF + c0, v1);
            tc::tmem_ld8(tbase + 2 * kNTF + c0, v2);
            tc::tmem_ld8(tbase + 3 * kNTF + c0, v3);
            tc::tmem_ld8(tbase + 4 * kNTF + c0, v4);
            tc::tmem_ld_wait();
            if (c0 + kFSub >= cend) {  // this warp's last accumulator values are in registers
              tc::fence_before_sync();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(acce + set);
              released = true;
            }
            const int ncol = min(kFSub, np - c0);
            __syncwarp();  // the previous sub-chunk's reads of the stage are done
#pragma unroll
            for (int c = 0; c < kFSub; ++c) {
              int64_t x = kDMaxFxLm;
              if (c < ncol) {  // warp-uniform
                if (valid) {
                  x = mdd[c0 + c] + P;
                  x += static_cast<int64_t>(static_cast<int32_t>(v0[c])) * -2;
                  x += static_cast<int64_t>(static_cast<int32_t>(v1[c])) * -512;
                  x += static_cast<int64_t>(static_cast<int32_t>(v2[c])) * -131072;
                  x += static_cast<int64_t>(static_cast<int32_t>(v3[c])) * -33554432LL;
                  x += static_cast<int64_t>(static_cast<int32_t>(v4[c])) * -8589934592LL;
                }
                if (slot < L) __stcs(reinterpret_cast<long long*>(mr[c0 + c] + toff), static_cast<long long>(x));
              }
              stg[c * (kFStageRow / 2) + lane] = x;
            }
            __syncwarp();
            // group minima: lane = column (lane & 7) x part (lane >> 3) of eight slots
            const int col = lane & 7, part = lane >> 3;
            const int4* r4 = reinterpret_cast<const int4*>(stg + col * (kFStageRow / 2) + part * 8);
            int64_t m = kDMaxFxLm;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int4 w = r4[u];
              const int64_t a0 = (static_cast<int64_t>(w.y) << 32) | static_cast<uint32_t>(w.x);
              const int64_t a1 = (static_cast<int64_t>(w.w) << 32) | static_cast<uint32_t>(w.z);
              m = min(m, min(a0, a1));
            }
            m = min(m, static_cast<int64_t>(__shfl_xor_sync(kFull, static_cast<long long>(m), 8)));
            m = min(m, static_cast<int64_t>(__shfl_xor_sync(kFull, static_cast<long long>(m), 16)));
            if (part == 0 && col < ncol) a.gmin[mg[c0 + col] + t * 4 + qd] = m;
          }
          if (!released) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(acce + set);
          }
        } else if (mine && slot < L) {
          // a tile of padding only: D = d_max, nothing read
          for (int c = cg * kFColsPerWarp; c < min(np, (cg + 1) * kFColsPerWarp); ++c) {
            __stcs(reinterpret_cast<long long*>(mr[c] + toff), static_cast<long long>(kDMaxFxLm));
            if (lane == 0) a.gmin[mg[c] + t * 4 + qd] = kDMaxFxLm;  // group sentinel
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bempty + b);
      if (++b == a.nb) {
        b = 0;
        bph ^= 1;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kWarpMma) tc::tmem_dealloc(tmem, 512);
}

// int32 fixed-point coordinates -> three balanced int8 limb planes [3][n][dim]
__global__ void fx_limbs_kernel(const int32_t* __restrict__ X, int64_t n, int dim, int8_t* __restrict__ out) {
  const int64_t tot = n * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = __ldg(X + e);
    const int d0 = ((v + 128) & 255) - 128, w = (v - d0) >> 8;
    const int d1 = ((w + 128) & 255) - 128, d2 = (w - d1) >> 8;
    out[e] = static_cast<int8_t>(d0);
    out[tot + e] = static_cast<int8_t>(d1);
    out[2 * tot + e] = static_cast<int8_t>(d2);
  }
}

}  // namespace

cudaError_t scan_list_major(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                            const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                            int32_t* trace_cand, cudaStream_t st, void (*prof)(int, cudaStream_t),
                            const int* list_hist) {
  if (nq <= 0) return cudaSuccess;
  if (!s->xhat || s->dim % 16 != 0) return cudaErrorInvalidValue;
  const int64_t npairs = nq * nprobe;
  const int L = s->L, ngroups = (L + kG - 1) / kG, kp = (s->dim + kPanel - 1) / kPanel;
  if (npairs >= (int64_t(1) << 31) || npairs * ngroups >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  // NT: pairs per item, 64 (measured: C4 main kernel 0.968 ms vs 1.009 at 128, C2 0.337 vs 0.357), or
  // less where three B operands would not fit 128 KB
  int NT = 64;
  const int64_t nt_opt = opt(V3DB_OPT_LM_NT);
  if (nt_opt == 32 || nt_opt == 64 || nt_opt == 128 || nt_opt == 256) NT = static_cast<int>(nt_opt);
  int nb = kNB;  // B buffers: 3, or 2 when three of the smallest NT do not fit (dim near 2048)
  while (NT > 32 && static_cast<uint32_t>(nb) * kp * NT * kPanel > 128u * 1024) NT >>= 1;
  if (static_cast<uint32_t>(nb) * kp * NT * kPanel > 128u * 1024) nb = 2;
  const int nacc = std::min(4, 512 / NT);  // a power of two
  const int lg_nacc = nacc == 4 ? 2 : nacc == 2 ? 1 : 0;
  const uint32_t b_bytes = static_cast<uint32_t>(kp) * NT * kPanel;
  // P terms of the item's list staged per B buffer (when they take <= 48 KB); the trace staged and
  // stored from a shared-memory stage when L % 4 == 0 and the stage fits beside >= 3 A stages
  int p_stride = L % 4 == 0 ? L : 0;  // (16-byte aligned rows: one bulk copy per item)
  if (static_cast<size_t>(nb) * 4 * p_stride > 48 * 1024) p_stride = 0;
  bool bulk = L % 4 == 0;
  int S = V3DB_LM_STAGES;
  auto smem_of = [&](int stages) {
    return 1024 + static_cast<size_t>(stages) * kAStageBytes + nb * b_bytes + nb * sizeof(PairMeta) * NT +
           static_cast<size_t>(nb) * 4 * NT + static_cast<size_t>(nb) * 4 * p_stride + (bulk ? kStageBytes : 0) +
           8 * (2 * stages + 2 * kNB + 2 * nacc + 2 * kIR) + 16 + 16 + sizeof(int4) * kIR;
  };
  while (S > 2 && smem_of(S) > 227 * 1024) --S;
  if (bulk && (S < 3 || smem_of(S) > 227 * 1024)) {
    bulk = false;
    S = V3DB_LM_STAGES;
    while (S > 2 && smem_of(S) > 227 * 1024) --S;
  }
  if (smem_of(S) > 227 * 1024) return cudaErrorInvalidConfiguration;

  CUtensorMap tmX;
  if (!make_tmap_i8(&tmX, s->xhat, static_cast<uint64_t>(s->nlist) * s->lm_Lp, s->dim, kTile, kPanel))
    return cudaErrorInvalidValue;

  // scratch: hist, cur, (unused), n_items, pairs, items, gmin + flags (+ trace when the caller passes none)
  const int nlist = s->nlist;
  const int64_t max_items = nlist + npairs / NT + 1;
  const size_t b_hist = al(sizeof(int) * nlist, 256), b_pairs = al(sizeof(int32_t) * npairs, 256),
               b_items = al(sizeof(int4) * max_items, 256),
               b_gmin = al(sizeof(int32_t) * npairs * ngroups, 256) + al(sizeof(int) * (nq + 1), 256),  // + flags
               b_trace = trace_cand ? 0 : al(sizeof(int32_t) * npairs * L, 256);
  uint8_t* base = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&base), 3 * b_hist + 256 + b_pairs + b_items + b_gmin + b_trace, st);
  if (e != cudaSuccess) return e;
  int* hist = reinterpret_cast<int*>(base);
  int* cur = reinterpret_cast<int*>(base + b_hist);
  int* n_items = reinterpret_cast<int*>(base + 3 * b_hist);  // (base + 2 b_hist: the items scan's CTA totals)
  int32_t* pairs = reinterpret_cast<int32_t*>(base + 3 * b_hist + 256);
  int4* items = reinterpret_cast<int4*>(base + 3 * b_hist + 256 + b_pairs);
  int32_t* gmin = reinterpret_cast<int32_t*>(base + 3 * b_hist + 256 + b_pairs + b_items);
  int32_t* trace = trace_cand ? trace_cand : reinterpret_cast<int32_t*>(base + 3 * b_hist + 256 + b_pairs + b_items + b_gmin);

  int dev = 0, sms = 148;
  e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess && !list_hist) e = cudaMemsetAsync(hist, 0, sizeof(int) * nlist, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(base, st);
    return e;
  }
  const unsigned pg = static_cast<unsigned>(std::min<int64_t>((npairs + 255) / 256, 4 * sms));
  if (!list_hist) {
    pair_hist_kernel<<<pg, 256, 0, st>>>(lists, npairs, hist);
    note_launch();
  }
  const int* hsrc = list_hist ? list_hist : hist;
  e = launch_scan_items(hsrc, s->counts, nlist, NT, cur, items, n_items, reinterpret_cast<int2*>(base + 2 * b_hist), st);
  if (e == cudaSuccess) e = launch_pair_scatter(lists, npairs, nlist, cur, pairs, st);
  note_launch(2);
  if (e != cudaSuccess) {
    cudaFreeAsync(base, st);
    return e;
  }
  if (prof) prof(2, st);

  LmArgs a;
  a.nprobe = nprobe;
  a.L = L;
  a.Lp = s->lm_Lp;
  a.dim = s->dim;
  a.kp = kp;
  a.NT = NT;
  a.nacc = nacc;
  a.S = S;
  a.ngroups = ngroups;
  a.queries = queries;
  a.pairs = pairs;
  a.items = items;
  a.n_items = n_items;
  a.next_item = opt(V3DB_OPT_LM_STATIC) == 1 ? nullptr : n_items + 1;  // (zeroed by the items scan)
  a.ldist = ldist;
  a.counts = s->counts;
  a.pterm = s->pterm;
  a.trace = trace;
  a.gmin = gmin;
  a.off_b = S * kAStageBytes;
  a.lg_nacc = lg_nacc;
  a.nb = nb;
  a.off_meta = a.off_b + nb * b_bytes;  // PairMeta is 16 B: 16-byte aligned (b_bytes is a multiple of 128)
  a.off_sd = a.off_meta + nb * sizeof(PairMeta) * NT;
  a.off_p = a.off_sd + nb * 4 * NT;
  a.off_stage = a.off_p + nb * 4 * p_stride;
  a.off_bar = static_cast<uint32_t>(al(a.off_stage + (bulk ? kStageBytes : 0), 8));
  a.p_stride = p_stride;
  a.bulk = bulk ? 1 : 0;
  a.b_bytes = b_bytes;
  const size_t smem = smem_of(S);
  e = cudaFuncSetAttribute(lm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) {
    const int64_t grid = std::min<int64_t>(sms, max_items);
    lm_kernel<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(tmX, a);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = debug_sync(st, "lm_kernel");
  if (prof) prof(3, st);
  if (e == cudaSuccess) {
    SelArgs<int32_t> sa;
    sa.nprobe = nprobe;
    sa.L = L;
    sa.ngroups = ngroups;
    sa.k = k;
    sa.lists = lists;
    sa.counts = s->counts;
    sa.ids = s->ids;
    sa.trace = trace;
    sa.gmin = gmin;
    sa.out_ids = out_ids;
    sa.out_dist = out_dist;
    e = launch_select(sa, nq, reinterpret_cast<int*>(gmin + npairs * ngroups), st);
  }
  if (e == cudaSuccess) e = debug_sync(st, "lm_select kernels");
  cudaFreeAsync(base, st);
  return e;
}

// NEXT-1 list-major: the fixed-point Steps 3-5 on the tensor cores (see lm_fx_kernel).  Requires
// s->xhat_fx (dim % 16 == 0, dim <= 256, nlist <= 32768).
cudaError_t scan_list_major_fx(const v3db_snapshot* s, const int32_t* queries, int64_t nq, int nprobe, int k,
                               const int32_t* lists, const int64_t* ldist, int32_t* out_ids, int64_t* out_dist,
                               int64_t* trace_cand, cudaStream_t st, void (*prof)(int, cudaStream_t)) {
  if (nq <= 0) return cudaSuccess;
  if (!s->xhat_fx || s->dim % 16 != 0) return cudaErrorInvalidValue;
  const int64_t npairs = nq * nprobe;
  const int L = s->L, ngroups = (L + kG - 1) / kG, kp = (s->dim + kPanel - 1) / kPanel, nlist = s->nlist;
  if (npairs >= (int64_t(1) << 31) || npairs * ngroups >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  const int nb = kFSetsLm == 1 ? 2 : kNB;  // B operand buffers
  const uint32_t b_bytes = 3u * kp * kNTF * kPanel;
  int p_stride = L % 2 == 0 ? L : 0;  // (16-byte aligned int64 rows: one bulk copy per item)
  if (static_cast<size_t>(nb) * 8 * p_stride > 48 * 1024) p_stride = 0;
  const uint32_t stage_bytes = kEpiWarps * kFSub * kFStageRow * 4;
  auto smem_of = [&](int stages) {
    return 1024 + static_cast<size_t>(stages) * kAStageBytes + nb * b_bytes + nb * kNTF * 20 +
           static_cast<size_t>(nb) * 8 * p_stride + stage_bytes +
           8 * (2 * stages + 2 * kNB + 2 * kFSetsLm + 2 * kIR) + 64 + 16 + sizeof(int4) * kIR;
  };
  int S = 9;
  while (S > 3 && smem_of(S) > 227 * 1024) --S;
  if (smem_of(S) > 227 * 1024) return cudaErrorInvalidConfiguration;

  CUtensorMap tmX;
  if (!make_tmap_i8(&tmX, s->xhat_fx, 3ull * nlist * s->lm_Lp, s->dim, kTile, kPanel)) return cudaErrorInvalidValue;

  const int64_t max_items = nlist + npairs / kNTF + 1;
  const size_t b_hist = al(sizeof(int) * nlist, 256), b_pairs = al(sizeof(int32_t) * npairs, 256),
               b_items = al(sizeof(int4) * max_items, 256), b_ql = al(3ull * nq * s->dim, 256),
               b_gmin = al(sizeof(int64_t) * npairs * ngroups, 256) + al(sizeof(int) * (nq + 1), 256),  // + flags
               b_trace = trace_cand ? 0 : al(sizeof(int64_t) * npairs * L, 256);
  uint8_t* base = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&base),
                                2 * b_hist + 512 + b_pairs + b_items + b_ql + b_gmin + b_trace, st);
  if (e != cudaSuccess) return e;
  int* hist = reinterpret_cast<int*>(base);
  int* cur = reinterpret_cast<int*>(base + b_hist);
  int* n_items = reinterpret_cast<int*>(base + 2 * b_hist);
  int2* agg = reinterpret_cast<int2*>(base + 2 * b_hist + 256);  // the items scan's CTA totals (<= 32)
  int32_t* pairs = reinterpret_cast<int32_t*>(base + 2 * b_hist + 512);
  int4* items = reinterpret_cast<int4*>(base + 2 * b_hist + 512 + b_pairs);
  int8_t* ql = reinterpret_cast<int8_t*>(base + 2 * b_hist + 512 + b_pairs + b_items);
  int64_t* gmin = reinterpret_cast<int64_t*>(base + 2 * b_hist + 512 + b_pairs + b_items + b_ql);
  int* flags = reinterpret_cast<int*>(gmin + npairs * ngroups);
  int64_t* trace = trace_cand ? trace_cand
                              : reinterpret_cast<int64_t*>(base + 2 * b_hist + 512 + b_pairs + b_items + b_ql + b_gmin);

  int dev = 0, sms = 148;
  e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, sizeof(int) * nlist, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(base, st);
    return e;
  }
  fx_limbs_kernel<<<static_cast<unsigned>(std::min<int64_t>((nq * s->dim + 255) / 256, 148 * 16)), 256, 0, st>>>(
      queries, nq, s->dim, ql);
  const unsigned pg = static_cast<unsigned>(std::min<int64_t>((npairs + 255) / 256, 4 * sms));
  pair_hist_kernel<<<pg, 256, 0, st>>>(lists, npairs, hist);
  e = launch_scan_items(hist, s->counts, nlist, kNTF, cur, items, n_items, agg, st);
  if (e == cudaSuccess) e = launch_pair_scatter(lists, npairs, nlist, cur, pairs, st);
  note_launch(4);
  if (e != cudaSuccess) {
    cudaFreeAsync(base, st);
    return e;
  }
  if (prof) prof(2, st);

  LmFxArgs a;
  a.nprobe = nprobe;
  a.L = L;
  a.Lp = s->lm_Lp;
  a.dim = s->dim;
  a.kp = kp;
  a.S = S;
  a.nb = nb;
  a.ngroups = ngroups;
  a.p_stride = p_stride;
  a.rows_x = static_cast<int64_t>(nlist) * s->lm_Lp;
  a.rows_q = nq;
  a.ql = ql;
  a.pairs = pairs;
  a.items = items;
  a.n_items = n_items;
  a.next_item = opt(V3DB_OPT_LM_STATIC) == 1 ? nullptr : n_items + 1;  // (zeroed by the items scan)
  a.ldist = ldist;
  a.counts = s->counts;
  a.pterm = s->pterm64;
  a.trace = trace;
  a.gmin = gmin;
  a.off_b = S * kAStageBytes;
  a.b_bytes = b_bytes;
  a.off_meta = a.off_b + nb * b_bytes;
  a.off_p = static_cast<uint32_t>(al(a.off_meta + nb * kNTF * 20, 16));
  a.off_stage = a.off_p + nb * 8 * p_stride;
  a.off_bar = static_cast<uint32_t>(al(a.off_stage + stage_bytes, 8));
  const size_t smem = smem_of(S);
  e = cudaFuncSetAttribute(lm_fx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) {
    const int64_t grid = std::min<int64_t>(sms, max_items);
    lm_fx_kernel<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(tmX, a);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = debug_sync(st, "lm_fx_kernel");
  if (prof) prof(3, st);
  if (e == cudaSuccess) {
    SelArgs<int64_t> sa;
    sa.nprobe = nprobe;
    sa.L = L;
    sa.ngroups = ngroups;
    sa.k = k;
    sa.lists = lists;
    sa.counts = s->counts;
    sa.ids = s->ids;
    sa.trace = trace;
    sa.gmin = gmin;
    sa.out_ids = out_ids;
    sa.out_dist = out_dist;
    e = launch_select(sa, nq, flags, st);
  }
  if (e == cudaSuccess) e = debug_sync(st, "lm_fx select kernels");
  cudaFreeAsync(base, st);
  return e;
}

}  // namespace v3db

#ifdef LM_EXP_TIMES
extern "C" int v3db_exp_lm_times(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, v3db::g_lm_times, sizeof(unsigned long long) * 512));
}
#endif

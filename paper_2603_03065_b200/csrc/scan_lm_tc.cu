// scan_lm_tc.cu -- the list-major Step 4 contraction on the 5th-gen tensor cores.
//
// One work item = one inverted list i and up to 128 of the (query, rank) pairs probing it.
// With xhat_{i,j} the slot's decoded reconstruction (concatenated codewords),
//   D_{i,j} = d_i + P_{i,j} - 2 <q, xhat_{i,j}>   (valid slot)      d_max  (padding)
// (DESIGN.md "LUT factorisation"), so per item the work is the int8 contraction
//   [128 pairs x D] (gathered queries)  .  [D x L] (decoded slots)  ->  int32 [128 x L]
// issued as tcgen05.mma.kind::i8, M=128, N=256 slots per chunk ("step"), K=32 per MMA.
//
// Warp roles (persistent CTA, one per SM):
//   warps 0-7   epilogue: TMEM -> registers (tcgen05.ld), D = d_i + P - 2 acc, padding
//               mask, trace row store, threshold emission (Step 5 candidates).
//               Thread (w%4)*32+lane owns one pair row; warps w and w+4 split 256 columns.
//   warps 8-15  producers: one step ahead, cp.async-prefetch the next item's query rows
//               (A, 128B-swizzled K-major, double-buffered), the next step's codes and
//               P_{i,j}; then write the step's pair metadata and DECODE its codes into the
//               128B-swizzled B operand directly in shared memory (warp per slot, lane per
//               codeword; the reconstruction never exists in HBM).
//   warp 16     one thread issues the MMAs and the tcgen05.commit arrivals.
// Pipelines (mbarriers): A [na] (full/empty), B stages (full/empty), accumulators (2 x 256
// TMEM columns, full/empty), per-step metadata ring [kRing] (full/empty).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "scan_lm_tc.cuh"
#include "tc_common.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

constexpr int kEW = 8, kPW = 8, kRing = 4;
constexpr int kStgWords = 36;  // epilogue staging row stride (words): conflict-free 16-B phases
constexpr int kThreads = 32 * (kEW + kPW + 1);
constexpr int kRows = 128, kChunk = 256, kPanel = 128;
constexpr uint32_t kAPanelBytes = kRows * kPanel, kBStageBytes = kChunk * kPanel;
constexpr int kProdBar = 2;  // named barrier among the producer warps (0 = __syncthreads)

struct Smem {  // offsets into the 1024-aligned dynamic shared memory
  uint32_t a, b, cb, codes, p, meta, info, stg, bars, end;
};

__host__ __device__ inline uint32_t codes_bytes(int M) { return (static_cast<uint32_t>(kChunk) * M + 15) & ~15u; }

__host__ __device__ inline Smem smem_layout(int kp, int na, int stages, int M, int Ks, int d, bool cb_in_smem) {
  Smem s;
  uint32_t o = 0;
  s.a = o;
  o += na * kp * kAPanelBytes;
  s.b = o;
  o += stages * kBStageBytes;
  s.cb = o;
  if (cb_in_smem) o += (static_cast<uint32_t>(M) * Ks * d + 15) & ~15u;
  s.codes = o;
  o += 3 * codes_bytes(M);  // ring of 3: prefetch(t+1) may not overwrite a buffer still being decoded
  s.p = o;
  o += kRing * kChunk * 4;
  s.meta = o;
  o += kRing * kRows * 16;
  s.info = o;
  o += kRing * 16;
  s.stg = o;
  o += kEW * 32 * kStgWords * 4;  // per epilogue warp: 32 rows x 32 values, transposed stores
  s.bars = o;
  o += 40 * 8;
  s.end = o;
  return s;
}

__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

struct Item {
  int li, p0, np, cnt;
};

__device__ __forceinline__ Item load_item(const LmTcArgs& a, int w) {
  const int4 v = a.items[w];
  return Item{v.x, v.y, v.z, v.w};
}

// Decode slots [0, nslots) x panel kp of a step: codes (shared) -> xhat rows of a B stage.
// Warp pw handles slots pw, pw+kPW, ...; lane l the l-th codeword of the panel.
template <int DS, bool CB_SMEM>
__device__ __forceinline__ void decode_panel(const LmTcArgs& a, const uint8_t* cds, const int8_t* cb, uint8_t* dst,
                                             int nslots, int kp, int pw, int lane) {
  const int kbeg = kp * kPanel;
  const int per = (min(a.dim, kbeg + kPanel) - kbeg) / DS;  // codewords of this panel (<= 32)
  if (lane >= per) return;
  const int m = kbeg / DS + lane;
  const int8_t* cbm = cb + static_cast<int64_t>(m) * a.Ks * DS;
  const int off = lane * DS;
  using W = typename std::conditional<DS == 4, uint32_t, typename std::conditional<DS == 8, uint2, uint4>::type>::type;
  for (int j = pw; j < nslots; j += 4 * kPW) {
    int c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = (j + u * kPW < nslots) ? cds[(j + u * kPW) * a.M + m] : 0;
    W w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      w[u] = CB_SMEM ? *reinterpret_cast<const W*>(cbm + c[u] * DS) : __ldg(reinterpret_cast<const W*>(cbm + c[u] * DS));
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j + u * kPW < nslots)
        *reinterpret_cast<W*>(dst + tc::sw128_offset(j + u * kPW, off >> 4) + (off & 15)) = w[u];
  }
}

// Any sub-block dimension: byte-wise decode.
__device__ __forceinline__ void decode_panel_generic(const LmTcArgs& a, const uint8_t* cds, const int8_t* cb,
                                                     uint8_t* dst, int nslots, int kp, int pt) {
  const int kbeg = kp * kPanel, w = min(a.dim, kbeg + kPanel) - kbeg;
  for (int e = pt; e < nslots * w; e += 32 * kPW) {
    const int j = e / w, u = e - j * w, col = kbeg + u;
    const int m = col / a.d;
    const int c = cds[j * a.M + m];
    dst[tc::sw128_offset(j, u >> 4) + (u & 15)] =
        static_cast<uint8_t>(cb[(static_cast<int64_t>(m) * a.Ks + c) * a.d + (col - m * a.d)]);
  }
}

template <int DS, bool CB_SMEM>
__global__ void __launch_bounds__(kThreads, 1) lm_tc_kernel(const LmTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const Smem SL = smem_layout(a.kp, a.na, a.stages, a.M, a.Ks, a.d, CB_SMEM);
  uint8_t* sA = smem + SL.a;
  uint8_t* sB = smem + SL.b;
  int8_t* sCB = reinterpret_cast<int8_t*>(smem + SL.cb);
  uint8_t* sCodes = smem + SL.codes;
  const uint32_t cbytes = codes_bytes(a.M);
  int32_t* sP = reinterpret_cast<int32_t*>(smem + SL.p);     // [kRing][256]
  int4* sMeta = reinterpret_cast<int4*>(smem + SL.meta);      // [kRing][128] (q, rank, d_i, tau_d)
  int4* sInfo = reinterpret_cast<int4*>(smem + SL.info);      // [kRing] (list, count, npairs, chunk)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL.bars);
  uint64_t* a_full = bars;            // [2]
  uint64_t* a_empty = bars + 2;       // [2]
  uint64_t* acc_full = bars + 4;      // [2]
  uint64_t* acc_empty = bars + 6;     // [2]
  uint64_t* pf_full = bars + 8;       // [kRing]
  uint64_t* pf_empty = bars + 12;     // [kRing]
  uint64_t* b_full = bars + 16;       // [stages <= 4]
  uint64_t* b_empty = bars + 20;      // [stages <= 4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 39);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int total_items = *a.n_items;
  const int my_items = total_items > static_cast<int>(blockIdx.x)
                           ? (total_items - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                           : 0;
  const int T = my_items * a.nchunk;  // steps of this CTA

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(a_full + s, 32 * kPW);
      tc::mbar_init(a_empty + s, 1);
      tc::mbar_init(acc_full + s, 1);
      tc::mbar_init(acc_empty + s, kEW);
    }
    for (int s = 0; s < kRing; ++s) {
      tc::mbar_init(pf_full + s, 32 * kPW);
      tc::mbar_init(pf_empty + s, kEW);
    }
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(b_full + s, 32 * kPW);
      tc::mbar_init(b_empty + s, 1);
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (CB_SMEM) {  // the whole codebook, once per CTA
    const int nb = a.M * a.Ks * a.d;
    for (int e = tid * 16; e < nb; e += kThreads * 16)
      *reinterpret_cast<uint4*>(sCB + e) = __ldg(reinterpret_cast<const uint4*>(a.cb + e));
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const int8_t* cb = CB_SMEM ? sCB : a.cb;

  if (warp >= kEW && warp < kEW + kPW) {
    // ================================ producers ================================
    const int pt = tid - 32 * kEW, pw = warp - kEW;  // 0..255, 0..7
    const int prow = pt & (kRows - 1), pseg = pt >> 7;  // A gather: row, segment parity
    Item cur{}, nxt{};
    int4 cur_pr = make_int4(-1, 0, 0, 0), nxt_pr = make_int4(-1, 0, 0, 0);  // (q, rank, d_i, tau)

    // gather item `it` (CTA-local index): pair row pt -> A buffer it % na (cp.async, zero-filled)
    auto gather_a = [&](int it, const Item& I, int4& pr) {
      const int ab = it % a.na, ause = it / a.na;
      pr = make_int4(-1, 0, 0, 0);
      if (prow < I.np) pr = a.pairs[I.p0 + prow];
      if (ause > 0) tc::mbar_wait(a_empty + ab, (ause - 1) & 1);
      if (prow < I.np) {
        const int8_t* qrow = a.queries + static_cast<int64_t>(pr.x) * a.dim;
        uint8_t* dstA = sA + ab * a.kp * kAPanelBytes;
        for (int seg = pseg; seg < a.kp * 8; seg += 2) {
          const int c0 = seg * 16;
          uint8_t* d = dstA + (seg >> 3) * kAPanelBytes + tc::sw128_offset(prow, seg & 7);
          if (a.dbg & 16) {
          } else if (a.q_vec) {
            tc::cp_async16(d, qrow + min(c0, a.dim - 16), c0 < a.dim ? 16 : 0);
          } else {
            for (int u = 0; u < 16; ++u) d[u] = (c0 + u < a.dim) ? static_cast<uint8_t>(qrow[c0 + u]) : 0;
          }
        }
      }
    };
    // codes and P of step t into sCodes[t % 3] / sP[t % kRing]
    auto prefetch_step = [&](int t, const Item& I) {
      const int nc = t % a.nchunk, slot = t % kRing, use = t / kRing;
      if (use > 0) tc::mbar_wait(pf_empty + slot, (use - 1) & 1);
      if (a.dbg & 32) return;
      const int j0 = nc * kChunk;
      const int64_t lbase = static_cast<int64_t>(I.li) * a.L;
      const int nslots = max(0, min(kChunk, I.cnt - j0));
      const int nbytes = nslots * a.M;
      const uint8_t* g = a.codes + (lbase + j0) * a.M;
      uint8_t* cds = sCodes + (t % 3) * cbytes;
      if (a.codes_vec) {
        for (int e = pt * 16; e < nbytes; e += 32 * kPW * 16) tc::cp_async16(cds + e, g + e, min(16, nbytes - e));
      } else {
        for (int e = pt; e < nbytes; e += 32 * kPW) cds[e] = g[e];
      }
      if (pt < kChunk / 4) {  // P_{i,j} for j0 .. j0+255 (clamped to the list)
        const int left = max(0, min(4, a.L - j0 - 4 * pt));
        int32_t* dp = sP + slot * kChunk + 4 * pt;
        if (a.p_vec && left > 0) {
          tc::cp_async16(dp, a.pterm + lbase + j0 + 4 * pt, 4 * left);
        } else {
          for (int u = 0; u < left; ++u) dp[u] = a.pterm[lbase + j0 + 4 * pt + u];
        }
      }
    };

    if (T > 0) {
      cur = load_item(a, blockIdx.x);
      gather_a(0, cur, cur_pr);
      prefetch_step(0, cur);
      tc::cp_async_commit();
    }
    int stage_ctr = 0;
    for (int t = 0; t < T; ++t) {
      const int it = t / a.nchunk, nc = t % a.nchunk, slot = t % kRing;
      // ---- prefetch step t+1 (and the next item's A when double-buffered)
      if (t + 1 < T) {
        const int it1 = (t + 1) / a.nchunk;
        if (it1 != it) {
          nxt = load_item(a, blockIdx.x + it1 * gridDim.x);
          if (a.na > 1) gather_a(it1, nxt, nxt_pr);
          prefetch_step(t + 1, nxt);
        } else {
          prefetch_step(t + 1, cur);
        }
        tc::cp_async_commit();
        tc::cp_async_wait<1>();
      } else {
        tc::cp_async_wait<0>();
      }
      if ((a.dbg & 8) && blockIdx.x == 0 && pt == 0 && t < 64) a.dbg_buf[t * 8 + 0] = clock64();
      bar_named(kProdBar, 32 * kPW);  // step t's codes / P (and A) have landed for every producer
      if ((a.dbg & 8) && blockIdx.x == 0 && pt == 0 && t < 64) a.dbg_buf[t * 8 + 1] = clock64();
      if (nc == 0) {
        tc::fence_async_smem();
        tc::mbar_arrive(a_full + (it % a.na));
      }
      // ---- step metadata for the epilogue
      if (pt < kRows) sMeta[slot * kRows + pt] = cur_pr;
      if (pt == 0) sInfo[slot] = make_int4(cur.li, cur.cnt, cur.np, nc);
      tc::mbar_arrive(pf_full + slot);
      // ---- decode the step, one K panel per B stage
      const int nslots = max(0, min(kChunk, cur.cnt - nc * kChunk));
      const uint8_t* cds = sCodes + (t % 3) * cbytes;
      for (int kp = 0; kp < a.kp; ++kp, ++stage_ctr) {
        const int s = stage_ctr % a.stages;
        if (stage_ctr >= a.stages) tc::mbar_wait(b_empty + s, ((stage_ctr / a.stages) - 1) & 1);
        uint8_t* dst = sB + s * kBStageBytes;
        if (a.dbg & 2) {
        } else if constexpr (DS > 0) decode_panel<DS, CB_SMEM>(a, cds, cb, dst, nslots, kp, pw, lane);
        else decode_panel_generic(a, cds, cb, dst, nslots, kp, pt);
        tc::fence_async_smem();
        tc::mbar_arrive(b_full + s);
      }
      if ((a.dbg & 8) && blockIdx.x == 0 && pt == 0 && t < 64) a.dbg_buf[t * 8 + 2] = clock64();
      // ---- move to the next item
      if (nc == a.nchunk - 1 && t + 1 < T) {
        cur = nxt;
        if (a.na > 1) {
          cur_pr = nxt_pr;
        } else {  // single A buffer: gather now (waits for this item's MMAs)
          gather_a(it + 1, cur, cur_pr);
          tc::cp_async_commit();
          tc::cp_async_wait<0>();
        }
      }
    }
  } else if (warp == kEW + kPW) {
    // ================================ MMA issuer ================================
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_s8(kRows, kChunk);
      int stage_ctr = 0;
      for (int t = 0; t < T; ++t) {
        const int it = t / a.nchunk, nc = t % a.nchunk, ab = t & 1, use = t >> 1;
        const int abuf = it % a.na;
        if (nc == 0) {
          tc::mbar_wait(a_full + abuf, (it / a.na) & 1);
          tc::fence_after_sync();
        }
        if (use > 0) {
          tc::mbar_wait(acc_empty + ab, (use - 1) & 1);
          tc::fence_after_sync();
        }
        for (int kp = 0; kp < a.kp; ++kp, ++stage_ctr) {
          const int s = stage_ctr % a.stages;
          tc::mbar_wait(b_full + s, (stage_ctr / a.stages) & 1);
          tc::fence_after_sync();
          const int nk = min(4, (a.dim - kp * kPanel + 31) / 32);
          const uint32_t aa = tc::smem_u32(sA + (abuf * a.kp + kp) * kAPanelBytes);
          const uint32_t ba = tc::smem_u32(sB + s * kBStageBytes);
          if (!(a.dbg & 256))
            for (int k = 0; k < nk; ++k)
              tc::mma_s8(tmem + ab * kChunk, tc::desc_sw128(aa + 32 * k), tc::desc_sw128(ba + 32 * k), idesc,
                         (kp | k) != 0);
          tc::mma_commit(b_empty + s);
        }
        tc::mma_commit(acc_full + ab);
        if (nc == a.nchunk - 1) tc::mma_commit(a_empty + abuf);
        if ((a.dbg & 8) && blockIdx.x == 0 && t < 64) a.dbg_buf[t * 8 + 3] = clock64();
      }
    }
  } else if (warp < kEW) {
    // ================================ epilogue ================================
    const int r = (warp & 3) * 32 + lane, half = warp >> 2;
    const bool vec_store = a.vec_store != 0;
    int32_t* stg = reinterpret_cast<int32_t*>(smem + SL.stg) + warp * 32 * kStgWords;
    for (int t = 0; t < T; ++t) {
      const int ab = t & 1, use = t >> 1, slot = t % kRing;
      tc::mbar_wait(pf_full + slot, (t / kRing) & 1);
      if ((a.dbg & 8) && blockIdx.x == 0 && tid == 0 && t < 64) a.dbg_buf[t * 8 + 4] = clock64();
      tc::mbar_wait(acc_full + ab, use & 1);
      tc::fence_after_sync();
      if ((a.dbg & 8) && blockIdx.x == 0 && tid == 0 && t < 64) a.dbg_buf[t * 8 + 5] = clock64();
      const int4 info = sInfo[slot];
      const int4 meta = sMeta[slot * kRows + r];
      const int li = info.x, cnt = info.y, np = info.z;
      const bool live = r < np;
      const int64_t lbase = static_cast<int64_t>(li) * a.L;
      int32_t* drow =
          (a.dst && live) ? a.dst + (static_cast<int64_t>(meta.x) * a.dst_nprobe + meta.y) * a.L : nullptr;
      const int32_t* P = sP + slot * kChunk;
      int nemit = 0;
#pragma unroll 1
      for (int b = 0; b < 4; ++b) {
        const int cl = half * 128 + b * 32;   // column within the step
        const int j0 = info.w * kChunk + cl;  // slot index
        if (j0 >= a.L) break;                 // warp-uniform
        uint32_t v[32];
        if (!(a.dbg & 128)) {
          tc::tmem_ld32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + ab * kChunk + cl, v);
          tc::tmem_ld_wait();
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u) v[u] = u;
        }
        if (!__any_sync(0xffffffffu, live)) continue;  // warp-uniform: no pair row of this warp is live
        int32_t D[32];
#pragma unroll
        for (int u = 0; u < 32; ++u)
          D[u] = (j0 + u < cnt) ? meta.z + P[cl + u] - 2 * static_cast<int>(v[u]) : kDMax;
        if (!(a.dbg & 1) && a.dst) {
          if (vec_store && j0 + 32 <= a.L) {
            // transpose through shared memory: each store instruction writes 4 full 128-B rows
#pragma unroll
            for (int u = 0; u < 32; u += 4)
              *reinterpret_cast<int4*>(stg + lane * kStgWords + u) = make_int4(D[u], D[u + 1], D[u + 2], D[u + 3]);
            __syncwarp();
            const int rl = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int row = 4 * i + rl;
              int32_t* rp = reinterpret_cast<int32_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(drow), row));
              const int4 val = *reinterpret_cast<const int4*>(stg + row * kStgWords + c4);
              if (rp) *reinterpret_cast<int4*>(rp + j0 + c4) = val;
            }
            __syncwarp();
          } else if (drow) {
#pragma unroll
            for (int u = 0; u < 32; ++u)
              if (j0 + u < a.L) drow[j0 + u] = D[u];
          }
        }
        if (a.emit && live) {
#pragma unroll
          for (int u = 0; u < 32; ++u) nemit += (j0 + u < cnt && D[u] <= meta.w) ? 1 : 0;
        }
      }
      // Step 5 candidates of this row: one atomic for the step, then re-read TMEM (warp-wide,
      // tcgen05.ld is .sync.aligned) to write them as (D << 32 | list * L + slot).
      const bool mine = a.emit && live && nemit > 0 && !(a.dbg & 4);
      if (__any_sync(0xffffffffu, mine)) {
        int pos = mine ? atomicAdd(a.cand_cnt + meta.x, nemit) : 0;
        uint64_t* dstc = a.cand_buf + (mine ? static_cast<int64_t>(meta.x) * a.cap : 0);
        const uint32_t slot_base = static_cast<uint32_t>(lbase) + static_cast<uint32_t>(info.w * kChunk);
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
          const int cl = half * 128 + b * 32;
          const int j0 = info.w * kChunk + cl;
          if (j0 >= a.L) break;  // warp-uniform
          uint32_t v[32];
          tc::tmem_ld32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + ab * kChunk + cl, v);
          tc::tmem_ld_wait();
          if (!mine) continue;
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int Dv = meta.z + P[cl + u] - 2 * static_cast<int>(v[u]);
            if (j0 + u < cnt && Dv <= meta.w) {
              if (pos < a.cap) dstc[pos] = (static_cast<uint64_t>(static_cast<uint32_t>(Dv)) << 32) | (slot_base + cl + u);
              ++pos;
            }
          }
        }
      }
      if ((a.dbg & 8) && blockIdx.x == 0 && tid == 0 && t < 64) a.dbg_buf[t * 8 + 6] = clock64();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(acc_empty + ab);
        tc::mbar_arrive(pf_empty + slot);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

template <int DS, bool CBS>
cudaError_t launch_variant(const LmTcArgs& a, size_t smem, int grid, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(lm_tc_kernel<DS, CBS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  lm_tc_kernel<DS, CBS><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool lm_tc_config(const v3db_snapshot* s, LmTcArgs* a, size_t* smem_bytes) {
  a->dim = s->dim;
  a->kp = (s->dim + kPanel - 1) / kPanel;
  a->M = s->M;
  a->Ks = s->Ks;
  a->d = s->d;
  a->L = s->L;
  a->nlist = s->nlist;
  a->nchunk = (s->L + kChunk - 1) / kChunk;
  const size_t budget = 225 * 1024;
  const char* fst = getenv("V3DB_LM_STAGES");  // performance / debugging override
  const int st_max = fst ? atoi(fst) : 4;
  for (int na = 2; na >= 1; --na)
    for (int cbs = 1; cbs >= 0; --cbs)
      for (int st = st_max; st >= 2; --st) {
        const Smem L = smem_layout(a->kp, na, st, s->M, s->Ks, s->d, cbs != 0);
        if (L.end + 1024 <= budget) {
          a->na = na;
          a->stages = st;
          a->cb_in_smem = cbs;
          *smem_bytes = L.end + 1024;
          return true;
        }
      }
  return false;
}

cudaError_t launch_lm_tc(const LmTcArgs& a_in, size_t smem, cudaStream_t st) {
  LmTcArgs a = a_in;
  const char* dbg = getenv("V3DB_LM_DEBUG");
  a.dbg = dbg ? atoi(dbg) : 0;
  a.dbg_buf = nullptr;
  if (a.dbg & 8) cudaMalloc(&a.dbg_buf, 64 * 8 * sizeof(long long));
  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const bool cbs = a.cb_in_smem != 0;
  const int DS = (a.d == 4 || a.d == 8 || a.d == 16) ? a.d : 0;
  if (DS == 4) e = cbs ? launch_variant<4, true>(a, smem, sms, st) : launch_variant<4, false>(a, smem, sms, st);
  else if (DS == 8) e = cbs ? launch_variant<8, true>(a, smem, sms, st) : launch_variant<8, false>(a, smem, sms, st);
  else if (DS == 16) e = cbs ? launch_variant<16, true>(a, smem, sms, st) : launch_variant<16, false>(a, smem, sms, st);
  else e = cbs ? launch_variant<0, true>(a, smem, sms, st) : launch_variant<0, false>(a, smem, sms, st);
  note_launch();
  if (a.dbg_buf) {  // performance experiment: dump CTA 0's step timeline
    long long h[64 * 8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, a.dbg_buf, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(a.dbg_buf);
    static int call = 0;
    char name[64];
    snprintf(name, sizeof(name), "gpurun_out/lm_timeline_%d.txt", call++);
    if (FILE* f = fopen(name, "w")) {
      for (int t = 0; t < 64; ++t) {
        for (int c = 0; c < 7; ++c) fprintf(f, "%lld ", h[t * 8 + c] - h[0]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  return e;
}

}  // namespace v3db

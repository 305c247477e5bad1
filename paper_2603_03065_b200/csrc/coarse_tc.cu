// coarse_tc.cu -- Steps 1-2 (and the build's B2 ranking) on the 5th-gen tensor cores.
//
//   d_i = dist(x, mu_i) = ||x||^2 + ||mu_i||^2 - 2 <x, mu_i>
//   out = the R smallest (d_i, i), ascending                          (R9)
//
// <x, mu_i> is an int8 contraction [rows x D] . [D x nlist] -> int32 (exact), issued as
// tcgen05.mma.kind::i8 (M=128 rows, N=256 centroids, K=32) with both operands brought into
// 128B-swizzled shared memory by TMA and the accumulators in TMEM (two 256-column buffers,
// so the epilogue of one centroid chunk overlaps the MMAs of the next).  Warp 4 is the
// TMA producer + single-thread MMA issuer; warps 0-7 are the epilogue: thread (w%4)*32+lane
// owns one row, warps w and w+4 split the 256 columns of a chunk.
//
// Exact top-R without materialising the [rows x nlist] distance matrix, in two passes of
// the (cheap) contraction:
//   pass 1: per row, the minimum distance of every group of G consecutive lists
//           (ngroups = nlist/G >= 2R);  tau_row = the R-th smallest group minimum.
//           tau_row >= the row's true R-th smallest distance (R distinct lists reach it).
//   pass 2: every (d_i, i) with d_i <= tau_row is appended to the row's candidate list
//           (at least R of them, typically a few R).
//   select: the exact R smallest (d, i) keys of the candidates (warp top-k, topk.cuh).
// A row whose candidate list overflows (pathological ties) is recomputed by a plain SIMT
// kernel.  Shapes the TMA path does not cover (dim % 16 != 0, dim > 768) use the mma.sync
// kernel of coarse_topk.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "tc_common.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {

cudaError_t coarse_topk_mma(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* cnorm, int nlist,
                            int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st);

namespace {

constexpr int kRows = 128;        // rows per tile (UMMA M)
constexpr int kChunk = 256;       // centroids per MMA chunk (UMMA N)
constexpr int kPanel = 128;       // bytes of K per swizzled panel
constexpr int kEpiWarps = 16;     // epilogue: warp w -> TMEM lanes 32*(w%4), columns 64*(w/4) of a chunk
constexpr int kProdWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr uint32_t kAPanelBytes = kRows * kPanel;     // 16 KB
constexpr uint32_t kBStageBytes = kChunk * kPanel;    // 32 KB

struct CoarseArgs {
  int64_t n, items;  // rows, work items (row tile x chunk)
  int dim, nlist, kp, stages, nchunks, G, ngroups, capc;
  const int8_t* X;
  const int32_t* cnorm;
  int32_t* gmin;        // pass 1: [n][ngroups] group-minimum distances
  const int32_t* tau;   // pass 2: [n] threshold distance
  uint64_t* cand;       // pass 2: [n][capc] candidate keys
  int* ccnt;            // pass 2: [n] candidate counts
};

// Persistent: CTA b owns the contiguous work items [b*per, (b+1)*per) of the row-major
// (row tile, chunk) order, so a CTA switches row tiles at most a few times.  Warp 16 issues the
// TMA loads (A once per row tile, B per (chunk, K panel) into a ring), warp 17 issues the MMAs
// into two TMEM accumulators, warps 0-15 run the epilogue (TMEM -> registers -> distances).
// GT: compile-time group size (32, 16, 8, 4) or 0 = runtime a.G (any power of two <= 32).
template <int PASS, int GT>
__global__ void __launch_bounds__(kThreads, 1) coarse_tc_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                const __grid_constant__ CUtensorMap tmMu,
                                                                const CoarseArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array (an integer round trip would
  // make every access through `smem` a generic-address LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                   // kp panels of [128][128]
  uint8_t* sB = smem + a.kp * kAPanelBytes;             // stages of [256][128]
  int* sCn = reinterpret_cast<int*>(sB + a.stages * kBStageBytes);  // [kEpiWarps][64] ||mu||^2
  uint64_t* bars = reinterpret_cast<uint64_t*>(sCn + kEpiWarps * 64);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 1;
  uint64_t* full = bars + 2;                            // [stages]
  uint64_t* empty = full + a.stages;                    // [stages]
  uint64_t* accf = empty + a.stages;                    // [2]
  uint64_t* acce = accf + 2;                            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t per = (a.items + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per, i1 = min(a.items, i0 + per);

  if (tid == 0) {
    tc::mbar_init(a_full, 1);
    tc::mbar_init(a_empty, 1);
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(accf + s, 1);
      tc::mbar_init(acce + s, kEpiWarps);
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProdWarp) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0 && i0 < i1) {
      tc::tma_prefetch(&tmX);
      tc::tma_prefetch(&tmMu);
      int64_t cur_rt = -1;
      int nA = 0, s = 0, u = 0;  // A loads so far; B stage index / ring pass
      for (int64_t it = i0; it < i1; ++it) {
        const int64_t rt = it / a.nchunks;
        const int c = static_cast<int>(it - rt * a.nchunks);
        if (rt != cur_rt) {
          if (nA > 0) tc::mbar_wait(a_empty, (nA - 1) & 1);  // every MMA reading the old tile is done
          tc::mbar_expect_tx(a_full, a.kp * kAPanelBytes);
          for (int p = 0; p < a.kp; ++p) tc::tma_load_2d(sA + p * kAPanelBytes, &tmX, a_full, p * kPanel, (int)(rt * kRows));
          ++nA;
          cur_rt = rt;
        }
        for (int p = 0; p < a.kp; ++p) {
          if (u > 0) tc::mbar_wait(empty + s, (u - 1) & 1);
          tc::mbar_expect_tx(full + s, kBStageBytes);
          tc::tma_load_2d(sB + s * kBStageBytes, &tmMu, full + s, p * kPanel, c * kChunk);
          if (++s == a.stages) {
            s = 0;
            ++u;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && i0 < i1) {
      constexpr uint32_t idesc = tc::idesc_s8(kRows, kChunk);
      int64_t cur_rt = -1;
      int nA = 0, s = 0, u = 0;
      for (int64_t it = i0; it < i1; ++it) {
        const int64_t rt = it / a.nchunks;
        const int j = static_cast<int>(it - i0), acc = j & 1, use = j >> 1;
        if (rt != cur_rt) {
          tc::mbar_wait(a_full, nA & 1);
          tc::fence_after_sync();
          ++nA;
          cur_rt = rt;
        }
        if (use > 0) {  // the epilogue drained this accumulator
          tc::mbar_wait(acce + acc, (use - 1) & 1);
          tc::fence_after_sync();
        }
        for (int p = 0; p < a.kp; ++p) {
          tc::mbar_wait(full + s, u & 1);
          tc::fence_after_sync();
          const int nk = min(4, (a.dim - p * kPanel + 31) / 32);
          const uint32_t a_addr = tc::smem_u32(sA + p * kAPanelBytes);
          const uint32_t b_addr = tc::smem_u32(sB + s * kBStageBytes);
          for (int k = 0; k < nk; ++k)
            tc::mma_s8(tmem + acc * kChunk, tc::desc_sw128(a_addr + k * 32), tc::desc_sw128(b_addr + k * 32), idesc,
                       (p | k) != 0);
          tc::mma_commit(empty + s);
          if (++s == a.stages) {
            s = 0;
            ++u;
          }
        }
        tc::mma_commit(accf + acc);
        // last item of this row tile in our range: the A buffer is free once these MMAs finish
        if (it + 1 == i1 || (it + 1) / a.nchunks != rt) tc::mma_commit(a_empty);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-15)
    const int q = warp & 3, h = warp >> 2;       // TMEM lane quadrant, 64-column quarter
    const int r = q * 32 + lane;                  // row within the tile
    int* cn = sCn + warp * 64;
    int64_t cur_rt = -1;
    int xn = 0, tau_d = 0;
    int64_t row = 0;
    bool live = false;
    for (int64_t it = i0; it < i1; ++it) {
      const int64_t rt = it / a.nchunks;
      const int c = static_cast<int>(it - rt * a.nchunks);
      const int j = static_cast<int>(it - i0), acc = j & 1, use = j >> 1;
      const int col0 = c * kChunk + h * 64;       // first list of this warp's 64 columns
      // ||mu||^2 of the 64 columns (warp-uniform per column: read back as broadcasts)
      __syncwarp();
      if constexpr (PASS == 3) {  // packed column terms 32 ||mu_i||^2 + (i mod 32); padding: +inf
        cn[lane] = col0 + lane < a.nlist ? 32 * __ldg(a.cnorm + col0 + lane) + lane : 0x7fffffff;
        cn[lane + 32] = col0 + 32 + lane < a.nlist ? 32 * __ldg(a.cnorm + col0 + 32 + lane) + lane : 0x7fffffff;
      } else {
        cn[lane] = col0 + lane < a.nlist ? __ldg(a.cnorm + col0 + lane) : 0;
        cn[lane + 32] = col0 + 32 + lane < a.nlist ? __ldg(a.cnorm + col0 + 32 + lane) : 0;
      }
      if (rt != cur_rt) {  // ||x||^2 of this thread's row (from global: the A tile may be reloaded)
        cur_rt = rt;
        row = rt * kRows + r;
        live = row < a.n;
        xn = 0;
        if (live && PASS != 3) {
          const int8_t* xr = a.X + row * a.dim;
          for (int u2 = 0; u2 < a.dim; u2 += 4) {
            const int v = *reinterpret_cast<const int*>(xr + u2);
            xn = __dp4a(v, v, xn);
          }
          if (PASS == 2) tau_d = a.tau[row];
        }
      }
      tc::mbar_wait_sleep(accf + acc, use & 1);
      tc::fence_after_sync();
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * kChunk + h * 64;
      const bool work = live && col0 < a.nlist;
      int gacc = 0x7fffffff;  // GT == 0 with G > 4: running minimum across the 4-element folds
      // In place: v[u] <- e = ||mu||^2 - 2 <x, mu> of one 32-column block (d = xn + e); padded
      // columns -> +inf.  Then Pass 1 stores group minima, Pass 2 appends candidates d <= tau.
      auto block = [&](int cb) {
        const int4* c4 = reinterpret_cast<const int4*>(cn + cb);
#pragma unroll
        for (int u4 = 0; u4 < 8; ++u4) {
          const int4 cc = c4[u4];
          v[4 * u4] = static_cast<uint32_t>(cc.x - 2 * static_cast<int>(v[4 * u4]));
          v[4 * u4 + 1] = static_cast<uint32_t>(cc.y - 2 * static_cast<int>(v[4 * u4 + 1]));
          v[4 * u4 + 2] = static_cast<uint32_t>(cc.z - 2 * static_cast<int>(v[4 * u4 + 2]));
          v[4 * u4 + 3] = static_cast<uint32_t>(cc.w - 2 * static_cast<int>(v[4 * u4 + 3]));
        }
        if (col0 + cb + 32 > a.nlist) {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (col0 + cb + u >= a.nlist) v[u] = 0x7fffffffu;
        }
        auto E = [&](int u) { return static_cast<int>(v[u]); };
        if constexpr (PASS == 1) {
          if constexpr (GT > 0) {
#pragma unroll
            for (int g0 = 0; g0 < 32; g0 += GT) {
              int best = min(min(E(g0), E(g0 + 1)), min(E(g0 + 2), E(g0 + 3)));
#pragma unroll
              for (int u = 4; u < GT; u += 2) best = min(best, min(E(g0 + u), E(g0 + u + 1)));
              const int gstart = col0 + cb + g0;
              if (gstart < a.nlist) a.gmin[row * a.ngroups + gstart / GT] = best + xn;
            }
          } else {
            const int G = a.G;  // any power of two <= 32
            for (int u = 0; u < 32; ++u) {
              gacc = min(gacc, E(u));
              if (((u + 1) & (G - 1)) == 0) {
                const int gstart = col0 + cb + u + 1 - G;
                if (gstart < a.nlist) a.gmin[row * a.ngroups + gstart / G] = gacc + xn;
                gacc = 0x7fffffff;
              }
            }
          }
        } else {
          // a block whose minimum is above tau has no candidate (the common case); otherwise one
          // atomic reserves room for all of the block's candidates
          int mn = min(min(E(0), E(1)), min(E(2), E(3)));
#pragma unroll
          for (int u = 4; u < 32; u += 2) mn = min(mn, min(E(u), E(u + 1)));
          const int lim = tau_d - xn;
          if (mn <= lim) {
            uint32_t mask = 0;
#pragma unroll
            for (int u = 0; u < 32; ++u) mask |= (E(u) <= lim ? 1u : 0u) << u;
            int pos = atomicAdd(a.ccnt + row, __popc(mask));
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              if ((mask >> u) & 1u) {
                if (pos < a.capc) a.cand[row * a.capc + pos] = step2_key(E(u) + xn, col0 + cb + u);
                ++pos;
              }
            }
          }
        }
      };
      if constexpr (PASS == 3) {
        // packed key p = 32 e + (i mod 32), e = ||mu_i||^2 - 2 <x, mu_i> = d_i - ||x||^2 (exact:
        // |32 e| < 2^31 for dim <= 1024; padding columns: acc = 0, p = +inf); per 32-list block the
        // KB = GT smallest keys (an insertion network: 2 KB - 1 IMNMX per column)
        constexpr int KB = GT;
        static_assert(KB == 2 || KB == 4 || KB == 8, "keys per block");
        int m[2][KB];
        auto topk = [&](int cb, int(&mk)[KB]) {
          const int4* c4 = reinterpret_cast<const int4*>(cn + cb);
#pragma unroll
          for (int z = 0; z < KB; ++z) mk[z] = 0x7fffffff;
#pragma unroll
          for (int u4 = 0; u4 < 8; ++u4) {
            const int4 cc = c4[u4];
            const int cw[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              int t = cw[w] - 64 * static_cast<int>(v[4 * u4 + w]);
#pragma unroll
              for (int z = 0; z < KB - 1; ++z) {
                const int hi = max(mk[z], t);
                mk[z] = min(mk[z], t);
                t = hi;
              }
              mk[KB - 1] = min(mk[KB - 1], t);
            }
          }
        };
        tc::tmem_ld32(taddr, v);
        tc::tmem_ld_wait();
        topk(0, m[0]);
        tc::tmem_ld32(taddr + 32, v);
        tc::tmem_ld_wait();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(acce + acc);  // accumulator columns consumed
        topk(32, m[1]);
        if (live) {  // blocks 8c + 2h and 8c + 2h + 1 of the row: their KB smallest keys each
          int4* dst = reinterpret_cast<int4*>(a.gmin + KB * (row * a.ngroups + c * 8 + h * 2));
          if constexpr (KB == 2) {
            dst[0] = make_int4(m[0][0], m[0][1], m[1][0], m[1][1]);
          } else if constexpr (KB == 4) {
            dst[0] = make_int4(m[0][0], m[0][1], m[0][2], m[0][3]);
            dst[1] = make_int4(m[1][0], m[1][1], m[1][2], m[1][3]);
          } else {
            dst[0] = make_int4(m[0][0], m[0][1], m[0][2], m[0][3]);
            dst[1] = make_int4(m[0][4], m[0][5], m[0][6], m[0][7]);
            dst[2] = make_int4(m[1][0], m[1][1], m[1][2], m[1][3]);
            dst[3] = make_int4(m[1][4], m[1][5], m[1][6], m[1][7]);
          }
        }
        continue;
      }
      // two 32-column TMEM loads, processed one after the other (32 live registers)
      tc::tmem_ld32(taddr, v);
      tc::tmem_ld_wait();
      if (work) block(0);
      tc::tmem_ld32(taddr + 32, v);
      tc::tmem_ld_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acce + acc);  // accumulator columns consumed
      if (work) block(32);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// tau_row = the R-th smallest of the row's group minima (exact 4-pass radix select, one warp per
// row); resets the candidate counters.  >= the row's true R-th smallest distance: R distinct lists
// reach it.  Fewer than R groups: no filtering.
__global__ void __launch_bounds__(256) tau_kernel(int64_t n, int ngroups, int R, const int32_t* __restrict__ gmin,
                                                 int32_t* __restrict__ tau, int* __restrict__ ccnt) {
  __shared__ int hist[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= n) return;
  int* hw = hist[warp];
  const int32_t* g = gmin + row * ngroups;
  if (ngroups < R) {
    if (lane == 0) {
      tau[row] = 0x7fffffff;
      ccnt[row] = 0;
    }
    return;
  }
  uint32_t prefix = 0;
  int kk = R;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int b = lane; b < 256; b += 32) hw[b] = 0;
    __syncwarp();
    for (int i = lane; i < ngroups; i += 32) {
      const uint32_t v = static_cast<uint32_t>(g[i]);
      if (pass == 0 || (v >> (shift + 8)) == prefix) atomicAdd(&hw[(v >> shift) & 255], 1);
    }
    __syncwarp();
    int hb[8], sum = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      hb[b] = hw[lane * 8 + b];
      sum += hb[b];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int cum = incl - sum, bin = -1, newk = 0;
    if (cum < kk && kk <= incl) {
      bin = lane * 8;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        if (cum + hb[b] >= kk) break;
        cum += hb[b];
        ++bin;
      }
      newk = kk - cum;
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, bin >= 0)) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    kk = __shfl_sync(0xffffffffu, newk, src);
    __syncwarp();
    prefix = (prefix << 8) | static_cast<uint32_t>(bin);
  }
  if (lane == 0) {
    tau[row] = static_cast<int32_t>(prefix);
    ccnt[row] = 0;
  }
}

// Exact R smallest candidate keys per row; rows whose list overflowed are flagged.
template <int KR>
__global__ void __launch_bounds__(256) select_kernel(int64_t n, int R, int capc, const uint64_t* __restrict__ cand,
                                                    const int* __restrict__ ccnt, int32_t* __restrict__ out_idx,
                                                    int32_t* __restrict__ out_dist, int* __restrict__ flags,
                                                    int* __restrict__ hist) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= n) return;
  const int cnt = ccnt[row];
  if (cnt > capc) {
    if (lane == 0) flags[row] = 1;
    return;
  }
  if (lane == 0) flags[row] = 0;
  WarpTopK<KR> top;
  top.init(R);
  const uint64_t* c = cand + row * capc;
  for (int b = 0; b < cnt; b += 32) top.offer((b + lane < cnt) ? c[b + lane] : ~0ull);
  top.store([&](int j, uint64_t key) {
    out_idx[row * R + j] = static_cast<int32_t>(key & 0xffffffffu);
    out_dist[row * R + j] = static_cast<int32_t>(key >> 32);
    if (hist) atomicAdd(hist + static_cast<uint32_t>(key), 1);
  });
}

// Plain exact recomputation of flagged rows (warp per row, all nlist distances).
template <int KR>
__global__ void __launch_bounds__(256) fallback_kernel(const int8_t* __restrict__ X, int64_t n, int dim,
                                                      const int8_t* __restrict__ mu, int nlist, int R,
                                                      const int* __restrict__ flags, int32_t* __restrict__ out_idx,
                                                      int32_t* __restrict__ out_dist, int* __restrict__ hist) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= n || flags[row] == 0) return;
  WarpTopK<KR> top;
  top.init(R);
  const int8_t* x = X + row * dim;
  for (int b = 0; b < nlist; b += 32) {
    uint64_t key = ~0ull;
    const int i = b + lane;
    if (i < nlist) {
      const int8_t* m = mu + static_cast<int64_t>(i) * dim;
      int d = 0;
      for (int u = 0; u < dim; ++u) {
        const int df = static_cast<int>(x[u]) - static_cast<int>(m[u]);
        d += df * df;
      }
      key = step2_key(d, i);
    }
    top.offer(key);
  }
  top.store([&](int j, uint64_t key) {
    out_idx[row * R + j] = static_cast<int32_t>(key & 0xffffffffu);
    out_dist[row * R + j] = static_cast<int32_t>(key >> 32);
    if (hist) atomicAdd(hist + static_cast<uint32_t>(key), 1);
  });
}

__global__ void list_hist_kernel(const int32_t* __restrict__ idx, int64_t n, int* __restrict__ hist) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(hist + __ldg(idx + p), 1);
}

// Step 2 from the group minima (one warp per row): tau = the R-th smallest group minimum (exact
// radix select; >= the row's R-th smallest distance, R distinct lists reach it), then the lists
// of every group whose minimum is <= tau -- and only those -- get their exact distance
// ||x||^2 + ||mu_i||^2 - 2 <x, mu_i> recomputed (dp4a against the L2-resident centroids) and the R
// smallest (d, i) keys kept (warp top-k, the total order R9).  A row with more than kPickCap
// selected groups (massive ties) recomputes every list.  Replaces the second contraction pass.
constexpr int kPickCap = 512;   // selected groups per row
template <int KR>
__global__ void __launch_bounds__(256) pick_kernel(const int8_t* __restrict__ X, int64_t n, int dim,
                                                  const int8_t* __restrict__ mu, const int32_t* __restrict__ cnorm,
                                                  int nlist, int G, int ngroups, int R,
                                                  const int32_t* __restrict__ gmin, int32_t* __restrict__ out_idx,
                                                  int32_t* __restrict__ out_dist, int* __restrict__ hist) {
  extern __shared__ __align__(16) uint8_t psm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  int* wh = reinterpret_cast<int*>(psm) + warp * 256;                       // [8][256] radix histograms
  int* sel = reinterpret_cast<int*>(psm) + 8 * 256 + warp * kPickCap;       // [8][kPickCap] groups
  int4* xs = reinterpret_cast<int4*>(psm + 4 * (8 * 256 + 8 * kPickCap)) + warp * (dim >> 4);  // [8][dim]
  if (row >= n) return;
  const int32_t* g = gmin + row * ngroups;
  const int8_t* x = X + row * dim;
  for (int u = lane; u < (dim >> 4); u += 32) xs[u] = *reinterpret_cast<const int4*>(x + 16 * u);
  int xn = 0;
  for (int u = lane; u < (dim >> 2); u += 32) {
    const int v = *reinterpret_cast<const int*>(x + 4 * u);
    xn = __dp4a(v, v, xn);
  }
  xn = __reduce_add_sync(0xffffffffu, xn);
  // tau >= the R-th smallest group minimum: linear 256-bin histograms over [lo, hi] of the row's
  // group minima, refined inside the bin that holds rank R until it holds <= 8 or is one value
  // wide; tau = that bin's upper edge.  Fewer groups than R: every list.
  uint32_t tau = 0xffffffffu;
  if (ngroups >= R) {
    int mn = 0x7fffffff, mx = 0;
    for (int i = lane; i < ngroups; i += 32) {
      const int v = g[i];
      mn = min(mn, v);
      mx = max(mx, v);
    }
    uint32_t lo = static_cast<uint32_t>(__reduce_min_sync(0xffffffffu, mn));
    uint32_t span = static_cast<uint32_t>(__reduce_max_sync(0xffffffffu, mx)) - lo + 1u;
    int kk = R;
    for (;;) {
      const int bits = 32 - __clz((span - 1u) | 1u);
      const int sh = bits > 8 ? bits - 8 : 0;
      for (int b = lane; b < 256; b += 32) wh[b] = 0;
      __syncwarp();
      for (int i = lane; i < ngroups; i += 32) {
        const uint32_t v = static_cast<uint32_t>(g[i]) - lo;
        if (v < span) atomicAdd(&wh[v >> sh], 1);
      }
      __syncwarp();
      int hb[8], sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        hb[b] = wh[lane * 8 + b];
        sum += hb[b];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int cum = incl - sum, bin = -1, newk = 0, cb = 0;
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
        newk = kk - cum;
      }
      const int src = __ffs(__ballot_sync(0xffffffffu, bin >= 0)) - 1;
      bin = __shfl_sync(0xffffffffu, bin, src);
      kk = __shfl_sync(0xffffffffu, newk, src);
      cb = __shfl_sync(0xffffffffu, cb, src);
      __syncwarp();
      lo += static_cast<uint32_t>(bin) << sh;
      span = 1u << sh;
      if (sh == 0 || cb <= 8) break;
    }
    tau = lo + span - 1u;
  }
  // the selected groups
  int nsel = 0;
  for (int i0 = 0; i0 < ngroups; i0 += 32) {
    const int i = i0 + lane;
    const bool take = i < ngroups && static_cast<uint32_t>(g[i]) <= tau;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    const int pos = nsel + __popc(bal & ((1u << lane) - 1u));
    if (take && pos < kPickCap) sel[pos] = i;
    nsel += __popc(bal);
  }
  __syncwarp();
  const bool all = nsel > kPickCap;  // massive ties: recompute every list
  const int ncand = all ? nlist : nsel * G, lgG = 31 - __clz(G);
  WarpTopK<KR> top;
  top.init(R);
  auto list_at = [&](int c) {
    if (c >= ncand) return -1;
    const int i = all ? c : (sel[c >> lgG] << lgG) + (c & (G - 1));  // G is a power of two
    return i < nlist ? i : -1;
  };
  for (int c0 = 0; c0 < ncand; c0 += 64) {  // two candidate lists per lane: their loads interleave
    const int i0 = list_at(c0 + lane), i1 = list_at(c0 + 32 + lane);
    const int4* m0 = reinterpret_cast<const int4*>(mu + static_cast<int64_t>(max(i0, 0)) * dim);
    const int4* m1 = reinterpret_cast<const int4*>(mu + static_cast<int64_t>(max(i1, 0)) * dim);
    int d0 = 0, d1 = 0;
    const int c0n = i0 >= 0 ? __ldg(cnorm + i0) : 0, c1n = i1 >= 0 ? __ldg(cnorm + i1) : 0;
    for (int u = 0; u < (dim >> 4); ++u) {
      const int4 a = xs[u];
      const int4 b0 = i0 >= 0 ? __ldg(m0 + u) : make_int4(0, 0, 0, 0);
      const int4 b1 = i1 >= 0 ? __ldg(m1 + u) : make_int4(0, 0, 0, 0);
      d0 = __dp4a(a.x, b0.x, __dp4a(a.y, b0.y, __dp4a(a.z, b0.z, __dp4a(a.w, b0.w, d0))));
      d1 = __dp4a(a.x, b1.x, __dp4a(a.y, b1.y, __dp4a(a.z, b1.z, __dp4a(a.w, b1.w, d1))));
    }
    d0 = xn + c0n - 2 * d0;
    d1 = xn + c1n - 2 * d1;
    const bool open = all || ngroups < R;
    top.offer(i0 >= 0 && (open || static_cast<uint32_t>(d0) <= tau) ? step2_key(d0, i0) : ~0ull);
    top.offer(i1 >= 0 && (open || static_cast<uint32_t>(d1) <= tau) ? step2_key(d1, i1) : ~0ull);
  }
  top.store([&](int j, uint64_t key) {
    out_idx[row * R + j] = static_cast<int32_t>(key & 0xffffffffu);
    out_dist[row * R + j] = static_cast<int32_t>(key >> 32);
    if (hist) atomicAdd(hist + static_cast<uint32_t>(key), 1);
  });
}

// Step 2 from the single contraction pass (PASS 3), one warp per row.  S = the stored keys, the
// two smallest of every block of 32 consecutive lists.  tau >= the R-th smallest e over S (linear-bin
// histogram refinement as in pick_kernel), hence >= the row's true R-th smallest e.  A list of the
// row's true top R that is not in S lies in a block whose two stored keys are both below it, so that
// block's second key has e <= tau: every such block is recomputed exactly (dp4a against the
// L2-resident centroids).  The candidates -- stored keys with e <= tau outside the recomputed
// blocks, and the recomputed lists with e <= tau -- contain the true top R, which is ranked on
// (d_i, i) (R9).  A row whose candidates or recomputed blocks overflow the caches is ranked by brute
// force over every list (the same warp).
constexpr int kMergeWarps = 4;
constexpr int kRecCap = 32;  // recomputed blocks per row
__device__ __forceinline__ uint64_t merge_key(int e, int i) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(e + (1 << 30))) << 32) | static_cast<uint32_t>(i);
}
// NV: int4 per lane held in registers: KB = 2 keys per block -> two blocks per int4 (nblk / 2 <= 32 NV);
// KB = 4 -> one block per int4 (nblk <= 32 NV); KB = 8 -> half a block per int4 (2 nblk <= 32 NV).
// KB >= R: every list of the row's true top R is among the stored keys (a list missing from its block
// has KB >= R smaller keys in that block alone), so no block is recomputed.
template <int KR, int NV, int KB>
#ifndef V3DB_MERGE_MINB
#define V3DB_MERGE_MINB 1
#endif
__global__ void __launch_bounds__(32 * kMergeWarps, V3DB_MERGE_MINB) merge_kernel(const int8_t* __restrict__ X, int64_t n, int dim,
                                                                const int8_t* __restrict__ mu,
                                                                const int32_t* __restrict__ cnorm, int nlist,
                                                                int nblk, int R, int cap,
                                                                const int32_t* __restrict__ bk,
                                                                int32_t* __restrict__ out_idx,
                                                                int32_t* __restrict__ out_dist, int* __restrict__ hist) {
  extern __shared__ __align__(16) uint8_t msm[];
  constexpr unsigned kFull = 0xffffffffu;
  constexpr int kInf = 0x7fffffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kMergeWarps + warp;
  int* wh = reinterpret_cast<int*>(msm) + warp * 256;                              // [256] histogram
  int* rb = reinterpret_cast<int*>(msm) + kMergeWarps * 256 + warp * kRecCap;      // recomputed blocks
  int4* xs = reinterpret_cast<int4*>(msm + 4 * kMergeWarps * (256 + kRecCap)) + warp * (dim >> 4);  // the row
  // per warp: cap keys, then cap 16-bit bin-order indices (cap / 4 key slots)
  uint64_t* keys = reinterpret_cast<uint64_t*>(msm + 4 * kMergeWarps * (256 + kRecCap) + kMergeWarps * dim) +
                   warp * (cap + cap / 4);
  if (row >= n) return;
  const int8_t* x = X + row * dim;
  const int nv4 = KB == 2 ? nblk >> 1 : KB == 4 ? nblk : 2 * nblk;  // int4s per row
  const bool complete = KB >= R;                                        // no block to recompute
  const int4* src = reinterpret_cast<const int4*>(bk + row * nblk * KB);
  int4 v[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const int i = 32 * u + lane;
    v[u] = i < nv4 ? __ldg(src + i) : make_int4(kInf, kInf, kInf, kInf);
  }
  int xn = 0;
  for (int u = lane; u < (dim >> 4); u += 32) {
    const int4 w = __ldg(reinterpret_cast<const int4*>(x) + u);
    xs[u] = w;
    xn = __dp4a(w.x, w.x, __dp4a(w.y, w.y, __dp4a(w.z, w.z, __dp4a(w.w, w.w, xn))));
  }
  xn = __reduce_add_sync(kFull, xn);
  const unsigned lt = (1u << lane) - 1u;
  int mn = kInf, mx = -kInf, cntv = 0;
  int s1 = kInf, s2 = kInf;  // this lane's two smallest stored e (kInf: fewer)
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const int w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = w[t] != kInf ? w[t] >> 5 : kInf;
      const int hi = max(s1, e);
      s1 = min(s1, e);
      s2 = min(s2, hi);
      if (w[t] != kInf) {
        mx = max(mx, e);
        ++cntv;
      }
    }
  }
  mn = __reduce_min_sync(kFull, s1);
  mx = __reduce_max_sync(kFull, mx);
  cntv = __reduce_add_sync(kFull, cntv);
  // A tighter upper end for the refinement below: the 32 lanes' smallest (R <= 32) or second
  // smallest (R <= 64) keys are 32 or 64 stored keys, so the R-th smallest stored e is at most
  // their maximum.  The first histogram then spans [mn, that] instead of every stored key: finer
  // bins (usually one pass instead of two) and an atomic only for the few keys inside.
  if (R <= 64) {
    const int ub = __reduce_max_sync(kFull, R <= 32 ? s1 : s2);
    if (ub != kInf) mx = min(mx, ub);
  }
  int tau = kInf;  // fewer than R stored keys: every block with two lists is recomputed
  if (cntv >= R) {
    int lo = mn, kk = R;
    uint32_t span = static_cast<uint32_t>(mx - mn) + 1u;
    for (;;) {
      const int bits = 32 - __clz((span - 1u) | 1u);
      const int sh = bits > 8 ? bits - 8 : 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) wh[lane * 8 + b] = 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const int w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t rel = static_cast<uint32_t>((w[t] >> 5) - lo);
          if (w[t] != kInf && rel < span) atomicAdd(&wh[rel >> sh], 1);
        }
      }
      __syncwarp();
      int hb[8], sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        hb[b] = wh[lane * 8 + b];
        sum += hb[b];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int cum = incl - sum, bin = -1, newk = 0, cb = 0;
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
        newk = kk - cum;
      }
      const int srcl = __ffs(__ballot_sync(kFull, bin >= 0)) - 1;
      bin = __shfl_sync(kFull, bin, srcl);
      kk = __shfl_sync(kFull, newk, srcl);
      cb = __shfl_sync(kFull, cb, srcl);
      __syncwarp();
      lo += bin << sh;
      span = 1u << sh;
      if (sh == 0 || cb <= 8) break;
    }
    tau = lo + static_cast<int>(span - 1u);
  }
  // candidates: stored keys with e <= tau of the blocks kept; the blocks to recompute
  int nc = 0, nr = 0;
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const int i = 32 * u + lane;
    const int w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
    if constexpr (KB == 8) {  // half a block per int4; complete (R <= 8)
      const int b = i >> 1;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int mk = w[t];
        const bool take = mk != kInf && (mk >> 5) <= tau;
        const unsigned bal = __ballot_sync(kFull, take);
        const int pos = nc + __popc(bal & lt);
        if (take && pos < cap) keys[pos] = merge_key(mk >> 5, b * 32 + (mk & 31));
        nc += __popc(bal);
      }
    } else {
#pragma unroll
    for (int hb = 0; hb < 4 / KB; ++hb) {
      const int b = (4 / KB) * i + hb, last = w[hb * KB + KB - 1];
      // a block whose KB-th key has e <= tau may hold more candidates than it stored: recompute it
      const bool rec = !complete && last != kInf && (last >> 5) <= tau;
      unsigned bal = __ballot_sync(kFull, rec);
      int pos = nr + __popc(bal & lt);
      if (rec && pos < kRecCap) rb[pos] = b;
      nr += __popc(bal);
#pragma unroll
      for (int t = 0; t < KB; ++t) {
        const int mk = w[hb * KB + t];
        const bool take = !rec && mk != kInf && (mk >> 5) <= tau;
        bal = __ballot_sync(kFull, take);
        pos = nc + __popc(bal & lt);
        if (take && pos < cap) keys[pos] = merge_key(mk >> 5, b * 32 + (mk & 31));
        nc += __popc(bal);
      }
    }
    }
  }
  __syncwarp();
  bool over = nr > kRecCap;
  if (!over) {
    // lane = list of the block; two blocks per step, 8 independent 16-byte loads each in flight
    const int nu = dim >> 4;
    for (int t = 0; t < nr; t += 2) {
      int li[2], dot[2] = {0, 0}, cnl[2];
      const int4* m4[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        li[h] = t + h < nr ? rb[t + h] * 32 + lane : nlist;
        m4[h] = reinterpret_cast<const int4*>(mu + static_cast<int64_t>(min(li[h], nlist - 1)) * dim);
        cnl[h] = li[h] < nlist ? __ldg(cnorm + li[h]) : 0;  // in flight with the centroid loads
      }
      for (int u0 = 0; u0 < nu; u0 += 8) {
        int4 q[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int w = 0; w < 8; ++w)
            q[h][w] = li[h] < nlist && u0 + w < nu ? __ldg(m4[h] + u0 + w) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (u0 + w < nu) {
            const int4 p = xs[u0 + w];
#pragma unroll
            for (int h = 0; h < 2; ++h)
              dot[h] = __dp4a(p.x, q[h][w].x, __dp4a(p.y, q[h][w].y, __dp4a(p.z, q[h][w].z, __dp4a(p.w, q[h][w].w, dot[h]))));
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = li[h] < nlist ? cnl[h] - 2 * dot[h] : 0;
        const bool take = li[h] < nlist && e <= tau;
        const unsigned bal = __ballot_sync(kFull, take);
        const int pos = nc + __popc(bal & lt);
        if (take && pos < cap) keys[pos] = merge_key(e, li[h]);
        nc += __popc(bal);
      }
    }
  }
  over = over || nc > cap;
  __syncwarp();
  if (!over) {
    // counting sort of the nc keys by e over 256 bins of [lo, hi], then the rank inside each bin
    // (ordered (e, i) keys: R9); ord (the recomputed-block list is dead) holds the bin order
    int elo = kInf, ehi = -kInf;
    for (int j = lane; j < nc; j += 32) {
      const int ej = static_cast<int>(keys[j] >> 32) - (1 << 30);
      elo = min(elo, ej);
      ehi = max(ehi, ej);
    }
    elo = __reduce_min_sync(kFull, elo);
    ehi = __reduce_max_sync(kFull, ehi);
    const uint32_t espan = static_cast<uint32_t>(ehi - elo);
    const int bits = 32 - __clz(espan | 1u), sh = bits > 8 ? bits - 8 : 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) wh[lane * 8 + b] = 0;
    __syncwarp();
    for (int j = lane; j < nc; j += 32)
      atomicAdd(&wh[static_cast<uint32_t>(static_cast<int>(keys[j] >> 32) - (1 << 30) - elo) >> sh], 1);
    __syncwarp();
    {
      int hb[8], sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        hb[b] = wh[lane * 8 + b];
        sum += hb[b];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - sum;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        wh[lane * 8 + b] = run;  // exclusive start; advanced to the bin's end by the scatter
        run += hb[b];
      }
    }
    __syncwarp();
    uint16_t* ord = reinterpret_cast<uint16_t*>(keys + cap);
    for (int j = lane; j < nc; j += 32) {
      const int b = static_cast<uint32_t>(static_cast<int>(keys[j] >> 32) - (1 << 30) - elo) >> sh;
      ord[atomicAdd(&wh[b], 1)] = static_cast<uint16_t>(j);
    }
    __syncwarp();
    for (int p = lane; p < nc; p += 32) {
      const uint64_t kj = keys[ord[p]];
      const int b = static_cast<uint32_t>(static_cast<int>(kj >> 32) - (1 << 30) - elo) >> sh;
      const int s0 = b ? wh[b - 1] : 0, s1 = wh[b];
      int rank = s0;
      for (int f = s0; f < s1; ++f) rank += keys[ord[f]] < kj ? 1 : 0;
      if (rank < R) {
        const int li = static_cast<int>(static_cast<uint32_t>(kj));
        out_idx[row * R + rank] = li;
        out_dist[row * R + rank] = xn + static_cast<int>(kj >> 32) - (1 << 30);
        if (hist) atomicAdd(hist + li, 1);
      }
    }
    for (int j = nc + lane; j < R; j += 32) {  // fewer lists than R (not reached: R <= nlist)
      out_idx[row * R + j] = -1;
      out_dist[row * R + j] = kInf;
    }
    return;
  }
  WarpTopK<KR> top;  // overflow: every list, exactly
  top.init(R);
  for (int b = 0; b < nlist; b += 32) {
    uint64_t key = ~0ull;
    const int i = b + lane;
    if (i < nlist) {
      const int8_t* m = mu + static_cast<int64_t>(i) * dim;
      int d = 0;
      for (int u = 0; u < dim; ++u) {
        const int df = static_cast<int>(x[u]) - static_cast<int>(m[u]);
        d += df * df;
      }
      key = step2_key(d, i);
    }
    top.offer(key);
  }
  top.store([&](int j, uint64_t key) {
    out_idx[row * R + j] = static_cast<int32_t>(key & 0xffffffffu);
    out_dist[row * R + j] = static_cast<int32_t>(key >> 32);
    if (hist) atomicAdd(hist + static_cast<uint32_t>(key), 1);
  });
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

bool make_tmap_i8(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint32_t box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t coarse_topk(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* cnorm, int nlist,
                        int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st, int* list_hist) {
  if (n <= 0) return cudaSuccess;
  const int kp = (dim + kPanel - 1) / kPanel;
  const size_t fixed = 1024 + static_cast<size_t>(kp) * kAPanelBytes + kEpiWarps * 64 * 4 + 64 * 8;
  // (A tiles of more than ~12 K panels leave no room for two B stages: the mma.sync kernel then)
  const int stages = fixed + 2 * kBStageBytes > 227 * 1024
                         ? 0
                         : static_cast<int>(std::min<size_t>(6, (227 * 1024 - fixed) / kBStageBytes));
  const bool tc_ok = dim % 16 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(mu) % 16 == 0 && stages >= 2 && !opt(V3DB_OPT_COARSE_SIMT);
  CUtensorMap tmX, tmMu;
  if (!tc_ok || !make_tmap_i8(&tmX, X, n, dim, kRows, kPanel) || !make_tmap_i8(&tmMu, mu, nlist, dim, kChunk, kPanel)) {
    cudaError_t em = coarse_topk_mma(X, n, dim, mu, cnorm, nlist, R, out_idx, out_dist, st);
    if (em == cudaSuccess && list_hist) {
      list_hist_kernel<<<static_cast<unsigned>(std::min<int64_t>((n * R + 255) / 256, 1184)), 256, 0, st>>>(out_idx, n * R,
                                                                                                       list_hist);
      note_launch();
      em = cudaGetLastError();
    }
    return em;
  }

  // Step 2 by recomputing the selected groups (pick_kernel): G <= kPickG lists per group with >= 2R
  // groups when nlist allows (small groups: few lists recomputed); R > 128 keeps the second
  // contraction pass (tau / pass 2 / select)
  // Recomputing ~R groups of G lists per row beats a second pass over every list when that is
  // small (measured: C1 0.069 vs 0.089 ms, C2 0.068 vs 0.101; C3 0.32 vs 0.20, C4 0.56 vs 0.46)
  const int64_t copt = opt(V3DB_OPT_COARSE_2PASS);
  // default: one contraction pass keeping each 32-list block's two smallest keys, then merge_kernel
  // (2 launches); the group-minimum paths remain as options (1, 4 / 8 / 16 / 32) and for dim > 1024
  const bool top2 = copt == 0 && dim <= 1024 && R <= 1024 && nlist <= 32768;  // (merge: <= 16 int4 per lane)
  const bool pick = !top2 && R <= 128 && copt != 1 &&
                    (copt != 0 || static_cast<int64_t>(R) * 8 * dim <= 32768);
  const int gmax = pick ? (copt == 4 || copt == 8 || copt == 16 || copt == 32 ? static_cast<int>(copt) : 8) : 32;
  int G = 1;
  while (G * 2 <= gmax && static_cast<int64_t>(G * 2) * 2 * R <= nlist) G *= 2;
  const int nchunks0 = (nlist + kChunk - 1) / kChunk;
  // top2: ngroups = blocks per row (8 per 256-list chunk), two keys each
  const int ngroups = top2 ? nchunks0 * 8 : (nlist + G - 1) / G;
  const int capc = pick || top2 ? 0 : ngroups < R ? std::max(nlist, 4 * R + 128) : 4 * R + 128;

  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t rtiles = (n + kRows - 1) / kRows;
  const int nchunks = (nlist + kChunk - 1) / kChunk;
  const int64_t items = rtiles * nchunks;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(items, sms));

  // keys kept per 32-list block: 2, or 4 where recomputing a block is expensive (dim > 256: the merge
  // then rarely recomputes); V3DB_OPT_COARSE_KEYS forces either
  const int64_t kopt = opt(V3DB_OPT_COARSE_KEYS);
  // 8 (or the smallest of 2 / 4 / 8 >= R) where R <= 8: the stored keys then hold the whole top R and
  // the merge recomputes nothing (C1, C2: R = 8)
  const int KB = kopt == 2 || kopt == 4 || (kopt == 8 && R <= 8 && nlist <= 16384) ? static_cast<int>(kopt)
                 : R <= 2                           ? 2
                 : R <= 4                           ? 4
                 : R <= 8 && nlist <= 16384         ? 8  // (merge: <= 32 int4 per lane)
                 : dim > 256                        ? 4
                                                    : 2;
  const size_t b_g = align256(sizeof(int32_t) * n * ngroups * (top2 ? KB : 1)), b_t = align256(sizeof(int32_t) * n),
               b_c = align256(sizeof(uint64_t) * n * capc), b_n = align256(sizeof(int) * n);
  uint8_t* base = nullptr;
  e = scratch_alloc(reinterpret_cast<void**>(&base), b_g + b_t + b_c + 2 * b_n, st);
  if (e != cudaSuccess) return e;
  CoarseArgs a;
  a.n = n;
  a.items = items;
  a.dim = dim;
  a.nlist = nlist;
  a.kp = kp;
  a.stages = stages;
  a.nchunks = nchunks;
  a.G = G;
  a.ngroups = ngroups;
  a.capc = capc;
  a.X = X;
  a.cnorm = cnorm;
  a.gmin = reinterpret_cast<int32_t*>(base);
  a.tau = reinterpret_cast<int32_t*>(base + b_g);
  a.cand = reinterpret_cast<uint64_t*>(base + b_g + b_t);
  a.ccnt = reinterpret_cast<int*>(base + b_g + b_t + b_c);
  int* flags = reinterpret_cast<int*>(base + b_g + b_t + b_c + b_n);

  const size_t smem = fixed + static_cast<size_t>(stages) * kBStageBytes;
  const unsigned rb = static_cast<unsigned>((n + 7) / 8);
  auto pass1 = [&]<int GT>() {
    cudaError_t e1 = cudaFuncSetAttribute(coarse_tc_kernel<1, GT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e1 == cudaSuccess) coarse_tc_kernel<1, GT><<<grid, kThreads, smem, st>>>(tmX, tmMu, a);
    return e1;
  };
  if (top2) {
    auto pass3 = [&](auto kern) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) kern<<<grid, kThreads, smem, st>>>(tmX, tmMu, a);
    };
    if (KB == 8) pass3(coarse_tc_kernel<3, 8>);
    else if (KB == 4) pass3(coarse_tc_kernel<3, 4>);
    else pass3(coarse_tc_kernel<3, 2>);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = debug_sync(st, "coarse pass (block top-2)");
    const int cap = (2 * R + 64 + 3) & ~3;  // (a multiple of 4: cap / 4 key slots hold the 16-bit bin order)
    const size_t msmem = 4 * kMergeWarps * (256 + kRecCap) + static_cast<size_t>(kMergeWarps) * dim +
                         sizeof(uint64_t) * kMergeWarps * (cap + cap / 4);
    const int nv4 = KB == 2 ? ngroups / 2 : KB == 4 ? ngroups : 2 * ngroups;
    if (e == cudaSuccess) {
      dispatch_kr(R, [&]<int KR>() {
        auto run = [&](auto kern) {
          e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem));
          if (e == cudaSuccess)
            kern<<<static_cast<unsigned>((n + kMergeWarps - 1) / kMergeWarps), 32 * kMergeWarps, msmem, st>>>(
                X, n, dim, mu, cnorm, nlist, ngroups, R, cap, a.gmin, out_idx, out_dist, list_hist);
        };
        auto by_nv = [&]<int KBT>() {
          if (nv4 <= 32) run(merge_kernel<KR, 1, KBT>);
          else if (nv4 <= 64) run(merge_kernel<KR, 2, KBT>);
          else if (nv4 <= 128) run(merge_kernel<KR, 4, KBT>);
          else if (nv4 <= 256) run(merge_kernel<KR, 8, KBT>);
          else if (nv4 <= 512) run(merge_kernel<KR, 16, KBT>);
          else run(merge_kernel<KR, 32, KBT>);
        };
        if (KB == 8) by_nv.template operator()<8>();
        else if (KB == 4) by_nv.template operator()<4>();
        else by_nv.template operator()<2>();
      });
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    note_launch(2);
    cudaFreeAsync(base, st);
    return e;
  }
  e = cudaFuncSetAttribute(coarse_tc_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    switch (G) {
      case 32: e = pass1.template operator()<32>(); break;
      case 16: e = pass1.template operator()<16>(); break;
      case 8: e = pass1.template operator()<8>(); break;
      case 4: e = pass1.template operator()<4>(); break;
      default: e = pass1.template operator()<0>(); break;
    }
  }
  if (e == cudaSuccess && pick) {
    if ((e = debug_sync(st, "coarse pass 1")) != cudaSuccess) {
      cudaFreeAsync(base, st);
      return e;
    }
    const size_t psmem = 4 * (8 * 256 + 8 * kPickCap) + 8 * static_cast<size_t>(dim);
    dispatch_kr(R, [&]<int KR>() {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(pick_kernel<KR>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(psmem));
      if (e == cudaSuccess)
        pick_kernel<KR><<<rb, 256, psmem, st>>>(X, n, dim, mu, cnorm, nlist, G, ngroups, R, a.gmin, out_idx, out_dist,
                                                list_hist);
    });
    note_launch(2);
    if (e == cudaSuccess) e = cudaGetLastError();
  } else if (e == cudaSuccess) {
    if ((e = debug_sync(st, "coarse pass 1")) != cudaSuccess) {
      cudaFreeAsync(base, st);
      return e;
    }
    tau_kernel<<<rb, 256, 0, st>>>(n, ngroups, R, a.gmin, const_cast<int32_t*>(a.tau), a.ccnt);
    coarse_tc_kernel<2, 0><<<grid, kThreads, smem, st>>>(tmX, tmMu, a);
    dispatch_kr(R, [&]<int KR>() {
      select_kernel<KR><<<rb, 256, 0, st>>>(n, R, capc, a.cand, a.ccnt, out_idx, out_dist, flags, list_hist);
      fallback_kernel<KR><<<rb, 256, 0, st>>>(X, n, dim, mu, nlist, R, flags, out_idx, out_dist, list_hist);
    });
    note_launch(5);
    e = cudaGetLastError();
  }
  cudaFreeAsync(base, st);
  return e;
}

}  // namespace v3db

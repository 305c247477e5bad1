// fx_coarse_tc.cu -- Steps 1-2 of PAPER.md §4.2 (and the build's B2 ranking) for the paper's 16-bit
// fixed point (NEXT-1) on the 5th-gen tensor cores.
//
// Coordinates are integers in [-65535, 65535].  Each is split into three balanced base-256 digits
//     v = v_0 + 256 v_1 + 65536 v_2,   v_0, v_1 in [-128, 127], v_2 in {-1, 0, 1}
// so <x, mu> = sum_{s,t} 256^(s+t) <x_s, mu_t> is nine int8 contractions; grouped by u = s + t they
// are five exact int32 accumulators acc_u (each |acc_u| <= 3 * 128^2 * dim < 2^31 for dim <= 1024),
// issued as tcgen05.mma.kind::i8 (M = 128 rows, N = 32 centroids, K = 32) with every limb tile brought
// into 128B-swizzled shared memory by TMA.  The epilogue forms, in int64 and exactly, the packed key
//     p = 32 e + (i mod 32),   e = ||mu_i||^2 - 2 <x, mu_i> = d_i - ||x||^2,
// as 32 ||mu_i||^2 + (i mod 32) + sum_u acc_u * (-64 * 256^u) (|p| < 2^49), and keeps the two smallest
// keys of every block of 32 consecutive lists -- the same single-pass scheme as the int8 coarse step
// (coarse_tc.cu): fx_merge_tc_kernel then takes tau >= the R-th smallest stored e, recomputes exactly
// the blocks whose second key is <= tau (they may hide more), and ranks the candidates on (d_i, i)
// (R9).  Distances are exact int64 throughout, so the result equals the oracle bit for bit.
//
// Warps: 0-11 epilogue (three groups of four TMEM lane quadrants; group g drains the work items
// j = g mod 3 of the CTA, each in its own set of five 32-column accumulators), 12 TMA producer,
// 13 MMA issuer.  dim <= 256 (the three limb tiles of a 128-row block stay resident).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "tc_common.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

constexpr int kFRows = 128;                       // rows per tile (UMMA M)
constexpr int kFCols = 96;                        // centroids per work item (UMMA N) = three blocks
constexpr int kFBlk = 32;                         // lists per block (two keys kept per block)
constexpr int kFPanel = 128;                      // bytes of K per swizzled panel
constexpr int kFSets = 1;                         // accumulator sets (5 x 96 columns: 480 of TMEM's 512)
constexpr int kFEpi = 12;                         // epilogue warps
constexpr int kFProd = kFEpi, kFMma = kFEpi + 1;
constexpr int kFThreads = 32 * (kFEpi + 2);
constexpr uint32_t kFAPanel = kFRows * kFPanel;   // 16 KB
constexpr uint32_t kFBStage = kFCols * kFPanel;   // 4 KB
constexpr int64_t kInf64 = 0x7fffffffffffffffLL;

struct FxTcArgs {
  int64_t n, items;
  int dim, nlist, kp, stages, nchunks, rows_p, cols_p;  // rows_p / cols_p: padded rows per limb
  const int64_t* cnorm;                                 // ||mu_i||^2
  int64_t* bk;                                          // [n][nchunks][2] block (min, second min)
};

// balanced base-256 digits of v (|v| <= 65535 + 65535): v = d0 + 256 d1 + 65536 d2
__device__ __forceinline__ void limbs3(int v, int& d0, int& d1, int& d2) {
  d0 = ((v + 128) & 255) - 128;
  const int w = (v - d0) >> 8;
  d1 = ((w + 128) & 255) - 128;
  d2 = (w - d1) >> 8;
}

// X [n][dim] int32 -> XL [3][rows_p][dim] int8 (rows >= n stay zero)
__global__ void limb_split_kernel(const int32_t* __restrict__ X, int64_t n, int dim, int64_t rows_p,
                                  int8_t* __restrict__ XL) {
  const int64_t tot = n * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int d0, d1, d2;
    limbs3(__ldg(X + e), d0, d1, d2);
    XL[e] = static_cast<int8_t>(d0);
    XL[rows_p * dim + e] = static_cast<int8_t>(d1);
    XL[2 * rows_p * dim + e] = static_cast<int8_t>(d2);
  }
}

__global__ void __launch_bounds__(kFThreads, 1) fx_coarse_tc_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                    const __grid_constant__ CUtensorMap tmMu,
                                                                    const FxTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                             // [3][kp][128 x 128 B]
  uint8_t* sB = smem + 3 * a.kp * kFAPanel;                       // [stages][32 x 128 B]
  int64_t* sCn = reinterpret_cast<int64_t*>(sB + a.stages * kFBStage);  // [kFEpi][32] packed column terms
  uint64_t* bars = reinterpret_cast<uint64_t*>(sCn + kFEpi * kFBlk);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 1;
  uint64_t* full = bars + 2;                  // [stages]
  uint64_t* empty = full + a.stages;          // [stages]
  uint64_t* accf = empty + a.stages;          // [kFSets]
  uint64_t* acce = accf + kFSets;             // [kFSets]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + kFSets);

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
    for (int s = 0; s < kFSets; ++s) {
      tc::mbar_init(accf + s, 1);
      tc::mbar_init(acce + s, kFEpi);  // every epilogue warp drains the item
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == kFProd) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0 && i0 < i1) {
      tc::tma_prefetch(&tmX);
      tc::tma_prefetch(&tmMu);
      int64_t cur_rt = -1;
      int nA = 0, s = 0, u = 0;
      for (int64_t it = i0; it < i1; ++it) {
        const int64_t rt = it / a.nchunks;
        const int c = static_cast<int>(it - rt * a.nchunks);
        if (rt != cur_rt) {
          if (nA > 0) tc::mbar_wait(a_empty, (nA - 1) & 1);
          tc::mbar_expect_tx(a_full, 3 * a.kp * kFAPanel);
          for (int l = 0; l < 3; ++l)
            for (int p = 0; p < a.kp; ++p)
              tc::tma_load_2d(sA + (l * a.kp + p) * kFAPanel, &tmX, a_full, p * kFPanel,
                              static_cast<int>(l * a.rows_p + rt * kFRows));
          ++nA;
          cur_rt = rt;
        }
        for (int p = 0; p < a.kp; ++p)  // (the MMA issuer's order: panel-major, limb-minor)
          for (int t = 0; t < 3; ++t) {
            if (u > 0) tc::mbar_wait(empty + s, (u - 1) & 1);
            tc::mbar_expect_tx(full + s, kFBStage);
            tc::tma_load_2d(sB + s * kFBStage, &tmMu, full + s, p * kFPanel, t * a.cols_p + c * kFCols);
            if (++s == a.stages) {
              s = 0;
              ++u;
            }
          }
      }
    }
  } else if (warp == kFMma) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && i0 < i1) {
      constexpr uint32_t idesc = tc::idesc_s8(kFRows, kFCols);
      int64_t cur_rt = -1;
      int nA = 0, s = 0, u = 0;
      // two consecutive items of one row tile at a time (one K panel): their MMAs alternate, so
      // updates of one accumulator are six MMAs apart (the tensor pipe executes in issue order)
      for (int64_t it = i0; it < i1;) {
        const int64_t rt = it / a.nchunks;
        const int ni = (kFSets > 1 && a.kp == 1 && it + 1 < i1 && (it + 1) / a.nchunks == rt) ? 2 : 1;
        if (rt != cur_rt) {
          tc::mbar_wait(a_full, nA & 1);
          tc::fence_after_sync();
          ++nA;
          cur_rt = rt;
        }
        uint32_t acc[2];
        int sets[2];
        for (int h = 0; h < ni; ++h) {
          const int j = static_cast<int>(it + h - i0), set = j % kFSets, use = j / kFSets;
          if (use > 0) tc::mbar_wait(acce + set, (use - 1) & 1);
          acc[h] = tmem + set * (5 * kFCols);
          sets[h] = set;
        }
        if (ni == 1) acc[1] = acc[0];
        tc::fence_after_sync();
        for (int p = 0; p < a.kp; ++p) {
          int st[2][3];
          for (int h = 0; h < ni; ++h)
            for (int t = 0; t < 3; ++t) {
              st[h][t] = s;
              tc::mbar_wait(full + s, u & 1);
              if (++s == a.stages) {
                s = 0;
                ++u;
              }
            }
          tc::fence_after_sync();
          const int nk = min(4, (a.dim - p * kFPanel + 31) / 32);
          // descriptors computed once per panel; a K step of 32 bytes adds 2 to the start field
          uint64_t dA[3], dB[2][3];
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            dA[l] = tc::desc_sw128(tc::smem_u32(sA + (l * a.kp + p) * kFAPanel));
            dB[0][l] = tc::desc_sw128(tc::smem_u32(sB + st[0][l] * kFBStage));
            dB[1][l] = ni == 2 ? tc::desc_sw128(tc::smem_u32(sB + st[1][l] * kFBStage)) : dB[0][l];
          }
          for (int k = 0; k < nk; ++k) {
            const uint32_t first = (p == 0 && k == 0) ? 1u : 0u;  // the items' first K step
            // the nine limb products in an order that spaces each accumulator's updates (u = sl + t:
            // 2 1 3 2 0 4 2 1 3); accumulate except on an accumulator's first product of the item
#define FX_MMA(SL, T, FIRSTPAIR)                                                                              \
  do {                                                                                                        \
    tc::mma_s8(acc[0] + ((SL) + (T)) * kFCols, dA[SL] + 2 * k, dB[0][T] + 2 * k, idesc,                       \
               (FIRSTPAIR) ? (first ^ 1u) : 1u);                                                              \
    if (ni == 2)                                                                                              \
      tc::mma_s8(acc[1] + ((SL) + (T)) * kFCols, dA[SL] + 2 * k, dB[1][T] + 2 * k, idesc,                     \
                 (FIRSTPAIR) ? (first ^ 1u) : 1u);                                                            \
  } while (0)
            FX_MMA(2, 0, true);   // u = 2
            FX_MMA(1, 0, true);   // u = 1
            FX_MMA(2, 1, true);   // u = 3
            FX_MMA(1, 1, false);  // u = 2
            FX_MMA(0, 0, true);   // u = 0
            FX_MMA(2, 2, true);   // u = 4
            FX_MMA(0, 2, false);  // u = 2
            FX_MMA(0, 1, false);  // u = 1
            FX_MMA(1, 2, false);  // u = 3
#undef FX_MMA
          }
          for (int h = 0; h < ni; ++h)
            for (int t = 0; t < 3; ++t) tc::mma_commit(empty + st[h][t]);
        }
        for (int h = 0; h < ni; ++h) tc::mma_commit(accf + sets[h]);
        if (it + ni == i1 || (it + ni) / a.nchunks != rt) tc::mma_commit(a_empty);
        it += ni;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-11)
    // warp = TMEM lane quadrant q x block blk (32 of the item's 96 columns); thread = row
    const int q = warp & 3, blk = warp >> 2;
    const int r = q * 32 + lane;
    int64_t* cn = sCn + warp * kFBlk;
    for (int64_t it = i0; it < i1; ++it) {
      const int j = static_cast<int>(it - i0), set = j % kFSets, use = j / kFSets;
      const int64_t rt = it / a.nchunks;
      const int c = static_cast<int>(it - rt * a.nchunks);
      const int col0 = c * kFCols + blk * kFBlk;
      const int64_t row = rt * kFRows + r;
      __syncwarp();
      // packed column terms 32 ||mu_i||^2 + (i mod 32); padding columns +inf (their limbs are zero)
      cn[lane] = col0 + lane < a.nlist ? 32 * __ldg(a.cnorm + col0 + lane) + lane : kInf64;
      __syncwarp();
#if defined(FXEXP) && FXEXP == 3  // experiment: spinning wait
      tc::mbar_wait(accf + set, use & 1);
#else
      tc::mbar_wait_sleep(accf + set, use & 1);
#endif
      tc::fence_after_sync();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + set * (5 * kFCols) + blk * kFBlk;
      int64_t m1 = kInf64, m2 = kInf64;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        uint32_t v0[8], v1[8], v2[8], v3[8], v4[8];
        tc::tmem_ld8(tbase + 0 * kFCols + qq * 8, v0);
        tc::tmem_ld8(tbase + 1 * kFCols + qq * 8, v1);
        tc::tmem_ld8(tbase + 2 * kFCols + qq * 8, v2);
        tc::tmem_ld8(tbase + 3 * kFCols + qq * 8, v3);
        tc::tmem_ld8(tbase + 4 * kFCols + qq * 8, v4);
        tc::tmem_ld_wait();
        if (qq == 3) {  // every accumulator value of this thread is in registers: release the set
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(acce + set);
        }
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const int64_t base = cn[qq * 8 + cc];
          int64_t pk = base;
          if (base != kInf64) {
            pk += static_cast<int64_t>(static_cast<int32_t>(v0[cc])) * -64;
            pk += static_cast<int64_t>(static_cast<int32_t>(v1[cc])) * -16384;
            pk += static_cast<int64_t>(static_cast<int32_t>(v2[cc])) * -4194304;
            pk += static_cast<int64_t>(static_cast<int32_t>(v3[cc])) * -1073741824LL;
            pk += static_cast<int64_t>(static_cast<int32_t>(v4[cc])) * -274877906944LL;  // -64 * 2^32
          }
          const int64_t t = max(m1, pk);
          m1 = min(m1, pk);
          m2 = min(m2, t);
        }
      }
      if (row < a.n)
        *reinterpret_cast<longlong2*>(a.bk + 2 * (row * (a.nchunks * 3) + c * 3 + blk)) = make_longlong2(m1, m2);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// Step 2 from the stored keys (one warp per row): the fixed-point counterpart of merge_kernel
// (coarse_tc.cu) on int64 keys p = 32 e + (i mod 32).
constexpr int kFxMergeWarps = 4;
constexpr int kFxRecCap = 32;
struct FxKey {
  int64_t e;
  int32_t i;
};

// NV: the row's stored key pairs per lane held in registers (nblk <= 32 NV).
template <int KR, int NV>
__global__ void __launch_bounds__(32 * kFxMergeWarps) fx_merge_tc_kernel(
    const int32_t* __restrict__ X, int64_t n, int dim, const int32_t* __restrict__ mu,
    const int64_t* __restrict__ cnorm, int nlist, int nblk, int rstride, int R, int cap,
    const int64_t* __restrict__ bk, int sh, int32_t* __restrict__ out_idx, int64_t* __restrict__ out_dist) {
  extern __shared__ __align__(16) uint8_t msm[];
  constexpr unsigned kFull = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kFxMergeWarps + warp;
  int* wh = reinterpret_cast<int*>(msm) + warp * 256;
  int* rb = reinterpret_cast<int*>(msm) + kFxMergeWarps * 256 + warp * kFxRecCap;
  FxKey* keys = reinterpret_cast<FxKey*>(msm + 4 * kFxMergeWarps * (256 + kFxRecCap)) + warp * cap;
  // per warp: one recomputed block's 32 centroid rows, then the row x ([33][dim] int32)
  int4* stage = reinterpret_cast<int4*>(msm + 4 * kFxMergeWarps * (256 + kFxRecCap) + sizeof(FxKey) * kFxMergeWarps * cap) +
                static_cast<size_t>(warp) * 33 * (dim >> 2);
  if (row >= n) return;
  const int32_t* x = X + row * dim;
  long long xn = 0;
  for (int u = lane; u < dim; u += 32) {
    const long long v = __ldg(x + u);
    xn += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xn += __shfl_xor_sync(kFull, xn, o);
  const longlong2* src = reinterpret_cast<const longlong2*>(bk + 2 * row * rstride);
  longlong2 kv[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) kv[u] = 32 * u + lane < nblk ? __ldg(src + 32 * u + lane) : make_longlong2(kInf64, kInf64);
  const unsigned lt = (1u << lane) - 1u;
  // extent of e over the stored keys (e = p >> 5)
  long long mn = kInf64, mx = -kInf64;
  int cntv = 0;
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const longlong2 v = kv[u];
    if (v.x != kInf64) {
      mn = min(mn, v.x >> 5);
      mx = max(mx, v.x >> 5);
      ++cntv;
    }
    if (v.y != kInf64) {
      mn = min(mn, v.y >> 5);
      mx = max(mx, v.y >> 5);
      ++cntv;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  }
  cntv = __reduce_add_sync(kFull, cntv);
  long long tau = kInf64;
  if (cntv >= R) {
    long long lo = mn;
    unsigned long long span = static_cast<unsigned long long>(mx - mn) + 1ull;
    int kk = R;
    for (;;) {
      const int bits = 64 - __clzll(static_cast<long long>((span - 1ull) | 1ull));
      const int shb = bits > 8 ? bits - 8 : 0;
      for (int b = lane; b < 256; b += 32) wh[b] = 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        const longlong2 v = kv[u];
        const long long w[2] = {v.x, v.y};
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const unsigned long long rel = static_cast<unsigned long long>((w[t] >> 5) - lo);
          if (w[t] != kInf64 && rel < span) atomicAdd(&wh[static_cast<int>(rel >> shb)], 1);
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
      lo += static_cast<long long>(bin) << shb;
      span = 1ull << shb;
      if (shb == 0 || cb <= 8) break;
    }
    tau = lo + static_cast<long long>(span - 1ull);
  }
  int nc = 0, nr = 0;
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    const int b = 32 * u + lane;
    const longlong2 v = kv[u];
    const bool rec = v.y != kInf64 && (v.y >> 5) <= tau;
    unsigned bal = __ballot_sync(kFull, rec);
    int pos = nr + __popc(bal & lt);
    if (rec && pos < kFxRecCap) rb[pos] = b;
    nr += __popc(bal);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const long long mk = t ? v.y : v.x;
      const bool take = !rec && mk != kInf64 && (mk >> 5) <= tau;
      bal = __ballot_sync(kFull, take);
      pos = nc + __popc(bal & lt);
      if (take && pos < cap) keys[pos] = FxKey{mk >> 5, b * 32 + static_cast<int>(mk & 31)};
      nc += __popc(bal);
    }
  }
  __syncwarp();
  bool over = nr > kFxRecCap;
  if (!over) {
    // lane = list of the block: exact int64 e.  The block's 32 rows (dim int32 each) arrive in shared
    // memory by cp.async -- all of a row's 16-byte pieces in flight at once, no registers held -- and
    // lane l reads its row's pieces in the rotated order (u + l) mod nu (conflict-free banks).
    const int nu = dim >> 2;
    int4* xs = stage + 32 * nu;
    for (int c = lane; c < nu; c += 32) xs[c] = __ldg(reinterpret_cast<const int4*>(x) + c);
    for (int t = 0; t < nr; ++t) {
      const int li = rb[t] * 32 + lane;
      const bool ok = li < nlist;
      const int4* m4 = reinterpret_cast<const int4*>(mu + static_cast<int64_t>(ok ? li : 0) * dim);
      int4* mine = stage + lane * nu;
      for (int c = 0; c < nu; ++c) tc::cp_async16(mine + c, m4 + c, ok ? 16 : 0);
      tc::cp_async_commit();
      const long long cnl = ok ? __ldg(cnorm + li) : 0;
      tc::cp_async_wait<0>();
      __syncwarp();
      long long dot = 0;
      int c = lane % nu;
      for (int u = 0; u < nu; ++u) {
        const int4 q = mine[c], p = xs[c];
        dot += static_cast<long long>(p.x) * q.x + static_cast<long long>(p.y) * q.y +
               static_cast<long long>(p.z) * q.z + static_cast<long long>(p.w) * q.w;
        if (++c == nu) c = 0;
      }
      const long long e = cnl - 2 * dot;
      const bool take = ok && e <= tau;
      const unsigned bal = __ballot_sync(kFull, take);
      const int pos = nc + __popc(bal & lt);
      if (take && pos < cap) keys[pos] = FxKey{e, li};
      nc += __popc(bal);
      __syncwarp();  // every lane is done with the stage before the next block's copies
    }
  }
  over = over || nc > cap;
  __syncwarp();
  if (!over) {
    // the (e, i) order as one unsigned compare: (e - emin) << 20 | i (e - emin < 2^44 for dim <= 256,
    // i < 2^20 lists), written over each key's e field
    long long emin = kInf64;
    for (int j = lane; j < nc; j += 32) emin = min(emin, static_cast<long long>(keys[j].e));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emin = min(emin, __shfl_xor_sync(kFull, emin, o));
    __syncwarp();
    for (int j = lane; j < nc; j += 32)
      keys[j].e = static_cast<long long>((static_cast<uint64_t>(keys[j].e - emin) << 20) | static_cast<uint32_t>(keys[j].i));
    __syncwarp();
    for (int j = lane; j < nc; j += 32) {
      const uint64_t kj = static_cast<uint64_t>(keys[j].e);
      int rank = 0;
      for (int f = 0; f < nc; ++f) rank += static_cast<uint64_t>(keys[f].e) < kj ? 1 : 0;
      if (rank < R) {
        out_idx[row * R + rank] = static_cast<int32_t>(kj & 0xfffff);
        out_dist[row * R + rank] = xn + emin + static_cast<long long>(kj >> 20);
      }
    }
    for (int j = nc + lane; j < R; j += 32) {  // fewer lists than R (not reached: R <= nlist)
      out_idx[row * R + j] = -1;
      out_dist[row * R + j] = kInf64;
    }
    return;
  }
  // overflow (massive ties): every list, exactly, on (d << sh | i) keys
  WarpTopK<KR> top;
  top.init(R);
  for (int b = 0; b < nlist; b += 32) {
    uint64_t key = ~0ull;
    const int i = b + lane;
    if (i < nlist) {
      const int32_t* m = mu + static_cast<int64_t>(i) * dim;
      long long d = 0;
      for (int u = 0; u < dim; ++u) {
        const long long df = static_cast<long long>(x[u]) - m[u];
        d += df * df;
      }
      key = (static_cast<uint64_t>(d) << sh) | static_cast<uint32_t>(i);
    }
    top.offer(key);
  }
  top.store([&](int j, uint64_t key) {
    out_idx[row * R + j] = static_cast<int32_t>(key & ((1ull << sh) - 1));
    out_dist[row * R + j] = static_cast<int64_t>(key >> sh);
  });
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

bool fx_coarse_tc_supported(int dim, int nlist, int R) {
  // (the merge holds a row's nlist / 32 stored key pairs in registers: nlist <= 32768)
  return dim % 16 == 0 && dim <= 256 && R <= 1024 && nlist <= 32768 && opt(V3DB_OPT_FX_COARSE) == 0;  // (i < 2^20)
}

// The R nearest lists (exact int64 distances, (d, i) order) of every row of X, on the tensor cores.
cudaError_t fx_topk_tc(const int32_t* X, int64_t n, int dim, const int32_t* mu, const int64_t* mnorm, int nlist,
                       int R, int sh, int32_t* out_idx, int64_t* out_dist, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int kp = (dim + kFPanel - 1) / kFPanel;
  const int64_t rows_p = (n + kFRows - 1) / kFRows * kFRows;
  const int nchunks = (nlist + kFCols - 1) / kFCols;
  const int cols_p = nchunks * kFCols;
  const size_t fixed = 1024 + 3 * static_cast<size_t>(kp) * kFAPanel + kFEpi * kFBlk * 8 + 64 * 8;
  const int stages = static_cast<int>(std::min<size_t>(24, (227 * 1024 - fixed) / kFBStage));
  if (stages < 4) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const size_t b_xl = al256(3 * static_cast<size_t>(rows_p) * dim), b_ml = al256(3 * static_cast<size_t>(cols_p) * dim),
               b_bk = al256(sizeof(int64_t) * 2 * n * nchunks * 3);
  uint8_t* base = nullptr;
  e = scratch_alloc(reinterpret_cast<void**>(&base), b_xl + b_ml + b_bk, st);
  if (e != cudaSuccess) return e;
  int8_t* XL = reinterpret_cast<int8_t*>(base);
  int8_t* ML = reinterpret_cast<int8_t*>(base + b_xl);
  int64_t* bk = reinterpret_cast<int64_t*>(base + b_xl + b_ml);
  e = cudaMemsetAsync(base, 0, b_xl + b_ml, st);  // zero padding rows of every limb
  if (e == cudaSuccess) {
    limb_split_kernel<<<static_cast<unsigned>(std::min<int64_t>((n * dim + 255) / 256, 148 * 16)), 256, 0, st>>>(
        X, n, dim, rows_p, XL);
    limb_split_kernel<<<static_cast<unsigned>(std::min<int64_t>((static_cast<int64_t>(nlist) * dim + 255) / 256, 148 * 16)),
                        256, 0, st>>>(mu, nlist, dim, cols_p, ML);
    note_launch(2);
    e = cudaGetLastError();
  }
  CUtensorMap tmX, tmMu;
  if (e == cudaSuccess && (!make_tmap_i8(&tmX, XL, 3 * static_cast<uint64_t>(rows_p), dim, kFRows, kFPanel) ||
                           !make_tmap_i8(&tmMu, ML, 3 * static_cast<uint64_t>(cols_p), dim, kFCols, kFPanel)))
    e = cudaErrorInvalidValue;
  if (e == cudaSuccess) {
    FxTcArgs a;
    a.n = n;
    a.items = (rows_p / kFRows) * nchunks;
    a.dim = dim;
    a.nlist = nlist;
    a.kp = kp;
    a.stages = stages;
    a.nchunks = nchunks;
    a.rows_p = static_cast<int>(rows_p);
    a.cols_p = cols_p;
    a.cnorm = mnorm;
    a.bk = bk;
    const size_t smem = fixed + static_cast<size_t>(stages) * kFBStage;
    e = cudaFuncSetAttribute(fx_coarse_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) {
      fx_coarse_tc_kernel<<<static_cast<unsigned>(std::min<int64_t>(a.items, sms)), kFThreads, smem, st>>>(tmX, tmMu, a);
      note_launch();
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = debug_sync(st, "fx coarse (tensor cores)");
  if (e == cudaSuccess) {
    const int cap = 2 * R + 64;
    const size_t msmem = 4 * kFxMergeWarps * (256 + kFxRecCap) + sizeof(FxKey) * kFxMergeWarps * cap +
                         sizeof(int32_t) * kFxMergeWarps * 33 * static_cast<size_t>(dim);  // + block stages
    const int nblk = (nlist + kFBlk - 1) / kFBlk;  // blocks of 32 lists holding a list (row stride 3 nchunks)
    dispatch_kr(R, [&]<int KR>() {
      auto run = [&](auto kern) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem));
        if (e == cudaSuccess)
          kern<<<static_cast<unsigned>((n + kFxMergeWarps - 1) / kFxMergeWarps), 32 * kFxMergeWarps, msmem, st>>>(
              X, n, dim, mu, mnorm, nlist, nblk, nchunks * 3, R, cap, bk, sh, out_idx, out_dist);
      };
      if (nblk <= 32) run(fx_merge_tc_kernel<KR, 1>);
      else if (nblk <= 64) run(fx_merge_tc_kernel<KR, 2>);
      else if (nblk <= 128) run(fx_merge_tc_kernel<KR, 4>);
      else if (nblk <= 256) run(fx_merge_tc_kernel<KR, 8>);
      else if (nblk <= 512) run(fx_merge_tc_kernel<KR, 16>);
      else run(fx_merge_tc_kernel<KR, 32>);
    });
    note_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  cudaFreeAsync(base, st);
  return e;
}

}  // namespace v3db

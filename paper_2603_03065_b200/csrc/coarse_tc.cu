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

constexpr int kRows = 128;        // rows per CTA (UMMA M)
constexpr int kChunk = 256;       // centroids per MMA chunk (UMMA N)
constexpr int kPanel = 128;       // bytes of K per swizzled panel
constexpr int kEpiWarps = 8;      // warps 0-7 epilogue (TMEM lanes 32*(w%4), column half w/4)
constexpr int kThreads = 32 * (kEpiWarps + 1);  // + warp 8: TMA producer / MMA issuer
constexpr uint32_t kAPanelBytes = kRows * kPanel;     // 16 KB
constexpr uint32_t kBStageBytes = kChunk * kPanel;    // 32 KB

struct CoarseArgs {
  int64_t n;
  int dim, nlist, kp, stages, nsplit, G, ngroups, capc;
  const int32_t* cnorm;
  int32_t* gmin;        // pass 1: [n][ngroups] group-minimum distances
  const int32_t* tau;   // pass 2: [n] threshold distance
  uint64_t* cand;       // pass 2: [n][capc] candidate keys
  int* ccnt;            // pass 2: [n] candidate counts
};

template <int PASS>
__global__ void __launch_bounds__(kThreads, 1) coarse_tc_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                const __grid_constant__ CUtensorMap tmMu,
                                                                const CoarseArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // kp panels of [128][128]
  uint8_t* sB = smem + a.kp * kAPanelBytes;             // stages of [256][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + a.stages * kBStageBytes);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;                            // [stages]
  uint64_t* empty = full + a.stages;                    // [stages]
  uint64_t* accf = empty + a.stages;                    // [2]
  uint64_t* acce = accf + 2;                            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  int* sCn = reinterpret_cast<int*>(bars + 32);         // [2][kChunk] ||mu||^2 of the chunk

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRows;
  const int nchunks = (a.nlist + kChunk - 1) / kChunk;
  const int cpc = (nchunks + a.nsplit - 1) / a.nsplit;
  const int c_begin = blockIdx.y * cpc;
  const int nch = max(0, min(nchunks, c_begin + cpc) - c_begin);

  if (tid == 32 * kEpiWarps) {
    tc::mbar_init(a_full, 1);
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

  if (nch > 0) {
    if (warp == kEpiWarps) {
      if (lane == 0) {
        tc::tma_prefetch(&tmX);
        tc::tma_prefetch(&tmMu);
        tc::mbar_expect_tx(a_full, a.kp * kAPanelBytes);
        for (int p = 0; p < a.kp; ++p) tc::tma_load_2d(sA + p * kAPanelBytes, &tmX, a_full, p * kPanel, (int)row0);
        const int n_it = nch * a.kp;
        auto load_b = [&](int it) {
          const int s = it % a.stages, c = c_begin + it / a.kp, p = it % a.kp;
          tc::mbar_expect_tx(full + s, kBStageBytes);
          tc::tma_load_2d(sB + s * kBStageBytes, &tmMu, full + s, p * kPanel, c * kChunk);
        };
        for (int it = 0; it < min(a.stages, n_it); ++it) load_b(it);
        tc::mbar_wait(a_full, 0);
        tc::fence_after_sync();
        constexpr uint32_t idesc = tc::idesc_s8(kRows, kChunk);
        for (int it = 0; it < n_it; ++it) {
          const int c = it / a.kp, p = it % a.kp, s = it % a.stages;
          const int acc = c & 1, use = c >> 1;
          if (p == 0 && use > 0) {
            tc::mbar_wait(acce + acc, (use - 1) & 1);
            tc::fence_after_sync();
          }
          tc::mbar_wait(full + s, (it / a.stages) & 1);
          tc::fence_after_sync();
          const int nk = min(4, (a.dim - p * kPanel + 31) / 32);
          const uint32_t a_addr = tc::smem_u32(sA + p * kAPanelBytes);
          const uint32_t b_addr = tc::smem_u32(sB + s * kBStageBytes);
          for (int k = 0; k < nk; ++k)
            tc::mma_s8(tmem + acc * kChunk, tc::desc_sw128(a_addr + k * 32), tc::desc_sw128(b_addr + k * 32), idesc,
                       (p | k) != 0);
          tc::mma_commit(empty + s);
          if (p == a.kp - 1) tc::mma_commit(accf + acc);
          if (it >= 1 && it - 1 + a.stages < n_it) {  // refill the stage of the previous iteration
            const int pit = it - 1, ps = pit % a.stages;
            tc::mbar_wait(empty + ps, (pit / a.stages) & 1);
            load_b(pit + a.stages);
          }
        }
      }
    } else {
      // ---------------- epilogue: thread r owns row row0 + r, half h of each chunk ----------------
      const int r = (warp & 3) * 32 + lane, half = warp >> 2;
      const int64_t row = row0 + r;
      const bool live = row < a.n;
      const int et = warp * 32 + lane;  // 0..255
      // ||mu||^2 of the first chunk into sCn[0]
      {
        const int col = c_begin * kChunk + et;
        sCn[et] = col < a.nlist ? __ldg(a.cnorm + col) : 0;
      }
      tc::mbar_wait(a_full, 0);
      int xn = 0;
      for (int p = 0; p < a.kp; ++p)
        for (int c = 0; c < 8; ++c) {
          const uint4 v = *reinterpret_cast<const uint4*>(sA + p * kAPanelBytes + tc::sw128_offset(r, c));
          xn = __dp4a(static_cast<int>(v.x), static_cast<int>(v.x), xn);
          xn = __dp4a(static_cast<int>(v.y), static_cast<int>(v.y), xn);
          xn = __dp4a(static_cast<int>(v.z), static_cast<int>(v.z), xn);
          xn = __dp4a(static_cast<int>(v.w), static_cast<int>(v.w), xn);
        }
      int tau_d = 0;
      if (PASS == 2 && live) tau_d = a.tau[row];
      for (int c = 0; c < nch; ++c) {
        const int acc = c & 1, use = c >> 1;
        // prefetch the next chunk's norms (published by the named barrier below)
        const int ncol = (c_begin + c + 1) * kChunk + et;
        const int cn_next = (c + 1 < nch && ncol < a.nlist) ? __ldg(a.cnorm + ncol) : 0;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));   // sCn[c&1] complete
        const int* cn = sCn + (c & 1) * kChunk + half * (kChunk / 2);
        tc::mbar_wait(accf + acc, use & 1);
        tc::fence_after_sync();
        const int colbase = (c_begin + c) * kChunk + half * (kChunk / 2);
#pragma unroll 1
        for (int b = 0; b < kChunk / 64; ++b) {
          const int col0 = colbase + b * 32;
          if (col0 >= a.nlist) break;  // warp-uniform
          uint32_t v[32];
          tc::tmem_ld32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + acc * kChunk +
                            half * (kChunk / 2) + b * 32, v);
          tc::tmem_ld_wait();
          if (!live) continue;
          const int* cnb = cn + b * 32;
          if (PASS == 1) {
            int best = 0x7fffffff;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              if (col0 + u < a.nlist) best = min(best, xn + cnb[u] - 2 * static_cast<int>(v[u]));
              if (((u + 1) & (a.G - 1)) == 0) {  // end of a group of G lists
                const int gstart = col0 + u + 1 - a.G;
                if (gstart < a.nlist) a.gmin[row * a.ngroups + gstart / a.G] = best;
                best = 0x7fffffff;
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              const int col = col0 + u;
              const int d = xn + cnb[u] - 2 * static_cast<int>(v[u]);
              if (d <= tau_d && col < a.nlist) {
                const int pos = atomicAdd(a.ccnt + row, 1);
                if (pos < a.capc) a.cand[row * a.capc + pos] = step2_key(d, col);
              }
            }
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(acce + acc);
        sCn[((c + 1) & 1) * kChunk + et] = cn_next;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// tau_row = R-th smallest group minimum (distance only); resets the candidate counters.
template <int KR>
__global__ void __launch_bounds__(256) tau_kernel(int64_t n, int ngroups, int R, const int32_t* __restrict__ gmin,
                                                 int32_t* __restrict__ tau, int* __restrict__ ccnt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= n) return;
  WarpTopK<KR> top;
  top.init(R);
  const int32_t* g = gmin + row * ngroups;
  for (int b = 0; b < ngroups; b += 32)
    top.offer((b + lane < ngroups) ? step2_key(g[b + lane], b + lane) : ~0ull);
  if (lane == 0) {
    tau[row] = static_cast<int32_t>(top.thr >> 32);
    ccnt[row] = 0;
  }
}

// Exact R smallest candidate keys per row; rows whose list overflowed are flagged.
template <int KR>
__global__ void __launch_bounds__(256) select_kernel(int64_t n, int R, int capc, const uint64_t* __restrict__ cand,
                                                    const int* __restrict__ ccnt, int32_t* __restrict__ out_idx,
                                                    int32_t* __restrict__ out_dist, int* __restrict__ flags) {
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
  });
}

// Plain exact recomputation of flagged rows (warp per row, all nlist distances).
template <int KR>
__global__ void __launch_bounds__(256) fallback_kernel(const int8_t* __restrict__ X, int64_t n, int dim,
                                                      const int8_t* __restrict__ mu, int nlist, int R,
                                                      const int* __restrict__ flags, int32_t* __restrict__ out_idx,
                                                      int32_t* __restrict__ out_dist) {
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
                        int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int kp = (dim + kPanel - 1) / kPanel;
  const int stages = std::min(4, static_cast<int>((200 * 1024 - kp * kAPanelBytes) / kBStageBytes));
  const char* force = getenv("V3DB_FORCE_COARSE_MMA");
  const bool tc_ok = dim % 16 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(mu) % 16 == 0 && stages >= 2 && !(force && force[0] == '1');
  CUtensorMap tmX, tmMu;
  if (!tc_ok || !make_tmap_i8(&tmX, X, n, dim, kRows, kPanel) || !make_tmap_i8(&tmMu, mu, nlist, dim, kChunk, kPanel))
    return coarse_topk_mma(X, n, dim, mu, cnorm, nlist, R, out_idx, out_dist, st);

  int G = 1;
  while (G * 2 <= 32 && static_cast<int64_t>(G * 2) * 2 * R <= nlist) G *= 2;
  const int ngroups = (nlist + G - 1) / G;
  const int capc = 4 * R + 128;

  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t rtiles = (n + kRows - 1) / kRows;
  const int nchunks = (nlist + kChunk - 1) / kChunk;
  const int nsplit = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nchunks, (2 * sms + rtiles - 1) / rtiles)));

  const size_t b_g = align256(sizeof(int32_t) * n * ngroups), b_t = align256(sizeof(int32_t) * n),
               b_c = align256(sizeof(uint64_t) * n * capc), b_n = align256(sizeof(int) * n);
  uint8_t* base = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&base), b_g + b_t + b_c + 2 * b_n, st);
  if (e != cudaSuccess) return e;
  CoarseArgs a;
  a.n = n;
  a.dim = dim;
  a.nlist = nlist;
  a.kp = kp;
  a.stages = stages;
  a.nsplit = nsplit;
  a.G = G;
  a.ngroups = ngroups;
  a.capc = capc;
  a.cnorm = cnorm;
  a.gmin = reinterpret_cast<int32_t*>(base);
  a.tau = reinterpret_cast<int32_t*>(base + b_g);
  a.cand = reinterpret_cast<uint64_t*>(base + b_g + b_t);
  a.ccnt = reinterpret_cast<int*>(base + b_g + b_t + b_c);
  int* flags = reinterpret_cast<int*>(base + b_g + b_t + b_c + b_n);

  const size_t smem = 1024 + kp * kAPanelBytes + stages * kBStageBytes + 32 * 8 + 2 * kChunk * 4;
  const dim3 grid(static_cast<unsigned>(rtiles), nsplit);
  const unsigned rb = static_cast<unsigned>((n + 7) / 8);
  e = cudaFuncSetAttribute(coarse_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(coarse_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    coarse_tc_kernel<1><<<grid, kThreads, smem, st>>>(tmX, tmMu, a);
    if ((e = debug_sync(st, "coarse pass 1")) != cudaSuccess) {
      cudaFreeAsync(base, st);
      return e;
    }
    dispatch_kr(R, [&]<int KR>() { tau_kernel<KR><<<rb, 256, 0, st>>>(n, ngroups, R, a.gmin, const_cast<int32_t*>(a.tau), a.ccnt); });
    coarse_tc_kernel<2><<<grid, kThreads, smem, st>>>(tmX, tmMu, a);
    dispatch_kr(R, [&]<int KR>() {
      select_kernel<KR><<<rb, 256, 0, st>>>(n, R, capc, a.cand, a.ccnt, out_idx, out_dist, flags);
      fallback_kernel<KR><<<rb, 256, 0, st>>>(X, n, dim, mu, nlist, R, flags, out_idx, out_dist);
    });
    note_launch(5);
    e = cudaGetLastError();
  }
  cudaFreeAsync(base, st);
  return e;
}

}  // namespace v3db

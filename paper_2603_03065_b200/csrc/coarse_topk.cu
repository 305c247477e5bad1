// coarse_topk.cu -- Step 1 (centroid distances) fused with Step 2 (probe selection).
//
//   d_i = dist(q, mu_i) = ||q||^2 + ||mu_i||^2 - 2 <q, mu_i>
//   P(q) = the R smallest (d_i, i), ascending                         (R9)
//
// The inner products are an int8 x int8 -> int32 dense contraction [rows x dim] . [dim x
// nlist] on the tensor cores (exact: |<q,mu>| <= dim*128^2 < 2^31).  The [rows x nlist]
// distance matrix is never written to HBM: each CTA keeps, per row, an exact sorted
// top-R list of composite keys in shared memory and streams the centroid tiles past it
// (threshold-pruned warp insertion, topk.cuh).  The same kernel ranks database vectors
// for the build (B2 needs each vector's lists in (e, i) order).
//
// This file holds the mma.sync (m16n8k32 s8) implementation, used for shapes the tcgen05
// path of coarse_tc.cu does not cover (dim % 16 != 0, dim > 768, unaligned rows).
#include <cuda_runtime.h>
#include <stdint.h>

#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

constexpr int kThreads = 256;
constexpr int kBN = 128;           // centroids per tile
constexpr int kKC = 128;           // K chunk (bytes of dim) staged per centroid tile
constexpr int kCsStride = kKC + 16;
constexpr int kDsStride = kBN + 8;

__device__ __forceinline__ void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Copy a [rows x cols] int8 block (row stride `src_stride` bytes in global memory,
// starting at column `c0`) into shared memory with row stride `dst_stride`, zero-filling
// rows >= valid_rows and columns >= valid_cols.  cols is a multiple of 16.
__device__ __forceinline__ void load_block(int8_t* dst, int dst_stride, const int8_t* src, int64_t src_stride,
                                           int rows, int cols, int valid_rows, int valid_cols, bool vec_ok) {
  const int segs = cols >> 4;
  for (int s = threadIdx.x; s < rows * segs; s += kThreads) {
    const int r = s / segs, c = (s - r * segs) << 4;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < valid_rows) {
      const int8_t* p = src + r * src_stride + c;
      if (vec_ok && c + 16 <= valid_cols) {
        v = __ldg(reinterpret_cast<const uint4*>(p));
      } else {
        uint8_t b[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) b[u] = (c + u < valid_cols) ? static_cast<uint8_t>(p[u]) : 0;
        v.x = b[0] | (b[1] << 8) | (b[2] << 16) | (uint32_t(b[3]) << 24);
        v.y = b[4] | (b[5] << 8) | (b[6] << 16) | (uint32_t(b[7]) << 24);
        v.z = b[8] | (b[9] << 8) | (b[10] << 16) | (uint32_t(b[11]) << 24);
        v.w = b[12] | (b[13] << 8) | (b[14] << 16) | (uint32_t(b[15]) << 24);
      }
    }
    *reinterpret_cast<uint4*>(dst + r * dst_stride + c) = v;
  }
}

template <int BM>
__global__ void __launch_bounds__(kThreads) coarse_topk_kernel(const int8_t* __restrict__ X, int64_t n, int dim,
                                                               int dp, const int8_t* __restrict__ mu,
                                                               const int32_t* __restrict__ cnorm, int nlist, int R,
                                                               int32_t* __restrict__ out_idx,
                                                               int32_t* __restrict__ out_dist, bool vec_ok) {
  constexpr int NT = (BM == 64) ? 8 : 2;  // n-tiles of 8 per warp
  extern __shared__ __align__(16) uint8_t smem[];
  const int xs_stride = dp + 16;
  uint64_t* T = reinterpret_cast<uint64_t*>(smem);                          // [BM][R]
  int32_t* Ds = reinterpret_cast<int32_t*>(T + BM * R);                      // [BM][kDsStride]
  int32_t* xnorm = Ds + BM * kDsStride;                                      // [BM]
  int8_t* Xs = reinterpret_cast<int8_t*>(xnorm + BM);                        // [BM][xs_stride]
  int8_t* Cs = Xs + BM * xs_stride;                                          // [kBN][kCsStride]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int valid_rows = static_cast<int>(n - row0 < BM ? n - row0 : BM);

  // Stage the row tile (zero padded to dp) and its squared norms; init the top-R lists.
  load_block(Xs, xs_stride, X + row0 * dim, dim, BM, dp, valid_rows, dim, vec_ok);
  for (int j = threadIdx.x; j < BM * R; j += kThreads) T[j] = ~0ull;
  __syncthreads();
  for (int r = warp; r < BM; r += kThreads / 32) {
    int acc = 0;
    for (int c = lane; c < dp; c += 32) {
      const int v = Xs[r * xs_stride + c];
      acc += v * v;
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if (lane == 0) xnorm[r] = acc;
  }

  const int wr = (BM == 64) ? (warp & 3) * 16 : 0;
  const int wc = (BM == 64) ? (warp >> 2) * 64 : warp * 16;
  constexpr int kRowsPerWarp = BM / (kThreads / 32);

  // per-warp top-R thresholds for its rows (T[r][R-1])
  uint64_t thr[kRowsPerWarp];
#pragma unroll
  for (int q = 0; q < kRowsPerWarp; ++q) thr[q] = ~0ull;

  for (int col0 = 0; col0 < nlist; col0 += kBN) {
    const int valid_cols = nlist - col0 < kBN ? nlist - col0 : kBN;
    int acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;

    for (int kc = 0; kc < dp; kc += kKC) {
      const int kw = dp - kc < kKC ? dp - kc : kKC;
      __syncthreads();  // previous users of Cs are done
      load_block(Cs, kCsStride, mu + static_cast<int64_t>(col0) * dim + kc, dim, kBN, kw, valid_cols,
                 dim - kc, vec_ok);
      __syncthreads();
      for (int kk = 0; kk < kw; kk += 32) {
        const int8_t* xa = Xs + (wr + g) * xs_stride + kc + kk + 4 * t4;
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(xa);
        const uint32_t a1 = *reinterpret_cast<const uint32_t*>(xa + 8 * xs_stride);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(xa + 16);
        const uint32_t a3 = *reinterpret_cast<const uint32_t*>(xa + 8 * xs_stride + 16);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int8_t* cb = Cs + (wc + t * 8 + g) * kCsStride + kk + 4 * t4;
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(cb);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(cb + 16);
          mma_s8(acc[t], a0, a1, a2, a3, b0, b1);
        }
      }
    }

    // Epilogue: exact integer distances into the shared tile.
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int c = wc + t * 8 + 2 * t4;
      const int r = wr + g;
      const int cn0 = (col0 + c < nlist) ? cnorm[col0 + c] : 0;
      const int cn1 = (col0 + c + 1 < nlist) ? cnorm[col0 + c + 1] : 0;
      Ds[r * kDsStride + c] = xnorm[r] + cn0 - 2 * acc[t][0];
      Ds[r * kDsStride + c + 1] = xnorm[r] + cn1 - 2 * acc[t][1];
      Ds[(r + 8) * kDsStride + c] = xnorm[r + 8] + cn0 - 2 * acc[t][2];
      Ds[(r + 8) * kDsStride + c + 1] = xnorm[r + 8] + cn1 - 2 * acc[t][3];
    }
    __syncthreads();

    // Selection: warp w owns rows w, w+8, ...; one candidate per lane per step.
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q) {
      const int r = warp + q * (kThreads / 32);
      uint64_t* Tr = T + r * R;
      for (int c = lane; c < kBN; c += 32) {
        const uint64_t key = (c < valid_cols) ? step2_key(Ds[r * kDsStride + c], col0 + c) : ~0ull;
        thr[q] = warp_offer(Tr, R, thr[q], key);
      }
    }
  }
  __syncthreads();

  for (int j = threadIdx.x; j < valid_rows * R; j += kThreads) {
    const int r = j / R, p = j - r * R;
    const uint64_t key = T[r * R + p];
    out_idx[(row0 + r) * R + p] = static_cast<int32_t>(key & 0xffffffffu);
    out_dist[(row0 + r) * R + p] = static_cast<int32_t>(key >> 32);
  }
}

template <int BM>
size_t smem_bytes(int dp, int R) {
  return sizeof(uint64_t) * BM * R + sizeof(int32_t) * BM * kDsStride + sizeof(int32_t) * BM +
         static_cast<size_t>(BM) * (dp + 16) + static_cast<size_t>(kBN) * kCsStride;
}

template <int BM>
cudaError_t launch(const int8_t* X, int64_t n, int dim, int dp, const int8_t* mu, const int32_t* cnorm, int nlist,
                   int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st) {
  const size_t smem = smem_bytes<BM>(dp, R);
  // 16-byte vector loads need 16-byte aligned rows
  const bool vec_ok = (dim % 16 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(mu) % 16 == 0);
  cudaError_t e = cudaFuncSetAttribute(coarse_topk_kernel<BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t blocks = (n + BM - 1) / BM;
  coarse_topk_kernel<BM><<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(X, n, dim, dp, mu, cnorm, nlist, R,
                                                                                 out_idx, out_dist, vec_ok);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t coarse_topk_mma(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* cnorm, int nlist,
                            int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int dp = (dim + 31) & ~31;
  if (R <= 128 && smem_bytes<64>(dp, R) <= 227 * 1024)
    return launch<64>(X, n, dim, dp, mu, cnorm, nlist, R, out_idx, out_dist, st);
  return launch<16>(X, n, dim, dp, mu, cnorm, nlist, R, out_idx, out_dist, st);
}

}  // namespace v3db

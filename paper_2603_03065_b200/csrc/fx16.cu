// fx16.cu -- NEXT-1: the five-step semantics on the paper's own 16-bit
// fixed-point representation: coordinates round((2^16-1) v / v_max) in
// [-65535, 65535] (int32), all distances exact in int64 (d_max = 2^63 - 1), codewords the residual
// sub-vectors themselves (R19).  Same steps and readings as the int8 path; different arithmetic
// (DESIGN.md §6.6):
//   * Step 1-2 (and the build ranking), fx_coarse_kernel: <x, mu> via IEEE-double FMAs -- exact,
//     every partial sum is an integer below dim * 65535^2 < 2^53 -- in 64 x 128 tiles whose keys
//     (d << sh | i, sh from the distance bound) update each row's top-R list in shared memory; the
//     distance matrix never reaches HBM (a materialised matrix + warp top-R only for R > 128);
//   * Steps 3-5, scan_fx_kernel: one CTA per query, the factorised table
//     A_q[m][c] = -2 <C_{m,c}, q^{(m)}> in int64 (conflict-free rotated layout for M % 8 == 0,
//     Ks = 256), D = d_i + P_{i,j} + sum_m A_q[m][c_m] per slot, every D to the trace, buffered
//     per-warp top-k on (D << sh5 | slot) keys with a CTA-wide admission bound, a rank merge, and
//     an exact re-selection by item id when ties at the k-th distance straddle the lists (R10).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

__global__ void abs_max_kernel(const int32_t* __restrict__ x, int64_t n, int* __restrict__ out) {
  int m = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = x[i];
    m = max(m, v == INT32_MIN ? INT32_MAX : abs(v));
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void encode_fp_kernel(const float* __restrict__ x, int64_t n, double v_max, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double y = __ddiv_rn(__dmul_rn(static_cast<double>(x[i]), 65535.0), v_max);
    // half away from zero (R18) on |y|: floor plus one when the fractional part (exact in IEEE
    // double) is >= 1/2 -- floor(|y| + 0.5) would round the double just below 0.5 up
    const double a = fabs(y), f = floor(a);
    const int32_t r = static_cast<int32_t>(f) + (__dsub_rn(a, f) >= 0.5 ? 1 : 0);
    out[i] = y < 0.0 ? -r : r;
  }
}

__global__ void gather32_kernel(const int32_t* __restrict__ db, int dim, const int32_t* __restrict__ rows, int nrows,
                                int32_t* __restrict__ out, int64_t* __restrict__ norms) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const int32_t* src = db + static_cast<int64_t>(rows[r]) * dim;
  long long acc = 0;
  for (int u = lane; u < dim; u += 32) {
    const int v = src[u];
    out[static_cast<int64_t>(r) * dim + u] = v;
    acc += static_cast<long long>(v) * v;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (norms && lane == 0) norms[r] = acc;
}

// out[r][c] = ||x_r||^2 + ||mu_c||^2 - 2 <x_r, mu_c> (int64, exact): 64 x 64 tile per CTA of 256
// threads, 4 x 4 outputs per thread, the dot products in double (exact below 2^53).
__global__ void __launch_bounds__(256) dist_matrix_kernel(const int32_t* __restrict__ X, int64_t n, int dim,
                                                          const int32_t* __restrict__ mu,
                                                          const int64_t* __restrict__ mnorm, int nlist,
                                                          int64_t* __restrict__ out) {
  __shared__ double As[32][65], Bs[32][65];  // [k][row] / [k][col]
  __shared__ long long xn_s[64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64;
  const int c0 = blockIdx.x * 64;
  double acc[4][4] = {};
  long long xn_part = 0;
  for (int k0 = 0; k0 < dim; k0 += 32) {
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int rr = e / 32, kk = e % 32;
      const int64_t r = r0 + rr;
      const int k = k0 + kk;
      const int xv = (r < n && k < dim) ? X[r * dim + k] : 0;
      As[kk][rr] = static_cast<double>(xv);
      const int c = c0 + rr;
      Bs[kk][rr] = (c < nlist && k < dim) ? static_cast<double>(mu[static_cast<int64_t>(c) * dim + k]) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 64) {
      for (int kk = 0; kk < 32; ++kk) {
        const long long v = static_cast<long long>(As[kk][threadIdx.x]);
        xn_part += v * v;
      }
    }
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty + 16 * i];
        b[i] = Bs[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 64) xn_s[threadIdx.x] = xn_part;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 16 * i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx + 16 * j;
      if (c >= nlist) continue;
      out[r * nlist + c] = xn_s[ty + 16 * i] + mnorm[c] - 2 * static_cast<long long>(acc[i][j]);
    }
  }
}

// R smallest (d, i) of each row of the distance matrix: warp per row, keys d << sh | i.
template <int KR>
__global__ void __launch_bounds__(256) row_topk_kernel(const int64_t* __restrict__ dm, int64_t n, int nlist, int R,
                                                       int sh, int32_t* __restrict__ out_idx,
                                                       int64_t* __restrict__ out_dist) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (r >= n) return;
  WarpTopK<KR> top;
  top.init(R);
  const int64_t* row = dm + r * nlist;
  for (int b = 0; b < nlist; b += 32) {
    const int i = b + lane;
    top.offer(i < nlist ? (static_cast<uint64_t>(row[i]) << sh) | static_cast<uint32_t>(i) : ~0ull);
  }
  const uint64_t mask = (uint64_t(1) << sh) - 1;
  top.store([&](int j, uint64_t key) {
    out_idx[r * R + j] = static_cast<int32_t>(key & mask);
    out_dist[r * R + j] = static_cast<int64_t>(key >> sh);
  });
}

// Fused Step 1 + Step 2 (and the build ranking): a CTA owns 64 rows of X and sweeps every
// centroid tile (64 x 64 distances, 4 x 4 per thread, dot products in double -- exact below
// 2^53), then each warp feeds 8 rows' tile keys (d << sh | i) to those rows' ascending top-R lists
// in shared memory.  The distance matrix never reaches HBM.  R <= 128.  With a centroid split
// (gridDim.y = S > 1, small batches) CTA (x, y) sweeps centroid tiles [y * span, (y + 1) * span) and
// writes its partial lists as keys to part [n][S][R]; fx_merge_kernel selects the final R.
template <int KR, int NJ>
__global__ void __launch_bounds__(256, 2) fx_coarse_kernel(const int32_t* __restrict__ X, int64_t n, int dim,
                                                        const int32_t* __restrict__ mu,
                                                        const int64_t* __restrict__ mnorm, int nlist, int R, int sh,
                                                        int span, int32_t* __restrict__ out_idx,
                                                        int64_t* __restrict__ out_dist, uint64_t* __restrict__ part) {
  constexpr int CW = 16 * NJ;       // centroids per tile: 4 rows x NJ columns per thread
  // dynamic: As [32][65] (k, row) | Bs [32][CW + 1] (k, col) -- reused as the key tile [64][65],
  // 64 columns at a time -- | T [64][R]
  __shared__ long long xn_s[64];
  extern __shared__ __align__(16) uint64_t dyn[];
  auto As = reinterpret_cast<double (*)[65]>(dyn);
  auto Bs = reinterpret_cast<double (*)[CW + 1]>(dyn + 32 * 65);
  uint64_t* T = dyn + 32 * 65 + 32 * (CW + 1);
  uint64_t* tile = dyn;
  static_assert(32 * 65 + 32 * (CW + 1) >= 64 * 65, "key tile alias");
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4, warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
  for (int e = tid; e < 64 * R; e += 256) T[e] = ~0ull;
  for (int rr = warp; rr < 64; rr += 8) {  // ||x_r||^2, exact
    const int64_t r = r0 + rr;
    long long acc = 0;
    if (r < n)
      for (int u = lane; u < dim; u += 32) {
        const long long v = X[r * dim + u];
        acc += v * v;
      }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) xn_s[rr] = acc;
  }
  uint64_t thr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) thr[i] = ~0ull;
  const int c_end = min(nlist, static_cast<int>(blockIdx.y + 1) * span);
  for (int c0 = blockIdx.y * span; c0 < c_end; c0 += CW) {
    double acc[4][NJ] = {};
    for (int k0 = 0; k0 < dim; k0 += 32) {
      if (dim % 32 == 0) {  // 16-byte loads, all issued before the conversions and stores
        constexpr int NA = 64 * 8 / 256, NB = CW * 8 / 256;
        int4 va[NA], vb[NB];
#pragma unroll
        for (int x = 0; x < NA; ++x) {
          const int e = tid + x * 256, rr = e >> 3, kq = (e & 7) * 4;
          const int64_t r = r0 + rr;
          va[x] = r < n ? __ldg(reinterpret_cast<const int4*>(X + r * dim + k0 + kq)) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int x = 0; x < NB; ++x) {
          const int e = tid + x * 256, cc = e >> 3, kq = (e & 7) * 4;
          const int c = c0 + cc;
          vb[x] = c < nlist ? __ldg(reinterpret_cast<const int4*>(mu + static_cast<int64_t>(c) * dim + k0 + kq))
                            : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int x = 0; x < NA; ++x) {
          const int e = tid + x * 256, rr = e >> 3, kq = (e & 7) * 4;
          As[kq][rr] = va[x].x;
          As[kq + 1][rr] = va[x].y;
          As[kq + 2][rr] = va[x].z;
          As[kq + 3][rr] = va[x].w;
        }
#pragma unroll
        for (int x = 0; x < NB; ++x) {
          const int e = tid + x * 256, cc = e >> 3, kq = (e & 7) * 4;
          Bs[kq][cc] = vb[x].x;
          Bs[kq + 1][cc] = vb[x].y;
          Bs[kq + 2][cc] = vb[x].z;
          Bs[kq + 3][cc] = vb[x].w;
        }
      } else {
        for (int e = tid; e < 64 * 32; e += 256) {
          const int rr = e >> 5, kk = e & 31;
          const int64_t r = r0 + rr;
          const int k = k0 + kk;
          As[kk][rr] = (r < n && k < dim) ? static_cast<double>(X[r * dim + k]) : 0.0;
        }
        for (int e = tid; e < CW * 32; e += 256) {
          const int cc = e >> 5, kk = e & 31;
          const int c = c0 + cc, k = k0 + kk;
          Bs[kk][cc] = (c < nlist && k < dim) ? static_cast<double>(mu[static_cast<int64_t>(c) * dim + k]) : 0.0;
        }
      }
      __syncthreads();
#pragma unroll 4
      for (int kk = 0; kk < 32; ++kk) {
        double av[4], bv[NJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];  // rows ty + 16 i: broadcast
#pragma unroll
        for (int j = 0; j < NJ; ++j) bv[j] = Bs[kk][tx + 16 * j];  // columns tx + 16 j: conflict-free
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int h = 0; h < NJ / 4; ++h) {  // 64 columns at a time through the key tile
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = c0 + 64 * h + tx + 16 * j;
          uint64_t key = ~0ull;
          if (r0 + rr < n && c < nlist) {
            const long long dd = xn_s[rr] + mnorm[c] - 2 * static_cast<long long>(acc[i][4 * h + j]);
            key = (static_cast<uint64_t>(dd) << sh) | static_cast<uint32_t>(c);
          }
          tile[rr * 65 + tx + 16 * j] = key;
        }
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = warp * 8 + i;
        const uint64_t k0 = tile[rr * 65 + lane], k1 = tile[rr * 65 + 32 + lane];
        if (!__any_sync(0xffffffffu, k0 < thr[i] || k1 < thr[i])) continue;
        // the row's list into registers (WarpTopK: insertion by ballots + shuffles), back to smem
        WarpTopK<KR> top;
        top.k = R;
        top.thr = thr[i];
#pragma unroll
        for (int r = 0; r < KR; ++r) top.v[r] = r * 32 + lane < R ? T[rr * R + r * 32 + lane] : ~0ull;
        top.offer(k0);
        top.offer(k1);
#pragma unroll
        for (int r = 0; r < KR; ++r)
          if (r * 32 + lane < R) T[rr * R + r * 32 + lane] = top.v[r];
        thr[i] = top.thr;
      }
      __syncthreads();  // `tile` aliases As / Bs
    }
  }
  __syncthreads();
  const uint64_t mask = (uint64_t(1) << sh) - 1;
  for (int e = tid; e < 64 * R; e += 256) {
    const int rr = e / R, j = e - rr * R;
    const int64_t r = r0 + rr;
    if (r >= n) continue;
    if (part) {
      part[(r * gridDim.y + blockIdx.y) * R + j] = T[e];
    } else {
      out_idx[r * R + j] = static_cast<int32_t>(T[e] & mask);
      out_dist[r * R + j] = static_cast<int64_t>(T[e] >> sh);
    }
  }
}

// The R smallest of each row's S partial lists (warp per row).
template <int KR>
__global__ void __launch_bounds__(256) fx_merge_kernel(const uint64_t* __restrict__ part, int64_t n, int S, int R,
                                                       int sh, int32_t* __restrict__ out_idx,
                                                       int64_t* __restrict__ out_dist) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (r >= n) return;
  WarpTopK<KR> top;
  top.init(R);
  const uint64_t* row = part + r * S * R;
  for (int b = 0; b < S * R; b += 32) top.offer(b + lane < S * R ? row[b + lane] : ~0ull);
  const uint64_t mask = (uint64_t(1) << sh) - 1;
  top.store([&](int j, uint64_t key) {
    out_idx[r * R + j] = static_cast<int32_t>(key & mask);
    out_dist[r * R + j] = static_cast<int64_t>(key >> sh);
  });
}

__global__ void codebook32_kernel(const int32_t* __restrict__ db, const int32_t* __restrict__ mu,
                                  const int32_t* __restrict__ list_of, int dim, int M, int Ks,
                                  const int32_t* __restrict__ rows, int32_t* __restrict__ cb) {
  const int d = dim / M;
  const int64_t total = static_cast<int64_t>(M) * Ks * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(e % d);
    const int64_t mc = e / d;
    const int m = static_cast<int>(mc / Ks);
    const int row = rows[mc];
    const int col = m * d + u;
    cb[e] = db[static_cast<int64_t>(row) * dim + col] - mu[static_cast<int64_t>(list_of[row]) * dim + col];  // R19
  }
}

// code_t[m] = argmin_c dist(r_t^{(m)}, C_{m,c}) (int64, lowest c on ties); ids / codes placement.
__global__ void encode32_kernel(const int32_t* __restrict__ db, int64_t n, int dim, const int32_t* __restrict__ mu,
                                const int32_t* __restrict__ list_of, const int32_t* __restrict__ flat_pos,
                                const int32_t* __restrict__ cb, int M, int Ks, uint8_t* __restrict__ codes,
                                int32_t* __restrict__ ids) {
  const int d = dim / M;
  const int64_t total = n * M;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = e / M;
    const int m = static_cast<int>(e - t * M);
    const int li = list_of[t];
    long long best = kDMaxFx;
    int bestc = 0;
    for (int c = 0; c < Ks; ++c) {
      long long acc = 0;
      const int32_t* cw = cb + (static_cast<int64_t>(m) * Ks + c) * d;
      for (int u = 0; u < d; ++u) {
        const long long r = static_cast<long long>(db[t * dim + m * d + u]) - mu[static_cast<int64_t>(li) * dim + m * d + u];
        const long long df = r - cw[u];
        acc += df * df;
      }
      if (acc < best) {
        best = acc;
        bestc = c;
      }
    }
    const int64_t pos = flat_pos[t];
    codes[pos * M + m] = static_cast<uint8_t>(bestc);
    if (m == 0) ids[pos] = static_cast<int32_t>(t);
  }
}

// codes_rot16 (see slot_dist_rot_w): byte s of group g of slot j = code of subspace
// off_g + ((s + j) mod gs), groups of gs = 16 and a trailing group of 8 when M % 16 == 8.
__global__ void rotate16_kernel(const uint8_t* __restrict__ codes, int64_t slots, int L, int M,
                                uint8_t* __restrict__ out) {
  const int64_t total = slots * M;
  const int m16 = M & ~15;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t slot = e / M;
    const int p = static_cast<int>(e - slot * M);
    const int j = static_cast<int>(slot % L);
    const int off = p < m16 ? (p & ~15) : m16, gs = p < m16 ? 16 : 8;
    out[e] = codes[slot * M + off + ((p - off + j) & (gs - 1))];
  }
}

// P_{i,j} = ||xhat||^2 + 2 <mu_i, xhat> (int64); 0 for padding.
__global__ void slot_terms64_kernel(const int32_t* __restrict__ mu, const int32_t* __restrict__ cb,
                                    const uint8_t* __restrict__ codes, const int32_t* __restrict__ ids, int nlist, int L,
                                    int dim, int M, int Ks, int64_t* __restrict__ pterm) {
  const int d = dim / M;
  const int64_t total = static_cast<int64_t>(nlist) * L;
  for (int64_t sidx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; sidx < total;
       sidx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    long long acc = 0;
    if (ids[sidx] != -1) {
      const int32_t* mui = mu + (sidx / L) * dim;
      for (int m = 0; m < M; ++m) {
        const int32_t* cw = cb + (static_cast<int64_t>(m) * Ks + codes[sidx * M + m]) * d;
        for (int u = 0; u < d; ++u) acc += static_cast<long long>(cw[u]) * cw[u] + 2LL * mui[m * d + u] * cw[u];
      }
    }
    pterm[sidx] = acc;
  }
}

// Offer one key per lane to the warp's ascending list T[0..R) (warp_offer) and track `mino`, the
// smallest key that is NOT in the list afterwards: rejected keys and the entry a full list drops
// on insertion (its old T[R-1] == thr).  Every key is offered exactly once and leaves only
// through one of those two doors, so at the end min(mino over warps and merge) is the smallest
// key outside the final top-k.
__device__ __forceinline__ uint64_t offer_track(uint64_t* T, int R, uint64_t thr, uint64_t key, uint64_t& mino) {
  if (key >= thr) mino = key < mino ? key : mino;
  unsigned mask = __ballot_sync(0xffffffffu, key < thr);
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
    if (kk < thr) {
      mino = thr < mino ? thr : mino;  // the entry the insertion drops
      thr = warp_insert(T, R, kk);
    } else {
      mino = kk < mino ? kk : mino;
    }
  }
  return thr;
}

// offer_track with a CTA-wide admission bound: *gthr is the smallest k-th key over all warps'
// lists -- a valid bound for every warp, since the warp owning it holds k smaller keys, so no key
// at or above it can be in the final top-k.  Keys at or above it are rejected (and tracked like
// any other rejection); a warp whose own k-th key drops publishes it with atomicMin.
__device__ __forceinline__ uint64_t offer_shared(uint64_t* T, int R, uint64_t thr, uint64_t key, uint64_t& mino,
                                                 unsigned long long* gthr) {
  // lane 0's read, broadcast: lanes not yet reconverged could otherwise read different values
  uint64_t eff = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile unsigned long long*>(gthr), 0);
  eff = thr < eff ? thr : eff;
  if (key >= eff) mino = key < mino ? key : mino;
  unsigned mask = __ballot_sync(0xffffffffu, key < eff);
  if (!mask) return thr;
  const uint64_t old = thr;
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
    if (kk < eff) {
      mino = thr < mino ? thr : mino;  // the entry the insertion drops
      thr = warp_insert(T, R, kk);
      eff = thr < eff ? thr : eff;
    } else {
      mino = kk < mino ? kk : mino;
    }
  }
  if (thr < old && (threadIdx.x & 31) == 0) atomicMin(gthr, static_cast<unsigned long long>(thr));
  return thr;
}

// Buffered per-warp top-k (k <= 256): keys below the admission bound are appended to the warp's
// buffer T[0..cap) (ballot + prefix count, no per-key insertion); when fewer than 32 free slots
// remain, the buffer is sorted (warp bitonic network) and cut back to its k smallest -- the cut
// keys are tracked like rejections (mino) and T[k-1] becomes the warp's bound.
__device__ __forceinline__ uint64_t warp_compact(uint64_t* T, int cap, int k, int& bcnt, uint64_t& mino) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int i = bcnt + lane; i < cap; i += 32) T[i] = ~0ull;
  __syncwarp();
  for (int size = 2; size <= cap; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (cap >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const uint64_t x = T[lo], y = T[hi];
        if ((x > y) == ((lo & size) == 0)) {
          T[lo] = y;
          T[hi] = x;
        }
      }
      __syncwarp();
    }
  const uint64_t cut = T[k];  // cap > k: the smallest key cut off
  mino = cut < mino ? cut : mino;
  bcnt = bcnt < k ? bcnt : k;
  return bcnt >= k ? T[k - 1] : ~0ull;
}

__device__ __forceinline__ uint64_t offer_buffered(uint64_t* T, int cap, int k, uint64_t thr, uint64_t key,
                                                   uint64_t& mino, int& bcnt, unsigned long long* gthr) {
  uint64_t eff = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile unsigned long long*>(gthr), 0);
  eff = thr < eff ? thr : eff;
  const bool pass = key < eff;
  if (!pass) mino = key < mino ? key : mino;
  const unsigned bal = __ballot_sync(0xffffffffu, pass);
  if (!bal) return thr;
  const int lane = threadIdx.x & 31;
  V3DB_DCHECK(bcnt + __popc(bal) <= cap);
  if (pass) T[bcnt + __popc(bal & ((1u << lane) - 1))] = key;
  bcnt += __popc(bal);
  if (bcnt > cap - 32) {
    const uint64_t old = thr;
    thr = warp_compact(T, cap, k, bcnt, mino);
    if (thr < old && lane == 0) atomicMin(gthr, static_cast<unsigned long long>(thr));
  }
  return thr;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Four table lookups of one 32-bit code word (subspaces m0..m0+3).
template <int KS>
__device__ __forceinline__ long long lut4(const int64_t* A, int Ks, int m0, uint32_t w) {
  const int ks = KS ? KS : Ks;
  return A[(m0 + 0) * ks + (w & 0xff)] + A[(m0 + 1) * ks + ((w >> 8) & 0xff)] +
         A[(m0 + 2) * ks + ((w >> 16) & 0xff)] + A[(m0 + 3) * ks + (w >> 24)];
}

// D_{i,j} = d_i + P_{i,j} + sum_m A_q[m][c_m] (acc enters as d_i + P_{i,j}); codes read with the
// widest aligned vector loads M allows.
template <int MT, int KS>
__device__ __forceinline__ long long slot_dist(const int64_t* A, const uint8_t* cp, int M, int Ks, long long acc) {
  if constexpr (MT > 0 && MT % 16 == 0) {
#pragma unroll
    for (int v = 0; v < MT / 16; ++v) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(cp) + v);
      acc += lut4<KS>(A, Ks, 16 * v, w.x) + lut4<KS>(A, Ks, 16 * v + 4, w.y) + lut4<KS>(A, Ks, 16 * v + 8, w.z) +
             lut4<KS>(A, Ks, 16 * v + 12, w.w);
    }
  } else if constexpr (MT > 0 && MT % 8 == 0) {
#pragma unroll
    for (int v = 0; v < MT / 8; ++v) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(cp) + v);
      acc += lut4<KS>(A, Ks, 8 * v, w.x) + lut4<KS>(A, Ks, 8 * v + 4, w.y);
    }
  } else {
    for (int m = 0; m < M; ++m) acc += A[m * Ks + cp[m]];
  }
  return acc;
}

// Conflict-free variant (M % 8 == 0, Ks == 256): subspaces in groups of 16 (and a trailing
// group of 8 when M % 16 == 8).  Group g's table is stored [c][gs] (row c holds the gs subspaces
// side by side, 8 B each: 128 B = all 32 banks for gs = 16) and the codes codes_rot16 hold, for
// slot j, byte s of group g = the code of subspace off_g + ((s + j) mod gs).  Lane l (== j mod 32)
// at step s then reads column (l + s) mod gs: for gs = 16 the 16 lanes of each half-warp hit 16
// distinct bank pairs whatever the codes are -- 2 wavefronts per LDS.64, the minimum; for gs = 8
// lanes l and l + 8 share a column and collide only when their rows have the same parity.
// rot8[s] = ((lane + s) & 15) * 8.  w = the slot's M code bytes as 32-bit words.
template <int MT>
__device__ __forceinline__ void load_code_words(const uint8_t* p, uint32_t (&w)[MT / 4]) {
  if constexpr (MT % 16 == 0) {
#pragma unroll
    for (int g = 0; g < MT / 16; ++g) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p) + g);
      w[4 * g] = x.x;
      w[4 * g + 1] = x.y;
      w[4 * g + 2] = x.z;
      w[4 * g + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int g = 0; g < MT / 8; ++g) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p) + g);
      w[2 * g] = x.x;
      w[2 * g + 1] = x.y;
    }
  }
}

template <int MT>
__device__ __forceinline__ long long slot_dist_rot_w(const int64_t* A, const uint32_t (&w)[MT / 4],
                                                     const uint32_t (&rot8)[16], long long acc) {
  constexpr int G16 = MT / 16;
#pragma unroll
  for (int g = 0; g < G16; ++g) {
    const char* Ab = reinterpret_cast<const char*>(A + g * 256 * 16);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const uint32_t c = (w[4 * g + (t >> 2)] >> (8 * (t & 3))) & 0xffu;
      acc += *reinterpret_cast<const long long*>(Ab + (c << 7) + rot8[t]);
    }
  }
  if constexpr (MT % 16 == 8) {
    const char* Ab = reinterpret_cast<const char*>(A + G16 * 256 * 16);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t c = (w[4 * G16 + (t >> 2)] >> (8 * (t & 3))) & 0xffu;
      acc += *reinterpret_cast<const long long*>(Ab + (c << 6) + (rot8[t] & 0x38u));
    }
  }
  return acc;
}

template <int MT>
__device__ __forceinline__ long long slot_dist_rot(const int64_t* A, const uint8_t* cp, const uint32_t (&rot8)[16],
                                                   long long acc) {
  uint32_t w[MT / 4];
  load_code_words<MT>(cp, w);
  return slot_dist_rot_w<MT>(A, w, rot8, acc);
}

// Steps 3-5 for one query per CTA of NW = 8 warps (16 measured slower: C4 16.7 -> 17.3 ms).
struct FxScanArgs {
  const int32_t* queries;
  int dim, M, Ks, L, nprobe, k, sh5;
  int cap;                   // per-warp list stride: the buffer size (k <= 256, buffered) or k
  const int32_t* cb;         // [M][Ks][d]
  const uint8_t* codes;      // canonical [nlist][L][M] (ROT: codes_rot16, same shape)
  const int64_t* pterm;      // [nlist][L]
  const int32_t* ids;
  const int32_t* counts;
  const int32_t* lists;      // [nq][nprobe]
  const int64_t* ldist;      // [nq][nprobe]
  int32_t* out_ids;
  int64_t* out_dist;
  int64_t* trace;            // [nq][nprobe][L] or null
  int64_t* Ag;               // [nq][M][Ks] when the table does not fit in shared memory, else null
  const int32_t* order;      // L2-aware query order (minhash_order) or null
};

// Shared memory: A [M][Ks] int64 (unless GA) | tops [W][k] u64 | resD [k] i64 | resI [k] i32 |
// q [dim] i32 | wmin [1] u64.
template <int MT, int KS, bool GA, bool ROT, int NW>
__global__ void __launch_bounds__(32 * NW) scan_fx_kernel(const FxScanArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int W = NW, NT = 32 * W;
  const int M = MT ? MT : a.M;
  const int Ks = KS ? KS : a.Ks;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t qi = a.order ? a.order[blockIdx.x] : blockIdx.x;
  const int k = a.k, L = a.L, nprobe = a.nprobe, d = a.dim / M;
  int64_t* A = GA ? a.Ag + static_cast<int64_t>(blockIdx.x) * M * Ks : reinterpret_cast<int64_t*>(smem);
  uint64_t* tops = reinterpret_cast<uint64_t*>(smem + (GA ? 0 : sizeof(int64_t) * M * Ks));
  const int S = a.cap;  // per-warp list stride
  const bool buffered = S > k;
  long long* resD = reinterpret_cast<long long*>(tops + W * S);
  int32_t* resI = reinterpret_cast<int32_t*>(resD + k);
  int32_t* qs = resI + k;
  uint64_t* wmin = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(qs + a.dim) + 15) & ~uintptr_t(15));
  const int32_t* q = a.queries + qi * a.dim;
  for (int u = tid; u < a.dim; u += NT) qs[u] = q[u];
  for (int e = tid; e < W * S; e += NT) tops[e] = ~0ull;
  if (tid == 0) wmin[1] = ~0ull;  // gthr
  __syncthreads();
  // Step 3, factorised: A_q[m][c] = -2 <C_{m,c}, q^{(m)}>
  for (int e = tid; e < M * Ks; e += NT) {
    const int m = e / Ks;
    const int32_t* cw = a.cb + static_cast<int64_t>(e) * d;
    long long acc = 0;
    for (int u = 0; u < d; ++u) acc += static_cast<long long>(__ldg(cw + u)) * qs[m * d + u];
    if constexpr (ROT) {
      const int c = e - m * Ks;
      constexpr int G16 = MT / 16;
      if (m < 16 * G16) A[((m >> 4) * Ks + c) * 16 + (m & 15)] = -2 * acc;
      else A[G16 * Ks * 16 + c * 8 + (m - 16 * G16)] = -2 * acc;  // trailing group of 8
    } else {
      A[e] = -2 * acc;
    }
  }
  __syncthreads();
  // Steps 4-5: every probed slot, per-warp exact top-k on (D << sh5 | slot)
  const int32_t* qlists = a.lists + qi * nprobe;
  const int64_t* qld = a.ldist + qi * nprobe;
  int64_t* trace = a.trace ? a.trace + qi * nprobe * static_cast<int64_t>(L) : nullptr;
  uint64_t* T = tops + warp * S;
  uint64_t thr = ~0ull, mino = ~0ull;
  int bcnt = 0;
  uint32_t rot8[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) rot8[t] = ((lane + t) & 15) << 3;
  auto dist = [&](int64_t slot, long long acc) -> long long {
    if constexpr (ROT) return slot_dist_rot<MT>(A, a.codes + slot * M, rot8, acc);
    else return slot_dist<MT, KS>(A, a.codes + slot * M, M, Ks, acc);
  };
  if constexpr (ROT) {
    // software-pipelined: the codes and P term of the warp's next 32-slot chunk are loaded while
    // the current chunk is scanned (the chunk sequence runs over (probe rank, slot) like below)
    constexpr int NWD = MT / 4;
    auto lim_of = [&](int r) { return trace ? L : a.counts[qlists[r]]; };
    auto load = [&](int r, int jj, uint32_t (&w)[NWD], long long& p) {
      const int li = qlists[r];
      const int j = jj + lane;
      if (j < a.counts[li]) {
        const int64_t slot = static_cast<int64_t>(li) * L + j;
        load_code_words<MT>(a.codes + slot * MT, w);
        p = __ldg(a.pterm + slot);
      }
    };
    int rho = 0, j0 = warp * 32;
    while (rho < nprobe && j0 >= lim_of(rho)) ++rho;
    uint32_t cw[NWD];
    long long cp = 0;
    if (rho < nprobe) load(rho, j0, cw, cp);
    while (rho < nprobe) {
      int nrho = rho, nj0 = j0 + W * 32;
      while (nrho < nprobe && nj0 >= lim_of(nrho)) {
        ++nrho;
        nj0 = warp * 32;
      }
      uint32_t nw[NWD];
      long long np = 0;
      if (nrho < nprobe) load(nrho, nj0, nw, np);
      const int cnt = a.counts[qlists[rho]];
      const int j = j0 + lane;
      long long D = kDMaxFx;
      if (j < cnt) D = slot_dist_rot_w<MT>(A, cw, rot8, qld[rho] + cp);
      if (trace && j < L) trace[static_cast<int64_t>(rho) * L + j] = D;
      const uint64_t key = j < cnt ? (static_cast<uint64_t>(D) << a.sh5) | static_cast<uint32_t>(rho * L + j) : ~0ull;
      if (buffered) thr = offer_buffered(T, S, k, thr, key, mino, bcnt, reinterpret_cast<unsigned long long*>(wmin + 1));
      else thr = offer_shared(T, k, thr, key, mino, reinterpret_cast<unsigned long long*>(wmin + 1));
      rho = nrho;
      j0 = nj0;
#pragma unroll
      for (int g = 0; g < NWD; ++g) cw[g] = nw[g];
      cp = np;
    }
  } else
  for (int rho = 0; rho < nprobe; ++rho) {
    const int li = qlists[rho];
    const long long di = qld[rho];
    const int cnt = a.counts[li];
    const int64_t base = static_cast<int64_t>(li) * L;
    const int lim = trace ? L : cnt;
    for (int j0 = warp * 32; j0 < lim; j0 += W * 32) {
      const int j = j0 + lane;
      long long D = kDMaxFx;
      if (j < cnt) D = dist(base + j, di + __ldg(a.pterm + base + j));
      if (trace && j < L) trace[static_cast<int64_t>(rho) * L + j] = D;
      const uint64_t key = j < cnt ? (static_cast<uint64_t>(D) << a.sh5) | static_cast<uint32_t>(rho * L + j) : ~0ull;
      if (buffered) thr = offer_buffered(T, S, k, thr, key, mino, bcnt, reinterpret_cast<unsigned long long*>(wmin + 1));
      else thr = offer_shared(T, k, thr, key, mino, reinterpret_cast<unsigned long long*>(wmin + 1));
    }
  }
  if (buffered) warp_compact(T, S, k, bcnt, mino);  // T[0..k): the warp's k smallest, ascending
  uint64_t* fin = reinterpret_cast<uint64_t*>(resD);  // the merged list (resD is free until resolved)
  if (tid == 0) wmin[0] = ~0ull;
  for (int e = tid; e < k; e += NT) fin[e] = ~0ull;
  __syncthreads();
  mino = warp_min_u64(mino);
  if (lane == 0 && mino != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(wmin), mino);
  // merge the W sorted lists by rank: the keys are distinct (slot in the low bits), so a key's
  // final position is the number of smaller keys over all lists (binary search in each)
  uint64_t lost = ~0ull;
  for (int e = tid; e < W * k; e += NT) {
    const uint64_t key = tops[(e / k) * S + e % k];
    if (key == ~0ull) continue;
    int rank = 0;
    for (int w = 0; w < W; ++w) {
      const uint64_t* Lw = tops + w * S;
      int lo = 0, hi = k;  // first index with Lw[idx] >= key
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (Lw[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      rank += lo;
    }
    if (rank < k) fin[rank] = key;
    else lost = key < lost ? key : lost;
  }
  lost = warp_min_u64(lost);
  if (lane == 0 && lost != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(wmin), lost);
  __syncthreads();
  const uint64_t tau = fin[k - 1];
  const uint64_t smallest_out = wmin[0];
  const uint64_t slot_mask = (uint64_t(1) << a.sh5) - 1;
  __syncthreads();  // everyone has read fin[k - 1] before it is resolved in place
  // resolve the list entries: (D, item), in place (thread e reads fin[e] before writing resD[e])
  for (int e = tid; e < k; e += NT) {
    const uint64_t key = fin[e];
    if (key != ~0ull) {
      const int slot = static_cast<int>(key & slot_mask);
      const int rho = slot / L;
      resD[e] = static_cast<long long>(key >> a.sh5);
      resI[e] = a.ids[static_cast<int64_t>(qlists[rho]) * L + (slot - rho * L)];
    } else {
      resD[e] = kDMaxFx;
      resI[e] = -1;
    }
  }
  __syncthreads();
  const long long Dtau = static_cast<long long>(tau >> a.sh5);
  // ties at the k-th distance that straddle the list boundary need the id order over all of them
  const bool straddle = tau != ~0ull && smallest_out != ~0ull && (smallest_out >> a.sh5) == (tau >> a.sh5);
  // list entries placed by their rank among themselves: the valid ones (a prefix of the key-sorted
  // list) -- or, when ties straddle, those with D < Dtau (also a prefix)
  int n_keep = 0;
  for (int e = 0; e < k; ++e)
    if (resI[e] != -1 && (!straddle || resD[e] < Dtau)) n_keep = e + 1;
  for (int e = tid; e < n_keep; e += NT) {
    const long long D = resD[e];
    const int32_t id = resI[e];
    int rank = 0;
    for (int f = 0; f < n_keep; ++f) rank += (resD[f] < D || (resD[f] == D && resI[f] < id)) ? 1 : 0;
    a.out_ids[qi * k + rank] = id;
    a.out_dist[qi * k + rank] = D;
  }
  if (!straddle) {  // fewer than k valid candidates: (-1, d_max) tail
    for (int r = n_keep + tid; r < k; r += NT) {
      a.out_ids[qi * k + r] = -1;
      a.out_dist[qi * k + r] = kDMaxFx;
    }
    return;
  }
  // Rare path: the need = k - n_keep smallest items among ALL candidates with D == Dtau
  // (recomputed; per-warp top-need on item ids, then merged in warp 0).
  const int need = k - n_keep;
  __syncthreads();
  for (int e = tid; e < W * k; e += NT) tops[e] = ~0ull;
  __syncthreads();
  thr = ~0ull;
  uint64_t dummy = ~0ull;
  for (int rho = 0; rho < nprobe; ++rho) {
    const int li = qlists[rho];
    const long long di = qld[rho];
    const int cnt = a.counts[li];
    const int64_t base = static_cast<int64_t>(li) * L;
    for (int j0 = warp * 32; j0 < cnt; j0 += W * 32) {
      const int j = j0 + lane;
      uint64_t key = ~0ull;
      if (j < cnt) {
        const long long D = dist(base + j, di + __ldg(a.pterm + base + j));
        if (D == Dtau) key = static_cast<uint32_t>(a.ids[base + j]);
      }
      thr = offer_track(tops + warp * k, need, thr, key, dummy);
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < W; ++w)
      for (int b = 0; b < need; b += 32)
        thr = offer_track(tops, need, thr, b + lane < need ? tops[w * k + b + lane] : ~0ull, dummy);
  }
  __syncthreads();
  for (int r = tid; r < need; r += NT) {
    a.out_ids[qi * k + n_keep + r] = static_cast<int32_t>(tops[r]);
    a.out_dist[qi * k + n_keep + r] = Dtau;
  }
}

int bits_for(long double v) {
  int b = 0;
  while (b < 63 && std::ldexp(1.0L, b) <= v) ++b;
  return b;
}

}  // namespace

// Key shifts: Step 2 keys d << sh2 | i need d < 2^(64-sh2); Step 5 keys D << sh5 | slot likewise.
int fx_shift2(int dim) { return 64 - bits_for(static_cast<long double>(dim) * 131070.0L * 131070.0L); }
int fx_shift5(int dim) { return 64 - bits_for(static_cast<long double>(dim) * 262140.0L * 262140.0L); }

cudaError_t rotate_codes16(const uint8_t* codes, int64_t slots, int L, int M, uint8_t* out, cudaStream_t st) {
  rotate16_kernel<<<static_cast<int>(std::min<int64_t>((slots * M + 255) / 256, 148 * 64)), 256, 0, st>>>(codes, slots,
                                                                                                      L, M, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t abs_max32(const int32_t* x, int64_t n, int* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  abs_max_kernel<<<blocks, 256, 0, st>>>(x, n, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t encode_fixed_point(const float* x, int64_t n, double v_max, int32_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  encode_fp_kernel<<<blocks, 256, 0, st>>>(x, n, v_max, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t gather_rows32(const int32_t* db, int dim, const int32_t* rows, int nrows, int32_t* out, int64_t* norms,
                          cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  gather32_kernel<<<(nrows * 32 + 255) / 256, 256, 0, st>>>(db, dim, rows, nrows, out, norms);
  note_launch();
  return cudaGetLastError();
}

// R nearest lists of every row of X (exact int64 distances); scratch: the [rows x nlist] matrix.
cudaError_t fx_topk(const int32_t* X, int64_t n, int dim, const int32_t* mu, const int64_t* mnorm, int nlist, int R,
                    int32_t* out_idx, int64_t* out_dist, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int sh = fx_shift2(dim);
  if (sh < 1 || nlist > (1 << std::min(sh, 30))) return cudaErrorInvalidValue;
  if (fx_coarse_tc_supported(dim, nlist, R)) return fx_topk_tc(X, n, dim, mu, mnorm, nlist, R, sh, out_idx, out_dist, st);
  if (R <= 128) {
    constexpr int NJ = 8, CW = 16 * NJ;
    const size_t smem = sizeof(uint64_t) * (32 * 65 + 32 * (CW + 1) + 64 * R);
    cudaError_t e = cudaFuncSetAttribute(fx_coarse_kernel<1, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fx_coarse_kernel<2, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fx_coarse_kernel<4, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int ctiles = (nlist + CW - 1) / CW;
    for (int64_t lo = 0; lo < n; lo += int64_t(1) << 24) {  // grid.x chunks
      const int64_t rows = std::min<int64_t>(int64_t(1) << 24, n - lo);
      const int64_t rtiles = (rows + 63) / 64;
      // centroid split so that small batches still fill 148 SMs x 2 CTAs (>= 2 tiles per CTA)
      const int S = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((4 * 148 + rtiles - 1) / rtiles,
                                                                             ctiles / 2)));
      const int span = ((ctiles + S - 1) / S) * CW;
      const int Sr = (nlist + span - 1) / span;
      uint64_t* part = nullptr;
      if (Sr > 1) {
        e = scratch_alloc(reinterpret_cast<void**>(&part), sizeof(uint64_t) * rows * Sr * R, st);
        if (e != cudaSuccess) return e;
      }
      const dim3 grid(static_cast<unsigned>(rtiles), Sr);
      if (R <= 32)
        fx_coarse_kernel<1, NJ><<<grid, 256, smem, st>>>(X + lo * dim, rows, dim, mu, mnorm, nlist, R, sh, span,
                                                     out_idx + lo * R, out_dist + lo * R, part);
      else if (R <= 64)
        fx_coarse_kernel<2, NJ><<<grid, 256, smem, st>>>(X + lo * dim, rows, dim, mu, mnorm, nlist, R, sh, span,
                                                     out_idx + lo * R, out_dist + lo * R, part);
      else
        fx_coarse_kernel<4, NJ><<<grid, 256, smem, st>>>(X + lo * dim, rows, dim, mu, mnorm, nlist, R, sh, span,
                                                     out_idx + lo * R, out_dist + lo * R, part);
      note_launch();
      if (Sr > 1) {
        dispatch_kr(R, [&]<int KR>() {
          fx_merge_kernel<KR><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(part, rows, Sr, R, sh,
                                                                                   out_idx + lo * R,
                                                                                   out_dist + lo * R);
        });
        note_launch();
        cudaFreeAsync(part, st);
      }
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // R > 128: the [rows x nlist] distance matrix in HBM, then a warp per row
  const int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(n, (int64_t(1) << 30) / nlist));  // <= 8 GB
  int64_t* dm = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&dm), sizeof(int64_t) * chunk * nlist, st);
  if (e != cudaSuccess) return e;
  for (int64_t lo = 0; lo < n && e == cudaSuccess; lo += chunk) {
    const int64_t rows = std::min(chunk, n - lo);
    dist_matrix_kernel<<<dim3((nlist + 63) / 64, static_cast<unsigned>((rows + 63) / 64)), 256, 0, st>>>(
        X + lo * dim, rows, dim, mu, mnorm, nlist, dm);
    const unsigned rb = static_cast<unsigned>((rows + 7) / 8);
    dispatch_kr(R, [&]<int KR>() {
      row_topk_kernel<KR><<<rb, 256, 0, st>>>(dm, rows, nlist, R, sh, out_idx + lo * R, out_dist + lo * R);
    });
    note_launch(2);
    e = cudaGetLastError();
  }
  cudaFreeAsync(dm, st);
  return e;
}

cudaError_t fx_build_tail(const int32_t* db, int64_t n, int dim, const int32_t* mu, const int32_t* list_of,
                          const int32_t* flat_pos, int M, int Ks, const int32_t* codeword_rows, int nlist, int L,
                          int32_t* cb, uint8_t* codes, int32_t* ids, int64_t* pterm, cudaStream_t st) {
  const int64_t tcb = static_cast<int64_t>(dim) * Ks;
  codebook32_kernel<<<static_cast<int>(std::min<int64_t>((tcb + 255) / 256, 4096)), 256, 0, st>>>(
      db, mu, list_of, dim, M, Ks, codeword_rows, cb);
  encode32_kernel<<<static_cast<int>(std::min<int64_t>((n * M + 255) / 256, 148 * 64)), 256, 0, st>>>(
      db, n, dim, mu, list_of, flat_pos, cb, M, Ks, codes, ids);
  const int64_t slots = static_cast<int64_t>(nlist) * L;
  slot_terms64_kernel<<<static_cast<int>(std::min<int64_t>((slots + 255) / 256, 8192)), 256, 0, st>>>(
      mu, cb, codes, ids, nlist, L, dim, M, Ks, pterm);
  note_launch(3);
  return cudaGetLastError();
}

// smem = table bytes (0 when GA) + fx_rest(8).
size_t fx_rest(const FxScanArgs& a, int nw) {
  return sizeof(uint64_t) * nw * a.cap + 12 * static_cast<size_t>(a.k) + 4 * static_cast<size_t>(a.dim + 4) + 16 + 64;
}

template <int MT, int KS, bool GA, bool ROT = false>
cudaError_t launch_scan_fx(const FxScanArgs& a, int64_t nq, size_t smem8, cudaStream_t st) {
  // A table too large for two CTAs per SM leaves one CTA of 8 warps per SM: then 12 warps when
  // their per-warp lists still fit (option V3DB_OPT_FX_W12 = 8 forces 8 warps)
  if constexpr (MT == 96 && ROT) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t smem12 = smem8 - fx_rest(a, 8) + fx_rest(a, 12);
    if (smem8 > 114 * 1024 && smem12 <= static_cast<size_t>(optin) && opt(V3DB_OPT_FX_W12) != 8) {
      auto kern = scan_fx_kernel<MT, KS, GA, ROT, 12>;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem12));
      if (e != cudaSuccess) return e;
      kern<<<static_cast<unsigned>(nq), 384, smem12, st>>>(a);
      note_launch();
      return cudaGetLastError();
    }
  }
  auto kern = scan_fx_kernel<MT, KS, GA, ROT, 8>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem8));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(nq), 256, smem8, st>>>(a);
  note_launch();
  return cudaGetLastError();
}

template <int MT>
cudaError_t launch_scan_fx_m(const FxScanArgs& a, int64_t nq, size_t smem, cudaStream_t st, bool rot) {
  if constexpr (MT % 8 == 0) {
    if (rot) return launch_scan_fx<MT, 256, false, true>(a, nq, smem, st);
  }
  return a.Ks == 256 ? launch_scan_fx<MT, 256, false>(a, nq, smem, st) : launch_scan_fx<MT, 0, false>(a, nq, smem, st);
}

static cudaError_t fx_scan_launch(const v3db_snapshot* s, FxScanArgs& a, int64_t nq, size_t smem, cudaStream_t st);

cudaError_t fx_scan(const v3db_snapshot* s, const int32_t* queries, int64_t nq, int nprobe, int k, const int32_t* lists,
                    const int64_t* ldist, int32_t* out_ids, int64_t* out_dist, int64_t* trace, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  FxScanArgs a;
  a.queries = queries;
  a.dim = s->dim;
  a.M = s->M;
  a.Ks = s->Ks;
  a.L = s->L;
  a.nprobe = nprobe;
  a.k = k;
  a.sh5 = fx_shift5(s->dim);
  a.cap = k;
  if (k <= 256) {  // buffered per-warp top-k: a power of two >= 2k + 32
    a.cap = 64;
    while (a.cap < 2 * k + 32) a.cap <<= 1;
  }
  a.cb = s->codebooks32;
  a.codes = s->codes;
  a.pterm = s->pterm64;
  a.ids = s->ids;
  a.counts = s->counts;
  a.lists = lists;
  a.ldist = ldist;
  a.out_ids = out_ids;
  a.out_dist = out_dist;
  a.trace = trace;
  a.Ag = nullptr;
  a.order = nullptr;
  if (a.sh5 < 1 || static_cast<int64_t>(nprobe) * s->L > (int64_t(1) << std::min(a.sh5, 31))) return cudaErrorInvalidValue;
  const size_t abytes = sizeof(int64_t) * s->M * s->Ks;
  const size_t rest = fx_rest(a, 8);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const bool a_smem = abytes + rest <= static_cast<size_t>(optin);
  if (!a_smem) {  // the table in per-query global scratch
    void* scratch = nullptr;
    cudaError_t e = scratch_alloc(&scratch, abytes * nq, st);
    if (e != cudaSuccess) return e;
    a.Ag = static_cast<int64_t*>(scratch);
    e = launch_scan_fx<0, 0, true>(a, nq, rest, st);  // canonical codes
    cudaFreeAsync(scratch, st);
    return e;
  }
  const size_t smem = abytes + rest;
  // the int8 scan's L2-aware query order, under the same condition (snapshot codes beyond L2)
  const int64_t sched = opt(V3DB_OPT_SCHED);
  const bool want = sched ? sched == 1
                          : (nq >= 2048 && static_cast<int64_t>(s->nlist) * s->L * s->M > (int64_t(64) << 20));
  if (want) {
    void* sbuf = nullptr;
    cudaError_t e = scratch_alloc(&sbuf, sizeof(int32_t) * (2 * nq + s->nlist), st);
    if (e != cudaSuccess) return e;
    e = minhash_order(lists, nq, nprobe, s->nlist, static_cast<int32_t*>(sbuf), st);
    if (e == cudaSuccess) {
      a.order = static_cast<int32_t*>(sbuf) + nq;
      e = fx_scan_launch(s, a, nq, smem, st);
    }
    cudaFreeAsync(sbuf, st);
    return e;
  }
  return fx_scan_launch(s, a, nq, smem, st);
}

bool fx_rot_supported(int M, int Ks) {
  return Ks == 256 && (M == 8 || M == 16 || M == 24 || M == 32 || M == 64 || M == 96);
}

static cudaError_t fx_scan_launch(const v3db_snapshot* s, FxScanArgs& a, int64_t nq, size_t smem, cudaStream_t st) {
  const bool rot = s->codes_rot16 != nullptr && fx_rot_supported(s->M, s->Ks);  // built iff supported
  if (rot) a.codes = s->codes_rot16;
  switch (s->M) {
    case 8: return launch_scan_fx_m<8>(a, nq, smem, st, rot);
    case 16: return launch_scan_fx_m<16>(a, nq, smem, st, rot);
    case 24: return launch_scan_fx_m<24>(a, nq, smem, st, rot);
    case 32: return launch_scan_fx_m<32>(a, nq, smem, st, rot);
    case 64: return launch_scan_fx_m<64>(a, nq, smem, st, rot);
    case 96: return launch_scan_fx_m<96>(a, nq, smem, st, rot);
    default:
      a.codes = s->codes;  // the generic loop reads the canonical layout
      return launch_scan_fx<0, 0, false>(a, nq, smem, st);
  }
}

}  // namespace v3db

// fx16.cu -- NEXT-1: the five-step semantics on the paper's own 16-bit
// fixed-point representation: coordinates round((2^16-1) v / v_max) in
// [-65535, 65535] (int32), all distances exact in int64 (d_max = 2^63 - 1), codewords the residual
// sub-vectors themselves (R19).  Same steps and readings as the int8 path; different arithmetic:
//   * Step 1 (and the build ranking): <x, mu> via IEEE-double FMAs -- exact, every partial sum is
//     an integer below dim * 65535^2 < 2^53 -- in a tiled kernel that writes the [rows x nlist]
//     int64 distance matrix; a warp per row then keeps the R smallest (d, i) as 64-bit composite
//     keys (d << sh | i, sh from the distance bound);
//   * Steps 3-5: one CTA per query, the factorised table A_q[m][c] = -2 <C_{m,c}, q^{(m)}> in int64
//     (shared memory), D = d_i + P_{i,j} + sum_m A_q[m][c_m] per slot, every D to the trace, per-warp
//     threshold top-k on (D << sh5 | slot) keys for the k-th D, then the exact (D, item) order of
//     the candidates with D <= that value (ties resolved by item id, R10).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
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
    const double r = y >= 0.0 ? floor(__dadd_rn(y, 0.5)) : -floor(__dadd_rn(-y, 0.5));  // half away from zero (R18)
    out[i] = static_cast<int32_t>(r);
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
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
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
    const int64_t r = r0 + ty * 4 + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c >= nlist) continue;
      out[r * nlist + c] = xn_s[ty * 4 + i] + mnorm[c] - 2 * static_cast<long long>(acc[i][j]);
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

// Steps 3-5 for one query per CTA (256 threads).
struct FxScanArgs {
  const int32_t* queries;
  int dim, M, Ks, L, nprobe, k, sh5, cap;
  const int32_t* cb;         // [M][Ks][d]
  const uint8_t* codes;      // canonical [nlist][L][M]
  const int64_t* pterm;      // [nlist][L]
  const int32_t* ids;
  const int32_t* counts;
  const int32_t* lists;      // [nq][nprobe]
  const int64_t* ldist;      // [nq][nprobe]
  int32_t* out_ids;
  int64_t* out_dist;
  int64_t* dbuf;             // [nq][nprobe][L]: the trace (or scratch)
  int64_t* Ag;               // [nq][M][Ks] when the table does not fit in shared memory, else null
  int* overflow;             // set when ties exceed the final buffer
};

__global__ void __launch_bounds__(256) scan_fx_kernel(const FxScanArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int W = 8;
  const int64_t qi = blockIdx.x;
  int64_t* A = a.Ag ? a.Ag + qi * a.M * a.Ks : reinterpret_cast<int64_t*>(smem);           // [M][Ks]
  uint64_t* tops = reinterpret_cast<uint64_t*>(smem + (a.Ag ? 0 : sizeof(int64_t) * a.M * a.Ks));  // [W][k]
  int64_t* bd = reinterpret_cast<int64_t*>(tops + W * a.k);      // [cap] final candidates: D
  int32_t* bi = reinterpret_cast<int32_t*>(bd + a.cap);          // [cap] item
  int* s_cnt = bi + a.cap;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int d = a.dim / a.M, L = a.L, nprobe = a.nprobe;
  const int32_t* q = a.queries + qi * a.dim;
  for (int e = tid; e < a.M * a.Ks; e += 256) {
    const int m = e / a.Ks;
    const int32_t* cw = a.cb + static_cast<int64_t>(e) * d;
    long long acc = 0;
    for (int u = 0; u < d; ++u) acc += static_cast<long long>(cw[u]) * q[m * d + u];
    A[e] = -2 * acc;
  }
  for (int e = tid; e < W * a.k; e += 256) tops[e] = ~0ull;
  if (tid == 0) *s_cnt = 0;
  __syncthreads();
  uint64_t* T = tops + warp * a.k;
  uint64_t thr = ~0ull;
  int64_t* drow = a.dbuf + qi * nprobe * static_cast<int64_t>(L);
  for (int rho = 0; rho < nprobe; ++rho) {
    const int li = a.lists[qi * nprobe + rho];
    const long long di = a.ldist[qi * nprobe + rho];
    const int cnt = a.counts[li];
    const int64_t base = static_cast<int64_t>(li) * L;
    for (int j0 = warp * 32; j0 < L; j0 += W * 32) {
      const int j = j0 + lane;
      long long D = kDMaxFx;
      if (j < cnt) {
        long long acc = di + a.pterm[base + j];
        const uint8_t* cp = a.codes + (base + j) * a.M;
        for (int m = 0; m < a.M; ++m) acc += A[m * a.Ks + cp[m]];
        D = acc;
      }
      if (j < L) drow[static_cast<int64_t>(rho) * L + j] = D;
      const uint64_t key = j < cnt ? (static_cast<uint64_t>(D) << a.sh5) | static_cast<uint32_t>(rho * L + j) : ~0ull;
      thr = warp_offer(T, a.k, thr, key);
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < W; ++w)
      for (int b = 0; b < a.k; b += 32) thr = warp_offer(tops, a.k, thr, b + lane < a.k ? tops[w * a.k + b + lane] : ~0ull);
  }
  __syncthreads();
  // tau = D of the k-th smallest (D, slot) key: every candidate of the final top-k has D <= tau
  const uint64_t kth = tops[a.k - 1];
  const long long tau = kth == ~0ull ? kDMaxFx - 1 : static_cast<long long>(kth >> a.sh5);
  __syncthreads();
  // Step 5 in the exact (D, item) order among the candidates with D <= tau (R10)
  for (int rho = 0; rho < nprobe; ++rho) {
    const int li = a.lists[qi * nprobe + rho];
    const int cnt = a.counts[li];
    for (int j = tid; j < cnt; j += 256) {
      const long long D = drow[static_cast<int64_t>(rho) * L + j];
      if (D <= tau) {
        const int pos = atomicAdd(s_cnt, 1);
        if (pos < a.cap) {
          bd[pos] = D;
          bi[pos] = a.ids[static_cast<int64_t>(li) * L + j];
        }
      }
    }
  }
  __syncthreads();
  const int n = *s_cnt;
  if (n > a.cap) {
    if (tid == 0) atomicExch(a.overflow, 1);
    return;
  }
  for (int e = tid; e < n; e += 256) {
    const long long D = bd[e];
    const int32_t id = bi[e];
    int rank = 0;
    for (int f = 0; f < n; ++f) rank += (bd[f] < D || (bd[f] == D && bi[f] < id)) ? 1 : 0;
    if (rank < a.k) {
      a.out_ids[qi * a.k + rank] = id;
      a.out_dist[qi * a.k + rank] = D;
    }
  }
  for (int r = n + tid; r < a.k; r += 256) {
    a.out_ids[qi * a.k + r] = -1;
    a.out_dist[qi * a.k + r] = kDMaxFx;
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
  const int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(n, (int64_t(1) << 30) / nlist));  // <= 8 GB
  int64_t* dm = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dm), sizeof(int64_t) * chunk * nlist, st);
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
  a.cap = std::max(4096, 4 * k);
  a.cb = s->codebooks32;
  a.codes = s->codes;
  a.pterm = s->pterm64;
  a.ids = s->ids;
  a.counts = s->counts;
  a.lists = lists;
  a.ldist = ldist;
  a.out_ids = out_ids;
  a.out_dist = out_dist;
  if (a.sh5 < 1 || static_cast<int64_t>(nprobe) * s->L > (int64_t(1) << std::min(a.sh5, 31))) return cudaErrorInvalidValue;
  // the table A_q stays in shared memory up to 96 KiB (M * Ks <= 12288), else per-query scratch
  const size_t abytes = sizeof(int64_t) * s->M * s->Ks;
  const bool a_smem = abytes <= 96 * 1024;
  void* scratch = nullptr;
  const size_t tb = trace ? 0 : sizeof(int64_t) * nq * nprobe * s->L;
  const size_t ab = a_smem ? 0 : abytes * nq;
  cudaError_t e = cudaMallocAsync(&scratch, tb + ab + 256, st);
  if (e != cudaSuccess) return e;
  a.overflow = static_cast<int*>(scratch);
  a.dbuf = trace ? trace : reinterpret_cast<int64_t*>(static_cast<uint8_t*>(scratch) + 256);
  a.Ag = a_smem ? nullptr : reinterpret_cast<int64_t*>(static_cast<uint8_t*>(scratch) + 256 + tb);
  e = cudaMemsetAsync(a.overflow, 0, sizeof(int), st);
  const size_t smem = (a_smem ? abytes : 0) + sizeof(uint64_t) * 8 * k + (8 + 4) * static_cast<size_t>(a.cap) + 16;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(scan_fx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    scan_fx_kernel<<<static_cast<unsigned>(nq), 256, smem, st>>>(a);
    note_launch();
    e = cudaGetLastError();
  }
  int ovf = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ovf, a.overflow, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(scratch, st);
  if (e == cudaSuccess && ovf) return cudaErrorNotSupported;  // ties beyond the final buffer
  return e;
}

}  // namespace v3db

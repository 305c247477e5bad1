// build_kernels.cu -- offline index shaping kernels (BUILD rows of SURVEY.md §8(a)).
//
//   B1 gather_rows      mu_i = db[centroid_rows[i]], ||mu_i||^2          (BASELINE.json rule)
//   B4 make_codebooks   C_{m,c} = sat_[-127,127](db[row] - mu_{list(row)})^{(m)}   (R5)
//   B3+B5 encode_and_place  residual r_t = db[t] - mu_{list(t)} (int16, unclamped),
//                       code_t[m] = argmin_c dist(r_t^{(m)}, C_{m,c}), lowest c (R6),
//                       written to the slot chosen by the host greedy (B2/B6)
//   slot_terms          P_{i,j} = ||xhat_ij||^2 + 2 <mu_i, xhat_ij>, the per-slot term of the
//                       exact identity d~_ij = d_i + P_ij + sum_m A_q[m][c_m] used by the scan
//                       (DESIGN.md "LUT factorisation"); 0 for padding slots.
//   rotate_codes        codes_rot: the layout the rotated-LUT scan reads (DESIGN.md "Rotated LUT
//                       layout"); transpose_codebooks: cbT [Ks][M][d].
// PQ of residuals: PAPER.md:97-100; fixed-shape lists: PAPER.md:292-294, 331-340.
#include <cuda_runtime.h>
#include <stdint.h>

#include "v3db_internal.cuh"

namespace v3db {
namespace {

__global__ void gather_rows_kernel(const int8_t* __restrict__ db, int dim, const int32_t* __restrict__ rows,
                                   int nrows, int8_t* __restrict__ out, int32_t* __restrict__ norms) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nrows) return;
  const int8_t* src = db + static_cast<int64_t>(rows[warp]) * dim;
  int acc = 0;
  for (int u = lane; u < dim; u += 32) {
    const int v = src[u];
    out[static_cast<int64_t>(warp) * dim + u] = static_cast<int8_t>(v);
    acc += v * v;
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  if (norms && lane == 0) norms[warp] = acc;
}

__global__ void codebook_kernel(const int8_t* __restrict__ db, const int8_t* __restrict__ mu,
                                const int32_t* __restrict__ list_of, int dim, int M, int Ks,
                                const int32_t* __restrict__ codeword_rows, int8_t* __restrict__ cb) {
  const int d = dim / M;
  const int64_t total = static_cast<int64_t>(M) * Ks * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(e % d);
    const int64_t mc = e / d;                    // m * Ks + c
    const int m = static_cast<int>(mc / Ks);
    const int row = codeword_rows[mc];
    const int col = m * d + u;
    int v = static_cast<int>(db[static_cast<int64_t>(row) * dim + col]) -
            static_cast<int>(mu[static_cast<int64_t>(list_of[row]) * dim + col]);
    v = v < -127 ? -127 : (v > 127 ? 127 : v);
    cb[e] = static_cast<int8_t>(v);
  }
}

// One block = 256 consecutive vectors x one subspace m (blockIdx.y).  The subspace's
// codebook (Ks x d int8) is staged in shared memory; every lane reads the same codeword
// at the same time (broadcast).
template <int DS>
__global__ void __launch_bounds__(256) encode_kernel(const int8_t* __restrict__ db, int64_t n, int dim,
                                                     const int8_t* __restrict__ mu,
                                                     const int32_t* __restrict__ list_of,
                                                     const int32_t* __restrict__ flat_pos,
                                                     const int8_t* __restrict__ cb, int M, int Ks,
                                                     uint8_t* __restrict__ codes, int32_t* __restrict__ ids) {
  extern __shared__ int8_t sC[];  // [Ks][d]
  const int d = dim / M;
  const int m = blockIdx.y;
  for (int e = threadIdx.x; e < Ks * d; e += blockDim.x) sC[e] = cb[static_cast<int64_t>(m) * Ks * d + e];
  __syncthreads();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int li = list_of[t];
  int r[DS];
#pragma unroll
  for (int u = 0; u < DS; ++u) {
    r[u] = 0;
    if (u < d) {
      const int col = m * d + u;
      r[u] = static_cast<int>(db[t * dim + col]) - static_cast<int>(mu[static_cast<int64_t>(li) * dim + col]);
    }
  }
  int best = 0x7fffffff, bestc = 0;
  for (int c = 0; c < Ks; ++c) {
    int acc = 0;
#pragma unroll
    for (int u = 0; u < DS; ++u) {
      if (u < d) {
        const int diff = r[u] - static_cast<int>(sC[c * d + u]);
        acc += diff * diff;
      }
    }
    if (acc < best) {  // strict: the lowest c wins ties (R6)
      best = acc;
      bestc = c;
    }
  }
  const int64_t pos = flat_pos[t];
  codes[pos * M + m] = static_cast<uint8_t>(bestc);
  if (m == 0) ids[pos] = static_cast<int32_t>(t);
}

__global__ void slot_terms_kernel(const int8_t* __restrict__ mu, const int8_t* __restrict__ cb,
                                  const uint8_t* __restrict__ codes, const int32_t* __restrict__ ids, int nlist,
                                  int L, int dim, int M, int Ks, int32_t* __restrict__ pterm) {
  const int d = dim / M;
  const int64_t total = static_cast<int64_t>(nlist) * L;
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < total;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int acc = 0;
    if (ids[s] != -1) {
      const int8_t* mui = mu + (s / L) * dim;
      for (int m = 0; m < M; ++m) {
        const int8_t* cw = cb + (static_cast<int64_t>(m) * Ks + codes[s * M + m]) * d;
        for (int u = 0; u < d; ++u) {
          const int x = cw[u];
          acc += x * x + 2 * static_cast<int>(mui[m * d + u]) * x;
        }
      }
    }
    pterm[s] = acc;
  }
}

// Byte off_g + s of slot j holds the code of subspace off_g + (j + s) mod G_g for rotation group g
// (lane l = j mod 32 reads table column l + s, which holds that subspace; kLutP64 has the one group
// [0, M)).  kLutW32 additionally pre-compensates the row
// wrap of columns l + s >= 32: the stored byte is (code - 1) mod 256 there.  Each 32-slot chunk
// is stored unit-transposed: byte pos of slot j lives at chunk + (pos/U)*32*U + (j%32)*U + pos%U.
__global__ void rotate_kernel(const uint8_t* __restrict__ codes, const int32_t* __restrict__ pterm, int nlist,
                              int L, int Lp, int M, int mode, int G, int U, uint8_t* __restrict__ out,
                              int32_t* __restrict__ pout) {
  const int64_t total = static_cast<int64_t>(nlist) * Lp * M;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sp = e / M;                       // padded slot index i*Lp + jp
    const int pos = static_cast<int>(e - sp * M);
    const int i = static_cast<int>(sp / Lp), jp = static_cast<int>(sp - static_cast<int64_t>(i) * Lp);
    const int lane = jp & 31;
    int v = 0;
    if (jp < L) {
      int off = 0, Gg = M;
      if (mode == kLutW32) {
        int g = 0;
        while (pos >= rot_goff(M, g + 1) && g + 1 < rot_ngroups(M)) ++g;
        off = rot_goff(M, g);
        Gg = rot_gsize(M, g);
      }
      const int s = pos - off;
      v = codes[(static_cast<int64_t>(i) * L + jp) * M + off + (lane + s) % Gg];
      if (mode == kLutW32 && lane + s >= 32) v = (v + 255) & 255;
    }
    const int64_t chunk = sp >> 5;                  // (i*Lp + jp) / 32: chunks never straddle lists
    out[chunk * 32 * M + (pos / U) * 32 * U + lane * U + pos % U] = static_cast<uint8_t>(v);
    if (pos == 0) pout[sp] = jp < L ? pterm[static_cast<int64_t>(i) * L + jp] : 0;
  }
}

// xhat[i][jp][u] = C_{m, code_{i,jp,m}}[u - m d] (m = u / d): the reconstruction of slot (i, jp)
// (concatenated codewords) for valid slots, 0 for padding slots and jp >= L.
// 16 bytes per thread (dim % 16 == 0).
__global__ void xhat_kernel(const uint8_t* __restrict__ codes, const int32_t* __restrict__ counts,
                            const int8_t* __restrict__ cb, int nlist, int L, int Lp, int dim, int M, int Ks,
                            int8_t* __restrict__ out) {
  const int d = dim / M, cpr = dim / 16;
  const int64_t total = static_cast<int64_t>(nlist) * Lp * cpr;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sp = e / cpr;
    const int c = static_cast<int>(e - sp * cpr);
    const int i = static_cast<int>(sp / Lp), jp = static_cast<int>(sp - static_cast<int64_t>(i) * Lp);
    alignas(16) int8_t v[16];
    if (jp < __ldg(counts + i)) {
      const uint8_t* cd = codes + (static_cast<int64_t>(i) * L + jp) * M;
      for (int b = 0; b < 16; ++b) {
        const int u = c * 16 + b, m = u / d;
        v[b] = cb[(static_cast<int64_t>(m) * Ks + cd[m]) * d + (u - m * d)];
      }
    } else {
      for (int b = 0; b < 16; ++b) v[b] = 0;
    }
    *reinterpret_cast<int4*>(out + sp * dim + c * 16) = *reinterpret_cast<const int4*>(v);
  }
}

// Fixed point: xl[l][i][jp][u] = limb l of C_{m, code_{i,jp,m}}[u - m d] (balanced base-256 digits,
// v = v_0 + 256 v_1 + 65536 v_2) for valid slots, 0 for padding slots and jp >= L.
__global__ void xhat_fx_kernel(const uint8_t* __restrict__ codes, const int32_t* __restrict__ counts,
                               const int32_t* __restrict__ cb, int nlist, int L, int Lp, int dim, int M, int Ks,
                               int8_t* __restrict__ out) {
  const int d = dim / M;
  const int64_t plane = static_cast<int64_t>(nlist) * Lp * dim;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < plane;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t sp = e / dim;
    const int u = static_cast<int>(e - sp * dim);
    const int i = static_cast<int>(sp / Lp), jp = static_cast<int>(sp - static_cast<int64_t>(i) * Lp);
    int v = 0;
    if (jp < __ldg(counts + i)) {
      const int m = u / d;
      v = __ldg(cb + (static_cast<int64_t>(m) * Ks + codes[(static_cast<int64_t>(i) * L + jp) * M + m]) * d + (u - m * d));
    }
    const int d0 = ((v + 128) & 255) - 128, w = (v - d0) >> 8;
    const int d1 = ((w + 128) & 255) - 128, d2 = (w - d1) >> 8;
    out[e] = static_cast<int8_t>(d0);
    out[plane + e] = static_cast<int8_t>(d1);
    out[2 * plane + e] = static_cast<int8_t>(d2);
  }
}

__global__ void transpose_cb_kernel(const int8_t* __restrict__ cb, int M, int Ks, int d, int8_t* __restrict__ cbT) {
  const int total = M * Ks * d;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int u = e % d, mc = e / d, m = mc / Ks, c = mc - m * Ks;
    cbT[(static_cast<int64_t>(c) * M + m) * d + u] = cb[e];
  }
}

__global__ void pair_dist_kernel(const int8_t* __restrict__ X, int64_t n, int dim, const int8_t* __restrict__ mu,
                                 const int32_t* __restrict__ lists, int32_t* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  (void)warp;
  if (r >= n) return;
  const int8_t* x = X + r * dim;
  const int8_t* m = mu + static_cast<int64_t>(lists[r]) * dim;
  int acc = 0;
  for (int u = lane; u < dim; u += 32) {
    const int df = static_cast<int>(x[u]) - static_cast<int>(m[u]);
    acc += df * df;
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  if (lane == 0) out[r] = acc;
}

__global__ void delta_keys_kernel(const int32_t* __restrict__ e_t, const int32_t* __restrict__ e_i, int64_t n,
                                  int64_t P, uint64_t* __restrict__ keys) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < P;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t key = ~0ull;
    if (r < n) {
      const uint32_t d = static_cast<uint32_t>(e_t[r] - e_i[r]) ^ 0x80000000u;  // signed -> unsigned order
      key = (static_cast<uint64_t>(d) << 32) | static_cast<uint32_t>(r);
    }
    keys[r] = key;
  }
}

}  // namespace

cudaError_t pair_dist(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* lists, int32_t* out,
                      cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pair_dist_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(X, n, dim, mu, lists, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t delta_keys(const int32_t* e_t, const int32_t* e_i, int64_t n, int64_t P, uint64_t* keys, cudaStream_t st) {
  const int blocks = static_cast<int>((P + 255) / 256 < 16384 ? (P + 255) / 256 : 16384);
  delta_keys_kernel<<<blocks, 256, 0, st>>>(e_t, e_i, n, P, keys);
  note_launch();
  return cudaGetLastError();
}

cudaError_t rotate_codes(const uint8_t* codes, const int32_t* pterm, int nlist, int L, int M, int mode, int G,
                         uint8_t* codes_rot, int32_t* pterm_rot, cudaStream_t st) {
  const int Lp = (L + 31) & ~31;
  const int64_t total = static_cast<int64_t>(nlist) * Lp * M;
  const int blocks = static_cast<int>((total + 255) / 256 < 16384 ? (total + 255) / 256 : 16384);
  rotate_kernel<<<blocks, 256, 0, st>>>(codes, pterm, nlist, L, Lp, M, mode, G, rot_unit(M), codes_rot, pterm_rot);
  note_launch();
  return cudaGetLastError();
}

cudaError_t make_xhat(const uint8_t* codes, const int32_t* counts, const int8_t* cb, int nlist, int L, int Lp,
                      int dim, int M, int Ks, int8_t* xhat, cudaStream_t st) {
  if (dim % 16 != 0) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(nlist) * Lp * (dim / 16);
  const int blocks = static_cast<int>((total + 255) / 256 < 32768 ? (total + 255) / 256 : 32768);
  xhat_kernel<<<blocks, 256, 0, st>>>(codes, counts, cb, nlist, L, Lp, dim, M, Ks, xhat);
  note_launch();
  return cudaGetLastError();
}

cudaError_t make_xhat_fx(const uint8_t* codes, const int32_t* counts, const int32_t* cb, int nlist, int L, int Lp,
                         int dim, int M, int Ks, int8_t* xl, cudaStream_t st) {
  const int64_t plane = static_cast<int64_t>(nlist) * Lp * dim;
  const int blocks = static_cast<int>((plane + 255) / 256 < 32768 ? (plane + 255) / 256 : 32768);
  xhat_fx_kernel<<<blocks, 256, 0, st>>>(codes, counts, cb, nlist, L, Lp, dim, M, Ks, xl);
  note_launch();
  return cudaGetLastError();
}

cudaError_t transpose_codebooks(const int8_t* cb, int M, int Ks, int d, int8_t* cbT, cudaStream_t st) {
  const int total = M * Ks * d;
  transpose_cb_kernel<<<(total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024, 256, 0, st>>>(cb, M, Ks, d, cbT);
  note_launch();
  return cudaGetLastError();
}

cudaError_t gather_rows(const int8_t* db, int dim, const int32_t* rows, int nrows, int8_t* out, int32_t* norms,
                        cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  gather_rows_kernel<<<(nrows * 32 + 255) / 256, 256, 0, st>>>(db, dim, rows, nrows, out, norms);
  note_launch();
  return cudaGetLastError();
}

cudaError_t make_codebooks(const int8_t* db, const int8_t* mu, const int32_t* list_of, int dim, int M, int Ks,
                           const int32_t* codeword_rows, int8_t* codebooks, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(dim) * Ks;
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  codebook_kernel<<<blocks, 256, 0, st>>>(db, mu, list_of, dim, M, Ks, codeword_rows, codebooks);
  note_launch();
  return cudaGetLastError();
}

cudaError_t encode_and_place(const int8_t* db, int64_t n, int dim, const int8_t* mu, const int32_t* list_of,
                             const int32_t* flat_pos, const int8_t* codebooks, int M, int Ks, uint8_t* codes,
                             int32_t* ids, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int d = dim / M;
  dim3 grid(static_cast<unsigned>((n + 255) / 256), M);
  const size_t smem = static_cast<size_t>(Ks) * d;
#define V3DB_ENC(DS)                                                                                         \
  encode_kernel<DS><<<grid, 256, smem, st>>>(db, n, dim, mu, list_of, flat_pos, codebooks, M, Ks, codes, ids); \
  break;
  switch (d <= 4 ? 4 : d <= 8 ? 8 : d <= 16 ? 16 : d <= 32 ? 32 : 64) {
    case 4: V3DB_ENC(4)
    case 8: V3DB_ENC(8)
    case 16: V3DB_ENC(16)
    case 32: V3DB_ENC(32)
    default: V3DB_ENC(64)
  }
#undef V3DB_ENC
  note_launch();
  return cudaGetLastError();
}

cudaError_t slot_terms(const int8_t* mu, const int8_t* codebooks, const uint8_t* codes, const int32_t* ids,
                       int nlist, int L, int dim, int M, int Ks, int32_t* pterm, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(nlist) * L;
  const int blocks = static_cast<int>((total + 255) / 256 < 8192 ? (total + 255) / 256 : 8192);
  slot_terms_kernel<<<blocks, 256, 0, st>>>(mu, codebooks, codes, ids, nlist, L, dim, M, Ks, pterm);
  note_launch();
  return cudaGetLastError();
}

}  // namespace v3db

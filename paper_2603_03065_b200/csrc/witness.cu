// witness.cu -- the prover witness of a batch of (challenged) queries: the sequences the
// multiset-based design of PAPER.md §4.7 takes from the off-circuit run.
//   S^sorted_{idx,dist}   all n_list pairs (i, d_i) in (d_i, i) order
//   l^{(m)}_{i,j}         LUT_{i,m,v^{(m)}_{i,j}} of every probed slot and subspace
//                         -- the literal Step-3 tables, not the factorised
//                         per-query table of the hot path
//   S^sorted_{item,dist}  all N_sel candidate pairs (item, D) in (D, item) order
// On demand, per challenged query: 6.3 MB of selected entries per C4
// query.  Sorting uses composite 64-bit keys (R9 / R10 total orders) and a segmented bitonic
// network in global memory (one launch per step).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

// keys[q][i] = (d_i << 32) | i for i < nlist (Step 1), ~0 up to P.
__global__ void list_keys_kernel(const int8_t* __restrict__ queries, int64_t nq, int dim,
                                 const int8_t* __restrict__ mu, int nlist, int P, uint64_t* __restrict__ keys) {
  const int64_t total = nq * P;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / P;
    const int i = static_cast<int>(e - q * P);
    uint64_t key = ~0ull;
    if (i < nlist) {
      const int8_t* x = queries + q * dim;
      const int8_t* m = mu + static_cast<int64_t>(i) * dim;
      int d = 0;
      for (int u = 0; u < dim; ++u) {
        const int df = static_cast<int>(x[u]) - static_cast<int>(m[u]);
        d += df * df;
      }
      key = step2_key(d, i);
    }
    keys[e] = key;
  }
}

// One step (size, stride) of an ascending bitonic sort of every P-key segment.
__global__ void bitonic_step_kernel(uint64_t* __restrict__ keys, int64_t pairs, int P, int size, int stride) {
  const int half = P >> 1;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < pairs;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t seg = t / half;
    const int loc = static_cast<int>(t - seg * half);
    const int lo = 2 * loc - (loc & (stride - 1)), hi = lo + stride;
    uint64_t* k = keys + seg * P;
    const uint64_t a = k[lo], b = k[hi];
    if ((a > b) == ((lo & size) == 0)) {
      k[lo] = b;
      k[hi] = a;
    }
  }
}

// The steps of a bitonic sort whose stride is below the tile, in shared memory: one CTA per
// tile of `tile` keys (a power of two dividing P, so a tile never straddles a segment).  The
// direction of a compare-exchange depends on the key's index within its segment, exactly as in
// bitonic_step_kernel.  size_lo..size_hi: the merge sizes to run (strides size/2 .. 1 each, only
// those below the tile).
__global__ void __launch_bounds__(512) bitonic_tile_kernel(uint64_t* __restrict__ keys, int P, int tile, int size_lo,
                                                           int size_hi) {
  extern __shared__ uint64_t sk[];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * tile;
  const int off = static_cast<int>(base % P);
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sk[e] = keys[base + e];
  __syncthreads();
  for (int size = size_lo; size <= size_hi; size <<= 1) {
    for (int stride = min(size, tile) >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (tile >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const uint64_t a = sk[lo], b = sk[hi];
        if ((a > b) == (((off + lo) & size) == 0)) {
          sk[lo] = b;
          sk[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x) keys[base + e] = sk[e];
}

// Per (query, probe rank): the literal Step-3 table LUT_{i,m,c} = dist(C_{m,c}, (q - mu_i)^{(m)})
// in shared memory, then for every slot j the selected entries l^{(m)}_{i,j} (Step 4 witness) and
// the Step-5 key of the masked candidate distance D_{i,j}.
__global__ void __launch_bounds__(256) lut_witness_kernel(
    const int8_t* __restrict__ queries, int dim, const int8_t* __restrict__ mu, const int8_t* __restrict__ cb, int M,
    int Ks, int L, const uint8_t* __restrict__ codes, const int32_t* __restrict__ ids,
    const uint64_t* __restrict__ list_keys, int P1, int nprobe, int32_t* __restrict__ lut_sel, uint64_t* __restrict__ cand_keys,
    int P2) {
  extern __shared__ int32_t lut[];  // [M][Ks]
  int* res = lut + M * Ks;          // [dim] q - mu_i
  const int64_t q = blockIdx.y;
  const int rho = blockIdx.x;
  const int i = static_cast<int>(list_keys[q * P1 + rho] & 0xffffffffu);  // P(q)[rho]
  const int d = dim / M;
  for (int u = threadIdx.x; u < dim; u += blockDim.x)
    res[u] = static_cast<int>(queries[q * dim + u]) - static_cast<int>(mu[static_cast<int64_t>(i) * dim + u]);
  __syncthreads();
  for (int e = threadIdx.x; e < M * Ks; e += blockDim.x) {
    const int m = e / Ks;
    const int8_t* cw = cb + static_cast<int64_t>(e) * d;
    int acc = 0;
    for (int u = 0; u < d; ++u) {
      const int df = static_cast<int>(cw[u]) - res[m * d + u];
      acc += df * df;
    }
    lut[e] = acc;
  }
  __syncthreads();
  const int64_t sbase = static_cast<int64_t>(i) * L;
  if (lut_sel) {
    int32_t* out = lut_sel + (q * nprobe + rho) * static_cast<int64_t>(L) * M;
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(L) * M; e += blockDim.x) {
      const int m = static_cast<int>(e % M);
      out[e] = lut[m * Ks + codes[sbase * M + e]];
    }
  }
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const int32_t id = ids[sbase + j];
    int32_t D = kDMax;
    if (id != -1) {
      int acc = 0;
      for (int m = 0; m < M; ++m) acc += lut[m * Ks + codes[(sbase + j) * M + m]];
      D = acc;
    }
    cand_keys[q * P2 + static_cast<int64_t>(rho) * L + j] = step5_key(D, id);
  }
}

__global__ void fill_kernel(uint64_t* __restrict__ keys, int64_t nq, int P, int from) {
  const int64_t total = nq * P;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (e % P >= from) keys[e] = ~0ull;
}

__global__ void unpack_kernel(const uint64_t* __restrict__ keys, int64_t nq, int P, int n, bool step5,
                              int32_t* __restrict__ item, int32_t* __restrict__ dist) {
  const int64_t total = nq * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / n;
    const uint64_t key = keys[q * P + (e - q * n)];
    if (item) item[e] = step5 ? step5_id(key) : static_cast<int32_t>(key & 0xffffffffu);
    if (dist) dist[e] = static_cast<int32_t>(key >> 32);
  }
}

int64_t pow2_at_least(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace

// Ascending sort of every P-key segment (P a power of two): bitonic network.  Steps whose stride
// is below the 4096-key tile run in shared memory (bitonic_tile_kernel: all sizes up to the tile
// in one launch, then one launch per larger size); only the larger strides are global passes
// (one launch each) -- 15 launches instead of 136 for a 2^16-key segment.
cudaError_t segmented_sort(uint64_t* keys, int64_t nseg, int P, cudaStream_t st) {
  const int64_t pairs = nseg * (P / 2);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((pairs + 255) / 256, 148 * 16));
  const int tile = std::min(P, 4096);
  const int64_t tiles = nseg * (P / tile);
  const size_t smem = sizeof(uint64_t) * tile;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(bitonic_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  bitonic_tile_kernel<<<static_cast<unsigned>(tiles), 512, smem, st>>>(keys, P, tile, 2, tile);
  note_launch();
  for (int size = 2 * tile; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride >= tile; stride >>= 1) {
      bitonic_step_kernel<<<grid, 256, 0, st>>>(keys, pairs, P, size, stride);
      note_launch();
    }
    bitonic_tile_kernel<<<static_cast<unsigned>(tiles), 512, smem, st>>>(keys, P, tile, size, size);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t witness_batch(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int32_t* list_order,
                          int32_t* list_dist, int32_t* lut_sel, int32_t* cand_items, int32_t* cand_dist,
                          cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  const int64_t nsel = static_cast<int64_t>(nprobe) * s->L;
  // segments of up to 2^30 keys (segmented_sort's int segment length; larger ones are refused)
  if (pow2_at_least(s->nlist) > (int64_t(1) << 30) || pow2_at_least(nsel) > (int64_t(1) << 30))
    return cudaErrorInvalidValue;
  const int P1 = static_cast<int>(pow2_at_least(s->nlist));
  const int P2 = static_cast<int>(pow2_at_least(nsel));
  uint64_t* keys1 = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&keys1), sizeof(uint64_t) * (nq * P1 + nq * P2), st);
  if (e != cudaSuccess) return e;
  uint64_t* keys2 = keys1 + nq * P1;
  const unsigned g = 148 * 8;
  list_keys_kernel<<<g, 256, 0, st>>>(queries, nq, s->dim, s->centroids, s->nlist, P1, keys1);
  note_launch();
  e = segmented_sort(keys1, nq, P1, st);  // Step 2's full order
  if (e == cudaSuccess) {
    const size_t smem = sizeof(int32_t) * (static_cast<size_t>(s->M) * s->Ks + s->dim);
    e = cudaFuncSetAttribute(lut_witness_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) {
      fill_kernel<<<g, 256, 0, st>>>(keys2, nq, P2, static_cast<int>(nsel));
      lut_witness_kernel<<<dim3(nprobe, static_cast<unsigned>(nq)), 256, smem, st>>>(
          queries, s->dim, s->centroids, s->codebooks, s->M, s->Ks, s->L, s->codes, s->ids, keys1, P1, nprobe, lut_sel,
          keys2, P2);
      note_launch(2);
      e = segmented_sort(keys2, nq, P2, st);  // Step 5's full order
    }
  }
  if (e == cudaSuccess && (list_order || list_dist)) {
    unpack_kernel<<<g, 256, 0, st>>>(keys1, nq, P1, s->nlist, false, list_order, list_dist);
    note_launch();
  }
  if (e == cudaSuccess && (cand_items || cand_dist)) {
    unpack_kernel<<<g, 256, 0, st>>>(keys2, nq, P2, static_cast<int>(nsel), true, cand_items, cand_dist);
    note_launch();
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFreeAsync(keys1, st);
  return e;
}

}  // namespace v3db

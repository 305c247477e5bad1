// scan_lut.cu -- Steps 3-5 of PAPER.md §4.2, generic query-major scan: one CTA per query.
// Serves every shape; the rotated-LUT kernel of scan_rot.cu replaces it where its
// conflict-free table geometry applies.
//
// Step 3 defines, per probed list i, LUT_{i,m,c} = dist(C_{m,c}, (q-mu_i)^{(m)}).
// Summed over the M sub-blocks selected by a slot's code this is (exact integer identity,
// DESIGN.md "LUT factorisation"):
//   d~_{i,j} = sum_m LUT_{i,m,c_m} = d_i + P_{i,j} + sum_m A_q[m][c_m]
//   with d_i = dist(q, mu_i) (Step 1), P_{i,j} = ||xhat_ij||^2 + 2<mu_i, xhat_ij> (per slot,
//   built once) and A_q[m][c] = -2 <C_{m,c}, q^{(m)}> (per query, shared by all probed lists).
// So each CTA builds ONE table A_q [M][Ks] int32 in shared memory instead of nprobe tables,
// then streams the probed lists' codes from HBM (Step 4): padding slots
// (f = 0, i.e. slot >= count_i) get D = d_max; every D is written to the trace; a
// threshold-pruned warp top-k on (D, id) keys (Step 5) loads ids lazily.
#include <cuda_runtime.h>
#include <stdint.h>

#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Load the M code bytes of one slot as 32-bit words (M % 4 == 0).
template <int M>
__device__ __forceinline__ void load_codes(const uint8_t* p, uint32_t (&w)[M / 4]) {
  if constexpr (M % 16 == 0) {
#pragma unroll
    for (int v = 0; v < M / 16; ++v) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p) + v);
      w[4 * v] = x.x; w[4 * v + 1] = x.y; w[4 * v + 2] = x.z; w[4 * v + 3] = x.w;
    }
  } else if constexpr (M % 8 == 0) {
#pragma unroll
    for (int v = 0; v < M / 8; ++v) {
      const uint2 x = __ldg(reinterpret_cast<const uint2*>(p) + v);
      w[2 * v] = x.x; w[2 * v + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < M / 4; ++v) w[v] = __ldg(reinterpret_cast<const uint32_t*>(p) + v);
  }
}

// MC > 0: compile-time M (multiple of 4).  MC == 0: runtime M, byte loads.
template <int MC>
__global__ void __launch_bounds__(kThreads) scan_qm_kernel(
    const int8_t* __restrict__ queries, int dim, int M_rt, int Ks, int L, const int8_t* __restrict__ cb,
    const uint8_t* __restrict__ codes, const int32_t* __restrict__ pterm, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ counts, int nprobe, int k, const int32_t* __restrict__ lists,
    const int32_t* __restrict__ ldist, int32_t* __restrict__ out_ids, int32_t* __restrict__ out_dist,
    int32_t* __restrict__ trace) {
  const int M = MC > 0 ? MC : M_rt;
  const int d = dim / M;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* tops = reinterpret_cast<uint64_t*>(smem);           // [kWarps][k]
  int32_t* A = reinterpret_cast<int32_t*>(tops + kWarps * k);   // [M][Ks]
  int2* probe = reinterpret_cast<int2*>(A + M * Ks);            // [nprobe] (list, d_i)
  int8_t* qs = reinterpret_cast<int8_t*>(probe + nprobe);       // [dim]

  const int64_t qi = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = threadIdx.x; u < dim; u += kThreads) qs[u] = queries[qi * dim + u];
  for (int r = threadIdx.x; r < nprobe; r += kThreads)
    probe[r] = make_int2(lists[qi * nprobe + r], ldist[qi * nprobe + r]);
  for (int e = threadIdx.x; e < kWarps * k; e += kThreads) tops[e] = ~0ull;
  __syncthreads();

  // Step 3 (factorised): A_q[m][c] = -2 <C_{m,c}, q^{(m)}>
  for (int e = threadIdx.x; e < M * Ks; e += kThreads) {
    const int m = e / Ks;
    const int8_t* cw = cb + static_cast<int64_t>(e) * d;
    const int8_t* qm = qs + m * d;
    int acc = 0;
    for (int u = 0; u < d; ++u) acc += static_cast<int>(cw[u]) * static_cast<int>(qm[u]);
    A[e] = -2 * acc;
  }
  __syncthreads();

  // Steps 4-5: stream the probed lists.
  uint64_t* T = tops + warp * k;
  uint64_t thr = ~0ull;
  for (int rho = 0; rho < nprobe; ++rho) {
    const int li = probe[rho].x;
    const int di = probe[rho].y;
    const int cnt = counts[li];
    const int64_t base = static_cast<int64_t>(li) * L;
    int32_t* tr = trace ? trace + (qi * nprobe + rho) * static_cast<int64_t>(L) : nullptr;
    for (int j0 = warp * 32; j0 < L; j0 += kThreads) {
      const int j = j0 + lane;
      int32_t D = kDMax;
      if (j < cnt) {
        int32_t sum = di + __ldg(pterm + base + j);
        if constexpr (MC > 0) {
          uint32_t w[MC / 4];
          load_codes<MC>(codes + (base + j) * MC, w);
#pragma unroll
          for (int m = 0; m < MC; ++m) sum += A[m * Ks + ((w[m >> 2] >> (8 * (m & 3))) & 0xff)];
        } else {
          const uint8_t* cp = codes + (base + j) * M;
          for (int m = 0; m < M; ++m) sum += A[m * Ks + __ldg(cp + m)];
        }
        D = sum;
      }
      if (tr && j < L) tr[j] = D;
      uint64_t key = ~0ull;
      if (j < L && static_cast<uint32_t>(D) <= static_cast<uint32_t>(thr >> 32))
        key = step5_key(D, j < cnt ? __ldg(ids + base + j) : -1);   // lazy id load
      thr = warp_offer(T, k, thr, key);
    }
  }
  __syncthreads();

  // Merge the per-warp lists into warp 0's.
  if (warp == 0) {
    for (int w = 1; w < kWarps; ++w) {
      const uint64_t* Tw = tops + w * k;
      for (int b = 0; b < k; b += 32) {
        const uint64_t key = (b + lane < k) ? Tw[b + lane] : ~0ull;
        thr = warp_offer(tops, k, thr, key);
      }
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += kThreads) {
    const uint64_t key = tops[r];
    out_ids[qi * k + r] = step5_id(key);
    out_dist[qi * k + r] = static_cast<int32_t>(key >> 32);
  }
}

}  // namespace

cudaError_t scan_generic(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                         const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                         int32_t* trace, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  const size_t smem = sizeof(uint64_t) * kWarps * k + sizeof(int32_t) * s->M * s->Ks + sizeof(int2) * nprobe +
                      ((s->dim + 15) & ~15);
#define V3DB_SCAN(MC)                                                                                            \
  {                                                                                                              \
    cudaError_t e = cudaFuncSetAttribute(scan_qm_kernel<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                         static_cast<int>(smem));                                                \
    if (e != cudaSuccess) return e;                                                                              \
    scan_qm_kernel<MC><<<static_cast<unsigned>(nq), kThreads, smem, st>>>(                                       \
        queries, s->dim, s->M, s->Ks, s->L, s->codebooks, s->codes, s->pterm, s->ids, s->counts, nprobe, k,     \
        lists, ldist, out_ids, out_dist, trace);                                                                 \
    break;                                                                                                       \
  }
  switch (s->M) {
    case 4: V3DB_SCAN(4)
    case 8: V3DB_SCAN(8)
    case 16: V3DB_SCAN(16)
    case 24: V3DB_SCAN(24)
    case 32: V3DB_SCAN(32)
    case 64: V3DB_SCAN(64)
    case 96: V3DB_SCAN(96)
    default: V3DB_SCAN(0)
  }
#undef V3DB_SCAN
  note_launch();
  return cudaGetLastError();
}

}  // namespace v3db

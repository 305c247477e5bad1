// scan_list_major.cu -- Steps 3-5 of PAPER.md §4.2, list-major.
//
// A batch of Q queries probes Q*nprobe (query, list) pairs but only nlist distinct lists;
// at C4 every list is probed ~64 times per batch.  The query-major scan re-reads a list's
// codes once per probing query (25.8 GB per C4 batch); this path groups the pairs by list
// and reads each probed list ONCE per batch.
//
// Per slot the exact identity of DESIGN.md "LUT factorisation", with the reconstruction
// xhat_{i,j} = (C_{0,c_0} | ... | C_{M-1,c_{M-1}}) (D = Md):
//   d~_{i,j} = sum_m LUT_{i,m,c_m} = dist(q - mu_i, xhat_ij) = d_i + P_{i,j} - 2 <q, xhat_ij>
// so for one list and the G queries probing it, Step 4 is the int8 contraction
//   [G x D] (gathered queries) . [D x L] (the list's decoded slots)  -> int32 [G x L]
// run on the tensor cores, plus a per-row (d_i) and per-column (P_{i,j}) add and the
// padding mask (f = 0 -> d_max).  Every D_{i,j} goes to the trace.
//
// Step 5 stays exact with per-query thresholds:
//   round 0: the tensor-core scan of ranks [0, r0) (r0 = max(ceil(k/L), ceil(nprobe/8)))
//            writes those D rows;
//   seed:    per query, a monotone histogram of the r0*L values gives tau_q = the upper edge
//            of the bin holding the k-th smallest -- at least k candidates have D <= tau_q --
//            and those valid candidates are appended to the query's buffer;
//   round 1: the scan of ranks [r0, nprobe) appends every valid candidate with D <= tau_q;
//   final:   the exact top-k (D, id) of the buffer, padded with (d_max, -1) if fewer than k
//            valid candidates exist (R11).  A candidate not in the buffer has D > tau_q, so it
//            ranks below k buffered ones.  A query whose buffer overflows (capacity `cap`) is
//            recomputed by the query-major kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "scan_lm_tc.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {
namespace {

// ---------------------------------------------------------------------------- grouping

__global__ void hist_kernel(const int32_t* __restrict__ lists, int64_t nq, int nprobe, int r0, int r1,
                            int* __restrict__ cnt) {
  const int per = r1 - r0;
  const int64_t total = nq * per;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / per;
    const int r = r0 + static_cast<int>(e - q * per);
    atomicAdd(cnt + lists[q * nprobe + r], 1);
  }
}

// One CTA: exclusive scans of the pair counts and of the work-item counts per list.
__global__ void __launch_bounds__(1024) plan_kernel(const int* __restrict__ cnt, int nlist, int tm,
                                                    int* __restrict__ list_off, int* __restrict__ item_off,
                                                    int* __restrict__ cursor) {
  __shared__ int s_p[32], s_i[32];
  const int per = (nlist + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(nlist, b + per);
  int sp = 0, si = 0;
  for (int i = b; i < e; ++i) {
    sp += cnt[i];
    si += (cnt[i] + tm - 1) / tm;
  }
  // block-wide exclusive scan of (sp, si)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ip = sp, ii = si;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ip, o), c = __shfl_up_sync(0xffffffffu, ii, o);
    if (lane >= o) {
      ip += a;
      ii += c;
    }
  }
  if (lane == 31) {
    s_p[warp] = ip;
    s_i[warp] = ii;
  }
  __syncthreads();
  if (warp == 0) {
    int vp = lane < (blockDim.x >> 5) ? s_p[lane] : 0, vi = lane < (blockDim.x >> 5) ? s_i[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, vp, o), c = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) {
        vp += a;
        vi += c;
      }
    }
    s_p[lane] = vp;
    s_i[lane] = vi;
  }
  __syncthreads();
  int op = ip - sp + (warp > 0 ? s_p[warp - 1] : 0);
  int oi = ii - si + (warp > 0 ? s_i[warp - 1] : 0);
  for (int i = b; i < e; ++i) {
    list_off[i] = op;
    cursor[i] = op;
    item_off[i] = oi;
    op += cnt[i];
    oi += (cnt[i] + tm - 1) / tm;
  }
  if (threadIdx.x == blockDim.x - 1) {
    list_off[nlist] = op;
    item_off[nlist] = oi;
  }
}

// Pair records (query, rank, d_i, tau_q) grouped by list (order inside a list is arbitrary;
// every consumer is order-independent).
__global__ void scatter_kernel(const int32_t* __restrict__ lists, const int32_t* __restrict__ ldist,
                               const int32_t* __restrict__ tau_d, int64_t nq, int nprobe, int r0, int r1,
                               int* __restrict__ cursor, int4* __restrict__ pairs) {
  const int per = r1 - r0;
  const int64_t total = nq * per;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / per;
    const int r = r0 + static_cast<int>(e - q * per);
    const int pos = atomicAdd(cursor + lists[q * nprobe + r], 1);
    pairs[pos] = make_int4(static_cast<int>(q), r, ldist[q * nprobe + r], tau_d ? tau_d[q] : 0);
  }
}

// Work-item table: (list, first pair, number of pairs <= tm, valid slots of the list).
__global__ void items_kernel(int nlist, int tm, const int* __restrict__ list_off, const int* __restrict__ item_off,
                             const int32_t* __restrict__ counts, int4* __restrict__ items) {
  const int li = blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= nlist) return;
  const int p0 = list_off[li], n = list_off[li + 1] - p0, w0 = item_off[li];
  for (int c = 0; c * tm < n; ++c) items[w0 + c] = make_int4(li, p0 + c * tm, min(tm, n - c * tm), counts[li]);
}

// ---------------------------------------------------------------------------- seed threshold

// Monotone bins of a non-negative D: 16 exact bins below 16, then 16 bins per octave.
__device__ __forceinline__ int dbin(int D) {
  if (D < 16) return D < 0 ? 0 : D;
  const int e = 31 - __clz(D);
  return 16 + (e - 4) * 16 + ((D >> (e - 4)) & 15);
}
__device__ __forceinline__ int dbin_hi(int b) {  // largest D in bin b
  if (b < 16) return b;
  const int e = (b - 16) / 16 + 4, m = (b - 16) % 16;
  const int64_t hi = (static_cast<int64_t>(17 + m) << (e - 4)) - 1;
  return hi > 0x7fffffff ? 0x7fffffff : static_cast<int>(hi);
}
constexpr int kBins = 448;

// Warp per query: tau_q from the histogram of its r0*L round-0 distances; append the valid
// candidates with D <= tau_q to the buffer.
__global__ void __launch_bounds__(256) seed_kernel(int64_t nq, int k, int r0, int L, int nprobe,
                                                  const int32_t* __restrict__ rows, int rows_nprobe,
                                                  const int32_t* __restrict__ lists, const int32_t* __restrict__ counts,
                                                  uint64_t* __restrict__ cand_buf,
                                                  int* __restrict__ cand_cnt, int cap, int32_t* __restrict__ tau_d) {
  __shared__ int hist[8][kBins];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (q >= nq) return;
  int* h = hist[warp];
  for (int b = lane; b < kBins; b += 32) h[b] = 0;
  __syncwarp();
  for (int rho = 0; rho < r0; ++rho) {
    const int32_t* src = rows + (q * rows_nprobe + rho) * static_cast<int64_t>(L);
    for (int j = lane; j < L; j += 32) atomicAdd(h + dbin(src[j]), 1);
  }
  __syncwarp();
  // first bin whose cumulative count reaches k
  constexpr int per = kBins / 32;
  int loc = 0;
  for (int b = 0; b < per; ++b) loc += h[lane * per + b];
  int inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, inc >= k);
  const int src_lane = __ffs(hit) - 1;  // exists: r0 * L >= k
  int bin = 0;
  if (lane == src_lane) {
    int c = inc - loc;
    for (bin = lane * per; bin < lane * per + per; ++bin) {
      c += h[bin];
      if (c >= k) break;
    }
  }
  bin = __shfl_sync(0xffffffffu, bin, src_lane);
  const int tq = dbin_hi(bin);
  // append the valid candidates with D <= tau_q (warp-aggregated positions)
  int n = 0;
  for (int rho = 0; rho < r0; ++rho) {
    const int li = lists[q * nprobe + rho];
    const int cnt = counts[li];
    const int32_t* src = rows + (q * rows_nprobe + rho) * static_cast<int64_t>(L);
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      const int D = j < cnt ? src[j] : 0x7fffffff;
      const bool take = j < cnt && D <= tq;
      const unsigned m = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int pos = n + __popc(m & ((1u << lane) - 1));
        if (pos < cap)
          cand_buf[q * cap + pos] = (static_cast<uint64_t>(static_cast<uint32_t>(D)) << 32) |
                                    static_cast<uint32_t>(li * L + j);
      }
      n += __popc(m);
    }
  }
  if (lane == 0) {
    cand_cnt[q] = n;
    tau_d[q] = tq;
  }
}

// ---------------------------------------------------------------------------- final top-k

// Candidates are (D << 32 | list * L + slot); the Step-5 key (D, item) is formed here.
template <int KR>
__global__ void __launch_bounds__(256) final_select_kernel(int64_t nq, int k, int cap, const int32_t* __restrict__ ids,
                                                          const uint64_t* __restrict__ cand_buf,
                                                          const int* __restrict__ cand_cnt,
                                                          int32_t* __restrict__ out_ids,
                                                          int32_t* __restrict__ out_dist, int* __restrict__ flags) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (q >= nq) return;
  const int n = cand_cnt[q];
  if (n > cap) {  // overflow: recomputed by the query-major fallback
    if (lane == 0) flags[q] = 1;
    return;
  }
  if (lane == 0) flags[q] = 0;
  WarpTopK<KR> top;
  top.init(k);
  const uint64_t* buf = cand_buf + q * cap;
  for (int b = 0; b < n; b += 32) {
    uint64_t key = ~0ull;
    if (b + lane < n) {
      const uint64_t c = buf[b + lane];
      key = step5_key(static_cast<int32_t>(c >> 32), __ldg(ids + static_cast<uint32_t>(c)));
    }
    top.offer(key);
  }
  const uint64_t pad = step5_key(kDMax, -1);  // fewer than k valid candidates (R11)
  top.store([&](int j, uint64_t key) {
    if (key == ~0ull) key = pad;
    out_ids[q * k + j] = step5_id(key);
    out_dist[q * k + j] = static_cast<int32_t>(key >> 32);
  });
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

cudaError_t scan_list_major(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                            const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                            int32_t* trace, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  const int L = s->L, nlist = s->nlist;
  LmTcArgs a{};
  size_t lm_smem = 0;
  if (!lm_tc_config(s, &a, &lm_smem))
    return scan_query_major(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace, st);
  // seed ranks: enough slots for k candidates, and at least 1/8 of the probed lists -- the
  // probed lists of a query are often about equally close, so one list gives a loose tau
  const int r0 = std::min(nprobe, std::max((k + L - 1) / L, (nprobe + 7) / 8));
  const int cap = std::min(16384, std::max(1024, 40 * k));
  const int64_t np0 = nq * r0, np1 = nq * (nprobe - r0);

  // scratch (stream-ordered pool)
  const size_t b_buf = align256(sizeof(uint64_t) * nq * cap), b_q = align256(sizeof(int) * nq),
               b_lc = align256(sizeof(int) * nlist), b_off = align256(sizeof(int) * (nlist + 1)),
               b_p0 = align256(sizeof(int4) * std::max<int64_t>(1, np0)),
               b_p1 = align256(sizeof(int4) * std::max<int64_t>(1, np1)),
               b_it0 = align256(sizeof(int4) * std::max<int64_t>(1, np0 + nlist)),
               b_it1 = align256(sizeof(int4) * std::max<int64_t>(1, np1 + nlist)),
               b_rows = trace ? 0 : align256(sizeof(int32_t) * nq * r0 * L);
  uint8_t* base = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base),
                                  b_buf + 3 * b_q + 2 * (2 * b_lc + 2 * b_off) + b_p0 + b_p1 + b_it0 + b_it1 + b_rows,
                                  st);
  if (e != cudaSuccess) return e;
  uint8_t* p = base;
  auto take = [&](size_t b) { uint8_t* r = p; p += b; return r; };
  uint64_t* cand_buf = reinterpret_cast<uint64_t*>(take(b_buf));
  int* cand_cnt = reinterpret_cast<int*>(take(b_q));
  int32_t* tau_d = reinterpret_cast<int32_t*>(take(b_q));
  int* flags = reinterpret_cast<int*>(take(b_q));
  int4* pairs[2] = {reinterpret_cast<int4*>(take(b_p0)), reinterpret_cast<int4*>(take(b_p1))};
  int4* items[2] = {reinterpret_cast<int4*>(take(b_it0)), reinterpret_cast<int4*>(take(b_it1))};
  int32_t* rows0 = trace ? trace : reinterpret_cast<int32_t*>(take(b_rows));
  const int rows0_np = trace ? nprobe : r0;

  a.queries = queries;
  a.q_vec = (s->dim % 16 == 0) && (reinterpret_cast<uintptr_t>(queries) % 16 == 0);
  a.codes_vec = (static_cast<int64_t>(L) * s->M % 16 == 0) && (reinterpret_cast<uintptr_t>(s->codes) % 16 == 0);
  a.p_vec = (L % 4 == 0) && (reinterpret_cast<uintptr_t>(s->pterm) % 16 == 0);
  a.cb = s->codebooks;
  a.codes = s->codes;
  a.pterm = s->pterm;
  a.counts = s->counts;
  a.cand_buf = cand_buf;
  a.cand_cnt = cand_cnt;
  a.cap = cap;

  for (int round = 0; round < 2 && e == cudaSuccess; ++round) {
    const int rlo = round == 0 ? 0 : r0, rhi = round == 0 ? r0 : nprobe;
    const int64_t npairs = nq * (rhi - rlo);
    if (npairs > 0) {
      int* lcnt = reinterpret_cast<int*>(take(b_lc));
      int* cursor = reinterpret_cast<int*>(take(b_lc));
      int* list_off = reinterpret_cast<int*>(take(b_off));
      int* item_off = reinterpret_cast<int*>(take(b_off));
      const int gb = static_cast<int>(std::min<int64_t>((npairs + 255) / 256, 148 * 16));
      e = cudaMemsetAsync(lcnt, 0, sizeof(int) * nlist, st);
      if (e == cudaSuccess) {
        hist_kernel<<<gb, 256, 0, st>>>(lists, nq, nprobe, rlo, rhi, lcnt);
        plan_kernel<<<1, 1024, 0, st>>>(lcnt, nlist, 128, list_off, item_off, cursor);
        scatter_kernel<<<gb, 256, 0, st>>>(lists, ldist, round == 1 ? tau_d : nullptr, nq, nprobe, rlo, rhi, cursor,
                                           pairs[round]);
        items_kernel<<<(nlist + 255) / 256, 256, 0, st>>>(nlist, 128, list_off, item_off, s->counts, items[round]);
        note_launch(4);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = debug_sync(st, "grouping");
      }
      if (e == cudaSuccess) {
        a.pairs = pairs[round];
        a.items = items[round];
        a.n_items = item_off + nlist;
        a.emit = round;
        a.dst = round == 0 ? rows0 : trace;
        a.dst_nprobe = round == 0 ? rows0_np : nprobe;
        a.vec_store = (L % 4 == 0) && (a.dst == nullptr || (reinterpret_cast<uintptr_t>(a.dst) % 16) == 0);
        e = launch_lm_tc(a, lm_smem, st);
        if (e == cudaSuccess) e = debug_sync(st, round == 0 ? "lm_tc round 0" : "lm_tc round 1");
      }
    }
    if (round == 0 && e == cudaSuccess) {
      seed_kernel<<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(nq, k, r0, L, nprobe, rows0, rows0_np, lists,
                                                                       s->counts, cand_buf, cand_cnt, cap, tau_d);
      note_launch();
      e = cudaGetLastError();
      if (e == cudaSuccess) e = debug_sync(st, "seed");
    }
  }
  if (e == cudaSuccess) {
    dispatch_kr(k, [&]<int KR>() {
      final_select_kernel<KR><<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(nq, k, cap, s->ids, cand_buf, cand_cnt,
                                                                                  out_ids, out_dist, flags);
    });
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = debug_sync(st, "final_select");
  }
  if (e == cudaSuccess) {
    QmExtra f;
    f.mode = kModeFallback;
    f.flags = flags;
    e = scan_query_major(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, nullptr, st, f);
  }
  cudaFreeAsync(base, st);
  return e;
}

}  // namespace v3db

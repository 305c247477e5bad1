// scan_rot.cu -- Steps 3-5 of PAPER.md §4.2 with a conflict-free rotated LUT (one CTA per query).
//
// Step 3 builds, per probed list i, LUT_{i,m,c} = dist(C_{m,c}, (q-mu_i)^{(m)}).
// Summed over the codes of a slot this is the exact integer identity (DESIGN.md "LUT
// factorisation")
//     d~_{i,j} = d_i + P_{i,j} + sum_m A_q[m][c_m],    A_q[m][c] = -2 <C_{m,c}, q^{(m)}>,
// so the CTA builds ONE table A_q per query in shared memory.  Step 4 streams
// the probed lists' codes; padding slots (f = 0) get D = d_max and whole chunks of padding are
// never read.  Step 5 keeps an exact top-k on (D, item) keys.
//
// Rotated LUT.  The M subspaces are split into groups of
// G in {32, 16, 8, 4} consecutive subspaces (greedy: M = 24 -> 16 + 8).  Lane l of a warp handles
// slot j = 32c + l of a chunk.  At step s of group g it reads subspace off_g + (l + s) mod G from
// table COLUMN l + s, so the 32 lanes of every LDS hit 32 distinct banks whatever the codes are.
// The slot's code bytes are stored pre-rotated (codes_rot, built once) so byte off_g + s of the
// register words is the right code.  Two table geometries:
//   kLutP64 (one group, G = M <= 32): rows of 64 int32 columns, column col = subspace col mod G;
//            address = code*256 + 4l + 4s = PRMT(code byte, 4l) + immediate.        1 ALU op
//   kLutW32 (any M % 4 == 0): per group, 257 rows of 32 columns; a lane whose column l+s passes
//            32 wraps into the next row, which the stored byte pre-compensates ((code - 1) mod
//            256; row 256 duplicates row 0):  address = ((byte << 7) | 4l) + immediate.  2 ALU ops
//
// Streaming.  A producer warp (one lane) walks the probed lists'
// VALID 32-slot chunks in probe order and packs them into CTA-wide stages of SEG chunks; each
// stage is filled by one cp.async.bulk (TMA bulk copy) of codes per list piece (~1-2 pieces per
// stage) plus per-chunk descriptors, completion on the stage's `full` mbarrier (expect-tx, copies,
// descriptors, then the producer's arrival); the consumer warps split the stage's chunks, read each
// chunk's P terms from global memory (__ldg, L2) and release the stage on its `empty` mbarrier.  codes_rot stores each chunk
// unit-transposed ([unit][lane][U bytes]) so the lanes' stage reads are conflict-free LDS.128/64/32.
// Chunks holding only padding are never read: their trace entries (d_max) are written up front.
//
// Top-k.  Candidates with D <= tau are appended to a shared buffer
// (warp-aggregated).  When an append lifts the count above a high-water mark, a compaction is
// requested and every consumer warp joins it at its next stage end (no periodic barrier): a
// 4-pass radix select finds the k-th smallest D, tau = that D and only entries with D <= tau stay
// (>= k of them, so every dropped key has k keys at or below it).  Item ids are resolved only for
// tie overflow and for the final (D, id) sort.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "tc_common.cuh"
#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {

int plan_lut(int M, int Ks, int d, int* G) {
  *G = 0;
  if (M < 4 || M % 4 != 0 || M > 128 || d % 4 != 0 || Ks < 1 || Ks > 256) return 0;
  const bool want_w32 = opt(V3DB_OPT_LUT_W32) != 0;  // test/bench option: W32 where P64 applies
  // P64: one rotation group of all M <= 32 subspaces; lane l reads column l + s < 64 at step s,
  // which holds subspace (l + s) mod M (columns m, m + M, ... replicate subspace m)
  const bool p64_ok = M <= 32 && (M == 4 || M == 8 || M == 12 || M == 16 || M == 20 || M == 24 || M == 28 || M == 32);
  const bool w32_ok = M == 8 || M == 12 || M == 16 || M == 24 || M == 32 || M == 48 || M == 64 || M == 96 || M == 128;
  // default: P64 (1 ALU op per lookup) wherever it applies; W32 (2 ALU ops, half the table) for
  // the other shapes.  Measured with 256-codeword tables (P64: 64 KB table, 2 stages of 16 chunks;
  // W32: 33 KB, 4 stages): C4 scan 6.43 vs 6.58 ms, C1 0.455 vs 0.474 ms (DESIGN.md "Rotated LUT
  // layout")
  if (p64_ok && !want_w32) {
    *G = M;
    return kLutP64;
  }
  if (w32_ok) {
    *G = rot_gsize(M, 0);
    return kLutW32;
  }
  return 0;
}


namespace {

constexpr uint32_t kFull = 0xffffffffu;
// Low 16 bits of the shared-window address of dynamic shared memory: the first 1 KB of a CTA's
// window is reserved on sm_90+ (cudaDevAttrReservedSharedMemoryPerBlock), so it starts at 0x400;
// checked at kernel entry.
constexpr uint32_t kSmemLo = 0x400;

__device__ __forceinline__ int32_t lds32(uint32_t addr) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
constexpr uint32_t kTauInit = 0x7ffffffeu;  // accept every valid D (< d_max)

template <int M, int MODE, int VAR = 0>
struct Geo {
  static constexpr int NG = rot_ngroups(M);
  static constexpr int NW = M / 4;                                   // 32-bit code words per slot
  static constexpr int U = M % 16 == 0 ? 16 : M % 8 == 0 ? 8 : 4;    // bytes per lane per unit
  static constexpr int NT = (MODE == kLutW32 && NG * kW32GroupBytes > 96 * 1024) ? 512 : 256;  // consumers
  static constexpr int NTOT = NT + 32;                              // + the producer warp
  static constexpr int MINB = NT == 512 ? 1 : 2;
};

struct RotArgs {
  const int8_t* queries;
  int dim, d, Ks, L, Lp, nprobe, k, cap, NS, SEG;
  int first_mult;         // first compaction at first_mult * k buffered candidates (capped by hw)
  int direct_max;         // final selection by direct ranking when at most this many are buffered
  uint32_t off_stage, off_desc, off_vc, off_buf, off_hist, off_probe, off_q, off_int, off_bar, stage_bytes;
  const int8_t* cbT;
  const uint8_t* codes;   // codes_rot [nlist][Lp/32][unit][lane][U]
  const int32_t* pterm;   // pterm_rot [nlist][Lp]
  const int32_t* ids;     // [nlist][L]
  const int32_t* counts;
  const int32_t* lists;
  const int32_t* ldist;
  int32_t* out_ids;
  int32_t* out_dist;
  int32_t* trace;
  const int32_t* order;   // [nq] query processed by CTA b (L2-aware schedule), or null = identity
};

// Named barrier 1 among the NT consumer threads (the producer warp never joins).
template <int NT>
__device__ __forceinline__ void bar_c() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// Exact sort of buf[0, P) ascending (bitonic network; P a power of two).  All threads call.
template <int NT>
__device__ __forceinline__ void bitonic_sort(uint64_t* buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (P >> 1); t += NT) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const uint64_t a = buf[lo], b = buf[hi];
        const bool asc = (lo & size) == 0;
        if ((a > b) == asc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      bar_c<NT>();
    }
  }
}

// Buffer keys: (D << 32) | low.  low = flat slot rho*L + j (< 2^31, bit 31 clear) until the item is
// resolved, then id ^ 0x80000000 (bit 31 set for every id >= 0; padding is never buffered) -- the
// Step-5 key of R10.  Items are resolved only where the (D, id) order is needed: ties that would
// overflow the buffer, and the final sort.
__device__ __forceinline__ uint64_t resolve_key(uint64_t key, const int4* probe, const RotArgs& a) {
  const uint32_t lo = static_cast<uint32_t>(key);
  if (lo & 0x80000000u) return key;
  const int rho = static_cast<int>(lo / static_cast<uint32_t>(a.L));
  const int j = static_cast<int>(lo - static_cast<uint32_t>(rho) * a.L);
  const int32_t id = __ldg(a.ids + static_cast<int64_t>(probe[rho].x) * a.L + j);
  return (key & 0xffffffff00000000ull) | (static_cast<uint32_t>(id) ^ 0x80000000u);
}

// Compaction of buf[0, n) (all consumer threads; n uniform): if n > k only the entries with
// D <= (the k-th smallest D, exact 4-pass 8-bit radix select) stay -- at least k of them, so every
// dropped key has k keys at or below it.  If ties at that D leave more than `limit`, or `final`,
// the items are resolved and sorted by (D, id) and the first min(n, k) kept (sorted).  Returns the
// new count; *tau = the D threshold for later appends.
template <int NT, int CAPM>
__device__ int compact(uint64_t* buf, int* hist, int* s_int, const int4* probe, const RotArgs& a, int n, int limit,
                       bool final, uint32_t* tau) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t kv[CAPM];
#pragma unroll
  for (int r = 0; r < CAPM; ++r) kv[r] = tid + r * NT < n ? buf[tid + r * NT] : ~0ull;
  int kept = n;
  if (n > a.k) {
    // Radix select (8-bit digits) of the k-th smallest D.  Every buffered D is <= *tau once tau is
    // set, so the leading digits above tau's top bit are 0 for all entries: those passes are
    // skipped.  Two histograms alternate (warp 0 scans one while the others clear the next), so a
    // pass costs two barriers.
    uint32_t prefix = 0;
    int kk = a.k;
    const uint32_t bound = *tau;  // kTauInit (all ones) before the first compaction
    const int top = 32 - __clz(bound | 1u);
    const int pass0 = 3 - (top - 1) / 8;
    for (int b = tid; b < 256; b += NT) hist[b] = 0;
    bar_c<NT>();
#pragma unroll 1
    for (int pass = pass0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass, par = (pass - pass0) & 1;
      int* H = hist + 256 * par;
#pragma unroll
      for (int r = 0; r < CAPM; ++r) {
        const uint32_t D = static_cast<uint32_t>(kv[r] >> 32);
        if (tid + r * NT < n && (pass == 0 || (D >> (shift + 8)) == prefix)) atomicAdd(&H[(D >> shift) & 255], 1);
      }
      bar_c<NT>();
      if (warp != 0) {
        int* Hn = hist + 256 * (par ^ 1);  // the next pass's histogram (last read one pass ago)
        for (int b = tid - 32; b < 256; b += NT - 32) Hn[b] = 0;
      } else {
        int h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          h[b] = H[lane * 8 + b];
          sum += h[b];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += v;
        }
        int cum = incl - sum;  // exclusive prefix of this lane's 8 bins
        if (cum < kk && kk <= incl) {
          int bin = lane * 8;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (cum + h[b] >= kk) break;
            cum += h[b];
            ++bin;
          }
          s_int[8 + 2 * par] = bin;
          s_int[9 + 2 * par] = kk - cum;
        }
      }
      bar_c<NT>();
      prefix = (prefix << 8) | static_cast<uint32_t>(s_int[8 + 2 * par]);
      kk = s_int[9 + 2 * par];
      // no barrier: the next pass writes the other histogram and the other s_int pair
    }
    *tau = prefix;  // exact k-th smallest D
    if (tid == 0) s_int[12] = 0;
    bar_c<NT>();
#pragma unroll
    for (int r = 0; r < CAPM; ++r) {
      const bool keep = tid + r * NT < n && static_cast<uint32_t>(kv[r] >> 32) <= prefix;
      const uint32_t bal = __ballot_sync(kFull, keep);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&s_int[12], __popc(bal));
      base = __shfl_sync(kFull, base, 0);
      if (keep) buf[base + __popc(bal & ((1u << lane) - 1u))] = kv[r];
    }
    bar_c<NT>();
    kept = s_int[12];
  }
  if (final) {  // resolve: the caller orders the survivors by (D, id) (rank_scatter)
    for (int e = tid; e < kept; e += NT) buf[e] = resolve_key(buf[e], probe, a);
  } else if (kept > limit) {  // ties: exact (D, id) order, keep the first k
    for (int e = tid; e < kept; e += NT) buf[e] = resolve_key(buf[e], probe, a);
    int P = 1;
    while (P < kept) P <<= 1;
    for (int e = kept + tid; e < P; e += NT) buf[e] = ~0ull;
    bar_c<NT>();
    bitonic_sort<NT>(buf, P);
    kept = a.k;
  }
  bar_c<NT>();
  return kept;
}

// (g, off_g, size_g) of subspace m: compile-time constants selected by m (W32 groups).
template <int M, int X = 1>
__device__ __forceinline__ void rot_group_of(int m, int& g, int& goff, int& Gg) {
  if constexpr (X < rot_ngroups(M)) {
    constexpr int o = rot_goff(M, X), z = rot_gsize(M, X);
    if (m >= o) {
      g = X;
      goff = o;
      Gg = z;
    }
    rot_group_of<M, X + 1>(m, g, goff, Gg);
  }
}

template <int M, int MODE, int G_IDX>
__device__ __forceinline__ void lut_sum(const uint32_t (&w)[M / 4], uint32_t lane4, int32_t& acc) {
  constexpr int off = rot_goff(M, G_IDX), Gg = MODE == kLutP64 ? M : rot_gsize(M, G_IDX);
  constexpr int TGB = MODE == kLutW32 ? kW32GroupBytes : 0;
#pragma unroll
  for (int s2 = 0; s2 < Gg; ++s2) {
    const int pos = off + s2;
    const uint32_t wd = w[pos >> 2];
    uint32_t ad;
    if constexpr (MODE == kLutP64) {
      ad = __byte_perm(wd, lane4, 0x7604u | ((pos & 3) << 4));  // code << 8 | lane4
    } else {
      const int b = pos & 3;
      const uint32_t sh = (b == 0) ? (wd << 7) : (wd >> (8 * b - 7));
      ad = (sh & 0x7f80u) | lane4;
    }
    acc += lds32(ad + (kSmemLo + G_IDX * TGB + 4 * s2));
  }
  if constexpr (MODE == kLutW32 && G_IDX + 1 < rot_ngroups(M)) lut_sum<M, MODE, G_IDX + 1>(w, lane4, acc);
}

template <int M, int MODE, int CAPM, int VAR>
__global__ void __launch_bounds__(Geo<M, MODE, VAR>::NTOT, Geo<M, MODE, VAR>::MINB) scan_rot_kernel(const RotArgs a) {
  using C = Geo<M, MODE, VAR>;
  constexpr int NT = C::NT, W = NT / 32, NW = C::NW, U = C::U;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem + a.off_stage;                        // [NS][SEG*32*M codes | SEG*128 P]
  int* vcoff = reinterpret_cast<int*>(smem + a.off_vc);        // [nprobe+1] prefix sums of valid chunks
  int4* dsc = reinterpret_cast<int4*>(smem + a.off_desc);      // [NS][SEG] chunk descriptors
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem + a.off_buf);
  int* hist = reinterpret_cast<int*>(smem + a.off_hist);
  int4* probe = reinterpret_cast<int4*>(smem + a.off_probe);  // (list, d_i, count, 0)
  int8_t* qs = reinterpret_cast<int8_t*>(smem + a.off_q);
  int* s_int = reinterpret_cast<int*>(smem + a.off_int);     // [0] count [1] request [2] done, [8..12] scratch
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* empty = full + a.NS;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t qi = a.order ? a.order[blockIdx.x] : blockIdx.x;
  const int L = a.L, nprobe = a.nprobe, NS = a.NS, SEG = a.SEG;

  for (int u = tid; u < a.dim; u += C::NTOT) qs[u] = a.queries[qi * a.dim + u];
  for (int r = tid; r < nprobe; r += C::NTOT) {
    const int li = a.lists[qi * nprobe + r];
    probe[r] = make_int4(li, a.ldist[qi * nprobe + r], __ldg(a.counts + li), 0);
  }
  if (tid < 16) s_int[tid] = 0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, W);
    }
  }
  tc::mbar_fence_init();
  __syncthreads();
  // valid-chunk prefix sums: the g-th valid chunk of the query (probe order) is chunk
  // g - vcoff[rho] of probe rho, vcoff[rho] <= g < vcoff[rho + 1]
  if (warp == 0) {
    int carry = 0;
    for (int r0 = 0; r0 < nprobe; r0 += 32) {
      const int r = r0 + lane;
      const int cv = r < nprobe ? (probe[r].z + 31) >> 5 : 0;
      int incl = cv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      if (r < nprobe) vcoff[r] = carry + incl - cv;
      carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) vcoff[nprobe] = carry;
  }
  __syncthreads();
  const int TV = vcoff[nprobe];               // valid chunks of this query
  const int NSTG = (TV + SEG - 1) / SEG;      // stages: [t*SEG, min(TV, (t+1)*SEG))

  if (warp == W) {
    // ------------------------------------------------ producer: one lane issues every stage
    if (lane == 0) {
      int rho = 0, s = 0;
      uint32_t eph = 0;  // parity of the empty-barrier phase to wait for (per ring pass)
      for (int t = 0; t < NSTG; ++t) {
        if (t >= NS) tc::mbar_wait_sleep(empty + s, eph);  // consumers released the previous fill
        uint8_t* st = stages + static_cast<uint32_t>(s) * a.stage_bytes;
        const int g0 = t * SEG, g1 = min(TV, g0 + SEG);
        // expect the stage's bytes (no arrival yet), issue the copies and write the chunk
        // descriptors, THEN arrive: the arrival's release orders the descriptor stores before any
        // consumer's acquire of the completed phase (the copies' complete_tx alone would not)
        tc::mbar_expect_tx_only(full + s, static_cast<uint32_t>(g1 - g0) * 32u * M);
        // one codes copy per piece (a run of valid chunks of one list)
        for (int g = g0; g < g1;) {
          while (vcoff[rho + 1] <= g) ++rho;
          const int jc = g - vcoff[rho];
          const int m = min(g1 - g, vcoff[rho + 1] - g);
          const int4 pr = probe[rho];
          const int64_t slot0 = static_cast<int64_t>(pr.x) * a.Lp + jc * 32;
          const uint32_t i = static_cast<uint32_t>(g - g0);
          // per-chunk descriptors: (d_i, rho*L + 32*jc (trace / flat offset), valid slots | slots << 8,
          // P-term offset list*Lp + 32*jc)
          V3DB_DCHECK(i + m <= static_cast<uint32_t>(SEG) && (i + m) * 32u * M <= a.stage_bytes);
          for (int x = 0; x < m; ++x)
            dsc[s * SEG + i + x] = make_int4(pr.y, rho * L + (jc + x) * 32,
                                             min(32, pr.z - (jc + x) * 32) | (min(32, L - (jc + x) * 32) << 8),
                                             static_cast<int>(slot0) + x * 32);
          bulk_g2s(st + i * 32u * M, a.codes + slot0 * M, static_cast<uint32_t>(m) * 32u * M, full + s);
          g += m;
        }
        tc::mbar_arrive(full + s);
        if (++s == NS) {
          s = 0;
          if (t + 1 > NS) eph ^= 1u;
        }
      }
    }
    return;
  }

  // ------------------------------------------------ consumers
  // trace of chunks that hold only padding: D = d_max (never read from HBM)
  if (a.trace) {
    for (int r = warp; r < nprobe; r += W) {
      const int cv = (probe[r].z + 31) >> 5;
      int32_t* tr = a.trace + (qi * nprobe + r) * static_cast<int64_t>(L);
      for (int j = cv * 32 + lane; j < L; j += 32) __stcs(tr + j, kDMax);
    }
  }

  // Step 3 (factorised): A_q[m][c] = -2 <C_{m,c}, q^{(m)}>, written into the rotated tables.
  // Eight entries per thread per step with their codebook loads issued together (latency-bound
  // otherwise: one L2 round trip per entry).
  {
    int32_t* T = reinterpret_cast<int32_t*>(smem);
    const int dw = a.d >> 2, MK = M * a.Ks;
    auto put = [&](int e, int32_t A) {
      const int m = e % M, cc = e / M;
      if constexpr (MODE == kLutP64) {
#pragma unroll
        for (int col = m; col < 64; col += M) T[cc * 64 + col] = A;
      } else if constexpr (M % 32 == 0) {  // groups of 32: one column per subspace
        int32_t* Tg = T + (m >> 5) * (kW32GroupBytes / 4);
        Tg[cc * 32 + (m & 31)] = A;
        if (cc == 0) Tg[256 * 32 + (m & 31)] = A;  // row 256 duplicates row 0 (wrap of code 0)
      } else {
        // the group of subspace m by compile-time selects (rot_goff / rot_gsize of a runtime group
        // index are evaluated as loops at run time: ~25 % of C3's instructions)
        constexpr int G0 = rot_gsize(M, 0);
        int g = 0, goff = 0, Gg = G0;
        rot_group_of<M>(m, g, goff, Gg);
        const int r = m - goff;
        int32_t* Tg = T + g * (kW32GroupBytes / 4);
        for (int col = r; col < 32; col += Gg) {
          Tg[cc * 32 + col] = A;
          if (cc == 0) Tg[256 * 32 + col] = A;  // row 256 duplicates row 0 (wrap of code 0)
        }
      }
    };
    const int* cbw = reinterpret_cast<const int*>(a.cbT);   // [Ks][M][dw] words
    const int* qw = reinterpret_cast<const int*>(qs);       // [M][dw] words
    constexpr int UB = 8;
    for (int e0 = tid; e0 < MK; e0 += UB * NT) {
      int acc[UB];
#pragma unroll
      for (int x = 0; x < UB; ++x) acc[x] = 0;
      if (dw == 1) {
        int cwv[UB];
#pragma unroll
        for (int x = 0; x < UB; ++x) cwv[x] = e0 + x * NT < MK ? __ldg(cbw + e0 + x * NT) : 0;
#pragma unroll
        for (int x = 0; x < UB; ++x) acc[x] = __dp4a(cwv[x], qw[(e0 + x * NT) % M], 0);
      } else if (dw == 2) {
        int2 cwv[UB];
#pragma unroll
        for (int x = 0; x < UB; ++x)
          cwv[x] = e0 + x * NT < MK ? __ldg(reinterpret_cast<const int2*>(cbw) + e0 + x * NT) : make_int2(0, 0);
#pragma unroll
        for (int x = 0; x < UB; ++x) {
          const int m = (e0 + x * NT) % M;
          acc[x] = __dp4a(cwv[x].y, qw[2 * m + 1], __dp4a(cwv[x].x, qw[2 * m], 0));
        }
      } else {
#pragma unroll
        for (int x = 0; x < UB; ++x) {
          const int e = e0 + x * NT;
          if (e < MK) {
            const int m = e % M;
            for (int u = 0; u < dw; ++u) acc[x] = __dp4a(__ldg(cbw + static_cast<int64_t>(e) * dw + u), qw[m * dw + u], acc[x]);
          }
        }
      }
#pragma unroll
      for (int x = 0; x < UB; ++x)
        if (e0 + x * NT < MK) put(e0 + x * NT, -2 * acc[x]);
    }
  }
  bar_c<NT>();

  // LUT addressing: the address register is built by one PRMT (P64) or SHF+LOP3 (W32) with the
  // lane's column and the high half of the shared-window address OR-ed in; the low half of the
  // dynamic shared-memory base (kSmemLo) and the step offset go into the LDS immediate.
  const uint32_t sbase = tc::smem_u32(smem);
  if ((sbase & 0xffffu) != kSmemLo) __trap();  // layout assumption
  // lane4 = 4 * lane | high half of the window address, kept in ONE register: read back from shared
  // memory so the compiler cannot split the OR into two instructions per lookup
  if (tid < 32) s_int[32 + tid] = static_cast<int>(4u * tid | (sbase & 0xffff0000u));
  bar_c<NT>();
  const uint32_t lane4 = static_cast<uint32_t>(*reinterpret_cast<volatile int*>(&s_int[32 + lane]));
  int32_t* trq = a.trace ? a.trace + qi * nprobe * static_cast<int64_t>(L) + lane : nullptr;  // this query's trace
  // Candidate buffer: s_int[0] = entries (monotonic between compactions), s_int[1] = compaction
  // requested, s_int[2] = consumer warps done.  A warp whose append lifts the count above `hw`
  // (or above k before tau is set) requests a compaction; every consumer warp joins at its next
  // stage end, so after the request each warp appends at most its share of one stage
  // (ceil(SEG/W) chunks): W * ceil(SEG/W) * 32 entries of headroom above hw.
  const int hw = a.cap - W * ((SEG + W - 1) / W) * 32;
  const int first = min(hw, a.first_mult * a.k);  // the first compaction (sets tau) once this many are buffered
  uint32_t tau = kTauInit;
  volatile int* vs = s_int;
  auto collective_compact = [&]() {  // all consumer threads
    bar_c<NT>();                     // every warp stopped appending
    uint32_t t2 = tau;
    const int kept = compact<NT, CAPM>(buf, hist, s_int, probe, a, s_int[0], hw, false, &t2);
    tau = t2;
    if (tid == 0) {
      s_int[0] = kept;
      s_int[1] = 0;
    }
    bar_c<NT>();
  };

  uint32_t fph = 0;
  // one chunk's code words (rotated, chunk-transposed) from the stage
  auto load_w = [&](const uint8_t* cp, uint32_t(&w)[NW]) {
#pragma unroll
    for (int u = 0; u < M / U; ++u) {
      const uint8_t* p = cp + u * 32 * U + lane * U;
      if constexpr (U == 16) {
        const uint4 x = *reinterpret_cast<const uint4*>(p);
        w[4 * u] = x.x; w[4 * u + 1] = x.y; w[4 * u + 2] = x.z; w[4 * u + 3] = x.w;
      } else if constexpr (U == 8) {
        const uint2 x = *reinterpret_cast<const uint2*>(p);
        w[2 * u] = x.x; w[2 * u + 1] = x.y;
      } else {
        w[u] = *reinterpret_cast<const uint32_t*>(p);
      }
    }
  };
  // masked D to the trace, candidate append (Step 5 buffer)
  auto emit = [&](const int4 dd, int32_t acc) {
    const bool valid = lane < (dd.z & 0xff);  // lanes past the valid slots read stale stage bytes
    const int32_t D = valid ? acc : kDMax;
    const int off = dd.y + lane;               // rho*L + j
    if (trq && lane < (dd.z >> 8)) __stcs(trq + dd.y, D);
    const bool pass = valid && static_cast<uint32_t>(D) <= tau;
    const uint32_t bal = __ballot_sync(kFull, pass);
    if (bal) {
      int base = 0;
      if (lane == 0) {
        const int cnt = __popc(bal);
        base = atomicAdd(&s_int[0], cnt);
        V3DB_DCHECK(base + cnt <= a.cap);  // headroom argument above (hw)
        if (base + cnt > (tau == kTauInit ? first : hw)) vs[1] = 1;
      }
      base = __shfl_sync(kFull, base, 0);
      if (pass)
        buf[base + __popc(bal & ((1u << lane) - 1u))] =
            (static_cast<uint64_t>(static_cast<uint32_t>(D)) << 32) | static_cast<uint32_t>(off);
    }
  };
  for (int t = 0, s = 0; t < NSTG; ++t) {
    tc::mbar_wait_sleep(full + s, fph);
    const uint8_t* st = stages + static_cast<uint32_t>(s) * a.stage_bytes;
    const int4* ds = dsc + s * SEG;
    const int n = min(TV, t * SEG + SEG) - t * SEG;
    // two chunks (i, i + W) per pass: their loads and 2M lookups interleave
    for (int i = warp; i < n; i += 2 * W) {
      const bool two = i + W < n;  // warp-uniform
      const int4 d0 = ds[i];
      const int4 d1 = ds[two ? i + W : i];
      // P terms straight from global memory (L2), issued first: used after the lookups
      const int32_t p0 = __ldg(a.pterm + d0.w + lane);
      const int32_t p1 = two ? __ldg(a.pterm + d1.w + lane) : 0;
      uint32_t w0[NW], w1[NW];
      load_w(st + static_cast<uint32_t>(i) * 32u * M, w0);
      int32_t acc0 = d0.x;
      if (two) {
        load_w(st + static_cast<uint32_t>(i + W) * 32u * M, w1);
        int32_t acc1 = d1.x;
        lut_sum<M, MODE, 0>(w0, lane4, acc0);
        lut_sum<M, MODE, 0>(w1, lane4, acc1);
        emit(d0, acc0 + p0);
        emit(d1, acc1 + p1);
      } else {
        lut_sum<M, MODE, 0>(w0, lane4, acc0);
        emit(d0, acc0 + p0);
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(empty + s);  // this warp is done with the stage
    if (++s == NS) {
      s = 0;
      fph ^= 1u;
    }
    if (vs[1]) collective_compact();  // warp-uniform (one broadcast read)
  }
  // wait for the other consumer warps, joining any compaction they request meanwhile
  __syncwarp();
  if (lane == 0) atomicAdd(&s_int[2], 1);
  for (;;) {
    __syncwarp();
    const int req = vs[1], done = vs[2];
    if (req) {
      collective_compact();
      continue;
    }
    if (done == W) break;
    __nanosleep(64);
  }
  bar_c<NT>();
  const int n_base = s_int[0];

  // Final Step 5: the k smallest (D, item) keys, (d_max, -1) past the valid candidates (R11).
  // The survivors (resolved, distinct keys) are placed by rank: one pass, one barrier.
  // Few survivors: resolve them all and place by rank directly (no radix select, no barriers
  // beyond one); many: cut to the k smallest D (ties kept) first.
  int n = n_base;
  if (n_base <= a.direct_max) {
    for (int e = tid; e < n_base; e += NT) buf[e] = resolve_key(buf[e], probe, a);
    bar_c<NT>();
  } else {
    uint32_t t2 = tau;
    n = compact<NT, CAPM>(buf, hist, s_int, probe, a, n_base, a.k, true, &t2);
  }
  for (int e = tid; e < n; e += NT) {
    const uint64_t key = buf[e];
    int rank = 0;
    for (int f = 0; f < n; ++f) rank += buf[f] < key ? 1 : 0;  // broadcast reads
    if (rank < a.k) {
      a.out_ids[qi * a.k + rank] = step5_id(key);
      a.out_dist[qi * a.k + rank] = static_cast<int32_t>(key >> 32);
    }
  }
  for (int r = n + tid; r < a.k; r += NT) {
    a.out_ids[qi * a.k + r] = -1;
    a.out_dist[qi * a.k + r] = kDMax;
  }
}

template <int M, int MODE, int CAPM, int VAR>
cudaError_t launch_cap(const RotArgs& a, int64_t nq, size_t smem, cudaStream_t st) {
  using C = Geo<M, MODE, VAR>;
  cudaError_t e = cudaFuncSetAttribute(scan_rot_kernel<M, MODE, CAPM, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  scan_rot_kernel<M, MODE, CAPM, VAR><<<static_cast<unsigned>(nq), C::NTOT, smem, st>>>(a);
  note_launch();
  return cudaGetLastError();
}

template <int M, int MODE, int VAR = 0>
cudaError_t launch(RotArgs a, int64_t nq, int smem_budget, cudaStream_t st) {
  using C = Geo<M, MODE, VAR>;
  constexpr int NT = C::NT;
  auto al = [](uint32_t x, uint32_t b) { return (x + b - 1) / b * b; };
  const uint32_t lut = MODE == kLutP64 ? static_cast<uint32_t>(a.Ks) * 256u : C::NG * kW32GroupBytes;
  const uint32_t chunk = 32u * M;  // codes of one 32-slot chunk (P terms are read from L2)
  // (SEG, NS, cap): the first candidate that fits the per-CTA budget; 2-3 stages in flight suffice.
  static const int cand[][3] = {{16, 4, 1024}, {16, 3, 1024}, {16, 2, 1024}, {8, 4, 1024}, {8, 3, 1024},
                                {8, 2, 1024}};
  int SEG = 8, NS = 2, cap = 1024;
  size_t smem = 0;
  const int e_seg = static_cast<int>(opt(V3DB_OPT_SCAN_SEG));  // experiments: force (SEG, NS, cap)
  const int e_ns = static_cast<int>(opt(V3DB_OPT_SCAN_NS));
  const int e_cap = static_cast<int>(opt(V3DB_OPT_SCAN_CAP));
  for (const auto& c : cand) {
    const int seg = e_seg > 0 ? e_seg : c[0], ns = e_ns > 0 ? e_ns : c[1];
    // headroom: one stage share of every consumer warp above the high-water mark, which must be >= k
    const int head = (NT / 32) * ((seg + NT / 32 - 1) / (NT / 32)) * 32;
    int cp = e_cap > 0 ? e_cap : c[2];
    while (cp < a.k + head) cp *= 2;
    const size_t need = al(lut, 128) + static_cast<size_t>(ns) * al(seg * chunk, 128) + al(4u * (a.nprobe + 1), 16) + 16u * ns * seg +
                        8u * cp + 512 * 4 + 16u * a.nprobe + al(a.dim, 16) + 256 + 16u * ns;
    SEG = seg;
    NS = ns;
    cap = cp;
    smem = need;
    if (need <= static_cast<size_t>(smem_budget) || (e_seg > 0 && e_ns > 0)) break;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  a.SEG = SEG;
  a.NS = NS;
  a.cap = cap;
  a.stage_bytes = al(SEG * chunk, 128);
  uint32_t o = al(lut, 128);
  a.off_stage = o;
  o += NS * a.stage_bytes;
  a.off_desc = o;
  o += 16u * NS * SEG;
  a.off_vc = o;
  o += al(4u * (a.nprobe + 1), 16);
  a.off_buf = o;
  o += 8u * cap;
  a.off_hist = o;
  o += 512 * 4;  // two alternating radix histograms
  a.off_probe = o;
  o += 16u * a.nprobe;
  a.off_q = o;
  o += al(a.dim, 16);
  a.off_int = o;
  o += 256;
  a.off_bar = o;
  const int capm = cap / NT;
  if (capm <= 2) return launch_cap<M, MODE, 2, VAR>(a, nq, smem, st);
  if (capm <= 4) return launch_cap<M, MODE, 4, VAR>(a, nq, smem, st);
  if (capm <= 8) return launch_cap<M, MODE, 8, VAR>(a, nq, smem, st);
  return launch_cap<M, MODE, 16, VAR>(a, nq, smem, st);
}

template <int M, int MODE, int VAR = 0>
int budget() {
  using C = Geo<M, MODE, VAR>;
  return (228 * 1024) / C::MINB - 1024;  // per-CTA share of the SM (1 KB reserved per CTA)
}

// L2-aware schedule: CTAs run in blockIdx order, ~300 at a time, so
// queries whose probe sets overlap should be adjacent.  List ids are a random sample of the
// database, so min(probe list ids) is a MinHash of the probe set: two queries get the same key with
// probability = the Jaccard similarity of their probe sets.  A counting sort by that key groups
// them; the results do not depend on the order (each CTA writes its own query's rows).
__global__ void minhash_kernel(const int32_t* __restrict__ lists, int64_t nq, int nprobe, int32_t* __restrict__ key,
                               int* __restrict__ hist) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nq) return;
  int m = 0x7fffffff;
  for (int r = 0; r < nprobe; ++r) m = min(m, __ldg(lists + q * nprobe + r));
  key[q] = m;
  atomicAdd(hist + m, 1);
}

// exclusive scan of hist[0, n) in place (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) scan_hist_kernel(int* __restrict__ hist, int n) {
  __shared__ int part[1024];
  const int per = (n + 1023) / 1024, b = threadIdx.x * per, e = min(n, b + per);
  int sum = 0;
  for (int i = b; i < e; ++i) sum += hist[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = part[threadIdx.x] - sum;
  for (int i = b; i < e; ++i) {
    const int c = hist[i];
    hist[i] = run;
    run += c;
  }
}

__global__ void scatter_kernel(const int32_t* __restrict__ key, int64_t nq, int* __restrict__ offs,
                               int32_t* __restrict__ order) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nq) return;
  order[atomicAdd(offs + key[q], 1)] = static_cast<int32_t>(q);
}

cudaError_t scan_dispatch(const v3db_snapshot* s, RotArgs& a, int64_t nq, cudaStream_t st) {
#define V3DB_ROT(MM, MODE) return launch<MM, MODE>(a, nq, budget<MM, MODE>(), st);
  if (s->lut_mode == kLutP64) {
    switch (s->M) {
      case 4: V3DB_ROT(4, kLutP64)
      case 8: V3DB_ROT(8, kLutP64)
      case 12: V3DB_ROT(12, kLutP64)
      case 16: V3DB_ROT(16, kLutP64)
      case 20: V3DB_ROT(20, kLutP64)
      case 24: V3DB_ROT(24, kLutP64)
      case 28: V3DB_ROT(28, kLutP64)
      case 32: V3DB_ROT(32, kLutP64)
      default: return cudaErrorInvalidValue;
    }
  }
  switch (s->M) {
    case 8: V3DB_ROT(8, kLutW32)
    case 12: V3DB_ROT(12, kLutW32)
    case 16: V3DB_ROT(16, kLutW32)
    case 24: V3DB_ROT(24, kLutW32)
    case 32: V3DB_ROT(32, kLutW32)
    case 48: V3DB_ROT(48, kLutW32)
    case 64: V3DB_ROT(64, kLutW32)
    case 96: V3DB_ROT(96, kLutW32)
    case 128: V3DB_ROT(128, kLutW32)
    default: return cudaErrorInvalidValue;
  }
#undef V3DB_ROT
}


}  // namespace

// The L2-aware query order (see minhash_kernel): scratch [2 nq + nlist] int32; the order is
// written to scratch + nq.
cudaError_t minhash_order(const int32_t* lists, int64_t nq, int nprobe, int nlist, int32_t* scratch, cudaStream_t st) {
  int32_t* key = scratch;
  int32_t* order = key + nq;
  int* hist = order + nq;
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int) * nlist, st);
  if (e != cudaSuccess) return e;
  const unsigned g = static_cast<unsigned>((nq + 255) / 256);
  minhash_kernel<<<g, 256, 0, st>>>(lists, nq, nprobe, key, hist);
  scan_hist_kernel<<<1, 1024, 0, st>>>(hist, nlist);
  scatter_kernel<<<g, 256, 0, st>>>(key, nq, hist, order);
  note_launch(3);
  return cudaGetLastError();
}

cudaError_t scan_rotated(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                         const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                         int32_t* trace, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  if (s->lut_mode == 0) return cudaErrorInvalidValue;
  RotArgs a;
  a.queries = queries;
  a.dim = s->dim;
  a.d = s->d;
  a.Ks = s->Ks;
  a.L = s->L;
  a.Lp = (s->L + 31) & ~31;
  a.nprobe = nprobe;
  a.k = k;
  a.cbT = s->cbT;
  a.codes = s->codes_rot;
  a.pterm = s->pterm_rot;
  a.ids = s->ids;
  a.counts = s->counts;
  a.lists = lists;
  a.ldist = ldist;
  a.out_ids = out_ids;
  a.out_dist = out_dist;
  a.trace = trace;
  a.order = nullptr;
  {
    const int64_t f = opt(V3DB_OPT_SCAN_FIRST);  // experiments
    a.first_mult = f > 0 ? static_cast<int>(f) : 16;  // measured: 16 vs 4 -0.8 % at C4, -1.8 % at C3, flat at C1/C2
    const int64_t dm = opt(V3DB_OPT_SCAN_DIRECT);  // experiments (-1 = never rank directly)
    a.direct_max = dm > 0 ? static_cast<int>(dm) : dm < 0 ? 0 : 256;  // measured: C1 scan -10 %, C2/C3 -2 %, C4 flat
  }
  // L2-aware schedule when the probed lists do not fit in L2 anyway and the batch is large
  const int64_t sched = opt(V3DB_OPT_SCHED);
  const bool want = sched ? sched == 1
                          : (nq >= 2048 && static_cast<int64_t>(s->nlist) * s->L * s->M > (int64_t(64) << 20));
  void* sbuf = nullptr;
  if (want) {
    cudaError_t e = scratch_alloc(&sbuf, sizeof(int32_t) * (2 * nq + s->nlist), st);
    if (e != cudaSuccess) return e;
    e = minhash_order(lists, nq, nprobe, s->nlist, static_cast<int32_t*>(sbuf), st);
    if (e != cudaSuccess) {
      cudaFreeAsync(sbuf, st);
      return e;
    }
    a.order = static_cast<int32_t*>(sbuf) + nq;
  }
  cudaError_t res = scan_dispatch(s, a, nq, st);
  if (sbuf) cudaFreeAsync(sbuf, st);
  return res;
}

}  // namespace v3db

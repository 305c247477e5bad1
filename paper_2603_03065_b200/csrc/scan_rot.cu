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
// Rotated LUT.  Lane l of a warp handles slot j = 32c + l of a
// chunk.  At step s it reads subspace m = gG + (l + s) mod G (G | 32 subspaces per group) from
// table COLUMN l + s, so the 32 lanes of every LDS hit 32 distinct banks whatever the codes are.
// The slot's code bytes are stored pre-rotated (codes_rot, built once) so byte s of the
// register word is the right code.  Two table geometries:
//   kLutP64 (G = M <= 32): rows of 64 int32 columns, column col = subspace col mod G;
//            address = code*256 + 4l + 4s = PRMT(code byte, 4l) + immediate.        1 ALU op
//   kLutW32 (G = gcd(M,32), M/G groups): rows of 32 columns, 257 rows per group; a lane whose
//            column l+s passes 32 wraps into the next row, which the stored byte pre-compensates
//            ((code - 1) mod 256; row 256 duplicates row 0):
//            address = ((byte << 7) | 4l) + immediate.                                2 ALU ops
// Top-k: candidates with D <= tau go to a shared buffer of (D, slot) keys (warp-aggregated
// append).  Between rounds (one 32-slot chunk per warp) the CTA compacts the buffer when it could
// overflow during the next round: item ids are resolved, the buffer is sorted by (D, item) and
// truncated to k, and tau = D of the k-th key.  Every key excluded by tau has k keys at or below
// it, so the final top-k is exact.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "topk.cuh"
#include "v3db_internal.cuh"

namespace v3db {

int plan_lut(int M, int Ks, int d, int* G) {
  *G = 0;
  if (M < 4 || M % 4 != 0 || d % 4 != 0 || Ks < 1 || Ks > 256) return 0;
  const int g = (M % 32 == 0) ? 32 : (M % 16 == 0) ? 16 : (M % 8 == 0) ? 8 : 4;
  const char* force = getenv("V3DB_LUT_MODE");  // test hook: "w32" forces the wrap geometry
  const bool want_w32 = force && force[0] == 'w';
  if (!want_w32 && g == M && (M == 4 || M == 8 || M == 16 || M == 32) && Ks * 256 <= 65536) {
    *G = g;
    return kLutP64;
  }
  if ((M == 8 || M == 16 || M == 24 || M == 32 || M == 48 || M == 64 || M == 96 || M == 128) &&
      (M / g) * kW32GroupBytes <= 200 * 1024) {
    *G = g;
    return kLutW32;
  }
  return 0;
}

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kTauInit = 0x7ffffffeu;  // accept every valid D (< d_max)

template <int M, int MODE>
struct Geo {
  static constexpr int G = (M % 32 == 0) ? 32 : (M % 16 == 0) ? 16 : (M % 8 == 0) ? 8 : 4;
  static constexpr int NG = M / G;
  static constexpr int NW = M / 4;  // 32-bit code words per slot
  static constexpr int TGB = (MODE == kLutW32) ? kW32GroupBytes : 0;  // bytes per group table
  static constexpr int NT = (MODE == kLutW32 && NG * kW32GroupBytes > 100 * 1024) ? 512 : 256;
  static constexpr int MINB = (MODE == kLutP64) ? 3 : (NT == 512 ? 1 : 2);
};

template <int M>
__device__ __forceinline__ void load_codes(const uint8_t* p, uint32_t (&w)[M / 4]) {
  if constexpr (M % 16 == 0) {
#pragma unroll
    for (int v = 0; v < M / 16; ++v) {
      uint4 x;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "l"(p + 16 * v));
      w[4 * v] = x.x; w[4 * v + 1] = x.y; w[4 * v + 2] = x.z; w[4 * v + 3] = x.w;
    }
  } else if constexpr (M % 8 == 0) {
#pragma unroll
    for (int v = 0; v < M / 8; ++v) {
      uint2 x;
      asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(x.x), "=r"(x.y) : "l"(p + 8 * v));
      w[2 * v] = x.x; w[2 * v + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < M / 4; ++v)
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(w[v]) : "l"(p + 4 * v));
  }
}

__device__ __forceinline__ int32_t ld_nc_i32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

struct RotArgs {
  const int8_t* queries;
  int dim, d, Ks, L, nprobe, k, cap;
  const int8_t* cbT;
  const uint8_t* codes;   // codes_rot
  const int32_t* pterm;
  const int32_t* ids;
  const int32_t* counts;
  const int32_t* lists;
  const int32_t* ldist;
  int32_t* out_ids;
  int32_t* out_dist;
  int32_t* trace;
};

// Shared-memory layout (bytes): [LUT tables][buf: cap x u64][probe: nprobe x int4][q: dim][scalars]
__host__ __device__ inline uint32_t lut_bytes(int mode, int M, int G, int Ks) {
  return mode == kLutP64 ? static_cast<uint32_t>(Ks) * 256u : static_cast<uint32_t>(M / G) * kW32GroupBytes;
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
      __syncthreads();
    }
  }
}

// Resolve item ids of the unresolved entries [nres, n), sort, keep the first min(n, k), set tau.
template <int NT>
__device__ void compact(uint64_t* buf, const int4* probe, int* s_int, const RotArgs& a, int n) {
  const int nres = s_int[1];
  for (int e = nres + static_cast<int>(threadIdx.x); e < n; e += NT) {
    const uint64_t key = buf[e];
    const uint32_t flat = static_cast<uint32_t>(key);
    const int rho = static_cast<int>(flat / static_cast<uint32_t>(a.L));
    const int j = static_cast<int>(flat - static_cast<uint32_t>(rho) * a.L);
    const int32_t id = __ldg(a.ids + static_cast<int64_t>(probe[rho].x) * a.L + j);
    buf[e] = (key & 0xffffffff00000000ull) | (static_cast<uint32_t>(id) ^ 0x80000000u);
  }
  int P = 1;
  while (P < n) P <<= 1;
  for (int e = n + static_cast<int>(threadIdx.x); e < P; e += NT) buf[e] = ~0ull;
  __syncthreads();
  bitonic_sort<NT>(buf, P);
  if (threadIdx.x == 0) {
    const int keep = n < a.k ? n : a.k;
    s_int[0] = keep;
    s_int[1] = keep;
    if (n >= a.k) s_int[2] = static_cast<int>(buf[a.k - 1] >> 32);
  }
  __syncthreads();
}

template <int M, int MODE>
__global__ void __launch_bounds__(Geo<M, MODE>::NT, Geo<M, MODE>::MINB) scan_rot_kernel(const RotArgs a) {
  using C = Geo<M, MODE>;
  constexpr int NT = C::NT, W = NT / 32, G = C::G, NG = C::NG, NW = C::NW;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lbytes = lut_bytes(MODE, M, G, a.Ks);
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem + lbytes);
  int4* probe = reinterpret_cast<int4*>(buf + a.cap);                // (list, d_i, count, 0)
  int8_t* qs = reinterpret_cast<int8_t*>(probe + a.nprobe);
  int* s_int = reinterpret_cast<int*>(qs + ((a.dim + 15) & ~15));   // [0] count [1] resolved [2] tau

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t qi = blockIdx.x;
  const int L = a.L, nprobe = a.nprobe;

  for (int u = tid; u < a.dim; u += NT) qs[u] = a.queries[qi * a.dim + u];
  for (int r = tid; r < nprobe; r += NT) {
    const int li = a.lists[qi * nprobe + r];
    probe[r] = make_int4(li, a.ldist[qi * nprobe + r], __ldg(a.counts + li), 0);
  }
  if (tid == 0) {
    s_int[0] = 0;
    s_int[1] = 0;
    s_int[2] = static_cast<int>(kTauInit);
  }
  __syncthreads();

  const int cpl = (L + 31) >> 5;              // 32-slot chunks per list
  const int nchunks = nprobe * cpl;
  const int nrounds = (nchunks + W - 1) / W;
  const uint32_t lane4 = 4u * lane;

  // chunk c = round * W + warp  ->  (rho, jc); advanced incrementally
  int c = warp, rho = warp / cpl, jc = warp - (warp / cpl) * cpl;

  // prefetch the first chunk while the LUT is built
  uint32_t cur[NW];
  int32_t pcur = 0;
  auto fetch = [&](int c_, int rho_, int jc_, uint32_t(&w)[NW], int32_t& p) {
#pragma unroll
    for (int v = 0; v < NW; ++v) w[v] = 0;
    p = 0;
    if (c_ < nchunks) {
      const int4 pr = probe[rho_];
      const int j = jc_ * 32 + lane;
      if (j < pr.z) {
        const int64_t slot = static_cast<int64_t>(pr.x) * L + j;
        load_codes<M>(a.codes + slot * M, w);
        p = ld_nc_i32(a.pterm + slot);
      }
    }
  };
  fetch(c, rho, jc, cur, pcur);

  // Step 3 (factorised): A_q[m][c] = -2 <C_{m,c}, q^{(m)}>, written into the rotated tables.
  {
    int32_t* T = reinterpret_cast<int32_t*>(smem);
    const int d = a.d;
    for (int e = tid; e < M * a.Ks; e += NT) {
      const int m = e % M, cc = e / M;
      const int8_t* cw = a.cbT + (static_cast<int64_t>(cc) * M + m) * d;
      const int8_t* qm = qs + m * d;
      int acc = 0;
      for (int u = 0; u < d; u += 4)
        acc = __dp4a(*reinterpret_cast<const int*>(cw + u), *reinterpret_cast<const int*>(qm + u), acc);
      const int32_t A = -2 * acc;
      const int g = m / G, r = m - g * G;
      if constexpr (MODE == kLutP64) {
#pragma unroll
        for (int col = r; col < 64; col += G) T[cc * 64 + col] = A;
      } else {
        int32_t* Tg = T + g * (kW32GroupBytes / 4);
#pragma unroll
        for (int col = r; col < 32; col += G) {
          Tg[cc * 32 + col] = A;
          if (cc == 0) Tg[256 * 32 + col] = A;  // row 256 duplicates row 0 (wrap of code 0)
        }
      }
    }
  }
  __syncthreads();

  uint32_t tau = kTauInit;
  int n_buf = 0;  // entries in buf (CTA-uniform: counted with __syncthreads_count)
  const int64_t trace_base = qi * nprobe;
  for (int round = 0; round < nrounds; ++round) {
    // next chunk of this warp
    int c2 = c + W, rho2 = rho, jc2 = jc + W;
    while (jc2 >= cpl) {
      jc2 -= cpl;
      ++rho2;
    }
    uint32_t nxt[NW];
    int32_t pnxt;
    fetch(c2, rho2, jc2, nxt, pnxt);

    bool pass = false;
    if (c < nchunks) {
      const int4 pr = probe[rho];
      const int j = jc * 32 + lane;
      int32_t D = kDMax;
      if (jc * 32 < pr.z) {  // warp-uniform: the chunk holds valid slots
        int32_t acc = pr.y + pcur;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
#pragma unroll
          for (int s = 0; s < G; ++s) {
            const int pos = g * G + s;
            const uint32_t w = cur[pos >> 2];
            uint32_t ad;
            if constexpr (MODE == kLutP64) {
              ad = __byte_perm(w, lane4, 0x5504u | ((pos & 3) << 4));
            } else {
              const int b = pos & 3;
              const uint32_t sh = (b == 0) ? (w << 7) : (w >> (8 * b - 7));
              ad = (sh & 0x7f80u) | lane4;
            }
            acc += *reinterpret_cast<const int32_t*>(smem + (g * C::TGB + 4 * s) + ad);
          }
        }
        if (j < pr.z) D = acc;
      }
      if (a.trace && j < L) __stcs(a.trace + (trace_base + rho) * L + j, D);
      pass = j < pr.z && static_cast<uint32_t>(D) <= tau;
      const uint32_t bal = __ballot_sync(kFull, pass);
      if (bal) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_int[0], __popc(bal));
        base = __shfl_sync(kFull, base, 0);
        if (pass)
          buf[base + __popc(bal & ((1u << lane) - 1u))] =
              (static_cast<uint64_t>(static_cast<uint32_t>(D)) << 32) | static_cast<uint32_t>(rho * L + j);
      }
    }
    n_buf += __syncthreads_count(pass);           // barrier: this round's appends are visible
    if (n_buf > a.cap - NT || round == nrounds - 1) {  // CTA-uniform
      compact<NT>(buf, probe, s_int, a, n_buf);
      n_buf = n_buf < a.k ? n_buf : a.k;
      tau = static_cast<uint32_t>(s_int[2]);        // written only inside compact()
    }
    c = c2;
    rho = rho2;
    jc = jc2;
#pragma unroll
    for (int v = 0; v < NW; ++v) cur[v] = nxt[v];
    pcur = pnxt;
  }

  // Step 5 output: the first k keys of the buffer, (d_max, -1) past the valid candidates (R11).
  const int kept = n_buf;
  for (int r = tid; r < a.k; r += NT) {
    int32_t id = -1, dd = kDMax;
    if (r < kept) {
      const uint64_t key = buf[r];
      id = step5_id(key);
      dd = static_cast<int32_t>(key >> 32);
    }
    a.out_ids[qi * a.k + r] = id;
    a.out_dist[qi * a.k + r] = dd;
  }
}

template <int M, int MODE>
cudaError_t launch(const RotArgs& a, int64_t nq, size_t smem, cudaStream_t st) {
  using C = Geo<M, MODE>;
  cudaError_t e = cudaFuncSetAttribute(scan_rot_kernel<M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  scan_rot_kernel<M, MODE><<<static_cast<unsigned>(nq), C::NT, smem, st>>>(a);
  note_launch();
  return cudaGetLastError();
}

template <int MODE>
int threads_for(int M, int G) {
  return (MODE == kLutW32 && (M / G) * kW32GroupBytes > 100 * 1024) ? 512 : 256;
}

}  // namespace

cudaError_t scan_rotated(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                         const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                         int32_t* trace, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  if (s->lut_mode == 0) return cudaErrorInvalidValue;
  const int nt = s->lut_mode == kLutP64 ? 256 : threads_for<kLutW32>(s->M, s->lut_g);
  // buffer: after a compaction at most k entries; one round appends at most nt
  int cap = 512;
  while (cap < k + 2 * nt) cap <<= 1;
  RotArgs a;
  a.queries = queries;
  a.dim = s->dim;
  a.d = s->d;
  a.Ks = s->Ks;
  a.L = s->L;
  a.nprobe = nprobe;
  a.k = k;
  a.cap = cap;
  a.cbT = s->cbT;
  a.codes = s->codes_rot;
  a.pterm = s->pterm;
  a.ids = s->ids;
  a.counts = s->counts;
  a.lists = lists;
  a.ldist = ldist;
  a.out_ids = out_ids;
  a.out_dist = out_dist;
  a.trace = trace;
  const size_t smem = lut_bytes(s->lut_mode, s->M, s->lut_g, s->Ks) + sizeof(uint64_t) * cap +
                      sizeof(int4) * nprobe + ((s->dim + 15) & ~15) + 16;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  if (s->lut_mode == kLutP64) {
    switch (s->M) {
      case 4: return launch<4, kLutP64>(a, nq, smem, st);
      case 8: return launch<8, kLutP64>(a, nq, smem, st);
      case 16: return launch<16, kLutP64>(a, nq, smem, st);
      case 32: return launch<32, kLutP64>(a, nq, smem, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (s->M) {
    case 8: return launch<8, kLutW32>(a, nq, smem, st);
    case 16: return launch<16, kLutW32>(a, nq, smem, st);
    case 24: return launch<24, kLutW32>(a, nq, smem, st);
    case 32: return launch<32, kLutW32>(a, nq, smem, st);
    case 48: return launch<48, kLutW32>(a, nq, smem, st);
    case 64: return launch<64, kLutW32>(a, nq, smem, st);
    case 96: return launch<96, kLutW32>(a, nq, smem, st);
    case 128: return launch<128, kLutW32>(a, nq, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace v3db

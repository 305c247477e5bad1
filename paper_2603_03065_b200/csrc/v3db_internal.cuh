// v3db_internal.cuh -- shared declarations of libv3db's CUDA kernels (sm_100a).
//
// Device layouts:
//   centroids  int8  [nlist][dim]          mu_i
//   cnorm      int32 [nlist]               ||mu_i||^2
//   codebooks  int8  [M][Ks][d]            C_{m,c}
//   ids        int32 [nlist][L]            item_{i,j}, -1 = padding
//   codes      uint8 [nlist][L][M]         v^PQ_{i,j}
//   counts     int32 [nlist]               valid slots (valid slots come first, R7)
//   pterm      int32 [nlist][L]            P_{i,j} = ||xhat_ij||^2 + 2<mu_i, xhat_ij>
//   list_of    int32 [n]                   final list of every vector (export/tests)
//   codes_rot  uint8 [nlist][Lp/32][M/U][32][U]  codes re-ordered for the conflict-free rotated
//                                          LUT scan: per 32-slot chunk, unit-transposed (U = 16/8/4
//                                          bytes), bytes rotated per slot (DESIGN.md "Rotated LUT
//                                          layout"); Lp = L rounded up to 32
//   pterm_rot  int32 [nlist][Lp]           P_{i,j} with the padded list stride
//   cbT        int8  [Ks][M][d]            codebooks, codeword-major (coalesced LUT build)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "v3db.h"

struct v3db_snapshot {
  int64_t n = 0;
  int dim = 0, nlist = 0, L = 0, M = 0, Ks = 0, d = 0;
  int64_t total_valid = 0;
  int device = 0;
  int8_t* centroids = nullptr;
  int32_t* cnorm = nullptr;
  int8_t* codebooks = nullptr;
  int32_t* ids = nullptr;
  uint8_t* codes = nullptr;
  int32_t* counts = nullptr;
  int32_t* pterm = nullptr;
  int32_t* list_of = nullptr;
  // rotated-LUT scan (scan_rot.cu): lut_mode 0 = not supported for this shape (generic scan),
  // kLutP64 / kLutW32 = table geometry; lut_g = subspaces per rotation group.
  int lut_mode = 0, lut_g = 0;
  uint8_t* codes_rot = nullptr;
  int32_t* pterm_rot = nullptr;
  int8_t* cbT = nullptr;
  // list-major tensor-core scan (scan_lm.cu): xhat [nlist][lm_Lp][dim] int8 = the reconstruction
  // of every slot (0 for padding), lm_Lp = L rounded up to 128 (one UMMA tile of slots); null when
  // the shape is not supported (dim % 16 != 0).
  int8_t* xhat = nullptr;
  int lm_Lp = 0;
  // NEXT-1 (fx16.cu): 16-bit fixed-point snapshot.  When fx != 0 the int8
  // fields centroids / cnorm / codebooks / pterm are unused and these hold the data instead.
  int fx = 0;
  int32_t* centroids32 = nullptr;  // [nlist][dim]
  int64_t* cnorm64 = nullptr;      // [nlist]
  int32_t* codebooks32 = nullptr;  // [M][Ks][d]
  int64_t* pterm64 = nullptr;      // [nlist][L]
  uint8_t* codes_rot16 = nullptr;  // [nlist][L][M], per-slot rotated in groups of 16 (+ 8) (M % 8 == 0, Ks == 256)
  // fixed-point list-major scan: the reconstruction of every slot as three balanced int8 limb planes
  // [3][nlist][lm_Lp][dim] (0 for padding); null unless dim % 16 == 0, dim <= 256, nlist <= 32768
  int8_t* xhat_fx = nullptr;
};

// Device-side invariant checks: traps in the debug build (libv3db_debug.so, -DV3DB_DEBUG), no
// code in the release build.  Used on every shared-memory buffer append / stage write whose bound
// rests on a protocol argument rather than on a per-write guard.
#ifdef V3DB_DEBUG
#define V3DB_DCHECK(cond)  \
  do {                     \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define V3DB_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace v3db {

// Counts every kernel launch of the library (v3db_kernel_launches).
void note_launch(int n = 1);
// Process-wide implementation options (v3db_set_option; V3DB_OPT_* keys, 0 = default).
int64_t opt(int key);
// Stream-ordered scratch from the library's own device memory pool (free with cudaFreeAsync).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
// Debugging aid (debug build libv3db_debug.so only, env V3DB_SYNC_CHECK=1): synchronize the
// stream after a launch and return the first error tagged with the kernel name (through
// v3db_last_error).  No-op in the release build.
cudaError_t debug_sync(cudaStream_t st, const char* what);

constexpr int32_t kDMax = 0x7fffffff;  // d_max = 2^31 - 1 (reading R8)

// Step 1 + Step 2 (and build ranking B2): for each row x of X [n][dim], the R smallest
// composite keys (dist(x, mu_i), i), ascending -> out_idx/out_dist [n][R].
// list_hist (optional, pre-zeroed [nlist]): += 1 for every output list (the list-major scan's
// grouping histogram).
cudaError_t coarse_topk(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* cnorm,
                        int nlist, int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st,
                        int* list_hist = nullptr);

// Build kernels (build_kernels.cu).
cudaError_t gather_rows(const int8_t* db, int dim, const int32_t* rows, int nrows, int8_t* out,
                        int32_t* norms_or_null, cudaStream_t st);
cudaError_t make_codebooks(const int8_t* db, const int8_t* mu, const int32_t* list_of, int dim,
                           int M, int Ks, const int32_t* codeword_rows, int8_t* codebooks,
                           cudaStream_t st);
cudaError_t encode_and_place(const int8_t* db, int64_t n, int dim, const int8_t* mu,
                             const int32_t* list_of, const int32_t* flat_pos, const int8_t* codebooks,
                             int M, int Ks, uint8_t* codes, int32_t* ids, cudaStream_t st);
cudaError_t slot_terms(const int8_t* mu, const int8_t* codebooks, const uint8_t* codes,
                       const int32_t* ids, int nlist, int L, int dim, int M, int Ks, int32_t* pterm,
                       cudaStream_t st);

// Rotated-LUT geometry.
constexpr int kLutP64 = 1;   // one group of M <= 32 subspaces, rows of 64 int32 columns (PRMT addressing)
constexpr int kLutW32 = 2;   // rot_ngroups(M) groups of 257 rows x 32 columns (wrap addressing)
constexpr int kW32GroupBytes = 257 * 32 * 4;
// Chooses the geometry for (M, Ks, d): returns the mode (0 = generic scan) and sets *G (the first
// group's size; informational).
int plan_lut(int M, int Ks, int d, int* G);
// Bytes per lane per unit of the chunk-transposed codes_rot layout.
__host__ __device__ constexpr int rot_unit(int M) { return M % 16 == 0 ? 16 : M % 8 == 0 ? 8 : 4; }
// Rotation groups of the W32 geometry: M (a multiple of 4) split greedily into groups of 32, 16,
// 8, 4 consecutive subspaces (M = 24 -> 16 + 8).  Group g covers [rot_goff(M,g), +rot_gsize(M,g)).
__host__ __device__ constexpr int rot_ngroups(int M) {
  int n = 0;
  for (int r = M, sz = 32; r > 0;) {
    if (r >= sz) {
      r -= sz;
      ++n;
    } else {
      sz >>= 1;
    }
  }
  return n;
}
__host__ __device__ constexpr int rot_gsize(int M, int g) {
  for (int r = M, sz = 32, i = 0; r > 0;) {
    if (r >= sz) {
      if (i == g) return sz;
      r -= sz;
      ++i;
    } else {
      sz >>= 1;
    }
  }
  return 0;
}
__host__ __device__ constexpr int rot_goff(int M, int g) {
  int o = 0;
  for (int i = 0; i < g; ++i) o += rot_gsize(M, i);
  return o;
}
// Build: codes_rot / pterm_rot from the canonical codes / pterm, and cbT.
cudaError_t rotate_codes(const uint8_t* codes, const int32_t* pterm, int nlist, int L, int M, int mode, int G,
                         uint8_t* codes_rot, int32_t* pterm_rot, cudaStream_t st);
cudaError_t make_xhat(const uint8_t* codes, const int32_t* counts, const int8_t* cb, int nlist, int L, int Lp,
                      int dim, int M, int Ks, int8_t* xhat, cudaStream_t st);
cudaError_t make_xhat_fx(const uint8_t* codes, const int32_t* counts, const int32_t* cb, int nlist, int L, int Lp,
                         int dim, int M, int Ks, int8_t* xl, cudaStream_t st);
// Steps 3-5 of the fixed-point path, list-major on the tensor cores (scan_lm.cu).  Requires s->xhat_fx.
cudaError_t scan_list_major_fx(const v3db_snapshot* s, const int32_t* queries, int64_t nq, int nprobe, int k,
                               const int32_t* lists, const int64_t* ldist, int32_t* out_ids, int64_t* out_dist,
                               int64_t* trace_cand, cudaStream_t st, void (*prof)(int, cudaStream_t));
cudaError_t transpose_codebooks(const int8_t* cb, int M, int Ks, int d, int8_t* cbT, cudaStream_t st);

// Steps 3-5, generic query-major scan (scan_lut.cu): any shape, per-query LUT [M][Ks] in shared
// memory (not conflict-free).
cudaError_t scan_generic(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                         const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                         int32_t* trace_cand, cudaStream_t st);

// Steps 3-5, rotated-LUT scan (scan_rot.cu): conflict-free LUT lookups, padding chunks skipped,
// buffered exact top-k.  Requires s->lut_mode != 0.
cudaError_t scan_rotated(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                         const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                         int32_t* trace_cand, cudaStream_t st);

// Steps 3-5, list-major tensor-core scan (scan_lm.cu): D_{i,j} = d_i + P_{i,j} - 2 <q, xhat_{i,j}> as
// tcgen05 kind::i8 tiles per (list, 128 slots, <= NT probing queries), every D to the trace (a
// library scratch trace when the caller passes none), 32-slot group minima, then an exact per-query
// selection.  Requires s->xhat.  prof(i) records profiling marks 2 (after grouping) and 3 (after
// the contraction kernel).
// list_hist: the per-list count of (query, rank) pairs that coarse_topk accumulated (or null:
// computed here).
cudaError_t scan_list_major(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int k,
                            const int32_t* lists, const int32_t* ldist, int32_t* out_ids, int32_t* out_dist,
                            int32_t* trace_cand, cudaStream_t st, void (*prof)(int, cudaStream_t),
                            const int* list_hist = nullptr);

// Ascending sort of nseg segments of P (a power of two) 64-bit keys (witness.cu).
cudaError_t segmented_sort(uint64_t* keys, int64_t nseg, int P, cudaStream_t st);

// Alg. 1 support (build_kernels.cu): dist(X[r], mu[lists[r]]) for every row r.
cudaError_t pair_dist(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* lists, int32_t* out,
                      cudaStream_t st);
// keys[r] = (uint32(delta[r] + 2^31) << 32) | r, delta = e_t - e_i; P - n padding keys = ~0.
cudaError_t delta_keys(const int32_t* e_t, const int32_t* e_i, int64_t n, int64_t P, uint64_t* keys, cudaStream_t st);

// Prover witness of a batch of queries (witness.cu; §4.7).  Outputs may be null.
cudaError_t witness_batch(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe, int32_t* list_order,
                          int32_t* list_dist, int32_t* lut_sel, int32_t* cand_items, int32_t* cand_dist,
                          cudaStream_t st);

// NEXT-1, the 16-bit fixed-point path (fx16.cu).
constexpr int64_t kDMaxFx = 0x7fffffffffffffffLL;  // d_max = 2^63 - 1 (R18)
int fx_shift2(int dim);  // key shift of Step-2 keys d << sh | i
int fx_shift5(int dim);  // key shift of Step-5 keys D << sh | slot
cudaError_t encode_fixed_point(const float* x, int64_t n, double v_max, int32_t* out, cudaStream_t st);
// max |v| over n int32 values -> *out (device int, pre-zeroed by the caller)
cudaError_t abs_max32(const int32_t* x, int64_t n, int* out, cudaStream_t st);
cudaError_t gather_rows32(const int32_t* db, int dim, const int32_t* rows, int nrows, int32_t* out, int64_t* norms,
                          cudaStream_t st);
cudaError_t fx_topk(const int32_t* X, int64_t n, int dim, const int32_t* mu, const int64_t* mnorm, int nlist, int R,
                    int32_t* out_idx, int64_t* out_dist, cudaStream_t st);
// The fixed-point Steps 1-2 on the tensor cores (fx_coarse_tc.cu): three int8 limbs per coordinate,
// five int32 accumulators, exact int64 keys; where fx_coarse_tc_supported (dim % 16 == 0, dim <= 256).
bool fx_coarse_tc_supported(int dim, int nlist, int R);
cudaError_t fx_topk_tc(const int32_t* X, int64_t n, int dim, const int32_t* mu, const int64_t* mnorm, int nlist,
                       int R, int sh, int32_t* out_idx, int64_t* out_dist, cudaStream_t st);
cudaError_t fx_build_tail(const int32_t* db, int64_t n, int dim, const int32_t* mu, const int32_t* list_of,
                          const int32_t* flat_pos, int M, int Ks, const int32_t* codeword_rows, int nlist, int L,
                          int32_t* cb, uint8_t* codes, int32_t* ids, int64_t* pterm, cudaStream_t st);
// L2-aware query order (scan_rot.cu): queries grouped by the MinHash min(probe list ids);
// scratch [2 nq + nlist] int32, the order lands in scratch + nq.
cudaError_t minhash_order(const int32_t* lists, int64_t nq, int nprobe, int nlist, int32_t* scratch, cudaStream_t st);
// The fx16 scan instantiations that read the rotated code copy (codes_rot16 is built only for these).
bool fx_rot_supported(int M, int Ks);
cudaError_t rotate_codes16(const uint8_t* codes, int64_t slots, int L, int M, uint8_t* out, cudaStream_t st);
cudaError_t fx_scan(const v3db_snapshot* s, const int32_t* queries, int64_t nq, int nprobe, int k, const int32_t* lists,
                    const int64_t* ldist, int32_t* out_ids, int64_t* out_dist, int64_t* trace, cudaStream_t st);

}  // namespace v3db

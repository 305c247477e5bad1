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
};

namespace v3db {

// Counts every kernel launch of the library (v3db_kernel_launches).
void note_launch(int n = 1);
// Debugging aid (env V3DB_SYNC_CHECK=1): synchronize the stream after a launch and return the
// first error tagged with the kernel name (through v3db_last_error).  No-op otherwise.
cudaError_t debug_sync(cudaStream_t st, const char* what);

constexpr int32_t kDMax = 0x7fffffff;  // d_max = 2^31 - 1 (reading R8)

// Step 1 + Step 2 (and build ranking B2): for each row x of X [n][dim], the R smallest
// composite keys (dist(x, mu_i), i), ascending -> out_idx/out_dist [n][R].
cudaError_t coarse_topk(const int8_t* X, int64_t n, int dim, const int8_t* mu, const int32_t* cnorm,
                        int nlist, int R, int32_t* out_idx, int32_t* out_dist, cudaStream_t st);

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

// Steps 3-5, query-major scan (scan_lut.cu).  Modes: final top-k over all ranks; seed (ranks
// [0, rho_end): write the exact top-k keys into cand_buf[q][0..k), cand_cnt[q] = k and the
// k-th key into tau[q]); fallback (final, only queries with flags[q] != 0, no trace).
constexpr int kModeFinal = 0, kModeSeed = 1, kModeFallback = 2;
struct QmExtra {
  int rho_begin = 0, rho_end = -1, mode = kModeFinal;
  uint64_t* cand_buf = nullptr;
  int cap = 0;
  int* cand_cnt = nullptr;
  uint64_t* tau = nullptr;
  const int* flags = nullptr;
};
cudaError_t scan_query_major(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe,
                             int k, const int32_t* lists, const int32_t* ldist, int32_t* out_ids,
                             int32_t* out_dist, int32_t* trace_cand, cudaStream_t st,
                             const QmExtra& x = QmExtra());

// Steps 3-5, list-major scan (scan_list_major.cu): groups the (query, rank) pairs by list and
// reads each probed list once per batch; exact top-k via per-query thresholds.
cudaError_t scan_list_major(const v3db_snapshot* s, const int8_t* queries, int64_t nq, int nprobe,
                            int k, const int32_t* lists, const int32_t* ldist, int32_t* out_ids,
                            int32_t* out_dist, int32_t* trace_cand, cudaStream_t st);

}  // namespace v3db

// scan_lm_tc.cuh -- arguments of the tcgen05 list-major scan kernel (scan_lm_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "v3db_internal.cuh"

namespace v3db {

struct LmTcArgs {
  const int8_t* queries;
  int dim, kp, M, Ks, d, L, nlist, nchunk, stages, na, cb_in_smem;
  int q_vec, codes_vec, p_vec;  // 16-byte cp.async allowed for query rows / codes / P rows
  const int8_t* cb;
  const uint8_t* codes;
  const int32_t* pterm;
  const int32_t* counts;
  const int4* pairs;      // (query, rank, d_i, tau_q), grouped by list
  const int4* items;      // [n_items] (list, first pair, npairs, count of the list)
  const int* n_items;     // device scalar
  uint64_t* cand_buf;     // [Q][cap] candidates (D << 32 | list * L + slot)
  int* cand_cnt;          // [Q]
  int cap;
  int emit;
  int32_t* dst;           // rows of D: dst + (q * dst_nprobe + rank) * L, or null
  int dst_nprobe;
  int vec_store;          // 16-byte row stores allowed (L % 4 == 0, dst aligned)
  int dbg;                // performance experiments only (V3DB_LM_DEBUG): 1 no trace, 2 no decode, 4 no emission,
                          // 8 record per-step clock64 timestamps of CTA 0 into dbg_buf
  long long* dbg_buf;
};

// Fills the shape fields of `a` and the dynamic shared memory size; false if the shape
// does not fit the kernel's shared-memory budget.
bool lm_tc_config(const v3db_snapshot* s, LmTcArgs* a, size_t* smem_bytes);
cudaError_t launch_lm_tc(const LmTcArgs& a, size_t smem, cudaStream_t st);

}  // namespace v3db

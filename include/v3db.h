/*
 * v3db.h -- C ABI of the B200-native fixed-shape IVF-PQ query path of V3DB
 * (arxiv 2603.03065).  Implemented by libv3db.so (paper_2603_03065_b200/csrc/).
 *
 * Scope: build a fixed-shape IVF-PQ snapshot from a database
 * ("Index shaping", §4.1, snapshot contents
 * PAPER.md:331-340), then run the five-step query semantics (§4.2)
 * on a batch of queries, returning the top-k items plus the witness trace that the
 * multiset-based prover consumes (§4.7).  The commitment `com`
 * is out of scope: the opaque snapshot handle stands in for it.
 *
 * Arithmetic: int8 inputs, exact integer distances (int32 results).  Every distance of
 * every config fits in int32 (bounds in DESIGN.md), so results are bit-identical to the
 * paper's field arithmetic with range bounds.
 *
 * Conventions for every entry point:
 *   - Return value: v3db_status (0 == V3DB_OK).  On a non-OK status nothing is written
 *     to any output and v3db_last_error() returns a thread-local message.
 *   - "DEVICE" pointers are CUDA device pointers on the current device (e.g. torch CUDA
 *     tensors' data_ptr()); "HOST" pointers are CPU memory.  The caller owns every
 *     input/output buffer; the library never frees them.  The library owns a snapshot
 *     until v3db_free().
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Query work is enqueued on it asynchronously; outputs are valid after the stream
 *     synchronizes.  The library never aborts or exits; CUDA errors map to V3DB_ECUDA.
 *   - A snapshot is immutable after build, so concurrent v3db_query_batch calls on the
 *     same snapshot from different streams/threads are safe.
 *   - No CPU fallback: every query step runs in this library's CUDA kernels.
 */
#ifndef V3DB_H
#define V3DB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct v3db_snapshot* v3db_snapshot_t; /* opaque; library-owned device memory */

typedef enum v3db_status {
  V3DB_OK = 0,
  V3DB_EINVAL = 1,      /* NULL required pointer, shape/range violation, bad handle */
  V3DB_EINFEASIBLE = 2, /* n > nlist * list_cap: the capacity bound |X_i| <= n cannot hold */
  V3DB_ENOMEM = 3,      /* device or host allocation failed */
  V3DB_ECUDA = 4        /* any other CUDA error (message from cudaGetErrorString) */
} v3db_status;

/* Library limits (argument validation returns V3DB_EINVAL beyond them). */
#define V3DB_MAX_DIM 2048
#define V3DB_MAX_NPROBE 1024
#define V3DB_MAX_K 1024

/*
 * v3db_build_snapshot -- offline index shaping
 * with BASELINE.json's rules (readings R1-R8):
 *   B1 mu_i = db[centroid_rows[i]]                        ("seeded-sampled database vectors")
 *   B2 for t = 0..n-1 in order: append t to the first list, in the ranking by
 *      (dist(db[t], mu_i), i), whose count is < list_cap  (nearest list, lowest index on
 *      ties, overflow to the next-nearest list with room)
 *   B3 residual r_t = db[t] - mu_{list(t)}  (int16, not clamped)
 *   B4 C_{m,c} = saturate_[-127,127]( r_{codeword_rows[m*ks+c]}[m*d .. m*d+d) )
 *   B5 code_t[m] = argmin_c dist(r_t^{(m)}, C_{m,c}), lowest c on ties
 *   B6 list i: members in ascending t in slots 0..count_i-1, then padding slots with
 *      item -1 (validity flag f = 0) and code 0
 *
 *   db            DEVICE int8 [n][dim], row-major.  Read only during the call.
 *   n             number of vectors N_0; nlist <= n < 2^31.
 *   dim           D, 1..V3DB_MAX_DIM, multiple of m.
 *   nlist         n_list >= 1;  list_cap = n (per-list capacity) >= 1;
 *                 nlist * list_cap < 2^31.
 *   m, ks         M sub-quantizers (d = dim/m), K codewords per sub-quantizer, 1..256.
 *   centroid_rows HOST int32 [nlist], distinct, each in [0, n).
 *   codeword_rows HOST int32 [m][ks]; row m distinct, each in [0, n).
 *   stream        work is enqueued on it; the call synchronizes it before returning.
 *   out           set to the new handle only on V3DB_OK.
 * Errors: EINVAL (NULL pointer, bad shape, duplicate/out-of-range rows), EINFEASIBLE
 * (n > nlist*list_cap), ENOMEM, ECUDA.
 */
int v3db_build_snapshot(const int8_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap,
                        int32_t m, int32_t ks, const int32_t* centroid_rows,
                        const int32_t* codeword_rows, void* stream, v3db_snapshot_t* out);

/* Shaping rules for v3db_build_snapshot_ex (B2). */
#define V3DB_SHAPE_GREEDY 0    /* BASELINE.json: nearest list, overflow to the next-nearest with room  */
#define V3DB_SHAPE_REBALANCE 1 /* the paper's Alg. 1 on the nearest-centroid lists  */

/*
 * v3db_build_snapshot_ex -- v3db_build_snapshot with an explicit shaping rule:
 *   V3DB_SHAPE_GREEDY     B2 as above (what v3db_build_snapshot does);
 *   V3DB_SHAPE_REBALANCE  capacity-constrained cluster rebalancing, Alg. 1 of PAPER.md:296-325:
 *                         start from every vector's nearest list (lowest index on ties); while a
 *                         list holds more than list_cap vectors: for every vector v of an overfull
 *                         list i take t* = its nearest list with room (lowest index on ties) and
 *                         Delta = dist(v, mu_t*) - dist(v, mu_i); sort these moves by Delta (stable
 *                         over (i, v) ascending); apply each in order if i is still overfull and t*
 *                         still has room.  B3-B6 are unchanged.
 *   stats    HOST int64 [2] or NULL <- {vectors moved from their nearest list, rounds of the loop}.
 * Errors as v3db_build_snapshot, plus EINVAL for an unknown rule.
 */
int v3db_build_snapshot_ex(const int8_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap,
                           int32_t m, int32_t ks, const int32_t* centroid_rows,
                           const int32_t* codeword_rows, int32_t rule, int64_t* stats, void* stream,
                           v3db_snapshot_t* out);

/*
 * v3db_query_batch -- Steps 1-5 of PAPER.md:351-428 for nq queries, all on the GPU.
 *   Step 1 d_i = dist(q, mu_i) for every list
 *   Step 2 P(q) = the nprobe smallest (d_i, i), in that order (ties -> lower i, R9) (:362-381)
 *   Step 3 LUT_{i,m,c} = dist(C_{m,c}, (q - mu_i)^{(m)})                     (:383-390)
 *   Step 4 D_{i,j} = f_ij * sum_m LUT_{i,m,code_ij[m]} + (1 - f_ij) * d_max, d_max = 2^31-1
 *                                                                           (:392-408)
 *   Step 5 the k smallest (D, item) pairs of the N_sel = nprobe*L candidates, ascending,
 *          ties -> lower item as signed int32 (R10)                          (:410-428)
 *
 *   s               snapshot from v3db_build_snapshot.
 *   queries         DEVICE int8 [nq][dim].
 *   nq              >= 0 (0 is a no-op).
 *   nprobe          1..min(nlist, V3DB_MAX_NPROBE).
 *   k               1..min(nprobe*L, V3DB_MAX_K).
 *   out_ids         DEVICE int32 [nq][k]: items, ascending (D, item).  If fewer than k valid
 *                   candidates exist, the tail is -1 (R11).
 *   out_dist        DEVICE int32 [nq][k]: D of each returned item (d_max with item -1).
 *   trace_lists     DEVICE int32 [nq][nprobe] or NULL: P(q) in probe order.
 *   trace_list_dist DEVICE int32 [nq][nprobe] or NULL: d_i of those lists.
 *   trace_cand_dist DEVICE int32 [nq][nprobe][L] or NULL: masked D_{i,j} of every slot
 *                   of every probed list, in probe-rank then slot order (S^orig_{item,dist},
 *                   R12); items are ids[trace_lists[q][r]][j] of the snapshot.
 *   stream          asynchronous; outputs valid after the stream synchronizes.
 * Errors: EINVAL (NULL handle/required pointer, nprobe/k out of range), ENOMEM, ECUDA.
 */
int v3db_query_batch(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe,
                     int32_t k, int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists,
                     int32_t* trace_list_dist, int32_t* trace_cand_dist, void* stream);

/* Scan-kernel selection for v3db_query_batch_ex (results are bit-identical for all). */
#define V3DB_SCAN_AUTO 0       /* LIST_MAJOR where supported, else ROTATED, else GENERIC          */
#define V3DB_SCAN_GENERIC 1    /* per-query LUT [M][Ks] in shared memory, any shape               */
#define V3DB_SCAN_ROTATED 2    /* conflict-free rotated LUT (M % 4 == 0, d % 4 == 0, M <= 128)    */
#define V3DB_SCAN_LIST_MAJOR 3 /* Steps 3-4 as the exact identity d_i + P_ij - 2 <q, xhat_ij>:   */
                               /* tcgen05 int8 tiles per (list, probing queries)                 */
                               /* (dim % 16 == 0, nlist <= 32768)                                */

/* v3db_query_batch_ex -- v3db_query_batch with an explicit scan kernel (`algo`, one of
 * V3DB_SCAN_*).  EINVAL for an unknown algo, or a kernel the snapshot's shape does not
 * support.  LIST_MAJOR computes every D_{i,j} of Step 4 from the identity
 *   sum_m LUT_{i,m,code_m} = dist(q - mu_i, xhat_ij) = d_i + P_ij - 2 <q, xhat_ij>
 * (xhat_ij the slot's reconstruction; P_ij = ||xhat||^2 + 2 <mu_i, xhat>), exact
 * in int32, so every output equals the literal Steps 3-4 bit for bit; with
 * trace_cand_dist NULL it writes the candidate distances to library scratch
 * (4 * nq * nprobe * L bytes) because its Step 5 reads them back. */
int v3db_query_batch_ex(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe,
                        int32_t k, int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists,
                        int32_t* trace_list_dist, int32_t* trace_cand_dist, int32_t algo,
                        void* stream);

/*
 * v3db_query_batch_host -- the same computation with HOST buffers (end-to-end entry):
 * copies queries host->device, runs v3db_query_batch on `stream` with library-owned
 * device buffers, copies the requested outputs device->host, and synchronizes the stream
 * before returning.  Pointers have the layouts of v3db_query_batch but are HOST memory
 * (pinned memory makes the copies asynchronous DMA).  trace pointers may be NULL.
 */
int v3db_query_batch_host(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe,
                          int32_t k, int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists,
                          int32_t* trace_list_dist, int32_t* trace_cand_dist, void* stream);

/*
 * v3db_witness_batch -- the prover witness of nq (challenged) queries: the values the
 * multiset-based design takes from the off-circuit run of Steps 1-5 (§4.7,
 * PAPER.md:614-657).  Per query, all in DEVICE memory, any may be NULL:
 *   list_order [nq][nlist], list_dist [nq][nlist]   S^sorted_{idx,dist}: every list i with its
 *                          d_i = dist(q, mu_i), ascending (d_i, i) (R9); the first
 *                          nprobe are P(q) (equal to v3db_query_batch's trace_lists)
 *   lut_sel [nq][nprobe][L][M]   l^{(m)}_{i,j} = LUT_{i,m,v^{(m)}_{i,j}}: the literal Step-3 entry
 *                           selected by each probed slot's code, padding slots
 *                          included (code 0)
 *   cand_items [nq][nprobe*L], cand_dist [nq][nprobe*L]   S^sorted_{item,dist}: all N_sel
 *                          candidates (item, D) ascending (D, item) (R10); the
 *                          first k are v3db_query_batch's out_ids / out_dist
 * nq in [0, 65535].  Asynchronous on `stream`.  Errors: EINVAL (NULL handle/queries, nq or nprobe out
 * of range), ENOMEM, ECUDA.  Not on the query hot path (on demand, a few MB per query).
 */
int v3db_witness_batch(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe,
                       int32_t* list_order, int32_t* list_dist, int32_t* lut_sel, int32_t* cand_items,
                       int32_t* cand_dist, void* stream);

/* ---- NEXT-1: the paper's 16-bit fixed-point representation ----
 * PAPER.md:781-782 (§5 setup): v_max, the maximum absolute coordinate over all involved vectors,
 * is rescaled to 2^16 - 1 and each coordinate v is encoded as the nearest integer to
 * (2^16 - 1) v / v_max (the paper's round-to-nearest bracket).  Readings (R18, R19):
 * coordinates become int32 values in [-65535, 65535] (the sign kept, exact ties rounded away from
 * zero, computed in IEEE double as (v * 65535) / v_max, the fraction compared exactly with 1/2);
 * every distance is the exact squared L2 in int64 and d_max = 2^63 - 1;
 * codewords are the residual sub-vectors themselves (int32, no saturation).  The five steps and
 * the build rules are those of the int8 path with this arithmetic; shaping is the greedy rule. */

/* v3db_encode_fixed_point -- out[i] = round_half_away(x[i] * 65535 / v_max), DEVICE float32 x
 * [count] -> DEVICE int32 out [count].  Asynchronous on `stream`.  EINVAL: NULL pointer with
 * count > 0, count < 0, v_max not positive finite.  |x| <= v_max keeps |out| <= 65535. */
int v3db_encode_fixed_point(const float* x, int64_t count, double v_max, int32_t* out, void* stream);

/* v3db_build_snapshot_fx -- v3db_build_snapshot on an int32 DEVICE database [n][dim] whose
 * coordinates lie in [-65535, 65535] (EINVAL otherwise).  Same validation, ownership and errors
 * as v3db_build_snapshot, plus EINVAL when nlist exceeds the composite-key bound at this dim
 * (2^(64 - bits(dim * 131070^2)), 2^20 at dim 768).  Synchronous. */
int v3db_build_snapshot_fx(const int32_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap,
                           int32_t m, int32_t ks, const int32_t* centroid_rows,
                           const int32_t* codeword_rows, void* stream, v3db_snapshot_t* out);

/* v3db_query_batch_fx -- Steps 1-5 on a fixed-point snapshot: int32 DEVICE queries [nq][dim] in
 * [-65535, 65535]; out_ids int32 [nq][k]; out_dist, trace_list_dist, trace_cand_dist int64 with
 * the layouts of v3db_query_batch (padding / missing entries: id -1, distance 2^63 - 1).  EINVAL
 * as v3db_query_batch, for an int8 snapshot, out-of-range queries, or nprobe * list_cap above the
 * Step-5 key bound (2^(64 - bits(dim * 262140^2))); ENOMEM, ECUDA.  Ties at the k-th distance are
 * resolved exactly by item id however many there are.  The range check of the queries reads one
 * word back, so the call returns after that check (the kernels stay asynchronous on `stream`). */
int v3db_query_batch_fx(v3db_snapshot_t s, const int32_t* queries, int64_t nq, int32_t nprobe,
                        int32_t k, int32_t* out_ids, int64_t* out_dist, int32_t* trace_lists,
                        int64_t* trace_list_dist, int64_t* trace_cand_dist, void* stream);

/* v3db_query_batch_fx_host -- the end-to-end fixed-point entry: HOST float32 queries [nq][dim]
 * copied host->device, encoded with v_max (v3db_encode_fixed_point), v3db_query_batch_fx with
 * library-owned device buffers, the requested outputs copied device->host (layouts and types of
 * v3db_query_batch_fx, HOST memory; pinned memory makes the copies asynchronous DMA); synchronizes
 * `stream` before returning.  trace pointers may be NULL.  Errors as v3db_query_batch_fx, plus
 * EINVAL for v_max not positive finite. */
int v3db_query_batch_fx_host(v3db_snapshot_t s, const float* queries, int64_t nq, double v_max,
                             int32_t nprobe, int32_t k, int32_t* out_ids, int64_t* out_dist,
                             int32_t* trace_lists, int64_t* trace_list_dist, int64_t* trace_cand_dist,
                             void* stream);

/* v3db_snapshot_kind -- V3DB_KIND_INT8 or V3DB_KIND_FX16 (negative status on a NULL handle).
 * v3db_query_batch* / v3db_witness_batch reject FX16 snapshots, v3db_query_batch_fx INT8 ones;
 * v3db_snapshot_export returns int32 CENTROIDS / CODEBOOKS for FX16 snapshots. */
#define V3DB_KIND_INT8 0
#define V3DB_KIND_FX16 1
int v3db_snapshot_kind(v3db_snapshot_t s);

/* v3db_free -- release a snapshot.  NULL-safe.  The caller must not free a snapshot with
 * query work still in flight on any stream. */
void v3db_free(v3db_snapshot_t s);

/* v3db_snapshot_info -- HOST int64 [8] <- {n, dim, nlist, list_cap, m, ks, d, total_valid}. */
int v3db_snapshot_info(v3db_snapshot_t s, int64_t* out8);

/* Field ids for v3db_snapshot_export. */
#define V3DB_FIELD_CENTROIDS 0 /* int8  [nlist][dim]        mu                          */
#define V3DB_FIELD_CODEBOOKS 1 /* int8  [m][ks][d]          C_{m,c}                     */
#define V3DB_FIELD_IDS 2       /* int32 [nlist][list_cap]   item_{i,j}, -1 = padding     */
#define V3DB_FIELD_CODES 3     /* uint8 [nlist][list_cap][m] v^PQ_{i,j}                  */
#define V3DB_FIELD_COUNTS 4    /* int32 [nlist]             valid slots per list         */
#define V3DB_FIELD_LIST_OF 5   /* int32 [n]                 final list of every vector   */

/* v3db_snapshot_export -- test-only introspection (never on the timed path): copy one
 * canonical snapshot array into HOST memory.  `bytes` must equal the field's exact size.
 * Synchronous.  EINVAL for an unknown field or a size mismatch. */
int v3db_snapshot_export(v3db_snapshot_t s, int32_t field, void* host_dst, size_t bytes);

/* Profiling hooks (used by bench.py; off by default, never change results).
 * v3db_profile_enable(1) makes every v3db_query_batch* call record CUDA events on its
 * stream around each kernel; v3db_profile_read waits for the most recent call's events and
 * writes up to n (<= 5) elapsed times in milliseconds: [0] Steps 1-2 (coarse top-nprobe
 * kernels), [1] Steps 3-5 (everything after Steps 1-2), [2] the scan's main kernel alone (the
 * list-major contraction / the rotated or generic scan), [3] the scan's prologue (pair grouping or
 * L2-aware query order), [4] the scan's epilogue (list-major Step-5 selection; 0 for the
 * query-major scans, whose kernel includes Step 5).  Not thread-safe: profile one
 * stream at a time.  v3db_kernel_launches returns the number of kernels this library has
 * launched since load (all entry points). */
int v3db_profile_enable(int32_t on);
int v3db_profile_read(float* out_ms, int32_t n);
int64_t v3db_kernel_launches(void);

/* v3db_set_option / v3db_get_option -- process-wide implementation choices (never change a
 * result: every choice is exact; tests use them to reach every code path, bench/tools to
 * measure alternatives).  0 is the default everywhere.  Set them between calls, not while
 * work is being enqueued from another thread.  EINVAL for an unknown key.
 *   V3DB_OPT_LUT_W32      1: the W32 rotated table even where P64 applies (read at build)
 *   V3DB_OPT_COARSE_SIMT  1: Steps 1-2 / build ranking on the mma.sync kernel (not tcgen05)
 *   V3DB_OPT_SCHED        L2-aware query order of the query-major scans: 0 auto, 1 on, 2 off
 *   V3DB_OPT_FX_NOROT     1: no rotated fixed-point code copy (read at fx16 build)
 *   V3DB_OPT_FX_W12       fx16 scan warps per CTA (0 = auto)
 *   V3DB_OPT_SCAN_SEG / _NS / _CAP / _FIRST / _DIRECT   rotated-LUT scan geometry (0 = auto)
 *   V3DB_OPT_LM_NT        list-major scan: (query, rank) pairs per work item, 32/64/128/256
 *                         (0 = auto: the largest whose B operand fits)
 *   V3DB_OPT_AUTO_SCAN    the kernel V3DB_SCAN_AUTO picks where several apply (0 = list-major,
 *                         else one of the V3DB_SCAN_* values)
 *   V3DB_OPT_COARSE_2PASS Steps 1-2 on the tensor cores: 0 auto (one contraction pass keeping
 *                         the two smallest keys of every block of 32 lists, then an exact merge that
 *                         recomputes the blocks that may hide more -- dim <= 1024; otherwise the
 *                         group-minimum pass below), 1 the group-minimum pass then a second
 *                         contraction pass, 4 / 8 / 16 / 32 the group-minimum pass then the
 *                         recomputation of the selected groups of at most that many lists
 *   V3DB_OPT_SELECT_CTA   list-major Step 5: 0 auto (one warp per query when the probed lists
 *                         hold >= 8 k groups of 32 slots, else one CTA per query), 1 always one
 *                         CTA of 256 threads per query, 2 always one warp per query (all exact;
 *                         the streaming CTA path takes the queries they flag)
 *   V3DB_OPT_FX_COARSE    fixed-point Steps 1-2 / build ranking: 0 auto (tensor cores: three int8
 *                         limbs per coordinate, where dim % 16 == 0 and dim <= 256), 1 always the
 *                         FP64-FMA kernel (exact below 2^53)
 *   V3DB_OPT_FX_SCAN      fixed-point Steps 3-5: 0 auto (list-major on the tensor cores, int8 limbs,
 *                         where the snapshot holds the limb planes: dim % 16 == 0, dim <= 256,
 *                         nlist <= 32768), 1 always the literal per-query int64 LUT scan
 *   V3DB_OPT_COARSE_KEYS  keys kept per 32-list block by the single-pass Steps 1-2: 0 auto (the
 *                         smallest of 2 / 4 / 8 that is >= nprobe where nprobe <= 8 -- nlist <= 16384
 *                         for 8 -- so that the kept keys hold the whole top nprobe and no block is
 *                         recomputed; otherwise 2 for dim <= 256, 4 above, where recomputing a block
 *                         in the merge is expensive), 2, 4 or 8 (8 only where nprobe <= 8)
 *   V3DB_OPT_LM_STATIC    list-major scans (int8 and fixed point): 0 the CTAs of the main kernel
 *                         draw their work items from a grid-wide counter (a CTA takes its next item
 *                         when it is ready for one), 1 the static round-robin deal (item j to CTA
 *                         j mod grid) */
#define V3DB_OPT_LUT_W32 0
#define V3DB_OPT_COARSE_SIMT 1
#define V3DB_OPT_SCHED 2
#define V3DB_OPT_FX_NOROT 3
#define V3DB_OPT_FX_W12 4
#define V3DB_OPT_SCAN_SEG 5
#define V3DB_OPT_SCAN_NS 6
#define V3DB_OPT_SCAN_CAP 7
#define V3DB_OPT_SCAN_FIRST 8
#define V3DB_OPT_SCAN_DIRECT 9
#define V3DB_OPT_LM_NT 10
#define V3DB_OPT_AUTO_SCAN 11
#define V3DB_OPT_COARSE_2PASS 12
#define V3DB_OPT_SELECT_CTA 13
#define V3DB_OPT_FX_COARSE 14
#define V3DB_OPT_FX_SCAN 15
#define V3DB_OPT_COARSE_KEYS 16
#define V3DB_OPT_LM_STATIC 17
#define V3DB_OPT_COUNT 18
int v3db_set_option(int32_t key, int64_t value);
int64_t v3db_get_option(int32_t key);

/* v3db_last_error -- thread-local message for the last non-OK status on this thread
 * ("" if none).  The pointer stays valid until the next call on the same thread. */
const char* v3db_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* V3DB_H */

// v3db_api.cu -- the C ABI declared in include/v3db.h: argument validation, snapshot
// ownership, the host side of the build (the ordered greedy placement B2), and the
// stream-ordered launch sequence of the query path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <mutex>
#include <stdlib.h>
#include <string>
#include <unordered_set>
#include <vector>

#include "v3db_internal.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? V3DB_ENOMEM : V3DB_ECUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define V3DB_CUDA(call)                               \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// Device buffer owned by the host code of one call.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t count) { return cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * (count ? count : 1)); }
};

template <typename T>
struct HostPinned {
  T* p = nullptr;
  ~HostPinned() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t alloc(size_t count) { return cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(T) * (count ? count : 1)); }
};

void free_snapshot(v3db_snapshot* s) {
  if (!s) return;
  cudaFree(s->centroids);
  cudaFree(s->cnorm);
  cudaFree(s->codebooks);
  cudaFree(s->ids);
  cudaFree(s->codes);
  cudaFree(s->counts);
  cudaFree(s->pterm);
  cudaFree(s->list_of);
  cudaFree(s->codes_rot);
  cudaFree(s->pterm_rot);
  cudaFree(s->cbT);
  cudaFree(s->centroids32);
  cudaFree(s->cnorm64);
  cudaFree(s->codebooks32);
  cudaFree(s->pterm64);
  cudaFree(s->codes_rot16);
  cudaFree(s->xhat_fx);
  cudaFree(s->xhat);
  delete s;
}

int check_device(const v3db_snapshot* s) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != s->device)
    return fail(V3DB_EINVAL, "snapshot belongs to CUDA device " + std::to_string(s->device) +
                                 " but the current device is " + std::to_string(dev));
  return V3DB_OK;
}

// Profiling state (v3db_profile_*): events around each query kernel on the call's stream.
// Marks: 0 call start, 1 after Steps 1-2, 2 after the scan's prologue (grouping / query order),
// 3 after the scan's main kernel, 4 call end (after the selection).
struct Profiler {
  std::mutex mu;
  bool on = false;
  bool created = false;
  bool recorded = false;
  int marked = 0;  // bit i: mark i recorded in the current call
  cudaEvent_t ev[5];
};
Profiler g_prof;
std::atomic<int64_t> g_launches{0};

void prof_record(int i, cudaStream_t st) {
  if (!g_prof.on) return;
  if (i == 0) g_prof.marked = 0;
  cudaEventRecord(g_prof.ev[i], st);
  g_prof.marked |= 1 << i;
  if (i == 4) g_prof.recorded = true;
}
// around a scan implementation that may record marks 2 and 3 itself
void prof_scan_begin(cudaStream_t st) {
  prof_record(1, st);
  prof_record(2, st);
}
void prof_scan_end(cudaStream_t st) {
  if (g_prof.on && !(g_prof.marked & 8)) prof_record(3, st);
  prof_record(4, st);
}

}  // namespace

namespace v3db {
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

std::atomic<int64_t> g_opts[V3DB_OPT_COUNT];
int64_t opt(int key) { return g_opts[key].load(std::memory_order_relaxed); }

#ifdef V3DB_DEBUG
// Debug build only (libv3db_debug.so): V3DB_SYNC_CHECK=1 synchronizes after each launch group
// and reports the first error tagged with the kernel name.
cudaError_t debug_sync(cudaStream_t st, const char* what) {
  static const bool on = [] {
    const char* e = getenv("V3DB_SYNC_CHECK");
    return e && e[0] == '1';
  }();
  if (!on) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) g_err = std::string("after ") + what + ": " + cudaGetErrorString(e);
  return e;
}
#else
cudaError_t debug_sync(cudaStream_t, const char*) { return cudaSuccess; }
#endif

// The library's own stream-ordered pool per device (query scratch): freed blocks stay in it
// instead of going back to the driver at every synchronization, without touching the device's
// default pool that the application (torch) may configure.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) {
        pools[dev] = nullptr;
        return e;
      }
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, st);
}
}  // namespace v3db

int v3db_set_option(int32_t key, int64_t value) {
  g_err.clear();
  if (key < 0 || key >= V3DB_OPT_COUNT) return fail(V3DB_EINVAL, "unknown option key");
  v3db::g_opts[key].store(value, std::memory_order_relaxed);
  return V3DB_OK;
}

int64_t v3db_get_option(int32_t key) {
  if (key < 0 || key >= V3DB_OPT_COUNT) return 0;
  return v3db::opt(key);
}

// B2, the ordered greedy placement (BASELINE.json configs[0]): every vector, in ascending t, goes
// to the nearest list with room.  rank(lo, rows, R, d_idx, d_dist) writes each row's R nearest lists
// (ascending (e, i)) on the GPU; when all R are full, exact(t, e) gives e_t,i for every list.
template <class RankFn, class ExactFn>
int place_greedy(int64_t n, int nlist, int L, RankFn rank, ExactFn exact, size_t dist_bytes, cudaStream_t st,
                 std::vector<int32_t>& list_of, std::vector<int32_t>& flat_pos, std::vector<int32_t>& counts) {
  const int R = std::min(nlist, 64);
  const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 18);
  DevBuf<int32_t> d_rank;
  DevBuf<uint8_t> d_rdist;
  HostPinned<int32_t> h_rank;
  V3DB_CUDA(d_rank.alloc(static_cast<size_t>(chunk) * R));
  V3DB_CUDA(d_rdist.alloc(static_cast<size_t>(chunk) * R * dist_bytes));
  V3DB_CUDA(h_rank.alloc(static_cast<size_t>(chunk) * R));
  std::vector<int64_t> e;
  for (int64_t lo = 0; lo < n; lo += chunk) {
    const int64_t rows = std::min(chunk, n - lo);
    V3DB_CUDA(rank(lo, rows, R, d_rank.p, static_cast<void*>(d_rdist.p)));
    V3DB_CUDA(cudaMemcpyAsync(h_rank.p, d_rank.p, sizeof(int32_t) * rows * R, cudaMemcpyDeviceToHost, st));
    V3DB_CUDA(cudaStreamSynchronize(st));
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t t = lo + r;
      int chosen = -1;
      const int32_t* rk = h_rank.p + r * R;
      for (int a = 0; a < R; ++a) {
        if (counts[rk[a]] < L) {
          chosen = rk[a];
          break;
        }
      }
      if (chosen < 0) {  // all R nearest lists are full: exact full ranking on the host
        e.resize(nlist);
        V3DB_CUDA(exact(t, e));
        int64_t best = INT64_MAX;
        for (int i = 0; i < nlist; ++i) {
          if (counts[i] < L && e[i] < best) {  // strict: lowest index on ties
            best = e[i];
            chosen = i;
          }
        }
        if (chosen < 0) return fail(V3DB_EINFEASIBLE, "no list with room (internal)");
      }
      list_of[t] = chosen;
      flat_pos[t] = chosen * L + counts[chosen];  // B6: members in ascending t
      ++counts[chosen];
    }
  }
  return V3DB_OK;
}

// Alg. 1 (capacity-constrained rebalancing) on the nearest-centroid assignment;
// readings R17: t* ties -> lowest list, M sorted stably by Delta over (cluster, vector)
// construction order.  GPU: nearest lists, t* over the free lists (the coarse top-1 kernel against
// the gathered free centroids), Delta, the sort; host: the guarded sequential apply.
int place_rebalance(const int8_t* db, int64_t n, int dim, int nlist, int L, const int8_t* mu, const int32_t* cnorm,
                    cudaStream_t st, std::vector<int32_t>& list_of, std::vector<int32_t>& counts, int64_t* moved,
                    int64_t* rounds) {
  const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 20);
  {
    DevBuf<int32_t> d_idx, d_dist;
    V3DB_CUDA(d_idx.alloc(chunk));
    V3DB_CUDA(d_dist.alloc(chunk));
    for (int64_t lo = 0; lo < n; lo += chunk) {
      const int64_t rows = std::min(chunk, n - lo);
      V3DB_CUDA(v3db::coarse_topk(db + lo * dim, rows, dim, mu, cnorm, nlist, 1, d_idx.p, d_dist.p, st));
      V3DB_CUDA(cudaMemcpyAsync(list_of.data() + lo, d_idx.p, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost, st));
    }
    V3DB_CUDA(cudaStreamSynchronize(st));
  }
  const std::vector<int32_t> init = list_of;
  std::fill(counts.begin(), counts.end(), 0);
  for (int64_t t = 0; t < n; ++t) ++counts[list_of[t]];
  *rounds = 0;
  for (;;) {
    std::vector<int32_t> F;
    std::vector<char> over(nlist, 0);
    bool any = false;
    for (int i = 0; i < nlist; ++i) {
      if (counts[i] > L) over[i] = 1, any = true;
      if (counts[i] < L) F.push_back(i);
    }
    if (!any) break;
    if (F.empty()) return fail(V3DB_EINFEASIBLE, "no free list (internal)");
    ++*rounds;
    // M in (cluster ascending, vector ascending) order: counting sort of the overfull members
    std::vector<int64_t> start(nlist + 1, 0);
    for (int64_t t = 0; t < n; ++t)
      if (over[list_of[t]]) ++start[list_of[t] + 1];
    for (int i = 0; i < nlist; ++i) start[i + 1] += start[i];
    const int64_t mm = start[nlist];
    std::vector<int32_t> vs(mm), src(mm);
    for (int64_t t = 0; t < n; ++t) {
      const int32_t i = list_of[t];
      if (over[i]) {
        vs[start[i]] = static_cast<int32_t>(t);
        src[start[i]++] = i;
      }
    }
    int64_t P = 1;
    while (P < mm) P <<= 1;
    if (P > (int64_t(1) << 30)) return fail(V3DB_EINVAL, "Alg. 1: more than 2^30 candidate moves in one round");
    DevBuf<int32_t> d_F, d_cnF, d_vs, d_src, d_tpos, d_et, d_ei;
    DevBuf<int8_t> d_muF, d_X;
    DevBuf<uint64_t> d_keys;
    const int nf = static_cast<int>(F.size());
    V3DB_CUDA(d_F.alloc(nf));
    V3DB_CUDA(d_cnF.alloc(nf));
    V3DB_CUDA(d_muF.alloc(static_cast<size_t>(nf) * dim));
    V3DB_CUDA(d_vs.alloc(mm));
    V3DB_CUDA(d_src.alloc(mm));
    V3DB_CUDA(d_tpos.alloc(mm));
    V3DB_CUDA(d_et.alloc(mm));
    V3DB_CUDA(d_ei.alloc(mm));
    V3DB_CUDA(d_X.alloc(static_cast<size_t>(mm) * dim));
    V3DB_CUDA(d_keys.alloc(P));
    V3DB_CUDA(cudaMemcpyAsync(d_F.p, F.data(), sizeof(int32_t) * nf, cudaMemcpyHostToDevice, st));
    V3DB_CUDA(cudaMemcpyAsync(d_vs.p, vs.data(), sizeof(int32_t) * mm, cudaMemcpyHostToDevice, st));
    V3DB_CUDA(cudaMemcpyAsync(d_src.p, src.data(), sizeof(int32_t) * mm, cudaMemcpyHostToDevice, st));
    V3DB_CUDA(v3db::gather_rows(mu, dim, d_F.p, nf, d_muF.p, d_cnF.p, st));       // free centroids
    V3DB_CUDA(v3db::gather_rows(db, dim, d_vs.p, static_cast<int>(mm), d_X.p, nullptr, st));  // candidate vectors
    V3DB_CUDA(v3db::pair_dist(d_X.p, mm, dim, mu, d_src.p, d_ei.p, st));           // ||v - mu_i||^2
    V3DB_CUDA(v3db::coarse_topk(d_X.p, mm, dim, d_muF.p, d_cnF.p, nf, 1, d_tpos.p, d_et.p, st));  // t*, ||v - mu_t*||^2
    V3DB_CUDA(v3db::delta_keys(d_et.p, d_ei.p, mm, P, d_keys.p, st));
    V3DB_CUDA(v3db::segmented_sort(d_keys.p, 1, static_cast<int>(P), st));       // sort M by (Delta, position)
    std::vector<uint64_t> keys(mm);
    std::vector<int32_t> tpos(mm);
    V3DB_CUDA(cudaMemcpyAsync(keys.data(), d_keys.p, sizeof(uint64_t) * mm, cudaMemcpyDeviceToHost, st));
    V3DB_CUDA(cudaMemcpyAsync(tpos.data(), d_tpos.p, sizeof(int32_t) * mm, cudaMemcpyDeviceToHost, st));
    V3DB_CUDA(cudaStreamSynchronize(st));
    for (int64_t a = 0; a < mm; ++a) {  // the guarded moves, in order
      const int64_t r = static_cast<int64_t>(keys[a] & 0xffffffffu);
      const int32_t v = vs[r], i = src[r], t = F[tpos[r]];
      if (counts[i] > L && counts[t] < L && list_of[v] == i) {
        list_of[v] = t;
        --counts[i];
        ++counts[t];
      }
    }
  }
  *moved = 0;
  for (int64_t t = 0; t < n; ++t) *moved += list_of[t] != init[t];
  return V3DB_OK;
}

extern "C" {

int v3db_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_err.clear();
  if (on && !g_prof.created) {
    for (auto& e : g_prof.ev) V3DB_CUDA(cudaEventCreate(&e));
    g_prof.created = true;
  }
  g_prof.on = on != 0;
  g_prof.recorded = false;
  return V3DB_OK;
}

int v3db_profile_read(float* out_ms, int32_t n) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_err.clear();
  if (!out_ms || n < 0) return fail(V3DB_EINVAL, "NULL pointer");
  if (!g_prof.recorded) return fail(V3DB_EINVAL, "no profiled query call recorded");
  V3DB_CUDA(cudaEventSynchronize(g_prof.ev[4]));
  static const int span[5][2] = {{0, 1}, {1, 4}, {2, 3}, {1, 2}, {3, 4}};
  for (int i = 0; i < n && i < 5; ++i) V3DB_CUDA(cudaEventElapsedTime(&out_ms[i], g_prof.ev[span[i][0]], g_prof.ev[span[i][1]]));
  return V3DB_OK;
}

int64_t v3db_kernel_launches(void) { return g_launches.load(); }

const char* v3db_last_error(void) { return g_err.c_str(); }

void v3db_free(v3db_snapshot_t s) { free_snapshot(s); }

static int validate_build(int64_t n, int32_t dim, int32_t nlist, int32_t list_cap, int32_t m, int32_t ks,
                          const int32_t* centroid_rows, const int32_t* codeword_rows, v3db_snapshot_t* out) {
  if (!centroid_rows || !codeword_rows || !out) return fail(V3DB_EINVAL, "NULL required pointer");
  if (dim < 1 || dim > V3DB_MAX_DIM) return fail(V3DB_EINVAL, "dim out of range [1, V3DB_MAX_DIM]");
  if (m < 1 || dim % m) return fail(V3DB_EINVAL, "dim must be a positive multiple of m (D = Md, PAPER.md:331)");
  if (dim / m > 64) return fail(V3DB_EINVAL, "sub-block dimension d = dim/m > 64 is not supported");
  if (ks < 1 || ks > 256) return fail(V3DB_EINVAL, "ks out of range [1, 256]");
  if (static_cast<int64_t>(m) * ks > 32768) return fail(V3DB_EINVAL, "m * ks > 32768 (per-query LUT > 128 KiB)");
  if (nlist < 1 || list_cap < 1) return fail(V3DB_EINVAL, "nlist and list_cap must be >= 1");
  if (static_cast<int64_t>(nlist) * list_cap >= (int64_t(1) << 31)) return fail(V3DB_EINVAL, "nlist * list_cap >= 2^31");
  if (n < nlist || n >= (int64_t(1) << 31)) return fail(V3DB_EINVAL, "n must satisfy nlist <= n < 2^31");
  if (n > static_cast<int64_t>(nlist) * list_cap)
    return fail(V3DB_EINFEASIBLE, "n > nlist * list_cap: capacity bound |X_i| <= n cannot hold (PAPER.md:290)");
  {
    std::unordered_set<int32_t> seen;
    for (int i = 0; i < nlist; ++i) {
      if (centroid_rows[i] < 0 || centroid_rows[i] >= n || !seen.insert(centroid_rows[i]).second)
        return fail(V3DB_EINVAL, "centroid_rows must be nlist distinct rows in [0, n)");
    }
    for (int mm = 0; mm < m; ++mm) {
      seen.clear();
      for (int c = 0; c < ks; ++c) {
        const int32_t r = codeword_rows[mm * ks + c];
        if (r < 0 || r >= n || !seen.insert(r).second)
          return fail(V3DB_EINVAL, "codeword_rows[m] must be ks distinct rows in [0, n)");
      }
    }
  }
  return V3DB_OK;
}

int v3db_build_snapshot(const int8_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap, int32_t m,
                        int32_t ks, const int32_t* centroid_rows, const int32_t* codeword_rows, void* stream,
                        v3db_snapshot_t* out) {
  return v3db_build_snapshot_ex(db, n, dim, nlist, list_cap, m, ks, centroid_rows, codeword_rows, V3DB_SHAPE_GREEDY,
                                nullptr, stream, out);
}

int v3db_build_snapshot_ex(const int8_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap, int32_t m,
                           int32_t ks, const int32_t* centroid_rows, const int32_t* codeword_rows, int32_t rule,
                           int64_t* stats, void* stream, v3db_snapshot_t* out) {
  g_err.clear();
  if (rule != V3DB_SHAPE_GREEDY && rule != V3DB_SHAPE_REBALANCE) return fail(V3DB_EINVAL, "unknown shaping rule");
  if (!db) return fail(V3DB_EINVAL, "NULL required pointer");
  int vrc = validate_build(n, dim, nlist, list_cap, m, ks, centroid_rows, codeword_rows, out);
  if (vrc != V3DB_OK) return vrc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int d = dim / m;
  const int L = list_cap;

  v3db_snapshot* s = new (std::nothrow) v3db_snapshot();
  if (!s) return fail(V3DB_ENOMEM, "host allocation failed");
  struct Guard {
    v3db_snapshot* s;
    ~Guard() { free_snapshot(s); }
  } guard{s};
  s->n = n;
  s->dim = dim;
  s->nlist = nlist;
  s->L = L;
  s->M = m;
  s->Ks = ks;
  s->d = d;
  V3DB_CUDA(cudaGetDevice(&s->device));
  const int64_t slots = static_cast<int64_t>(nlist) * L;
  V3DB_CUDA(cudaMalloc(&s->centroids, static_cast<size_t>(nlist) * dim));
  V3DB_CUDA(cudaMalloc(&s->cnorm, sizeof(int32_t) * nlist));
  V3DB_CUDA(cudaMalloc(&s->codebooks, static_cast<size_t>(m) * ks * d));
  V3DB_CUDA(cudaMalloc(&s->ids, sizeof(int32_t) * slots));
  V3DB_CUDA(cudaMalloc(&s->codes, static_cast<size_t>(slots) * m));
  V3DB_CUDA(cudaMalloc(&s->counts, sizeof(int32_t) * nlist));
  V3DB_CUDA(cudaMalloc(&s->pterm, sizeof(int32_t) * slots));
  V3DB_CUDA(cudaMalloc(&s->list_of, sizeof(int32_t) * n));

  // B1: centroids and their squared norms.
  DevBuf<int32_t> d_rows;
  V3DB_CUDA(d_rows.alloc(nlist));
  V3DB_CUDA(cudaMemcpyAsync(d_rows.p, centroid_rows, sizeof(int32_t) * nlist, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(v3db::gather_rows(db, dim, d_rows.p, nlist, s->centroids, s->cnorm, st));

  std::vector<int32_t> list_of(n), flat_pos(n), counts(nlist, 0);
  int64_t moved = 0, rounds = 0;
  if (rule == V3DB_SHAPE_GREEDY) {
    // B2: GPU ranks each vector's R nearest lists by (e, i); host places in ascending t.
    std::vector<int8_t> mu_host;
    std::vector<int8_t> row(dim);
    int rc = place_greedy(
        n, nlist, L,
        [&](int64_t lo, int64_t rows, int R, int32_t* d_rank, void* d_rdist) {
          return v3db::coarse_topk(db + lo * dim, rows, dim, s->centroids, s->cnorm, nlist, R, d_rank,
                                   static_cast<int32_t*>(d_rdist), st);
        },
        [&](int64_t t, std::vector<int64_t>& e) -> cudaError_t {  // exact e_t,i for every list (host)
          cudaError_t ce = cudaSuccess;
          if (mu_host.empty()) {
            mu_host.resize(static_cast<size_t>(nlist) * dim);
            ce = cudaMemcpy(mu_host.data(), s->centroids, mu_host.size(), cudaMemcpyDeviceToHost);
          }
          if (ce == cudaSuccess) ce = cudaMemcpy(row.data(), db + t * dim, dim, cudaMemcpyDeviceToHost);
          for (int i = 0; i < nlist && ce == cudaSuccess; ++i) {
            int64_t acc = 0;
            for (int u = 0; u < dim; ++u) {
              const int64_t df = int64_t(row[u]) - int64_t(mu_host[static_cast<size_t>(i) * dim + u]);
              acc += df * df;
            }
            e[i] = acc;
          }
          return ce;
        },
        sizeof(int32_t), st, list_of, flat_pos, counts);
    if (rc != V3DB_OK) return rc;

  } else {
    int rc = place_rebalance(db, n, dim, nlist, L, s->centroids, s->cnorm, st, list_of, counts, &moved, &rounds);
    if (rc != V3DB_OK) return rc;
    std::fill(counts.begin(), counts.end(), 0);
    for (int64_t t = 0; t < n; ++t) {  // B6: members in ascending t
      const int32_t i = list_of[t];
      flat_pos[t] = i * L + counts[i]++;
    }
  }
  if (stats) {
    stats[0] = moved;
    stats[1] = rounds;
  }

  // B3-B6 on the GPU.
  DevBuf<int32_t> d_pos, d_cwrows;
  V3DB_CUDA(d_pos.alloc(n));
  V3DB_CUDA(d_cwrows.alloc(static_cast<size_t>(m) * ks));
  V3DB_CUDA(cudaMemcpyAsync(s->list_of, list_of.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(d_pos.p, flat_pos.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(d_cwrows.p, codeword_rows, sizeof(int32_t) * m * ks, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(s->counts, counts.data(), sizeof(int32_t) * nlist, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemsetAsync(s->ids, 0xff, sizeof(int32_t) * slots, st));  // padding item -1 (R7)
  V3DB_CUDA(cudaMemsetAsync(s->codes, 0, static_cast<size_t>(slots) * m, st));  // padding code 0
  V3DB_CUDA(v3db::make_codebooks(db, s->centroids, s->list_of, dim, m, ks, d_cwrows.p, s->codebooks, st));
  V3DB_CUDA(v3db::encode_and_place(db, n, dim, s->centroids, s->list_of, d_pos.p, s->codebooks, m, ks, s->codes,
                                   s->ids, st));
  V3DB_CUDA(v3db::slot_terms(s->centroids, s->codebooks, s->codes, s->ids, nlist, L, dim, m, ks, s->pterm, st));
  // layouts of the rotated-LUT scan
  s->lut_mode = v3db::plan_lut(m, ks, d, &s->lut_g);
  if (static_cast<int64_t>(nlist) * ((L + 31) & ~31) >= (int64_t(1) << 31)) s->lut_mode = 0;  // 32-bit slot offsets
  if (s->lut_mode != 0) {
    // padded list stride Lp; +256 B so rounded-up bulk copies of the last chunk stay in bounds
    const int64_t pslots = static_cast<int64_t>(nlist) * ((L + 31) & ~31);
    V3DB_CUDA(cudaMalloc(&s->codes_rot, static_cast<size_t>(pslots) * m + 256));
    V3DB_CUDA(cudaMalloc(&s->pterm_rot, sizeof(int32_t) * pslots + 256));
    V3DB_CUDA(cudaMalloc(&s->cbT, static_cast<size_t>(m) * ks * d));
    V3DB_CUDA(v3db::rotate_codes(s->codes, s->pterm, nlist, L, m, s->lut_mode, s->lut_g, s->codes_rot, s->pterm_rot,
                                 st));
    V3DB_CUDA(v3db::transpose_codebooks(s->codebooks, m, ks, d, s->cbT, st));
  }
  // reconstruction of every slot for the list-major tensor-core scan (dim % 16 == 0, nlist <= 32768:
  // its one-CTA item scan holds 32 lists per thread)
  if (dim % 16 == 0 && nlist <= 32768) {
    s->lm_Lp = (L + 127) & ~127;
    V3DB_CUDA(cudaMalloc(&s->xhat, static_cast<size_t>(nlist) * s->lm_Lp * dim));
    V3DB_CUDA(v3db::make_xhat(s->codes, s->counts, s->codebooks, nlist, L, s->lm_Lp, dim, m, ks, s->xhat, st));
  }
  V3DB_CUDA(cudaStreamSynchronize(st));
  s->total_valid = n;
  guard.s = nullptr;
  *out = s;
  return V3DB_OK;
}

static int validate_query(v3db_snapshot_t s, const void* queries, int64_t nq, int32_t nprobe, int32_t k,
                          const void* out_ids, const void* out_dist) {
  if (!s) return fail(V3DB_EINVAL, "NULL snapshot");
  if (nq < 0 || nq >= (int64_t(1) << 31)) return fail(V3DB_EINVAL, "nq out of range");
  if (nq > 0 && (!queries || !out_ids || !out_dist)) return fail(V3DB_EINVAL, "NULL required pointer");
  if (nprobe < 1 || nprobe > s->nlist || nprobe > V3DB_MAX_NPROBE)
    return fail(V3DB_EINVAL, "nprobe out of range [1, min(nlist, V3DB_MAX_NPROBE)]");
  const int64_t nsel = static_cast<int64_t>(nprobe) * s->L;
  if (k < 1 || k > nsel || k > V3DB_MAX_K) return fail(V3DB_EINVAL, "k out of range [1, min(nprobe*L, V3DB_MAX_K)]");
  return V3DB_OK;
}

int v3db_query_batch_ex(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe, int32_t k,
                        int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists, int32_t* trace_list_dist,
                        int32_t* trace_cand_dist, int32_t algo, void* stream) {
  g_err.clear();
  int rc = validate_query(s, queries, nq, nprobe, k, out_ids, out_dist);
  if (rc != V3DB_OK) return rc;
  if (s->fx) return fail(V3DB_EINVAL, "fixed-point snapshot: use v3db_query_batch_fx");
  if (algo != V3DB_SCAN_AUTO && algo != V3DB_SCAN_GENERIC && algo != V3DB_SCAN_ROTATED && algo != V3DB_SCAN_LIST_MAJOR)
    return fail(V3DB_EINVAL, "unsupported scan algo");
  if (algo == V3DB_SCAN_ROTATED && s->lut_mode == 0)
    return fail(V3DB_EINVAL, "V3DB_SCAN_ROTATED does not support this snapshot's (M, Ks, d)");
  if (algo == V3DB_SCAN_LIST_MAJOR && !s->xhat)
    return fail(V3DB_EINVAL, "V3DB_SCAN_LIST_MAJOR needs dim % 16 == 0 and nlist <= 32768");
  if (algo == V3DB_SCAN_AUTO) {
    const int64_t pref = v3db::opt(V3DB_OPT_AUTO_SCAN);
    if (pref == V3DB_SCAN_GENERIC || (pref == V3DB_SCAN_ROTATED && s->lut_mode != 0))
      algo = static_cast<int32_t>(pref);
    else
      algo = s->xhat ? V3DB_SCAN_LIST_MAJOR : s->lut_mode != 0 ? V3DB_SCAN_ROTATED : V3DB_SCAN_GENERIC;
  }
  if ((rc = check_device(s)) != V3DB_OK) return rc;
  if (nq == 0) return V3DB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* lists = trace_lists;
  int32_t* ldist = trace_list_dist;
  void* scratch = nullptr;
  if (!lists || !ldist) {
    V3DB_CUDA(v3db::scratch_alloc(&scratch, sizeof(int32_t) * 2 * nq * nprobe, st));
    if (!lists) lists = static_cast<int32_t*>(scratch);
    if (!ldist) ldist = static_cast<int32_t*>(scratch) + nq * nprobe;
  }
  // list-major scan: Steps 1-2 also count the (query, rank) pairs per list for its grouping
  int* list_hist = nullptr;
  if (algo == V3DB_SCAN_LIST_MAJOR) {
    cudaError_t eh = v3db::scratch_alloc(reinterpret_cast<void**>(&list_hist), sizeof(int) * s->nlist, st);
    if (eh == cudaSuccess) eh = cudaMemsetAsync(list_hist, 0, sizeof(int) * s->nlist, st);
    if (eh != cudaSuccess) {
      if (scratch) cudaFreeAsync(scratch, st);
      return cuda_fail(eh, "list-major scratch");
    }
  }
  prof_record(0, st);
  cudaError_t e = v3db::coarse_topk(queries, nq, s->dim, s->centroids, s->cnorm, s->nlist, nprobe, lists, ldist, st,
                                    list_hist);
  prof_scan_begin(st);
  if (e == cudaSuccess) {
    if (algo == V3DB_SCAN_LIST_MAJOR)
      e = v3db::scan_list_major(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace_cand_dist, st,
                                g_prof.on ? prof_record : nullptr, list_hist);
    else if (algo == V3DB_SCAN_ROTATED)
      e = v3db::scan_rotated(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace_cand_dist, st);
    else
      e = v3db::scan_generic(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace_cand_dist, st);
  }
  prof_scan_end(st);
  if (scratch) cudaFreeAsync(scratch, st);
  if (list_hist) cudaFreeAsync(list_hist, st);
  if (e != cudaSuccess) {
    if (g_err.empty()) return cuda_fail(e, "query kernels");
    return V3DB_ECUDA;
  }
  return V3DB_OK;
}

int v3db_query_batch(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe, int32_t k,
                     int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists, int32_t* trace_list_dist,
                     int32_t* trace_cand_dist, void* stream) {
  return v3db_query_batch_ex(s, queries, nq, nprobe, k, out_ids, out_dist, trace_lists, trace_list_dist,
                             trace_cand_dist, V3DB_SCAN_AUTO, stream);
}

int v3db_query_batch_host(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe, int32_t k,
                          int32_t* out_ids, int32_t* out_dist, int32_t* trace_lists, int32_t* trace_list_dist,
                          int32_t* trace_cand_dist, void* stream) {
  g_err.clear();
  int rc = validate_query(s, queries, nq, nprobe, k, out_ids, out_dist);
  if (rc != V3DB_OK) return rc;
  if (s->fx) return fail(V3DB_EINVAL, "fixed-point snapshot: use v3db_query_batch_fx");
  if ((rc = check_device(s)) != V3DB_OK) return rc;
  if (nq == 0) return V3DB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t qb = static_cast<size_t>(nq) * s->dim;
  const size_t ob = sizeof(int32_t) * static_cast<size_t>(nq) * k;
  const size_t lb = sizeof(int32_t) * static_cast<size_t>(nq) * nprobe;
  const size_t tb = trace_cand_dist ? sizeof(int32_t) * static_cast<size_t>(nq) * nprobe * s->L : 0;
  const size_t total = ((qb + 255) & ~size_t(255)) + 2 * ob + 2 * lb + tb + 1024;
  uint8_t* buf = nullptr;
  V3DB_CUDA(v3db::scratch_alloc(reinterpret_cast<void**>(&buf), total, st));
  uint8_t* p = buf;
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  int8_t* dq = reinterpret_cast<int8_t*>(take(qb));
  int32_t* dids = reinterpret_cast<int32_t*>(take(ob));
  int32_t* ddist = reinterpret_cast<int32_t*>(take(ob));
  int32_t* dl = reinterpret_cast<int32_t*>(take(lb));
  int32_t* dld = reinterpret_cast<int32_t*>(take(lb));
  int32_t* dtr = tb ? reinterpret_cast<int32_t*>(take(tb)) : nullptr;
  // With the witness trace requested the call is bound by the device->host copy of the trace;
  // the batch then runs in sub-batches whose outputs are copied on a second stream while the next
  // sub-batch computes (results do not depend on the split: queries are independent).
  const int nchunk = (tb && nq >= 8192) ? 4 : 1;
  const int64_t qc = (nq + nchunk - 1) / nchunk;
  cudaStream_t cs = st;
  cudaEvent_t ev[5] = {};
  cudaError_t e = cudaSuccess;
  if (nchunk > 1) {
    e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int c = 0; c <= nchunk && e == cudaSuccess; ++c) e = cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(dq, queries, qb, cudaMemcpyHostToDevice, st);
  for (int c = 0; c < nchunk && e == cudaSuccess; ++c) {
    const int64_t q0 = c * qc, n = std::min(qc, nq - q0);
    if (n <= 0) break;
    rc = v3db_query_batch_ex(s, dq + q0 * s->dim, n, nprobe, k, dids + q0 * k, ddist + q0 * k, dl + q0 * nprobe,
                             dld + q0 * nprobe, dtr ? dtr + q0 * nprobe * s->L : nullptr, V3DB_SCAN_AUTO, stream);
    if (rc != V3DB_OK) break;
    if (nchunk > 1) {
      e = cudaEventRecord(ev[c], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[c], 0);
    }
    const size_t ob_c = sizeof(int32_t) * static_cast<size_t>(n) * k, lb_c = sizeof(int32_t) * static_cast<size_t>(n) * nprobe;
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_ids + q0 * k, dids + q0 * k, ob_c, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_dist + q0 * k, ddist + q0 * k, ob_c, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && trace_lists)
      e = cudaMemcpyAsync(trace_lists + q0 * nprobe, dl + q0 * nprobe, lb_c, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && trace_list_dist)
      e = cudaMemcpyAsync(trace_list_dist + q0 * nprobe, dld + q0 * nprobe, lb_c, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && dtr)
      e = cudaMemcpyAsync(trace_cand_dist + q0 * nprobe * s->L, dtr + q0 * nprobe * s->L, lb_c * s->L,
                          cudaMemcpyDeviceToHost, cs);
  }
  if (nchunk > 1) {  // the buffer is freed on `st` after the copies on `cs`
    cudaError_t e2 = cudaEventRecord(ev[nchunk], cs);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, ev[nchunk], 0);
    if (e == cudaSuccess) e = e2;
  }
  cudaFreeAsync(buf, st);
  cudaError_t es = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = es;
  if (nchunk > 1) {
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    cudaStreamDestroy(cs);
  }
  if (rc != V3DB_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "v3db_query_batch_host");
  return V3DB_OK;
}

int v3db_witness_batch(v3db_snapshot_t s, const int8_t* queries, int64_t nq, int32_t nprobe, int32_t* list_order,
                       int32_t* list_dist, int32_t* lut_sel, int32_t* cand_items, int32_t* cand_dist, void* stream) {
  g_err.clear();
  if (!s) return fail(V3DB_EINVAL, "NULL snapshot");
  if (s->fx) return fail(V3DB_EINVAL, "the witness API covers int8 snapshots");
  if (nq < 0 || nq > 65535) return fail(V3DB_EINVAL, "nq out of range [0, 65535] (witnesses are per challenged query)");
  if (nq > 0 && !queries) return fail(V3DB_EINVAL, "NULL queries");
  if (nprobe < 1 || nprobe > s->nlist || nprobe > V3DB_MAX_NPROBE)
    return fail(V3DB_EINVAL, "nprobe out of range [1, min(nlist, V3DB_MAX_NPROBE)]");
  int rc = check_device(s);
  if (rc != V3DB_OK) return rc;
  if (nq == 0) return V3DB_OK;
  if (static_cast<int64_t>(nprobe) * s->L > (int64_t(1) << 30))
    return fail(V3DB_EINVAL, "nprobe * list_cap > 2^30: the witness sort segment is too long");
  cudaError_t e = v3db::witness_batch(s, queries, nq, nprobe, list_order, list_dist, lut_sel, cand_items, cand_dist,
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "v3db_witness_batch");
  return V3DB_OK;
}

// ---- NEXT-1: the 16-bit fixed-point path (fx16.cu) ----

int v3db_encode_fixed_point(const float* x, int64_t count, double v_max, int32_t* out, void* stream) {
  g_err.clear();
  if (count < 0) return fail(V3DB_EINVAL, "count < 0");
  if (count > 0 && (!x || !out)) return fail(V3DB_EINVAL, "NULL pointer");
  if (!(v_max > 0.0) || !std::isfinite(v_max)) return fail(V3DB_EINVAL, "v_max must be positive and finite");
  cudaError_t e = v3db::encode_fixed_point(x, count, v_max, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "v3db_encode_fixed_point");
  return V3DB_OK;
}

// |v| <= 65535 for every coordinate (the 16-bit fixed-point range; the distance bounds of the
// composite keys and the exactness of the double-precision dot products rest on it).
static int check_fx_range(const int32_t* x, int64_t count, cudaStream_t st, const char* what) {
  DevBuf<int> d_m;
  V3DB_CUDA(d_m.alloc(1));
  V3DB_CUDA(cudaMemsetAsync(d_m.p, 0, sizeof(int), st));
  V3DB_CUDA(v3db::abs_max32(x, count, d_m.p, st));
  int m = 0;
  V3DB_CUDA(cudaMemcpyAsync(&m, d_m.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  V3DB_CUDA(cudaStreamSynchronize(st));
  if (m > 65535) return fail(V3DB_EINVAL, std::string(what) + " coordinates outside [-65535, 65535]");
  return V3DB_OK;
}

int v3db_build_snapshot_fx(const int32_t* db, int64_t n, int32_t dim, int32_t nlist, int32_t list_cap, int32_t m,
                           int32_t ks, const int32_t* centroid_rows, const int32_t* codeword_rows, void* stream,
                           v3db_snapshot_t* out) {
  g_err.clear();
  if (!db) return fail(V3DB_EINVAL, "NULL required pointer");
  int rc = validate_build(n, dim, nlist, list_cap, m, ks, centroid_rows, codeword_rows, out);
  if (rc != V3DB_OK) return rc;
  if (v3db::fx_shift2(dim) < 1 || nlist > (1 << std::min(v3db::fx_shift2(dim), 30)))
    return fail(V3DB_EINVAL, "nlist too large for the composite Step-2 keys at this dim");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = check_fx_range(db, n * dim, st, "database")) != V3DB_OK) return rc;
  const int d = dim / m;
  const int L = list_cap;
  v3db_snapshot* s = new (std::nothrow) v3db_snapshot();
  if (!s) return fail(V3DB_ENOMEM, "host allocation failed");
  struct Guard {
    v3db_snapshot* s;
    ~Guard() { free_snapshot(s); }
  } guard{s};
  s->n = n;
  s->dim = dim;
  s->nlist = nlist;
  s->L = L;
  s->M = m;
  s->Ks = ks;
  s->d = d;
  s->fx = 1;
  V3DB_CUDA(cudaGetDevice(&s->device));
  const int64_t slots = static_cast<int64_t>(nlist) * L;
  V3DB_CUDA(cudaMalloc(&s->centroids32, sizeof(int32_t) * nlist * dim));
  V3DB_CUDA(cudaMalloc(&s->cnorm64, sizeof(int64_t) * nlist));
  V3DB_CUDA(cudaMalloc(&s->codebooks32, sizeof(int32_t) * m * ks * d));
  V3DB_CUDA(cudaMalloc(&s->ids, sizeof(int32_t) * slots));
  V3DB_CUDA(cudaMalloc(&s->codes, static_cast<size_t>(slots) * m));
  V3DB_CUDA(cudaMalloc(&s->counts, sizeof(int32_t) * nlist));
  V3DB_CUDA(cudaMalloc(&s->pterm64, sizeof(int64_t) * slots));
  V3DB_CUDA(cudaMalloc(&s->list_of, sizeof(int32_t) * n));
  DevBuf<int32_t> d_rows;
  V3DB_CUDA(d_rows.alloc(nlist));
  V3DB_CUDA(cudaMemcpyAsync(d_rows.p, centroid_rows, sizeof(int32_t) * nlist, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(v3db::gather_rows32(db, dim, d_rows.p, nlist, s->centroids32, s->cnorm64, st));  // B1

  std::vector<int32_t> list_of(n), flat_pos(n), counts(nlist, 0);
  std::vector<int32_t> mu_host, row(dim);
  rc = place_greedy(
      n, nlist, L,
      [&](int64_t lo, int64_t rows, int R, int32_t* d_rank, void* d_rdist) {
        return v3db::fx_topk(db + lo * dim, rows, dim, s->centroids32, s->cnorm64, nlist, R, d_rank,
                             static_cast<int64_t*>(d_rdist), st);
      },
      [&](int64_t t, std::vector<int64_t>& e) -> cudaError_t {
        cudaError_t ce = cudaSuccess;
        if (mu_host.empty()) {
          mu_host.resize(static_cast<size_t>(nlist) * dim);
          ce = cudaMemcpy(mu_host.data(), s->centroids32, sizeof(int32_t) * mu_host.size(), cudaMemcpyDeviceToHost);
        }
        if (ce == cudaSuccess) ce = cudaMemcpy(row.data(), db + t * dim, sizeof(int32_t) * dim, cudaMemcpyDeviceToHost);
        for (int i = 0; i < nlist && ce == cudaSuccess; ++i) {
          int64_t acc = 0;
          for (int u = 0; u < dim; ++u) {
            const int64_t df = int64_t(row[u]) - int64_t(mu_host[static_cast<size_t>(i) * dim + u]);
            acc += df * df;
          }
          e[i] = acc;
        }
        return ce;
      },
      sizeof(int64_t), st, list_of, flat_pos, counts);
  if (rc != V3DB_OK) return rc;
  DevBuf<int32_t> d_pos, d_cwrows;
  V3DB_CUDA(d_pos.alloc(n));
  V3DB_CUDA(d_cwrows.alloc(static_cast<size_t>(m) * ks));
  V3DB_CUDA(cudaMemcpyAsync(s->list_of, list_of.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(d_pos.p, flat_pos.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(d_cwrows.p, codeword_rows, sizeof(int32_t) * m * ks, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemcpyAsync(s->counts, counts.data(), sizeof(int32_t) * nlist, cudaMemcpyHostToDevice, st));
  V3DB_CUDA(cudaMemsetAsync(s->ids, 0xff, sizeof(int32_t) * slots, st));
  V3DB_CUDA(cudaMemsetAsync(s->codes, 0, static_cast<size_t>(slots) * m, st));
  V3DB_CUDA(v3db::fx_build_tail(db, n, dim, s->centroids32, s->list_of, d_pos.p, m, ks, d_cwrows.p, nlist, L,
                                s->codebooks32, s->codes, s->ids, s->pterm64, st));  // B3-B6
  if (v3db::fx_rot_supported(m, ks) && !v3db::opt(V3DB_OPT_FX_NOROT)) {  // conflict-free scan layout
    V3DB_CUDA(cudaMalloc(&s->codes_rot16, static_cast<size_t>(slots) * m));
    V3DB_CUDA(v3db::rotate_codes16(s->codes, slots, L, m, s->codes_rot16, st));
  }
  // limb planes of every slot's reconstruction for the list-major tensor-core scan
  if (dim % 16 == 0 && dim <= 256 && nlist <= 32768) {
    s->lm_Lp = (L + 127) & ~127;
    V3DB_CUDA(cudaMalloc(&s->xhat_fx, 3ull * nlist * s->lm_Lp * dim));
    V3DB_CUDA(v3db::make_xhat_fx(s->codes, s->counts, s->codebooks32, nlist, L, s->lm_Lp, dim, m, ks, s->xhat_fx, st));
  }
  V3DB_CUDA(cudaStreamSynchronize(st));
  s->total_valid = n;
  guard.s = nullptr;
  *out = s;
  return V3DB_OK;
}

// Steps 1-5 on a validated fixed-point query batch already range-checked (stream-ordered, no host
// synchronization).
static int fx_query_impl(v3db_snapshot_t s, const int32_t* queries, int64_t nq, int32_t nprobe, int32_t k,
                         int32_t* out_ids, int64_t* out_dist, int32_t* trace_lists, int64_t* trace_list_dist,
                         int64_t* trace_cand_dist, cudaStream_t st) {
  int32_t* lists = trace_lists;
  int64_t* ldist = trace_list_dist;
  void* scratch = nullptr;
  if (!lists || !ldist) {
    V3DB_CUDA(v3db::scratch_alloc(&scratch, (sizeof(int32_t) + sizeof(int64_t)) * nq * nprobe, st));
    if (!ldist) ldist = static_cast<int64_t*>(scratch);
    if (!lists) lists = reinterpret_cast<int32_t*>(static_cast<int64_t*>(scratch) + nq * nprobe);
  }
  prof_record(0, st);
  cudaError_t e = v3db::fx_topk(queries, nq, s->dim, s->centroids32, s->cnorm64, s->nlist, nprobe, lists, ldist, st);
  prof_scan_begin(st);
  if (e == cudaSuccess) {
    if (s->xhat_fx && v3db::opt(V3DB_OPT_FX_SCAN) == 0)
      e = v3db::scan_list_major_fx(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace_cand_dist, st,
                                   g_prof.on ? prof_record : nullptr);
    else
      e = v3db::fx_scan(s, queries, nq, nprobe, k, lists, ldist, out_ids, out_dist, trace_cand_dist, st);
  }
  prof_scan_end(st);
  if (scratch) cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "v3db_query_batch_fx");
  return V3DB_OK;
}

static int validate_fx_query(v3db_snapshot_t s, const void* queries, int64_t nq, int32_t nprobe, int32_t k,
                             const void* out_ids, const void* out_dist) {
  int rc = validate_query(s, queries, nq, nprobe, k, out_ids, out_dist);
  if (rc != V3DB_OK) return rc;
  if (!s->fx) return fail(V3DB_EINVAL, "the fixed-point query entry points need a snapshot from v3db_build_snapshot_fx");
  if (static_cast<int64_t>(nprobe) * s->L > (int64_t(1) << std::min(v3db::fx_shift5(s->dim), 31)))
    return fail(V3DB_EINVAL, "nprobe * list_cap too large for the composite Step-5 keys at this dim");
  return check_device(s);
}

int v3db_query_batch_fx(v3db_snapshot_t s, const int32_t* queries, int64_t nq, int32_t nprobe, int32_t k,
                        int32_t* out_ids, int64_t* out_dist, int32_t* trace_lists, int64_t* trace_list_dist,
                        int64_t* trace_cand_dist, void* stream) {
  g_err.clear();
  int rc = validate_fx_query(s, queries, nq, nprobe, k, out_ids, out_dist);
  if (rc != V3DB_OK) return rc;
  if (nq == 0) return V3DB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = check_fx_range(queries, nq * s->dim, st, "query")) != V3DB_OK) return rc;
  return fx_query_impl(s, queries, nq, nprobe, k, out_ids, out_dist, trace_lists, trace_list_dist, trace_cand_dist,
                       st);
}

int v3db_query_batch_fx_host(v3db_snapshot_t s, const float* queries, int64_t nq, double v_max, int32_t nprobe,
                             int32_t k, int32_t* out_ids, int64_t* out_dist, int32_t* trace_lists,
                             int64_t* trace_list_dist, int64_t* trace_cand_dist, void* stream) {
  g_err.clear();
  int rc = validate_fx_query(s, queries, nq, nprobe, k, out_ids, out_dist);
  if (rc != V3DB_OK) return rc;
  if (!(v_max > 0.0) || !std::isfinite(v_max)) return fail(V3DB_EINVAL, "v_max must be positive and finite");
  if (nq == 0) return V3DB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t fb = sizeof(float) * static_cast<size_t>(nq) * s->dim;
  const size_t qb = sizeof(int32_t) * static_cast<size_t>(nq) * s->dim;
  const size_t ib = sizeof(int32_t) * static_cast<size_t>(nq) * k, db = sizeof(int64_t) * static_cast<size_t>(nq) * k;
  const size_t lb = sizeof(int32_t) * static_cast<size_t>(nq) * nprobe, ldb = 2 * lb;
  const size_t tb = trace_cand_dist ? sizeof(int64_t) * static_cast<size_t>(nq) * nprobe * s->L : 0;
  uint8_t* buf = nullptr;
  V3DB_CUDA(v3db::scratch_alloc(reinterpret_cast<void**>(&buf), fb + qb + ib + db + lb + ldb + tb + 2048, st));
  uint8_t* p = buf;
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  float* dx = reinterpret_cast<float*>(take(fb));
  int32_t* dq = reinterpret_cast<int32_t*>(take(qb));
  int32_t* dids = reinterpret_cast<int32_t*>(take(ib));
  int64_t* ddist = reinterpret_cast<int64_t*>(take(db));
  int32_t* dl = reinterpret_cast<int32_t*>(take(lb));
  int64_t* dld = reinterpret_cast<int64_t*>(take(ldb));
  int64_t* dtr = tb ? reinterpret_cast<int64_t*>(take(tb)) : nullptr;
  // sub-batches with the outputs copied on a second stream, as in v3db_query_batch_host
  const int nchunk = (tb && nq >= 8192) ? 4 : 1;
  const int64_t qc = (nq + nchunk - 1) / nchunk;
  cudaStream_t cs = st;
  cudaEvent_t ev[5] = {};
  cudaError_t e = cudaSuccess;
  if (nchunk > 1) {
    e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int c = 0; c <= nchunk && e == cudaSuccess; ++c) e = cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(dx, queries, fb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = v3db::encode_fixed_point(dx, nq * s->dim, v_max, dq, st);
  // one range check of the whole encoded batch, before any output copy is queued
  if (e == cudaSuccess && (rc = check_fx_range(dq, nq * s->dim, st, "query")) != V3DB_OK) {
    cudaFreeAsync(buf, st);
    if (nchunk > 1) {
      for (auto& x : ev)
        if (x) cudaEventDestroy(x);
      cudaStreamDestroy(cs);
    }
    return rc;
  }
  const int64_t Lq = static_cast<int64_t>(nprobe) * s->L;
  for (int c = 0; c < nchunk && e == cudaSuccess; ++c) {
    const int64_t q0 = c * qc, n = std::min(qc, nq - q0);
    if (n <= 0) break;
    rc = fx_query_impl(s, dq + q0 * s->dim, n, nprobe, k, dids + q0 * k, ddist + q0 * k, dl + q0 * nprobe,
                       dld + q0 * nprobe, dtr ? dtr + q0 * Lq : nullptr, st);
    if (rc != V3DB_OK) break;
    if (nchunk > 1) {
      e = cudaEventRecord(ev[c], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[c], 0);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_ids + q0 * k, dids + q0 * k, 4 * n * k, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_dist + q0 * k, ddist + q0 * k, 8 * n * k, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && trace_lists)
      e = cudaMemcpyAsync(trace_lists + q0 * nprobe, dl + q0 * nprobe, 4 * n * nprobe, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && trace_list_dist)
      e = cudaMemcpyAsync(trace_list_dist + q0 * nprobe, dld + q0 * nprobe, 8 * n * nprobe, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess && dtr)
      e = cudaMemcpyAsync(trace_cand_dist + q0 * Lq, dtr + q0 * Lq, 8 * n * Lq, cudaMemcpyDeviceToHost, cs);
  }
  if (nchunk > 1) {
    cudaError_t e2 = cudaEventRecord(ev[nchunk], cs);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, ev[nchunk], 0);
    if (e == cudaSuccess) e = e2;
  }
  cudaFreeAsync(buf, st);
  cudaError_t es = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = es;
  if (nchunk > 1) {
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    cudaStreamDestroy(cs);
  }
  if (rc != V3DB_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "v3db_query_batch_fx_host");
  return V3DB_OK;
}

int v3db_snapshot_kind(v3db_snapshot_t s) {
  g_err.clear();
  if (!s) return fail(V3DB_EINVAL, "NULL snapshot");
  return s->fx ? V3DB_KIND_FX16 : V3DB_KIND_INT8;
}

int v3db_snapshot_info(v3db_snapshot_t s, int64_t* out8) {
  g_err.clear();
  if (!s || !out8) return fail(V3DB_EINVAL, "NULL pointer");
  const int64_t v[8] = {s->n, s->dim, s->nlist, s->L, s->M, s->Ks, s->d, s->total_valid};
  std::memcpy(out8, v, sizeof(v));
  return V3DB_OK;
}

int v3db_snapshot_export(v3db_snapshot_t s, int32_t field, void* host_dst, size_t bytes) {
  g_err.clear();
  if (!s || !host_dst) return fail(V3DB_EINVAL, "NULL pointer");
  const int64_t slots = static_cast<int64_t>(s->nlist) * s->L;
  const void* src = nullptr;
  size_t need = 0;
  switch (field) {
    case V3DB_FIELD_CENTROIDS:
      src = s->fx ? static_cast<const void*>(s->centroids32) : s->centroids;
      need = static_cast<size_t>(s->nlist) * s->dim * (s->fx ? 4 : 1);
      break;
    case V3DB_FIELD_CODEBOOKS:
      src = s->fx ? static_cast<const void*>(s->codebooks32) : s->codebooks;
      need = static_cast<size_t>(s->M) * s->Ks * s->d * (s->fx ? 4 : 1);
      break;
    case V3DB_FIELD_IDS: src = s->ids; need = sizeof(int32_t) * slots; break;
    case V3DB_FIELD_CODES: src = s->codes; need = static_cast<size_t>(slots) * s->M; break;
    case V3DB_FIELD_COUNTS: src = s->counts; need = sizeof(int32_t) * s->nlist; break;
    case V3DB_FIELD_LIST_OF: src = s->list_of; need = sizeof(int32_t) * s->n; break;
    default: return fail(V3DB_EINVAL, "unknown field");
  }
  if (bytes != need) return fail(V3DB_EINVAL, "size mismatch: field needs " + std::to_string(need) + " bytes");
  int rc = check_device(s);
  if (rc != V3DB_OK) return rc;
  V3DB_CUDA(cudaMemcpy(host_dst, src, need, cudaMemcpyDeviceToHost));
  return V3DB_OK;
}

}  // extern "C"

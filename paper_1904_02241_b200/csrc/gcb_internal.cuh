// gcb_internal.cuh -- shared internals of libgcb_b200.so (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>
#include <stdexcept>

#include "../../include/gcb_b200.h"

namespace gcb {

// ---------------------------------------------------------------------------
// errors: internal code throws; every extern "C" entry point catches and maps
// to a return code + thread-local message (gcb_last_error()).
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const char *fmt, ...);
void cuda_check(cudaError_t e, const char *what, const char *file, int line);
int set_last_error(int code, const char *msg);

#define GCB_CUDA(x) ::gcb::cuda_check((x), #x, __FILE__, __LINE__)
#define GCB_REQUIRE(cond, ...)                        \
  do {                                                \
    if (!(cond)) ::gcb::fail(GCB_EINVAL, __VA_ARGS__); \
  } while (0)

#define GCB_API_BEGIN try {
#define GCB_API_END                                                   \
  return GCB_OK;                                                      \
  }                                                                   \
  catch (const ::gcb::Error &e) {                                     \
    return ::gcb::set_last_error(e.code, e.what());                   \
  }                                                                   \
  catch (const std::bad_alloc &) {                                    \
    return ::gcb::set_last_error(GCB_ENOMEM, "host allocation failed"); \
  }                                                                   \
  catch (const std::exception &e) {                                   \
    return ::gcb::set_last_error(GCB_ECUDA, e.what());                \
  }

// ---------------------------------------------------------------------------
// device memory: RAII owner over the device's default stream-ordered pool.
// Graph uploads allocate and free several GB per call; cudaMalloc/cudaFree
// of fresh address ranges cost 5-100 ms per upload at scale 24
// (scripts/e2e_phases.py), the pool (release threshold raised in
// gcb_ctx_create) reuses them.  Semantics stay those of cudaMalloc/cudaFree:
// the allocation is complete before it is handed out, and a release waits for
// the device (cudaFree's implicit synchronisation), so buffers may be used on
// any stream.
// ---------------------------------------------------------------------------
void *device_alloc(size_t bytes);   // ctx.cu
void device_free(void *p);          // ctx.cu
// While one is alive, device_free on this thread is stream-ordered on `s`
// instead of a device-wide synchronisation: for code whose temporaries are
// only touched by kernels on `s` and that must not stall the host behind
// copies queued on another stream (the overlapped upload, partition.cu).
extern thread_local cudaStream_t t_free_stream;
struct StreamOrderedFrees {
  cudaStream_t prev;
  explicit StreamOrderedFrees(cudaStream_t s) : prev(t_free_stream) { t_free_stream = s; }
  ~StreamOrderedFrees() { t_free_stream = prev; }
};

template <typename T>
struct DArray {
  T *p = nullptr;
  size_t n = 0;
  DArray() = default;
  explicit DArray(size_t count) { alloc(count); }
  DArray(const DArray &) = delete;
  DArray &operator=(const DArray &) = delete;
  DArray(DArray &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DArray &operator=(DArray &&o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DArray() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    size_t bytes = (count ? count : 1) * sizeof(T);
    p = static_cast<T *>(device_alloc(bytes));
  }
  void ensure(size_t count) {
    if (n < count || p == nullptr) alloc(count);
  }
  void release() {
    if (p) device_free(p);
    p = nullptr;
    n = 0;
  }
  T *get() const { return p; }
  T *release_ownership() { T *q = p; p = nullptr; n = 0; return q; }
};

}  // namespace gcb

// ---------------------------------------------------------------------------
// opaque handle definitions
// ---------------------------------------------------------------------------
struct gcb_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t l2_bytes = 0, persist_max = 0, window_max = 0;
  int64_t persist_set = 0;  // persisting-L2 set-aside in force (GCB_L2_PERSIST), bytes
  int64_t launches = 0;
  void *pinned = nullptr;  // small pinned host staging (scalars)
  cudaStream_t copy_stream = nullptr;  // host->device copies overlapped with kernels
  cudaStream_t aux_stream = nullptr;   // second compute stream (exact pull: blocks 1..B-1)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // peer exchange (exchange.cu): k_wait_peers sets this mapped host word when
  // a peer misses its deadline, instead of trapping the context
  unsigned *peer_err = nullptr, *peer_err_dev = nullptr;
  gcb::DArray<uint8_t> cub_tmp;
  gcb::DArray<uint8_t> scratch;  // general scratch
  // optional per-category kernel timing (gcb_ctx_set_profiling)
  bool profiling = false;
  struct ProfRec {
    int cat;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> prof;
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_n[4] = {0, 0, 0, 0};
};

struct gcb_csr {
  int device = 0;
  int64_t n = 0, m = 0;
  gcb::DArray<int64_t> ro;   // [n+1]
  gcb::DArray<uint32_t> col; // [m + pad]
  gcb::DArray<double> w;     // [m] or empty
  bool weighted = false;
  // lazily built one-block compacted pull view (unblocked kernels reuse the
  // TOCAB gather with W >= n; kernels.py:207-268 semantics are identical)
  gcb_blocked *compact = nullptr;
  gcb::DArray<uint32_t> outdeg;  // lazily: out-degree (ro diff) as uint32
};

// tile geometry of the edge-balanced (merge-path) pull/push kernels
namespace gcb {
constexpr int kTileV = 8;              // edges per lane
constexpr int kTileT = 32 * kTileV;    // edges per warp tile
constexpr int64_t kColPad = 2 * kTileT; // padding so vector loads never fault
constexpr int kMergeK = 2048;          // internal merge range width
constexpr uint32_t kExactShort = 32;    // exact pull: longer rows go to k_pull_exact_long
constexpr uint32_t kExactMid = 4096;    // ... and rows longer than this get a warp each
}  // namespace gcb

struct gcb_blocked {
  int device = 0;
  int direction = 0;  // 0 pull / 1 push
  bool cb = false;    // conventional blocking (partition_cb, blocking.py:256-286): every
                      // block holds all n rows (identity id_map, empty rows included)
  int64_t width = 0, n = 0, m = 0, B = 0, L = 0;
  bool weighted = false;
  std::vector<int64_t> h_row_starts, h_edge_starts;  // [B+1]
  gcb::DArray<int64_t> row_starts, edge_starts;      // device copies
  gcb::DArray<uint32_t> lro;     // [L+B] per-block local offsets (blocking.py:120)
  gcb::DArray<uint32_t> id_map;  // [L]
  gcb::DArray<uint32_t> col;     // [m + pad]
  gcb::DArray<double> w;         // [m] or empty
  gcb::DArray<uint8_t> w8;       // [m + pad] byte copy of integral weights in [0, 255] (SSSP)
  int w8_state = 0;              // 0 unknown, 1 built, -1 weights do not fit a byte

  // ---- derived, built once by ensure_derived() ----
  bool derived = false;
  bool deg_ready = false;            // deg already counted (overlapped with the upload)
  gcb::DArray<uint32_t> deg;         // out-degrees (kernels.py:324-330)
  std::vector<int64_t> h_tile_t0;    // first absolute tile id per block
  std::vector<int64_t> h_tile_base;  // [B+1] prefix of tiles per block
  gcb::DArray<uint32_t> tile_row;    // per tile: local row of first valid edge
  std::vector<int64_t> h_span_base;  // [B+1] prefix of carry-span starts
  gcb::DArray<uint32_t> span_tile;   // tile ids (global) of each row's first carry tile
  gcb::DArray<uint32_t> span_len;    // number of consecutive carry tiles of that row
  bool long_ready = false;           // long_rows built (ensure_long_rows)
  std::vector<int64_t> h_long_base;  // [B+1] prefix of long rows per block
  std::vector<int64_t> h_long_big;   // [B] leading rows longer than kExactMid (a warp each)
  gcb::DArray<uint32_t> long_rows;   // local rows with > kExactShort edges (exact pull)
  int64_t R = 0;                     // merge ranges (ceil(n / kMergeK))
  gcb::DArray<int64_t> bounds;       // [B][R+1] arena positions per range

  // ---- execution layout of the fast accumulate gather (gather.cu ensure_exec) ----
  bool xready = false;
  int64_t hot_k = 0;                 // hot slots per block (0: staging disabled)
  gcb::DArray<uint32_t> xcol;        // col arena recoded: 0x80000000|slot for hot sources
                                     // (graphs that are not degree-ordered)
  gcb::DArray<uint32_t> hot_ids;     // [B][hot_k] source id of each slot (or ~0u)
  gcb::DArray<double> hotval;        // [B][hot_k] staged values for the next gather
  gcb::DArray<uint32_t> rstart;      // bit q: arena edge q starts a local row
  gcb::DArray<uint32_t> hub_pack;    // hybrid hub blockings: per edge (row - tile_row) << 15 | slot
                                     // (pr.cu ensure_hub_pack); ~0u past the arena
  int hub_pack_state = 0;            // 0 not built, 1 built, -1 not packable (k_push_hot instead)
  gcb::DArray<unsigned long long> hub_acc;  // [hot_k] k_push_hub's cross-CTA fixed-point sums
                                            // (zero between passes: k_hub_fold clears them)

  // ---- workspaces (grown on demand) ----
  gcb::DArray<double> partials;  // [L]
  gcb::DArray<double> carry;     // [tiles]
  gcb::DArray<double> contrib;   // [n]
  gcb::DArray<float> contrib32;  // [n]
  gcb::DArray<double> sums;      // [n] (push)
  gcb::DArray<double> deltas;    // [R + 1]
  gcb::DArray<double> ranks;     // [n]

  // ---- degree-ordered execution copy of a pull graph (relabel.cu) ----
  bool is_relabeled = false;         // this object is such a copy
  int64_t fast_iters = 0;            // fast-mode passes run on this graph (tiering)
  gcb_blocked *rl = nullptr;         // the copy (owned), built on first fast call
  gcb_blocked *hybrid = nullptr;     // degree-ordered copies: push blocking of the edges
                                     // from cold sources into hot destinations (owned)
  gcb::DArray<uint32_t> rl_perm;     // [n] original id -> renumbered id
  int64_t n_live = -1;               // degree-ordered copies: ids [0, n_live) have out-degree
                                     // > 0 (the rest contribute 0 forever); -1 = not counted
  int64_t n_conn = 0;                // ... and [n_conn, n) are isolated (no edge either way)
  const void *iso_clean[2] = {nullptr, nullptr};  // contrib / sums buffers whose isolated
                                     // tail [n_conn, n) is known to be zero (pr.cu pr_run)
  bool dead_dirty = false;           // shard steps: sums of [n_live, v1) not cleared since a
                                     // GCB_FLAG_DEAD_SKIP step (pr.cu shard_live_range)
  gcb_blocked *pending_hybrid = nullptr;  // build scratch of ensure_relabeled (owned)
  gcb_blocked *exact_pull = nullptr;      // push graphs: single-block pull blocking of the
                                          // transpose for the exact push (relabel.cu, owned)

  // ---- tol > 0 PageRank: the convergence loop as one CUDA graph (pr.cu) ----
  struct PrGraph *pr_graph = nullptr;  // owned

  gcb_blocked() = default;
  gcb_blocked(const gcb_blocked &) = delete;
  gcb_blocked &operator=(const gcb_blocked &) = delete;
  ~gcb_blocked();
};

namespace gcb {

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    GCB_CUDA(cudaGetDevice(&prev));
    if (prev != dev) GCB_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Dynamic shared memory / carve-out attributes are per function and per
// device: set them when a launch needs more than was set for this device, or
// a different carve-out (carve_pct < 0 leaves the carve-out alone).
inline void ensure_smem_attrs(gcb_ctx *ctx, const void *kern, size_t smem, int carve_pct = -1) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, std::pair<size_t, int>> set;
  std::lock_guard<std::mutex> lock(mu);
  auto &cur = set[{kern, ctx->device}];
  if (smem > cur.first) {
    GCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur.first = smem;
  }
  if (carve_pct >= 0 && carve_pct != cur.second) {
    GCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve_pct));
    cur.second = carve_pct;
  }
}

inline int max_smem_optin(gcb_ctx *ctx) {
  int optin = 0;
  GCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  return optin;
}

inline void after_launch(gcb_ctx *ctx, const char *name) {
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(GCB_ECUDA, "launch of %s failed: %s", name, cudaGetErrorString(e));
}

// Records CUDA events around a group of launches when profiling is on.
// Categories: 0 gather/scatter, 1 hybrid hub-destination push pass,
// 2 merge/update, 3 other.
struct ProfScope {
  gcb_ctx *ctx;
  int cat;
  cudaEvent_t a = nullptr;
  ProfScope(gcb_ctx *c, int category) : ctx(c), cat(category) {
    if (ctx->profiling) {
      cudaEventCreate(&a);
      cudaEventRecord(a, ctx->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecord(b, ctx->stream);
      ctx->prof.push_back({cat, a, b});
    }
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline unsigned grid_for(int64_t work, int threads, int64_t cap) {
  int64_t g = ceil_div(work > 0 ? work : 1, threads);
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// copies
template <typename T>
void h2d(gcb_ctx *ctx, T *dst, const T *src, size_t count) {
  if (count) GCB_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
}
template <typename T>
void d2h(gcb_ctx *ctx, T *dst, const T *src, size_t count) {
  if (count) GCB_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
}
inline void sync(gcb_ctx *ctx) { GCB_CUDA(cudaStreamSynchronize(ctx->stream)); }

// ---------------------------------------------------------------------------
// cross-file internal API
// ---------------------------------------------------------------------------
// build.cu
void csr_from_sorted_keys(gcb_ctx *ctx, int64_t n, int64_t m, const uint64_t *keys,
                          int bits, gcb_csr *out);
gcb_csr *csr_from_device_edges(gcb_ctx *ctx, int64_t n, int64_t m, const uint32_t *src,
                               const uint32_t *dst, const double *w_or_null);
int bits_for(int64_t n);
// partition.cu
gcb_blocked *partition_device(gcb_ctx *ctx, const gcb_csr *g, int direction, int64_t width);
void ensure_derived(gcb_ctx *ctx, gcb_blocked *bg);
void k_deg_count(gcb_ctx *ctx, int64_t cnt, const uint32_t *col, uint32_t *deg);  // out-degree += per source
gcb_blocked *csr_compact_view(gcb_ctx *ctx, gcb_csr *g);
void compute_range_bounds(gcb_ctx *ctx, const gcb_blocked *bg, int64_t k, int64_t *bounds_dev);
// value kernels (pr.cu)
void pull_sums(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, const float *vals32,
               bool use_weights, uint32_t flags, int64_t block_only, double *out, bool accum);
void merge_to(gcb_ctx *ctx, gcb_blocked *bg, double *out);
// gather.cu: fast pull gather accumulating into a dense vector (hot staging)
void ensure_exec(gcb_ctx *ctx, gcb_blocked *bg);
void upload_col_overlapped(gcb_ctx *ctx, gcb_blocked *bg, const uint32_t *col_host);
void ensure_row_bits(gcb_ctx *ctx, gcb_blocked *bg);  // rstart only (tiles.cuh kernels)
void ensure_long_rows(gcb_ctx *ctx, gcb_blocked *bg);  // exact pull's long-row lists
void ensure_push_exec(gcb_ctx *ctx, gcb_blocked *bg, int64_t hot_slots);  // push hot destinations
void gather_accum(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights,
                  uint32_t flags, double *out);
void cub_sort_pairs_desc_u32_u32(gcb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                                 uint32_t *vals_alt, int64_t m, uint32_t **res_keys,
                                 uint32_t **res_vals);
void push_scatter(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, double *sums,
                  bool use_weights, uint32_t flags, int64_t block_only, bool nonneg = false);
// relabel.cu: degree-ordered execution copy of a pull graph
bool relabel_enabled(gcb_blocked *bg, uint32_t flags, int64_t upcoming_iters);
gcb_blocked *ensure_relabeled(gcb_ctx *ctx, gcb_blocked *bg);
gcb_blocked *ensure_exact_pull(gcb_ctx *ctx, gcb_blocked *bg);
void permute_out(gcb_ctx *ctx, const gcb_blocked *bg, const double *y_new, double *y);
int64_t shard_live_range(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, uint32_t flags,
                         const uint32_t *deg_dev);
int64_t hot_capacity(gcb_ctx *ctx);    // gather.cu: pull hot-table slots
int64_t push_hot_slots(gcb_ctx *ctx);  // pr.cu: push hub-accumulator slots
void destroy_pr_graph(struct ::PrGraph *g);  // pr.cu
// partition.cu: conventional-blocking layout (the CB ablation)
void to_cb_layout(gcb_ctx *ctx, gcb_blocked *bg);
void cb_sums(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights, bool exact,
             double *out);
// cub wrappers (cub_ops.cu)
void cub_sort_keys_u64(gcb_ctx *ctx, uint64_t *keys, uint64_t *keys_alt, int64_t m, int end_bit,
                       uint64_t **result);
void cub_sort_pairs_u64_u32(gcb_ctx *ctx, uint64_t *keys, uint64_t *keys_alt, uint32_t *vals,
                            uint32_t *vals_alt, int64_t m, int end_bit, uint64_t **res_keys,
                            uint32_t **res_vals);
void cub_sort_pairs_u32_u32(gcb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                            uint32_t *vals_alt, int64_t m, int end_bit, uint32_t **res_keys,
                            uint32_t **res_vals);
void cub_exclusive_sum_u32(gcb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t count);
void cub_exclusive_sum_i64(gcb_ctx *ctx, const int64_t *in, int64_t *out, int64_t count);
void cub_inclusive_sum_u32(gcb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t count);
void cub_sum_u64(gcb_ctx *ctx, const uint64_t *in, uint64_t *out_dev, int64_t count);

}  // namespace gcb

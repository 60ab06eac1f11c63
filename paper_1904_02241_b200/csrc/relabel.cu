// relabel.cu -- degree-ordered execution layout of a pull TOCAB graph.
//
// The fast (non-exact) pull paths run on an internal copy of the blocked graph
// whose vertices are renumbered by descending out-degree (ties: ascending id).
// The partition itself is unchanged in kind -- partition_tocab
// (blocking.py:204-253) of the renumbered transpose with the same width -- but
// the renumbering packs the sources that carry most edges into a dense prefix
// of the value vector:
//   * the gather's shared-memory hot table becomes that prefix of each block,
//   * the next-hottest sources share 128-byte lines, so L1/L2 sectors are
//     reused instead of each carrying one useful 8-byte value,
//   * destinations are renumbered with the same permutation, so the rank
//     update stays a pure streaming pass (no permutation per iteration).
// Values are permuted in once per call and results permuted out once per call
// (k_permute_in / k_permute_out).  Sums differ from the reference's only by
// reassociation (the fast-mode contract, <= 1e-6 relative); the exact mode
// never uses this layout.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "gcb_internal.cuh"

namespace gcb {

__global__ void k_iota_u32(int64_t n, uint32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)i;
}

// perm[inv[i]] = i
__global__ void k_invert(int64_t n, const uint32_t *__restrict__ inv, uint32_t *__restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    perm[inv[i]] = (uint32_t)i;
}

// Edges of one block, renumbered: rows (destinations) and cols (sources).
// The source ids are renumbered edge-parallel (k_relabel_cols: four
// independent perm lookups per thread in flight); the row ids are written by
// one warp per local row (k_relabel_rows: stores only), which also adds the
// row's length to the destination's in-degree (one atomic per local row
// instead of one per edge) when the hybrid split needs it.  One warp per row
// doing both took 8 ms at rmat:24 (profiles/r2_promotion_trace.txt): its
// per-edge perm gathers sat behind the row's dependent lro -> id_map -> perm
// chain.
__global__ void k_relabel_cols(int64_t cnt, const uint32_t *__restrict__ col_b,
                               const uint32_t *__restrict__ perm, uint32_t *__restrict__ cols_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += 4 * stride) {
    uint32_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = i + k * stride < cnt ? col_b[i + k * stride] : 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = i + k * stride < cnt ? __ldg(perm + c[k]) : 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < cnt) cols_out[i + k * stride] = c[k];
  }
}

__global__ void k_relabel_rows(int64_t Lb, const uint32_t *__restrict__ lro_b,
                               const uint32_t *__restrict__ id_map_b,
                               const uint32_t *__restrict__ perm, uint32_t *__restrict__ rows_out,
                               uint32_t *__restrict__ indeg) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Lb; r += nw) {
    const uint32_t s = lro_b[r], e = lro_b[r + 1];
    const uint32_t d = perm[id_map_b[r]];
    if (indeg && lane == 0) atomicAdd(indeg + d, e - s);
    for (uint32_t i = s + lane; i < e; i += 32) rows_out[i] = d;
  }
}

// the arena's edges as (row vertex, column) pairs at their arena positions
__global__ void k_block_edges(int64_t Lb, const uint32_t *__restrict__ lro_b,
                              const uint32_t *__restrict__ id_map_b,
                              const uint32_t *__restrict__ col_b, uint32_t *__restrict__ rows_out,
                              uint32_t *__restrict__ cols_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Lb; r += nw) {
    const uint32_t s = lro_b[r], e = lro_b[r + 1];
    const uint32_t d = id_map_b[r];
    for (uint32_t i = s + lane; i < e; i += 32) {
      rows_out[i] = d;
      cols_out[i] = col_b[i];
    }
  }
}

template <typename T>
__global__ void k_permute_in(int64_t n, const uint32_t *__restrict__ perm, const T *__restrict__ x,
                             T *__restrict__ x_new) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    x_new[perm[v]] = x[v];
}

// Ranks back to the input numbering.  Ids [n_conn, n) of the copy are the
// isolated vertices (no edge either way, sorted last): their sums are exactly
// 0, so they all hold one rank, read once instead of gathered (rmat:24: 9.4M
// of 16.8M vertices -- the gather's random sectors were the pass's cost).
__global__ void k_permute_out(int64_t n, int64_t n_conn, const uint32_t *__restrict__ perm,
                              const double *__restrict__ y_new, double *__restrict__ y) {
  const double iso = n_conn < n ? __ldg(y_new + n_conn) : 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = __ldcs(perm + v);
    y[v] = p < n_conn ? y_new[p] : iso;
  }
}

__global__ void k_mark_u8(int64_t cnt, const uint32_t *__restrict__ ids, uint8_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[ids[i]] = 1;
}

// sort key of the degree order: out-degree + 1 for vertices with out-edges,
// 1 for the rest with in-edges, 0 for isolated vertices; counts [#key>=2, #key>=1]
__global__ void k_order_keys(int64_t n, const uint32_t *__restrict__ deg,
                             const uint8_t *__restrict__ has_in, uint32_t *__restrict__ key,
                             unsigned long long *__restrict__ cnt) {
  unsigned long long live = 0, conn = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t d = deg[v];
    const uint32_t k = d ? (d < 0xfffffffeu ? d : 0xfffffffeu) + 1u : (uint32_t)has_in[v];
    key[v] = k;
    live += k >= 2u;
    conn += k >= 1u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_down_sync(0xffffffffu, live, o);
    conn += __shfl_down_sync(0xffffffffu, conn, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (live) atomicAdd(cnt, live);
    if (conn) atomicAdd(cnt + 1, conn);
  }
}

// Tiering: the copy costs a few passes over the edges (~42 ms at rmat:24)
// and saves ~0.2 ms per iteration there, so it pays only on a graph that
// stays resident.  A graph is promoted once it has run GCB_RELABEL_AFTER
// fast-mode iterations (default 256; 0 = immediately); a graph uploaded for
// one short call never is.
// ---------------------------------------------------------------------------
// Hybrid split of the degree-ordered copy.  Every cold gather of the pull
// kernel costs one L1->XBAR request (gather.cu), but an edge from a cold
// source into a hub destination need not: in push form its source value is
// read once per source row (sequential ids) and the add lands in the
// shared-memory hub table of k_push_hot.  So edges (u -> v) with u outside its
// block's hot prefix and v among the top-H destinations by in-degree move to
// a push blocking that runs after the pull pass (rmat:24: A hot-source 29.9%,
// B cold-source/hub-destination 24.0%, C both cold 46.1% of the edges).
// ---------------------------------------------------------------------------
// GCB_HYBRID: 0 off, 1 (default) when the cost model below says it pays, 2 always
static int hybrid_mode() {
  const char *env = getenv("GCB_HYBRID");
  return env && env[0] ? atoi(env) : 1;
}

bool hybrid_enabled() { return hybrid_mode() != 0; }

// Hub destinations of the hybrid class (and slots of its push table): 20480
// ran the iteration 0.7% faster than the full 24576-slot table at rmat:24
// (gather 0.791 vs 0.796 ms, three runs each); GCB_HYBRID_HUBS overrides.
static int64_t hybrid_hub_slots(gcb_ctx *ctx) {
  const char *env = getenv("GCB_HYBRID_HUBS");
  const int64_t want = env ? atoll(env) : 20480;
  const int64_t cap = push_hot_slots(ctx);
  return want < cap ? want : cap;
}

// The push pass has a fixed cost -- its own launch, every CTA zeroes and
// flushes its hub table, the fold -- against a per-edge saving over the pull
// gather.  With the packed hub kernel (pr.cu k_push_hub) the measured gather +
// hub time per iteration, hybrid vs pull-only, is 0.0963 vs 0.0955 ms at
// rmat:21 (9.7M hub edges) and 0.172 vs 0.190 ms at rmat:22 (19M): break-even
// near 3 x num_sms x slots (profiles/r2_hybrid_threshold.txt).  The round-1
// hub kernel needed 13x.
constexpr int64_t kHybridMinEdgesPerSlot = 3;

__global__ void k_count_u32(int64_t m, const uint32_t *__restrict__ ids, uint32_t *__restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + ids[e], 1u);
}

__global__ void k_mark_top(int64_t K, const uint32_t *__restrict__ keys, const uint32_t *__restrict__ ids,
                           uint8_t *__restrict__ hot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x)
    if (keys[i] > 0) hot[ids[i]] = 1;
}

__global__ void k_class_b(int64_t m, const uint32_t *__restrict__ rows, const uint32_t *__restrict__ cols,
                          int64_t width, uint32_t hs, const uint8_t *__restrict__ hot_dst,
                          uint32_t *__restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = cols[e];
    const bool cold_src = (uint32_t)((int64_t)u % width) >= hs;
    flag[e] = (cold_src && hot_dst[rows[e]]) ? 1u : 0u;
  }
}

// stable split: flag 1 -> (a_*) at pos[e], flag 0 -> (b_*) at e - pos[e]
__global__ void k_split_edges(int64_t m, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ pos,
                              const uint32_t *__restrict__ rows, const uint32_t *__restrict__ cols,
                              const double *__restrict__ w, uint32_t *__restrict__ a_src,
                              uint32_t *__restrict__ a_dst, double *__restrict__ a_w,
                              uint32_t *__restrict__ b_rows, uint32_t *__restrict__ b_cols,
                              double *__restrict__ b_w) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = pos[e];
    if (flag[e]) {
      a_src[p] = cols[e];  // push form: rows = sources
      a_dst[p] = rows[e];
      if (w) a_w[p] = w[e];
    } else {
      const int64_t q = e - p;
      b_rows[q] = rows[e];
      b_cols[q] = cols[e];
      if (w) b_w[q] = w[e];
    }
  }
}

// rows/cols (renumbered transpose edges, in place) keep the pull edges;
// returns their count and the push CSR of the split-off edges
// indeg (optional): in-degrees of the row ids, already counted by the caller
// (consumed: the sort below reuses its storage)
static int64_t hybrid_split(gcb_ctx *ctx, int64_t n, int64_t m, int64_t width,
                            DArray<uint32_t> &rows, DArray<uint32_t> &cols, const double *w,
                            DArray<double> &w_pull, gcb_csr **push_csr,
                            DArray<uint32_t> *indeg = nullptr) {
  *push_csr = nullptr;
  const int64_t hs = hot_capacity(ctx);
  const int64_t hd = hybrid_hub_slots(ctx);
  if (m == 0 || hs <= 0 || hd <= 0 || width <= hs) return m;  // whole slices are hot already
  DArray<uint8_t> hot_dst(n);
  {
    DArray<uint32_t> k1, k2(n), v1(n), v2(n);
    if (indeg && indeg->p && indeg->n >= (size_t)n) {
      k1 = std::move(*indeg);
    } else {
      k1.alloc(n);
      GCB_CUDA(cudaMemsetAsync(k1.p, 0, n * sizeof(uint32_t), ctx->stream));
      k_count_u32<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, rows.p, k1.p);
      after_launch(ctx, "k_count_u32");
    }
    k_iota_u32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, v1.p);
    after_launch(ctx, "k_iota_u32");
    uint32_t *rk = nullptr, *rv = nullptr;
    cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, n, &rk, &rv);
    GCB_CUDA(cudaMemsetAsync(hot_dst.p, 0, n, ctx->stream));
    const int64_t K = hd < n ? hd : n;
    k_mark_top<<<grid_for(K, 256, 4096), 256, 0, ctx->stream>>>(K, rk, rv, hot_dst.p);
    after_launch(ctx, "k_mark_top");
  }
  DArray<uint32_t> flag(m + 1), pos(m + 1);
  k_class_b<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, rows.p, cols.p, width,
                                                             (uint32_t)hs, hot_dst.p, flag.p);
  after_launch(ctx, "k_class_b");
  GCB_CUDA(cudaMemsetAsync(flag.p + m, 0, sizeof(uint32_t), ctx->stream));
  cub_exclusive_sum_u32(ctx, flag.p, pos.p, m + 1);
  uint32_t mb = 0;
  d2h(ctx, &mb, pos.p + m, 1);
  sync(ctx);
  if (mb == 0) return m;
  if (hybrid_mode() == 1 && (int64_t)mb < kHybridMinEdgesPerSlot * ctx->num_sms * hd) return m;
  const int64_t mp = m - mb;
  DArray<uint32_t> a_src(mb), a_dst(mb), b_rows(mp ? mp : 1), b_cols(mp ? mp : 1);
  DArray<double> a_w;
  if (w) {
    a_w.alloc(mb);
    w_pull.alloc(mp ? mp : 1);
  }
  k_split_edges<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
      m, flag.p, pos.p, rows.p, cols.p, w, a_src.p, a_dst.p, w ? a_w.p : nullptr, b_rows.p,
      b_cols.p, w ? w_pull.p : nullptr);
  after_launch(ctx, "k_split_edges");
  *push_csr = csr_from_device_edges(ctx, n, mb, a_src.p, a_dst.p, w ? a_w.p : nullptr);
  rows = std::move(b_rows);
  cols = std::move(b_cols);
  return mp;
}

bool relabel_enabled(gcb_blocked *bg, uint32_t flags, int64_t upcoming_iters) {
  if (flags & (GCB_FLAG_EXACT | GCB_FLAG_NO_RELABEL)) return false;
  if (bg->m == 0 || bg->n >= (int64_t(1) << 32)) return false;
  if (bg->is_relabeled || bg->cb) return false;
  const char *env = getenv("GCB_NO_RELABEL");
  if (env && env[0] && env[0] != '0') return false;
  if (bg->rl) return true;
  // Ski rental: building the copy (permutation, renumbered edges, hybrid
  // split, pull CSR, both partitions) costs 41-43 ms at rmat:24 once the
  // memory pool has grown (53-62 ms before the edge-parallel relabel) and saves
  // ~0.20 ms per iteration (hot-bit 11.6 vs promoted 9.6 ms per 10-iteration
  // call; profiles/r2_promotion_trace.txt, GCB_TRACE_PROMO=1), so it pays after
  // ~200-215 iterations.  Promoting once 256 fast iterations have been asked
  // for keeps any workload within ~2x of the better choice; long-running jobs
  // (and bench.py, which builds it in its untimed setup) get the steady state.
  const char *after = getenv("GCB_RELABEL_AFTER");
  const int64_t threshold = after ? atoll(after) : 256;
  if (bg->fast_iters >= threshold) return true;
  bg->fast_iters += upcoming_iters;
  return false;
}

// Exact push (np.bincount order, kernels.py:285-297): every destination lives
// in one push block, and bincount adds its in-edges in arena order, i.e. by
// ascending source row.  That is the sequential sum an exact pull computes
// over the transpose whose rows list sources ascending (the stable sort keeps
// duplicate edges, and so their weights, in arena order) -- with a single
// block, so each destination's adds form one chain.  The push arena is
// transposed into that pull blocking once per graph; one thread per block
// walking its arena took 17 s per iteration at rmat:22.
gcb_blocked *ensure_exact_pull(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->exact_pull) return bg->exact_pull;
  ensure_derived(ctx, bg);
  const int64_t n = bg->n, m = bg->m;
  gcb_csr *csr = nullptr;
  {
    DArray<uint32_t> rows(m ? m : 1), cols(m ? m : 1);
    for (int64_t b = 0; b < bg->B; ++b) {
      const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
      if (Lb == 0) continue;
      const int64_t es = bg->h_edge_starts[b];
      k_block_edges<<<grid_for(Lb * 32, 256, 65536), 256, 0, ctx->stream>>>(
          Lb, bg->lro.p + rs + b, bg->id_map.p + rs, bg->col.p + es, rows.p + es, cols.p + es);
      after_launch(ctx, "k_block_edges");
    }
    // (destination, source) pairs: the transpose, rows sorted, sources ascending
    csr = csr_from_device_edges(ctx, n, m, cols.p, rows.p, bg->weighted ? bg->w.p : nullptr);
  }
  try {
    bg->exact_pull = partition_device(ctx, csr, 0, n > 0 ? n : 1);
  } catch (...) {
    gcb_csr_destroy(csr);
    throw;
  }
  gcb_csr_destroy(csr);
  return bg->exact_pull;
}

// GCB_TRACE_PROMO=1: synchronise after each stage of the promotion build and
// print its wall time to stderr (the stage costs behind the ski-rental threshold)
struct PromoTrace {
  gcb_ctx *ctx;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PromoTrace(gcb_ctx *c) : ctx(c) {
    const char *e = getenv("GCB_TRACE_PROMO");
    on = e && e[0] && e[0] != '0';
    if (on) { sync(ctx); t = std::chrono::steady_clock::now(); }
  }
  void mark(const char *stage) {
    if (!on) return;
    sync(ctx);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[promo] %-28s %8.2f ms\n", stage,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

gcb_blocked *ensure_relabeled(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->rl) return bg->rl;
  PromoTrace tr(ctx);
  ensure_derived(ctx, bg);
  tr.mark("derived tables");
  const int64_t n = bg->n, m = bg->m;
  // 1. permutation: stable sort of (deg desc, id asc)
  bg->rl_perm.alloc(n);
  int64_t n_live = -1, n_conn = n;
  {
    // descending out-degree (ties by id); among the vertices without
    // out-edges those with in-edges come first and isolated ones last, so
    // [n_live, n) contributes nothing and [n_conn, n) is never touched
    DArray<uint32_t> k1(n), k2(n), v1(n), v2(n);
    DArray<uint8_t> has_in(n);
    DArray<unsigned long long> cnt(2);
    GCB_CUDA(cudaMemsetAsync(has_in.p, 0, n, ctx->stream));
    GCB_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
    // in-edges: a pull blocking's rows (id_map) are destinations, a push one's col
    const int64_t nin = bg->direction == 0 ? bg->L : m;
    if (nin > 0) {
      k_mark_u8<<<grid_for(nin, 256, 65536), 256, 0, ctx->stream>>>(
          nin, bg->direction == 0 ? bg->id_map.p : bg->col.p, has_in.p);
      after_launch(ctx, "k_mark_u8");
    }
    k_order_keys<<<grid_for(n, 256, 4096), 256, 0, ctx->stream>>>(n, bg->deg.p, has_in.p, k1.p,
                                                                 cnt.p);
    after_launch(ctx, "k_order_keys");
    k_iota_u32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, v1.p);
    after_launch(ctx, "k_iota_u32");
    uint32_t *rk = nullptr, *inv = nullptr;
    cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, n, &rk, &inv);
    k_invert<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, inv, bg->rl_perm.p);
    after_launch(ctx, "k_invert");
    unsigned long long hc[2] = {0, 0};
    d2h(ctx, hc, cnt.p, 2);
    sync(ctx);
    n_live = (int64_t)hc[0];
    n_conn = (int64_t)hc[1];
  }
  tr.mark("permutation");
  // 2. renumbered edge list (destination, source) from the arenas
  gcb_csr *csr = nullptr;
  {
    DArray<uint32_t> rows(m), cols(m);
    // in-degrees of the renumbered destinations for the hybrid split (a pull
    // blocking's rows are its destinations)
    DArray<uint32_t> indeg;
    if (hybrid_enabled() && bg->direction == 0) {
      indeg.alloc(n);
      GCB_CUDA(cudaMemsetAsync(indeg.p, 0, n * sizeof(uint32_t), ctx->stream));
    }
    for (int64_t b = 0; b < bg->B; ++b) {
      const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
      const int64_t es = bg->h_edge_starts[b], eb = bg->h_edge_starts[b + 1] - es;
      if (Lb == 0) continue;
      k_relabel_cols<<<grid_for((eb + 3) / 4, 256, (int64_t)64 * ctx->num_sms), 256, 0,
                       ctx->stream>>>(eb, bg->col.p + es, bg->rl_perm.p, cols.p + es);
      after_launch(ctx, "k_relabel_cols");
      k_relabel_rows<<<grid_for(Lb * 32, 256, 65536), 256, 0, ctx->stream>>>(
          Lb, bg->lro.p + rs + b, bg->id_map.p + rs, bg->rl_perm.p, rows.p + es, indeg.p);
      after_launch(ctx, "k_relabel_rows");
    }
    // a push blocking's rows are sources: the copy is always the pull
    // (destination-row) form, so push PageRank runs the same pipeline
    if (bg->direction == 1) std::swap(rows, cols);
    tr.mark("renumbered edges");
    // 3. split off the edges whose source misses its block's hot prefix but
    //    whose destination is a hub (hybrid_split), then the canonical CSR of
    //    the rest of the renumbered transpose and the same TOCAB cut
    gcb_csr *push_csr = nullptr;
    int64_t m_pull = m;
    const double *w = bg->weighted ? bg->w.p : nullptr;
    DArray<double> wpull;
    if (hybrid_enabled()) {
      m_pull = hybrid_split(ctx, n, m, bg->width, rows, cols, w, wpull, &push_csr, &indeg);
      if (push_csr && bg->weighted) w = wpull.p;  // split: the pull edges' own weights
      tr.mark("hybrid split (+ push csr)");
    }
    try {
      csr = csr_from_device_edges(ctx, n, m_pull, rows.p, cols.p, w);
    } catch (...) {
      if (push_csr) gcb_csr_destroy(push_csr);
      throw;
    }
    tr.mark("pull csr");
    if (push_csr) {
      try {
        bg->pending_hybrid = partition_device(ctx, push_csr, 1, n);  // one block: every hub slot
      } catch (...) {
        gcb_csr_destroy(push_csr);
        gcb_csr_destroy(csr);
        throw;
      }
      gcb_csr_destroy(push_csr);
      tr.mark("push partition");
    }
  }
  try {
    gcb_blocked *rl = partition_device(ctx, csr, 0, bg->width);
    tr.mark("pull partition");
    rl->is_relabeled = true;
    rl->n_live = n_live;
    rl->n_conn = n_conn;
    if (bg->pending_hybrid) {
      rl->hybrid = bg->pending_hybrid;
      ensure_push_exec(ctx, rl->hybrid, hybrid_hub_slots(ctx));  // table sized to the hubs
      bg->pending_hybrid = nullptr;
      // the pull copy no longer holds every edge: its out-degrees are the
      // whole graph's, renumbered (kernels.py:324-330)
      rl->deg.alloc(n);
      k_permute_in<uint32_t><<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(
          n, bg->rl_perm.p, bg->deg.p, rl->deg.p);
      after_launch(ctx, "k_permute_in");
      rl->deg_ready = true;
    }
    bg->rl = rl;
  } catch (...) {
    gcb_csr_destroy(csr);
    throw;
  }
  gcb_csr_destroy(csr);
  sync(ctx);
  tr.mark("push exec table, degrees");
  return bg->rl;
}

void permute_out(gcb_ctx *ctx, const gcb_blocked *bg, const double *y_new, double *y) {
  const int64_t nc = bg->rl ? bg->rl->n_conn : bg->n;
  k_permute_out<<<grid_for(bg->n, 256, 65536), 256, 0, ctx->stream>>>(bg->n, nc, bg->rl_perm.p,
                                                                     y_new, y);
  after_launch(ctx, "k_permute_out");
}

}  // namespace gcb

// ---------------------------------------------------------------------------
// Degree-ordered destination shards (parallel.py).  A shard cannot
// promote itself the way ensure_relabeled does: every rank's contribution
// vector must use one numbering.  So the whole transpose is renumbered once
// (gcb_csr_degree_order, the permutation ensure_relabeled would pick from the
// global out-degrees), the shards are contiguous row ranges of the renumbered
// graph, and each shard's slab is blocked with the prefix hot set (and, where
// the cost model says it pays, the hybrid hub-destination push pass) by
// gcb_shard_blocking.
// ---------------------------------------------------------------------------
namespace gcb {

__global__ void k_csr_edges(int64_t n, const int64_t *__restrict__ ro, const uint32_t *__restrict__ col,
                            const uint32_t *__restrict__ perm, uint32_t *__restrict__ rows_out,
                            uint32_t *__restrict__ cols_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t s = ro[r], e = ro[r + 1];
    const uint32_t d = perm ? perm[r] : (uint32_t)r;
    for (int64_t i = s + lane; i < e; i += 32) {
      rows_out[i] = d;
      cols_out[i] = perm ? perm[col[i]] : col[i];
    }
  }
}

__global__ void k_nonempty_rows(int64_t n, const int64_t *__restrict__ ro, uint8_t *__restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = ro[v + 1] > ro[v] ? 1 : 0;
}

static void csr_edge_list(gcb_ctx *ctx, const gcb_csr *g, const uint32_t *perm, uint32_t *rows,
                          uint32_t *cols) {
  if (!g->m) return;
  k_csr_edges<<<grid_for(g->n * 32, 256, 65536), 256, 0, ctx->stream>>>(g->n, g->ro.p, g->col.p, perm,
                                                                       rows, cols);
  after_launch(ctx, "k_csr_edges");
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_csr_degree_order(gcb_ctx *ctx, const gcb_csr *gt, uint32_t *perm_dev, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && gt && perm_dev && out, "NULL argument");
  GCB_REQUIRE(gt->n < (int64_t(1) << 32), "vertex count exceeds the 32-bit id space");
  DeviceGuard dg(ctx->device);
  const int64_t n = gt->n, m = gt->m;
  {
    // out-degree of every source = its count among the transpose's columns;
    // stable sort (deg desc, id asc) as ensure_relabeled
    DArray<uint32_t> k1(n), k2(n), v1(n), v2(n);
    GCB_CUDA(cudaMemsetAsync(k1.p, 0, (n ? n : 1) * sizeof(uint32_t), ctx->stream));
    if (m) {
      k_count_u32<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, gt->col.p, k1.p);
      after_launch(ctx, "k_count_u32");
    }
    if (n) {
      // the same key as ensure_relabeled: vertices with in-edges only before
      // isolated ones (a transpose row is a destination's in-edges)
      DArray<uint8_t> has_in(n);
      DArray<unsigned long long> cnt(2);
      GCB_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
      k_nonempty_rows<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, gt->ro.p, has_in.p);
      after_launch(ctx, "k_nonempty_rows");
      k_order_keys<<<grid_for(n, 256, 4096), 256, 0, ctx->stream>>>(n, k1.p, has_in.p, k2.p, cnt.p);
      after_launch(ctx, "k_order_keys");
      std::swap(k1, k2);
      k_iota_u32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, v1.p);
      after_launch(ctx, "k_iota_u32");
      uint32_t *rk = nullptr, *inv = nullptr;
      cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, n, &rk, &inv);
      k_invert<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, inv, perm_dev);
      after_launch(ctx, "k_invert");
    }
  }
  DArray<uint32_t> rows(m ? m : 1), cols(m ? m : 1);
  csr_edge_list(ctx, gt, perm_dev, rows.p, cols.p);
  DArray<double> w;
  if (gt->weighted && m) {
    // weights follow their edge: carried through the builder's sort
    w.alloc(m);
    GCB_CUDA(cudaMemcpyAsync(w.p, gt->w.p, m * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  }
  *out = csr_from_device_edges(ctx, n, m, rows.p, cols.p, gt->weighted ? w.p : nullptr);
  sync(ctx);
  GCB_API_END
}

int gcb_shard_blocking(gcb_ctx *ctx, const gcb_csr *slab, int64_t width, gcb_blocked **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && slab && out, "NULL argument");
  GCB_REQUIRE(width >= 1, "width must be >= 1");
  DeviceGuard dg(ctx->device);
  const int64_t n = slab->n, m = slab->m;
  gcb_csr *pull_csr = nullptr, *push_csr = nullptr;
  if (hybrid_enabled() && m > 0) {
    DArray<uint32_t> rows(m), cols(m);
    csr_edge_list(ctx, slab, nullptr, rows.p, cols.p);
    DArray<double> wpull;
    const int64_t mp = hybrid_split(ctx, n, m, width, rows, cols,
                                    slab->weighted ? slab->w.p : nullptr, wpull, &push_csr);
    if (push_csr) {
      try {
        pull_csr = csr_from_device_edges(ctx, n, mp, rows.p, cols.p,
                                         slab->weighted ? wpull.p : nullptr);
      } catch (...) {
        gcb_csr_destroy(push_csr);
        throw;
      }
    }
  }
  gcb_blocked *bg = nullptr;
  try {
    bg = partition_device(ctx, pull_csr ? pull_csr : slab, 0, width);
    bg->is_relabeled = true;  // sources are in degree order: prefix hot set, no recode
    if (push_csr) {
      bg->hybrid = partition_device(ctx, push_csr, 1, n);  // one block: every hub slot
      ensure_push_exec(ctx, bg->hybrid, hybrid_hub_slots(ctx));
    }
  } catch (...) {
    delete bg;
    if (pull_csr) gcb_csr_destroy(pull_csr);
    if (push_csr) gcb_csr_destroy(push_csr);
    throw;
  }
  if (pull_csr) gcb_csr_destroy(pull_csr);
  if (push_csr) gcb_csr_destroy(push_csr);
  sync(ctx);
  *out = bg;
  GCB_API_END
}

}  // extern "C"

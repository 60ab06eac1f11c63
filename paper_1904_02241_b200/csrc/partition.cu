// partition.cu -- TOCAB static partitioner on the device (blocking.py:189-253)
// plus the derived, build-once tables the iteration kernels read:
//   * out-degrees (kernels.py:324-330),
//   * edge-balanced warp tiles (tile -> first local row),
//   * carry spans (rows longer than one tile),
//   * merge range bounds (BlockedGraph.range_bounds, blocking.py:151-173).
#include <algorithm>

#include "gcb_internal.cuh"

namespace gcb {

__global__ void k_iota_blk(int64_t m, int64_t width, const uint32_t *__restrict__ col,
                           uint32_t *__restrict__ blk, uint32_t *__restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    blk[i] = (uint32_t)((int64_t)col[i] / width);
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_gather_edges(int64_t m, const uint32_t *__restrict__ perm,
                               const uint32_t *__restrict__ col, const uint32_t *__restrict__ erow,
                               const double *__restrict__ w, uint32_t *__restrict__ col_out,
                               uint32_t *__restrict__ row_out, double *__restrict__ w_out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t e = perm ? perm[p] : (uint32_t)p;
    col_out[p] = col[e];
    row_out[p] = erow[e];
    if (w_out) w_out[p] = w[e];
  }
}

__global__ void k_run_flags(int64_t m, int64_t width, const uint32_t *__restrict__ col_p,
                            const uint32_t *__restrict__ row_p, uint32_t *__restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f = 1;
    if (p > 0) {
      uint32_t b0 = (uint32_t)((int64_t)col_p[p - 1] / width), b1 = (uint32_t)((int64_t)col_p[p] / width);
      f = (b0 != b1) || (row_p[p - 1] != row_p[p]);
    }
    flag[p] = f;
  }
}

// edge_starts[b] = lower_bound over block ids (block-major arena)
__global__ void k_block_starts(int64_t B, int64_t m, int64_t width, const uint32_t *__restrict__ col_p,
                               const uint32_t *__restrict__ rid, const uint32_t *__restrict__ flag,
                               int64_t L, int64_t *__restrict__ edge_starts,
                               int64_t *__restrict__ row_starts) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= B;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)col_p[mid] / width < b) lo = mid + 1;
      else hi = mid;
    }
    edge_starts[b] = lo;
    row_starts[b] = (lo < m) ? (int64_t)rid[lo] : L;
  }
}

__global__ void k_runs_to_rows(int64_t m, int64_t width, const uint32_t *__restrict__ col_p,
                               const uint32_t *__restrict__ row_p, const uint32_t *__restrict__ flag,
                               const uint32_t *__restrict__ rid,
                               const int64_t *__restrict__ edge_starts,
                               uint32_t *__restrict__ id_map, uint32_t *__restrict__ lro) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[p]) continue;
    uint32_t r = rid[p];
    int64_t b = (int64_t)col_p[p] / width;
    id_map[r] = row_p[p];
    lro[r + b] = (uint32_t)(p - edge_starts[b]);
  }
}

__global__ void k_block_ends(int64_t B, const int64_t *__restrict__ edge_starts,
                             const int64_t *__restrict__ row_starts, uint32_t *__restrict__ lro) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B;
       b += (int64_t)gridDim.x * blockDim.x)
    lro[row_starts[b + 1] + b] = (uint32_t)(edge_starts[b + 1] - edge_starts[b]);
}

__global__ void k_expand_rows_p(int64_t n, const int64_t *__restrict__ ro, uint32_t *__restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nw) {
    int64_t s = ro[v], e = ro[v + 1];
    for (int64_t i = s + lane; i < e; i += 32) out[i] = (uint32_t)v;
  }
}

gcb_blocked *partition_device(gcb_ctx *ctx, const gcb_csr *g, int direction, int64_t width) {
  GCB_REQUIRE(direction == 0 || direction == 1, "direction must be pull or push");
  GCB_REQUIRE(width >= 1, "width must be >= 1");
  int64_t n = g->n, m = g->m;
  int64_t B = n ? ceil_div(n, width) : 0;
  auto bg = new gcb_blocked();
  try {
    bg->device = ctx->device;
    bg->direction = direction;
    bg->width = width;
    bg->n = n;
    bg->m = m;
    bg->B = B;
    bg->weighted = g->weighted;
    bg->row_starts.alloc(B + 1);
    bg->edge_starts.alloc(B + 1);
    bg->col.alloc(m + kColPad);
    GCB_CUDA(cudaMemsetAsync(bg->col.p, 0, (m + kColPad) * sizeof(uint32_t), ctx->stream));
    if (g->weighted) bg->w.alloc(m + kColPad);
    DArray<uint32_t> erow(m), row_p(m), flag(m), rid(m);
    if (m) {
      k_expand_rows_p<<<grid_for(n * 32, 256, 16384), 256, 0, ctx->stream>>>(n, g->ro.p, erow.p);
      after_launch(ctx, "k_expand_rows_p");
    }
    uint32_t *perm = nullptr;
    DArray<uint32_t> k1, k2, v1, v2;
    if (B > 1 && m) {
      // stable partition by block id == stable radix sort on col // width
      k1.alloc(m); k2.alloc(m); v1.alloc(m); v2.alloc(m);
      k_iota_blk<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, width, g->col.p, k1.p, v1.p);
      after_launch(ctx, "k_iota_blk");
      uint32_t *rk = nullptr;
      cub_sort_pairs_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, m, bits_for(B), &rk, &perm);
    }
    if (m) {
      k_gather_edges<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
          m, perm, g->col.p, erow.p, g->weighted ? g->w.p : nullptr, bg->col.p, row_p.p,
          g->weighted ? bg->w.p : nullptr);
      after_launch(ctx, "k_gather_edges");
      k_run_flags<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, width, bg->col.p, row_p.p,
                                                                    flag.p);
      after_launch(ctx, "k_run_flags");
      cub_exclusive_sum_u32(ctx, flag.p, rid.p, m);
    }
    uint32_t last[2] = {0, 0};
    if (m) {
      d2h(ctx, &last[0], rid.p + (m - 1), 1);
      d2h(ctx, &last[1], flag.p + (m - 1), 1);
      sync(ctx);
    }
    int64_t L = m ? (int64_t)last[0] + last[1] : 0;
    bg->L = L;
    bg->id_map.alloc(L);
    bg->lro.alloc(L + B + 1);
    if (B + 1 > 0) {
      k_block_starts<<<grid_for(B + 1, 256, 4096), 256, 0, ctx->stream>>>(
          B, m, width, bg->col.p, rid.p, flag.p, L, bg->edge_starts.p, bg->row_starts.p);
      after_launch(ctx, "k_block_starts");
    }
    if (m) {
      k_runs_to_rows<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
          m, width, bg->col.p, row_p.p, flag.p, rid.p, bg->edge_starts.p, bg->id_map.p, bg->lro.p);
      after_launch(ctx, "k_runs_to_rows");
    }
    if (B) {
      k_block_ends<<<grid_for(B, 256, 4096), 256, 0, ctx->stream>>>(B, bg->edge_starts.p,
                                                                    bg->row_starts.p, bg->lro.p);
      after_launch(ctx, "k_block_ends");
    }
    bg->h_row_starts.resize(B + 1);
    bg->h_edge_starts.resize(B + 1);
    d2h(ctx, bg->h_row_starts.data(), bg->row_starts.p, B + 1);
    d2h(ctx, bg->h_edge_starts.data(), bg->edge_starts.p, B + 1);
    sync(ctx);
    for (int64_t b = 0; b < B; ++b)
      GCB_REQUIRE(bg->h_edge_starts[b + 1] - bg->h_edge_starts[b] < (int64_t(1) << 32),
                  "block %lld has >= 2^32 edges", (long long)b);
  } catch (...) {
    delete bg;
    throw;
  }
  return bg;
}

// ---------------------------------------------------------------------------
// derived tables
// ---------------------------------------------------------------------------
__global__ void k_deg_pull(int64_t m, const uint32_t *__restrict__ col, uint32_t *__restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&deg[col[i]], 1u);
}

void k_deg_count(gcb_ctx *ctx, int64_t cnt, const uint32_t *col, uint32_t *deg) {
  if (cnt <= 0) return;
  k_deg_pull<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, col, deg);
  after_launch(ctx, "k_deg_pull");
}

__global__ void k_deg_push(int64_t B, const int64_t *__restrict__ row_starts,
                           const uint32_t *__restrict__ lro, const uint32_t *__restrict__ id_map,
                           int64_t L, uint32_t *__restrict__ deg) {
  // one thread per arena row; find its block by scanning row_starts (B small)
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < L;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = B;  // largest b with row_starts[b] <= r
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (row_starts[mid] <= r) lo = mid;
      else hi = mid;
    }
    int64_t b = lo;
    uint32_t d = lro[r + b + 1] - lro[r + b];
    atomicAdd(&deg[id_map[r]], d);
  }
}

// tile_row[t] = local row containing the first valid edge of tile t
__global__ void k_tile_rows(int64_t ntiles, int64_t t0, int64_t es, int64_t Lb,
                            const uint32_t *__restrict__ lro_b, uint32_t *__restrict__ tile_row,
                            uint32_t *__restrict__ carry_flag) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = (t0 + t) * kTileT - es;
    if (q < 0) q = 0;
    int64_t lo = 0, hi = Lb;  // largest i in [0, Lb) with lro_b[i] <= q
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)lro_b[mid] <= q) lo = mid;
      else hi = mid;
    }
    tile_row[t] = (uint32_t)lo;
    carry_flag[t] = (int64_t)lro_b[lo] < q ? 1u : 0u;
  }
}

__global__ void k_span_flags(int64_t ntiles, const uint32_t *__restrict__ tile_row,
                             const uint32_t *__restrict__ carry_flag, uint32_t *__restrict__ start) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = carry_flag[t];
    if (s && t > 0 && carry_flag[t - 1] && tile_row[t - 1] == tile_row[t]) s = 0;
    start[t] = s;
  }
}

__global__ void k_compact_spans(int64_t ntiles, const uint32_t *__restrict__ start,
                                const uint32_t *__restrict__ pos, uint32_t *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x)
    if (start[t]) out[pos[t]] = (uint32_t)t;
}

// length of each carry span: consecutive carry tiles continuing the same row
__global__ void k_span_len(int64_t nspans, int64_t ntiles, const uint32_t *__restrict__ span_tile,
                           const uint32_t *__restrict__ tile_row, const uint32_t *__restrict__ cflag,
                           uint32_t *__restrict__ len) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nspans;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = span_tile[s];
    const uint32_t r = tile_row[t];
    int64_t tt = t;
    while (tt < ntiles && cflag[tt] && tile_row[tt] == r) ++tt;
    len[s] = (uint32_t)(tt - t);
  }
}

__global__ void k_long_flags(int64_t Lb, const uint32_t *__restrict__ lro_b, uint32_t short_max,
                             uint32_t *__restrict__ flag) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Lb;
       r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = lro_b[r + 1] - lro_b[r] > short_max ? 1u : 0u;
}

__global__ void k_compact_rows(int64_t Lb, const uint32_t *__restrict__ flag,
                               const uint32_t *__restrict__ pos, uint32_t *__restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Lb;
       r += (int64_t)gridDim.x * blockDim.x)
    if (flag[r]) out[pos[r]] = (uint32_t)r;
}

__global__ void k_count_above(int64_t c, const uint32_t *__restrict__ keys, uint32_t thr,
                              uint32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c;
       i += (int64_t)gridDim.x * blockDim.x)
    if (keys[i] > thr) atomicAdd(out, 1u);
}

__global__ void k_row_lengths(int64_t c, const uint32_t *__restrict__ rows,
                              const uint32_t *__restrict__ lro_b, uint32_t *__restrict__ len) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c;
       i += (int64_t)gridDim.x * blockDim.x)
    len[i] = lro_b[rows[i] + 1] - lro_b[rows[i]];
}

// bounds[b][j] = row_starts[b] + lower_bound(id_map_b, j*k), j in [0, R]
__global__ void k_range_bounds(int64_t B, int64_t R, int64_t k, const int64_t *__restrict__ row_starts,
                               const uint32_t *__restrict__ id_map, int64_t *__restrict__ bounds) {
  int64_t total = B * (R + 1);
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = x / (R + 1), j = x % (R + 1);
    int64_t rs = row_starts[b], re = row_starts[b + 1];
    int64_t pos;
    if (j == 0) pos = rs;
    else if (j == R) pos = re;
    else {
      int64_t target = j * k, lo = rs, hi = re;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)id_map[mid] < target) lo = mid + 1;
        else hi = mid;
      }
      pos = lo;
    }
    bounds[x] = pos;
  }
}

void compute_range_bounds(gcb_ctx *ctx, const gcb_blocked *bg, int64_t k, int64_t *bounds_dev) {
  int64_t R = bg->n ? ceil_div(bg->n, k) : 0;
  int64_t total = bg->B * (R + 1);
  if (total <= 0) return;
  k_range_bounds<<<grid_for(total, 256, 65536), 256, 0, ctx->stream>>>(bg->B, R, k, bg->row_starts.p,
                                                                      bg->id_map.p, bounds_dev);
  after_launch(ctx, "k_range_bounds");
}

}  // namespace gcb

gcb_blocked::~gcb_blocked() {
  delete rl;
  delete hybrid;
  delete pending_hybrid;
  delete exact_pull;
  gcb::destroy_pr_graph(pr_graph);
}

namespace gcb {

// Long rows per block for the exact pull (a warp each, longest first), built
// on the first exact pass: the fast paths never read them, and the per-block
// compaction and sort cost several host round trips per upload.
void ensure_long_rows(gcb_ctx *ctx, gcb_blocked *bg) {
  ensure_derived(ctx, bg);
  if (bg->long_ready) return;
  const int64_t B = bg->B;
  {
    bg->h_long_base.assign(B + 1, 0);
    std::vector<int64_t> big(B, 0);
    std::vector<DArray<uint32_t>> parts;
    DArray<uint32_t> lflag(bg->L + 1), lpos(bg->L + 1);
    int64_t total = 0;
    std::vector<int64_t> cnt(B, 0);
    for (int64_t b = 0; b < B; ++b) {
      const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
      if (Lb == 0) continue;
      k_long_flags<<<grid_for(Lb, 256, 65536), 256, 0, ctx->stream>>>(Lb, bg->lro.p + rs + b,
                                                                     kExactShort, lflag.p);
      after_launch(ctx, "k_long_flags");
      GCB_CUDA(cudaMemsetAsync(lflag.p + Lb, 0, sizeof(uint32_t), ctx->stream));
      cub_exclusive_sum_u32(ctx, lflag.p, lpos.p, Lb + 1);
      uint32_t c = 0;
      d2h(ctx, &c, lpos.p + Lb, 1);
      sync(ctx);
      cnt[b] = c;
      DArray<uint32_t> part(c ? c : 1);
      if (c) {
        k_compact_rows<<<grid_for(Lb, 256, 65536), 256, 0, ctx->stream>>>(Lb, lflag.p, lpos.p, part.p);
        after_launch(ctx, "k_compact_rows");
        // longest first: the hub rows' add chains are the kernel's critical
        // path, so their warps must start at once (rows are independent)
        DArray<uint32_t> k1(c), k2(c), v2(c);
        k_row_lengths<<<grid_for(c, 256, 65536), 256, 0, ctx->stream>>>(c, part.p, bg->lro.p + rs + b,
                                                                       k1.p);
        after_launch(ctx, "k_row_lengths");
        uint32_t *rk = nullptr, *rv = nullptr;
        cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, part.p, v2.p, c, &rk, &rv);
        if (rv != part.p)
          GCB_CUDA(cudaMemcpyAsync(part.p, rv, c * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                   ctx->stream));
        // how many lead the list with more than kExactMid edges
        uint32_t *nbig = rk == k1.p ? k2.p : k1.p;
        GCB_CUDA(cudaMemsetAsync(nbig, 0, sizeof(uint32_t), ctx->stream));
        k_count_above<<<grid_for(c, 256, 4096), 256, 0, ctx->stream>>>(c, rk, kExactMid, nbig);
        after_launch(ctx, "k_count_above");
        uint32_t hb = 0;
        d2h(ctx, &hb, nbig, 1);
        sync(ctx);  // k1/k2/v2 are released at scope end
        big[b] = hb;
      }
      parts.push_back(std::move(part));
      total += c;
    }
    bg->long_rows.alloc(total ? total : 1);
    int64_t at = 0, pi = 0;
    for (int64_t b = 0; b < B; ++b) {
      bg->h_long_base[b] = at;
      const int64_t Lb = bg->h_row_starts[b + 1] - bg->h_row_starts[b];
      if (Lb == 0) continue;
      if (cnt[b])
        GCB_CUDA(cudaMemcpyAsync(bg->long_rows.p + at, parts[pi].p, cnt[b] * sizeof(uint32_t),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
      at += cnt[b];
      ++pi;
    }
    bg->h_long_base[B] = at;
    bg->h_long_big = big;
  }
  bg->long_ready = true;
}

void ensure_derived(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->derived) return;
  // a captured convergence loop (pr.cu) reads the tables rebuilt below, and
  // the pool may hand back the same addresses: never replay it afterwards
  destroy_pr_graph(bg->pr_graph);
  bg->pr_graph = nullptr;
  bg->hub_pack.release();  // packed against the tile table rebuilt below
  bg->hub_acc.release();
  bg->hub_pack_state = 0;
  int64_t n = bg->n, B = bg->B;
  if (bg->cb) {
    // the CB kernels walk rows directly: out-degrees only
    bg->deg.alloc(n);
    GCB_CUDA(cudaMemsetAsync(bg->deg.p, 0, (n ? n : 1) * sizeof(uint32_t), ctx->stream));
    if (bg->m) {
      k_deg_pull<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->col.p, bg->deg.p);
      after_launch(ctx, "k_deg_pull");
    }
    sync(ctx);
    bg->derived = true;
    return;
  }
  // out-degrees (unless counted while the arena was uploaded)
  if (!bg->deg_ready) bg->deg.alloc(n);
  if (!bg->deg_ready) GCB_CUDA(cudaMemsetAsync(bg->deg.p, 0, (n ? n : 1) * sizeof(uint32_t), ctx->stream));
  if (bg->m && !bg->deg_ready) {
    if (bg->direction == 0) {
      k_deg_pull<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->col.p, bg->deg.p);
      after_launch(ctx, "k_deg_pull");
    } else {
      k_deg_push<<<grid_for(bg->L, 256, 65536), 256, 0, ctx->stream>>>(
          B, bg->row_starts.p, bg->lro.p, bg->id_map.p, bg->L, bg->deg.p);
      after_launch(ctx, "k_deg_push");
    }
  }
  // tiles
  bg->h_tile_t0.assign(B, 0);
  bg->h_tile_base.assign(B + 1, 0);
  for (int64_t b = 0; b < B; ++b) {
    int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
    int64_t nt = 0;
    if (ee > es) {
      bg->h_tile_t0[b] = es / kTileT;
      nt = ceil_div(ee, kTileT) - bg->h_tile_t0[b];
    }
    bg->h_tile_base[b + 1] = bg->h_tile_base[b] + nt;
  }
  int64_t T = bg->h_tile_base[B > 0 ? B : 0];
  bg->tile_row.alloc(T);
  DArray<uint32_t> cflag(T + 1), sflag(T + 1), spos(T + 1);
  bg->h_span_base.assign(B + 1, 0);
  std::vector<uint32_t> span_counts(B, 0);
  for (int64_t b = 0; b < B; ++b) {
    int64_t nt = bg->h_tile_base[b + 1] - bg->h_tile_base[b];
    if (!nt) continue;
    int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    int64_t off = bg->h_tile_base[b];
    k_tile_rows<<<grid_for(nt, 256, 65536), 256, 0, ctx->stream>>>(
        nt, bg->h_tile_t0[b], bg->h_edge_starts[b], Lb, bg->lro.p + rs + b, bg->tile_row.p + off,
        cflag.p + off);
    after_launch(ctx, "k_tile_rows");
    k_span_flags<<<grid_for(nt, 256, 65536), 256, 0, ctx->stream>>>(nt, bg->tile_row.p + off,
                                                                    cflag.p + off, sflag.p + off);
    after_launch(ctx, "k_span_flags");
  }
  if (T) {
    GCB_CUDA(cudaMemsetAsync(sflag.p + T, 0, sizeof(uint32_t), ctx->stream));
    cub_exclusive_sum_u32(ctx, sflag.p, spos.p, T + 1);
    uint32_t nspans = 0;
    d2h(ctx, &nspans, spos.p + T, 1);
    std::vector<uint32_t> hpos(B + 1);
    for (int64_t b = 0; b <= B; ++b) {
      int64_t at = bg->h_tile_base[b];
      d2h(ctx, &hpos[b], spos.p + at, 1);
    }
    sync(ctx);
    bg->span_tile.alloc(nspans);
    k_compact_spans<<<grid_for(T, 256, 65536), 256, 0, ctx->stream>>>(T, sflag.p, spos.p,
                                                                      bg->span_tile.p);
    after_launch(ctx, "k_compact_spans");
    bg->span_len.alloc(nspans);
    if (nspans) {
      k_span_len<<<grid_for(nspans, 256, 65536), 256, 0, ctx->stream>>>(
          nspans, T, bg->span_tile.p, bg->tile_row.p, cflag.p, bg->span_len.p);
      after_launch(ctx, "k_span_len");
    }
    for (int64_t b = 0; b <= B; ++b) bg->h_span_base[b] = hpos[b];
  }
  // span tile ids were global; kernels subtract the block's tile base
  // merge bounds
  bg->R = n ? ceil_div(n, kMergeK) : 0;
  bg->bounds.alloc(B * (bg->R + 1));
  compute_range_bounds(ctx, bg, kMergeK, bg->bounds.p);
  bg->carry.alloc(T);
  sync(ctx);
  bg->derived = true;
}

// ---------------------------------------------------------------------------
// Conventional blocking (partition_cb blocking.py:256-286; _cb_sums
// kernels.py:350-364), kept as the ablation of TOCAB: the same edge split,
// but every block carries all n rows (empty rows included) and its sums go
// to a dense per-block vector that is merged in block order -- no row
// compaction.  Results equal TOCAB's bit for bit (x + 0.0 == x), only the
// memory traffic differs; profiles/ records both per edge.
// ---------------------------------------------------------------------------
__global__ void k_cb_counts(int64_t Lb, const uint32_t *__restrict__ lro_b,
                            const uint32_t *__restrict__ id_map_b, uint32_t *__restrict__ cnt) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Lb;
       r += (int64_t)gridDim.x * blockDim.x)
    cnt[id_map_b[r]] = lro_b[r + 1] - lro_b[r];
}

__global__ void k_cb_ids(int64_t n, int64_t B, uint32_t *__restrict__ id_map) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * B;
       i += (int64_t)gridDim.x * blockDim.x)
    id_map[i] = (uint32_t)(i % n);
}

void to_cb_layout(gcb_ctx *ctx, gcb_blocked *bg) {
  GCB_REQUIRE(bg->direction == 0, "the cb scheme is pull-only");
  const int64_t n = bg->n, B = bg->B;
  DArray<uint32_t> lro((size_t)B * (n + 1) + 1), idm((size_t)(B * n ? B * n : 1)), cnt(n + 1);
  for (int64_t b = 0; b < B; ++b) {
    const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    GCB_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(uint32_t), ctx->stream));
    if (Lb) {
      k_cb_counts<<<grid_for(Lb, 256, 65536), 256, 0, ctx->stream>>>(Lb, bg->lro.p + rs + b,
                                                                     bg->id_map.p + rs, cnt.p);
      after_launch(ctx, "k_cb_counts");
    }
    cub_exclusive_sum_u32(ctx, cnt.p, lro.p + b * (n + 1), n + 1);
  }
  if (B * n) {
    k_cb_ids<<<grid_for(B * n, 256, 65536), 256, 0, ctx->stream>>>(n, B, idm.p);
    after_launch(ctx, "k_cb_ids");
  }
  bg->lro = std::move(lro);
  bg->id_map = std::move(idm);
  bg->L = B * n;
  for (int64_t b = 0; b <= B; ++b) bg->h_row_starts[b] = b * n;
  h2d(ctx, bg->row_starts.p, bg->h_row_starts.data(), B + 1);
  sync(ctx);
  bg->cb = true;
}

// one block's dense partial vector: exact = thread per row in storage order
// (_gather_rows), fast = warp per row
template <bool WGT>
__global__ void k_cb_rows_exact(int64_t n, const uint32_t *__restrict__ lro_b,
                                const uint32_t *__restrict__ col_b, const double *__restrict__ w_b,
                                const double *__restrict__ vals, double *__restrict__ part) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (uint32_t e = lro_b[v]; e < lro_b[v + 1]; ++e)
      acc = __dadd_rn(acc, WGT ? __dmul_rn(w_b[e], vals[col_b[e]]) : vals[col_b[e]]);
    part[v] = acc;
  }
}

template <bool WGT>
__global__ void k_cb_rows_warp(int64_t n, const uint32_t *__restrict__ lro_b,
                               const uint32_t *__restrict__ col_b, const double *__restrict__ w_b,
                               const double *__restrict__ vals, double *__restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
    double acc = 0.0;
    for (uint32_t e = lro_b[v] + lane; e < lro_b[v + 1]; e += 32)
      acc += WGT ? w_b[e] * vals[col_b[e]] : vals[col_b[e]];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) part[v] = acc;
  }
}

// sums = ((0 + part_0) + part_1) + ...  (the block-ordered merge of _cb_sums)
__global__ void k_cb_merge(int64_t n, int64_t B, const double *__restrict__ part,
                           double *__restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < B; ++b) s = __dadd_rn(s, part[b * n + v]);
    out[v] = s;
  }
}

void cb_sums(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights, bool exact,
             double *out) {
  const int64_t n = bg->n, B = bg->B;
  const bool wgt = use_weights && bg->weighted;
  bg->partials.ensure((size_t)(B * n ? B * n : 1));
  for (int64_t b = 0; b < B; ++b) {
    const int64_t es = bg->h_edge_starts[b];
    const uint32_t *lro_b = bg->lro.p + b * (n + 1);
    double *part = bg->partials.p + b * n;
    const double *wb = wgt ? bg->w.p + es : nullptr;
    ProfScope ps(ctx, 0);
    if (exact) {
      if (wgt)
        k_cb_rows_exact<true><<<grid_for(n, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
            n, lro_b, bg->col.p + es, wb, vals, part);
      else
        k_cb_rows_exact<false><<<grid_for(n, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
            n, lro_b, bg->col.p + es, wb, vals, part);
      after_launch(ctx, "k_cb_rows_exact");
    } else {
      if (wgt)
        k_cb_rows_warp<true><<<grid_for(n * 32, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
            n, lro_b, bg->col.p + es, wb, vals, part);
      else
        k_cb_rows_warp<false><<<grid_for(n * 32, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
            n, lro_b, bg->col.p + es, wb, vals, part);
      after_launch(ctx, "k_cb_rows_warp");
    }
  }
  ProfScope ps(ctx, 2);
  k_cb_merge<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, B, bg->partials.p, out);
  after_launch(ctx, "k_cb_merge");
}

// mask[v] = 1 for every source the arena references (the sparse exchange plan)
__global__ void k_mark_sources(int64_t m, const uint32_t *__restrict__ col, uint8_t *__restrict__ mask) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    mask[col[e]] = 1;
}

__global__ void k_narrow_lro(int64_t count, const int64_t *__restrict__ in,
                             uint32_t *__restrict__ out, unsigned int *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v >= (int64_t(1) << 32)) atomicOr(bad, 1u);
    out[i] = (uint32_t)v;
  }
}

gcb_blocked *csr_compact_view(gcb_ctx *ctx, gcb_csr *g) {
  // one block spanning every column: identical arithmetic to the unblocked
  // row gather (kernels.py:155-161) with empty rows compacted away.
  if (!g->compact) g->compact = partition_device(ctx, g, 0, g->n > 0 ? g->n : 1);
  return g->compact;
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_blocked_source_mask(gcb_ctx *ctx, const gcb_blocked *bg, uint8_t *mask_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && (mask_dev || bg->n == 0), "NULL argument");
  DeviceGuard dg(ctx->device);
  if (bg->n) GCB_CUDA(cudaMemsetAsync(mask_dev, 0, bg->n, ctx->stream));
  if (bg->m) {
    k_mark_sources<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->col.p, mask_dev);
    after_launch(ctx, "k_mark_sources");
  }
  sync(ctx);
  GCB_API_END
}

int gcb_partition_cb(gcb_ctx *ctx, const gcb_csr *g, int64_t width, gcb_blocked **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out, "NULL argument");
  DeviceGuard dg(ctx->device);
  gcb_blocked *bg = partition_device(ctx, g, 0, width);
  try {
    to_cb_layout(ctx, bg);
  } catch (...) {
    delete bg;
    throw;
  }
  *out = bg;
  GCB_API_END
}

int gcb_blocked_mark_cb(gcb_ctx *ctx, gcb_blocked *bg) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg, "NULL argument");
  GCB_REQUIRE(bg->direction == 0, "the cb scheme is pull-only");
  for (int64_t b = 0; b <= bg->B; ++b)
    GCB_REQUIRE(bg->h_row_starts[b] == b * bg->n, "cb blocks must hold all n rows");
  GCB_REQUIRE(!bg->derived, "mark the scheme before the first computation");
  bg->cb = true;
  GCB_API_END
}

int gcb_partition_tocab(gcb_ctx *ctx, const gcb_csr *g, int direction, int64_t width,
                        gcb_blocked **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out, "NULL argument");
  DeviceGuard dg(ctx->device);
  *out = partition_device(ctx, g, direction, width);
  GCB_API_END
}

int gcb_blocked_upload(gcb_ctx *ctx, int direction, int64_t width, int64_t n, int64_t m,
                       int64_t num_blocks, const int64_t *row_starts_host,
                       const int64_t *lro_arena_host, const uint32_t *id_map_host,
                       const int64_t *edge_starts_host, const uint32_t *col_arena_host,
                       const double *weight_arena_host_or_null, gcb_blocked **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && out && row_starts_host && edge_starts_host, "NULL argument");
  GCB_REQUIRE(direction == 0 || direction == 1, "direction must be pull or push");
  GCB_REQUIRE(width >= 1 && n >= 0 && m >= 0 && num_blocks >= 0, "bad sizes");
  DeviceGuard dg(ctx->device);
  int64_t B = num_blocks, L = row_starts_host[B];
  GCB_REQUIRE(edge_starts_host[B] == m, "edge_starts disagrees with num_edges");
  for (int64_t b = 0; b < B; ++b)
    GCB_REQUIRE(edge_starts_host[b + 1] - edge_starts_host[b] < (int64_t(1) << 32),
                "block %lld has >= 2^32 edges", (long long)b);
  auto bg = new gcb_blocked();
  try {
    bg->device = ctx->device;
    bg->direction = direction;
    bg->width = width;
    bg->n = n;
    bg->m = m;
    bg->B = B;
    bg->L = L;
    bg->weighted = weight_arena_host_or_null != nullptr;
    bg->h_row_starts.assign(row_starts_host, row_starts_host + B + 1);
    bg->h_edge_starts.assign(edge_starts_host, edge_starts_host + B + 1);
    bg->row_starts.alloc(B + 1);
    bg->edge_starts.alloc(B + 1);
    bg->lro.alloc(L + B + 1);
    bg->id_map.alloc(L);
    bg->col.alloc(m + kColPad);
    GCB_CUDA(cudaMemsetAsync(bg->col.p + m, 0, kColPad * sizeof(uint32_t), ctx->stream));
    h2d(ctx, bg->row_starts.p, row_starts_host, B + 1);
    h2d(ctx, bg->edge_starts.p, edge_starts_host, B + 1);
    {
      // int64 reference lro -> per-block uint32 on the device (range-checked)
      DArray<int64_t> tmp(L + B);
      DArray<unsigned int> bad(1);
      GCB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned int), ctx->stream));
      h2d(ctx, tmp.p, lro_arena_host, L + B);
      if (L + B) {
        k_narrow_lro<<<grid_for(L + B, 256, 65536), 256, 0, ctx->stream>>>(L + B, tmp.p, bg->lro.p,
                                                                            bad.p);
        after_launch(ctx, "k_narrow_lro");
      }
      unsigned int hbad = 0;
      d2h(ctx, &hbad, bad.p, 1);
      sync(ctx);
      GCB_REQUIRE(hbad == 0, "local row offset out of the 32-bit range");
    }
    h2d(ctx, bg->id_map.p, id_map_host, L);
    // col (the bulk of the bytes): from pinned memory, a pull blocking's copy is
    // chunked on a second stream and the out-degree count plus the whole fast
    // execution layout are built under it (gather.cu upload_col_overlapped).
    // Not for a blocking shaped like the cb scheme (every block holds all n
    // rows): gcb_blocked_mark_cb may still follow, before anything is derived.
    cudaPointerAttributes pa;
    const bool pinned_col = m > 0 && cudaPointerGetAttributes(&pa, col_arena_host) == cudaSuccess &&
                            pa.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    bool cb_shaped = B > 0;
    for (int64_t b = 0; b <= B && cb_shaped; ++b) cb_shaped = bg->h_row_starts[b] == b * n;
    if (direction == 0 && pinned_col && !cb_shaped) {
      upload_col_overlapped(ctx, bg, col_arena_host);
    } else {
      h2d(ctx, bg->col.p, col_arena_host, m);
    }
    if (bg->weighted) {
      bg->w.alloc(m + kColPad);
      h2d(ctx, bg->w.p, weight_arena_host_or_null, m);
    }
    sync(ctx);
  } catch (...) {
    delete bg;
    throw;
  }
  *out = bg;
  GCB_API_END
}

int gcb_blocked_info(const gcb_blocked *bg, int *direction, int64_t *width, int64_t *n, int64_t *m,
                     int64_t *num_blocks, int64_t *total_local_rows, int *weighted) {
  GCB_API_BEGIN
  GCB_REQUIRE(bg, "NULL blocking");
  if (direction) *direction = bg->direction;
  if (width) *width = bg->width;
  if (n) *n = bg->n;
  if (m) *m = bg->m;
  if (num_blocks) *num_blocks = bg->B;
  if (total_local_rows) *total_local_rows = bg->L;
  if (weighted) *weighted = bg->weighted ? 1 : 0;
  GCB_API_END
}

int gcb_blocked_download(gcb_ctx *ctx, const gcb_blocked *bg, int64_t *row_starts_host,
                         int64_t *lro_arena_host, uint32_t *id_map_host, int64_t *edge_starts_host,
                         uint32_t *col_arena_host, double *weight_arena_host_or_null) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg, "NULL argument");
  DeviceGuard dg(ctx->device);
  if (row_starts_host) std::copy(bg->h_row_starts.begin(), bg->h_row_starts.end(), row_starts_host);
  if (edge_starts_host)
    std::copy(bg->h_edge_starts.begin(), bg->h_edge_starts.end(), edge_starts_host);
  if (lro_arena_host) {
    std::vector<uint32_t> tmp(bg->L + bg->B);
    d2h(ctx, tmp.data(), bg->lro.p, bg->L + bg->B);
    sync(ctx);
    for (size_t i = 0; i < tmp.size(); ++i) lro_arena_host[i] = tmp[i];
  }
  if (id_map_host) d2h(ctx, id_map_host, bg->id_map.p, bg->L);
  if (col_arena_host) d2h(ctx, col_arena_host, bg->col.p, bg->m);
  if (weight_arena_host_or_null && bg->weighted) d2h(ctx, weight_arena_host_or_null, bg->w.p, bg->m);
  sync(ctx);
  GCB_API_END
}

int gcb_blocked_range_bounds(gcb_ctx *ctx, gcb_blocked *bg, int64_t k, int64_t *bounds_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && bounds_host, "NULL argument");
  GCB_REQUIRE(k >= 1, "range width k must be >= 1");
  DeviceGuard dg(ctx->device);
  int64_t R = bg->n ? ceil_div(bg->n, k) : 0;
  int64_t total = bg->B * (R + 1);
  DArray<int64_t> d(total);
  compute_range_bounds(ctx, bg, k, d.p);
  d2h(ctx, bounds_host, d.p, total);
  sync(ctx);
  GCB_API_END
}

int gcb_blocked_destroy(gcb_blocked *bg) {
  GCB_API_BEGIN
  if (!bg) return GCB_OK;
  DeviceGuard dg(bg->device);
  delete bg;
  GCB_API_END
}

}  // extern "C"

// traversal.cu -- level-synchronous BFS with the push / blocked-pull direction
// switch (traversal.py:93-209), frontier SSSP over integer weights, and weakly
// connected components.
//
// Frontier representation: a dense per-vertex flag array for the next level
// (so the push step needs no atomics and the level queue comes out ascending
// after a stream compaction, exactly the order np.unique / flatnonzero give in
// traversal.py:135 and :172) plus a bitmap of the current frontier for the
// pull step (n/8 bytes: 2 MiB at scale 24, L2-resident).
#include <algorithm>
#include <climits>

#include "gcb_internal.cuh"
#include "tiles.cuh"

namespace gcb {

constexpr int32_t kInfDepth = INT32_MAX;
constexpr int64_t kInfDist = INT64_MAX;

// BFS push step (forward_push_step traversal.py:121-140): k_bfs_push_eb below,
// one thread per frontier edge; unvisited destinations get next[v] = 1.

// --------------------------------------------------------------------------
// BFS blocked pull step (forward_pull_step traversal.py:143-176): per TOCAB
// block of the transpose, each still-unvisited local row scans its in-range
// sources against the frontier bitmap.  Depth only, so the row may stop at
// the first hit (the reference sums the whole row; "sum > 0" == "any").
// Warp per 32 local rows; lanes cooperate on long rows.
// --------------------------------------------------------------------------
__global__ void k_bfs_pull_block(int64_t Lb, const uint32_t *__restrict__ lro_b,
                                 const uint32_t *__restrict__ id_map_b,
                                 const uint32_t *__restrict__ col_b,
                                 const uint32_t *__restrict__ front_bits,
                                 const int32_t *__restrict__ depth, uint8_t *__restrict__ next) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Lb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = id_map_b[i];
    // found in an earlier block of this level (blocks run in order), or visited
    if (next[v] || depth[v] != kInfDepth) continue;
    const uint32_t e1 = lro_b[i + 1];
    for (uint32_t e = lro_b[i]; e < e1; ++e) {
      const uint32_t u = col_b[e];
      if (front_bits[u >> 5] >> (u & 31) & 1u) {
        next[v] = 1;
        break;
      }
    }
  }
}

// Every block's rows in one launch (the per-block launches of a pull level
// were 8 small kernels with a gap each at rmat:24, W = 2^21).  Global row r
// of block b reads lro[r + b] and the col arena from edge_starts[b]; rows
// go in block order, so most rows of later blocks still see the next[] flags
// their vertex got from an earlier block.
constexpr int kMaxPullBlocks = 64;
__global__ void k_bfs_pull_all(int64_t L, int B, const int64_t *__restrict__ row_starts,
                               const int64_t *__restrict__ edge_starts,
                               const uint32_t *__restrict__ lro, const uint32_t *__restrict__ id_map,
                               const uint32_t *__restrict__ col, const uint32_t *__restrict__ front_bits,
                               const int32_t *__restrict__ depth, uint8_t *__restrict__ next) {
  __shared__ int64_t s_rs[kMaxPullBlocks + 1], s_es[kMaxPullBlocks + 1];
  for (int i = threadIdx.x; i <= B; i += blockDim.x) {
    s_rs[i] = row_starts[i];
    s_es[i] = i < B ? edge_starts[i] : 0;
  }
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < L;
       r += (int64_t)gridDim.x * blockDim.x) {
    int b = 0;
    while (b + 1 < B && s_rs[b + 1] <= r) ++b;
    const uint32_t v = id_map[r];
    if (next[v] || depth[v] != kInfDepth) continue;
    const uint32_t *col_b = col + s_es[b];
    const uint32_t e1 = lro[r + b + 1];
    for (uint32_t e = lro[r + b]; e < e1; ++e) {
      const uint32_t u = col_b[e];
      if (front_bits[u >> 5] >> (u & 31) & 1u) {
        next[v] = 1;
        break;
      }
    }
  }
}

static gcb_blocked *default_pull_blocking(gcb_ctx *ctx, const gcb_csr *g,
                                          gcb_blocked **owned) {
  // traversal.py:186-187: partition_tocab(transpose(g), "pull", max(1, n // 8))
  gcb_csr *gt = nullptr;
  int rc = gcb_csr_transpose(ctx, g, &gt);
  if (rc != GCB_OK) fail(rc, "%s", gcb_last_error());
  try {
    *owned = partition_device(ctx, gt, 0, std::max<int64_t>(1, g->n / 8));
  } catch (...) {
    gcb_csr_destroy(gt);
    throw;
  }
  gcb_csr_destroy(gt);
  return *owned;
}

// Level commit (compact_commit below): a CTA of 256 threads x 16 vertices
// (one 16-byte vector of next-frontier flags each) covers 4096 vertices.
constexpr int kCmpT = 256, kCmpV = 16, kCmpChunk = kCmpT * kCmpV;

struct Frontier {
  DArray<uint8_t> next;  // padded to a multiple of kCmpChunk; the pad stays 0
  DArray<uint32_t> flags, pos, bits;
  DArray<uint32_t> qdeg, qoff;  // edge-balanced push: queue degrees and their prefix
  DArray<unsigned long long> degsum;
  explicit Frontier(int64_t n) {
    next.alloc((size_t)ceil_div(n > 0 ? n : 1, kCmpChunk) * kCmpChunk);
    flags.alloc(n + 1);
    pos.alloc(n + 1);
    bits.alloc((n + 31) / 32 + 1);
    qdeg.alloc(n + 1);
    qoff.alloc(n + 1);
    degsum.alloc(1);
  }
};

// What a committed vertex v gets besides its queue slot (null = skip).
struct CommitOps {
  int32_t level = 0;
  int32_t *depth = nullptr;  // depth[v] = level
  double *sigma = nullptr;   // sigma[v] += sig_add[v]; sig_add[v] = 0
  double *sig_add = nullptr;
  uint32_t *bits = nullptr;  // bitmap of the committed level (every word rewritten)
  const int64_t *ro = nullptr;
  unsigned long long *degsum = nullptr;  // += out-degree of every committed vertex
};

// bit k = flag byte k of the 16 is nonzero
__device__ __forceinline__ uint32_t flag_mask16(uint4 w) {
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if ((x[j] >> (8 * b)) & 0xffu) m |= 1u << (4 * j + b);
  return m;
}

__global__ void __launch_bounds__(kCmpT) k_cmp_count(const uint8_t *__restrict__ next,
                                                     uint32_t *__restrict__ cnt) {
  __shared__ uint32_t s_w[kCmpT / 32];
  const int64_t v0 = (int64_t)blockIdx.x * kCmpChunk + threadIdx.x * kCmpV;
  const uint32_t c = __reduce_add_sync(0xffffffffu,
                                       (unsigned)__popc(flag_mask16(*reinterpret_cast<const uint4 *>(next + v0))));
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < kCmpT / 32; ++i) t += s_w[i];
    cnt[blockIdx.x] = t;
  }
}

// queue[off[cta] + rank of v among the CTA's flagged vertices] = v, in vertex
// order; clears the flags and applies op
__global__ void __launch_bounds__(kCmpT) k_cmp_commit(int64_t n, uint8_t *__restrict__ next,
                                                      const uint32_t *__restrict__ off,
                                                      uint32_t *__restrict__ queue, CommitOps op) {
  __shared__ uint32_t s_w[kCmpT / 32];
  __shared__ unsigned long long s_sum;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v0 = (int64_t)blockIdx.x * kCmpChunk + threadIdx.x * kCmpV;
  uint4 *np = reinterpret_cast<uint4 *>(next + v0);
  const uint32_t m = flag_mask16(*np);
  const uint32_t c = __popc(m);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  uint32_t pos = off[blockIdx.x] + incl - c;
  for (int i = 0; i < warp; ++i) pos += s_w[i];
  unsigned long long local = 0;
  if (m) {
    *np = make_uint4(0u, 0u, 0u, 0u);
    // unrolled over the 16 slots (predicated): the out-degree loads of all
    // flagged vertices are in flight together (a serial loop over the set
    // bits waited one row-offset round trip per vertex: 84 us for the third
    // BFS level at rmat:24)
#pragma unroll
    for (int k = 0; k < kCmpV; ++k) {
      if (!((m >> k) & 1u)) continue;
      const int64_t v = v0 + k;
      queue[pos + __popc(m & ((1u << k) - 1u))] = (uint32_t)v;
      if (op.depth) op.depth[v] = op.level;
      if (op.sigma) {
        op.sigma[v] = __dadd_rn(op.sigma[v], op.sig_add[v]);
        op.sig_add[v] = 0.0;
      }
      if (op.degsum) local += (unsigned long long)(__ldg(op.ro + v + 1) - __ldg(op.ro + v));
    }
  }
  if (op.bits) {
    const uint32_t hi = __shfl_down_sync(FULL, m, 1);
    if (!(lane & 1) && v0 < n) op.bits[v0 >> 5] = m | (hi << 16);
  }
  if (op.degsum) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) local += __shfl_down_sync(FULL, local, d);
    if (lane == 0 && local) atomicAdd(&s_sum, local);
    __syncthreads();
    if (threadIdx.x == 0 && s_sum) atomicAdd(op.degsum, s_sum);
  }
}

// Commit the flagged next frontier: count per CTA, scan the CTA counts, write
// (replaces flags -> u32 copy -> n-element scan -> commit: 135-175 us per
// level at rmat:24).  Returns the committed count and, with want_degsum, the
// committed vertices' out-degree sum.
static int64_t compact_commit(gcb_ctx *ctx, Frontier &F, int64_t n, CommitOps op, uint32_t *queue,
                              bool want_degsum, uint64_t *degsum) {
  const int64_t nb = ceil_div(n, kCmpChunk);
  if (nb == 0) return 0;
  k_cmp_count<<<(unsigned)nb, kCmpT, 0, ctx->stream>>>(F.next.p, F.flags.p);
  after_launch(ctx, "k_cmp_count");
  GCB_CUDA(cudaMemsetAsync(F.flags.p + nb, 0, sizeof(uint32_t), ctx->stream));
  cub_exclusive_sum_u32(ctx, F.flags.p, F.pos.p, nb + 1);
  if (want_degsum) {
    GCB_CUDA(cudaMemsetAsync(F.degsum.p, 0, sizeof(unsigned long long), ctx->stream));
    op.degsum = F.degsum.p;
  } else {
    op.degsum = nullptr;
  }
  k_cmp_commit<<<(unsigned)nb, kCmpT, 0, ctx->stream>>>(n, F.next.p, F.pos.p, queue, op);
  after_launch(ctx, "k_cmp_commit");
  uint32_t *h = (uint32_t *)ctx->pinned;
  unsigned long long *hs = (unsigned long long *)((char *)ctx->pinned + 64);
  d2h(ctx, h, F.pos.p + nb, 1);
  if (want_degsum) d2h(ctx, hs, F.degsum.p, 1);
  sync(ctx);
  if (degsum) *degsum = want_degsum ? *hs : 0;
  return (int64_t)*h;
}

// Edge-balanced push (a frontier holding one hub -- vertex 0 of rmat:24 has
// 370K out-edges -- left a warp-per-vertex push on one warp for 3.4 ms):
// qoff = exclusive prefix of the queue's out-degrees; one thread per frontier
// edge finds its vertex by binary search (push levels are small by the
// direction rule, <= capacity/value_bytes edges).
__global__ void k_queue_degrees(int64_t qsize, const uint32_t *__restrict__ queue,
                                const int64_t *__restrict__ ro, uint32_t *__restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= qsize;
       i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = i < qsize ? (uint32_t)(ro[queue[i] + 1] - ro[queue[i]]) : 0u;
}

static void queue_offsets(gcb_ctx *ctx, const gcb_csr *g, const uint32_t *queue, int64_t qsize,
                          Frontier &F) {
  k_queue_degrees<<<grid_for(qsize + 1, 256, 65536), 256, 0, ctx->stream>>>(qsize, queue, g->ro.p,
                                                                         F.qdeg.p);
  after_launch(ctx, "k_queue_degrees");
  cub_exclusive_sum_u32(ctx, F.qdeg.p, F.qoff.p, qsize + 1);
}

// largest i in [0, qsize) with qoff[i] <= idx
__device__ __forceinline__ int64_t locate_edge(uint32_t idx, const uint32_t *__restrict__ qoff,
                                               int64_t qsize) {
  int64_t lo = 0, hi = qsize;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (qoff[mid] <= idx) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k_bfs_push_eb(int64_t total, int64_t qsize, const uint32_t *__restrict__ queue,
                              const uint32_t *__restrict__ qoff, const int64_t *__restrict__ ro,
                              const uint32_t *__restrict__ col, const int32_t *__restrict__ depth,
                              uint8_t *__restrict__ next) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = locate_edge((uint32_t)x, qoff, qsize);
    const uint32_t v = col[ro[queue[i]] + (x - qoff[i])];
    if (depth[v] == kInfDepth) next[v] = 1;
  }
}

// flags -> queue slice at `out`; returns (count, degree sum) after a sync
static void commit_level(gcb_ctx *ctx, const gcb_csr *g, Frontier &F, int32_t level,
                         uint32_t *out, int32_t *depth, int64_t *count, uint64_t *degsum) {
  CommitOps op;
  op.level = level;
  op.depth = depth;
  op.bits = F.bits.p;
  op.ro = g->ro.p;
  *count = compact_commit(ctx, F, g->n, op, out, true, degsum);
}

__global__ void k_fill_i32(int64_t n, int32_t v, int32_t *p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_fill_i64(int64_t n, int64_t v, int64_t *p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_seed(int64_t src, int32_t *depth, uint32_t *queue, uint32_t *bits) {
  depth[src] = 0;
  queue[0] = (uint32_t)src;
  bits[src >> 5] = 1u << (src & 31);
}

// levels_host (optional, pinned): each committed level's queue slice is copied
// back on the copy stream while the next level runs (the caller waits for the
// copy stream)
static void bfs_run(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg, int64_t source, int mode,
                    int64_t capacity, int64_t value_bytes, int32_t *depth_dev, uint32_t *levels_dev,
                    std::vector<int64_t> &level_sizes, std::vector<uint8_t> &dirs,
                    uint32_t *levels_host = nullptr) {
  const int64_t n = g->n;
  if (levels_host && !ctx->copy_stream)
    GCB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  Frontier F(n);
  k_fill_i32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, kInfDepth, depth_dev);
  after_launch(ctx, "k_fill_i32");
  GCB_CUDA(cudaMemsetAsync(F.next.p, 0, F.next.n, ctx->stream));
  GCB_CUDA(cudaMemsetAsync(F.bits.p, 0, ((n + 31) / 32 + 1) * sizeof(uint32_t), ctx->stream));
  k_seed<<<1, 1, 0, ctx->stream>>>(source, depth_dev, levels_dev, F.bits.p);
  after_launch(ctx, "k_seed");
  int64_t qoff = 0, qsize = 1;
  uint64_t work = (uint64_t)0;
  {
    int64_t h[2];
    d2h(ctx, &h[0], g->ro.p + source, 2);
    sync(ctx);
    work = (uint64_t)(h[1] - h[0]);
  }
  level_sizes.push_back(1);
  int32_t level = 0;
  while (qsize > 0) {
    bool pull;
    if (mode == GCB_BFS_FORCE_PUSH) pull = false;
    else if (mode == GCB_BFS_FORCE_PULL) pull = true;
    else pull = (unsigned __int128)work * (unsigned __int128)value_bytes > (unsigned __int128)capacity;
    dirs.push_back(pull ? 1 : 0);
    if (!pull) {
      if (work) {
        queue_offsets(ctx, g, levels_dev + qoff, qsize, F);
        k_bfs_push_eb<<<grid_for((int64_t)work, 256, (int64_t)ctx->num_sms * 32), 256, 0,
                        ctx->stream>>>((int64_t)work, qsize, levels_dev + qoff, F.qoff.p, g->ro.p,
                                       g->col.p, depth_dev, F.next.p);
        after_launch(ctx, "k_bfs_push_eb");
      }
    } else {
      if (bg->B <= kMaxPullBlocks && !getenv("GCB_BFS_PULL_PER_BLOCK")) {
        if (bg->L)
          k_bfs_pull_all<<<grid_for(bg->L, 256, (int64_t)ctx->num_sms * 16), 256, 0,
                           ctx->stream>>>(bg->L, (int)bg->B, bg->row_starts.p, bg->edge_starts.p,
                                          bg->lro.p, bg->id_map.p, bg->col.p, F.bits.p, depth_dev,
                                          F.next.p);
        after_launch(ctx, "k_bfs_pull_all");
      } else {
        for (int64_t b = 0; b < bg->B; ++b) {
          const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
          if (!Lb) continue;
          const int64_t es = bg->h_edge_starts[b];
          k_bfs_pull_block<<<grid_for(Lb, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
              Lb, bg->lro.p + rs + b, bg->id_map.p + rs, bg->col.p + es, F.bits.p, depth_dev,
              F.next.p);
          after_launch(ctx, "k_bfs_pull_block");
        }
      }
    }
    int64_t cnt = 0;
    uint64_t ds = 0;
    commit_level(ctx, g, F, level + 1, levels_dev + qoff + qsize, depth_dev, &cnt, &ds);
    if (levels_host) {
      // commit_level synchronised the stream: the slice is final
      if (qoff == 0)
        GCB_CUDA(cudaMemcpyAsync(levels_host, levels_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                 ctx->copy_stream));
      if (cnt)
        GCB_CUDA(cudaMemcpyAsync(levels_host + qoff + qsize, levels_dev + qoff + qsize,
                                 cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->copy_stream));
    }
    qoff += qsize;
    qsize = cnt;
    work = ds;
    level += 1;
    if (qsize) level_sizes.push_back(qsize);
  }
}

// --------------------------------------------------------------------------
// SSSP (integer weights): frontier Bellman-Ford.  A round relaxes the out-
// edges of every vertex whose distance dropped in the previous round, either
// pushing with 64-bit atomicMin or pulling over the TOCAB blocks of the
// transpose (min over frontier in-neighbours).  The fixpoint is the unique
// shortest-distance vector, independent of direction and relaxation order.
// --------------------------------------------------------------------------

__global__ void k_sssp_push_eb(int64_t total, int64_t qsize, const uint32_t *__restrict__ queue,
                               const uint32_t *__restrict__ qoff, const int64_t *__restrict__ ro,
                               const uint32_t *__restrict__ col, const double *__restrict__ w,
                               long long *__restrict__ dist, uint8_t *__restrict__ next) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = locate_edge((uint32_t)x, qoff, qsize);
    const uint32_t u = queue[i];
    const int64_t k = ro[u] + (x - qoff[i]);
    const uint32_t v = col[k];
    const long long nd = dist[u] + (long long)w[k];
    if (nd < dist[v]) {
      const long long old = atomicMin(&dist[v], nd);
      if (nd < old) next[v] = 1;
    }
  }
}

// Edge-balanced form of the pull round (the thread-per-row kernel above left
// a hub row of ~370K in-edges to one thread: 679 ms for SSSP at rmat:24).
// Warp per 256-edge tile; candidate dist[u] + w for frontier sources u;
// per-row min via tiles.cuh; every row piece lands with a 64-bit atomicMin
// (idempotent, so pieces of rows that cross tiles need no special case).
__global__ void __launch_bounds__(256)
    k_sssp_pull_tiles(const uint32_t *__restrict__ col, const double *__restrict__ w,
                      const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ id_map_b,
                      const uint32_t *__restrict__ tile_row, int64_t es, int64_t ee, int64_t t0,
                      int64_t ntiles, const uint32_t *__restrict__ front_bits,
                      long long *__restrict__ dist, uint8_t *__restrict__ next) {
  constexpr int V = kTileV;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
    const int64_t abase = (t0 + t) * kTileT;
    const uint4 *cp = reinterpret_cast<const uint4 *>(col + abase + lane * V);
    const uint4 ca = __ldcs(cp), cb = __ldcs(cp + 1);
    const uint32_t c[V] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    const uint32_t fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    const uint32_t r0 = tile_row[t];
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < kTileT ? (int)(ee - abase) : kTileT;
    const TileBits tb = tile_bits(fw, llo, lhi, lane);
    long long cand[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      cand[k] = LLONG_MAX;
      if ((tb.vm >> k) & 1u) {
        const uint32_t u = c[k];
        if ((front_bits[u >> 5] >> (u & 31)) & 1u) {
          const long long du = dist[u];
          if (du != LLONG_MAX) cand[k] = du + (long long)w[abase + lane * V + k];
        }
      }
    }
    tile_reduce<long long>(
        cand, tb, r0, lane, LLONG_MAX, [](long long a, long long b) { return a < b ? a : b; },
        [&](uint32_t row, long long x, uint32_t) {
          if (x == LLONG_MAX) return;
          const uint32_t v = id_map_b[row];
          if (x < dist[v]) {
            const long long old = atomicMin(&dist[v], x);
            if (x < old) next[v] = 1;
          }
        });
  }
}

// The pull round, pipelined (k_sssp_pull_tiles left every tile a chain of
// dependent round trips -- col, bitmap word, dist, weight -- and ran 364 us per
// rmat:24 block at 80% long-scoreboard stalls, IPC 0.86):
//   * the next tile's arena words, row-start bits, first row and weights are
//     loaded while this tile is processed;
//   * weights come as one vector per lane: 8 bytes when the graph's weights
//     are integers in [0, 255] (an execution copy, ensure_w8), else 64 bytes
//     of f64 -- streamed for every edge instead of one scattered 8-byte load
//     per frontier edge;
//   * the 8 frontier tests, then the 8 dist loads, are issued before any is
//     used.
template <bool W8>
__global__ void __launch_bounds__(256, 4)
    k_sssp_pull_pipe(const uint32_t *__restrict__ col, const double *__restrict__ w,
                     const uint8_t *__restrict__ w8, const uint32_t *__restrict__ rstart,
                     const uint32_t *__restrict__ id_map_b, const uint32_t *__restrict__ tile_row,
                     int64_t es, int64_t ee, int64_t t0, int64_t ntiles,
                     const uint32_t *__restrict__ front_bits, long long *__restrict__ dist,
                     uint8_t *__restrict__ next) {
  constexpr int V = kTileV;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= ntiles) return;
  auto load = [&](int64_t tt, uint32_t (&c)[V], uint32_t &fw, uint32_t &r0, uint64_t &wb,
                  double (&wd)[V]) {
    const int64_t abase = (t0 + tt) * kTileT;
    const uint4 *cp = reinterpret_cast<const uint4 *>(col + abase + lane * V);
    const uint4 ca = __ldcs(cp), cb = __ldcs(cp + 1);
    c[0] = ca.x; c[1] = ca.y; c[2] = ca.z; c[3] = ca.w;
    c[4] = cb.x; c[5] = cb.y; c[6] = cb.z; c[7] = cb.w;
    fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    r0 = tile_row[tt];
    if (W8) {
      wb = __ldcs(reinterpret_cast<const unsigned long long *>(w8 + abase + lane * V));
    } else {
      const double2 *wp = reinterpret_cast<const double2 *>(w + abase + lane * V);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 x = __ldcs(wp + j);
        wd[2 * j] = x.x;
        wd[2 * j + 1] = x.y;
      }
    }
  };
  uint32_t c[V], fw, r0;
  uint64_t wb = 0;
  double wd[V];
  load(t, c, fw, r0, wb, wd);
  for (; t < ntiles; t += nw) {
    const int64_t abase = (t0 + t) * kTileT;
    const int64_t tn = t + nw;
    uint32_t cn[V], fwn = 0, r0n = 0;
    uint64_t wbn = 0;
    double wdn[V];
    if (tn < ntiles) load(tn, cn, fwn, r0n, wbn, wdn);
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < kTileT ? (int)(ee - abase) : kTileT;
    const TileBits tb = tile_bits(fw, llo, lhi, lane);
    uint32_t fm = 0;  // frontier sources among the lane's valid edges
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const uint32_t u = c[k];
      const uint32_t word = ((tb.vm >> k) & 1u) ? __ldg(front_bits + (u >> 5)) : 0u;
      fm |= ((word >> (u & 31)) & 1u) << k;
    }
    long long du[V];
#pragma unroll
    // through L1 (block 0's hub sources are read by many tiles of a CTA: 6.0 ->
    // 5.8 ms at rmat:24, profiles/r2_sssp_dist_l1_ab.txt).  A line cached before
    // another CTA lowered dist[u] in this launch gives an older, larger distance:
    // still a path length, and the improved u is in the next frontier anyway,
    // so the fixed point (unique shortest distances) is unchanged.
    for (int k = 0; k < V; ++k) du[k] = ((fm >> k) & 1u) ? __ldg(dist + c[k]) : LLONG_MAX;
    long long cand[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const long long wk = W8 ? (long long)((wb >> (8 * k)) & 0xffu) : (long long)wd[k];
      cand[k] = du[k] != LLONG_MAX ? du[k] + wk : LLONG_MAX;
    }
    tile_reduce<long long>(
        cand, tb, r0, lane, LLONG_MAX, [](long long a, long long b) { return a < b ? a : b; },
        [&](uint32_t row, long long x, uint32_t) {
          if (x == LLONG_MAX) return;
          const uint32_t v = id_map_b[row];
          if (x < dist[v]) {
            const long long old = atomicMin(&dist[v], x);
            if (x < old) next[v] = 1;
          }
        });
#pragma unroll
    for (int k = 0; k < V; ++k) {
      c[k] = cn[k];
      if (!W8) wd[k] = wdn[k];
    }
    fw = fwn;
    r0 = r0n;
    wb = wbn;
  }
}

__global__ void k_w8_check(int64_t m, const double *__restrict__ w, unsigned *__restrict__ bad) {
  unsigned b = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double x = w[e];
    b |= !(x >= 0.0 && x <= 255.0 && x == (double)(int)x);
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

__global__ void k_w8_copy(int64_t m, const double *__restrict__ w, uint8_t *__restrict__ w8) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    w8[e] = (uint8_t)(int)w[e];
}

// Byte copy of a blocking's weights when every weight is an integer in
// [0, 255] (U[1, 255] at the configs[3] sizes); built once.
static const uint8_t *ensure_w8(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->w8_state) return bg->w8_state > 0 ? bg->w8.p : nullptr;
  bg->w8_state = -1;
  if (!bg->weighted || bg->m == 0) return nullptr;
  DArray<unsigned> bad(1);
  GCB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned), ctx->stream));
  k_w8_check<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->w.p, bad.p);
  after_launch(ctx, "k_w8_check");
  unsigned h = 1;
  d2h(ctx, &h, bad.p, 1);
  sync(ctx);
  if (h) return nullptr;
  bg->w8.alloc(bg->m + kColPad);
  GCB_CUDA(cudaMemsetAsync(bg->w8.p + bg->m, 0, kColPad, ctx->stream));
  k_w8_copy<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->w.p, bg->w8.p);
  after_launch(ctx, "k_w8_copy");
  bg->w8_state = 1;
  return bg->w8.p;
}

// --------------------------------------------------------------------------
// CC: lock-free union-find, always hooking the larger root under the smaller
// one, so every final root is its component's minimum vertex id.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t uf_find(uint32_t *parent, uint32_t x) {
  while (true) {
    const uint32_t p = __ldcg(parent + x);
    if (p == x) return x;
    const uint32_t gp = __ldcg(parent + p);
    if (gp != p) parent[x] = gp;  // path halving (benign race: gp <= p < x)
    x = p;
  }
}

__global__ void k_cc_init(int64_t n, uint32_t *parent) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    parent[v] = (uint32_t)v;
}

// union of a and b (roots or not): hook the larger root under the smaller
__device__ __forceinline__ void uf_union(uint32_t *parent, uint32_t a, uint32_t b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    const uint32_t hi = a > b ? a : b, lo = a > b ? b : a;
    const uint32_t old = atomicCAS(&parent[hi], hi, lo);
    if (old == hi) return;
    a = old;
    b = lo;
  }
}

// Afforest-style sampling round: every vertex joins its r-th out-neighbour
__global__ void k_cc_sample(int64_t n, int r, const int64_t *__restrict__ ro,
                            const uint32_t *__restrict__ col, uint32_t *parent) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = ro[u] + r;
    if (e < ro[u + 1]) uf_union(parent, (uint32_t)u, col[e]);
  }
}

// pointer jumping: every vertex points at its root
__global__ void k_cc_flatten(int64_t n, uint32_t *parent) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)v;
    while (true) {
      const uint32_t p = __ldcg(parent + x);
      if (p == x) break;
      x = p;
    }
    parent[v] = x;
  }
}

// every edge (u, v), edge-balanced (a hub row no longer serialises on one
// warp); after the sampling rounds most endpoints already point straight at
// the giant root, so the common case is two reads and no atomics.  A warp
// takes a group of kCcGroup consecutive edges and walks them 32 at a time:
// the lanes load the ends of the next 32 rows once, and each lane finds its
// edge's row by a 5-step shuffle binary search over them.  No per-edge source
// array: materialising src[] wrote and re-read 1.07 GB at rmat:24, and its
// warp-per-32-rows writer (k_cc_src) took 0.82 ms behind the hub rows.
constexpr int64_t kCcGroup = 1024;

// grp_row[g] = the row holding edge g * kCcGroup (thread per row; the rows
// of hub vertices cover several groups)
__global__ void k_cc_group_rows(int64_t n, const int64_t *__restrict__ ro,
                                uint32_t *__restrict__ grp_row) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = ro[u], e = ro[u + 1];
    for (int64_t g = (s + kCcGroup - 1) / kCcGroup; g * kCcGroup < e; ++g) grp_row[g] = (uint32_t)u;
  }
}

__global__ void k_cc_edges(int64_t n, int64_t m, const int64_t *__restrict__ ro,
                           const uint32_t *__restrict__ grp_row, const uint32_t *__restrict__ col,
                           uint32_t *parent) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g * kCcGroup < m;
       g += nw) {
    int64_t base = g * kCcGroup;
    const int64_t gend = base + kCcGroup < m ? base + kCcGroup : m;
    // window: the ends of rows uw .. uw + 31 (one coalesced load), kept while
    // it covers the edges; uw starts at the row holding edge `base`
    uint32_t uw = grp_row[g];
    auto ends = [&](uint32_t r0) {
      return (int64_t)r0 + lane + 1 <= n ? __ldg(ro + r0 + lane + 1) : INT64_MAX;
    };
    int64_t rend = ends(uw), wend = __shfl_sync(FULL, rend, 31);
    while (base < gend) {
      // every window row ends at or before base (empty rows): the next 32
      while (wend <= base) {
        uw += 32;
        rend = ends(uw);
        wend = __shfl_sync(FULL, rend, 31);
      }
      // up to 64 edges per pass, two per lane, so two independent load
      // chains are in flight
      const int64_t lim = gend < wend ? gend : wend;
      const int step = lim - base < 64 ? (int)(lim - base) : 64;
      const int64_t p0 = base + lane, p1 = p0 + 32;
      const bool ok0 = lane < step, ok1 = lane + 32 < step;
      const uint32_t v0 = ok0 ? __ldcs(col + p0) : 0u, v1 = ok1 ? __ldcs(col + p1) : 0u;
      // row of an edge: the first window row whose end exceeds it (per-lane
      // shuffle binary search)
      int lo0 = 0, hi0 = 31, lo1 = 0, hi1 = 31;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int mid0 = (lo0 + hi0) >> 1, mid1 = (lo1 + hi1) >> 1;
        const int64_t x0 = __shfl_sync(FULL, rend, mid0), x1 = __shfl_sync(FULL, rend, mid1);
        if (x0 > p0) hi0 = mid0;
        else lo0 = mid0 + 1;
        if (x1 > p1) hi1 = mid1;
        else lo1 = mid1 + 1;
      }
      const uint32_t u0 = uw + (uint32_t)lo0, u1 = uw + (uint32_t)lo1;
      const uint32_t pu0 = ok0 ? __ldcg(parent + u0) : 0u, pv0 = ok0 ? __ldcg(parent + v0) : 0u;
      const uint32_t pu1 = ok1 ? __ldcg(parent + u1) : 0u, pv1 = ok1 ? __ldcg(parent + v1) : 0u;
      if (pu0 != pv0) uf_union(parent, pu0, pv0);
      if (pu1 != pv1) uf_union(parent, pu1, pv1);
      base += step;
    }
  }
}

__global__ void k_cc_compress(int64_t n, uint32_t *parent, unsigned long long *count) {
  unsigned long long local = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)v;
    while (parent[x] != x) x = parent[x];
    parent[v] = x;
    local += (x == (uint32_t)v);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) local += __shfl_down_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(count, local);
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_bfs(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int64_t source, int mode,
            int64_t capacity_bytes, int64_t value_bytes, int32_t *depth_host,
            uint32_t *level_verts_host, int64_t *level_sizes_host, uint8_t *directions_host,
            int64_t max_levels, int64_t *num_levels, int64_t *num_expansions) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && depth_host && num_levels && num_expansions, "NULL argument");
  GCB_REQUIRE(source >= 0 && source < g->n, "source %lld out of range", (long long)source);
  GCB_REQUIRE(mode >= 0 && mode <= 2, "unknown direction mode");
  GCB_REQUIRE(capacity_bytes >= 1 && value_bytes >= 1, "capacity and value size must be positive");
  DeviceGuard dg(ctx->device);
  gcb_blocked *owned = nullptr;
  gcb_blocked *bg = bg_pull;
  if (mode != GCB_BFS_FORCE_PUSH && !bg) bg = default_pull_blocking(ctx, g, &owned);
  try {
    if (bg) {
      GCB_REQUIRE(bg->n == g->n && bg->direction == 0, "g_blocked must be a pull blocking of g");
      ensure_derived(ctx, bg);
    }
    DArray<int32_t> depth(g->n ? g->n : 1);
    DArray<uint32_t> levels(g->n ? g->n : 1);
    std::vector<int64_t> sizes;
    std::vector<uint8_t> dirs;
    {
      ProfScope ps(ctx, 3);  // device span of the traversal (bench.py ms_device)
      bfs_run(ctx, g, bg, source, mode, capacity_bytes, value_bytes, depth.p, levels.p, sizes,
              dirs, level_verts_host);
    }
    d2h(ctx, depth_host, depth.p, g->n);
    sync(ctx);
    if (level_verts_host) GCB_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    *num_levels = (int64_t)sizes.size();
    *num_expansions = (int64_t)dirs.size();
    for (int64_t i = 0; i < (int64_t)sizes.size() && i < max_levels; ++i) {
      if (level_sizes_host) level_sizes_host[i] = sizes[i];
    }
    for (int64_t i = 0; i < (int64_t)dirs.size() && i < max_levels; ++i)
      if (directions_host) directions_host[i] = dirs[i];
  } catch (...) {
    if (owned) gcb_blocked_destroy(owned);
    throw;
  }
  if (owned) gcb_blocked_destroy(owned);
  GCB_API_END
}

int gcb_sssp(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int64_t source, int mode,
             int64_t capacity_bytes, int64_t value_bytes, int64_t *dist_host,
             uint8_t *directions_host, int64_t max_rounds, int64_t *rounds) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && dist_host && rounds, "NULL argument");
  GCB_REQUIRE(g->weighted, "SSSP needs integer edge weights on the graph");
  GCB_REQUIRE(source >= 0 && source < g->n, "source %lld out of range", (long long)source);
  GCB_REQUIRE(mode >= 0 && mode <= 2, "unknown direction mode");
  DeviceGuard dg(ctx->device);
  gcb_blocked *bg = bg_pull;
  if (mode == GCB_BFS_FORCE_PULL) GCB_REQUIRE(bg, "force-pull SSSP needs a weighted pull blocking");
  if (bg) {
    GCB_REQUIRE(bg->n == g->n && bg->direction == 0 && bg->weighted,
                "g_blocked must be a weighted pull blocking of g");
    ensure_row_bits(ctx, bg);
  }
  const uint8_t *w8 = bg ? ensure_w8(ctx, bg) : nullptr;
  const int64_t n = g->n;
  DArray<int64_t> dist(n ? n : 1);
  DArray<uint32_t> queue(n ? n : 1);
  Frontier F(n);
  int64_t qsize = 1, r = 0;
  {
  ProfScope ps(ctx, 3);  // device span of the traversal (bench.py ms_device)
  k_fill_i64<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, kInfDist, dist.p);
  after_launch(ctx, "k_fill_i64");
  GCB_CUDA(cudaMemsetAsync(F.next.p, 0, F.next.n, ctx->stream));
  GCB_CUDA(cudaMemsetAsync(F.bits.p, 0, ((n + 31) / 32 + 1) * sizeof(uint32_t), ctx->stream));
  {
    int64_t zero = 0;
    uint32_t s32 = (uint32_t)source, bit = 1u << (source & 31);
    h2d(ctx, dist.p + source, &zero, 1);
    h2d(ctx, queue.p, &s32, 1);
    h2d(ctx, F.bits.p + (source >> 5), &bit, 1);
    sync(ctx);
  }
  uint64_t work;
  {
    int64_t h[2];
    d2h(ctx, &h[0], g->ro.p + source, 2);
    sync(ctx);
    work = (uint64_t)(h[1] - h[0]);
  }
  while (qsize > 0) {
    bool pull;
    if (mode == GCB_BFS_FORCE_PUSH || !bg) pull = false;
    else if (mode == GCB_BFS_FORCE_PULL) pull = true;
    else pull = (unsigned __int128)work * (unsigned __int128)value_bytes > (unsigned __int128)capacity_bytes;
    if (directions_host && r < max_rounds) directions_host[r] = pull ? 1 : 0;
    if (!pull) {
      if (work) {
        queue_offsets(ctx, g, queue.p, qsize, F);
        k_sssp_push_eb<<<grid_for((int64_t)work, 256, (int64_t)ctx->num_sms * 32), 256, 0,
                         ctx->stream>>>((int64_t)work, qsize, queue.p, F.qoff.p, g->ro.p, g->col.p,
                                        g->w.p, (long long *)dist.p, F.next.p);
        after_launch(ctx, "k_sssp_push_eb");
      }
    } else {
      for (int64_t b = 0; b < bg->B; ++b) {
        const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
        if (!Lb) continue;
        const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
        const unsigned gsp = grid_for(nt * 32, 256, (int64_t)ctx->num_sms * 8);
        const char *sp = getenv("GCB_SSSP_PULL");  // A/B knob: 0 = the round-1 kernel
        if (sp && sp[0] == '0') {
          k_sssp_pull_tiles<<<gsp, 256, 0, ctx->stream>>>(
              bg->col.p, bg->w.p, bg->rstart.p, bg->id_map.p + rs, bg->tile_row.p + tb,
              bg->h_edge_starts[b], bg->h_edge_starts[b + 1], bg->h_tile_t0[b], nt, F.bits.p,
              (long long *)dist.p, F.next.p);
        } else if (w8) {
          k_sssp_pull_pipe<true><<<gsp, 256, 0, ctx->stream>>>(
              bg->col.p, nullptr, w8, bg->rstart.p, bg->id_map.p + rs, bg->tile_row.p + tb,
              bg->h_edge_starts[b], bg->h_edge_starts[b + 1], bg->h_tile_t0[b], nt, F.bits.p,
              (long long *)dist.p, F.next.p);
        } else {
          k_sssp_pull_pipe<false><<<gsp, 256, 0, ctx->stream>>>(
              bg->col.p, bg->w.p, nullptr, bg->rstart.p, bg->id_map.p + rs, bg->tile_row.p + tb,
              bg->h_edge_starts[b], bg->h_edge_starts[b + 1], bg->h_tile_t0[b], nt, F.bits.p,
              (long long *)dist.p, F.next.p);
        }
        after_launch(ctx, "k_sssp_pull");
      }
    }
    // compact next flags into the queue
    CommitOps op;
    op.bits = F.bits.p;
    op.ro = g->ro.p;
    uint64_t ds = 0;
    qsize = compact_commit(ctx, F, n, op, queue.p, true, &ds);
    work = ds;
    ++r;
  }
  }
  d2h(ctx, dist_host, dist.p, n);
  sync(ctx);
  *rounds = r;
  GCB_API_END
}

int gcb_cc(gcb_ctx *ctx, const gcb_csr *g, uint32_t *labels_host, int64_t *num_components) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && labels_host, "NULL argument");
  DeviceGuard dg(ctx->device);
  const int64_t n = g->n;
  DArray<uint32_t> parent(n ? n : 1);
  DArray<unsigned long long> cnt(1);
  {
  ProfScope ps(ctx, 3);  // device span of the labelling (bench.py ms_device)
  GCB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
  k_cc_init<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, parent.p);
  after_launch(ctx, "k_cc_init");
  if (g->m) {
    // Afforest (Sutton et al.): two sampled neighbours per vertex, flatten,
    // then the remaining edges with a cheap already-joined test
    for (int r = 0; r < 2; ++r) {
      k_cc_sample<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, r, g->ro.p, g->col.p,
                                                                  parent.p);
      after_launch(ctx, "k_cc_sample");
      k_cc_flatten<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, parent.p);
      after_launch(ctx, "k_cc_flatten");
    }
    const int64_t groups = (g->m + kCcGroup - 1) / kCcGroup;
    DArray<uint32_t> grp_row(groups);
    k_cc_group_rows<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, g->ro.p, grp_row.p);
    after_launch(ctx, "k_cc_group_rows");
    k_cc_edges<<<grid_for(groups * 32, 256, (int64_t)ctx->num_sms * 64), 256, 0, ctx->stream>>>(
        n, g->m, g->ro.p, grp_row.p, g->col.p, parent.p);
    after_launch(ctx, "k_cc_edges");
  }
  k_cc_compress<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, parent.p, cnt.p);
  after_launch(ctx, "k_cc_compress");
  }
  unsigned long long hc = 0;
  d2h(ctx, labels_host, parent.p, n);
  d2h(ctx, &hc, cnt.p, 1);
  sync(ctx);
  if (num_components) *num_components = (int64_t)hc;
  GCB_API_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Single level steps with path counts (forward_push_step traversal.py:121-140,
// forward_pull_step traversal.py:143-176).  sigma values are integer-valued
// doubles (< 2^53), so the atomic sums are exact in any order.
// ---------------------------------------------------------------------------
namespace gcb {


// edge-balanced form (see k_bfs_push_eb)
__global__ void k_step_push_eb(int64_t total, int64_t qsize, const uint32_t *__restrict__ queue,
                               const uint32_t *__restrict__ qoff, const int64_t *__restrict__ ro,
                               const uint32_t *__restrict__ col, const int32_t *__restrict__ depth,
                               const double *__restrict__ sigma, uint8_t *__restrict__ next,
                               double *__restrict__ sig_add) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = locate_edge((uint32_t)x, qoff, qsize);
    const uint32_t u = queue[i];
    const uint32_t v = col[ro[u] + (x - qoff[i])];
    if (depth[v] == kInfDepth) {
      next[v] = 1;
      if (sigma) atomicAdd(sig_add + v, sigma[u]);
    }
  }
}

// per block: unvisited rows sum sigma (or 1) over in-range frontier sources
__global__ void k_step_pull(int64_t Lb, const uint32_t *__restrict__ lro_b,
                            const uint32_t *__restrict__ id_map_b, const uint32_t *__restrict__ col_b,
                            const uint32_t *__restrict__ front_bits, const int32_t *__restrict__ depth,
                            const double *__restrict__ sigma, uint8_t *__restrict__ next,
                            double *__restrict__ sig_add) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Lb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = id_map_b[i];
    if (depth[v] != kInfDepth) continue;
    double s = 0.0;
    for (uint32_t e = lro_b[i]; e < lro_b[i + 1]; ++e) {
      const uint32_t u = col_b[e];
      if (front_bits[u >> 5] >> (u & 31) & 1u) {
        if (!sigma) {
          s = 1.0;
          break;
        }
        s += sigma[u];
      }
    }
    if (s > 0.0) {
      next[v] = 1;
      if (sigma) atomicAdd(sig_add + v, s);
    }
  }
}

__global__ void k_set_bits(int64_t q, const uint32_t *__restrict__ queue, uint32_t *__restrict__ bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicOr(bits + (queue[i] >> 5), 1u << (queue[i] & 31));
}

}  // namespace gcb

extern "C" int gcb_bfs_step(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int direction,
                            int32_t *depth_host, double *sigma_host_or_null,
                            const uint32_t *frontier_host, int64_t frontier_size, int32_t level,
                            uint32_t *next_host, int64_t *next_size) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && depth_host && next_size && (frontier_host || frontier_size == 0), "NULL argument");
  GCB_REQUIRE(direction == 0 || direction == 1, "direction must be push (0) or pull (1)");
  GCB_REQUIRE(direction == 0 ? g != nullptr : bg_pull != nullptr, "missing graph for the step");
  DeviceGuard dg(ctx->device);
  const int64_t n = direction == 0 ? g->n : bg_pull->n;
  DArray<int32_t> depth(n ? n : 1);
  DArray<double> sigma, sig_add;
  DArray<uint32_t> queue(frontier_size ? frontier_size : 1), out(n ? n : 1);
  Frontier F(n);
  h2d(ctx, depth.p, depth_host, n);
  h2d(ctx, queue.p, frontier_host, frontier_size);
  GCB_CUDA(cudaMemsetAsync(F.next.p, 0, F.next.n, ctx->stream));
  if (sigma_host_or_null) {
    sigma.alloc(n ? n : 1);
    sig_add.alloc(n ? n : 1);
    h2d(ctx, sigma.p, sigma_host_or_null, n);
    GCB_CUDA(cudaMemsetAsync(sig_add.p, 0, (n ? n : 1) * sizeof(double), ctx->stream));
  }
  double *sg = sigma_host_or_null ? sigma.p : nullptr;
  if (direction == 0) {
    if (frontier_size) {
      queue_offsets(ctx, g, queue.p, frontier_size, F);
      uint32_t total = 0;
      d2h(ctx, &total, F.qoff.p + frontier_size, 1);
      sync(ctx);
      if (total) {
        k_step_push_eb<<<grid_for(total, 256, (int64_t)ctx->num_sms * 32), 256, 0, ctx->stream>>>(
            total, frontier_size, queue.p, F.qoff.p, g->ro.p, g->col.p, depth.p, sg, F.next.p,
            sig_add.p);
        after_launch(ctx, "k_step_push_eb");
      }
    }
  } else {
    gcb_blocked *bg = bg_pull;
    GCB_REQUIRE(bg->direction == 0, "g_blocked must be a pull blocking");
    ensure_derived(ctx, bg);
    GCB_CUDA(cudaMemsetAsync(F.bits.p, 0, ((n + 31) / 32 + 1) * sizeof(uint32_t), ctx->stream));
    if (frontier_size) {
      k_set_bits<<<grid_for(frontier_size, 256, 4096), 256, 0, ctx->stream>>>(frontier_size, queue.p,
                                                                             F.bits.p);
      after_launch(ctx, "k_set_bits");
    }
    for (int64_t b = 0; b < bg->B; ++b) {
      const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
      if (!Lb) continue;
      k_step_pull<<<grid_for(Lb, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          Lb, bg->lro.p + rs + b, bg->id_map.p + rs, bg->col.p + bg->h_edge_starts[b], F.bits.p,
          depth.p, sg, F.next.p, sig_add.p);
      after_launch(ctx, "k_step_pull");
    }
  }
  CommitOps op;
  op.level = level + 1;
  op.depth = depth.p;
  op.sigma = sg;
  op.sig_add = sg ? sig_add.p : nullptr;
  const int64_t cnt = compact_commit(ctx, F, n, op, out.p, false, nullptr);
  *next_size = cnt;
  d2h(ctx, depth_host, depth.p, n);
  if (sigma_host_or_null) d2h(ctx, sigma_host_or_null, sigma.p, n);
  if (next_host) d2h(ctx, next_host, out.p, cnt);
  sync(ctx);
  GCB_API_END
}

// ---------------------------------------------------------------------------
// Betweenness centrality (bc / bc_single_source / bc_backward,
// traversal.py:212-278): a forward sweep with path counts (the BFS steps
// above, push or blocked pull per choose_direction) then the dependency pass
// deepest level first:
//   delta[v] = sum over out-edges v->w with depth[w] == depth[v] + 1 of
//              (sigma[v] / sigma[w]) * (1 + delta[w])        (traversal.py:224-234)
// delta[source] = 0; centrality accumulates delta over the sources in order.
// Exact mode sums each vertex's out-edges sequentially in CSR order (the
// np.bincount order of traversal.py:233) -> bit-identical; fast mode reduces
// each vertex's edges across a warp (|err| ~ 1e-16 relative).
// ---------------------------------------------------------------------------
namespace gcb {

__device__ __forceinline__ double bc_term(double sv, double sw, double dw) {
  return __dmul_rn(__ddiv_rn(sv, sw), __dadd_rn(1.0, dw));
}

// thread per vertex of the level, sequential in CSR order (exact); vertices
// with more than kExactShort out-edges are k_bc_back_exact_long's
__global__ void k_bc_back_exact(int64_t cnt, const uint32_t *__restrict__ verts, int32_t level,
                                const int64_t *__restrict__ ro, const uint32_t *__restrict__ col,
                                const int32_t *__restrict__ depth, const double *__restrict__ sigma,
                                double *__restrict__ delta) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = verts[i];
    if (ro[v + 1] - ro[v] > (int64_t)kExactShort) continue;
    const double sv = sigma[v];
    double acc = 0.0;
    for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
      const uint32_t w = col[e];
      if (depth[w] == level + 1) acc = __dadd_rn(acc, bc_term(sv, sigma[w], delta[w]));
    }
    delta[v] = __dadd_rn(delta[v], acc);
  }
}

// Exact dependency sum of a vertex with many out-edges (a hub took ~100 ms on
// one thread, a dependent round trip per edge).  A warp per such vertex: the
// lanes load steps of 256 edges (8 each), software-pipelined -- column ids two
// steps ahead, depth/sigma/delta of the successors one step ahead -- turn them
// into terms (a non-successor's term is +0.0, which leaves the non-negative
// sum unchanged bit for bit), stage them in the warp's shared-memory slot,
// and the chain adds them in CSR order, as the reference loop does.
__global__ void k_bc_back_exact_long(int64_t cnt, const uint32_t *__restrict__ verts,
                                     int32_t level, const int64_t *__restrict__ ro,
                                     const uint32_t *__restrict__ col,
                                     const int32_t *__restrict__ depth,
                                     const double *__restrict__ sigma,
                                     double *__restrict__ delta) {
  __shared__ double s_buf[8][256];  // 256-thread CTAs: one slot per warp
  double *buf = s_buf[threadIdx.x >> 5];
  constexpr uint32_t kNone = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += nw) {
    const uint32_t v = verts[i];
    const int64_t e0 = ro[v], e1 = ro[v + 1];
    if (e1 - e0 <= (int64_t)kExactShort) continue;
    const double sv = sigma[v];
    auto load_cols = [&](int64_t base, uint32_t (&c)[8]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t e = base + q * 32 + lane;
        c[q] = e < e1 ? col[e] : kNone;
      }
    };
    auto load_succ = [&](const uint32_t (&c)[8], int (&d)[8], double (&sw)[8], double (&dw)[8]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        d[q] = -1;
        if (c[q] != kNone) {
          d[q] = depth[c[q]];
          sw[q] = sigma[c[q]];
          dw[q] = delta[c[q]];
        }
      }
    };
    uint32_t c1[8], c2[8];
    int d0[8], d1[8];
    double s0[8], s1[8], w0[8], w1[8];
    load_cols(e0, c1);
    load_succ(c1, d0, s0, w0);  // step 0
    load_cols(e0 + 256, c1);    // step 1's columns
    double acc = 0.0;
    for (int64_t base = e0; base < e1; base += 256) {
      if (base + 256 < e1) {
        load_succ(c1, d1, s1, w1);  // step s+1
        load_cols(base + 512, c2);  // step s+2
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        buf[q * 32 + lane] = d0[q] == level + 1 ? bc_term(sv, s0[q], w0[q]) : 0.0;
      __syncwarp();
      const int n = (int)(e1 - base < 256 ? e1 - base : 256);
      if (n == 256) {
#pragma unroll 64
        for (int k = 0; k < 256; ++k) acc = __dadd_rn(acc, buf[k]);
      } else {
        for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, buf[k]);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        d0[q] = d1[q];
        s0[q] = s1[q];
        w0[q] = w1[q];
        c1[q] = c2[q];
      }
    }
    if (lane == 0) delta[v] = __dadd_rn(delta[v], acc);
  }
}

// fast mode, long vertices: a CTA per vertex (from the level's compacted
// list of long vertices), each thread sums a strided share of the edges with
// 4 gathers in flight, then a block reduction -- no add chain, so a hub's
// 370K out-edges no longer set the pass's critical path
__global__ void k_bc_long_flags(int64_t cnt, const uint32_t *__restrict__ verts,
                                const int64_t *__restrict__ ro, uint32_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = verts[i];
    flag[i] = ro[v + 1] - ro[v] > (int64_t)kExactShort ? 1u : 0u;
  }
}

__global__ void k_bc_compact(int64_t cnt, const uint32_t *__restrict__ verts,
                             const uint32_t *__restrict__ flag, const uint32_t *__restrict__ pos,
                             uint32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[pos[i]] = verts[i];
}

__global__ void __launch_bounds__(256)
    k_bc_back_cta(int64_t nlong, const uint32_t *__restrict__ longv, int32_t level,
                  const int64_t *__restrict__ ro, const uint32_t *__restrict__ col,
                  const int32_t *__restrict__ depth, const double *__restrict__ sigma,
                  double *__restrict__ delta) {
  __shared__ double red[8];
  for (int64_t j = blockIdx.x; j < nlong; j += gridDim.x) {
    const uint32_t v = longv[j];
    const int64_t e0 = ro[v], e1 = ro[v + 1];
    const double sv = sigma[v];
    double acc = 0.0;
    int64_t e = e0 + threadIdx.x;
    for (; e + 3 * 256 < e1; e += 4 * 256) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = col[e + k * 256];
      int d[4];
      double sw[4], dw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        d[k] = depth[w[k]];
        sw[k] = sigma[w[k]];
        dw[k] = delta[w[k]];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (d[k] == level + 1) acc += bc_term(sv, sw[k], dw[k]);
    }
    for (; e < e1; e += 256) {
      const uint32_t w = col[e];
      if (depth[w] == level + 1) acc += bc_term(sv, sigma[w], delta[w]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += red[k];
      delta[v] = delta[v] + t;
    }
    __syncthreads();
  }
}

// warp per vertex of the level (fast)
__global__ void k_bc_back_warp(int64_t cnt, const uint32_t *__restrict__ verts, int32_t level,
                               const int64_t *__restrict__ ro, const uint32_t *__restrict__ col,
                               const int32_t *__restrict__ depth, const double *__restrict__ sigma,
                               double *__restrict__ delta) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += nw) {
    const uint32_t v = verts[i];
    const double sv = sigma[v];
    double acc = 0.0;
    for (int64_t e = ro[v] + lane; e < ro[v + 1]; e += 32) {
      const uint32_t w = col[e];
      if (depth[w] == level + 1) acc += bc_term(sv, sigma[w], delta[w]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) delta[v] = delta[v] + acc;
  }
}

// centrality += delta (delta[source] counted as 0), delta cleared for the next source
__global__ void k_bc_accum(int64_t n, int64_t source, double *__restrict__ delta,
                           double *__restrict__ cent) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const double d = v == source ? 0.0 : delta[v];
    cent[v] = __dadd_rn(cent[v], d);
    delta[v] = 0.0;
  }
}

// blocked pull step with path counts on warp tiles: every row sums sigma over
// its frontier in-neighbours (tiles.cuh); unvisited rows with a hit are
// discovered and take the sum (forward_pull_step traversal.py:143-176)
__global__ void __launch_bounds__(256)
    k_bc_pull_tiles(const uint32_t *__restrict__ col, const uint32_t *__restrict__ rstart,
                    const uint32_t *__restrict__ id_map_b, const uint32_t *__restrict__ tile_row,
                    int64_t es, int64_t ee, int64_t t0, int64_t ntiles,
                    const uint32_t *__restrict__ front_bits, const int32_t *__restrict__ depth,
                    const double *__restrict__ sigma, uint8_t *__restrict__ next,
                    double *__restrict__ sig_add) {
  constexpr int V = kTileV;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
    const int64_t abase = (t0 + t) * kTileT;
    const uint4 *cp = reinterpret_cast<const uint4 *>(col + abase + lane * V);
    const uint4 ca = __ldcs(cp), cb = __ldcs(cp + 1);
    const uint32_t c[V] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    const uint32_t fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    const uint32_t r0 = tile_row[t];
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < kTileT ? (int)(ee - abase) : kTileT;
    const TileBits tb = tile_bits(fw, llo, lhi, lane);
    double s[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const uint32_t u = c[k];
      s[k] = (((tb.vm >> k) & 1u) && ((front_bits[u >> 5] >> (u & 31)) & 1u)) ? sigma[u] : 0.0;
    }
    tile_reduce<double>(
        s, tb, r0, lane, 0.0, [](double a, double b) { return a + b; },
        [&](uint32_t row, double x, uint32_t) {
          if (!(x > 0.0)) return;
          const uint32_t v = id_map_b[row];
          if (depth[v] != kInfDepth) return;
          next[v] = 1;
          atomicAdd(sig_add + v, x);
        });
  }
}

__global__ void k_bc_seed(int64_t src, int32_t *depth, double *sigma, uint32_t *queue,
                          uint32_t *bits) {
  depth[src] = 0;
  sigma[src] = 1.0;
  queue[0] = (uint32_t)src;
  bits[src >> 5] = 1u << (src & 31);
}

// dependency pass over per-level ascending vertex lists (levels[off[l]:off[l+1]])
static void bc_backward_dev(gcb_ctx *ctx, const gcb_csr *g, const int32_t *depth,
                            const double *sigma, const uint32_t *levels,
                            const std::vector<int64_t> &off, bool exact, double *delta) {
  const int64_t L = (int64_t)off.size() - 1;  // number of non-empty levels
  DArray<uint32_t> flag, pos, longv;  // fast mode: the level's long vertices
  for (int64_t l = L - 2; l >= 0; --l) {
    const int64_t cnt = off[l + 1] - off[l];
    if (!cnt) continue;
    // fast: short vertices a thread each, long ones a CTA each (16 ms for 4
    // sources at rmat:24); exact: the order-keeping kernels (23 ms); the older
    // warp-per-vertex fast form (31 ms) stays behind GCB_BC_WARP=1
    const char *wenv = getenv("GCB_BC_WARP");
    if (!exact && !(wenv && wenv[0] == '1')) {
      // fast: thread per short vertex, a CTA per long one
      k_bc_back_exact<<<grid_for(cnt, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          cnt, levels + off[l], (int32_t)l, g->ro.p, g->col.p, depth, sigma, delta);
      after_launch(ctx, "k_bc_back_exact");
      flag.ensure(cnt + 1);
      pos.ensure(cnt + 1);
      longv.ensure(cnt);
      k_bc_long_flags<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, levels + off[l],
                                                                         g->ro.p, flag.p);
      after_launch(ctx, "k_bc_long_flags");
      GCB_CUDA(cudaMemsetAsync(flag.p + cnt, 0, sizeof(uint32_t), ctx->stream));
      cub_exclusive_sum_u32(ctx, flag.p, pos.p, cnt + 1);
      uint32_t *hn = (uint32_t *)ctx->pinned;
      d2h(ctx, hn, pos.p + cnt, 1);
      sync(ctx);
      const int64_t nl = *hn;
      if (nl) {
        k_bc_compact<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, levels + off[l],
                                                                         flag.p, pos.p, longv.p);
        after_launch(ctx, "k_bc_compact");
        k_bc_back_cta<<<(unsigned)std::min<int64_t>(nl, (int64_t)ctx->num_sms * 8), 256, 0,
                        ctx->stream>>>(nl, longv.p, (int32_t)l, g->ro.p, g->col.p, depth, sigma,
                                       delta);
        after_launch(ctx, "k_bc_back_cta");
      }
    } else if (exact || !(wenv && wenv[0] == '1')) {
      k_bc_back_exact<<<grid_for(cnt, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          cnt, levels + off[l], (int32_t)l, g->ro.p, g->col.p, depth, sigma, delta);
      after_launch(ctx, "k_bc_back_exact");
      k_bc_back_exact_long<<<grid_for(cnt * 32, 256, (int64_t)ctx->num_sms * 16), 256, 0,
                             ctx->stream>>>(cnt, levels + off[l], (int32_t)l, g->ro.p, g->col.p,
                                            depth, sigma, delta);
      after_launch(ctx, "k_bc_back_exact_long");
    } else {
      k_bc_back_warp<<<grid_for(cnt * 32, 256, (int64_t)ctx->num_sms * 16), 256, 0, ctx->stream>>>(
          cnt, levels + off[l], (int32_t)l, g->ro.p, g->col.p, depth, sigma, delta);
      after_launch(ctx, "k_bc_back_warp");
    }
  }
}

// forward sweep with path counts; fills depth / sigma / per-level queues
static void bc_forward_dev(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg, int64_t source, int mode,
                           int64_t capacity, int64_t value_bytes, Frontier &F, int32_t *depth,
                           double *sigma, double *sig_add, uint32_t *levels,
                           std::vector<int64_t> &off, std::vector<uint8_t> *dirs = nullptr) {
  const int64_t n = g->n;
  k_fill_i32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, kInfDepth, depth);
  after_launch(ctx, "k_fill_i32");
  GCB_CUDA(cudaMemsetAsync(sigma, 0, n * sizeof(double), ctx->stream));
  GCB_CUDA(cudaMemsetAsync(F.bits.p, 0, ((n + 31) / 32 + 1) * sizeof(uint32_t), ctx->stream));
  k_bc_seed<<<1, 1, 0, ctx->stream>>>(source, depth, sigma, levels, F.bits.p);
  after_launch(ctx, "k_bc_seed");
  uint64_t work;
  {
    int64_t *h = (int64_t *)ctx->pinned;
    d2h(ctx, h, g->ro.p + source, 2);
    sync(ctx);
    work = (uint64_t)(h[1] - h[0]);
  }
  off.assign(1, 0);
  off.push_back(1);
  int64_t qoff = 0, qsize = 1;
  int32_t level = 0;
  while (qsize > 0) {
    bool pull;
    if (mode == GCB_BFS_FORCE_PUSH || !bg) pull = false;
    else if (mode == GCB_BFS_FORCE_PULL) pull = true;
    else pull = (unsigned __int128)work * (unsigned __int128)value_bytes > (unsigned __int128)capacity;
    if (dirs) dirs->push_back(pull ? 1 : 0);
    if (!pull) {
      if (work) {
        queue_offsets(ctx, g, levels + qoff, qsize, F);
        k_step_push_eb<<<grid_for((int64_t)work, 256, (int64_t)ctx->num_sms * 32), 256, 0,
                         ctx->stream>>>((int64_t)work, qsize, levels + qoff, F.qoff.p, g->ro.p,
                                        g->col.p, depth, sigma, F.next.p, sig_add);
        after_launch(ctx, "k_step_push_eb");
      }
    } else {
      for (int64_t b = 0; b < bg->B; ++b) {
        const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
        if (!Lb) continue;
        const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
        k_bc_pull_tiles<<<grid_for(nt * 32, 256, (int64_t)ctx->num_sms * 8), 256, 0,
                          ctx->stream>>>(bg->col.p, bg->rstart.p, bg->id_map.p + rs,
                                         bg->tile_row.p + tb, bg->h_edge_starts[b],
                                         bg->h_edge_starts[b + 1], bg->h_tile_t0[b], nt, F.bits.p,
                                         depth, sigma, F.next.p, sig_add);
        after_launch(ctx, "k_bc_pull_tiles");
      }
    }
    CommitOps op;
    op.level = level + 1;
    op.depth = depth;
    op.sigma = sigma;
    op.sig_add = sig_add;
    op.bits = F.bits.p;
    op.ro = g->ro.p;
    uint64_t ds = 0;
    const int64_t cnt = compact_commit(ctx, F, n, op, levels + qoff + qsize, true, &ds);
    qoff += qsize;
    qsize = cnt;
    work = ds;
    ++level;
    if (qsize) off.push_back(qoff + qsize);
  }
}

__global__ void k_level_hist(int64_t n, const int32_t *__restrict__ depth,
                             unsigned long long *__restrict__ hist, int32_t maxd) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = depth[v];
    if (d >= 0 && d <= maxd) atomicAdd(hist + d, 1ull);
  }
}

__global__ void k_depth_keys(int64_t n, const int32_t *__restrict__ depth, uint32_t *__restrict__ key,
                             uint32_t *__restrict__ val) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = (uint32_t)depth[v];  // INF_DEPTH sorts last
    val[v] = (uint32_t)v;
  }
}

__global__ void k_max_depth(int64_t n, const int32_t *__restrict__ depth, int *__restrict__ out) {
  int mx = -1;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = depth[v];
    if (d != kInfDepth && d > mx) mx = d;
  }
  atomicMax(out, mx);
}

}  // namespace gcb

extern "C" int gcb_bc(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, const int64_t *sources_host,
                      int64_t num_sources, int mode, int64_t capacity_bytes, int64_t value_bytes,
                      uint32_t flags, double *centrality_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && centrality_host && (sources_host || num_sources == 0), "NULL argument");
  GCB_REQUIRE(mode >= 0 && mode <= 2, "unknown direction mode");
  DeviceGuard dg(ctx->device);
  const int64_t n = g->n;
  for (int64_t i = 0; i < num_sources; ++i)
    GCB_REQUIRE(sources_host[i] >= 0 && sources_host[i] < n, "source %lld out of range",
                (long long)sources_host[i]);
  gcb_blocked *owned = nullptr;
  gcb_blocked *bg = bg_pull;
  try {
    if (mode != GCB_BFS_FORCE_PUSH && !bg && n > 0) bg = default_pull_blocking(ctx, g, &owned);
    if (bg) {
      GCB_REQUIRE(bg->n == n && bg->direction == 0, "g_blocked must be a pull blocking of g");
      ensure_row_bits(ctx, bg);
    }
    DArray<int32_t> depth(n ? n : 1);
    DArray<double> sigma(n ? n : 1), sig_add(n ? n : 1), delta(n ? n : 1), cent(n ? n : 1);
    DArray<uint32_t> levels(n ? n : 1);
    Frontier F(n);
    GCB_CUDA(cudaMemsetAsync(F.next.p, 0, F.next.n, ctx->stream));
    GCB_CUDA(cudaMemsetAsync(sig_add.p, 0, (n ? n : 1) * sizeof(double), ctx->stream));
    GCB_CUDA(cudaMemsetAsync(delta.p, 0, (n ? n : 1) * sizeof(double), ctx->stream));
    GCB_CUDA(cudaMemsetAsync(cent.p, 0, (n ? n : 1) * sizeof(double), ctx->stream));
    const bool exact = flags & GCB_FLAG_EXACT;
    std::vector<int64_t> off;
    for (int64_t i = 0; i < num_sources; ++i) {
      const int64_t s = sources_host[i];
      bc_forward_dev(ctx, g, bg, s, mode, capacity_bytes, value_bytes, F, depth.p, sigma.p,
                     sig_add.p, levels.p, off);
      bc_backward_dev(ctx, g, depth.p, sigma.p, levels.p, off, exact, delta.p);
      k_bc_accum<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, s, delta.p, cent.p);
      after_launch(ctx, "k_bc_accum");
    }
    if (n) d2h(ctx, centrality_host, cent.p, n);
    sync(ctx);
  } catch (...) {
    if (owned) gcb_blocked_destroy(owned);
    throw;
  }
  if (owned) gcb_blocked_destroy(owned);
  GCB_API_END
}

// bc_single_source (traversal.py:239-254) on the device: the forward sweep with
// path counts and the dependency pass, results copied back once (the
// step-by-step form moved depth/sigma across PCIe on every level: 84 ms at
// rmat:22 from the hub)
extern "C" int gcb_bc_single_source(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull,
                                    int64_t source, int mode, int64_t capacity_bytes,
                                    int64_t value_bytes, uint32_t flags, double *delta_host,
                                    int32_t *depth_host, double *sigma_host,
                                    uint32_t *level_verts_host, int64_t *level_sizes_host,
                                    uint8_t *directions_host, int64_t max_levels,
                                    int64_t *num_levels, int64_t *num_expansions) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && delta_host && depth_host && sigma_host && num_levels && num_expansions,
              "NULL argument");
  GCB_REQUIRE(mode >= 0 && mode <= 2, "unknown direction mode");
  const int64_t n = g->n;
  GCB_REQUIRE(source >= 0 && source < n, "source %lld out of range", (long long)source);
  DeviceGuard dg(ctx->device);
  gcb_blocked *owned = nullptr;
  gcb_blocked *bg = bg_pull;
  try {
    if (mode != GCB_BFS_FORCE_PUSH && !bg) bg = default_pull_blocking(ctx, g, &owned);
    if (bg) {
      GCB_REQUIRE(bg->n == n && bg->direction == 0, "g_blocked must be a pull blocking of g");
      ensure_row_bits(ctx, bg);
    }
    DArray<int32_t> depth(n);
    DArray<double> sigma(n), sig_add(n), delta(n);
    DArray<uint32_t> levels(n);
    Frontier F(n);
    GCB_CUDA(cudaMemsetAsync(F.next.p, 0, F.next.n, ctx->stream));
    GCB_CUDA(cudaMemsetAsync(sig_add.p, 0, n * sizeof(double), ctx->stream));
    GCB_CUDA(cudaMemsetAsync(delta.p, 0, n * sizeof(double), ctx->stream));
    std::vector<int64_t> off;
    std::vector<uint8_t> dirs;
    bc_forward_dev(ctx, g, bg, source, mode, capacity_bytes, value_bytes, F, depth.p, sigma.p,
                   sig_add.p, levels.p, off, &dirs);
    bc_backward_dev(ctx, g, depth.p, sigma.p, levels.p, off, flags & GCB_FLAG_EXACT, delta.p);
    const double zero = 0.0;
    h2d(ctx, delta.p + source, &zero, 1);
    const int64_t nl = (int64_t)off.size() - 1;
    d2h(ctx, delta_host, delta.p, n);
    d2h(ctx, depth_host, depth.p, n);
    d2h(ctx, sigma_host, sigma.p, n);
    if (level_verts_host && nl > 0) d2h(ctx, level_verts_host, levels.p, off.back());
    sync(ctx);
    *num_levels = nl;
    *num_expansions = (int64_t)dirs.size();
    for (int64_t i = 0; i < nl && i < max_levels; ++i)
      if (level_sizes_host) level_sizes_host[i] = off[i + 1] - off[i];
    for (int64_t i = 0; i < (int64_t)dirs.size() && i < max_levels; ++i)
      if (directions_host) directions_host[i] = dirs[i];
  } catch (...) {
    if (owned) gcb_blocked_destroy(owned);
    throw;
  }
  if (owned) gcb_blocked_destroy(owned);
  GCB_API_END
}

extern "C" int gcb_bc_backward(gcb_ctx *ctx, const gcb_csr *g, const int32_t *depth_host,
                               const double *sigma_host, int64_t source, uint32_t flags,
                               double *delta_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && depth_host && sigma_host && delta_host, "NULL argument");
  DeviceGuard dg(ctx->device);
  const int64_t n = g->n;
  if (n == 0) return GCB_OK;
  DArray<int32_t> depth(n);
  DArray<double> sigma(n), delta(n);
  DArray<uint32_t> k1(n), k2(n), v1(n), v2(n);
  DArray<int> mx(1);
  h2d(ctx, depth.p, depth_host, n);
  h2d(ctx, sigma.p, sigma_host, n);
  GCB_CUDA(cudaMemsetAsync(delta.p, 0, n * sizeof(double), ctx->stream));
  GCB_CUDA(cudaMemsetAsync(mx.p, 0xff, sizeof(int), ctx->stream));  // -1
  k_max_depth<<<grid_for(n, 256, 4096), 256, 0, ctx->stream>>>(n, depth.p, mx.p);
  after_launch(ctx, "k_max_depth");
  int maxd = -1;
  d2h(ctx, &maxd, mx.p, 1);
  sync(ctx);
  if (maxd >= 0) {
    // per-level ascending vertex lists: stable sort by depth (INF last)
    k_depth_keys<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, depth.p, k1.p, v1.p);
    after_launch(ctx, "k_depth_keys");
    uint32_t *rk = nullptr, *rv = nullptr;
    cub_sort_pairs_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, n, 32, &rk, &rv);
    DArray<unsigned long long> hist(maxd + 1);
    GCB_CUDA(cudaMemsetAsync(hist.p, 0, (maxd + 1) * sizeof(unsigned long long), ctx->stream));
    k_level_hist<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, depth.p, hist.p, maxd);
    after_launch(ctx, "k_level_hist");
    std::vector<unsigned long long> h(maxd + 1);
    d2h(ctx, h.data(), hist.p, maxd + 1);
    sync(ctx);
    std::vector<int64_t> off(1, 0);
    for (int d = 0; d <= maxd; ++d) off.push_back(off.back() + (int64_t)h[d]);
    bc_backward_dev(ctx, g, depth.p, sigma.p, rv, off, flags & GCB_FLAG_EXACT, delta.p);
    const double zero = 0.0;
    if (source >= 0 && source < n) h2d(ctx, delta.p + source, &zero, 1);
  }
  d2h(ctx, delta_host, delta.p, n);
  sync(ctx);
  GCB_API_END
}

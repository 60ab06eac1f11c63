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
#include <cstdlib>

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
// One warp per local row.
__global__ void k_relabel_block(int64_t Lb, const uint32_t *__restrict__ lro_b,
                                const uint32_t *__restrict__ id_map_b,
                                const uint32_t *__restrict__ col_b, const uint32_t *__restrict__ perm,
                                uint32_t *__restrict__ rows_out, uint32_t *__restrict__ cols_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Lb; r += nw) {
    const uint32_t s = lro_b[r], e = lro_b[r + 1];
    const uint32_t d = perm[id_map_b[r]];
    for (uint32_t i = s + lane; i < e; i += 32) {
      rows_out[i] = d;
      cols_out[i] = perm[col_b[i]];
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

template <typename T>
__global__ void k_permute_out(int64_t n, const uint32_t *__restrict__ perm,
                              const T *__restrict__ y_new, T *__restrict__ y) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    y[v] = y_new[perm[v]];
}

// Tiering: the copy costs a few passes over the edges (tens of ms at
// rmat:24) and saves ~0.07 ms per iteration there, so it pays only on a graph
// that stays resident.  A graph is promoted once it has run
// GCB_RELABEL_AFTER fast-mode iterations (default 20; 0 = immediately); a
// graph uploaded for one short call never is.
bool relabel_enabled(gcb_blocked *bg, uint32_t flags, int64_t upcoming_iters) {
  if (flags & (GCB_FLAG_EXACT | GCB_FLAG_NO_RELABEL)) return false;
  if (bg->direction != 0 || bg->m == 0 || bg->n >= (int64_t(1) << 32)) return false;
  if (bg->is_relabeled || bg->cb) return false;
  const char *env = getenv("GCB_NO_RELABEL");
  if (env && env[0] && env[0] != '0') return false;
  if (bg->rl) return true;
  const char *after = getenv("GCB_RELABEL_AFTER");
  const int64_t threshold = after ? atoll(after) : 20;
  if (bg->fast_iters >= threshold) return true;
  bg->fast_iters += upcoming_iters;
  return false;
}

gcb_blocked *ensure_relabeled(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->rl) return bg->rl;
  ensure_derived(ctx, bg);
  const int64_t n = bg->n, m = bg->m;
  // 1. permutation: stable sort of (deg desc, id asc)
  bg->rl_perm.alloc(n);
  {
    DArray<uint32_t> k1(n), k2(n), v1(n), v2(n);
    GCB_CUDA(cudaMemcpyAsync(k1.p, bg->deg.p, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    k_iota_u32<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, v1.p);
    after_launch(ctx, "k_iota_u32");
    uint32_t *rk = nullptr, *inv = nullptr;
    cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, n, &rk, &inv);
    k_invert<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, inv, bg->rl_perm.p);
    after_launch(ctx, "k_invert");
  }
  // 2. renumbered edge list (destination, source) from the arenas
  gcb_csr *csr = nullptr;
  {
    DArray<uint32_t> rows(m), cols(m);
    for (int64_t b = 0; b < bg->B; ++b) {
      const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
      const int64_t es = bg->h_edge_starts[b];
      if (Lb == 0) continue;
      k_relabel_block<<<grid_for(Lb * 32, 256, 65536), 256, 0, ctx->stream>>>(
          Lb, bg->lro.p + rs + b, bg->id_map.p + rs, bg->col.p + es, bg->rl_perm.p, rows.p + es,
          cols.p + es);
      after_launch(ctx, "k_relabel_block");
    }
    // 3. canonical CSR of the renumbered transpose, then the same TOCAB cut
    csr = csr_from_device_edges(ctx, n, m, rows.p, cols.p, bg->weighted ? bg->w.p : nullptr);
  }
  try {
    gcb_blocked *rl = partition_device(ctx, csr, 0, bg->width);
    rl->is_relabeled = true;
    bg->rl = rl;
  } catch (...) {
    gcb_csr_destroy(csr);
    throw;
  }
  gcb_csr_destroy(csr);
  return bg->rl;
}

void permute_in(gcb_ctx *ctx, const gcb_blocked *bg, const double *x, double *x_new) {
  k_permute_in<double><<<grid_for(bg->n, 256, 65536), 256, 0, ctx->stream>>>(bg->n, bg->rl_perm.p,
                                                                            x, x_new);
  after_launch(ctx, "k_permute_in");
}

void permute_out(gcb_ctx *ctx, const gcb_blocked *bg, const double *y_new, double *y) {
  k_permute_out<double><<<grid_for(bg->n, 256, 65536), 256, 0, ctx->stream>>>(bg->n, bg->rl_perm.p,
                                                                             y_new, y);
  after_launch(ctx, "k_permute_out");
}

}  // namespace gcb

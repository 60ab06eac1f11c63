// gather.cu -- the fast TOCAB pull gather (K2) that accumulates straight into
// a dense per-vertex vector, optionally with the block's hottest sources
// staged in shared memory.
//
// Bottleneck model (ncu, profiles/): a random 8-byte gather through L1TEX
// costs one wavefront per distinct 128-byte line, ~2 SM cycles each when a
// warp load touches 32 lines, so the plain gather runs at ~1 edge per 2 cycles
// per SM (L1/TEX throughput 59-79%, DRAM 13-15%).  Two levers:
//   * memory-level parallelism: the next tile's tile_row / col_idx / row-end
//     chunk are prefetched while the current tile's gathers are in flight;
//   * hot staging: the top-K sources (by out-degree) of each TOCAB block are
//     copied into shared memory once per launch; R-MAT blocks are
//     self-similar, so the top ~16-26K sources of a 2^22-wide block carry
//     ~40-49% of its edges (scale 24), and those edges become LDS.
// Execution layout (built once, ensure_exec): xcol = col arena with every
// hot source replaced by 0x80000000 | slot; hot_ids[b][slot] = source id.
// The reference arena (col) is kept for downloads and the other kernels.
//
// Rows that cross a tile boundary are combined with f64 atomics (RED) on the
// destination's sum; all other rows use a plain read-modify-write (a row's
// destination appears once per block and blocks are stream-ordered).  The
// order of the RED contributions is not fixed, so this path is deterministic
// only up to reassociation of long rows (|err| ~ 1e-16 relative); the exact
// mode (pr.cu, k_pull_exact) is the bit-reproducible path.
#include <cstdlib>

#include "gcb_internal.cuh"
#include "ldst.cuh"

namespace gcb {

#ifndef GCB_GWARPS
#define GCB_GWARPS 32
#endif
constexpr int kGWarps = GCB_GWARPS;  // warps per CTA (1 CTA per SM)
constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kHotBit = 0x80000000u;
constexpr int kEndsPerWarp = kTileT + 32;

struct TileGeom {
  int64_t abase, lbase, llo, lhi;
};

__device__ __forceinline__ TileGeom tile_geom(int64_t t, int64_t t0, int64_t es, int64_t ee) {
  TileGeom g;
  g.abase = (t0 + t) * kTileT;
  g.lbase = g.abase - es;
  g.llo = g.lbase > 0 ? g.lbase : 0;
  g.lhi = (g.lbase + kTileT < ee - es) ? g.lbase + kTileT : ee - es;
  return g;
}

template <bool WGT, bool HOT>
__global__ void __launch_bounds__(kGWarps * 32, 1)
    k_gather(const uint32_t *__restrict__ xcol, const double *__restrict__ w,
             const uint32_t *__restrict__ lro_b, const uint32_t *__restrict__ id_map_b,
             const uint32_t *__restrict__ tile_row, int64_t es, int64_t ee, int64_t t0,
             int64_t ntiles, uint32_t Lb, const double *__restrict__ vals,
             const double *__restrict__ hotval_b, int hot_k, double *__restrict__ out) {
  constexpr int V = kTileV;
  extern __shared__ __align__(16) unsigned char smem[];
  double *s_hot = reinterpret_cast<double *>(smem);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *ends = reinterpret_cast<uint32_t *>(smem + (size_t)hot_k * 8) + wid * kEndsPerWarp;
  const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
  const unsigned FULL = 0xffffffffu;
  const int64_t stride = (int64_t)gridDim.x * kGWarps;

  if (HOT) {
    const double2 *src = reinterpret_cast<const double2 *>(hotval_b);
    double2 *dst = reinterpret_cast<double2 *>(s_hot);
    for (int i = threadIdx.x; i < hot_k / 2; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
  }

  int64_t t = (int64_t)blockIdx.x * kGWarps + wid;
  if (t < ntiles) {
  // software pipeline: tile t's row id, col chunk and first row-end chunk
  uint32_t r0 = tile_row[t];
  uint4 ca, cb;
  {
    const TileGeom g = tile_geom(t, t0, es, ee);
    const uint4 *cp = reinterpret_cast<const uint4 *>(xcol + g.abase + lane * V);
    ca = ld_stream_u4(cp, pol_stream);
    cb = ld_stream_u4(cp + 1, pol_stream);
  }
  uint32_t e0 = (r0 + 1 + lane <= Lb) ? lro_b[r0 + 1 + lane] : 0xffffffffu;
  uint32_t r0_start = lro_b[r0];

  for (; t < ntiles; t += stride) {
    const TileGeom g = tile_geom(t, t0, es, ee);
    const int64_t tn = t + stride;
    const bool has_next = tn < ntiles;
    uint32_t r0n = 0;
    uint4 can = make_uint4(0, 0, 0, 0), cbn = make_uint4(0, 0, 0, 0);
    if (has_next) {
      r0n = tile_row[tn];
      const TileGeom gn = tile_geom(tn, t0, es, ee);
      const uint4 *cp = reinterpret_cast<const uint4 *>(xcol + gn.abase + lane * V);
      can = ld_stream_u4(cp, pol_stream);
      cbn = ld_stream_u4(cp + 1, pol_stream);
    }

    // gathers of the current tile
    const uint32_t c[V] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    const int64_t q0 = g.lbase + (int64_t)lane * V;
    double v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t q = q0 + k;
      double x = 0.0;
      if (q >= g.llo && q < g.lhi) {
        if (HOT && (c[k] & kHotBit)) x = s_hot[c[k] & ~kHotBit];
        else x = ld_keep(vals + c[k], pol_keep);
      }
      v[k] = x;
    }
    if (WGT) {
      const double2 *wp = reinterpret_cast<const double2 *>(w + g.abase + lane * V);
#pragma unroll
      for (int k2 = 0; k2 < V / 2; ++k2) {
        const double2 ww = ld_stream_d2(wp + k2, pol_stream);
        v[2 * k2] = __dmul_rn(ww.x, v[2 * k2]);
        v[2 * k2 + 1] = __dmul_rn(ww.y, v[2 * k2 + 1]);
      }
    }
    // next tile's row-end chunk + row start (depends on r0n, overlaps the gathers)
    uint32_t e0n = 0xffffffffu, r0n_start = 0;
    if (has_next) {
      e0n = (r0n + 1 + lane <= Lb) ? lro_b[r0n + 1 + lane] : 0xffffffffu;
      r0n_start = lro_b[r0n];
    }

    // row-end table of the current tile; j_last = row holding lhi - 1
    ends[lane] = e0;
    unsigned below = __ballot_sync(FULL, e0 < (uint32_t)g.lhi);
    int j_last = __popc(below), nload = 32;
    while (below == FULL && nload < kTileT) {
      const uint32_t idx = r0 + 1 + nload + lane;
      const uint32_t e = idx <= Lb ? lro_b[idx] : 0xffffffffu;
      ends[nload + lane] = e;
      below = __ballot_sync(FULL, e < (uint32_t)g.lhi);
      j_last += __popc(below);
      nload += 32;
    }
    __syncwarp();
    const bool first_partial = (int64_t)r0_start < g.llo;
    const bool last_partial = (int64_t)ends[j_last] > g.lhi;

    auto emit = [&](int jj, double x) {
      const uint32_t vid = id_map_b[r0 + jj];
      if ((jj == 0 && first_partial) || (jj == j_last && last_partial)) {
        atomicAdd(out + vid, x);
      } else {
        out[vid] = __dadd_rn(out[vid], x);
      }
    };

    const int64_t qf = q0 > g.llo ? q0 : g.llo;
    const bool lane_valid = (qf < g.lhi) && (q0 + V > g.llo);
    int j = 0;
    if (lane_valid) {
      int lo = 0, hi = nload;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)ends[mid] > qf) hi = mid;
        else lo = mid + 1;
      }
      j = lo;
    }
    const int head_j = j;
    double head_sum = 0.0, acc = 0.0;
    bool head_closed = false;
    uint32_t endj = ends[j];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t q = q0 + k;
      if (q < g.llo || q >= g.lhi) continue;
      if ((uint32_t)q >= endj) {
        if (j == head_j) {
          head_sum = acc;
          head_closed = true;
        } else {
          emit(j, acc);
        }
        acc = 0.0;
        ++j;
        endj = ends[j];
      }
      acc = __dadd_rn(acc, v[k]);
    }
    int key = lane_valid ? j : -1 - lane;
    double val = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int k2 = __shfl_up_sync(FULL, key, d);
      const double v2 = __shfl_up_sync(FULL, val, d);
      if (lane >= d && k2 == key) val = __dadd_rn(v2, val);
    }
    int pk = __shfl_up_sync(FULL, key, 1);
    const double pv = __shfl_up_sync(FULL, val, 1);
    if (lane == 0) pk = -1000;
    int nh = __shfl_down_sync(FULL, lane_valid ? head_j : -1000, 1);
    if (lane == 31) nh = -1000;
    if (lane_valid) {
      if (head_closed) emit(head_j, (pk == head_j) ? __dadd_rn(pv, head_sum) : head_sum);
      if (nh != j) emit(j, val);
    }
    __syncwarp();
    // rotate the pipeline
    r0 = r0n;
    ca = can;
    cb = cbn;
    e0 = e0n;
    r0_start = r0n_start;
  }
  }  // t < ntiles
}

// hotval[b][s] = vals[hot_ids[b][s]]
__global__ void k_fill_hot(int64_t count, const uint32_t *__restrict__ ids,
                           const double *__restrict__ vals, double *__restrict__ hotval) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = ids[i];
    hotval[i] = v != kNone ? vals[v] : 0.0;
  }
}

__global__ void k_iota_range(int64_t lo, int64_t cnt, uint32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(lo + i);
}

__global__ void k_pick_hot(int64_t K, int64_t cnt, const uint32_t *__restrict__ keys,
                           const uint32_t *__restrict__ ids, uint32_t *__restrict__ hot_ids_b,
                           uint32_t *__restrict__ slot_of) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < K;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (s < cnt && keys[s] > 0) {
      hot_ids_b[s] = ids[s];
      slot_of[ids[s]] = (uint32_t)s;
    } else {
      hot_ids_b[s] = kNone;
    }
  }
}

__global__ void k_recode(int64_t m, const uint32_t *__restrict__ col,
                         const uint32_t *__restrict__ slot_of, uint32_t *__restrict__ xcol) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = col[e];
    const uint32_t s = slot_of[c];
    xcol[e] = s != kNone ? (kHotBit | s) : c;
  }
}

static size_t ends_bytes() { return (size_t)kGWarps * kEndsPerWarp * sizeof(uint32_t); }

template <bool WGT, bool HOT>
static void set_smem_attr(size_t bytes) {
  static size_t done = 0;
  if (bytes > done) {
    GCB_CUDA(cudaFuncSetAttribute(k_gather<WGT, HOT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done = bytes;
  }
}

// Hot-table size: GCB_HOT_K (slots per block; 0 disables), else what fits in
// the opt-in shared memory next to the row-end tables.
static int64_t hot_slots(gcb_ctx *ctx) {
  int optin = 0;
  GCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  int64_t K = ((int64_t)optin - (int64_t)ends_bytes() - 256) / 8;
  const char *env = getenv("GCB_HOT_K");
  if (env) {
    const int64_t want = atoll(env);
    if (want < K) K = want;
  } else if (K > 8192) {
    // measured at scale 24 (W = 2^22): 8K slots beat 0 / 16K / 24K -- a larger
    // carve-out shrinks the L1 that the cold gathers and row tables rely on
    K = 8192;
  }
  return K < 0 ? 0 : (K / 64) * 64;
}

void ensure_exec(gcb_ctx *ctx, gcb_blocked *bg) {
  ensure_derived(ctx, bg);
  if (bg->xready) return;
  int64_t K = hot_slots(ctx);
  const bool can = bg->direction == 0 && bg->n < (int64_t(1) << 31) && bg->m > 0 && K >= 64;
  if (can) {
    const int64_t B = bg->B, n = bg->n;
    if (bg->width < K) K = ((bg->width + 63) / 64) * 64;  // whole slice fits: every source hot
    bg->hot_k = K;
    bg->hot_ids.alloc(B * K);
    bg->hotval.alloc(B * K);
    DArray<uint32_t> slot_of(n), k1(bg->width), k2(bg->width), v1(bg->width), v2(bg->width);
    GCB_CUDA(cudaMemsetAsync(slot_of.p, 0xff, n * sizeof(uint32_t), ctx->stream));
    for (int64_t b = 0; b < B; ++b) {
      const int64_t lo = b * bg->width, hi = (lo + bg->width < n) ? lo + bg->width : n;
      const int64_t cnt = hi - lo;
      GCB_CUDA(cudaMemcpyAsync(k1.p, bg->deg.p + lo, cnt * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, ctx->stream));
      k_iota_range<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(lo, cnt, v1.p);
      after_launch(ctx, "k_iota_range");
      uint32_t *rk = nullptr, *rv = nullptr;
      cub_sort_pairs_desc_u32_u32(ctx, k1.p, k2.p, v1.p, v2.p, cnt, &rk, &rv);
      k_pick_hot<<<grid_for(K, 256, 4096), 256, 0, ctx->stream>>>(K, cnt, rk, rv,
                                                                  bg->hot_ids.p + b * K, slot_of.p);
      after_launch(ctx, "k_pick_hot");
    }
    bg->xcol.alloc(bg->m + kColPad);
    GCB_CUDA(cudaMemsetAsync(bg->xcol.p + bg->m, 0, kColPad * sizeof(uint32_t), ctx->stream));
    k_recode<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->col.p, slot_of.p,
                                                                   bg->xcol.p);
    after_launch(ctx, "k_recode");
    sync(ctx);
  } else {
    bg->hot_k = 0;
  }
  bg->xready = true;
}

template <bool WGT, bool HOT>
static void launch_gather(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, const double *vals,
                          double *out) {
  const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
  const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
  const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
  const int hot_k = HOT ? (int)bg->hot_k : 0;
  const size_t smem = (size_t)hot_k * 8 + ends_bytes();
  set_smem_attr<WGT, HOT>(smem);
  int64_t grid = ceil_div(nt, kGWarps);
  if (grid > ctx->num_sms) grid = ctx->num_sms;
  k_gather<WGT, HOT><<<(unsigned)(grid < 1 ? 1 : grid), kGWarps * 32, smem, ctx->stream>>>(
      HOT ? bg->xcol.p : bg->col.p, WGT ? bg->w.p : nullptr, bg->lro.p + rs + b, bg->id_map.p + rs,
      bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt, (uint32_t)Lb, vals,
      HOT ? bg->hotval.p + b * bg->hot_k : nullptr, hot_k, out);
  after_launch(ctx, "k_gather");
}

static void fill_hot(gcb_ctx *ctx, gcb_blocked *bg, const double *vals) {
  ProfScope ps(ctx, 3);
  const int64_t cnt = bg->B * bg->hot_k;
  k_fill_hot<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, bg->hot_ids.p, vals,
                                                                 bg->hotval.p);
  after_launch(ctx, "k_fill_hot");
}

// out[v] += sum over the rows of v in every block (block order); the caller
// clears out first.
void gather_accum(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights,
                  uint32_t flags, double *out) {
  ensure_exec(ctx, bg);
  const bool wgt = use_weights && bg->weighted;
  const bool hot = bg->hot_k > 0;
  if (hot) fill_hot(ctx, bg, vals);
  (void)flags;
  for (int64_t b = 0; b < bg->B; ++b) {
    if (bg->h_row_starts[b + 1] == bg->h_row_starts[b]) continue;
    ProfScope ps(ctx, 0);
    if (wgt && hot) launch_gather<true, true>(ctx, bg, b, vals, out);
    else if (wgt) launch_gather<true, false>(ctx, bg, b, vals, out);
    else if (hot) launch_gather<false, true>(ctx, bg, b, vals, out);
    else launch_gather<false, false>(ctx, bg, b, vals, out);
  }
}

}  // namespace gcb

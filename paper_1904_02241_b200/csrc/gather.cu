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

// ---------------------------------------------------------------------------
// k_pull_prefix: the gather for the degree-ordered layout (relabel.cu).
//
// ncu (profiles/r1b_*) put the hot-staged kernel at the L1TEX sector ceiling
// (~0.9 global sectors per SM cycle; a pure random-gather microbenchmark tops
// out at 0.95, scripts/mb_gather.cu), so every change here removes sectors or
// instructions:
//   * hot table = the block's first H sources (the hottest, by construction)
//     copied contiguously into shared memory: no recoded arena, no fill pass;
//   * col_idx streamed with one 256-bit load per lane (8 edges = one full
//     32-byte sector; the two 128-bit loads it replaces touched 2 sectors);
//   * row boundaries come from a 1-bit-per-edge row-start bitmap (32 bytes per
//     256-edge tile, one sector per warp) instead of lro tables + a binary
//     search in shared memory.  Local rows are never empty (blocking.py:
//     189-201), so row(q) = tile_row + #row starts in (first, q].
// Reduction and emission are as in k_gather: in-lane runs, a segmented
// shuffle scan over lane tails, plain read-modify-write for rows inside the
// tile and f64 RED for rows that cross a tile boundary.
// ---------------------------------------------------------------------------
// One source value: the block's hot prefix from shared memory, everything
// else from L2 (evict_last keeps the block's value slice resident; no L1
// allocation, cold lines would only evict each other).  Predicated loads, no
// branch: the compiler's if/else cost a BSSY/BSYNC pair per edge.
__device__ __forceinline__ double gather_one(const double *vals, uint32_t c, uint32_t lo,
                                             uint32_t hot, uint32_t s_hot, uint64_t pol) {
  const uint32_t h = c - lo;
  double x;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.lt.u32 p, %1, %2;\n\t"
      "@p ld.shared.f64 %0, [%3];\n\t"
      "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%4], %5;\n\t}"
      : "=d"(x)
      : "r"(h), "r"(hot), "r"(s_hot + h * 8u), "l"(vals + c), "l"(pol));
  return x;
}

// ASSIGN: out is all zero before this launch (first block of the pass), so a
// row that lies inside one tile is stored (out[v] = x) instead of
// read-modify-written -- no dependent load on the emit path.
template <bool WGT, bool ASSIGN, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    k_pull_prefix(const uint32_t *__restrict__ col, const double *__restrict__ w,
                  const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ id_map_b,
                  const uint32_t *__restrict__ tile_row, int64_t es, int64_t ee, int64_t t0,
                  int64_t ntiles, uint32_t lo, int hot, uint32_t Lb,
                  const double *__restrict__ vals, double *__restrict__ out) {
  constexpr int V = kTileV;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // per-warp cache of the destination ids of the tile's first 32 rows
  uint32_t *s_ids = reinterpret_cast<uint32_t *>(smem) + wid * 32;
  double *s_hot = reinterpret_cast<double *>(smem + NW * 32 * sizeof(uint32_t));
  const uint32_t s_hot_addr = (uint32_t)__cvta_generic_to_shared(s_hot);
  const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
  const unsigned FULL = 0xffffffffu;
  const int64_t stride = (int64_t)gridDim.x * NW;

  for (int i = threadIdx.x; i < hot; i += blockDim.x) s_hot[i] = __ldcg(vals + lo + i);
  __syncthreads();

  int64_t t = (int64_t)blockIdx.x * NW + wid;
  if (t >= ntiles) return;
  // software pipeline: tile t's col chunk, bitmap words, first row and its ids
  uint32_t c[V], fw, r0, idl;
  {
    const int64_t abase = (t0 + t) * kTileT;
    ld_stream_u32x8(col + abase + lane * V, pol_stream, c);
    fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    r0 = tile_row[t];
    idl = r0 + lane < Lb ? id_map_b[r0 + lane] : 0u;
  }
  for (; t < ntiles; t += stride) {
    const int64_t abase = (t0 + t) * kTileT;
    const int64_t tn = t + stride;
    const bool has_next = tn < ntiles;
    uint32_t cn[V] = {0, 0, 0, 0, 0, 0, 0, 0}, fwn = 0, r0n = 0;
    if (has_next) {
      const int64_t nb = (t0 + tn) * kTileT;
      ld_stream_u32x8(col + nb + lane * V, pol_stream, cn);
      fwn = rstart[(nb >> 5) + (lane < 8 ? lane : 8)];
      r0n = tile_row[tn];
    }
    // gathers first: everything below overlaps their latency
    double v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = gather_one(vals, c[k], lo, (uint32_t)hot, s_hot_addr, pol_keep);
    if (WGT) {
      double ww[V];
      ld_stream_f64x4(w + abase + lane * V, pol_stream, ww);
      ld_stream_f64x4(w + abase + lane * V + 4, pol_stream, ww + 4);
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = __dmul_rn(ww[k], v[k]);
    }
    // valid tile positions [llo, lhi); lane's valid k in [a, z)
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < kTileT ? (int)(ee - abase) : kTileT;
    const int a = llo - lane * V, z = lhi - lane * V;
    const uint32_t vm = (z <= 0 || a >= V) ? 0u
                        : ((0xffu >> (V - (z < V ? z : V))) & (0xffu << (a > 0 ? a : 0)));
    // row-start bits of the lane's edges (valid ones; the tile's first valid
    // edge dropped -- its row is r0)
    const uint32_t wl = __shfl_sync(FULL, fw, lane >> 2);
    uint32_t bits = (wl >> ((lane & 3) * 8)) & vm;
    if (a >= 0 && a < V) bits &= ~(1u << a);
    const bool first_start = (__shfl_sync(FULL, fw, llo >> 5) >> (llo & 31)) & 1u;
    const bool last_cont = (lhi == kTileT) && !(__shfl_sync(FULL, fw, 8) & 1u);
    // next tile's id cache (its first row is known by now)
    uint32_t idn = 0;
    if (has_next && r0n + lane < Lb) idn = id_map_b[r0n + lane];

    if (__all_sync(FULL, bits == 0)) {
      // the whole tile lies in row r0: a plain warp reduction, one emit
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < V; ++k) acc = __dadd_rn(acc, ((vm >> k) & 1u) ? v[k] : 0.0);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, d));
      const uint32_t vid = __shfl_sync(FULL, idl, 0);
      if (lane == 0) {
        if (!first_start || last_cont) atomicAdd(out + vid, acc);
        else if (ASSIGN) out[vid] = acc;
        else out[vid] = __dadd_rn(out[vid], acc);
      }
    } else {
      s_ids[lane] = idl;
      // exclusive prefix of row starts over lanes
      const int cnt = __popc(bits);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
      }
      const uint32_t r_last = r0 + (uint32_t)__shfl_sync(FULL, incl, 31);
      __syncwarp();
      const bool lane_valid = vm != 0;
      const int kf = lane_valid ? __ffs(vm) - 1 : 0;
      uint32_t j = r0 + (uint32_t)(incl - cnt) + ((bits >> kf) & 1u);
      const uint32_t sb = bits & ~((2u << kf) - 1u);  // row starts after the lane's first edge

      auto emit = [&](uint32_t row, double x) {
        const uint32_t rr = row - r0;
        const uint32_t vid = rr < 32 ? s_ids[rr] : id_map_b[row];
        if ((row == r0 && !first_start) || (row == r_last && last_cont)) atomicAdd(out + vid, x);
        else if (ASSIGN) out[vid] = x;
        else out[vid] = __dadd_rn(out[vid], x);
      };

      const uint32_t head_j = j;
      double head_sum = 0.0, acc = 0.0;
      bool head_closed = false;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if ((sb >> k) & 1u) {
          if (!head_closed) {
            head_sum = acc;
            head_closed = true;
          } else {
            emit(j, acc);
          }
          acc = 0.0;
          ++j;
        }
        acc = __dadd_rn(acc, ((vm >> k) & 1u) ? v[k] : 0.0);
      }
      // segmented inclusive scan of the lane tails (key = tail row)
      const int key = lane_valid ? (int)j : -1 - lane;
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
      int nh = __shfl_down_sync(FULL, lane_valid ? (int)head_j : -1000, 1);
      if (lane == 31) nh = -1000;
      if (lane_valid) {
        if (head_closed) emit(head_j, (pk == (int)head_j) ? __dadd_rn(pv, head_sum) : head_sum);
        if (nh != (int)j) emit(j, val);
      }
      __syncwarp();
    }
    // rotate the pipeline
#pragma unroll
    for (int k = 0; k < V; ++k) c[k] = cn[k];
    fw = fwn;
    r0 = r0n;
    idl = idn;
  }
}

// rstart bit q = arena edge q is the first edge of its local row; bit m is a
// sentinel (set) so the last tile of the last block sees its row closed.
__global__ void k_row_start_bits(int64_t Lb, int64_t es, const uint32_t *__restrict__ lro_b,
                                 uint32_t *__restrict__ bits) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= Lb;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = es + lro_b[r];
    atomicOr(bits + (q >> 5), 1u << (q & 31));
  }
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

// ---- degree-ordered layout: row-start bitmap + prefix hot table ----
// Shared-memory carve-out of the prefix gather (KB; one of the sm_100
// configurations) and the hot slots that fill it.  The rest of the 256 KB
// unified array is L1, where the warm tier lives and the cold misses are
// staged: a larger table starves them (scripts/mb_gather.cu: random LDG at
// 0.93 / 0.86 / 0.50 per SM cycle with 0 / 128 / 192 KB of shared memory).
static int prefix_carveout_kb() {
  const char *env = getenv("GCB_CARVE_KB");
  return env ? atoi(env) : 100;
}
static int64_t prefix_hot_slots(gcb_ctx *ctx, int nw) {
  int optin = 0;
  GCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  int64_t budget = (int64_t)prefix_carveout_kb() * 1024;
  if (budget > optin + 1024) budget = optin + 1024;
  // 1 KB per CTA is reserved by the system; the id caches take kGWarps * 128 B
  int64_t K = (budget - 1024 - (int64_t)nw * 128) / 8;
  const char *env = getenv("GCB_HOT_K");
  if (env && atoll(env) < K) K = atoll(env);
  return K < 0 ? 0 : K;
}

static void ensure_prefix_exec(gcb_ctx *ctx, gcb_blocked *bg) {
  ensure_derived(ctx, bg);
  if (bg->rready) return;
  const int64_t words = (bg->m + kColPad) / 32 + 16;
  bg->rstart.alloc(words);
  GCB_CUDA(cudaMemsetAsync(bg->rstart.p, 0, words * sizeof(uint32_t), ctx->stream));
  for (int64_t b = 0; b < bg->B; ++b) {
    const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    if (Lb == 0) continue;
    k_row_start_bits<<<grid_for(Lb + 1, 256, 65536), 256, 0, ctx->stream>>>(
        Lb, bg->h_edge_starts[b], bg->lro.p + rs + b, bg->rstart.p);
    after_launch(ctx, "k_row_start_bits");
  }
  sync(ctx);
  bg->rready = true;
}

template <bool WGT, bool ASSIGN, int NW>
static void launch_prefix_nw(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, const double *vals,
                             double *out) {
  const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
  const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
  const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
  const int64_t lo = b * bg->width, hi = (lo + bg->width < bg->n) ? lo + bg->width : bg->n;
  const int64_t hot_cap = prefix_hot_slots(ctx, NW);
  const int hot = (int)(hot_cap < hi - lo ? hot_cap : hi - lo);
  const size_t smem = (size_t)hot * 8 + NW * 32 * sizeof(uint32_t);
  static size_t done = 0;
  if (smem > done) {
    GCB_CUDA(cudaFuncSetAttribute(k_pull_prefix<WGT, ASSIGN, NW>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int pct = (int)(100.0 * prefix_carveout_kb() / 228.0 + 0.99);
    if (pct > 100) pct = 100;
    GCB_CUDA(cudaFuncSetAttribute(k_pull_prefix<WGT, ASSIGN, NW>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    done = smem;
  }
  int64_t grid = ceil_div(nt, NW);
  if (grid > ctx->num_sms) grid = ctx->num_sms;
  k_pull_prefix<WGT, ASSIGN, NW><<<(unsigned)(grid < 1 ? 1 : grid), NW * 32, smem, ctx->stream>>>(
      bg->col.p, WGT ? bg->w.p : nullptr, bg->rstart.p, bg->id_map.p + rs, bg->tile_row.p + tb, es,
      ee, bg->h_tile_t0[b], nt, (uint32_t)lo, hot, (uint32_t)Lb, vals, out);
  after_launch(ctx, "k_pull_prefix");
}

static int prefix_warps() {
  const char *env = getenv("GCB_PWARPS");
  return env ? atoi(env) : 32;
}

template <bool WGT, bool ASSIGN>
static void launch_prefix(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, const double *vals, double *out) {
  switch (prefix_warps()) {
    case 16: launch_prefix_nw<WGT, ASSIGN, 16>(ctx, bg, b, vals, out); break;
    case 24: launch_prefix_nw<WGT, ASSIGN, 24>(ctx, bg, b, vals, out); break;
    default: launch_prefix_nw<WGT, ASSIGN, 32>(ctx, bg, b, vals, out); break;
  }
}

// out[v] += sum over the rows of v in every block (block order); the caller
// clears out first.
void gather_accum(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights,
                  uint32_t flags, double *out) {
  if (bg->is_relabeled && getenv("GCB_OLD_PREFIX") == nullptr) {
    ensure_prefix_exec(ctx, bg);
    const bool wgt = use_weights && bg->weighted;
    bool first = true;  // out is zero before the first launch (callers clear it)
    for (int64_t b = 0; b < bg->B; ++b) {
      if (bg->h_row_starts[b + 1] == bg->h_row_starts[b]) continue;
      ProfScope ps(ctx, 0);
      if (wgt && first) launch_prefix<true, true>(ctx, bg, b, vals, out);
      else if (wgt) launch_prefix<true, false>(ctx, bg, b, vals, out);
      else if (first) launch_prefix<false, true>(ctx, bg, b, vals, out);
      else launch_prefix<false, false>(ctx, bg, b, vals, out);
      first = false;
    }
    return;
  }
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

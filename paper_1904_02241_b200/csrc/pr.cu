// pr.cu -- TOCAB value kernels on sm_100a and their drivers:
//   K2 pull gather  (kernels.py:155-161, 275-282, 333-347)
//   K3 block merge  (accumulate_ranges kernels.py:300-321)
//   K1+update       (kernels.py:185-191, 398-399)
//   K4 push scatter (kernels.py:285-297)
//   K5 SpMV         (kernels.py:412-487), K2/K4 with weights.
//
// Iteration structure (pull): the blocks are gathered one launch at a time in
// block order; each finished row is added straight into a dense f64 sums
// vector at id_map[row] (sums[v] = ((0 + p_b0) + p_b1) + ... -- the
// reference's block-ordered merge, kernels.py:310-320, without materialising
// the partials arena), then one elementwise kernel applies the rank update,
// the L1 delta, the next contributions and clears sums.  No two rows of a
// block share a destination, and blocks are stream-ordered, so the
// read-modify-write needs no atomics.
//
// Two arithmetic modes:
//   exact (GCB_FLAG_EXACT): one thread per local row adds in storage order with
//     __dadd_rn/__dmul_rn, blocks merge in order from 0.0, the update is
//     base + (d * s) with two roundings -> bit-identical to the reference.
//   fast (default): edge-balanced warp tiles (merge-path): each lane owns
//     kTileV consecutive edges, streams col_idx with 16-byte evict-first loads,
//     gathers the L2-resident vertex values with evict-last loads, reduces
//     in-lane then across lanes with a segmented shuffle scan.  Degree skew is
//     irrelevant to load balance.  Results differ from the sequential order by
//     reassociation only (|err| ~ 1e-15 relative).
#include <cmath>
#include <cstdlib>

#include "gcb_internal.cuh"

namespace gcb {

}  // namespace gcb

#include "ldst.cuh"
#include "pr_math.cuh"
#include "tiles.cuh"

namespace gcb {

constexpr int kWarps = 8;  // warps per CTA in the tile kernels

// ---------------------------------------------------------------------------
// K2 fast: edge-balanced pull gather over one block.
//   row_sum(r) = sum_{e in row r} w_e * vals[col_e]  (w_e = 1 if unweighted)
//   ACCUM: out[id_map_b[r]] += row_sum(r)   (dense sums / y vector)
//   else : out[r] = row_sum(r)              (partials of this block)
// Rows crossing a tile boundary: the tile where the row starts emits its
// portion as above; every later tile writes its portion to carry_b[t]; the
// warp-per-span fix-up adds the carries afterwards.
// ---------------------------------------------------------------------------
template <typename VT, bool WGT, bool ACCUM>
__global__ void __launch_bounds__(kWarps * 32)
    k_pull_tiles(const uint32_t *__restrict__ col, const double *__restrict__ w,
                 const uint32_t *__restrict__ lro_b, const uint32_t *__restrict__ id_map_b,
                 const uint32_t *__restrict__ tile_row, int64_t es, int64_t ee, int64_t t0,
                 int64_t ntiles, uint32_t Lb, const VT *__restrict__ vals, double *__restrict__ out,
                 double *__restrict__ carry_b) {
  constexpr int V = kTileV, T = kTileT;
  __shared__ uint32_t s_ends[kWarps][T + 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *ends = s_ends[wid];
  const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
  const unsigned FULL = 0xffffffffu;

  for (int64_t t = (int64_t)blockIdx.x * kWarps + wid; t < ntiles;
       t += (int64_t)gridDim.x * kWarps) {
    const int64_t abase = (t0 + t) * T;
    const int64_t lbase = abase - es;
    const int64_t llo = lbase > 0 ? lbase : 0;
    const int64_t lhi = (lbase + T < ee - es) ? lbase + T : ee - es;
    const uint32_t r0 = tile_row[t];
    const bool r0_carried = (int64_t)lro_b[r0] < llo;

    // streaming loads first (independent of the row table)
    uint32_t c[V];
    {
      const uint4 *cp = reinterpret_cast<const uint4 *>(col + abase + lane * V);
      uint4 a = ld_stream_u4(cp, pol_stream), b = ld_stream_u4(cp + 1, pol_stream);
      c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
      c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
    }
    const int64_t q0 = lbase + (int64_t)lane * V;
    double v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t q = q0 + k;
      v[k] = (q >= llo && q < lhi) ? ld_keep(vals + c[k], pol_keep) : 0.0;
    }
    if (WGT) {
      const double2 *wp = reinterpret_cast<const double2 *>(w + abase + lane * V);
#pragma unroll
      for (int k2 = 0; k2 < V / 2; ++k2) {
        double2 ww = ld_stream_d2(wp + k2, pol_stream);
        v[2 * k2] = __dmul_rn(ww.x, v[2 * k2]);
        v[2 * k2 + 1] = __dmul_rn(ww.y, v[2 * k2 + 1]);
      }
    }

    // row-end table for this tile: ends[j] = lro_b[r0 + 1 + j]
    int nload = 0;
    while (true) {
      const uint32_t idx = r0 + 1 + nload + lane;
      const uint32_t e = idx <= Lb ? lro_b[idx] : 0xffffffffu;
      ends[nload + lane] = e;
      const unsigned below = __ballot_sync(FULL, e < (uint32_t)lhi);
      nload += 32;
      if (below != FULL || nload >= T) break;
    }
    __syncwarp();

    auto emit = [&](int jj, double x) {
      if (jj == 0 && r0_carried) {
        carry_b[t] = x;
      } else if (ACCUM) {
        double *p = out + id_map_b[r0 + jj];
        *p = __dadd_rn(*p, x);
      } else {
        out[r0 + jj] = x;
      }
    };

    const int64_t qf = q0 > llo ? q0 : llo;
    const bool lane_valid = (qf < lhi) && (q0 + V > llo);
    int j = 0;
    if (lane_valid) {  // first j with ends[j] > qf
      int lo = 0, hi = nload;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
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
      if (q < llo || q >= lhi) continue;
      if ((uint32_t)q >= endj) {
        if (j == head_j) {
          head_sum = acc;
          head_closed = true;
        } else {
          emit(j, acc);  // middle row: starts and ends in this lane
        }
        acc = 0.0;
        ++j;
        endj = ends[j];
      }
      acc = __dadd_rn(acc, v[k]);
    }

    // segmented inclusive scan over lanes keyed by the tail row
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
  }
}

// Carry fix-up: one warp per row spanning several tiles; lanes sum the
// carries in a fixed strided order, a fixed shuffle tree combines them.
template <bool ACCUM>
__global__ void k_fixup(int64_t nspans, const uint32_t *__restrict__ span_tile,
                        const uint32_t *__restrict__ span_len, int64_t tile_base,
                        const uint32_t *__restrict__ tile_row, const uint32_t *__restrict__ id_map_b,
                        const double *__restrict__ carry_b, double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < nspans; s += nw) {
    const int64_t t = (int64_t)span_tile[s] - tile_base;
    const uint32_t len = span_len[s];
    double acc = 0.0;
    for (uint32_t i = lane; i < len; i += 32) acc = __dadd_rn(acc, carry_b[t + i]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, d));
    if (lane == 0) {
      const uint32_t r = tile_row[t];
      double *p = ACCUM ? out + id_map_b[r] : out + r;
      *p = __dadd_rn(*p, acc);
    }
  }
}

// K2 exact: storage-order sums (kernels.py:155-170), bit-identical.  Rows of
// up to kExactShort edges: one thread per row (k_pull_exact).  Longer rows
// (listed per block, longest first, by ensure_long_rows) go to
// k_pull_exact_long: up to kExactMid edges one row per lane, longer ones a
// warp each whose lanes gather in parallel while one add chain walks the
// values in edge order -- every row's rounding sequence is the sequential
// one.  (One thread per row left the 370K-edge hub row of rmat:24 on a single
// thread: 28 ms per exact iteration.)
template <bool WGT, bool ACCUM>
__device__ __forceinline__ void exact_store(double *out, const uint32_t *id_map_b, int64_t i, double s) {
  if (ACCUM) {
    double *p = out + id_map_b[i];
    *p = __dadd_rn(*p, s);
  } else {
    out[i] = s;
  }
}

template <bool WGT, bool ACCUM>
__global__ void k_pull_exact(const uint32_t *__restrict__ col_b, const double *__restrict__ w_b,
                             const uint32_t *__restrict__ lro_b, const uint32_t *__restrict__ id_map_b,
                             int64_t Lb, const double *__restrict__ vals, double *__restrict__ out,
                             uint32_t short_max) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Lb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e0 = lro_b[i], e1 = lro_b[i + 1];
    if (e1 - e0 > short_max) continue;  // k_pull_exact_long
    double s = 0.0;
    for (uint32_t e = e0; e < e1; ++e) {
      double x = vals[col_b[e]];
      if (WGT) x = __dmul_rn(w_b[e], x);
      s = __dadd_rn(s, x);
    }
    exact_store<WGT, ACCUM>(out, id_map_b, i, s);
  }
}

// Rows of kExactShort..kExactMid edges, 32 per warp, one per lane: each lane
// runs its own row's chain, so one warp-DADD serves 32 rows (the FP64 pipe
// issues ~1.75 warp-DADDs per SM-cycle whatever the active mask), with the
// lane's column ids two steps and its values one step ahead of its adds.
// Rows come sorted by length, so a warp's 32 rows are about equally long.
template <bool WGT, bool ACCUM>
__device__ __forceinline__ void exact_rows_by_lane(const uint32_t *__restrict__ col_b,
                                                   const double *__restrict__ w_b,
                                                   const uint32_t *__restrict__ lro_b,
                                                   const uint32_t *__restrict__ id_map_b,
                                                   const uint32_t *__restrict__ rows, int64_t nrows,
                                                   const double *__restrict__ vals,
                                                   double *__restrict__ out, int lane) {
  constexpr int S = 8;
  const bool act = lane < nrows;
  const uint32_t i = act ? rows[lane] : 0u;
  const uint32_t e0 = act ? lro_b[i] : 0u, e1 = act ? lro_b[i + 1] : 0u;
  const uint32_t steps = (e1 - e0 + S - 1) / S;
  const uint32_t wsteps = __reduce_max_sync(0xffffffffu, steps);
  auto load_cols = [&](uint32_t e, uint32_t (&c)[S], double (&w)[S]) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      c[k] = e + k < e1 ? col_b[e + k] : 0xffffffffu;
      if (WGT) w[k] = e + k < e1 ? w_b[e + k] : 0.0;
    }
  };
  auto load_vals = [&](const uint32_t (&c)[S], const double (&w)[S], double (&x)[S]) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      x[k] = 0.0;
      if (c[k] != 0xffffffffu) {
        x[k] = vals[c[k]];
        if (WGT) x[k] = __dmul_rn(w[k], x[k]);
      }
    }
  };
  uint32_t c1[S], c2[S];
  double w1[S], w2[S], x[S], nx[S];
  load_cols(e0, c1, w1);
  load_vals(c1, w1, x);
  load_cols(e0 + S, c1, w1);
  double acc = 0.0;
  for (uint32_t st = 0; st < wsteps; ++st) {
    const uint32_t e = e0 + st * S;
    load_vals(c1, w1, nx);
    load_cols(e + 2 * S, c2, w2);
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (e + k < e1) acc = __dadd_rn(acc, x[k]);
#pragma unroll
    for (int k = 0; k < S; ++k) {
      x[k] = nx[k];
      c1[k] = c2[k];
      if (WGT) w1[k] = w2[k];
    }
  }
  if (act) exact_store<WGT, ACCUM>(out, id_map_b, i, acc);
}

// Rows longer than kExactShort.  The first nbig rows of the (longest-first)
// list, longer than kExactMid, get a warp each; the rest go 32 per warp,
// one per lane (exact_rows_by_lane).  Work items: the big rows first, then
// the 32-row groups, over a grid-stride of warps.
template <bool WGT, bool ACCUM>
__global__ void k_pull_exact_long(const uint32_t *__restrict__ col_b, const double *__restrict__ w_b,
                                  const uint32_t *__restrict__ lro_b,
                                  const uint32_t *__restrict__ id_map_b,
                                  const uint32_t *__restrict__ long_rows, int64_t nlong,
                                  int64_t nbig, const double *__restrict__ vals,
                                  double *__restrict__ out) {
  __shared__ double s_buf[8][256];  // one 256-value slot per warp (256-thread CTAs)
  double *buf = s_buf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = nbig + (nlong - nbig + 31) / 32;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < items; j += nw) {
    if (j >= nbig) {
      const int64_t first = nbig + (j - nbig) * 32;
      exact_rows_by_lane<WGT, ACCUM>(col_b, w_b, lro_b, id_map_b, long_rows + first,
                                     nlong - first, vals, out, lane);
      continue;
    }
    const uint32_t i = long_rows[j];
    const uint32_t b0 = lro_b[i], b1 = lro_b[i + 1];
    double acc = 0.0;
    // Steps of 256 edges (8 per lane).  Software pipeline over steps: the
    // column ids of step s+2 and the gathered values of step s+1 are in
    // flight while step s's 256 values are added in edge order, so neither
    // the col load nor the value gather sits in front of the add chain -- the
    // chain (8.7 cycles per f64 add, scripts/mb_dadd.cu) is the hub rows'
    // critical path.  The step's values go through the warp's shared-memory
    // slot, read back with independent LDS (a SHFL per add sat on the chain).
    constexpr uint32_t kNone = 0xffffffffu;
    auto load_cols = [&](uint32_t base, uint32_t (&c)[8], double (&w)[8]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t e = base + q * 32 + lane;
        c[q] = e < b1 ? col_b[e] : kNone;
        if (WGT) w[q] = e < b1 ? w_b[e] : 0.0;
      }
    };
    auto load_vals = [&](const uint32_t (&c)[8], const double (&w)[8], double (&x)[8]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        x[q] = 0.0;
        if (c[q] != kNone) {
          x[q] = vals[c[q]];
          if (WGT) x[q] = __dmul_rn(w[q], x[q]);
        }
      }
    };
    uint32_t c1[8], c2[8];
    double w1[8], w2[8], x[8], nx[8];
    load_cols(b0, c1, w1);
    load_vals(c1, w1, x);                 // step 0
    load_cols(b0 + 256, c1, w1);          // step 1's columns
    for (uint32_t base = b0; base < b1; base += 256) {
      if (base + 256 < b1) {
        load_vals(c1, w1, nx);            // step s+1 (columns arrived a step ago)
        load_cols(base + 512, c2, w2);    // step s+2
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) buf[q * 32 + lane] = x[q];
      __syncwarp();
      const int cnt = (int)(b1 - base < 256u ? b1 - base : 256u);
      if (cnt == 256) {
#pragma unroll 64
        for (int k = 0; k < 256; ++k) acc = __dadd_rn(acc, buf[k]);
      } else {
        for (int k = 0; k < cnt; ++k) acc = __dadd_rn(acc, buf[k]);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        x[q] = nx[q];
        c1[q] = c2[q];
        if (WGT) w1[q] = w2[q];
      }
    }
    if (lane == 0) exact_store<WGT, ACCUM>(out, id_map_b, i, acc);
  }
}

// ---------------------------------------------------------------------------
// K3: range-tiled merge of an explicit partials arena (accumulate_ranges,
// kernels.py:300-321; PAPER Fig. 5).  One CTA per kMergeK-wide destination
// range; block-ordered shared-memory accumulation from 0.0.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
    k_merge(int64_t n, int64_t B, int64_t R, const int64_t *__restrict__ bounds,
            const uint32_t *__restrict__ id_map, const double *__restrict__ partial,
            double *__restrict__ out) {
  __shared__ double buf[kMergeK];
  const int64_t j = blockIdx.x;
  const int64_t lo = j * kMergeK;
  const int64_t hi = (lo + kMergeK < n) ? lo + kMergeK : n;
  const int width = (int)(hi - lo);
  for (int i0 = 0; i0 < kMergeK; i0 += blockDim.x) {  // CTA-uniform trip count
    const int i = i0 + threadIdx.x;
    if (i < kMergeK) buf[i] = 0.0;
  }
  __syncthreads();
  for (int64_t b = 0; b < B; ++b) {
    const int64_t s = bounds[b * (R + 1) + j], e = bounds[b * (R + 1) + j + 1];
    // a CTA-uniform trip count: every warp reaches the barrier converged
    // (synccheck flagged the data-dependent exits of a p < e loop here)
    for (int64_t q = s; q < e; q += blockDim.x) {
      const int64_t p = q + threadIdx.x;
      if (p < e) {
        const int idx = (int)(id_map[p] - lo);
        buf[idx] = __dadd_rn(buf[idx], partial[p]);
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < width; i += blockDim.x) out[lo + i] = buf[i];
}

// deterministic single-CTA sum of per-CTA partials
__global__ void k_reduce_sum(const double *__restrict__ in, int64_t count, double *__restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += in[i];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_down_sync(0xffffffffu, x, d);
    if (threadIdx.x == 0) *out = x;
  }
}

// compute_contributions kernels.py:185-191 as a standalone operator
__global__ void k_contributions(int64_t n, const double *__restrict__ ranks,
                                const int64_t *__restrict__ deg, double *__restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = deg[v] > 0 ? __ddiv_rn(ranks[v], (double)deg[v]) : 0.0;
}

// ranks = r0; contributions = r0 / deg (VertexValueSet.initial kernels.py:80-89);
// sums = 0.  One 4-vertex quad per thread with 256-bit stores, like the
// update.  ranks == nullptr (tol == 0): the ranks are first read after the
// last iteration writes them, so they are not initialised.
__global__ void k_pr_init(int64_t n, double r0, const uint32_t *__restrict__ deg,
                          double *__restrict__ ranks, double *__restrict__ contrib,
                          float *__restrict__ contrib32, double *__restrict__ sums) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4 *D = reinterpret_cast<const uint4 *>(deg);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint4 d = __ldcs(D + i);
    const uint32_t dg[4] = {d.x, d.y, d.z, d.w};
    double c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = dg[k] ? __ddiv_rn(r0, (double)dg[k]) : 0.0;
    if (ranks) st_f64x4(ranks + 4 * i, r0, r0, r0, r0);
    if (contrib) st_f64x4(contrib + 4 * i, c[0], c[1], c[2], c[3]);
    if (contrib32)
      reinterpret_cast<float4 *>(contrib32)[i] =
          make_float4(__double2float_rn(c[0]), __double2float_rn(c[1]), __double2float_rn(c[2]),
                      __double2float_rn(c[3]));
    st_f64x4(sums + 4 * i, 0.0, 0.0, 0.0, 0.0);
  }
  for (int64_t v = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (ranks) ranks[v] = r0;
    const uint32_t dg = deg[v];
    const double c = dg ? __ddiv_rn(r0, (double)dg) : 0.0;
    if (contrib) contrib[v] = c;
    if (contrib32) contrib32[v] = __double2float_rn(c);
    sums[v] = 0.0;
  }
}

__global__ void k_count_nonzero_u32(int64_t n, const uint32_t *__restrict__ x,
                                    unsigned long long *__restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += x[i] != 0u;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// rank update (kernels.py:398-399) fused with the L1 delta (399), the next
// iteration's contributions (185-191) and clearing sums for the next pass.
// One 4-vertex quad per thread (update_grid): 256-bit loads and stores, the
// CTA reduces its delta once at the end.  The arithmetic is pr_math.cuh's.
// RANKS = false (tol == 0, every iteration but the last): the intermediate
// ranks are dead -- the next iteration reads only the contributions, and the
// L1 delta (kernels.py:399) is compared with tol = 0, which it can never fall
// below -- so neither the old ranks are read nor the new ones written: 28 B
// per vertex instead of 44.  The contributions are computed from the same
// r' = base + d*s, so every result stays bit-identical.
template <bool EXACT, bool RANKS>
__global__ void __launch_bounds__(512, 2)
    k_pr_update2(int64_t n, double base, double damping, double *__restrict__ sums,
                 double *__restrict__ ranks, const uint32_t *__restrict__ deg,
                 double *__restrict__ contrib, float *__restrict__ contrib32,
                 double *__restrict__ deltas) {
  __shared__ double red[16];
  double dsum = 0.0;
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4 *D = reinterpret_cast<const uint4 *>(deg);
  auto store = [&](int64_t i, const double *nr, const double *c) {
    if (RANKS) st_f64x4(ranks + 4 * i, nr[0], nr[1], nr[2], nr[3]);
    st_f64x4(sums + 4 * i, 0.0, 0.0, 0.0, 0.0);
    if (contrib) st_f64x4(contrib + 4 * i, c[0], c[1], c[2], c[3]);
    if (contrib32)
      reinterpret_cast<float4 *>(contrib32)[i] =
          make_float4(__double2float_rn(c[0]), __double2float_rn(c[1]), __double2float_rn(c[2]),
                      __double2float_rn(c[3]));
  };
  // deltas == nullptr (tol == 0): the delta is dead, the old ranks are not read
  const bool want_delta = RANKS && deltas;
  auto old = [&](int64_t i, double *o) {
    if (want_delta) ld_rw_f64x4(ranks + 4 * i, o);
    else o[0] = o[1] = o[2] = o[3] = 0.0;
  };
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n4; i += 2 * stride) {
    const int64_t k = i + stride;
    double sa[4], sb[4], oa[4], ob[4], nr[4], c[4];
    ld_rw_f64x4(sums + 4 * i, sa);
    ld_rw_f64x4(sums + 4 * k, sb);
    old(i, oa);
    old(k, ob);
    const uint4 da = __ldcs(D + i), db = __ldcs(D + k);
    pr_quad<EXACT>(sa, oa, da, base, damping, nr, c, dsum);
    store(i, nr, c);
    pr_quad<EXACT>(sb, ob, db, base, damping, nr, c, dsum);
    store(k, nr, c);
  }
  if (i < n4) {
    double sa[4], oa[4], nr[4], c[4];
    ld_rw_f64x4(sums + 4 * i, sa);
    old(i, oa);
    pr_quad<EXACT>(sa, oa, D[i], base, damping, nr, c, dsum);
    store(i, nr, c);
  }
  for (int64_t v = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    const double nr = __dadd_rn(base, __dmul_rn(damping, sums[v]));
    if (want_delta) dsum += fabs(nr - ranks[v]);
    const double c = deg[v] ? div_deg<EXACT>(nr, deg[v]) : 0.0;
    if (RANKS) ranks[v] = nr;
    sums[v] = 0.0;
    if (contrib) contrib[v] = c;
    if (contrib32) contrib32[v] = __double2float_rn(c);
  }
  if (!want_delta) return;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dsum;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_down_sync(0xffffffffu, x, d);
    if (threadIdx.x == 0) deltas[blockIdx.x] = x;
  }
}

static unsigned update_grid(gcb_ctx *ctx, int64_t n) {
  // one 4-vertex quad per thread: 111 us at rmat:24 against 125 us with two
  // persistent CTAs per SM (scripts/mb_stream.cu)
  return grid_for((n + 3) / 4, 512, (int64_t)(1 << 20) * ctx->num_sms);
}

static void launch_update(gcb_ctx *ctx, bool exact, int64_t n, double base, double damping,
                          double *sums, double *ranks, const uint32_t *deg, double *contrib,
                          float *contrib32, double *deltas, bool with_ranks = true) {
  const unsigned g = update_grid(ctx, n);
#define GCB_UPD(E, R)                                                                           \
  k_pr_update2<E, R><<<g, 512, 0, ctx->stream>>>(n, base, damping, sums, ranks, deg, contrib,   \
                                                 contrib32, deltas)
  if (exact) {
    if (with_ranks) GCB_UPD(true, true);
    else GCB_UPD(true, false);
  } else {
    if (with_ranks) GCB_UPD(false, true);
    else GCB_UPD(false, false);
  }
#undef GCB_UPD
  after_launch(ctx, "k_pr_update2");
}

// ---------------------------------------------------------------------------
// K4: push scatter.  fast: edge-balanced tiles + f64 atomics into the block's
// destination range (L2-resident); exact: one thread per block walks its
// edges in storage order (np.bincount order, kernels.py:290-296).
// ---------------------------------------------------------------------------
// Push scatter on warp tiles with the row-start bitmap (tiles.cuh): the
// values of the tile's first 32 source rows are fetched by the lanes up front
// (one id_map + one vals load each, overlapped) and each edge takes its row's
// value by shuffle; the loop of k_push_tiles reloaded id_map -> vals on every
// row change (ncu: 55% long-scoreboard stalls, 11% issue).  Destinations are
// accumulated with f64 RED into the block's (L2-resident) range.
template <bool WGT>
__global__ void __launch_bounds__(256)
    k_push_bits(const uint32_t *__restrict__ col, const double *__restrict__ w,
                const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ tile_row,
                int64_t es, int64_t ee, int64_t t0, int64_t ntiles, uint32_t Lb,
                const uint32_t *__restrict__ id_map_b, const double *__restrict__ vals,
                double *__restrict__ sums) {
  constexpr int V = kTileV, T = kTileT;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t pol_stream = policy_evict_first();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
    const int64_t abase = (t0 + t) * T;
    uint32_t c[V];
    ld_stream_u32x8(col + abase + lane * V, pol_stream, c);
    const uint32_t fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    const uint32_t r0 = tile_row[t];
    const double rv = r0 + lane < Lb ? vals[id_map_b[r0 + lane]] : 0.0;
    double ww[V];
    if (WGT) {
      ld_stream_f64x4(w + abase + lane * V, pol_stream, ww);
      ld_stream_f64x4(w + abase + lane * V + 4, pol_stream, ww + 4);
    }
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < T ? (int)(ee - abase) : T;
    const TileBits tb = tile_bits(fw, llo, lhi, lane);
    // exclusive prefix of row starts over lanes -> the row of the lane's first edge
    const int cnt = __popc(tb.bits);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    const int kf = tb.vm ? __ffs(tb.vm) - 1 : 0;
    uint32_t rr = (uint32_t)(incl - cnt) + ((tb.bits >> kf) & 1u);  // row - r0
#pragma unroll
    for (int k = 0; k < V; ++k) {
      if (k > kf && ((tb.bits >> k) & 1u)) ++rr;
      double x = __shfl_sync(FULL, rv, rr & 31);
      if (!((tb.vm >> k) & 1u)) continue;
      if (rr >= 32) x = vals[id_map_b[r0 + rr]];
      if (WGT) x = __dmul_rn(ww[k], x);
      atomicAdd(sums + c[k], x);
    }
  }
}

// Push scatter with hub destinations accumulated in shared memory: the
// arena is recoded (ensure_push_exec) so an edge into one of the block's top
// in-degree destinations carries 0x80000000 | slot; those adds go to the
// CTA's accumulator (shared-memory atomic) and every CTA flushes its
// non-zero slots with one global RED each at the end.
// FIX (non-negative values, i.e. PageRank contributions): the hub table is
// 64-bit fixed point (2^-62 units) so the shared-memory adds are native
// integer atomics -- f64 adds on shared memory compile to a CAS loop
// (ATOMS.CAST.SPIN) that serialises on the hottest hubs.  Sums stay below 1
// (rank mass), so a CTA's slot cannot overflow; each term is rounded to
// 2^-62 absolute, and integer adds make the slot order-independent.
#ifndef GCB_FIX_BITS
#define GCB_FIX_BITS 62  // experiment builds override (Makefile `variant`)
#endif
constexpr double kFixScale = (double)(1ull << GCB_FIX_BITS);  // 2^62
constexpr double kFixInv = 1.0 / kFixScale;

// 64-bit shared adds (f64 or u64) are CAS loops on sm_100 (ATOMS.CAST.SPIN);
// 32-bit ATOMS.ADD is native.  A 64-bit fixed-point slot is therefore two
// 32-bit words: the low add returns the old word, which tells whether it
// wrapped, and the carry rides with the high add -- the pair always holds
// the exact 64-bit sum.
__device__ __forceinline__ void fix_add(unsigned *lo, unsigned *hi, uint32_t slot,
                                        unsigned long long add) {
  const unsigned alo = (unsigned)add, ahi = (unsigned)(add >> 32);
  const unsigned old = atomicAdd(lo + slot, alo);
  const unsigned carry = (old + alo < old) ? 1u : 0u;
  if (ahi + carry) atomicAdd(hi + slot, ahi + carry);
}

template <bool WGT, bool FIX = false>
__global__ void __launch_bounds__(1024, 1)
    k_push_hot(const uint32_t *__restrict__ xcol, const double *__restrict__ w,
               const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ tile_row,
               int64_t es, int64_t ee, int64_t t0, int64_t ntiles, uint32_t Lb,
               const uint32_t *__restrict__ id_map_b, const uint32_t *__restrict__ hot_ids_b,
               int hot, const double *__restrict__ vals, double *__restrict__ sums) {
  constexpr int V = kTileV, T = kTileT;
  constexpr uint32_t kHot = 0x80000000u;
  extern __shared__ double s_acc[];
  unsigned *s_lo = reinterpret_cast<unsigned *>(s_acc), *s_hi = s_lo + hot;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t pol_stream = policy_evict_first();
  for (int i = threadIdx.x; i < hot; i += blockDim.x) s_acc[i] = 0.0;  // also 0 in fixed point
  __syncthreads();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
    const int64_t abase = (t0 + t) * T;
    uint32_t c[V];
    ld_stream_u32x8(xcol + abase + lane * V, pol_stream, c);
    const uint32_t fw = rstart[(abase >> 5) + (lane < 8 ? lane : 8)];
    const uint32_t r0 = tile_row[t];
    const double rv = r0 + lane < Lb ? vals[id_map_b[r0 + lane]] : 0.0;
    double ww[V];
    if (WGT) {
      ld_stream_f64x4(w + abase + lane * V, pol_stream, ww);
      ld_stream_f64x4(w + abase + lane * V + 4, pol_stream, ww + 4);
    }
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < T ? (int)(ee - abase) : T;
    const TileBits tb = tile_bits(fw, llo, lhi, lane);
    const int cnt = __popc(tb.bits);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += y;
    }
    const int kf = tb.vm ? __ffs(tb.vm) - 1 : 0;
    uint32_t rr = (uint32_t)(incl - cnt) + ((tb.bits >> kf) & 1u);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      if (k > kf && ((tb.bits >> k) & 1u)) ++rr;
      double x = __shfl_sync(FULL, rv, rr & 31);
      if (!((tb.vm >> k) & 1u)) continue;
      if (rr >= 32) x = vals[id_map_b[r0 + rr]];
      if (WGT) x = __dmul_rn(ww[k], x);
      if (c[k] & kHot) {
        if (FIX) fix_add(s_lo, s_hi, c[k] & ~kHot, __double2ull_rn(x * kFixScale));
        else atomicAdd(s_acc + (c[k] & ~kHot), x);
      } else {
        atomicAdd(sums + c[k], x);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hot; i += blockDim.x) {
    const double v =
        FIX ? (double)(((unsigned long long)s_hi[i] << 32) | s_lo[i]) * kFixInv : s_acc[i];
    if (v != 0.0) atomicAdd(sums + hot_ids_b[i], v);
  }
}

// The hybrid hub pass (relabel.cu hybrid_split): every edge runs from a cold
// source into a hub destination, and a cold source has few such edges, so a
// 256-edge tile spans many source rows (rmat:22: median 5, 10% of tiles over
// 64).  Its execution layout is packed once per graph (ensure_hub_pack): each
// arena edge holds (its row - the tile's first row) << 15 | its hub slot, so
// the kernel needs no row-start bitmap, no tile scan and no recode test --
// an edge is one LDS.64 of its row's value and the two 32-bit shared atomics
// of fix_add.  A tile's row values are fetched two pipeline stages ahead
// (tile_row three tiles ahead, the id_map words of tile t+2, the values of
// tile t+1, two rows per lane), converted to the table's fixed point once per
// row and parked in the warp's slice of shared memory; rows 64..127 of a long
// tile are loaded when it starts, and edges of rows past 128 take a second,
// warp-uniform loop.  The bitmap form of this pass spent 432 warp
// instructions per tile and stalled on its id_map -> value chain (ncu,
// profiles/r2_hub_ncu.txt).
constexpr int kHubRows = 128;         // row values per warp parked in shared memory
constexpr uint32_t kPackNone = ~0u;   // hub_pack entry past the arena
constexpr int kPackSlotBits = 15;     // slots < 2^15 - 32 (the 32 lane dummies follow)

// fix_add on shared-memory addresses (a_lo / a_hi: the slot's two words).
// Unpredicated: an edge that must not add is aimed at its lane's dummy slot
// with 0 (no branch around the atomics, and no two lanes share a dummy).
__device__ __forceinline__ void fix_add_s(uint32_t a_lo, uint32_t a_hi, unsigned long long add) {
  const unsigned alo = (unsigned)add, ahi = (unsigned)(add >> 32);
  unsigned old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a_lo), "r"(alo));
  const unsigned carry = (old + alo < old) ? 1u : 0u;
  asm volatile("red.shared.add.u32 [%0], %1;" : : "r"(a_hi), "r"(ahi + carry));
}

// two fix_add_s with both low-word atomics issued first
__device__ __forceinline__ void fix_add2_s(uint32_t a_lo, uint32_t a_hi, unsigned long long add_a,
                                           uint32_t b_lo, uint32_t b_hi, unsigned long long add_b) {
  const unsigned alo = (unsigned)add_a, ahi = (unsigned)(add_a >> 32);
  const unsigned blo = (unsigned)add_b, bhi = (unsigned)(add_b >> 32);
  unsigned olda, oldb;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(olda) : "r"(a_lo), "r"(alo));
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(oldb) : "r"(b_lo), "r"(blo));
  const unsigned ca = (olda + alo < olda) ? 1u : 0u, cb = (oldb + blo < oldb) ? 1u : 0u;
  asm volatile("red.shared.add.u32 [%0], %1;" : : "r"(a_hi), "r"(ahi + ca));
  asm volatile("red.shared.add.u32 [%0], %1;" : : "r"(b_hi), "r"(bhi + cb));
}

__device__ __forceinline__ unsigned long long to_fix(double x) {
  return __double2ull_rn(x * kFixScale);
}

// the tile loop of k_push_hub (one warp, tiles t, t + stride, ...)
__device__ __forceinline__ void hub_tiles(const uint32_t *__restrict__ pack,
                                          const uint32_t *__restrict__ tile_row, uint32_t ntiles,
                                          uint32_t Lb, const uint32_t *__restrict__ id_map_b,
                                          const double *__restrict__ vals, uint32_t s_lo_addr,
                                          uint32_t s_hi_addr, unsigned long long *s_rows,
                                          uint32_t dummy, uint32_t t, uint32_t stride, int lane,
                                          uint64_t pol_stream) {
  constexpr int V = kTileV, T = kTileT;
  constexpr uint32_t kSlotMask = (1u << kPackSlotBits) - 1u;
  const unsigned FULL = 0xffffffffu;
  auto row_id = [&](uint32_t r) { return r < Lb ? __ldg(id_map_b + r) : 0u; };
  auto words = [&](uint32_t tt, uint32_t (&w)[V]) {
    ld_stream_u32x8(pack + (size_t)tt * T + lane * V, pol_stream, w);
  };
  // pipeline: tile t's words and row values, tile t+1's row ids, the first
  // rows of tiles t+1 and t+2
  uint32_t c[V];
  words(t, c);
  uint32_t r0 = tile_row[t], r0n = 0, r0nn = 0, idA = 0, idB = 0;
  if (t + stride < ntiles) {
    r0n = tile_row[t + stride];
    idA = row_id(r0n + lane);
    idB = row_id(r0n + 32 + lane);
    if (t + 2 * stride < ntiles) r0nn = tile_row[t + 2 * stride];
  }
  double rvA = __ldg(vals + row_id(r0 + lane)), rvB = __ldg(vals + row_id(r0 + 32 + lane));
  for (; t < ntiles; t += stride) {
    const uint32_t tn = t + stride, tnn = tn + stride;
    uint32_t cn[V], idAn = 0, idBn = 0, r0nnn = 0;
    double rvAn = 0.0, rvBn = 0.0;
#pragma unroll
    for (int k = 0; k < V; ++k) cn[k] = kPackNone;
    if (tn < ntiles) {  // tile t+1: words and values (its ids landed an iteration ago)
      words(tn, cn);
      rvAn = __ldg(vals + idA);
      rvBn = __ldg(vals + idB);
    }
    if (tnn < ntiles) {  // tile t+2: row ids; tile t+3: first row
      idAn = row_id(r0nn + lane);
      idBn = row_id(r0nn + 32 + lane);
      if (tnn + stride < ntiles) r0nnn = tile_row[tnn + stride];
    }
    // this tile's row values, fixed point, in the warp's slice
    __syncwarp();  // the previous tile's readers are done with the slice
    s_rows[lane] = to_fix(rvA);
    s_rows[32 + lane] = to_fix(rvB);
    uint32_t lane_max = 0;  // entries are in bank order, not row order (ensure_hub_pack)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (c[k] != kPackNone) lane_max = max(lane_max, c[k] >> kPackSlotBits);
    const uint32_t rr_max = __reduce_max_sync(FULL, lane_max);
    if (rr_max >= 64) {
      const double xc = __ldg(vals + row_id(r0 + 64 + lane));
      const double xd = rr_max >= 96 ? __ldg(vals + row_id(r0 + 96 + lane)) : 0.0;
      s_rows[64 + lane] = to_fix(xc);
      s_rows[96 + lane] = to_fix(xd);
    }
    __syncwarp();
    uint32_t omask = 0;  // edges of rows past kHubRows
    // two edges per step: both low-word atomics are in flight before either
    // carry is needed
#pragma unroll
    for (int k = 0; k < V; k += 2) {
      unsigned long long f[2];
      uint32_t slot[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t e = c[k + j];
        const uint32_t rr = e >> kPackSlotBits;
        const bool add = rr < (uint32_t)kHubRows;  // kPackNone: rr = 2^17 - 1
        if (!add && e != kPackNone) omask |= 1u << (k + j);
        f[j] = add ? s_rows[rr] : 0ull;
        slot[j] = (add ? (e & kSlotMask) : dummy) * 4u;
      }
      fix_add2_s(s_lo_addr + slot[0], s_hi_addr + slot[0], f[0], s_lo_addr + slot[1],
                 s_hi_addr + slot[1], f[1]);
    }
    if (__any_sync(FULL, omask != 0u)) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (!((omask >> k) & 1u)) continue;
        const uint32_t e = c[k];
        const double x = __ldg(vals + __ldg(id_map_b + r0 + (e >> kPackSlotBits)));
        const uint32_t slot = (e & kSlotMask) * 4u;
        fix_add_s(s_lo_addr + slot, s_hi_addr + slot, to_fix(x));
      }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) c[k] = cn[k];
    r0 = r0n;
    r0n = r0nn;
    r0nn = r0nnn;
    idA = idAn;
    idB = idBn;
    rvA = rvAn;
    rvB = rvBn;
  }
}

// Each CTA adds its table into hub_acc (u64 fixed point: coalesced 64-bit
// integer REDs, no id lookup on the flush path, and the cross-CTA sum is
// order-independent); k_hub_fold then adds hub_acc into sums once.
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    k_push_hub(const uint32_t *__restrict__ pack, const uint32_t *__restrict__ tile_row,
               uint32_t ntiles, uint32_t Lb, const uint32_t *__restrict__ id_map_b, int hot,
               const double *__restrict__ vals, unsigned long long *__restrict__ hub_acc) {
  extern __shared__ double smem_d[];
  // hub table: hot slots + one dummy slot per lane, low words then high words
  const int slots = hot + 32;
  unsigned *s_lo = reinterpret_cast<unsigned *>(smem_d), *s_hi = s_lo + slots;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // per-warp row-value slices after the table
  unsigned long long *s_rows = reinterpret_cast<unsigned long long *>(smem_d + slots) + wid * kHubRows;
  const uint64_t pol_stream = policy_evict_first();
  for (int i = threadIdx.x; i < slots; i += blockDim.x) smem_d[i] = 0.0;
  __syncthreads();
  const uint32_t t = blockIdx.x * NW + wid;
  if (t < ntiles)
    hub_tiles(pack, tile_row, ntiles, Lb, id_map_b, vals, (uint32_t)__cvta_generic_to_shared(s_lo),
              (uint32_t)__cvta_generic_to_shared(s_hi), s_rows, (uint32_t)(hot + lane), t,
              gridDim.x * NW, lane, pol_stream);
  __syncthreads();
  for (int i = threadIdx.x; i < hot; i += blockDim.x) {
    const unsigned long long v = ((unsigned long long)s_hi[i] << 32) | s_lo[i];
    if (v) atomicAdd(hub_acc + i, v);
  }
}

// sums[hub] += hub_acc[slot] (fixed point -> f64), and hub_acc back to zero
__global__ void k_hub_fold(int hot, const uint32_t *__restrict__ hot_ids_b,
                           unsigned long long *__restrict__ hub_acc, double *__restrict__ sums) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hot; i += gridDim.x * blockDim.x) {
    const unsigned long long v = hub_acc[i];
    if (v) {
      const uint32_t id = hot_ids_b[i];
      sums[id] = __dadd_rn(sums[id], (double)v * kFixInv);
      hub_acc[i] = 0ull;
    }
  }
}

// hub_pack[q] = (row(q) - tile_row[tile(q)]) << 15 | slot(q) for the arena edges of a
// single-block hub blocking; *bad counts edges the format cannot hold
__global__ void k_hub_pack(int64_t Lb, const uint32_t *__restrict__ lro_b,
                           const uint32_t *__restrict__ tile_row_b, const uint32_t *__restrict__ xcol,
                           uint32_t slot_cap, uint32_t *__restrict__ pack,
                           unsigned long long *__restrict__ bad) {
  constexpr uint32_t kHot = 0x80000000u;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nb = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < Lb; r += nw) {
    const uint32_t s = lro_b[r], e = lro_b[r + 1];
    for (uint32_t q = s + lane; q < e; q += 32) {
      const uint32_t rr = (uint32_t)r - tile_row_b[q / kTileT];
      const uint32_t x = xcol[q], slot = x & ~kHot;
      const bool ok = (x & kHot) && rr < 256u && slot < slot_cap;
      pack[q] = ok ? (rr << kPackSlotBits) | slot : 0u;
      nb += !ok;
    }
  }
  if (nb) atomicAdd(bad, nb);
}

// Reorders every 256-entry tile of hub_pack by shared-memory bank of its slot
// (slot mod 32).  Lane l runs entries 8l..8l+7 in steps k = 0..7, so step k
// takes sorted positions k, 8+k, ..., and no two edges of one step share a bank
// unless a bank holds more than 8 of the tile's edges: the atomics of a step
// go out in one wavefront instead of ~3.7 (ncu, r2_hub_ncu.txt).  Integer
// fixed-point adds commute and every entry carries its own row offset, so any
// order within a tile gives the same table.  One warp per tile.
__global__ void __launch_bounds__(256) k_hub_bank_sort(int64_t ntiles, uint32_t *__restrict__ pack) {
  __shared__ uint32_t s_ent[8][kTileT];
  __shared__ uint32_t s_cnt[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * 8 + w;
  if (t >= ntiles) return;
  uint32_t *tile = pack + t * kTileT;
  s_cnt[w][lane] = 0;
  __syncwarp();
  uint32_t e[kTileV], b[kTileV];
#pragma unroll
  for (int k = 0; k < kTileV; ++k) {
    e[k] = tile[lane * kTileV + k];
    b[k] = (e[k] == kPackNone ? 31u : e[k]) & 31u;
    atomicAdd(&s_cnt[w][b[k]], 1u);
  }
  __syncwarp();
  // exclusive prefix of the 32 bank counts (lane = bank)
  const uint32_t cnt = s_cnt[w][lane];
  uint32_t incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  __syncwarp();
  s_cnt[w][lane] = incl - cnt;  // cursor of each bank
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kTileV; ++k) s_ent[w][atomicAdd(&s_cnt[w][b[k]], 1u)] = e[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kTileV; ++k) tile[lane * kTileV + k] = s_ent[w][lane * kTileV + k];
}

// Builds the packed hub layout once per blocking: single-block push blockings
// whose every edge is a recoded hub (relabel.cu hybrid_split guarantees it:
// the blocking holds only hub destinations); anything else keeps k_push_hot.
static bool ensure_hub_pack(gcb_ctx *ctx, gcb_blocked *bg) {
  if (bg->hub_pack_state) return bg->hub_pack_state > 0;
  bg->hub_pack_state = -1;
  const int64_t cap = (int64_t(1) << kPackSlotBits) - 32;
  if (bg->B != 1 || bg->hot_k <= 0 || bg->hot_k > cap || bg->m == 0 || !bg->xcol.p ||
      bg->h_edge_starts[0] != 0 || bg->h_tile_t0[0] != 0)
    return false;
  bg->hub_pack.alloc(bg->m + kColPad);
  GCB_CUDA(cudaMemsetAsync(bg->hub_pack.p + bg->m, 0xff, kColPad * sizeof(uint32_t), ctx->stream));
  DArray<unsigned long long> bad(1);
  GCB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), ctx->stream));
  const int64_t Lb = bg->h_row_starts[1] - bg->h_row_starts[0];
  k_hub_pack<<<grid_for(Lb * 32, 256, 65536), 256, 0, ctx->stream>>>(
      Lb, bg->lro.p, bg->tile_row.p, bg->xcol.p, (uint32_t)bg->hot_k, bg->hub_pack.p, bad.p);
  after_launch(ctx, "k_hub_pack");
  const int64_t ntiles = bg->h_tile_base[1] - bg->h_tile_base[0];
  const char *ns = getenv("GCB_HUB_NOSORT");  // A/B knob: keep the arena order
  if (!(ns && ns[0] == '1')) {
    k_hub_bank_sort<<<(unsigned)ceil_div(ntiles, 8), 256, 0, ctx->stream>>>(ntiles, bg->hub_pack.p);
    after_launch(ctx, "k_hub_bank_sort");
  }
  unsigned long long h = 0;
  d2h(ctx, &h, bad.p, 1);
  sync(ctx);
  if (h) {
    bg->hub_pack.release();
    return false;
  }
  bg->hub_pack_state = 1;
  return true;
}

__global__ void k_add_range(int64_t lo, int64_t hi, const double *__restrict__ local,
                            double *__restrict__ sums) {
  for (int64_t v = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi;
       v += (int64_t)gridDim.x * blockDim.x)
    sums[v] = __dadd_rn(sums[v], local[v]);
}

// ---------------------------------------------------------------------------
// drivers
// ---------------------------------------------------------------------------
template <typename K, typename... Args>
static void launch_window(gcb_ctx *ctx, K kernel, unsigned grid, unsigned block, const void *win,
                          size_t win_bytes, bool use_window, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  if (use_window && win_bytes > 0 && ctx->window_max > 0 && ctx->persist_max > 0) {
    size_t nb = win_bytes < (size_t)ctx->window_max ? win_bytes : (size_t)ctx->window_max;
    float ratio = (float)((double)ctx->persist_max / (double)nb);
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<void *>(win);
    attr[0].val.accessPolicyWindow.num_bytes = nb;
    attr[0].val.accessPolicyWindow.hitRatio = ratio > 1.0f ? 1.0f : ratio;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  GCB_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  ctx->launches++;
}

static unsigned tile_grid(gcb_ctx *ctx, int64_t ntiles) {
  int64_t cap = (int64_t)ctx->num_sms * 8;
  int64_t g = ceil_div(ntiles, kWarps);
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename VT, bool WGT, bool ACCUM>
static void launch_pull_tiles(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, const VT *vals, double *out,
                              bool window) {
  const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
  const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
  const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
  const int64_t vlo = b * bg->width;
  const int64_t vhi = (vlo + bg->width < bg->n) ? vlo + bg->width : bg->n;
  launch_window(ctx, k_pull_tiles<VT, WGT, ACCUM>, tile_grid(ctx, nt), kWarps * 32, vals + vlo,
                (size_t)(vhi - vlo) * sizeof(VT), window, (const uint32_t *)bg->col.p,
                (const double *)(WGT ? bg->w.p : nullptr), (const uint32_t *)(bg->lro.p + rs + b),
                (const uint32_t *)(bg->id_map.p + rs), (const uint32_t *)(bg->tile_row.p + tb), es,
                ee, bg->h_tile_t0[b], nt, (uint32_t)Lb, vals, ACCUM ? out : out + rs,
                bg->carry.p + tb);
}

// Pull gather of every block (or block_only) in block order.
//   accum: out is a dense n-vector, out[id_map[row]] += row_sum (sums / y)
//   else : out is the partials arena, out[arena_row] = row_sum
void pull_sums(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, const float *vals32,
               bool use_weights, uint32_t flags, int64_t block_only, double *out, bool accum) {
  ensure_derived(ctx, bg);
  const bool exact = flags & GCB_FLAG_EXACT;
  if (bg->cb) {
    GCB_REQUIRE(accum && block_only < 0 && vals && !vals32,
                "the cb scheme supports whole-graph pull passes only");
    cb_sums(ctx, bg, vals, use_weights, exact, out);  // partition.cu: the CB ablation
    return;
  }
  if (accum && !exact && vals && !vals32 && block_only < 0) {
    gather_accum(ctx, bg, vals, use_weights, flags, out);  // gather.cu: hot-staged path
    return;
  }
  const bool window = !(flags & GCB_FLAG_NO_L2_WINDOW);
  const bool wgt = use_weights && bg->weighted;
  for (int64_t b = 0; b < bg->B; ++b) {
    if (block_only >= 0 && b != block_only) continue;
    const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    if (Lb == 0) continue;
    const int64_t es = bg->h_edge_starts[b];
    const uint32_t *lro_b = bg->lro.p + rs + b;
    const uint32_t *idm_b = bg->id_map.p + rs;
    ProfScope ps_gather(ctx, 0);
    if (exact || !(vals || vals32)) {
      ensure_long_rows(ctx, bg);
      const unsigned g = grid_for(Lb, 256, (int64_t)ctx->num_sms * 16);
      const double *wb = wgt ? bg->w.p + es : nullptr;
      double *o = accum ? out : out + rs;
      const uint32_t *lr = bg->long_rows.p + bg->h_long_base[b];
      const int64_t nl = bg->h_long_base[b + 1] - bg->h_long_base[b];
      const int64_t nb = bg->h_long_big[b];
      const unsigned gl = grid_for((nb + (nl - nb + 31) / 32) * 32, 256, (int64_t)ctx->num_sms * 16);
      if (wgt && accum) {
        k_pull_exact<true, true><<<g, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
        if (nl) k_pull_exact_long<true, true><<<gl, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      } else if (wgt) {
        k_pull_exact<true, false><<<g, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
        if (nl) k_pull_exact_long<true, false><<<gl, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      } else if (accum) {
        k_pull_exact<false, true><<<g, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
        if (nl) k_pull_exact_long<false, true><<<gl, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      } else {
        k_pull_exact<false, false><<<g, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
        if (nl) k_pull_exact_long<false, false><<<gl, 256, 0, ctx->stream>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      }
      after_launch(ctx, "k_pull_exact");
      continue;
    }
    if (vals32) {
      if (wgt && accum) launch_pull_tiles<float, true, true>(ctx, bg, b, vals32, out, window);
      else if (wgt) launch_pull_tiles<float, true, false>(ctx, bg, b, vals32, out, window);
      else if (accum) launch_pull_tiles<float, false, true>(ctx, bg, b, vals32, out, window);
      else launch_pull_tiles<float, false, false>(ctx, bg, b, vals32, out, window);
    } else {
      if (wgt && accum) launch_pull_tiles<double, true, true>(ctx, bg, b, vals, out, window);
      else if (wgt) launch_pull_tiles<double, true, false>(ctx, bg, b, vals, out, window);
      else if (accum) launch_pull_tiles<double, false, true>(ctx, bg, b, vals, out, window);
      else launch_pull_tiles<double, false, false>(ctx, bg, b, vals, out, window);
    }
    const int64_t sb = bg->h_span_base[b], ns = bg->h_span_base[b + 1] - sb;
    if (ns > 0) {
      ProfScope ps_fix(ctx, 1);
      const int64_t tb = bg->h_tile_base[b];
      const unsigned g = grid_for(ns * 32, 256, (int64_t)ctx->num_sms * 8);
      if (accum)
        k_fixup<true><<<g, 256, 0, ctx->stream>>>(ns, bg->span_tile.p + sb, bg->span_len.p + sb, tb,
                                                  bg->tile_row.p + tb, idm_b, bg->carry.p + tb, out);
      else
        k_fixup<false><<<g, 256, 0, ctx->stream>>>(ns, bg->span_tile.p + sb, bg->span_len.p + sb, tb,
                                                   bg->tile_row.p + tb, idm_b, bg->carry.p + tb,
                                                   out + rs);
      after_launch(ctx, "k_fixup");
    }
  }
}

void merge_to(gcb_ctx *ctx, gcb_blocked *bg, double *out);

// Exact pull pass of a multi-block graph into zeroed sums.  Accumulating
// block by block serialises the blocks' long-row kernels, and each is bound by
// its hub row's dependent add chain (rmat:24: 2.26 + 0.73 ms).  Instead every
// block writes its partials (the same per-row sums) to the partials arena --
// block 0 on the main stream, the others on the auxiliary stream, so the
// chains overlap -- and the block-ordered merge (k_merge, accumulate_ranges
// kernels.py:300-321) forms ((0 + p_0) + p_1) + ..., the value accumulating
// into zeroed sums gives, bit for bit.
static void exact_pull_concurrent(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool wgt,
                                  double *out) {
  ensure_long_rows(ctx, bg);
  bg->partials.ensure(bg->L ? bg->L : 1);
  if (!ctx->aux_stream) {
    GCB_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    GCB_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    GCB_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  }
  GCB_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
  GCB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->fork_ev, 0));
  // block 0's long rows (the hub chains, the critical path) start first on the
  // main stream; every short-row pass and the other blocks run beside them
  for (int64_t b = 0; b < bg->B; ++b) {
    const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    if (Lb == 0) continue;
    cudaStream_t st = b == 0 ? ctx->stream : ctx->aux_stream;
    cudaStream_t sst = ctx->aux_stream;
    const int64_t es = bg->h_edge_starts[b];
    const uint32_t *lro_b = bg->lro.p + rs + b;
    const uint32_t *idm_b = bg->id_map.p + rs;
    const double *wb = wgt ? bg->w.p + es : nullptr;
    double *o = bg->partials.p + rs;
    const uint32_t *lr = bg->long_rows.p + bg->h_long_base[b];
    const int64_t nl = bg->h_long_base[b + 1] - bg->h_long_base[b];
    const int64_t nb = bg->h_long_big[b];
    const unsigned g = grid_for(Lb, 256, (int64_t)ctx->num_sms * 16);
    const unsigned gl = grid_for((nb + (nl - nb + 31) / 32) * 32, 256, (int64_t)ctx->num_sms * 16);
    if (wgt) {
      if (nl) k_pull_exact_long<true, false><<<gl, 256, 0, st>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      k_pull_exact<true, false><<<g, 256, 0, sst>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
    } else {
      if (nl) k_pull_exact_long<false, false><<<gl, 256, 0, st>>>(bg->col.p + es, wb, lro_b, idm_b, lr, nl, nb, vals, o);
      k_pull_exact<false, false><<<g, 256, 0, sst>>>(bg->col.p + es, wb, lro_b, idm_b, Lb, vals, o, kExactShort);
    }
    after_launch(ctx, "k_pull_exact");
  }
  GCB_CUDA(cudaEventRecord(ctx->join_ev, ctx->aux_stream));
  GCB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
  merge_to(ctx, bg, out);
}

void merge_to(gcb_ctx *ctx, gcb_blocked *bg, double *out) {
  ensure_derived(ctx, bg);
  if (bg->R == 0) return;
  k_merge<<<(unsigned)bg->R, 512, 0, ctx->stream>>>(bg->n, bg->B, bg->R, bg->bounds.p, bg->id_map.p,
                                                    bg->partials.p, out);
  after_launch(ctx, "k_merge");
}

// Hub accumulator slots per block (f64 in shared memory).  rmat:24 push,
// ms per iteration: none 3.69, 1K 1.75, 4K 1.48, 16K 1.28, 24K 1.07, 27K 1.07
// -- REDs need no L1 staging, so unlike the pull gather the table can take
// most of the shared memory.
int64_t push_hot_slots(gcb_ctx *ctx) {
  int optin = 0;
  GCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const char *env = getenv("GCB_PUSH_HOT");
  int64_t K = env ? atoll(env) : 24576;
  const int64_t cap = ((int64_t)optin - 1024) / 8;
  return K < cap ? K : cap;
}

void push_scatter(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, double *sums, bool use_weights,
                  uint32_t flags, int64_t block_only, bool nonneg) {
  ensure_derived(ctx, bg);
  if (!(flags & GCB_FLAG_EXACT)) ensure_push_exec(ctx, bg, push_hot_slots(ctx));
  const bool wgt = use_weights && bg->weighted;
  if (flags & GCB_FLAG_EXACT) {
    // bincount order == exact pull of the transpose (relabel.cu ensure_exact_pull);
    // per-block exact scatters go through gcb_process_block_push
    GCB_REQUIRE(block_only < 0, "exact push_scatter covers whole graphs");
    if (bg->m == 0) return;
    pull_sums(ctx, ensure_exact_pull(ctx, bg), vals, nullptr, use_weights, flags, -1, sums, true);
    return;
  }
  for (int64_t b = 0; b < bg->B; ++b) {
    if (block_only >= 0 && b != block_only) continue;
    const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
    if (Lb == 0) continue;
    const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
    const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
    if (bg->hot_k > 0) {
      const int hot = (int)bg->hot_k;
      const size_t smem = (size_t)hot * sizeof(double);
      ensure_smem_attrs(ctx, (const void *)k_push_hot<true>, smem);
      ensure_smem_attrs(ctx, (const void *)k_push_hot<false>, smem);
      ensure_smem_attrs(ctx, (const void *)k_push_hot<false, true>, smem);
      const unsigned gh = grid_for(nt * 32, 1024, (int64_t)ctx->num_sms);
      constexpr int kHubNW = 32;
      const size_t smem_hub = (size_t)(hot + 32) * sizeof(double) +
                              (size_t)kHubNW * kHubRows * sizeof(unsigned long long);
      const char *hv = getenv("GCB_HUB_KERNEL");
      if (nonneg && !wgt && !getenv("GCB_NO_FIX") && !(hv && hv[0] == '0') &&
          smem_hub <= (size_t)max_smem_optin(ctx) && ensure_hub_pack(ctx, bg)) {
        ensure_smem_attrs(ctx, (const void *)k_push_hub<kHubNW>, smem_hub);
        if (!bg->hub_acc.p) {
          bg->hub_acc.alloc(hot);
          GCB_CUDA(cudaMemsetAsync(bg->hub_acc.p, 0, hot * sizeof(unsigned long long), ctx->stream));
        }
        k_push_hub<kHubNW><<<gh, kHubNW * 32, smem_hub, ctx->stream>>>(
            bg->hub_pack.p, bg->tile_row.p, (uint32_t)nt, (uint32_t)Lb, bg->id_map.p, hot, vals,
            bg->hub_acc.p);
        after_launch(ctx, "k_push_hub");
        k_hub_fold<<<grid_for(hot, 256, 1024), 256, 0, ctx->stream>>>(hot, bg->hot_ids.p,
                                                                      bg->hub_acc.p, sums);
        after_launch(ctx, "k_hub_fold");
        continue;
      }
      if (nonneg && !wgt && !getenv("GCB_NO_FIX"))
        k_push_hot<false, true><<<gh, 1024, smem, ctx->stream>>>(
            bg->xcol.p, nullptr, bg->rstart.p, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt,
            (uint32_t)Lb, bg->id_map.p + rs, bg->hot_ids.p + b * bg->hot_k, hot, vals, sums);
      else if (wgt)
        k_push_hot<true><<<gh, 1024, smem, ctx->stream>>>(
            bg->xcol.p, bg->w.p, bg->rstart.p, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt,
            (uint32_t)Lb, bg->id_map.p + rs, bg->hot_ids.p + b * bg->hot_k, hot, vals, sums);
      else
        k_push_hot<false><<<gh, 1024, smem, ctx->stream>>>(
            bg->xcol.p, nullptr, bg->rstart.p, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt,
            (uint32_t)Lb, bg->id_map.p + rs, bg->hot_ids.p + b * bg->hot_k, hot, vals, sums);
      after_launch(ctx, "k_push_hot");
      continue;
    }
    const unsigned g = grid_for(nt * 32, 256, (int64_t)ctx->num_sms * 8);
    if (wgt)
      k_push_bits<true><<<g, 256, 0, ctx->stream>>>(
          bg->col.p, bg->w.p, bg->rstart.p, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt,
          (uint32_t)Lb, bg->id_map.p + rs, vals, sums);
    else
      k_push_bits<false><<<g, 256, 0, ctx->stream>>>(
          bg->col.p, nullptr, bg->rstart.p, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt,
          (uint32_t)Lb, bg->id_map.p + rs, vals, sums);
    after_launch(ctx, "k_push_bits");
  }
}

}  // namespace gcb

// The tol > 0 convergence loop (kernels.py:257-266 / 397-404) as one CUDA graph:
// a WHILE conditional node whose body is one iteration's launches plus
// k_pr_check, which tests delta < tol on the device and sets the loop
// condition, so iterations 2.. run with no host round trip (the host loop
// read delta back after every iteration: +24 us per iteration at rmat:24).
// The body is captured once per blocking and reused while the buffers it
// was captured with stay the same.
struct PrGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  gcb::DArray<int> state;  // [iterations run, converged, iteration budget]
  static constexpr int kKey = 24;
  const void *key[kKey] = {};
  double kd[2] = {0, 0};
  uint32_t kflags = 0;
  int kdir = -1;
};

namespace gcb {

void destroy_pr_graph(PrGraph *g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

__global__ void k_pr_check(cudaGraphConditionalHandle h, const double *__restrict__ delta,
                           double tol, int *__restrict__ state) {
  const int k = ++state[0];
  const bool done = *delta < tol;
  if (done) state[1] = 1;
  cudaGraphSetConditional(h, (!done && k < state[2]) ? 1u : 0u);
}

static bool graph_loops_enabled(gcb_ctx *ctx) {
  const char *env = getenv("GCB_NO_GRAPH");
  return !ctx->profiling && !(env && env[0] && env[0] != '0');
}

// Runs up to `budget` more iterations of `iterate` inside one graph launch;
// returns false (nothing run) when the graph cannot be built, and the caller
// keeps the host loop.
template <class F>
static bool pr_graph_loop(gcb_ctx *ctx, gcb_blocked *bg, F &&iterate, const void *const *key,
                          double damping, double tol, uint32_t flags, const double *delta_dev,
                          int budget, int *ran, int *conv) {
  PrGraph *g = bg->pr_graph;
  bool same = g && g->kd[0] == damping && g->kd[1] == tol && g->kflags == flags &&
              g->kdir == bg->direction;
  for (int i = 0; same && i < PrGraph::kKey; ++i) same = g->key[i] == key[i];
  if (!same) {
    destroy_pr_graph(g);
    bg->pr_graph = g = nullptr;
    PrGraph *ng = new PrGraph();
    cudaStream_t cs = nullptr, saved = ctx->stream;
    bool ok = false, capturing = false;
    try {
      ng->state.alloc(3);
      if (cudaGraphCreate(&ng->graph, 0) != cudaSuccess) throw 0;
      cudaGraphConditionalHandle h;
      if (cudaGraphConditionalHandleCreate(&h, ng->graph, 1, cudaGraphCondAssignDefault) != cudaSuccess)
        throw 0;
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = h;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      if (cudaGraphAddNode(&node, ng->graph, nullptr, 0, &p) != cudaSuccess) throw 0;
      cudaGraph_t body = p.conditional.phGraph_out[0];
      if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) throw 0;
      if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed) != cudaSuccess)
        throw 0;
      capturing = true;
      ctx->stream = cs;
      iterate(true);  // tol > 0: every iteration needs its delta
      k_pr_check<<<1, 1, 0, cs>>>(h, delta_dev, tol, ng->state.p);
      after_launch(ctx, "k_pr_check");
      ctx->stream = saved;
      capturing = false;
      if (cudaStreamEndCapture(cs, &body) != cudaSuccess) throw 0;
      if (cudaGraphInstantiate(&ng->exec, ng->graph, 0) != cudaSuccess) throw 0;
      ok = true;
    } catch (...) {
      // any failure (no conditional-node support, an operation the capture
      // rejects): the caller keeps the host loop
      ok = false;
    }
    ctx->stream = saved;
    if (capturing) {
      cudaGraph_t dropped = nullptr;
      cudaStreamEndCapture(cs, &dropped);
    }
    if (cs) cudaStreamDestroy(cs);
    if (!ok) {
      destroy_pr_graph(ng);
      cudaGetLastError();  // clear the (non-sticky) error of the failed build
      return false;
    }
    for (int i = 0; i < PrGraph::kKey; ++i) ng->key[i] = key[i];
    ng->kd[0] = damping;
    ng->kd[1] = tol;
    ng->kflags = flags;
    ng->kdir = bg->direction;
    bg->pr_graph = g = ng;
  }
  int *hs = (int *)ctx->pinned;
  hs[0] = 0;
  hs[1] = 0;
  hs[2] = budget;
  GCB_CUDA(cudaMemcpyAsync(g->state.p, hs, 3 * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  GCB_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
  ctx->launches++;
  GCB_CUDA(cudaMemcpyAsync(hs, g->state.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  *ran = hs[0];
  *conv = hs[1];
  return true;
}

// PageRank driver shared by pr_blocked / pr_baseline (kernels.py:207-268, 367-405)
static void pr_run(gcb_ctx *ctx, gcb_blocked *bg, double damping, double tol, int max_iters,
                   uint32_t flags, const uint32_t *deg_override, double *ranks_dev, int *iters,
                   int *conv) {
  GCB_REQUIRE(damping > 0.0 && damping < 1.0, "damping must lie in (0, 1)");
  GCB_REQUIRE(tol >= 0.0, "tol must be >= 0");
  GCB_REQUIRE(max_iters >= 1, "max_iters must be >= 1");
  GCB_REQUIRE(bg->n > 0, "PageRank needs at least one vertex");
  ensure_derived(ctx, bg);
  const int64_t n = bg->n;
  const bool exact = flags & GCB_FLAG_EXACT;
  const bool push = bg->direction == 1;
  if (!(flags & GCB_FLAG_F32_VALUES) && !deg_override && relabel_enabled(bg, flags, max_iters)) {
    // run on the degree-ordered copy (relabel.cu); ranks come back in input order
    gcb_blocked *rl = ensure_relabeled(ctx, bg);
    rl->ranks.ensure(n);
    pr_run(ctx, rl, damping, tol, max_iters, flags, nullptr, rl->ranks.p, iters, conv);
    permute_out(ctx, bg, rl->ranks.p, ranks_dev);
    return;
  }
  const bool f32 = (flags & GCB_FLAG_F32_VALUES) && !exact && !push;
  const uint32_t *deg = deg_override ? deg_override : bg->deg.p;
  bg->contrib.ensure(n);
  if (f32) bg->contrib32.ensure(n);
  bg->sums.ensure(n);
  // one 4-vertex quad per thread: enough loads in flight to run at HBM speed
  // (a capped grid-stride loop left this pass latency-bound, 0.26 IPC in ncu)
  const unsigned upd_grid = grid_for((n + 3) / 4, 256, 1 << 20);
  const int64_t nslots = (int64_t)upd_grid > 3 * (int64_t)ctx->num_sms ? (int64_t)upd_grid
                                                                         : 3 * (int64_t)ctx->num_sms;
  bg->deltas.ensure(nslots + 2);
  double *delta_dev = bg->deltas.p + bg->deltas.n - 1;
  const double r0 = 1.0 / (double)n;
  const double base = (1.0 - damping) / (double)n;
  double *contrib = f32 ? nullptr : bg->contrib.p;
  float *contrib32 = f32 ? bg->contrib32.p : nullptr;
  // Live range of the degree-ordered copy.  Its ids are sorted by descending
  // out-degree, so [n_live, n) is every vertex with out-degree 0: its
  // contribution is 0 in every iteration (kernels.py:185-191), and with
  // tol == 0 its intermediate ranks are never read (no delta; only the last
  // iteration's ranks are returned).  Those iterations update [0, n_live)
  // only (rmat:24: 7.38M of 16.8M vertices -- most R-MAT vertices are
  // isolated); the last one updates the rest after clearing the sums the
  // skipped updates did not clear.  [n_conn, n) are isolated vertices: their
  // sums stay 0 and all share one rank, so the last update stops at n_conn + 1
  // (permute_out fills them from that one value), and once a buffer pair has
  // been initialised in full their zero contributions and sums are not
  // rewritten.  The ranks are unchanged: the skipped work is dead.
  int64_t n_upd = n, n_fin = n, n_init = n;
  if (bg->is_relabeled && tol == 0.0 && !exact && !push && !f32 && !deg_override) {
    if (bg->n_live < 0) {
      DArray<unsigned long long> cnt(1);
      GCB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
      k_count_nonzero_u32<<<grid_for(n, 256, 4096), 256, 0, ctx->stream>>>(n, deg, cnt.p);
      after_launch(ctx, "k_count_nonzero_u32");
      unsigned long long h = 0;
      d2h(ctx, &h, cnt.p, 1);
      sync(ctx);
      bg->n_live = (int64_t)h;
    }
    const char *lv = getenv("GCB_FULL_UPDATE");  // A/B knob: 1 updates every vertex
    if (!(lv && lv[0] == '1')) {
      n_upd = bg->n_live;
      if (bg->n_conn > 0 && bg->n_conn < n) {
        n_fin = bg->n_conn + 1;
        if (bg->iso_clean[0] == bg->contrib.p && bg->iso_clean[1] == bg->sums.p) n_init = n_fin;
      }
    }
  }
  {
    ProfScope ps(ctx, 3);
    k_pr_init<<<grid_for((n_init + 3) / 4, 256, 1 << 20), 256, 0, ctx->stream>>>(
        n_init, r0, deg, tol > 0.0 ? ranks_dev : nullptr, contrib ? contrib : bg->contrib.p,
        contrib32, bg->sums.p);
    after_launch(ctx, "k_pr_init");
    if (n_init == n) {
      bg->iso_clean[0] = bg->contrib.p;
      bg->iso_clean[1] = bg->sums.p;
    }
  }
  // one iteration's launches (no host synchronisation: also the graph body);
  // with_ranks = false only where the ranks and delta are dead (tol == 0, not
  // the last iteration: see k_pr_update2)
  auto iterate = [&](bool with_ranks) {
    if (!push && exact && !bg->cb && bg->B >= 1 && contrib) {
      ProfScope ps(ctx, 0);
      exact_pull_concurrent(ctx, bg, contrib, false, bg->sums.p);
    } else if (!push) {
      pull_sums(ctx, bg, contrib, contrib32, false, flags, -1, bg->sums.p, true);
      if (bg->hybrid) {  // relabel.cu: cold-source -> hot-destination edges
        ProfScope ps(ctx, 1);
        push_scatter(ctx, bg->hybrid, contrib, bg->sums.p, false, flags, -1, true);
      }
    } else {
      ProfScope ps(ctx, 0);
      // plain push PageRank keeps the f64 table: measured 1.09 ms vs 1.19 ms per
      // iteration with the fixed-point one at rmat:24 (its hub slots see far
      // more adds per CTA than the hybrid's, and the two-word add costs more)
      push_scatter(ctx, bg, bg->contrib.p, bg->sums.p, false, flags, -1, false);
    }
    {
      ProfScope ps(ctx, 2);
      launch_update(ctx, exact, with_ranks ? n_fin : n_upd, base, damping, bg->sums.p, ranks_dev, deg,
                    contrib ? contrib : (push ? bg->contrib.p : nullptr), contrib32,
                    tol > 0.0 ? bg->deltas.p : nullptr, with_ranks);
    }
    if (tol > 0.0) {
      k_reduce_sum<<<1, 1024, 0, ctx->stream>>>(bg->deltas.p, update_grid(ctx, n), delta_dev);
      after_launch(ctx, "k_reduce_sum");
    }
  };
  double *hdelta = (double *)ctx->pinned;
  int it = 0, cv = 0;
  const char *kr = getenv("GCB_KEEP_RANKS");  // 1: full update every iteration (A/B knob)
  const bool keep_ranks = kr && kr[0] == '1';
  for (int k = 0; k < max_iters; ++k) {
    const bool last = tol > 0.0 || k == max_iters - 1 || keep_ranks;
    if (last && k > 0 && n_upd < n_fin)
      GCB_CUDA(cudaMemsetAsync(bg->sums.p + n_upd, 0, (n_fin - n_upd) * sizeof(double),
                               ctx->stream));
    iterate(last);
    ++it;
    if (tol > 0.0) {
      d2h(ctx, hdelta, delta_dev, 1);
      sync(ctx);
      if (*hdelta < tol) {
        cv = 1;
        break;
      }
      // the first iteration built every lazy structure: the rest can loop on
      // the device
      if (k == 0 && max_iters > 1 && graph_loops_enabled(ctx)) {
        // every buffer the captured launches read or write: a rebuilt layout
        // (other table sizes, say) or another output vector means a new graph
        const gcb_blocked *hy = bg->hybrid;
        const void *key[PrGraph::kKey] = {bg, ranks_dev, deg, contrib, contrib32, bg->sums.p,
                                          bg->deltas.p, hy, bg->xcol.p, bg->hotval.p,
                                          bg->hot_ids.p, bg->rstart.p, bg->tile_row.p,
                                          (const void *)(intptr_t)bg->hot_k,
                                          hy ? hy->xcol.p : nullptr,
                                          hy ? (const void *)(intptr_t)hy->hot_k : nullptr,
                                          // the exact pull's buffers
                                          bg->partials.p, bg->bounds.p, bg->long_rows.p,
                                          bg->carry.p, bg->span_tile.p, bg->span_len.p,
                                          (const void *)(intptr_t)bg->direction,
                                          (const void *)(intptr_t)bg->B};
        int ran = 0, c2 = 0;
        if (pr_graph_loop(ctx, bg, iterate, key, damping, tol, flags, delta_dev, max_iters - 1,
                          &ran, &c2)) {
          it += ran;
          cv = c2;
          break;
        }
      }
    }
  }
  *iters = it;
  *conv = cv;
}

// Shard steps with GCB_FLAG_DEAD_SKIP on a degree-ordered shard (ids sorted by
// descending out-degree: [n_live, n) have none): the step's ranks and delta
// are dead, so only [v0, min(v1, n_live)) is updated; the sums of the rest are
// then not cleared, and the next step without the flag (the last iteration)
// clears them before its gather.  Returns the end of the range to update.
int64_t shard_live_range(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, uint32_t flags,
                         const uint32_t *deg_dev) {
  const bool skip = (flags & GCB_FLAG_DEAD_SKIP) && bg->is_relabeled && !(flags & GCB_FLAG_EXACT);
  if (skip || bg->dead_dirty) {
    if (bg->n_live < 0) {
      DArray<unsigned long long> cnt(1);
      GCB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
      k_count_nonzero_u32<<<grid_for(bg->n, 256, 4096), 256, 0, ctx->stream>>>(bg->n, deg_dev,
                                                                                cnt.p);
      after_launch(ctx, "k_count_nonzero_u32");
      unsigned long long h = 0;
      d2h(ctx, &h, cnt.p, 1);
      sync(ctx);
      bg->n_live = (int64_t)h;
    }
  }
  const int64_t live = bg->n_live < 0 ? v1 : (bg->n_live < v0 ? v0 : (bg->n_live > v1 ? v1 : bg->n_live));
  if (!skip) {
    if (bg->dead_dirty && live < v1)
      GCB_CUDA(cudaMemsetAsync(bg->sums.p + live, 0, (v1 - live) * sizeof(double), ctx->stream));
    bg->dead_dirty = false;
    return v1;
  }
  if (live < v1) bg->dead_dirty = true;
  return live;
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_compute_contributions(gcb_ctx *ctx, int64_t n, const double *ranks_host,
                              const int64_t *out_degrees_host, double *out_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && ((ranks_host && out_degrees_host && out_host) || n == 0), "NULL argument");
  DeviceGuard dg(ctx->device);
  if (n == 0) return GCB_OK;
  DArray<double> r(n), o(n);
  DArray<int64_t> d(n);
  h2d(ctx, r.p, ranks_host, n);
  h2d(ctx, d.p, out_degrees_host, n);
  k_contributions<<<grid_for(n, 256, 65536), 256, 0, ctx->stream>>>(n, r.p, d.p, o.p);
  after_launch(ctx, "k_contributions");
  d2h(ctx, out_host, o.p, n);
  sync(ctx);
  GCB_API_END
}

int gcb_pr_blocked_dev(gcb_ctx *ctx, gcb_blocked *bg, double damping, double tol, int max_iters,
                       uint32_t flags, double *ranks_dev, int *iterations, int *converged) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && ranks_dev && iterations && converged, "NULL argument");
  DeviceGuard dg(ctx->device);
  pr_run(ctx, bg, damping, tol, max_iters, flags, nullptr, ranks_dev, iterations, converged);
  GCB_API_END
}

int gcb_pr_blocked(gcb_ctx *ctx, gcb_blocked *bg, double damping, double tol, int max_iters,
                   int64_t k, uint32_t flags, double *ranks_host, int *iterations, int *converged) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && ranks_host && iterations && converged, "NULL argument");
  GCB_REQUIRE(k >= 1, "range width k must be >= 1");
  DeviceGuard dg(ctx->device);
  bg->ranks.ensure(bg->n ? bg->n : 1);
  pr_run(ctx, bg, damping, tol, max_iters, flags, nullptr, bg->ranks.p, iterations, converged);
  d2h(ctx, ranks_host, bg->ranks.p, bg->n);
  sync(ctx);
  GCB_API_END
}

static gcb_blocked *compact_for(gcb_ctx *ctx, const gcb_csr *g_const, int direction) {
  gcb_csr *g = const_cast<gcb_csr *>(g_const);
  gcb_blocked *v = csr_compact_view(ctx, g);
  if (v->direction != direction) {
    // same arena, other degree semantics: rebuild the derived tables
    v->direction = direction;
    v->derived = false;
  }
  return v;
}

int gcb_pr_baseline(gcb_ctx *ctx, const gcb_csr *g, int direction, double damping, double tol,
                    int max_iters, uint32_t flags, const int64_t *out_degrees_host_or_null,
                    double *ranks_host, int *iterations, int *converged) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && ranks_host && iterations && converged, "NULL argument");
  GCB_REQUIRE(direction == 0 || direction == 1, "direction must be pull or push");
  DeviceGuard dg(ctx->device);
  gcb_blocked *v = compact_for(ctx, g, direction);
  DArray<uint32_t> dover;
  if (out_degrees_host_or_null) {
    std::vector<uint32_t> d32(g->n);
    for (int64_t i = 0; i < g->n; ++i) {
      GCB_REQUIRE(out_degrees_host_or_null[i] >= 0 && out_degrees_host_or_null[i] < (int64_t(1) << 32),
                  "out_degrees out of range");
      d32[i] = (uint32_t)out_degrees_host_or_null[i];
    }
    dover.alloc(g->n);
    h2d(ctx, dover.p, d32.data(), g->n);
  }
  v->ranks.ensure(v->n ? v->n : 1);
  pr_run(ctx, v, damping, tol, max_iters, flags, out_degrees_host_or_null ? dover.p : nullptr,
         v->ranks.p, iterations, converged);
  d2h(ctx, ranks_host, v->ranks.p, v->n);
  sync(ctx);
  GCB_API_END
}

int gcb_process_block_pull(gcb_ctx *ctx, gcb_blocked *bg, int64_t block, const double *contrib_host,
                           uint32_t flags, double *out_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && contrib_host && out_host, "NULL argument");
  if (block < 0 || block >= bg->B) fail(GCB_EINDEX, "%lld", (long long)block);
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->contrib.ensure(bg->n ? bg->n : 1);
  bg->partials.ensure(bg->L > 0 ? bg->L : 1);
  h2d(ctx, bg->contrib.p, contrib_host, bg->n);
  const int64_t rs = bg->h_row_starts[block], Lb = bg->h_row_starts[block + 1] - rs;
  GCB_CUDA(cudaMemsetAsync(bg->partials.p + rs, 0, (Lb ? Lb : 1) * sizeof(double), ctx->stream));
  pull_sums(ctx, bg, bg->contrib.p, nullptr, false, flags, block, bg->partials.p, false);
  d2h(ctx, out_host, bg->partials.p + rs, Lb);
  sync(ctx);
  GCB_API_END
}

int gcb_process_block_push(gcb_ctx *ctx, gcb_blocked *bg, int64_t block, const double *contrib_host,
                           uint32_t flags, double *sums_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && contrib_host && sums_host, "NULL argument");
  if (block < 0 || block >= bg->B) fail(GCB_EINDEX, "%lld", (long long)block);
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  const int64_t n = bg->n;
  bg->contrib.ensure(n ? n : 1);
  DArray<double> local(n ? n : 1), dsums(n ? n : 1);
  h2d(ctx, bg->contrib.p, contrib_host, n);
  h2d(ctx, dsums.p, sums_host, n);
  GCB_CUDA(cudaMemsetAsync(local.p, 0, (n ? n : 1) * sizeof(double), ctx->stream));
  // unweighted, like the reference (kernels.py:291-293).  Exact: the block's
  // destinations [lo, hi) get exactly their bincount sums from the exact pull
  // over the transpose (every destination lives in one push block); the rows
  // of other blocks land in `local` too but are not added below.
  if ((flags & GCB_FLAG_EXACT) && bg->m > 0)
    pull_sums(ctx, ensure_exact_pull(ctx, bg), bg->contrib.p, nullptr, false, flags, -1, local.p,
              true);
  else
    push_scatter(ctx, bg, bg->contrib.p, local.p, false, flags, block);
  const int64_t lo = block * bg->width, hi = (lo + bg->width < n) ? lo + bg->width : n;
  if (hi > lo) {
    k_add_range<<<grid_for(hi - lo, 256, 4096), 256, 0, ctx->stream>>>(lo, hi, local.p, dsums.p);
    after_launch(ctx, "k_add_range");
  }
  d2h(ctx, sums_host, dsums.p, n);
  sync(ctx);
  GCB_API_END
}

int gcb_accumulate_ranges(gcb_ctx *ctx, gcb_blocked *bg, const double *partials_host, int64_t k,
                          double *out_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && out_host && (partials_host || bg->L == 0), "NULL argument");
  GCB_REQUIRE(k >= 1, "range width k must be >= 1");
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->partials.ensure(bg->L > 0 ? bg->L : 1);
  h2d(ctx, bg->partials.p, partials_host, bg->L);
  DArray<double> y(bg->n ? bg->n : 1);
  merge_to(ctx, bg, y.p);
  d2h(ctx, out_host, y.p, bg->n);
  sync(ctx);
  GCB_API_END
}

// y = pull gather of x over a blocking, accumulated block by block.  SpMV
// stays on the input numbering: the degree-ordered copy would need x and y
// permuted on every call (two random passes over n values), which cost more
// than its faster gather saves -- rmat:22 device SpMV 0.242 ms promoted
// against 0.199 ms without.  PageRank keeps its vectors in the copy's order
// across iterations, so only pr_run promotes.
static void pull_spmv(gcb_ctx *ctx, gcb_blocked *bg, const double *x, bool weights, uint32_t flags,
                      double *y) {
  GCB_CUDA(cudaMemsetAsync(y, 0, (bg->n ? bg->n : 1) * sizeof(double), ctx->stream));
  pull_sums(ctx, bg, x, nullptr, weights, flags, -1, y, true);
}

int gcb_segment_row_sums(gcb_ctx *ctx, const gcb_csr *g, const double *values_host, int use_weights,
                         uint32_t flags, double *out_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out_host && (values_host || g->n == 0), "NULL argument");
  DeviceGuard dg(ctx->device);
  gcb_blocked *v = compact_for(ctx, g, 0);
  DArray<double> x(g->n ? g->n : 1), y(g->n ? g->n : 1);
  h2d(ctx, x.p, values_host, g->n);
  pull_spmv(ctx, v, x.p, use_weights != 0, flags, y.p);
  d2h(ctx, out_host, y.p, g->n);
  sync(ctx);
  GCB_API_END
}

int gcb_spmv(gcb_ctx *ctx, const gcb_csr *g, const double *x_host, int direction, uint32_t flags,
             double *y_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && y_host && (x_host || g->n == 0), "NULL argument");
  GCB_REQUIRE(direction == 0 || direction == 1, "direction must be pull or push");
  DeviceGuard dg(ctx->device);
  gcb_blocked *v = compact_for(ctx, g, direction);
  DArray<double> x(g->n ? g->n : 1), y(g->n ? g->n : 1);
  h2d(ctx, x.p, x_host, g->n);
  if (direction == 0) {
    pull_spmv(ctx, v, x.p, true, flags, y.p);
  } else {
    GCB_CUDA(cudaMemsetAsync(y.p, 0, (g->n ? g->n : 1) * sizeof(double), ctx->stream));
    push_scatter(ctx, v, x.p, y.p, true, flags, -1);
  }
  d2h(ctx, y_host, y.p, g->n);
  sync(ctx);
  GCB_API_END
}

static void spmv_blocked_dev(gcb_ctx *ctx, gcb_blocked *bg, const double *x, uint32_t flags,
                             double *y) {
  ensure_derived(ctx, bg);
  if (bg->direction == 0) {
    pull_spmv(ctx, bg, x, true, flags, y);
  } else {
    GCB_CUDA(cudaMemsetAsync(y, 0, (bg->n ? bg->n : 1) * sizeof(double), ctx->stream));
    push_scatter(ctx, bg, x, y, true, flags, -1);
  }
}

int gcb_spmv_blocked(gcb_ctx *ctx, gcb_blocked *bg, const double *x_host, int64_t k, uint32_t flags,
                     double *y_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && y_host && (x_host || bg->n == 0), "NULL argument");
  GCB_REQUIRE(k >= 1, "range width k must be >= 1");
  DeviceGuard dg(ctx->device);
  DArray<double> x(bg->n ? bg->n : 1), y(bg->n ? bg->n : 1);
  h2d(ctx, x.p, x_host, bg->n);
  spmv_blocked_dev(ctx, bg, x.p, flags, y.p);
  d2h(ctx, y_host, y.p, bg->n);
  sync(ctx);
  GCB_API_END
}

int gcb_spmv_blocked_dev(gcb_ctx *ctx, gcb_blocked *bg, const double *x_dev, uint32_t flags,
                         double *y_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && y_dev && (x_dev || bg->n == 0), "NULL argument");
  DeviceGuard dg(ctx->device);
  spmv_blocked_dev(ctx, bg, x_dev, flags, y_dev);
  GCB_API_END
}

// ---------------------------------------------------------------------------
// Destination-sharded PageRank: rank r owns vertices [v0, v1) of
// the transpose; its blocking holds only those rows, the contribution vector
// is the full n-vector kept in sync by the caller's all-gather of every
// rank's [v0, v1) slice.  deg_dev = global out-degrees (gcb_csr_col_counts).
// ---------------------------------------------------------------------------
int gcb_pr_shard_init(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, const uint32_t *deg_dev,
                      double *contrib_dev, double *ranks_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && deg_dev && contrib_dev && ranks_dev, "NULL argument");
  GCB_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= bg->n && bg->n > 0 && (v0 % 4) == 0, "bad shard range");
  GCB_REQUIRE(bg->direction == 0, "sharded PageRank runs on a pull blocking");
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->sums.ensure(bg->n);
  GCB_CUDA(cudaMemsetAsync(bg->sums.p, 0, bg->n * sizeof(double), ctx->stream));
  const int64_t cnt = v1 - v0;
  if (cnt) {
    k_pr_init<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(
        cnt, 1.0 / (double)bg->n, deg_dev + v0, ranks_dev + v0, contrib_dev + v0, nullptr,
        bg->sums.p + v0);
    after_launch(ctx, "k_pr_init");
  }
  GCB_API_END
}

int gcb_pr_shard_step(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, double damping,
                      uint32_t flags, const uint32_t *deg_dev, double *contrib_dev,
                      double *ranks_dev, double *delta_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && deg_dev && contrib_dev && ranks_dev, "NULL argument");
  GCB_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= bg->n && (v0 % 4) == 0, "bad shard range");
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->sums.ensure(bg->n);
  const int64_t u1 = shard_live_range(ctx, bg, v0, v1, flags, deg_dev);
  const bool dead_skip = u1 < v1 || (flags & GCB_FLAG_DEAD_SKIP);
  const int64_t cnt = u1 - v0;
  const unsigned grid = update_grid(ctx, cnt);
  bg->deltas.ensure((int64_t)grid + 2);
  // gather reads the full contribution vector, then the owned slice is
  // updated in place (stream order keeps the two phases apart)
  pull_sums(ctx, bg, contrib_dev, nullptr, false, flags, -1, bg->sums.p, true);
  if (bg->hybrid) {  // degree-ordered shard (gcb_shard_blocking): hub-destination edges
    ProfScope ps(ctx, 1);
    push_scatter(ctx, bg->hybrid, contrib_dev, bg->sums.p, false, flags, -1, true);
  }
  if (cnt) {
    ProfScope ps(ctx, 2);
    launch_update(ctx, flags & GCB_FLAG_EXACT, cnt, (1.0 - damping) / (double)bg->n, damping,
                  bg->sums.p + v0, ranks_dev + v0, deg_dev + v0, contrib_dev + v0, nullptr,
                  delta_dev ? bg->deltas.p : nullptr,  // no delta wanted: old ranks unread
                  !(dead_skip && !delta_dev));         // dead-skip steps: ranks dead too
  }
  if (delta_dev) {
    if (cnt) {
      k_reduce_sum<<<1, 1024, 0, ctx->stream>>>(bg->deltas.p, grid, delta_dev);
      after_launch(ctx, "k_reduce_sum");
    } else {
      GCB_CUDA(cudaMemsetAsync(delta_dev, 0, sizeof(double), ctx->stream));
    }
  }
  GCB_API_END
}

}  // extern "C"

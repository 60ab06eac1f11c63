// gather.cu -- the fast TOCAB pull gather (K2): every block's rows are
// summed straight into a dense per-vertex vector (sums[id_map[row]] += row
// sum), with the block's hottest sources staged in shared memory.
//
// What bounds it (ncu + microbenchmarks, profiles/ and scripts/mb_*.cu):
//   * every cold gather is one L1TEX->XBAR request; the SM issues at most ~1
//     per cycle (l1tex__m_l1tex2xbar_req_cycles_active reaches 94% in a pure
//     random-gather loop at 0.93 gathers/SM-cycle, scripts/mb_gather.cu);
//   * a shared-memory hit costs no request (random LDS: ~3.7 per SM-cycle,
//     scripts/mb_smem.cu), so the hot table is the only way below that floor;
//   * but misses are staged in L1 lines: the random-LDG rate falls to 0.86 /
//     0.50 / 0.23 per SM-cycle with 128 / 192 / 220 KB of shared memory, so
//     the table is sized to a 124 KB carve-out (~15K f64 slots);
//   * TMA tile::gather4 (0.5/cycle) and DSMEM (0.2-0.6/cycle) are slower.
// So the kernel is built to issue nothing but the cold gathers on the
// request path, and as few instructions as possible around them:
//   * col_idx: one 256-bit load per lane (8 edges = one full sector);
//   * row boundaries: a 1-bit-per-edge row-start bitmap (one 32-byte sector
//     per 256-edge tile) -- local rows are never empty (blocking.py:189-201),
//     so row(q) = tile_row + #row starts in (first, q];
//   * hot test + LDS/LDG as predicated loads (no divergent branches);
//   * tiles inside a single row (47% at rmat:24) take a plain warp reduction;
//     the rest use in-lane runs + a segmented shuffle scan over lane tails;
//   * ASSIGN: the first block of a pass stores rows (sums is zero) instead of
//     read-modify-writing them; rows that cross a tile use f64 RED.
// The order of the RED contributions is not fixed, so this path is
// deterministic only up to reassociation (|err| ~ 1e-16 relative); the exact
// mode (pr.cu, k_pull_exact) is the bit-reproducible path.
//
// Hot sets: on the degree-ordered copy (relabel.cu) the hot sources of a
// block are its first `hot` ids, read straight from the value vector; on any
// other pull graph the top-`hot` sources by out-degree are recoded in an
// execution copy of the arena (xcol = 0x80000000 | slot) and their values
// gathered into hotval once per pass (k_fill_hot).
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "gcb_internal.cuh"
#include "ldst.cuh"
#include "tiles.cuh"

namespace gcb {

constexpr int kGWarps = 32;  // warps per CTA (1 CTA per SM)
constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kHotBit = 0x80000000u;
constexpr double kL2KeepMB = 32.0;  // evict_last head of a degree-ordered value slice

// One source value: a hot source from shared memory, everything else from
// L2 (evict_last keeps the block's value slice resident; no L1 allocation --
// cold lines would only evict each other).  Predicated loads, no branch: the
// compiler's if/else cost a BSSY/BSYNC pair per edge.
//   HOTBIT: c is an xcol entry, hot iff bit 31 is set (slot = low bits);
//   else  : c is a source id, hot iff c - lo < hot (degree-ordered prefix).
#ifdef GCB_ABLATE
// timing ablations (instrumented build only): bit 0 drop the row stores,
// bit 1 drop the cold gathers, bit 2 one warp sum per tile instead of the
// per-row reduction
__constant__ int c_abl;
#define ABL(b) ((c_abl >> (b)) & 1)
#else
#define ABL(b) 0
#endif

template <bool HOTBIT, bool HINT = true, bool LO0 = false>
__device__ __forceinline__ double gather_one(const double *vals, uint32_t c, uint32_t lo,
                                             uint32_t hot, uint32_t s_hot, uint64_t pol) {
  // LO0: the block's sources start at id 0 (block 0), so the slot is the id
  const uint32_t h = HOTBIT ? (c ^ kHotBit) : (LO0 ? c : c - lo);
  double x;
  if (ABL(1) && h >= hot) return 0.0;
  if (HINT)
    asm("{\n\t.reg .pred p;\n\t"
        "setp.lt.u32 p, %1, %2;\n\t"
        "@p ld.shared.f64 %0, [%3];\n\t"
        "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%4], %5;\n\t}"
        : "=d"(x)
        : "r"(h), "r"(hot), "r"(s_hot + h * 8u), "l"(vals + c), "l"(pol));
  else  // no per-load policy: the launch's access-policy window governs L2
    asm("{\n\t.reg .pred p;\n\t"
        "setp.lt.u32 p, %1, %2;\n\t"
        "@p ld.shared.f64 %0, [%3];\n\t"
        "@!p ld.global.nc.L1::no_allocate.f64 %0, [%4];\n\t}"
        : "=d"(x)
        : "r"(h), "r"(hot), "r"(s_hot + h * 8u), "l"(vals + c));
  return x;
}

// ASSIGN: out is all zero before this launch (first block of the pass), so a
// row that lies inside one tile is stored (out[v] = x) instead of
// read-modify-written -- no dependent load on the emit path.
// L2 policy of the cold gathers: mode 0 evict_last over everything; modes 1/2
// a range policy over the block's value slice (policy_range, ldst.cuh)
struct RangePolicy {
  int mode;
  uint32_t keep, total;
};

template <bool WGT, bool ASSIGN, bool HOTBIT, int NW, bool HINT = true, bool LO0 = false>
__global__ void __launch_bounds__(NW * 32, 1)
    k_pull_hot(const uint32_t *__restrict__ col, const double *__restrict__ w,
               const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ id_map_b,
               const uint32_t *__restrict__ tile_row, int64_t es, int64_t ee, int64_t t0,
               int64_t ntiles, uint32_t lo, int hot, uint32_t Lb, const double *__restrict__ hot_src,
               const double *__restrict__ vals, double *__restrict__ out, RangePolicy rp) {
  constexpr int V = kTileV;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // per-warp cache of the destination ids of the tile's first 32 rows
  uint32_t *s_ids = reinterpret_cast<uint32_t *>(smem) + wid * 32;
  double *s_hot = reinterpret_cast<double *>(smem + NW * 32 * sizeof(uint32_t));
  const uint32_t s_hot_addr = (uint32_t)__cvta_generic_to_shared(s_hot);
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep =
      rp.mode ? policy_range(vals + lo, rp.keep, rp.total, rp.mode) : policy_evict_last();
  const unsigned FULL = 0xffffffffu;
  const int64_t stride = (int64_t)gridDim.x * NW;

  // stage the hot table: 8 loads in flight per thread (one at a time, the
  // ~15 rounds of a 1024-thread CTA each waited a full L2/DRAM latency)
  for (int i0 = threadIdx.x; i0 < hot; i0 += 8 * blockDim.x) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * blockDim.x;
      x[j] = i < hot ? __ldcg(hot_src + i) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * blockDim.x;
      if (i < hot) s_hot[i] = x[j];
    }
  }
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
    for (int k = 0; k < V; ++k)
      v[k] = gather_one<HOTBIT, HINT, LO0>(vals, c[k], lo, (uint32_t)hot, s_hot_addr, pol_keep);
    if (WGT) {
      double ww[V];
      ld_stream_f64x4(w + abase + lane * V, pol_stream, ww);
      ld_stream_f64x4(w + abase + lane * V + 4, pol_stream, ww + 4);
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = __dmul_rn(ww[k], v[k]);
    }
    // valid tile positions [llo, lhi); row-start bits of the lane's edges
    const int llo = es > abase ? (int)(es - abase) : 0;
    const int lhi = ee - abase < kTileT ? (int)(ee - abase) : kTileT;
    const TileBits tbits = tile_bits(fw, llo, lhi, lane);
    // next tile's id cache (its first row is known by now)
    uint32_t idn = 0;
    if (has_next && r0n + lane < Lb) idn = id_map_b[r0n + lane];
    s_ids[lane] = idl;
    __syncwarp();
    if (ABL(2)) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < V; ++k) acc += v[k];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(FULL, acc, d);
      if (lane == 0 && !ABL(0)) atomicAdd(out + s_ids[0], acc);
    } else
    tile_reduce<double>(
        v, tbits, r0, lane, 0.0, [](double x, double y) { return __dadd_rn(x, y); },
        [&](uint32_t row, double x, uint32_t r_last) {
          const uint32_t rr = row - r0;
          if (ABL(0)) {
            if (x == 123.456) out[0] = x;  // keeps the reduction alive
            return;
          }
          const uint32_t vid = rr < 32 ? s_ids[rr] : id_map_b[row];
          if ((row == r0 && !tbits.first_start) || (row == r_last && tbits.last_cont))
            atomicAdd(out + vid, x);
          else if (ASSIGN) out[vid] = x;
          else out[vid] = __dadd_rn(out[vid], x);
        });
    __syncwarp();
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

__global__ void k_count_ids(int64_t m, const uint32_t *__restrict__ ids, uint32_t *__restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + ids[e], 1u);
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

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Shared-memory carve-out (KB; an sm_100 configuration) and the hot slots
// that fill it; the rest of the 256 KB array is L1 (see the header).
static int carveout_kb() {
  const char *env = getenv("GCB_CARVE_KB");
  return env ? atoi(env) : 124;  // 124 vs 132 KB: 0.789 vs 0.791 ms gather at rmat:24
}
int64_t hot_capacity(gcb_ctx *ctx) {
  int optin = 0;
  GCB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  int64_t budget = (int64_t)carveout_kb() * 1024;
  if (budget > optin + 1024) budget = optin + 1024;
  // 1 KB per CTA is reserved by the system; the id caches take kGWarps * 128 B
  int64_t K = (budget - 1024 - (int64_t)kGWarps * 128) / 8;
  const char *env = getenv("GCB_HOT_K");
  if (env && atoll(env) < K) K = atoll(env);
  return K < 0 ? 0 : K;
}

// Row-start bitmap of the arena (tiles.cuh).  Built once.
void ensure_row_bits(gcb_ctx *ctx, gcb_blocked *bg) {
  ensure_derived(ctx, bg);
  if (bg->rstart.p) return;
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
}

// Hot set of every block from the out-degrees in bg->deg as the stream
// reaches this point: the top-K sources of block b's range get slots
// [b*K, b*K + K) and slot_of[source] = slot (slot_of is all ~0 on entry).
struct HotScratch {
  DArray<uint32_t> slot_of, k1, k2, v1, v2;
  HotScratch(int64_t n, int64_t width) : slot_of(n), k1(width), k2(width), v1(width), v2(width) {}
};
static void select_hot(gcb_ctx *ctx, gcb_blocked *bg, int64_t K, HotScratch &hs) {
  GCB_CUDA(cudaMemsetAsync(hs.slot_of.p, 0xff, bg->n * sizeof(uint32_t), ctx->stream));
  for (int64_t b = 0; b < bg->B; ++b) {
    const int64_t lo = b * bg->width, hi = (lo + bg->width < bg->n) ? lo + bg->width : bg->n;
    const int64_t cnt = hi - lo;
    GCB_CUDA(cudaMemcpyAsync(hs.k1.p, bg->deg.p + lo, cnt * sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    k_iota_range<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(lo, cnt, hs.v1.p);
    after_launch(ctx, "k_iota_range");
    uint32_t *rk = nullptr, *rv = nullptr;
    cub_sort_pairs_desc_u32_u32(ctx, hs.k1.p, hs.k2.p, hs.v1.p, hs.v2.p, cnt, &rk, &rv);
    k_pick_hot<<<grid_for(K, 256, 4096), 256, 0, ctx->stream>>>(K, cnt, rk, rv,
                                                                bg->hot_ids.p + b * K, hs.slot_of.p);
    after_launch(ctx, "k_pick_hot");
  }
}

static void recode_range(gcb_ctx *ctx, gcb_blocked *bg, const uint32_t *slot_of, int64_t off,
                         int64_t cnt) {
  if (cnt <= 0) return;
  k_recode<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, bg->col.p + off, slot_of,
                                                               bg->xcol.p + off);
  after_launch(ctx, "k_recode");
}

static int64_t pull_hot_slots(gcb_ctx *ctx, const gcb_blocked *bg) {
  int64_t K = hot_capacity(ctx);
  if (K > bg->width) K = bg->width;
  if (bg->m == 0) K = 0;  // nothing to gather: no table (and no recode)
  return K;
}

static void alloc_hot_tables(gcb_ctx *ctx, gcb_blocked *bg, int64_t K) {
  GCB_REQUIRE(bg->n < (int64_t(1) << 31), "hot recode needs vertex ids below 2^31");
  bg->hot_ids.alloc(bg->B * K);
  bg->hotval.alloc(bg->B * K);
  bg->xcol.alloc(bg->m + kColPad);
  GCB_CUDA(cudaMemsetAsync(bg->xcol.p + bg->m, 0, kColPad * sizeof(uint32_t), ctx->stream));
}

// Row-start bitmap + (non-degree-ordered graphs) hot recode.  Built once.
void ensure_exec(gcb_ctx *ctx, gcb_blocked *bg) {
  ensure_derived(ctx, bg);
  if (bg->xready) return;
  ensure_row_bits(ctx, bg);
  const int64_t K = pull_hot_slots(ctx, bg);
  bg->hot_k = K;
  if (!bg->is_relabeled && K > 0) {
    alloc_hot_tables(ctx, bg, K);
    HotScratch hs(bg->n, bg->width);
    select_hot(ctx, bg, K, hs);
    recode_range(ctx, bg, hs.slot_of.p, 0, bg->m);
  }
  sync(ctx);
  bg->xready = true;
}

// The col arena of a pull TOCAB blocking from pinned host memory, with the
// whole execution layout built under the transfer (gcb_blocked_upload).
// The copy is ~20 ms at rmat:24 (1.07 GB over PCIe), the layout build ~3 ms
// after it (tile tables, row-start bitmap, per-block hot-set sort, recode),
// and the out-degree count needs every edge.  So:
//   * col goes over in chunks on the copy stream, each block's chunks in an
//     order that sends a strided sample (every 4th chunk of every block) first;
//   * the tile tables and the row-start bitmap (they need lro only) run while
//     the first chunks are in flight;
//   * each chunk's out-degrees are counted as it lands; once the sample has
//     landed the hot set of every block is picked from the sampled degrees,
//     and from then on each chunk is recoded as it lands.
// The hot set only decides which loads are served from shared memory: the
// ranks are the same for any hot set (the gather's add order does not depend
// on it).  With fewer than 8 chunks there is no sample: the hot set is picked
// from the exact degrees after the last chunk, as ensure_exec does.
void upload_col_overlapped(gcb_ctx *ctx, gcb_blocked *bg, const uint32_t *col_host) {
  const int64_t n = bg->n, m = bg->m;
  if (!ctx->copy_stream)
    GCB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  int64_t chunk = int64_t(16) << 20;  // 64 MB of col per copy
  if (const char *e = getenv("GCB_UPLOAD_CHUNK")) chunk = atoll(e) > 0 ? atoll(e) : chunk;
  // chunk list: block by block; the sample (every 4th chunk of each block,
  // its first included) goes first
  struct Piece { int64_t off, cnt; };
  std::vector<Piece> sample, rest;
  int64_t total = 0;
  for (int64_t b = 0; b < bg->B; ++b) {
    const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
    for (int64_t off = es, j = 0; off < ee; off += chunk, ++j) {
      const Piece pc{off, ee - off < chunk ? ee - off : chunk};
      (j % 4 == 0 ? sample : rest).push_back(pc);
      ++total;
    }
  }
  if (total < 8) {  // small upload: exact degrees, no sample
    for (const Piece &pc : sample) rest.push_back(pc);
    sample.clear();
  }
  std::vector<Piece> order(sample);
  order.insert(order.end(), rest.begin(), rest.end());

  // every allocation before the first copy is queued (an allocation waits for
  // the legacy stream; frees below are stream-ordered)
  bg->deg.alloc(n);
  GCB_CUDA(cudaMemsetAsync(bg->deg.p, 0, (n ? n : 1) * sizeof(uint32_t), ctx->stream));
  const int64_t K = pull_hot_slots(ctx, bg);
  const bool recode = K > 0;
  std::unique_ptr<HotScratch> hs;
  if (recode) {
    alloc_hot_tables(ctx, bg, K);
    hs.reset(new HotScratch(n, bg->width));
  }
  bg->deg_ready = true;  // counted below, in stream order
  {
    cudaEvent_t ready;
    GCB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    GCB_CUDA(cudaEventRecord(ready, ctx->stream));
    GCB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
    cudaEventDestroy(ready);
  }
  std::vector<cudaEvent_t> landed(order.size());
  for (size_t i = 0; i < order.size(); ++i) {
    GCB_CUDA(cudaMemcpyAsync(bg->col.p + order[i].off, col_host + order[i].off,
                             order[i].cnt * sizeof(uint32_t), cudaMemcpyHostToDevice,
                             ctx->copy_stream));
    GCB_CUDA(cudaEventCreateWithFlags(&landed[i], cudaEventDisableTiming));
    GCB_CUDA(cudaEventRecord(landed[i], ctx->copy_stream));
  }
  StreamOrderedFrees frees(ctx->stream);
  ensure_derived(ctx, bg);   // tile tables: lro only (its syncs wait for this stream alone)
  ensure_row_bits(ctx, bg);
  auto count = [&](size_t i) {
    GCB_CUDA(cudaStreamWaitEvent(ctx->stream, landed[i], 0));
    cudaEventDestroy(landed[i]);  // released once the wait is satisfied
    k_deg_count(ctx, order[i].cnt, bg->col.p + order[i].off, bg->deg.p);
  };
  for (size_t i = 0; i < sample.size(); ++i) count(i);
  if (recode && !sample.empty()) {
    select_hot(ctx, bg, K, *hs);
    for (size_t i = 0; i < sample.size(); ++i) recode_range(ctx, bg, hs->slot_of.p, order[i].off, order[i].cnt);
  }
  for (size_t i = sample.size(); i < order.size(); ++i) {
    count(i);
    if (recode && !sample.empty()) recode_range(ctx, bg, hs->slot_of.p, order[i].off, order[i].cnt);
  }
  if (recode && sample.empty()) {
    select_hot(ctx, bg, K, *hs);
    recode_range(ctx, bg, hs->slot_of.p, 0, m);
  }
  bg->hot_k = K;
  hs.reset();
  bg->xready = true;
}

// Push blockings (pr.cu k_push_hot): the per-block top destinations by
// in-degree (= bincount of the arena's col) get a shared-memory accumulator
// slot; the arena is recoded like the pull hot-bit layout.  Atomics on a hub
// destination otherwise serialise on one L2 slice (ncu: lts tag requests 84%
// max vs 45% mean across slices).
void ensure_push_exec(gcb_ctx *ctx, gcb_blocked *bg, int64_t K) {
  ensure_derived(ctx, bg);
  if (bg->xready) return;
  const int64_t B = bg->B, n = bg->n;
  ensure_row_bits(ctx, bg);
  if (K > bg->width) K = bg->width;
  if (bg->m == 0) K = 0;
  bg->hot_k = K;
  if (K > 0) {
    GCB_REQUIRE(n < (int64_t(1) << 31), "hot recode needs vertex ids below 2^31");
    DArray<uint32_t> indeg(n);
    GCB_CUDA(cudaMemsetAsync(indeg.p, 0, n * sizeof(uint32_t), ctx->stream));
    k_count_ids<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(bg->m, bg->col.p, indeg.p);
    after_launch(ctx, "k_count_ids");
    bg->hot_ids.alloc(B * K);
    DArray<uint32_t> slot_of(n), k1(bg->width), k2(bg->width), v1(bg->width), v2(bg->width);
    GCB_CUDA(cudaMemsetAsync(slot_of.p, 0xff, n * sizeof(uint32_t), ctx->stream));
    for (int64_t b = 0; b < B; ++b) {
      const int64_t lo = b * bg->width, hi = (lo + bg->width < n) ? lo + bg->width : n;
      const int64_t cnt = hi - lo;
      GCB_CUDA(cudaMemcpyAsync(k1.p, indeg.p + lo, cnt * sizeof(uint32_t),
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
  }
  sync(ctx);
  bg->xready = true;
}

template <bool WGT, bool ASSIGN, bool HOTBIT>
static void launch_block(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, const double *vals,
                         double *out) {
  const int64_t rs = bg->h_row_starts[b], Lb = bg->h_row_starts[b + 1] - rs;
  const int64_t es = bg->h_edge_starts[b], ee = bg->h_edge_starts[b + 1];
  const int64_t tb = bg->h_tile_base[b], nt = bg->h_tile_base[b + 1] - tb;
  const int64_t lo = b * bg->width, hi = (lo + bg->width < bg->n) ? lo + bg->width : bg->n;
  const int hot = HOTBIT ? (int)bg->hot_k : (int)(bg->hot_k < hi - lo ? bg->hot_k : hi - lo);
  const size_t smem = (size_t)hot * 8 + kGWarps * 32 * sizeof(uint32_t);
  const int pct = (int)(100.0 * carveout_kb() / 228.0 + 0.99);
  ensure_smem_attrs(ctx, (const void *)k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps>, smem,
                    pct > 100 ? 100 : pct);
#ifdef GCB_ABLATE
  {
    const char *e = getenv("GCB_ABL");
    const int abl = e ? atoi(e) : 0;
    GCB_CUDA(cudaMemcpyToSymbolAsync(c_abl, &abl, sizeof(int), 0, cudaMemcpyHostToDevice,
                                     ctx->stream));
  }
#endif
  int64_t grid = ceil_div(nt, kGWarps);
  if (grid > ctx->num_sms) grid = ctx->num_sms;
  const double *hot_src = HOTBIT ? bg->hotval.p + b * bg->hot_k : vals + lo;
  // L2 residency of the cold gathers (north star (1)): on the degree-ordered
  // copy the block's value slice is sorted by out-degree, so its head holds
  // the most-read cold values.  By default a range policy -- the
  // per-instruction form of an access-policy window (createpolicy.range) --
  // marks the first kL2KeepMB of the slice evict_last and leaves the tail at
  // normal priority.  With a persisting set-aside (GCB_L2_PERSIST=<MB>, ctx.cu)
  // the launch carries a real access-policy window over that head instead
  // (below): as fast at 48 MB (7.186 vs 7.19 ms per step at rmat:24) but 1.6x
  // the DRAM traffic (profiles/r2_l2_window_attr.txt).  For the range policy,
  // marking the tail evict_first ran slower, as did a 16 MB head
  // (profiles/r2_l2_window.txt).  GCB_L2_RANGE="<MB>:<mode>" overrides it (mode
  // 1: tail evict_first, 2: tail unchanged, 0: whole slice evict_last); the
  // hot-bit layout has no sorted slice and keeps evict_last.
  RangePolicy rp{0, 0, 0};
  {
    double mb = kL2KeepMB;
    int mode = HOTBIT ? 0 : 2;
    if (const char *e = getenv("GCB_L2_RANGE")) {
      if (sscanf(e, "%lf:%d", &mb, &mode) != 2 || mode < 0 || mode > 2) mode = 0;
    }
    const uint64_t total = (uint64_t)(hi - lo) * 8u;
    uint64_t keep = (uint64_t)(mb * 1048576.0);
    if (keep > total) keep = total;
    if (mode && keep < total && total < (uint64_t(1) << 32))
      rp = RangePolicy{mode, (uint32_t)keep, (uint32_t)total};
  }
  // With a persisting set-aside in force (GCB_L2_PERSIST=<MB>) the head of a
  // degree-ordered value slice -- its most-read cold values -- is pinned by a
  // launch access-policy window instead of the per-load range policy
  // (measured against it in profiles/r2_l2_window_attr.txt).
  const bool window = !HOTBIT && ctx->persist_set > 0 && ctx->window_max > 0;
  if (window) {
    uint64_t wbytes = (uint64_t)(hi - lo) * 8u;
    if (wbytes > (uint64_t)ctx->persist_set) wbytes = (uint64_t)ctx->persist_set;
    if (wbytes > (uint64_t)ctx->window_max) wbytes = (uint64_t)ctx->window_max;
    ensure_smem_attrs(ctx, (const void *)k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps, false>, smem,
                      pct > 100 ? 100 : pct);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(grid < 1 ? 1 : grid));
    cfg.blockDim = dim3(kGWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<double *>(vals + lo);
    attr[0].val.accessPolicyWindow.num_bytes = (size_t)wbytes;
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    // accesses past the window's hit fraction stay normal (streaming evicted
    // the slice's tail early: ncu DRAM per launch 1.79 GB against 1.08 GB)
    attr[0].val.accessPolicyWindow.missProp =
        getenv("GCB_L2_WINDOW_STREAM") ? cudaAccessPropertyStreaming : cudaAccessPropertyNormal;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GCB_CUDA(cudaLaunchKernelEx(&cfg, k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps, false>,
                                (const uint32_t *)(HOTBIT ? bg->xcol.p : bg->col.p),
                                (const double *)(WGT ? bg->w.p : nullptr),
                                (const uint32_t *)bg->rstart.p, (const uint32_t *)(bg->id_map.p + rs),
                                (const uint32_t *)(bg->tile_row.p + tb), es, ee, bg->h_tile_t0[b], nt,
                                (uint32_t)lo, hot, (uint32_t)Lb, hot_src, vals, out, rp));
  } else if (!HOTBIT && lo == 0 && !getenv("GCB_NO_LO0")) {
    ensure_smem_attrs(ctx, (const void *)k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps, true, true>,
                      smem, pct > 100 ? 100 : pct);
    k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps, true, true>
        <<<(unsigned)(grid < 1 ? 1 : grid), kGWarps * 32, smem, ctx->stream>>>(
            HOTBIT ? bg->xcol.p : bg->col.p, WGT ? bg->w.p : nullptr, bg->rstart.p,
            bg->id_map.p + rs, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt, (uint32_t)lo,
            hot, (uint32_t)Lb, hot_src, vals, out, rp);
  } else {
    k_pull_hot<WGT, ASSIGN, HOTBIT, kGWarps>
        <<<(unsigned)(grid < 1 ? 1 : grid), kGWarps * 32, smem, ctx->stream>>>(
            HOTBIT ? bg->xcol.p : bg->col.p, WGT ? bg->w.p : nullptr, bg->rstart.p,
            bg->id_map.p + rs, bg->tile_row.p + tb, es, ee, bg->h_tile_t0[b], nt, (uint32_t)lo,
            hot, (uint32_t)Lb, hot_src, vals, out, rp);
  }
  after_launch(ctx, "k_pull_hot");
}

template <bool HOTBIT>
static void launch_block_any(gcb_ctx *ctx, gcb_blocked *bg, int64_t b, bool wgt, bool assign,
                             const double *vals, double *out) {
  if (wgt && assign) launch_block<true, true, HOTBIT>(ctx, bg, b, vals, out);
  else if (wgt) launch_block<true, false, HOTBIT>(ctx, bg, b, vals, out);
  else if (assign) launch_block<false, true, HOTBIT>(ctx, bg, b, vals, out);
  else launch_block<false, false, HOTBIT>(ctx, bg, b, vals, out);
}

// out[v] += sum over the rows of v in every block (block order); the caller
// clears out first (the first non-empty block stores instead of adding).
void gather_accum(gcb_ctx *ctx, gcb_blocked *bg, const double *vals, bool use_weights,
                  uint32_t flags, double *out) {
  (void)flags;
  ensure_exec(ctx, bg);
  const bool wgt = use_weights && bg->weighted;
  const bool hotbit = !bg->is_relabeled && bg->hot_k > 0;
  if (hotbit) {
    ProfScope ps(ctx, 3);
    const int64_t cnt = bg->B * bg->hot_k;
    k_fill_hot<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(cnt, bg->hot_ids.p, vals,
                                                                   bg->hotval.p);
    after_launch(ctx, "k_fill_hot");
  }
  bool first = true;
  for (int64_t b = 0; b < bg->B; ++b) {
    if (bg->h_row_starts[b + 1] == bg->h_row_starts[b]) continue;
    ProfScope ps(ctx, 0);
    if (hotbit) launch_block_any<true>(ctx, bg, b, wgt, first, vals, out);
    else launch_block_any<false>(ctx, bg, b, wgt, first, vals, out);
    first = false;
  }
}

// Census of one block's arena for the request model: edges whose source is
// served from the shared-memory hot table (HOTBIT: recoded entries; else the
// block's degree-ordered prefix [lo, lo + hot)).
__global__ void k_count_hot(int64_t es, int64_t ee, const uint32_t *__restrict__ col, bool hotbit,
                            uint32_t lo, uint32_t hot, unsigned long long *__restrict__ out) {
  unsigned long long c = 0;
  for (int64_t e = es + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ee;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = col[e];
    c += hotbit ? (x >> 31) : ((x - lo) < hot ? 1u : 0u);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_blocked_gather_census(gcb_ctx *ctx, gcb_blocked *bg, int64_t *out4) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && out4, "NULL argument");
  GCB_REQUIRE(bg->direction == 0 && !bg->cb, "the census is of a pull TOCAB blocking");
  DeviceGuard dg(ctx->device);
  // the layout the fast pull runs: the degree-ordered copy once promoted
  gcb_blocked *x = bg->rl ? bg->rl : bg;
  ensure_exec(ctx, x);
  const bool hotbit = !x->is_relabeled && x->hot_k > 0;
  DArray<unsigned long long> cnt(1);
  GCB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
  for (int64_t b = 0; b < x->B && x->hot_k > 0; ++b) {
    const int64_t es = x->h_edge_starts[b], ee = x->h_edge_starts[b + 1];
    if (ee == es) continue;
    const int64_t lo = b * x->width, hi = (lo + x->width < x->n) ? lo + x->width : x->n;
    const int64_t hot = x->hot_k < hi - lo ? x->hot_k : hi - lo;
    k_count_hot<<<grid_for(ee - es, 256, 65536), 256, 0, ctx->stream>>>(
        es, ee, hotbit ? x->xcol.p : x->col.p, hotbit, (uint32_t)lo, (uint32_t)hot, cnt.p);
    after_launch(ctx, "k_count_hot");
  }
  unsigned long long h = 0;
  d2h(ctx, &h, cnt.p, 1);
  sync(ctx);
  out4[0] = (int64_t)h;                          // hot-table edges (shared memory)
  out4[1] = x->m - (int64_t)h;                   // cold edges: one L2 request each
  out4[2] = x->hybrid ? x->hybrid->m : 0;        // hub-destination edges (push pass)
  out4[3] = x->is_relabeled ? 1 : 0;             // layout: 1 degree-ordered, 0 hot-bit
  GCB_API_END
}

}  // extern "C"

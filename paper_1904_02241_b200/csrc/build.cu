// build.cu -- device CSR construction: upload/download, from_edges (stable
// radix sort), transpose, symmetrize, and the bit-exact PCG64 R-MAT generator.
// Reference: graph.py:45-151 (CsrGraph, from_edges, transpose, symmetrize) and
// graph.py:371-386 (_generate_rmat).
#include <cstring>

#include "gcb_internal.cuh"

namespace gcb {

int bits_for(int64_t n) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < n) ++b;
  return b;
}

// ---------------------------------------------------------------------------
// 128-bit LCG arithmetic for PCG64 (numpy's default bit generator)
// ---------------------------------------------------------------------------
struct U128 {
  uint64_t lo, hi;
};

__host__ __device__ inline U128 u128_mul(U128 a, U128 b) {
  U128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  unsigned __int128 x = ((unsigned __int128)a.hi << 64) | a.lo;
  unsigned __int128 y = ((unsigned __int128)b.hi << 64) | b.lo;
  unsigned __int128 z = x * y;
  r.lo = (uint64_t)z;
  r.hi = (uint64_t)(z >> 64);
#endif
  return r;
}

__host__ __device__ inline U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

struct Affine {  // x -> mult * x + plus  (mod 2^128)
  U128 mult, plus;
};

__host__ __device__ inline U128 affine_apply(const Affine &f, U128 x) {
  return u128_add(u128_mul(f.mult, x), f.plus);
}

// g after f
__host__ __device__ inline Affine affine_then(const Affine &f, const Affine &g) {
  Affine r;
  r.mult = u128_mul(g.mult, f.mult);
  r.plus = u128_add(u128_mul(g.mult, f.plus), g.plus);
  return r;
}

__host__ __device__ inline U128 pcg_mult() { return U128{0x4385DF649FCCF645ULL, 0x2360ED051FC65DA4ULL}; }

__device__ inline double pcg_next_double(U128 &s, const U128 &inc) {
  s = u128_add(u128_mul(s, pcg_mult()), inc);
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
  return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

// jump tables: tab[k] = 2^k LCG steps
static void make_jump_table(U128 inc, Affine *tab) {
  Affine cur = {pcg_mult(), inc};
  for (int k = 0; k < 64; ++k) {
    tab[k] = cur;
    cur = affine_then(cur, cur);
  }
}

static Affine jump_by(const Affine *tab, uint64_t delta) {
  Affine acc = {{1, 0}, {0, 0}};
  for (int k = 0; k < 64; ++k)
    if (delta >> k & 1) acc = affine_then(acc, tab[k]);
  return acc;
}

constexpr int kRmatEPT = 16;  // edges per thread

// Each thread owns kRmatEPT consecutive edges; level l of edge i consumes draw
// l*m + i (graph.py:380-385: one rng.random(m) per level, MSB first).
__global__ void k_rmat_keys(int scale, int64_t m, U128 s0, U128 inc, const Affine *__restrict__ tab,
                            Affine jump_m, double t_a, double t_ab, double t_abc, int transposed,
                            uint64_t *__restrict__ keys) {
  int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRmatEPT;
  if (i0 >= m) return;
  int cnt = (m - i0 < kRmatEPT) ? (int)(m - i0) : kRmatEPT;
  // state after i0 steps: compose 2^k jumps
  Affine acc = {{1, 0}, {0, 0}};
  for (int k = 0; k < 63; ++k)
    if ((uint64_t)i0 >> k & 1) acc = affine_then(acc, tab[k]);
  U128 start = affine_apply(acc, s0);
  uint32_t src[kRmatEPT], dst[kRmatEPT];
#pragma unroll
  for (int j = 0; j < kRmatEPT; ++j) src[j] = dst[j] = 0;
  for (int l = 0; l < scale; ++l) {
    U128 s = start;
#pragma unroll
    for (int j = 0; j < kRmatEPT; ++j) {
      if (j < cnt) {
        double r = pcg_next_double(s, inc);
        uint32_t sb = r >= t_ab;
        uint32_t db = ((r >= t_a) && (r < t_ab)) || (r >= t_abc);
        src[j] = (src[j] << 1) | sb;
        dst[j] = (dst[j] << 1) | db;
      }
    }
    start = affine_apply(jump_m, start);
  }
#pragma unroll
  for (int j = 0; j < kRmatEPT; ++j)
    if (j < cnt)
      keys[i0 + j] = transposed ? ((uint64_t)dst[j] << scale) | src[j]
                                : ((uint64_t)src[j] << scale) | dst[j];
}

__global__ void k_keys_from_edges(int64_t m, int bits, const uint32_t *__restrict__ src,
                                  const uint32_t *__restrict__ dst, uint64_t *__restrict__ keys,
                                  uint32_t *__restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = ((uint64_t)src[i] << bits) | dst[i];
    if (idx) idx[i] = (uint32_t)i;
  }
}

__global__ void k_row_offsets_from_keys(int64_t n, int64_t m, int bits,
                                        const uint64_t *__restrict__ keys,
                                        int64_t *__restrict__ ro) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    // lower_bound(keys, v << bits)
    uint64_t target = (uint64_t)v << bits;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    ro[v] = (v == n) ? m : lo;
  }
}

__global__ void k_col_from_keys(int64_t m, uint64_t mask, const uint64_t *__restrict__ keys,
                                uint32_t *__restrict__ col, const uint32_t *__restrict__ perm,
                                const double *__restrict__ w_in, double *__restrict__ w_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    col[i] = (uint32_t)(keys[i] & mask);
    if (w_out) w_out[i] = w_in[perm[i]];
  }
}

// warp per row: edge_src[e] = row(e)
__global__ void k_expand_rows(int64_t n, const int64_t *__restrict__ ro, uint32_t *__restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nw) {
    int64_t s = ro[v], e = ro[v + 1];
    for (int64_t i = s + lane; i < e; i += 32) out[i] = (uint32_t)v;
  }
}

void csr_from_sorted_keys(gcb_ctx *ctx, int64_t n, int64_t m, const uint64_t *keys, int bits,
                          gcb_csr *out) {
  out->ro.alloc(n + 1);
  out->col.alloc(m + kColPad);
  GCB_CUDA(cudaMemsetAsync(out->col.p, 0, (m + kColPad) * sizeof(uint32_t), ctx->stream));
  k_row_offsets_from_keys<<<grid_for(n + 1, 256, 65536), 256, 0, ctx->stream>>>(n, m, bits, keys,
                                                                                out->ro.p);
  after_launch(ctx, "k_row_offsets_from_keys");
  if (m) {
    k_col_from_keys<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
        m, (bits >= 64) ? ~0ULL : ((1ULL << bits) - 1), keys, out->col.p, nullptr, nullptr,
        nullptr);
    after_launch(ctx, "k_col_from_keys");
  }
}

// from_edges graph.py:110-130 on device arrays (ids already validated < n).
gcb_csr *csr_from_device_edges(gcb_ctx *ctx, int64_t n, int64_t m, const uint32_t *src,
                               const uint32_t *dst, const double *w_or_null) {
  GCB_REQUIRE(m < (int64_t(1) << 32), "edge count %lld exceeds the 32-bit edge id space",
              (long long)m);
  GCB_REQUIRE(n <= (int64_t(1) << 32), "vertex count exceeds the 32-bit id space");
  int bits = bits_for(n);
  auto g = new gcb_csr();
  try {
    g->device = ctx->device;
    g->n = n;
    g->m = m;
    DArray<uint64_t> k1(m), k2(m);
    DArray<uint32_t> v1, v2;
    bool weighted = w_or_null != nullptr;
    if (weighted) {
      v1.alloc(m);
      v2.alloc(m);
    }
    if (m) {
      k_keys_from_edges<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
          m, bits, src, dst, k1.p, weighted ? v1.p : nullptr);
      after_launch(ctx, "k_keys_from_edges");
    }
    uint64_t *keys = k1.p;
    uint32_t *perm = nullptr;
    int end_bit = bits * 2;
    if (weighted) cub_sort_pairs_u64_u32(ctx, k1.p, k2.p, v1.p, v2.p, m, end_bit, &keys, &perm);
    else cub_sort_keys_u64(ctx, k1.p, k2.p, m, end_bit, &keys);
    csr_from_sorted_keys(ctx, n, m, keys, bits, g);
    if (weighted) {
      g->w.alloc(m + kColPad);
      g->weighted = true;
      if (m) {
        k_col_from_keys<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
            m, (1ULL << bits) - 1, keys, g->col.p, perm, w_or_null, g->w.p);
        after_launch(ctx, "k_col_from_keys(w)");
      }
    }
    sync(ctx);  // temporaries die at scope exit
  } catch (...) {
    delete g;
    throw;
  }
  return g;
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_csr_upload(gcb_ctx *ctx, int64_t n, int64_t m, const int64_t *row_offsets_host,
                   const uint32_t *col_host, const double *weights_host_or_null, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && out && row_offsets_host && (col_host || m == 0), "NULL argument");
  GCB_REQUIRE(n >= 0 && m >= 0, "negative size");
  DeviceGuard dg(ctx->device);
  auto g = new gcb_csr();
  try {
    g->device = ctx->device;
    g->n = n;
    g->m = m;
    g->ro.alloc(n + 1);
    g->col.alloc(m + kColPad);
    GCB_CUDA(cudaMemsetAsync(g->col.p, 0, (m + kColPad) * sizeof(uint32_t), ctx->stream));
    h2d(ctx, g->ro.p, row_offsets_host, n + 1);
    h2d(ctx, g->col.p, col_host, m);
    if (weights_host_or_null) {
      g->weighted = true;
      g->w.alloc(m + kColPad);
      h2d(ctx, g->w.p, weights_host_or_null, m);
    }
    sync(ctx);
  } catch (...) {
    delete g;
    throw;
  }
  *out = g;
  GCB_API_END
}

int gcb_csr_from_edges(gcb_ctx *ctx, int64_t n, int64_t m, const int64_t *src_host,
                       const int64_t *dst_host, const double *weights_host_or_null,
                       gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && out && ((src_host && dst_host) || m == 0), "NULL argument");
  GCB_REQUIRE(n >= 0 && m >= 0, "negative size");
  DeviceGuard dg(ctx->device);
  std::vector<uint32_t> s32(m), d32(m);
  for (int64_t i = 0; i < m; ++i) {
    GCB_REQUIRE(src_host[i] >= 0 && dst_host[i] >= 0, "negative vertex id");
    GCB_REQUIRE(src_host[i] < n && dst_host[i] < n, "vertex id out of range");
    s32[i] = (uint32_t)src_host[i];
    d32[i] = (uint32_t)dst_host[i];
  }
  DArray<uint32_t> ds(m), dd(m);
  DArray<double> dw;
  h2d(ctx, ds.p, s32.data(), m);
  h2d(ctx, dd.p, d32.data(), m);
  if (weights_host_or_null) {
    dw.alloc(m);
    h2d(ctx, dw.p, weights_host_or_null, m);
  }
  *out = csr_from_device_edges(ctx, n, m, ds.p, dd.p, weights_host_or_null ? dw.p : nullptr);
  GCB_API_END
}

int gcb_csr_generate_rmat(gcb_ctx *ctx, int scale, int64_t edge_factor, uint64_t state_hi,
                          uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double t_a,
                          double t_ab, double t_abc, int transposed, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && out, "NULL argument");
  GCB_REQUIRE(scale >= 1 && scale <= 31, "rmat scale must be in [1, 31]");
  GCB_REQUIRE(edge_factor >= 1, "edge_factor must be >= 1");
  DeviceGuard dg(ctx->device);
  int64_t n = int64_t(1) << scale;
  int64_t m = edge_factor * n;
  GCB_REQUIRE(m < (int64_t(1) << 32), "edge count exceeds the 32-bit edge id space");
  U128 s0 = {state_lo, state_hi}, inc = {inc_lo, inc_hi};
  Affine tab[64];
  make_jump_table(inc, tab);
  Affine jm = jump_by(tab, (uint64_t)m);
  DArray<Affine> dtab(64);
  h2d(ctx, dtab.p, tab, 64);
  DArray<uint64_t> k1(m), k2(m);
  int64_t threads = ceil_div(m, kRmatEPT);
  k_rmat_keys<<<(unsigned)ceil_div(threads, 256), 256, 0, ctx->stream>>>(
      scale, m, s0, inc, dtab.p, jm, t_a, t_ab, t_abc, transposed, k1.p);
  after_launch(ctx, "k_rmat_keys");
  uint64_t *keys = nullptr;
  cub_sort_keys_u64(ctx, k1.p, k2.p, m, 2 * scale, &keys);
  auto g = new gcb_csr();
  try {
    g->device = ctx->device;
    g->n = n;
    g->m = m;
    csr_from_sorted_keys(ctx, n, m, keys, scale, g);
    sync(ctx);
  } catch (...) {
    delete g;
    throw;
  }
  *out = g;
  GCB_API_END
}

int gcb_csr_transpose(gcb_ctx *ctx, const gcb_csr *g, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out, "NULL argument");
  DeviceGuard dg(ctx->device);
  DArray<uint32_t> src(g->m);
  if (g->m) {
    k_expand_rows<<<grid_for(g->n * 32, 256, 16384), 256, 0, ctx->stream>>>(g->n, g->ro.p, src.p);
    after_launch(ctx, "k_expand_rows");
  }
  // transpose == from_edges(col, edge_sources) (graph.py:133-138)
  *out = csr_from_device_edges(ctx, g->n, g->m, g->col.p, src.p, g->weighted ? g->w.p : nullptr);
  GCB_API_END
}

__global__ void k_symm_edges(int64_t m, const uint32_t *__restrict__ src,
                             const uint32_t *__restrict__ dst, const uint32_t *__restrict__ pos,
                             uint32_t *__restrict__ s2, uint32_t *__restrict__ d2,
                             const double *__restrict__ w, double *__restrict__ w2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = src[i], d = dst[i];
    s2[i] = s;
    d2[i] = d;
    if (w2) w2[i] = w[i];
    if (s != d) {
      int64_t j = m + pos[i];
      s2[j] = d;
      d2[j] = s;
      if (w2) w2[j] = w[i];
    }
  }
}

__global__ void k_nonloop_flags(int64_t m, const uint32_t *__restrict__ src,
                                const uint32_t *__restrict__ dst, uint32_t *__restrict__ f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    f[i] = src[i] != dst[i];
}

int gcb_csr_symmetrize(gcb_ctx *ctx, const gcb_csr *g, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out, "NULL argument");
  DeviceGuard dg(ctx->device);
  int64_t m = g->m;
  DArray<uint32_t> src(m), flags(m + 1), pos(m + 1);
  if (m) {
    k_expand_rows<<<grid_for(g->n * 32, 256, 16384), 256, 0, ctx->stream>>>(g->n, g->ro.p, src.p);
    after_launch(ctx, "k_expand_rows");
    k_nonloop_flags<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(m, src.p, g->col.p, flags.p);
    after_launch(ctx, "k_nonloop_flags");
  }
  GCB_CUDA(cudaMemsetAsync(flags.p + m, 0, sizeof(uint32_t), ctx->stream));
  cub_exclusive_sum_u32(ctx, flags.p, pos.p, m + 1);
  uint32_t extra = 0;
  d2h(ctx, &extra, pos.p + m, 1);
  sync(ctx);
  int64_t m2 = m + extra;
  DArray<uint32_t> s2(m2), d2(m2);
  DArray<double> w2;
  if (g->weighted) w2.alloc(m2);
  if (m) {
    k_symm_edges<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
        m, src.p, g->col.p, pos.p, s2.p, d2.p, g->weighted ? g->w.p : nullptr,
        g->weighted ? w2.p : nullptr);
    after_launch(ctx, "k_symm_edges");
  }
  *out = csr_from_device_edges(ctx, g->n, m2, s2.p, d2.p, g->weighted ? w2.p : nullptr);
  GCB_API_END
}

int gcb_csr_info(const gcb_csr *g, int64_t *n, int64_t *m, int *weighted) {
  GCB_API_BEGIN
  GCB_REQUIRE(g, "NULL graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (weighted) *weighted = g->weighted ? 1 : 0;
  GCB_API_END
}

int gcb_csr_download(gcb_ctx *ctx, const gcb_csr *g, int64_t *row_offsets_host, uint32_t *col_host,
                     double *weights_host_or_null) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g, "NULL argument");
  DeviceGuard dg(ctx->device);
  if (row_offsets_host) d2h(ctx, row_offsets_host, g->ro.p, g->n + 1);
  if (col_host) d2h(ctx, col_host, g->col.p, g->m);
  if (weights_host_or_null && g->weighted) d2h(ctx, weights_host_or_null, g->w.p, g->m);
  sync(ctx);
  GCB_API_END
}

int gcb_csr_set_weights(gcb_ctx *ctx, gcb_csr *g, const double *weights_host) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && weights_host, "NULL argument");
  DeviceGuard dg(ctx->device);
  g->w.alloc(g->m + kColPad);
  h2d(ctx, g->w.p, weights_host, g->m);
  g->weighted = true;
  sync(ctx);
  GCB_API_END
}

int gcb_csr_destroy(gcb_csr *g) {
  GCB_API_BEGIN
  if (!g) return GCB_OK;
  DeviceGuard dg(g->device);
  if (g->compact) gcb_blocked_destroy(g->compact);
  delete g;
  GCB_API_END
}

__global__ void k_slab_offsets(int64_t n, int64_t v0, int64_t v1, const int64_t *__restrict__ ro,
                               int64_t *__restrict__ out) {
  const int64_t lo = ro[v0], hi = ro[v1];
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = ro[v];
    x = x < lo ? lo : (x > hi ? hi : x);
    out[v] = x - lo;
  }
}

__global__ void k_col_counts(int64_t m, const uint32_t *__restrict__ col, uint32_t *__restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[i], 1u);
}

// rows [v0, v1) of g kept, every other row emptied (same n x n shape): the
// slab a destination shard owns
int gcb_csr_row_slab(gcb_ctx *ctx, const gcb_csr *g, int64_t v0, int64_t v1, gcb_csr **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && out, "NULL argument");
  GCB_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= g->n, "bad row range");
  DeviceGuard dg(ctx->device);
  int64_t se[2];
  d2h(ctx, &se[0], g->ro.p + v0, 1);
  d2h(ctx, &se[1], g->ro.p + v1, 1);
  sync(ctx);
  const int64_t m = se[1] - se[0];
  auto s = new gcb_csr();
  try {
    s->device = ctx->device;
    s->n = g->n;
    s->m = m;
    s->ro.alloc(g->n + 1);
    s->col.alloc(m + kColPad);
    GCB_CUDA(cudaMemsetAsync(s->col.p + m, 0, kColPad * sizeof(uint32_t), ctx->stream));
    k_slab_offsets<<<grid_for(g->n + 1, 256, 65536), 256, 0, ctx->stream>>>(g->n, v0, v1, g->ro.p,
                                                                           s->ro.p);
    after_launch(ctx, "k_slab_offsets");
    if (m) GCB_CUDA(cudaMemcpyAsync(s->col.p, g->col.p + se[0], m * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
    if (g->weighted) {
      s->weighted = true;
      s->w.alloc(m + kColPad);
      if (m) GCB_CUDA(cudaMemcpyAsync(s->w.p, g->w.p + se[0], m * sizeof(double),
                                      cudaMemcpyDeviceToDevice, ctx->stream));
    }
    sync(ctx);
  } catch (...) {
    delete s;
    throw;
  }
  *out = s;
  GCB_API_END
}

// counts[v] = occurrences of v among the column ids (for the transpose: the
// forward out-degrees, kernels.py:199-204); counts_dev is a device uint32[n]
int gcb_csr_col_counts(gcb_ctx *ctx, const gcb_csr *g, uint32_t *counts_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && g && counts_dev, "NULL argument");
  DeviceGuard dg(ctx->device);
  GCB_CUDA(cudaMemsetAsync(counts_dev, 0, (g->n ? g->n : 1) * sizeof(uint32_t), ctx->stream));
  if (g->m) {
    k_col_counts<<<grid_for(g->m, 256, 65536), 256, 0, ctx->stream>>>(g->m, g->col.p, counts_dev);
    after_launch(ctx, "k_col_counts");
  }
  GCB_API_END
}

}  // extern "C"

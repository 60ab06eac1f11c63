// exchange.cu -- destination-sharded PageRank with the contribution exchange
// fused into the rank update over peer memory (BASELINE north star:
// "PageRank/SpMV shard by destination-vertex range with the vertex-value
// vector all-gathered over NVLink").
//
// Rank r owns rows [v0, v1) of the transpose.  Instead of an update kernel
// followed by an NCCL collective, k_pr_update_p2p computes each owned
// contribution and stores it straight into the contribution buffer of every
// rank whose slab reads that source (need mask, bit p = rank p reads v), over
// NVLink through CUDA IPC mappings of the peers' buffers.  The stores overlap
// the update's own HBM stream tile by tile; no staging buffer, no separate
// collective launch.  Then k_signal_peers publishes the epoch to every peer
// with a system-scope release, and the next step's k_wait_peers acquires all
// peers' epochs before the gather reads the vector.
//
// Two contribution buffers alternate by epoch: step e gathers buffer (e-1)%2
// and writes buffer e%2.  A rank that runs ahead cannot overwrite values a
// slower peer is still gathering: it writes buffer e%2 only after waiting for
// every peer's epoch e-1, which each peer signals after its gather e-1.
//
// Entries of a buffer this rank never reads stay stale (the gather cannot
// observe them), exactly as with the sparse all-to-all exchange.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "gcb_internal.cuh"
#include "ldst.cuh"
#include "pr_math.cuh"

namespace gcb {

__global__ void k_reduce_sum(const double *__restrict__ in, int64_t count, double *__restrict__ out);

// the update of the owned quads (k_pr_update2's arithmetic, pr_math.cuh) with
// every contribution also stored into the peers that read it
template <bool EXACT>
__global__ void __launch_bounds__(512, 2)
    k_pr_update_p2p(int64_t cnt, int64_t v0, double base, double damping,
                    double *__restrict__ sums, double *__restrict__ ranks,
                    const uint32_t *__restrict__ deg, double *const *__restrict__ out,
                    const uint8_t *__restrict__ need, int P, int self,
                    double *__restrict__ deltas) {
  __shared__ double red[16];
  double dsum = 0.0;
  double *mine = out[self];
  const int64_t n4 = cnt >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double s[4], o[4], nr[4], c[4];
    ld_rw_f64x4(sums + v0 + 4 * i, s);
    ld_rw_f64x4(ranks + v0 + 4 * i, o);
    const uint4 d = __ldcs(reinterpret_cast<const uint4 *>(deg + v0) + i);
    pr_quad<EXACT>(s, o, d, base, damping, nr, c, dsum);
    st_f64x4(ranks + v0 + 4 * i, nr[0], nr[1], nr[2], nr[3]);
    st_f64x4(sums + v0 + 4 * i, 0.0, 0.0, 0.0, 0.0);
    st_f64x4(mine + v0 + 4 * i, c[0], c[1], c[2], c[3]);
    const uint32_t nm = reinterpret_cast<const uint32_t *>(need)[i];  // 4 masks
    if (nm) {
      const uint32_t any = (nm | (nm >> 8) | (nm >> 16) | (nm >> 24)) & 0xffu;
      for (int p = 0; p < P; ++p) {
        if (!((any >> p) & 1u)) continue;
        // the whole 32-byte quad as one full-sector store even when the peer
        // reads only some of its four entries: the others land on entries the
        // peer never reads (measured: per-entry 8-byte stores cost more)
        st_f64x4(out[p] + v0 + 4 * i, c[0], c[1], c[2], c[3]);
      }
    }
  }
  for (int64_t v = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < cnt; v += stride) {
    const double nr = __dadd_rn(base, __dmul_rn(damping, sums[v0 + v]));
    dsum += fabs(nr - ranks[v0 + v]);
    const uint32_t dg = deg[v0 + v];
    const double c = dg ? div_deg<EXACT>(nr, dg) : 0.0;
    ranks[v0 + v] = nr;
    sums[v0 + v] = 0.0;
    mine[v0 + v] = c;
    for (int p = 0; p < P; ++p)
      if ((need[v] >> p) & 1u) out[p][v0 + v] = c;
  }
  // the peer stores must be visible system-wide before k_signal_peers
  // publishes the epoch
  __threadfence_system();
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

// init (VertexValueSet.initial, kernels.py:80-89) of the owned slice, with the
// contributions published to the peers like the update's
__global__ void k_pr_init_p2p(int64_t cnt, int64_t v0, double r0, const uint32_t *__restrict__ deg,
                              double *__restrict__ ranks, double *__restrict__ sums,
                              double *const *__restrict__ out, const uint8_t *__restrict__ need,
                              int P, int self) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < cnt;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t dg = deg[v0 + v];
    const double c = dg ? __ddiv_rn(r0, (double)dg) : 0.0;
    ranks[v0 + v] = r0;
    sums[v0 + v] = 0.0;
    out[self][v0 + v] = c;
    for (int p = 0; p < P; ++p)
      if ((need[v] >> p) & 1u) out[p][v0 + v] = c;
  }
  __threadfence_system();
}

// flags[p][self] = epoch for every peer p (release at system scope)
__global__ void k_signal_peers(uint32_t *const *flags, int P, int self, uint32_t epoch) {
  const int p = threadIdx.x;
  if (p >= P || p == self) return;
  __threadfence_system();
  cuda::atomic_ref<uint32_t, cuda::thread_scope_system> f(flags[p][self]);
  f.store(epoch, cuda::memory_order_release);
}

// wait until every peer q has published epoch >= `epoch` into mine[q].  A
// peer that misses the deadline (GCB_PEER_TIMEOUT_S, default 120 s) sets
// *err and the kernel returns: the context stays usable and the host raises
// at the next step or at gcb_peer_check (a __trap would destroy the context)
__global__ void k_wait_peers(uint32_t *mine, int P, int self, uint32_t epoch,
                             uint64_t timeout_ns, volatile unsigned *err) {
  const int q = threadIdx.x;
  if (q >= P || q == self) return;
  cuda::atomic_ref<uint32_t, cuda::thread_scope_system> f(mine[q]);
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while ((int32_t)(f.load(cuda::memory_order_acquire) - epoch) < 0) {
    if (*err) return;  // an earlier wait already gave up
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      *err = 1u + (unsigned)q;
      __threadfence_system();
      return;
    }
  }
}

static uint64_t peer_timeout_ns() {
  const char *env = getenv("GCB_PEER_TIMEOUT_S");
  const double s = env && env[0] ? atof(env) : 120.0;
  return (uint64_t)((s > 0 ? s : 120.0) * 1e9);
}

// raise (once) what a previous k_wait_peers recorded
static void check_peer_error(gcb_ctx *ctx) {
  if (!ctx->peer_err) {
    GCB_CUDA(cudaHostAlloc((void **)&ctx->peer_err, sizeof(unsigned), cudaHostAllocMapped));
    *ctx->peer_err = 0;
    GCB_CUDA(cudaHostGetDevicePointer((void **)&ctx->peer_err_dev, ctx->peer_err, 0));
  }
  const unsigned e = *(volatile unsigned *)ctx->peer_err;
  if (e) {
    *(volatile unsigned *)ctx->peer_err = 0;
    fail(GCB_ECUDA, "peer exchange: rank %u did not publish its epoch within GCB_PEER_TIMEOUT_S "
                    "(results of the steps since are invalid)", e - 1);
  }
}

// The NCCL fallback exchange (parallel.SparseExchange): pack the values the
// peers read into the all_to_all send buffer, and scatter the received ones
// into the full vector.  32-bit indices (half the index bytes of torch's
// int64 index_select / index_copy_), 4 per thread.
__global__ void k_index_pack(int64_t cnt, const uint32_t *__restrict__ idx,
                             const double *__restrict__ full, double *__restrict__ out) {
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k < cnt) out[i + k] = __ldg(full + __ldcs(idx + i + k));
  }
}
__global__ void k_index_unpack(int64_t cnt, const uint32_t *__restrict__ idx,
                               const double *__restrict__ in, double *__restrict__ full) {
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k < cnt) full[__ldcs(idx + i + k)] = __ldcs(in + i + k);
  }
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_index_pack_f64(gcb_ctx *ctx, const double *full_dev, const uint32_t *idx_dev, int64_t count,
                       double *out_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && (count == 0 || (full_dev && idx_dev && out_dev)), "NULL argument");
  GCB_REQUIRE(count >= 0, "negative count");
  if (!count) return GCB_OK;
  DeviceGuard dg(ctx->device);
  k_index_pack<<<grid_for((count + 3) / 4, 256, (int64_t)ctx->num_sms * 8), 256, 0, ctx->stream>>>(
      count, idx_dev, full_dev, out_dev);
  after_launch(ctx, "k_index_pack");
  GCB_API_END
}

int gcb_index_unpack_f64(gcb_ctx *ctx, const double *in_dev, const uint32_t *idx_dev, int64_t count,
                         double *full_dev) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && (count == 0 || (full_dev && idx_dev && in_dev)), "NULL argument");
  GCB_REQUIRE(count >= 0, "negative count");
  if (!count) return GCB_OK;
  DeviceGuard dg(ctx->device);
  k_index_unpack<<<grid_for((count + 3) / 4, 256, (int64_t)ctx->num_sms * 8), 256, 0,
                   ctx->stream>>>(count, idx_dev, in_dev, full_dev);
  after_launch(ctx, "k_index_unpack");
  GCB_API_END
}

int gcb_ipc_alloc(gcb_ctx *ctx, int64_t bytes, void **ptr, unsigned char *handle) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && ptr && handle && bytes > 0, "NULL argument or empty allocation");
  DeviceGuard dg(ctx->device);
  // plain cudaMalloc: pool (cudaMallocAsync) memory is not IPC-exportable
  void *p = nullptr;
  GCB_CUDA(cudaMalloc(&p, (size_t)bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    GCB_CUDA(e);
  }
  GCB_CUDA(cudaMemset(p, 0, (size_t)bytes));
  std::memcpy(handle, &h, sizeof(h));
  *ptr = p;
  GCB_API_END
}

int gcb_ipc_free(gcb_ctx *ctx, void *ptr) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx, "NULL argument");
  DeviceGuard dg(ctx->device);
  if (ptr) GCB_CUDA(cudaFree(ptr));
  GCB_API_END
}

int gcb_ipc_open(gcb_ctx *ctx, const unsigned char *handle, void **ptr) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && handle && ptr, "NULL argument");
  DeviceGuard dg(ctx->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  GCB_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  GCB_API_END
}

int gcb_ipc_close(gcb_ctx *ctx, void *ptr) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx, "NULL argument");
  DeviceGuard dg(ctx->device);
  if (ptr) GCB_CUDA(cudaIpcCloseMemHandle(ptr));
  GCB_API_END
}

int gcb_peer_check(gcb_ctx *ctx) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx, "NULL argument");
  DeviceGuard dg(ctx->device);
  sync(ctx);
  check_peer_error(ctx);
  GCB_API_END
}

int gcb_pr_shard_init_p2p(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1,
                          const uint32_t *deg_dev, double *ranks_dev, double *const *out_dev,
                          const uint8_t *need_dev, int num_ranks, int rank,
                          uint32_t *const *flags_dev, uint32_t epoch) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && deg_dev && ranks_dev && out_dev && flags_dev, "NULL argument");
  GCB_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= bg->n && bg->n > 0 && (v0 % 4) == 0, "bad shard range");
  GCB_REQUIRE(num_ranks >= 1 && num_ranks <= 8 && rank >= 0 && rank < num_ranks,
              "1..8 ranks (need masks are 8 bits)");
  GCB_REQUIRE(bg->direction == 0, "sharded PageRank runs on a pull blocking");
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->sums.ensure(bg->n);
  GCB_CUDA(cudaMemsetAsync(bg->sums.p, 0, bg->n * sizeof(double), ctx->stream));
  const int64_t cnt = v1 - v0;
  if (cnt) {
    GCB_REQUIRE(need_dev, "NULL need mask");
    k_pr_init_p2p<<<grid_for(cnt, 256, 65536), 256, 0, ctx->stream>>>(
        cnt, v0, 1.0 / (double)bg->n, deg_dev, ranks_dev, bg->sums.p, out_dev, need_dev,
        num_ranks, rank);
    after_launch(ctx, "k_pr_init_p2p");
  }
  k_signal_peers<<<1, 32, 0, ctx->stream>>>(flags_dev, num_ranks, rank, epoch);
  after_launch(ctx, "k_signal_peers");
  GCB_API_END
}

int gcb_pr_shard_step_p2p(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, double damping,
                          uint32_t flags, const uint32_t *deg_dev, const double *contrib_in,
                          double *ranks_dev, double *delta_dev, double *const *out_dev,
                          const uint8_t *need_dev, int num_ranks, int rank,
                          uint32_t *const *flags_dev, uint32_t *my_flags_dev, uint32_t epoch) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && deg_dev && contrib_in && ranks_dev && out_dev && flags_dev &&
                  my_flags_dev,
              "NULL argument");
  GCB_REQUIRE(0 <= v0 && v0 <= v1 && v1 <= bg->n && (v0 % 4) == 0, "bad shard range");
  GCB_REQUIRE(num_ranks >= 1 && num_ranks <= 8 && rank >= 0 && rank < num_ranks,
              "1..8 ranks (need masks are 8 bits)");
  DeviceGuard dg(ctx->device);
  ensure_derived(ctx, bg);
  bg->sums.ensure(bg->n);
  // dead-skip steps (GCB_FLAG_DEAD_SKIP): ids without out-edges are read by no
  // slab (their need masks are 0), so their stores are skipped with them
  const int64_t cnt = shard_live_range(ctx, bg, v0, v1, flags, deg_dev) - v0;
  const unsigned grid = grid_for((cnt + 3) / 4, 512, (int64_t)(1 << 20) * ctx->num_sms);
  bg->deltas.ensure((int64_t)grid + 2);
  check_peer_error(ctx);
  // every peer's contributions of the previous epoch have landed
  k_wait_peers<<<1, 32, 0, ctx->stream>>>(my_flags_dev, num_ranks, rank, epoch - 1,
                                          peer_timeout_ns(), ctx->peer_err_dev);
  after_launch(ctx, "k_wait_peers");
  pull_sums(ctx, bg, contrib_in, nullptr, false, flags, -1, bg->sums.p, true);
  if (bg->hybrid) {  // degree-ordered shard (gcb_shard_blocking): hub-destination edges
    ProfScope ps(ctx, 1);
    push_scatter(ctx, bg->hybrid, contrib_in, bg->sums.p, false, flags, -1, true);
  }
  if (cnt) {
    GCB_REQUIRE(need_dev, "NULL need mask");
    ProfScope ps(ctx, 2);
    const double base = (1.0 - damping) / (double)bg->n;
    if (flags & GCB_FLAG_EXACT)
      k_pr_update_p2p<true><<<grid, 512, 0, ctx->stream>>>(cnt, v0, base, damping, bg->sums.p,
                                                           ranks_dev, deg_dev, out_dev, need_dev,
                                                           num_ranks, rank, bg->deltas.p);
    else
      k_pr_update_p2p<false><<<grid, 512, 0, ctx->stream>>>(cnt, v0, base, damping, bg->sums.p,
                                                            ranks_dev, deg_dev, out_dev, need_dev,
                                                            num_ranks, rank, bg->deltas.p);
    after_launch(ctx, "k_pr_update_p2p");
  }
  k_signal_peers<<<1, 32, 0, ctx->stream>>>(flags_dev, num_ranks, rank, epoch);
  after_launch(ctx, "k_signal_peers");
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

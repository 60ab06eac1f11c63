/*
 * gcb_b200.h -- C ABI of the B200-native TOCAB engine (libgcb_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (arxiv 1904.02241 "GraphCage", package `gcb`) is pure Python/numba, so its
 * boundary is the Python module API; the innermost operator is the numba
 * signature `_gather_rows(values, col, offsets, lo, hi, out)` at
 * /root/reference/pkg/src/gcb/kernels.py:155-161.  Each entry point below
 * names the reference function it replaces (file:line under
 * /root/reference/pkg/src/gcb/).  The Python package
 * `paper_1904_02241_b200` binds these with ctypes (INTEGRATION.md shows the
 * binding a maintainer of the reference would add).
 *
 * Conventions
 *  - Every function returns GCB_OK (0) or an error code; gcb_last_error()
 *    returns a thread-local message for the last failure.
 *      GCB_EINVAL (1) -> ValueError, GCB_ECUDA (2) -> RuntimeError,
 *      GCB_ENOMEM (3) -> MemoryError, GCB_EINDEX (4) -> IndexError,
 *      GCB_EFORMAT (5) -> GraphFormatError (a ValueError), GCB_EIO (6) -> OSError.
 *  - Plain pointers and sizes only.  Pointers named *_host are host memory,
 *    borrowed for the duration of the call; pointers named *_dev are device
 *    memory on the context's device.  Host-buffer calls are synchronous on
 *    return.  _dev calls are stream-ordered on the context stream and return
 *    without synchronising unless stated.
 *  - Graph state lives on the device in opaque handles (gcb_csr,
 *    gcb_blocked) owned by the caller and released with *_destroy.
 *  - Vertex ids are uint32 (graph.py:4-6); CSR row offsets int64; edge weights
 *    float64; every floating-point result is float64 (kernels.py:83-89).
 */
#ifndef GCB_B200_H
#define GCB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define GCB_OK 0
#define GCB_EINVAL 1
#define GCB_ECUDA 2
#define GCB_ENOMEM 3
#define GCB_EINDEX 4
#define GCB_EFORMAT 5
#define GCB_EIO 6

#define GCB_DIR_PULL 0
#define GCB_DIR_PUSH 1

/* flags for the value kernels */
#define GCB_FLAG_EXACT 1u        /* reference operation order, bit-exact      */
#define GCB_FLAG_F32_VALUES 2u   /* f32 copy of the gathered vector (f64 sums) */
#define GCB_FLAG_NO_L2_WINDOW 4u /* disable the per-block access-policy window */
#define GCB_FLAG_NO_GRAPH 8u     /* launch eagerly instead of a CUDA graph     */
#define GCB_FLAG_NO_RELABEL 16u  /* fast pull paths: keep the input numbering  */
#define GCB_FLAG_DEAD_SKIP 32u   /* shard steps on degree-ordered shards, tol = 0,
                                    not the last iteration: ranks and delta are
                                    dead, update only owned ids with out-edges */

/* BFS direction modes (DirectionPolicy.MODES, traversal.py:46-61) */
#define GCB_BFS_AUTO 0
#define GCB_BFS_FORCE_PUSH 1
#define GCB_BFS_FORCE_PULL 2

typedef struct gcb_ctx gcb_ctx;
typedef struct gcb_csr gcb_csr;
typedef struct gcb_blocked gcb_blocked;

/* ---- runtime ----------------------------------------------------------- */
const char *gcb_last_error(void);
int gcb_version(void);
int gcb_ctx_create(int device, gcb_ctx **out);
int gcb_ctx_destroy(gcb_ctx *ctx);
/* run on an external stream (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the context's own stream */
int gcb_ctx_set_stream(gcb_ctx *ctx, void *cuda_stream);
int gcb_ctx_sync(gcb_ctx *ctx);
/* L2 facts the partitioner sizes blocks from (SURVEY 7 "hard parts") */
int gcb_ctx_info(gcb_ctx *ctx, int64_t *num_sms, int64_t *l2_bytes,
                 int64_t *persist_max_bytes, int64_t *window_max_bytes);
/* persisting-L2 set-aside this context made (GCB_L2_PERSIST; 0 = none, the
 * pull gather then uses its per-load range policy instead of a window) */
int gcb_ctx_l2_set_aside(gcb_ctx *ctx, int64_t *bytes);
/* number of this library's kernel launches issued on ctx so far */
int gcb_ctx_launch_count(gcb_ctx *ctx, int64_t *count);
/* CUDA-event timing of kernel groups on the ctx stream (bench.py roofline):
 * categories 0 gather/scatter, 1 carry fix-up, 2 merge/update, 3 other.
 * read_profile synchronises, returns ms[4] / launches-groups[4], resets. */
int gcb_ctx_set_profiling(gcb_ctx *ctx, int enable);
int gcb_ctx_read_profile(gcb_ctx *ctx, double *ms_out, int64_t *count_out);

/* ---- CSR graphs (graph.py) -------------------------------------------- */
/* CsrGraph(n, m, row_offsets, col_indices, edge_weights) graph.py:45-107:
 * upload an already-canonical CSR (validation is the caller's). */
int gcb_csr_upload(gcb_ctx *ctx, int64_t n, int64_t m, const int64_t *row_offsets_host,
                   const uint32_t *col_host, const double *weights_host_or_null,
                   gcb_csr **out);
/* from_edges graph.py:110-130: stable lexsort by (src, dst) on the device. */
int gcb_csr_from_edges(gcb_ctx *ctx, int64_t n, int64_t m, const int64_t *src_host,
                       const int64_t *dst_host, const double *weights_host_or_null,
                       gcb_csr **out);
/* _generate_rmat graph.py:371-386 bit-exactly on the device.  (state, inc) is
 * numpy's PCG64 state after seeding (np.random.PCG64(seed).state), split in
 * 64-bit halves; t_a / t_ab / t_abc are the f64 thresholds of graph.py:378-383. */
int gcb_csr_generate_rmat(gcb_ctx *ctx, int scale, int64_t edge_factor,
                          uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                          uint64_t inc_lo, double t_a, double t_ab, double t_abc,
                          int transposed, gcb_csr **out);
/* transpose graph.py:133-138 / symmetrize graph.py:141-151 */
int gcb_csr_transpose(gcb_ctx *ctx, const gcb_csr *g, gcb_csr **out);
int gcb_csr_symmetrize(gcb_ctx *ctx, const gcb_csr *g, gcb_csr **out);
int gcb_csr_info(const gcb_csr *g, int64_t *n, int64_t *m, int *weighted);
int gcb_csr_download(gcb_ctx *ctx, const gcb_csr *g, int64_t *row_offsets_host,
                     uint32_t *col_host, double *weights_host_or_null);
/* rows [v0, v1) of g, all other rows emptied (n x n): a destination shard's
 * slab of the transpose */
int gcb_csr_row_slab(gcb_ctx *ctx, const gcb_csr *g, int64_t v0, int64_t v1, gcb_csr **out);
/* counts_dev[v] (device uint32[n]) = occurrences of v in the column ids;
 * for the transpose these are the forward out-degrees (kernels.py:199-204) */
int gcb_csr_col_counts(gcb_ctx *ctx, const gcb_csr *g, uint32_t *counts_dev);
/* set/replace the edge weights of a device CSR (storage order) */
int gcb_csr_set_weights(gcb_ctx *ctx, gcb_csr *g, const double *weights_host);
int gcb_csr_destroy(gcb_csr *g);

/* ---- TOCAB blocking (blocking.py) --------------------------------------- */
/* partition_tocab blocking.py:204-253 on the device (bit-identical arenas). */
int gcb_partition_tocab(gcb_ctx *ctx, const gcb_csr *g, int direction, int64_t width,
                        gcb_blocked **out);
/* partition_cb blocking.py:256-286 (the conventional-blocking ablation): the
 * same edge split as a pull TOCAB partition, but every block holds all n rows
 * (identity id_map, empty rows included; row_starts[b] = b*n, a block's lro
 * segment has n+1 entries).  pr_blocked / spmv_blocked on it run _cb_sums
 * (kernels.py:350-364): a dense partial vector per block, merged in block order. */
int gcb_partition_cb(gcb_ctx *ctx, const gcb_csr *g, int64_t width, gcb_blocked **out);
/* mask_dev[n] (device bytes) = 1 for every source the blocking's edges read:
 * the per-rank need set of the sparse contribution exchange. */
int gcb_blocked_source_mask(gcb_ctx *ctx, const gcb_blocked *bg, uint8_t *mask_dev);
/* Request model of the fast pull gather (no reference counterpart; feeds
 * bench.py's roofline.request_frac): out4 = {edges served from the
 * shared-memory hot table, cold edges (one L2 request each), hub-destination
 * edges of the hybrid push pass, 1 if the degree-ordered copy is the layout}.
 * Counts the layout the fast pull runs (the promoted copy when one exists). */
int gcb_blocked_gather_census(gcb_ctx *ctx, gcb_blocked *bg, int64_t *out4);
/* Marks an uploaded pull blocking as cb-scheme (arenas already in that layout). */
int gcb_blocked_mark_cb(gcb_ctx *ctx, gcb_blocked *bg);
/* BlockedGraph(...) blocking.py:86-110 from host arenas (int64 lro converted
 * to per-block uint32 local offsets on the device). */
int gcb_blocked_upload(gcb_ctx *ctx, int direction, int64_t width, int64_t n, int64_t m,
                       int64_t num_blocks, const int64_t *row_starts_host,
                       const int64_t *lro_arena_host, const uint32_t *id_map_host,
                       const int64_t *edge_starts_host, const uint32_t *col_arena_host,
                       const double *weight_arena_host_or_null, gcb_blocked **out);
int gcb_blocked_info(const gcb_blocked *bg, int *direction, int64_t *width, int64_t *n,
                     int64_t *m, int64_t *num_blocks, int64_t *total_local_rows,
                     int *weighted);
int gcb_blocked_download(gcb_ctx *ctx, const gcb_blocked *bg, int64_t *row_starts_host,
                         int64_t *lro_arena_host, uint32_t *id_map_host,
                         int64_t *edge_starts_host, uint32_t *col_arena_host,
                         double *weight_arena_host_or_null);
/* BlockedGraph.range_bounds blocking.py:151-173 ([B, ceil(n/k)+1] int64) */
int gcb_blocked_range_bounds(gcb_ctx *ctx, gcb_blocked *bg, int64_t k,
                             int64_t *bounds_host);
int gcb_blocked_destroy(gcb_blocked *bg);
/* GCB container (blocking.py:327-441), written from and read into device
 * arenas (csrc/gcbio.cu): write_gcb blocking.py:341-365 and read_gcb
 * blocking.py:368-441, byte-identical files and the same checks in the same
 * order (truncated, CRC, magic, direction, block table, trailing bytes, edge
 * totals; GCB_EFORMAT).  The CRC-32 (zlib's) is computed on the device. */
int gcb_blocked_save(gcb_ctx *ctx, gcb_blocked *bg, const char *path);
int gcb_blocked_load(gcb_ctx *ctx, const char *path, gcb_blocked **out);
int gcb_blocked_scheme(const gcb_blocked *bg, int *is_cb);
/* zlib.crc32 of a host buffer, computed on the device (the container's check) */
int gcb_crc32(gcb_ctx *ctx, const void *data_host, int64_t len, uint32_t *crc);

/* ---- value kernels (kernels.py) ----------------------------------------- */
/* compute_contributions kernels.py:185-191: out = deg > 0 ? rank / deg : 0 */
int gcb_compute_contributions(gcb_ctx *ctx, int64_t n, const double *ranks_host,
                              const int64_t *out_degrees_host, double *out_host);
/* pr_blocked kernels.py:367-405 (tocab pull / push).  k (kernels.py:47) is
 * validated (k >= 1) but results are k-invariant bitwise, as in the reference. */
int gcb_pr_blocked(gcb_ctx *ctx, gcb_blocked *bg, double damping, double tol,
                   int max_iters, int64_t k, uint32_t flags, double *ranks_host,
                   int *iterations, int *converged);
/* same, device-resident: ranks_dev[n] receives the ranks; no host sync when
 * tol == 0 (iterations = max_iters).  Used by bench.py's device-timed leg. */
int gcb_pr_blocked_dev(gcb_ctx *ctx, gcb_blocked *bg, double damping, double tol,
                       int max_iters, uint32_t flags, double *ranks_dev,
                       int *iterations, int *converged);
/* pr_baseline kernels.py:207-268: unblocked pull over the transpose / push
 * over the forward graph.  out_degrees_host may be NULL (kernels.py:199-204). */
int gcb_pr_baseline(gcb_ctx *ctx, const gcb_csr *g, int direction, double damping,
                    double tol, int max_iters, uint32_t flags,
                    const int64_t *out_degrees_host_or_null, double *ranks_host,
                    int *iterations, int *converged);
/* Destination-sharded PageRank (multi-GPU).  Rank r owns
 * [v0, v1) (v0 % 4 == 0) and a pull blocking of its row slab; contrib_dev and
 * ranks_dev are full n-vectors on the device, deg_dev the global
 * out-degrees.  init sets ranks/contributions of the owned slice; step
 * gathers over the full contribution vector, then updates the owned slice of
 * ranks and contributions in place and (if delta_dev) writes the slice's L1
 * delta.  The caller all-gathers the owned contribution slices between steps
 * (NCCL).  Both calls are stream-ordered and do not synchronise. */
int gcb_pr_shard_init(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1,
                      const uint32_t *deg_dev, double *contrib_dev, double *ranks_dev);
int gcb_pr_shard_step(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, double damping,
                      uint32_t flags, const uint32_t *deg_dev, double *contrib_dev,
                      double *ranks_dev, double *delta_dev);
/* Degree-ordered destination shards (parallel.py): gcb_csr_degree_order
 * renumbers a transpose CSR by descending out-degree (ties: ascending id;
 * perm_dev[old] = new, uint32[n]) -- the permutation the single-GPU promotion
 * (relabel.cu) picks -- so all ranks share one numbering.  gcb_shard_blocking
 * blocks one shard's row slab of that graph (pull, `width`) with the prefix
 * hot set and, where the cost model says it pays, the hybrid hub-destination
 * push pass that gcb_pr_shard_step(_p2p) then runs after the pull gather.
 * Fast mode only (the reference's summation order is that of the original
 * numbering). */
int gcb_csr_degree_order(gcb_ctx *ctx, const gcb_csr *gt, uint32_t *perm_dev, gcb_csr **out);
int gcb_shard_blocking(gcb_ctx *ctx, const gcb_csr *slab, int64_t width, gcb_blocked **out);
/* The NCCL exchange between gcb_pr_shard_step calls (parallel.SparseExchange,
 * SURVEY 8e): out[i] = full[idx[i]] packs the values the peers read into the
 * all_to_all send buffer; full[idx[i]] = in[i] scatters the received ones.
 * Device pointers, uint32 indices, stream-ordered on the ctx stream. */
int gcb_index_pack_f64(gcb_ctx *ctx, const double *full_dev, const uint32_t *idx_dev,
                       int64_t count, double *out_dev);
int gcb_index_unpack_f64(gcb_ctx *ctx, const double *in_dev, const uint32_t *idx_dev,
                         int64_t count, double *full_dev);
/* The same step with the contribution exchange fused into the update over
 * peer memory (csrc/exchange.cu), replacing the NCCL exchange between
 * gcb_pr_shard_step calls.  Buffers come from gcb_ipc_alloc and are mapped in
 * every rank with gcb_ipc_open (CUDA IPC; NVLink P2P across GPUs).
 *   out_dev[p]   device array of num_ranks pointers: rank p's contribution
 *                buffer of this epoch's parity (the caller alternates two)
 *   need_dev     uint8[v1 - v0]: bit p = rank p's slab reads that source
 *   flags_dev[p] device array of num_ranks pointers to each rank's uint32[P]
 *                epoch flags; my_flags_dev is this rank's own
 * init publishes epoch `epoch`; step waits for every peer's epoch - 1,
 * gathers contrib_in (the other buffer), updates the owned slice, stores each
 * contribution into the peers that read it and publishes `epoch`.  Stream-
 * ordered, no host synchronisation.  A peer that misses its deadline
 * (GCB_PEER_TIMEOUT_S, default 120 s) makes the wait kernel record the fact
 * and return instead of hanging the device; the next step call, or
 * gcb_peer_check (which synchronises the ctx stream), returns GCB_ECUDA. */
int gcb_ipc_alloc(gcb_ctx *ctx, int64_t bytes, void **ptr, unsigned char *handle64);
int gcb_ipc_free(gcb_ctx *ctx, void *ptr);
int gcb_ipc_open(gcb_ctx *ctx, const unsigned char *handle64, void **ptr);
int gcb_ipc_close(gcb_ctx *ctx, void *ptr);
int gcb_pr_shard_init_p2p(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1,
                          const uint32_t *deg_dev, double *ranks_dev, double *const *out_dev,
                          const uint8_t *need_dev, int num_ranks, int rank,
                          uint32_t *const *flags_dev, uint32_t epoch);
int gcb_peer_check(gcb_ctx *ctx);
int gcb_pr_shard_step_p2p(gcb_ctx *ctx, gcb_blocked *bg, int64_t v0, int64_t v1, double damping,
                          uint32_t flags, const uint32_t *deg_dev, const double *contrib_in,
                          double *ranks_dev, double *delta_dev, double *const *out_dev,
                          const uint8_t *need_dev, int num_ranks, int rank,
                          uint32_t *const *flags_dev, uint32_t *my_flags_dev, uint32_t epoch);
/* process_block_pull kernels.py:275-282: partials of block b (n_local f64) */
int gcb_process_block_pull(gcb_ctx *ctx, gcb_blocked *bg, int64_t block,
                           const double *contrib_host, uint32_t flags,
                           double *out_host);
/* process_block_push kernels.py:285-297: sums[lo:hi] += block b scatter */
int gcb_process_block_push(gcb_ctx *ctx, gcb_blocked *bg, int64_t block,
                           const double *contrib_host, uint32_t flags,
                           double *sums_host);
/* accumulate_ranges kernels.py:300-321 */
int gcb_accumulate_ranges(gcb_ctx *ctx, gcb_blocked *bg, const double *partials_host,
                          int64_t k, double *out_host);
/* segment_row_sums kernels.py:173-182 over a device CSR */
int gcb_segment_row_sums(gcb_ctx *ctx, const gcb_csr *g, const double *values_host,
                         int use_weights, uint32_t flags, double *out_host);
/* spmv kernels.py:412-428 and spmv_blocked kernels.py:431-487 */
int gcb_spmv(gcb_ctx *ctx, const gcb_csr *g, const double *x_host, int direction,
             uint32_t flags, double *y_host);
int gcb_spmv_blocked(gcb_ctx *ctx, gcb_blocked *bg, const double *x_host, int64_t k,
                     uint32_t flags, double *y_host);
int gcb_spmv_blocked_dev(gcb_ctx *ctx, gcb_blocked *bg, const double *x_dev,
                         uint32_t flags, double *y_dev);

/* ---- traversal (traversal.py) ------------------------------------------- */
/* bfs traversal.py:201-209 with choose_direction traversal.py:93-99.
 * g = forward CSR; bg_pull = partition_tocab(transpose(g), "pull", W) or NULL
 * (then width max(1, n/8) as traversal.py:186-187).  Outputs: depth[n]
 * (INT32_MAX = unvisited), level_verts[n] (level queues concatenated, each
 * ascending), level_sizes[max_levels], directions[max_levels] (0 push,
 * 1 blocked-pull, one per expansion), *num_levels (non-empty levels),
 * *num_expansions. */
int gcb_bfs(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int64_t source,
            int mode, int64_t capacity_bytes, int64_t value_bytes, int32_t *depth_host,
            uint32_t *level_verts_host, int64_t *level_sizes_host,
            uint8_t *directions_host, int64_t max_levels, int64_t *num_levels,
            int64_t *num_expansions);
/* One level of the forward sweep: direction 0 = forward_push_step
 * traversal.py:121-140 over g, 1 = forward_pull_step traversal.py:143-176
 * over bg_pull.  depth[n] (in/out), sigma[n] (in/out, NULL = no path counts),
 * frontier = current queue; writes the next queue (ascending) to next_host
 * and its length to *next_size; discovered vertices get depth level + 1. */
int gcb_bfs_step(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int direction,
                 int32_t *depth_host, double *sigma_host_or_null, const uint32_t *frontier_host,
                 int64_t frontier_size, int32_t level, uint32_t *next_host, int64_t *next_size);
/* SSSP with non-negative integer weights (named by BASELINE.json; no
 * reference code).  The weights are the graphs' edge weights
 * (integral float64 < 2^53): g = weighted forward CSR, bg_pull =
 * partition_tocab(transpose(g), "pull", W) carrying the same weights, or NULL
 * (push-only).  Frontier Bellman-Ford; the per-round direction switch is
 * choose_direction's rule (traversal.py:93-99).  dist[n] int64, INT64_MAX =
 * unreachable; *rounds = relaxation rounds; directions_host (may be NULL)
 * receives one byte per round (0 push, 1 pull). */
int gcb_sssp(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int64_t source, int mode,
             int64_t capacity_bytes, int64_t value_bytes, int64_t *dist_host,
             uint8_t *directions_host, int64_t max_rounds, int64_t *rounds);
/* Weakly connected components, labels = min vertex id. */
int gcb_cc(gcb_ctx *ctx, const gcb_csr *g, uint32_t *labels_host, int64_t *num_components);
/* Betweenness centrality (bc traversal.py:257-278): for each source in order,
 * a forward sweep with path counts (push / blocked-pull per choose_direction,
 * bg_pull NULL = partition_tocab(transpose(g), "pull", max(1, n // 8))) and
 * the dependency pass (bc_backward traversal.py:212-236); centrality[n] =
 * sum of the per-source dependencies (ordered pairs, endpoints excluded).
 * flags: GCB_FLAG_EXACT sums every vertex's out-edges in CSR order
 * (bit-identical to the reference); default = warp reductions. */
int gcb_bc(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, const int64_t *sources_host,
           int64_t num_sources, int mode, int64_t capacity_bytes, int64_t value_bytes,
           uint32_t flags, double *centrality_host);
/* bc_single_source traversal.py:239-254: forward sweep with path counts and
 * the dependency pass on the device; delta (delta[source] = 0), the final
 * depth / sigma, the per-level vertex lists (concatenated, sizes in
 * level_sizes_host) and the per-expansion directions (1 = blocked pull) */
int gcb_bc_single_source(gcb_ctx *ctx, const gcb_csr *g, gcb_blocked *bg_pull, int64_t source,
                         int mode, int64_t capacity_bytes, int64_t value_bytes, uint32_t flags,
                         double *delta_host, int32_t *depth_host, double *sigma_host,
                         uint32_t *level_verts_host, int64_t *level_sizes_host,
                         uint8_t *directions_host, int64_t max_levels, int64_t *num_levels,
                         int64_t *num_expansions);
/* bc_backward traversal.py:212-236 for a given forward state: depth[n]
 * (INT32_MAX = unreached), sigma[n]; writes delta[n] with delta[source] = 0. */
int gcb_bc_backward(gcb_ctx *ctx, const gcb_csr *g, const int32_t *depth_host,
                    const double *sigma_host, int64_t source, uint32_t flags, double *delta_host);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* GCB_B200_H */

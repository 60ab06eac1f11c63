// cub_ops.cu -- thin wrappers over CUB (CUDA toolkit library) used only by the
// one-off preprocessing path (CSR build, partitioner); never by the per-
// iteration hot path.
#include <cub/cub.cuh>

#include "gcb_internal.cuh"

namespace gcb {

namespace {
template <typename F>
void run_cub(gcb_ctx *ctx, F &&f) {
  size_t bytes = 0;
  GCB_CUDA(f(nullptr, bytes));
  ctx->cub_tmp.ensure(bytes + 256);
  bytes = ctx->cub_tmp.n;
  GCB_CUDA(f(ctx->cub_tmp.p, bytes));
  ctx->launches++;
}
}  // namespace

void cub_sort_keys_u64(gcb_ctx *ctx, uint64_t *keys, uint64_t *keys_alt, int64_t m, int end_bit,
                       uint64_t **result) {
  cub::DoubleBuffer<uint64_t> db(keys, keys_alt);
  if (m > 0)
    run_cub(ctx, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortKeys(t, b, db, m, 0, end_bit, ctx->stream);
    });
  *result = db.Current();
}

void cub_sort_pairs_u64_u32(gcb_ctx *ctx, uint64_t *keys, uint64_t *keys_alt, uint32_t *vals,
                            uint32_t *vals_alt, int64_t m, int end_bit, uint64_t **res_keys,
                            uint32_t **res_vals) {
  cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
  if (m > 0)
    run_cub(ctx, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, end_bit, ctx->stream);
    });
  *res_keys = dk.Current();
  *res_vals = dv.Current();
}

void cub_sort_pairs_u32_u32(gcb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                            uint32_t *vals_alt, int64_t m, int end_bit, uint32_t **res_keys,
                            uint32_t **res_vals) {
  cub::DoubleBuffer<uint32_t> dk(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
  if (m > 0 && end_bit > 0)
    run_cub(ctx, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, end_bit, ctx->stream);
    });
  *res_keys = dk.Current();
  *res_vals = dv.Current();
}

void cub_sort_pairs_desc_u32_u32(gcb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                                 uint32_t *vals_alt, int64_t m, uint32_t **res_keys,
                                 uint32_t **res_vals) {
  cub::DoubleBuffer<uint32_t> dk(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
  if (m > 0)
    run_cub(ctx, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairsDescending(t, b, dk, dv, m, 0, 32, ctx->stream);
    });
  *res_keys = dk.Current();
  *res_vals = dv.Current();
}

void cub_exclusive_sum_u32(gcb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t count) {
  if (count <= 0) return;
  run_cub(ctx, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, in, out, count, ctx->stream);
  });
}

void cub_exclusive_sum_i64(gcb_ctx *ctx, const int64_t *in, int64_t *out, int64_t count) {
  if (count <= 0) return;
  run_cub(ctx, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, in, out, count, ctx->stream);
  });
}

void cub_inclusive_sum_u32(gcb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t count) {
  if (count <= 0) return;
  run_cub(ctx, [&](void *t, size_t &b) {
    return cub::DeviceScan::InclusiveSum(t, b, in, out, count, ctx->stream);
  });
}

void cub_sum_u64(gcb_ctx *ctx, const uint64_t *in, uint64_t *out_dev, int64_t count) {
  run_cub(ctx, [&](void *t, size_t &b) {
    return cub::DeviceReduce::Sum(t, b, in, out_dev, count, ctx->stream);
  });
}

}  // namespace gcb

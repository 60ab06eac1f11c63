// tiles.cuh -- the edge-balanced warp-tile machinery shared by the pull
// kernels (sum: gather.cu k_pull_hot; min-plus: traversal.cu SSSP pull).
//
// A warp owns a 256-edge tile of a block's arena (lane = 8 consecutive
// edges).  Row boundaries come from the row-start bitmap (bit q = arena edge
// q opens a local row; local rows are never empty, blocking.py:189-201), so
// row(q) = tile_row + #row starts in (first valid edge, q].  tile_reduce
// combines the lane's 8 values into per-row results with in-lane runs plus a
// segmented shuffle scan over lane tails, and calls emit(row, value, r_last)
// once per row piece in the tile; r_last is the tile's last row, so callers
// can tell pieces of rows that cross a tile edge (row == r0 && !first_start,
// row == r_last && last_cont).
#pragma once

#include <cstdint>

#include "gcb_internal.cuh"

namespace gcb {

struct TileBits {
  uint32_t vm;       // lane's valid edges (bit k = edge 8*lane + k in [llo, lhi))
  uint32_t bits;     // lane's row starts among valid edges, tile's first valid edge dropped
  bool first_start;  // the tile's first valid edge opens its row
  bool last_cont;    // the tile's last row continues into the next tile
};

// fw: lanes 0..7 hold bitmap words 0..7 of the tile, lanes 8..31 word 8
// (the first word of the next tile); llo/lhi: valid tile positions.
__device__ __forceinline__ TileBits tile_bits(uint32_t fw, int llo, int lhi, int lane) {
  constexpr int V = kTileV;
  const unsigned FULL = 0xffffffffu;
  TileBits t;
  const int a = llo - lane * V, z = lhi - lane * V;
  t.vm = (z <= 0 || a >= V) ? 0u
                            : ((0xffu >> (V - (z < V ? z : V))) & (0xffu << (a > 0 ? a : 0)));
  const uint32_t wl = __shfl_sync(FULL, fw, lane >> 2);
  uint32_t bits = (wl >> ((lane & 3) * 8)) & t.vm;
  if (a >= 0 && a < V) bits &= ~(1u << a);
  t.bits = bits;
  t.first_start = (__shfl_sync(FULL, fw, llo >> 5) >> (llo & 31)) & 1u;
  t.last_cont = (lhi == kTileT) && !(__shfl_sync(FULL, fw, 8) & 1u);
  return t;
}

// Per-row reduction of a tile.  Comb(a, b) must be associative; ident is its
// identity.  Whole-warp call (every lane, converged).
template <typename T, class Comb, class Emit>
__device__ __forceinline__ void tile_reduce(const T (&v)[kTileV], const TileBits &tb, uint32_t r0,
                                            int lane, T ident, Comb comb, Emit emit) {
  constexpr int V = kTileV;
  const unsigned FULL = 0xffffffffu;
  if (__all_sync(FULL, tb.bits == 0)) {
    // the whole tile lies in row r0: a plain warp reduction, one emit
    T acc = ident;
#pragma unroll
    for (int k = 0; k < V; ++k) acc = comb(acc, ((tb.vm >> k) & 1u) ? v[k] : ident);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc = comb(acc, __shfl_xor_sync(FULL, acc, d));
    if (lane == 0) emit(r0, acc, r0);
    return;
  }
  // exclusive prefix of row starts over lanes
  const int cnt = __popc(tb.bits);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += y;
  }
  const uint32_t r_last = r0 + (uint32_t)__shfl_sync(FULL, incl, 31);
  const bool lane_valid = tb.vm != 0;
  const int kf = lane_valid ? __ffs(tb.vm) - 1 : 0;
  uint32_t j = r0 + (uint32_t)(incl - cnt) + ((tb.bits >> kf) & 1u);
  const uint32_t sb = tb.bits & ~((2u << kf) - 1u);  // row starts after the lane's first edge

  const uint32_t head_j = j;
  T head = ident, acc = ident;
  bool head_closed = false;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    if ((sb >> k) & 1u) {
      if (!head_closed) {
        head = acc;
        head_closed = true;
      } else {
        emit(j, acc, r_last);
      }
      acc = ident;
      ++j;
    }
    acc = comb(acc, ((tb.vm >> k) & 1u) ? v[k] : ident);
  }
  // segmented inclusive scan of the lane tails (key = tail row)
  const int key = lane_valid ? (int)j : -1 - lane;
  T val = acc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int k2 = __shfl_up_sync(FULL, key, d);
    const T v2 = __shfl_up_sync(FULL, val, d);
    if (lane >= d && k2 == key) val = comb(v2, val);
  }
  int pk = __shfl_up_sync(FULL, key, 1);
  const T pv = __shfl_up_sync(FULL, val, 1);
  if (lane == 0) pk = -1000;
  int nh = __shfl_down_sync(FULL, lane_valid ? (int)head_j : -1000, 1);
  if (lane == 31) nh = -1000;
  if (lane_valid) {
    if (head_closed) emit(head_j, (pk == (int)head_j) ? comb(pv, head) : head, r_last);
    if (nh != (int)j) emit(j, val, r_last);
  }
}

}  // namespace gcb

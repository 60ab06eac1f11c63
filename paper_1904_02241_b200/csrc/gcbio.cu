// gcbio.cu -- the GCB container (blocking.py:327-441) written from and read
// into device arenas: SURVEY 8f row 2, "persist device partitions, with a
// CRC32 check and a byte-identical format".
//
// File layout (little endian, the reference's): header "GCB1", u8
// direction, u8 flags (bit 0 weights, bit 1 cb scheme), u16 0, u64 n, m,
// width, B; per block u64 n_local, u64 n_edges, u32 id_map[n_local],
// u64 local_row_offsets[n_local + 1], u32 col[n_edges], f64 w[n_edges] if
// weighted; trailing u32 zlib CRC-32 of every preceding byte.
//
// Save: the body is packed on the device (every section starts at a 4-byte
// aligned offset: header 40 B, block header 16 B, sections 4/8 B per entry),
// its CRC-32 computed on the device, then streamed to the file through two
// pinned buffers (the D2H of chunk k+1 overlaps the write of chunk k).
// Load: the file is streamed into a device body buffer the same way, the
// CRC is checked on the device before anything is parsed, the block table is
// walked on the host (16 bytes per block, read from the file), and the
// arenas are unpacked by device kernels straight into a gcb_blocked.
//
// CRC-32 (reflected, poly 0xEDB88320, init/final ~0) is linear over GF(2):
// with raw(s, M) = the table recurrence from state s over M,
//     raw(s, A || B) = Z_|B|(raw(s, A)) ^ raw(0, B),
// where Z_k (k zero bytes) is a 32x32 bit matrix.  The device computes
// raw(0, .) of every 8 KiB chunk -- one warp per chunk, each lane 256 bytes
// staged through shared memory, the 32 lane results folded by a tree of
// Z_256 .. Z_4096 -- and the host folds the chunk results with Z_8192
// (Horner) and runs the < 8 KiB tail bytewise.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gcb_internal.cuh"

namespace gcb {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr int kLaneBytes = 256;                 // bytes per lane
constexpr int64_t kChunk = 32 * kLaneBytes;     // 8 KiB per warp
constexpr int kCrcWarps = 4;                    // warps per CTA
constexpr int kMagicLen = 4;
constexpr int64_t kHeaderBytes = 40;  // "<4sBBH4Q"
constexpr uint8_t kFlagWeights = 1, kFlagCb = 2;

struct CrcTables {
  uint32_t byte[256];      // one-byte recurrence step
  uint32_t zmat[5][32];    // Z_{256 << j}: column i = image of bit i
};
__constant__ CrcTables c_crc;

// ---- host-side GF(2) helpers ----------------------------------------------
static uint32_t crc_byte_step(uint32_t c) {
  for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (kCrcPoly & (0u - (c & 1u)));
  return c;
}

struct HostCrc {
  uint32_t table[256];
  uint32_t z_chunk[4][256];  // Z_kChunk applied through 4 byte tables
  CrcTables dev;
  HostCrc() {
    for (uint32_t i = 0; i < 256; ++i) table[i] = crc_byte_step(i);
    // Z_k columns by running k zero bytes from each basis vector
    auto zeros = [&](uint32_t s, int64_t k) {
      for (int64_t i = 0; i < k; ++i) s = table[s & 0xffu] ^ (s >> 8);
      return s;
    };
    std::memcpy(dev.byte, table, sizeof(table));
    for (int j = 0; j < 5; ++j)
      for (int i = 0; i < 32; ++i) dev.zmat[j][i] = zeros(1u << i, (int64_t)kLaneBytes << j);
    uint32_t col[32];
    for (int i = 0; i < 32; ++i) col[i] = zeros(1u << i, kChunk);
    for (int b = 0; b < 4; ++b)
      for (uint32_t v = 0; v < 256; ++v) {
        uint32_t r = 0;
        for (int i = 0; i < 8; ++i)
          if ((v >> i) & 1u) r ^= col[8 * b + i];
        z_chunk[b][v] = r;
      }
  }
  uint32_t shift_chunk(uint32_t s) const {
    return z_chunk[0][s & 0xffu] ^ z_chunk[1][(s >> 8) & 0xffu] ^ z_chunk[2][(s >> 16) & 0xffu] ^
           z_chunk[3][s >> 24];
  }
  uint32_t bytes(uint32_t s, const uint8_t *p, int64_t k) const {
    for (int64_t i = 0; i < k; ++i) s = table[(s ^ p[i]) & 0xffu] ^ (s >> 8);
    return s;
  }
};

static const HostCrc &host_crc() {
  static const HostCrc h;
  return h;
}

static void ensure_crc_constants(gcb_ctx *ctx) {
  static std::mutex mu;
  static uint64_t done = 0;  // bit d: device d has the tables
  std::lock_guard<std::mutex> lk(mu);
  const uint64_t bit = uint64_t(1) << (ctx->device & 63);
  if (done & bit) return;
  GCB_CUDA(cudaMemcpyToSymbolAsync(c_crc, &host_crc().dev, sizeof(CrcTables), 0,
                                   cudaMemcpyHostToDevice, ctx->stream));
  done |= bit;
}

// ---- device CRC of whole chunks -------------------------------------------
__device__ __forceinline__ uint32_t zmul(int j, uint32_t s) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) r ^= c_crc.zmat[j][i] & (0u - ((s >> i) & 1u));
  return r;
}

// out[c] = raw(0, body[c * kChunk, (c + 1) * kChunk)) for c < nchunks
__global__ void __launch_bounds__(kCrcWarps * 32)
    k_crc_chunks(const uint8_t *__restrict__ body, int64_t nchunks, uint32_t *__restrict__ out) {
  // per warp: 32 lanes x 256 bytes, padded by one word per lane so that the
  // lanes' word k sit in different banks
  constexpr int LW = kLaneBytes / 4 + 1;
  __shared__ uint32_t s_tab[256];
  __shared__ uint32_t s_buf[kCrcWarps][32 * LW];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tab[i] = c_crc.byte[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *buf = s_buf[wid];
  const int64_t nw = (int64_t)gridDim.x * kCrcWarps;
  for (int64_t c = (int64_t)blockIdx.x * kCrcWarps + wid; c < nchunks; c += nw) {
    const uint4 *src = reinterpret_cast<const uint4 *>(body + c * kChunk);
    // coalesced 16-byte loads: word w of the chunk -> lane w / 64, slot w % 64
#pragma unroll 4
    for (int k = 0; k < kChunk / 16 / 32; ++k) {
      const int q = k * 32 + lane;  // uint4 index within the chunk
      const uint4 v = __ldcs(src + q);
      const int w = q * 4, ln = w / (kLaneBytes / 4), sl = w % (kLaneBytes / 4);
      uint32_t *d = buf + ln * LW + sl;
      d[0] = v.x;
      d[1] = v.y;
      d[2] = v.z;
      d[3] = v.w;
    }
    __syncwarp();
    uint32_t s = 0;
    const uint32_t *mine = buf + lane * LW;
#pragma unroll 8
    for (int k = 0; k < kLaneBytes / 4; ++k) {
      uint32_t x = mine[k];
      s = s_tab[(s ^ x) & 0xffu] ^ (s >> 8);
      s = s_tab[(s ^ (x >> 8)) & 0xffu] ^ (s >> 8);
      s = s_tab[(s ^ (x >> 16)) & 0xffu] ^ (s >> 8);
      s = s_tab[(s ^ (x >> 24)) & 0xffu] ^ (s >> 8);
    }
    __syncwarp();
    // fold pairs: raw(A || B) = Z_|B|(raw(A)) ^ raw(B), |B| = 256 << j
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const uint32_t other = __shfl_down_sync(0xffffffffu, s, 1 << j);
      if ((lane & ((2 << j) - 1)) == 0) s = zmul(j, s) ^ other;
    }
    if (lane == 0) out[c] = s;
  }
}

// zlib.crc32 of body[0, len): device chunks + host fold and tail.  host_tail
// must hold the bytes [nchunks * kChunk, len) (the caller has them).
static uint32_t crc32_device(gcb_ctx *ctx, const uint8_t *body_dev, int64_t len,
                             const uint8_t *host_tail) {
  const HostCrc &hc = host_crc();
  const int64_t nchunks = len / kChunk;
  uint32_t s = 0xffffffffu;
  if (nchunks) {
    ensure_crc_constants(ctx);
    DArray<uint32_t> part(nchunks);
    const unsigned grid = grid_for(ceil_div(nchunks, kCrcWarps), 1, (int64_t)ctx->num_sms * 8);
    k_crc_chunks<<<grid, kCrcWarps * 32, 0, ctx->stream>>>(body_dev, nchunks, part.p);
    after_launch(ctx, "k_crc_chunks");
    std::vector<uint32_t> h(nchunks);
    d2h(ctx, h.data(), part.p, nchunks);
    sync(ctx);
    for (int64_t c = 0; c < nchunks; ++c) s = hc.shift_chunk(s) ^ h[c];
  }
  s = hc.bytes(s, host_tail, len - nchunks * kChunk);
  return s ^ 0xffffffffu;
}

// ---- layout ---------------------------------------------------------------
struct GcbLayout {
  int64_t body = 0;                 // bytes before the CRC
  std::vector<int64_t> blk;         // [B] offset of each block header
};

static GcbLayout layout_of(const std::vector<int64_t> &rs, const std::vector<int64_t> &es,
                           bool weighted) {
  GcbLayout L;
  const int64_t B = (int64_t)rs.size() - 1;
  L.blk.resize(B);
  int64_t at = kHeaderBytes;
  for (int64_t b = 0; b < B; ++b) {
    L.blk[b] = at;
    const int64_t nl = rs[b + 1] - rs[b], ne = es[b + 1] - es[b];
    at += 16 + 4 * nl + 8 * (nl + 1) + 4 * ne + (weighted ? 8 * ne : 0);
  }
  L.body = at;
  return L;
}

__device__ __forceinline__ int64_t block_of(const int64_t *__restrict__ starts, int64_t B,
                                            int64_t i) {
  int64_t lo = 0, hi = B;  // last b with starts[b] <= i
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (starts[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Section offsets of block b, derived from its header offset.
struct Sections {
  int64_t id, lro, col, w;
};
__device__ __forceinline__ Sections sections(int64_t boff, int64_t nl, int64_t ne) {
  Sections s;
  s.id = boff + 16;
  s.lro = s.id + 4 * nl;
  s.col = s.lro + 8 * (nl + 1);
  s.w = s.col + 4 * ne;
  return s;
}

// ---- pack (save) ----------------------------------------------------------
__global__ void k_pack_rows(int64_t B, const int64_t *__restrict__ rs, const int64_t *__restrict__ es,
                            const int64_t *__restrict__ boff, const uint32_t *__restrict__ id_map,
                            const uint32_t *__restrict__ lro, uint8_t *__restrict__ body) {
  const int64_t L = rs[B];
  // every arena row i (id_map) and every lro entry j of the L + B segment
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < L + B;
       j += (int64_t)gridDim.x * blockDim.x) {
    // lro entry j lies in block b's segment [rs[b] + b, rs[b + 1] + b + 1)
    int64_t lo = 0, hi = B;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rs[mid] + mid <= j) lo = mid;
      else hi = mid;
    }
    const int64_t b = lo, nl = rs[b + 1] - rs[b], ne = es[b + 1] - es[b];
    const Sections s = sections(boff[b], nl, ne);
    const int64_t k = j - (rs[b] + b);
    uint32_t *d = reinterpret_cast<uint32_t *>(body + s.lro + 8 * k);
    d[0] = lro[j];
    d[1] = 0u;
    if (k < nl) reinterpret_cast<uint32_t *>(body + s.id)[k] = id_map[rs[b] + k];
    if (k == 0) {
      uint32_t *h = reinterpret_cast<uint32_t *>(body + boff[b]);
      h[0] = (uint32_t)nl;
      h[1] = (uint32_t)((uint64_t)nl >> 32);
      h[2] = (uint32_t)ne;
      h[3] = (uint32_t)((uint64_t)ne >> 32);
    }
  }
}

__global__ void k_pack_edges(int64_t B, int64_t m, const int64_t *__restrict__ rs,
                             const int64_t *__restrict__ es, const int64_t *__restrict__ boff,
                             const uint32_t *__restrict__ col, const double *__restrict__ w,
                             uint8_t *__restrict__ body) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = block_of(es, B, e);
    const int64_t nl = rs[b + 1] - rs[b], ne = es[b + 1] - es[b], k = e - es[b];
    const Sections s = sections(boff[b], nl, ne);
    reinterpret_cast<uint32_t *>(body + s.col)[k] = col[e];
    if (w) {
      const unsigned long long x = __double_as_longlong(w[e]);
      uint32_t *d = reinterpret_cast<uint32_t *>(body + s.w + 8 * k);
      d[0] = (uint32_t)x;
      d[1] = (uint32_t)(x >> 32);
    }
  }
}

// ---- unpack (load) --------------------------------------------------------
__global__ void k_unpack_rows(int64_t B, const int64_t *__restrict__ rs, const int64_t *__restrict__ es,
                              const int64_t *__restrict__ boff, const uint8_t *__restrict__ body,
                              uint32_t *__restrict__ id_map, uint32_t *__restrict__ lro,
                              unsigned *__restrict__ bad) {
  const int64_t L = rs[B];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < L + B;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = B;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rs[mid] + mid <= j) lo = mid;
      else hi = mid;
    }
    const int64_t b = lo, nl = rs[b + 1] - rs[b], ne = es[b + 1] - es[b];
    const Sections s = sections(boff[b], nl, ne);
    const int64_t k = j - (rs[b] + b);
    const uint32_t *x = reinterpret_cast<const uint32_t *>(body + s.lro + 8 * k);
    if (x[1] != 0u) atomicOr(bad, 1u);  // offsets >= 2^32: not representable here
    lro[j] = x[0];
    if (k < nl) id_map[rs[b] + k] = reinterpret_cast<const uint32_t *>(body + s.id)[k];
  }
}

__global__ void k_unpack_edges(int64_t B, int64_t m, const int64_t *__restrict__ rs,
                               const int64_t *__restrict__ es, const int64_t *__restrict__ boff,
                               const uint8_t *__restrict__ body, uint32_t *__restrict__ col,
                               double *__restrict__ w) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = block_of(es, B, e);
    const int64_t nl = rs[b + 1] - rs[b], ne = es[b + 1] - es[b], k = e - es[b];
    const Sections s = sections(boff[b], nl, ne);
    col[e] = reinterpret_cast<const uint32_t *>(body + s.col)[k];
    if (w) {
      const uint32_t *x = reinterpret_cast<const uint32_t *>(body + s.w + 8 * k);
      w[e] = __longlong_as_double((long long)(((unsigned long long)x[1] << 32) | x[0]));
    }
  }
}

// ---- file streaming through two pinned buffers ------------------------------
struct FileCloser {
  FILE *f;
  ~FileCloser() {
    if (f) fclose(f);
  }
};

struct PinnedPair {
  void *p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  size_t bytes;
  explicit PinnedPair(size_t b) : bytes(b) {
    for (int i = 0; i < 2; ++i) {
      GCB_CUDA(cudaMallocHost(&p[i], bytes));
      GCB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~PinnedPair() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
};

constexpr size_t kStage = size_t(32) << 20;

[[noreturn]] static void io_fail(const char *what, const char *path) {
  const int e = errno;
  fail(GCB_EIO, "%s: %s (%s) [errno %d]", path, what, strerror(e), e);
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gcb_blocked_save(gcb_ctx *ctx, gcb_blocked *bg, const char *path) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && bg && path, "NULL argument");
  DeviceGuard dg(ctx->device);
  const int64_t B = bg->B;
  const GcbLayout lay = layout_of(bg->h_row_starts, bg->h_edge_starts, bg->weighted);
  const int64_t len = lay.body;
  DArray<uint8_t> body(len);
  {
    uint8_t hdr[kHeaderBytes] = {};
    std::memcpy(hdr, "GCB1", kMagicLen);
    hdr[4] = (uint8_t)bg->direction;
    hdr[5] = (uint8_t)((bg->weighted ? kFlagWeights : 0) | (bg->cb ? kFlagCb : 0));
    const uint64_t f[4] = {(uint64_t)bg->n, (uint64_t)bg->m, (uint64_t)bg->width, (uint64_t)B};
    std::memcpy(hdr + 8, f, sizeof(f));
    h2d(ctx, body.p, hdr, kHeaderBytes);
  }
  if (B) {
    DArray<int64_t> boff(B);
    h2d(ctx, boff.p, lay.blk.data(), B);
    k_pack_rows<<<grid_for(bg->L + B, 256, 65536), 256, 0, ctx->stream>>>(
        B, bg->row_starts.p, bg->edge_starts.p, boff.p, bg->id_map.p, bg->lro.p, body.p);
    after_launch(ctx, "k_pack_rows");
    if (bg->m) {
      k_pack_edges<<<grid_for(bg->m, 256, 65536), 256, 0, ctx->stream>>>(
          B, bg->m, bg->row_starts.p, bg->edge_starts.p, boff.p, bg->col.p,
          bg->weighted ? bg->w.p : nullptr, body.p);
      after_launch(ctx, "k_pack_edges");
    }
    sync(ctx);  // boff is released at scope end
  }
  FILE *f = fopen(path, "wb");
  if (!f) io_fail("cannot open for writing", path);
  FileCloser fc{f};
  // stream the body out, the D2H of the next chunk overlapping this write;
  // the CRC runs on the device first and needs only the tail on the host
  const int64_t tail_at = (len / kChunk) * kChunk;
  std::vector<uint8_t> tail(len - tail_at);
  if (!tail.empty()) d2h(ctx, tail.data(), body.p + tail_at, (int64_t)tail.size());
  const uint32_t crc = crc32_device(ctx, body.p, len, tail.data());
  PinnedPair pp(kStage);
  const int64_t nst = ceil_div(len, (int64_t)kStage);
  auto issue = [&](int64_t i) {
    const int64_t off = i * (int64_t)kStage, cnt = len - off < (int64_t)kStage ? len - off : kStage;
    GCB_CUDA(cudaMemcpyAsync(pp.p[i & 1], body.p + off, cnt, cudaMemcpyDeviceToHost, ctx->stream));
    GCB_CUDA(cudaEventRecord(pp.ev[i & 1], ctx->stream));
  };
  if (nst) issue(0);
  for (int64_t i = 0; i < nst; ++i) {
    if (i + 1 < nst) issue(i + 1);
    GCB_CUDA(cudaEventSynchronize(pp.ev[i & 1]));
    const int64_t off = i * (int64_t)kStage, cnt = len - off < (int64_t)kStage ? len - off : kStage;
    if (fwrite(pp.p[i & 1], 1, (size_t)cnt, f) != (size_t)cnt) io_fail("write failed", path);
  }
  const uint8_t c4[4] = {(uint8_t)crc, (uint8_t)(crc >> 8), (uint8_t)(crc >> 16),
                         (uint8_t)(crc >> 24)};
  if (fwrite(c4, 1, 4, f) != 4) io_fail("write failed", path);
  if (fflush(f) != 0) io_fail("write failed", path);
  GCB_API_END
}

int gcb_blocked_load(gcb_ctx *ctx, const char *path, gcb_blocked **out) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && path && out, "NULL argument");
  DeviceGuard dg(ctx->device);
  FILE *f = fopen(path, "rb");
  if (!f) io_fail("cannot open", path);
  FileCloser fc{f};
  if (fseeko(f, 0, SEEK_END) != 0) io_fail("seek failed", path);
  const int64_t size = (int64_t)ftello(f);
  if (size < kHeaderBytes + 4) fail(GCB_EFORMAT, "%s: truncated container", path);
  const int64_t len = size - 4;
  // stream the body into the device, H2D of chunk k overlapping the read of k+1
  DArray<uint8_t> body(len);
  const int64_t tail_at = (len / kChunk) * kChunk;
  std::vector<uint8_t> tail(len - tail_at);
  uint8_t c4[4];
  {
    if (fseeko(f, 0, SEEK_SET) != 0) io_fail("seek failed", path);
    PinnedPair pp(kStage);
    const int64_t nst = ceil_div(len, (int64_t)kStage);
    for (int64_t i = 0; i < nst; ++i) {
      const int64_t off = i * (int64_t)kStage;
      const int64_t cnt = len - off < (int64_t)kStage ? len - off : (int64_t)kStage;
      GCB_CUDA(cudaEventSynchronize(pp.ev[i & 1]));  // buffer free again
      uint8_t *hb = (uint8_t *)pp.p[i & 1];
      if (fread(hb, 1, (size_t)cnt, f) != (size_t)cnt) io_fail("read failed", path);
      // the tail bytes of the CRC are folded on the host
      const int64_t lo = off > tail_at ? off : tail_at, hi = off + cnt;
      if (hi > lo) std::memcpy(tail.data() + (lo - tail_at), hb + (lo - off), (size_t)(hi - lo));
      GCB_CUDA(cudaMemcpyAsync(body.p + off, hb, (size_t)cnt, cudaMemcpyHostToDevice, ctx->stream));
      GCB_CUDA(cudaEventRecord(pp.ev[i & 1], ctx->stream));
    }
    if (fread(c4, 1, 4, f) != 4) io_fail("read failed", path);
  }
  const uint32_t stored = (uint32_t)c4[0] | ((uint32_t)c4[1] << 8) | ((uint32_t)c4[2] << 16) |
                          ((uint32_t)c4[3] << 24);
  if (crc32_device(ctx, body.p, len, tail.data()) != stored)
    fail(GCB_EFORMAT, "%s: CRC mismatch, file is corrupt", path);
  // header and block table, walked on the host (blocking.py:376-420 checks)
  auto pread_at = [&](int64_t at, void *dst, size_t cnt) {
    if (fseeko(f, at, SEEK_SET) != 0 || fread(dst, 1, cnt, f) != cnt) io_fail("read failed", path);
  };
  uint8_t hdr[kHeaderBytes];
  pread_at(0, hdr, kHeaderBytes);
  if (std::memcmp(hdr, "GCB1", kMagicLen) != 0) {
    char m4[32];
    snprintf(m4, sizeof(m4), "b'%c%c%c%c'", hdr[0], hdr[1], hdr[2], hdr[3]);
    fail(GCB_EFORMAT, "%s: bad magic %s", path, m4);
  }
  if (hdr[4] > 1) fail(GCB_EFORMAT, "%s: bad direction byte %d", path, (int)hdr[4]);
  uint64_t hf[4];
  std::memcpy(hf, hdr + 8, sizeof(hf));
  const int64_t n = (int64_t)hf[0], m = (int64_t)hf[1], width = (int64_t)hf[2], B = (int64_t)hf[3];
  const bool weighted = hdr[5] & kFlagWeights, cb = hdr[5] & kFlagCb;
  GCB_REQUIRE(n >= 0 && m >= 0 && width >= 1 && B >= 0 && B <= len / 16, "%s: bad header", path);
  std::vector<int64_t> rs(B + 1, 0), es(B + 1, 0), boff(B);
  int64_t at = kHeaderBytes;
  for (int64_t b = 0; b < B; ++b) {
    if (at + 16 > len) fail(GCB_EFORMAT, "%s: truncated block table", path);
    uint64_t ne2[2];
    pread_at(at, ne2, 16);
    boff[b] = at;
    const int64_t nl = (int64_t)ne2[0], ne = (int64_t)ne2[1];
    const int64_t sec = 4 * nl + 8 * (nl + 1) + 4 * ne + (weighted ? 8 * ne : 0);
    if (nl < 0 || ne < 0 || nl > len || ne > len || at + 16 + sec > len)
      fail(GCB_EFORMAT, "%s: truncated block table", path);
    uint64_t last;
    pread_at(at + 16 + 4 * nl + 8 * nl, &last, 8);
    if ((uint64_t)ne != last) fail(GCB_EFORMAT, "%s: block %lld edge count disagrees", path, (long long)b);
    rs[b + 1] = rs[b] + nl;
    es[b + 1] = es[b] + ne;
    at += 16 + sec;
  }
  if (at != len) fail(GCB_EFORMAT, "%s: trailing bytes after last block", path);
  if (es[B] != m) fail(GCB_EFORMAT, "%s: total edges disagree with header", path);
  for (int64_t b = 0; b < B; ++b)
    GCB_REQUIRE(es[b + 1] - es[b] < (int64_t(1) << 32), "block %lld has >= 2^32 edges", (long long)b);
  auto bg = new gcb_blocked();
  try {
    const int64_t L = rs[B];
    bg->device = ctx->device;
    bg->direction = hdr[4];
    bg->width = width;
    bg->n = n;
    bg->m = m;
    bg->B = B;
    bg->L = L;
    bg->weighted = weighted;
    bg->h_row_starts = rs;
    bg->h_edge_starts = es;
    bg->row_starts.alloc(B + 1);
    bg->edge_starts.alloc(B + 1);
    bg->lro.alloc(L + B + 1);
    bg->id_map.alloc(L);
    bg->col.alloc(m + kColPad);
    GCB_CUDA(cudaMemsetAsync(bg->col.p + m, 0, kColPad * sizeof(uint32_t), ctx->stream));
    if (weighted) bg->w.alloc(m + kColPad);
    h2d(ctx, bg->row_starts.p, rs.data(), B + 1);
    h2d(ctx, bg->edge_starts.p, es.data(), B + 1);
    if (B) {
      DArray<int64_t> dboff(B);
      DArray<unsigned> bad(1);
      GCB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned), ctx->stream));
      h2d(ctx, dboff.p, boff.data(), B);
      k_unpack_rows<<<grid_for(L + B, 256, 65536), 256, 0, ctx->stream>>>(
          B, bg->row_starts.p, bg->edge_starts.p, dboff.p, body.p, bg->id_map.p, bg->lro.p, bad.p);
      after_launch(ctx, "k_unpack_rows");
      if (m) {
        k_unpack_edges<<<grid_for(m, 256, 65536), 256, 0, ctx->stream>>>(
            B, m, bg->row_starts.p, bg->edge_starts.p, dboff.p, body.p, bg->col.p,
            weighted ? bg->w.p : nullptr);
        after_launch(ctx, "k_unpack_edges");
      }
      unsigned hbad = 0;
      d2h(ctx, &hbad, bad.p, 1);
      sync(ctx);
      GCB_REQUIRE(hbad == 0, "local row offset out of the 32-bit range");
    }
    if (cb) {
      GCB_REQUIRE(bg->direction == 0, "the cb scheme is pull-only");
      for (int64_t b = 0; b <= B; ++b)
        GCB_REQUIRE(rs[b] == b * n, "cb blocks must hold all n rows");
      bg->cb = true;
    }
    sync(ctx);
  } catch (...) {
    delete bg;
    throw;
  }
  *out = bg;
  GCB_API_END
}

int gcb_blocked_scheme(const gcb_blocked *bg, int *is_cb) {
  GCB_API_BEGIN
  GCB_REQUIRE(bg && is_cb, "NULL argument");
  *is_cb = bg->cb ? 1 : 0;
  GCB_API_END
}

int gcb_crc32(gcb_ctx *ctx, const void *data_host, int64_t len, uint32_t *crc) {
  GCB_API_BEGIN
  GCB_REQUIRE(ctx && crc && (data_host || len == 0) && len >= 0, "NULL argument");
  DeviceGuard dg(ctx->device);
  DArray<uint8_t> d(len ? len : 1);
  if (len) h2d(ctx, d.p, (const uint8_t *)data_host, len);
  const int64_t tail_at = (len / kChunk) * kChunk;
  *crc = crc32_device(ctx, d.p, len, (const uint8_t *)data_host + tail_at);
  GCB_API_END
}

}  // extern "C"

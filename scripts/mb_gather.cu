// mb_gather.cu -- microbenchmark: random 8-byte gathers from an L2-resident
// vector on B200, via (a) LDG (L1TEX path) and (b) TMA tile::gather4 (TMA
// unit -> smem, bypassing the LSU/L1TEX tag stage).  Decides how the TOCAB
// gather fetches cold source values.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o mb_gather mb_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void k_fill_idx(uint32_t *idx, int64_t M, uint32_t N, uint64_t seed, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    uint32_t v = (uint32_t)(x % N);
    if (mode == 1) {  // power-law-ish: square of a uniform in [0,1)
      double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      v = (uint32_t)(u * u * u * N);
      if (v >= N) v = N - 1;
    }
    idx[i] = v;
  }
}

template <typename T>
__global__ void k_fill_vals(T *v, int64_t N) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (T)(i & 1023) * (T)0.5;
}

// (a) LDG: 8 gathers in flight per thread (idx as 2x uint4 per thread-iteration)
template <typename T, bool NA>
__global__ void __launch_bounds__(1024, 1) k_ldg(const T *__restrict__ vals, const uint32_t *__restrict__ idx,
                                                 int64_t M, double *__restrict__ out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; b < M; b += stride) {
    uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + b));
    uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + b) + 1);
    uint32_t ii[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (NA) {
        if (sizeof(T) == 8) {
          double d;
          asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(d) : "l"(vals + ii[k]));
          x[k] = (T)d;
        } else {
          float f;
          asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(f) : "l"(vals + ii[k]));
          x[k] = (T)f;
        }
      } else {
        x[k] = __ldg(vals + ii[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += (double)x[k];
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (a2) LDG with S bytes of (unused) dynamic smem: L1 capacity vs throughput
template <typename T>
__global__ void __launch_bounds__(1024, 1) k_ldg_sm(const T *__restrict__ vals, const uint32_t *__restrict__ idx,
                                                    int64_t M, double *__restrict__ out) {
  extern __shared__ double dummy[];
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; b < M; b += stride) {
    uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + b));
    uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + b) + 1);
    uint32_t ii[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    T x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ldg(vals + ii[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += (double)x[k];
  }
  if (acc == -1.0) dummy[threadIdx.x] = acc;
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// (a3) LDGSTS (cp.async 8B) into a per-thread smem ring of D stages x 8 values
template <int D, bool CG>
__global__ void __launch_bounds__(512, 1) k_ldgsts(const double *__restrict__ vals, const uint32_t *__restrict__ idx,
                                                   int64_t M, double *__restrict__ out) {
  extern __shared__ double ring[];  // [D][8][blockDim]
  const int T = blockDim.x, tid = threadIdx.x;
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * T * 8;
  int64_t b = ((int64_t)blockIdx.x * T + tid) * 8;
  // prologue
  uint32_t ii[D][8];
#pragma unroll
  for (int s = 0; s < D; ++s) {
    const int64_t bb = b + s * stride;
    if (bb < M) {
      uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + bb));
      uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + bb) + 1);
      uint32_t t8[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(ring + ((s * 8 + k) * T + tid));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(vals + t8[k]));
      }
    }
    asm volatile("cp.async.commit_group;");
  }
  int s = 0;
  for (; b < M; b += stride) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1));
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += ring[(s * 8 + k) * T + tid];
    const int64_t bb = b + (int64_t)D * stride;
    if (bb < M) {
      uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + bb));
      uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + bb) + 1);
      uint32_t t8[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(ring + ((s * 8 + k) * T + tid));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(vals + t8[k]));
      }
    }
    asm volatile("cp.async.commit_group;");
    if (++s == D) s = 0;
  }
  asm volatile("cp.async.wait_all;");
  out[(int64_t)blockIdx.x * T + tid] = acc;
}

// (b) TMA gather4.  Tensor: [N/2 rows][2 f64] (16-byte rows).  Each warp owns
// a ring of D stages; a stage = 128 edges = 32 gather4 (one per lane) = 2 KB.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity));
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <int D, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    k_tma(const __grid_constant__ CUtensorMap map, const uint32_t *__restrict__ idx, int64_t M,
          double *__restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char *ring = smem + (size_t)wid * D * 4096;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)WARPS * D * 4096) + wid * D;
  if (lane == 0)
    for (int s = 0; s < D; ++s) mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t nchunks = M / 128;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + wid, nw = (int64_t)gridDim.x * WARPS;
  double acc = 0;
  // prologue: issue D chunks
  int64_t issue = gw;
  uint4 pend[D];
#pragma unroll
  for (int s = 0; s < D; ++s) {
    if (issue < nchunks) {
      uint4 q = __ldcs(reinterpret_cast<const uint4 *>(idx + issue * 128) + lane);
      pend[s] = q;
      if (lane == 0) mbar_expect_tx(bars + s, 4096);
      __syncwarp();
      tma_gather4(ring + s * 4096 + lane * 128, &map, bars + s, 0, q.x >> 2, q.y >> 2, q.z >> 2,
                  q.w >> 2);
    }
    issue += nw;
  }
  uint32_t phase = 0;
  int64_t c = gw;
  for (int s = 0; c < nchunks; c += nw) {
    mbar_wait(bars + s, phase);
    const uint4 q = pend[s];
    const double *row = reinterpret_cast<const double *>(ring + s * 4096 + lane * 128);
    acc += row[0 + (q.x & 3)] + row[4 + (q.y & 3)] + row[8 + (q.z & 3)] + row[12 + (q.w & 3)];
    __syncwarp();
    const int64_t nx = c + (int64_t)D * nw;
    if (nx < nchunks) {
      uint4 q2 = __ldcs(reinterpret_cast<const uint4 *>(idx + nx * 128) + lane);
      pend[s] = q2;
      if (lane == 0) mbar_expect_tx(bars + s, 4096);
      __syncwarp();
      tma_gather4(ring + s * 4096 + lane * 128, &map, bars + s, 0, q2.x >> 2, q2.y >> 2, q2.z >> 2,
                  q2.w >> 2);
    }
    if (++s == D) {
      s = 0;
      phase ^= 1;
    }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char **argv) {
  const uint32_t N = argc > 1 ? atoi(argv[1]) : (8u << 20);  // vertices (f64)
  const int64_t M = argc > 2 ? atoll(argv[2]) : (int64_t(128) << 20);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *vals;
  float *vals32;
  uint32_t *idx;
  double *out;
  CK(cudaMalloc(&vals, (size_t)N * 8));
  CK(cudaMalloc(&vals32, (size_t)N * 4));
  CK(cudaMalloc(&idx, (size_t)M * 4));
  CK(cudaMalloc(&out, (size_t)sms * 4096 * 8));
  k_fill_vals<double><<<1024, 256>>>(vals, N);
  k_fill_vals<float><<<1024, 256>>>(vals32, N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int R = 5;
    for (int r = 0; r < R; ++r) launch();
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-34s %8.3f ms  %7.1f Ggathers/s  (%.2f per SM-cycle @1.965GHz)\n", name, ms,
           M / ms / 1e6, M / (ms * 1e-3) / (sms * 1.965e9));
  };
  // TMA map: [N/2][2] f64
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &qr));
  CUtensorMap map;
  cuuint64_t dims[2] = {4, N / 4};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, vals, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)cr);
  for (int mode = 0; mode < 2; ++mode) {
    k_fill_idx<<<4096, 256>>>(idx, M, N, 12345, mode);
    CK(cudaDeviceSynchronize());
    printf("--- N=%u (%u MB f64) M=%lld idx %s\n", N, N / 131072, (long long)M,
           mode ? "power-law (u^3)" : "uniform");
    timeit("ldg f64", [&] { k_ldg<double, false><<<sms, 1024>>>(vals, idx, M, out); });
    timeit("ldg f64 no_allocate", [&] { k_ldg<double, true><<<sms, 1024>>>(vals, idx, M, out); });
    timeit("ldg f32", [&] { k_ldg<float, false><<<sms, 1024>>>(vals32, idx, M, out); });
    for (int S : {0, 65536, 131072, 196608, 225280}) {
      char nm[64];
      snprintf(nm, 64, "ldg f64 smem %dK", S / 1024);
      CK(cudaFuncSetAttribute(k_ldg_sm<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, S));
      timeit(nm, [&] { k_ldg_sm<double><<<sms, 1024, S>>>(vals, idx, M, out); });
    }
    {
      constexpr int D = 4;
      size_t S = (size_t)D * 8 * 512 * 8;
      CK(cudaFuncSetAttribute(k_ldgsts<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S));
      timeit("ldgsts 8B D4 512thr (128K ring)", [&] { k_ldgsts<D, false><<<sms, 512, S>>>(vals, idx, M, out); });
    }
    {
      constexpr int D = 6;
      size_t S = (size_t)D * 8 * 512 * 8;
      CK(cudaFuncSetAttribute(k_ldgsts<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S));
      timeit("ldgsts 8B D6 512thr (192K ring)", [&] { k_ldgsts<D, false><<<sms, 512, S>>>(vals, idx, M, out); });
    }
    {
      constexpr int D = 2;
      size_t S = (size_t)D * 8 * 512 * 8;
      CK(cudaFuncSetAttribute(k_ldgsts<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S));
      timeit("ldgsts 8B D2 512thr (64K ring)", [&] { k_ldgsts<D, false><<<sms, 512, S>>>(vals, idx, M, out); });
    }
    timeit("ldg f64 2cta/sm 512thr", [&] { k_ldg<double, false><<<sms * 2, 512>>>(vals, idx, M, out); });
  }
  // streaming reference: idx read only
  return 0;
}

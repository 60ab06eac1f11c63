// mb_mixed.cu -- microbenchmark: does a second on-chip tier in a cluster
// peer's shared memory (DSMEM) add gather throughput beside the random L2
// gathers of the TOCAB pull, or does it share their request path?
// Each lane issues 8 random 8-byte loads per step; a fraction p of them go to
// the peer CTA's 124 KB table over DSMEM (ld.shared::cluster), a fraction q
// to the CTA's own table (LDS), the rest to a 64 MB L2-resident vector
// (LDG, evict_last, no L1 allocation) -- the pull kernel's three tiers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mixed mb_mixed.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

// idx: bit 31 = DSMEM (peer table slot), bit 30 = own table slot, else vector index
__global__ void k_fill(uint32_t *idx, int64_t M, uint32_t N, uint32_t T, uint32_t p256,
                       uint32_t q256, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    const uint32_t sel = (uint32_t)(x >> 56);
    const uint32_t r = (uint32_t)(x & 0xffffffffu);
    if (sel < p256) idx[i] = 0x80000000u | (r % T);
    else if (sel < p256 + q256) idx[i] = 0x40000000u | (r % T);
    else idx[i] = r % N;
  }
}

template <int CL>
__global__ void __launch_bounds__(1024, 1)
    k_mixed(const uint32_t *__restrict__ idx, int64_t M, int T, const double *__restrict__ vec,
            double *__restrict__ out) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < T; i += blockDim.x) tab[i] = (double)(i & 255) + blockIdx.x;
  cg::cluster_group cl = cg::this_cluster();
  if (CL > 1) cl.sync(); else __syncthreads();
  const double *peer = CL > 1 ? cl.map_shared_rank(tab, (cl.block_rank() + 1) % CL) : tab;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; b < M; b += stride) {
    uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + b));
    uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + b) + 1);
    uint32_t ii[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t v = ii[k];
      if (v & 0x80000000u) x[k] = peer[v & 0x3fffffffu];
      else if (v & 0x40000000u) x[k] = tab[v & 0x3fffffffu];
      else
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(x[k]) : "l"(vec + v), "l"(pol));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += x[k];
  }
  if (CL > 1) cl.sync();
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t M = int64_t(256) << 20;
  const uint32_t N = 8u << 20;  // 64 MB of f64: L2-resident
  const int T = 15872;          // 124 KB table per CTA
  uint32_t *idx;
  double *out, *vec;
  CK(cudaMalloc(&idx, M * 4));
  CK(cudaMalloc(&vec, (size_t)N * 8));
  CK(cudaMemset(vec, 0, (size_t)N * 8));
  CK(cudaMalloc(&out, (size_t)sms * 1024 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto kern, int cl, double p, double q) {
    const int grid = (sms / cl) * cl;
    size_t sm = (size_t)T * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 55));
    k_fill<<<4096, 256>>>(idx, M, N, T, (uint32_t)(p * 256), (uint32_t)(q * 256), 7);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)idx, M, T, (const double *)vec, out));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r)
      CK(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)idx, M, T, (const double *)vec, out));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double per = M / (ms * 1e-3) / (grid * 1.965e9);
    const double l2 = per * (1.0 - p - q);
    printf("%-34s p_dsmem %.3f q_lds %.3f  %8.3f ms  all %.3f  L2-part %.3f  per SM-cycle\n", name,
           p, q, ms, per, l2);
  };
  run("L2 only", k_mixed<1>, 1, 0.0, 0.0);
  run("L2 + own table 30%", k_mixed<1>, 1, 0.0, 0.30);
  run("L2 + own 30% (cluster 2 launch)", k_mixed<2>, 2, 0.0, 0.30);
  for (double p : {0.0625, 0.125, 0.25, 0.5})
    run("L2 + own 30% + peer DSMEM", k_mixed<2>, 2, p, 0.30);
  for (double p : {0.125, 0.25})
    run("L2 + peer DSMEM (no own)", k_mixed<2>, 2, p, 0.0);
  return 0;
}

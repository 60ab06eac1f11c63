// mb_smem.cu -- microbenchmark: random 8-byte gathers from (a) the CTA's own
// shared memory and (b) distributed shared memory across a thread-block
// cluster (DSMEM), to size the on-chip tiers of the TOCAB gather.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_smem mb_smem.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void k_fill_idx(uint32_t *idx, int64_t M, uint32_t N, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    idx[i] = (uint32_t)(x % N);
  }
}

// T entries per CTA table; idx in [0, CL*T); CL = cluster size (1 = local only)
template <int CL>
__global__ void __launch_bounds__(1024, 1) k_gather_sm(const uint32_t *__restrict__ idx, int64_t M, int T,
                                                       double *__restrict__ out) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < T; i += blockDim.x) tab[i] = (double)(i & 255) + blockIdx.x;
  cg::cluster_group cl = cg::this_cluster();
  if (CL > 1) cl.sync(); else __syncthreads();
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; b < M; b += stride) {
    uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + b));
    uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + b) + 1);
    uint32_t ii[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (CL > 1) {
        const uint32_t r = ii[k] / T, o = ii[k] - r * T;
        const double *p = cl.map_shared_rank(tab, r);
        x[k] = p[o];
      } else {
        x[k] = tab[ii[k]];
      }
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
  const int64_t M = int64_t(128) << 20;
  uint32_t *idx;
  double *out;
  CK(cudaMalloc(&idx, M * 4));
  CK(cudaMalloc(&out, (size_t)sms * 2 * 1024 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int T = 24576;  // 192 KB per CTA
  auto run = [&](const char *name, auto kern, int cl, int grid) {
    size_t sm = (size_t)T * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_fill_idx<<<4096, 256>>>(idx, M, (uint32_t)T * cl, 7);
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
    CK(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)idx, M, T, out));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) CK(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)idx, M, T, out));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-28s grid %4d  %8.3f ms  %7.1f Ggathers/s (%.2f per SM-cycle @1.965GHz)\n", name, grid, ms,
           M / ms / 1e6, M / (ms * 1e-3) / (grid * 1.965e9));
  };
  run("local smem (cluster 1)", k_gather_sm<1>, 1, sms);
  run("dsmem cluster 2", k_gather_sm<2>, 2, (sms / 2) * 2);
  run("dsmem cluster 4", k_gather_sm<4>, 4, 128);
  run("dsmem cluster 8", k_gather_sm<8>, 8, 128);
  return 0;
}

// mb_atoms.cu -- microbenchmark: shared-memory atomic adds into a 20480-slot
// table (the hybrid hub pass's accumulator, pr.cu k_push_hub) at random slots,
// to tell whether that pass is bound by its shared atomics:
//   u32    one 32-bit ATOMS.ADD per add
//   fix64  the two-word 64-bit fixed point of fix_add (low add + carry-in high add)
//   f64    atomicAdd(double) on shared memory (a CAS loop on sm_100)
//   fix64_skewed  fix64 with a power-law slot distribution (rmat hubs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_atoms mb_atoms.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void k_fill_idx(uint32_t *idx, int64_t M, uint32_t N, uint64_t seed, int skew) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    if (skew) {  // ~ Zipf: slot = N * u^3
      const double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      idx[i] = (uint32_t)(N * u * u * u) % N;
    } else {
      idx[i] = (uint32_t)(x % N);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_atoms(const uint32_t *__restrict__ idx, int64_t M, int T,
                                                   unsigned long long *__restrict__ out) {
  extern __shared__ unsigned smem[];
  unsigned *lo = smem, *hi = smem + T;
  double *tf = reinterpret_cast<double *>(smem);
  for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; b < M; b += stride) {
    uint4 a = __ldcs(reinterpret_cast<const uint4 *>(idx + b));
    uint4 c = __ldcs(reinterpret_cast<const uint4 *>(idx + b) + 1);
    uint32_t ii[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const unsigned long long add = 0x0000000A12345678ull + ii[k];
      if (MODE == 0) {
        atomicAdd(lo + ii[k], (unsigned)add);
      } else if (MODE == 1) {
        const unsigned alo = (unsigned)add, ahi = (unsigned)(add >> 32);
        const unsigned old = atomicAdd(lo + ii[k], alo);
        const unsigned carry = (old + alo < old) ? 1u : 0u;
        if (ahi + carry) atomicAdd(hi + ii[k], ahi + carry);
      } else {
        atomicAdd(tf + ii[k], 1e-8 * (double)ii[k]);
      }
    }
  }
  __syncthreads();
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < T; i += blockDim.x) s += lo[i] + hi[i];
  atomicAdd(out, s);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const int T = 20480;
  const int64_t M = int64_t(1) << 28;
  uint32_t *idx;
  unsigned long long *out;
  CK(cudaMalloc(&idx, M * 4));
  CK(cudaMalloc(&out, 8));
  const size_t smem = (size_t)T * 8;
  CK(cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char *names[3] = {"u32", "fix64", "f64"};
  for (int skew = 0; skew < 2; ++skew) {
    k_fill_idx<<<4096, 256>>>(idx, M, T, 12345, skew);
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        CK(cudaEventRecord(e0));
        if (mode == 0) k_atoms<0><<<sms, 1024, smem>>>(idx, M, T, out);
        if (mode == 1) k_atoms<1><<<sms, 1024, smem>>>(idx, M, T, out);
        if (mode == 2) k_atoms<2><<<sms, 1024, smem>>>(idx, M, T, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r && ms < best) best = ms;
      }
      const double per = (double)M / (best * 1e-3) / sms / (clk * 1e3);
      printf("%-6s %-7s %8.3f ms  %.3f adds per SM-cycle (%d SMs, %.0f MHz)\n", names[mode],
             skew ? "skewed" : "uniform", best, per, sms, clk / 1e3);
    }
  }
  return 0;
}

// mb_dadd.cu -- microbenchmark: latency of a dependent f64 add chain on B200
// (the critical path of exact-mode hub rows), with the addend from a register,
// from shared memory (LDS) and from a warp shuffle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dadd mb_dadd.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_chain(int n, const double *in, double *out, long long *cyc, int mode) {
  __shared__ double s[256];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = in[i];
  __syncwarp();
  double acc = 0.0, x = in[lane];
  const long long t0 = clock64();
  if (mode == 0) {
    const double a = in[1];
    for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, a);
  } else if (mode == 1) {
    for (int k = 0; k < n; k += 256)
#pragma unroll 64
      for (int j = 0; j < 256; ++j) acc = __dadd_rn(acc, s[j]);
  } else {
    for (int k = 0; k < n; k += 32)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, x, j));
  }
  const long long t1 = clock64();
  if (lane == 0) {
    out[0] = acc;
    cyc[mode] = t1 - t0;
  }
}

// throughput: every warp runs its own dependent chain (all 32 lanes, as the
// exact long-row kernel does); reports warp-level DADDs per SM-cycle
__global__ void k_tput(int n, const double *in, double *out) {
  double acc = 0.0;
  const double a = in[threadIdx.x & 255];
  for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, a);
  if (acc == 12345.0) out[0] = acc;
}

// the same, but only lane 0 of each warp runs the chain (the other lanes idle)
__global__ void k_tput_lane0(int n, const double *in, double *out) {
  if ((threadIdx.x & 31) != 0) return;
  double acc = 0.0;
  const double a = in[threadIdx.x & 255];
  for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, a);
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  double *in, *out;
  long long *cyc;
  cudaMalloc(&in, 256 * 8);
  cudaMalloc(&out, 8);
  cudaMallocManaged(&cyc, 3 * 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1e-3 * (i + 1);
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 1 << 20;
  const char *names[3] = {"register", "shared (LDS)", "shuffle"};
  for (int mode = 0; mode < 3; ++mode) {
    k_chain<<<1, 32>>>(n, in, out, cyc, mode);
    k_chain<<<1, 32>>>(n, in, out, cyc, mode);
    cudaDeviceSynchronize();
    printf("dependent DADD chain, addend from %-13s: %.2f cycles per add\n", names[mode],
           (double)cyc[mode] / n);
  }
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int m = 1 << 16;
  for (int wps : {4, 8, 16, 32, 64}) {  // warps per SM
    const int ctas = sms * (wps / 4);
    k_tput<<<ctas, 128>>>(m, in, out);
    cudaEventRecord(e0);
    k_tput<<<ctas, 128>>>(m, in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%2d chaining warps per SM: %.3f warp-DADD per SM-cycle (%.1f cycles per add per warp)\n",
           wps, (double)m * wps / cycles, cycles / m);
    k_tput_lane0<<<ctas, 128>>>(m, in, out);
    cudaEventRecord(e0);
    k_tput_lane0<<<ctas, 128>>>(m, in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double c2 = ms * 1e-3 * clk * 1e3;
    printf("   lane 0 only:            %.3f warp-DADD per SM-cycle (%.1f cycles per add per warp)\n",
           (double)m * wps / c2, c2 / m);
  }
  return 0;
}

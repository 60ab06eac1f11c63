// mb_stream.cu -- microbenchmark: streaming bandwidth of the PageRank update's
// access shape (R read streams + W write streams of f64, 16M elements) on
// B200, to separate the HBM limit from kernel structure.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_stream mb_stream.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int R, int W>
__global__ void __launch_bounds__(512) k_stream(int64_t n4, double **in, double **out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double a, b, c, d;
      asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                   : "l"(in[r] + 4 * i));
      acc[0] += a; acc[1] += b; acc[2] += c; acc[3] += d;
    }
#pragma unroll
    for (int w = 0; w < W; ++w)
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(out[w] + 4 * i), "d"(acc[0]),
                   "d"(acc[1]), "d"(acc[2]), "d"(acc[3])
                   : "memory");
  }
}

// the PageRank update shape: sums, ranks, deg(u32) in; ranks, sums(0), contrib out
template <int MATH>
__global__ void __launch_bounds__(512) k_upd(int64_t n4, double *sums, double *ranks,
                                             const uint32_t *deg, double *contrib, double *deltas) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double dsum = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double s[4], o[4], nr[4], c[4];
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(s[0]), "=d"(s[1]), "=d"(s[2]), "=d"(s[3]) : "l"(sums + 4 * i));
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(ranks + 4 * i));
    uint4 d = __ldcs(reinterpret_cast<const uint4 *>(deg) + i);
    uint32_t dg[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (MATH == 0) {
        nr[k] = s[k] + o[k];
        c[k] = nr[k] + dg[k];
      } else {
        nr[k] = __dadd_rn(0.15 / 16777216.0, __dmul_rn(0.85, s[k]));
        dsum += fabs(nr[k] - o[k]);
        if (MATH == 1) {
          double q = (double)__frcp_rn((float)dg[k]);
          const double dd = (double)dg[k];
          q = fma(fma(-dd, q, 1.0), q, q);
          q = fma(fma(-dd, q, 1.0), q, q);
          c[k] = dg[k] ? nr[k] * q : 0.0;
        } else {
          c[k] = dg[k] ? __ddiv_rn(nr[k], (double)dg[k]) : 0.0;
        }
      }
    }
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(ranks + 4 * i), "d"(nr[0]), "d"(nr[1]), "d"(nr[2]), "d"(nr[3]) : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(sums + 4 * i), "d"(0.0), "d"(0.0), "d"(0.0), "d"(0.0) : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(contrib + 4 * i), "d"(c[0]), "d"(c[1]), "d"(c[2]), "d"(c[3]) : "memory");
  }
  if (dsum == 12345.0) deltas[0] = dsum;
}

int main() {
  const int64_t n = int64_t(1) << 24;
  double *buf[6];
  for (auto &b : buf) cudaMalloc(&b, n * 8);
  double **din, **dout;
  cudaMalloc(&din, 3 * sizeof(double *));
  cudaMalloc(&dout, 3 * sizeof(double *));
  cudaMemcpy(din, buf, 3 * sizeof(double *), cudaMemcpyHostToDevice);
  cudaMemcpy(dout, buf + 3, 3 * sizeof(double *), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto kern, int R, int W, int grid) {
    kern<<<grid, 512>>>(n / 4, din, dout);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) kern<<<grid, 512>>>(n / 4, din, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    double bytes = (double)(R + W) * n * 8;
    printf("%-10s grid %6d  %8.1f us  %7.1f GB/s\n", name, grid, ms * 1e3, bytes / ms / 1e6);
  };
  for (int g : {sms * 2, sms * 4, sms * 8, (int)(n / 4 / 512)}) {
    run("1R1W", k_stream<1, 1>, 1, 1, g);
    run("2R2W", k_stream<2, 2>, 2, 2, g);
    run("3R3W", k_stream<3, 3>, 3, 3, g);
    run("2R3W", k_stream<2, 3>, 2, 3, g);
  }
  uint32_t *deg;
  cudaMalloc(&deg, n * 4);
  cudaMemset(deg, 1, n * 4);
  auto runu = [&](const char *name, auto kern, int grid) {
    kern<<<grid, 512>>>(n / 4, buf[0], buf[1], deg, buf[2], buf[3]);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) kern<<<grid, 512>>>(n / 4, buf[0], buf[1], deg, buf[2], buf[3]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-22s grid %6d  %8.1f us  %7.1f GB/s (44 B/vertex)\n", name, grid, ms * 1e3, 44.0 * n / ms / 1e6);
  };
  for (int g : {sms * 2, sms * 8, (int)(n / 4 / 512)}) {
    runu("update no-math", k_upd<0>, g);
    runu("update rcp-newton", k_upd<1>, g);
    runu("update ddiv", k_upd<2>, g);
  }
  return 0;
}

// ldst.cuh -- cache-hinted global loads shared by the gather kernels.
#pragma once

#include <cstdint>

namespace gcb {

// ---------------------------------------------------------------------------
// cache-policy loads (createpolicy: evict_first for streams read once,
// evict_last for the per-block vertex-value slice)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Range policy (the per-instruction form of an access-policy window):
// evict_last for [base, base + keep), the secondary priority for
// [base + keep, base + total) -- mode 1: evict_first, mode 2: evict_unchanged.
__device__ __forceinline__ uint64_t policy_range(const void *base, uint32_t keep, uint32_t total,
                                                 int mode) {
  uint64_t p;
  if (mode == 1)
    asm("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
        : "=l"(p)
        : "l"(base), "r"(keep), "r"(total));
  else
    asm("createpolicy.range.global.L2::evict_last.L2::evict_unchanged.b64 %0, [%1], %2, %3;"
        : "=l"(p)
        : "l"(base), "r"(keep), "r"(total));
  return p;
}
__device__ __forceinline__ uint4 ld_stream_u4(const void *ptr, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const void *ptr, uint64_t pol) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
      : "=d"(r.x), "=d"(r.y)
      : "l"(ptr), "l"(pol));
  return r;
}
// 256-bit loads (sm_100+: LDG.E.256): one full 32-byte sector per lane
__device__ __forceinline__ void ld_stream_u32x8(const void *ptr, uint64_t pol, uint32_t (&c)[8]) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]),
        "=r"(c[7])
      : "l"(ptr), "l"(pol));
}
__device__ __forceinline__ void ld_stream_f64x4(const void *ptr, uint64_t pol, double *d) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3])
      : "l"(ptr), "l"(pol));
}
// read-write streams (the same thread stores the line back): no .nc
__device__ __forceinline__ void ld_rw_f64x4(const double *ptr, double *d) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3])
               : "l"(ptr));
}
__device__ __forceinline__ void st_f64x4(double *ptr, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(ptr), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ double ld_keep(const double *p, uint64_t pol) {
  double r;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
// L1 tiers for the degree-ordered gather: warm sources stay in L1, cold ones
// do not displace them
__device__ __forceinline__ double ld_warm(const double *p, uint64_t pol) {
  double r;
  asm("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_cold(const double *p, uint64_t pol) {
  double r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_keep(const float *p, uint64_t pol) {
  float r;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return (double)r;
}

}  // namespace gcb

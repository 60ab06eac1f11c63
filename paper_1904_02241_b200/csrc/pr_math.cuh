// pr_math.cuh -- the per-vertex PageRank update arithmetic (kernels.py:398-399
// and compute_contributions 185-191), shared by the single-GPU update
// (pr.cu k_pr_update2) and the sharded peer-exchange update (exchange.cu), so
// both round identically.
#pragma once

#include <cstdint>

namespace gcb {

// Fast mode replaces the IEEE divide by deg with a Newton-refined reciprocal
// (<= 2 ulp); the exact mode keeps __ddiv_rn.
template <bool EXACT>
__device__ __forceinline__ double div_deg(double r, uint32_t dg) {
  if (EXACT) return __ddiv_rn(r, (double)dg);
  const double d = (double)dg;
  double q = (double)__frcp_rn((float)dg);
  q = fma(fma(-d, q, 1.0), q, q);
  q = fma(fma(-d, q, 1.0), q, q);
  return r * q;
}

// r' = base + d*s with two roundings, |r' - r| into dsum, c' = r'/deg (0 if dangling)
template <bool EXACT>
__device__ __forceinline__ void pr_quad(const double *s, const double *o, const uint4 d, double base,
                                        double damping, double *nr, double *c, double &dsum) {
  const uint32_t dg[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    nr[k] = __dadd_rn(base, __dmul_rn(damping, s[k]));
    dsum += fabs(nr[k] - o[k]);
    c[k] = dg[k] ? div_deg<EXACT>(nr[k], dg[k]) : 0.0;
  }
}

}  // namespace gcb

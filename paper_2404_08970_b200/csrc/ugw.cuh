// ugw.cuh -- entropic unbalanced GW (Remark 3, readings
// R32-R35 in DESIGN.md).  The hot-path kernels do the heavy work: the DP gradient (with the
// realised marginals of the plan in the constant term), and the safe-path Sinkhorn kernels with
// kappa = rho~/(rho~ + eps~).  This file holds the scalar statistics the UGW iteration needs.
#pragma once
#include "common.cuh"
#include "fused.cuh"  // ex2_ftz
#include "grad2.cuh"  // TSrc2

namespace gw {

// The plan statistics a = T 1, ct = (C o T) 1 and b = T^T 1 of the implicit plan
// T_ip = 2^((fmaf(C, -ch, gh_p) + fh_i) + fmaf(C, -cl, gl_p + fl_i)) (the Gibbs form of every other pass,
// C = the cost buffer) come from one read of C: k_ugw_moments (grad2.cuh, the moments pass's tiling).

// Fixed-order sums for the UGW scalars (one CTA):
//   out = {m(a), <a, log(a/u)>, <b, log(b/v)>, <a, f'>, <b, g'>, <ct, 1>, <a, log u>, <b, log v>}
// with 0 log 0 = 0 and rows / columns of zero weight skipped.
__global__ void __launch_bounds__(1024) k_ugw_scalars(const double* __restrict__ a, const double* __restrict__ lu,
                                                      const double* __restrict__ fa, const double* __restrict__ ct,
                                                      int64_t n, const double* __restrict__ b,
                                                      const double* __restrict__ lv, const double* __restrict__ gb,
                                                      int64_t m, double* __restrict__ out) {
  __shared__ double sm[32];
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ai = a[i];
    s[0] += ai;
    s[5] += ct[i];
    if (ai > 0.0 && lu[i] != -INFINITY) {
      s[1] += ai * (log(ai) - lu[i]);
      s[3] += ai * fa[i];
      s[6] += ai * lu[i];
    }
  }
  for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
    const double bp = b[p];
    if (bp > 0.0 && lv[p] != -INFINITY) {
      s[2] += bp * (log(bp) - lv[p]);
      s[4] += bp * gb[p];
      s[7] += bp * lv[p];
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double v = block_sum<32>(s[k], sm);
    if (threadIdx.x == 0) out[k] = v;
  }
}

// out_i = x_i + s w_i  (w = log weights: -inf stays -inf)
__global__ void k_ugw_axpy(const double* __restrict__ x, const double* __restrict__ w, double s, int64_t n,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (w[i] == -INFINITY) ? -INFINITY : fma(s, w[i], x[i]);
}

// x_i += c (finite entries only)
__global__ void k_ugw_addc(double* __restrict__ x, double c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (isfinite(x[i])) x[i] += c;
}

}  // namespace gw

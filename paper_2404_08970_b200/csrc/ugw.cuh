// ugw.cuh -- entropic unbalanced GW (Remark 3, readings
// R32-R35 in DESIGN.md).  The hot-path kernels do the heavy work: the DP gradient (with the
// realised marginals of the plan in the constant term), and the safe-path Sinkhorn kernels with
// kappa = rho~/(rho~ + eps~).  This file holds the plan statistics the UGW iteration needs.
#pragma once
#include "common.cuh"
#include "fused.cuh"  // ex2_ftz
#include "grad2.cuh"  // TSrc2

namespace gw {

// Row statistics of the implicit plan T_ip = 2^((fmaf(C, -ch, gh_p) + fh_i) + fmaf(C, -cl, gl_p + fl_i))
// (the Gibbs form of every other pass, C = the cost buffer): a_i = sum_p T_ip, ct_i = sum_p C_ip T_ip.
// Warp per row, float4 loads; fp32 lane sums flushed to fp64 every 256 columns.
constexpr int URPW = 4;  // rows per warp
__global__ void __launch_bounds__(256) k_ugw_rowstats(TSrc2 S, int64_t nl, int64_t m, double* __restrict__ a,
                                                      double* __restrict__ ct) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * URPW;
  for (int rr = 0; rr < URPW; ++rr) {
    const int64_t i = r0 + rr;
    if (i >= nl) break;
    const float Fh = S.fh[i], Fl = S.fl[i];
    const float* row = S.T + i * S.ld;
    double sa = 0.0, sc = 0.0;
    for (int64_t c0 = 4 * (int64_t)lane; c0 < m; c0 += 128 * 64) {
      float pa = 0.f, pc = 0.f;
      for (int u0 = 0; u0 < 64; u0 += 8) {
        if (c0 + 128 * u0 >= m) break;  // uniform
        float4 g4[8];  // the loads of 8 steps first
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int64_t q = c0 + 128 * (u0 + v);
          g4[v] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q + 3 < m) {
            g4[v] = *reinterpret_cast<const float4*>(row + q);
          } else if (q < m) {
            float gt[4] = {0.f, 0.f, 0.f, 0.f};
            for (int e = 0; e < 4 && q + e < m; ++e) gt[e] = row[q + e];
            g4[v] = make_float4(gt[0], gt[1], gt[2], gt[3]);
          }
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int64_t q = c0 + 128 * (u0 + v);
          const float gv[4] = {g4[v].x, g4[v].y, g4[v].z, g4[v].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (q + e < m) {
              const float g = gv[e];
              const float t = ex2_ftz((fmaf(g, -S.ch, S.gh[q + e]) + Fh) + fmaf(g, -S.cl, S.gl[q + e] + Fl));
              pa += t;
              pc = fmaf(g, t, pc);
            }
          }
        }
      }
      sa += (double)pa;
      sc += (double)pc;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, d);
      sc += __shfl_xor_sync(0xffffffffu, sc, d);
    }
    if (lane == 0) {
      a[i] = sa;
      ct[i] = sc;
    }
  }
}

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

// sink.cuh -- log-domain Sinkhorn for the entropic-OT subproblem (PAPER.md:108-114,
// Remark 1 PAPER.md:127-133) on a cost G (N x M fp32), never materialising exp(-G/eps).
//
// One iteration (reading R7): f-update then g-update,
//   f_i = eps ln p_i - eps LSE_p((g_p - G_ip)/eps),   g_p = eps ln q_p - eps LSE_i((f_i - G_ip)/eps).
// Work is in log2 units: a_ip = g_p log2e/eps - G_ip log2e/eps with the dual scaled and split
// into fp32 hi + lo parts (so the per-column rounding of g is below fp32 ulp), exponent by
// MUFU ex2, max-shifted (online) log-sum-exp, fp64 duals.
#pragma once
#include "common.cuh"

namespace gw {

// ---------------------------------------------------------------------------------
// Row half-step (robust "safe" path).  kappa = 1 (balanced); kappa = rho/(rho + eps) gives the
// unbalanced update of UGW's subproblem (reading R34) in the same absorbed form.  A CTA of 256 threads owns RROWS rows and walks
// the columns in chunks of 2048 (8 per thread), so each chunk's dual constants gh/gl are
// loaded once per RROWS rows (L2 traffic 8/RROWS B per element on top of the 4 B of G).
// Online max-shifted LSE per row in registers.
//   fout_i = eps ln p_i - eps ln2 LSE2_p(a_ip),   a_ip = g_p log2e/eps - G_ip log2e/eps
// and the violation of the current plan's row (the plan (fcur, g)):
//   |sum_p T_ip - p_i| = p_i |2^{(fcur_i - fout_i) log2e / eps} - 1|
// ---------------------------------------------------------------------------------
constexpr int RROWS = 16;

__global__ void __launch_bounds__(256) k_sink_row(const float* __restrict__ G, int64_t ld, int64_t nl, int64_t m,
                                                  const float* __restrict__ gh, const float* __restrict__ gl,
                                                  float c2f, const double* __restrict__ fcur,
                                                  double* __restrict__ fout, const double* __restrict__ lp,
                                                  double eps, float* __restrict__ fh, float* __restrict__ fl,
                                                  float* __restrict__ viol, const int* __restrict__ stop,
                                                  const int* __restrict__ skip_if_fast, double kappa = 1.0) {
  if (stop && *stop) return;
  if (skip_if_fast && *skip_if_fast) return;  // a skipped launch costs one small wave (grid-stride)
  __shared__ float smm[RROWS][8], sms[RROWS][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t r0 = (int64_t)blockIdx.x * RROWS; r0 < nl; r0 += (int64_t)gridDim.x * RROWS) {
  const int nr = (int)min((int64_t)RROWS, nl - r0);
  LSE2 st[RROWS];
#pragma unroll
  for (int r = 0; r < RROWS; ++r) st[r] = LSE2{-INFINITY, 0.f};
  for (int64_t q = 8 * (int64_t)threadIdx.x; q < m; q += 8 * 256) {
    float hv[8], lv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool v = q + k < m;
      hv[k] = v ? gh[q + k] : -INFINITY;
      lv[k] = v ? gl[q + k] : 0.f;
    }
    // rows in groups of 4: the group's 8 float4 loads are issued before their arithmetic
#pragma unroll
    for (int r4 = 0; r4 < RROWS; r4 += 4) {
      float4 x0[4], x1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        x1[u] = x0[u];
        if (r4 + u < nr) {
          const float* gr = G + (r0 + r4 + u) * ld + q;
          x0[u] = __ldcs(reinterpret_cast<const float4*>(gr));
          if (q + 4 < m) x1[u] = __ldcs(reinterpret_cast<const float4*>(gr + 4));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r4 + u;
        if (r < nr) {
          const float gv[8] = {x0[u].x, x0[u].y, x0[u].z, x0[u].w, x1[u].x, x1[u].y, x1[u].z, x1[u].w};
          float av[8];
          float cm = -INFINITY;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            av[k] = (q + k < m) ? fmaf(gv[k], -c2f, hv[k]) + lv[k] : -INFINITY;
            cm = fmaxf(cm, av[k]);
          }
          LSE2 s = st[r];
          if (cm > s.m) {
            s.s = (s.m == -INFINITY) ? 0.f : s.s * exp2f(s.m - cm);
            s.m = cm;
          }
          if (s.m != -INFINITY) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += exp2f(av[k] - s.m);
            s.s += acc;
          }
          st[r] = s;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RROWS; ++r) {
    LSE2 s = lse_warp(st[r]);
    if (lane == 0) { smm[r][w] = s.m; sms[r][w] = s.s; }
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    const int r = threadIdx.x;
    const int64_t row = r0 + r;
    LSE2 s{smm[r][0], sms[r][0]};
    for (int k = 1; k < 8; ++k) s = lse_merge(s, LSE2{smm[r][k], sms[r][k]});
    const double l2e_eps = GW_LOG2E / eps;
    const double lse2 = (double)s.m + log2((double)s.s);
    const double fo = fcur[row];
    const double fn = (lp[row] == -INFINITY) ? -INFINITY : eps * lp[row] - kappa * (eps * GW_LN2 * lse2);
    fout[row] = fn;
    const double fs = fn * l2e_eps;
    const float h = (float)fs;
    fh[row] = h;
    fl[row] = isfinite(fs) ? (float)(fs - (double)h) : 0.f;
    if (viol) {
      const double pi = exp(lp[row]);
      double v = (pi > 0.0) ? pi * fabs(exp2((fo - fn) * l2e_eps) - 1.0) : 0.0;
      if (!(v == v)) v = 3.0e38;
      atomic_max_nonneg(viol, (float)fmin(v, 3.0e38));
    }
  }
  __syncthreads();  // smm / sms are reused by the next row group
  }
}

// ---------------------------------------------------------------------------------
// Column half-step, pass 1: per (row block, column) online LSE of b_ip = f_i log2e/eps -
// G_ip log2e/eps.  Thread = 4 consecutive columns (float4), CTA = 1024 columns, rows
// [rb*RB, (rb+1)*RB).  Partials (m, s) to part[rb][q].
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sink_col(const float* __restrict__ G, int64_t ld, int64_t nl, int64_t m,
                                                  const float* __restrict__ fh, const float* __restrict__ fl,
                                                  float c2f, int64_t RB, float2* __restrict__ part,
                                                  const int* __restrict__ stop, const int* __restrict__ skip_if_fast) {
  if (stop && *stop) return;
  if (skip_if_fast && *skip_if_fast) return;  // a skipped launch costs one small wave (grid-stride)
  const int64_t ncb = (m + 1023) / 1024, nrb = (nl + RB - 1) / RB;
  for (int64_t item = blockIdx.x; item < ncb * nrb; item += gridDim.x) {
  const int64_t q0 = ((item % ncb) * 256 + threadIdx.x) * 4;
  if (q0 >= m) continue;
  const int64_t rb = item / ncb;
  const int64_t rs = rb * RB, re = min(nl, rs + RB);
  LSE2 st[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) st[k] = LSE2{-INFINITY, 0.f};
  const float* base = G + q0;
  int64_t r = rs;
  for (; r + 8 <= re; r += 8) {  // 8 rows' loads in flight per thread
    float4 x[8];
    float fr[8], fo[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcs(reinterpret_cast<const float4*>(base + (r + u) * ld));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      fr[u] = fh[r + u];
      fo[u] = fl[r + u];
    }
    float a[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u][0] = fmaf(x[u].x, -c2f, fr[u]) + fo[u];
      a[u][1] = fmaf(x[u].y, -c2f, fr[u]) + fo[u];
      a[u][2] = fmaf(x[u].z, -c2f, fr[u]) + fo[u];
      a[u][3] = fmaf(x[u].w, -c2f, fr[u]) + fo[u];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float cm = a[0][k];
#pragma unroll
      for (int u = 1; u < 8; ++u) cm = fmaxf(cm, a[u][k]);
      if (cm > st[k].m) {
        st[k].s = (st[k].m == -INFINITY) ? 0.f : st[k].s * exp2f(st[k].m - cm);
        st[k].m = cm;
      }
      if (st[k].m != -INFINITY) {
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += exp2f(a[u][k] - st[k].m);
        st[k].s += acc;
      }
    }
  }
  for (; r < re; ++r) {
    const float4 x = __ldcs(reinterpret_cast<const float4*>(base + r * ld));
    const float fr = fh[r], lo = fl[r];
    const float a[4] = {fmaf(x.x, -c2f, fr) + lo, fmaf(x.y, -c2f, fr) + lo, fmaf(x.z, -c2f, fr) + lo,
                        fmaf(x.w, -c2f, fr) + lo};
#pragma unroll
    for (int k = 0; k < 4; ++k) st[k] = lse_merge(st[k], LSE2{a[k], 1.f});
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (q0 + k < m) part[rb * m + q0 + k] = make_float2(st[k].m, st[k].s);
  }
}

// Column half-step, pass 2a: merge this rank's row-block partials in fixed order, in fp64:
// lse[q] = max_rb M, lse[m + q] = sum_rb S_rb 2^(M_rb - max).
// pack: write the pair as ONE 8-byte {float M, float S} per column (M is a max of fp32 values, exact in
// fp32; S in [1, nrb] rounded once to fp32), so the pairs fit the multi-rank loop's M-double payload.
__global__ void k_sink_colmerge(const float2* __restrict__ part, int nrb, int64_t m, double* __restrict__ lse,
                                const int* __restrict__ stop, const int* __restrict__ skip_if_fast,
                                bool pack = false) {
  if (stop && *stop) return;
  if (skip_if_fast && *skip_if_fast) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  double M = -INFINITY;
  for (int rb = 0; rb < nrb; ++rb) M = fmax(M, (double)part[(int64_t)rb * m + q].x);
  double S = 0.0;
  if (M != -INFINITY)
    for (int rb = 0; rb < nrb; ++rb) {
      const float2 v = part[(int64_t)rb * m + q];
      if (v.x != -INFINITY) S += (double)v.y * exp2((double)v.x - M);
    }
  if (pack) {
    reinterpret_cast<float2*>(lse)[q] = make_float2((float)M, (float)S);
  } else {
    lse[q] = M;
    lse[m + q] = S;
  }
}

// Column half-step, pass 2b: merge the R ranks' (M, S) pairs (gath [R][2m]) in rank order and
// update g (identical on every rank).
// gstride: doubles between two ranks' payloads in gath (0: 2m; the multi-rank fixed-count loop gathers
// the column sums and the LSE pairs in one payload, so its pairs sit at a larger stride).
__global__ void k_sink_colfin(const double* __restrict__ gath, int R, int64_t m, const double* __restrict__ lq,
                              double eps, double* __restrict__ g, float* __restrict__ gh, float* __restrict__ gl,
                              const int* __restrict__ stop, const int* __restrict__ skip_if_fast,
                              float* __restrict__ dev, double kappa = 1.0, int64_t gstride = 0,
                              bool packed = false) {
  if (stop && *stop) return;
  if (skip_if_fast && *skip_if_fast) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  const int64_t gs_ = gstride > 0 ? gstride : 2 * m;
  // rank r's pair: {M, S} doubles at [r gs_ + q], [r gs_ + m + q], or packed {float M, float S} at
  // 8-byte slot r gs_ + q (k_sink_colmerge's pack)
  auto Mof = [&](int r) -> double {
    return packed ? (double)reinterpret_cast<const float2*>(gath + (int64_t)r * gs_)[q].x : gath[(int64_t)r * gs_ + q];
  };
  auto Sof = [&](int r) -> double {
    return packed ? (double)reinterpret_cast<const float2*>(gath + (int64_t)r * gs_)[q].y
                  : gath[(int64_t)r * gs_ + m + q];
  };
  double M = -INFINITY;
  for (int r = 0; r < R; ++r) M = fmax(M, Mof(r));
  double S = 0.0;
  if (M != -INFINITY)
    for (int r = 0; r < R; ++r) {
      const double Mr = Mof(r);
      if (Mr != -INFINITY) S += Sof(r) * exp2(Mr - M);
    }
  const double lse2 = M + log2(S);
  const double gn = (lq[q] == -INFINITY) ? -INFINITY : eps * lq[q] - kappa * (eps * GW_LN2 * lse2);
  if (dev) {  // |log2(colsum / q)| of the half-step plan: decides the next iteration's path
    double d = fabs((gn - g[q]) * (GW_LOG2E / eps));
    if (!(d == d)) d = 3.0e38;
    float dv = (float)fmin(d, 3.0e38);
    dv = warp_max(dv);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dev, dv);
  }
  g[q] = gn;
  const double gs = gn * (GW_LOG2E / eps);
  const float h = (float)gs;
  gh[q] = h;
  gl[q] = isfinite(gs) ? (float)(gs - (double)h) : 0.f;
}

// One rank: pass 2a + 2b in one launch (merge the row-block partials, then update g).
__global__ void k_sink_colmergefin(const float2* __restrict__ part, int nrb, int64_t m, const double* __restrict__ lq,
                                   double eps, double* __restrict__ g, float* __restrict__ gh, float* __restrict__ gl,
                                   const int* __restrict__ stop, const int* __restrict__ skip_if_fast,
                                   float* __restrict__ dev, double kappa = 1.0) {
  if (stop && *stop) return;
  if (skip_if_fast && *skip_if_fast) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  double M = -INFINITY;
  for (int rb = 0; rb < nrb; ++rb) M = fmax(M, (double)part[(int64_t)rb * m + q].x);
  double S = 0.0;
  if (M != -INFINITY)
    for (int rb = 0; rb < nrb; ++rb) {
      const float2 v = part[(int64_t)rb * m + q];
      if (v.x != -INFINITY) S += (double)v.y * exp2((double)v.x - M);
    }
  // (M, S) exactly as k_sink_colmerge + k_sink_colfin with R = 1
  const double lse2 = M + log2(S);
  const double gn = (lq[q] == -INFINITY) ? -INFINITY : eps * lq[q] - kappa * (eps * GW_LN2 * lse2);
  if (dev) {
    double d = fabs((gn - g[q]) * (GW_LOG2E / eps));
    if (!(d == d)) d = 3.0e38;
    float dv = (float)fmin(d, 3.0e38);
    dv = warp_max(dv);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dev, dv);
  }
  g[q] = gn;
  const double gs = gn * (GW_LOG2E / eps);
  const float h = (float)gs;
  gh[q] = h;
  gl[q] = isfinite(gs) ? (float)(gs - (double)h) : 0.f;
}

// Fused path: this rank's column sums of the half-step plan, clusters summed in fixed order.
// CTA = 32 columns x 8 warps: warp w sums clusters w, w + 8, ... for lane's column, then the 8
// warp sums are added in warp order (deterministic; 8x the parallelism of a thread per column,
// which matters when there are many clusters, i.e. small problems with one CTA per cluster).
// Multi-rank (rowflag != null): the same launch also checks this rank's row sums S_i (finite, above
// 2^-100, as k_sink_fast_check) and ORs a bad row into *rowflag -- an int in the payload slot after
// the M column sums, so the speculation flag travels in the column-sum all-gather (one collective
// per iteration).  Rows are covered grid-stride by all threads.
// csflag / lq (one rank): also validate the column sums here (k_sink_fast_check's column test, on the
// columns with q > 0) and OR a failure into *csflag -- with rowflag == csflag the whole check of the
// speculative iteration happens in this launch.
__global__ void __launch_bounds__(256) k_sink_colsum(const double* __restrict__ part, int ncl, int64_t m,
                                                     double* __restrict__ out, const int* __restrict__ mode,
                                                     const int* __restrict__ stop, const float* __restrict__ Srow = nullptr,
                                                     int64_t nl = 0, int* __restrict__ rowflag = nullptr,
                                                     int* __restrict__ csflag = nullptr,
                                                     const double* __restrict__ lq = nullptr) {
  if (*mode != 1 || (stop && *stop)) return;
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (rowflag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
      const float S = Srow[i];
      bad |= !(S > 7.9e-31f && S < 3.0e38f);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(rowflag, 1);
  }
  const int64_t q = blockIdx.x * (int64_t)32 + lane;
  double CS = 0.0;
  if (q < m)
    for (int c = w; c < ncl; c += 8) CS += part[(int64_t)c * m + q];
  red[w][lane] = CS;
  __syncthreads();
  if (w == 0) {
    bool bad = false;
    if (q < m) {
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) v += red[k][lane];
      out[q] = v;
      if (csflag && lq[q] != -INFINITY) bad = !(v > 7.9e-31 && v < 1e300);
    }
    if (csflag && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(csflag, 1);
  }
}

// Tolerance rule (reading R8): the row half-step of iteration k+1 measured the violation of
// the plan after iteration k into *viol (written to ftmp).  If it is <= tol, stop with f
// unchanged (iteration k+1 is discarded); otherwise commit ftmp -> f.
// it_dev (nullable): the iteration count before this check, read from the device (graph-resident loop)
__global__ void k_sink_commit(const float* __restrict__ viol, double tol, int* __restrict__ stop,
                              const double* __restrict__ ftmp, double* __restrict__ f, int64_t nl,
                              int* __restrict__ iters, int it_before, const int* __restrict__ it_dev = nullptr) {
  if (*stop) return;
  const bool done = (double)(*viol) <= tol;
  __syncthreads();
  if (done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { *stop = 1; *iters = it_dev ? *it_dev : it_before; }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = ftmp[i];
}

// End of one round of the graph-resident tolerance loop (reading R8): `step` more iterations done;
// loop again unless the tolerance stopped the solve or the cap is reached (a device flag, no host sync).
__global__ void k_tol_round_end(int* __restrict__ cnt, int step, int cap, const int* __restrict__ stop,
                                cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    *cnt += step;
    cudaGraphSetConditional(h, (!*stop && *cnt < cap) ? 1u : 0u);
  }
}

}  // namespace gw

// vec.cuh -- O(N + M) kernels: validation, set-up, 1-D dynamic programmes.
#pragma once
#include "common.cuh"

namespace gw {

// ---------------------------------------------------------------------------------
// Validation + moments of one (support, marginal) pair, one CTA of 1024 threads.
// out[0..7] = {unsorted, negative, nonfinite, S0 = sum w, S1 = sum xc w, S2 = sum xc^2 w,
//              xmid, x_{n-1}}, xc = x - xmid, xmid = (x_0 + x_{n-1}) / 2.
// Fixed-order reduction => deterministic (SPEC.md:68-76 validate_measure).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_validate(const double* __restrict__ x0, const double* __restrict__ w0,
                                                   int64_t n0, const double* __restrict__ x1,
                                                   const double* __restrict__ w1, int64_t n1,
                                                   double* __restrict__ out) {
  __shared__ double sm[32];
  const double* x = blockIdx.x == 0 ? x0 : x1;
  const double* w = blockIdx.x == 0 ? w0 : w1;
  const int64_t n = blockIdx.x == 0 ? n0 : n1;
  double* o = out + 8 * blockIdx.x;
  const double xmid = 0.5 * (x[0] + x[n - 1]);
  double uns = 0, neg = 0, nf = 0, s0 = 0, s1 = 0, s2 = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double xi = x[i], wi = w[i];
    if (!isfinite(xi) || !isfinite(wi)) nf = 1;
    if (i + 1 < n && !(x[i + 1] >= xi)) uns = 1;
    if (wi < 0) neg = 1;
    const double xc = xi - xmid;
    s0 += wi;
    s1 += xc * wi;
    s2 += xc * xc * wi;
  }
  uns = block_sum<32>(uns, sm);
  neg = block_sum<32>(neg, sm);
  nf = block_sum<32>(nf, sm);
  s0 = block_sum<32>(s0, sm);
  s1 = block_sum<32>(s1, sm);
  s2 = block_sum<32>(s2, sm);
  if (threadIdx.x == 0) {
    o[0] = uns; o[1] = neg; o[2] = nf; o[3] = s0; o[4] = s1; o[5] = s2; o[6] = xmid; o[7] = x[n - 1];
  }
}

// ---------------------------------------------------------------------------------
// Set-up of one (support, marginal) pair (grid-stride):
//   xc = x - xmid (centred; GW is translation invariant),
//   wn = w / S0 (renormalised copy), lw = ln wn,
//   c_i = sum_j (x_i - x_j)^2 wn_j = xc_i^2 - 2 xc_i mu1 + mu2   ((D o D) u
//   at k = 1, by moments of the normalised marginal; mu_k = S_k / S0).
// ---------------------------------------------------------------------------------
__global__ void k_prep(const double* __restrict__ x, const double* __restrict__ w, int64_t n,
                       const double* __restrict__ mom, double* __restrict__ xc, double* __restrict__ wn,
                       double* __restrict__ lw, double* __restrict__ cvec, bool normalize = true,
                       float* __restrict__ wf = nullptr, float* __restrict__ xf = nullptr) {
  // normalize = false (unbalanced GW): wn = w as given (mass S0), cvec = (D o D) w = S0 (v^2 - 2 v mu1 + mu2)
  const double xmid = mom[6], S0 = mom[3];
  const double mu1 = mom[4] / S0, mu2 = mom[5] / S0, inv = normalize ? 1.0 / S0 : 1.0, cs = normalize ? 1.0 : S0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i] - xmid;
    const double wv = w[i] * inv;
    xc[i] = v;
    wn[i] = wv;
    lw[i] = log(wv);
    cvec[i] = cs * (v * v - 2.0 * v * mu1 + mu2);
    if (wf) wf[i] = (float)wv;  // fp32 copies (the fp32 gradient path's T^0 = p q^T, centred y)
    if (xf) xf[i] = (float)v;
  }
}

// ---------------------------------------------------------------------------------
// 1-D dynamic programme on a sorted support s (k_scan1d_tot / k_scan1d_out below):
//   lower_i = sum_{j<i} (s_i - s_j) v_j                      (the paper's L v at k = 1,
//   dist_i  = sum_j |s_i - s_j| v_j = 2 lower_i + Sv - s_i V   PAPER.md:219-243; D = L + L^T)
// with V = sum v, Sv = sum s v.  Chunked: local pass, fixed-order scan of chunk states,
// second local pass.  Either output may be null.  tot (nullable) = {V, Sv}.
// ---------------------------------------------------------------------------------
struct Scan1D {
  const double* v;
  const double* s;
  int64_t n;
  double* lower;
  double* dist;
  double* tot;
};
struct Scan1DBatch {
  Scan1D d[6];
};

// ---------------------------------------------------------------------------------
// Spread over K CTAs per vector (one CTA per vector would be 4 CTAs on 148 SMs and a 64-step
// fp64 warp-scan chain per pass at n = 65536).  Segment k
// of vector v is [k L, (k+1) L), L a multiple of 1024; warp w owns the contiguous 1/32 of it.
//   k_scan1d_tot: each warp's total state -> wt[((v K) + k) 32 + w]   (3 doubles: P, A, s)
//   k_scan1d_out: the warp's exclusive prefix = fixed-order fold of the warp totals before it,
//                 the grand total = fold of all of them; then the output walk.
// ---------------------------------------------------------------------------------
constexpr int SCAN_KMAX = 32;

__device__ __forceinline__ void scan1d_seg(const Scan1D& D, int K, int k, int w, int64_t& i0, int64_t& i1) {
  const int64_t L = ((D.n + K - 1) / K + 1023) / 1024 * 1024;
  const int64_t C = L / 32;
  i0 = (int64_t)k * L + (int64_t)w * C;
  i1 = min(D.n, i0 + C);
}

__global__ void __launch_bounds__(1024) k_scan1d_tot(Scan1DBatch B, int K, double* __restrict__ wt) {
  const int v = blockIdx.y, k = blockIdx.x;
  if (k >= K) return;
  const Scan1D D = B.d[v];
  const int64_t n = D.n;
  if (n <= 0) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t i0, i1;
  scan1d_seg(D, K, k, w, i0, i1);
  constexpr int SU = 4;
  PA<double> run{0.0, 0.0, i0 < n ? D.s[i0] : D.s[n - 1]};
  for (int64_t b4 = i0; b4 < i1; b4 += 32 * SU) {
    double sv[SU], vv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int64_t i = b4 + 32 * u + lane;
      sv[u] = D.s[min(i, i1 - 1)];
      vv[u] = i < i1 ? D.v[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      if (b4 + 32 * u >= i1) break;  // uniform across the warp
      PA<double> ex;
      const PA<double> inc = pa_warp_scan(PA<double>{vv[u], 0.0, sv[u]}, ex);
      PA<double> st;
      st.P = __shfl_sync(0xffffffffu, inc.P, 31);
      st.A = __shfl_sync(0xffffffffu, inc.A, 31);
      st.s = __shfl_sync(0xffffffffu, inc.s, 31);
      run = pa_combine(run, st);
    }
  }
  if (lane == 0) {
    double* o = wt + 3 * (((int64_t)v * K + k) * 32 + w);
    o[0] = run.P; o[1] = run.A; o[2] = run.s;
  }
}

__global__ void __launch_bounds__(1024) k_scan1d_out(Scan1DBatch B, int K, const double* __restrict__ wt) {
  __shared__ double sw[3 * 32 * SCAN_KMAX];
  __shared__ double sseg[3 * SCAN_KMAX], spre[3 * 32], stot[3];
  const int v = blockIdx.y, k = blockIdx.x;
  const Scan1D D = B.d[v];
  const int64_t n = D.n;
  if (n <= 0) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = K * 32;
  for (int e = threadIdx.x; e < 3 * nw; e += 1024) sw[e] = wt[3 * (int64_t)v * nw + e];
  __syncthreads();
  // fixed-order two-level fold (every CTA of the vector folds the same entries in the same order):
  // lane j of warp 0 folds segment j's 32 warp totals; lane 0 folds the segment totals (-> the
  // segment prefixes and the grand total); warp w's lane 0 adds its segment's warps before it.
  if (w == 0) {
    if (lane < K) {
      const double* e = sw + 3 * 32 * lane;
      PA<double> t{e[0], e[1], e[2]};
#pragma unroll 4
      for (int j = 1; j < 32; ++j) t = pa_combine(t, PA<double>{e[3 * j], e[3 * j + 1], e[3 * j + 2]});
      sseg[3 * lane] = t.P; sseg[3 * lane + 1] = t.A; sseg[3 * lane + 2] = t.s;
    }
    __syncwarp();
    if (lane == 0) {
      PA<double> run{0.0, 0.0, sw[2]}, segpre = run;
      for (int j = 0; j < K; ++j) {
        if (j == k) segpre = run;
        run = pa_combine(run, PA<double>{sseg[3 * j], sseg[3 * j + 1], sseg[3 * j + 2]});
      }
      stot[0] = run.P; stot[1] = run.A; stot[2] = run.s;
      spre[0] = segpre.P; spre[1] = segpre.A; spre[2] = segpre.s;
    }
  }
  __syncthreads();
  if (lane == 0 && w > 0) {
    PA<double> pre{spre[0], spre[1], spre[2]};
    const double* e = sw + 3 * 32 * k;
    for (int j = 0; j < w; ++j) pre = pa_combine(pre, PA<double>{e[3 * j], e[3 * j + 1], e[3 * j + 2]});
    spre[3 * w] = pre.P; spre[3 * w + 1] = pre.A; spre[3 * w + 2] = pre.s;
  }
  __syncthreads();
  const double V = stot[0], Sv = stot[2] * stot[0] - stot[1];
  int64_t i0, i1;
  scan1d_seg(D, K, k, w, i0, i1);
  PA<double> run{spre[3 * w], spre[3 * w + 1], spre[3 * w + 2]};
  constexpr int SU = 4;
  for (int64_t b4 = i0; b4 < i1; b4 += 32 * SU) {
    double sv[SU], vv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int64_t i = b4 + 32 * u + lane;
      sv[u] = D.s[min(i, i1 - 1)];
      vv[u] = i < i1 ? D.v[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      if (b4 + 32 * u >= i1) break;  // uniform across the warp
      const int64_t i = b4 + 32 * u + lane;
      const double si = sv[u];
      PA<double> ex;
      const PA<double> inc = pa_warp_scan(PA<double>{vv[u], 0.0, si}, ex);
      const double lo = pa_eval(pa_combine(run, ex), si);
      if (i < i1) {
        if (D.lower) D.lower[i] = lo;
        if (D.dist) D.dist[i] = 2.0 * lo + Sv - si * V;
      }
      PA<double> st;
      st.P = __shfl_sync(0xffffffffu, inc.P, 31);
      st.A = __shfl_sync(0xffffffffu, inc.A, 31);
      st.s = __shfl_sync(0xffffffffu, inc.s, 31);
      run = pa_combine(run, st);
    }
  }
  if (D.tot && k == 0 && threadIdx.x == 0) { D.tot[0] = V; D.tot[1] = Sv; }
}

// Test-only fault injection (SURVEY §4.2 tier T6, env GWDP_FAULT): perturb one entry so that the
// parity tests must fail -- evidence that they would catch a wrong carry or column sum.
__global__ void k_fault_scale(double* __restrict__ v, int64_t i, double f) {
  if (blockIdx.x == 0 && threadIdx.x == 0) v[i] *= f;
}

// fp32 hi/lo split of s * v (log2-domain dual scaling used by the Sinkhorn kernels)
__global__ void k_split(const double* __restrict__ v, int64_t n, double scale, float* __restrict__ hi,
                        float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = v[i] * scale;
    const float h = (float)s;
    hi[i] = h;
    lo[i] = isfinite(s) ? (float)(s - (double)h) : 0.f;
  }
}

__global__ void k_scale(const double* __restrict__ v, int64_t n, double scale, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v[i] * scale;
}

__global__ void k_scale_f(const double* __restrict__ v, int64_t n, double scale, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)(v[i] * scale);
}

__global__ void k_to_float(const double* __restrict__ v, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)v[i];
}

__global__ void k_fill_int(int* __restrict__ v, int val) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *v = val;
}

__global__ void k_fill(double* __restrict__ v, int64_t n, double val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = val;
}

// ---------------------------------------------------------------------------------
// Objective assembly from the gradient pass's reductions (deterministic, fixed order).
// With G' = 2(c 1^T + 1 c'^T) - 4 V (prescribed c, c'), V = D_X T D_Y:
//   <V, T> = (2<c, a> + 2<c', b> - <G', T>) / 4,
//   E(T)   = a^T (D_X o D_X) a + b^T (D_Y o D_Y) b - 2 <V, T>      (PAPER.md:86 expanded)
// and a^T (D o D) a = 2 (A0 A2 - A1^2), A_k = sum xc^k a (moments; k = 1).
// viol = max(|a - p|_inf, |b - q|_inf).
// k_obj_partial: this rank's row sums a = T 1 (local rows) and tile sums ->
//   part[8] = {A0, A1, A2, <c, a>, max|a - p|, <G', T>, H, <C o C, T>}
// k_obj_final: sums the R ranks' partials in rank order, adds the column part (b = T^T 1 is
// global) -> out = {E, viol, <G', T>, H, -, -, <C o C, T>, -}.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_obj_partial(const double* __restrict__ a, const double* __restrict__ xc,
                                                      const double* __restrict__ p, const double* __restrict__ c,
                                                      int64_t n, const double* __restrict__ tile_obj, int64_t ntile,
                                                      const double* __restrict__ tile_ent,
                                                      const double* __restrict__ tile_cc, double* __restrict__ part) {
  __shared__ double sm[32];
  double A0 = 0, A1 = 0, A2 = 0, ca = 0, va = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ai = a[i], xi = xc[i];
    A0 += ai; A1 += ai * xi; A2 += ai * xi * xi; ca += c[i] * ai;
    va = fmax(va, fabs(ai - p[i]));
  }
  double go = 0, he = 0, cc = 0;
  for (int64_t i = threadIdx.x; i < ntile; i += blockDim.x) {
    go += tile_obj[i];
    if (tile_ent) he += tile_ent[i];
    if (tile_cc) cc += tile_cc[i];
  }
  A0 = block_sum<32>(A0, sm); A1 = block_sum<32>(A1, sm); A2 = block_sum<32>(A2, sm);
  ca = block_sum<32>(ca, sm);
  go = block_sum<32>(go, sm); he = block_sum<32>(he, sm); cc = block_sum<32>(cc, sm);
  __shared__ double smx[32];
  double vmax = va;
  for (int d = 16; d > 0; d >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, d));
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) smx[0] = fmax(smx[0], smx[k]);
    part[0] = A0; part[1] = A1; part[2] = A2; part[3] = ca; part[4] = smx[0];
    part[5] = go; part[6] = he; part[7] = cc;
  }
}

__global__ void __launch_bounds__(1024) k_obj_final(const double* __restrict__ parts, int R,
                                                    const double* __restrict__ b, const double* __restrict__ yc,
                                                    const double* __restrict__ q, const double* __restrict__ c2,
                                                    int64_t m, double* __restrict__ out) {
  __shared__ double sm[32];
  double B0 = 0, B1 = 0, B2 = 0, cb = 0, vb = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double bi = b[i], yi = yc[i];
    B0 += bi; B1 += bi * yi; B2 += bi * yi * yi; cb += c2[i] * bi;
    vb = fmax(vb, fabs(bi - q[i]));
  }
  B0 = block_sum<32>(B0, sm); B1 = block_sum<32>(B1, sm); B2 = block_sum<32>(B2, sm);
  cb = block_sum<32>(cb, sm);
  __shared__ double smx[32];
  double vmax = vb;
  for (int d = 16; d > 0; d >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, d));
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) smx[0] = fmax(smx[0], smx[k]);
    double A0 = 0, A1 = 0, A2 = 0, ca = 0, va = 0, go = 0, he = 0, cc = 0;
    for (int r = 0; r < R; ++r) {
      const double* pr = parts + 8 * r;
      A0 += pr[0]; A1 += pr[1]; A2 += pr[2]; ca += pr[3]; va = fmax(va, pr[4]);
      go += pr[5]; he += pr[6]; cc += pr[7];
    }
    const double VT = (2.0 * ca + 2.0 * cb - go) / 4.0;
    const double E = 2.0 * (A0 * A2 - A1 * A1) + 2.0 * (B0 * B2 - B1 * B1) - 2.0 * VT;
    out[0] = E;
    out[1] = fmax(va, smx[0]);
    out[2] = go;
    out[3] = he;
    out[6] = cc;
  }
}

}  // namespace gw

// small.cuh -- cluster-resident Sinkhorn for problems whose cost matrix fits in one thread-block
// cluster's shared memory (C1, N = M = 256, is launch-bound).
//
// The multi-kernel iteration of sink.cuh / fused.cuh costs ~10 launches (~28 us) per Sinkhorn
// iteration at these sizes, whatever the bytes.  Here ONE launch runs all `iters` iterations of
// a solve's inner loop: a cluster of CL CTAs (CL = 1 .. 16) holds G in shared memory (CTA r owns a
// contiguous block of rows), and per iteration
//   f-update  (reading R7 order)  warp per own row, max-shifted LSE over the row in smem;
//   g-update  thread per column, LSE partials (max, sum) over the CTA's rows, written to this
//             CTA's double-buffered partials; ONE cluster barrier; every CTA reads all CL partials
//             through DSMEM (mapa + ld.shared::cluster) and combines them in CTA order, so g is
//             bit-identical in every CTA.
// Same update as k_sink_row / k_sink_colfin (log-domain, fp64 duals, exponent in log2 units):
//   f_i = eps ln p_i - kappa eps ln2 LSE2_p((g_p - G_ip) log2e/eps),
//   g_p = eps ln q_p - kappa eps ln2 LSE2_i((f_i - G_ip) log2e/eps),   kappa = 1 (balanced).
// The exponent arguments are formed in fp64 (the matrix is small); each LSE is two passes (the
// max, then the sum of exp2f(a - max): independent exponentials, no rescaling chain).
#pragma once
#include "common.cuh"
#include "fused.cuh"  // cluster helpers

namespace gw {

constexpr int SNT = 512;  // threads per CTA

__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

struct SmallArgs {
  const float* G;
  int64_t ld, nl, m;
  int rows;       // rows per CTA (last CTA may hold fewer)
  int mp;         // smem row pitch (floats; even, so the fp64 arrays after the tile are aligned)
  const double *lp, *lq;
  double eps, kappa;
  int iters;
  double *f, *g;  // in: warm start, out: final duals
};

// dynamic smem: Gs [rows][mp] fp32 | gS [m] | part [2][2][m] (max, sum; double-buffered) | fS [rows] | lpS [rows]
__host__ __device__ inline size_t small_smem_bytes(int rows, int mp, int64_t m) {
  return sizeof(float) * (size_t)rows * mp + sizeof(double) * ((size_t)m * 5 + 2 * (size_t)rows);
}

__global__ void __launch_bounds__(SNT, 1) k_sink_small(SmallArgs a) {
  extern __shared__ __align__(16) float sraw[];
  const uint32_t cr = cluster_rank();
  const uint32_t CL = gridDim.x;  // one cluster: every CTA of the grid
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int NWp = SNT / 32;
  const int64_t m = a.m;
  const int64_t r0 = (int64_t)cr * a.rows;
  const int nr = (int)max((int64_t)0, min((int64_t)a.rows, a.nl - r0));
  float* Gs = sraw;
  double* gS = reinterpret_cast<double*>(Gs + (size_t)a.rows * a.mp);
  double* part = gS + m;                 // [2 buffers][2 (max, sum)][m]
  double* fS = part + 4 * m;
  double* lpS = fS + a.rows;
  const double c = GW_LOG2E / a.eps;
  const double kep = a.kappa * a.eps * GW_LN2;
  // stage G (this CTA's rows), the duals and ln p
  for (int r = 0; r < nr; ++r)
    for (int64_t q = t; q < m; q += SNT) Gs[(size_t)r * a.mp + q] = a.G[(r0 + r) * a.ld + q];
  for (int64_t q = t; q < m; q += SNT) gS[q] = a.g[q];
  for (int r = t; r < nr; r += SNT) {
    fS[r] = a.f[r0 + r];
    lpS[r] = a.lp[r0 + r];
  }
  __syncthreads();
  cluster_arrive();
  cluster_wait();  // every CTA's shared memory is live before any DSMEM access
  for (int it = 0; it < a.iters; ++it) {
    // ---- f-update: warp per own row; two passes (max, then sum of 2^(a - max)) ----
    for (int r = w; r < nr; r += NWp) {
      const float* row = Gs + (size_t)r * a.mp;
      double mx = -INFINITY;
      for (int64_t q = lane; q < m; q += 32) mx = fmax(mx, (gS[q] - (double)row[q]) * c);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      float sm = 0.f;
      if (mx != -INFINITY)
        for (int64_t q = lane; q < m; q += 32) sm += exp2f((float)((gS[q] - (double)row[q]) * c - mx));
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, d);
      if (lane == 0) {
        const double lse2 = (mx == -INFINITY) ? -INFINITY : mx + log2((double)sm);
        fS[r] = (lpS[r] == -INFINITY) ? -INFINITY : a.eps * lpS[r] - kep * lse2;
      }
    }
    __syncthreads();
    // ---- g-update: column partials (max, sum) over this CTA's rows ----
    double* pb = part + (size_t)(it & 1) * 2 * m;
    for (int64_t q = t; q < m; q += SNT) {
      double mx = -INFINITY;
      for (int r = 0; r < nr; ++r) mx = fmax(mx, (fS[r] - (double)Gs[(size_t)r * a.mp + q]) * c);
      float sm = 0.f;
      if (mx != -INFINITY)
        for (int r = 0; r < nr; ++r) sm += exp2f((float)((fS[r] - (double)Gs[(size_t)r * a.mp + q]) * c - mx));
      pb[q] = mx;
      pb[m + q] = (double)sm;
    }
    cluster_arrive();
    cluster_wait();  // every CTA's partials of this iteration are written
    for (int64_t q = t; q < m; q += SNT) {
      double Mk[16], Sk[16];
      double M = -INFINITY;
      for (uint32_t k = 0; k < CL; ++k) {
        Mk[k] = ld_dsmem_f64(mapa(pb + q, k));
        Sk[k] = ld_dsmem_f64(mapa(pb + m + q, k));
        M = fmax(M, Mk[k]);
      }
      double S = 0.0;
      if (M != -INFINITY)
        for (uint32_t k = 0; k < CL; ++k)
          if (Mk[k] != -INFINITY) S += Sk[k] * (double)exp2f((float)(Mk[k] - M));
      const double lq = a.lq[q];
      const double lse2 = (M == -INFINITY) ? -INFINITY : M + log2(S);
      gS[q] = (lq == -INFINITY) ? -INFINITY : a.eps * lq - kep * lse2;
    }
    __syncthreads();
  }
  for (int r = t; r < nr; r += SNT) a.f[r0 + r] = fS[r];
  if (cr == 0)
    for (int64_t q = t; q < m; q += SNT) a.g[q] = gS[q];
  cluster_arrive();
  cluster_wait();  // no CTA exits while a peer may still read its partials
}

}  // namespace gw

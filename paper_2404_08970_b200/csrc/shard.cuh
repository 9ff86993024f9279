// shard.cuh -- the exchange steps of the row-sharded path.
//
// Rank r owns rows [row0_r, row0_r + nl_r) of T / G; ranks hold consecutive row ranges in rank
// order.  Every exchange is an all-gather of a small per-rank payload followed by a combine in
// rank order, so all ranks compute bit-identical replicated results and the result does not
// depend on the transport (NCCL or host callbacks).
//
//   column carries  : per column the state (sum_j T_jq, sum_j (x_ref - x_j) T_jq) of the ranks
//                     above (gap-weighted pair combine, the k = 1 DP of PAPER.md:237-243 with gaps)
//   block-strip     : the same for the per-strip sums of the row carries (k_blkscan_w tails)
//   row moments     : T 1 and the row-direction A_end are gathered whole (n doubles) and the 1-D
//                     DPs D_X (.) run over the global support
//   objective       : 8 partial sums per rank
//   Sinkhorn        : per-rank column sums (fused path) or per-column LSE pairs (safe path),
//                     merged in rank order
#pragma once
#include "common.cuh"

namespace gw {

// rank table on the device: tab[2r] = row0_r, tab[2r+1] = nl_r
// Exclusive column state of the ranks above `rank` (re-referenced to x_row0 of `rank`) and the
// global totals (referenced at x_{n-1}).  gath: [R][2m] = {btot_r (m), cxend_r (m)}.
__global__ void k_cols_ranks(const double* __restrict__ gath, int R, int rank, const int64_t* __restrict__ tab,
                             const double* __restrict__ xc, int64_t m, double* __restrict__ inP,
                             double* __restrict__ inX, double* __restrict__ btot, double* __restrict__ cxend) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  double CP = 0.0, CX = 0.0, s = 0.0;
  bool have = false;
  for (int r = 0; r < R; ++r) {
    if (r == rank) {
      inP[q] = CP;
      inX[q] = have ? CX + (xc[tab[2 * rank]] - s) * CP : 0.0;
    }
    const int64_t nlr = tab[2 * r + 1];
    if (nlr == 0) continue;
    const double P = gath[(int64_t)r * 2 * m + q], A = gath[(int64_t)r * 2 * m + m + q];
    const double ss = xc[tab[2 * r] + nlr - 1];
    if (!have) {
      CP = P; CX = A; s = ss; have = true;
    } else {
      CX = CX + (ss - s) * CP + A;
      CP += P;
      s = ss;
    }
  }
  btot[q] = CP;
  cxend[q] = CX;
}

// cS[b][q] += inP[q];  cX[b][q] += inX[q] + (x_{r0(b)} - x_row0) inP[q]
__global__ void k_cols_apply(int nb, int64_t m, const double* __restrict__ xl, const double* __restrict__ inP,
                             const double* __restrict__ inX, double* __restrict__ cS, double* __restrict__ cX) {
  const int64_t total = (int64_t)nb * m;
  const double x0 = xl[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / m, q = e - b * m;
    const double P = inP[q];
    cS[e] += P;
    cX[e] += inX[q] + (xl[b * 256] - x0) * P;
  }
}

// Block-strip tails: gath [R][ns][4] = {SP, SA, XP, XA} of each rank after its last block
// (referenced at its last row).  in4[s] = state of the ranks above, re-referenced to x_row0.
__global__ void k_bs_ranks(const double* __restrict__ gath, int R, int rank, const int64_t* __restrict__ tab,
                           const double* __restrict__ xc, int ns, double* __restrict__ in4) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  double SP = 0.0, SA = 0.0, XP = 0.0, XA = 0.0, ref = 0.0;
  bool have = false;
  for (int r = 0; r < rank; ++r) {
    const int64_t nlr = tab[2 * r + 1];
    if (nlr == 0) continue;
    const double* g = gath + ((int64_t)r * ns + s) * 4;
    const double ss = xc[tab[2 * r] + nlr - 1];
    if (!have) {
      SP = g[0]; SA = g[1]; XP = g[2]; XA = g[3]; ref = ss; have = true;
    } else {
      XP = XP + (ss - ref) * SP + g[2];
      XA = XA + (ss - ref) * SA + g[3];
      SP += g[0];
      SA += g[1];
      ref = ss;
    }
  }
  const double d = have ? xc[tab[2 * rank]] - ref : 0.0;
  in4[4 * s + 0] = SP;
  in4[4 * s + 1] = SA;
  in4[4 * s + 2] = XP + d * SP;
  in4[4 * s + 3] = XA + d * SA;
}

__global__ void k_bs_apply(int nb, int ns, const double* __restrict__ xl, const double* __restrict__ in4,
                           double* __restrict__ bs) {
  const int64_t total = (int64_t)nb * ns;
  const double x0 = xl[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / ns, s = e - b * ns;
    const double d = xl[b * 256] - x0;
    const double* v = in4 + 4 * s;
    double* o = bs + 4 * e;
    o[0] += v[0];
    o[1] += v[1];
    o[2] += v[2] + d * v[0];
    o[3] += v[3] + d * v[1];
  }
}

// gath [R][stride] (rank r's first nl_r entries are its rows) -> global vector v[row0_r + i]
__global__ void k_unpad(const double* __restrict__ gath, int R, int64_t stride, const int64_t* __restrict__ tab,
                        double* __restrict__ v) {
  for (int r = 0; r < R; ++r) {
    const int64_t r0 = tab[2 * r], nlr = tab[2 * r + 1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nlr; i += (int64_t)gridDim.x * blockDim.x)
      v[r0 + i] = gath[(int64_t)r * stride + i];
  }
}

// max over R gathered floats (violation), written to *out
__global__ void k_max_f(const float* __restrict__ gath, int R, float* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float v = 0.f;
    for (int r = 0; r < R; ++r) v = fmaxf(v, gath[r]);
    *out = v;
  }
}

}  // namespace gw

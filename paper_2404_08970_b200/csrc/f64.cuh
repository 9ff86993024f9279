// fp64 matrix storage (GW_F64; C1 = configs[0] runs with fp64 matrices, reading
// R28 as revised in round 2).  Every N x M matrix (T, G) is float64 and every step of the hot path
// runs in fp64: the paper's dynamic programme for G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y
// as a row scan (B = T D_Y) and a column scan (D_X B), and the
// log-domain Sinkhorn updates with max-shifted fp64 LSEs.
// k = 1 (|x - x'|) on 1-D supports.  This is the precision path (C1: parity ~1e-12 with the
// float64 oracle), not the bandwidth path: the plan is kept explicit (one more N x M buffer), rows
// are one warp each, columns one thread each over 64-row blocks, all loads coalesced.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "small.cuh"  // cluster helpers, SNT, ld_dsmem_f64

namespace gw {

constexpr int F64_RB = 64;  // rows per column block (column scans and column LSE partials)
constexpr int F64_CH = 16;  // rows whose loads a column thread issues before consuming them

// a marginal deviation for a max-reduction: NaN counts as +inf (fmax would drop it)
__device__ __forceinline__ double dev64(double d) { return d == d ? fabs(d) : INFINITY; }

// T^0 = p q^T (reading R5)
__global__ void k64_product(const double* __restrict__ pl, const double* __restrict__ q, int64_t nl, int64_t m,
                            double* __restrict__ T, int64_t ldT) {
  for (int64_t i = blockIdx.x; i < nl; i += gridDim.x) {
    const double pi = pl[i];
    for (int64_t p = threadIdx.x; p < m; p += blockDim.x) T[i * ldT + p] = pi * q[p];
  }
}

// T_ip = exp((f_i + g_p - G_ip) / eps): the Gibbs form of the subproblem's solution
__global__ void k64_gibbs(const double* __restrict__ G, int64_t ldG, const double* __restrict__ f,
                          const double* __restrict__ g, double eps, int64_t nl, int64_t m, double* __restrict__ T,
                          int64_t ldT) {
  for (int64_t i = blockIdx.x; i < nl; i += gridDim.x) {
    const double fi = f[i];
    for (int64_t p = threadIdx.x; p < m; p += blockDim.x) T[i * ldT + p] = exp((fi + g[p] - G[i * ldG + p]) / eps);
  }
}

// Supplied moments (gw_moments): row totals in the centred y coordinates, Q_c = T y - ymid T 1.
__global__ void k64_momrows(const double* __restrict__ rs, const double* __restrict__ rys, double ymid, int64_t nl,
                            double* __restrict__ rin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    rin[i] = rs[i];
    rin[nl + i] = rys[i] - ymid * rs[i];
  }
}
// ... and the column totals' sources for the 1-D DPs over y: T^T 1 and T^T x_c = T^T x - xmid T^T 1.
__global__ void k64_momcols(const double* __restrict__ cs, const double* __restrict__ cxs, double xmid, int64_t m,
                            double* __restrict__ v) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    v[p] = cs[p];
    v[m + p] = cxs[p] - xmid * cs[p];
  }
}

// Distance power k (|x - x'|^k, PAPER.md:229-259 / reading R17), with kappa_r = C(k, r) (-1)^r:
//   (D v)_p = sum_q |y_p - y_q|^k v_q = sum_r kappa_r y_p^(k-r) [S_r^<(p) + (-1)^k (S_r^tot - S_r^<(p))],
//   S_r^<(p) = sum_{q<p} y_q^r v_q   (the q = p term vanishes),
// i.e. odd k: sum_r kappa_r y_p^(k-r) (2 S_r^< - S_r^tot); even k: sum_r kappa_r y_p^(k-r) S_r^tot (no scan).
// k = 1 is the paper's gap recursion: 2 (y_p P_< - Q_<) + Q_tot - y_p P_tot.  Supports are centred.
__host__ __device__ constexpr double kappa64(int k, int r) {
  double c = 1.0;
  for (int j = 0; j < r; ++j) c = c * (k - j) / (j + 1);
  return (r & 1) ? -c : c;
}
template <int K>
__device__ __forceinline__ void pow64(double x, double (&v)[K + 1]) {
  v[0] = 1.0;
#pragma unroll
  for (int r = 1; r <= K; ++r) v[r] = v[r - 1] * x;
}

// a2, the row direction: B = T D_Y row by row, one warp per row, ONE read of the row.  Odd k: fp64
// warp scans of the k + 1 power sums with running carries; the kernel writes
// B'_ip = 2 sum_r kappa_r y_p^(k-r) S_r^<(p) and the row totals S_r^tot (the final carries); the column
// kernels add the deferred term -sum_r kappa_r y_p^(k-r) S_r^tot(i) when they read B' (b64 below).
// Even k: only the totals (B is then the deferred term alone; nothing is written).  B may alias T (each
// lane reads its element before writing it).  rin (nullable, k = 1): supplied totals [P_tot | Q_tot];
// rtot (out): [k + 1][nl].
template <int K>
__global__ void k64_row(const double* T, int64_t ldT, int64_t nl, int64_t m, const double* __restrict__ yc,
                        const double* __restrict__ rin, double* B, int64_t ldB, double* __restrict__ rtot) {
  constexpr int NS = K + 1;
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= nl) return;
  const double* t = T + i * ldT;
  double* b = B + i * ldB;
  double cr[NS];
#pragma unroll
  for (int r = 0; r < NS; ++r) cr[r] = 0.0;
  if (K % 2 == 0) {  // totals only
#pragma unroll 4
    for (int64_t p = lane; p < m; p += 32) {
      const double v = t[p], y = yc[p];
      double yp = 1.0;
#pragma unroll
      for (int r = 0; r < NS; ++r) {
        cr[r] += yp * v;
        yp *= y;
      }
    }
#pragma unroll
    for (int r = 0; r < NS; ++r) cr[r] = warp_sum(cr[r]);
  } else {
    constexpr int U = K == 1 ? 4 : 2;  // chunks of 32 columns loaded ahead of the (serial) scans
    for (int64_t p0 = 0; p0 < m; p0 += 32 * U) {
      double v[U], yv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + 32 * u + lane;
        v[u] = p < m ? t[p] : 0.0;
        yv[u] = p < m ? yc[p] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + 32 * u + lane;
        double yp[NS], a[NS];
        pow64<K>(yv[u], yp);
#pragma unroll
        for (int r = 0; r < NS; ++r) a[r] = yp[r] * v[u];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {  // inclusive warp scans
#pragma unroll
          for (int r = 0; r < NS; ++r) {
            const double o = __shfl_up_sync(0xffffffffu, a[r], d);
            if (lane >= d) a[r] += o;
          }
        }
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < NS; ++r) {
          double e = __shfl_up_sync(0xffffffffu, a[r], 1);
          if (lane == 0) e = 0.0;
          acc += kappa64(K, r) * yp[K - r] * (cr[r] + e);
          cr[r] += __shfl_sync(0xffffffffu, a[r], 31);
        }
        if (p < m) b[p] = 2.0 * acc;
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < NS; ++r) rtot[r * nl + i] = (K == 1 && rin) ? rin[r * nl + i] : cr[r];
  }
}

// B_ip: (odd k) B'_ip plus the deferred term, or (even k) the term alone; yq = powers of y_p
template <int K>
__device__ __forceinline__ double b64(double bp, const double* __restrict__ rtot, int64_t nl, int64_t i,
                                      const double (&yq)[K + 1]) {
  double d = 0.0;
#pragma unroll
  for (int r = 0; r <= K; ++r) d += kappa64(K, r) * yq[K - r] * rtot[r * nl + i];
  return (K & 1) ? bp - d : d;
}

// a3, the column direction: per 64-row block and column, the power sums
// S_r = sum_j x_j^r B_jp (r = 0..k) over the block's rows.  part: [nb][k + 1][m].
template <int K>
__global__ void k64_colpart(const double* __restrict__ B, int64_t ldB, int64_t nl, int64_t m,
                            const double* __restrict__ xl, const double* __restrict__ yc,
                            const double* __restrict__ rtot, double* __restrict__ part) {
  constexpr int NS = K + 1, CH = K == 1 ? F64_CH : 8;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t blk = blockIdx.y;
  if (p >= m) return;
  const int64_t i0 = blk * F64_RB, i1 = min(nl, i0 + F64_RB);
  double yq[NS];
  pow64<K>(yc[p], yq);
  double S[NS];
#pragma unroll
  for (int r = 0; r < NS; ++r) S[r] = 0.0;
  for (int64_t c0 = i0; c0 < i1; c0 += CH) {  // CH loads in flight per thread
    double bv[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) bv[u] = ((K & 1) && c0 + u < i1) ? B[(c0 + u) * ldB + p] : 0.0;
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c0 + u < i1) {
        const double bb = b64<K>(bv[u], rtot, nl, c0 + u, yq);
        const double x = xl[c0 + u];
        double xp = 1.0;
#pragma unroll
        for (int r = 0; r < NS; ++r) {
          S[r] += xp * bb;
          xp *= x;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NS; ++r) part[(NS * blk + r) * m + p] = S[r];
}

// Exclusive prefix of the block partials over blocks (in place, block order); tot = this rank's totals
// [NS][m].  One thread per column (coalesced across the warp), several blocks' loads in flight.
template <int NS>
__global__ void k64_colscan(double* __restrict__ part, int nb, int64_t m, double* __restrict__ tot) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= m) return;
  constexpr int CH = NS <= 2 ? 16 : 4;
  double S[NS];
#pragma unroll
  for (int r = 0; r < NS; ++r) S[r] = 0.0;
  for (int k0 = 0; k0 < nb; k0 += CH) {
    double v[CH][NS];
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int r = 0; r < NS; ++r) v[j][r] = k0 + j < nb ? part[(NS * (int64_t)(k0 + j) + r) * m + p] : 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (k0 + j < nb) {
#pragma unroll
        for (int r = 0; r < NS; ++r) {
          part[(NS * (int64_t)(k0 + j) + r) * m + p] = S[r];
          S[r] += v[j][r];
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NS; ++r) tot[r * m + p] = S[r];
}

// Row shards: off = sum of the ranks before this one, glob = sum over all ranks (rank order).
// gath: [R][len]; glob_set: the global totals were supplied (gw_moments): only off is written.
__global__ void k64_rankoff(const double* __restrict__ gath, int R, int rank, int64_t len, double* __restrict__ off,
                            double* __restrict__ glob, bool glob_set) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= len) return;
  double o = 0.0, t = 0.0;
  for (int r = 0; r < R; ++r) {
    const double v = gath[(int64_t)r * len + e];
    if (r < rank) o += v;
    t += v;
  }
  off[e] = o;
  if (!glob_set) glob[e] = t;
}

// a3 + a4: (D_X B)_ip = sum_r kappa_r x_i^(k-r) (odd k: 2 S_r^<(i) - S_r^tot; even k: S_r^tot) with the
// column power sums S_r of B, then G_ip = 2 (c_i + c'_p) - 4 (D_X T D_Y)_ip
// or, with the feature cost (Remark 2),
// (1 - alpha) C_ip^2 + alpha (2 (c_i + c'_p) - 4 (D_X T D_Y)_ip).  G holds B' (k64_row, odd k) on entry and
// is overwritten in place.  OBJ: per (block, column) partials of sum T (D_X T D_Y), sum T,
// sum T (ln T - 1), sum T C^2 into obj [nb][4][m] (T explicit, not aliased).
template <int K, bool OBJ, bool FGW>
__global__ void k64_colapply(double* G, int64_t ldG, const double* __restrict__ T, int64_t ldT, int64_t nl,
                             int64_t m, const double* __restrict__ xl, const double* __restrict__ part,
                             const double* __restrict__ off, const double* __restrict__ glob,
                             const double* __restrict__ cl, const double* __restrict__ c2,
                             const double* __restrict__ fxl, const double* __restrict__ fy, double alpha,
                             const double* __restrict__ yc, const double* __restrict__ rtot, double* __restrict__ obj) {
  constexpr int NS = K + 1;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t blk = blockIdx.y;
  if (p >= m) return;
  const int64_t i0 = blk * F64_RB, i1 = min(nl, i0 + F64_RB);
  double S[NS], St[NS], yq[NS];
#pragma unroll
  for (int r = 0; r < NS; ++r) {
    S[r] = off[r * m + p] + part[(NS * blk + r) * m + p];
    St[r] = glob[r * m + p];
  }
  pow64<K>(yc[p], yq);
  const double cp = c2[p];
  const double fyp = FGW ? fy[p] : 0.0;
  double o0 = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0;
  constexpr int CHA = K == 1 ? 8 : 4;  // (16 rows at k = 1: 168 registers, 18 % of the warps resident)
  for (int64_t c0 = i0; c0 < i1; c0 += CHA) {
    double bv[CHA], tv[CHA];
#pragma unroll
    for (int u = 0; u < CHA; ++u) {
      bv[u] = c0 + u < i1 ? G[(c0 + u) * ldG + p] : 0.0;
      if (OBJ) tv[u] = c0 + u < i1 ? T[(c0 + u) * ldT + p] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CHA; ++u) {
      const int64_t i = c0 + u;
      if (i >= i1) break;
      const double x = xl[i];
      const double b = b64<K>(bv[u], rtot, nl, i, yq);
      double xp[NS];
      pow64<K>(x, xp);
      double db = 0.0;
#pragma unroll
      for (int r = 0; r < NS; ++r) db += kappa64(K, r) * xp[K - r] * ((K & 1) ? 2.0 * S[r] - St[r] : St[r]);
#pragma unroll
      for (int r = 0; r < NS; ++r) S[r] += xp[r] * b;
      double gv = 2.0 * (cl[i] + cp) - 4.0 * db;
      double cc = 0.0;
      if (FGW) {
        const double d = fxl[i] - fyp;
        cc = d * d;
        gv = (1.0 - alpha) * cc + alpha * gv;
      }
      G[i * ldG + p] = gv;
      if (OBJ) {
        const double t = tv[u];
        o0 += t * db;
        o1 += t;
        if (t > 0.0) o2 += t * (log(t) - 1.0);
        o3 += t * cc;
      }
    }
  }
  if (OBJ) {
    obj[(4 * blk + 0) * m + p] = o0;
    obj[(4 * blk + 1) * m + p] = o1;
    obj[(4 * blk + 2) * m + p] = o2;
    obj[(4 * blk + 3) * m + p] = o3;
  }
}

// Objective pieces, step 1: per column, the block partials summed in block order.
// pay[p] = (T^T 1)_p over this rank's rows; tmp[k][p] (k = 0, 1, 2) = the column's sums of
// T (D_X T D_Y), T (ln T - 1), T C^2.
__global__ void k64_objcols(const double* __restrict__ obj, int nb, int64_t m, double* __restrict__ pay,
                            double* __restrict__ tmp) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= m) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int k = 0; k < nb; ++k) {
    s0 += obj[(4 * (int64_t)k + 0) * m + p];
    s1 += obj[(4 * (int64_t)k + 1) * m + p];
    s2 += obj[(4 * (int64_t)k + 2) * m + p];
    s3 += obj[(4 * (int64_t)k + 3) * m + p];
  }
  pay[p] = s1;
  tmp[p] = s0;
  tmp[m + p] = s2;
  tmp[2 * m + p] = s3;
}

__device__ __forceinline__ double bsum1024(double v, double* sm) { return block_sum<32, double>(v, sm); }
__device__ __forceinline__ double bmax1024(double v, double* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sm[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = warp_max(sm[lane]);
    if (lane == 0) sm[0] = t;
  }
  __syncthreads();
  t = sm[0];
  __syncthreads();
  return t;
}

constexpr int F64_PAYS = 16;  // scalars after the m column sums in the objective payload

// Objective pieces, step 2 (one CTA of 1024): this rank's scalars into pay[m .. m + 16):
//   {sum T DTD, sum T (ln T - 1), sum T C^2, max_i |a_i - p_i|, A_0 .. A_2k}
// with a = T 1 (the row pass's S_0^tot) and A_r = sum_i a_i x_i^r (centred x).
template <int K>
__global__ void __launch_bounds__(1024) k64_objlocal(const double* __restrict__ tmp, int64_t m, const double* __restrict__ a,
                             const double* __restrict__ xl, const double* __restrict__ pl, int64_t nl,
                             double* __restrict__ pay) {
  __shared__ double sm[32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
    s0 += tmp[p];
    s1 += tmp[m + p];
    s2 += tmp[2 * m + p];
  }
  double A[2 * K + 1], dv = 0.0;
#pragma unroll
  for (int r = 0; r <= 2 * K; ++r) A[r] = 0.0;
  for (int64_t i = threadIdx.x; i < nl; i += blockDim.x) {
    const double v = a[i], x = xl[i];
    double xp = v;
#pragma unroll
    for (int r = 0; r <= 2 * K; ++r) {
      A[r] += xp;
      xp *= x;
    }
    dv = fmax(dv, dev64(v - pl[i]));
  }
  s0 = bsum1024(s0, sm); s1 = bsum1024(s1, sm); s2 = bsum1024(s2, sm);
#pragma unroll
  for (int r = 0; r <= 2 * K; ++r) A[r] = bsum1024(A[r], sm);
  dv = bmax1024(dv, sm);
  if (threadIdx.x == 0) {
    double* o = pay + m;
    o[0] = s0; o[1] = s1; o[2] = s2; o[3] = dv;
#pragma unroll
    for (int r = 0; r <= 2 * K; ++r) o[4 + r] = A[r];
  }
}

// Objective pieces, step 3 (one CTA of 1024): the ranks' payloads [R][m + 16] combined in rank order;
//   E(T) = a (D_X o D_X) a + b (D_Y o D_Y) b - 2 <D_X T D_Y, T>
// with sum_ij |x_i - x_j|^2k a_i a_j = sum_r kappa_r(2k) A_(2k-r) A_r (an even power: no split), likewise
// b = T^T 1 over y.  out: [0] E, [1] max(|T1 - p|, |T^T 1 - q|), [3] H = sum T (ln T - 1), [6] sum T C^2.
template <int K>
__global__ void __launch_bounds__(1024) k64_objglobal(const double* __restrict__ gath, int R, int64_t m, const double* __restrict__ yc,
                              const double* __restrict__ qn, double* __restrict__ out) {
  __shared__ double sm[32];
  const int64_t st = m + F64_PAYS;
  double B[2 * K + 1], dv = 0.0;
#pragma unroll
  for (int r = 0; r <= 2 * K; ++r) B[r] = 0.0;
  for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
    double b = 0.0;
    for (int r = 0; r < R; ++r) b += gath[r * st + p];
    const double y = yc[p];
    double yp = b;
#pragma unroll
    for (int r = 0; r <= 2 * K; ++r) {
      B[r] += yp;
      yp *= y;
    }
    dv = fmax(dv, dev64(b - qn[p]));
  }
#pragma unroll
  for (int r = 0; r <= 2 * K; ++r) B[r] = bsum1024(B[r], sm);
  dv = bmax1024(dv, sm);
  if (threadIdx.x == 0) {
    double s[4 + 2 * K + 1];
    for (int k = 0; k < 4 + 2 * K + 1; ++k) s[k] = 0.0;
    for (int r = 0; r < R; ++r) {
      const double* o = gath + r * st + m;
      for (int k = 0; k < 4 + 2 * K + 1; ++k) s[k] = k == 3 ? fmax(s[3], o[3]) : s[k] + o[k];
    }
    double Ea = 0.0, Eb = 0.0;
    for (int r = 0; r <= 2 * K; ++r) {
      Ea += kappa64(2 * K, r) * s[4 + 2 * K - r] * s[4 + r];
      Eb += kappa64(2 * K, r) * B[2 * K - r] * B[r];
    }
    out[0] = Ea + Eb - 2.0 * s[0];
    out[1] = fmax(s[3], dv);
    out[2] = 0.0;
    out[3] = s[1];
    out[4] = out[5] = 0.0;
    out[6] = s[2];
    out[7] = 0.0;
  }
}

// ---- Sinkhorn, max-shifted log-sum-exp in fp64 ----------------
struct L64 {
  double m, s;  // max and sum of 2^(v - m), v in log2 units
};
__device__ __forceinline__ L64 l64_merge(L64 a, L64 b) {
  const double mx = fmax(a.m, b.m);
  if (mx == -INFINITY) return L64{-INFINITY, 0.0};
  return L64{mx, a.s * exp2(a.m - mx) + b.s * exp2(b.m - mx)};
}

// F values at once: one max, one rescale of the running sum, F exponentials
template <int F>
__device__ __forceinline__ void l64_chunk(L64& a, const double (&v)[F]) {
  double mx = v[0];
#pragma unroll
  for (int u = 1; u < F; ++u) mx = fmax(mx, v[u]);
  if (mx == -INFINITY) return;
  if (mx > a.m) {
    a.s *= exp2(a.m - mx);  // a.m = -inf: 0
    a.m = mx;
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < F; ++u) s += exp2(v[u] - a.m);
  a.s += s;
}

// The exponents are formed as (f_i + g_p - G_ip) * c2, c2 = log2(e) / eps (no fp64 division per element;
// 2^x instead of e^x), LSE = ln 2 (m + log2 s): within ~|v| ulp of the oracle's (.)/eps and exp.
// Rows, one warp each: LSE_p of v_p = (f_i + g_p - G_ip) / eps.
//   mode 0 (a5, f-update): f_i = eps ln p_i - eps LSE_p((g_p - G_ip) / eps)
//   mode 1 (violation):    dev_i = |sum_p T_ip - p_i| with T = exp((f + g - G) / eps)
__global__ void k64_rowlse(const double* __restrict__ G, int64_t ldG, int64_t nl, int64_t m,
                           const double* __restrict__ g, double eps, double* __restrict__ f,
                           const double* __restrict__ lpl, const double* __restrict__ pl, int mode,
                           double* __restrict__ dev) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= nl) return;
  const double fi = mode == 1 ? f[i] : 0.0;
  const double c2 = GW_LOG2E / eps;
  const double* Gi = G + i * ldG;
  L64 a{-INFINITY, 0.0};
  constexpr int U = 4;  // 4 coalesced warp loads in flight
  for (int64_t p0 = lane; p0 < m; p0 += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + 32 * u;
      v[u] = p < m ? Gi[p] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + 32 * u;
      v[u] = p < m ? (fi + g[p] - v[u]) * c2 : -INFINITY;
    }
    l64_chunk<U>(a, v);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    L64 o{__shfl_xor_sync(0xffffffffu, a.m, d), __shfl_xor_sync(0xffffffffu, a.s, d)};
    a = l64_merge(a, o);
  }
  if (lane == 0) {
    const double lse = (a.m + log2(a.s)) * GW_LN2;
    if (mode == 0) f[i] = eps * lpl[i] - eps * lse;
    else dev[i] = dev64(exp(lse) - pl[i]);
  }
}

// Columns: per (column, 64-row block) LSE pair of v_i = (f_i + g_p - G_ip) / eps (g nullable: 0).
__global__ void k64_colpart_lse(const double* __restrict__ G, int64_t ldG, int64_t nl, int64_t m,
                                const double* __restrict__ f, const double* __restrict__ g, double eps,
                                double2* __restrict__ part) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t blk = blockIdx.y;
  if (p >= m) return;
  const int64_t i0 = blk * F64_RB, i1 = min(nl, i0 + F64_RB);
  const double gp = g ? g[p] : 0.0;
  const double c2 = GW_LOG2E / eps;
  L64 a{-INFINITY, 0.0};
  constexpr int CH = 8;
  for (int64_t c0 = i0; c0 < i1; c0 += CH) {
    double v[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) v[u] = c0 + u < i1 ? G[(c0 + u) * ldG + p] : 0.0;
#pragma unroll
    for (int u = 0; u < CH; ++u) v[u] = c0 + u < i1 ? (f[c0 + u] + gp - v[u]) * c2 : -INFINITY;
    l64_chunk<CH>(a, v);
  }
  part[blk * m + p] = make_double2(a.m, a.s);
}
// The blocks' pairs merged (one warp per column: lane segments, then a fixed butterfly):
// pay[p] = max, pay[m + p] = sum (this rank's rows).
__global__ void k64_colcomb(const double2* __restrict__ part, int nb, int64_t m, double* __restrict__ pay) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (p >= m) return;
  L64 a{-INFINITY, 0.0};
  for (int k = lane; k < nb; k += 32) {
    const double2 v = part[(int64_t)k * m + p];
    a = l64_merge(a, L64{v.x, v.y});
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    L64 o{__shfl_xor_sync(0xffffffffu, a.m, d), __shfl_xor_sync(0xffffffffu, a.s, d)};
    a = l64_merge(a, o);
  }
  if (lane == 0) {
    pay[p] = a.m;
    pay[m + p] = a.s;
  }
}
// The ranks' pairs [R][stride] merged in rank order.
//   mode 0 (a6, g-update): g_p = eps ln q_p - eps LSE_i((f_i - G_ip) / eps)
//   mode 1 (violation):    dev_p = |sum_i T_ip - q_p|
__global__ void k64_colfinal(const double* __restrict__ gath, int R, int64_t stride, int64_t m, double eps,
                             const double* __restrict__ lq, const double* __restrict__ qn, double* __restrict__ g,
                             int mode, double* __restrict__ dev) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= m) return;
  L64 a{-INFINITY, 0.0};
  for (int r = 0; r < R; ++r) a = l64_merge(a, L64{gath[r * stride + p], gath[r * stride + m + p]});
  const double lse = (a.m + log2(a.s)) * GW_LN2;
  if (mode == 0) g[p] = eps * lq[p] - eps * lse;
  else dev[p] = dev64(exp(lse) - qn[p]);
}

// max of v[0 .. n) into *out (one CTA of 1024)
__global__ void __launch_bounds__(1024) k64_max(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double sm[32];
  double d = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d = fmax(d, v[i]);
  d = bmax1024(d, sm);
  if (threadIdx.x == 0) *out = d;
}
// violation = max(column deviations, every rank's row maximum gath[r * stride + 2m]) (one CTA of 1024)
__global__ void __launch_bounds__(1024) k64_viol(const double* __restrict__ coldev, int64_t m, const double* __restrict__ gath, int R,
                         int64_t stride, double* __restrict__ out) {
  __shared__ double sm[32];
  double d = 0.0;
  for (int64_t p = threadIdx.x; p < m; p += blockDim.x) d = fmax(d, coldev[p]);
  d = bmax1024(d, sm);
  if (threadIdx.x == 0) {
    for (int r = 0; r < R; ++r) d = fmax(d, gath[r * stride + 2 * m]);
    *out = d;
  }
}


// ---- cluster-resident fp64 Sinkhorn (small problems; C1) --------------------------------------------
// The fp64 analogue of small.cuh: G (this CTA's rows, fp64) in shared memory, ALL `iters` iterations of
// a fixed-count inner loop in one launch; per iteration the f-update (warp per own row, two-pass
// max-shifted LSE) and the g-update (thread per column: (max, sum) over the CTA's rows, one cluster
// barrier, the CL partials merged in CTA order through DSMEM, so g is bit-identical in every CTA).
// Same formulas as k64_rowlse / k64_colfinal: exponent (g_p - G_ip) log2e/eps in fp64, exp2 in fp64,
// LSE = ln 2 (max + log2 sum).
struct Small64Args {
  const double* G;
  int64_t ld, nl, m;
  int rows;  // rows per CTA (the last CTA may hold fewer)
  const double *lp, *lq;
  double eps;
  int iters;
  double *f, *g;  // in: warm start, out: final duals
};

// dynamic smem: Gs [rows][m] | gS [m] | part [2][2][m] (max, sum; double-buffered) | fS [rows] | lpS [rows]
__host__ __device__ inline size_t small64_smem_bytes(int rows, int64_t m) {
  return sizeof(double) * ((size_t)rows * m + 5 * (size_t)m + 2 * (size_t)rows);
}

__global__ void __launch_bounds__(SNT, 1) k64_sink_small(Small64Args a) {
  extern __shared__ __align__(16) double dsm[];
  const uint32_t cr = cluster_rank();
  const uint32_t CL = gridDim.x;  // one cluster: every CTA of the grid
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int NWp = SNT / 32;
  const int64_t m = a.m;
  const int64_t r0 = (int64_t)cr * a.rows;
  const int nr = (int)max((int64_t)0, min((int64_t)a.rows, a.nl - r0));
  double* Gs = dsm;
  double* gS = Gs + (size_t)a.rows * m;
  double* part = gS + m;  // [2 buffers][2 (max, sum)][m]
  double* fS = part + 4 * m;
  double* lpS = fS + a.rows;
  const double c2 = GW_LOG2E / a.eps;
  for (int r = 0; r < nr; ++r)
    for (int64_t q = t; q < m; q += SNT) Gs[(size_t)r * m + q] = a.G[(r0 + r) * a.ld + q];
  for (int64_t q = t; q < m; q += SNT) gS[q] = a.g[q];
  for (int r = t; r < nr; r += SNT) {
    fS[r] = a.f[r0 + r];
    lpS[r] = a.lp[r0 + r];
  }
  __syncthreads();
  cluster_arrive();
  cluster_wait();  // every CTA's shared memory is live before any DSMEM access
  for (int it = 0; it < a.iters; ++it) {
    for (int r = w; r < nr; r += NWp) {  // f-update
      const double* row = Gs + (size_t)r * m;
      double mx = -INFINITY;
      for (int64_t q = lane; q < m; q += 32) mx = fmax(mx, (gS[q] - row[q]) * c2);
      mx = warp_max(mx);
      double sm = 0.0;
      if (mx != -INFINITY)
        for (int64_t q = lane; q < m; q += 32) sm += exp2((gS[q] - row[q]) * c2 - mx);
      sm = warp_sum(sm);
      if (lane == 0) fS[r] = a.eps * lpS[r] - a.eps * ((mx + log2(sm)) * GW_LN2);
    }
    __syncthreads();
    double* pb = part + (size_t)(it & 1) * 2 * m;
    for (int64_t q = t; q < m; q += SNT) {  // g-update: this CTA's column partials
      double mx = -INFINITY;
      for (int r = 0; r < nr; ++r) mx = fmax(mx, (fS[r] - Gs[(size_t)r * m + q]) * c2);
      double sm = 0.0;
      if (mx != -INFINITY)
        for (int r = 0; r < nr; ++r) sm += exp2((fS[r] - Gs[(size_t)r * m + q]) * c2 - mx);
      pb[q] = mx;
      pb[m + q] = sm;
    }
    cluster_arrive();
    cluster_wait();  // every CTA's partials of this iteration are written
    for (int64_t q = t; q < m; q += SNT) {
      L64 acc{-INFINITY, 0.0};
      for (uint32_t k = 0; k < CL; ++k)
        acc = l64_merge(acc, L64{ld_dsmem_f64(mapa(pb + q, k)), ld_dsmem_f64(mapa(pb + m + q, k))});
      gS[q] = a.eps * a.lq[q] - a.eps * ((acc.m + log2(acc.s)) * GW_LN2);
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

// polyk.cuh -- the gradient for a general distance power k >= 3 (PAPER.md:65-80
// and the (k+1)-state recursion of PAPER.md:229-259; sorted supports by reading R1).
//
// Split each 1-D product at the diagonal.  For j < i, (x_i - x_j)^k = sum_r C(k,r) (-1)^r x_i^{k-r} x_j^r,
// and for j > i the same expansion carries the sign (-1)^k.  With the power sums S_r^<(i) =
// sum_{j<i} x_j^r v_j and their totals S_r:
//   (D v)_i = sum_r C(k,r) (-1)^r x_i^{k-r} (2 S_r^<(i) - S_r)    (k odd)
//           = sum_r C(k,r) (-1)^r x_i^{k-r} S_r                    (k even)
// (the diagonal contributes 0^k = 0 and may sit on either side).  These are the paper's k+1 states
// per position, carried as power sums about the centre of the support instead of
// gap-shifted binomial states: on centred supports every term of the recombination is O(width^k)
// (bounded cancellation), and every state and product is fp64.
//
// D_X T D_Y on GK x GK tiles:
//   k_gk_sums   per tile: row power sums (weights y^r) and column power sums (weights x^r) of T;
//   carries     exclusive prefix over column tiles per row (k_gk_scan_tiles); the column power sums of
//               W = T D_Y over row tiles are D_Y applied to T's column power sums (k_gk_apply on
//               (N/GK)(k+1) vectors of length M), then an exclusive prefix over row tiles;
//   k_gk_main   the tile in shared memory: a thread-per-row scan forms W (fp32, in place), then a
//               thread-per-column scan forms V = D_X W and G = 2c + 2c' - 4V (coalesced stores).
// Bytes: 2 reads + 1 write of the N x M matrix, plus ~3 (k+1) N M / GK fp64 carries.
#pragma once
#include "common.cuh"
#include "fused.cuh"  // ex2_ftz
#include "grad2.cuh"  // TSrc2, T_* modes

namespace gw {

constexpr int GK = 128;   // tile side = threads per CTA
constexpr int GKQ = GK + 4;  // smem row pitch in floats: 16-B rows for the bulk copies, and float4 row
                             // reads by a thread-per-row scan hit 8 distinct 16-B bank groups

__host__ __device__ constexpr double gk_binom(int n, int r) {
  double v = 1.0;
  for (int i = 1; i <= r; ++i) v = v * (double)(n - r + i) / (double)i;
  return v;
}

// one plan entry, the same fp32 expression as every other pass (grad2.cuh / poly.cuh)
template <int MODE>
__device__ __forceinline__ float gk_regen(const TSrc2& S, int64_t i, int64_t q, float gq, float glq) {
  if (MODE == T_EXPLICIT) return S.T[i * S.ld + q];
  if (MODE == T_PRODUCT) return S.fh[i] * gq;
  const float g = S.T[i * S.ld + q];
  const float a = (fmaf(g, -S.ch, gq) + S.fh[i]) + fmaf(g, -S.cl, glq + S.fl[i]);
  return ex2_ftz(a);
}

// powers s^r (r <= K) and recombination coefficients C(K,r) (-1)^r s^{K-r} of one coordinate
template <int K>
__device__ __forceinline__ void gk_powers(double s, double* pw, double* cf, int stride) {
  double v[K + 1];
  v[0] = 1.0;
#pragma unroll
  for (int r = 1; r <= K; ++r) v[r] = v[r - 1] * s;
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    pw[r * stride] = v[r];
    cf[r * stride] = ((r & 1) ? -1.0 : 1.0) * gk_binom(K, r) * v[K - r];
  }
}

// dynamic smem: the fp32 tile [GK][GKQ] first (16-B aligned), then fp64 tables
// kappa_r = C(K,r) (-1)^r: the scans carry kappa_r h_r so that sum_r kappa_r s^{K-r} h_r is a Horner
// evaluation in s (K FMAs, no coefficient tables)
template <int K>
__device__ __forceinline__ double gk_kappa(int r) { return ((r & 1) ? -1.0 : 1.0) * gk_binom(K, r); }

// acc_r += v s^r  (r = 0..K)
template <int K>
__device__ __forceinline__ void gk_accum(double (&acc)[K + 1], double v, double s) {
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    acc[r] += v;
    v *= s;
  }
}
// sum_r h~_r s^{K-r}
template <int K>
__device__ __forceinline__ double gk_horner(const double (&h)[K + 1], double s) {
  double v = h[0];
#pragma unroll
  for (int r = 1; r <= K; ++r) v = fma(v, s, h[r]);
  return v;
}
// h~_r += kappa_r v s^r
template <int K>
__device__ __forceinline__ void gk_update(double (&h)[K + 1], double v, double s) {
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    h[r] = fma(gk_kappa<K>(r), v, h[r]);
    v *= s;
  }
}

// dynamic smem: the fp32 tile [GK][GKQ] first (16-B aligned), then fp64 per-row / per-column values
constexpr size_t gk_smem_bytes() { return sizeof(float) * GK * GKQ + sizeof(double) * 4 * GK; }

// The plan tile [r0, r0 + GK) x [c0, c0 + GK) into shared memory, zero outside the matrix.  EXPLICIT /
// GIBBS: one bulk copy (cp.async.bulk, complete_tx on an mbarrier) per row, so the whole 64 KB tile is
// in flight at once; then each thread regenerates its column in place (GIBBS: the same fp32
// expression as every other pass).  PRODUCT: p_i q_q directly.
template <int MODE>
__device__ __forceinline__ void gk_load_tile(const TSrc2& S, int64_t nl, int64_t m, int64_t r0, int64_t c0,
                                             float* tile) {
  __shared__ uint64_t bar;
  __shared__ float fhs[GK], fls[GK];
  const int t = threadIdx.x;
  const int rows = (int)(nl - r0 < GK ? nl - r0 : GK);
  const int cols = (int)(m - c0 < GK ? m - c0 : GK);
  if (MODE != T_EXPLICIT) fhs[t] = t < rows ? S.fh[r0 + t] : 0.f;
  if (MODE == T_GIBBS) fls[t] = t < rows ? S.fl[r0 + t] : 0.f;
  if (MODE != T_PRODUCT) {
    const uint32_t rb = 4u * (uint32_t)((cols + 3) & ~3);  // ld % 4 == 0: stays inside the row
    if (t == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&bar, rb * (uint32_t)rows);
    }
    __syncthreads();
    if (t < rows) tma_load_1d(tile + t * GKQ, S.T + (r0 + t) * S.ld + c0, rb, &bar);
    mbar_wait(&bar, 0);
  } else {
    __syncthreads();
  }
  const bool qv = t < cols;
  float gq = 0.f, glq = 0.f;
  if (qv && MODE != T_EXPLICIT) gq = S.gh[c0 + t];
  if (qv && MODE == T_GIBBS) glq = S.gl[c0 + t];
#pragma unroll 4
  for (int rr = 0; rr < GK; ++rr) {
    float v = 0.f;
    if (qv && rr < rows) {
      if (MODE == T_EXPLICIT) {
        v = tile[rr * GKQ + t];
      } else if (MODE == T_PRODUCT) {
        v = fhs[rr] * gq;
      } else {
        const float g = tile[rr * GKQ + t];
        v = ex2_ftz((fmaf(g, -S.ch, gq) + fhs[rr]) + fmaf(g, -S.cl, glq + fls[rr]));
      }
    }
    tile[rr * GKQ + t] = v;
  }
}

// Pass 1: per tile (blockIdx.x = column tile, blockIdx.y = row tile)
//   colpart[ty][r][q] = sum_{i in tile rows} x_i^r T_iq,   rowpart[tx][r][i] = sum_{q in tile cols} y_q^r T_iq
template <int K, int MODE>
__global__ void __launch_bounds__(GK) k_gk_sums(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                const double* __restrict__ yc, double* __restrict__ rowpart,
                                                double* __restrict__ colpart) {
  extern __shared__ float4 gk_smem[];
  float* tile = reinterpret_cast<float*>(gk_smem);            // [GK][GKQ]
  double* xs = reinterpret_cast<double*>(tile + GK * GKQ);    // [GK] x of the tile's rows
  double* ys = xs + GK;                                       // [GK] y of the tile's columns
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * GK, c0 = (int64_t)blockIdx.x * GK;
  xs[t] = r0 + t < nl ? xl[r0 + t] : 0.0;
  ys[t] = c0 + t < m ? yc[c0 + t] : 0.0;
  gk_load_tile<MODE>(S, nl, m, r0, c0, tile);
  __syncthreads();
  double U[K + 1];
#pragma unroll
  for (int r = 0; r <= K; ++r) U[r] = 0.0;
  for (int rr = 0; rr < GK; ++rr) gk_accum<K>(U, (double)tile[rr * GKQ + t], xs[rr]);
  if (c0 + t < m)
#pragma unroll
    for (int r = 0; r <= K; ++r) colpart[((int64_t)blockIdx.y * (K + 1) + r) * m + c0 + t] = U[r];
#pragma unroll
  for (int r = 0; r <= K; ++r) U[r] = 0.0;
  for (int c = 0; c < GK; c += 4) {
    const float4 t4 = *reinterpret_cast<const float4*>(tile + t * GKQ + c);
    gk_accum<K>(U, (double)t4.x, ys[c]);
    gk_accum<K>(U, (double)t4.y, ys[c + 1]);
    gk_accum<K>(U, (double)t4.z, ys[c + 2]);
    gk_accum<K>(U, (double)t4.w, ys[c + 3]);
  }
  if (r0 + t < nl)
#pragma unroll
    for (int r = 0; r <= K; ++r) rowpart[((int64_t)blockIdx.x * (K + 1) + r) * nl + r0 + t] = U[r];
}

// In-place exclusive prefix over the tile index of part[nt][len2] (fixed order); totals -> tot[len2].
// Eight tiles' loads are issued before their stores (independent addresses, latency overlapped).
__global__ void k_gk_scan_tiles(double* __restrict__ part, int nt, int64_t len2, double* __restrict__ tot) {
  constexpr int U = 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len2; e += (int64_t)gridDim.x * blockDim.x) {
    double run = 0.0;
    for (int k0 = 0; k0 < nt; k0 += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = k0 + u < nt ? part[(int64_t)(k0 + u) * len2 + e] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u < nt) part[(int64_t)(k0 + u) * len2 + e] = run;
        run += v[u];
      }
    }
    tot[e] = run;
  }
}

// The same exclusive prefix over tiles, segmented for parallelism (the sequential walk over hundreds of
// tiles per element is load-latency bound): the nt tiles are split into nseg segments; pass A sums each
// segment (segtot[seg][e]), pass B adds the segments before it (fixed order) and walks its own tiles.
// Fixed summation order -> deterministic.
__global__ void k_gk_scan_seg_a(const double* __restrict__ part, int nt, int64_t len2, int nseg,
                                double* __restrict__ segtot) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int sg = blockIdx.y;
  if (e >= len2) return;
  const int per = (nt + nseg - 1) / nseg, t0 = sg * per, t1 = min(nt, t0 + per);
  constexpr int U = 8;
  double run = 0.0;
  for (int k0 = t0; k0 < t1; k0 += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = k0 + u < t1 ? part[(int64_t)(k0 + u) * len2 + e] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) run += v[u];
  }
  segtot[(int64_t)sg * len2 + e] = run;
}
__global__ void k_gk_scan_seg_b(double* __restrict__ part, int nt, int64_t len2, int nseg,
                                const double* __restrict__ segtot, double* __restrict__ tot) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int sg = blockIdx.y;
  if (e >= len2) return;
  const int per = (nt + nseg - 1) / nseg, t0 = sg * per, t1 = min(nt, t0 + per);
  double run = 0.0;
  for (int s2 = 0; s2 < sg; ++s2) run += segtot[(int64_t)s2 * len2 + e];
  constexpr int U = 8;
  for (int k0 = t0; k0 < t1; k0 += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = k0 + u < t1 ? part[(int64_t)(k0 + u) * len2 + e] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k0 + u < t1) part[(int64_t)(k0 + u) * len2 + e] = run;
      run += v[u];
    }
  }
  if (sg == nseg - 1) {
    double all = 0.0;
    for (int s2 = 0; s2 < nseg; ++s2) all += segtot[(int64_t)s2 * len2 + e];
    tot[e] = all;
  }
}

// Z[b] = D^(K) U[b] along a sorted centred support s (length m), one CTA per vector: a totals sweep,
// then a chunked block scan of the K+1 power sums (8 consecutive entries per thread per step).
template <int K>
__global__ void __launch_bounds__(256) k_gk_apply(const double* __restrict__ U, int64_t m,
                                                  const double* __restrict__ s, double* __restrict__ Z) {
  constexpr int NT = 256, E = 8, STEP = NT * E;
  __shared__ double wsum[NT / 32][K + 1];
  __shared__ double sm[32];
  const double* u = U + (int64_t)blockIdx.x * m;
  double* z = Z + (int64_t)blockIdx.x * m;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double tot[K + 1];
  {
    double acc[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) acc[r] = 0.0;
    for (int64_t q = t; q < m; q += NT) {
      const double y = s[q];
      double v = u[q];
#pragma unroll
      for (int r = 0; r <= K; ++r) {
        acc[r] += v;
        v *= y;
      }
    }
#pragma unroll
    for (int r = 0; r <= K; ++r) tot[r] = block_sum<NT / 32>(acc[r], sm);
  }
  double carry[K + 1];
#pragma unroll
  for (int r = 0; r <= K; ++r) carry[r] = 0.0;
  for (int64_t base = 0; base < m; base += STEP) {
    const int64_t q0 = base + (int64_t)t * E;
    double uv[E], sv[E], loc[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) loc[r] = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t q = q0 + e;
      uv[e] = q < m ? u[q] : 0.0;
      sv[e] = q < m ? s[q] : 0.0;
      double v = uv[e];
#pragma unroll
      for (int r = 0; r <= K; ++r) {
        loc[r] += v;
        v *= sv[e];
      }
    }
    double inc[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      double v = loc[r];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
      }
      inc[r] = v;
      if (lane == 31) wsum[w][r] = v;
    }
    __syncthreads();
    double run[K + 1], btot[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      double pre = 0.0, all = 0.0;
      for (int ww = 0; ww < NT / 32; ++ww) {
        if (ww < w) pre += wsum[ww][r];
        all += wsum[ww][r];
      }
      run[r] = carry[r] + pre + (inc[r] - loc[r]);
      btot[r] = all;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t q = q0 + e;
      double pw[K + 1], cf[K + 1];
      gk_powers<K>(sv[e], pw, cf, 1);
      double zv = 0.0;
#pragma unroll
      for (int r = 0; r <= K; ++r) zv = fma(cf[r], (K & 1) ? 2.0 * run[r] - tot[r] : tot[r], zv);
      if (q < m) z[q] = zv;
#pragma unroll
      for (int r = 0; r <= K; ++r) run[r] = fma(pw[r], uv[e], run[r]);
    }
#pragma unroll
    for (int r = 0; r <= K; ++r) carry[r] += btot[r];
  }
}

// Pass 2: G = alpha (2c 1^T + 2 1 c'^T - 4 D_X T D_Y) [+ (1 - alpha)(fx_i - fy_q)^2]  (STORE)
// and / or the tile's <D_X T D_Y, T> (OBJ -> tile_obj[tile]).
//   rowpre[tx][r][i], rowtot[r][i]: power sums of row i over the columns before tile tx / all columns
//   colpre[ty][r][q], coltot[r][q]: power sums (weights x^r) of column q of W = T D_Y over the rows
//                                   before row tile ty (this rank) / all rows (all ranks)
//   colcarry[r][q] (nullable): the same sums over the rows of the ranks above
template <int K, int MODE, bool STORE, bool OBJ, bool FGW>
__global__ void __launch_bounds__(GK) k_gk_main(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                const double* __restrict__ yc, const double* __restrict__ rowpre,
                                                const double* __restrict__ rowtot, const double* __restrict__ colpre,
                                                const double* __restrict__ coltot, const double* __restrict__ cl,
                                                const double* __restrict__ c2, double alpha,
                                                const double* __restrict__ fx, const double* __restrict__ fy,
                                                float* __restrict__ G, int64_t ldG, double* __restrict__ tile_obj,
                                                const double* __restrict__ colcarry) {
  extern __shared__ float4 gk_smem[];
  float* tile = reinterpret_cast<float*>(gk_smem);          // [GK][GKQ]
  double* xs = reinterpret_cast<double*>(tile + GK * GKQ);  // x of the tile's rows
  double* ys = xs + GK;                                     // y of the tile's columns
  double* crow = ys + GK;                                   // 2 alpha c_i
  double* frow = crow + GK;                                 // fx_i
  constexpr bool ODD = K & 1;
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * GK, c0 = (int64_t)blockIdx.x * GK;
  const int64_t i_t = r0 + t, q = c0 + t;
  xs[t] = i_t < nl ? xl[i_t] : 0.0;
  ys[t] = q < m ? yc[q] : 0.0;
  crow[t] = i_t < nl ? 2.0 * alpha * cl[i_t] : 0.0;
  frow[t] = (FGW && i_t < nl) ? fx[i_t] : 0.0;
  gk_load_tile<MODE>(S, nl, m, r0, c0, tile);
  __syncthreads();
  // thread = row: W_iq = sum_r kappa_r y_q^{K-r} h_r,  h_r = 2 S_r^<(q) - S_r (odd k) or S_r (even k)
  if (i_t < nl) {
    double h[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      const double tt = rowtot[(int64_t)r * nl + i_t];
      h[r] = gk_kappa<K>(r) * (ODD ? 2.0 * rowpre[((int64_t)blockIdx.x * (K + 1) + r) * nl + i_t] - tt : tt);
    }
    float* trow = tile + t * GKQ;
    for (int c = 0; c < GK; c += 4) {
      const float4 t4 = *reinterpret_cast<const float4*>(trow + c);
      const double tv[4] = {(double)t4.x, (double)t4.y, (double)t4.z, (double)t4.w};
      float wo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double y = ys[c + e];
        wo[e] = (float)gk_horner<K>(h, y);
        if (ODD) gk_update<K>(h, 2.0 * tv[e], y);
      }
      *reinterpret_cast<float4*>(trow + c) = make_float4(wo[0], wo[1], wo[2], wo[3]);
    }
  }
  __syncthreads();
  // thread = column: V_iq = sum_r kappa_r x_i^{K-r} h'_r,  h'_r from the column power sums of W
  double acc = 0.0;
  if (q < m) {
    double h[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
      const double tt = coltot[(int64_t)r * m + q];
      double pre = colpre[((int64_t)blockIdx.y * (K + 1) + r) * m + q];
      if (colcarry) pre += colcarry[(int64_t)r * m + q];  // rows of the ranks above
      h[r] = gk_kappa<K>(r) * (ODD ? 2.0 * pre - tt : tt);
    }
    const double c2q = 2.0 * alpha * c2[q];
    const double fyq = FGW ? fy[q] : 0.0;
    const double a4 = -4.0 * alpha, a1 = 1.0 - alpha;
    float gq = 0.f, glq = 0.f;
    if (OBJ && MODE != T_EXPLICIT) gq = S.gh[q];
    if (OBJ && MODE == T_GIBBS) glq = S.gl[q];
    const int rows = (int)(nl - r0 < GK ? nl - r0 : GK);
    for (int rr = 0; rr < rows; ++rr) {
      const double x = xs[rr];
      const double v = gk_horner<K>(h, x);
      if (ODD) gk_update<K>(h, 2.0 * (double)tile[rr * GKQ + t], x);
      const int64_t i = r0 + rr;
      if (OBJ) acc = fma(v, (double)gk_regen<MODE>(S, i, q, gq, glq), acc);
      if (STORE) {
        double g = fma(a4, v, crow[rr] + c2q);
        if (FGW) {
          const double d = frow[rr] - fyq;
          g = fma(a1 * d, d, g);
        }
        G[i * ldG + q] = (float)g;
      }
    }
  }
  if (OBJ) {
    __shared__ double sm[32];
    acc = block_sum<GK / 32>(acc, sm);
    if (t == 0) tile_obj[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = acc;
  }
}

// c = (D o D) w for D = |s - s'|^K, i.e. the even power P = 2K: sum_r C(P,r) (-1)^r s_i^{P-r} mu_r with
// mu_r = sum_j s_j^r w_j (centred supports; one CTA, fixed-order reductions).
template <int P>
__global__ void __launch_bounds__(1024) k_gk_const(const double* __restrict__ s, const double* __restrict__ w,
                                                   int64_t n, double* __restrict__ c) {
  __shared__ double sm[32];
  __shared__ double mu[P + 1];
  double acc[P + 1];
#pragma unroll
  for (int r = 0; r <= P; ++r) acc[r] = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double v = w[i];
    const double si = s[i];
#pragma unroll
    for (int r = 0; r <= P; ++r) {
      acc[r] += v;
      v *= si;
    }
  }
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    const double v = block_sum<32>(acc[r], sm);
    if (threadIdx.x == 0) mu[r] = v;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = s[i];
    double v = 0.0, sp = 1.0;
    for (int r = P; r >= 0; --r) {  // sum_r C(P,r) (-1)^r mu_r s_i^{P-r}, from r = P down
      v += ((r & 1) ? -1.0 : 1.0) * gk_binom(P, r) * mu[r] * sp;
      sp *= si;
    }
    c[i] = v;
  }
}

// E(T) = a^T (D_X o D_X) a + b^T (D_Y o D_Y) b - 2 <D_X T D_Y, T>  with a = T1, b = T^T 1 (realised).
// The power-2K quadratic forms by moments: sum_r C(P,r) (-1)^r mu_r mu_{P-r}.
// Partial (per rank): part = {mu_0(a) .. mu_P(a) over this rank's rows, sum of the tile <V, T> sums}.
template <int K>
__global__ void __launch_bounds__(1024) k_gk_obj_partial(const double* __restrict__ a, const double* __restrict__ xl,
                                                         int64_t nl, const double* __restrict__ tile_obj,
                                                         int64_t ntile, double* __restrict__ part) {
  constexpr int P = 2 * K;
  __shared__ double sm[32];
  double ua[P + 1];
#pragma unroll
  for (int r = 0; r <= P; ++r) ua[r] = 0.0;
  for (int64_t i = threadIdx.x; i < nl; i += blockDim.x) {
    double v = a[i];
    const double x = xl[i];
#pragma unroll
    for (int r = 0; r <= P; ++r) {
      ua[r] += v;
      v *= x;
    }
  }
  double go = 0.0;
  for (int64_t i = threadIdx.x; i < ntile; i += blockDim.x) go += tile_obj[i];
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    const double v = block_sum<32>(ua[r], sm);
    if (threadIdx.x == 0) part[r] = v;
  }
  go = block_sum<32>(go, sm);
  if (threadIdx.x == 0) part[P + 1] = go;
}

// Final: the R ranks' partials (gathered [R][P + 2]) summed in rank order; b = T^T 1 over all
// rows (bparts [R][m], summed in rank order) -> out[0] = E.
template <int K>
__global__ void __launch_bounds__(1024) k_gk_obj_final(const double* __restrict__ parts, int R,
                                                       const double* __restrict__ bparts, const double* __restrict__ yc,
                                                       int64_t m, double* __restrict__ out) {
  constexpr int P = 2 * K;
  __shared__ double sm[32];
  __shared__ double mub[P + 1];
  double ub[P + 1];
#pragma unroll
  for (int r = 0; r <= P; ++r) ub[r] = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    double v = 0.0;
    for (int rk = 0; rk < R; ++rk) v += bparts[(int64_t)rk * m + i];
    const double y = yc[i];
#pragma unroll
    for (int r = 0; r <= P; ++r) {
      ub[r] += v;
      v *= y;
    }
  }
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    const double v = block_sum<32>(ub[r], sm);
    if (threadIdx.x == 0) mub[r] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mua[P + 1], go = 0.0;
    for (int r = 0; r <= P; ++r) mua[r] = 0.0;
    for (int rk = 0; rk < R; ++rk) {
      for (int r = 0; r <= P; ++r) mua[r] += parts[(int64_t)rk * (P + 2) + r];
      go += parts[(int64_t)rk * (P + 2) + P + 1];
    }
    double Ea = 0.0, Eb = 0.0;
    for (int r = 0; r <= P; ++r) {
      const double cf = ((r & 1) ? -1.0 : 1.0) * gk_binom(P, r);
      Ea += cf * mua[r] * mua[P - r];
      Eb += cf * mub[r] * mub[P - r];
    }
    out[0] = Ea + Eb - 2.0 * go;
  }
}

// Multi-rank column carries: g = [R][len] (each rank's column totals); carry = sum over the ranks
// before `rank`, tot = sum over all (rank order).
__global__ void k_gk_ranks(const double* __restrict__ g, int R, int rank, int64_t len, double* __restrict__ carry,
                           double* __restrict__ tot) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    double c = 0.0, t = 0.0;
    for (int r = 0; r < R; ++r) {
      const double v = g[(int64_t)r * len + e];
      if (r < rank) c += v;
      t += v;
    }
    carry[e] = c;
    tot[e] = t;
  }
}

}  // namespace gw

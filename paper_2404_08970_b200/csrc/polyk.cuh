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
// D_X T D_Y on GR x GR regions (one CTA each, staged through shared memory as 2 x 2 tiles of GK x GK):
//   k_gk_sums   per region: row power sums (weights y^r) and column power sums (weights x^r) of T;
//   carries     exclusive prefix over column regions per row (k_gk_scan_tiles); the column power sums
//               of W = T D_Y over row regions are D_Y applied to T's column power sums (k_gk_apply on
//               (N/GR)(k+1) vectors of length M), then an exclusive prefix over row regions;
//   k_gk_main   per tile in shared memory: a thread-per-row scan forms W (fp32, in place), then a
//               thread-per-column scan forms V = D_X W and G = 2c + 2c' - 4V (coalesced stores).
// Bytes: 2 reads + 1 write of the N x M matrix, plus ~3 (k+1) N M / GR fp64 carries.
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

// Tile-centred fp32 arithmetic.  Inside a GK x GK tile every power and every state is taken about the
// centre of the tile's own coordinate range (cx: the tile's rows, cy: its columns), so |x - cx| is at
// most half the tile's width: the recombination sum_j a_j s^j of a tile-centred polynomial has no
// cancellation beyond the terms' own size (a_0 = the value at the centre dominates), and fp32 state +
// fp32 FFMA give errors of a few fp32 ulps of (width^k x mass), far inside the gradient tolerance.  The
// cross-tile carries stay in fp64 about the global centre; each thread converts them to its tile's
// centre once per tile (a Taylor shift, O(k^2) fp64 operations per row or column per tile).
//
// per-coordinate table stride in floats (K + 1 values, padded for 8-B / 16-B shared loads)
template <int K>
__host__ __device__ constexpr int gk_kp() { return (K + 1 + 1) & ~1; }

// dynamic smem: the fp32 tile [GK][GKQ] first (16-B aligned), then one fp32 table [GK][KP] (rebuilt
// between the row and the column pass) and five fp32 per-coordinate vectors [GK]; with the static
// shared memory at most 73.5 KB (k = 5): three CTAs per SM
template <int K>
constexpr size_t gk_smem_bytes() { return sizeof(float) * (GK * GKQ + GK * gk_kp<K>() + 5 * GK); }

// Taylor shift in fp64: c[0..K] ascending coefficients of P(y) -> those of P(c + s) in s
template <int K>
__device__ __forceinline__ void gk_shift(double (&a)[K + 1], double c) {
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = K - 1; j >= i; --j) a[j] = fma(c, a[j + 1], a[j]);
}

// KP consecutive fp32 table entries (16-B loads when KP % 4 == 0, else 8-B)
template <int KP>
__device__ __forceinline__ void gk_ld_tab(const float* p, float (&v)[KP]) {
  if constexpr (KP % 4 == 0) {
#pragma unroll
    for (int i = 0; i < KP; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(p + i);
      v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < KP; i += 2) {
      const float2 t = *reinterpret_cast<const float2*>(p + i);
      v[i] = t.x; v[i + 1] = t.y;
    }
  }
}

// sum_j a_j s^j (fp32 Horner)
template <int K>
__device__ __forceinline__ float gk_horner_f(const float (&a)[K + 1], float s) {
  float v = a[K];
#pragma unroll
  for (int j = K - 1; j >= 0; --j) v = fmaf(v, s, a[j]);
  return v;
}

// centre of the sorted coordinates v[i0 .. i0 + cnt) (0 for an empty range)
__device__ __forceinline__ double gk_centre(const double* __restrict__ v, int64_t i0, int cnt) {
  return cnt > 0 ? 0.5 * (v[i0] + v[i0 + cnt - 1]) : 0.0;
}

// The plan tile [r0, r0 + GK) x [c0, c0 + GK) into shared memory, zero outside the matrix.  EXPLICIT /
// GIBBS: one bulk copy (cp.async.bulk, complete_tx on the mbarrier `bar`, phase `parity`) per row, so
// the whole 64 KB tile is in flight at once; then each thread regenerates its column in place (GIBBS:
// the same fp32 expression as every other pass).  PRODUCT: p_i q_q directly.  The caller has passed a
// barrier after every thread's last access to `tile` (and fenced its generic writes to the async proxy).
template <int MODE>
__device__ __forceinline__ void gk_load_tile(const TSrc2& S, int64_t nl, int64_t m, int64_t r0, int64_t c0,
                                             float* tile, uint64_t* bar, uint32_t parity) {
  __shared__ float fhs[GK], fls[GK];
  const int t = threadIdx.x;
  const int rows = (int)(nl - r0 < GK ? nl - r0 : GK);
  const int cols = (int)(m - c0 < GK ? m - c0 : GK);
  if (MODE != T_EXPLICIT) fhs[t] = t < rows ? S.fh[r0 + t] : 0.f;
  if (MODE == T_GIBBS) fls[t] = t < rows ? S.fl[r0 + t] : 0.f;
  if (MODE != T_PRODUCT) {
    const uint32_t rb = 4u * (uint32_t)((cols + 3) & ~3);  // ld % 4 == 0: stays inside the row
    if (t == 0) mbar_expect_tx(bar, rb * (uint32_t)rows);
    __syncthreads();
    if (t < rows) tma_load_1d(tile + t * GKQ, S.T + (r0 + t) * S.ld + c0, rb, bar);
    mbar_wait(bar, parity);
  } else {
    __syncthreads();
  }
  const bool qv = t < cols;
  if (MODE == T_EXPLICIT) {
    // the bulk copies filled [0, rows) x [0, 4 ceil(cols / 4)); only a ragged tile has entries to zero
    if (rows < GK || cols < GK) {
      for (int rr = 0; rr < GK; ++rr)
        if (!qv || rr >= rows) tile[rr * GKQ + t] = 0.f;
    }
    return;
  }
  float gq = 0.f, glq = 0.f;
  if (qv) gq = S.gh[c0 + t];
  if (qv && MODE == T_GIBBS) glq = S.gl[c0 + t];
#pragma unroll 4
  for (int rr = 0; rr < GK; ++rr) {
    float v = 0.f;
    if (qv && rr < rows) {
      if (MODE == T_PRODUCT) {
        v = fhs[rr] * gq;
      } else {
        const float g = tile[rr * GKQ + t];
        v = ex2_ftz((fmaf(g, -S.ch, gq) + fhs[rr]) + fmaf(g, -S.cl, glq + fls[rr]));
      }
    }
    tile[rr * GKQ + t] = v;
  }
}

// A CTA owns a GR x GR region (GNS x GNS tiles of GK x GK, staged through shared memory one tile at a
// time): the carries between CTAs are per region, 1 / GNS as many as per tile, and the states are taken
// about the region's centres (|x - cx| <= half the region's width).
constexpr int GNS = 4;        // tiles per region side
constexpr int GR = GNS * GK;  // region side

// before a tile buffer is refilled: generic-proxy writes to it ordered before the async-proxy (TMA)
// writes, and every thread past its last read
__device__ __forceinline__ void gk_tile_release() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

// sum_j C(r,j) c^{r-j} d_j for r = 0..K (the power sums of the centred coordinates about 0)
template <int K>
__device__ __forceinline__ void gk_uncentre(const double (&u)[K + 1], double c, double (&o)[K + 1]) {
#pragma unroll
  for (int r = 0; r <= K; ++r) {
    double v = 0.0, cp = 1.0;
#pragma unroll
    for (int j = r; j >= 0; --j) {
      v = fma(gk_binom(r, j) * cp, u[j], v);
      cp *= c;
    }
    o[r] = v;
  }
}

// Pass 1: per region (blockIdx.x = column region, blockIdx.y = row region)
//   colpart[ry][r][q] = sum_{i in region rows} x_i^r T_iq,   rowpart[rx][r][i] = sum_{q in region cols} y_q^r T_iq
// (global centred coordinates, fp64), accumulated in fp32 about the region's centres and shifted back:
//   sum_i x_i^r T_iq = sum_j C(r,j) cx^{r-j} U_j,  U_j = sum_i (x_i - cx)^j T_iq.
template <int K, int MODE>
__global__ void __launch_bounds__(GK) k_gk_sums(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                const double* __restrict__ yc, double* __restrict__ rowpart,
                                                double* __restrict__ colpart) {
  constexpr int KP = gk_kp<K>();
  extern __shared__ float4 gk_smem[];
  __shared__ uint64_t bar;
  float* tile = reinterpret_cast<float*>(gk_smem);  // [GK][GKQ]
  float* pwt = tile + GK * GKQ;                      // [GK][KP] (x_i - cx)^j, then (y_q - cy)^j
  const int t = threadIdx.x;
  const int64_t R0 = (int64_t)blockIdx.y * GR, C0 = (int64_t)blockIdx.x * GR;
  const double cx = gk_centre(xl, R0, (int)min((int64_t)GR, nl - R0));
  const double cy = gk_centre(yc, C0, (int)min((int64_t)GR, m - C0));
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto powers = [&](float sv) {
    float pv = 1.f;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      pwt[t * KP + j] = j <= K ? pv : 0.f;
      pv *= sv;
    }
  };
  // column sums of the region's column tiles over all its row tiles: each tile's fp32 partial is folded
  // into an fp64 accumulator (the fp32 sums run over 128 terms at most)
  double U[GNS][K + 1];
#pragma unroll
  for (int cs = 0; cs < GNS; ++cs)
#pragma unroll
    for (int j = 0; j <= K; ++j) U[cs][j] = 0.0;
  uint32_t ph = 0;
#pragma unroll 1
  for (int rs = 0; rs < GNS; ++rs) {
    const int64_t r0 = R0 + rs * GK;
    if (r0 >= nl) break;  // uniform
    const int rows = (int)min((int64_t)GK, nl - r0);
    double R[K + 1];  // row sums of row r0 + t over the region's column tiles (fp64 fold per tile)
#pragma unroll
    for (int j = 0; j <= K; ++j) R[j] = 0.0;
#pragma unroll
    for (int cs = 0; cs < GNS; ++cs) {
      const int64_t c0 = C0 + cs * GK;
      if (c0 >= m) break;  // uniform
      const int cols = (int)min((int64_t)GK, m - c0);
      gk_tile_release();
      powers(t < rows ? (float)(xl[r0 + t] - cx) : 0.f);
      gk_load_tile<MODE>(S, nl, m, r0, c0, tile, &bar, ph);
      if (MODE != T_PRODUCT) ph ^= 1u;
      __syncthreads();
      // thread = column t: U_j += sum_rr (x_rr - cx)^j T[rr][t]
      {
        float u[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) u[j] = 0.f;
#pragma unroll 4
        for (int rr = 0; rr < GK; ++rr) {
          float pw[KP];
          gk_ld_tab<KP>(pwt + rr * KP, pw);
          const float v = tile[rr * GKQ + t];
#pragma unroll
          for (int j = 0; j <= K; ++j) u[j] = fmaf(v, pw[j], u[j]);
        }
#pragma unroll
        for (int j = 0; j <= K; ++j) U[cs][j] += (double)u[j];
      }
      __syncthreads();
      powers(t < cols ? (float)(yc[c0 + t] - cy) : 0.f);
      __syncthreads();
      // thread = row t: R_j += sum_c (y_c - cy)^j T[t][c]
      {
        float u[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) u[j] = 0.f;
        const float* trow = tile + t * GKQ;
#pragma unroll 2
        for (int cc = 0; cc < GK; cc += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(trow + cc);
          const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float pw[KP];
            gk_ld_tab<KP>(pwt + (cc + e) * KP, pw);
#pragma unroll
            for (int j = 0; j <= K; ++j) u[j] = fmaf(tv[e], pw[j], u[j]);
          }
        }
#pragma unroll
        for (int j = 0; j <= K; ++j) R[j] += (double)u[j];
      }
    }
    if (t < rows) {
      double o[K + 1];
      gk_uncentre<K>(R, cy, o);
#pragma unroll
      for (int r = 0; r <= K; ++r) rowpart[((int64_t)blockIdx.x * (K + 1) + r) * nl + r0 + t] = o[r];
    }
  }
#pragma unroll
  for (int cs = 0; cs < GNS; ++cs) {
    const int64_t q = C0 + cs * GK + t;
    if (q < m) {
      double o[K + 1];
      gk_uncentre<K>(U[cs], cx, o);
#pragma unroll
      for (int r = 0; r <= K; ++r) colpart[((int64_t)blockIdx.y * (K + 1) + r) * m + q] = o[r];
    }
  }
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
// and / or the region's <D_X T D_Y, T> (OBJ -> tile_obj[region]).
//   rowpre[rx][r][i], rowtot[r][i]: power sums of row i over the columns before region rx / all columns
//   colpre[ry][r][q], coltot[r][q]: power sums (weights x^r) of column q of W = T D_Y over the rows
//                                   before row region ry (this rank) / all rows (all ranks)
//   colcarry[r][q] (nullable): the same sums over the rows of the ranks above
// Each thread turns its fp64 carry polynomial sum_r h_r y^{K-r} into fp32 coefficients a_j about the
// region's centre (gk_shift), then walks the region's two tiles in order: W = sum_j a_j s^j, and (odd
// k) crossing column c flips that column's sign: a_j += 2 T_c C(K,j) (-s_c)^{K-j}  (the table tab[c][j]).
// The column states of the region's column tiles stay in registers from one row tile to the next.
template <int K, int MODE, bool STORE, bool OBJ, bool FGW>
__global__ void __launch_bounds__(GK) k_gk_main(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                const double* __restrict__ yc, const double* __restrict__ rowpre,
                                                const double* __restrict__ rowtot, const double* __restrict__ colpre,
                                                const double* __restrict__ coltot, const double* __restrict__ cl,
                                                const double* __restrict__ c2, double alpha,
                                                const double* __restrict__ fx, const double* __restrict__ fy,
                                                float* __restrict__ G, int64_t ldG, double* __restrict__ tile_obj,
                                                const double* __restrict__ colcarry) {
  constexpr int KP = gk_kp<K>();
  constexpr bool ODD = K & 1;
  extern __shared__ float4 gk_smem[];
  __shared__ uint64_t bar;
  float* tile = reinterpret_cast<float*>(gk_smem);  // [GK][GKQ]
  float* tab = tile + GK * GKQ;                      // [GK][KP] crossing table: columns, then rows
  float* sys = tab + GK * KP;                        // [GK] y_q - cy
  float* sxs = sys + GK;                             // [GK] x_i - cx
  float2* sxc = reinterpret_cast<float2*>(sxs + GK);  // [GK] {x_i - cx, 2 alpha c_i} (8-B aligned)
  float* fxs = sxs + 3 * GK;                         // [GK] fx_i (FGW)
  const int t = threadIdx.x;
  const int64_t R0 = (int64_t)blockIdx.y * GR, C0 = (int64_t)blockIdx.x * GR;
  const double cx = gk_centre(xl, R0, (int)min((int64_t)GR, nl - R0));
  const double cy = gk_centre(yc, C0, (int)min((int64_t)GR, m - C0));
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto crossing = [&](float sv) {  // 2 C(K,j) (-s)^{K-j}
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      float v = 0.f;
      if (j <= K) {
        v = (float)(2.0 * gk_binom(K, j));
        for (int e = j; e < K; ++e) v *= -sv;
      }
      tab[t * KP + j] = v;
    }
  };
  const float a4 = (float)(-4.0 * alpha), a1 = (float)(1.0 - alpha);
  float b[GNS][K + 1], e0[GNS];  // column states of the region's column tiles (constant term split as for a)
  double acc = 0.0;
  uint32_t ph = 0;
#pragma unroll 1
  for (int rs = 0; rs < GNS; ++rs) {
    const int64_t r0 = R0 + rs * GK;
    if (r0 >= nl) break;  // uniform
    const int rows = (int)min((int64_t)GK, nl - r0);
    const int64_t i_t = r0 + t;
    // row state of row r0 + t.  The constant coefficient is split: a[0] keeps the carried value, d0
    // collects the crossings' constant terms 2 T_c (-s_c)^K -- hundreds of increments far smaller than
    // a[0] would each round at a[0]'s ulp (a random walk of ~sqrt(GR) ulps); apart they do not.  The
    // higher coefficients meet powers of |s| <= half the region's width, where that rounding is negligible.
    float a[K + 1], d0 = 0.f;
#pragma unroll
    for (int cs = 0; cs < GNS; ++cs) {
      const int64_t c0 = C0 + cs * GK;
      if (c0 >= m) break;  // uniform
      const int cols = (int)min((int64_t)GK, m - c0);
      const int64_t q = c0 + t;
      gk_tile_release();
      {
        const float sx = t < rows ? (float)(xl[i_t] - cx) : 0.f;
        const float sy = t < cols ? (float)(yc[q] - cy) : 0.f;
        sxs[t] = sx;
        sys[t] = sy;
        sxc[t] = make_float2(sx, t < rows ? (float)(2.0 * alpha * cl[i_t]) : 0.f);
        if (FGW) fxs[t] = t < rows ? (float)fx[i_t] : 0.f;
        if (ODD) crossing(sy);
      }
      gk_load_tile<MODE>(S, nl, m, r0, c0, tile, &bar, ph);
      if (MODE != T_PRODUCT) ph ^= 1u;
      __syncthreads();
      // thread = row: W_iq for the tile's columns, in place
      if (t < rows) {
        if (cs == 0) {
          double h[K + 1];  // ascending in y: P(y) = sum_d h_d y^d, h_d = kappa_{K-d} (2 S^<_{K-d} - S_{K-d})
#pragma unroll
          for (int d = 0; d <= K; ++d) {
            const int r = K - d;
            const double tt = rowtot[(int64_t)r * nl + i_t];
            h[d] = gk_kappa<K>(r) * (ODD ? 2.0 * rowpre[((int64_t)blockIdx.x * (K + 1) + r) * nl + i_t] - tt : tt);
          }
          gk_shift<K>(h, cy);
#pragma unroll
          for (int j = 0; j <= K; ++j) a[j] = (float)h[j];
          d0 = 0.f;
        }
        float* trow = tile + t * GKQ;
#pragma unroll 2
        for (int cc = 0; cc < GK; cc += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(trow + cc);
          const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
          float wo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            wo[e] = gk_horner_f<K>(a, sys[cc + e]) + d0;
            if (ODD) {
              float tb[KP];
              gk_ld_tab<KP>(tab + (cc + e) * KP, tb);
              d0 = fmaf(tv[e], tb[0], d0);
#pragma unroll
              for (int j = 1; j <= K; ++j) a[j] = fmaf(tv[e], tb[j], a[j]);
            }
          }
          *reinterpret_cast<float4*>(trow + cc) = make_float4(wo[0], wo[1], wo[2], wo[3]);
        }
      }
      __syncthreads();
      if (ODD) {
        crossing(sxs[t]);
        __syncthreads();
      }
      // thread = column: V_iq = D_X W over the tile's rows, G
      if (t < cols) {
        if (rs == 0) {
          double h[K + 1];
#pragma unroll
          for (int d = 0; d <= K; ++d) {
            const int r = K - d;
            const double tt = coltot[(int64_t)r * m + q];
            double pre = colpre[((int64_t)blockIdx.y * (K + 1) + r) * m + q];
            if (colcarry) pre += colcarry[(int64_t)r * m + q];  // rows of the ranks above
            h[d] = gk_kappa<K>(r) * (ODD ? 2.0 * pre - tt : tt);
          }
          gk_shift<K>(h, cx);
#pragma unroll
          for (int j = 0; j <= K; ++j) b[cs][j] = (float)h[j];
          e0[cs] = 0.f;
        }
        const float c2q = (float)(2.0 * alpha * c2[q]);
        const float fyq = FGW ? (float)fy[q] : 0.f;
        float gq = 0.f, glq = 0.f;
        if (OBJ && MODE != T_EXPLICIT) gq = S.gh[q];
        if (OBJ && MODE == T_GIBBS) glq = S.gl[q];
        float* gp = G + r0 * ldG + q;
#pragma unroll 2
        for (int rr = 0; rr < rows; ++rr, gp += ldG) {
          const float2 xc = sxc[rr];
          const float v = gk_horner_f<K>(b[cs], xc.x) + e0[cs];
          if (ODD) {
            float tb[KP];
            gk_ld_tab<KP>(tab + rr * KP, tb);
            const float w = tile[rr * GKQ + t];
            e0[cs] = fmaf(w, tb[0], e0[cs]);
#pragma unroll
            for (int j = 1; j <= K; ++j) b[cs][j] = fmaf(w, tb[j], b[cs][j]);
          }
          if (OBJ) acc = fma((double)v, (double)gk_regen<MODE>(S, r0 + rr, q, gq, glq), acc);
          if (STORE) {
            // the constant 2 alpha (c_i + c'_q) in fp32: one rounding of a term no larger than ~max|G|
            float g = fmaf(a4, v, xc.y + c2q);
            if (FGW) {
              const float d = fxs[rr] - fyq;
              g = fmaf(a1 * d, d, g);
            }
            __stcs(gp, g);
          }
        }
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

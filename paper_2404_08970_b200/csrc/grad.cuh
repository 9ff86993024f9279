// grad.cuh -- the DP GW gradient  G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y  in O(N M)
// (PAPER.md:120-126 decomposition; PAPER.md:190-259 fast multiply) for sorted 1-D
// supports with |x - x'| distance (k = 1, reading R1/R17).
//
// Formulation (every scan is a sum of non-negative terms):
//   A_jp   = sum_{q<p} (y_p - y_q) T_jq              row-direction scan   (paper's L on rows)
//   A''_ip = sum_{j<i} (x_i - x_j) A_jp              column-direction scan (paper's L on columns)
//   T D_Y  = 2A + Qtot 1^T - Ptot y^T,   D_X A = 2A'' + 1 U_A^T - x S_A^T
//   =>  D_X T D_Y = 4A'' + 2(1 U_A^T - x S_A^T) + (D_X Qtot) 1^T - (D_X Ptot) y^T
// with Ptot = T1, Qtot = Ty, S_A = L_y(T^T 1), U_A = L_y(T^T x): every correction is a
// 1-D DP of the four moment vectors (the paper's L^T parts).
//
// Tiles of TR x TC (rows x columns).  Three passes (12 N M bytes of fp32):
//   k_grad_moments : per (row, strip) and (block, column) partial moments of T
//   k_rowcarry / k_colcarry / k_blkscan_w : exclusive carries (fp64, in place)
//   k_grad_main    : row scan (warp per row, fp32 in-tile, fp32-rounded fp64 carries),
//                    column scan (thread per column), fp64 epilogue, fp32 store.
// T is explicit (gw_grad_dp), regenerated from the Gibbs form exp((f+g-G)/eps) (solver),
// or the product p q^T (T^0, reading R5).
#pragma once
#include "common.cuh"

namespace gw {

constexpr int TC = 256;   // tile columns (one per thread in the column phase)
constexpr int TR = 256;   // tile rows
constexpr int SUB = 32;   // rows per sub-strip of the main pass
constexpr int NT = 256;   // threads per CTA
constexpr int NWARP = NT / 32;

enum { T_EXPLICIT = 0, T_GIBBS = 1, T_PRODUCT = 2 };

struct TSrc {
  const float* T;    // explicit: T;  gibbs: G (the cost whose Gibbs plan is T)
  int64_t ld;
  const double* fs;  // gibbs: f * log2e / eps (local rows);  product: p (local rows)
  const double* gs;  // gibbs: g * log2e / eps (columns);     product: q
  double c2;         // gibbs: log2e / eps
};

// 8 consecutive columns q0..q0+7 of local row j (masked beyond m; caller guarantees j valid).
// Gibbs arguments are formed in fp64 (reading R19: MUFU ex2 for the fp32 exp only).
template <int MODE>
__device__ __forceinline__ void load_row8(const TSrc& S, int64_t j, int64_t q0, int64_t m, const double* gsl,
                                          double fsj, float* v) {
  if (MODE == T_PRODUCT) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (q0 + k < m) ? (float)(fsj * gsl[k]) : 0.f;
    return;
  }
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* row = S.T + j * S.ld + q0;
  if (q0 < m) a = __ldcs(reinterpret_cast<const float4*>(row));
  if (q0 + 4 < m) b = __ldcs(reinterpret_cast<const float4*>(row + 4));
  float t[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (q0 + k >= m) {
      v[k] = 0.f;
    } else if (MODE == T_GIBBS) {
      v[k] = exp2f((float)(fsj + gsl[k] - (double)t[k] * S.c2));
    } else {
      v[k] = t[k];
    }
  }
}

// ---------------------------------------------------------------------------------
// Pass 1: moments.  Tile (s = blockIdx.x, b = blockIdx.y).  Warp w owns rows w, w+8, ...
//   rP[s][j] = sum_{q in s} T_jq,   rA[s][j] = sum_{q in s} (ye_s - y_q) T_jq
//   cS[b][q] = sum_{j in b} T_jq,   cX[b][q] = sum_{j in b} (xe_b - x_j) T_jq
// with ye_s = y[min(c0 + TC, m - 1)], xe_b = x[min(r0 + TR, n - 1)] (the next tile's
// first point).  fp32 partial sums inside the tile, fp64 outputs.
// ---------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(NT) k_grad_moments(TSrc S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                     const double* __restrict__ yc, double* __restrict__ rP,
                                                     double* __restrict__ rA, double* __restrict__ cS,
                                                     double* __restrict__ cX) {
  __shared__ __align__(16) float red[2][NWARP][TC];
  const int s = blockIdx.x, b = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)s * TC, r0 = (int64_t)b * TR;
  const int64_t q0 = c0 + 8 * lane;
  const double ye = yc[min(c0 + TC, m - 1)];
  float dy[8];
  double gsl[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t q = q0 + k;
    dy[k] = q < m ? (float)(ye - yc[q]) : 0.f;
    gsl[k] = (MODE != T_EXPLICIT && q < m) ? S.gs[q] : 0.0;
  }
  const double xe = xl[min(r0 + TR, nl - 1)];
  float cs[8], cx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { cs[k] = 0.f; cx[k] = 0.f; }

  constexpr int U = 4;  // rows in flight per warp
  for (int rr = w; rr < TR; rr += NWARP * U) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = r0 + rr + u * NWARP;
      if (j < nl) {
        const double fsj = (MODE != T_EXPLICIT) ? S.fs[j] : 0.0;
        load_row8<MODE>(S, j, q0, m, gsl, fsj, v[u]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[u][k] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = r0 + rr + u * NWARP;
      float sP = 0.f, sA = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) { sP += v[u][k]; sA = fmaf(dy[k], v[u][k], sA); }
      sP = warp_sum(sP);
      sA = warp_sum(sA);
      if (j < nl) {
        if (lane == 0) { rP[s * nl + j] = (double)sP; rA[s * nl + j] = (double)sA; }
        const float dx = (float)(xe - xl[j]);
#pragma unroll
        for (int k = 0; k < 8; ++k) { cs[k] += v[u][k]; cx[k] = fmaf(dx, v[u][k], cx[k]); }
      }
    }
  }
  float4* r0p = reinterpret_cast<float4*>(&red[0][w][8 * lane]);
  float4* r1p = reinterpret_cast<float4*>(&red[1][w][8 * lane]);
  r0p[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
  r0p[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
  r1p[0] = make_float4(cx[0], cx[1], cx[2], cx[3]);
  r1p[1] = make_float4(cx[4], cx[5], cx[6], cx[7]);
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t q = c0 + t;
  if (q < m) {
    double a = 0.0, bx = 0.0;
#pragma unroll
    for (int ww = 0; ww < NWARP; ++ww) { a += red[0][ww][t]; bx += red[1][ww][t]; }
    cS[b * m + q] = a;
    cX[b * m + q] = bx;
  }
}

// ---------------------------------------------------------------------------------
// Carries (fp64, exclusive, written in place over the partials).
// Column carries, one thread per column q, walking the row blocks b:
//   CP_b(q) = sum_{j < r0(b)} T_jq,   CX_b(q) = sum_{j < r0(b)} (x_{r0(b)} - x_j) T_jq
//   CX_{b+1} = CX_b + (x_{r0(b+1)} - x_{r0(b)}) CP_b + cX[b]    (positive recursion)
// Totals: btot = T^T 1, cxend = sum_j (x_{n-1} - x_j) T_jq.
// ---------------------------------------------------------------------------------
__global__ void k_colcarry(int64_t nl, int64_t m, int nb, const double* __restrict__ xl, double* __restrict__ cS,
                           double* __restrict__ cX, double* __restrict__ btot, double* __restrict__ cxend) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  double CP = 0.0, CX = 0.0;
  constexpr int U = 16;  // blocks in flight: the loads of a group are independent, the recursion is not
  for (int b0 = 0; b0 < nb; b0 += U) {
    double s1[U], sx[U];
    double dx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int b = b0 + u;
      s1[u] = b < nb ? cS[(int64_t)b * m + q] : 0.0;
      sx[u] = b < nb ? cX[(int64_t)b * m + q] : 0.0;
      dx[u] = b < nb ? xl[min((int64_t)(b + 1) * TR, nl - 1)] - xl[(int64_t)b * TR] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int b = b0 + u;
      if (b < nb) {
        cS[(int64_t)b * m + q] = CP;
        cX[(int64_t)b * m + q] = CX;
        CX = CX + dx[u] * CP + sx[u];
        CP += s1[u];
      }
    }
  }
  btot[q] = CP;
  cxend[q] = CX;
}

// Row carries, one CTA per row block (thread = row), walking the strips s:
//   P_c0(j) = sum_{q < c0} T_jq,   A_c0(j) = sum_{q < c0} (y_{c0} - y_q) T_jq
// plus per-(block, strip) sums over the block's rows of {P_c0, A_c0, (xe_b - x_j) P_c0,
// (xe_b - x_j) A_c0} -> blk (the column-direction carry of the row carries).
// Totals: Ptot = T 1, Aend = sum_q (y_{m-1} - y_q) T_jq.
__global__ void __launch_bounds__(TR, 2) k_rowcarry(int64_t nl, int64_t m, int ns, const double* __restrict__ xl,
                                                 const double* __restrict__ yc, double* __restrict__ rP,
                                                 double* __restrict__ rA, double* __restrict__ blk,
                                                 double* __restrict__ Ptot, double* __restrict__ Aend) {
  constexpr int U = 8;  // strips in flight
  __shared__ double red[U][NWARP][4];
  const int b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t j = (int64_t)b * TR + t;
  const bool jv = j < nl;
  const double xe = xl[min((int64_t)(b + 1) * TR, nl - 1)];
  const double dxe = jv ? xe - xl[j] : 0.0;
  double P = 0.0, A = 0.0;
  for (int sc = 0; sc < ns; sc += U) {
    const int cnt = min(U, ns - sc);
    double rp[U], ra[U], dy[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      rp[k] = (jv && k < cnt) ? rP[(int64_t)(sc + k) * nl + j] : 0.0;
      ra[k] = (jv && k < cnt) ? rA[(int64_t)(sc + k) * nl + j] : 0.0;
      dy[k] = k < cnt ? yc[min((int64_t)(sc + k + 1) * TC, m - 1)] - yc[(int64_t)(sc + k) * TC] : 0.0;
    }
    double vals[4 * U];  // [strip k][P, A, dxe P, dxe A] of this row, reduced over the warp below
#pragma unroll
    for (int k = 0; k < U; ++k) {
      vals[4 * k] = vals[4 * k + 1] = vals[4 * k + 2] = vals[4 * k + 3] = 0.0;
      if (k < cnt) {
        const int s = sc + k;
        if (jv) {
          rP[(int64_t)s * nl + j] = P;
          rA[(int64_t)s * nl + j] = A;
        }
        vals[4 * k] = P; vals[4 * k + 1] = A; vals[4 * k + 2] = dxe * P; vals[4 * k + 3] = dxe * A;
        A = A + dy[k] * P + ra[k];
        P += rp[k];
      }
    }
    // recursive halving over the warp (31 shuffles for the 32 sums instead of 32 x 5): afterwards
    // lane L holds the warp sum of vals[L]; fixed lane structure => deterministic
    static_assert(4 * U == 32, "one value per lane after the halving");
#pragma unroll
    for (int off = 16, h = 16; off >= 1; off >>= 1, h >>= 1) {
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < h) {
          const double send = hi ? vals[i] : vals[h + i];
          const double keep = hi ? vals[h + i] : vals[i];
          vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
    }
    red[lane >> 2][w][lane & 3] = vals[0];
    __syncthreads();
    if (t < cnt * 4) {
      const int k = t >> 2, e = t & 3;
      double acc = 0.0;
      for (int ww = 0; ww < NWARP; ++ww) acc += red[k][ww][e];
      blk[((int64_t)b * ns + sc + k) * 4 + e] = acc;
    }
    __syncthreads();
  }
  if (jv) { Ptot[j] = P; Aend[j] = A; }
}

// Block-strip carries: for each strip s, exclusive prefix over row blocks of blk,
//   bs[b][s] = { sum_{j<r0} P_c0(j), sum_{j<r0} A_c0(j),
//                sum_{j<r0} (x_{r0} - x_j) P_c0(j), sum_{j<r0} (x_{r0} - x_j) A_c0(j) }.
// tail (nullable): [ns][4] the state after the last block (referenced at the last local row), the
// per-rank payload of the multi-rank exchange (shard.cuh).
// Warp per strip (a serial walk over the row blocks per thread is a 256-step dependent chain at
// N = 65536).  Both recurrences are PA scans over the row blocks (element of block
// b: {P, A} = {blk.x, blk.z} resp. {blk.y, blk.w}, positioned at X(b+1), X(b) = x of the block's
// first row, X(nb) = x of the last local row): lane L folds blocks 8L .. 8L+7 of a round of 256,
// a warp scan combines the lanes, and the outputs are evaluated at X(b) (pa_eval).
__global__ void __launch_bounds__(256) k_blkscan_w(int64_t nl, int nb, int ns, const double* __restrict__ xl,
                                                   const double* __restrict__ blk, double* __restrict__ bs,
                                                   double* __restrict__ tail) {
  constexpr int PER = 8;
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= ns) return;  // uniform per warp
  auto X = [&](int b) { return xl[min((int64_t)b * TR, nl - 1)]; };
  PA<double> runP{0.0, 0.0, X(0)}, runA = runP;
  for (int r0 = 0; r0 < nb; r0 += 32 * PER) {
    const int b0 = r0 + lane * PER;
    double4 tv[PER];
    double xs[PER + 1];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int b = b0 + u;
      tv[u] = b < nb ? *reinterpret_cast<const double4*>(blk + ((int64_t)b * ns + s) * 4) : make_double4(0, 0, 0, 0);
      xs[u] = X(min(b, nb));
    }
    xs[PER] = X(min(b0 + PER, nb));
    PA<double> lp{0.0, 0.0, xs[0]}, la = lp;
#pragma unroll
    for (int u = 0; u < PER; ++u)
      if (b0 + u < nb) {
        lp = pa_combine(lp, PA<double>{tv[u].x, tv[u].z, xs[u + 1]});
        la = pa_combine(la, PA<double>{tv[u].y, tv[u].w, xs[u + 1]});
      }
    PA<double> exP, exA;
    const PA<double> incP = pa_warp_scan(lp, exP);
    const PA<double> incA = pa_warp_scan(la, exA);
    PA<double> stP = pa_combine(runP, exP), stA = pa_combine(runA, exA);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int b = b0 + u;
      if (b < nb) {
        *reinterpret_cast<double4*>(bs + ((int64_t)b * ns + s) * 4) =
            make_double4(stP.P, stA.P, pa_eval(stP, xs[u]), pa_eval(stA, xs[u]));
        stP = pa_combine(stP, PA<double>{tv[u].x, tv[u].z, xs[u + 1]});
        stA = pa_combine(stA, PA<double>{tv[u].y, tv[u].w, xs[u + 1]});
      }
    }
    const PA<double> tP{__shfl_sync(0xffffffffu, incP.P, 31), __shfl_sync(0xffffffffu, incP.A, 31),
                        __shfl_sync(0xffffffffu, incP.s, 31)};
    const PA<double> tA{__shfl_sync(0xffffffffu, incA.P, 31), __shfl_sync(0xffffffffu, incA.A, 31),
                        __shfl_sync(0xffffffffu, incA.s, 31)};
    runP = pa_combine(runP, tP);
    runA = pa_combine(runA, tA);
  }
  if (tail && lane == 0) {
    const double xe = X(nb);
    *reinterpret_cast<double4*>(tail + 4 * (int64_t)s) = make_double4(runP.P, runA.P, pa_eval(runP, xe), pa_eval(runA, xe));
  }
}

// ---------------------------------------------------------------------------------
// Pass 3: main.  Tile (s, b).  Per element (i, p), tile-relative xh_i = x_i - x_r0,
// yh_p = y_p - y_c0:
//   G_ip = R_i + K_p + xh_i u_p + yh_p v_i - 16 A''loc(i, p)
//   R_i = 2 c_i + 4 (D_X Aend)_i - 4 (y_{m-1} - y_c0)(D_X Ptot)_i,   v_i = 4 (D_X Ptot)_i
//   K_p = 2 c'_p - 16 AA0_p - 8 (x_{n-1} - x_r0) S_A(p) + 8 W_A(p),  u_p = 8 S_A(p) - 16 SA0_p
//   SA0_p = sum_{j<r0} A_jp,  AA0_p = sum_{j<r0} (x_r0 - x_j) A_jp   (column state at the tile top)
//   A''loc(i, p) = sum_{r0 <= j < i} (x_i - x_j) A_jp
// (W_A = L_y(cxend), so U_A = x_{n-1} S_A - W_A.)  Epilogue in fp64.
// ---------------------------------------------------------------------------------
struct MainArgs {
  TSrc S;
  int64_t nl, m;
  int nb, ns;
  const double* xl;    // centred x of local rows
  const double* yc;    // centred y
  const double* cl;    // c (local rows)
  const double* c2;    // c' (m)
  const double* DP;    // D_X Ptot (local rows)
  const double* DA;    // D_X Aend (local rows)
  const double* SAg;   // S_A (m)
  const double* WAg;   // W_A (m)
  const double* rP;    // row carries  [ns][nl]
  const double* rA;
  const double* cS;    // column carries [nb][m]
  const double* cX;
  const double* bs;    // [nb][ns][4]
  double xlast, ylast;
  float* G;
  int64_t ldG;
  double* tile_obj;    // [nb*ns]  sum G' T per tile (OBJ)
  double* tile_ent;    // [nb*ns]  sum T (ln T - 1) per tile (OBJ)
  double* tile_cc;     // [nb*ns]  sum (fx_i - fy_p)^2 T per tile (OBJ, FGW)
  // FGW (Remark 2): G = (1-alpha)(fx_i - fy_p)^2 + alpha * G_gw
  const double* fx;    // local rows (nullable -> GW)
  const double* fy;
  double alpha;
  // tau != eps: the cost gets + beta ln T of the plan it was regenerated
  // from, beta = eps - tau (k_grad_store2<.., TAU>)
  double beta;
};

// dynamic shared memory: sA [SUB][TC] (+ sT [SUB][TC] when OBJ)
template <bool OBJ>
constexpr size_t main_dyn_smem() { return (OBJ ? 2 : 1) * (size_t)SUB * TC * sizeof(float); }

template <int MODE, bool STORE, bool OBJ>
__global__ void __launch_bounds__(NT) k_grad_main(MainArgs a) {
  extern __shared__ __align__(16) float dyn[];
  float (*sA)[TC] = reinterpret_cast<float (*)[TC]>(dyn);
  float (*sT)[TC] = reinterpret_cast<float (*)[TC]>(dyn + SUB * TC);
  __shared__ double sR[TR], sV[TR], sXd[TR + 1], sF[TR], sFx[TR];
  __shared__ float sPc[TR], sAc[TR];
  __shared__ double sm[3 * NWARP];

  const int s = blockIdx.x, b = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t c0 = (int64_t)s * TC, r0 = (int64_t)b * TR;
  const int64_t nl = a.nl, m = a.m;
  const double yc0 = a.yc[c0], xr0 = a.xl[r0];
  const bool fgw = a.fx != nullptr;

  // ---- prologue: column state at the tile top (thread t = column c0 + t) ----
  const int64_t q = c0 + t;
  const bool qv = q < m;
  const int64_t qq = qv ? q : m - 1;
  const double yq = a.yc[qq];
  double Kq, uq, yhq, fyq = 0.0;
  {
    const double CPq = qv ? a.cS[(int64_t)b * m + q] : 0.0;
    const double CXq = qv ? a.cX[(int64_t)b * m + q] : 0.0;
    PA<double> tot;
    PA<double> e1 = pa_block_scan_excl<NWARP>(PA<double>{CPq, 0.0, yq}, sm, tot);
    PA<double> e2 = pa_block_scan_excl<NWARP>(PA<double>{CXq, 0.0, yq}, sm, tot);
    const double* bsv = a.bs + ((int64_t)b * a.ns + s) * 4;
    const double SA0 = bsv[1] + (yq - yc0) * bsv[0] + pa_eval(e1, yq);
    const double AA0 = bsv[3] + (yq - yc0) * bsv[2] + pa_eval(e2, yq);
    const double SAq = a.SAg[qq];
    Kq = 2.0 * a.c2[qq] - 16.0 * AA0 - 8.0 * (a.xlast - xr0) * SAq + 8.0 * a.WAg[qq];
    uq = 8.0 * SAq - 16.0 * SA0;
    yhq = yq - yc0;
    if (fgw) fyq = a.fy[qq];
  }
  // ---- row data of the tile (thread t = row r0 + t) ----
  {
    const int64_t j = r0 + t;
    const int64_t jj = j < nl ? j : nl - 1;
    const double dp = a.DP[jj];
    sR[t] = 2.0 * a.cl[jj] + 4.0 * a.DA[jj] - 4.0 * (a.ylast - yc0) * dp;
    sV[t] = 4.0 * dp;
    sXd[t] = a.xl[jj] - xr0;
    sPc[t] = (float)a.rP[(int64_t)s * nl + jj];
    sAc[t] = (float)a.rA[(int64_t)s * nl + jj];
    sF[t] = (MODE != T_EXPLICIT) ? a.S.fs[jj] : 0.0;
    sFx[t] = fgw ? a.fx[jj] : 0.0;
    if (t == TR - 1) sXd[TR] = sXd[TR - 1];
  }
  // per-lane row-phase constants: columns q0..q0+7
  const int64_t q0 = c0 + 8 * lane;
  float yh[8];
  double gsl[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t qk = min(q0 + k, m - 1);
    yh[k] = (float)(a.yc[qk] - yc0);
    gsl[k] = (MODE != T_EXPLICIT && q0 + k < m) ? a.S.gs[q0 + k] : 0.0;
  }
  __syncthreads();

  double SAloc = 0.0, AAloc = 0.0;  // column state of the tile (fp64: sequential over TR rows)
  double acc_obj = 0.0, acc_ent = 0.0, acc_cc = 0.0;
  const double alpha = a.alpha;

  for (int sub = 0; sub < TR / SUB; ++sub) {
    const int rbase = sub * SUB;
    if (r0 + rbase >= nl) break;  // uniform
    // ---- phase A: row scans, warp w owns sub-strip rows w*4 .. w*4+3 ----
    float v[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rho = w * 4 + u;
      const int64_t j = r0 + rbase + rho;
      if (j < nl) {
        load_row8<MODE>(a.S, j, q0, m, gsl, sF[rbase + rho], v[u]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[u][k] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rho = w * 4 + u;
      float P = 0.f, A = 0.f, sref = yh[0];
      float loc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        loc[k] = A + (yh[k] - sref) * P;
        P += v[u][k];
        A = loc[k];
        sref = yh[k];
      }
      PA<float> ex;
      pa_warp_scan(PA<float>{P, A, sref}, ex);
      const float Pc = sPc[rbase + rho], Ac = sAc[rbase + rho];
      float out[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) out[k] = loc[k] + pa_eval(ex, yh[k]) + Ac + yh[k] * Pc;
      float4* dst = reinterpret_cast<float4*>(&sA[rho][8 * lane]);
      dst[0] = make_float4(out[0], out[1], out[2], out[3]);
      dst[1] = make_float4(out[4], out[5], out[6], out[7]);
      if (OBJ) {
        float4* dt = reinterpret_cast<float4*>(&sT[rho][8 * lane]);
        dt[0] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
        dt[1] = make_float4(v[u][4], v[u][5], v[u][6], v[u][7]);
        if (MODE == T_GIBBS) {
          // H(T) = sum T (ln T - 1) with ln T = (f + g - G)/eps
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float tv = v[u][k];
            if (tv > 0.f) acc_ent += (double)tv * ((double)__log2f(tv) * GW_LN2 - 1.0);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float tv = v[u][k];
            if (tv > 0.f) acc_ent += (double)tv * (log((double)tv) - 1.0);
          }
        }
      }
    }
    __syncthreads();
    // ---- phase B: column scans, thread t owns column c0 + t ----
#pragma unroll 4
    for (int rho = 0; rho < SUB; ++rho) {
      const int ri = rbase + rho;
      const int64_t i = r0 + ri;
      if (i >= nl) break;
      const float Av = sA[rho][t];
      const double gw = sR[ri] + Kq + sXd[ri] * uq + yhq * sV[ri] - 16.0 * AAloc;
      double gv = gw, cc = 0.0;
      if (fgw) {
        const double d = sFx[ri] - fyq;
        cc = d * d;
        gv = (1.0 - alpha) * cc + alpha * gw;
      }
      if (STORE && qv) a.G[i * a.ldG + q] = (float)gv;
      if (OBJ && qv) {
        const double tv = (double)sT[rho][t];
        acc_obj += gw * tv;
        if (fgw) acc_cc += cc * tv;
      }
      const double SAi = SAloc + (double)Av;
      AAloc = fma(sXd[ri + 1] - sXd[ri], SAi, AAloc);
      SAloc = SAi;
    }
    __syncthreads();
  }
  if (OBJ) {
    const double so = block_sum<NWARP>(acc_obj, sm);
    const double se = block_sum<NWARP>(acc_ent, sm);
    const double sc = block_sum<NWARP>(acc_cc, sm);
    if (t == 0) {
      a.tile_obj[(int64_t)b * a.ns + s] = so;
      a.tile_ent[(int64_t)b * a.ns + s] = se;
      a.tile_cc[(int64_t)b * a.ns + s] = sc;
    }
  }
}

// Materialise T = exp((f + g - G) / eps) (fp64 argument, fp32 store) or T = p q^T.
template <int MODE>
__global__ void k_materialize(TSrc S, int64_t nl, int64_t m, float* __restrict__ T, int64_t ldT) {
  const int64_t total = nl * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, q = e - i * m;
    float v;
    if (MODE == T_PRODUCT) v = (float)(S.fs[i] * S.gs[q]);
    else v = exp2f((float)(S.fs[i] + S.gs[q] - (double)S.T[i * S.ld + q] * S.c2));
    T[i * ldT + q] = v;
  }
}

}  // namespace gw

// grad2.cuh -- streaming kernels of the DP gradient (rows a1-a4 of SURVEY §8a):
//   k_grad_moments3 : per (row, strip) row partials and per (block, column) column partials of T
//   k_grad_store2   : the main pass, G = R_i + K'_p + xh_i u'_p + yh_p v_i - 16 A''_sub  (fp32 out)
// Same tiling, carries and formulas as grad.cuh (TR x TC = 256 x 256 tiles; the derivation is in
// grad.cuh and DESIGN.md §3), re-laid out so that every per-element step is a handful of fp32
// instructions:
//   * a tile is processed in sub-strips of G2SUB = 32 rows; a sub-strip is loaded with coalesced
//     128-bit loads one sub-strip ahead (registers), T is regenerated on the way into shared
//     memory (fp32 hi/lo duals, below), and stored in a padded layout (row stride 272 floats,
//     64-column segments at stride 68) on which the row pass, the column pass and the staging
//     stores are all bank-conflict free;
//   * row direction: thread = (row, 64-column segment), a sequential gap-weighted scan
//     (PAPER.md:237-243 with gaps, reading R1) with no shuffles; the 4 segment states are
//     combined by a 2-step shuffle scan and applied in the column pass;
//   * column direction: thread = 2 adjacent columns (packed fp32x2), fp32 state inside a
//     sub-strip, fp64 state across sub-strips.
// Precision: tile-level carries and moments stay fp64 (grad.cuh); inside a sub-strip every term
// is a sum of non-negative contributions (no cancellation); the assembly adds O(1) terms in
// fp32 (absolute error ~1e-7 against the 1e-5 max|G| tolerance).
//
// T regeneration (MODE == T_GIBBS, the solver path): T_ip = 2^(F_i + g_p - G_ip c),
// c = log2e/eps, with every quantity split into fp32 hi + lo parts:
//   a = [fma(G, -c_hi, g_hi) + F_hi] + [fma(G, -c_lo, g_lo + F_lo)].
// The first fma rounds once (the only inexact step, an unbiased <= 1/2 ulp of |g_hi - G c_hi|,
// ~1e-4 in log2 units at eps = 1e-3); "+ F_hi" is exact where T is not negligible (Sterbenz);
// the lo bracket carries the dual and c residuals, so T has no systematic per-row or
// per-column bias.
#pragma once
#include "common.cuh"
#include "fused.cuh"  // ffma2 / fadd2
#include "grad.cuh"

namespace gw {

constexpr int G2T = 128;               // threads per CTA
constexpr int G2SUB = 32;              // rows per sub-strip
constexpr int G2SEG = 68;              // floats per 64-column segment in shared memory (64 + 4 pad)
constexpr int G2RS = 4 * G2SEG;        // row stride (272 floats = 68 16-B chunks, = 4 mod 8)

struct TSrc2 {
  const float* T;    // explicit: T;  gibbs: G
  int64_t ld;
  const float *fh, *fl;  // gibbs: f log2e/eps hi/lo (local rows);  product: p (fp32, local rows) in fh
  const float *gh, *gl;  // gibbs: g log2e/eps hi/lo (columns);     product: q (fp32) in gh
  float ch, cl;          // gibbs: log2e/eps hi/lo
};

__device__ __forceinline__ int g2_phys(int col) { return (col >> 6) * G2SEG + (col & 63); }

// Sub-strip loader: warp w loads rows w, w+4, ... (8 rows); per row 2 x 32 lanes x float4 = 256
// columns.  Values stay in registers until g2_stage() writes them to shared memory.
template <int MODE>
struct G2Loader {
  float4 v[16];
  __device__ __forceinline__ void load(const TSrc2& S, int64_t r0, int64_t c0, int64_t nl, int64_t m, int sub) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if constexpr (MODE != T_PRODUCT) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = r0 + sub * G2SUB + w + 4 * u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t q = c0 + 128 * h + 4 * lane;
          if (i < nl && q < m) v[2 * u + h] = __ldcs(reinterpret_cast<const float4*>(S.T + i * S.ld + q));
          else v[2 * u + h] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
};

// Regenerate T from the loaded values (MODE) and write it to the padded shared-memory tile.
// OBJ: also copy T to sT2 and accumulate the entropy sum T (ln T - 1) into *ent;
// on the Gibbs path ln T is the exponent itself (a ln 2), so no logarithm is taken.
template <int MODE, bool OBJ = false, bool LNT = false>
__device__ __forceinline__ void g2_stage(const G2Loader<MODE>& L, const TSrc2& S, float* __restrict__ sT, int64_t r0,
                                         int64_t c0, int64_t nl, int64_t m, int sub, float* __restrict__ sT2 = nullptr,
                                         float* ent = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t q = c0 + 128 * h + 4 * lane;
    float2 gh0 = make_float2(0.f, 0.f), gh1 = gh0, gl0 = gh0, gl1 = gh0;
    if (MODE != T_EXPLICIT) {
      gh0 = make_float2(q < m ? S.gh[q] : 0.f, q + 1 < m ? S.gh[q + 1] : 0.f);
      gh1 = make_float2(q + 2 < m ? S.gh[q + 2] : 0.f, q + 3 < m ? S.gh[q + 3] : 0.f);
      if (MODE == T_GIBBS) {
        gl0 = make_float2(q < m ? S.gl[q] : 0.f, q + 1 < m ? S.gl[q + 1] : 0.f);
        gl1 = make_float2(q + 2 < m ? S.gl[q + 2] : 0.f, q + 3 < m ? S.gl[q + 3] : 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int rl = w + 4 * u;
      const int64_t i = r0 + sub * G2SUB + rl;
      float4 t, lt = make_float4(0.f, 0.f, 0.f, 0.f);  // LNT: ln T
      if (MODE == T_EXPLICIT) {
        t = L.v[2 * u + h];
        if (LNT) lt = make_float4(logf(t.x), logf(t.y), logf(t.z), logf(t.w));
      } else if (MODE == T_PRODUCT) {
        const float pi = i < nl ? S.fh[i] : 0.f;
        t = make_float4(pi * gh0.x, pi * gh0.y, pi * gh1.x, pi * gh1.y);
        if (LNT) {
          const float lpi = logf(pi);
          lt = make_float4(lpi + logf(gh0.x), lpi + logf(gh0.y), lpi + logf(gh1.x), lpi + logf(gh1.y));
        }
      } else {
        const float4 g = L.v[2 * u + h];
        const float Fh = i < nl ? S.fh[i] : 0.f, Fl = i < nl ? S.fl[i] : 0.f;
        const float2 F2 = make_float2(Fh, Fh), Fl2 = make_float2(Fl, Fl);
        const float2 nch = make_float2(-S.ch, -S.ch), ncl = make_float2(-S.cl, -S.cl);
        const float2 g01 = make_float2(g.x, g.y), g23 = make_float2(g.z, g.w);
        const float2 a0 = fadd2(fadd2(ffma2(g01, nch, gh0), F2), ffma2(g01, ncl, fadd2(gl0, Fl2)));
        const float2 a1 = fadd2(fadd2(ffma2(g23, nch, gh1), F2), ffma2(g23, ncl, fadd2(gl1, Fl2)));
        t = make_float4(ex2_ftz(a0.x), ex2_ftz(a0.y), ex2_ftz(a1.x), ex2_ftz(a1.y));
        if (LNT) {
          constexpr float ln2 = 0.6931471805599453f;
          lt = make_float4(a0.x * ln2, a0.y * ln2, a1.x * ln2, a1.y * ln2);
        }
        if (OBJ && i < nl) {
          constexpr float ln2 = 0.6931471805599453f;
          const float av[4] = {a0.x, a0.y, a1.x, a1.y}, tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (tv[e] > 0.f && q + e < m) *ent += tv[e] * fmaf(av[e], ln2, -1.f);
        }
      }
      if (OBJ && MODE != T_GIBBS && i < nl) {
        const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (tv[e] > 0.f && q + e < m) *ent += tv[e] * (__logf(tv[e]) - 1.f);
      }
      if (i >= nl) t = lt = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q + 3 >= m) {
        if (q >= m) t.x = lt.x = 0.f;
        if (q + 1 >= m) t.y = lt.y = 0.f;
        if (q + 2 >= m) t.z = lt.z = 0.f;
        if (q + 3 >= m) t.w = lt.w = 0.f;
      }
      *reinterpret_cast<float4*>(sT + rl * G2RS + g2_phys(128 * h + 4 * lane)) = t;
      if (OBJ) *reinterpret_cast<float4*>(sT2 + rl * G2RS + g2_phys(128 * h + 4 * lane)) = t;
      if (LNT) *reinterpret_cast<float4*>(sT2 + rl * G2RS + g2_phys(128 * h + 4 * lane)) = lt;
    }
  }
}

// Interior tiles (all 256 rows and columns real): loads with a running row pointer, T
// regeneration with the tile's column duals held in registers (gq: g_hi, gq2: g_lo of the
// lane's 8 columns) and the row duals from shared memory, no masks.
template <int MODE>
__device__ __forceinline__ void g2_load_fast(G2Loader<MODE>& L, const TSrc2& S, int64_t r0, int64_t c0, int sub) {
  if constexpr (MODE != T_PRODUCT) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float* p = S.T + (r0 + sub * G2SUB + w) * S.ld + c0 + 4 * lane;
    const int64_t step = 4 * S.ld;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      L.v[2 * u] = __ldcs(reinterpret_cast<const float4*>(p));
      L.v[2 * u + 1] = __ldcs(reinterpret_cast<const float4*>(p + 128));
      p += step;
    }
  }
}

template <int MODE, bool OBJ, bool LNT = false>
__device__ __forceinline__ void g2_stage_fast(const G2Loader<MODE>& L, const TSrc2& S, float* __restrict__ sT,
                                              const float2 (&gq)[2][2], const float2 (&gq2)[2][2],
                                              const float* __restrict__ sF, const float* __restrict__ sFl, int sub,
                                              float* __restrict__ sT2, float* ent) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float2 entv = make_float2(0.f, 0.f);  // OBJ, Gibbs: two interleaved fp32 partial sums of T (ln T - 1)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int phys = g2_phys(128 * h + 4 * lane);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int rl = w + 4 * u;
      float4 t, lt = make_float4(0.f, 0.f, 0.f, 0.f);  // LNT: ln T
      if (MODE == T_EXPLICIT) {
        t = L.v[2 * u + h];
        if (LNT) lt = make_float4(logf(t.x), logf(t.y), logf(t.z), logf(t.w));
      } else if (MODE == T_PRODUCT) {
        const float pi = sF[sub * G2SUB + rl];
        t = make_float4(pi * gq[h][0].x, pi * gq[h][0].y, pi * gq[h][1].x, pi * gq[h][1].y);
        if (LNT) {
          const float lpi = logf(pi);
          lt = make_float4(lpi + logf(gq[h][0].x), lpi + logf(gq[h][0].y), lpi + logf(gq[h][1].x),
                           lpi + logf(gq[h][1].y));
        }
      } else {
        const float4 g = L.v[2 * u + h];
        const float Fh = sF[sub * G2SUB + rl], Fl = sFl[sub * G2SUB + rl];
        const float2 F2 = make_float2(Fh, Fh), Fl2 = make_float2(Fl, Fl);
        const float2 nch = make_float2(-S.ch, -S.ch), ncl = make_float2(-S.cl, -S.cl);
        const float2 g01 = make_float2(g.x, g.y), g23 = make_float2(g.z, g.w);
        const float2 a0 = fadd2(fadd2(ffma2(g01, nch, gq[h][0]), F2), ffma2(g01, ncl, fadd2(gq2[h][0], Fl2)));
        const float2 a1 = fadd2(fadd2(ffma2(g23, nch, gq[h][1]), F2), ffma2(g23, ncl, fadd2(gq2[h][1], Fl2)));
        t = make_float4(ex2_ftz(a0.x), ex2_ftz(a0.y), ex2_ftz(a1.x), ex2_ftz(a1.y));
        if (LNT) {
          constexpr float ln2 = 0.6931471805599453f;
          lt = make_float4(a0.x * ln2, a0.y * ln2, a1.x * ln2, a1.y * ln2);
        }
        if (OBJ) {
          // T (ln T - 1) with ln T = a ln 2, packed, no branch: a clamped at -200 (T = 0 there) so that a
          // zero-mass column's a = -inf contributes 0 x finite
          const float2 l2 = make_float2(0.6931471805599453f, 0.6931471805599453f), m1 = make_float2(-1.f, -1.f);
          const float2 A0 = make_float2(fmaxf(a0.x, -200.f), fmaxf(a0.y, -200.f));
          const float2 A1 = make_float2(fmaxf(a1.x, -200.f), fmaxf(a1.y, -200.f));
          entv = ffma2(make_float2(t.x, t.y), ffma2(A0, l2, m1), entv);
          entv = ffma2(make_float2(t.z, t.w), ffma2(A1, l2, m1), entv);
        }
      }
      if (OBJ && MODE != T_GIBBS) {
        const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (tv[e] > 0.f) *ent += tv[e] * (__logf(tv[e]) - 1.f);
      }
      *reinterpret_cast<float4*>(sT + rl * G2RS + phys) = t;
      if (OBJ) *reinterpret_cast<float4*>(sT2 + rl * G2RS + phys) = t;
      if (LNT) *reinterpret_cast<float4*>(sT2 + rl * G2RS + phys) = lt;
    }
  }
  if (OBJ && MODE == T_GIBBS) *ent += entv.x + entv.y;
}

// ---------------------------------------------------------------------------------
// Main pass (STORE only; the objective pass keeps grad.cuh's k_grad_main<.., OBJ>).
// Per tile (same quantities as k_grad_main, see grad.cuh):
//   G_ip = R_i + K_p + xh_i u_p + yh_p v_i - 16 A''loc(i, p),
// with, per sub-strip starting at tile row i0 (column state SAtop, AAtop in fp64),
//   A''loc(i, p) = AAtop + (xh_i - xh_i0) SAtop + AAsub(i, p)
//   => G_ip = R_i + K'_p + xh_i u'_p + yh_p v_i - 16 AAsub(i, p),
//      K'_p = K_p - 16 AAtop + 16 xh_i0 SAtop,  u'_p = u_p - 16 SAtop.
// FGW (Remark 2): G = (1 - alpha) (fx_i - fy_p)^2 + alpha G_gw; the alpha is
// folded into the constants and sqrt(1 - alpha) into the features.
// ---------------------------------------------------------------------------------
// OBJ (the objective pass over the final plan): nothing is stored; per tile the fp64 sums
// <G, T> (GW gradient, prescribed c), sum T (ln T - 1) and <(fx - fy)^2, T> go to
// a.tile_obj / tile_ent / tile_cc for k_obj_partial (the constants are then not alpha-scaled).
// TAU (tau != eps): the stored cost is G + beta ln T (beta = eps - tau) with ln T
// of the plan the tile was regenerated from, kept in the dynamic buffer (a.beta).
template <int MODE, bool FGW, bool OBJ = false, bool TAU = false>
__global__ void __launch_bounds__(G2T, 3) k_grad_store2(MainArgs a, TSrc2 S) {
  __shared__ __align__(16) float sT[G2SUB * G2RS];  // T, then the local row scans (exclusive, per segment)
  extern __shared__ __align__(16) float sTobj[];     // OBJ: a copy of T (dynamic, G2SUB * G2RS floats)
  __shared__ __align__(16) float4 sRow[TR];         // {R_i, xh_i, v_i, dx_i} (alpha-scaled for FGW)
  __shared__ __align__(16) float2 sEx[G2SUB][4];    // per (row, segment): {P, A} exclusive state of the row
                                                    // before the segment (incl. the strip carry), at the
                                                    // segment's reference point
  __shared__ __align__(16) float sDy[4 * G2SEG];    // gaps y_q - y_{q-1} inside a segment (0 at a segment start);
                                                    // segments G2SEG apart: the row pass's 4 segments of a
                                                    // quarter-warp then fall in distinct banks
  __shared__ float sFx[TR];
  __shared__ __align__(8) float2 sCar[TR];          // strip carry of each row: {P_c0, A_c0} (fp32)
  __shared__ float sSref[4];                        // y (tile-relative) of each segment's last column
  __shared__ float sF[TR], sFl[TR];                 // row duals (hi, lo) / p (product) of the tile's rows
  __shared__ double sm[3 * (G2T / 32)];

  const int s = blockIdx.x, b = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t c0 = (int64_t)s * TC, r0 = (int64_t)b * TR;
  const int64_t nl = a.nl, m = a.m;
  const bool interior = (r0 + TR <= nl) && (c0 + TC <= m);  // uniform: no masks on this tile
  float2 gq[2][2], gq2[2][2];                       // column duals of the lane's staging columns
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t q = c0 + 128 * h + 4 * lane;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      gq[h][e] = make_float2(0.f, 0.f);
      gq2[h][e] = gq[h][e];
      if (MODE != T_EXPLICIT && interior) {
        gq[h][e] = make_float2(S.gh[q + 2 * e], S.gh[q + 2 * e + 1]);
        if (MODE == T_GIBBS) gq2[h][e] = make_float2(S.gl[q + 2 * e], S.gl[q + 2 * e + 1]);
      }
    }
  }
  const double yc0 = a.yc[c0], xr0 = a.xl[r0];
  const double alpha = (FGW && !OBJ) ? a.alpha : 1.0;
  const double fscale = (FGW && !OBJ) ? sqrt(1.0 - a.alpha) : 1.0;  // features: (1 - alpha)(fx - fy)^2
  double acc_obj = 0.0, acc_ent = 0.0, acc_cc = 0.0;

  // ---- prologue: column state at the tile top, columns q = c0 + 2t + e (e = 0, 1) ----
  double Kq[2], uq[2];
  float yhq[2], dYs[2], fyq[2];
  {
    double CP[2], CX[2], yq[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t q = c0 + 2 * t + e;
      const bool qv = q < m;
      yq[e] = a.yc[qv ? q : m - 1];
      CP[e] = qv ? a.cS[(int64_t)b * m + q] : 0.0;
      CX[e] = qv ? a.cX[(int64_t)b * m + q] : 0.0;
    }
    // block-exclusive scans of (CP, 0, y) and (CX, 0, y) over the tile's columns, 2 per thread
    PA<double> tot;
    const PA<double> v1 = pa_combine(PA<double>{CP[0], 0.0, yq[0]}, PA<double>{CP[1], 0.0, yq[1]});
    const PA<double> v2 = pa_combine(PA<double>{CX[0], 0.0, yq[0]}, PA<double>{CX[1], 0.0, yq[1]});
    PA<double> e1 = pa_block_scan_excl<G2T / 32>(v1, sm, tot);
    PA<double> e2 = pa_block_scan_excl<G2T / 32>(v2, sm, tot);
    const double* bsv = a.bs + ((int64_t)b * a.ns + s) * 4;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t q = c0 + 2 * t + e;
      const int64_t qq = q < m ? q : m - 1;
      const double SA0 = bsv[1] + (yq[e] - yc0) * bsv[0] + pa_eval(e1, yq[e]);
      const double AA0 = bsv[3] + (yq[e] - yc0) * bsv[2] + pa_eval(e2, yq[e]);
      const double SAq = a.SAg[qq];
      Kq[e] = alpha * (2.0 * a.c2[qq] - 16.0 * AA0 - 8.0 * (a.xlast - xr0) * SAq + 8.0 * a.WAg[qq]);
      uq[e] = alpha * (8.0 * SAq - 16.0 * SA0);
      yhq[e] = (float)(yq[e] - yc0);
      fyq[e] = FGW ? (float)(fscale * a.fy[qq]) : 0.f;
      // step to the next exclusive state for e = 1
      e1 = pa_combine(e1, PA<double>{CP[e], 0.0, yq[e]});
      e2 = pa_combine(e2, PA<double>{CX[e], 0.0, yq[e]});
    }
    // gap to the previous column inside the segment (0 at a segment start: the segment's
    // reference point is its first column)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = 2 * t + e;
      const int64_t q = c0 + col;
      sDy[(col >> 6) * G2SEG + (col & 63)] = ((col & 63) == 0 || q >= m) ? 0.f : (float)(a.yc[q] - a.yc[q - 1]);
      // yh_p - yh_ref(segment): distance from the previous segment's last column (ex-state
      // reference) to this column; for segment 0 the reference is y_c0 (strip carry)
      const int sgc = col >> 6;
      const double yref = sgc == 0 ? yc0 : a.yc[min(c0 + 64 * sgc - 1, m - 1)];
      dYs[e] = (float)(a.yc[min(q, m - 1)] - yref);
    }
  }
  // ---- row data of the tile ----
  for (int k = t; k < TR; k += G2T) {
    const int64_t j = r0 + k;
    const int64_t jj = j < nl ? j : nl - 1;
    const double dp = a.DP[jj];
    const double R = 2.0 * a.cl[jj] + 4.0 * a.DA[jj] - 4.0 * (a.ylast - yc0) * dp;
    const double xh = a.xl[jj] - xr0;
    const double xn = (j + 1 < nl) ? a.xl[j + 1] - xr0 : xh;
    sRow[k] = make_float4((float)(alpha * R), (float)xh, (float)(alpha * 4.0 * dp), (float)(xn - xh));
    sFx[k] = FGW ? (float)(fscale * a.fx[jj]) : 0.f;
    sCar[k] = make_float2((float)a.rP[(int64_t)s * nl + jj], (float)a.rA[(int64_t)s * nl + jj]);
    sF[k] = (MODE != T_EXPLICIT) ? S.fh[jj] : 0.f;
    sFl[k] = (MODE == T_GIBBS) ? S.fl[jj] : 0.f;
  }
  if (t < 4) sSref[t] = (float)(a.yc[min(c0 + 64 * t + 63, m - 1)] - yc0);
  const int nsub = (int)min((int64_t)(TR / G2SUB), (nl - r0 + G2SUB - 1) / G2SUB);
  const int rrow = w * 8 + (lane >> 2), sg = lane & 3;
  const int cphys = g2_phys(2 * t), csg = (2 * t) >> 6;
  const float m16 = (float)(-16.0 * alpha);
  double SAtop[2] = {0.0, 0.0}, AAtop[2] = {0.0, 0.0};
  G2Loader<MODE> L;
  if (interior) g2_load_fast<MODE>(L, S, r0, c0, 0);
  else L.load(S, r0, c0, nl, m, 0);
  for (int sub = 0; sub < nsub; ++sub) {
    __syncthreads();  // previous sub-strip fully consumed; prologue smem visible
    {
      float ent = 0.f;
      if (interior) g2_stage_fast<MODE, OBJ, TAU>(L, S, sT, gq, gq2, sF, sFl, sub, sTobj, &ent);
      else g2_stage<MODE, OBJ, TAU>(L, S, sT, r0, c0, nl, m, sub, sTobj, &ent);
      if (OBJ) acc_ent += (double)ent;
    }
    if (sub + 1 < nsub) {
      if (interior) g2_load_fast<MODE>(L, S, r0, c0, sub + 1);
      else L.load(S, r0, c0, nl, m, sub + 1);
    }
    __syncthreads();
    // ---- row pass: exclusive gap-weighted scan of this thread's segment, in place ----
    {
      float* rowp = sT + rrow * G2RS + sg * G2SEG;
      const float* dyp = sDy + sg * G2SEG;
      float P = 0.f, A = 0.f;
#pragma unroll 4
      for (int k = 0; k < 16; ++k) {
        const float4 v = *reinterpret_cast<const float4*>(rowp + 4 * k);
        const float4 d = *reinterpret_cast<const float4*>(dyp + 4 * k);
        float4 o;
        o.x = fmaf(d.x, P, A); P += v.x; A = o.x;
        o.y = fmaf(d.y, P, A); P += v.y; A = o.y;
        o.z = fmaf(d.z, P, A); P += v.z; A = o.z;
        o.w = fmaf(d.w, P, A); P += v.w; A = o.w;
        *reinterpret_cast<float4*>(rowp + 4 * k) = o;
      }
      // segment state (P, A) referenced at its last column; exclusive scan over the 4 segments,
      // seeded with the strip carry (Pc, Ac at y_c0) for segment 0:
      //   combine(a, b) = (a.P + b.P, a.A + (b.s - a.s) a.P + b.A)
      const float2 car = sCar[sub * G2SUB + rrow];
      const float Pc = car.x, Ac = car.y;
      // reference points: s_{-1} = y_c0, s_k = y of segment k's last column (clamped to m-1)
      const float sref = sSref[sg];
      float eP = P, eA = A, es = sref;  // inclusive state of this segment
      // Hillis-Steele over 4 lanes (lanes 4r..4r+3 hold segments 0..3 of one row)
#pragma unroll
      for (int d = 1; d < 4; d <<= 1) {
        const float oP = __shfl_up_sync(0xffffffffu, eP, d);
        const float oA = __shfl_up_sync(0xffffffffu, eA, d);
        const float os = __shfl_up_sync(0xffffffffu, es, d);
        if (sg >= d) {
          eA = oA + (es - os) * oP + eA;
          eP = oP + eP;
        }
      }
      // exclusive = inclusive of the previous segment; seed = strip carry at yh = 0
      float xP = __shfl_up_sync(0xffffffffu, eP, 1), xA = __shfl_up_sync(0xffffffffu, eA, 1);
      const float xs = __shfl_up_sync(0xffffffffu, es, 1);
      if (sg == 0) { xP = 0.f; xA = 0.f; }
      // carry (Pc, Ac at 0) combined with the exclusive state (xP, xA at xs): value at the
      // segment's reference point yr (y_c0 for segment 0, else xs)
      const float yr = sg == 0 ? 0.f : xs;
      const float outA = Ac + yr * Pc + xA;
      const float outP = Pc + xP;
      sEx[rrow][sg] = make_float2(outP, outA);
    }
    __syncthreads();
    // ---- column pass ----
    {
      float Kf[2], uf[2];
      const float xh0 = sRow[sub * G2SUB].y;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        Kf[e] = (float)(Kq[e] - 16.0 * alpha * AAtop[e] + 16.0 * alpha * (double)xh0 * SAtop[e]);
        uf[e] = (float)(uq[e] - 16.0 * alpha * SAtop[e]);
      }
      const float2 K2 = make_float2(Kf[0], Kf[1]), u2 = make_float2(uf[0], uf[1]);
      const float2 yh2 = make_float2(yhq[0], yhq[1]), dY2 = make_float2(dYs[0], dYs[1]);
      const float2 fy2 = make_float2(fyq[0], fyq[1]);
      const float2 m162 = make_float2(m16, m16);
      float2 SA = make_float2(0.f, 0.f), AA = SA;
      float* Gp = a.G + (r0 + sub * G2SUB) * a.ldG + c0 + 2 * t;
      const bool q0v = c0 + 2 * t < m, q1v = c0 + 2 * t + 1 < m;
      const int nr = (int)min((int64_t)G2SUB, nl - (r0 + sub * G2SUB));
      // OBJ: the sub-strip's <G, T> and feature terms in fp32 (<= G2SUB non-negative products per
      // lane, relative rounding <= G2SUB ulps), folded into the fp64 sums after the sub-strip
      float2 ob = make_float2(0.f, 0.f), oc = ob;
#pragma unroll 4
      for (int rl = 0; rl < nr; ++rl) {
        const float2 loc = *reinterpret_cast<const float2*>(sT + rl * G2RS + cphys);
        const float2 ex = sEx[rl][csg];
        const float4 rc = sRow[sub * G2SUB + rl];
        // A_ip = loc + ex.A + (y_p - y_ref) ex.P   (all terms >= 0)
        const float2 Av = ffma2(dY2, make_float2(ex.x, ex.x), fadd2(loc, make_float2(ex.y, ex.y)));
        float2 g = fadd2(K2, make_float2(rc.x, rc.x));
        g = ffma2(make_float2(rc.y, rc.y), u2, g);
        g = ffma2(yh2, make_float2(rc.z, rc.z), g);
        g = ffma2(AA, m162, g);
        if (OBJ) {
          const float2 tv = *reinterpret_cast<const float2*>(sTobj + rl * G2RS + cphys);
          ob = ffma2(g, tv, ob);
          if (FGW) {
            const float fx = sFx[sub * G2SUB + rl];
            const float2 d = fadd2(make_float2(fx, fx), make_float2(-fy2.x, -fy2.y));
            oc = ffma2(make_float2(d.x * d.x, d.y * d.y), tv, oc);
          }
        } else {
          if (FGW) {
            const float fx = sFx[sub * G2SUB + rl];
            const float2 d = fadd2(make_float2(fx, fx), make_float2(-fy2.x, -fy2.y));
            g = ffma2(d, d, g);
          }
          if (TAU) {
            const float2 lv = *reinterpret_cast<const float2*>(sTobj + rl * G2RS + cphys);
            const float bt = (float)a.beta;
            g = ffma2(lv, make_float2(bt, bt), g);
          }
            if (q1v) *reinterpret_cast<float2*>(Gp) = g;
          else if (q0v) Gp[0] = g.x;
          Gp += a.ldG;
        }
        SA = fadd2(SA, Av);
        AA = ffma2(make_float2(rc.w, rc.w), SA, AA);
      }
      if (OBJ) {
        acc_obj += (double)ob.x + (double)ob.y;
        if (FGW) acc_cc += (double)oc.x + (double)oc.y;
      }
      // fold the sub-strip into the fp64 column state: AAtop(i0 + 32) = AAtop + (x_end - x_i0) SAtop + AAsub
      const float xend = nr > 0 ? sRow[sub * G2SUB + nr - 1].y + sRow[sub * G2SUB + nr - 1].w : xh0;
      AAtop[0] += (double)(xend - xh0) * SAtop[0] + (double)AA.x;
      AAtop[1] += (double)(xend - xh0) * SAtop[1] + (double)AA.y;
      SAtop[0] += (double)SA.x;
      SAtop[1] += (double)SA.y;
    }
  }
  if (OBJ) {
    // fixed-order CTA reductions (columns beyond m and rows beyond nl contribute exact zeros)
    const double so = block_sum<G2T / 32>(acc_obj, sm);
    const double se = block_sum<G2T / 32>(acc_ent, sm);
    const double sc = block_sum<G2T / 32>(acc_cc, sm);
    if (t == 0) {
      a.tile_obj[(int64_t)b * a.ns + s] = so;
      a.tile_ent[(int64_t)b * a.ns + s] = se;
      a.tile_cc[(int64_t)b * a.ns + s] = sc;
    }
  }
}

}  // namespace gw

namespace gw {

// ---------------------------------------------------------------------------------
// Moments without shared-memory staging (outputs as k_grad_moments in grad.cuh):
//   rP[s][j] = sum_{q in s} T_jq,   rA[s][j] = sum_{q in s} (ye_s - y_q) T_jq
//   cS[b][q] = sum_{j in b} T_jq,   cX[b][q] = sum_{j in b} (xe_b - x_j) T_jq
// CTA = 256 threads, tile 256 x 256: warp w owns rows w, w+8, ..., lane L owns columns
// c0 + 8L .. c0 + 8L + 7 (two coalesced float4 per row).  Per row the lane's 8 values give its
// partial (P, A) of the row and feed its 8 column accumulators (fp32 over the tile's rows).
// Rows are taken 4 at a time: the 8 lane partials (4 rows x {P, A}) are reduced over the warp by
// recursive halving (9 shuffles instead of 40); fixed lane structure => deterministic.
// ---------------------------------------------------------------------------------
template <int MODE, bool COSTW = false>
__device__ __forceinline__ void moments3_body(const TSrc2& S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                              const double* __restrict__ yc, double* __restrict__ rP,
                                              double* __restrict__ rA, double* __restrict__ cS,
                                              double* __restrict__ cX) {
  __shared__ float red[2][8][TC];
  const int s = blockIdx.x, b = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)s * TC, r0 = (int64_t)b * TR;
  const int64_t q0 = c0 + 8 * lane;
  const double ye = yc[min(c0 + TC, m - 1)];
  const double xe = xl[min(r0 + TR, nl - 1)];
  float2 dy[4], gh[4], gl[4], cs[4], cx[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t q = q0 + 2 * k;
    dy[k] = make_float2(q < m ? (float)(ye - yc[q]) : 0.f, q + 1 < m ? (float)(ye - yc[q + 1]) : 0.f);
    gh[k] = make_float2(0.f, 0.f);
    gl[k] = gh[k];
    if (MODE != T_EXPLICIT) {
      gh[k] = make_float2(q < m ? S.gh[q] : 0.f, q + 1 < m ? S.gh[q + 1] : 0.f);
      if (MODE == T_GIBBS) gl[k] = make_float2(q < m ? S.gl[q] : 0.f, q + 1 < m ? S.gl[q + 1] : 0.f);
    }
    cs[k] = make_float2(0.f, 0.f);
    cx[k] = cs[k];
  }
  const float2 nch = make_float2(-S.ch, -S.ch), ncl = make_float2(-S.cl, -S.cl);
  const bool colsok = q0 + 8 <= m;  // all 8 columns of this lane are real
  const int nrows = (int)min((int64_t)TR, nl - r0);
  for (int rr = 0; rr < TR; rr += 32) {  // 4 rows per warp per group (8 warps x 4 = 32 rows)
    if (rr >= nrows) break;              // uniform
    float2 tv[4][4];                     // [row u][float2 k]
    float F[4], Fl[4], dxr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rl = rr + w + 8 * u;
      const int64_t j = r0 + rl;
      const bool jv = rl < nrows;
      F[u] = 0.f; Fl[u] = 0.f;
      if (MODE != T_EXPLICIT && jv) {
        F[u] = S.fh[j];
        if (MODE == T_GIBBS) Fl[u] = S.fl[j];
      }
      dxr[u] = jv ? (float)(xe - xl[j]) : 0.f;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
      if (MODE != T_PRODUCT && jv) {
        const float* row = S.T + j * S.ld + q0;
        if (q0 < m) a = __ldcs(reinterpret_cast<const float4*>(row));
        if (q0 + 4 < m) c = __ldcs(reinterpret_cast<const float4*>(row + 4));
      }
      tv[u][0] = make_float2(a.x, a.y); tv[u][1] = make_float2(a.z, a.w);
      tv[u][2] = make_float2(c.x, c.y); tv[u][3] = make_float2(c.z, c.w);
    }
    float part[8];  // [u][P, A]
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rl = rr + w + 8 * u;
      const bool jv = rl < nrows;
      float2 P2 = make_float2(0.f, 0.f), A2 = P2;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 graw = tv[u][k];  // the loaded value (GIBBS: the cost)
        float2 t = graw;
        if (MODE == T_GIBBS) {
          const float2 aa = fadd2(fadd2(ffma2(t, nch, gh[k]), make_float2(F[u], F[u])),
                                  ffma2(t, ncl, fadd2(gl[k], make_float2(Fl[u], Fl[u]))));
          t = make_float2(ex2_ftz(aa.x), ex2_ftz(aa.y));
        } else if (MODE == T_PRODUCT) {
          t = make_float2(F[u] * gh[k].x, F[u] * gh[k].y);
        }
        if (!jv) t = make_float2(0.f, 0.f);
        if (!colsok) {
          const int64_t q = q0 + 2 * k;
          if (q >= m) t.x = 0.f;
          if (q + 1 >= m) t.y = 0.f;
        }
        P2 = fadd2(P2, t);
        A2 = ffma2(COSTW ? graw : dy[k], t, A2);
        cs[k] = fadd2(cs[k], t);
        if (!COSTW) cx[k] = ffma2(make_float2(dxr[u], dxr[u]), t, cx[k]);
      }
      part[2 * u] = P2.x + P2.y;
      part[2 * u + 1] = A2.x + A2.y;
    }
    // recursive halving over the warp: 8 values -> lanes with (lane & 3) == 0 hold value lane >> 2
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool hi = lane & 16;
      const float send = hi ? part[i] : part[4 + i];
      const float keep = hi ? part[4 + i] : part[i];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool hi = lane & 8;
      const float send = hi ? part[i] : part[2 + i];
      const float keep = hi ? part[2 + i] : part[i];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool hi = lane & 4;
      const float send = hi ? part[0] : part[1];
      const float keep = hi ? part[1] : part[0];
      part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 2);
    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
    if ((lane & 3) == 0) {
      const int idx = lane >> 2;  // = 4 bit4 + 2 bit3 + bit2
      const int u = idx >> 1;
      const int rl = rr + w + 8 * u;
      const int64_t j = r0 + rl;
      if (rl < nrows) {
        if (idx & 1) rA[(int64_t)s * nl + j] = (double)part[0];
        else rP[(int64_t)s * nl + j] = (double)part[0];
      }
    }
  }
  // column partials: fixed-order sum over the 8 warps
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    red[0][w][8 * lane + 2 * k] = cs[k].x;
    red[0][w][8 * lane + 2 * k + 1] = cs[k].y;
    if (!COSTW) {
      red[1][w][8 * lane + 2 * k] = cx[k].x;
      red[1][w][8 * lane + 2 * k + 1] = cx[k].y;
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t q = c0 + t;
  if (q < m) {
    double a = 0.0, bx = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) {
      a += red[0][ww][t];
      if (!COSTW) bx += red[1][ww][t];
    }
    cS[b * m + q] = a;
    if (!COSTW) cX[b * m + q] = bx;
  }
}

// Gibbs mode (an ex2 per element, 126 registers): the compiler's own allocation, 2 CTAs per SM.
template <int MODE>
__global__ void __launch_bounds__(256) k_grad_moments3(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                       const double* __restrict__ yc, double* __restrict__ rP,
                                                       double* __restrict__ rA, double* __restrict__ cS,
                                                       double* __restrict__ cX) {
  moments3_body<MODE>(S, nl, m, xl, yc, rP, rA, cS, cX);
}

// Explicit T and the product plan: capped at 85 registers for 3 CTAs per SM (24 warps: more loads
// in flight; 11.4 -> 10.3 ms for the whole k = 1 gradient at N = M = 65536).
template <int MODE>
__global__ void __launch_bounds__(256, 3) k_grad_moments3o(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                           const double* __restrict__ yc, double* __restrict__ rP,
                                                           double* __restrict__ rA, double* __restrict__ cS,
                                                           double* __restrict__ cX) {
  moments3_body<MODE>(S, nl, m, xl, yc, rP, rA, cS, cX);
}

// UGW plan statistics in one read of the cost (Remark 3, reading R33; ugw.cuh): per (row, strip)
//   rP[s][j] = sum_{q in s} T_jq,  rC[s][j] = sum_{q in s} C_jq T_jq,  and per (block, column)
//   cS[b][q] = sum_{j in b} T_jq  of the Gibbs plan T = exp2(...) regenerated from the cost C.
__global__ void __launch_bounds__(256) k_ugw_moments(TSrc2 S, int64_t nl, int64_t m, const double* __restrict__ xl,
                                                     const double* __restrict__ yc, double* __restrict__ rP,
                                                     double* __restrict__ rC, double* __restrict__ cS) {
  moments3_body<T_GIBBS, true>(S, nl, m, xl, yc, rP, rC, cS, nullptr);
}

}  // namespace gw

namespace gw {

// ---------------------------------------------------------------------------------
// The gradient on the product plan T^0 = p q^T (the first outer iteration, PAPER.md:120-126 with a
// rank-1 plan): D_X T D_Y = (D_X p)(D_Y q)^T, so
//   G_ip = 2 c_i + 2 c'_p - 4 a_i b_p,   a = D_X p,  b = D_Y q   (1-D DPs)
// -- one write of G (4 N M bytes) instead of the general moments + main passes.  Thread: one float4 of
// columns x 32 rows; fp32 assembly of O(max|G|) terms as in the main pass (two roundings).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_grad_product(float* __restrict__ G, int64_t ld, int64_t nl, int64_t m,
                                                      const double* __restrict__ a, const double* __restrict__ c,
                                                      const double* __restrict__ b, const double* __restrict__ c2) {
  const int64_t q = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int64_t i0 = (int64_t)blockIdx.y * 32;
  if (q >= m) return;
  float bq[4], dq[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    bq[e] = q + e < m ? (float)b[q + e] : 0.f;
    dq[e] = q + e < m ? (float)(2.0 * c2[q + e]) : 0.f;
  }
  const bool full = q + 3 < m;
  const int nr = (int)min((int64_t)32, nl - i0);
  for (int r = 0; r < nr; ++r) {
    const int64_t i = i0 + r;
    const float A = (float)(-4.0 * a[i]), C = (float)(2.0 * c[i]);
    float g[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) g[e] = fmaf(A, bq[e], C + dq[e]);
    float* gp = G + i * ld + q;
    if (full) __stcs(reinterpret_cast<float4*>(gp), make_float4(g[0], g[1], g[2], g[3]));
    else
      for (int e = 0; e < 4 && q + e < m; ++e) gp[e] = g[e];
  }
}

}  // namespace gw

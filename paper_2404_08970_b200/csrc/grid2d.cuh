// grid2d.cuh -- the GW gradient on 2-D tensor grids at k = 1 (PAPER.md:280-360,
// the paper's Table 3 workload).
//
// Points i = a nx + b <-> (s_a, s_b) of an nx x nx grid with axis s (reading R31); Manhattan
// distance D_ij = |s_a - s_a'| + |s_b - s_b'|, i.e. D = D1 (x) J + J (x) D1 (k = 1).
// Then, with the four marginal matrices of the plan (T as a 4-index tensor T[a][b][c][d],
// columns q = c ny + d of the ny x ny grid of y)
//   T^AC[a][c] = sum_{b,d} T,  T^AD[a][d] = sum_{b,c} T,  T^BC[b][c] = sum_{a,d} T,  T^BD[b][d] = sum_{a,c} T,
//   (D_X T D_Y)[(a,b),(c,d)] = V_AC[a][c] + V_AD[a][d] + V_BC[b][c] + V_BD[b][d],  V_.. = D1x T^.. D1y.
// So the O(N M) gradient is one reduction pass over T (per-row sums over d and over c), tiny
// n^3 products, and one write pass; no scans.  The constant term c = (D o D) p and the objective
// use the same marginals: (D o D) p = sum_a' D1^2 P_A + sum_b' D1^2 P_B + 2 (D1 mat(p) D1).
#pragma once
#include "common.cuh"
#include "fused.cuh"  // ex2_ftz
#include "grad2.cuh"  // TSrc2, T_* modes

namespace gw {

constexpr int G2D_MAXN = 256;  // axis length limit (M = ny^2 <= 65536 per row)

// axis sortedness / finiteness and weight signs / sum; out[8] like k_validate
__global__ void __launch_bounds__(1024) k_g2_validate(const double* __restrict__ s, int64_t ns,
                                                      const double* __restrict__ w, int64_t nw,
                                                      double* __restrict__ out) {
  __shared__ double sm[32];
  double uns = 0, neg = 0, nf = 0, s0 = 0;
  for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
    if (!isfinite(s[i])) nf = 1;
    if (i + 1 < ns && !(s[i + 1] >= s[i])) uns = 1;
  }
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) {
    const double wi = w[i];
    if (!isfinite(wi)) nf = 1;
    if (wi < 0) neg = 1;
    s0 += wi;
  }
  uns = block_sum<32>(uns, sm);
  neg = block_sum<32>(neg, sm);
  nf = block_sum<32>(nf, sm);
  s0 = block_sum<32>(s0, sm);
  if (threadIdx.x == 0) {
    out[0] = uns; out[1] = neg; out[2] = nf; out[3] = s0;
    out[4] = 0; out[5] = 0; out[6] = 0.5 * (s[0] + s[ns - 1]); out[7] = 0;
  }
}

// wn = w / S0, lw = ln wn; axc = axis - mid
__global__ void k_g2_prep(const double* __restrict__ w, int64_t nw, const double* __restrict__ s, int64_t ns,
                          const double* __restrict__ mom, double* __restrict__ wn, double* __restrict__ lw,
                          double* __restrict__ sc) {
  const double inv = 1.0 / mom[3], mid = mom[6];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = w[i] * inv;
    wn[i] = v;
    lw[i] = log(v);
    if (i < ns) sc[i] = s[i] - mid;
  }
}

// WA[a] = sum_b w[a n + b], WB[b] = sum_a w[a n + b]  (fixed order)
__global__ void k_g2_wmarg(const double* __restrict__ w, int n, double* __restrict__ WA, double* __restrict__ WB) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    double v = 0.0;
    for (int b = 0; b < n; ++b) v += w[(int64_t)t * n + b];
    WA[t] = v;
  } else if (t < 2 * n) {
    const int b = t - n;
    double v = 0.0;
    for (int a = 0; a < n; ++a) v += w[(int64_t)a * n + b];
    WB[b] = v;
  }
}

// out[r][c] = sum_{c'} Min[r][c'] |sy_c - sy_c'|     (R x C times the C x C axis distance)
__global__ void k_g2_mul_right(const double* __restrict__ Min, int R, int C, const double* __restrict__ sy,
                               double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R * C) return;
  const int r = e / C, c = e - r * C;
  const double y = sy[c];
  double v = 0.0;
  for (int k = 0; k < C; ++k) v += Min[(int64_t)r * C + k] * fabs(y - sy[k]);
  out[e] = v;
}

// out[r][c] = sum_{r'} |sx_r - sx_r'| Min[r'][c]
__global__ void k_g2_mul_left(const double* __restrict__ sx, int R, const double* __restrict__ Min, int C,
                              double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R * C) return;
  const int r = e / C, c = e - r * C;
  const double x = sx[r];
  double v = 0.0;
  for (int k = 0; k < R; ++k) v += fabs(x - sx[k]) * Min[(int64_t)k * C + c];
  out[e] = v;
}

// out[a] = sum_a' (s_a - s_a')^2 W[a']
__global__ void k_g2_sqmv(const double* __restrict__ s, int n, const double* __restrict__ W, double* __restrict__ out) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  double v = 0.0;
  for (int k = 0; k < n; ++k) {
    const double d = s[a] - s[k];
    v += d * d * W[k];
  }
  out[a] = v;
}

// c[(a,b)] = vA[a] + vB[b] + 2 DWD[a][b]
__global__ void k_g2_const(const double* __restrict__ vA, const double* __restrict__ vB,
                           const double* __restrict__ DWD, int n, double* __restrict__ c) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * n) return;
  const int a = (int)(i / n), b = (int)(i - (int64_t)a * n);
  c[i] = vA[a] + vB[b] + 2.0 * DWD[i];
}

// Per-row reductions of the plan: RC[i][c] = sum_d T[i,(c,d)], RD[i][d] = sum_c T[i,(c,d)]
// (+ the row's entropy sum T (ln T - 1) when OBJ).  One CTA per row, thread d of the row's
// ny x ny view (coalesced over d), column sums in fp32 over <= 256 terms, fp64 outputs.
template <int MODE, bool OBJ>
__global__ void __launch_bounds__(G2D_MAXN) k_g2_rowred(TSrc2 S, int ny, double* __restrict__ RC,
                                                        double* __restrict__ RD, double* __restrict__ Hrow,
                                                        const double* __restrict__ fx, const double* __restrict__ fy,
                                                        double* __restrict__ CCrow) {
  __shared__ float wp[G2D_MAXN][G2D_MAXN / 32 + 1];
  const int64_t i = blockIdx.x;
  const int d = threadIdx.x, lane = d & 31, w = d >> 5;
  const bool dv = d < ny;
  float Fh = 0.f, Fl = 0.f;
  if (MODE != T_EXPLICIT) Fh = S.fh[i];
  if (MODE == T_GIBBS) Fl = S.fl[i];
  const float* row = (MODE == T_PRODUCT) ? nullptr : S.T + i * S.ld;
  float rd = 0.f, ent = 0.f, cc = 0.f;
  const float fxi = (OBJ && fx) ? (float)fx[i] : 0.f;
  float gq = 0.f, glq = 0.f;  // (column duals are per q: loaded per element below)
  constexpr int U = 8;        // loads of U columns c in flight per thread
  for (int c0 = 0; c0 < ny; c0 += U) {
    float raw[U], gqv[U], glv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      const int64_t q = (int64_t)c * ny + d;
      const bool ok = dv && c < ny;
      raw[u] = (ok && MODE != T_PRODUCT) ? row[q] : 0.f;
      gqv[u] = (ok && MODE != T_EXPLICIT) ? S.gh[q] : 0.f;
      glv[u] = (ok && MODE == T_GIBBS) ? S.gl[q] : 0.f;
    }
    float tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      float t = 0.f;
      if (dv && c < ny) {
        const int64_t q = (int64_t)c * ny + d;
        if (MODE == T_EXPLICIT) {
          t = raw[u];
        } else if (MODE == T_PRODUCT) {
          t = Fh * gqv[u];
        } else {
          gq = gqv[u];
          glq = glv[u];
          const float a = (fmaf(raw[u], -S.ch, gq) + Fh) + fmaf(raw[u], -S.cl, glq + Fl);
          t = ex2_ftz(a);
          if (OBJ && t > 0.f) ent += t * fmaf(a, 0.6931471805599453f, -1.f);
        }
        if (OBJ && MODE != T_GIBBS && t > 0.f) ent += t * (__logf(t) - 1.f);
        if (OBJ && fx) {
          const float df = fxi - (float)fy[q];
          cc = fmaf(df * df, t, cc);
        }
      }
      rd += t;
      tv[u] = t;
    }
    // warp sums of the U = 8 columns by recursive halving (9 shuffles for 8 sums instead of 40): lanes
    // with (lane & 3) == 0 end with column c0 + (lane >> 2); fixed lane structure -> deterministic
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) {  // lane bit 16 -> 4 values, bit 8 -> 2, bit 4 -> 1
      const int bit = 4 * h;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const bool hi = lane & bit;
        const float send = hi ? tv[k] : tv[h + k];
        const float keep = hi ? tv[h + k] : tv[k];
        tv[k] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
      }
    }
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 2);
    tv[0] += __shfl_xor_sync(0xffffffffu, tv[0], 1);
    if ((lane & 3) == 0 && c0 + (lane >> 2) < ny) wp[c0 + (lane >> 2)][w] = tv[0];
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) / 32;
  if (dv) {
    double v = 0.0;
    for (int k = 0; k < nw; ++k) v += (double)wp[d][k];
    RC[i * ny + d] = v;
    RD[i * ny + d] = (double)rd;
  }
  if (OBJ) {
    __shared__ double se[G2D_MAXN / 32], sc[G2D_MAXN / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ent += __shfl_xor_sync(0xffffffffu, ent, o);
      cc += __shfl_xor_sync(0xffffffffu, cc, o);
    }
    if (lane == 0) { se[w] = (double)ent; sc[w] = (double)cc; }
    __syncthreads();
    if (d == 0) {
      double h = 0.0, hc = 0.0;
      for (int k = 0; k < nw; ++k) { h += se[k]; hc += sc[k]; }
      Hrow[i] = h;
      if (fx) CCrow[i] = hc;
    }
  }
}

// The same row reductions (no OBJ terms) for ny = 4 TPR with TPR in {32, 64}: 128-bit loads.  Thread
// (phase, j) of the 256 covers d = 4j .. 4j + 3 of the c-rows c = phase + P k (P = 256 / TPR phases),
// eight c-rows' float4 in flight per thread (4x the bytes per load of the scalar kernel, which is
// load-latency bound); the 8 per-thread c-row partials are reduced over the warp by recursive halving,
// the TPR / 32 warps of a c-row and the P phases of a d are combined through shared memory in fixed
// order -> deterministic.
template <int MODE, int TPR>
__global__ void __launch_bounds__(256) k_g2_rowred4(TSrc2 S, double* __restrict__ RC, double* __restrict__ RD) {
  constexpr int NY = 4 * TPR, P = 256 / TPR, WPR = TPR / 32;  // WPR warps per c-row
  // c-rows per thread per batch (GIBBS loads the cost and both column-dual words: 4 keep the double
  // buffer in registers)
  constexpr int B = MODE == T_GIBBS ? 4 : 8;
  constexpr int LB = B == 8 ? 3 : 2;
  __shared__ float wp[NY][WPR];
  __shared__ float4 rdp[P][TPR];
  const int64_t i = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31;
  const int phase = t / TPR, j = t % TPR, wr = j / 32;  // wr: this warp's index within its c-row
  float Fh = 0.f, Fl = 0.f;
  if (MODE != T_EXPLICIT) Fh = S.fh[i];
  if (MODE == T_GIBBS) Fl = S.fl[i];
  const float4* row = (MODE == T_PRODUCT) ? nullptr : reinterpret_cast<const float4*>(S.T + i * S.ld);
  float4 rd = make_float4(0.f, 0.f, 0.f, 0.f);
  // software pipeline: the next batch's loads are issued before this batch's arithmetic (left to
  // itself the compiler sinks each load to its use at 32 registers: 4 loads in flight, not 8)
  float4 nraw[B], ng1[B], ng2[B];
  auto load = [&](int cb) {
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int c = cb + phase + P * k;
      const int64_t q4 = (int64_t)c * TPR + j;  // float4 index of (c, 4j)
      nraw[k] = MODE != T_PRODUCT ? __ldcs(row + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (MODE != T_EXPLICIT) ng1[k] = reinterpret_cast<const float4*>(S.gh)[q4];
      if (MODE == T_GIBBS) ng2[k] = reinterpret_cast<const float4*>(S.gl)[q4];
    }
  };
  load(0);
  for (int cb = 0; cb < NY; cb += P * B) {
    float4 raw[B], g1[B], g2[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      raw[k] = nraw[k];
      if (MODE != T_EXPLICIT) g1[k] = ng1[k];
      if (MODE == T_GIBBS) g2[k] = ng2[k];
    }
    if (cb + P * B < NY) load(cb + P * B);
    float v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      float4 tt;
      if (MODE == T_EXPLICIT) {
        tt = raw[k];
      } else if (MODE == T_PRODUCT) {
        tt = make_float4(Fh * g1[k].x, Fh * g1[k].y, Fh * g1[k].z, Fh * g1[k].w);
      } else {
        const float2 nch = make_float2(-S.ch, -S.ch), ncl = make_float2(-S.cl, -S.cl);
        const float2 F2 = make_float2(Fh, Fh), Fl2 = make_float2(Fl, Fl);
        const float2 a0 = fadd2(fadd2(ffma2(make_float2(raw[k].x, raw[k].y), nch, make_float2(g1[k].x, g1[k].y)), F2),
                                ffma2(make_float2(raw[k].x, raw[k].y), ncl, fadd2(make_float2(g2[k].x, g2[k].y), Fl2)));
        const float2 a1 = fadd2(fadd2(ffma2(make_float2(raw[k].z, raw[k].w), nch, make_float2(g1[k].z, g1[k].w)), F2),
                                ffma2(make_float2(raw[k].z, raw[k].w), ncl, fadd2(make_float2(g2[k].z, g2[k].w), Fl2)));
        tt = make_float4(ex2_ftz(a0.x), ex2_ftz(a0.y), ex2_ftz(a1.x), ex2_ftz(a1.y));
      }
      rd.x += tt.x; rd.y += tt.y; rd.z += tt.z; rd.w += tt.w;
      v[k] = (tt.x + tt.y) + (tt.z + tt.w);
    }
    // the warp's sums of the B c-rows by recursive halving: lanes whose low 5 - LB bits are zero end
    // with k = lane >> (5 - LB)
    int bit = 16;
#pragma unroll
    for (int h = B / 2; h >= 1; h >>= 1, bit >>= 1) {
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const bool hi = lane & bit;
        const float send = hi ? v[k] : v[h + k];
        const float keep = hi ? v[h + k] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
      }
    }
#pragma unroll
    for (int bb = 16 >> LB; bb >= 1; bb >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], bb);
    if ((lane & ((1 << (5 - LB)) - 1)) == 0) wp[cb + phase + P * (lane >> (5 - LB))][wr] = v[0];
  }
  rdp[phase][j] = rd;
  __syncthreads();
  // RC[c] = sum of the c-row's warp partials; RD[d] = sum over the phases (fixed order)
  for (int c = t; c < NY; c += 256) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < WPR; ++w) a += (double)wp[c][w];
    RC[i * NY + c] = a;
  }
  for (int d = t; d < NY; d += 256) {
    double a = 0.0;
#pragma unroll
    for (int ph = 0; ph < P; ++ph) {
      const float4 r4 = rdp[ph][d >> 2];
      const int e = d & 3;
      a += (double)(e == 0 ? r4.x : e == 1 ? r4.y : e == 2 ? r4.z : r4.w);
    }
    RD[i * NY + d] = a;
  }
}

// T^AC[a][c] = sum_b RC[(a,b)][c], T^BC[b][c] = sum_a RC, T^AD[a][d] = sum_b RD, T^BD[b][d] = sum_a RD,
// over this rank's rows [row0, row0 + nl) (RC, RD hold those rows; the ranks' partial matrices are
// all-gathered and summed in rank order).
__global__ void k_g2_marg(const double* __restrict__ RC, const double* __restrict__ RD, int nx, int ny, int64_t row0,
                          int64_t nl, double* __restrict__ TAC, double* __restrict__ TAD, double* __restrict__ TBC,
                          double* __restrict__ TBD) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 4 * nx * ny) return;
  const int which = e / (nx * ny), k = e - which * nx * ny;
  const int r = k / ny, col = k - r * ny;
  const double* src = (which == 0 || which == 2) ? RC : RD;
  double v = 0.0;
  for (int o = 0; o < nx; ++o) {  // which < 2: sum over b for fixed a = r; else over a for fixed b = r
    const int64_t i = which < 2 ? (int64_t)r * nx + o : (int64_t)o * nx + r;
    if (i >= row0 && i < row0 + nl) v += src[(i - row0) * ny + col];
  }
  double* dst = which == 0 ? TAC : which == 1 ? TAD : which == 2 ? TBC : TBD;
  dst[k] = v;
}

// G[i][q] = alpha (2 c_i + 2 c'_q - 4 (VAC[a][c] + VAD[a][d] + VBC[b][c] + VBD[b][d])) [+ (1-alpha)(fx_i - fy_q)^2]
// A CTA covers 2048 columns (8 per thread at stride 256: coalesced stores, and the per-row vector
// reads rd[d] hit consecutive shared-memory words) x G2SR rows; each thread keeps its
// columns' c'_q (and fy_q) in registers across the rows.  Per row the CTA forms the row's two
// ny-vectors in shared memory (double-buffered), the next row's V entries already in flight
// (loaded one row ahead into registers).  The terms are O(1) and cancel (G near its minimum is much
// smaller than c_i), so each element is summed in fp64 and rounded to fp32 once.
constexpr int G2SR = 32;
constexpr int G2SC = 8;  // columns per thread
// k_g2_store4: columns per thread (more columns per barrier; FGW keeps 16: its feature terms double the
// per-column registers)
template <bool FGW>
__host__ __device__ constexpr int g2sc4() { return FGW ? 16 : 32; }
template <bool FGW>
__global__ void __launch_bounds__(256) k_g2_store(const double* __restrict__ cX, const double* __restrict__ cY,
                                                  const double* __restrict__ VAC, const double* __restrict__ VAD,
                                                  const double* __restrict__ VBC, const double* __restrict__ VBD,
                                                  int nx, int ny, int64_t row0, int64_t nl, int64_t m, double alpha,
                                                  const double* __restrict__ fx, const double* __restrict__ fy,
                                                  float* __restrict__ G, int64_t ldG) {
  __shared__ double rc[2][G2D_MAXN], rd[2][G2D_MAXN];
  const int t = threadIdx.x;
  const int64_t qb = (int64_t)G2SC * blockIdx.x * blockDim.x + t;  // columns qb + 256 k
  const bool act = qb < m;
  const double a2 = 2.0 * alpha, a1 = 1.0 - alpha, a4 = -4.0 * alpha;
  double cy[G2SC], fyv[G2SC];
  int cc[G2SC], dd[G2SC];
#pragma unroll
  for (int k = 0; k < G2SC; ++k) {
    const int64_t q = act ? min(qb + 256 * k, m - 1) : 0;
    cc[k] = (int)(q / ny);
    dd[k] = (int)(q - (int64_t)cc[k] * ny);
    cy[k] = a2 * cY[q];
    fyv[k] = FGW ? fy[q] : 0.0;
  }
  const int64_t il0 = (int64_t)blockIdx.y * G2SR, il1 = min(nl, il0 + G2SR);
  const bool vt = t < ny;  // this thread forms entry t of the row's two vectors
  double vac = 0, vbc = 0, vad = 0, vbd = 0, cxi = 0;
  // grid coordinates (a, b) of row i = a nx + b, advanced incrementally (no division per row)
  int fa = (int)((row0 + il0) / nx), fb = (int)((row0 + il0) - (int64_t)fa * nx);
  auto fetch = [&](int64_t il) {
    const int64_t i = row0 + il;
    if (vt) {
      vac = VAC[(int64_t)fa * ny + t]; vbc = VBC[(int64_t)fb * ny + t];
      vad = VAD[(int64_t)fa * ny + t]; vbd = VBD[(int64_t)fb * ny + t];
      cxi = cX[i];
    }
    if (++fb == nx) { fb = 0; ++fa; }
  };
  if (il0 < il1) fetch(il0);
  for (int64_t il = il0; il < il1; ++il) {
    const int buf = (int)(il & 1);
    if (vt) {
      rc[buf][t] = fma(a4, vac + vbc, a2 * cxi);
      rd[buf][t] = a4 * (vad + vbd);
    }
    if (il + 1 < il1) fetch(il + 1);  // in flight during this row's stores
    __syncthreads();                  // (double buffer: the next row writes the other half)
    if (act) {
      const int64_t i = row0 + il;
      const double fxi = FGW ? fx[i] : 0.0;
      float o[G2SC];
#pragma unroll
      for (int k = 0; k < G2SC; ++k) {
        double v = rc[buf][cc[k]] + rd[buf][dd[k]] + cy[k];
        if (FGW) {
          const double d = fxi - fyv[k];
          v = fma(a1 * d, d, v);
        }
        o[k] = (float)v;
      }
      float* dst = G + il * ldG + qb;
#pragma unroll
      for (int k = 0; k < G2SC; ++k)
        if (qb + 256 * k < m) __stcs(dst + 256 * k, o[k]);
    }
  }
}

// The same store with 4 consecutive columns per thread group (ny % 4 == 0: the 4 share c, and d..d+3
// are consecutive): one rc read, two double2 rd reads and ONE 16-byte store per 4 elements; row grid
// coordinates advance incrementally (no division per row).  A CTA covers 256 g2sc4 columns: 32 per
// thread (16 with FGW) amortise each row's barrier and shared-memory staging over 8192 stores (3.78 ->
// 3.22 ms per store pass in ncu at 256^2 x 256^2, 8 columns per thread before).  (Reading the V rows straight
// from L1 without the shared-memory staging measured slower: 10.1 vs 8.4 ms per gradient.)
template <bool FGW>
__global__ void __launch_bounds__(256) k_g2_store4(const double* __restrict__ cX, const double* __restrict__ cY,
                                                   const double* __restrict__ VAC, const double* __restrict__ VAD,
                                                   const double* __restrict__ VBC, const double* __restrict__ VBD,
                                                   int nx, int ny, int64_t row0, int64_t nl, int64_t m, double alpha,
                                                   const double* __restrict__ fx, const double* __restrict__ fy,
                                                   float* __restrict__ G, int64_t ldG) {
  __shared__ __align__(16) double rc[2][G2D_MAXN], rd[2][G2D_MAXN];
  const int t = threadIdx.x;
  constexpr int NG = g2sc4<FGW>() / 4;  // groups of 4 columns per thread
  const int64_t qb = (int64_t)g2sc4<FGW>() * 256 * blockIdx.x + 4 * t;  // groups at qb + 1024 k
  const double a2 = 2.0 * alpha, a1 = 1.0 - alpha, a4 = -4.0 * alpha;
  double cy[NG][4], fyv[NG][4];
  int cc[NG], dd[NG];
  bool gv[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int64_t q = qb + 1024 * k;
    gv[k] = q < m;
    const int64_t qq = gv[k] ? q : 0;
    cc[k] = (int)(qq / ny);
    dd[k] = (int)(qq - (int64_t)cc[k] * ny);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      cy[k][e] = gv[k] ? a2 * cY[qq + e] : 0.0;
      fyv[k][e] = (FGW && gv[k]) ? fy[qq + e] : 0.0;
    }
  }
  const int64_t il0 = (int64_t)blockIdx.y * G2SR, il1 = min(nl, il0 + G2SR);
  const bool vt = t < ny;
  double vac = 0, vbc = 0, vad = 0, vbd = 0, cxi = 0;
  int fa = (int)((row0 + il0) / nx), fb = (int)((row0 + il0) - (int64_t)fa * nx);
  auto fetch = [&](int64_t il) {
    const int64_t i = row0 + il;
    if (vt) {
      vac = VAC[(int64_t)fa * ny + t]; vbc = VBC[(int64_t)fb * ny + t];
      vad = VAD[(int64_t)fa * ny + t]; vbd = VBD[(int64_t)fb * ny + t];
      cxi = cX[i];
    }
    if (++fb == nx) { fb = 0; ++fa; }
  };
  if (il0 < il1) fetch(il0);
  for (int64_t il = il0; il < il1; ++il) {
    const int buf = (int)(il & 1);
    if (vt) {
      rc[buf][t] = fma(a4, vac + vbc, a2 * cxi);
      rd[buf][t] = a4 * (vad + vbd);
    }
    if (il + 1 < il1) fetch(il + 1);
    __syncthreads();
    const int64_t i = row0 + il;
    const double fxi = FGW ? fx[i] : 0.0;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      if (!gv[k]) continue;
      const double r = rc[buf][cc[k]];
      const double2 d01 = *reinterpret_cast<const double2*>(&rd[buf][dd[k]]);
      const double2 d23 = *reinterpret_cast<const double2*>(&rd[buf][dd[k] + 2]);
      const double dv[4] = {d01.x, d01.y, d23.x, d23.y};
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double v = (r + dv[e]) + cy[k][e];
        if (FGW) {
          const double df = fxi - fyv[k][e];
          v = fma(a1 * df, df, v);
        }
        o[e] = (float)v;
      }
      __stcs(reinterpret_cast<float4*>(G + il * ldG + qb + 1024 * k), make_float4(o[0], o[1], o[2], o[3]));
    }
  }
}

// column sums of the plan (2-D objective / violation): part[chunk][q] over row chunks of 256
template <int MODE>
__global__ void __launch_bounds__(256) k_g2_colsum(TSrc2 S, int64_t nl, int64_t m, double* __restrict__ part) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * 256;
  if (q >= m) return;
  const int64_t r1 = min(nl, r0 + 256);
  double acc = 0.0;
  float ghq = 0.f, glq = 0.f;
  if (MODE != T_EXPLICIT) ghq = S.gh[q];
  if (MODE == T_GIBBS) glq = S.gl[q];
  for (int64_t i0 = r0; i0 < r1; i0 += 8) {
    float g8[8];  // 8 rows' loads first
#pragma unroll
    for (int v = 0; v < 8; ++v) g8[v] = (MODE != T_PRODUCT && i0 + v < r1) ? S.T[(i0 + v) * S.ld + q] : 0.f;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int64_t i = i0 + v;
      if (i >= r1) break;
      float t;
      if (MODE == T_EXPLICIT) {
        t = g8[v];
      } else if (MODE == T_PRODUCT) {
        t = S.fh[i] * ghq;
      } else {
        t = ex2_ftz((fmaf(g8[v], -S.ch, ghq) + S.fh[i]) + fmaf(g8[v], -S.cl, glq + S.fl[i]));
      }
      acc += (double)t;
    }
  }
  part[(int64_t)blockIdx.y * m + q] = acc;
}

__global__ void k_g2_colsum_reduce(const double* __restrict__ part, int nchunk, int64_t m, double* __restrict__ b) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m) return;
  double v = 0.0;
  for (int k = 0; k < nchunk; ++k) v += part[(int64_t)k * m + q];
  b[q] = v;
}

// a_i = sum_c RC[i][c] (row sums of the plan)
__global__ void k_g2_rowsum(const double* __restrict__ RC, int64_t nl, int ny, double* __restrict__ a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double v = 0.0;
  for (int c = 0; c < ny; ++c) v += RC[i * ny + c];
  a[i] = v;
}

// Objective at 2-D:  out = {E, viol, -, H, -, -, -, -}
//   E = a^T cA + b^T cB - 2 (<VAC, TAC> + <VAD, TAD> + <VBC, TBC> + <VBD, TBD>)
// with cA = (D o D) a, cB = (D o D) b computed by the constant-term kernels on the realised marginals.
__global__ void __launch_bounds__(1024) k_g2_objective(const double* __restrict__ a, const double* __restrict__ cA,
                                                       const double* __restrict__ p, int64_t n,
                                                       const double* __restrict__ b, const double* __restrict__ cB,
                                                       const double* __restrict__ q, int64_t m,
                                                       const double* __restrict__ VT, const double* __restrict__ TT,
                                                       int nxny4, const double* __restrict__ Hrow,
                                                       const double* __restrict__ CCrow, double* __restrict__ out) {
  __shared__ double sm[32];
  double ea = 0, eb = 0, vt = 0, h = 0, va = 0, vb = 0, ccs = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    ea += a[i] * cA[i];
    h += Hrow[i];
    if (CCrow) ccs += CCrow[i];
    va = fmax(va, fabs(a[i] - p[i]));
  }
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    eb += b[i] * cB[i];
    vb = fmax(vb, fabs(b[i] - q[i]));
  }
  for (int i = threadIdx.x; i < nxny4; i += blockDim.x) vt += VT[i] * TT[i];
  ea = block_sum<32>(ea, sm);
  eb = block_sum<32>(eb, sm);
  vt = block_sum<32>(vt, sm);
  h = block_sum<32>(h, sm);
  ccs = block_sum<32>(ccs, sm);
  __shared__ double smx[32];
  double vmax = fmax(va, vb);
  for (int o = 16; o > 0; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) smx[0] = fmax(smx[0], smx[k]);
    out[0] = ea + eb - 2.0 * vt;
    out[1] = smx[0];
    out[2] = vt;
    out[3] = h;
    out[6] = ccs;
  }
}

}  // namespace gw

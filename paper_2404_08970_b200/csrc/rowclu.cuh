// rowclu.cuh -- the solver's DP gradient in ONE read of the cost and ONE write of G (8 N M bytes,
// SURVEY §8(d) M1), k = 1, one rank.
//
// G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y, evaluated in the order D_X (T D_Y):
//   B = T D_Y,  B_ip = sum_q T_iq |y_q - y_p| = y_p (2 P_<p - R_i) - (2 Y_<p - (Ty)_i)        (row DP)
//     with P_<p = sum_{q<p} T_iq, Y_<p = sum_{q<p} y_q T_iq, R_i = (T 1)_i, (Ty)_i  -- all of ROW i only;
//   (D_X B)_ip = sum_j |x_i - x_j| B_jp = x_i U_ip - Z_ip                                    (column DP)
//     with U_ip = 2 sum_{j<i} B_jp - sum_j B_jp,  Z_ip = 2 sum_{j<i} x_j B_jp - sum_j x_j B_jp
// (the j = i and q = p terms cancel; ties contribute |.| = 0 either way).  This is the paper's
// forward/backward pair of 1-D recursions run along rows, then along columns.
//
// Why one read suffices on the solver path: a thread-block cluster spans whole rows (as in the fused
// Sinkhorn kernel), so the row DP of row i needs only row i (its totals R_i, (Ty)_i and the prefix
// offsets of the CTAs / warps to its left arrive through DSMEM); a cluster owns a contiguous row range
// and walks it top-down, so the column DP needs only the state U, Z at the cluster's first row.  That
// state is a 1-D DP of the COLUMN partials of T over the rows above:
//   sum_{j in S} B_jp = (D_Y (T_S^T 1))_p,   sum_{j in S} x_j B_jp = (D_Y (T_S^T x))_p,
// and the column partials of the final plan T^l per cluster are exactly the last Sinkhorn sweep's
// half-step column sums rescaled by the column update: T^l = diag(w) E diag(q/CS), so
// sum_{i in c} T^l_ip = (q_p / CS_p) sum_{i in c} e_ip w_i (and likewise with x_i).  The last sweep of
// every inner loop runs the XM instantiation of k_sink_fused2 (fused.cuh), which accumulates both
// sums per cluster with the exponent in the same (Gibbs-regeneration) form as this kernel.
//
// Precision: the row DP is fp32 over one row with hierarchical sums (thread 16 -> warp scan -> 8 x CL
// partials; every term non-negative) and one rounding of each prefix against the row total; the column
// state is fp64 (shared memory) re-based every RC_FLUSH rows with fp32 increments in between; the
// assembly V = x_i U + Zn is one fp32 fma on O(max|G|) terms.
//
// RCX_* macros are timing-only switches of the standalone harness scripts/rc_bench.cu (they remove one
// part of the kernel, giving wrong results); the product build never defines them.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "fused.cuh"

namespace gw {

#ifndef RC_NT_DEF
#define RC_NT_DEF 256
#endif
constexpr int RC_NT = RC_NT_DEF;        // threads per CTA
constexpr int RC_W = 4096;              // columns per CTA
constexpr int RC_KC = RC_W / RC_NT;     // contiguous columns per thread (16 or 8)
constexpr int RC_KP = RC_KC / 2;        // column pairs per thread
constexpr int RC_NCH = RC_KC / 4;       // 16-B chunks per thread and row
constexpr int RC_TPL = 32 / RC_KC;      // threads per 128-B line
constexpr int RC_RS = 7;                // TMA ring stages (rows of the CTA slice, 16 KB each)
constexpr int RC_FLUSH = 32;            // rows between fp32 -> fp64 column-state re-basing

struct RcArgs {
  float* G;                   // in: the cost G^l (the plan is regenerated from it); out: G^{l+1} (in place)
  int64_t ld, nl, m, rows_per_cluster;
  const float *fh, *fl, *gh, *gl;  // f log2e/eps, g log2e/eps of T^l: fp32 hi / lo
  float ch, cl;                    // log2e/eps hi / lo
  const float* dxf;  // x_{i+1} - x_i (fp32, local rows; 0 for the last)
  const double* xc;  // centred x (fp64, local rows)
  const float* ccx;  // 2 c_i (fp32, local rows)
  const float* yf;   // centred y (fp32)
  const float* ccy;  // 2 c'_p (fp32)
  const double* U0;  // [ncl][m] column state U at each cluster's first row
  const double* Zn0; // [ncl][m] -Z there (V = x U + Zn = (D_X B) at that row)
};

__host__ __device__ constexpr size_t rc_dyn_smem() {
  return 1024 + (size_t)RC_RS * RC_W * sizeof(float) + (size_t)2 * RC_KC * RC_NT * sizeof(double) +
         (size_t)2 * RC_KC * RC_NT * sizeof(float);
}

// TMA tile load of one 4096-column row slice as a [128][32] fp32 box, 128-byte swizzle: the 16-B chunk
// j of 128-B line r lands at r*128 + 16 (j ^ (r & 7)), so the 16 contiguous columns of a thread (half a
// line) are read with four conflict-free LDS.128
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// One CTA = 256 threads x 16 contiguous columns; a cluster of CL CTAs spans a row; cluster cid owns
// rows [cid rpc, (cid + 1) rpc) and walks them top-down in PAIRS of rows.  Per pair step P (no CTA-wide
// barrier, as in k_sink_fused2): produce(P) -- regenerate T on rows 2P, 2P+1, the threads' totals, one
// warp scan of the four values, the warp totals of both rows in ONE 16-byte st.async to every CTA of
// the cluster -- then consume(P - 1): the (rank, warp) partials of the previous pair give R, (Ty) and
// this warp's offset for both rows (one butterfly of eight values); the row DP gives B, G is stored, and
// the column state advances down the two rows.  The two rows' chains interleave (latency per row
// halved; the kernel is latency bound at 2 warps per scheduler).
template <int CL>
__global__ void __launch_bounds__(RC_NT, 1) k_grad_rc(const __grid_constant__ CUtensorMap tmap, RcArgs a) {
  constexpr int NW = RC_NT / 32;
  constexpr int NX = CL * NW;               // partials per row pair
  constexpr int NXP = NX < 32 ? 32 : NX;    // padded so that every lane reads a slot
  constexpr int PER = NXP / 32;             // partials per lane
  constexpr int NSLOT = 4;
  extern __shared__ unsigned char rc_raw[];
  // 1024-B aligned ring (128-byte swizzle); offset from the shared base keeps the shared address space
  float* ring = reinterpret_cast<float*>(rc_raw + ((1024u - (smem_u32(rc_raw) & 1023u)) & 1023u));
  double* U64 = reinterpret_cast<double*>(ring + (size_t)RC_RS * RC_W);  // [16][NT]  U
  double* V64 = U64 + RC_KC * RC_NT;                                       // [16][NT]  V = D_X B
  float4* sgh = reinterpret_cast<float4*>(V64 + RC_KC * RC_NT);           // [4][NT]  g_hi (16 columns)
  float4* sgl = sgh + RC_NCH * RC_NT;                                      // [NCH][NT]  g_lo
  __shared__ __align__(8) uint64_t full[RC_RS];
  __shared__ unsigned int scnt[RC_RS];
  __shared__ __align__(8) uint64_t xbar[NSLOT];
  __shared__ __align__(16) float4 xs[NSLOT][NXP];  // {T row 0, yT row 0, T row 1, yT row 1}
  // the pair's totals and the exclusive prefixes of this CTA's warps, reduced by ONE designated warp
  // (P mod NW) and published through a CTA-local mbarrier
  __shared__ __align__(16) float4 red[NSLOT][NW + 1];
  __shared__ __align__(8) uint64_t rbar[NSLOT];

  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t cr = blockIdx.x % CL;
  const int64_t cid = blockIdx.x / CL;
  const int64_t m = a.m, ld = a.ld;
  const int64_t c0 = (int64_t)cr * RC_W;
  const int64_t ncol = max((int64_t)0, min((int64_t)RC_W, m - c0));
  const int64_t rb = cid * a.rows_per_cluster;
  const int64_t re = min(a.nl, rb + a.rows_per_cluster);
  const int nrows = (int)max((int64_t)0, re - rb);
  const int npairs = (nrows + 1) >> 1;
  const int64_t q0 = c0 + (int64_t)RC_KC * t;  // this thread's first column
  const int nv = (int)max((int64_t)0, min((int64_t)RC_KC, m - q0));
  constexpr uint32_t xbytes = 16u * NX;
  constexpr uint32_t tbytes = RC_W * 4u;

  // padding slots (never written by peers) read as zero
  for (int i = NX + t; i < NXP; i += RC_NT)
    for (int s = 0; s < NSLOT; ++s) xs[s][i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t == 0) {
    for (int s = 0; s < RC_RS; ++s) {
      mbar_init(&full[s], 1);
      scnt[s] = 0u;
    }
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&xbar[s], 1);
      mbar_init(&rbar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NSLOT && s < npairs; ++s) mbar_expect_tx(&xbar[s], xbytes);
  }
  __syncthreads();
  cluster_arrive();
  cluster_wait();
  const int cy = (int)(c0 / 32);
  if (t == 0 && ncol > 0) {
    for (int r = 0; r < RC_RS && r < nrows; ++r) {
      mbar_expect_tx(&full[r], tbytes);
      tma_load_3d(ring + (size_t)r * RC_W, &tmap, 0, cy, (int)(rb + r), &full[r]);
    }
  }

  // column state (pairs of adjacent columns): U = Uf + u, V = Vf + v with fp64 bases U64, V64 every
  // RC_FLUSH rows; Wf = 2c'_p - 4 Vf.  Down the column: G_i = Wf + 2c_i - 4 v;  U += 2 B_i;
  // V += (x_{i+1} - x_i) U  (V_{i+1} - V_i = dx_i (2 sum_{j<=i} B_j - sum_j B_j), PAPER.md:237-243 on columns)
  float2 y2[RC_KP], Uf[RC_KP], Wf[RC_KP], u2[RC_KP], v2[RC_KP];
  const double* U0 = a.U0 + cid * m;
  const double* Zn0 = a.Zn0 + cid * m;
  const double x0 = nrows > 0 ? a.xc[rb] : 0.0;
  {
    float gh[RC_KC], gl[RC_KC];
#pragma unroll
    for (int k = 0; k < RC_KP; ++k) {
      float yv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = 2 * k + h;
        const int64_t q = q0 + kk;
        const bool ok = kk < nv;
        gh[kk] = ok ? a.gh[q] : 0.f;
        gl[kk] = ok ? a.gl[q] : 0.f;
        yv[h] = ok ? a.yf[q] : 0.f;
        const double U = ok ? U0[q] : 0.0, V = ok ? fma(x0, U0[q], Zn0[q]) : 0.0;
        const double cp = ok ? (double)a.ccy[q] : 0.0;
        U64[kk * RC_NT + t] = U;
        V64[kk * RC_NT + t] = V;
        if (h == 0) { Uf[k].x = (float)U; Wf[k].x = (float)(cp - 4.0 * V); }
        else { Uf[k].y = (float)U; Wf[k].y = (float)(cp - 4.0 * V); }
      }
      y2[k] = make_float2(yv[0], yv[1]);
      u2[k] = make_float2(0.f, 0.f);
      v2[k] = u2[k];
    }
#pragma unroll
    for (int c = 0; c < RC_NCH; ++c) {
      sgh[c * RC_NT + t] = make_float4(gh[4 * c], gh[4 * c + 1], gh[4 * c + 2], gh[4 * c + 3]);
      sgl[c * RC_NT + t] = make_float4(gl[4 * c], gl[4 * c + 1], gl[4 * c + 2], gl[4 * c + 3]);
    }
  }
  const float2 nch = make_float2(-a.ch, -a.ch), ncl = make_float2(-a.cl, -a.cl);
  const float* __restrict__ fh = a.fh + rb;
  const float* __restrict__ fl = a.fl + rb;
  const float* __restrict__ dxf = a.dxf + rb;
  const float* __restrict__ ccx = a.ccx + rb;
  float* __restrict__ Gout = a.G + rb * ld + q0;
  const uint32_t peer = (uint32_t)min(lane, CL - 1);
  const uint32_t rx0 = mapa(&xs[0][cr * NW + wid], peer), rbar0 = mapa(&xbar[0], peer);
  constexpr uint32_t XSTRIDE = sizeof(xs[0]), BSTRIDE = sizeof(uint64_t);
  // swizzled offsets (floats) of the thread's four 16-B chunks inside a stage
  const int rl = t / RC_TPL;
  int chunk_off[RC_NCH];
#pragma unroll
  for (int c = 0; c < RC_NCH; ++c) chunk_off[c] = rl * 32 + (((RC_NCH * (t % RC_TPL) + c) ^ (rl & 7)) << 2);

  // per-row scalars {F_hi, F_lo, x_{i+1} - x_i, 2 c_i}: lane l holds those of row 32 g + l of the current
  // 32-row group g (and prefetches group g + 1), broadcast by shuffles -- no global-load latency per row
  float4 rcur = make_float4(0.f, 0.f, 0.f, 0.f), rnxt = rcur;
  auto rload = [&](int g) {
    const int r = 32 * g + lane;
    return r < nrows ? make_float4(fh[r], fl[r], dxf[r], ccx[r]) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  rnxt = rload(0);

  // regenerate the plan on one row of the pair (stage st) into tv
  auto regen = [&](int j, float Fh, float Fl, float2 (&tv)[RC_KP]) {
    const int st = j % RC_RS;
    mbar_wait(&full[st], (uint32_t)((j / RC_RS) & 1));
    const float* sp = ring + (size_t)st * RC_W;
    float4 gv[RC_NCH];
#pragma unroll
    for (int c = 0; c < RC_NCH; ++c) gv[c] = *reinterpret_cast<const float4*>(sp + chunk_off[c]);
    const float2 F2 = make_float2(Fh, Fh), L2 = make_float2(Fl, Fl);
#pragma unroll
    for (int c = 0; c < RC_NCH; ++c) {
      const float4 h4 = sgh[c * RC_NT + t], l4 = sgl[c * RC_NT + t];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 2 * c + e;
        const float2 g = e ? make_float2(gv[c].z, gv[c].w) : make_float2(gv[c].x, gv[c].y);
        const float2 gh = e ? make_float2(h4.z, h4.w) : make_float2(h4.x, h4.y);
        const float2 gl = e ? make_float2(l4.z, l4.w) : make_float2(l4.x, l4.y);
#ifdef RCX_NOREGEN
        tv[k] = g;
#else
        const float2 ae = fadd2(fadd2(ffma2(g, nch, gh), F2), ffma2(g, ncl, fadd2(gl, L2)));
        tv[k] = make_float2(ex2_ftz(ae.x), ex2_ftz(ae.y));
#endif
      }
    }
    if (nv < RC_KC) {
#pragma unroll
      for (int k = 0; k < RC_KP; ++k) {
        if (2 * k >= nv) tv[k].x = 0.f;
        if (2 * k + 1 >= nv) tv[k].y = 0.f;
      }
    }
  };
  auto release = [&](int j) {  // the last warp to release a stage refills it with row j + RS
    const int st = j % RC_RS;
    if (atomicAdd(&scnt[st], 1u) == NW - 1) {
      scnt[st] = 0u;
      const int nxt = j + RC_RS;
      if (nxt < nrows) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], tbytes);
        tma_load_3d(ring + (size_t)st * RC_W, &tmap, 0, cy, (int)(rb + nxt), &full[st]);
      }
    }
  };

  // produce pair P: plan values of both rows, the lane-exclusive warp prefixes `off` = {T0, yT0, T1, yT1}
  // of the thread's first column, and the rows' {dx, 2 c_i} in `xc`
  auto produce = [&](int P, float2 (&t0)[RC_KP], float2 (&t1)[RC_KP], float4& off, float4& xc) {
    const int j0 = 2 * P, j1 = j0 + 1;
    if ((j0 & 31) == 0) {
      rcur = rnxt;
      rnxt = rload((j0 >> 5) + 1);
    }
    const int s0 = j0 & 31;
    const float Fh0 = __shfl_sync(0xffffffffu, rcur.x, s0), Fl0 = __shfl_sync(0xffffffffu, rcur.y, s0);
    const float Fh1 = __shfl_sync(0xffffffffu, rcur.x, s0 + 1), Fl1 = __shfl_sync(0xffffffffu, rcur.y, s0 + 1);
    xc = make_float4(__shfl_sync(0xffffffffu, rcur.z, s0), __shfl_sync(0xffffffffu, rcur.w, s0),
                     __shfl_sync(0xffffffffu, rcur.z, s0 + 1), __shfl_sync(0xffffffffu, rcur.w, s0 + 1));
    if (ncol > 0) {
      regen(j0, Fh0, Fl0, t0);
      if (j1 < nrows) regen(j1, Fh1, Fl1, t1);
      else {
#pragma unroll
        for (int k = 0; k < RC_KP; ++k) t1[k] = make_float2(0.f, 0.f);
      }
      __syncwarp();
      if (lane == 0) {
        release(j0);
        if (j1 < nrows) release(j1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < RC_KP; ++k) t0[k] = t1[k] = make_float2(0.f, 0.f);
    }
    // thread totals {sum t, sum y t} of both rows, pairwise
    float2 p0 = make_float2(0.f, 0.f), q0s = p0, p1 = p0, q1s = p0;
#pragma unroll
    for (int k = 0; k < RC_KP; ++k) {
      p0 = fadd2(p0, t0[k]);
      q0s = ffma2(y2[k], t0[k], q0s);
      p1 = fadd2(p1, t1[k]);
      q1s = ffma2(y2[k], t1[k], q1s);
    }
    float4 it = make_float4(p0.x + p0.y, q0s.x + q0s.y, p1.x + p1.y, q1s.x + q1s.y);
#ifndef RCX_NOSCAN
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // warp inclusive scan of the four totals
      const float u0 = __shfl_up_sync(0xffffffffu, it.x, d), u1 = __shfl_up_sync(0xffffffffu, it.y, d);
      const float u2s = __shfl_up_sync(0xffffffffu, it.z, d), u3 = __shfl_up_sync(0xffffffffu, it.w, d);
      if (lane >= d) { it.x += u0; it.y += u1; it.z += u2s; it.w += u3; }
    }
    off = make_float4(__shfl_up_sync(0xffffffffu, it.x, 1), __shfl_up_sync(0xffffffffu, it.y, 1),
                      __shfl_up_sync(0xffffffffu, it.z, 1), __shfl_up_sync(0xffffffffu, it.w, 1));
    if (lane == 0) off = make_float4(0.f, 0.f, 0.f, 0.f);
#else
    off = it;
#endif
    const float4 w4 = make_float4(__shfl_sync(0xffffffffu, it.x, 31), __shfl_sync(0xffffffffu, it.y, 31),
                                  __shfl_sync(0xffffffffu, it.z, 31), __shfl_sync(0xffffffffu, it.w, 31));
    const int xsl = P & (NSLOT - 1);
    if (lane < CL)
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                       rx0 + XSTRIDE * xsl),
                   "f"(w4.x), "f"(w4.y), "f"(w4.z), "f"(w4.w), "r"(rbar0 + BSTRIDE * xsl)
                   : "memory");
  };

  // one row of the consumed pair: row DP -> B, G stored, column state advanced
  auto row_out = [&](int jp, const float2 (&tv)[RC_KP], float a0, float b0, float dx, float ci) {
    const float2 two = make_float2(2.f, 2.f), mtwo = make_float2(-2.f, -2.f), m4 = make_float2(-4.f, -4.f);
    const float2 a02 = make_float2(a0, a0), b02 = make_float2(b0, b0);
    const float2 ci2 = make_float2(ci, ci), dx2 = make_float2(dx, dx);
    float2 Gv[RC_KP];
    float lp = 0.f, ly = 0.f;  // in-thread exclusive prefixes (sum t, sum y t)
#pragma unroll
    for (int k = 0; k < RC_KP; ++k) {
      float2 lpk, lyk;
      lpk.x = lp;
      lyk.x = ly;
      lp += tv[k].x;
      ly = fmaf(y2[k].x, tv[k].x, ly);
      lpk.y = lp;
      lyk.y = ly;
      lp += tv[k].y;
      ly = fmaf(y2[k].y, tv[k].y, ly);
      const float2 av = ffma2(two, lpk, a02);
      const float2 bv = ffma2(mtwo, lyk, b02);
      const float2 B = ffma2(y2[k], av, bv);                 // B_ip = y_p a - b
      Gv[k] = fadd2(ffma2(m4, v2[k], Wf[k]), ci2);           // 2c'_p - 4 V + 2c_i
      u2[k] = ffma2(two, B, u2[k]);                          // U_{i+1}
      v2[k] = ffma2(dx2, fadd2(Uf[k], u2[k]), v2[k]);        // V_{i+1} = V_i + dx_i U_{i+1}
    }
#ifdef RCX_NOSTORE
    if (ncol < 0) {
#else
    if (ncol > 0) {
#endif
      float* gp = Gout + (int64_t)jp * ld;
      if (nv == RC_KC) {  // two 256-bit stores: each lane writes whole 32-B sectors
#pragma unroll
        for (int h = 0; h < RC_KC / 8; ++h)
          asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(gp + 8 * h),
                       "f"(Gv[4 * h].x), "f"(Gv[4 * h].y), "f"(Gv[4 * h + 1].x), "f"(Gv[4 * h + 1].y),
                       "f"(Gv[4 * h + 2].x), "f"(Gv[4 * h + 2].y), "f"(Gv[4 * h + 3].x), "f"(Gv[4 * h + 3].y)
                       : "memory");
      } else {
#pragma unroll
        for (int k = 0; k < RC_KP; ++k) {
          if (2 * k < nv) gp[2 * k] = Gv[k].x;
          if (2 * k + 1 < nv) gp[2 * k + 1] = Gv[k].y;
        }
      }
    }
    if ((jp & (RC_FLUSH - 1)) == RC_FLUSH - 1) {  // re-base the column state in fp64
#pragma unroll
      for (int k = 0; k < RC_KP; ++k) {
        double* U = U64 + (2 * k) * RC_NT + t;
        double* V = V64 + (2 * k) * RC_NT + t;
        const double U_0 = U[0] + (double)u2[k].x, U_1 = U[RC_NT] + (double)u2[k].y;
        const double V_0 = V[0] + (double)v2[k].x, V_1 = V[RC_NT] + (double)v2[k].y;
        U[0] = U_0; U[RC_NT] = U_1; V[0] = V_0; V[RC_NT] = V_1;
        const int64_t q = q0 + 2 * k;
        const double cp0 = 2 * k < nv ? (double)a.ccy[q] : 0.0, cp1 = 2 * k + 1 < nv ? (double)a.ccy[q + 1] : 0.0;
        Uf[k] = make_float2((float)U_0, (float)U_1);
        Wf[k] = make_float2((float)(cp0 - 4.0 * V_0), (float)(cp1 - 4.0 * V_1));
        u2[k] = make_float2(0.f, 0.f);
        v2[k] = u2[k];
      }
    }
  };

  // consume pair Pp: totals and this warp's offsets for both rows, then the two rows in order
  auto consume = [&](int Pp, const float2 (&t0)[RC_KP], const float2 (&t1)[RC_KP], float4 off, float4 xc) {
    const int psl = Pp & (NSLOT - 1);
    float4 tot, pre;
#ifndef RCX_NOEXCH
    if (wid == (Pp & (NW - 1))) {
      // designated warp: lane l holds entries [l PER, (l + 1) PER) in column order; inclusive scan
      mbar_wait(&xbar[psl], (uint32_t)((Pp / NSLOT) & 1));
      float4 e[PER], run = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        e[i] = xs[psl][lane * PER + i];
        run.x += e[i].x; run.y += e[i].y; run.z += e[i].z; run.w += e[i].w;
      }
      if (lane == 0 && Pp + NSLOT < npairs) mbar_expect_tx(&xbar[psl], xbytes);  // xs[psl] consumed
      float4 inc = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float u0 = __shfl_up_sync(0xffffffffu, inc.x, d), u1 = __shfl_up_sync(0xffffffffu, inc.y, d);
        const float u2s = __shfl_up_sync(0xffffffffu, inc.z, d), u3 = __shfl_up_sync(0xffffffffu, inc.w, d);
        if (lane >= d) { inc.x += u0; inc.y += u1; inc.z += u2s; inc.w += u3; }
      }
      float4 ex = make_float4(__shfl_up_sync(0xffffffffu, inc.x, 1), __shfl_up_sync(0xffffffffu, inc.y, 1),
                              __shfl_up_sync(0xffffffffu, inc.z, 1), __shfl_up_sync(0xffffffffu, inc.w, 1));
      if (lane == 0) ex = make_float4(0.f, 0.f, 0.f, 0.f);
      tot = make_float4(__shfl_sync(0xffffffffu, inc.x, 31), __shfl_sync(0xffffffffu, inc.y, 31),
                        __shfl_sync(0xffffffffu, inc.z, 31), __shfl_sync(0xffffffffu, inc.w, 31));
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int idx = lane * PER + i;
        if (idx >= (int)cr * NW && idx < (int)cr * NW + NW) red[psl][idx - (int)cr * NW] = ex;
        ex.x += e[i].x; ex.y += e[i].y; ex.z += e[i].z; ex.w += e[i].w;
      }
      if (lane == 0) red[psl][NW] = tot;
      __syncwarp();
      pre = red[psl][wid];
      if (lane == 0) mbar_arrive(&rbar[psl]);
    } else {
      mbar_wait(&rbar[psl], (uint32_t)((Pp / NSLOT) & 1));
      tot = red[psl][NW];
      pre = red[psl][wid];
    }
#else
    tot = pre = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
    // a = 2 P_<p - R_i,  nb = (Ty)_i - 2 Y_<p  at the thread's first column
    const int jp0 = 2 * Pp, jp1 = jp0 + 1;
    row_out(jp0, t0, fmaf(2.f, pre.x + off.x, -tot.x), fmaf(-2.f, pre.y + off.y, tot.y), xc.x, xc.y);
    if (jp1 < nrows) row_out(jp1, t1, fmaf(2.f, pre.z + off.z, -tot.z), fmaf(-2.f, pre.w + off.w, tot.w), xc.z, xc.w);
  };

  float2 tA0[RC_KP], tA1[RC_KP], tB0[RC_KP], tB1[RC_KP];
  float4 offA, offB, xcA, xcB;
  for (int P = 0; P <= npairs; P += 2) {
    if (P < npairs) produce(P, tA0, tA1, offA, xcA);
    if (P > 0) consume(P - 1, tB0, tB1, offB, xcB);
    if (P + 1 <= npairs) {
      if (P + 1 < npairs) produce(P + 1, tB0, tB1, offB, xcB);
      consume(P, tA0, tA1, offA, xcA);
    }
  }
  cluster_arrive();
  cluster_wait();
}

// x_{i+1} - x_i (fp32) of the local rows, 0 for the last
__global__ void k_rc_dx(const double* __restrict__ x, int64_t nl, float* __restrict__ dx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = i + 1 < nl ? (float)(x[i + 1] - x[i]) : 0.f;
}

// Column partials of T^l per cluster -> the signed prefix vectors whose D_Y gives each cluster's
// starting column state (grid-stride over columns, fixed order over clusters):
//   r_p = q_p / CS_p,  v_c = r (2 sum_{c'<c} part_c' - sum_c' part_c'),  vx_c likewise with partx
__global__ void k_rc_vec(const double* __restrict__ part, const double* __restrict__ partx, int ncl, int64_t m,
                         const double* __restrict__ cs, const double* __restrict__ lq, double* __restrict__ V,
                         double* __restrict__ VX) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    const double r = (lq[p] == -INFINITY) ? 0.0 : exp(lq[p]) / cs[p];
    double tot = 0.0, totx = 0.0;
    for (int c = 0; c < ncl; ++c) {
      tot += part[(int64_t)c * m + p];
      totx += partx[(int64_t)c * m + p];
    }
    double run = 0.0, runx = 0.0;
    for (int c = 0; c < ncl; ++c) {
      V[(int64_t)c * m + p] = r * (2.0 * run - tot);
      VX[(int64_t)c * m + p] = r * (2.0 * runx - totx);
      run += part[(int64_t)c * m + p];
      runx += partx[(int64_t)c * m + p];
    }
  }
}

// out_c = sgn * D_Y v_c, one CTA (1024 threads) per vector (blockIdx.x = vector index):
//   (D_Y v)_p = y_p (2 S_<p - S) - (2 Y_<p - Y),  S_<p = sum_{q<p} v_q,  Y_<p = sum_{q<p} y_q v_q  (fp64)
// vectors [0, ncl): v = V, sgn = +1 -> U0;  [ncl, 2 ncl): v = VX, sgn = -1 -> Zn0
__global__ void __launch_bounds__(1024) k_rc_dy(const double* __restrict__ V, const double* __restrict__ VX, int ncl,
                                                int64_t m, const double* __restrict__ y, double* __restrict__ U0,
                                                double* __restrict__ Zn0) {
  __shared__ double ws[2][32];
  __shared__ double tot[2];
  const int b = blockIdx.x;
  const bool isx = b >= ncl;
  const int c = isx ? b - ncl : b;
  const double* v = (isx ? VX : V) + (int64_t)c * m;
  double* out = (isx ? Zn0 : U0) + (int64_t)c * m;
  const double sg = isx ? -1.0 : 1.0;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t chunk = (m + 1023) / 1024;
  const int64_t lo = min(m, (int64_t)t * chunk), hi = min(m, lo + chunk);
  double s = 0.0, sy = 0.0;
  for (int64_t q = lo; q < hi; ++q) {
    s += v[q];
    sy += y[q] * v[q];
  }
  // block exclusive scan of (s, sy)
  double is = s, iy = sy;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double us = __shfl_up_sync(0xffffffffu, is, d), uy = __shfl_up_sync(0xffffffffu, iy, d);
    if (lane >= d) { is += us; iy += uy; }
  }
  if (lane == 31) { ws[0][w] = is; ws[1][w] = iy; }
  __syncthreads();
  if (w == 0) {
    double a0 = ws[0][lane], a1 = ws[1][lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double u0 = __shfl_up_sync(0xffffffffu, a0, d), u1 = __shfl_up_sync(0xffffffffu, a1, d);
      if (lane >= d) { a0 += u0; a1 += u1; }
    }
    ws[0][lane] = a0;
    ws[1][lane] = a1;
    if (lane == 31) { tot[0] = a0; tot[1] = a1; }
  }
  __syncthreads();
  double S = (w ? ws[0][w - 1] : 0.0) + (is - s), Y = (w ? ws[1][w - 1] : 0.0) + (iy - sy);
  const double St = tot[0], Yt = tot[1];
  for (int64_t q = lo; q < hi; ++q) {
    out[q] = sg * (y[q] * (2.0 * S - St) - (2.0 * Y - Yt));
    S += v[q];
    Y += y[q] * v[q];
  }
}

}  // namespace gw

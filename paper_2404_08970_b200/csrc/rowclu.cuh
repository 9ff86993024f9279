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
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "fused.cuh"

namespace gw {

constexpr int RC_NT = 256;              // threads per CTA
constexpr int RC_KC = 16;               // contiguous columns per thread
constexpr int RC_W = RC_NT * RC_KC;     // 4096 columns per CTA
constexpr int RC_RS = 8;                // TMA ring stages (rows of the CTA slice, 16 KB each)
constexpr int RC_FLUSH = 32;            // rows between fp32 -> fp64 column-state re-basing

struct RcArgs {
  float* G;                   // in: the cost G^l (the plan is regenerated from it); out: G^{l+1} (in place)
  int64_t ld, nl, m, rows_per_cluster;
  const float *fh, *fl, *gh, *gl;  // f log2e/eps, g log2e/eps of T^l: fp32 hi / lo
  float ch, cl;                    // log2e/eps hi / lo
  const float* xf;   // centred x (fp32, local rows)
  const float* ccx;  // 2 c_i (fp32, local rows)
  const float* yf;   // centred y (fp32)
  const float* ccy;  // 2 c'_p (fp32)
  const double* U0;  // [ncl][m] column state U at each cluster's first row
  const double* Zn0; // [ncl][m] -Z there
};

__host__ __device__ constexpr size_t rc_dyn_smem() {
  return 1024 + (size_t)RC_RS * RC_W * sizeof(float) + (size_t)2 * RC_KC * RC_NT * sizeof(double);
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
// rows [cid rpc, (cid + 1) rpc) and walks them top-down.  Per row j (no CTA-wide barrier, as in
// k_sink_fused2): produce(j) -- regenerate T, the thread's in-row exclusive prefixes, a warp scan, the
// warp totals st.async'ed to every CTA of the cluster -- then consume(j - 1): the (rank, warp) partials
// of row j - 1 give R, (Ty) and this warp's offset; the row DP gives B, the column state gives
// V = x U + Zn, G = 2c_i + 2c'_p - 4 V is stored, and U, Zn advance by 2B, -2xB.
template <int CL>
__global__ void __launch_bounds__(RC_NT, 1) k_grad_rc(const __grid_constant__ CUtensorMap tmap, RcArgs a) {
  constexpr int NW = RC_NT / 32;
  constexpr int NX = CL * NW;               // partials per row
  constexpr int NXP = NX < 32 ? 32 : NX;    // padded so that every lane reads a slot
  constexpr int PER = NXP / 32;             // partials per lane
  constexpr int NSLOT = 4;
  extern __shared__ unsigned char rc_raw[];
  float* ring = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(rc_raw) + 1023) & ~uintptr_t(1023));
  double* U64 = reinterpret_cast<double*>(ring + (size_t)RC_RS * RC_W);  // [16][NT]
  double* Z64 = U64 + RC_KC * RC_NT;                                       // [16][NT]  (-Z)
  __shared__ __align__(8) uint64_t full[RC_RS];
  __shared__ unsigned int scnt[RC_RS];
  __shared__ __align__(8) uint64_t xbar[NSLOT];
  __shared__ __align__(16) float2 xs[NSLOT][NXP];

  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t cr = blockIdx.x % CL;
  const int64_t cid = blockIdx.x / CL;
  const int64_t m = a.m, ld = a.ld;
  const int64_t c0 = (int64_t)cr * RC_W;
  const int64_t ncol = max((int64_t)0, min((int64_t)RC_W, m - c0));
  const int64_t rb = cid * a.rows_per_cluster;
  const int64_t re = min(a.nl, rb + a.rows_per_cluster);
  const int nrows = (int)max((int64_t)0, re - rb);
  const int64_t q0 = c0 + (int64_t)RC_KC * t;  // this thread's first column
  const int nv = (int)max((int64_t)0, min((int64_t)RC_KC, m - q0));
  constexpr uint32_t xbytes = 8u * NX;
  constexpr uint32_t tbytes = RC_W * 4u;

  // padding slots (never written by peers) read as zero
  for (int i = NX + t; i < NXP; i += RC_NT)
    for (int s = 0; s < NSLOT; ++s) xs[s][i] = make_float2(0.f, 0.f);
  if (t == 0) {
    for (int s = 0; s < RC_RS; ++s) {
      mbar_init(&full[s], 1);
      scnt[s] = 0u;
    }
    for (int s = 0; s < NSLOT; ++s) mbar_init(&xbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NSLOT && s < nrows; ++s) mbar_expect_tx(&xbar[s], xbytes);
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

  // per-column constants and the column state (pairs of adjacent columns)
  float2 gh2[8], gl2[8], y2[8], cp2[8], Uf[8], Zf[8], u2[8], z2[8];
  const double* U0 = a.U0 + cid * m;
  const double* Zn0 = a.Zn0 + cid * m;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float v[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 2 * k + h;
      const int64_t q = q0 + kk;
      const bool ok = kk < nv;
      v[h][0] = ok ? a.gh[q] : 0.f;
      v[h][1] = ok ? a.gl[q] : 0.f;
      v[h][2] = ok ? a.yf[q] : 0.f;
      v[h][3] = ok ? a.ccy[q] : 0.f;
      const double U = ok ? U0[q] : 0.0, Z = ok ? Zn0[q] : 0.0;
      U64[kk * RC_NT + t] = U;
      Z64[kk * RC_NT + t] = Z;
      if (h == 0) { Uf[k].x = (float)U; Zf[k].x = (float)Z; }
      else { Uf[k].y = (float)U; Zf[k].y = (float)Z; }
    }
    gh2[k] = make_float2(v[0][0], v[1][0]);
    gl2[k] = make_float2(v[0][1], v[1][1]);
    y2[k] = make_float2(v[0][2], v[1][2]);
    cp2[k] = make_float2(v[0][3], v[1][3]);
    u2[k] = make_float2(0.f, 0.f);
    z2[k] = u2[k];
  }
  const float2 nch = make_float2(-a.ch, -a.ch), ncl = make_float2(-a.cl, -a.cl);
  const float* __restrict__ fh = a.fh + rb;
  const float* __restrict__ fl = a.fl + rb;
  const float* __restrict__ xf = a.xf + rb;
  const float* __restrict__ ccx = a.ccx + rb;
  float* __restrict__ Gout = a.G + rb * ld + q0;
  const uint32_t peer = (uint32_t)min(lane, CL - 1);
  const uint32_t rx0 = mapa(&xs[0][cr * NW + wid], peer), rbar0 = mapa(&xbar[0], peer);
  constexpr uint32_t XSTRIDE = sizeof(xs[0]), BSTRIDE = sizeof(uint64_t);
  const int me = (int)cr * NW + wid;  // this warp's index in the row's column order
  // swizzled offsets (floats) of the thread's four 16-B chunks inside a stage
  const int rl = t >> 1;
  int chunk_off[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) chunk_off[c] = rl * 32 + (((4 * (t & 1) + c) ^ (rl & 7)) << 2);

  // per-row scalars {F_hi, F_lo, x_i, 2 c_i}: lane l holds those of row 32 g + l of the current 32-row
  // group g (and prefetches group g + 1), broadcast by shuffles -- no global-load latency per row
  float4 rcur = make_float4(0.f, 0.f, 0.f, 0.f), rnxt = rcur;
  auto rload = [&](int g) {
    const int r = 32 * g + lane;
    return r < nrows ? make_float4(fh[r], fl[r], xf[r], ccx[r]) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  rnxt = rload(0);

  // produce row j: the plan values t of the thread's 16 columns (pairs), the lane-exclusive warp prefix
  // `off` = (sum T, sum yT) of the thread's first column, and the row's {x_i, 2 c_i}
  auto produce = [&](int j, float2 (&tv)[8], float2& off, float2& xc) {
    if ((j & 31) == 0) {
      rcur = rnxt;
      rnxt = rload((j >> 5) + 1);
    }
    const int src = j & 31;
    const float Fh = __shfl_sync(0xffffffffu, rcur.x, src), Fl = __shfl_sync(0xffffffffu, rcur.y, src);
    xc = make_float2(__shfl_sync(0xffffffffu, rcur.z, src), __shfl_sync(0xffffffffu, rcur.w, src));
    if (ncol > 0) {
      const int st = j % RC_RS;
      mbar_wait(&full[st], (uint32_t)((j / RC_RS) & 1));
      const float* sp = ring + (size_t)st * RC_W;
      float4 gv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) gv[c] = *reinterpret_cast<const float4*>(sp + chunk_off[c]);
      const float2 F2 = make_float2(Fh, Fh), L2 = make_float2(Fl, Fl);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 g4 = gv[k >> 1];
        const float2 g = (k & 1) ? make_float2(g4.z, g4.w) : make_float2(g4.x, g4.y);
        const float2 ae = fadd2(fadd2(ffma2(g, nch, gh2[k]), F2), ffma2(g, ncl, fadd2(gl2[k], L2)));
        tv[k] = make_float2(ex2_ftz(ae.x), ex2_ftz(ae.y));
      }
      if (nv < RC_KC) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (2 * k >= nv) tv[k].x = 0.f;
          if (2 * k + 1 >= nv) tv[k].y = 0.f;
        }
      }
      __syncwarp();
      if (lane == 0) {  // release the stage; the last warp refills it with row j + RS
        if (atomicAdd(&scnt[st], 1u) == NW - 1) {
          scnt[st] = 0u;
          const int nxt = j + RC_RS;
          if (nxt < nrows) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[st], tbytes);
            tma_load_3d(ring + (size_t)st * RC_W, &tmap, 0, cy, (int)(rb + nxt), &full[st]);
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) tv[k] = make_float2(0.f, 0.f);
    }
    // thread totals (sum t, sum y t), pairwise
    float2 sp2 = make_float2(0.f, 0.f), sy2 = sp2;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sp2 = fadd2(sp2, tv[k]);
      sy2 = ffma2(y2[k], tv[k], sy2);
    }
    const float s = sp2.x + sp2.y, sy = sy2.x + sy2.y;
    // warp inclusive scan of the thread totals -> lane-exclusive prefix, warp total
    float it = s, iy = sy;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const float ut = __shfl_up_sync(0xffffffffu, it, d), uy = __shfl_up_sync(0xffffffffu, iy, d);
      if (lane >= d) { it += ut; iy += uy; }
    }
    const float et = __shfl_up_sync(0xffffffffu, it, 1), ey = __shfl_up_sync(0xffffffffu, iy, 1);
    off = lane ? make_float2(et, ey) : make_float2(0.f, 0.f);
    const float wt = __shfl_sync(0xffffffffu, it, 31), wy = __shfl_sync(0xffffffffu, iy, 31);
    const int xsl = j & (NSLOT - 1);
    if (lane < CL) st_async_v2f32(rx0 + XSTRIDE * xsl, wt, wy, rbar0 + BSTRIDE * xsl);
  };

  // consume row jp (local index): row DP, column DP, store
  auto consume = [&](int jp, const float2 (&tv)[8], float2 off, float2 xc) {
    const int psl = jp & (NSLOT - 1);
    mbar_wait(&xbar[psl], (uint32_t)((jp / NSLOT) & 1));
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);  // {tot T, tot yT, prefix T, prefix yT}
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int idx = lane * PER + i;
      const float2 v = xs[psl][idx];
      acc.x += v.x;
      acc.y += v.y;
      if (idx < me) {
        acc.z += v.x;
        acc.w += v.y;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, d);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, d);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, d);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, d);
    }
    if (t == 0 && jp + NSLOT < nrows) mbar_expect_tx(&xbar[psl], xbytes);
    const float xi = xc.x, ci = xc.y;
    // a_k = 2 P_<p - R_i,  nb_k = (Ty)_i - 2 Y_<p   at the thread's columns
    const float a0 = fmaf(2.f, acc.z + off.x, -acc.x);
    const float b0 = fmaf(-2.f, acc.w + off.y, acc.y);
    const float2 a02 = make_float2(a0, a0), b02 = make_float2(b0, b0);
    const float2 two = make_float2(2.f, 2.f), mtwo = make_float2(-2.f, -2.f), m4 = make_float2(-4.f, -4.f);
    const float2 x2 = make_float2(xi, xi), ci2 = make_float2(ci, ci), m2x = make_float2(-2.f * xi, -2.f * xi);
    float2 Gv[8];
    float lp = 0.f, ly = 0.f;  // in-thread exclusive prefixes (sum t, sum y t)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
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
      const float2 B = ffma2(y2[k], av, bv);                       // B_ip = y_p a - b
      const float2 V = ffma2(x2, fadd2(Uf[k], u2[k]), fadd2(Zf[k], z2[k]));  // x_i U + Zn
      Gv[k] = ffma2(m4, V, fadd2(cp2[k], ci2));                    // 2c'_p + 2c_i - 4 V
      u2[k] = ffma2(two, B, u2[k]);
      z2[k] = ffma2(m2x, B, z2[k]);
    }
    if (ncol > 0) {
      float* gp = Gout + (int64_t)jp * ld;
      if (nv == RC_KC) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<float4*>(gp + 4 * c) = make_float4(Gv[2 * c].x, Gv[2 * c].y, Gv[2 * c + 1].x, Gv[2 * c + 1].y);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (2 * k < nv) gp[2 * k] = Gv[k].x;
          if (2 * k + 1 < nv) gp[2 * k + 1] = Gv[k].y;
        }
      }
    }
    if ((jp & (RC_FLUSH - 1)) == RC_FLUSH - 1) {  // re-base the column state in fp64
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double* U = U64 + (2 * k) * RC_NT + t;
        double* Z = Z64 + (2 * k) * RC_NT + t;
        const double U_0 = U[0] + (double)u2[k].x, U_1 = U[RC_NT] + (double)u2[k].y;
        const double Z_0 = Z[0] + (double)z2[k].x, Z_1 = Z[RC_NT] + (double)z2[k].y;
        U[0] = U_0; U[RC_NT] = U_1; Z[0] = Z_0; Z[RC_NT] = Z_1;
        Uf[k] = make_float2((float)U_0, (float)U_1);
        Zf[k] = make_float2((float)Z_0, (float)Z_1);
        u2[k] = make_float2(0.f, 0.f);
        z2[k] = u2[k];
      }
    }
  };

  float2 tA[8], tB[8], offA, offB, xcA, xcB;
  for (int j = 0; j <= nrows; j += 2) {
    if (j < nrows) produce(j, tA, offA, xcA);
    if (j > 0) consume(j - 1, tB, offB, xcB);
    if (j + 1 <= nrows) {
      if (j + 1 < nrows) produce(j + 1, tB, offB, xcB);
      consume(j, tA, offA, xcA);
    }
  }
  cluster_arrive();
  cluster_wait();
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

// fused.cuh -- one-read Sinkhorn iteration (f-update + g-update fused, PAPER.md:108-114,
// reading R7), the "fast" path used once the duals are within 2^20 of their targets.
//
// Absorbed duals: with F_i = f_i log2e/eps and a_ip = (g_p - G_ip) log2e/eps,
//   e_ip = 2^(a_ip + F_i) = T_ip (the current plan),   S_i = sum_p e_ip  (its row sums),
//   f_i <- f_i + eps (ln p_i - ln S_i)                                   (row half-step)
//   w_i = p_i / S_i,  CS_p = sum_i e_ip w_i  (column sums of the half-step plan),
//   g_p <- g_p + eps (ln q_p - ln CS_p)                                  (column half-step)
// so every element of G is read ONCE per iteration and exponentiated ONCE.
//
// Layout: a thread-block cluster of CL CTAs spans a row (CTA rank r owns columns
// [r W, (r+1) W), W = 4 K FT); clusters own contiguous row ranges.  Per row:
//   TMA bulk copy (cp.async.bulk, mbarrier complete_tx) of the CTA's row slice into a
//   FSTAGES-deep shared-memory ring -> e values in registers -> CTA partial of S_i ->
//   DSMEM store of the partial into every peer CTA (mapa + st.shared::cluster) ->
//   split cluster barrier (arrive.release now, wait.acquire one row later, so the exchange
//   latency hides behind the next row) -> S_i (fixed rank order: identical in all CTAs)
//   -> column accumulation e_ip w_i (fp32 per 32 rows, then fp64).
// Column partials per cluster -> part[cluster][col] (fp64), merged in fixed order by
// k_sink_colfin_fast: deterministic, no float atomics.
#pragma once
#include "common.cuh"

namespace gw {

constexpr int FT = 512;       // threads per CTA
constexpr int FNW = FT / 32;  // warps per CTA
constexpr int FSTAGES = 4;    // TMA ring depth (rows)
constexpr int FFLUSH = 32;    // rows between fp32 -> fp64 column-accumulator flushes
constexpr int FPF = 8;        // L2 prefetch distance (rows) beyond the shared-memory ring

struct FusedArgs {
  const float* G;
  int64_t ld, nl, m;
  float c2f;                  // log2e / eps
  const float* gh;            // g log2e/eps, fp32 hi / lo (m)
  const float* gl;
  const float* fh;            // f log2e/eps, fp32 hi / lo (local rows)
  const float* fl;
  const float* pf;            // p (local rows, fp32)
  float* Srow;                // out: S_i = row sums of the plan entering the iteration
  double* part;               // [nclusters][m] column sums of the half-step plan
  int64_t rows_per_cluster;
  const int* mode;            // run only if *mode == 1
  const int* stop;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t mapa(const void* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
// asynchronous remote store that completes `8` transaction bytes on the receiver's mbarrier:
// no fence / cluster barrier needed for the receiver to observe it after its mbarrier phase
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
// fixed-order warp sum (tree to lane 0, then broadcast): bit-identical in every lane and warp
__device__ __forceinline__ float warp_sum_fixed(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  return __shfl_sync(0xffffffffu, v, 0);
}

// dynamic shared memory: the TMA ring [FSTAGES][W] fp32 + fp64 column accumulators [W]
template <int K>
constexpr size_t fused_dyn_smem() {
  return (size_t)FSTAGES * 4 * K * FT * sizeof(float) + (size_t)4 * K * FT * sizeof(double);
}

// Per row, no CTA-wide barrier: every warp (a) exponentiates its 4K columns from the ring
// stage, (b) releases the stage (empty mbarrier), (c) sends its partial of S_i to every
// cluster rank with st.async (complete_tx on the receiver's slot mbarrier), then (d) waits
// for the previous row's CL x FNW partials, reduces them in a fixed order (bit-identical in
// every warp of every CTA) and accumulates e_ip w_i for its columns.  Warp 0 lane 0 refills
// ring stages one row behind and prefetches FPF further rows into L2.
//
// Exponent (log2 units): a = fma(G_ip, -log2e/eps, gh_p) + F_i with the fp32 hi parts of the
// scaled duals only: the fma carries the one rounding of the large terms and "+ F" cancels
// exactly.  Dropping the lo parts (|lo| <= ulp/2 ~ 2^-20 relative) biases each row by 2^{Fl_i}
// and each column by 2^{gl_p}; the row / column normalisations of the iteration absorb both, so
// the fp64 duals' plan differs from the fixed point by <= 2^-19 relative per entry (marginal
// violation ~1e-5 * p_i).
template <int K, bool FULL>
__device__ __forceinline__ float fused_exp_row(const float4* __restrict__ st, const float (&ghv)[K][4], float c2f,
                                               float F, float (&ec)[K][4], int t, int64_t c0, int64_t m) {
  float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float4 gv = st[t + FT * k];
    const float g4[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      float e = ex2_ftz(fmaf(g4[jj], -c2f, ghv[k][jj]) + F);
      if (!FULL && c0 + 4 * (t + FT * k) + jj >= m) e = 0.f;
      ec[k][jj] = e;
      ps[jj] += e;
    }
  }
  return (ps[0] + ps[1]) + (ps[2] + ps[3]);
}

template <int K, int CL>
struct FusedCtx {
  static constexpr int W = 4 * K * FT;
  static constexpr int NSLOT = 4;           // exchange slots (power of 2)
  static constexpr int NX = CL * FNW;       // partials per row
};

template <int K, int CL>
__global__ void __launch_bounds__(FT, 1) k_sink_fused(FusedArgs a) {
  if (*a.mode != 1 || (a.stop && *a.stop)) return;  // uniform across the cluster
  constexpr int W = FusedCtx<K, CL>::W;
  constexpr int NSLOT = FusedCtx<K, CL>::NSLOT;
  constexpr int NX = FusedCtx<K, CL>::NX;
  extern __shared__ __align__(128) float ring[];  // [FSTAGES][W], then acc64 [W] (fp64)
  double* acc64 = reinterpret_cast<double*>(ring + (size_t)FSTAGES * W);
  __shared__ __align__(8) uint64_t full[FSTAGES], empty[FSTAGES];
  __shared__ __align__(8) uint64_t xbar[NSLOT];
  __shared__ __align__(16) float xs[NSLOT][NX];  // [slot][rank * FNW + warp]

  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t cr = cluster_rank();
  const int64_t cid = cluster_id();
  const int64_t m = a.m;
  const int64_t c0 = (int64_t)cr * W;
  const int64_t ncol = max((int64_t)0, min((int64_t)W, m - c0));  // valid columns of this CTA
  const uint32_t bytes = (uint32_t)(((ncol + 3) & ~int64_t(3)) * 4);
  const int64_t rb = cid * a.rows_per_cluster;
  const int64_t re = min(a.nl, rb + a.rows_per_cluster);
  const int nrows = (int)max((int64_t)0, re - rb);
  constexpr uint32_t xbytes = 4u * NX;
  const float* __restrict__ fh = a.fh + rb;
  const float* __restrict__ pf = a.pf + rb;
  float* __restrict__ Srow = a.Srow + rb;
  const float* __restrict__ Gbase = a.G + rb * a.ld + c0;
  const int64_t ld = a.ld;

  float ghv[K][4];
  const bool full_tile = (ncol == W);
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = c0 + 4 * (t + FT * k) + j;
      ghv[k][j] = col < m ? a.gh[col] : 0.f;
    }
  if (t == 0) {
    for (int s = 0; s < FSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], FNW);
    }
    for (int s = 0; s < NSLOT; ++s) mbar_init(&xbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NSLOT && s < nrows; ++s) mbar_expect_tx(&xbar[s], xbytes);
  }
  __syncthreads();
  cluster_arrive();
  cluster_wait();  // every CTA's barriers are initialised and armed before any DSMEM traffic
  if (t == 0 && bytes > 0) {
    for (int s = 0; s < FSTAGES && s < nrows; ++s) {
      mbar_expect_tx(&full[s], bytes);
      tma_load_1d(ring + (size_t)s * W, Gbase + (int64_t)s * ld, bytes, &full[s]);
    }
    for (int r = FSTAGES; r < FSTAGES + FPF && r < nrows; ++r) prefetch_l2_bulk(Gbase + (int64_t)r * ld, bytes);
  }
  // lane c < CL of every warp sends to rank c: remote address of this warp's slot-0 entry and
  // of the slot-0 barrier (slot s sits at a fixed byte offset from slot 0 in every CTA)
  const uint32_t peer = (uint32_t)min(lane, CL - 1);
  const uint32_t rx0 = mapa(&xs[0][cr * FNW + wid], peer), rb0 = mapa(&xbar[0], peer);
  constexpr uint32_t XSTRIDE = sizeof(xs[0]), BSTRIDE = sizeof(uint64_t);
  float acc32[K][4];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc32[k][j] = 0.f; acc64[4 * (t + FT * k) + j] = 0.0; }
  const float c2f = a.c2f;
  float eA[K][4], eB[K][4];
  float pA = 0.f, pB = 0.f;

  // one row: exponentiate + send (row j), then consume the previous row (j - 1)
  auto step = [&](int j, float (&ecur)[K][4], float& pcur, float (&eprv)[K][4], float pprv) {
    const int st = j & (FSTAGES - 1);
    if (j < nrows) {
      const float F = fh[j];
      pcur = pf[j];
      float psum = 0.f;
      if (bytes > 0) {
        mbar_wait(&full[st], (uint32_t)((j / FSTAGES) & 1));
        const float4* sp = reinterpret_cast<const float4*>(ring + (size_t)st * W);
        psum = full_tile ? fused_exp_row<K, true>(sp, ghv, c2f, F, ecur, t, c0, m)
                         : fused_exp_row<K, false>(sp, ghv, c2f, F, ecur, t, c0, m);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with stage st
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) ecur[k][jj] = 0.f;
      }
      psum = warp_sum_fixed(psum);
      const int xsl = j & (NSLOT - 1);
      if (lane < CL) st_async_f32(rx0 + XSTRIDE * xsl, psum, rb0 + BSTRIDE * xsl);
    }
    if (j > 0) {
      const int jp = j - 1;
      // warp 0 lane 0 refills the stage of row j-1 with row j-1+FSTAGES (+ L2 prefetch)
      if (t == 0 && bytes > 0 && jp + FSTAGES < nrows) {
        const int rs = jp & (FSTAGES - 1);
        mbar_wait(&empty[rs], (uint32_t)((jp / FSTAGES) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[rs], bytes);
        tma_load_1d(ring + (size_t)rs * W, Gbase + (int64_t)(jp + FSTAGES) * ld, bytes, &full[rs]);
        if (jp + FSTAGES + FPF < nrows) prefetch_l2_bulk(Gbase + (int64_t)(jp + FSTAGES + FPF) * ld, bytes);
      }
      // row j-1: wait for its CL x FNW partials and reduce them in a fixed order
      const int psl = jp & (NSLOT - 1);
      mbar_wait(&xbar[psl], (uint32_t)((jp / NSLOT) & 1));
      float S = 0.f;
      if (NX >= 32) {
#pragma unroll
        for (int i = 0; i < NX / 32; ++i) S += xs[psl][lane + 32 * i];
      } else {
        S = lane < NX ? xs[psl][lane] : 0.f;
      }
      S = warp_sum_fixed(S);
      if (t == 0) {
        Srow[jp] = S;
        if (jp + NSLOT < nrows) mbar_expect_tx(&xbar[psl], xbytes);  // the slot now serves row j+3
      }
      const float wv = pprv * rcp_ftz(S);
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc32[k][jj] = fmaf(eprv[k][jj], wv, acc32[k][jj]);
      if ((j & (FFLUSH - 1)) == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            acc64[4 * (t + FT * k) + jj] += (double)acc32[k][jj];
            acc32[k][jj] = 0.f;
          }
      }
    }
  };
  // rows in pairs: the two e buffers swap roles, so no register copies
  for (int j = 0; j <= nrows; j += 2) {
    step(j, eA, pA, eB, pB);
    if (j + 1 <= nrows) step(j + 1, eB, pB, eA, pA);
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const double v = acc64[4 * (t + FT * k) + jj] + (double)acc32[k][jj];
      const int64_t col = c0 + 4 * (t + FT * k) + jj;
      if (col < m) a.part[cid * m + col] = v;
    }
  // no CTA may exit while a peer can still address its shared memory
  cluster_arrive();
  cluster_wait();
}

// Finish of the fused iteration (one thread per row and per column, fixed order):
//   rows    f_i <- f_i + eps (ln p_i - ln S_i);  viol = max_i |S_i - p_i|
//   columns CS_p = sum over clusters, g_p <- g_p + eps (ln q_p - ln CS_p);
//           |log2(CS_p / q_p)| -> dev (path decision).
__global__ void k_sink_fin_fast(const float* __restrict__ Srow, int64_t nl, const double* __restrict__ lp,
                                double* __restrict__ f, float* __restrict__ fh, float* __restrict__ fl,
                                float* __restrict__ viol, const double* __restrict__ part, int ncl, int64_t m,
                                const double* __restrict__ lq, double eps, double* __restrict__ g,
                                float* __restrict__ gh, float* __restrict__ gl, int* __restrict__ mode,
                                const int* __restrict__ stop, float* __restrict__ dev) {
  if (*mode != 1 || (stop && *stop)) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float dv = 0.f, vv = 0.f;
  if (q < m) {
    double CS = 0.0;
    for (int c = 0; c < ncl; ++c) CS += part[(int64_t)c * m + q];
    const double d = lq[q] - log(CS);  // ln(q / CS)
    const double gn = (lq[q] == -INFINITY) ? -INFINITY : g[q] + eps * d;
    g[q] = gn;
    const double gs = gn * (GW_LOG2E / eps);
    const float h = (float)gs;
    gh[q] = h;
    gl[q] = isfinite(gs) ? (float)(gs - (double)h) : 0.f;
    double ad = fabs(d * GW_LOG2E);
    if (!(ad == ad)) ad = 3.0e38;
    dv = (float)fmin(ad, 3.0e38);
  }
  if (q < nl) {
    // the kernel used only the fp32 hi part of f log2e/eps: S' = S 2^{-Fl}; the row
    // normalisation is then f <- f + eps (ln p - ln S') which absorbs the dropped lo part
    const double S = (double)Srow[q];
    const double fn = (lp[q] == -INFINITY) ? -INFINITY : f[q] + eps * (lp[q] - log(S));
    f[q] = fn;
    const double fs = fn * (GW_LOG2E / eps);
    const float h = (float)fs;
    fh[q] = h;
    fl[q] = isfinite(fs) ? (float)(fs - (double)h) : 0.f;
    double v = fabs(S - exp(lp[q]));
    if (!(v == v)) v = 3.0e38;
    vv = (float)fmin(v, 3.0e38);
  }
  dv = warp_max(dv);
  vv = warp_max(vv);
  if ((threadIdx.x & 31) == 0) {
    if (dv > 0.f) atomic_max_nonneg(dev, dv);
    if (viol && vv > 0.f) atomic_max_nonneg(viol, vv);
  }
  if (q == 0) atomicAdd(mode + 1, 1);  // count of fused iterations executed
}

// Path decision for the next iteration: fast (fused, absorbed duals) iff the last column
// correction was within 2^20 -> then every plan entry e_ip <= 2^20 and every column sum of
// the half-step plan stays within 2^{+-20} of q (no fp32 overflow or catastrophic underflow).
__global__ void k_sink_mode(float* __restrict__ dev, int* __restrict__ mode, float thresh) {
  if (threadIdx.x == 0) {
    *mode = (*dev <= thresh) ? 1 : 0;
    *dev = 0.f;
  }
}

}  // namespace gw

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
// [r W, (r+1) W), W = 4 K NT); clusters own contiguous row ranges.  Per row:
//   TMA bulk copy (cp.async.bulk, mbarrier complete_tx) of the CTA's row slice into a
//   FSTAGES-deep shared-memory ring -> e values in registers (packed fp32x2 FFMA2/FADD2,
//   MUFU.EX2) -> warp partial of S_i -> st.async of the partial into every peer CTA
//   (complete_tx on the receiver's slot mbarrier) -> consumed one row later, so the exchange
//   latency hides behind the next row -> S_i (fixed order: identical in all warps and CTAs)
//   -> column accumulation e_ip w_i (fp32 per FFLUSH rows, then fp64 in shared memory).
// Column partials per cluster -> part[cluster][col] (fp64), merged in fixed order by
// k_sink_fin_fast: deterministic, no float atomics.
#pragma once
#include "common.cuh"

namespace gw {

// TMA ring depth (rows): 5 stages of 32 KB at 256 threads; 4 at 512 threads, whose larger exchange
// slots would not leave room for a fifth next to the 64 KB of fp64 column accumulators
template <int NT>
__host__ __device__ constexpr int fstages() { return NT >= 512 ? 4 : 5; }
#ifndef FFLUSH_DEF
#define FFLUSH_DEF 64
#endif
// rows between fp32 -> fp64 column-accumulator flushes: a fp32 sum of <= 64 positive terms (relative error
// <= 63 u = 3.8e-6 worst case, ~sqrt(64) u typical), folded in fp64; the flush (F2F conversions) cost 2 %
// of the iteration at 32 rows, 1 % at 64 (profiles/r02_fused_poly_offload.jsonl)
constexpr int FFLUSH = FFLUSH_DEF;

struct FusedArgs {
  const float* G;
  int64_t ld, nl, m;
  float c2f;                  // log2e / eps
  const float* gh;            // g log2e/eps, fp32 hi / lo (m)
  const float* gl;
  const float* fh;            // f log2e/eps, fp32 hi / lo (local rows)
  const float* fl;
  const float* pf;            // balanced (kappa == 1): p (local rows, fp32); unbalanced: log2 u
  float kappa;                // 1: balanced; < 1: unbalanced row factor (UGW, reading R34)
  float* Srow;                // out: S_i = row sums of the plan entering the iteration
  double* part;               // [nclusters][m] column sums of the half-step plan
  int64_t rows_per_cluster;
  int64_t wcol;               // columns per CTA (k_sink_fused2; <= the stage capacity 4 K NT)
  const int* mode;            // run only if *mode == 1
  const int* stop;
  // XM instantiation (the last sweep of an inner loop on the 8 N M gradient path, rowclu.cuh): the
  // exponent in the Gibbs-regeneration form (lo parts of the duals and of log2e/eps included), and
  // the column sums of x_i e_ip w_i beside those of e_ip w_i
  float c2f_lo;               // lo part of log2e/eps
  const float* xr;            // centred x (fp32, local rows)
  double* partx;              // [nclusters][m]
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
// MUFU reciprocal (<= 1 ulp; reading R19b): the fused iteration's per-row factor w = p / S
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a 16-byte aligned range (bytes % 16 == 0): no registers, no completion to wait for
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
// Butterfly warp sum: every lane ends with the same bits (each step adds the same two values,
// only in commuted order), so lanes 0..CL-1 can send identical partials to the CL ranks.
__device__ __forceinline__ float warp_sum_bfly(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

#ifndef FUSED_POLY_K
#define FUSED_POLY_K 5  // a chunk (of K = 8) whose exponentials run on the FMA pipe
#endif
#ifndef FUSED_POLY_K2
#define FUSED_POLY_K2 -1  // a second chunk: {2, 5} gained 0.4 % at full clocks but lost 2 % under sw_power_cap (sustained harness)
#endif
#ifndef FUSED_POLY_K6
#define FUSED_POLY_K6 5  // K = 6 instances (rows of 24576, C5): one chunk in six (0.584 -> 0.568 ms)
#endif
// packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 -- two lanes per instruction)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.ftz.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.ftz.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// 2^x on the FMA pipe for a pair (offloads MUFU): x clamped to [-126, 128] (the lower bound NaN-propagating,
// so a NaN argument becomes 128), n = rint(x) by the 1.5 2^23 shift, f = x - n in [-1/2, 1/2], 2^f by a
// degree-5 polynomial (max rel. error 2.4e-7 in fp32 Horner, the size of MUFU ex2.approx's), n added to the
// exponent field.  n = 128 (overflow, or a NaN argument) gives inf / NaN, which the iteration's validity
// check rejects exactly as it rejects MUFU's inf / NaN.
__device__ __forceinline__ float clamp_ex2(float x) {
  float y;
  asm("{\n\t.reg .f32 t;\n\tmax.NaN.f32 t, %1, 0fC2FC0000;\n\tmin.f32 %0, t, 0f43000000;\n\t}"
      : "=f"(y) : "f"(x));  // max(x, -126) keeping NaN, then min(., 128) turning NaN into 128
  return y;
}
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x = make_float2(clamp_ex2(x.x), clamp_ex2(x.y));
  const float2 r = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 f = fadd2(x, make_float2(-(r.x - 12582912.f), -(r.y - 12582912.f)));
  float2 p = make_float2(0.0013276450335979462f, 0.0013276450335979462f);
  p = ffma2(p, f, make_float2(0.009675541892647743f, 0.009675541892647743f));
  p = ffma2(p, f, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = ffma2(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = ffma2(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = ffma2(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  // the low bits of r are n + 2^22 + 2^23, which the shift by 23 drops
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(r.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(r.y) << 23)));
}

// W = 4 K NT columns per CTA.  Dynamic shared memory: the TMA ring [FSTAGES][W] fp32, then the
// fp64 column accumulators [K][4][NT] (conflict-free: lane-contiguous doubles).
template <int K, int NT, bool XM = false>
constexpr size_t fused_dyn_smem() {
  return (size_t)fstages<NT>() * 4 * K * NT * sizeof(float) + (size_t)(XM ? 2 : 1) * 4 * K * NT * sizeof(double);
}

// Exponentiate one row slice: e = 2^(fma(G, -log2e/eps, gh) + F) for the thread's 4K columns
// (K float4 from the ring stage), packed fp32x2; returns the thread's partial row sum (pairwise
// tree, so the dependent-add chain is log2(K) deep instead of K).
template <int K, int NT, bool FULL>
__device__ __forceinline__ float fused_exp_row(const float4* __restrict__ sp, const float2 (&ghv)[K][2], float2 nc2,
                                               float2 F2, float2 (&ec)[K][2], int t, int64_t c0, int64_t m) {
  float2 ps[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float4 gv = sp[t + NT * k];
    const float2 a0 = fadd2(ffma2(make_float2(gv.x, gv.y), nc2, ghv[k][0]), F2);
    const float2 a1 = fadd2(ffma2(make_float2(gv.z, gv.w), nc2, ghv[k][1]), F2);
    float2 e0 = make_float2(ex2_ftz(a0.x), ex2_ftz(a0.y));
    float2 e1 = make_float2(ex2_ftz(a1.x), ex2_ftz(a1.y));
    if (!FULL) {
      const int64_t col = c0 + 4 * (t + NT * k);
      if (col >= m) e0.x = 0.f;
      if (col + 1 >= m) e0.y = 0.f;
      if (col + 2 >= m) e1.x = 0.f;
      if (col + 3 >= m) e1.y = 0.f;
    }
    ec[k][0] = e0;
    ec[k][1] = e1;
    ps[k] = fadd2(e0, e1);
  }
#pragma unroll
  for (int w = 1; w < K; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < K; k += 2 * w) ps[k] = fadd2(ps[k], ps[k + w]);
  return ps[0].x + ps[0].y;
}

// XM: the same with the Gibbs-regeneration exponent a = [fma(G, -c_hi, g_hi) + F_hi] +
// [fma(G, -c_lo, g_lo + F_lo)] (grad2.cuh), so that e is the plan the gradient regenerates
template <int K, int NT, bool FULL>
__device__ __forceinline__ float fused_exp_row_xm(const float4* __restrict__ sp, const float2 (&ghv)[K][2],
                                                  const float2 (&glv)[K][2], float2 nc2, float2 ncl2, float2 F2,
                                                  float2 Fl2, float2 (&ec)[K][2], int t, int64_t c0, int64_t m) {
  float2 ps[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float4 gv = sp[t + NT * k];
    const float2 g01 = make_float2(gv.x, gv.y), g23 = make_float2(gv.z, gv.w);
    const float2 a0 = fadd2(fadd2(ffma2(g01, nc2, ghv[k][0]), F2), ffma2(g01, ncl2, fadd2(glv[k][0], Fl2)));
    const float2 a1 = fadd2(fadd2(ffma2(g23, nc2, ghv[k][1]), F2), ffma2(g23, ncl2, fadd2(glv[k][1], Fl2)));
    float2 e0 = make_float2(ex2_ftz(a0.x), ex2_ftz(a0.y));
    float2 e1 = make_float2(ex2_ftz(a1.x), ex2_ftz(a1.y));
    if (!FULL) {
      const int64_t col = c0 + 4 * (t + NT * k);
      if (col >= m) e0.x = 0.f;
      if (col + 1 >= m) e0.y = 0.f;
      if (col + 2 >= m) e1.x = 0.f;
      if (col + 3 >= m) e1.y = 0.f;
    }
    ec[k][0] = e0;
    ec[k][1] = e1;
    ps[k] = fadd2(e0, e1);
  }
#pragma unroll
  for (int w = 1; w < K; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < K; k += 2 * w) ps[k] = fadd2(ps[k], ps[k + w]);
  return ps[0].x + ps[0].y;
}

__device__ __forceinline__ void st_async_v2f32(uint32_t raddr, float v0, float v1, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "f"(v0), "f"(v1), "r"(rbar)
               : "memory");
}

// One CTA = NT threads (NT/32 warps), each owning 4K columns (K float4 per row).  Without any
// CTA-wide barrier every warp (a) exponentiates its columns of a ring stage, (b) releases the stage
// -- the LAST warp to release it (shared counter) refills it by TMA with the row FSTAGES further on,
// so FSTAGES-1 rows stay in flight whatever the warps' relative progress -- (c) sends its partial row
// sums to every cluster rank with st.async, then (d) waits for the previous step's CL x NW partials,
// reduces them in a fixed order (bit-identical in every warp of every CTA) and accumulates e w.
// Rows are processed in PAIRS: one step exponentiates two rows and exchanges both partial row sums
// in one 8-byte st.async per peer, so the per-row exchange, barrier and loop overhead is paid once
// per two rows.
//
// Exponent (log2 units): a = fma(G_ip, -log2e/eps, gh_p) + F_i with the fp32 hi parts of the
// scaled duals only (reading R30): the fma carries the one rounding of the large terms and
// "+ F" cancels exactly; the dropped lo parts are per-row / per-column scalings that the
// iteration's normalisations absorb.
// UGW: the unbalanced row factor (a separate instantiation: the balanced kernel carries no trace of it)
// XM: Gibbs-regeneration exponent + column sums of x_i e_ip w_i (see FusedArgs; balanced only)
template <int K, int CL, int NT, bool UGW, bool XM = false>
__global__ void __launch_bounds__(NT, 1) k_sink_fused2(FusedArgs a) {
  static_assert(!(UGW && XM), "XM is balanced only");
  if (*a.mode != 1 || (a.stop && *a.stop)) return;  // uniform across the cluster
  constexpr int NW = NT / 32;
  constexpr int W = 4 * K * NT;
  constexpr int FSTAGES = fstages<NT>();
  constexpr int NSLOT = 4;       // exchange slots (pairs; power of 2)
  constexpr int NX = CL * NW;    // partial pairs per row pair
  extern __shared__ __align__(128) float ring[];  // [FSTAGES][W], then acc64 [K][4][NT] (fp64)
  double* acc64 = reinterpret_cast<double*>(ring + (size_t)FSTAGES * W);
  double* acc64x = acc64 + (size_t)4 * K * NT;  // XM only
  __shared__ __align__(8) uint64_t full[FSTAGES];
  __shared__ unsigned int scnt[FSTAGES];
  __shared__ __align__(8) uint64_t xbar[NSLOT];
  __shared__ __align__(16) float2 xs[NSLOT][NX];  // [slot][rank * NW + warp] = {S_j0 part, S_j1 part}

  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t cr = blockIdx.x % CL;
  const int64_t cid = blockIdx.x / CL;
  const int64_t m = a.m;
  const int64_t c0 = (int64_t)cr * a.wcol;
  const int64_t ncol = max((int64_t)0, min(a.wcol, m - c0));  // this CTA's columns (<= W)
  const uint32_t bytes = (uint32_t)(((ncol + 3) & ~int64_t(3)) * 4);
  const int64_t rb = cid * a.rows_per_cluster;
  const int64_t re = min(a.nl, rb + a.rows_per_cluster);
  const int nrows = (int)max((int64_t)0, re - rb);
  const int npairs = (nrows + 1) >> 1;
  constexpr uint32_t xbytes = 8u * NX;
  const float* __restrict__ Gbase = a.G + rb * a.ld + c0;
  const int64_t ld = a.ld;

  // A CTA slice narrower than the stage (wcol < W): stage slots beyond the loaded bytes are never
  // written by TMA; zero them once so that with g_hi = -inf on every column the CTA does not own,
  // e = 2^(0 c - inf + F) = 0 there.
  if (ncol < W) {
    for (int i = t; i < FSTAGES * W; i += NT) ring[i] = 0.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (t == 0) {
    for (int s = 0; s < FSTAGES; ++s) {
      mbar_init(&full[s], 1);
      scnt[s] = 0u;
    }
    for (int s = 0; s < NSLOT; ++s) mbar_init(&xbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NSLOT && s < npairs; ++s) mbar_expect_tx(&xbar[s], xbytes);
  }
  __syncthreads();
  cluster_arrive();
  cluster_wait();

  if (t == 0 && bytes > 0) {
    for (int r = 0; r < FSTAGES && r < nrows; ++r) {
      mbar_expect_tx(&full[r], bytes);
      tma_load_1d(ring + (size_t)r * W, Gbase + (int64_t)r * ld, bytes, &full[r]);
    }
  }
  const float* __restrict__ fh = a.fh + rb;
  const float* __restrict__ pf = a.pf + rb;
  float* __restrict__ Srow = a.Srow + rb;
  const uint32_t peer = (uint32_t)min(lane, CL - 1);
  const uint32_t rx0 = mapa(&xs[0][cr * NW + wid], peer), rb0 = mapa(&xbar[0], peer);
  constexpr uint32_t XSTRIDE = sizeof(xs[0]), BSTRIDE = sizeof(uint64_t);
  // per-element masks are only needed where the last loaded float4 straddles m (m % 4 != 0);
  // elsewhere every slot is a real column of this CTA or a zeroed slot with g_hi = -inf
  const bool full_tile = !((c0 + ncol >= m) && (m & 3));

  float2 ghv[K][2], acc[K][2];
  float2 glv[K][2], accx[K][2];  // XM only
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t lc = 4 * (t + NT * k) + 2 * h;  // column inside the CTA slice
      const int64_t col = c0 + lc;
      ghv[k][h].x = (lc < ncol && col < m) ? a.gh[col] : -INFINITY;
      ghv[k][h].y = (lc + 1 < ncol && col + 1 < m) ? a.gh[col + 1] : -INFINITY;
      acc[k][h] = make_float2(0.f, 0.f);
      acc64[(k * 4 + 2 * h) * NT + t] = 0.0;
      acc64[(k * 4 + 2 * h + 1) * NT + t] = 0.0;
      if (XM) {
        glv[k][h].x = (lc < ncol && col < m) ? a.gl[col] : 0.f;
        glv[k][h].y = (lc + 1 < ncol && col + 1 < m) ? a.gl[col + 1] : 0.f;
        accx[k][h] = make_float2(0.f, 0.f);
        acc64x[(k * 4 + 2 * h) * NT + t] = 0.0;
        acc64x[(k * 4 + 2 * h + 1) * NT + t] = 0.0;
      }
    }
  const float2 nc2 = make_float2(-a.c2f, -a.c2f);
  const float2 ncl2 = make_float2(-a.c2f_lo, -a.c2f_lo);  // XM only
  constexpr bool ugw = UGW;
  const float km1 = a.kappa - 1.f;
  float2 eA0[K][2], eA1[K][2], eB0[K][2], eB1[K][2];
  float2 pA = make_float2(0.f, 0.f), pB = pA;  // marginals of the pair's two rows
  float2 xA = pA, xB = pA;                       // XM: their x
  float2 Fnx = make_float2(nrows > 0 ? fh[0] : 0.f, nrows > 1 ? fh[1] : 0.f);
  float2 pnx = make_float2(nrows > 0 ? pf[0] : 0.f, nrows > 1 ? pf[1] : 0.f);
  const float* __restrict__ flr = a.fl + rb;
  const float* __restrict__ xr = XM ? a.xr + rb : nullptr;
  float2 Flnx = make_float2(0.f, 0.f), xnx = Flnx;
  if (XM) {
    Flnx = make_float2(nrows > 0 ? flr[0] : 0.f, nrows > 1 ? flr[1] : 0.f);
    xnx = make_float2(nrows > 0 ? xr[0] : 0.f, nrows > 1 ? xr[1] : 0.f);
  }

  // exponentiate row j into e (returns the thread's partial row sum) and release its stage
  auto do_row = [&](int j, float F, float Fl, float2 (&e)[K][2]) -> float {
    float psum = 0.f;
    if (bytes > 0) {
      const int st = j % FSTAGES;
      mbar_wait(&full[st], (uint32_t)((j / FSTAGES) & 1));
      const float4* sp = reinterpret_cast<const float4*>(ring + (size_t)st * W);
      if (XM)
        psum = full_tile ? fused_exp_row_xm<K, NT, true>(sp, ghv, glv, nc2, ncl2, make_float2(F, F),
                                                         make_float2(Fl, Fl), e, t, c0, m)
                         : fused_exp_row_xm<K, NT, false>(sp, ghv, glv, nc2, ncl2, make_float2(F, F),
                                                          make_float2(Fl, Fl), e, t, c0, m);
      else
        psum = full_tile ? fused_exp_row<K, NT, true>(sp, ghv, nc2, make_float2(F, F), e, t, c0, m)
                         : fused_exp_row<K, NT, false>(sp, ghv, nc2, make_float2(F, F), e, t, c0, m);
      __syncwarp();
      if (lane == 0) {  // the last warp to release a stage refills it
        const int nxt = j + FSTAGES;
        if (atomicAdd(&scnt[st], 1u) == NW - 1) {
          scnt[st] = 0u;
          if (nxt < nrows) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[st], bytes);
            tma_load_1d(ring + (size_t)st * W, Gbase + (int64_t)nxt * ld, bytes, &full[st]);
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) { e[k][0] = make_float2(0.f, 0.f); e[k][1] = e[k][0]; }
    }
    return psum;
  };

  // Step P: rows 2P, 2P+1 (exponentiate + send), then consume pair P-1.
  auto step = [&](int P, float2 (&c0e)[K][2], float2 (&c1e)[K][2], float2& pcur, float2& xcur, float2 (&v0)[K][2],
                  float2 (&v1)[K][2], float2 pprv, float2 xprv) {
    const int j0 = 2 * P, j1 = 2 * P + 1;
    if (j0 < nrows) {
      const float2 F = Fnx;
      pcur = pnx;
      float2 Fl = make_float2(0.f, 0.f);
      if (XM) {
        Fl = Flnx;
        xcur = xnx;
        if (j0 + 2 < nrows) Flnx.x = flr[j0 + 2], xnx.x = xr[j0 + 2];
        if (j1 + 2 < nrows) Flnx.y = flr[j1 + 2], xnx.y = xr[j1 + 2];
      }
      if (ugw) {  // the row factor's constant part log2 u + (kappa - 1) F (F: the hi part the row uses)
        pcur.x = fmaf(km1, F.x, pcur.x);
        pcur.y = fmaf(km1, F.y, pcur.y);
      }
      if (j0 + 2 < nrows) Fnx.x = fh[j0 + 2], pnx.x = pf[j0 + 2];
      if (j1 + 2 < nrows) Fnx.y = fh[j1 + 2], pnx.y = pf[j1 + 2];
      float s0, s1 = 0.f;
      if (bytes > 0 && full_tile && j1 < nrows) {
        // common case: wait for both stages, then exponentiate the two rows in one block so the
        // scheduler can interleave their independent chains
        const int st0 = j0 % FSTAGES, st1 = j1 % FSTAGES;
        mbar_wait(&full[st0], (uint32_t)((j0 / FSTAGES) & 1));
        mbar_wait(&full[st1], (uint32_t)((j1 / FSTAGES) & 1));
        const float4* sp0 = reinterpret_cast<const float4*>(ring + (size_t)st0 * W);
        const float4* sp1 = reinterpret_cast<const float4*>(ring + (size_t)st1 * W);
        float2 q0 = make_float2(0.f, 0.f), q1 = q0;
        const float2 F0 = make_float2(F.x, F.x), F1 = make_float2(F.y, F.y);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float4 g0 = sp0[t + NT * k], g1 = sp1[t + NT * k];
          float2 a00 = fadd2(ffma2(make_float2(g0.x, g0.y), nc2, ghv[k][0]), F0);
          float2 a01 = fadd2(ffma2(make_float2(g0.z, g0.w), nc2, ghv[k][1]), F0);
          float2 a10 = fadd2(ffma2(make_float2(g1.x, g1.y), nc2, ghv[k][0]), F1);
          float2 a11 = fadd2(ffma2(make_float2(g1.z, g1.w), nc2, ghv[k][1]), F1);
          if (XM) {  // the lo bracket of the Gibbs-regeneration exponent
            const float2 L0 = make_float2(Fl.x, Fl.x), L1 = make_float2(Fl.y, Fl.y);
            a00 = fadd2(a00, ffma2(make_float2(g0.x, g0.y), ncl2, fadd2(glv[k][0], L0)));
            a01 = fadd2(a01, ffma2(make_float2(g0.z, g0.w), ncl2, fadd2(glv[k][1], L0)));
            a10 = fadd2(a10, ffma2(make_float2(g1.x, g1.y), ncl2, fadd2(glv[k][0], L1)));
            a11 = fadd2(a11, ffma2(make_float2(g1.z, g1.w), ncl2, fadd2(glv[k][1], L1)));
          }
          if ((K >= 8 && (k == FUSED_POLY_K || k == FUSED_POLY_K2)) || (FUSED_POLY_K6 >= 0 && K == 6 && k == FUSED_POLY_K6)) {
            // chunk 5 of 8 (K = 8), 5 of 6 (K = 6) on the FMA pipe (ex2_poly2): MUFU.EX2 is the kernel's
            // busiest unit (XU 47 %); with the 64-row flush 2.86 -> 2.78 ms per iteration at C4 at full
            // clocks, 3.11 -> 3.07 ms under sw_power_cap (profiles/r02_fused_poly_offload.jsonl)
            c0e[k][0] = ex2_poly2(a00); c0e[k][1] = ex2_poly2(a01); c1e[k][0] = ex2_poly2(a10); c1e[k][1] = ex2_poly2(a11);
          } else {
            c0e[k][0] = make_float2(ex2_ftz(a00.x), ex2_ftz(a00.y));
            c0e[k][1] = make_float2(ex2_ftz(a01.x), ex2_ftz(a01.y));
            c1e[k][0] = make_float2(ex2_ftz(a10.x), ex2_ftz(a10.y));
            c1e[k][1] = make_float2(ex2_ftz(a11.x), ex2_ftz(a11.y));
          }
          q0 = fadd2(q0, fadd2(c0e[k][0], c0e[k][1]));
          q1 = fadd2(q1, fadd2(c1e[k][0], c1e[k][1]));
        }
        s0 = q0.x + q0.y;
        s1 = q1.x + q1.y;
        __syncwarp();
        if (lane == 0) {  // release both stages; the last warp to release a stage refills it
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int st = h ? st1 : st0, nxt = (h ? j1 : j0) + FSTAGES;
            if (atomicAdd(&scnt[st], 1u) == NW - 1) {
              scnt[st] = 0u;
              if (nxt < nrows) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&full[st], bytes);
                tma_load_1d(ring + (size_t)st * W, Gbase + (int64_t)nxt * ld, bytes, &full[st]);
              }
            }
          }
        }
      } else if (j1 < nrows) {
        s0 = do_row(j0, F.x, Fl.x, c0e);
        s1 = do_row(j1, F.y, Fl.y, c1e);
      } else {
        s0 = do_row(j0, F.x, Fl.x, c0e);
#pragma unroll
        for (int k = 0; k < K; ++k) { c1e[k][0] = make_float2(0.f, 0.f); c1e[k][1] = c1e[k][0]; }
        pcur.y = 0.f;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, d);
        s1 += __shfl_xor_sync(0xffffffffu, s1, d);
      }
      const int xsl = P & (NSLOT - 1);
      if (lane < CL) st_async_v2f32(rx0 + XSTRIDE * xsl, s0, s1, rb0 + BSTRIDE * xsl);
    }
    if (P > 0) {
      const int Pp = P - 1;
      const int psl = Pp & (NSLOT - 1);
      mbar_wait(&xbar[psl], (uint32_t)((Pp / NSLOT) & 1));
      float S0 = 0.f, S1 = 0.f;
      if (NX >= 32) {
#pragma unroll
        for (int i = 0; i < (NX + 31) / 32; ++i) {
          if (lane + 32 * i < NX) {
            const float2 v = xs[psl][lane + 32 * i];
            S0 += v.x;
            S1 += v.y;
          }
        }
      } else if (lane < NX) {
        const float2 v = xs[psl][lane];
        S0 = v.x;
        S1 = v.y;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        S0 += __shfl_xor_sync(0xffffffffu, S0, d);
        S1 += __shfl_xor_sync(0xffffffffu, S1, d);
      }
      const int jp0 = 2 * Pp, jp1 = 2 * Pp + 1;
      if (t == 0) {
        Srow[jp0] = S0;
        if (jp1 < nrows) Srow[jp1] = S1;
        if (Pp + NSLOT < npairs) mbar_expect_tx(&xbar[psl], xbytes);
      }
      // half-step row factor: balanced w = p (1/S) with the MUFU reciprocal (<= 1 ulp, reading R19b: the
      // IEEE __frcp_rn sequence on this latency-critical step cost 8% of the kernel); unbalanced (R34,
      // absorbed duals)
      // w = 2^(log2 u + (kappa - 1) F - kappa log2 S), i.e. f'_new = eps~ ln u - kappa eps~ (ln S - F ln 2)
      float w0, w1 = 0.f;
      if (!ugw) {
        w0 = pprv.x * rcp_approx(S0);
        if (jp1 < nrows) w1 = pprv.y * rcp_approx(S1);
      } else {
        w0 = ex2_ftz(fmaf(-a.kappa, lg2_ftz(S0), pprv.x));
        if (jp1 < nrows) w1 = ex2_ftz(fmaf(-a.kappa, lg2_ftz(S1), pprv.y));
      }
      const float2 w02 = make_float2(w0, w0), w12 = make_float2(w1, w1);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        acc[k][0] = ffma2(v1[k][0], w12, ffma2(v0[k][0], w02, acc[k][0]));
        acc[k][1] = ffma2(v1[k][1], w12, ffma2(v0[k][1], w02, acc[k][1]));
      }
      if (XM) {
        const float wx0 = w0 * xprv.x, wx1 = w1 * xprv.y;
        const float2 wx02 = make_float2(wx0, wx0), wx12 = make_float2(wx1, wx1);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          accx[k][0] = ffma2(v1[k][0], wx12, ffma2(v0[k][0], wx02, accx[k][0]));
          accx[k][1] = ffma2(v1[k][1], wx12, ffma2(v0[k][1], wx02, accx[k][1]));
        }
      }
      if ((Pp & (FFLUSH / 2 - 1)) == FFLUSH / 2 - 1) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            acc64[(k * 4 + 2 * h) * NT + t] += (double)acc[k][h].x;
            acc64[(k * 4 + 2 * h + 1) * NT + t] += (double)acc[k][h].y;
            acc[k][h] = make_float2(0.f, 0.f);
            if (XM) {
              acc64x[(k * 4 + 2 * h) * NT + t] += (double)accx[k][h].x;
              acc64x[(k * 4 + 2 * h + 1) * NT + t] += (double)accx[k][h].y;
              accx[k][h] = make_float2(0.f, 0.f);
            }
          }
      }
    }
  };
  for (int P = 0; P <= npairs; P += 2) {
    step(P, eA0, eA1, pA, xA, eB0, eB1, pB, xB);
    if (P + 1 <= npairs) step(P + 1, eB0, eB1, pB, xB, eA0, eA1, pA, xA);
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t lc = 4 * (t + NT * k) + 2 * h;
      const int64_t col = c0 + lc;
      const double v0 = acc64[(k * 4 + 2 * h) * NT + t] + (double)acc[k][h].x;
      const double v1 = acc64[(k * 4 + 2 * h + 1) * NT + t] + (double)acc[k][h].y;
      if (lc < ncol && col < m) a.part[cid * m + col] = v0;
      if (lc + 1 < ncol && col + 1 < m) a.part[cid * m + col + 1] = v1;
      if (XM) {
        const double x0 = acc64x[(k * 4 + 2 * h) * NT + t] + (double)accx[k][h].x;
        const double x1 = acc64x[(k * 4 + 2 * h + 1) * NT + t] + (double)accx[k][h].y;
        if (lc < ncol && col < m) a.partx[cid * m + col] = x0;
        if (lc + 1 < ncol && col + 1 < m) a.partx[cid * m + col + 1] = x1;
      }
    }
  cluster_arrive();
  cluster_wait();
}

// Finish of the fused iteration (one thread per row and per column, fixed order):
//   rows    f_i <- f_i + eps (ln p_i - ln S_i);  viol = max_i |S_i - p_i|
//   columns CS_p = sum over clusters, g_p <- g_p + eps (ln q_p - ln CS_p);
//           |log2(CS_p / q_p)| -> dev (path decision).
// Validity of a (speculative) fused iteration, before anything is committed: every row sum S_i and
// every column sum CS_p must be finite and above 2^-100 (no overflow of an exponential, no row or
// column whose terms all underflowed).  Then the absorbed-dual update equals the log-domain one up
// to fp32 rounding of sums of positive terms.  flag |= 1 otherwise (order-independent OR).
// part: ncl payloads of `stride` doubles (the M column sums, then -- multi-rank -- the rank's row flag
// as an int in the slot at M: rowflags_gathered).  One rank: the row sums are checked here.
__global__ void k_sink_fast_check(const float* __restrict__ Srow, int64_t nl, const double* __restrict__ part,
                                  int ncl, int64_t stride, int64_t m, const double* __restrict__ lq,
                                  int* __restrict__ flag, const int* __restrict__ mode, const int* __restrict__ stop,
                                  bool rowflags_gathered) {
  if (*mode != 1 || (stop && *stop)) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (!rowflags_gathered && q < nl) {
    const float S = Srow[q];
    bad |= !(S > 7.9e-31f && S < 3.0e38f);
  }
  if (rowflags_gathered && q == 0)
    for (int c = 0; c < ncl; ++c) bad |= *reinterpret_cast<const int*>(part + (int64_t)c * stride + m) != 0;
  if (q < m && lq[q] != -INFINITY) {
    double CS = 0.0;
    for (int c = 0; c < ncl; ++c) CS += part[(int64_t)c * stride + q];
    bad |= !(CS > 7.9e-31 && CS < 1e300);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// OR of the ranks' gathered validity flags (multi-rank), in place into flag[0]
__global__ void k_or_flags(int* __restrict__ flag, const int* __restrict__ gath, int R) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int v = 0;
    for (int r = 0; r < R; ++r) v |= gath[r];
    *flag = v;
  }
}

__global__ void k_sink_fin_fast(const float* __restrict__ Srow, int64_t nl, const double* __restrict__ lp,
                                double* __restrict__ f, float* __restrict__ fh, float* __restrict__ fl,
                                float* __restrict__ viol, const double* __restrict__ part, int ncl, int64_t stride,
                                int64_t m,
                                const double* __restrict__ lq, double eps, double* __restrict__ g,
                                float* __restrict__ gh, float* __restrict__ gl, int* __restrict__ mode,
                                const int* __restrict__ stop, float* __restrict__ dev, const int* __restrict__ flag,
                                double kappa = 1.0, cudaGraphConditionalHandle cond = 0, int use_cond = 0) {
  // inside a captured iteration: arm the conditional node that runs the safe path iff this iteration
  // was not committed here (path already safe, or the speculation failed its check)
  if (use_cond && blockIdx.x == 0 && threadIdx.x == 0)
    cudaGraphSetConditional(cond, (!(stop && *stop) && (*mode != 1 || *flag)) ? 1u : 0u);
  if (*mode != 1 || (stop && *stop)) return;
  if (*flag) {
    // speculation failed: nothing is committed and this iteration runs the safe path instead
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) *mode = 0;
    return;
  }
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float dv = 0.f, vv = 0.f;
  if (q < m) {
    double CS = 0.0;
    for (int c = 0; c < ncl; ++c) CS += part[(int64_t)c * stride + q];
    double d = lq[q] - log(CS);  // ln(q / CS)
    double gn;
    if (kappa == 1.0) {
      gn = (lq[q] == -INFINITY) ? -INFINITY : g[q] + eps * d;
    } else {  // unbalanced (R34, absorbed duals): g'_new = eps~ ln v - kappa eps~ (ln CS - gh ln 2)
      gn = (lq[q] == -INFINITY) ? -INFINITY : eps * lq[q] - kappa * eps * (log(CS) - (double)gh[q] * GW_LN2);
      d = (gn - g[q]) / eps;
    }
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
    double fn;
    if (kappa == 1.0) fn = (lp[q] == -INFINITY) ? -INFINITY : f[q] + eps * (lp[q] - log(S));
    else fn = (lp[q] == -INFINITY) ? -INFINITY : eps * lp[q] - kappa * eps * (log(S) - (double)fh[q] * GW_LN2);
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
__global__ void k_sink_mode(float* __restrict__ dev, int* __restrict__ mode, float thresh,
                            int* __restrict__ flag_reset = nullptr) {
  if (threadIdx.x == 0) {
    *mode = (*dev <= thresh) ? 1 : 0;
    *dev = 0.f;
    if (flag_reset) *flag_reset = 0;  // the next speculative iteration's validity flag starts clear
  }
}

// Multi-rank fixed-count loop (sink_run): end of one iteration slot, decided on the device (every rank
// reaches the same decision: the flag and the column corrections follow gathered data).  The slot
// committed an update unless its fused attempt failed the validity check (flag != 0: nothing was
// committed and the next slot runs the safe path).  Next path: fused iff this slot committed and its
// column correction was within 2^thresh.  stop once `target` updates are committed.
//   md: [0] path of the next slot, [5] committed updates, [6] target
__global__ void k_sink_slot_end(int* __restrict__ md, float* __restrict__ dev, const int* __restrict__ flag,
                                int* __restrict__ stop, float thresh) {
  if (threadIdx.x == 0) {
    if (!*stop) {
      const bool ok = *flag == 0;
      if (ok) md[5] += 1;
      md[0] = (ok && *dev <= thresh) ? 1 : 0;
      if (md[5] >= md[6]) *stop = 1;
    }
    *dev = 0.f;
  }
}

}  // namespace gw

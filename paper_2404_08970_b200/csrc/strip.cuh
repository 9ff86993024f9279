// strip.cuh -- one-read Sinkhorn iteration on ALL SMs: column strips + a grid-wide row-sum exchange.
//
// Same iteration as fused.cuh (f-update then g-update in one read of G, readings R7
// and R30; absorbed duals):
//   e_ip = 2^(fma(G_ip, -log2e/eps, gh_p) + F_i),  S_i = sum_p e_ip,  w_i = p_i / S_i,
//   CS_p = sum_i e_ip w_i   (column sums of the half-step plan).
// fused.cuh holds a row's e values in the registers of a thread-block cluster spanning the row, which
// needs clusters of 8 CTAs at M = 65536 -- and only 15 of those fit on the B200's GPCs (120 of 148
// SMs).  Here every SM works: CTA c of a persistent grid of one CTA per SM owns the column strip
// [c M/NB, (c+1) M/NB) of EVERY row (M/NB ~ 443 columns = 1.8 KB per row), so its column sums are
// complete locally, and the row sums are exchanged across the grid.  Per block b of SRB rows:
//   * compute warps (8): TMA bulk copies of the CTA's strip of the rows land in a ring buffer; e is
//     computed in place (warp per row); per-row partial sums -> global {value, tag} words;
//   * the reducer warp of CTA b mod NB waits for the NB partials of every row of block b, sums them
//     in a fixed order (deterministic) and publishes S as {value, tag} words;
//   * the consumer warp polls the published S of the next blocks (a 4-block window), forms
//     w = p / S into a shared-memory slot and signals an mbarrier;
//   * LAG blocks after exponentiating block b the compute warps accumulate e w of block b - LAG into
//     their column sums (fp32 per block, fp64 across blocks) and release its buffer to the TMA.
// The LAG blocks of e kept in shared memory hide the exchange latency.  All CTAs must be co-resident
// (cooperative launch; one CTA per SM); spin-waits are bounded (trap after ~seconds).
#pragma once
#include "common.cuh"
#include "fused.cuh"  // mbarrier / TMA / packed fp32x2 helpers

namespace gw {

constexpr int SNTH = 256;            // compute threads per CTA (8 warps)
constexpr int SNTX = SNTH + 64;      // + the consumer warp and the reducer warp
constexpr int SRB = 16;              // rows per block
constexpr int SPB = 16;              // exchange slots (ring of blocks; power of 2, >= lag + 2)
constexpr int SWB = 8;               // w slots (blocks the consumer warp may run ahead)
constexpr int SNBMAX = 160;          // CTAs (SMs) the reducer's unrolled loads cover

struct StripArgs {
  const float* G;
  int64_t ld, nl, m;
  float c2f;             // log2e / eps
  const float* gh;       // g log2e/eps (hi), m
  const float* fh;       // f log2e/eps (hi), local rows
  const float* pf;       // p (fp32), local rows
  float* Srow;           // out: S_i
  double* part;          // out: [m] column sums of the half-step plan (this rank's rows)
  unsigned long long* xp;  // [SPB][nb][SRB] partial row sums as {value, tag} words
  unsigned long long* xs;  // [SPB][SRB] row sums of a block as {value, tag} words (its reducer)
  unsigned* epoch;       // launch counter (tags); CTA 0 increments it on exit
  int nb;                // CTAs in the grid (<= SNBMAX)
  int nbuf, lag;         // ring depth and exchange lag (blocks)
  const int* mode;
  const int* stop;
};

// {value, tag} words ("flag in data"): an aligned 64-bit store / load is single-copy atomic, so a
// reader that sees the expected tag sees the value written with it -- no fences, no counters.
// tag = (launch << 20) + block: unique between the block's current writer, the previous user of its
// slot (block - SPB, same launch) and the previous launch (exchange buffers are zeroed per solve).
__device__ __forceinline__ unsigned long long ll_pack(float v, unsigned tag) {
  return ((unsigned long long)tag << 32) | __float_as_uint(v);
}
__device__ __forceinline__ void ll_store(unsigned long long* p, unsigned long long w) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ll_load(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ unsigned ll_tag(unsigned long long w) { return (unsigned)(w >> 32); }
__device__ __forceinline__ float ll_val(unsigned long long w) { return __uint_as_float((unsigned)w); }
__device__ __forceinline__ void bar_compute() {  // named barrier over the 8 compute warps only
  asm volatile("bar.sync 1, %0;" ::"n"(SNTH) : "memory");
}

// KF: float4 per lane per row in the exponentiation phase (the CTA's strip has nf4 <= 32 KF float4).
template <int KF>
__global__ void __launch_bounds__(SNTX, 1) k_sink_strip(StripArgs a) {
  if (*a.mode != 1 || (a.stop && *a.stop)) return;  // uniform across the grid
  constexpr int NW = SNTH / 32;
  constexpr int RPW = SRB / NW;  // rows per warp per block
  extern __shared__ __align__(128) float sdyn[];  // [nbuf][SRB][nf4] float4
  float4* ring = reinterpret_cast<float4*>(sdyn);
  __shared__ __align__(8) uint64_t full[16];      // TMA landed (per ring buffer)
  __shared__ __align__(8) uint64_t wready[SWB];   // w of a block is in sw[slot] (consumer warp)
  __shared__ __align__(8) uint64_t wfree[SWB];    // sw[slot] consumed (compute warps)
  __shared__ float sw[SWB][SRB];
  __shared__ double sacc[128 * 4];                // final fixed-order merge of the two row halves
  __shared__ unsigned sepoch;

  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int cta = blockIdx.x, NB = a.nb;
  const int64_t m = a.m, nl = a.nl;
  const int64_t M4 = (m + 3) >> 2;
  const int64_t f40 = (int64_t)cta * M4 / NB, f41 = (int64_t)(cta + 1) * M4 / NB;
  const int nf4 = (int)(f41 - f40);
  const int nblk = (int)((nl + SRB - 1) / SRB);
  const int nbuf = a.nbuf, lag = a.lag;
  const float* __restrict__ Gs = a.G + 4 * f40;
  const int64_t ld = a.ld;

  if (t == 0) {
    for (int s = 0; s < nbuf; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < SWB; ++s) {
      mbar_init(&wready[s], 1);
      mbar_init(&wfree[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sepoch = *reinterpret_cast<volatile unsigned*>(a.epoch);
  }
  __syncthreads();
  const unsigned tag0 = sepoch << 20;  // tag of block b: tag0 + b

  if (wid == NW + 1) {
    // ================= reducer warp: the blocks b = cta (mod NB) =================
    // lanes r and r + 16 own row r and sum the CTAs c = h, h + 2, ... (h = lane >> 4) in order
    constexpr int NV = SNBMAX / 4;  // words per lane per chunk (two chunks: c < 2 NV and c >= 2 NV)
    const int r = lane & 15, h = lane >> 4;
    for (int b = cta; b < nblk; b += NB) {
      const unsigned want = tag0 + (unsigned)b;
      const unsigned long long* src = a.xp + (size_t)(b & (SPB - 1)) * NB * SRB + r;
      float S = 0.f;
#pragma unroll 1
      for (int ch = 0; ch < 2; ++ch) {
        const int cb = h + 2 * NV * ch;
        unsigned long long v[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = cb + 2 * k;
          v[k] = c < NB ? ll_load(src + (size_t)c * SRB) : ll_pack(0.f, want);
        }
        long long spins = 0;
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            if (ll_tag(v[k]) != want) {
              ok = false;
              v[k] = ll_load(src + (size_t)(cb + 2 * k) * SRB);
            }
          }
          if (__all_sync(0xffffffffu, ok)) break;
          __nanosleep(32);
          if (++spins > (1ll << 26)) __trap();  // a lost CTA: fail loudly instead of hanging
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) S += ll_val(v[k]);
      }
      S += __shfl_xor_sync(0xffffffffu, S, 16);
      if (h == 0) {
        ll_store(a.xs + (size_t)(b & (SPB - 1)) * SRB + r, ll_pack(S, want));
        if ((int64_t)b * SRB + r < nl) a.Srow[(int64_t)b * SRB + r] = S;
      }
    }
    return;
  }
  if (wid == NW) {
    // ================= consumer warp: w = p / S of every block, in order =================
    // lanes r and r + 16 poll row r of the two blocks b0 + h and b0 + 2 + h of a 4-block window
    const int r = lane & 15, h = lane >> 4;
    int b0 = 0;
    long long spins = 0;
    while (b0 < nblk) {
      unsigned long long w2[2];
      float p2[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = b0 + 2 * j + h;
        w2[j] = b < nblk ? ll_load(a.xs + (size_t)(b & (SPB - 1)) * SRB + r) : 0ull;
        const int64_t i = (int64_t)b * SRB + r;
        p2[j] = (b < nblk && i < nl) ? a.pf[i] : 0.f;
      }
      int done = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // blocks b0 + q, in order, while ready
        const int b = b0 + q;
        const int j = q >> 1, hq = q & 1;
        if (b >= nblk) break;
        const bool mine = h == hq;
        const bool ok = ll_tag(w2[j]) == tag0 + (unsigned)b;
        const unsigned ball = __ballot_sync(0xffffffffu, mine && ok);
        if (__popc(ball) != 16) break;
        const int ws_ = b % SWB;
        if (b >= SWB) mbar_wait(&wfree[ws_], (uint32_t)(((b / SWB) - 1) & 1));
        if (mine) {
          const int64_t i = (int64_t)b * SRB + r;
          sw[ws_][r] = i < nl ? __fdiv_rn(p2[j], ll_val(w2[j])) : 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&wready[ws_]);
        ++done;
      }
      b0 += done;
      if (done == 0) {
        __nanosleep(20);
        if (++spins > (1ll << 27)) __trap();
      }
    }
    return;
  }

  // ================= compute warps =================
  // TMA producer: lane r of warp 0 copies row r of a block (SRB bulk copies of nf4 * 16 bytes)
  auto issue = [&](int blk) {
    const int64_t r0 = (int64_t)blk * SRB;
    const int rows = (int)min((int64_t)SRB, nl - r0);
    const uint32_t rb = (uint32_t)nf4 * 16u;
    float4* dst = ring + (size_t)(blk % nbuf) * SRB * nf4;
    if (lane == 0) mbar_expect_tx(&full[blk % nbuf], rb * rows);
    __syncwarp();
    if (lane < rows) tma_load_1d(dst + (size_t)lane * nf4, Gs + (r0 + lane) * ld, rb, &full[blk % nbuf]);
  };
  if (wid == 0 && nf4 > 0)
    for (int blk = 0; blk < nbuf && blk < nblk; ++blk) issue(blk);

  // this lane's columns (exponentiation phase): float4 k = lane + 32 j of the strip
  float4 ghv[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) {
    const int k = lane + 32 * j;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t col = 4 * (f40 + k) + e;
      v[e] = (k < nf4 && col < m) ? a.gh[col] : -INFINITY;
    }
    ghv[j] = make_float4(v[0], v[1], v[2], v[3]);
  }
  const float2 nc2 = make_float2(-a.c2f, -a.c2f);
  // consumption phase: thread t owns float4 column kc of the strip for rows [hh RB/2, (hh+1) RB/2)
  const int kc = t & 127, hh = t >> 7;
  float4 acc32 = make_float4(0.f, 0.f, 0.f, 0.f);
  double acc64[4] = {0.0, 0.0, 0.0, 0.0};
  float Fn[RPW];
#pragma unroll
  for (int u = 0; u < RPW; ++u) {
    const int64_t i = wid + NW * u;
    Fn[u] = i < nl ? a.fh[i] : 0.f;
  }

  for (int b = 0; b < nblk + lag; ++b) {
    // ---- exponentiate block b (warp per row), partial row sums -> xpart ----
    if (b < nblk) {
      const int slot = b & (SPB - 1);
      const int64_t r0 = (int64_t)b * SRB;
      float F[RPW];
#pragma unroll
      for (int u = 0; u < RPW; ++u) {
        F[u] = Fn[u];
        const int64_t i = r0 + SRB + wid + NW * u;
        Fn[u] = i < nl ? a.fh[i] : 0.f;
      }
      if (nf4 > 0) mbar_wait(&full[b % nbuf], (uint32_t)((b / nbuf) & 1));
      float4* buf = ring + (size_t)(b % nbuf) * SRB * nf4;
      float ps[RPW];
#pragma unroll
      for (int u = 0; u < RPW; ++u) {
        const int r = wid + NW * u;
        float4* row = buf + (size_t)r * nf4;
        const float2 F2 = make_float2(F[u], F[u]);
        float2 s2 = make_float2(0.f, 0.f);
        if (r0 + r < nl) {
#pragma unroll
          for (int j = 0; j < KF; ++j) {
            const int k = lane + 32 * j;
            if (k < nf4) {
              const float4 gv = row[k];
              const float2 a0 = fadd2(ffma2(make_float2(gv.x, gv.y), nc2, make_float2(ghv[j].x, ghv[j].y)), F2);
              const float2 a1 = fadd2(ffma2(make_float2(gv.z, gv.w), nc2, make_float2(ghv[j].z, ghv[j].w)), F2);
              const float4 ev = make_float4(ex2_ftz(a0.x), ex2_ftz(a0.y), ex2_ftz(a1.x), ex2_ftz(a1.y));
              row[k] = ev;
              s2 = fadd2(s2, fadd2(make_float2(ev.x, ev.y), make_float2(ev.z, ev.w)));
            }
          }
        }
        ps[u] = s2.x + s2.y;
      }
#pragma unroll
      for (int u = 0; u < RPW; ++u) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) ps[u] += __shfl_xor_sync(0xffffffffu, ps[u], d);
        if (lane == 0)
          ll_store(a.xp + ((size_t)slot * NB + cta) * SRB + wid + NW * u, ll_pack(ps[u], tag0 + (unsigned)b));
      }
    }
    // ---- accumulate block bc = b - lag: e w into the column sums ----
    const int bc = b - lag;
    if (bc >= 0) {
      const int ws_ = bc % SWB;
      mbar_wait(&wready[ws_], (uint32_t)((bc / SWB) & 1));
      const float4* buf = ring + (size_t)(bc % nbuf) * SRB * nf4;
      const int rows_c = (int)min((int64_t)SRB, nl - (int64_t)bc * SRB);  // rows past nl hold stale smem
      if (kc < nf4) {
#pragma unroll
        for (int u = 0; u < SRB / 2; ++u) {
          const int r = hh * (SRB / 2) + u;
          if (r >= rows_c) break;
          const float w = sw[ws_][r];
          const float4 ev = buf[(size_t)r * nf4 + kc];
          acc32.x = fmaf(ev.x, w, acc32.x);
          acc32.y = fmaf(ev.y, w, acc32.y);
          acc32.z = fmaf(ev.z, w, acc32.z);
          acc32.w = fmaf(ev.w, w, acc32.w);
        }
        acc64[0] += (double)acc32.x;
        acc64[1] += (double)acc32.y;
        acc64[2] += (double)acc32.z;
        acc64[3] += (double)acc32.w;
        acc32 = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // the e values were written to this buffer by the generic proxy; the TMA refill is an
      // async-proxy write: order them (every writer fences, then the barrier)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_compute();  // buffer of block bc and sw[ws_] consumed
      if (t == 0) mbar_arrive(&wfree[ws_]);
      const int nxt = bc + nbuf;
      if (wid == 0 && nxt < nblk && nf4 > 0) issue(nxt);
    }
  }
  // ---- column sums: fixed-order merge of the two row halves ----
  if (hh == 1 && kc < nf4)
#pragma unroll
    for (int e = 0; e < 4; ++e) sacc[kc * 4 + e] = acc64[e];
  bar_compute();
  if (hh == 0 && kc < nf4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t col = 4 * (f40 + kc) + e;
      if (col < m) a.part[col] = acc64[e] + sacc[kc * 4 + e];
    }
  }
  // every CTA read the epoch at its start (CTA 0 consumed every block, so every CTA produced them)
  if (cta == 0 && t == 0) atomicAdd(a.epoch, 1u);
}

}  // namespace gw

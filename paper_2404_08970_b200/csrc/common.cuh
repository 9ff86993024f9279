// common.cuh -- shared device helpers for the gwdp kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define GW_LOG2E 1.4426950408889634
#define GW_LN2 0.6931471805599453

namespace gw {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------------
// Second-order prefix state: for a segment of (support s_j, value v_j) pairs,
//   P = sum v_j,   A = sum (s_ref - s_j) v_j   measured at the segment's reference
// point s_ref (its last support point).  Every term is >= 0 for sorted supports and
// v >= 0, so the scan is cancellation-free.  Combining an earlier segment a with a
// later segment b:  (a.P + b.P,  a.A + (b.s - a.s) a.P + b.A,  b.s)  (associative).
// This is the k = 1 instance of the paper's recursion a_{i+1,2} = a_{i,2} + Delta a_{i,1}
// with gaps Delta = s_{i+1} - s_i (reading R1).
// ---------------------------------------------------------------------------------
template <typename R>
struct PA {
  R P, A, s;
};

template <typename R>
__device__ __forceinline__ PA<R> pa_combine(const PA<R>& a, const PA<R>& b) {
  PA<R> r;
  r.P = a.P + b.P;
  r.A = a.A + (b.s - a.s) * a.P + b.A;
  r.s = b.s;
  return r;
}

// value at support point s given the exclusive state e (all j before the point)
template <typename R>
__device__ __forceinline__ R pa_eval(const PA<R>& e, R s) {
  return e.A + (s - e.s) * e.P;
}

template <typename R>
__device__ __forceinline__ PA<R> pa_shfl_up(const PA<R>& v, int d) {
  PA<R> r;
  r.P = __shfl_up_sync(0xffffffffu, v.P, d);
  r.A = __shfl_up_sync(0xffffffffu, v.A, d);
  r.s = __shfl_up_sync(0xffffffffu, v.s, d);
  return r;
}

// inclusive warp scan; returns inclusive, writes exclusive (identity for lane 0)
template <typename R>
__device__ __forceinline__ PA<R> pa_warp_scan(PA<R> v, PA<R>& excl) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    PA<R> o = pa_shfl_up(v, d);
    if (lane >= d) v = pa_combine(o, v);
  }
  PA<R> e = pa_shfl_up(v, 1);
  if (lane == 0) { e.P = R(0); e.A = R(0); e.s = v.s; }
  excl = e;
  return v;
}

// Block-wide exclusive scan of PA<double> (NW warps).  smem: 3*NW doubles.
template <int NW>
__device__ __forceinline__ PA<double> pa_block_scan_excl(PA<double> v, double* sm, PA<double>& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  PA<double> ex;
  PA<double> inc = pa_warp_scan(v, ex);
  if (lane == 31) { sm[w] = inc.P; sm[NW + w] = inc.A; sm[2 * NW + w] = inc.s; }
  __syncthreads();
  // Every thread combines the warp totals before its warp (NW small, fixed order).
  // An empty segment (0, 0, s) is a left identity; on the right it only moves the
  // reference point, which pa_eval is invariant to.
  PA<double> pre; pre.P = 0.0; pre.A = 0.0; pre.s = sm[2 * NW];
  PA<double> tot = pre;
  for (int k = 0; k < NW; ++k) {
    PA<double> t; t.P = sm[k]; t.A = sm[NW + k]; t.s = sm[2 * NW + k];
    if (k < w) pre = pa_combine(pre, t);
    tot = pa_combine(tot, t);
  }
  total = tot;
  PA<double> r = pa_combine(pre, ex);
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------
// Deterministic block reductions (fixed tree order).
// ---------------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}
template <typename R>
__device__ __forceinline__ R warp_max(R v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

template <int NW, typename R>
__device__ __forceinline__ R block_sum(R v, R* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sm[w] = v;
  __syncthreads();
  R t = R(0);
  if (w == 0) {
    t = lane < NW ? sm[lane] : R(0);
    t = warp_sum(t);
    if (lane == 0) sm[0] = t;
  }
  __syncthreads();
  t = sm[0];
  __syncthreads();
  return t;
}

template <int NW>
__device__ __forceinline__ float block_max(float v, float* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sm[w] = v;
  __syncthreads();
  float t = -INFINITY;
  if (w == 0) {
    t = lane < NW ? sm[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) sm[0] = t;
  }
  __syncthreads();
  t = sm[0];
  __syncthreads();
  return t;
}

// log-sum-exp pair (max m, sum s of 2^(a - m)) in log2 units
struct LSE2 {
  float m, s;
};
__device__ __forceinline__ LSE2 lse_merge(LSE2 a, LSE2 b) {
  float m = fmaxf(a.m, b.m);
  if (m == -INFINITY) return LSE2{-INFINITY, 0.f};
  return LSE2{m, a.s * exp2f(a.m - m) + b.s * exp2f(b.m - m)};
}
__device__ __forceinline__ LSE2 lse_warp(LSE2 v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    LSE2 o{__shfl_xor_sync(0xffffffffu, v.m, d), __shfl_xor_sync(0xffffffffu, v.s, d)};
    v = lse_merge(v, o);
  }
  return v;
}

__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  // order-independent (max), valid for v >= 0 (and NaN flags as huge)
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
}

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}

}  // namespace gw

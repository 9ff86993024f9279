"""The fused Sinkhorn iteration's FMA-pipe exponential (csrc/fused.cuh ex2_poly2, reading R19c)
against exact 2^x and against the MUFU ex2.approx it stands in for: relative error within MUFU's bound
(<= 2.4e-7 ~ 2 ulp) on the arguments the iteration produces, overflow to inf / NaN at >= 128 and for a NaN
argument (which the validity check rejects, as it does MUFU's inf / NaN), and a floor of 2^-126 (never 0 /
negative / garbage) below.

A tiny test-only kernel is compiled here with nvcc from the product header (it is not in libgwdp.so).
"""

import ctypes as C
import os
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r"""
#include "%s/paper_2404_08970_b200/csrc/fused.cuh"
__global__ void k(const float* x, float* poly, float* mufu, int n) {
  const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    const float2 r = gw::ex2_poly2(make_float2(x[i], x[i + 1]));
    poly[i] = r.x; poly[i + 1] = r.y;
    mufu[i] = gw::ex2_ftz(x[i]); mufu[i + 1] = gw::ex2_ftz(x[i + 1]);
  }
}
extern "C" int run(const float* hx, float* hp, float* hm, int n) {
  float *x, *p, *m;
  cudaMalloc(&x, n * 4); cudaMalloc(&p, n * 4); cudaMalloc(&m, n * 4);
  cudaMemcpy(x, hx, n * 4, cudaMemcpyHostToDevice);
  k<<<(n / 2 + 255) / 256, 256>>>(x, p, m, n);
  cudaMemcpy(hp, p, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hm, m, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(x); cudaFree(p); cudaFree(m);
  return (int)cudaGetLastError();
}
"""


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = tempfile.mkdtemp()
    cu, so = os.path.join(d, "ex2poly.cu"), os.path.join(d, "ex2poly.so")
    open(cu, "w").write(SRC % ROOT)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", cu, "-o", so])
    L = C.CDLL(so)
    L.run.argtypes = [C.c_void_p] * 3 + [C.c_int]
    return L


def _eval(lib, x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.size % 2:
        x = np.append(x, np.float32(0))
    p, m = np.empty_like(x), np.empty_like(x)
    assert lib.run(x.ctypes.data, p.ctypes.data, m.ctypes.data, x.size) == 0
    return x, p, m


def test_ex2_poly_accuracy_matches_mufu_bound(lib):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-126.0, 127.5, 400_000), rng.uniform(-1, 1, 100_000),
                        np.arange(-126, 128, dtype=np.float64), np.arange(-126, 127) + 0.5])
    x, p, m = _eval(lib, x)
    ex = np.exp2(x.astype(np.float64))
    rel_p = np.abs(p / ex - 1)
    rel_m = np.abs(m / ex - 1)
    print("ex2_poly2 max rel err %.3e (MUFU ex2.approx %.3e)" % (rel_p.max(), rel_m.max()))
    assert rel_p.max() <= 3e-7
    assert rel_p.max() <= 1.5 * max(rel_m.max(), 2.0 ** -22)


def test_ex2_poly_overflow_and_floor(lib):
    hi = np.array([128.0, 129.0, 200.0, 1e30, np.inf], dtype=np.float32)
    _, p, m = _eval(lib, hi)
    assert np.all(~np.isfinite(p[:hi.size])), p  # inf / NaN: rejected by the fused iteration's check
    lo = np.array([-126.0, -126.4, -127.0, -150.0, -1e30, -np.inf], dtype=np.float32)
    _, p, _ = _eval(lib, lo)
    p = p[:lo.size]
    assert np.all(np.isfinite(p)) and np.all(p >= 2.0 ** -126 * 0.999) and np.all(p <= 2.0 ** -125.5)
    _, p, m = _eval(lib, np.array([np.nan, 1.0], dtype=np.float32))
    assert not np.isfinite(p[0]) and np.isnan(m[0])  # a NaN argument gives inf / NaN (rejected as MUFU's NaN)

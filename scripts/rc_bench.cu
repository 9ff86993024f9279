// standalone timing harness for k_grad_rc<16> at N = M = 65536 (random inputs; experiments only, not the product):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DRCX_NOSTORE|-DRCX_NOEXCH|-DRCX_NOREGEN|-DRCX_NOSCAN] scripts/rc_bench.cu -o rc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include "../paper_2404_08970_b200/csrc/rowclu.cuh"
using namespace gw;
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void fillf(float* p, size_t n, float v) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v * (float)((i * 2654435761u) % 1000) * 1e-3f; }
__global__ void filld(double* p, size_t n, double v) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v; }
int main(int argc, char** argv) {
  const int64_t n = 65536, m = 65536, ld = m;
  float* G; cudaMalloc(&G, n * ld * 4);
  fillf<<<1184, 256>>>(G, n * ld, 0.3f);
  float *fh, *fl, *gh, *gl, *dxf, *ccx, *yf, *ccy; double *xc, *U0, *Z0;
  cudaMalloc(&fh, n * 4); cudaMalloc(&fl, n * 4); cudaMalloc(&gh, m * 4); cudaMalloc(&gl, m * 4);
  cudaMalloc(&dxf, n * 4); cudaMalloc(&ccx, n * 4); cudaMalloc(&yf, m * 4); cudaMalloc(&ccy, m * 4);
  cudaMalloc(&xc, n * 8); cudaMalloc(&U0, 16 * m * 8); cudaMalloc(&Z0, 16 * m * 8);
  fillf<<<64, 256>>>(fh, n, -1.f); fillf<<<64, 256>>>(fl, n, 1e-6f); fillf<<<64, 256>>>(gh, m, -1.f); fillf<<<64, 256>>>(gl, m, 1e-6f);
  fillf<<<64, 256>>>(dxf, n, 1e-5f); fillf<<<64, 256>>>(ccx, n, 0.1f); fillf<<<64, 256>>>(yf, m, 0.5f); fillf<<<64, 256>>>(ccy, m, 0.1f);
  filld<<<64, 256>>>(xc, n, 0.0); filld<<<64, 256>>>(U0, 16 * m, 0.1); filld<<<64, 256>>>(Z0, 16 * m, 0.1);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  const cuuint64_t dims[3] = {32, (cuuint64_t)(ld / 32), (cuuint64_t)n};
  const cuuint64_t strides[2] = {128, (cuuint64_t)ld * 4};
  const cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
  ((EncodeTiledFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, G, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto kg = k_grad_rc<16>;
  cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rc_dyn_smem());
  cudaFuncSetAttribute(kg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(RC_NT); cfg.dynamicSmemBytes = rc_dyn_smem(); cfg.attrs = at; cfg.numAttrs = 1;
  cfg.gridDim = dim3(148 * 16);
  int ncl = 0; cudaOccupancyMaxActiveClusters(&ncl, (void*)kg, &cfg);
  cfg.gridDim = dim3(ncl * 16);
  RcArgs a; a.G = G; a.ld = ld; a.nl = n; a.m = m; a.rows_per_cluster = (n + ncl - 1) / ncl;
  a.fh = fh; a.fl = fl; a.gh = gh; a.gl = gl; a.ch = 1442.7f; a.cl = 1e-5f; a.dxf = dxf; a.xc = xc; a.ccx = ccx; a.yf = yf; a.ccy = ccy; a.U0 = U0; a.Zn0 = Z0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, kg, tm, a);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, kg, tm, a);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%s ncl=%d: %.3f ms per launch, %.0f GB/s over 8NM (err %s)\n", argc > 1 ? argv[1] : "", ncl, ms / 3, 8.0 * n * m / (ms / 3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

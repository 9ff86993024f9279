// gwdp.cu -- host side of the C ABI (include/gwdp.h): context, workspace, validation,
// the gradient pass, Sinkhorn and the entropic (F)GW mirror-descent loop.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <nvtx3/nvToolsExt.h>
#include <vector>

#include "../../include/gwdp.h"
#include "common.cuh"
#include "fused.cuh"
#include "rowclu.cuh"
#include "grad.cuh"
#include "grad2.cuh"
#include "shard.cuh"
#include "poly.cuh"
#include "grid2d.cuh"
#include "polyk.cuh"
#include "ugw.cuh"
#include "small.cuh"
#include "sink.cuh"
#include "vec.cuh"
#include "f64.cuh"

using namespace gw;

// The next Sinkhorn iteration tries the fused (absorbed-dual) path iff the last column correction
// |log2(CS/q)| was within 2^FUSED_THRESH (§5.3); a failed attempt is caught by k_sink_fast_check
#ifndef FUSED_THRESH
#define FUSED_THRESH 20.f
#endif

// ------------------------------------------------------------------------------ errors
static thread_local std::string g_err;

static gw_status fail(gw_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      return fail(e_ == cudaErrorMemoryAllocation ? GW_ERR_OOM : GW_ERR_CUDA, "%s: %s (%s:%d)", \
                  #x, cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)
#define TRY(x)                      \
  do {                              \
    gw_status s_ = (x);             \
    if (s_ != GW_OK) return s_;     \
  } while (0)
// every kernel launch is followed by KCHECK(); it also counts launches on the ctx `c`
#define KCHECK()                 \
  do {                           \
    CU(cudaGetLastError());      \
    ++c->launches;               \
  } while (0)

// ------------------------------------------------------------------------------ context
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

// Communicator: NCCL (gw_comm_init) or host callbacks (gw_comm_init_host).  The library uses a
// single collective, an all-gather of equal-sized per-rank payloads (shard.cuh combines them in
// rank order), so both transports give bit-identical results.
struct gw_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0;
  gw_allgather_fn host_ag = nullptr;
  void* user = nullptr;
  unsigned char* hsend = nullptr;  // pinned staging for the host transport
  unsigned char* hrecv = nullptr;
  size_t hcap = 0;
};

// Per-kernel-class CUDA-event timing (enabled by gw_ctx_profile; events on ctx's stream).
// slot 7 of gw_ctx_profile is the count of all kernel launches (no class of its own)
enum { PC_GRAD_MOMENTS = 0, PC_GRAD_CARRY, PC_GRAD_MAIN, PC_SINK_ROW, PC_SINK_COL, PC_SINK_FUSED, PC_OBJ, PC_LAUNCHES,
       PC_GRAD_ONEPASS, PC_SINK_XM, PC_N };
struct Prof {
  bool on = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  double ms[PC_N] = {0};
  long long cnt[PC_N] = {0};
};

struct gw_ctx {
  Prof prof;
  long long launches = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cap = nullptr;  // CUDA-graph capture stream (created on first use)
  cudaStream_t cap2 = nullptr;  // capture stream of a conditional node's body
  gw_comm* comm = nullptr;
  std::vector<Buf*> all;
  // vectors
  Buf stage, mom, xc, yc, pn, qn, lp, lq, cvx, cvy;
  Buf fs, gs, fh, fl, gh, gl, ftmp, viol, stop, iters, part, fpart, mode, srow, pfl;
  // gradient aux
  Buf rP, rA, cS, cX, blk, bs, btot, cxend, SAg, WAg, Ptot, Aend, DP, DA, tobj, tent, tcc, objout, scanwt;
  Buf fxs, fys;  // FGW features (staged)
  Buf pnf, qnf;  // fp32 marginals
  Buf yfb, pcoef, pc2s, pfx, pfy, ppart, pM, p4coef, p4c2;  // k = 2 and k = 4 (moments) paths
  Buf gkrp, gkrt, gkcp, gkz, gkct, gkctt, gkobj, gkseg;  // k >= 3 path
  Buf uga, ugb, ugct, ugpart, ugca, ugcb, ugfr, uggr, ugsc, ugrpart;  // UGW
  Buf g2rc, g2rd, g2h, g2cc, g2tt, g2vt, g2tmp, g2s, g2a, g2b, g2ca, g2cb, g2part;  // 2-D grids
  Buf xtab, xg1, xg2, xin, xvec, xtail, xpart;  // multi-rank exchange buffers
  Buf slse, slseg, scsl, scsg, sviolg, sun, sung;  // Sinkhorn column-sum exchange
  Buf sflag, sflagg;
  Buf fsc, gsc;  // scaled duals for the Gibbs regeneration
  Buf Gs;        // solver cost buffer
  Buf rcp, rcpx, rcv, rcvx, rcu, rcz, rcxf, rccx, rccy, rcflag, rcdx;  // 8 N M solver gradient (rowclu.cuh)
  Buf d64T, d64G, d64rt, d64part, d64tot, d64gath, d64obj, d64tmp, d64pay, d64pg, d64mc;  // GW_F64 (f64.cuh)
  Buf s64pay, s64gath, s64part, s64rdev, s64cdev;                                      // GW_F64 Sinkhorn
  double* hpin = nullptr;  // pinned host scratch (64 doubles)
  // one-shot debug export for the next solve (gw_solve_set_export)
  struct {
    int iter = 0;
    void *T = nullptr, *G = nullptr;
    int64_t ld = 0;
  } exp;
  gw_ctx() {
    Buf* b[] = {&stage, &mom, &xc, &yc, &pn, &qn, &lp, &lq, &cvx, &cvy, &fs, &gs, &fh, &fl, &gh, &gl,
                &ftmp, &viol, &stop, &iters, &part, &fpart, &mode, &srow, &pfl, &rP, &rA, &cS, &cX, &blk, &bs, &btot, &cxend,
                &SAg, &WAg, &Ptot, &Aend, &DP, &DA, &tobj, &tent, &tcc, &objout, &scanwt, &fxs, &fys, &fsc, &gsc, &Gs,
                &pnf, &qnf, &xtab, &xg1, &xg2, &xin, &xvec, &xtail, &xpart, &slse, &slseg, &scsl, &scsg, &sun, &sung,
                &sviolg, &sflag, &sflagg, &yfb, &pcoef, &pc2s, &pfx, &pfy, &ppart, &pM, &p4coef, &p4c2,
                &gkrp, &gkrt, &gkcp, &gkz, &gkct, &gkctt, &gkobj, &gkseg,
                &uga, &ugb, &ugct, &ugpart, &ugca, &ugcb, &ugfr, &uggr, &ugsc, &ugrpart,
                &g2rc, &g2rd, &g2h, &g2cc, &g2tt, &g2vt, &g2tmp, &g2s, &g2a, &g2b, &g2ca, &g2cb, &g2part,
                &rcp, &rcpx, &rcv, &rcvx, &rcu, &rcz, &rcxf, &rccx, &rccy, &rcflag, &rcdx,
                &d64T, &d64G, &d64rt, &d64part, &d64tot, &d64gath, &d64obj, &d64tmp, &d64pay, &d64pg, &d64mc,
                &s64pay, &s64gath, &s64part, &s64rdev, &s64cdev};
    for (Buf* x : b) all.push_back(x);
  }
};

static gw_status prof_event(gw_ctx* c, cudaEvent_t* e) {
  Prof& P = c->prof;
  if (P.used == P.pool.size()) {
    cudaEvent_t x;
    CU(cudaEventCreate(&x));
    P.pool.push_back(x);
  }
  *e = P.pool[P.used++];
  return GW_OK;
}
// Open / close a timed region of kernel class `cls` (no-ops when profiling is off).
#define PROF_BEGIN(c, cls)                                           \
  cudaEvent_t pb_##cls = nullptr;                                    \
  if ((c)->prof.on) {                                                \
    TRY(prof_event(c, &pb_##cls));                                   \
    CU(cudaEventRecord(pb_##cls, (c)->stream));                      \
  }
#define PROF_END(c, cls, nlaunch)                                    \
  if ((c)->prof.on) {                                                \
    cudaEvent_t pe_;                                                 \
    TRY(prof_event(c, &pe_));                                        \
    CU(cudaEventRecord(pe_, (c)->stream));                           \
    (c)->prof.ev.push_back({cls, {pb_##cls, pe_}});                  \
    (c)->prof.cnt[cls] += (nlaunch);                                 \
  }

template <typename T>
static gw_status ws(gw_ctx* c, Buf& b, size_t count, T** out) {
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = 16;
  if (b.cap < bytes) {
    if (b.p) {
      CU(cudaStreamSynchronize(c->stream));
      CU(cudaFree(b.p));
      b.p = nullptr;
      b.cap = 0;
    }
    size_t alloc = bytes + (bytes >> 4);  // slack to avoid regrowth churn
    CU(cudaMalloc(&b.p, alloc));
    b.cap = alloc;
  }
  *out = reinterpret_cast<T*>(b.p);
  return GW_OK;
}

static int grid_for(int64_t n, int tpb = 256, int cap = 148 * 16) {
  int64_t g = (n + tpb - 1) / tpb;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

extern "C" const char* gw_last_error(void) { return g_err.c_str(); }
extern "C" int gw_abi_version(void) { return GWDP_ABI_VERSION; }

extern "C" gw_status gw_ctx_create(gw_ctx** out, int device, void* cuda_stream, gw_comm* comm) {
  if (!out) return fail(GW_ERR_INVALID_ARG, "gw_ctx_create: out is null");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(GW_ERR_INVALID_ARG, "gw_ctx_create: bad device %d", device);
  CU(cudaSetDevice(device));
  gw_ctx* c = new gw_ctx();
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  c->comm = comm;
  if (cudaMallocHost(&c->hpin, 64 * sizeof(double)) != cudaSuccess) {
    delete c;
    return fail(GW_ERR_OOM, "gw_ctx_create: pinned alloc failed");
  }
  *out = c;
  return GW_OK;
}

extern "C" gw_status gw_ctx_trim(gw_ctx* c) {
  if (!c) return fail(GW_ERR_INVALID_ARG, "null ctx");
  CU(cudaSetDevice(c->device));
  CU(cudaStreamSynchronize(c->stream));
  for (Buf* b : c->all)
    if (b->p) {
      CU(cudaFree(b->p));
      b->p = nullptr;
      b->cap = 0;
    }
  return GW_OK;
}

// Profiling: enable != 0 turns event timing on (and resets the totals when enable == 2);
// out_ms / out_counts (host, nullable, `nslots` entries) receive the accumulated milliseconds
// and launch counts per kernel class {grad_moments, grad_carry, grad_main, sink_row,
// sink_col, other}.  Synchronises the stream when reading.
extern "C" gw_status gw_ctx_profile(gw_ctx* c, int enable, double* out_ms, int64_t* out_counts, int nslots) {
  if (!c) return fail(GW_ERR_INVALID_ARG, "null ctx");
  CU(cudaSetDevice(c->device));
  Prof& P = c->prof;
  if (out_ms || out_counts || enable == 2 || enable == 0) {
    CU(cudaStreamSynchronize(c->stream));
    for (auto& e : P.ev) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
      P.ms[e.first] += ms;
    }
    P.ev.clear();
    P.used = 0;
  }
  for (int k = 0; k < nslots && k < PC_N; ++k) {
    if (out_ms) out_ms[k] = k == PC_LAUNCHES ? 0.0 : P.ms[k];
    if (out_counts) out_counts[k] = k == PC_LAUNCHES ? c->launches : P.cnt[k];  // slot 7: all kernel launches
  }
  if (enable == 2) {
    for (int k = 0; k < PC_N; ++k) { P.ms[k] = 0; P.cnt[k] = 0; }
    c->launches = 0;
  }
  P.on = enable != 0;
  return GW_OK;
}

extern "C" gw_status gw_ctx_destroy(gw_ctx* c) {
  if (!c) return GW_OK;
  gw_status st = gw_ctx_trim(c);
  for (auto e : c->prof.pool) cudaEventDestroy(e);
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
  return st;
}

// ------------------------------------------------------------------------------ NCCL
extern "C" gw_status gw_get_unique_id(unsigned char id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(GW_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(id, &u, 128);
  return GW_OK;
}

extern "C" gw_status gw_comm_init(gw_comm** out, const unsigned char id[128], int nranks, int rank) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return fail(GW_ERR_INVALID_ARG, "gw_comm_init: bad args");
  gw_comm* c = new gw_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(GW_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return GW_OK;
}

extern "C" gw_status gw_comm_init_host(gw_comm** out, int nranks, int rank, gw_allgather_fn allgather, void* user) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !allgather))
    return fail(GW_ERR_INVALID_ARG, "gw_comm_init_host: bad args");
  gw_comm* c = new gw_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->host_ag = allgather;
  c->user = user;
  *out = c;
  return GW_OK;
}

extern "C" gw_status gw_comm_destroy(gw_comm* c) {
  if (!c) return GW_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->hsend) cudaFreeHost(c->hsend);
  if (c->hrecv) cudaFreeHost(c->hrecv);
  delete c;
  return GW_OK;
}

extern "C" gw_status gw_shard_rows(int64_t n, int nranks, int rank, int64_t* row0, int64_t* n_local) {
  if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !n_local)
    return fail(GW_ERR_INVALID_ARG, "gw_shard_rows: bad args");
  const int64_t base = n / nranks, extra = n % nranks;
  *n_local = base + (rank < extra ? 1 : 0);
  *row0 = rank * base + std::min<int64_t>(rank, extra);
  return GW_OK;
}

extern "C" gw_status gw_check_shards(const int64_t* table, int nranks, int64_t n) {
  if (!table || nranks < 1) return fail(GW_ERR_INVALID_ARG, "gw_check_shards: bad args");
  int64_t next = 0;
  for (int r = 0; r < nranks; ++r) {
    const int64_t r0 = table[2 * r], nl = table[2 * r + 1];
    if (nl < 0 || r0 != next)
      return fail(GW_ERR_DIM_MISMATCH, "rank %d holds rows [%lld, %lld): shards must be consecutive in rank order",
                  r, (long long)r0, (long long)(r0 + nl));
    next = r0 + nl;
  }
  if (next != n) return fail(GW_ERR_DIM_MISMATCH, "shards cover %lld rows, n = %lld", (long long)next, (long long)n);
  return GW_OK;
}

// NVTX ranges (host-side, for nsys / ncu --nvtx): solve, gradient, Sinkhorn, all-gather
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static int nranks_of(const gw_ctx* c) { return c->comm ? c->comm->nranks : 1; }

// Test-only fault injection (SURVEY §4.2 tier T6): GWDP_FAULT=<site> perturbs one value at that site.
static bool fault_is(const char* site) {
  const char* e = getenv("GWDP_FAULT");
  return e && strcmp(e, site) == 0;
}

// All-gather of `bytes` per rank from device `dsend` into device `drecv` ([nranks][bytes], rank
// order), ordered on ctx's stream.  Host transport: synchronises the stream around the callback.
static gw_status comm_allgather(gw_ctx* c, const void* dsend, void* drecv, size_t bytes) {
  NvtxRange nv("gw.allgather");
  gw_comm* k = c->comm;
  if (!k || k->nranks == 1) {
    if (dsend != drecv) CU(cudaMemcpyAsync(drecv, dsend, bytes, cudaMemcpyDeviceToDevice, c->stream));
    return GW_OK;
  }
  if (k->nccl) {
    ncclResult_t r = ncclAllGather(dsend, drecv, bytes, ncclInt8, k->nccl, c->stream);
    if (r != ncclSuccess) return fail(GW_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
    return GW_OK;
  }
  const size_t need = bytes * (size_t)k->nranks;
  if (k->hcap < need) {
    if (k->hsend) cudaFreeHost(k->hsend);
    if (k->hrecv) cudaFreeHost(k->hrecv);
    k->hsend = k->hrecv = nullptr;
    k->hcap = 0;
    CU(cudaMallocHost(&k->hsend, need));
    CU(cudaMallocHost(&k->hrecv, need));
    k->hcap = need;
  }
  CU(cudaMemcpyAsync(k->hsend, dsend, bytes, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (k->host_ag(k->hsend, k->hrecv, (int64_t)bytes, k->user) != 0)
    return fail(GW_ERR_NCCL, "host all-gather callback failed");
  CU(cudaMemcpyAsync(drecv, k->hrecv, need, cudaMemcpyHostToDevice, c->stream));
  return GW_OK;
}

// ------------------------------------------------------------------------------ set-up
struct Prepared {
  int64_t n, m, row0, nl;
  const double *x, *y, *p, *q;  // device views of the caller's vectors (staged if host)
  double *xc, *yc, *pn, *qn, *lp, *lq, *cx, *cy;
  float *pnf, *qnf;  // fp32 copies of the normalised marginals (T^0 = p q^T on the fp32 gradient path)
  float* yf;         // fp32 centred y (k = 2 path)
  double mass_p = 1.0, mass_q = 1.0;  // m(u), m(v): 1 except for ugw_solve (weights not normalised)
  double xlast, ylast;
  double xend_u = 0.0, yend_u = 0.0;  // x_{n-1}, y_{m-1} in the caller's (uncentred) coordinates
  int k = 1;         // distance power
  bool grid2d = false;  // GW_GRID2D: xc / yc are the centred axes (nx, ny entries)
  int nx = 0, ny = 0;
  // row shards of all ranks (multi-rank only): tab[2r] = row0_r, tab[2r+1] = nl_r
  int R = 1, rank = 0;
  int64_t maxnl = 0;
  std::vector<int64_t> tab;
  int64_t* dtab = nullptr;
};

static gw_status check_problem(const gw_problem* pb) {
  if (!pb) return fail(GW_ERR_INVALID_ARG, "problem is null");
  if (pb->n < 1 || pb->m < 1) return fail(GW_ERR_INVALID_ARG, "n, m must be >= 1 (got %lld, %lld)",
                                          (long long)pb->n, (long long)pb->m);
  if (pb->row0 < 0 || pb->n_local < 0 || pb->row0 + pb->n_local > pb->n)
    return fail(GW_ERR_DIM_MISMATCH, "row shard [%lld, %lld) outside [0, %lld)", (long long)pb->row0,
                (long long)(pb->row0 + pb->n_local), (long long)pb->n);
  if (!pb->x || !pb->y || !pb->p || !pb->q) return fail(GW_ERR_INVALID_ARG, "x, y, p, q must be non-null");
  if (pb->k < 1 || pb->k > GW_MAX_K)
    return fail(GW_ERR_UNSUPPORTED, "distance power k=%d: 1 <= k <= %d is implemented (R17)", pb->k, GW_MAX_K);
  if (pb->flags & GW_GRID2D) {
    const int64_t nx = (int64_t)llround(sqrt((double)pb->n)), ny = (int64_t)llround(sqrt((double)pb->m));
    if (nx * nx != pb->n || ny * ny != pb->m)
      return fail(GW_ERR_INVALID_ARG, "GW_GRID2D: n = %lld and m = %lld must be squares", (long long)pb->n,
                  (long long)pb->m);
    if (nx > G2D_MAXN || ny > G2D_MAXN)
      return fail(GW_ERR_UNSUPPORTED, "GW_GRID2D: grid side %lld / %lld exceeds %d", (long long)nx, (long long)ny,
                  G2D_MAXN);
    if (pb->k != 1) return fail(GW_ERR_UNSUPPORTED, "GW_GRID2D: only k = 1 (Manhattan distance) is implemented");
  }
  if (pb->loss != GW_LOSS_SQUARE) return fail(GW_ERR_UNSUPPORTED, "only the square loss is defined (PAPER.md:86)");
  if (pb->dtype != GW_F32 && pb->dtype != GW_F64) return fail(GW_ERR_INVALID_ARG, "dtype %d is not a gw_dtype", pb->dtype);
  if (pb->dtype == GW_F64 && (pb->flags & GW_GRID2D))
    return fail(GW_ERR_UNSUPPORTED, "GW_F64 storage: 1-D supports only (f64.cuh)");
  return GW_OK;
}

static gw_status check_matrix(const void* M, int64_t ld, int64_t m, const char* name) {
  if (!M) return fail(GW_ERR_INVALID_ARG, "%s is null", name);
  if (ld < m || (ld & 3)) return fail(GW_ERR_INVALID_ARG, "%s: ld=%lld must be >= m=%lld and a multiple of 4", name,
                                      (long long)ld, (long long)m);
  if (reinterpret_cast<uintptr_t>(M) & 15) return fail(GW_ERR_INVALID_ARG, "%s: base must be 16-byte aligned", name);
  return GW_OK;
}

// Validate (reading R16) and build the centred supports, normalised
// marginals, their logs and the constant-term vectors c, c'.
// (D o D) w for a 2-D grid (Manhattan, k = 1): sum_a' D1^2 W_A + sum_b' D1^2 W_B + 2 D1 mat(w) D1
static gw_status g2_sqconst(gw_ctx* c, const double* axis, int na, const double* w, double* out) {
  double *WAB, *vAB, *tmp, *dwd;
  TRY(ws(c, c->g2s, 4 * (size_t)na + 2 * (size_t)na * na, &WAB));
  vAB = WAB + 2 * na;
  tmp = vAB + 2 * na;
  dwd = tmp + (size_t)na * na;
  k_g2_wmarg<<<(2 * na + 255) / 256, 256, 0, c->stream>>>(w, na, WAB, WAB + na);
  KCHECK();
  k_g2_sqmv<<<(na + 255) / 256, 256, 0, c->stream>>>(axis, na, WAB, vAB);
  KCHECK();
  k_g2_sqmv<<<(na + 255) / 256, 256, 0, c->stream>>>(axis, na, WAB + na, vAB + na);
  KCHECK();
  const int nn = na * na;
  k_g2_mul_right<<<(nn + 255) / 256, 256, 0, c->stream>>>(w, na, na, axis, tmp);
  KCHECK();
  k_g2_mul_left<<<(nn + 255) / 256, 256, 0, c->stream>>>(axis, na, tmp, na, dwd);
  KCHECK();
  k_g2_const<<<(nn + 255) / 256, 256, 0, c->stream>>>(vAB, vAB + na, dwd, na, out);
  KCHECK();
  return GW_OK;
}

// The ranks' (row0, n_local) table (one all-gather), checked; P.R, P.rank, P.tab, P.dtab, P.maxnl.
static gw_status shard_table(gw_ctx* c, Prepared& P) {
  P.R = nranks_of(c);
  P.rank = c->comm ? c->comm->rank : 0;
  P.tab.assign(2 * (size_t)P.R, 0);
  if (P.R > 1) {
    int64_t* dt;
    TRY(ws(c, c->xtab, 2 * (size_t)P.R + 2, &dt));
    const int64_t mine[2] = {P.row0, P.nl};
    CU(cudaMemcpyAsync(dt + 2 * P.R, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
    TRY(comm_allgather(c, dt + 2 * P.R, dt, 2 * sizeof(int64_t)));
    CU(cudaMemcpyAsync(P.tab.data(), dt, 2 * sizeof(int64_t) * P.R, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    TRY(gw_check_shards(P.tab.data(), P.R, P.n));
    for (int r = 0; r < P.R; ++r)
      if (P.tab[2 * r + 1] == 0) return fail(GW_ERR_DIM_MISMATCH, "rank %d holds no rows (n >= nranks required)", r);
    P.dtab = dt;
    for (int r = 0; r < P.R; ++r) P.maxnl = std::max(P.maxnl, P.tab[2 * r + 1]);
  } else {
    // one rank holds the whole problem: a partial shard would silently treat the other rows of T as
    // zero mass (the carries, moments and column sums are local-only when R == 1)
    if (P.row0 != 0 || P.nl != P.n)
      return fail(GW_ERR_DIM_MISMATCH, "single-rank context: the shard must be (row0, n_local) = (0, %lld), got "
                  "(%lld, %lld)", (long long)P.n, (long long)P.row0, (long long)P.nl);
    P.tab[0] = P.row0;
    P.tab[1] = P.nl;
    P.maxnl = P.nl;
  }
  return GW_OK;
}

static gw_status prepare_2d(gw_ctx* c, const gw_problem* pb, Prepared& P) {
  const int64_t n = pb->n, m = pb->m;
  const int nx = (int)llround(sqrt((double)n)), ny = (int)llround(sqrt((double)m));
  P.n = n; P.m = m; P.row0 = pb->row0; P.nl = pb->n_local; P.k = 1; P.grid2d = true; P.nx = nx; P.ny = ny;
  const bool host = pb->flags & GW_HOST_VECTORS;
  if (host) {
    double* st;
    TRY(ws(c, c->stage, (size_t)(nx + n + ny + m), &st));
    CU(cudaMemcpyAsync(st, pb->x, nx * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + nx, pb->p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + nx + n, pb->y, ny * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + nx + n + ny, pb->q, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    P.x = st; P.p = st + nx; P.y = st + nx + n; P.q = st + nx + n + ny;
  } else {
    P.x = pb->x; P.p = pb->p; P.y = pb->y; P.q = pb->q;
  }
  double* mom;
  TRY(ws(c, c->mom, 16, &mom));
  k_g2_validate<<<1, 1024, 0, c->stream>>>(P.x, nx, P.p, n, mom);
  KCHECK();
  k_g2_validate<<<1, 1024, 0, c->stream>>>(P.y, ny, P.q, m, mom + 8);
  KCHECK();
  CU(cudaMemcpyAsync(c->hpin, mom, 16 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  const double* h = c->hpin;
  if (!(pb->flags & GW_NO_VALIDATE)) {
    if (h[2] != 0 || h[10] != 0) return fail(GW_ERR_NONFINITE, "non-finite entry in x, y, p or q");
    if (h[0] != 0 || h[8] != 0) return fail(GW_ERR_UNSORTED, "the grid axes x and y must be non-decreasing");
    if (h[1] != 0 || h[9] != 0) return fail(GW_ERR_NEGATIVE_WEIGHT, "p and q must be >= 0");
    if (fabs(h[3] - 1.0) > 1e-9 || fabs(h[11] - 1.0) > 1e-9)
      return fail(GW_ERR_NOT_NORMALIZED, "|sum p - 1| = %.3g, |sum q - 1| = %.3g exceed 1e-9 (SPEC.md:72)",
                  fabs(h[3] - 1.0), fabs(h[11] - 1.0));
  }
  double *xc, *yc, *pn, *qn, *lp, *lq, *cx, *cy;
  TRY(ws(c, c->xc, nx, &xc)); TRY(ws(c, c->yc, ny, &yc));
  TRY(ws(c, c->pn, n, &pn)); TRY(ws(c, c->qn, m, &qn));
  TRY(ws(c, c->lp, n, &lp)); TRY(ws(c, c->lq, m, &lq));
  TRY(ws(c, c->cvx, n, &cx)); TRY(ws(c, c->cvy, m, &cy));
  k_g2_prep<<<grid_for(n), 256, 0, c->stream>>>(P.p, n, P.x, nx, mom, pn, lp, xc);
  KCHECK();
  k_g2_prep<<<grid_for(m), 256, 0, c->stream>>>(P.q, m, P.y, ny, mom + 8, qn, lq, yc);
  KCHECK();
  TRY(g2_sqconst(c, xc, nx, pn, cx));
  TRY(g2_sqconst(c, yc, ny, qn, cy));
  P.xc = xc; P.yc = yc; P.pn = pn; P.qn = qn; P.lp = lp; P.lq = lq; P.cx = cx; P.cy = cy;
  P.yf = nullptr;
  TRY(ws(c, c->pnf, n, &P.pnf)); TRY(ws(c, c->qnf, m, &P.qnf));
  k_to_float<<<grid_for(n), 256, 0, c->stream>>>(pn, n, P.pnf);
  KCHECK();
  k_to_float<<<grid_for(m), 256, 0, c->stream>>>(qn, m, P.qnf);
  KCHECK();
  P.xlast = P.ylast = 0.0;
  return shard_table(c, P);
}

// unbalanced (ugw_solve only): p, q are positive measures of any mass; they are kept as given
// (P.pn = p, P.lp = log p, P.cx = (D o D) p) and their masses recorded in P.mass_p / P.mass_q.
static gw_status prepare(gw_ctx* c, const gw_problem* pb, Prepared& P, bool unbalanced = false) {
  TRY(check_problem(pb));
  if (pb->flags & GW_GRID2D) return prepare_2d(c, pb, P);
  const int64_t n = pb->n, m = pb->m;
  P.n = n; P.m = m; P.row0 = pb->row0; P.nl = pb->n_local;
  const bool host = pb->flags & GW_HOST_VECTORS;
  if (host) {
    double* st;
    TRY(ws(c, c->stage, (size_t)(2 * n + 2 * m), &st));
    CU(cudaMemcpyAsync(st, pb->x, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + n, pb->p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + 2 * n, pb->y, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(st + 2 * n + m, pb->q, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    P.x = st; P.p = st + n; P.y = st + 2 * n; P.q = st + 2 * n + m;
  } else {
    P.x = pb->x; P.p = pb->p; P.y = pb->y; P.q = pb->q;
  }
  double* mom;
  TRY(ws(c, c->mom, 16, &mom));
  k_validate<<<2, 1024, 0, c->stream>>>(P.x, P.p, n, P.y, P.q, m, mom);
  KCHECK();
  double *xc, *yc, *pn, *qn, *lp, *lq, *cx, *cy;
  TRY(ws(c, c->xc, n, &xc)); TRY(ws(c, c->yc, m, &yc));
  TRY(ws(c, c->pn, n, &pn)); TRY(ws(c, c->qn, m, &qn));
  TRY(ws(c, c->lp, n, &lp)); TRY(ws(c, c->lq, m, &lq));
  TRY(ws(c, c->cvx, n, &cx)); TRY(ws(c, c->cvy, m, &cy));
  CU(cudaMemcpyAsync(c->hpin, mom, 16 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  const double* h = c->hpin;
  if (!(pb->flags & GW_NO_VALIDATE)) {
    if (h[2] != 0 || h[10] != 0) return fail(GW_ERR_NONFINITE, "non-finite entry in x, y, p or q");
    if (h[0] != 0 || h[8] != 0) return fail(GW_ERR_UNSORTED, "x and y must be non-decreasing (reading R16)");
    if (h[1] != 0 || h[9] != 0) return fail(GW_ERR_NEGATIVE_WEIGHT, "p and q must be >= 0");
    if (!unbalanced && (fabs(h[3] - 1.0) > 1e-9 || fabs(h[11] - 1.0) > 1e-9))
      return fail(GW_ERR_NOT_NORMALIZED, "|sum p - 1| = %.3g, |sum q - 1| = %.3g exceed 1e-9 (SPEC.md:72)",
                  fabs(h[3] - 1.0), fabs(h[11] - 1.0));
  }
  if (unbalanced) {
    if (!(h[3] > 0.0) || !(h[11] > 0.0))
      return fail(GW_ERR_NOT_NORMALIZED, "ugw_solve: the masses m(u) = %.3g, m(v) = %.3g must be > 0", h[3], h[11]);
    P.mass_p = h[3];
    P.mass_q = h[11];
  }
  TRY(ws(c, c->yfb, m, &P.yf));
  TRY(ws(c, c->pnf, n, &P.pnf)); TRY(ws(c, c->qnf, m, &P.qnf));
  k_prep<<<grid_for(n), 256, 0, c->stream>>>(P.x, P.p, n, mom, xc, pn, lp, cx, !unbalanced, P.pnf);
  KCHECK();
  k_prep<<<grid_for(m), 256, 0, c->stream>>>(P.y, P.q, m, mom + 8, yc, qn, lq, cy, !unbalanced, P.qnf, P.yf);
  KCHECK();
  P.xc = xc; P.yc = yc; P.pn = pn; P.qn = qn; P.lp = lp; P.lq = lq; P.cx = cx; P.cy = cy;
  P.k = pb->k;
  if (P.k >= 3) {  // c = (D o D) p, D = |x - x'|^k: the even power 2k by moments (polyk.cuh)
    switch (P.k) {
      case 3: k_gk_const<6><<<1, 1024, 0, c->stream>>>(xc, pn, n, cx); k_gk_const<6><<<1, 1024, 0, c->stream>>>(yc, qn, m, cy); break;
      case 4: k_gk_const<8><<<1, 1024, 0, c->stream>>>(xc, pn, n, cx); k_gk_const<8><<<1, 1024, 0, c->stream>>>(yc, qn, m, cy); break;
      default: k_gk_const<10><<<1, 1024, 0, c->stream>>>(xc, pn, n, cx); k_gk_const<10><<<1, 1024, 0, c->stream>>>(yc, qn, m, cy); break;
    }
    KCHECK();
  }
  if (P.k == 2) {  // c = (D o D) p with D = |x - x'|^2, by moments up to order 4
    k_poly_const<<<1, 1024, 0, c->stream>>>(xc, pn, n, cx);
    KCHECK();
    k_poly_const<<<1, 1024, 0, c->stream>>>(yc, qn, m, cy);
    KCHECK();
  }
  // endpoints (k_validate's slot 7, read with the moments): x_{n-1} in the caller's coordinates and,
  // centred, x_{n-1} - xmid = (x_{n-1} - x_0) / 2
  P.xlast = h[7] - h[6];
  P.ylast = h[15] - h[14];
  P.xend_u = h[7];
  P.yend_u = h[15];
  return shard_table(c, P);
}

// ------------------------------------------------------------------------------ gradient
// Supplied moments (gw_moments): the plan's row totals T 1, T y (this rank's rows) and column totals
// T^T 1, T^T x (all rows), in the caller's coordinates, replace the totals the moments pass reduced:
//   Ptot = T 1,  Aend = sum_q (y_{m-1} - y_q) T_jq = y_{m-1} T 1 - T y,
//   btot = T^T 1,  cxend = sum_j (x_{n-1} - x_j) T_jq = x_{n-1} T^T 1 - T^T x.
__global__ void k_moments_rows(int64_t nl, const double* __restrict__ rs, const double* __restrict__ rys,
                               double yend, double* __restrict__ Ptot, double* __restrict__ Aend) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    Ptot[i] = rs[i];
    Aend[i] = yend * rs[i] - rys[i];
  }
}
__global__ void k_moments_cols(int64_t m, const double* __restrict__ cs, const double* __restrict__ cxs, double xend,
                               double* __restrict__ btot, double* __restrict__ cxend) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    btot[q] = cs[q];
    cxend[q] = xend * cs[q] - cxs[q];
  }
}

struct GradOut {
  double E, viol, go, H, cc;  // filled when OBJ
};

// One DP gradient pass over the (local) plan given by `S` (mode `mode`):
//   STORE -> G (ldG);  OBJ -> E(T), violation(T), H(T) via k_objective.
// The STORE-only pass (every gradient of the solver and gw_grad_dp) AND the OBJ-only objective pass
// run the streaming fp32 kernels of grad2.cuh with T supplied by S2 (fp32 hi/lo duals fh, fl, gh, gl);
// only the rare STORE+OBJ pass (GW_SOLVE_TRACE_OBJECTIVE) runs grad.cuh's kernels with S (fp64
// regeneration from the scaled duals).  Invariant relied on by the S2 passes: whenever sink_run returns,
// fh/fl == split(f log2e/eps) and gh/gl == split(g log2e/eps) of the COMMITTED duals.
static gw_status grad_pass_k1(gw_ctx* c, const Prepared& P, int mode, const TSrc& S, const TSrc2& S2, float* G,
                              int64_t ldG, bool store, bool obj, const double* fx, const double* fy, double alpha,
                              double* objout_dev, double beta = 0.0, const gw_moments* mom = nullptr) {
  const int64_t nl = P.nl, m = P.m, n = P.n;
  const int R = P.R;
  if (nl == 0) return GW_OK;  // single rank only: prepare() rejects empty shards when R > 1
  const int nb = (int)((nl + TR - 1) / TR), ns = (int)((m + TC - 1) / TC);
  double *rP, *rA, *cS, *cX, *blk, *bs, *btot, *cxend, *SAg, *WAg, *Ptot, *Aend, *DP, *DA, *tobj, *tent, *tcc;
  TRY(ws(c, c->rP, (size_t)ns * nl, &rP)); TRY(ws(c, c->rA, (size_t)ns * nl, &rA));
  TRY(ws(c, c->cS, (size_t)nb * m, &cS)); TRY(ws(c, c->cX, (size_t)nb * m, &cX));
  TRY(ws(c, c->blk, (size_t)nb * ns * 4, &blk)); TRY(ws(c, c->bs, (size_t)nb * ns * 4, &bs));
  TRY(ws(c, c->btot, 2 * (size_t)m, &btot));  // {btot | cxend}: one all-gather payload
  cxend = btot + m;
  TRY(ws(c, c->SAg, m, &SAg)); TRY(ws(c, c->WAg, m, &WAg));
  TRY(ws(c, c->Ptot, 2 * (size_t)P.maxnl, &Ptot));  // {Ptot | Aend}, padded to the largest shard
  Aend = Ptot + P.maxnl;
  TRY(ws(c, c->DP, (size_t)(R > 1 ? n : nl), &DP)); TRY(ws(c, c->DA, (size_t)(R > 1 ? n : nl), &DA));
  TRY(ws(c, c->tobj, (size_t)nb * ns, &tobj)); TRY(ws(c, c->tent, (size_t)nb * ns, &tent));
  TRY(ws(c, c->tcc, (size_t)nb * ns, &tcc));
  const double* xl = P.xc + P.row0;
  dim3 grid(ns, nb);
  // streaming kernels (grad2.cuh) for the STORE-only gradient and the OBJ-only objective pass; the
  // rare STORE+OBJ pass (GW_SOLVE_TRACE_OBJECTIVE) runs grad.cuh's kernels
  const bool fast = store != obj;
  // the objective pass is timed as its own class
  const int pc_mom = !obj ? PC_GRAD_MOMENTS : PC_OBJ, pc_main = !obj ? PC_GRAD_MAIN : PC_OBJ;
  PROF_BEGIN(c, pc_mom);
  if (fast) {
    switch (mode) {
      case T_EXPLICIT: k_grad_moments3o<T_EXPLICIT><<<grid, 256, 0, c->stream>>>(S2, nl, m, xl, P.yc, rP, rA, cS, cX); break;
      case T_GIBBS: k_grad_moments3<T_GIBBS><<<grid, 256, 0, c->stream>>>(S2, nl, m, xl, P.yc, rP, rA, cS, cX); break;
      default: k_grad_moments3o<T_PRODUCT><<<grid, 256, 0, c->stream>>>(S2, nl, m, xl, P.yc, rP, rA, cS, cX); break;
    }
  } else {
    switch (mode) {
      case T_EXPLICIT: k_grad_moments<T_EXPLICIT><<<grid, NT, 0, c->stream>>>(S, nl, m, xl, P.yc, rP, rA, cS, cX); break;
      case T_GIBBS: k_grad_moments<T_GIBBS><<<grid, NT, 0, c->stream>>>(S, nl, m, xl, P.yc, rP, rA, cS, cX); break;
      default: k_grad_moments<T_PRODUCT><<<grid, NT, 0, c->stream>>>(S, nl, m, xl, P.yc, rP, rA, cS, cX); break;
    }
  }
  KCHECK();
  PROF_END(c, pc_mom, !obj ? 1 : 0);
  PROF_BEGIN(c, PC_GRAD_CARRY);
  k_colcarry<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(nl, m, nb, xl, cS, cX, btot, cxend);
  KCHECK();
  k_rowcarry<<<nb, TR, 0, c->stream>>>(nl, m, ns, xl, P.yc, rP, rA, blk, Ptot, Aend);
  KCHECK();
  if (mom) {  // supplied row totals (this rank's rows) replace the reduced ones
    k_moments_rows<<<grid_for(nl), 256, 0, c->stream>>>(nl, mom->row_sum, mom->row_ysum, P.yend_u, Ptot, Aend);
    KCHECK();
    if (R == 1) {
      k_moments_cols<<<grid_for(m), 256, 0, c->stream>>>(m, mom->col_sum, mom->col_xsum, P.xend_u, btot, cxend);
      KCHECK();
    }
  }
  if (fault_is("carry") && ns > 1 && nl > 0) {  // test-only: one row carry doubled
    k_fault_scale<<<1, 32, 0, c->stream>>>(rP, (int64_t)1 * nl + nl / 2, 2.0);
    KCHECK();
  }
  double* tail = nullptr;
  if (R > 1) TRY(ws(c, c->xtail, 8 * (size_t)ns, &tail));
  k_blkscan_w<<<(ns + 7) / 8, 256, 0, c->stream>>>(nl, nb, ns, xl, blk, bs, tail);
  KCHECK();
  const double* DPsrc = Ptot;
  const double* DAsrc = Aend;
  const double* xs_rows = xl;
  int64_t nrows_dp = nl;
  if (R > 1) {
    // (1) column state of the ranks above + global column totals
    double *g1, *in;
    TRY(ws(c, c->xg1, 2 * (size_t)m * R, &g1));
    TRY(ws(c, c->xin, 2 * (size_t)m, &in));
    TRY(comm_allgather(c, btot, g1, 2 * sizeof(double) * (size_t)m));
    k_cols_ranks<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(g1, R, P.rank, P.dtab, P.xc, m, in, in + m, btot,
                                                                   cxend);
    KCHECK();
    if (mom) {  // supplied global column totals replace the gathered ones
      k_moments_cols<<<grid_for(m), 256, 0, c->stream>>>(m, mom->col_sum, mom->col_xsum, P.xend_u, btot, cxend);
      KCHECK();
    }
    k_cols_apply<<<grid_for((int64_t)nb * m, 256, 148 * 16), 256, 0, c->stream>>>(nb, m, xl, in, in + m, cS, cX);
    KCHECK();
    // (2) block-strip sums of the row carries of the ranks above
    double* g3;
    TRY(ws(c, c->xg2, std::max<size_t>(4 * (size_t)ns * R, 2 * (size_t)P.maxnl * R), &g3));
    TRY(comm_allgather(c, tail, g3, 4 * sizeof(double) * (size_t)ns));
    k_bs_ranks<<<(ns + 127) / 128, 128, 0, c->stream>>>(g3, R, P.rank, P.dtab, P.xc, ns, tail + 4 * ns);
    KCHECK();
    k_bs_apply<<<grid_for((int64_t)nb * ns, 256, 148 * 8), 256, 0, c->stream>>>(nb, ns, xl, tail + 4 * ns, bs);
    KCHECK();
    // (3) row totals of every rank -> the 1-D DPs D_X(.) over the global support
    double* vg;
    TRY(ws(c, c->xvec, 2 * (size_t)n, &vg));
    TRY(comm_allgather(c, Ptot, g3, 2 * sizeof(double) * (size_t)P.maxnl));
    k_unpad<<<grid_for(P.maxnl), 256, 0, c->stream>>>(g3, R, 2 * P.maxnl, P.dtab, vg);
    KCHECK();
    k_unpad<<<grid_for(P.maxnl), 256, 0, c->stream>>>(g3 + P.maxnl, R, 2 * P.maxnl, P.dtab, vg + n);
    KCHECK();
    DPsrc = vg;
    DAsrc = vg + n;
    xs_rows = P.xc;
    nrows_dp = n;
  }
  Scan1DBatch B;
  memset(&B, 0, sizeof(B));
  B.d[0] = Scan1D{btot, P.yc, m, SAg, nullptr, nullptr};
  B.d[1] = Scan1D{cxend, P.yc, m, WAg, nullptr, nullptr};
  B.d[2] = Scan1D{DPsrc, xs_rows, nrows_dp, nullptr, DP, nullptr};
  B.d[3] = Scan1D{DAsrc, xs_rows, nrows_dp, nullptr, DA, nullptr};
  {  // the four 1-D programmes, each over K CTAs (k_scan1d_tot / k_scan1d_out)
    const int64_t nmax = std::max<int64_t>(m, nrows_dp);
    const int K = (int)std::min<int64_t>(SCAN_KMAX, std::max<int64_t>(1, (nmax + 4095) / 4096));
    double* wt;
    TRY(ws(c, c->scanwt, (size_t)4 * K * 32 * 3, &wt));
    k_scan1d_tot<<<dim3(K, 4), 1024, 0, c->stream>>>(B, K, wt);
    KCHECK();
    k_scan1d_out<<<dim3(K, 4), 1024, 0, c->stream>>>(B, K, wt);
    KCHECK();
  }
  PROF_END(c, PC_GRAD_CARRY, 5);
  MainArgs a;
  a.S = S; a.nl = nl; a.m = m; a.nb = nb; a.ns = ns;
  a.xl = xl; a.yc = P.yc; a.cl = P.cx + P.row0; a.c2 = P.cy;
  a.DP = R > 1 ? DP + P.row0 : DP; a.DA = R > 1 ? DA + P.row0 : DA;
  a.SAg = SAg; a.WAg = WAg;
  a.rP = rP; a.rA = rA; a.cS = cS; a.cX = cX; a.bs = bs; a.xlast = P.xlast; a.ylast = P.ylast;
  a.G = G; a.ldG = ldG; a.tile_obj = tobj; a.tile_ent = tent; a.tile_cc = tcc;
  a.fx = fx ? fx + P.row0 : nullptr; a.fy = fy; a.alpha = alpha; a.beta = beta;
  PROF_BEGIN(c, pc_main);
#define LAUNCH_MAIN(MODE, ST, OB)                                                                  \
  do {                                                                                             \
    const size_t dsm = main_dyn_smem<OB>();                                                        \
    CU(cudaFuncSetAttribute(k_grad_main<MODE, ST, OB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            (int)dsm));                                                            \
    k_grad_main<MODE, ST, OB><<<grid, NT, dsm, c->stream>>>(a);                                    \
  } while (0)
#define LAUNCH_STORE2(MODE)                                                                           \
  do {                                                                                                \
    if (obj) {                                                                                        \
      const int dsm = G2SUB * G2RS * (int)sizeof(float);                                              \
      if (fx) {                                                                                       \
        CU(cudaFuncSetAttribute(k_grad_store2<MODE, true, true>,                                      \
                                cudaFuncAttributeMaxDynamicSharedMemorySize, dsm));                   \
        k_grad_store2<MODE, true, true><<<grid, G2T, dsm, c->stream>>>(a, S2);                        \
      } else {                                                                                        \
        CU(cudaFuncSetAttribute(k_grad_store2<MODE, false, true>,                                     \
                                cudaFuncAttributeMaxDynamicSharedMemorySize, dsm));                   \
        k_grad_store2<MODE, false, true><<<grid, G2T, dsm, c->stream>>>(a, S2);                       \
      }                                                                                               \
    } else if (beta != 0.0) {                                                                         \
      const int dsm = G2SUB * G2RS * (int)sizeof(float);                                              \
      if (fx) {                                                                                       \
        CU(cudaFuncSetAttribute(k_grad_store2<MODE, true, false, true>,                               \
                                cudaFuncAttributeMaxDynamicSharedMemorySize, dsm));                   \
        k_grad_store2<MODE, true, false, true><<<grid, G2T, dsm, c->stream>>>(a, S2);                 \
      } else {                                                                                        \
        CU(cudaFuncSetAttribute(k_grad_store2<MODE, false, false, true>,                              \
                                cudaFuncAttributeMaxDynamicSharedMemorySize, dsm));                   \
        k_grad_store2<MODE, false, false, true><<<grid, G2T, dsm, c->stream>>>(a, S2);                \
      }                                                                                               \
    } else if (fx) {                                                                                  \
      k_grad_store2<MODE, true><<<grid, G2T, 0, c->stream>>>(a, S2);                                  \
    } else {                                                                                          \
      k_grad_store2<MODE, false><<<grid, G2T, 0, c->stream>>>(a, S2);                                 \
    }                                                                                                 \
  } while (0)
  if (fast) {
    if (mode == T_EXPLICIT) LAUNCH_STORE2(T_EXPLICIT);
    else if (mode == T_GIBBS) LAUNCH_STORE2(T_GIBBS);
    else LAUNCH_STORE2(T_PRODUCT);
  } else if (mode == T_EXPLICIT) {
    if (store && obj) LAUNCH_MAIN(T_EXPLICIT, true, true);
    else if (store) LAUNCH_MAIN(T_EXPLICIT, true, false);
    else LAUNCH_MAIN(T_EXPLICIT, false, true);
  } else if (mode == T_GIBBS) {
    if (store && obj) LAUNCH_MAIN(T_GIBBS, true, true);
    else if (store) LAUNCH_MAIN(T_GIBBS, true, false);
    else LAUNCH_MAIN(T_GIBBS, false, true);
  } else {
    if (store && obj) LAUNCH_MAIN(T_PRODUCT, true, true);
    else if (store) LAUNCH_MAIN(T_PRODUCT, true, false);
    else LAUNCH_MAIN(T_PRODUCT, false, true);
  }
#undef LAUNCH_MAIN
#undef LAUNCH_STORE2
  KCHECK();
  PROF_END(c, pc_main, 1);
  if (obj) {
    double *part, *gpart;
    TRY(ws(c, c->xpart, 8 * (size_t)(R + 1), &part));
    gpart = part + 8;
    k_obj_partial<<<1, 1024, 0, c->stream>>>(Ptot, xl, P.pn + P.row0, P.cx + P.row0, nl, tobj, (int64_t)nb * ns,
                                             tent, fx ? tcc : nullptr, part);
    KCHECK();
    TRY(comm_allgather(c, part, gpart, 8 * sizeof(double)));
    k_obj_final<<<1, 1024, 0, c->stream>>>(gpart, R, btot, P.yc, P.qn, P.cy, m, objout_dev);
    KCHECK();
  }
  return GW_OK;
}

// k = 2 (poly.cuh): global moments M_rt of the plan (one read), then G by rows (one write) and/or
// E(T) from the moments.  Multi-rank: the per-CTA moment partials are all-gathered and summed in
// rank order.
static gw_status poly_moments(gw_ctx* c, const Prepared& P, int mode, const TSrc2& S2, bool obj, double** Mout) {
  const int64_t nl = P.nl, m = P.m;
  const int64_t rows_per_cta = (PT / 32) * PRPW;
  const int ncta = (int)std::max<int64_t>(1, (nl + rows_per_cta - 1) / rows_per_cta);
  // equal all-gather payloads: pad every rank's partials to the largest shard's CTA count
  const int maxcta = (int)std::max<int64_t>(ncta, (P.maxnl + rows_per_cta - 1) / rows_per_cta);
  double *part, *M;
  TRY(ws(c, c->ppart, (size_t)(PNM + 1) * maxcta * (P.R + 1), &part));
  TRY(ws(c, c->pM, PNM + 1, &M));
  if (maxcta > ncta)
    CU(cudaMemsetAsync(part + (size_t)(PNM + 1) * ncta, 0, sizeof(double) * (PNM + 1) * (maxcta - ncta), c->stream));
  const double* xl = P.xc + P.row0;
#define LAUNCH_PM(MODE)                                                                                    \
  do {                                                                                                     \
    if (obj) k_poly_moments<MODE, true><<<ncta, PT, 0, c->stream>>>(S2, nl, m, xl, P.yf, part);            \
    else k_poly_moments<MODE, false><<<ncta, PT, 0, c->stream>>>(S2, nl, m, xl, P.yf, part);               \
  } while (0)
  if (mode == T_EXPLICIT) LAUNCH_PM(T_EXPLICIT);
  else if (mode == T_GIBBS) LAUNCH_PM(T_GIBBS);
  else LAUNCH_PM(T_PRODUCT);
#undef LAUNCH_PM
  KCHECK();
  if (P.R > 1) {
    double* all = part + (size_t)(PNM + 1) * maxcta;
    TRY(comm_allgather(c, part, all, sizeof(double) * (PNM + 1) * (size_t)maxcta));
    k_poly_reduce<<<1, 32, 0, c->stream>>>(all, maxcta * P.R, M);
  } else {
    k_poly_reduce<<<1, 32, 0, c->stream>>>(part, ncta, M);
  }
  KCHECK();
  *Mout = M;
  return GW_OK;
}

// 2-D grids (grid2d.cuh): per-row reductions of the plan -> four marginal matrices -> V = D1x T.. D1y
// (tiny) -> G by rows; the objective from the same marginals plus the plan's row / column sums.
static gw_status grad_pass_2d(gw_ctx* c, const Prepared& P, int mode, const TSrc2& S2, float* G, int64_t ldG,
                              bool store, bool obj, const double* fx, const double* fy, double alpha,
                              double* objout_dev) {
  const int nx = P.nx, ny = P.ny;
  const int64_t n = P.n, m = P.m, nl = P.nl;
  const int nn = nx * ny;
  double *RC, *RD, *Hr, *CCr, *TT, *VT, *tmp;
  TRY(ws(c, c->g2rc, (size_t)std::max<int64_t>(nl, 1) * ny, &RC));
  TRY(ws(c, c->g2rd, (size_t)std::max<int64_t>(nl, 1) * ny, &RD));
  TRY(ws(c, c->g2h, (size_t)std::max<int64_t>(nl, 1), &Hr)); TRY(ws(c, c->g2cc, (size_t)std::max<int64_t>(nl, 1), &CCr));
  TRY(ws(c, c->g2tt, 4 * (size_t)nn, &TT)); TRY(ws(c, c->g2vt, 4 * (size_t)nn, &VT));
  TRY(ws(c, c->g2tmp, (size_t)nn, &tmp));
  const int bt = (ny + 31) / 32 * 32;
  const double* fxl = fx ? fx + P.row0 : nullptr;
  PROF_BEGIN(c, PC_GRAD_MOMENTS);
#define LAUNCH_RR(MODE, OB)                                                                                   \
  k_g2_rowred<MODE, OB><<<(unsigned)nl, bt, 0, c->stream>>>(S2, ny, RC, RD, Hr, OB ? fxl : nullptr, fy, CCr)
  if (nl > 0) {
    if (obj) {
      if (mode == T_EXPLICIT) LAUNCH_RR(T_EXPLICIT, true);
      else if (mode == T_GIBBS) LAUNCH_RR(T_GIBBS, true);
      else LAUNCH_RR(T_PRODUCT, true);
    } else if ((ny == 128 || ny == 256) && !getenv("GWDP_G2_SCALAR")) {
      // 128-bit loads (k_g2_rowred4): rows of 128^2 or 256^2 columns
#define LAUNCH_RR4(MODE, TPR) k_g2_rowred4<MODE, TPR><<<(unsigned)nl, 256, 0, c->stream>>>(S2, RC, RD)
      if (ny == 256) {
        if (mode == T_EXPLICIT) LAUNCH_RR4(T_EXPLICIT, 64);
        else if (mode == T_GIBBS) LAUNCH_RR4(T_GIBBS, 64);
        else LAUNCH_RR4(T_PRODUCT, 64);
      } else {
        if (mode == T_EXPLICIT) LAUNCH_RR4(T_EXPLICIT, 32);
        else if (mode == T_GIBBS) LAUNCH_RR4(T_GIBBS, 32);
        else LAUNCH_RR4(T_PRODUCT, 32);
      }
#undef LAUNCH_RR4
    } else {
      if (mode == T_EXPLICIT) LAUNCH_RR(T_EXPLICIT, false);
      else if (mode == T_GIBBS) LAUNCH_RR(T_GIBBS, false);
      else LAUNCH_RR(T_PRODUCT, false);
    }
  }
#undef LAUNCH_RR
  KCHECK();
  PROF_END(c, PC_GRAD_MOMENTS, obj ? 0 : 1);
  PROF_BEGIN(c, PC_GRAD_CARRY);
  k_g2_marg<<<(4 * nn + 255) / 256, 256, 0, c->stream>>>(RC, RD, nx, ny, P.row0, nl, TT, TT + nn, TT + 2 * nn,
                                                         TT + 3 * nn);
  KCHECK();
  if (P.R > 1) {  // the four marginal matrices of the whole plan: partials summed in rank order
    double* g;
    TRY(ws(c, c->xg1, 4 * (size_t)nn * (P.R + 1), &g));
    TRY(comm_allgather(c, TT, g, 4 * sizeof(double) * (size_t)nn));
    k_gk_ranks<<<grid_for(4 * (int64_t)nn), 256, 0, c->stream>>>(g, P.R, P.rank, 4 * (int64_t)nn,
                                                                 g + 4 * (size_t)nn * P.R, TT);
    KCHECK();
  }
  for (int k = 0; k < 4; ++k) {
    k_g2_mul_right<<<(nn + 255) / 256, 256, 0, c->stream>>>(TT + (size_t)k * nn, nx, ny, P.yc, tmp);
    KCHECK();
    k_g2_mul_left<<<(nn + 255) / 256, 256, 0, c->stream>>>(P.xc, nx, tmp, ny, VT + (size_t)k * nn);
    KCHECK();
  }
  PROF_END(c, PC_GRAD_CARRY, 4);
  if (obj) {
    // realised marginals a = T 1 (from the row reductions), b = T^T 1 (column pass); with R > 1
    // b's partials are summed and a, H, <C o C, T> per row are gathered into global vectors
    double *av, *bv, *cA, *cB, *part;
    TRY(ws(c, c->g2a, 3 * (size_t)n, &av)); TRY(ws(c, c->g2b, (size_t)m, &bv));
    TRY(ws(c, c->g2ca, (size_t)n, &cA)); TRY(ws(c, c->g2cb, (size_t)m, &cB));
    const int nch = (int)((nl + 255) / 256);
    TRY(ws(c, c->g2part, (size_t)std::max(nch, 1) * m, &part));
    double* al = av;  // this rank's rows (R == 1: the whole vector)
    k_g2_rowsum<<<grid_for(nl), 256, 0, c->stream>>>(RC, nl, ny, al);
    KCHECK();
    dim3 cg((unsigned)((m + 255) / 256), (unsigned)std::max(nch, 1));
    if (nl > 0) {
      if (mode == T_EXPLICIT) k_g2_colsum<T_EXPLICIT><<<cg, 256, 0, c->stream>>>(S2, nl, m, part);
      else if (mode == T_GIBBS) k_g2_colsum<T_GIBBS><<<cg, 256, 0, c->stream>>>(S2, nl, m, part);
      else k_g2_colsum<T_PRODUCT><<<cg, 256, 0, c->stream>>>(S2, nl, m, part);
      KCHECK();
    }
    k_g2_colsum_reduce<<<grid_for(m), 256, 0, c->stream>>>(part, nch, m, bv);
    KCHECK();
    const double *aF = av, *HF = Hr, *CF = CCr;
    if (P.R > 1) {
      double *g, *pk;
      const int64_t ml = P.maxnl;
      TRY(ws(c, c->xg2, 3 * (size_t)ml * (P.R + 1), &g));
      pk = g + 3 * (size_t)ml * P.R;
      CU(cudaMemsetAsync(pk, 0, 3 * sizeof(double) * (size_t)ml, c->stream));
      CU(cudaMemcpyAsync(pk, al, sizeof(double) * (size_t)nl, cudaMemcpyDeviceToDevice, c->stream));
      CU(cudaMemcpyAsync(pk + ml, Hr, sizeof(double) * (size_t)nl, cudaMemcpyDeviceToDevice, c->stream));
      if (fx) CU(cudaMemcpyAsync(pk + 2 * ml, CCr, sizeof(double) * (size_t)nl, cudaMemcpyDeviceToDevice, c->stream));
      TRY(comm_allgather(c, pk, g, 3 * sizeof(double) * (size_t)ml));
      double* full = av + n;  // [H | CC] after the first n entries of av's buffer
      k_unpad<<<grid_for(ml), 256, 0, c->stream>>>(g, P.R, 3 * ml, P.dtab, av);
      k_unpad<<<grid_for(ml), 256, 0, c->stream>>>(g + ml, P.R, 3 * ml, P.dtab, full);
      k_unpad<<<grid_for(ml), 256, 0, c->stream>>>(g + 2 * ml, P.R, 3 * ml, P.dtab, full + n);
      KCHECK();
      HF = full;
      CF = full + n;
      // b: the ranks' column sums in rank order
      double* gb;
      TRY(ws(c, c->xvec, (size_t)m * (P.R + 1), &gb));
      TRY(comm_allgather(c, bv, gb, sizeof(double) * (size_t)m));
      k_gk_ranks<<<grid_for(m), 256, 0, c->stream>>>(gb, P.R, P.rank, m, gb + (size_t)m * P.R, bv);
      KCHECK();
    }
    TRY(g2_sqconst(c, P.xc, nx, aF, cA));
    TRY(g2_sqconst(c, P.yc, ny, bv, cB));
    k_g2_objective<<<1, 1024, 0, c->stream>>>(aF, cA, P.pn, n, bv, cB, P.qn, m, VT, TT, 4 * nn, HF,
                                              fx ? CF : nullptr, objout_dev);
    KCHECK();
  }
  if (store && nl > 0) {
    PROF_BEGIN(c, PC_GRAD_MAIN);
    const dim3 sg((unsigned)((m + 256 * G2SC - 1) / (256 * G2SC)), (unsigned)((nl + G2SR - 1) / G2SR));
    const int sc4 = fx ? g2sc4<true>() : g2sc4<false>();
    const dim3 sg4((unsigned)((m + 256 * sc4 - 1) / (256 * sc4)), (unsigned)((nl + G2SR - 1) / G2SR));
    if (ny % 4 == 0) {  // 4 consecutive columns share their grid row c: vectorised stores
      if (fx) k_g2_store4<true><<<sg4, 256, 0, c->stream>>>(P.cx, P.cy, VT, VT + nn, VT + 2 * nn, VT + 3 * nn, nx, ny,
                                                          P.row0, nl, m, alpha, fx, fy, G, ldG);
      else k_g2_store4<false><<<sg4, 256, 0, c->stream>>>(P.cx, P.cy, VT, VT + nn, VT + 2 * nn, VT + 3 * nn, nx, ny,
                                                        P.row0, nl, m, alpha, nullptr, nullptr, G, ldG);
    } else if (fx) k_g2_store<true><<<sg, 256, 0, c->stream>>>(P.cx, P.cy, VT, VT + nn, VT + 2 * nn, VT + 3 * nn, nx, ny,
                                                       P.row0, nl, m, alpha, fx, fy, G, ldG);
    else k_g2_store<false><<<sg, 256, 0, c->stream>>>(P.cx, P.cy, VT, VT + nn, VT + 2 * nn, VT + 3 * nn, nx, ny,
                                                     P.row0, nl, m, alpha, nullptr, nullptr, G, ldG);
    KCHECK();
    PROF_END(c, PC_GRAD_MAIN, 1);
  }
  return GW_OK;
}

// General distance power k >= 3 (polyk.cuh): tile power sums -> carries -> one main pass.
template <int K, int MODE, bool STORE, bool OBJ, bool FGW>
static gw_status gk_main_launch(gw_ctx* c, dim3 grid, const TSrc2& S2, int64_t nl, int64_t m, const double* xl,
                                const double* yc, const double* rp, const double* rt, const double* Z,
                                const double* ct, const double* cl, const double* c2, double alpha, const double* fx,
                                const double* fy, float* G, int64_t ldG, double* tob, const double* carry) {
  auto kern = k_gk_main<K, MODE, STORE, OBJ, FGW>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gk_smem_bytes<K>()));
  kern<<<grid, GK, gk_smem_bytes<K>(), c->stream>>>(S2, nl, m, xl, yc, rp, rt, Z, ct, cl, c2, alpha, fx, fy, G, ldG,
                                                    tob, carry);
  KCHECK();
  return GW_OK;
}

// Exclusive prefix over the nt tiles of part[nt][len2] (+ totals): segmented when there are many tiles
static gw_status gk_scan_tiles(gw_ctx* c, double* part, int nt, int64_t len2, double* tot) {
  // one thread per element already fills the machine from ~128K elements (C4: 262144, where the segmented
  // form measured slower: 2.1 vs 1.6 ms per gradient); below that, segments add the parallelism
  if (nt <= 32 || len2 >= 131072) {
    k_gk_scan_tiles<<<grid_for(len2), 256, 0, c->stream>>>(part, nt, len2, tot);
    KCHECK();
    return GW_OK;
  }
  const int nseg = std::min(32, (nt + 15) / 16);
  double* seg;
  TRY(ws(c, c->gkseg, (size_t)nseg * len2, &seg));
  const dim3 g((unsigned)((len2 + 255) / 256), (unsigned)nseg);
  k_gk_scan_seg_a<<<g, 256, 0, c->stream>>>(part, nt, len2, nseg, seg);
  KCHECK();
  k_gk_scan_seg_b<<<g, 256, 0, c->stream>>>(part, nt, len2, nseg, seg, tot);
  KCHECK();
  return GW_OK;
}

template <int K, int MODE>
static gw_status grad_pass_gk_mode(gw_ctx* c, const Prepared& P, const TSrc2& S2, float* G, int64_t ldG, bool store,
                                   bool obj, const double* fx, const double* fy, double alpha, double* objout_dev) {
  const int64_t nl = P.nl, m = P.m;
  const int ntc = (int)((m + GR - 1) / GR), ntr = (int)((nl + GR - 1) / GR);  // regions (polyk.cuh)
  const size_t K1 = K + 1;
  double *rp, *rt, *cp, *Z, *ct, *ctt, *tob;
  TRY(ws(c, c->gkrp, (size_t)ntc * K1 * nl, &rp)); TRY(ws(c, c->gkrt, K1 * nl, &rt));
  TRY(ws(c, c->gkcp, (size_t)ntr * K1 * m, &cp)); TRY(ws(c, c->gkz, (size_t)ntr * K1 * m, &Z));
  TRY(ws(c, c->gkct, K1 * m, &ct)); TRY(ws(c, c->gkctt, K1 * m, &ctt));
  TRY(ws(c, c->gkobj, (size_t)ntc * ntr, &tob));
  const double* xl = P.xc + P.row0;
  const dim3 grid((unsigned)ntc, (unsigned)ntr);
  PROF_BEGIN(c, PC_GRAD_MOMENTS);
  auto ks = k_gk_sums<K, MODE>;
  CU(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gk_smem_bytes<K>()));
  ks<<<grid, GK, gk_smem_bytes<K>(), c->stream>>>(S2, nl, m, xl, P.yc, rp, cp);
  KCHECK();
  PROF_END(c, PC_GRAD_MOMENTS, 1);
  PROF_BEGIN(c, PC_GRAD_CARRY);
  TRY(gk_scan_tiles(c, rp, ntc, (int64_t)K1 * nl, rt));
  k_gk_apply<K><<<(unsigned)(ntr * K1), 256, 0, c->stream>>>(cp, m, P.yc, Z);
  KCHECK();
  TRY(gk_scan_tiles(c, Z, ntr, (int64_t)K1 * m, ct));
  // multi-rank: the column sums of W over the rows of the ranks above (carry) and over all rows
  // (ct, replaced by the global totals): one all-gather of (k+1) M fp64 per rank
  double* carry = nullptr;
  if (P.R > 1) {
    double *g, *tot;
    TRY(ws(c, c->xg1, K1 * (size_t)m * (P.R + 2), &g));
    carry = g + K1 * (size_t)m * P.R;
    tot = carry + K1 * (size_t)m;
    TRY(comm_allgather(c, ct, g, sizeof(double) * K1 * (size_t)m));
    k_gk_ranks<<<grid_for((int64_t)K1 * m), 256, 0, c->stream>>>(g, P.R, P.rank, (int64_t)K1 * m, carry, tot);
    KCHECK();
    ct = tot;
  }
  PROF_END(c, PC_GRAD_CARRY, 3);
  const double* cl = P.cx + P.row0;
  if (obj) {
    TRY((gk_main_launch<K, MODE, false, true, false>(c, grid, S2, nl, m, xl, P.yc, rp, rt, Z, ct, cl, P.cy, 1.0,
                                                     nullptr, nullptr, nullptr, 0, tob, carry)));
    // realised marginals: a = T 1 (row totals, power 0; this rank's rows), b = T^T 1 (column
    // totals of the plan over every rank: gathered and summed in rank order)
    TRY(gk_scan_tiles(c, cp, ntr, (int64_t)K1 * m, ctt));
    double *part, *gpart, *bg;
    TRY(ws(c, c->xpart, (size_t)(2 * K + 2) * (P.R + 1), &part));
    gpart = part + (2 * K + 2);
    k_gk_obj_partial<K><<<1, 1024, 0, c->stream>>>(rt, xl, nl, tob, (int64_t)ntc * ntr, part);
    KCHECK();
    TRY(comm_allgather(c, part, gpart, sizeof(double) * (2 * K + 2)));
    if (P.R > 1) {
      TRY(ws(c, c->xg2, (size_t)m * P.R, &bg));
      TRY(comm_allgather(c, ctt, bg, sizeof(double) * (size_t)m));  // power-0 row of ctt
    } else {
      bg = ctt;
    }
    k_gk_obj_final<K><<<1, 1024, 0, c->stream>>>(gpart, P.R, bg, P.yc, m, objout_dev);
    KCHECK();
  }
  if (store) {
    PROF_BEGIN(c, PC_GRAD_MAIN);
    if (fx)
      TRY((gk_main_launch<K, MODE, true, false, true>(c, grid, S2, nl, m, xl, P.yc, rp, rt, Z, ct, cl, P.cy, alpha,
                                                      fx + P.row0, fy, G, ldG, nullptr, carry)));
    else
      TRY((gk_main_launch<K, MODE, true, false, false>(c, grid, S2, nl, m, xl, P.yc, rp, rt, Z, ct, cl, P.cy, alpha,
                                                       nullptr, nullptr, G, ldG, nullptr, carry)));
    PROF_END(c, PC_GRAD_MAIN, 1);
  }
  return GW_OK;
}

template <int K>
static gw_status grad_pass_gk(gw_ctx* c, const Prepared& P, int mode, const TSrc2& S2, float* G, int64_t ldG,
                              bool store, bool obj, const double* fx, const double* fy, double alpha,
                              double* objout_dev) {
  if (mode == T_EXPLICIT)
    return grad_pass_gk_mode<K, T_EXPLICIT>(c, P, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
  if (mode == T_GIBBS) return grad_pass_gk_mode<K, T_GIBBS>(c, P, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
  return grad_pass_gk_mode<K, T_PRODUCT>(c, P, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
}

// k = 4 gradient (store only): the k = 2 moments pass (M_rt, r, t <= 4) + a degree-4 polynomial per row
// evaluated in fp64 (poly.cuh) -- 4NM read + 4NM write, no scans (the objective stays on polyk.cuh)
static gw_status grad_store_poly4(gw_ctx* c, const Prepared& P, int mode, const TSrc2& S2, float* G, int64_t ldG,
                                  const double* fx, const double* fy, double alpha) {
  const int64_t nl = P.nl, m = P.m;
  if (nl == 0) return GW_OK;
  double* M;
  PROF_BEGIN(c, PC_GRAD_MOMENTS);
  TRY(poly_moments(c, P, mode, S2, false, &M));
  PROF_END(c, PC_GRAD_MOMENTS, 1);
  PROF_BEGIN(c, PC_GRAD_MAIN);
  double *coef, *c2d;
  float *fxs = nullptr, *fys = nullptr;
  TRY(ws(c, c->p4coef, 5 * (size_t)std::max<int64_t>(nl, 1), &coef));
  TRY(ws(c, c->p4c2, (size_t)m, &c2d));
  k_poly4_rowcoef<<<grid_for(nl), 256, 0, c->stream>>>(M, P.xc + P.row0, P.cx + P.row0, nl, alpha, coef);
  KCHECK();
  k_scale<<<grid_for(m), 256, 0, c->stream>>>(P.cy, m, 2.0 * alpha, c2d);
  KCHECK();
  const dim3 grid((unsigned)((m + 1023) / 1024), (unsigned)((nl + PSR - 1) / PSR));
  if (fx) {
    TRY(ws(c, c->pfx, std::max<int64_t>(nl, 1), &fxs));
    TRY(ws(c, c->pfy, m, &fys));
    k_scale_f<<<grid_for(nl), 256, 0, c->stream>>>(fx + P.row0, nl, sqrt(1.0 - alpha), fxs);
    k_scale_f<<<grid_for(m), 256, 0, c->stream>>>(fy, m, sqrt(1.0 - alpha), fys);
    KCHECK();
    k_poly4_store<true><<<grid, 256, 0, c->stream>>>(coef, c2d, P.yc, fxs, fys, nl, m, G, ldG);
  } else {
    k_poly4_store<false><<<grid, 256, 0, c->stream>>>(coef, c2d, P.yc, nullptr, nullptr, nl, m, G, ldG);
  }
  KCHECK();
  PROF_END(c, PC_GRAD_MAIN, 1);
  return GW_OK;
}

static gw_status grad_pass(gw_ctx* c, const Prepared& P, int mode, const TSrc& S, const TSrc2& S2, float* G,
                           int64_t ldG, bool store, bool obj, const double* fx, const double* fy, double alpha,
                           double* objout_dev, double beta = 0.0, const gw_moments* mom = nullptr) {
  NvtxRange nv(obj && !store ? "gw.objective" : "gw.grad");
  if (beta != 0.0 && (P.grid2d || P.k != 1 || obj || !store))
    return fail(GW_ERR_UNSUPPORTED, "tau != eps: only the k = 1 1-D gradient store carries the (eps - tau) ln T term");
  if (beta != 0.0) return grad_pass_k1(c, P, mode, S, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev, beta);
  if (P.grid2d) return grad_pass_2d(c, P, mode, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
  if (P.k == 1) return grad_pass_k1(c, P, mode, S, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev, 0.0, mom);
  if (P.k == 4 && store && !obj) return grad_store_poly4(c, P, mode, S2, G, ldG, fx, fy, alpha);
  if (P.k >= 3) {
    if (P.nl == 0) return GW_OK;
    if (obj)  // violation, entropy and <C o C, T> from the k = 1 objective machinery; E(T) below
      TRY(grad_pass_k1(c, P, mode, S, S2, nullptr, 0, false, true, fx, fy, alpha, objout_dev));
    switch (P.k) {
      case 3: return grad_pass_gk<3>(c, P, mode, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
      case 4: return grad_pass_gk<4>(c, P, mode, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
      default: return grad_pass_gk<5>(c, P, mode, S2, G, ldG, store, obj, fx, fy, alpha, objout_dev);
    }
  }
  const int64_t nl = P.nl, m = P.m;
  if (obj) {
    // violation, entropy and <C o C, T> do not depend on k: the k = 1 objective machinery supplies
    // them; E(T) at k = 2 comes from the plan's moments.  Runs before the store: on the solver
    // path the plan is regenerated from the cost that the store overwrites.
    TRY(grad_pass_k1(c, P, mode, S, S2, nullptr, 0, false, true, fx, fy, alpha, objout_dev));
    double* M;
    TRY(poly_moments(c, P, mode, S2, true, &M));
    k_poly_objective<<<1, 32, 0, c->stream>>>(M, objout_dev);
    KCHECK();
  }
  if (store) {
    double* M;
    PROF_BEGIN(c, PC_GRAD_MOMENTS);
    TRY(poly_moments(c, P, mode, S2, false, &M));
    PROF_END(c, PC_GRAD_MOMENTS, 1);
    PROF_BEGIN(c, PC_GRAD_MAIN);
    float4* coef;
    float *c2s, *fxs = nullptr, *fys = nullptr;
    TRY(ws(c, c->pcoef, std::max<int64_t>(nl, 1), &coef));
    TRY(ws(c, c->pc2s, m, &c2s));
    k_poly_rowcoef<<<grid_for(nl), 256, 0, c->stream>>>(M, P.xc + P.row0, P.cx + P.row0, nl, alpha, coef);
    KCHECK();
    k_scale_f<<<grid_for(m), 256, 0, c->stream>>>(P.cy, m, 2.0 * alpha, c2s);
    KCHECK();
    if (fx) {
      TRY(ws(c, c->pfx, std::max<int64_t>(nl, 1), &fxs));
      TRY(ws(c, c->pfy, m, &fys));
      k_scale_f<<<grid_for(nl), 256, 0, c->stream>>>(fx + P.row0, nl, sqrt(1.0 - alpha), fxs);
      k_scale_f<<<grid_for(m), 256, 0, c->stream>>>(fy, m, sqrt(1.0 - alpha), fys);
      KCHECK();
      k_poly_store<true><<<dim3((unsigned)((m + 1023) / 1024), (unsigned)((nl + PSR - 1) / PSR)), 256, 0, c->stream>>>(
          coef, c2s, P.yf, fxs, fys, nl, m, G, ldG);
    } else {
      k_poly_store<false><<<dim3((unsigned)((m + 1023) / 1024), (unsigned)((nl + PSR - 1) / PSR)), 256, 0, c->stream>>>(
          coef, c2s, P.yf, nullptr, nullptr, nl, m, G, ldG);
    }
    KCHECK();
    PROF_END(c, PC_GRAD_MAIN, 1);
  }
  return GW_OK;
}

// ------------------------------------------------------------------------------ fp64 storage (GW_F64)
// f64.cuh: the same gradient and Sinkhorn steps with float64 matrices (C1 = configs[0]).  Multi-rank:
// the column prefixes / totals and the column LSE pairs are all-gathered and combined in rank order
// (as shard.cuh does for the fp32 path), so one and several ranks agree up to summation order.

// G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y (alpha, fx, fy: the FGW cost, Remark 2) for this rank's rows,
// distance power K (f64.cuh).  G may alias T unless obj.  obj: objout (device, 8 doubles) =
// {E, violation, -, H, -, -, sum T C^2, -} of the plan T (over all ranks).  mom (nullable, K = 1):
// supplied totals (gw_moments).
template <int K>
static gw_status grad64_k(gw_ctx* c, const Prepared& P, const double* T, int64_t ldT, double* G, int64_t ldG, bool obj,
                          const double* fx, const double* fy, double alpha, const gw_moments* mom, double* objout) {
  constexpr int NS = K + 1;
  const int64_t nl = P.nl, m = P.m;
  const int R = P.R;
  if (nl == 0) return GW_OK;  // single rank only: prepare() rejects empty shards when R > 1
  const int64_t nb = (nl + F64_RB - 1) / F64_RB;
  if (nb > 65535) return fail(GW_ERR_UNSUPPORTED, "GW_F64: at most %lld rows per rank", (long long)65535 * F64_RB);
  double *rtot, *part, *tot, *gath;
  TRY(ws(c, c->d64rt, (size_t)(NS + 2) * nl, &rtot));
  TRY(ws(c, c->d64part, (size_t)nb * NS * m, &part));
  TRY(ws(c, c->d64tot, 3 * (size_t)NS * m, &tot));
  TRY(ws(c, c->d64gath, (size_t)R * NS * m, &gath));
  double* rin = rtot + NS * nl;
  double* off = tot + NS * m;
  double* glob = tot + 2 * NS * m;
  const double* xl = P.xc + P.row0;
  NvtxRange nv("gw.grad64");
  PROF_BEGIN(c, PC_GRAD_MAIN);
  if (K == 1 && mom) {
    k64_momrows<<<grid_for(nl), 256, 0, c->stream>>>(mom->row_sum, mom->row_ysum, P.yend_u - P.ylast, nl, rin);
    KCHECK();
  }
  // a2: B' = (T D_Y)' into G (odd K) and the row power sums (one warp per row)
  k64_row<K><<<(unsigned)((nl * 32 + 255) / 256), 256, 0, c->stream>>>(T, ldT, nl, m, P.yc,
                                                                        (K == 1 && mom) ? rin : nullptr, G, ldG, rtot);
  KCHECK();
  // a3: column block power sums of B, their exclusive prefix, the ranks' offsets and totals
  const dim3 cg((unsigned)((m + 127) / 128), (unsigned)nb);
  k64_colpart<K><<<cg, 128, 0, c->stream>>>(G, ldG, nl, m, xl, P.yc, rtot, part);
  KCHECK();
  k64_colscan<NS><<<(unsigned)((m + 127) / 128), 128, 0, c->stream>>>(part, (int)nb, m, tot);
  KCHECK();
  TRY(comm_allgather(c, tot, gath, (size_t)NS * m * sizeof(double)));
  if (K == 1 && mom) {  // column totals of B = T D_Y from the supplied T^T 1, T^T x by 1-D DPs over y
    double* v;
    TRY(ws(c, c->d64mc, 2 * (size_t)m, &v));
    k64_momcols<<<grid_for(m), 256, 0, c->stream>>>(mom->col_sum, mom->col_xsum, P.xend_u - P.xlast, m, v);
    KCHECK();
    Scan1DBatch B;
    memset(&B, 0, sizeof(B));
    B.d[0] = Scan1D{v, P.yc, m, nullptr, glob, nullptr};
    B.d[1] = Scan1D{v + m, P.yc, m, nullptr, glob + m, nullptr};
    const int KS = (int)std::min<int64_t>(SCAN_KMAX, std::max<int64_t>(1, (m + 4095) / 4096));
    double* wt;
    TRY(ws(c, c->scanwt, (size_t)4 * KS * 32 * 3, &wt));
    k_scan1d_tot<<<dim3(KS, 2), 1024, 0, c->stream>>>(B, KS, wt);
    KCHECK();
    k_scan1d_out<<<dim3(KS, 2), 1024, 0, c->stream>>>(B, KS, wt);
    KCHECK();
  }
  k64_rankoff<<<(unsigned)((NS * m + 255) / 256), 256, 0, c->stream>>>(gath, R, P.rank, NS * m, off, glob,
                                                                       K == 1 && mom != nullptr);
  KCHECK();
  // a3 + a4: D_X B by the column scan, assembled into G in place
  double* ob = nullptr;
  if (obj) TRY(ws(c, c->d64obj, (size_t)nb * 4 * m, &ob));
  const double* fxl = fx ? fx + P.row0 : nullptr;
#define K64_APPLY(O, F)                                                                                           \
  k64_colapply<K, O, F><<<cg, 128, 0, c->stream>>>(G, ldG, T, ldT, nl, m, xl, part, off, glob, P.cx + P.row0, P.cy, \
                                                    fxl, fy, alpha, P.yc, rtot, ob)
  if (obj) {
    if (fx) K64_APPLY(true, true); else K64_APPLY(true, false);
  } else {
    if (fx) K64_APPLY(false, true); else K64_APPLY(false, false);
  }
#undef K64_APPLY
  KCHECK();
  PROF_END(c, PC_GRAD_MAIN, 5);
  if (obj) {  // a8: E(T), violation, H, sum T C^2
    double *tmp, *pay, *pg;
    const int64_t st = m + F64_PAYS;
    TRY(ws(c, c->d64tmp, 3 * (size_t)m, &tmp));
    TRY(ws(c, c->d64pay, (size_t)st, &pay));
    TRY(ws(c, c->d64pg, (size_t)R * st, &pg));
    k64_objcols<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(ob, (int)nb, m, pay, tmp);
    KCHECK();
    k64_objlocal<K><<<1, 1024, 0, c->stream>>>(tmp, m, rtot, xl, P.pn + P.row0, nl, pay);
    KCHECK();
    TRY(comm_allgather(c, pay, pg, (size_t)st * sizeof(double)));
    k64_objglobal<K><<<1, 1024, 0, c->stream>>>(pg, R, m, P.yc, P.qn, objout);
    KCHECK();
  }
  return GW_OK;
}

static gw_status grad64(gw_ctx* c, const Prepared& P, const double* T, int64_t ldT, double* G, int64_t ldG, bool obj,
                        const double* fx, const double* fy, double alpha, const gw_moments* mom, double* objout) {
  switch (P.k) {
    case 1: return grad64_k<1>(c, P, T, ldT, G, ldG, obj, fx, fy, alpha, mom, objout);
    case 2: return grad64_k<2>(c, P, T, ldT, G, ldG, obj, fx, fy, alpha, mom, objout);
    case 3: return grad64_k<3>(c, P, T, ldT, G, ldG, obj, fx, fy, alpha, mom, objout);
    case 4: return grad64_k<4>(c, P, T, ldT, G, ldG, obj, fx, fy, alpha, mom, objout);
    case 5: return grad64_k<5>(c, P, T, ldT, G, ldG, obj, fx, fy, alpha, mom, objout);
    default: return fail(GW_ERR_UNSUPPORTED, "GW_F64: distance power k = %d", P.k);
  }
}

// fp64 Sinkhorn state: the column exchange payload {max[m], sum[m], row deviation, pad} per rank.
struct Sink64 {
  double *pay, *gath, *rdev, *cdev, *vout;
  double2* part;
  int64_t stride = 0, nb = 0;
  cudaGraphExec_t gexec = nullptr;  // fixed-count loops: `gchunk` iterations captured once per solve
  int gchunk = 0;
  ~Sink64() {
    if (gexec) cudaGraphExecDestroy(gexec);
  }
};
static gw_status sink64_alloc(gw_ctx* c, const Prepared& P, Sink64& s) {
  s.stride = 2 * P.m + 2;
  s.nb = (std::max<int64_t>(P.nl, 1) + F64_RB - 1) / F64_RB;
  if (s.nb > 65535) return fail(GW_ERR_UNSUPPORTED, "GW_F64: at most %lld rows per rank", (long long)65535 * F64_RB);
  TRY(ws(c, c->s64pay, (size_t)s.stride + 2, &s.pay));
  s.vout = s.pay + s.stride;
  TRY(ws(c, c->s64gath, (size_t)P.R * s.stride, &s.gath));
  TRY(ws(c, c->s64part, (size_t)s.nb * P.m, &s.part));
  TRY(ws(c, c->s64rdev, (size_t)std::max<int64_t>(P.nl, 1), &s.rdev));
  TRY(ws(c, c->s64cdev, (size_t)P.m, &s.cdev));
  return GW_OK;
}
// column LSE pairs of (f_i + g_p - G_ip)/eps over this rank's rows, all-gathered (g nullable: 0)
static gw_status sink64_cols(gw_ctx* c, const Prepared& P, Sink64& s, const double* G, int64_t ldG, const double* f,
                             const double* g, double eps) {
  const int64_t m = P.m;
  k64_colpart_lse<<<dim3((unsigned)((m + 127) / 128), (unsigned)s.nb), 128, 0, c->stream>>>(G, ldG, P.nl, m, f, g,
                                                                                          eps, s.part);
  KCHECK();
  k64_colcomb<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>(s.part, (int)s.nb, m, s.pay);
  KCHECK();
  TRY(comm_allgather(c, s.pay, s.gath, (size_t)s.stride * sizeof(double)));
  return GW_OK;
}
// one iteration: f-update (a5) then g-update (a6), reading R7
static gw_status sink64_iter(gw_ctx* c, const Prepared& P, Sink64& s, const double* G, int64_t ldG, double* f,
                             double* g, double eps) {
  const int64_t nl = P.nl, m = P.m;
  k64_rowlse<<<(unsigned)((nl * 32 + 255) / 256), 256, 0, c->stream>>>(G, ldG, nl, m, g, eps, f, P.lp + P.row0,
                                                                       P.pn + P.row0, 0, nullptr);
  KCHECK();
  TRY(sink64_cols(c, P, s, G, ldG, f, nullptr, eps));
  k64_colfinal<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(s.gath, P.R, s.stride, m, eps, P.lq, P.qn, g, 0,
                                                                   nullptr);
  KCHECK();
  return GW_OK;
}
// violation max(|T1 - p|, |T^T 1 - q|) of the plan (f, g) into s.vout (device); host != null: read back
static gw_status sink64_viol(gw_ctx* c, const Prepared& P, Sink64& s, const double* G, int64_t ldG, const double* f,
                             const double* g, double eps, double* host) {
  const int64_t nl = P.nl, m = P.m;
  k64_rowlse<<<(unsigned)((nl * 32 + 255) / 256), 256, 0, c->stream>>>(G, ldG, nl, m, g, eps, const_cast<double*>(f),
                                                                       nullptr, P.pn + P.row0, 1, s.rdev);
  KCHECK();
  k64_max<<<1, 1024, 0, c->stream>>>(s.rdev, nl, s.pay + 2 * m);
  KCHECK();
  TRY(sink64_cols(c, P, s, G, ldG, f, g, eps));
  k64_colfinal<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(s.gath, P.R, s.stride, m, eps, P.lq, P.qn, nullptr,
                                                                   1, s.cdev);
  KCHECK();
  k64_viol<<<1, 1024, 0, c->stream>>>(s.cdev, m, s.gath, P.R, s.stride, s.vout);
  KCHECK();
  if (host) {
    CU(cudaMemcpyAsync(c->hpin + 56, s.vout, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *host = c->hpin[56];
  }
  return GW_OK;
}
// Cluster size for the cluster-resident fp64 Sinkhorn (f64.cuh k64_sink_small): G's rows in one cluster's
// shared memory, >= 16 rows per CTA where the rows allow (up to 16 CTAs); 0 if it does not fit.
static int small64_cluster(const Prepared& P, int* rows_out, size_t* bytes_out) {
  if (P.nl <= 0 || P.m <= 0) return 0;
  int want = 1;
  while (want < 16 && P.nl >= 16 * 2 * (int64_t)want) want *= 2;
  for (int CL : {1, 2, 4, 8, 16}) {
    if (CL < want) continue;
    const int64_t rows = (P.nl + CL - 1) / CL;
    const size_t bytes = small64_smem_bytes((int)std::min<int64_t>(rows, 1 << 20), P.m);
    if (rows > (1 << 20) || bytes > 220 * 1024) continue;
    if (CL > 1 && rows * (CL - 1) >= P.nl) continue;  // every CTA holds at least one row
    static std::atomic<int> ok[32];  // occupancy verdict per CL (0 = unknown, 1 = fits, -1 = does not)
    cudaFuncSetAttribute(k64_sink_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (CL > 8) cudaFuncSetAttribute(k64_sink_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (ok[CL].load() == 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(SNT);
      cfg.dynamicSmemBytes = 220 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      const cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k64_sink_small, &cfg);
      ok[CL].store((e == cudaSuccess && ncl >= 1) ? 1 : -1);
      cudaGetLastError();
    }
    if (ok[CL].load() < 0) continue;
    *rows_out = (int)rows;
    *bytes_out = bytes;
    return CL;
  }
  return 0;
}

// `iters` iterations; tol > 0: the plan's violation checked every check_every iterations, stop when
// <= tol (reading R8; the oracle's schedule exactly)
static gw_status sink64_run(gw_ctx* c, const Prepared& P, Sink64& s, const double* G, int64_t ldG, double* f,
                            double* g, double eps, int iters, double tol, int check_every, int* used, int* conv,
                            bool graph_ok = false) {
  NvtxRange nv("gw.sinkhorn64");
  *used = 0;
  *conv = 0;
  if (check_every < 1) check_every = 10;
  // Fixed-count loop on one rank with G small enough for one cluster's shared memory: every iteration in
  // ONE launch (k64_sink_small; GWDP_NO_SMALL=1 disables it)
  if (tol <= 0 && iters > 0 && P.R == 1 && getenv("GWDP_NO_SMALL") == nullptr) {
    int rows = 0;
    size_t bytes = 0;
    const int CL = small64_cluster(P, &rows, &bytes);
    if (CL > 0) {
      Small64Args sa{G, ldG, P.nl, P.m, rows, P.lp + P.row0, P.lq, eps, iters, f, g};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(SNT);
      cfg.dynamicSmemBytes = bytes;
      cfg.stream = c->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PROF_BEGIN(c, PC_SINK_ROW);
      CU(cudaLaunchKernelEx(&cfg, k64_sink_small, sa));
      KCHECK();
      PROF_END(c, PC_SINK_ROW, 1);
      *used = iters;
      return GW_OK;
    }
  }
  // Fixed-count loop inside a solve (the same G, f, g, eps every outer iteration): up to 100 iterations
  // captured once as a CUDA graph and replayed (C1's 256 x 256 iterations are launch bound: 4 kernels
  // each).  Host-transport all-gathers are not capturable.
  static const bool no_graph = getenv("GWDP_NO_GRAPH") != nullptr;
  if (graph_ok && tol <= 0 && iters > 0 && !no_graph && !c->prof.on &&
      (P.R == 1 || (c->comm && c->comm->nccl))) {
    const int chunk = std::min(iters, 100);
    if (!s.gexec || s.gchunk != chunk) {
      if (s.gexec) cudaGraphExecDestroy(s.gexec);
      s.gexec = nullptr;
      if (!c->cap) CU(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
      CU(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
      cudaStream_t saved = c->stream;
      c->stream = c->cap;
      gw_status st = GW_OK;
      for (int k = 0; k < chunk && st == GW_OK; ++k) st = sink64_iter(c, P, s, G, ldG, f, g, eps);
      c->stream = saved;
      cudaGraph_t gr = nullptr;
      const cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
      if (st != GW_OK) {
        if (gr) cudaGraphDestroy(gr);
        return st;
      }
      if (e != cudaSuccess) return fail(GW_ERR_CUDA, "fp64 Sinkhorn graph capture: %s", cudaGetErrorString(e));
      const cudaError_t ei = cudaGraphInstantiate(&s.gexec, gr, 0);
      cudaGraphDestroy(gr);
      if (ei != cudaSuccess) return fail(GW_ERR_CUDA, "fp64 Sinkhorn graph instantiate: %s", cudaGetErrorString(ei));
      s.gchunk = chunk;
    }
    int done = 0;
    for (; done + s.gchunk <= iters; done += s.gchunk) CU(cudaGraphLaunch(s.gexec, c->stream));
    for (; done < iters; ++done) TRY(sink64_iter(c, P, s, G, ldG, f, g, eps));
    *used = iters;
    return GW_OK;
  }
  for (int it = 1; it <= iters; ++it) {
    PROF_BEGIN(c, PC_SINK_ROW);
    TRY(sink64_iter(c, P, s, G, ldG, f, g, eps));
    PROF_END(c, PC_SINK_ROW, 4);
    *used = it;
    if (tol > 0 && it % check_every == 0) {
      double v = 0.0;
      TRY(sink64_viol(c, P, s, G, ldG, f, g, eps, &v));
      if (v <= tol) {
        *conv = 1;
        break;
      }
    }
  }
  return GW_OK;
}

extern "C" gw_status gw_grad_dp(gw_ctx* c, const gw_problem* pb, const void* T, int64_t ldT, void* G, int64_t ldG,
                                const gw_moments* mom) {
  if (!c) return fail(GW_ERR_INVALID_ARG, "null ctx");
  TRY(check_problem(pb));
  if (mom) {
    if (!mom->row_sum || !mom->row_ysum || !mom->col_sum || !mom->col_xsum)
      return fail(GW_ERR_INVALID_ARG, "gw_grad_dp: gw_moments needs all four vectors");
    if (pb->k != 1 || (pb->flags & GW_GRID2D))
      return fail(GW_ERR_UNSUPPORTED, "gw_grad_dp: precomputed moments are used by the k = 1 1-D gradient only");
  }
  TRY(check_matrix(T, ldT, pb->m, "T"));
  TRY(check_matrix(G, ldG, pb->m, "G"));
  CU(cudaSetDevice(c->device));
  Prepared P;
  TRY(prepare(c, pb, P));
  if (pb->dtype == GW_F64)
    return grad64(c, P, reinterpret_cast<const double*>(T), ldT, reinterpret_cast<double*>(G), ldG, false, nullptr,
                  nullptr, 1.0, mom, nullptr);
  TSrc S{reinterpret_cast<const float*>(T), ldT, nullptr, nullptr, 0.0};
  TSrc2 S2{reinterpret_cast<const float*>(T), ldT, nullptr, nullptr, nullptr, nullptr, 0.f, 0.f};
  TRY(grad_pass(c, P, T_EXPLICIT, S, S2, reinterpret_cast<float*>(G), ldG, true, false, nullptr, nullptr, 1.0,
                nullptr, 0.0, mom));
  return GW_OK;
}

// ------------------------------------------------------------------------------ Sinkhorn
struct SinkState {
  double *f, *g;     // fp64 duals (device)
  float *fh, *fl, *gh, *gl;
  double* ftmp;
  float* viol;
  int *stop, *iters;
  float2* part;
  int nrb;
  int64_t RB;
  // fused fast path
  int* mode;      // [0] = path of the current iteration (1 = fused), [1] = fused iterations run,
                  // [2] = dev (float), [5] / [6] = committed / target updates (multi-rank fixed-count loop)
  float* dev;     // max |log2(colsum/q)| of the last column half-step
  double* fpart;  // [ncl][m]
  float* Srow;    // [nl]
  float* pf;      // [nl] p as fp32
  int fK = 0, fCL = 0, fNT = 256, fncl = 0;  // fK == 0: fast path unavailable for this shape
  int64_t fW = 0;                            // columns per CTA
  int64_t frpc = 0;
  // column-sum exchange: this rank's column LSE pairs / column sums, and all ranks' (gathered)
  double *lse, *lseg, *csl, *csg;
  double *un = nullptr, *ung = nullptr;  // multi-rank fixed-count loop: payload (M + 1) and gathered
  float* violg;
  int *flag, *flagg;  // speculation validity flag (and the ranks' flags)
  cudaGraphExec_t gexec = nullptr;  // one fixed-count iteration, captured once per solve
  double g_eps = 0.0, g_kappa = 0.0;  // the scalars baked into gexec (UGW changes them per outer iteration)
  // 8 N M solver gradient (rowclu.cuh): the last sweep of an inner loop runs the XM instantiation over
  // rcncl clusters of rcCL CTAs (4096 columns each, rcrpc rows per cluster), the same partition as the
  // gradient's main pass; rcCL == 0: unavailable for this problem
  int rcCL = 0, rcncl = 0;
  int64_t rcrpc = 0;
  double *rcpart = nullptr, *rcpartx = nullptr;
  float *xf = nullptr, *ccx = nullptr, *ccy = nullptr, *dxf = nullptr;
  int* xmv = nullptr;               // set on the device when the XM sweep ran and was committed
  cudaGraphExec_t gexec_xm = nullptr;  // the same iteration with the XM sweep
};

static void sink_free(SinkState& s) {
  if (s.gexec) cudaGraphExecDestroy(s.gexec);
  if (s.gexec_xm) cudaGraphExecDestroy(s.gexec_xm);
  s.gexec = s.gexec_xm = nullptr;
}
// CUDA events owned by one call, destroyed on every exit path (errors included)
struct EventSet {
  std::vector<cudaEvent_t> v;
  ~EventSet() {
    for (auto e : v)
      if (e) cudaEventDestroy(e);
  }
  cudaError_t make(cudaEvent_t* out) {
    cudaEvent_t e = nullptr;
    const cudaError_t r = cudaEventCreate(&e);
    if (r == cudaSuccess) v.push_back(e);
    *out = e;
    return r;
  }
};
struct SinkGuard {  // releases the captured graph on every exit path of a solve
  SinkState& s;
  ~SinkGuard() { sink_free(s); }
};

template <int K, int CL, int NT>
static gw_status fused_config_t(gw_ctx* c, int* ncl) {
  auto kern = k_sink_fused2<K, CL, NT, false>;
  const size_t dsm = fused_dyn_smem<K, NT>();
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  CU(cudaFuncSetAttribute(k_sink_fused2<K, CL, NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = dsm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU(cudaOccupancyMaxActiveClusters(ncl, (void*)kern, &cfg));
  return GW_OK;
}

template <int K, int CL, int NT>
static gw_status fused_launch_t(gw_ctx* c, const FusedArgs& fa, int ncl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = fused_dyn_smem<K, NT>();
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (fa.kappa != 1.f) CU(cudaLaunchKernelEx(&cfg, k_sink_fused2<K, CL, NT, true>, fa));
  else CU(cudaLaunchKernelEx(&cfg, k_sink_fused2<K, CL, NT, false>, fa));
  return GW_OK;
}

// (K, CL, NT) dispatch: W = 4 K NT columns per CTA (W <= 8192); one cluster of CL CTAs spans a row.
//   NT = 256: K in {1, 2, 4, 8} with CL = 1, K = 8 with CL in {2, 4, 8}, K = 6 with CL in {4, 8}
//   NT = 512: K in {1, 2, 4} with CL = 1, K = 4 with CL in {2, 4, 8}
#define FUSED_DISPATCH(FN, ...)                                                   \
  switch ((NT / 256) * 256 + K * 16 + CL) {                                       \
    case 256 + 1 * 16 + 1: return FN<1, 1, 256>(__VA_ARGS__);                     \
    case 256 + 2 * 16 + 1: return FN<2, 1, 256>(__VA_ARGS__);                     \
    case 256 + 4 * 16 + 1: return FN<4, 1, 256>(__VA_ARGS__);                     \
    case 256 + 8 * 16 + 1: return FN<8, 1, 256>(__VA_ARGS__);                     \
    case 256 + 8 * 16 + 2: return FN<8, 2, 256>(__VA_ARGS__);                     \
    case 256 + 8 * 16 + 4: return FN<8, 4, 256>(__VA_ARGS__);                     \
    case 256 + 8 * 16 + 8: return FN<8, 8, 256>(__VA_ARGS__);                     \
    case 256 + 6 * 16 + 4: return FN<6, 4, 256>(__VA_ARGS__);                     \
    case 256 + 6 * 16 + 8: return FN<6, 8, 256>(__VA_ARGS__);                     \
    case 512 + 1 * 16 + 1: return FN<1, 1, 512>(__VA_ARGS__);                     \
    case 512 + 2 * 16 + 1: return FN<2, 1, 512>(__VA_ARGS__);                     \
    case 512 + 4 * 16 + 1: return FN<4, 1, 512>(__VA_ARGS__);                     \
    case 512 + 4 * 16 + 2: return FN<4, 2, 512>(__VA_ARGS__);                     \
    case 512 + 4 * 16 + 4: return FN<4, 4, 512>(__VA_ARGS__);                     \
    case 512 + 4 * 16 + 8: return FN<4, 8, 512>(__VA_ARGS__);                     \
    default: return fail(GW_ERR_UNSUPPORTED, "fused path: no instance K=%d CL=%d NT=%d", K, CL, NT); \
  }
static gw_status fused_config(gw_ctx* c, int K, int CL, int NT, int* ncl) { FUSED_DISPATCH(fused_config_t, c, ncl) }
static gw_status fused_launch(gw_ctx* c, int K, int CL, int NT, const FusedArgs& fa, int ncl) {
  FUSED_DISPATCH(fused_launch_t, c, fa, ncl)
}

// XM instantiation (K = 4, NT = 256: 4096 columns per CTA) and the gradient main pass, CL in {1,...,16}
template <int CL>
static gw_status rc_config_t(gw_ctx* c, int* ncl) {
  auto kx = k_sink_fused2<4, CL, 256, false, true>;
  auto kg = k_grad_rc<CL>;
  const size_t dx = fused_dyn_smem<4, 256, true>(), dg = rc_dyn_smem();
  CU(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dx));
  CU(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dg));
  if (CL > 8) {
    CU(cudaFuncSetAttribute(kx, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CU(cudaFuncSetAttribute(kg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 * CL);
  cfg.blockDim = dim3(256);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nx = 0, ng = 0;
  cfg.dynamicSmemBytes = dx;
  CU(cudaOccupancyMaxActiveClusters(&nx, (void*)kx, &cfg));
  cfg.dynamicSmemBytes = dg;
  CU(cudaOccupancyMaxActiveClusters(&ng, (void*)kg, &cfg));
  *ncl = std::min(nx, ng);
  return GW_OK;
}
template <int CL>
static gw_status rc_xm_launch_t(gw_ctx* c, const FusedArgs& fa, int ncl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * CL);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = fused_dyn_smem<4, 256, true>();
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU(cudaLaunchKernelEx(&cfg, k_sink_fused2<4, CL, 256, false, true>, fa));
  return GW_OK;
}
template <int CL>
static gw_status rc_grad_launch_t(gw_ctx* c, const CUtensorMap& tm, const RcArgs& ra, int ncl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * CL);
  cfg.blockDim = dim3(RC_NT);
  cfg.dynamicSmemBytes = rc_dyn_smem();
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CU(cudaLaunchKernelEx(&cfg, k_grad_rc<CL>, tm, ra));
  return GW_OK;
}
#define RC_DISPATCH(FN, CL, ...)                                                        \
  switch (CL) {                                                                         \
    case 1: return FN<1>(__VA_ARGS__);                                                  \
    case 2: return FN<2>(__VA_ARGS__);                                                  \
    case 4: return FN<4>(__VA_ARGS__);                                                  \
    case 8: return FN<8>(__VA_ARGS__);                                                  \
    case 16: return FN<16>(__VA_ARGS__);                                                \
    default: return fail(GW_ERR_UNSUPPORTED, "8NM gradient: no instance CL=%d", CL);   \
  }
static gw_status rc_config(gw_ctx* c, int CL, int* ncl) { RC_DISPATCH(rc_config_t, CL, c, ncl) }
static gw_status rc_xm_launch(gw_ctx* c, int CL, const FusedArgs& fa, int ncl) { RC_DISPATCH(rc_xm_launch_t, CL, c, fa, ncl) }
static gw_status rc_grad_launch(gw_ctx* c, int CL, const CUtensorMap& tm, const RcArgs& ra, int ncl) {
  RC_DISPATCH(rc_grad_launch_t, CL, c, tm, ra, ncl)
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// The solver's cost buffer as a 3-D tensor {32, ld / 32, nl} (fp32, 128-B lines) read in boxes of
// {32, 128, 1} = one 4096-column row slice, 128-byte swizzle (rowclu.cuh)
static gw_status rc_tensor_map(gw_ctx* c, const float* G, int64_t ld, int64_t nl, CUtensorMap* tm) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(GW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<EncodeTiledFn>(fn);
  }
  if (ld % 32 != 0 || (reinterpret_cast<uintptr_t>(G) & 15))
    return fail(GW_ERR_INVALID_ARG, "8NM gradient: the cost buffer needs ld %% 32 == 0 and 16-B alignment");
  const cuuint64_t dims[3] = {32, (cuuint64_t)(ld / 32), (cuuint64_t)std::max<int64_t>(nl, 1)};
  const cuuint64_t strides[2] = {128, (cuuint64_t)ld * 4};
  const cuuint32_t box[3] = {32, 128, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(G), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GW_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GW_OK;
}

// XM sweep validity: set when the last iteration ran the XM fused kernel and passed its check (before
// k_sink_fin_fast, which may switch *mode)
__global__ void k_xm_mark(const int* __restrict__ mode, const int* __restrict__ flag, const int* __restrict__ stop,
                          int* __restrict__ xmv) {
  if (threadIdx.x == 0) *xmv = (*mode == 1 && *flag == 0 && !(stop && *stop)) ? 1 : 0;
}

static gw_status sink_alloc(gw_ctx* c, const Prepared& P, SinkState& s) {
  TRY(ws(c, c->fh, P.nl, &s.fh)); TRY(ws(c, c->fl, P.nl, &s.fl));
  TRY(ws(c, c->gh, P.m, &s.gh)); TRY(ws(c, c->gl, P.m, &s.gl));
  TRY(ws(c, c->ftmp, P.nl, &s.ftmp));
  TRY(ws(c, c->viol, 4, &s.viol));
  TRY(ws(c, c->stop, 4, &s.stop));
  TRY(ws(c, c->iters, 4, &s.iters));
  // row blocks of the column half-step: enough CTAs to fill the machine (>= 4 waves)
  const int64_t colblocks = (P.m + 1023) / 1024;
  int64_t want = (148 * 8 + colblocks - 1) / colblocks;
  int64_t RB = (P.nl + want - 1) / std::max<int64_t>(want, 1);
  RB = std::max<int64_t>(16, (RB + 3) & ~int64_t(3));
  s.RB = RB;
  s.nrb = (int)std::max<int64_t>(1, (P.nl + RB - 1) / RB);
  TRY(ws(c, c->part, (size_t)s.nrb * P.m, &s.part));
  TRY(ws(c, c->slse, 2 * (size_t)P.m, &s.lse));
  TRY(ws(c, c->scsl, (size_t)P.m + 1, &s.csl));  // + the row-flag slot (multi-rank)
  TRY(ws(c, c->sflag, 4, &s.flag));
  TRY(ws(c, c->sflagg, (size_t)P.R + 4, &s.flagg));
  if (P.R > 1) {
    TRY(ws(c, c->slseg, 2 * (size_t)P.m * P.R, &s.lseg));
    TRY(ws(c, c->scsg, ((size_t)P.m + 1) * P.R, &s.csg));
    // the fixed-count loop's one payload per iteration: column sums or packed LSE pairs + row flag
    TRY(ws(c, c->sun, (size_t)P.m + 1, &s.un));
    TRY(ws(c, c->sung, ((size_t)P.m + 1) * P.R, &s.ung));
    TRY(ws(c, c->sviolg, (size_t)P.R, &s.violg));
  } else {
    s.lseg = s.lse;
    s.csg = s.csl;
    s.violg = nullptr;
  }
  // fused fast path: cluster of CL CTAs x W = 1024 K columns spans a row
  int* md;
  TRY(ws(c, c->mode, 8, &md));
  s.mode = md;
  s.dev = reinterpret_cast<float*>(md + 2);
  s.fK = 0;
  const char* env = getenv("GWDP_NO_FUSED");
  if (!(env && env[0] == '1') && P.nl > 0) {
    const char* nte = getenv("GWDP_FUSED_NT");
    const int NT = (nte && atoi(nte) == 512) ? 512 : 256;
    const int kmax = 8192 / (4 * NT);  // K at W = 8192 columns per CTA
    int K, CL;
    if (P.m <= 8192) {
      K = (int)((P.m + 4 * NT - 1) / (4 * NT));
      K = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : 8;
      if (K > kmax) K = kmax;
      CL = 1;
    } else {
      K = kmax;
      CL = (int)((P.m + 8191) / 8192);
    }
    if (CL == 3) CL = 4;
    if (CL > 4 && CL < 8) CL = 8;
    // clusters rounded up to 4 or 8 CTAs: narrower CTAs (K = 6, 6144 columns) when they still cover the
    // row, instead of idle CTAs (e.g. M = 24576: 4 x 6144 rather than 3 x 8192 + an empty fourth)
    if (NT == 256 && CL >= 4 && (int64_t)CL * 6 * 1024 >= P.m) K = 6;
    const int64_t wcol = 4 * (int64_t)K * NT;
    if (CL <= 8) {  // clusters must fit in a GPC: on B200 clusters of 8 leave 28 SMs idle
      int ncl = 0;
      TRY(fused_config(c, K, CL, NT, &ncl));
      if (ncl > 0) {
        ncl = (int)std::min<int64_t>(ncl, P.nl);
        s.fK = K; s.fCL = CL; s.fNT = NT; s.fncl = ncl; s.fW = wcol;
        s.frpc = (P.nl + ncl - 1) / ncl;
        TRY(ws(c, c->fpart, (size_t)ncl * P.m, &s.fpart));
        TRY(ws(c, c->srow, (size_t)P.nl, &s.Srow));
        TRY(ws(c, c->pfl, (size_t)P.nl, &s.pf));
        k_to_float<<<grid_for(P.nl), 256, 0, c->stream>>>(P.pn + P.row0, P.nl, s.pf);
        KCHECK();
      }
    }
  }
  // 8 N M solver gradient: one rank, k = 1 on 1-D supports, M <= 16 x 4096 (opt-in while it is slower
  // than the two-read path: GWDP_RC=1 enables it, GWDP_NO_RC=1 disables it)
  s.rcCL = 0;
  const char* nrc = getenv("GWDP_NO_RC");
  const char* yrc = getenv("GWDP_RC");
  if (!(nrc && nrc[0] == '1') && (yrc && yrc[0] == '1') && s.fK > 0 && P.R == 1 && P.k == 1 && !P.grid2d && P.nl > 0 && P.m <= 16 * RC_W) {
    int CL = 1;
    while ((int64_t)CL * RC_W < P.m) CL *= 2;
    int ncl = 0;
    TRY(rc_config(c, CL, &ncl));
    if (ncl > 0) {
      ncl = (int)std::min<int64_t>(ncl, P.nl);
      s.rcCL = CL;
      s.rcncl = ncl;
      s.rcrpc = (P.nl + ncl - 1) / ncl;
      TRY(ws(c, c->rcp, (size_t)ncl * P.m, &s.rcpart));
      TRY(ws(c, c->rcpx, (size_t)ncl * P.m, &s.rcpartx));
      TRY(ws(c, c->rcxf, (size_t)P.nl, &s.xf));
      TRY(ws(c, c->rccx, (size_t)P.nl, &s.ccx));
      TRY(ws(c, c->rccy, (size_t)P.m, &s.ccy));
      TRY(ws(c, c->rcflag, 4, &s.xmv));
      k_to_float<<<grid_for(P.nl), 256, 0, c->stream>>>(P.xc + P.row0, P.nl, s.xf);
      TRY(ws(c, c->rcdx, (size_t)P.nl, &s.dxf));
      k_rc_dx<<<grid_for(P.nl), 256, 0, c->stream>>>(P.xc + P.row0, P.nl, s.dxf);
      k_scale_f<<<grid_for(P.nl), 256, 0, c->stream>>>(P.cx + P.row0, P.nl, 2.0, s.ccx);
      k_scale_f<<<grid_for(P.m), 256, 0, c->stream>>>(P.cy, P.m, 2.0, s.ccy);
      KCHECK();
    }
  }
  return GW_OK;
}

// The gradient on the product plan T^0 = p q^T (k = 1, 1-D supports, GW): the closed form of
// k_grad_product (a = D_X p over all n rows, b = D_Y q by the 1-D programmes), one write of G.
static gw_status grad_product(gw_ctx* c, const Prepared& P, float* G, int64_t ldG) {
  const int64_t n = P.n, m = P.m, nl = P.nl;
  if (nl == 0) return GW_OK;
  double *a, *b;
  TRY(ws(c, c->DP, (size_t)n, &a));
  TRY(ws(c, c->DA, (size_t)m, &b));
  PROF_BEGIN(c, PC_GRAD_CARRY);
  Scan1DBatch B;
  memset(&B, 0, sizeof(B));
  B.d[0] = Scan1D{P.pn, P.xc, n, nullptr, a, nullptr};
  B.d[1] = Scan1D{P.qn, P.yc, m, nullptr, b, nullptr};
  const int K = (int)std::min<int64_t>(SCAN_KMAX, std::max<int64_t>(1, (std::max(n, m) + 4095) / 4096));
  double* wt;
  TRY(ws(c, c->scanwt, (size_t)4 * K * 32 * 3, &wt));
  k_scan1d_tot<<<dim3(K, 2), 1024, 0, c->stream>>>(B, K, wt);
  KCHECK();
  k_scan1d_out<<<dim3(K, 2), 1024, 0, c->stream>>>(B, K, wt);
  KCHECK();
  PROF_END(c, PC_GRAD_CARRY, 2);
  PROF_BEGIN(c, PC_GRAD_MAIN);
  const dim3 grid((unsigned)((m + 1023) / 1024), (unsigned)((nl + 31) / 32));
  k_grad_product<<<grid, 256, 0, c->stream>>>(G, ldG, nl, m, a + P.row0, P.cx + P.row0, b, P.cy);
  KCHECK();
  PROF_END(c, PC_GRAD_MAIN, 1);
  return GW_OK;
}

// The solver's gradient on the 8 N M path (rowclu.cuh), k = 1, one rank: requires that the last
// Sinkhorn iteration ran the XM sweep (s.rcpart / s.rcpartx / s.csl hold its column sums).
static gw_status grad_rc(gw_ctx* c, const Prepared& P, SinkState& s, float* G, int64_t ldG, const TSrc2& S2) {
  const int64_t nl = P.nl, m = P.m;
  const int ncl = s.rcncl;
  double *V, *VX, *U0, *Z0;
  TRY(ws(c, c->rcv, (size_t)ncl * m, &V));
  TRY(ws(c, c->rcvx, (size_t)ncl * m, &VX));
  TRY(ws(c, c->rcu, (size_t)ncl * m, &U0));
  TRY(ws(c, c->rcz, (size_t)ncl * m, &Z0));
  PROF_BEGIN(c, PC_GRAD_ONEPASS);
  k_rc_vec<<<grid_for(m), 256, 0, c->stream>>>(s.rcpart, s.rcpartx, ncl, m, s.csl, P.lq, V, VX);
  KCHECK();
  k_rc_dy<<<2 * ncl, 1024, 0, c->stream>>>(V, VX, ncl, m, P.yc, U0, Z0);
  KCHECK();
  CUtensorMap tm;
  TRY(rc_tensor_map(c, G, ldG, nl, &tm));
  RcArgs ra;
  ra.G = G; ra.ld = ldG; ra.nl = nl; ra.m = m; ra.rows_per_cluster = s.rcrpc;
  ra.fh = S2.fh; ra.fl = S2.fl; ra.gh = S2.gh; ra.gl = S2.gl; ra.ch = S2.ch; ra.cl = S2.cl;
  ra.dxf = s.dxf; ra.xc = P.xc + P.row0; ra.ccx = s.ccx; ra.yf = P.yf; ra.ccy = s.ccy; ra.U0 = U0; ra.Zn0 = Z0;
  TRY(rc_grad_launch(c, s.rcCL, tm, ra, ncl));
  KCHECK();
  PROF_END(c, PC_GRAD_ONEPASS, 1);
  return GW_OK;
}

static gw_status sink_split(gw_ctx* c, const Prepared& P, SinkState& s, double eps) {
  k_split<<<grid_for(P.nl), 256, 0, c->stream>>>(s.f, P.nl, GW_LOG2E / eps, s.fh, s.fl);
  KCHECK();
  k_split<<<grid_for(P.m), 256, 0, c->stream>>>(s.g, P.m, GW_LOG2E / eps, s.gh, s.gl);
  KCHECK();
  return GW_OK;
}

// Violation measured by a row half-step is a per-rank max: make it global (all ranks agree).
static gw_status sink_viol_global(gw_ctx* c, const Prepared& P, SinkState& s) {
  if (P.R == 1) return GW_OK;
  TRY(comm_allgather(c, s.viol, s.violg, sizeof(float)));
  k_max_f<<<1, 32, 0, c->stream>>>(s.violg, P.R, s.viol);
  KCHECK();
  return GW_OK;
}

// Cluster-resident Sinkhorn (small.cuh) for a cost matrix that fits in one cluster's shared
// memory.  The kernel is bound by its per-element fp64 / MUFU work on the cluster's SMs, so the
// cluster is as wide as the rows allow (>= 16 rows per CTA, up to 16 CTAs) once it fits; 0 if none.
static int small_cluster(gw_ctx* c, const Prepared& P, int* rows_out, size_t* bytes_out) {
  if (P.nl <= 0 || P.m <= 0) return 0;
  int want = 1;
  while (want < 16 && P.nl >= 16 * 2 * (int64_t)want) want *= 2;
  for (int CL : {1, 2, 4, 8, 16}) {
    if (CL < want) continue;
    const int64_t rows = (P.nl + CL - 1) / CL;
    if (rows > (1 << 20)) continue;
    const size_t bytes = small_smem_bytes((int)rows, (int)((P.m + 1) & ~int64_t(1)), P.m);
    if (bytes > 220 * 1024) continue;
    if (CL > 1 && rows * (CL - 1) >= P.nl) continue;  // every CTA holds at least one row
    static std::atomic<int> ok[32];  // occupancy verdict per CL (0 = unknown, 1 = fits, -1 = does not);
    const int key = CL;               // contexts on several host threads may race benignly (same value)
    // the attribute is the CAP (220 KB) for every launch: one value, so contexts on several host
    // threads never shrink it under each other's launches
    cudaFuncSetAttribute(k_sink_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (CL > 8) cudaFuncSetAttribute(k_sink_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (ok[key].load() == 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(SNT);
      cfg.dynamicSmemBytes = 220 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      const cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_sink_small, &cfg);
      ok[key].store((e == cudaSuccess && ncl >= 1) ? 1 : -1);
      cudaGetLastError();
    }
    if (ok[key].load() < 0) continue;
    *rows_out = (int)rows;
    *bytes_out = bytes;
    return CL;
  }
  return 0;
}

// `iters` Sinkhorn iterations on G.  tol > 0: check every `check_every` iterations (one
// host sync per check); returns the iterations used and whether tol was met.
// Multi-rank: f is per-shard, g replicated; every column half-step gathers the ranks' column
// sums (the only exchange), and every rank reaches the same path decision and stop flag.
// kappa (UGW, reading R34): the unbalanced updates f' = eps ln u - kappa eps LSE, g' likewise, in the
// absorbed-dual form (P.lp, P.lq = ln u, ln v); 1 = balanced.
static gw_status sink_run(gw_ctx* c, const Prepared& P, SinkState& s, const float* G, int64_t ldG, double eps,
                          int iters, double tol, int check_every, int* used, int* converged, bool reset_count = true,
                          double kappa = 1.0, bool xm = false) {
  NvtxRange nv("gw.sinkhorn");
  const int64_t nl = P.nl, m = P.m;
  const float c2f = (float)(GW_LOG2E / eps);
  // grid-stride launches: when the fused path runs, the skipped safe-path kernels cost one small wave
  const unsigned cgrid = (unsigned)std::min<int64_t>(((m + 1023) / 1024) * s.nrb, 148 * 4);
  const unsigned rgrid = (unsigned)std::min<int64_t>((nl + RROWS - 1) / RROWS, 148 * 4);
  CU(cudaMemsetAsync(s.stop, 0, sizeof(int), c->stream));
  CU(cudaMemsetAsync(s.flag, 0, sizeof(int), c->stream));  // the speculation flag starts clear
  if (reset_count) CU(cudaMemsetAsync(s.mode, 0, 4 * sizeof(int), c->stream));  // dev = 0; count = 0
  // first iteration: speculative fused path if available (validated before commit), else safe
  k_fill_int<<<1, 32, 0, c->stream>>>(s.mode, s.fK > 0 ? 1 : 0);
  KCHECK();
  *used = 0;
  *converged = 0;
  if (check_every < 1) check_every = 10;
  int done = 0;
  const bool tolmode = tol > 0;
  FusedArgs fa;
  fa.G = G; fa.ld = ldG; fa.nl = nl; fa.m = m; fa.c2f = c2f; fa.gh = s.gh; fa.gl = s.gl; fa.fh = s.fh;
  fa.fl = s.fl; fa.pf = s.pf; fa.Srow = s.Srow; fa.part = s.fpart; fa.rows_per_cluster = s.frpc;
  fa.mode = s.mode; fa.stop = s.stop; fa.wcol = s.fW;
  fa.kappa = (float)kappa;
  if (kappa != 1.0 && s.fK > 0) {  // the fused kernel's row term: log2 u (fp32) instead of p
    k_scale_f<<<grid_for(nl), 256, 0, c->stream>>>(P.lp + P.row0, nl, GW_LOG2E, s.pf);
    KCHECK();
  }
  // the fused one-read step of one iteration (speculative; a no-op unless *mode == 1)
  cudaGraphConditionalHandle cond_h = 0;  // set while capturing the single-rank iteration graph
  int use_cond = 0;
  // XM sweep (the last iteration of the inner loop on the 8 N M gradient path): only in the fixed-count
  // single-rank graph loop below; s.xmv tells the caller whether it ran and was committed
  xm = xm && s.rcCL > 0 && s.fK > 0 && P.R == 1 && kappa == 1.0 && tol <= 0;
  if (s.xmv) CU(cudaMemsetAsync(s.xmv, 0, sizeof(int), c->stream));
  FusedArgs fax = fa;
  if (xm) {
    const double cc = GW_LOG2E / eps;
    fax.c2f_lo = (float)(cc - (double)c2f);
    fax.xr = s.xf;
    fax.part = s.rcpart;
    fax.partx = s.rcpartx;
    fax.rows_per_cluster = s.rcrpc;
    fax.wcol = RC_W;
  }
  auto fused_step = [&](bool xmstep = false) -> gw_status {
    // Every iteration first tries the fused one-read path when *mode == 1 (speculatively at the
    // start of a solve); k_sink_fast_check validates it before anything is committed, and on
    // failure k_sink_fin_fast leaves f, g untouched and sets *mode = 0 so that the robust
    // two-kernel path below runs this same iteration.  No host sync.
    if (s.fK > 0) {
      PROF_BEGIN(c, PC_SINK_XM);
      PROF_BEGIN(c, PC_SINK_FUSED);
      if (xmstep) TRY(rc_xm_launch(c, s.rcCL, fax, s.rcncl));
      else TRY(fused_launch(c, s.fK, s.fCL, s.fNT, fa, s.fncl));
      KCHECK();
      double* const fpart = xmstep ? s.rcpart : s.fpart;
      const int fncl = xmstep ? s.rcncl : s.fncl;
      // one rank: column sums, check (rows + columns), commit.  R > 1: the rank's row check rides in
      // the column-sum payload (slot M), so ONE all-gather per iteration carries everything.
      const bool multi = P.R > 1;
      const int64_t stride = multi ? m + 1 : m;
      if (multi) {
        CU(cudaMemsetAsync(s.csl + m, 0, sizeof(double), c->stream));
        k_sink_colsum<<<(unsigned)((m + 31) / 32), 256, 0, c->stream>>>(
            fpart, fncl, m, s.csl, s.mode, s.stop, s.Srow, nl, reinterpret_cast<int*>(s.csl + m));
      } else {  // one rank: column sums + the whole validity check in one launch (flag cleared by k_sink_mode)
        k_sink_colsum<<<(unsigned)((m + 31) / 32), 256, 0, c->stream>>>(
            fpart, fncl, m, s.csl, s.mode, s.stop, s.Srow, nl, s.flag, s.flag, P.lq);
      }
      KCHECK();
      if (xmstep) {
        k_xm_mark<<<1, 32, 0, c->stream>>>(s.mode, s.flag, s.stop, s.xmv);
        KCHECK();
      }
      if (fault_is("colsum")) {  // test-only: one column sum of the half-step plan doubled
        k_fault_scale<<<1, 32, 0, c->stream>>>(s.csl, m / 2, 2.0);
        KCHECK();
      }
      TRY(comm_allgather(c, s.csl, s.csg, sizeof(double) * (size_t)stride));
      if (multi) {
        CU(cudaMemsetAsync(s.flag, 0, sizeof(int), c->stream));
        k_sink_fast_check<<<grid_for(std::max(m, nl), 256, 1 << 30), 256, 0, c->stream>>>(
            s.Srow, nl, s.csg, P.R, stride, m, P.lq, s.flag, s.mode, s.stop, multi);
        KCHECK();
      }
      k_sink_fin_fast<<<grid_for(std::max(m, nl), 256, 1 << 30), 256, 0, c->stream>>>(
          s.Srow, nl, P.lp + P.row0, s.f, s.fh, s.fl, nullptr, s.csg, P.R, stride, m, P.lq, eps, s.g, s.gh, s.gl,
          s.mode, s.stop, s.dev, s.flag, kappa, cond_h, use_cond);
      KCHECK();
      if (xmstep) {
        PROF_END(c, PC_SINK_XM, 2);
      } else {
        PROF_END(c, PC_SINK_FUSED, 2);
      }
    }
    return GW_OK;
  };
  // one iteration (check: the tolerance rule's violation check of the plan after `done` iterations)
  const int* commit_cnt = nullptr;  // graph-resident tolerance loop: the iteration count lives on the device
  auto iteration = [&](bool check, int done, bool xmstep = false) -> gw_status {
    if (!check) TRY(fused_step(xmstep));
    // iterations run the robust two-kernel path while *mode == 0 (decided on the device)
    const int* skip = check ? nullptr : s.mode;
    if (check) CU(cudaMemsetAsync(s.viol, 0, sizeof(float), c->stream));
    double* fout = check ? s.ftmp : s.f;
    PROF_BEGIN(c, PC_SINK_ROW);
    k_sink_row<<<rgrid, 256, 0, c->stream>>>(
        G, ldG, nl, m, s.gh, s.gl, c2f, s.f, fout, P.lp + P.row0, eps, s.fh, s.fl, check ? s.viol : nullptr, s.stop,
        skip, kappa);
    KCHECK();
    PROF_END(c, PC_SINK_ROW, 1);
    if (check) {
      TRY(sink_viol_global(c, P, s));
      k_sink_commit<<<grid_for(nl), 256, 0, c->stream>>>(s.viol, tol, s.stop, s.ftmp, s.f, nl, s.iters, done,
                                                         commit_cnt);
      KCHECK();
    }
    PROF_BEGIN(c, PC_SINK_COL);
    k_sink_col<<<cgrid, 256, 0, c->stream>>>(G, ldG, nl, m, s.fh, s.fl, c2f, s.RB, s.part, s.stop, skip);
    KCHECK();
    if (P.R == 1) {
      k_sink_colmergefin<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.part, s.nrb, m, P.lq, eps, s.g, s.gh,
                                                                            s.gl, s.stop, skip, s.dev, kappa);
      KCHECK();
    } else {
      k_sink_colmerge<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.part, s.nrb, m, s.lse, s.stop, skip);
      KCHECK();
      TRY(comm_allgather(c, s.lse, s.lseg, 2 * sizeof(double) * (size_t)m));
      k_sink_colfin<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.lseg, P.R, m, P.lq, eps, s.g, s.gh, s.gl,
                                                                       s.stop, skip, s.dev, kappa);
      KCHECK();
    }
    PROF_END(c, PC_SINK_COL, 2);
    k_sink_mode<<<1, 32, 0, c->stream>>>(s.dev, s.mode, s.fK > 0 ? FUSED_THRESH : -1.f, s.flag);
    KCHECK();
    return GW_OK;
  };
  // Fixed iteration counts on several ranks: every iteration SLOT issues exactly one all-gather of one
  // payload of M + 1 doubles: the fused path's column sums (+ this rank's row flag in slot M), or the
  // safe path's column LSE pairs packed as 8-byte {float max, float sum}; the kernels of the path not
  // taken exit at once (decided on the device, identically on every rank:
  // the decision follows gathered data).  A slot whose fused attempt fails the validity check commits
  // nothing and the next slot runs the safe path, so the committed updates are exactly those of the
  // single-rank loop; slots are replayed (a CUDA graph per solve over NCCL) until `iters` updates are
  // committed -- iters + SLACK slots per round, the device stops after the target, ONE host read per
  // round (no host sync inside the inner loop unless more than SLACK fused attempts fail).
  if (!tolmode && P.R > 1 && s.fK > 0) {
    const int64_t U = m + 1;
    double* uc = s.un;           // [0, m): column sums (fused) or packed LSE pairs (safe), [m]: row flag
    CU(cudaMemsetAsync(s.mode + 5, 0, 2 * sizeof(int), c->stream));
    k_fill_int<<<1, 32, 0, c->stream>>>(s.mode + 6, iters);
    KCHECK();
    auto slot = [&]() -> gw_status {
      CU(cudaMemsetAsync(s.flag, 0, sizeof(int), c->stream));
      CU(cudaMemsetAsync(uc + m, 0, sizeof(double), c->stream));
      PROF_BEGIN(c, PC_SINK_FUSED);
      TRY(fused_launch(c, s.fK, s.fCL, s.fNT, fa, s.fncl));
      KCHECK();
      k_sink_colsum<<<(unsigned)((m + 31) / 32), 256, 0, c->stream>>>(s.fpart, s.fncl, m, uc, s.mode, s.stop, s.Srow,
                                                                      nl, reinterpret_cast<int*>(uc + m));
      KCHECK();
      PROF_END(c, PC_SINK_FUSED, 2);
      // the safe path's local half (skipped unless *mode == 0): row update, then column LSE pairs
      PROF_BEGIN(c, PC_SINK_ROW);
      k_sink_row<<<rgrid, 256, 0, c->stream>>>(G, ldG, nl, m, s.gh, s.gl, c2f, s.f, s.f, P.lp + P.row0, eps, s.fh,
                                                s.fl, nullptr, s.stop, s.mode, kappa);
      KCHECK();
      PROF_END(c, PC_SINK_ROW, 1);
      PROF_BEGIN(c, PC_SINK_COL);
      k_sink_col<<<cgrid, 256, 0, c->stream>>>(G, ldG, nl, m, s.fh, s.fl, c2f, s.RB, s.part, s.stop, s.mode);
      KCHECK();
      k_sink_colmerge<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.part, s.nrb, m, uc, s.stop, s.mode, true);
      KCHECK();
      PROF_END(c, PC_SINK_COL, 1);
      TRY(comm_allgather(c, s.un, s.ung, sizeof(double) * (size_t)U));
      // safe path: g from the gathered LSE pairs (before the fused finish, which may switch *mode)
      k_sink_colfin<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.ung, P.R, m, P.lq, eps, s.g, s.gh, s.gl,
                                                                       s.stop, s.mode, s.dev, kappa, U, true);
      KCHECK();
      // fused path: validity of the speculative iteration (all ranks' row flags, the gathered column
      // sums), then commit -- or not, and switch to the safe path
      k_sink_fast_check<<<grid_for(std::max(m, nl), 256, 1 << 30), 256, 0, c->stream>>>(
          s.Srow, nl, s.ung, P.R, U, m, P.lq, s.flag, s.mode, s.stop, true);
      KCHECK();
      k_sink_fin_fast<<<grid_for(std::max(m, nl), 256, 1 << 30), 256, 0, c->stream>>>(
          s.Srow, nl, P.lp + P.row0, s.f, s.fh, s.fl, nullptr, s.ung, P.R, U, m, P.lq, eps, s.g, s.gh, s.gl,
          s.mode, s.stop, s.dev, s.flag, kappa);
      KCHECK();
      k_sink_slot_end<<<1, 32, 0, c->stream>>>(s.mode, s.dev, s.flag, s.stop, FUSED_THRESH);
      KCHECK();
      return GW_OK;
    };
    static const bool no_graph_mr = getenv("GWDP_NO_GRAPH") != nullptr;
    const bool graph = !no_graph_mr && !c->prof.on && c->comm && c->comm->nccl;  // host transport: not capturable
    if (graph && s.gexec && (s.g_eps != eps || s.g_kappa != kappa)) sink_free(s);
    if (graph && !s.gexec) {
      s.g_eps = eps;
      s.g_kappa = kappa;
      if (!c->cap) CU(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
      CU(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
      cudaStream_t saved = c->stream;
      c->stream = c->cap;
      const gw_status st = slot();
      c->stream = saved;
      cudaGraph_t gr = nullptr;
      const cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
      if (st != GW_OK) {
        if (gr) cudaGraphDestroy(gr);
        return st;
      }
      if (e != cudaSuccess) return fail(GW_ERR_CUDA, "Sinkhorn graph capture (multi-rank): %s", cudaGetErrorString(e));
      const cudaError_t ei = cudaGraphInstantiate(&s.gexec, gr, 0);
      cudaGraphDestroy(gr);
      if (ei != cudaSuccess) return fail(GW_ERR_CUDA, "Sinkhorn graph instantiate: %s", cudaGetErrorString(ei));
    }
    constexpr int SLACK = 4;
    int* hc = reinterpret_cast<int*>(c->hpin + 40);
    int committed = 0;
    for (int round = 0; committed < iters; ++round) {
      const int nslots = (iters - committed) + SLACK;
      for (int k = 0; k < nslots; ++k) {
        if (graph) CU(cudaGraphLaunch(s.gexec, c->stream));
        else TRY(slot());
      }
      CU(cudaMemcpyAsync(hc, s.mode + 5, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      committed = hc[0];
      if (round > 64) return fail(GW_ERR_CUDA, "multi-rank Sinkhorn: no progress (%d of %d updates)", committed, iters);
    }
    // the device stop flag is left set; later calls reset it
    CU(cudaMemsetAsync(s.stop, 0, sizeof(int), c->stream));
    *used = iters;
    return GW_OK;
  }
  // Fixed iteration counts, one rank, G small enough for one cluster's shared memory: every
  // iteration in ONE launch (small.cuh; GWDP_NO_SMALL=1 disables it)
  const bool no_small = getenv("GWDP_NO_SMALL") != nullptr;  // read per call (tests compare both paths)
  if (!tolmode && !no_small && P.R == 1 && iters > 0) {
    int rows = 0;
    size_t bytes = 0;
    const int CL = small_cluster(c, P, &rows, &bytes);
    if (CL > 0) {
      // even smem row pitch: the fp64 arrays after the fp32 tile stay 8-byte aligned
      SmallArgs sa{G, ldG, nl, m, rows, (int)((m + 1) & ~int64_t(1)), P.lp + P.row0, P.lq, eps, kappa, iters, s.f,
                   s.g};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(SNT);
      cfg.dynamicSmemBytes = bytes;
      cfg.stream = c->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PROF_BEGIN(c, PC_SINK_ROW);
      CU(cudaLaunchKernelEx(&cfg, k_sink_small, sa));
      KCHECK();
      PROF_END(c, PC_SINK_ROW, 1);
      TRY(sink_split(c, P, s, eps));
      *used = iters;
      return GW_OK;
    }
  }
  // Fixed iteration counts on one rank: the iteration's ~10 launches are captured once per solve
  // into a CUDA graph and replayed (the small configurations are launch-bound; GWDP_NO_GRAPH=1
  // disables it; not while per-kernel profiling is on, whose events time the launches).
  static const bool no_graph = getenv("GWDP_NO_GRAPH") != nullptr;
  if (!tolmode && !no_graph && !c->prof.on && P.R == 1 && iters >= 3) {
    if (s.gexec && (s.g_eps != eps || s.g_kappa != kappa)) sink_free(s);
    auto capture = [&](bool xmstep, cudaGraphExec_t* out) -> gw_status {
      if (!c->cap) CU(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
      static const bool no_cond = getenv("GWDP_NO_COND") != nullptr;
      cudaGraph_t graph = nullptr;
      gw_status st = GW_OK;
      cudaError_t e = cudaSuccess;
      cudaStream_t saved = c->stream;
      if (s.fK > 0 && !no_cond) {
        // fused step, then the safe path as the body of a conditional (IF) node armed by
        // k_sink_fin_fast, then the path decision: a committed fused iteration launches nothing else
        if (!c->cap2) CU(cudaStreamCreateWithFlags(&c->cap2, cudaStreamNonBlocking));
        CU(cudaGraphCreate(&graph, 0));
        CU(cudaGraphConditionalHandleCreate(&cond_h, graph, 0, cudaGraphCondAssignDefault));
        CU(cudaStreamBeginCaptureToGraph(c->cap, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        c->stream = c->cap;
        use_cond = 1;
        st = fused_step(xmstep);
        use_cond = 0;
        if (st == GW_OK) {
          cudaStreamCaptureStatus cs;
          const cudaGraphNode_t* deps = nullptr;
          size_t nd = 0;
          cudaGraph_t cg = nullptr;
          e = cudaStreamGetCaptureInfo(c->cap, &cs, nullptr, &cg, &deps, &nd);
          cudaGraphNodeParams cp = {};
          cp.type = cudaGraphNodeTypeConditional;
          cp.conditional.handle = cond_h;
          cp.conditional.type = cudaGraphCondTypeIf;
          cp.conditional.size = 1;
          cudaGraphNode_t cn = nullptr;
          if (e == cudaSuccess) e = cudaGraphAddNode(&cn, cg, deps, nd, &cp);
          if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(c->cap, &cn, 1, cudaStreamSetCaptureDependencies);
          if (e == cudaSuccess) {
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            e = cudaStreamBeginCaptureToGraph(c->cap2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
              c->stream = c->cap2;
              k_sink_row<<<rgrid, 256, 0, c->stream>>>(G, ldG, nl, m, s.gh, s.gl, c2f, s.f, s.f, P.lp + P.row0, eps,
                                                        s.fh, s.fl, nullptr, s.stop, nullptr, kappa);
              k_sink_col<<<cgrid, 256, 0, c->stream>>>(G, ldG, nl, m, s.fh, s.fl, c2f, s.RB, s.part, s.stop, nullptr);
              k_sink_colmergefin<<<grid_for(m, 256, 1 << 30), 256, 0, c->stream>>>(s.part, s.nrb, m, P.lq, eps, s.g,
                                                                                    s.gh, s.gl, s.stop, nullptr, s.dev,
                                                                                    kappa);
              cudaGraph_t bo = nullptr;
              e = cudaStreamEndCapture(c->cap2, &bo);
              c->stream = c->cap;
            }
          }
          k_sink_mode<<<1, 32, 0, c->stream>>>(s.dev, s.mode, FUSED_THRESH, s.flag);
        }
        c->stream = saved;
        cudaGraph_t go = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(c->cap, &go);
        if (e == cudaSuccess) e = e2;
      } else {
        CU(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
        c->stream = c->cap;
        st = iteration(false, 0);
        c->stream = saved;
        e = cudaStreamEndCapture(c->cap, &graph);
      }
      if (st != GW_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (e != cudaSuccess) return fail(GW_ERR_CUDA, "Sinkhorn graph capture: %s", cudaGetErrorString(e));
      const cudaError_t ei = cudaGraphInstantiate(out, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) return fail(GW_ERR_CUDA, "Sinkhorn graph instantiate: %s", cudaGetErrorString(ei));
      return GW_OK;
    };
    static const bool no_cond_x = getenv("GWDP_NO_COND") != nullptr;
    if (no_cond_x) xm = false;  // the XM sweep rides on the conditional-node graph only
    if (!s.gexec) {
      s.g_eps = eps;
      s.g_kappa = kappa;
      TRY(capture(false, &s.gexec));
    }
    if (xm && !s.gexec_xm) TRY(capture(true, &s.gexec_xm));
    for (int k = 0; k < iters; ++k) CU(cudaGraphLaunch((xm && k == iters - 1) ? s.gexec_xm : s.gexec, c->stream));
    *used = iters;
    return GW_OK;
  }
  // Tolerance rule on one rank (reading R8), graph-resident: a prologue of check_every iterations, then a
  // WHILE conditional node whose body is [the checking iteration (measure the violation of the current
  // plan; stop, or commit the measured row update as this iteration's) + check_every - 1 iterations] and
  // whose condition is set on the device (no stop, count below the cap): the same schedule as the host
  // loop below, with no host synchronisation inside it.  GWDP_NO_DEVLOOP=1 keeps the host loop.
  static const bool no_devloop = getenv("GWDP_NO_DEVLOOP") != nullptr;
  if (tolmode && P.R == 1 && !no_graph && !no_devloop && !c->prof.on && iters >= 2 * check_every &&
      iters % check_every == 0) {
    int* cnt = s.mode + 3;  // iterations done (device)
    if (!c->cap) CU(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    if (!c->cap2) CU(cudaStreamCreateWithFlags(&c->cap2, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    CU(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle hw;
    CU(cudaGraphConditionalHandleCreate(&hw, graph, 1, cudaGraphCondAssignDefault));
    cudaStream_t saved = c->stream;
    gw_status st = GW_OK;
    cudaError_t e = cudaStreamBeginCaptureToGraph(c->cap, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      c->stream = c->cap;
      k_fill_int<<<1, 32, 0, c->stream>>>(cnt, check_every);
      for (int k = 0; k < check_every && st == GW_OK; ++k) st = iteration(false, 0);
      if (st == GW_OK) {
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaGraph_t cg = nullptr;
        e = cudaStreamGetCaptureInfo(c->cap, &cs, nullptr, &cg, &deps, &nd);
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hw;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wn = nullptr;
        if (e == cudaSuccess) e = cudaGraphAddNode(&wn, cg, deps, nd, &cp);
        if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(c->cap, &wn, 1, cudaStreamSetCaptureDependencies);
        if (e == cudaSuccess) {
          e = cudaStreamBeginCaptureToGraph(c->cap2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal);
          if (e == cudaSuccess) {
            c->stream = c->cap2;
            commit_cnt = cnt;
            st = iteration(true, 0);
            commit_cnt = nullptr;
            for (int k = 1; k < check_every && st == GW_OK; ++k) st = iteration(false, 0);
            k_tol_round_end<<<1, 32, 0, c->stream>>>(cnt, check_every, iters, s.stop, hw);
            cudaGraph_t bo = nullptr;
            const cudaError_t eb = cudaStreamEndCapture(c->cap2, &bo);
            if (e == cudaSuccess) e = eb;
          }
        }
      }
      c->stream = saved;
      cudaGraph_t go = nullptr;
      const cudaError_t ee = cudaStreamEndCapture(c->cap, &go);
      if (e == cudaSuccess) e = ee;
    }
    cudaGraphExec_t ex = nullptr;
    if (st == GW_OK && e == cudaSuccess) e = cudaGraphInstantiate(&ex, graph, 0);
    cudaGraphDestroy(graph);
    if (st != GW_OK) {
      if (ex) cudaGraphExecDestroy(ex);
      return st;
    }
    if (e != cudaSuccess) return fail(GW_ERR_CUDA, "Sinkhorn tolerance-loop graph: %s", cudaGetErrorString(e));
    const cudaError_t el = cudaGraphLaunch(ex, c->stream);
    int hs[3];
    CU(cudaMemcpyAsync(hs, s.stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(hs + 1, s.iters, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(hs + 2, cnt, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    const cudaError_t es = cudaStreamSynchronize(c->stream);
    cudaGraphExecDestroy(ex);
    if (el != cudaSuccess || es != cudaSuccess)
      return fail(GW_ERR_CUDA, "Sinkhorn tolerance loop: %s", cudaGetErrorString(el != cudaSuccess ? el : es));
    if (hs[0]) {
      *used = hs[1];
      *converged = 1;
      k_split<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / eps, s.fh, s.fl);  // fh/fl == split(f)
      KCHECK();
      return GW_OK;
    }
    done = iters;  // the final check below
  }
  while (done < iters) {
    const int chunk = tolmode ? std::min(check_every, iters - done) : iters - done;
    for (int k = 0; k < chunk; ++k) {
      const bool check = tolmode && k == 0 && done > 0;  // violation of the plan after `done` iterations
      TRY(iteration(check, done, xm && !tolmode && done + k == iters - 1));
    }
    if (tolmode) {
      int hs[2];
      CU(cudaMemcpyAsync(hs, s.stop, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaMemcpyAsync(hs + 1, s.iters, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      if (hs[0]) {
        *used = hs[1];
        *converged = 1;
        // the measuring row half-step split the DISCARDED trial f' into fh/fl (k_sink_row always writes
        // them); k_sink_commit kept f: re-split it so that fh/fl == split(f) on every return
        k_split<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / eps, s.fh, s.fl);
        KCHECK();
        return GW_OK;
      }
    }
    done += chunk;
  }
  *used = done;
  if (tolmode) {
    // final check of the plan after `done` iterations (row half-step into ftmp, not committed)
    CU(cudaMemsetAsync(s.viol, 0, sizeof(float), c->stream));
    k_sink_row<<<rgrid, 256, 0, c->stream>>>(
        G, ldG, nl, m, s.gh, s.gl, c2f, s.f, s.ftmp, P.lp + P.row0, eps, s.fh, s.fl, s.viol, nullptr, nullptr, kappa);
    KCHECK();
    TRY(sink_viol_global(c, P, s));
    float hv;
    CU(cudaMemcpyAsync(&hv, s.viol, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *converged = (double)hv <= tol;
    // restore fh/fl for the committed f
    k_split<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / eps, s.fh, s.fl);
    KCHECK();
  }
  return GW_OK;
}

static gw_status stage_duals_in(gw_ctx* c, const gw_problem* pb, const Prepared& P, double* f, double* g,
                                double** fd, double** gd) {
  if (pb->flags & GW_HOST_VECTORS) {
    TRY(ws(c, c->fs, P.nl, fd));
    TRY(ws(c, c->gs, P.m, gd));
    if (f) CU(cudaMemcpyAsync(*fd, f, P.nl * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (g) CU(cudaMemcpyAsync(*gd, g, P.m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  } else {
    *fd = f;
    *gd = g;
  }
  return GW_OK;
}

static gw_status stage_duals_out(gw_ctx* c, const gw_problem* pb, const Prepared& P, double* f, double* g,
                                 const double* fd, const double* gd) {
  if (pb->flags & GW_HOST_VECTORS) {
    if (f) CU(cudaMemcpyAsync(f, fd, P.nl * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (g) CU(cudaMemcpyAsync(g, gd, P.m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return GW_OK;
}

static gw_status materialize(gw_ctx* c, const Prepared& P, int mode, const TSrc& S, void* T, int64_t ldT) {
  const int g = grid_for(P.nl * P.m, 256, 148 * 32);
  if (mode == T_PRODUCT) k_materialize<T_PRODUCT><<<g, 256, 0, c->stream>>>(S, P.nl, P.m, (float*)T, ldT);
  else k_materialize<T_GIBBS><<<g, 256, 0, c->stream>>>(S, P.nl, P.m, (float*)T, ldT);
  KCHECK();
  return GW_OK;
}

extern "C" gw_status sinkhorn_solve(gw_ctx* c, const gw_problem* pb, const void* G, int64_t ldG,
                                    const gw_sinkhorn_opts* o, double* f, double* g, void* T_out, int64_t ldT,
                                    gw_sinkhorn_info* info) {
  if (!c || !o) return fail(GW_ERR_INVALID_ARG, "null ctx or opts");
  if (!(o->eps > 0) || o->max_iter < 0) return fail(GW_ERR_CONFIG, "eps must be > 0 and max_iter >= 0");
  if (!f || !g) return fail(GW_ERR_INVALID_ARG, "f and g (warm start, in/out) must be non-null");
  TRY(check_problem(pb));
  TRY(check_matrix(G, ldG, pb->m, "G"));
  if (T_out) TRY(check_matrix(T_out, ldT, pb->m, "T_out"));
  CU(cudaSetDevice(c->device));
  Prepared P;
  TRY(prepare(c, pb, P));
  if (pb->dtype == GW_F64) {  // fp64 storage (f64.cuh)
    Sink64 s;
    TRY(sink64_alloc(c, P, s));
    double *fd, *gd;
    TRY(stage_duals_in(c, pb, P, f, g, &fd, &gd));
    const double* Gd = reinterpret_cast<const double*>(G);
    int used = 0, conv = 0;
    TRY(sink64_run(c, P, s, Gd, ldG, fd, gd, o->eps, o->max_iter, o->tol, o->check_every, &used, &conv));
    if (T_out) {
      k64_gibbs<<<grid_for(P.nl * P.m, 256, 148 * 32), 256, 0, c->stream>>>(Gd, ldG, fd, gd, o->eps, P.nl, P.m,
                                                                            reinterpret_cast<double*>(T_out), ldT);
      KCHECK();
    }
    if (info) {
      double v = 0.0;
      TRY(sink64_viol(c, P, s, Gd, ldG, fd, gd, o->eps, &v));
      info->iters = used;
      info->converged = o->tol > 0 ? (v <= o->tol) : 0;
      info->fused_iters = 0;
      info->marginal_violation = v;
    }
    TRY(stage_duals_out(c, pb, P, f, g, fd, gd));
    return GW_OK;
  }
  SinkState s;
  SinkGuard sguard{s};
  TRY(sink_alloc(c, P, s));
  TRY(stage_duals_in(c, pb, P, f, g, &s.f, &s.g));
  TRY(sink_split(c, P, s, o->eps));
  int used = 0, conv = 0;
  TRY(sink_run(c, P, s, reinterpret_cast<const float*>(G), ldG, o->eps, o->max_iter, o->tol, o->check_every, &used,
               &conv));
  if (T_out) {
    double *fs, *gs;
    TRY(ws(c, c->Ptot, P.nl, &fs));  // scratch
    TRY(ws(c, c->btot, P.m, &gs));
    k_scale<<<grid_for(P.nl), 256, 0, c->stream>>>(s.f, P.nl, GW_LOG2E / o->eps, fs);
    k_scale<<<grid_for(P.m), 256, 0, c->stream>>>(s.g, P.m, GW_LOG2E / o->eps, gs);
    KCHECK();
    TSrc S{reinterpret_cast<const float*>(G), ldG, fs, gs, GW_LOG2E / o->eps};
    TRY(materialize(c, P, T_GIBBS, S, T_out, ldT));
  }
  if (info) {
    // violation of the returned plan: a measuring row half-step (not committed)
    CU(cudaMemsetAsync(s.viol, 0, sizeof(float), c->stream));
    const float c2f = (float)(GW_LOG2E / o->eps);
    k_sink_row<<<(unsigned)((P.nl + RROWS - 1) / RROWS), 256, 0, c->stream>>>(
        reinterpret_cast<const float*>(G), ldG, P.nl, P.m, s.gh, s.gl, c2f, s.f, s.ftmp, P.lp + P.row0, o->eps, s.fh,
        s.fl, s.viol, nullptr, nullptr);
    KCHECK();
    TRY(sink_viol_global(c, P, s));
    float hv;
    CU(cudaMemcpyAsync(&hv, s.viol, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    int* md = reinterpret_cast<int*>(c->hpin + 40);
    CU(cudaMemcpyAsync(md, s.mode, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    info->iters = used;
    info->converged = o->tol > 0 ? ((double)hv <= o->tol) : 0;
    info->fused_iters = md[1];
    info->marginal_violation = hv;
  }
  TRY(stage_duals_out(c, pb, P, f, g, s.f, s.g));
  return GW_OK;
}

// Entropic (F)GW with fp64 storage (f64.cuh): the same mirror-descent schedule as solve_impl
// (Remark 1; Remark 2 for FGW; readings R5, R7, R8) with the plan kept explicit:
// T^l (fp64, one N x M buffer) and G^{l+1} (fp64, one N x M buffer); T^{l+1} = exp((f + g - G^{l+1})/eps).
static gw_status solve64(gw_ctx* c, const gw_problem* pb, const Prepared& P, const gw_solve_opts* o, const double* fx,
                         const double* fy, double alpha, const void* T0, void* T_out, int64_t ldT, double* f, double* g,
                         gw_result* res, double* trace, int ex_iter, void* ex_T, void* ex_G, int64_t ex_ld) {
  const int64_t nl = P.nl, m = P.m;
  const double eps = o->eps;
  const int64_t ld = (m + 31) & ~int64_t(31);
  double *Tb, *Gb, *objout;
  TRY(ws(c, c->d64T, (size_t)std::max<int64_t>(nl, 1) * ld, &Tb));
  TRY(ws(c, c->d64G, (size_t)std::max<int64_t>(nl, 1) * ld, &Gb));
  TRY(ws(c, c->objout, 16, &objout));
  Sink64 s;
  TRY(sink64_alloc(c, P, s));
  double *fd, *gd;
  if (pb->flags & GW_HOST_VECTORS) {
    TRY(stage_duals_in(c, pb, P, nullptr, nullptr, &fd, &gd));
  } else {
    fd = f;
    gd = g;
  }
  k_fill<<<grid_for(nl), 256, 0, c->stream>>>(fd, nl, 0.0);  // f = g = 0 before the first sweep (R7)
  k_fill<<<grid_for(m), 256, 0, c->stream>>>(gd, m, 0.0);
  KCHECK();
  EventSet evset;
  cudaEvent_t ev0, ev1;
  CU(evset.make(&ev0)); CU(evset.make(&ev1));
  CU(cudaEventRecord(ev0, c->stream));
  std::vector<cudaEvent_t> evs(2 * (size_t)o->outer_iters + 2);
  for (auto& e : evs) CU(evset.make(&e));
  const int eg = grid_for(nl * m, 256, 148 * 32);
  // T^0: the caller's T0 or p q^T (reading R5)
  if (T0) CU(cudaMemcpy2DAsync(Tb, ld * 8, T0, ldT * 8, m * 8, nl, cudaMemcpyDeviceToDevice, c->stream));
  else k64_product<<<eg, 256, 0, c->stream>>>(P.pn + P.row0, P.qn, nl, m, Tb, ld);
  KCHECK();
  const bool want_trace_obj = (o->flags & GW_SOLVE_TRACE_OBJECTIVE) != 0;
  std::vector<double> tr((size_t)std::max(o->outer_iters, 1) * 4, NAN);
  int inner_total = 0, conv_all = 1;
  for (int l = 0; l < o->outer_iters; ++l) {
    const bool exporting = ex_iter == l + 1;
    if (exporting && ex_T) CU(cudaMemcpy2DAsync(ex_T, ex_ld * 8, Tb, ld * 8, m * 8, nl, cudaMemcpyDeviceToDevice, c->stream));
    const bool obj = l > 0 && want_trace_obj;
    CU(cudaEventRecord(evs[2 * l], c->stream));
    TRY(grad64(c, P, Tb, ld, Gb, ld, obj, fx, fy, alpha, nullptr, objout));  // G^{l+1} = grad E(T^l)
    CU(cudaEventRecord(evs[2 * l + 1], c->stream));
    if (exporting && ex_G) CU(cudaMemcpy2DAsync(ex_G, ex_ld * 8, Gb, ld * 8, m * 8, nl, cudaMemcpyDeviceToDevice, c->stream));
    if (obj) {
      CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      tr[(size_t)(l - 1) * 4 + 0] = fx ? (1.0 - alpha) * c->hpin[6] + alpha * c->hpin[0] : c->hpin[0];
      tr[(size_t)(l - 1) * 4 + 1] = c->hpin[1];
    }
    int used = 0, conv = 0;
    TRY(sink64_run(c, P, s, Gb, ld, fd, gd, eps, o->inner.max_iter, o->inner.tol, o->inner.check_every, &used, &conv,
                   true));
    k64_gibbs<<<eg, 256, 0, c->stream>>>(Gb, ld, fd, gd, eps, nl, m, Tb, ld);  // T^{l+1}
    KCHECK();
    inner_total += used;
    if (o->inner.tol > 0 && !conv) conv_all = 0;
    tr[(size_t)l * 4 + 2] = used;
  }
  CU(cudaEventRecord(evs[2 * (size_t)o->outer_iters], c->stream));
  // final plan: objective, violation, entropy (one gradient pass; G is scratch now)
  TRY(grad64(c, P, Tb, ld, Gb, ld, true, fx, fy, alpha, nullptr, objout));
  if (T_out) CU(cudaMemcpy2DAsync(T_out, ldT * 8, Tb, ld * 8, m * 8, nl, cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaEventRecord(ev1, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  const double E = c->hpin[0], viol = c->hpin[1], H = c->hpin[3], ecc = c->hpin[6];
  if (!(std::isfinite(E) && std::isfinite(H) && std::isfinite(viol)))
    return fail(GW_ERR_NONFINITE, "non-finite result (E = %g, H = %g, violation = %g): eps too small for the "
                "cost scale, or non-finite inputs", E, H, viol);
  const double Eout = fx ? (1.0 - alpha) * ecc + alpha * E : E;
  if (o->outer_iters > 0) {
    tr[(size_t)(o->outer_iters - 1) * 4 + 0] = Eout;
    tr[(size_t)(o->outer_iters - 1) * 4 + 1] = viol;
  }
  float ms_grad = 0.f, ms_sink = 0.f, ms_total = 0.f;
  for (int l = 0; l < o->outer_iters; ++l) {
    float a = 0.f, b = 0.f;
    CU(cudaEventElapsedTime(&a, evs[2 * l], evs[2 * l + 1]));
    CU(cudaEventElapsedTime(&b, evs[2 * l + 1], evs[2 * l + 2]));
    ms_grad += a;
    ms_sink += b;
    tr[(size_t)l * 4 + 3] = a + b;
  }
  CU(cudaEventElapsedTime(&ms_total, ev0, ev1));
  res->gw_objective = Eout;
  res->entropic_objective = Eout + eps * H;
  res->marginal_violation = viol;
  res->outer_iters = o->outer_iters;
  res->inner_iters_total = inner_total;
  res->converged = (o->inner.tol > 0) ? conv_all : 0;
  res->inner_fused_total = 0;
  res->ms_grad = ms_grad;
  res->ms_sinkhorn = ms_sink;
  res->ms_total = ms_total;
  res->grad_onepass_total = 0;
  if (trace) memcpy(trace, tr.data(), sizeof(double) * 4 * (size_t)o->outer_iters);
  TRY(stage_duals_out(c, pb, P, f, g, fd, gd));
  return GW_OK;
}

// ------------------------------------------------------------------------------ solver
static gw_status solve_impl(gw_ctx* c, const gw_problem* pb, const gw_solve_opts* o, const double* fx_in,
                            const double* fy_in, double alpha, const void* T0, void* T_out, int64_t ldT, double* f,
                            double* g, gw_result* res, double* trace) {
  if (!c || !o || !res) return fail(GW_ERR_INVALID_ARG, "null ctx, opts or result");
  // the debug export request is one-shot: taken by this call whatever its outcome
  const auto ex = c->exp;
  c->exp.iter = 0;
  c->exp.T = c->exp.G = nullptr;
  if (!(o->eps > 0)) return fail(GW_ERR_CONFIG, "eps must be > 0");
  NvtxRange nv("gw.solve");
  // tau (0 means tau = eps, Remark 1): the Sinkhorn regulariser; tau != eps adds
  // (eps - tau) ln T^l to the cost (k = 1, 1-D supports, T0 = p q^T)
  const double tau = (o->tau == 0) ? o->eps : o->tau;
  if (!(tau > 0)) return fail(GW_ERR_CONFIG, "tau must be > 0");
  const bool tau_mode = tau != o->eps;
  if (tau_mode && T0) return fail(GW_ERR_UNSUPPORTED, "tau != eps with an explicit T0 (ln T0) is not implemented");
  if (o->outer_iters < 0 || o->inner.max_iter < 0) return fail(GW_ERR_CONFIG, "iteration counts must be >= 0");
  if (!f || !g) return fail(GW_ERR_INVALID_ARG, "f and g (outputs) must be non-null");
  TRY(check_problem(pb));
  if (T0) TRY(check_matrix(T0, ldT, pb->m, "T0"));
  if (T_out) TRY(check_matrix(T_out, ldT, pb->m, "T_out"));
  CU(cudaSetDevice(c->device));
  const double eps = o->eps;  // the problem's regulariser (entropic objective E + eps H)
  const double es = tau;      // the Sinkhorn regulariser (= eps unless tau != eps)
  const double beta = tau_mode ? eps - tau : 0.0;
  Prepared P;
  TRY(prepare(c, pb, P));
  if (tau_mode && (P.k != 1 || P.grid2d))
    return fail(GW_ERR_UNSUPPORTED, "tau != eps: k = 1 on 1-D supports only");
  const int64_t nl = P.nl, m = P.m;
  const double* fx = nullptr;
  const double* fy = nullptr;
  if (fx_in) {
    if (pb->flags & GW_HOST_VECTORS) {
      double *a, *b;
      TRY(ws(c, c->fxs, P.n, &a));
      TRY(ws(c, c->fys, m, &b));
      CU(cudaMemcpyAsync(a, fx_in, P.n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      CU(cudaMemcpyAsync(b, fy_in, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      fx = a; fy = b;
    } else {
      fx = fx_in; fy = fy_in;
    }
  }
  if (pb->dtype == GW_F64) {
    if (tau_mode) return fail(GW_ERR_UNSUPPORTED, "GW_F64 storage: tau != eps is not implemented");
    return solve64(c, pb, P, o, fx, fy, alpha, T0, T_out, ldT, f, g, res, trace, ex.iter, ex.T, ex.G, ex.ld);
  }
  // cost buffer
  const int64_t ldG = (m + 31) & ~int64_t(31);
  float* G;
  TRY(ws(c, c->Gs, (size_t)std::max<int64_t>(nl, 1) * ldG, &G));
  SinkState s;
  SinkGuard sguard{s};
  TRY(sink_alloc(c, P, s));
  if (pb->flags & GW_HOST_VECTORS) {
    TRY(stage_duals_in(c, pb, P, nullptr, nullptr, &s.f, &s.g));  // device scratch for host duals
  } else {
    s.f = f;  // the caller's device output buffers hold the duals throughout
    s.g = g;
  }
  // f = g = 0 before the first sweep (reading R7)
  k_fill<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, 0.0);
  k_fill<<<grid_for(m), 256, 0, c->stream>>>(s.g, m, 0.0);
  KCHECK();
  // scaled duals f log2e/eps, g log2e/eps for the Gibbs regeneration of T in the gradient
  double *Fs, *Gs2, *objout;
  TRY(ws(c, c->fsc, (size_t)std::max<int64_t>(nl, 1), &Fs));
  TRY(ws(c, c->gsc, (size_t)m, &Gs2));
  TRY(ws(c, c->objout, 16, &objout));

  EventSet evset;
  cudaEvent_t ev0, ev1;
  CU(evset.make(&ev0)); CU(evset.make(&ev1));
  CU(cudaEventRecord(ev0, c->stream));
  std::vector<cudaEvent_t> evs(2 * (size_t)o->outer_iters + 2);
  for (auto& e : evs) CU(evset.make(&e));

  int inner_total = 0, conv_all = 1;
  float ms_grad = 0.f, ms_sink = 0.f;
  std::vector<double> tr((size_t)std::max(o->outer_iters, 1) * 4, NAN);
  const bool want_trace_obj = (o->flags & GW_SOLVE_TRACE_OBJECTIVE) != 0;
  bool rc_next = false;  // the next gradient runs on the 8 N M path (rowclu.cuh)
  int onepass = 0;
  for (int l = 0; l < o->outer_iters; ++l) {
    // ---- gradient of T^{l} (l = 0: T0 or p q^T) ----
    int mode;
    TSrc S;
    TSrc2 S2;
    if (l == 0) {
      if (T0) {
        mode = T_EXPLICIT;
        S = TSrc{reinterpret_cast<const float*>(T0), ldT, nullptr, nullptr, 0.0};
        S2 = TSrc2{reinterpret_cast<const float*>(T0), ldT, nullptr, nullptr, nullptr, nullptr, 0.f, 0.f};
      } else {
        mode = T_PRODUCT;
        S = TSrc{nullptr, 0, P.pn + P.row0, P.qn, 0.0};
        S2 = TSrc2{nullptr, 0, P.pnf + P.row0, nullptr, P.qnf, nullptr, 0.f, 0.f};
      }
    } else {
      mode = T_GIBBS;
      k_scale<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / es, Fs);
      k_scale<<<grid_for(m), 256, 0, c->stream>>>(s.g, m, GW_LOG2E / es, Gs2);
      KCHECK();
      S = TSrc{G, ldG, Fs, Gs2, GW_LOG2E / es};
      // fp32 hi/lo split of the duals: the Sinkhorn state (fh, fl, gh, gl) is consistent with (f, g)
      const double cc = GW_LOG2E / es;
      const float ch = (float)cc;
      S2 = TSrc2{G, ldG, s.fh, s.fl, s.gh, s.gl, ch, (float)(cc - (double)ch)};
    }
    const bool obj = (l > 0) && want_trace_obj;
    const bool exporting = ex.iter == l + 1;
    if (exporting && ex.T) {  // debug export: the plan T^{l} this gradient is evaluated on
      if (mode == T_EXPLICIT) {
        CU(cudaMemcpy2DAsync(ex.T, ex.ld * 4, T0, ldT * 4, m * 4, nl, cudaMemcpyDeviceToDevice, c->stream));
      } else if (mode == T_PRODUCT) {
        TRY(materialize(c, P, T_PRODUCT, S, ex.T, ex.ld));
      } else {
        TRY(materialize(c, P, T_GIBBS, S, ex.T, ex.ld));
      }
    }
    CU(cudaEventRecord(evs[2 * l], c->stream));
    if (tau_mode && obj) {  // objective of T^l first, then the cost over the buffer it reads
      TRY(grad_pass(c, P, mode, S, S2, nullptr, 0, false, true, fx, fy, alpha, objout));
      TRY(grad_pass(c, P, mode, S, S2, G, ldG, true, false, fx, fy, alpha, nullptr, beta));
    } else if (mode == T_GIBBS && rc_next && !obj) {
      TRY(grad_rc(c, P, s, G, ldG, S2));  // one read + one write (rowclu.cuh)
      ++onepass;
    } else if (mode == T_PRODUCT && P.k == 1 && !P.grid2d && !fx && !tau_mode && !obj) {
      TRY(grad_product(c, P, G, ldG));  // closed form on T^0 = p q^T: one write
    } else {
      TRY(grad_pass(c, P, mode, S, S2, G, ldG, true, obj, fx, fy, alpha, objout, beta));
    }
    CU(cudaEventRecord(evs[2 * l + 1], c->stream));
    if (exporting && ex.G)  // debug export: the solver's own stored cost G^{l+1} = grad E(T^l)
      CU(cudaMemcpy2DAsync(ex.G, ex.ld * 4, G, ldG * 4, m * 4, nl, cudaMemcpyDeviceToDevice, c->stream));
    if (obj) {
      CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      const double E = c->hpin[0];
      tr[(size_t)(l - 1) * 4 + 0] = fx ? (1.0 - alpha) * c->hpin[6] + alpha * E : E;
      tr[(size_t)(l - 1) * 4 + 1] = c->hpin[1];
    }
    // ---- Sinkhorn on G^{l+1} with warm-started duals ----
    TRY(sink_split(c, P, s, es));
    int used = 0, conv = 0;
    // the next gradient on the 8 N M path needs the XM sweep as this inner loop's last iteration
    const bool want_xm = s.rcCL > 0 && l + 1 < o->outer_iters && !tau_mode && !fx && !want_trace_obj;
    TRY(sink_run(c, P, s, G, ldG, es, o->inner.max_iter, o->inner.tol, o->inner.check_every, &used, &conv,
                 l == 0, 1.0, want_xm));
    rc_next = false;
    if (want_xm) {  // did it run and commit? (one 4-byte read per outer iteration)
      int* hx = reinterpret_cast<int*>(c->hpin + 48);
      CU(cudaMemcpyAsync(hx, s.xmv, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      rc_next = hx[0] == 1;
    }
    inner_total += used;
    if (o->inner.tol > 0 && !conv) conv_all = 0;
    tr[(size_t)l * 4 + 2] = used;
  }
  CU(cudaEventRecord(evs[2 * (size_t)o->outer_iters], c->stream));
  // ---- final plan T^L: objective, violation, entropy (one read-only gradient pass) ----
  double E = 0.0, viol = 0.0, H = 0.0, ecc = 0.0;
  if (nl > 0) {
    int mode;
    TSrc S;
    if (o->outer_iters == 0) {
      if (T0) { mode = T_EXPLICIT; S = TSrc{reinterpret_cast<const float*>(T0), ldT, nullptr, nullptr, 0.0}; }
      else { mode = T_PRODUCT; S = TSrc{nullptr, 0, P.pn + P.row0, P.qn, 0.0}; }
    } else {
      mode = T_GIBBS;
      k_scale<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / es, Fs);
      k_scale<<<grid_for(m), 256, 0, c->stream>>>(s.g, m, GW_LOG2E / es, Gs2);
      KCHECK();
      S = TSrc{G, ldG, Fs, Gs2, GW_LOG2E / es};
    }
    TSrc2 S2{};
    if (mode == T_EXPLICIT) {
      S2 = TSrc2{reinterpret_cast<const float*>(T0), ldT, nullptr, nullptr, nullptr, nullptr, 0.f, 0.f};
    } else if (mode == T_PRODUCT) {
      S2 = TSrc2{nullptr, 0, P.pnf + P.row0, nullptr, P.qnf, nullptr, 0.f, 0.f};
    } else {
      const double cc = GW_LOG2E / es;
      const float ch = (float)cc;
      S2 = TSrc2{G, ldG, s.fh, s.fl, s.gh, s.gl, ch, (float)(cc - (double)ch)};
    }
    TRY(grad_pass(c, P, mode, S, S2, nullptr, 0, false, true, fx, fy, alpha, objout));
    // outer_iters == 0 with an explicit T0: the returned plan IS T0 (S has no duals to regenerate from)
    if (T_out && mode == T_EXPLICIT) CU(cudaMemcpy2DAsync(T_out, ldT * 4, T0, ldT * 4, m * 4, nl,
                                                          cudaMemcpyDeviceToDevice, c->stream));
    else if (T_out) TRY(materialize(c, P, mode, S, T_out, ldT));
    CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  int fused_total = 0;
  if (o->outer_iters > 0) CU(cudaMemcpyAsync(c->hpin + 32, s.mode, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaEventRecord(ev1, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (o->outer_iters > 0) fused_total = reinterpret_cast<int*>(c->hpin + 32)[1];
  if (nl > 0) {
    E = c->hpin[0]; viol = c->hpin[1]; H = c->hpin[3]; ecc = c->hpin[6];
  }
  if (nl > 0 && !(std::isfinite(E) && std::isfinite(H) && std::isfinite(viol)))
    return fail(GW_ERR_NONFINITE, "non-finite result (E = %g, H = %g, violation = %g): eps too small for the "
                "cost scale, or non-finite inputs", E, H, viol);
  const double Eout = fx ? (1.0 - alpha) * ecc + alpha * E : E;
  if (o->outer_iters > 0) {
    tr[(size_t)(o->outer_iters - 1) * 4 + 0] = Eout;
    tr[(size_t)(o->outer_iters - 1) * 4 + 1] = viol;
  }
  for (int l = 0; l < o->outer_iters; ++l) {
    float a = 0.f, b = 0.f;
    CU(cudaEventElapsedTime(&a, evs[2 * l], evs[2 * l + 1]));
    CU(cudaEventElapsedTime(&b, evs[2 * l + 1], evs[2 * l + 2]));
    ms_grad += a;
    ms_sink += b;
    tr[(size_t)l * 4 + 3] = a + b;
  }
  float ms_total = 0.f;
  CU(cudaEventElapsedTime(&ms_total, ev0, ev1));
  res->gw_objective = Eout;
  res->entropic_objective = Eout + eps * H;
  res->marginal_violation = viol;
  res->outer_iters = o->outer_iters;
  res->inner_iters_total = inner_total;
  res->converged = (o->inner.tol > 0) ? conv_all : 0;
  res->inner_fused_total = fused_total;
  res->ms_grad = ms_grad;
  res->ms_sinkhorn = ms_sink;
  res->ms_total = ms_total;
  res->grad_onepass_total = onepass;
  if (trace) memcpy(trace, tr.data(), sizeof(double) * 4 * (size_t)o->outer_iters);
  TRY(stage_duals_out(c, pb, P, f, g, s.f, s.g));
  return GW_OK;
}

extern "C" gw_status gw_solve_set_export(gw_ctx* c, int32_t outer_iter, void* T_prev, void* G_out, int64_t ld) {
  if (!c) return fail(GW_ERR_INVALID_ARG, "null ctx");
  if (outer_iter < 0) return fail(GW_ERR_CONFIG, "export: outer_iter must be >= 0 (0 clears)");
  if (outer_iter > 0 && !T_prev && !G_out) return fail(GW_ERR_INVALID_ARG, "export: both buffers are null");
  if (T_prev && (ld % 4 != 0 || (reinterpret_cast<uintptr_t>(T_prev) & 15)))
    return fail(GW_ERR_INVALID_ARG, "export: T_prev needs ld %% 4 == 0 and a 16-byte aligned base");
  if (G_out && (ld % 4 != 0 || (reinterpret_cast<uintptr_t>(G_out) & 15)))
    return fail(GW_ERR_INVALID_ARG, "export: G_out needs ld %% 4 == 0 and a 16-byte aligned base");
  c->exp.iter = outer_iter;
  c->exp.T = T_prev;
  c->exp.G = G_out;
  c->exp.ld = ld;
  return GW_OK;
}

extern "C" gw_status entropic_gw_solve(gw_ctx* c, const gw_problem* pb, const gw_solve_opts* o, const void* T0,
                                       void* T_out, int64_t ldT, double* f, double* g, gw_result* res,
                                       double* trace) {
  return solve_impl(c, pb, o, nullptr, nullptr, 1.0, T0, T_out, ldT, f, g, res, trace);
}

extern "C" gw_status fgw_solve(gw_ctx* c, const gw_problem* pb, const double* fx, const double* fy, double alpha,
                               const gw_solve_opts* o, const void* T0, void* T_out, int64_t ldT, double* f,
                               double* g, gw_result* res, double* trace) {
  if (!fx || !fy) return fail(GW_ERR_INVALID_ARG, "fgw_solve: fx and fy must be non-null");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(GW_ERR_CONFIG, "fgw_solve: alpha must be in [0, 1]");
  return solve_impl(c, pb, o, fx, fy, alpha, T0, T_out, ldT, f, g, res, trace);
}

// ------------------------------------------------------------------------------ UGW (f4)
// (D o D) w for the 1-D power-k distance: the even power 2k by moments (polyk.cuh)
static gw_status dd_const(gw_ctx* c, int k, const double* s, const double* w, int64_t n, double* out) {
  switch (k) {
    case 1: k_gk_const<2><<<1, 1024, 0, c->stream>>>(s, w, n, out); break;
    case 2: k_gk_const<4><<<1, 1024, 0, c->stream>>>(s, w, n, out); break;
    case 3: k_gk_const<6><<<1, 1024, 0, c->stream>>>(s, w, n, out); break;
    case 4: k_gk_const<8><<<1, 1024, 0, c->stream>>>(s, w, n, out); break;
    default: k_gk_const<10><<<1, 1024, 0, c->stream>>>(s, w, n, out); break;
  }
  KCHECK();
  return GW_OK;
}

struct UgwStats {
  double mass, A1, B1, KL;  // m(T), <a, log(a/u)>, <b, log(b/v)>, <T, log(T/(u v))>
};

// Statistics of the implicit plan T = 2^(((f' + g' - C) log2e / eps_t)) (absorbed duals in s):
// a = T 1, b = T^T 1 (device, into a_out / b_out) and the scalars (host).
static gw_status ugw_stats(gw_ctx* c, const Prepared& P, SinkState& s, const float* C, int64_t ldC, double eps_t,
                           double* a_out, double* b_out, UgwStats* st) {
  const int64_t nl = P.nl, m = P.m;
  const double cc = GW_LOG2E / eps_t;
  const float ch = (float)cc;
  const TSrc2 S2{C, ldC, s.fh, s.fl, s.gh, s.gl, ch, (float)(cc - (double)ch)};
  double *ct, *part, *rpart, *sc;
  TRY(ws(c, c->ugct, (size_t)std::max<int64_t>(nl, 1), &ct));
  // one read of the cost (k_ugw_moments): per 256-column strip row partials of a and ct, per 256-row
  // block column partials of b, then fixed-order sums over the strips / blocks
  const int nblk = (int)((nl + TR - 1) / TR), nstr = (int)((m + TC - 1) / TC);
  TRY(ws(c, c->ugpart, (size_t)std::max(nblk, 1) * m, &part));
  TRY(ws(c, c->ugrpart, 2 * (size_t)nstr * (size_t)std::max<int64_t>(nl, 1), &rpart));
  TRY(ws(c, c->ugsc, 8, &sc));
  if (nl > 0) {
    k_ugw_moments<<<dim3((unsigned)nstr, (unsigned)nblk), 256, 0, c->stream>>>(S2, nl, m, P.xc + P.row0, P.yc, rpart,
                                                                                rpart + (size_t)nstr * nl, part);
    KCHECK();
    k_g2_colsum_reduce<<<grid_for(nl), 256, 0, c->stream>>>(rpart, nstr, nl, a_out);
    k_g2_colsum_reduce<<<grid_for(nl), 256, 0, c->stream>>>(rpart + (size_t)nstr * nl, nstr, nl, ct);
    KCHECK();
  }
  k_g2_colsum_reduce<<<grid_for(m), 256, 0, c->stream>>>(part, nl > 0 ? nblk : 0, m, b_out);
  KCHECK();
  if (P.R > 1) {  // b over every rank's rows, summed in rank order
    double* gb;
    TRY(ws(c, c->xvec, (size_t)m * (P.R + 1), &gb));
    TRY(comm_allgather(c, b_out, gb, sizeof(double) * (size_t)m));
    k_gk_ranks<<<grid_for(m), 256, 0, c->stream>>>(gb, P.R, P.rank, m, gb + (size_t)m * P.R, b_out);
    KCHECK();
  }
  k_ugw_scalars<<<1, 1024, 0, c->stream>>>(a_out, P.lp + P.row0, s.f, ct, nl, b_out, P.lq, s.g, m, sc);
  KCHECK();
  // the row sums (entries 0, 1, 3, 5, 6) add over the ranks; the column sums (2, 4, 7) are replicated
  double* gsc;
  TRY(ws(c, c->xpart, 8 * (size_t)(P.R + 1), &gsc));
  TRY(comm_allgather(c, sc, gsc, 8 * sizeof(double)));
  CU(cudaMemcpyAsync(c->hpin, gsc, 8 * sizeof(double) * P.R, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  double h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = 0; r < P.R; ++r)
    for (int k : {0, 1, 3, 5, 6}) h[k] += c->hpin[8 * r + k];
  for (int k : {2, 4, 7}) h[k] = c->hpin[k];
  st->mass = h[0];
  st->A1 = h[1];
  st->B1 = h[2];
  st->KL = (h[3] + h[4] - h[5]) / eps_t - h[6] - h[7];
  return GW_OK;
}

// A per-row vector of this rank's rows -> the full vector on every rank (padded all-gather)
static gw_status ugw_gather_rows(gw_ctx* c, const Prepared& P, const double* local, double* full) {
  if (P.R == 1) {
    if (local != full) CU(cudaMemcpyAsync(full, local, sizeof(double) * (size_t)P.nl, cudaMemcpyDeviceToDevice,
                                          c->stream));
    return GW_OK;
  }
  const int64_t ml = P.maxnl;
  double* g;
  TRY(ws(c, c->xg2, (size_t)ml * (P.R + 1), &g));
  double* pk = g + (size_t)ml * P.R;
  CU(cudaMemsetAsync(pk, 0, sizeof(double) * (size_t)ml, c->stream));
  CU(cudaMemcpyAsync(pk, local, sizeof(double) * (size_t)P.nl, cudaMemcpyDeviceToDevice, c->stream));
  TRY(comm_allgather(c, pk, g, sizeof(double) * (size_t)ml));
  k_unpad<<<grid_for(ml), 256, 0, c->stream>>>(g, P.R, ml, P.dtab, full);
  KCHECK();
  return GW_OK;
}

// F_eps (reading R33) from E and the plan statistics (m(u) = m(v) = 1)
// R33 with KL(x (x) x | y (x) y) = 2 m(x) <x, log(x/y)> - m(x)^2 + m(y)^2; mu = m(u), mv = m(v)
static double ugw_F(double E, const UgwStats& st, double rho, double eps, double mu, double mv) {
  const double mm = st.mass;
  return E + rho * (2.0 * mm * st.A1 - mm * mm + mu * mu) + rho * (2.0 * mm * st.B1 - mm * mm + mv * mv) +
         eps * (2.0 * mm * st.KL - mm * mm + (mu * mv) * (mu * mv));
}

// Entropic UGW (Remark 3) with readings R32-R35: per outer iteration
//   C = grad E(T^) [realised marginals] + 2 g(T^)   (twice the paper's 1/2 grad E + g: the same
//       subproblem at 2 m(T^) eps and 2 m(T^) rho)
//   unbalanced Sinkhorn (kappa = rho / (rho + eps)) on C with warm-started duals, safe path
//   T^ <- sqrt(m(T^) / m(T)) T.
static gw_status ugw_impl(gw_ctx* c, const gw_problem* pb, double rho, const gw_solve_opts* o, const void* T0,
                          void* T_out, int64_t ldT, double* f, double* g, gw_result* res, double* trace) {
  if (!c || !o || !res) return fail(GW_ERR_INVALID_ARG, "null ctx, opts or result");
  if (!(o->eps > 0)) return fail(GW_ERR_CONFIG, "eps must be > 0");
  if (!(rho > 0) || !std::isfinite(rho)) return fail(GW_ERR_CONFIG, "ugw_solve: rho must be finite and > 0");
  if (o->tau != o->eps && o->tau != 0) return fail(GW_ERR_UNSUPPORTED, "tau != eps is not implemented (R6)");
  if (o->outer_iters < 0 || o->inner.max_iter < 0) return fail(GW_ERR_CONFIG, "iteration counts must be >= 0");
  if (!f || !g) return fail(GW_ERR_INVALID_ARG, "f and g (outputs) must be non-null");
  if (T0) return fail(GW_ERR_UNSUPPORTED, "ugw_solve: the iteration starts from u v (R35); T0 must be null");
  if (o->inner.tol > 0) return fail(GW_ERR_UNSUPPORTED, "ugw_solve: fixed inner iteration counts only");
  TRY(check_problem(pb));
  if (pb->flags & GW_GRID2D) return fail(GW_ERR_UNSUPPORTED, "ugw_solve: 2-D grids are not implemented");
  if (pb->dtype != GW_F32) return fail(GW_ERR_UNSUPPORTED, "ugw_solve: fp32 storage only");
  if (T_out) TRY(check_matrix(T_out, ldT, pb->m, "T_out"));
  CU(cudaSetDevice(c->device));
  const double eps = o->eps;
  Prepared P;
  TRY(prepare(c, pb, P, true));
  const double mu = P.mass_p, mv = P.mass_q, m0 = std::sqrt(mu * mv);
  const int64_t nl = P.nl, m = P.m;
  const int64_t ldG = (m + 31) & ~int64_t(31);
  float* G;
  TRY(ws(c, c->Gs, (size_t)std::max<int64_t>(nl, 1) * ldG, &G));
  SinkState s;
  SinkGuard sguard{s};
  TRY(sink_alloc(c, P, s));
  if (pb->flags & GW_HOST_VECTORS) {
    TRY(stage_duals_in(c, pb, P, nullptr, nullptr, &s.f, &s.g));
  } else {
    s.f = f;
    s.g = g;
  }
  double *av, *bv, *ca, *cb, *fr, *gr, *Fs, *Gs2, *objout, *afull;
  const int64_t n = P.n;
  TRY(ws(c, c->uga, (size_t)std::max<int64_t>(nl, 1) + (size_t)n, &av)); TRY(ws(c, c->ugb, (size_t)m, &bv));
  afull = av + std::max<int64_t>(nl, 1);
  TRY(ws(c, c->ugca, (size_t)n, &ca)); TRY(ws(c, c->ugcb, (size_t)m, &cb));
  TRY(ws(c, c->ugfr, (size_t)std::max<int64_t>(nl, 1), &fr)); TRY(ws(c, c->uggr, (size_t)m, &gr));
  TRY(ws(c, c->fsc, (size_t)std::max<int64_t>(nl, 1), &Fs)); TRY(ws(c, c->gsc, (size_t)m, &Gs2));
  TRY(ws(c, c->objout, 16, &objout));
  k_fill<<<grid_for(nl), 256, 0, c->stream>>>(fr, nl, 0.0);
  k_fill<<<grid_for(m), 256, 0, c->stream>>>(gr, m, 0.0);
  KCHECK();
  const bool want_trace_obj = (o->flags & GW_SOLVE_TRACE_OBJECTIVE) != 0;
  std::vector<double> tr((size_t)std::max(o->outer_iters, 1) * 4, NAN);
  EventSet evset;
  cudaEvent_t ev0, ev1;
  CU(evset.make(&ev0)); CU(evset.make(&ev1));
  CU(cudaEventRecord(ev0, c->stream));
  // T^0 = u v / m0, m0 = sqrt(m(u) m(v)) (R35): a = u sqrt(mv/mu), b = v sqrt(mu/mv), m(T^0) = m0
  UgwStats st{m0, 0.5 * m0 * std::log(mv / mu), 0.5 * m0 * std::log(mu / mv), -0.5 * m0 * std::log(mu * mv)};
  // the product form of T^0 for the gradient kernels: rows u / m0 (local, fp64 in Fs and fp32 in s.fh,
  // both free until the first Sinkhorn split), columns v
  auto product_src = [&](TSrc& S, TSrc2& S2) -> gw_status {
    k_scale<<<grid_for(nl), 256, 0, c->stream>>>(P.pn + P.row0, nl, 1.0 / m0, Fs);
    k_scale_f<<<grid_for(nl), 256, 0, c->stream>>>(P.pn + P.row0, nl, 1.0 / m0, s.fh);
    KCHECK();
    S = TSrc{nullptr, 0, Fs, P.qn, 0.0};
    S2 = TSrc2{nullptr, 0, s.fh, nullptr, P.qnf, nullptr, 0.f, 0.f};
    return GW_OK;
  };
  double eps_reg = 0.0;  // regulariser of the current implicit plan (l > 0)
  int inner_total = 0;
  // E of the current plan (objective pass on the Gibbs form, realised marginals)
  auto plan_E = [&](double* Eout, double* violout) -> gw_status {
    const double cc = GW_LOG2E / eps_reg;
    const float ch = (float)cc;
    k_scale<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, cc, Fs);
    k_scale<<<grid_for(m), 256, 0, c->stream>>>(s.g, m, cc, Gs2);
    KCHECK();
    const TSrc S{G, ldG, Fs, Gs2, cc};
    const TSrc2 S2{G, ldG, s.fh, s.fl, s.gh, s.gl, ch, (float)(cc - (double)ch)};
    TRY(grad_pass(c, P, T_GIBBS, S, S2, nullptr, 0, false, true, nullptr, nullptr, 1.0, objout));
    CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *Eout = c->hpin[0];
    if (violout) *violout = c->hpin[1];
    return GW_OK;
  };
  for (int l = 0; l < o->outer_iters; ++l) {
    // ---- cost C = grad E(T^) (realised a, b) + 2 g(T^) (R32) ----
    const double gconst = rho * st.A1 + rho * st.B1 + eps * st.KL;
    if (l > 0) {
      TRY(ugw_gather_rows(c, P, av, afull));
    } else {  // T^0: a = u sqrt(mv/mu) (all rows), b = v sqrt(mu/mv)
      k_scale<<<grid_for(n), 256, 0, c->stream>>>(P.pn, n, std::sqrt(mv / mu), afull);
      k_scale<<<grid_for(m), 256, 0, c->stream>>>(P.qn, m, std::sqrt(mu / mv), bv);
      KCHECK();
    }
    const double* aw = afull;
    const double* bw = bv;
    TRY(dd_const(c, P.k, P.xc, aw, n, ca));
    TRY(dd_const(c, P.k, P.yc, bw, m, cb));
    k_ugw_addc<<<grid_for(n), 256, 0, c->stream>>>(ca, gconst, n);
    KCHECK();
    Prepared P2 = P;
    P2.cx = ca;
    P2.cy = cb;
    int mode;
    TSrc S;
    TSrc2 S2;
    if (l == 0) {
      mode = T_PRODUCT;
      TRY(product_src(S, S2));
    } else {
      mode = T_GIBBS;
      const double cc = GW_LOG2E / eps_reg;
      const float ch = (float)cc;
      k_scale<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, cc, Fs);
      k_scale<<<grid_for(m), 256, 0, c->stream>>>(s.g, m, cc, Gs2);
      KCHECK();
      S = TSrc{G, ldG, Fs, Gs2, cc};
      S2 = TSrc2{G, ldG, s.fh, s.fl, s.gh, s.gl, ch, (float)(cc - (double)ch)};
    }
    TRY(grad_pass(c, P2, mode, S, S2, G, ldG, true, false, nullptr, nullptr, 1.0, nullptr));
    // ---- unbalanced Sinkhorn at eps~ = 2 m eps, rho~ = 2 m rho (R34), absorbed duals f' = f + eps~ ln u ----
    const double eps_t = 2.0 * st.mass * eps, rho_t = 2.0 * st.mass * rho;
    const double kap = rho_t / (rho_t + eps_t);
    const float c2f = (float)(GW_LOG2E / eps_t);
    k_ugw_axpy<<<grid_for(nl), 256, 0, c->stream>>>(fr, P.lp + P.row0, eps_t, nl, s.f);
    k_ugw_axpy<<<grid_for(m), 256, 0, c->stream>>>(gr, P.lq, eps_t, m, s.g);
    KCHECK();
    TRY(sink_split(c, P, s, eps_t));
    // the unbalanced subproblem on the hot path's Sinkhorn machinery: the one-read fused iteration
    // (speculative, validated on the device, falling back to the safe two-kernel path), the
    // cluster-resident loop for small problems, CUDA graphs / one collective per slot -- kappa
    // carried through every update (R34)
    int used = 0, conv = 0;
    TRY(sink_run(c, P, s, G, ldG, eps_t, o->inner.max_iter, 0.0, 10, &used, &conv, l == 0, kap));
    inner_total += o->inner.max_iter;
    // relative duals for the warm start (R34), then the mass rescaling (R35)
    k_ugw_axpy<<<grid_for(nl), 256, 0, c->stream>>>(s.f, P.lp + P.row0, -eps_t, nl, fr);
    k_ugw_axpy<<<grid_for(m), 256, 0, c->stream>>>(s.g, P.lq, -eps_t, m, gr);
    KCHECK();
    UgwStats sn;
    TRY(ugw_stats(c, P, s, G, ldG, eps_t, av, bv, &sn));
    const double scl = std::sqrt(st.mass / sn.mass), lsc = std::log(scl);
    k_ugw_addc<<<grid_for(nl), 256, 0, c->stream>>>(s.f, eps_t * lsc, nl);
    k_scale<<<grid_for(nl), 256, 0, c->stream>>>(av, nl, scl, av);
    k_scale<<<grid_for(m), 256, 0, c->stream>>>(bv, m, scl, bv);
    KCHECK();
    k_split<<<grid_for(nl), 256, 0, c->stream>>>(s.f, nl, GW_LOG2E / eps_t, s.fh, s.fl);
    KCHECK();
    st.mass = scl * sn.mass;
    st.A1 = scl * (sn.A1 + lsc * sn.mass);
    st.B1 = scl * (sn.B1 + lsc * sn.mass);
    st.KL = scl * (sn.KL + lsc * sn.mass);
    eps_reg = eps_t;
    tr[(size_t)l * 4 + 2] = o->inner.max_iter;
    tr[(size_t)l * 4 + 3] = st.mass;
    if (want_trace_obj && l + 1 < o->outer_iters) {
      double E;
      TRY(plan_E(&E, nullptr));
      tr[(size_t)l * 4 + 0] = ugw_F(E, st, rho, eps, mu, mv);
      tr[(size_t)l * 4 + 1] = E;
    }
  }
  // ---- final plan: E, F, violation (vs u, v; informational) ----
  double E = 0.0, viol = 0.0;
  if (o->outer_iters == 0) {
    TSrc S;
    TSrc2 S2;
    TRY(product_src(S, S2));
    TRY(grad_pass(c, P, T_PRODUCT, S, S2, nullptr, 0, false, true, nullptr, nullptr, 1.0, objout));
    CU(cudaMemcpyAsync(c->hpin, objout, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    E = c->hpin[0];
    viol = c->hpin[1];
    if (T_out) TRY(materialize(c, P, T_PRODUCT, S, T_out, ldT));
  } else {
    TRY(plan_E(&E, &viol));
    if (T_out) TRY(materialize(c, P, T_GIBBS, TSrc{G, ldG, Fs, Gs2, GW_LOG2E / eps_reg}, T_out, ldT));
  }
  const double F = ugw_F(E, st, rho, eps, mu, mv);
  if (o->outer_iters > 0) {
    tr[(size_t)(o->outer_iters - 1) * 4 + 0] = F;
    tr[(size_t)(o->outer_iters - 1) * 4 + 1] = E;
  }
  // the returned duals are the subproblem's final ones in R34's convention (relative to u v)
  CU(cudaMemcpyAsync(s.f, fr, nl * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemcpyAsync(s.g, gr, m * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (o->outer_iters > 0) CU(cudaMemcpyAsync(c->hpin + 32, s.mode, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaEventRecord(ev1, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  const int ugw_fused = o->outer_iters > 0 ? reinterpret_cast<int*>(c->hpin + 32)[1] : 0;
  float ms_total = 0.f;
  CU(cudaEventElapsedTime(&ms_total, ev0, ev1));
  res->grad_onepass_total = 0;
  res->gw_objective = E;
  res->entropic_objective = F;
  res->marginal_violation = viol;
  res->outer_iters = o->outer_iters;
  res->inner_iters_total = inner_total;
  res->converged = 0;
  res->inner_fused_total = o->outer_iters > 0 ? ugw_fused : 0;
  res->ms_grad = 0.0;
  res->ms_sinkhorn = 0.0;
  res->ms_total = ms_total;
  if (trace) memcpy(trace, tr.data(), sizeof(double) * 4 * (size_t)o->outer_iters);
  TRY(stage_duals_out(c, pb, P, f, g, s.f, s.g));
  return GW_OK;
}

extern "C" gw_status ugw_solve(gw_ctx* c, const gw_problem* pb, double rho, const gw_solve_opts* o, const void* T0,
                               void* T_out, int64_t ldT, double* f, double* g, gw_result* res, double* trace) {
  return ugw_impl(c, pb, rho, o, T0, T_out, ldT, f, g, res, trace);
}

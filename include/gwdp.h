/*
 * gwdp.h -- C ABI of the B200-native FGC entropic Gromov-Wasserstein hot path.
 *
 * Paper: "Efficient Gradient Computation for Gromov-Wasserstein" style FGC-GW,
 * arXiv 2404.08970 (PAPER.md in the reference).  Citations below are
 * "PAPER.md:<line>" (the paper's LaTeX source) and "SPEC.md:<line>".
 *
 * Problem (notation of SURVEY.md §0.3 / BASELINE.json):
 *   x in R^n (rows, marginal p), y in R^m (columns, marginal q), both
 *   NON-DECREASING; D_X[i,j] = |x_i - x_j|^k, D_Y[p,q] = |y_p - y_q|^k
 *   (generalised to sorted supports: reading R1 in DESIGN.md);
 *   plan T (n x m, the paper's Gamma), row-major.
 *   GW gradient (transpose typo fixed, reading R3):
 *     G = 2 (c 1^T + 1 c'^T) - 4 D_X T D_Y,  c = (D_X o D_X) p,  c' = (D_Y o D_Y) q.
 *   Entropic GW by mirror descent with tau = eps by default
 *   (Remark 1 PAPER.md:127-133; tau != eps: gw_solve_opts):
 *     T^l = argmin_{T in S(p,q)} <G(T^{l-1}), T> + eps H(T),  solved by log-domain
 *     Sinkhorn: f_i = eps ln p_i - eps LSE_p((g_p - G_ip)/eps),
 *               g_p = eps ln q_p - eps LSE_i((f_i - G_ip)/eps),
 *     T_ip = exp((f_i + g_p - G_ip)/eps).
 *
 * Conventions (all entry points):
 *   - Every pointer is a DEVICE pointer on ctx's device unless the problem's
 *     flags contain GW_HOST_VECTORS (then x, y, p, q, f, g, fx, fy are HOST
 *     pointers and the library stages them; N x M matrices are always device).
 *     The caller owns every argument; the library never frees or retains them.
 *   - N x M matrices: row-major fp32 (gw_dtype GW_F32), leading dimension
 *     ld >= m, ld % 4 == 0, 16-byte aligned base.  A rank holds only its
 *     n_local rows [row0, row0 + n_local).  Only the elements [0, n_local) x
 *     [0, m) of an output matrix are written: its padding columns [m, ld) and
 *     anything outside its rows are left untouched (tests/test_gpu_canary.py).
 *   - Work is enqueued on ctx's stream.  Calls that fill host structs
 *     (info, res, trace) synchronise that stream before returning.
 *   - Errors: a status is returned; no exception or abort crosses the ABI;
 *     gw_last_error() returns a thread-local message.  Argument and validation
 *     errors are detected before any output is written.  Asynchronous CUDA
 *     faults surface as GW_ERR_CUDA at the next synchronising call.
 *     Sinkhorn not reaching tol within max_iter is NOT an error
 *     (converged = 0).
 *   - Inputs are never mutated; marginals within 1e-9 of unit mass are
 *     renormalised in an internal copy.
 *   - Results are bitwise reproducible for fixed inputs, sizes and world size
 *     (fixed-order reductions, no float atomics on result paths).
 *   - Execution routes chosen inside (same results within the stated tolerances): the fused
 *     one-read Sinkhorn iteration with a device-validated safe fallback; for fixed iteration
 *     counts on one rank a cluster-resident kernel when G fits in one thread-block cluster's
 *     shared memory, else one CUDA graph replay per iteration; chunks of fused steps on
 *     several ranks.  Env switches (diagnostics only): GWDP_NO_SMALL, GWDP_NO_GRAPH,
 *     GWDP_NO_FUSED; GWDP_FAULT=carry|colsum is a test-only fault injection.
 */
#ifndef GWDP_H
#define GWDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GWDP_ABI_VERSION 2

typedef struct gw_ctx gw_ctx;    /* opaque: device, stream, workspace, optional comm */
typedef struct gw_comm gw_comm;  /* opaque: NCCL communicator, rank, world size      */

typedef enum {
  GW_OK = 0,
  GW_ERR_INVALID_ARG = 1,     /* null pointer, bad size, bad ld / alignment, eps <= 0 */
  GW_ERR_DIM_MISMATCH = 2,    /* shard does not fit (row0 + n_local > n)              */
  GW_ERR_UNSORTED = 3,        /* x or y not non-decreasing (reading R16)              */
  GW_ERR_NEGATIVE_WEIGHT = 4, /* p or q has a negative entry             */
  GW_ERR_NOT_NORMALIZED = 5,  /* |sum - 1| > 1e-9                        */
  GW_ERR_NONFINITE = 6,       /* NaN/Inf in inputs or produced          */
  GW_ERR_CONFIG = 7,          /* invalid options                                       */
  GW_ERR_UNSUPPORTED = 8,     /* k > GW_MAX_K, loss != square, GW_F64 on 2-D grids, tau != eps off k = 1, ... */
  GW_ERR_OOM = 9,
  GW_ERR_CUDA = 10,
  GW_ERR_NCCL = 11
} gw_status;

typedef enum { GW_LOSS_SQUARE = 0 } gw_loss;       /* the only loss the paper defines */
/* Storage of every N x M matrix (T, G, T0, T_out, export buffers) of a call.  GW_F32: the bandwidth
 * path (C2-C5).  GW_F64 (C1 = BASELINE configs[0], SURVEY.md §8 sizes table): every matrix float64 and
 * every step in fp64 (the DP gradient as a row scan and a column scan, the log-domain Sinkhorn updates,
 * the objective) -- parity ~1e-12 with the float64 oracle; 1-D supports, k = 1..GW_MAX_K (2-D grids,
 * ugw_solve, tau != eps: GW_ERR_UNSUPPORTED).  The solver keeps its plan explicit then (two
 * fp64 N x M buffers).  Any other value: GW_ERR_INVALID_ARG. */
typedef enum { GW_F32 = 0, GW_F64 = 1 } gw_dtype;

/* problem flags */
#define GW_NO_VALIDATE     0x1u  /* skip sortedness / marginal checks (caller guarantees them) */
#define GW_HOST_VECTORS    0x2u  /* x, y, p, q (and f, g, fx, fy outputs/inputs) are host pointers */
/* 2-D tensor grids (Table 3): n = nx^2 points (a, b) -> row a nx + b
 * at (x[a], x[b]) with x the SORTED axis of length nx (likewise y with ny, m = ny^2), Manhattan
 * distance |x_a - x_a'| + |x_b - x_b'| (reading R31; the paper's uniform grid is x_a = a h).
 * k = 1, nx, ny <= 256; p (n) and q (m) as usual; rows shard as in 1-D (row0, n_local). */
#define GW_GRID2D          0x4u
/* largest distance power: k = 1 (gap-weighted scans), k = 2 (moments), 3..5 (power-sum scans,
 * PAPER.md:229-259) */
#define GW_MAX_K           5

typedef struct {
  int64_t n, m;           /* global sizes: x in R^n (rows), y in R^m (columns)        */
  int64_t row0, n_local;  /* this rank's row shard; (0, n) on one GPU                  */
  const double *x, *y;    /* supports, non-decreasing (length n and m)                 */
  const double *p, *q;    /* marginals, >= 0, sum 1 within 1e-9 (length n and m)       */
  int32_t k;              /* distance power |x - x'|^k: 1 (hot path) .. GW_MAX_K (R17, f2) */
  int32_t loss;           /* gw_loss */
  int32_t dtype;          /* gw_dtype: GW_F32, or GW_F64 (1-D supports)                 */
  uint32_t flags;         /* GW_NO_VALIDATE | GW_HOST_VECTORS | GW_GRID2D              */
} gw_problem;

/* Optional precomputed moments of T (device, fp64, the caller's coordinates; nullable argument of
 * gw_grad_dp, k = 1 on 1-D supports): the plan's row totals T 1 and T y over this rank's rows and its
 * column totals T^T 1 and T^T x over ALL rows.  When given they replace the totals the moments pass
 * reduces -- the rank-2 term -4[(D_X (T y))_i - (D_X (T 1))_i y_p] and the column totals' 1-D DPs of
 * PAPER.md:122-126 / 190-259 are formed from them -- while the pass itself still runs for the per-tile
 * partials that feed the carries.  All four must be non-null (GW_ERR_INVALID_ARG); k != 1 or 2-D grids:
 * GW_ERR_UNSUPPORTED. */
typedef struct {
  const double *row_sum, *row_ysum;   /* T 1, T y over this shard's rows       */
  const double *col_sum, *col_xsum;   /* T^T 1, T^T x over ALL rows            */
} gw_moments;

typedef struct {
  double eps;           /* entropic regulariser, > 0                   */
  int32_t max_iter;     /* Sinkhorn iterations (f-update + g-update pairs)           */
  double tol;           /* stop when marginal violation <= tol; <= 0: run max_iter    */
  int32_t check_every;  /* violation check period (iterations) when tol > 0           */
} gw_sinkhorn_opts;

typedef struct {
  int32_t iters;               /* iterations performed                                */
  int32_t converged;           /* 1 if violation <= tol was observed                   */
  int32_t fused_iters;         /* iterations that ran the fused one-read path            */
  double marginal_violation;   /* max(|T1 - p|_inf, |T^T 1 - q|_inf) of the final plan */
} gw_sinkhorn_info;

/* solve flags */
#define GW_SOLVE_TRACE_OBJECTIVE 0x1u  /* fill trace[l*4+0] = E(T^l) for every l (costs one
                                          moments+reduce pass for the last l only)        */

typedef struct {
  double eps, tau;            /* tau: the step's KL weight; 0 or eps =
                                 Remark 1's tau = eps; tau != eps (k = 1, 1-D, T0 = NULL):
                                 cost grad E + (eps - tau) ln T^l at regulariser tau (R6) */
  int32_t outer_iters;        /* mirror-descent iterations L                           */
  gw_sinkhorn_opts inner;     /* inner.eps is ignored (eps above is used)              */
  uint32_t flags;             /* GW_SOLVE_* */
} gw_solve_opts;

typedef struct {
  double gw_objective;        /* E(T^L), realised marginals (R13)          */
  double entropic_objective;  /* E(T^L) + eps H(T^L)                  */
  double marginal_violation;  /* of T^L                                                 */
  int32_t outer_iters, inner_iters_total, converged;
  int32_t inner_fused_total;  /* Sinkhorn iterations that ran the fused one-read path    */
  double ms_grad, ms_sinkhorn, ms_total;
  int32_t grad_onepass_total; /* gradients evaluated in one read of the cost + one write  */
                              /* (8 N M bytes): k = 1, one rank          */
} gw_result;

/* ---- context / communicator ------------------------------------------------------ */

/* Create a context on `device`, enqueuing on `cuda_stream` (a cudaStream_t; NULL =
 * the legacy default stream).  `comm` may be NULL (single GPU). */
gw_status gw_ctx_create(gw_ctx **out, int device, void *cuda_stream, gw_comm *comm);
gw_status gw_ctx_destroy(gw_ctx *ctx);
/* Release the context's workspace (it is re-grown lazily). */
gw_status gw_ctx_trim(gw_ctx *ctx);
/* Kernel-class timing with CUDA events on ctx's stream (for measurement harnesses).
 * enable: 0 off, 1 on, 2 on + reset totals.  out_ms / out_counts (host, nullable) receive
 * `nslots` entries: {grad_moments, grad_carry, grad_main, sink_row, sink_col, sink_fused,
 * objective_pass, -, grad_onepass, sink_xm} accumulated since the last reset (sink_col,
 * sink_fused and sink_xm count their two launches per iteration; objective_pass counts one per
 * final-objective pass; grad_onepass: the one-read gradient, its carries included, one per
 * gradient; sink_xm: the last Sinkhorn iteration of an inner loop on that path); slot 7 has no
 * time: out_counts[7] = all kernel launches of the library since the last reset.
 * Synchronises ctx's stream. */
gw_status gw_ctx_profile(gw_ctx *ctx, int enable, double *out_ms, int64_t *out_counts, int nslots);
const char *gw_last_error(void);
int gw_abi_version(void);

/* ---- row sharding ------------------------------------------
 * Rank r of R owns rows [row0_r, row0_r + n_local_r) of every N x M matrix (its gw_problem's
 * row0 / n_local); shards must be non-empty and consecutive in rank order.  x, y, p, q and g are
 * replicated, f is per shard.  Every rank calls the same entry points in the same order with
 * identical n, m, x, y, p, q and options (collective semantics).  The only collective the library
 * issues is an all-gather of equal-sized per-rank payloads (column sums per Sinkhorn iteration,
 * column / block-strip carries and row moments per gradient, a few scalars per objective);
 * payloads are combined in rank order, so results are identical on every rank and do not
 * depend on the transport. */

/* NCCL transport: rank 0 gets a 128-byte id, the caller broadcasts it (e.g. with
 * torch.distributed), every rank calls gw_comm_init with the same id.  Collectives are
 * enqueued on the ctx stream (asynchronous). */
gw_status gw_get_unique_id(unsigned char id[128]);
gw_status gw_comm_init(gw_comm **out, const unsigned char id[128], int nranks, int rank);

/* Host-callback transport (same sharded code path; used for testing without NVLink and for
 * any host-side process group): `allgather` receives `bytes` bytes from this rank in `send`
 * (host memory) and must fill `recv` with nranks * bytes bytes, rank r's contribution at offset
 * r * bytes; it returns 0 on success.  Called synchronously from the thread driving the ctx,
 * after the ctx stream has been synchronised. */
typedef int (*gw_allgather_fn)(const void *send, void *recv, int64_t bytes, void *user);
gw_status gw_comm_init_host(gw_comm **out, int nranks, int rank, gw_allgather_fn allgather, void *user);
gw_status gw_comm_destroy(gw_comm *comm);

/* Balanced row shard: the first n % nranks ranks get one more row.  Host only (no GPU). */
gw_status gw_shard_rows(int64_t n, int nranks, int rank, int64_t *row0, int64_t *n_local);
/* Validate a shard table (table[2r] = row0_r, table[2r+1] = n_local_r): consecutive in rank order
 * and covering [0, n).  GW_ERR_DIM_MISMATCH otherwise.  Host only. */
gw_status gw_check_shards(const int64_t *table, int nranks, int64_t n);

/* ---- hot path ----------------------------------------------------------------------- */

/* G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y for the rows [row0, row0 + n_local)
 * in O(n m) by the paper's dynamic programme
 * realised as row and column prefix scans with fp64 carries.  With a multi-rank ctx every rank
 * passes its own rows of T and receives its rows of G.
 * T: device fp32 (n_local x m, ldT); G: device fp32 output (ldG), may alias T; both fp64 with GW_F64
 * (ldG == ldT).  c, c' use the PRESCRIBED p, q (reading R4).  mom (nullable): the
 * plan's row / column totals (gw_moments above).  Asynchronous. */
gw_status gw_grad_dp(gw_ctx *ctx, const gw_problem *prob, const void *T, int64_t ldT,
                     void *G, int64_t ldG, const gw_moments *mom);

/* Log-domain Sinkhorn on cost G, never materialising
 * exp(-G/eps).  f (n_local) and g (m) are in/out fp64 duals (warm start; pass
 * zeros for a cold start).  T_out (nullable): the plan exp((f+g-G)/eps), fp32,
 * ldT (G and T_out fp64 with GW_F64).  info (host, nullable).  Iteration = f-update then g-update (reading R7). */
gw_status sinkhorn_solve(gw_ctx *ctx, const gw_problem *prob, const void *G, int64_t ldG,
                         const gw_sinkhorn_opts *opts, double *f, double *g,
                         void *T_out, int64_t ldT, gw_sinkhorn_info *info);

/* Entropic GW by mirror descent (tau = eps unless opts->tau says otherwise).
 * T0: initial plan (device fp32, nullable -> p (x) q, reading R5); T_out: final plan
 * (nullable); both fp64 with GW_F64.  f, g: final duals (f has n_local entries, g has m).  res (host,
 * required).  trace (host, nullable): [outer_iters x 4] doubles per outer l:
 * {E(T^l) (NaN unless GW_SOLVE_TRACE_OBJECTIVE), violation of T^l,
 *  Sinkhorn iterations used, milliseconds}.  The iteration counts let the oracle
 * replay the schedule (reading R8). */
gw_status entropic_gw_solve(gw_ctx *ctx, const gw_problem *prob, const gw_solve_opts *opts,
                            const void *T0, void *T_out, int64_t ldT, double *f, double *g,
                            gw_result *res, double *trace);

/* Debug export for parity checks of the solver's own gradients.
 * Arms a ONE-SHOT request consumed by the next entropic_gw_solve / fgw_solve on ctx: at outer
 * iteration `outer_iter` (1-based; 0 clears the request) the library writes
 *   T_prev (nullable): the plan T^{l-1} the l-th gradient is evaluated on (p q^T or T0 for l = 1,
 *                      else exp((f + g - G^{l-1})/eps) materialised from the solver's duals), and
 *   G_out  (nullable): the solver's stored cost G^l = grad E(T^{l-1}) (FGW:
 *                      its cost) exactly as the Sinkhorn iterations consume it.
 * Both are this rank's n_local x m rows, fp32 (fp64 when the solve's problem is GW_F64) row-major
 * with leading dimension ld in elements (ld % 4 == 0, 16-byte aligned).  The request is taken by the next solve call whatever its outcome; a solve with
 * fewer outer iterations writes nothing.  Errors: GW_ERR_INVALID_ARG (null ctx, both buffers null,
 * bad ld / alignment), GW_ERR_CONFIG (outer_iter < 0).  Costs one extra N x M write each (debug only). */
gw_status gw_solve_set_export(gw_ctx *ctx, int32_t outer_iter, void *T_prev, void *G_out, int64_t ld);

/* Fused GW (Remark 2): cost (1-alpha) C o C + alpha G with the
 * feature cost C_ip = |fx_i - fy_p| (never stored), objective
 * (1-alpha) <C o C, T> + alpha E(T).  fx (n), fy (m).  Same conventions as
 * entropic_gw_solve. */
gw_status fgw_solve(gw_ctx *ctx, const gw_problem *prob, const double *fx, const double *fy,
                    double alpha, const gw_solve_opts *opts, const void *T0, void *T_out,
                    int64_t ldT, double *f, double *g, gw_result *res, double *trace);

/* Entropic unbalanced GW (Remark 3).  The paper fixes the functional and the
 * per-iteration subproblem  min_{G >= 0} <1/2 grad E(G^) + g(G^), G> + m(G^)(rho KL(G1|u) +
 * rho KL(G^T 1|v) + eps KL(G|u v))  but leaves g(G^) undefined; this build takes readings
 * R32-R35: g = rho <log(a/u),a> + rho <log(b/v),b> + eps <log(G^/(uv)),G^>, the
 * gradient with the REALISED marginals a = G^1, b = G^T1, unbalanced Sinkhorn with
 * kappa = rho~/(rho~+eps~) (opts->inner.max_iter fixed iterations; tol must be 0), G^0 = u v and
 * the mass rescaling sqrt(m(G^)/m(G)) after each subproblem.
 *   prob     p = u, q = v: nonnegative measures of ANY positive mass (not normalised here; the
 *            |sum - 1| check of the balanced solvers is skipped, m(u), m(v) > 0 is required);
 *            G^0 = u v / sqrt(m(u) m(v)) (R35).
 *   rho      > 0 (finite); opts->eps > 0, opts->tau = eps or 0; T0 must be NULL.
 *   T_out    nullable: the final plan (fp32, ldT).  f, g: the subproblem's final duals in R34's
 *            convention (G = exp((f + g - C)/eps~) u v before the rescaling).
 *   res      gw_objective = E(G) (realised marginals), entropic_objective = F_eps(G) (R33),
 *            marginal_violation = max(|G1 - u|, |G^T1 - v|) (informational: G is unbalanced).
 *   trace    [outer][4] = {F_eps, E, inner iterations, m(G)} per outer iteration (F_eps, E only
 *            with GW_SOLVE_TRACE_OBJECTIVE, and always for the last one).
 * 1-D supports (k = 1..GW_MAX_K), row-sharded like the other solvers; 2-D grids or tol > 0 ->
 * GW_ERR_UNSUPPORTED. */
gw_status ugw_solve(gw_ctx *ctx, const gw_problem *prob, double rho, const gw_solve_opts *opts,
                    const void *T0, void *T_out, int64_t ldT, double *f, double *g,
                    gw_result *res, double *trace);

#ifdef __cplusplus
}
#endif
#endif /* GWDP_H */

/*
 * lp.h -- C ABI of the B200-native restarted-PDHG LP engine
 * (raPDHG and r2HPDHG of MPAX, arXiv 2412.09734), fp64, sm_100a.
 *
 * The problem (Eq. (1)):
 *     min c'x   s.t.   G x >= h,   A x = b,   l <= x <= u,
 * is handed over already stacked as in its saddle form Eq. (2):
 *     K = [G; A]  (rows 0..m1-1 are the ">=" rows, rows m1..m1+m2-1 the "=" rows),
 *     q = (h; b).
 * "<=" rows are negated by the caller.  l may hold -inf, u +inf.
 *
 * The solver implements the iteration contract written down in DESIGN.md §3
 * (= SURVEY.md §8(c) c.2): Ruiz + Pock-Chambolle preconditioning, PDHG
 * steps Eq. (pdhg) with the adaptive step size, averaging
 * (raPDHG) or Halpern reflection Eq. (hrpdhg) (r2HPDHG), checks of
 * termination / restart every 64 iterations, primal-weight
 * update on restart, warm start and batches of same-shape
 * instances; plus the SURVEY §8(f) rows: infeasibility detection with
 * certificate rays (reading 35), feasibility polishing
 * (reading 36), the SPO+ layer (reading 37, lp_spo_plus),
 * the constant-step / partial-reflection variants (readings 34, 38), fp32 storage on the
 * grid path (reading 39), row- or column-sharded LPs with the axis chosen by
 * min(m, n) (reading 33), and per-decision logs for the parity tests.
 * Everything after argument checks runs in CUDA kernels on the handle's stream;
 * there is no CPU fallback.
 *
 * Conventions (all entry points):
 *  - Return value: an lp_error code (LP_OK = 0).  Output parameters are only
 *    written on LP_OK.  lp_last_error_detail() gives a thread-local message.
 *  - Solver outcome is an lp_status inside lp_result, never an error code.
 *  - memory: LP_HOST or LP_DEVICE tells where EVERY pointer of that call lives
 *    (device pointers must be in the current CUDA device's memory).
 *  - Ownership: lp_create* COPY their inputs into library-owned device memory;
 *    the caller keeps its arrays.  Results are COPIED OUT into caller buffers.
 *    The handle owns all device state until lp_destroy().
 *  - Streams: all work of a handle is ordered on the cuda_stream given at
 *    creation (NULL = legacy default stream).  lp_solve / lp_solve_batch block
 *    once, at the end, to fill lp_result; nothing synchronises per iteration.
 *  - Threads: a handle is not thread-safe; distinct handles are independent.
 */
#ifndef MPAX_B200_LP_H
#define MPAX_B200_LP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_ABI_VERSION 1

typedef struct lp_handle_s *lp_handle; /* opaque, library-owned */

enum lp_error {
  LP_OK = 0,
  LP_ERR_INVALID_ARGUMENT = -1, /* NULL where data is required, bad option value */
  LP_ERR_DIMENSION = -2,        /* inconsistent sizes, unsorted / out-of-range CSR */
  LP_ERR_NAN = -3,              /* NaN anywhere, or +-inf outside l/u */
  LP_ERR_CROSSED_BOUNDS = -4,   /* l_j > u_j, l_j = +inf or u_j = -inf */
  LP_ERR_BATCH_SHAPE = -5,      /* batch arrays inconsistent with the shared problem */
  LP_ERR_OUT_OF_MEMORY = -6,
  LP_ERR_CUDA = -7,             /* a CUDA call failed (detail names it) */
  LP_ERR_NCCL = -8,
  LP_ERR_NOT_SOLVED = -9,       /* lp_get_solution before a solve */
  LP_ERR_UNSUPPORTED = -10      /* path not available for this handle / build */
};

enum lp_status {
  LP_OPTIMAL = 1,          /* relative KKT termination test passed */
  LP_ITERATION_LIMIT = 2,  /* iteration_limit accepted steps reached */
  LP_NUMERICAL_ERROR = 3,  /* 100 consecutive line-search rejections */
  LP_PRIMAL_INFEASIBLE = 4,/* a dual ray certifies that no x satisfies the rows and bounds */
  LP_DUAL_INFEASIBLE = 5   /* a primal ray certifies that c'x is unbounded below */
};
/* Infeasibility detection ("termination, restart, and infeasibility
 * detection" every 64 iterations; tolerances P:530-531; reading 35).
 * At every check, after the optimality test and before the iteration limit, the
 * candidate rays d = z - z_b in ORIGINAL space -- z_b the iterate before the
 * last accepted step (raPDHG) or the epoch's Halpern anchor (r2HPDHG) -- are
 * scaled to unit 2-norm and tested:
 *   PRIMAL_INFEASIBLE: q'd_y + sum_{l finite} l lam^+ - sum_{u finite} u lam^- > eps_pi with
 *     lam = -K'd_y, and max((d_y)_G^-, lam^+ on l = -inf, lam^- on u = +inf) <= eps_pi;
 *   DUAL_INFEASIBLE: c'd_x < -eps_di and max(|A d_x|, (G d_x)^-, (d_x)^+ on finite u,
 *     (d_x)^- on finite l) <= eps_di.
 * On either status lp_get_solution returns the unit rays: x = d_x/|d_x|,
 * y = d_y/|d_y|, reduced_costs = -K'd_y/|d_y| (a zero ray is returned as 0); the
 * lp_result objectives / residuals describe the current iterate.  A negative
 * tolerance switches that test off. */

enum lp_algorithm { LP_RAPDHG = 0, LP_R2HPDHG = 1 };

/* Step-size rule (lp_options.step_rule).  ADAPTIVE is the line search of P:95
 * (DESIGN.md §3 reading 4).  CONSTANT uses eta = 0.998 / sigma_max(K~) with
 * sigma_max from 200 power iterations on K~'K~ (deterministic start vector), every
 * attempt accepted -- the constant-step r2HPDHG of the cited Halpern work (SURVEY
 * §8(f) row 4; reading 34). */
enum lp_step_rule { LP_STEP_ADAPTIVE = 0, LP_STEP_CONSTANT = 1 };

/* Storage precision of the solve (lp_options.precision; MPAX runs in fp32 by
 * default, fp64 with jax_enable_x64; every LP experiment of the paper is fp64).
 * LP_FP64: everything fp64.  LP_FP32 (grid path only, DESIGN.md
 * reading 39): K~, K~' and every iterate vector are STORED in fp32 -- half the bytes per
 * attempt -- while each element's arithmetic, every dot product and every reduction runs in
 * fp64 registers; inputs, setup (scaling) and the returned solution stay fp64.  Any other
 * path with LP_FP32 returns LP_ERR_UNSUPPORTED. */
enum lp_precision { LP_FP64 = 0, LP_FP32 = 1 };
enum lp_memory { LP_HOST = 0, LP_DEVICE = 1 };

/* Solve path selection (lp_options.path). */
enum lp_path {
  LP_PATH_AUTO = 0,     /* batch / small LP -> per-instance kernel; big LP -> grid kernel */
  LP_PATH_INSTANCE = 1, /* one CTA per instance, whole solve loop in-kernel (§8(a) a11) */
  LP_PATH_GRID = 2,     /* one LP over the whole GPU: fused SpMV phases (§8(a) a5-a9) */
  LP_PATH_DMMA = 3      /* batch sharing a dense K: fp64 tensor-core contraction (a12) */
};

/* The LP, K = [G; A] in CSR.  If dense != 0 the CSR holds every entry of the
 * row-major m x n matrix (nnz = m*n, col_idx[i*n+j] = j); the dense flag lets
 * a batch use the shared-A DMMA path. */
typedef struct {
  int64_t n;          /* columns (variables), >= 1 */
  int64_t m1, m2;     /* ">=" rows, "=" rows; m = m1 + m2 >= 0 */
  int64_t nnz;        /* stored entries of K */
  int32_t dense;      /* see above */
  int32_t memory;     /* LP_HOST or LP_DEVICE for every pointer below */
  const int64_t *row_ptr; /* m+1, row_ptr[0] = 0, row_ptr[m] = nnz */
  const int32_t *col_idx; /* nnz, strictly increasing within each row, in [0, n) */
  const double *values;   /* nnz, finite */
  const double *c;        /* n */
  const double *q;        /* m: (h; b) */
  const double *l, *u;    /* n: -inf <= l <= u <= +inf */
} lp_problem_desc;

/* Options (Appendix, plus the engine's path / logging switches). */
typedef struct {
  double eps_abs;               /* 1e-4 */
  double eps_rel;               /* 1e-4 */
  double eps_primal_infeasible; /* 1e-8; < 0 disables the test */
  double eps_dual_infeasible;   /* 1e-8; < 0 disables the test */
  double eps_feas_polish;       /* 1e-6 */
  int64_t iteration_limit;      /* INT64_MAX; accepted steps */
  int32_t check_frequency;      /* 64 */
  int32_t algorithm;            /* lp_algorithm, default LP_R2HPDHG */
  int32_t warm_start;           /* informational; a non-NULL x0 / y0 is what warm-starts */
  int32_t feasibility_polishing;/* 0; 1: polish OPTIMAL results (see below; every engine) */
  int32_t verbose;              /* 0; 1: one line per display_frequency-th check of every
                                   instance (device printf, flushed when the solve returns; every
                                   engine -- the sharded one prints from rank 0's first shard) */
  int32_t display_frequency;    /* 10, in checks */
  int32_t path;                 /* lp_path, default LP_PATH_AUTO */
  int32_t step_rule;            /* lp_step_rule, default LP_STEP_ADAPTIVE */
  double reflection;            /* r2HPDHG reflection rho in [0, 1], default 1: z <- a((1 + rho) PDHG(z)
                                   - rho z) + b z0; rho = 1 is the full reflection 2 PDHG(z) - z of
                                   P:64, rho < 1 the partial reflection of SURVEY §8(f) row 4
                                   (reading 38); unused by raPDHG */
  int32_t precision;            /* lp_precision, default LP_FP64 */
  int32_t sharded_exchange;     /* row-sharded engine: 0 = variant A, all-reduce of the
                                   K~'y partials, n-side update replicated on every GPU (default);
                                   1 = variant B, reduce-scatter of the partials, n-side update on
                                   each GPU's slice of n/p columns, all-gather of x' (and of the
                                   average before a check); other engines ignore it */
} lp_options;

/* Feasibility polishing (reading 36).
 * With feasibility_polishing = 1, every instance whose solve ends OPTIMAL is followed by
 * two sub-solves with the same algorithm and options (infeasibility detection off, at most
 * min(iteration_limit, 100000) accepted steps each): a primal polish of the LP with c = 0
 * from (x*, 0) until the primal residual alone satisfies
 * pres <= eps_feas_polish (1 + ||q||), and a dual polish with q = 0 from (proj(0), y*) until
 * dres <= eps_feas_polish (1 + ||c||).  The returned x is the primal polish's, y and the
 * reduced costs the dual polish's; primal_residual / dual_residual are theirs, the
 * objectives, gap and rel_kkt are recomputed on the original c, q, l, u; iterations,
 * attempts and restarts are summed over the three solves; `polish` flags the outcome. */

/* Per-instance outcome.  The objectives and residuals are those of the
 * returned (x, y) in ORIGINAL space (contract step 5/6):
 *   primal_residual = ||(q - Kx) with ">=" rows clipped at 0||_2,
 *   dual_residual   = ||lambda+ [l=-inf] + lambda- [u=+inf]||_2, lambda = c - K'y,
 *   gap = |pobj - dobj|,
 *   rel_kkt = max(pres/(1+||q||), dres/(1+||c||), gap/(1+|pobj|+|dobj|)). */
typedef struct {
  int32_t status;       /* lp_status */
  int32_t polish;       /* feasibility polishing: 0 not run, 1 both sub-solves passed, 2 one hit its limit */
  int64_t iterations;   /* accepted PDHG steps k */
  int64_t attempts;     /* line-search attempts j (>= iterations) */
  int64_t restarts;
  double primal_objective, dual_objective;
  double primal_residual, dual_residual, gap, rel_kkt;
  double omega, eta;    /* final primal weight and step size (scaled space) */
  double solve_seconds; /* device time of the whole solve call (all instances) */
} lp_result;

/* Fills o with the Appendix defaults: 1e-4, 1e-4, 1e-8, 1e-8, 1e-6,
 * INT64_MAX, 64, LP_R2HPDHG, 0, 0, 0, 10, LP_PATH_AUTO, LP_STEP_ADAPTIVE, 1.0, LP_FP64, 0. */
void lp_default_options(lp_options *o);

/* Create a single-LP handle: validates, uploads, builds
 * K~' (transpose) and the Ruiz(10) + Pock-Chambolle(alpha=1) scaling
 * on the device.  cuda_stream: a cudaStream_t or NULL. */
int lp_create(const lp_problem_desc *p, void *cuda_stream, lp_handle *out);

/* Create a batch handle for `batch` instances sharing K, l, u.
 * C: batch x n row-major costs (NULL: every instance uses shared->c);
 * Q: batch x m row-major right-hand sides (NULL: every instance uses shared->q).
 * `memory` applies to C and Q; shared->memory to the shared problem.
 * Preconditioning depends on K only, so it is shared; all other state is per
 * instance (contract step 6 "Batch"). */
int lp_create_batch(const lp_problem_desc *shared, int64_t batch, const double *C, const double *Q,
                    int32_t memory, void *cuda_stream, lp_handle *out);

/* Replace the per-instance costs / right-hand sides of a batch handle (same
 * shapes; NULL leaves that side unchanged).  Used for SPO+-style loops where K
 * is fixed and c changes every step.  The new values are validated
 * like lp_create's (LP_ERR_NAN for a NaN or infinity; the handle then holds the
 * rejected values and no solution until the next successful update).  Synchronous:
 * the caller's buffers may be freed on return.  LP_ERR_UNSUPPORTED on a sharded handle. */
int lp_update_batch(lp_handle h, const double *C, const double *Q, int32_t memory);

/* Solve a single-LP handle.  x0 (n) / y0 (m) are an optional warm start in
 * ORIGINAL space; NULL halves start at zero.  `memory`
 * applies to x0, y0.  `out` is a host struct; out->status is OPTIMAL,
 * PRIMAL_INFEASIBLE / DUAL_INFEASIBLE (then lp_get_solution returns the rays),
 * ITERATION_LIMIT or NUMERICAL_ERROR.  The kernel is picked by o->path (AUTO: the
 * persistent grid kernel for large single LPs, else the per-instance kernels). */
int lp_solve(lp_handle h, const lp_options *o, const double *x0, const double *y0, int32_t memory,
             lp_result *out);

/* Solve every instance of a batch handle.  X0 (batch x n), Y0 (batch x m)
 * optional warm starts.  `out` is a host array of `batch` results. */
int lp_solve_batch(lp_handle h, const lp_options *o, const double *X0, const double *Y0,
                   int32_t memory, lp_result *out);

/* ---- SPO+ layer ----
 * SPO+ loss and one subgradient over a batch: PAPER.md Eq. (spo+ loss) and
 * Eq. (spo+ gradient), as in the training step of P:198-215.  h must be a batch
 * handle with per-instance costs (lp_create_batch with C != NULL), or a single-LP handle;
 * its K, q, l, u describe the feasible set S and its costs are overwritten.
 *   C_pred (batch x n): predicted costs c^;  C_true (batch x n): realised costs c;
 *   X_true (batch x n): x*(c);  obj_true (batch): c'x*(c).
 * On the device: the handle's costs become 2c^ - c; the batch is solved with *o (warm != 0:
 * started from the handle's previous solutions, the warm start of P:263 / P:411; else cold);
 * then, per instance b with x_b the inner solution and obj_b its primal objective
 * (2c^_b - c_b)'x_b,
 *   loss[b] = -obj_b + 2 c^_b'x*(c_b) - obj_true[b],    grad[b] = 2 (x*(c_b) - x_b).
 * The caller averages over the batch.  out[b] receives the inner solve's result; the
 * inner solutions stay in the handle (lp_get_solutions).  All arrays live in `memory`
 * (LP_HOST / LP_DEVICE); loss and grad are written, the inputs are only read.
 * Errors: LP_ERR_BATCH_SHAPE if the handle shares one c across a batch > 1; as lp_solve_batch. */
int lp_spo_plus(lp_handle h, const lp_options *o, const double *C_pred, const double *C_true,
                const double *X_true, const double *obj_true, int32_t warm, int32_t memory, double *loss,
                double *grad, lp_result *out);

/* Copy out instance `instance`'s solution of the last solve, in original space:
 * x (n), y (m), reduced costs lambda = c - K'y (n).  Any pointer may be NULL.
 * memory = LP_HOST: synchronous (the data is in place on return).  memory = LP_DEVICE:
 * stream-ordered on the handle's stream (no host synchronisation; work queued on that
 * stream afterwards sees the data). */
int lp_get_solution(lp_handle h, int64_t instance, double *x, double *y, double *reduced_costs,
                    int32_t memory);

/* Copy out every instance: X (batch x n), Y (batch x m); either may be NULL.
 * Synchronous for LP_HOST, stream-ordered on the handle's stream for LP_DEVICE. */
int lp_get_solutions(lp_handle h, double *X, double *Y, int32_t memory);

/* Shapes of a handle: n, m1, m2, batch (any pointer may be NULL). */
int lp_get_shape(lp_handle h, int64_t *n, int64_t *m1, int64_t *m2, int64_t *batch);

/* Diagnostics used by the parity tests: the diagonal scalings Dr (m), Dc (n)
 * of step 1, and the scaled products K~ v (m) and K~' w (n) computed by the
 * solver's own SpMV kernels (bench.py's SpMV-pair leg).  Any pointer may be
 * NULL.  memory = LP_DEVICE: the buffers are device memory and are read /
 * written in place; LP_HOST: staged through device copies.  Blocks until the
 * products are written. */
int lp_get_scaling(lp_handle h, double *Dr, double *Dc, int32_t memory);

/* Decision log of the grid path (the parity tests' tool for finding the
 * first decision where the GPU and the oracle part ways).  att: att_cap x 4
 * doubles, one row per line-search attempt j = 1, 2, ... : (j, accepted, eta, eta_bar) with
 * eta the step tried and eta_bar = M / (2|I|) (contract step 3); chk: chk_cap x 6 doubles, one
 * row per check: (k, metric, ref, last, restart, outcome) with outcome 0 = no termination,
 * 1 = optimal (raPDHG: the average; r2HPDHG: the candidate), 2 = optimal (raPDHG: the current
 * iterate), 3 = infeasibility certificate; metric = 0 where the oracle logs 0 -- the same
 * records as the oracle's ora_log.  Rows past the capacity are dropped; rows not reached are
 * left untouched.  The buffers must be device-accessible (device or mapped pinned memory) and
 * stay valid through every later lp_solve on the handle; NULL / capacity 0 switches a log off.
 * Recorded by the grid path (one LP), by the sharded engines (every rank records the same,
 * replicated decisions) and by the register kernel of the small-LP batches (the C2 shapes:
 * m <= 32, n <= 64, rows <= 4 and columns <= 4 entries), which logs ONE instance, `instance` of
 * lp_set_decision_log_instance (default 0); any other path returns LP_ERR_UNSUPPORTED while a
 * log is set.  Polishing sub-solves are not logged.  Logging does not change any result. */
int lp_set_decision_log(lp_handle h, double *att, int64_t att_cap, double *chk, int64_t chk_cap);
int lp_set_decision_log_instance(lp_handle h, int64_t instance);

int lp_spmv_scaled(lp_handle h, const double *v, double *Kv, const double *w, double *KTw,
                   int32_t memory);

/* ---- one LP row-sharded across GPUs (§3.5) ----
 * Process `rank` of `nranks` (one process per GPU) passes ITS block of rows:
 * rows [global_row_offset, global_row_offset + m_local) of K = [G; A], with
 * local_rows->m1 = number of those rows that are ">=" rows (all of them come
 * first, as globally), local q, and the FULL c, l, u (n).  nccl_comm is a
 * borrowed ncclComm_t (NULL allowed when nranks == 1); the caller keeps it alive.
 * Column norms of the preconditioner and every cross-shard sum of the iteration
 * go through ncclAllReduce on the handle's stream.  lp_solve then takes x0 (n)
 * and y0 (this rank's m_local rows); lp_get_solution returns x, reduced costs (n)
 * and this rank's rows of y. */
int lp_create_sharded(const lp_problem_desc *local_rows, int64_t global_row_offset, int64_t m1_global,
                      int64_t m2_global, void *nccl_comm, int rank, int nranks, void *cuda_stream, lp_handle *out);

/* The same sharded engine with `shards` row blocks (balanced by nnz) on the
 * CURRENT device and a fixed-order device sum in place of NCCL: the partitioned
 * arithmetic of lp_create_sharded, testable on one GPU.  y covers all m rows. */
int lp_create_sharded_virtual(const lp_problem_desc *p, int32_t shards, void *cuda_stream, lp_handle *out);

/* ---- the sharding axis (reading 33) ----
 * Row sharding exchanges the n-long K~'y partials every attempt, column sharding the m-long
 * K~x' partials: the shorter vector should travel.  lp_shard_axis(m, n) = LP_SHARD_COLS iff
 * m < n, else LP_SHARD_ROWS.
 * Column-sharded engine: process `rank` passes ITS block of columns, columns
 * [global_col_offset, global_col_offset + n_local) of K as an m x n_local CSR with LOCAL
 * column indices (every row, m1 / m2 global), the FULL q (m) and its c, l, u (n_local).  Row
 * norms of the preconditioner and every cross-shard sum go through ncclAllReduce.  lp_solve
 * takes x0 (this rank's n_local columns) and y0 (m); lp_get_solution returns this rank's
 * columns of x and of the reduced costs and the full y.  The constant step rule's power
 * iteration all-reduces K~x partials and squared norms across the column shards.
 * lp_create_sharded_virtual_axis: `shards` blocks
 * of rows or columns (balanced by nnz; LP_SHARD_AUTO picks lp_shard_axis) on the current
 * device with the fixed-order device sum; x, y and the reduced costs then cover the whole LP. */
enum lp_shard_axis { LP_SHARD_ROWS = 0, LP_SHARD_COLS = 1, LP_SHARD_AUTO = 2 };
int lp_shard_axis(int64_t m, int64_t n);
int lp_create_sharded_cols(const lp_problem_desc *local_cols, int64_t global_col_offset, int64_t n_global,
                           void *nccl_comm, int rank, int nranks, void *cuda_stream, lp_handle *out);
int lp_create_sharded_virtual_axis(const lp_problem_desc *p, int32_t shards, int32_t axis, void *cuda_stream,
                                   lp_handle *out);

/* NCCL communicator helpers (so callers need no NCCL headers): rank 0 calls
 * lp_nccl_unique_id (128 bytes) and broadcasts it (e.g. torch.distributed),
 * then every rank calls lp_nccl_comm_init with its CUDA device current. */
int lp_nccl_unique_id(void *out_id128);
int lp_nccl_comm_init(void **comm, int nranks, const void *id128, int rank);
int lp_nccl_comm_destroy(void *comm);

/* Self-test of the division with a deferred slow path that the latency-bound kernels use for
 * the line-search ratio eta_bar = M / (2|I|) and the averaging weight eta / (W + eta)
 * (contract step 3-4): `count` operand pairs drawn on the device from a
 * counter-based hash of `seed` (random signs, exponents over the whole double range, and
 * zeros, infinities, NaNs, subnormals mixed in) are divided both ways.  *mismatches = pairs
 * where the fast path claimed success (ok) but its quotient is not bit-identical to the
 * IEEE quotient a / b; *slow = pairs that took the slow path.  Synchronous on the default
 * stream.  Returns LP_ERR_CUDA without a GPU. */
int lp_selftest_division(int64_t count, uint64_t seed, int64_t *mismatches, int64_t *slow);

/* Number of kernels this library has launched in the calling process so far
 * (bench.py reports the difference across its timed region). */
int64_t lp_kernel_launch_count(void);

const char *lp_error_string(int code);
const char *lp_last_error_detail(void); /* thread-local */
void lp_destroy(lp_handle h);           /* NULL is a no-op */

#ifdef __cplusplus
}
#endif
#endif

/*
 * mpax_oracle.c -- plain, slow, CPU reference ("oracle") for the restarted PDHG
 * LP iteration of MPAX (arXiv 2412.09734).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product (paper_2412_09734_b200/, the CUDA C-ABI library) shares no code,
 * header, table or helper with this file and never calls it.
 *
 * What it computes.  The LP of PAPER.md Eq. (1)
 *     min c'x  s.t.  Gx >= h, Ax = b, l <= x <= u,
 * through its saddle form Eq. (2) with K = [G; A], q = (h; b)
 * (rows 0..m1-1 are ">=" rows, the rest "=" rows), by
 *   raPDHG   -- PDHG Eq. (pdhg) + averaging and restarts
 *   r2HPDHG  -- Halpern PDHG with reflection Eq. (hrpdhg), restarted
 * with the enhancements of P:91-96 (preconditioning, adaptive restart, adaptive
 * step size, primal-weight update, termination on relative KKT error checked
 * every 64 iterations).  The paper names these enhancements but gives no
 * constants or formulas for them; every such choice follows the binding reading
 * "ORACLE-CONTRACT v1" written in SURVEY.md §8(c) (c.2 steps 0-6, c.3 readings)
 * and restated in DESIGN.md §3.  Each function below cites the passage it follows.
 *
 * Style: scalar loops in the contract's order and notation, fp64, IEEE round to
 * nearest, no FMA contraction (-ffp-contract=off), no blocking or fusion.  OpenMP
 * is used only (a) over rows of a sparse matrix-vector product, where each row's
 * sum is still a sequential loop, and (b) over independent batch instances; all
 * reductions are sequential, so results do not depend on the thread count.
 *
 * Parity status: every function is pinned by tests in
 * tests/test_oracle_*.py -- including the readings the paper leaves unquantified
 * (KKT_omega, omega0 / eta0, the restart candidate, the r2HPDHG epoch reference:
 * hand-derived values in tests/golden/readings.json) -- and
 * tests/test_oracle_mutations.py checks that 19 plausible one-line slips in this
 * file each fail a pin.  NOT pinned: the iteration / attempt / restart COUNTS of a
 * full solve, which are "parity unpinned" externally (the paper prints counts
 * only for datasets we do not have); only GPU == oracle applies to
 * them.
 */
#include <math.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double ora_time_t;   /* wall-clock seconds (timing only; fp64 in both builds) */

/* The fp32 build (liboracle_f32.so; reading 39).  MPAX's default precision is
 * single ("MPAX uses single-precision (FP32) by default, consistent with JAX's
 * standard setting"): in JAX every array and every operation of the solve is then float32, and
 * Python literals adopt the array dtype (weak typing).  This file compiled with -DORA_FP32 and
 * -fsingle-precision-constant is that program: every real (inputs, scaling, iterates,
 * reductions, step sizes, tolerances) is an IEEE single, every literal is rounded to single,
 * and the math library calls are their single-precision versions.  Integers (indices, counts)
 * are unchanged.  Defined after the system headers so their prototypes keep their types. */
#ifdef ORA_FP32
#define double float
#define sqrt sqrtf
#define fabs fabsf
#define fmin fminf
#define fmax fmaxf
#define pow powf
#define ORA_INF HUGE_VALF
#else
#define ORA_INF HUGE_VAL
#endif

#define ORA_POLISH_LIMIT 100000   /* accepted steps per polishing sub-solve (reading 36) */

enum { ORA_OK = 0, ORA_ERR_INVALID = -1, ORA_ERR_DIMENSION = -2, ORA_ERR_NAN = -3,
       ORA_ERR_CROSSED_BOUNDS = -4, ORA_ERR_OOM = -6 };
enum { ORA_OPTIMAL = 1, ORA_ITERATION_LIMIT = 2, ORA_NUMERICAL_ERROR = 3, ORA_PRIMAL_INFEASIBLE = 4,
       ORA_DUAL_INFEASIBLE = 5 };
enum { ORA_RAPDHG = 0, ORA_R2HPDHG = 1 };

/* ---------------------------------------------------------------- types -- */

/* The LP of Eq. (1), already stacked as K = [G; A], q = (h; b). */
typedef struct {
  int64_t n, m1, m2, nnz;
  const int64_t *row_ptr;  /* m+1 */
  const int32_t *col_idx;  /* nnz */
  const double *val;       /* nnz */
  const double *c, *q, *l, *u;
} ora_problem;

typedef struct {
  double eps_abs, eps_rel;      /* Appendix, default 1e-4 */
  int64_t iteration_limit;      /* Appendix */
  int32_t check_frequency;      /* P:96 "every 64 iterations" */
  int32_t algorithm;            /* ORA_RAPDHG / ORA_R2HPDHG */
  int32_t ruiz_iters;           /* contract c.3 #3: 10 */
  int32_t pock_chambolle;       /* contract c.3 #3: 1 = apply one PC(alpha=1) round */
  int32_t step_rule;            /* 0: adaptive line search (contract step 3); 1: constant step
                                   eta = 0.998 / sigma_max(K~) (DESIGN reading 34) */
  int32_t power_iters;          /* power-iteration steps for sigma_max(K~), default 200 */
  double eps_primal_infeasible; /* Appendix, default 1e-8 (< 0: test off) */
  double eps_dual_infeasible;   /* Appendix, default 1e-8 (< 0: test off) */
  double eps_feas_polish;       /* Appendix, default 1e-6 */
  int32_t feasibility_polishing;/* Appendix, default 0 (DESIGN reading 36) */
  int32_t polish_mode;          /* termination test: 0 relative KKT (contract step 5); 1 primal
                                   residual only; 2 dual residual only (the polishing sub-solves) */
  double reflection;            /* r2HPDHG reflection rho in [0, 1], default 1 (reading 38) */
} ora_options;

/* Infeasibility certificate test on ORIGINAL-space rays (reading 35;
 * SPEC S:419-427).  Both rays are judged after scaling to unit
 * 2-norm: d_y certifies primal infeasibility iff
 *     q'd_y + sum_{l_j finite} l_j lam_j^+ - sum_{u_j finite} u_j lam_j^-  >  eps_p,
 *     with lam = -K'd_y,  and  max( (d_y)_i^- for ">=" rows i,
 *                                  lam_j^+ for l_j = -inf, lam_j^- for u_j = +inf ) <= eps_p
 * (the Farkas alternative: K x >=/= q has no solution in the box); d_x certifies
 * dual infeasibility iff c'd_x < -eps_d and
 *     max( |(K d_x)_i| for "=" rows, (K d_x)_i^- for ">=" rows,
 *          (d_x)_j^+ for u_j finite, (d_x)_j^- for l_j finite ) <= eps_d
 * (a recession direction of the feasible set along which c'x decreases). */
typedef struct {
  int32_t primal_infeasible, dual_infeasible;
  double norm_dy, dual_ray_objective, dual_ray_violation;    /* after / for the unit scaling */
  double norm_dx, primal_ray_objective, primal_ray_violation;
} ora_certificate;

typedef struct {
  int32_t status, polish;       /* polish: 0 not run, 1 both polish solves converged, 2 one hit the limit */
  int64_t iterations, attempts, restarts;
  double primal_objective, dual_objective, primal_residual, dual_residual, gap, rel_kkt;
  double omega, eta;
} ora_result;

/* Optional decision log: one row per attempt
 * (j, acc, eta_used, eta_bar) and one row per check
 * (k, metric, ref, last, restart, pass). */
typedef struct {
  int64_t att_cap, att_len; double *att;
  int64_t chk_cap, chk_len; double *chk;
} ora_log;

typedef struct {
  double pres, dres, pobj, dobj, gap;
} ora_kkt;

typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t *rp; int32_t *ci; double *v;
} csr;

/* ------------------------------------------------------- linear algebra -- */

/* y = M x, row by row, entries in stored order (the matvec). */
static void csr_spmv(const csr *M, const double *x, double *y) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < M->nrows; ++i) {
    double s = 0.0;
    for (int64_t p = M->rp[i]; p < M->rp[i + 1]; ++p) s += M->v[p] * x[M->ci[p]];
    y[i] = s;
  }
}

/* CSR of the transpose by a stable counting sort on the column index. */
static int csr_transpose(const csr *M, csr *T) {
  T->nrows = M->ncols; T->ncols = M->nrows; T->nnz = M->nnz;
  T->rp = (int64_t *)calloc((size_t)T->nrows + 1, sizeof(int64_t));
  T->ci = (int32_t *)malloc((size_t)(M->nnz ? M->nnz : 1) * sizeof(int32_t));
  T->v = (double *)malloc((size_t)(M->nnz ? M->nnz : 1) * sizeof(double));
  if (!T->rp || !T->ci || !T->v) return ORA_ERR_OOM;
  for (int64_t p = 0; p < M->nnz; ++p) T->rp[M->ci[p] + 1] += 1;
  for (int64_t j = 0; j < T->nrows; ++j) T->rp[j + 1] += T->rp[j];
  int64_t *next = (int64_t *)malloc((size_t)(T->nrows + 1) * sizeof(int64_t));
  if (!next) return ORA_ERR_OOM;
  memcpy(next, T->rp, (size_t)(T->nrows + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < M->nrows; ++i)
    for (int64_t p = M->rp[i]; p < M->rp[i + 1]; ++p) {
      int64_t d = next[M->ci[p]]++;
      T->ci[d] = (int32_t)i; T->v[d] = M->v[p];
    }
  free(next);
  return ORA_OK;
}

static void csr_free(csr *M) { free(M->rp); free(M->ci); free(M->v); memset(M, 0, sizeof(*M)); }

static double dot(const double *a, const double *b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double norm2(const double *a, int64_t n) { return sqrt(dot(a, a, n)); }
static double dist2(const double *a, const double *b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) { double d = a[i] - b[i]; s += d * d; }
  return sqrt(s);
}
static double dmin(double a, double b) { return fmin(a, b); }
static double dmax(double a, double b) { return fmax(a, b); }

/* median(l, v, u) = min(max(v, l), u): proj_X of Eq. (pdhg), X = {l <= x <= u}. */
static double median3(double l, double v, double u) { return dmin(dmax(v, l), u); }

/* Largest singular value of M by power iteration on M'M (used by the
 * constant-step variant, DESIGN reading 34).  Deterministic start vector
 * v_j = frac(j * 2654435761 / 2^32) + 0.5 (integer hash, exact in double), normalised;
 * then `iters` times: u = M v, w = M'u, s = ||w||, v = w / s, sigma = sqrt(s).
 * Returns 0 for a zero matrix. */
static double power_sigma(const csr *M, const csr *MT, int32_t iters) {
  const int64_t n = M->ncols, m = M->nrows;
  double *v = (double *)malloc((size_t)n * sizeof(double));
  double *u = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *w = (double *)malloc((size_t)n * sizeof(double));
  for (int64_t j = 0; j < n; ++j) v[j] = (double)((uint32_t)((uint64_t)j * 2654435761ull)) / 4294967296.0 + 0.5;
  double nv = norm2(v, n);
  for (int64_t j = 0; j < n; ++j) v[j] /= nv;
  double sigma = 0.0;
  for (int32_t t = 0; t < iters; ++t) {
    csr_spmv(M, v, u);
    csr_spmv(MT, u, w);
    double sw = norm2(w, n);
    if (!(sw > 0.0)) { sigma = 0.0; break; }
    for (int64_t j = 0; j < n; ++j) v[j] = w[j] / sw;
    sigma = sqrt(sw);
  }
  free(v); free(u); free(w);
  return sigma;
}

/* ------------------------------------------------------------ Step 0 ----- */

/* Validation (contract step 0): consistent dimensions,
 * sorted in-range column indices, no NaN anywhere, +-inf only in l/u, l <= u.
 * Returns the first violation. */
int ora_validate(const ora_problem *p) {
  if (!p || p->n < 1 || p->m1 < 0 || p->m2 < 0 || p->nnz < 0) return ORA_ERR_DIMENSION;
  int64_t m = p->m1 + p->m2;
  if (m > 0 && (!p->row_ptr || (p->nnz > 0 && (!p->col_idx || !p->val)))) return ORA_ERR_INVALID;
  if (!p->c || !p->l || !p->u || (m > 0 && !p->q)) return ORA_ERR_INVALID;
  if (m > 0) {
    if (p->row_ptr[0] != 0 || p->row_ptr[m] != p->nnz) return ORA_ERR_DIMENSION;
    for (int64_t i = 0; i < m; ++i) {
      if (p->row_ptr[i + 1] < p->row_ptr[i]) return ORA_ERR_DIMENSION;
      for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) {
        if (p->col_idx[k] < 0 || p->col_idx[k] >= p->n) return ORA_ERR_DIMENSION;
        if (k > p->row_ptr[i] && p->col_idx[k] <= p->col_idx[k - 1]) return ORA_ERR_DIMENSION;
      }
    }
  } else if (p->nnz != 0) return ORA_ERR_DIMENSION;
  for (int64_t k = 0; k < p->nnz; ++k) if (!isfinite(p->val[k])) return ORA_ERR_NAN;
  for (int64_t j = 0; j < p->n; ++j) if (!isfinite(p->c[j])) return ORA_ERR_NAN;
  for (int64_t i = 0; i < m; ++i) if (!isfinite(p->q[i])) return ORA_ERR_NAN;
  for (int64_t j = 0; j < p->n; ++j) {
    if (isnan(p->l[j]) || isnan(p->u[j])) return ORA_ERR_NAN;
    if (p->l[j] == ORA_INF || p->u[j] == -ORA_INF) return ORA_ERR_CROSSED_BOUNDS;
    if (p->l[j] > p->u[j]) return ORA_ERR_CROSSED_BOUNDS;
  }
  return ORA_OK;
}

/* ------------------------------------------------------------ Step 1 ----- */

/* Diagonal preconditioning ("Ruiz scaling ... and Pock and Chambolle's
 * diagonal scaling"; contract step 1 and reading c.3 #3).  With
 * a_ij = (|K_ij| Dr_i) Dc_j over stored entries:
 *   Ruiz (ruiz_iters rounds): rho_i = max_j a_ij, gamma_j = max_i a_ij from the
 *     same Dr, Dc; Dr_i *= 1/sqrt(rho_i), Dc_j *= 1/sqrt(gamma_j) (1 if zero);
 *   Pock-Chambolle alpha = 1 (one round if pc): rho_i = sum_j a_ij,
 *     gamma_j = sum_i a_ij, same update.
 * Dr (m), Dc (n) are outputs. */
int ora_precondition(const ora_problem *p, int32_t ruiz_iters, int32_t pc, double *Dr, double *Dc) {
  int64_t m = p->m1 + p->m2, n = p->n;
  double *rho = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *gam = (double *)malloc((size_t)n * sizeof(double));
  if (!rho || !gam) { free(rho); free(gam); return ORA_ERR_OOM; }
  for (int64_t i = 0; i < m; ++i) Dr[i] = 1.0;
  for (int64_t j = 0; j < n; ++j) Dc[j] = 1.0;
  int32_t rounds = ruiz_iters + (pc ? 1 : 0);
  for (int32_t r = 0; r < rounds; ++r) {
    int use_sum = (r >= ruiz_iters);  /* the final round is Pock-Chambolle */
    for (int64_t i = 0; i < m; ++i) rho[i] = 0.0;
    for (int64_t j = 0; j < n; ++j) gam[j] = 0.0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) {
        int64_t j = p->col_idx[k];
        double a = (fabs(p->val[k]) * Dr[i]) * Dc[j];
        if (use_sum) { rho[i] += a; gam[j] += a; }
        else { rho[i] = dmax(rho[i], a); gam[j] = dmax(gam[j], a); }
      }
    for (int64_t i = 0; i < m; ++i) Dr[i] *= (rho[i] > 0.0 ? 1.0 / sqrt(rho[i]) : 1.0);
    for (int64_t j = 0; j < n; ++j) Dc[j] *= (gam[j] > 0.0 ? 1.0 / sqrt(gam[j]) : 1.0);
  }
  free(rho); free(gam);
  return ORA_OK;
}

/* The scaled problem the iterations run on ("iterations begin on the
 * scaled LP"): K~ = Dr K Dc entrywise as (K_ij Dr_i) Dc_j, c~ = c Dc, q~ = q Dr,
 * l~ = l / Dc, u~ = u / Dc (contract step 1). */
typedef struct {
  int64_t n, m, m1;
  csr K, KT;
  double *c, *q, *l, *u;        /* scaled */
  const double *Dr, *Dc;        /* shared with a batch */
  const double *c0, *q0, *l0, *u0;
  double nc0, nq0;              /* original ||c||, ||q|| for the termination test */
} scaled_lp;

static int scale_matrix(const ora_problem *p, const double *Dr, const double *Dc, csr *K, csr *KT) {
  int64_t m = p->m1 + p->m2;
  K->nrows = m; K->ncols = p->n; K->nnz = p->nnz;
  K->rp = (int64_t *)malloc((size_t)(m + 1) * sizeof(int64_t));
  K->ci = (int32_t *)malloc((size_t)(p->nnz ? p->nnz : 1) * sizeof(int32_t));
  K->v = (double *)malloc((size_t)(p->nnz ? p->nnz : 1) * sizeof(double));
  if (!K->rp || !K->ci || !K->v) return ORA_ERR_OOM;
  if (m == 0) K->rp[0] = 0;
  else memcpy(K->rp, p->row_ptr, (size_t)(m + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) {
      K->ci[k] = p->col_idx[k];
      K->v[k] = (p->val[k] * Dr[i]) * Dc[p->col_idx[k]];
    }
  return csr_transpose(K, KT);
}

static int build_scaled(const ora_problem *p, const double *Dr, const double *Dc,
                        const csr *Kshared, const csr *KTshared, scaled_lp *S) {
  memset(S, 0, sizeof(*S));
  S->n = p->n; S->m = p->m1 + p->m2; S->m1 = p->m1;
  S->Dr = Dr; S->Dc = Dc;
  if (Kshared) { S->K = *Kshared; S->KT = *KTshared; }
  else { int e = scale_matrix(p, Dr, Dc, &S->K, &S->KT); if (e) return e; }
  int64_t n = S->n, m = S->m;
  S->c = (double *)malloc((size_t)n * sizeof(double));
  S->l = (double *)malloc((size_t)n * sizeof(double));
  S->u = (double *)malloc((size_t)n * sizeof(double));
  S->q = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  if (!S->c || !S->l || !S->u || !S->q) return ORA_ERR_OOM;
  for (int64_t j = 0; j < n; ++j) {
    S->c[j] = p->c[j] * Dc[j];
    S->l[j] = p->l[j] / Dc[j];
    S->u[j] = p->u[j] / Dc[j];
  }
  for (int64_t i = 0; i < m; ++i) S->q[i] = p->q[i] * Dr[i];
  S->c0 = p->c; S->q0 = p->q; S->l0 = p->l; S->u0 = p->u;
  S->nc0 = norm2(p->c, n);
  S->nq0 = m ? norm2(p->q, m) : 0.0;
  return ORA_OK;
}

static void scaled_free(scaled_lp *S, int owns_matrix) {
  if (owns_matrix) { csr_free(&S->K); csr_free(&S->KT); }
  free(S->c); free(S->q); free(S->l); free(S->u);
}

/* ------------------------------------------------------- Step 3 pieces --- */

/* proj_Y of Eq. (pdhg): Y = {y : y_{1:m1} >= 0}. */
static void project_dual(double *y, int64_t m1) {
  for (int64_t i = 0; i < m1; ++i) y[i] = dmax(y[i], 0.0);
}

/* Adaptive step size ("heuristic line search"; contract step 3, reading
 * c.3 #4): M = omega dx2 + dy2 omega^-1, eta_bar = M / (2|I|) (+inf if I == 0),
 * accept iff eta <= eta_bar, eta_next = min((1-(j+1)^-0.3) eta_bar, (1+(j+1)^-0.6) eta).
 * omega^-1 = 1 / omega (reading 32: every x / omega of the iteration is x * omega^-1). */
void ora_step_size(double eta, double omega, double dx2, double dy2, double I, int64_t j,
                   double *eta_bar, int32_t *acc, double *eta_next) {
  double inv_omega = 1.0 / omega;
  double M = omega * dx2 + dy2 * inv_omega;
  double eb = (I != 0.0) ? M / (2.0 * fabs(I)) : ORA_INF;
  double jp1 = (double)(j + 1);
  *eta_bar = eb;
  *acc = (eta <= eb) ? 1 : 0;
  *eta_next = dmin((1.0 - pow(jp1, -0.3)) * eb, (1.0 + pow(jp1, -0.6)) * eta);
}

/* Halpern step with reflection, Eq. (hrpdhg):
 * z_{k+1} = (k+1)/(k+2) (2 w - z_k) + 1/(k+2) z_0 with w = PDHG(z_k). */
/* Partial reflection (DESIGN reading 38): z <- a((1 + rho) w - rho z) + b z0;
 * rho = 1 is the full reflection above (the same operations: 2 w and 1 z are exact). */
void ora_halpern_rho(int64_t len, int64_t k, double rho, const double *z, const double *w, const double *z0,
                     double *out) {
  double a = (double)(k + 1) / (double)(k + 2);
  double b = 1.0 / (double)(k + 2);
  for (int64_t i = 0; i < len; ++i) out[i] = a * ((1.0 + rho) * w[i] - rho * z[i]) + b * z0[i];
}

void ora_halpern(int64_t len, int64_t k, const double *z, const double *w, const double *z0, double *out) {
  double a = (double)(k + 1) / (double)(k + 2);
  double b = 1.0 / (double)(k + 2);
  for (int64_t i = 0; i < len; ++i) out[i] = a * (2.0 * w[i] - z[i]) + b * z0[i];
}

/* Step-size-weighted running average ("averaging"; contract step 4 raPDHG,
 * reading c.3 #16): W += eta; avg += (eta / W) (z - avg).  Returns the new W. */
double ora_average_update(int64_t len, double *avg, const double *z, double W, double eta) {
  double W1 = W + eta;
  double theta = eta / W1;
  for (int64_t i = 0; i < len; ++i) avg[i] += theta * (z[i] - avg[i]);
  return W1;
}

/* Restart criterion (contract step 5, reading c.3 #12):
 * restart iff k_in >= 0.36 k, or metric <= 0.2 ref, or
 * (metric <= 0.8 ref and metric > last). */
int32_t ora_restart_test(int64_t k_in, int64_t k, double metric, double ref, double last) {
  if ((double)k_in >= 0.36 * (double)k) return 1;
  if (metric <= 0.2 * ref) return 1;
  if (metric <= 0.8 * ref && metric > last) return 1;
  return 0;
}

/* Primal-weight update at a restart (contract step 5, reading c.3 #9):
 * omega <- sqrt(omega * dy/dx) when dx, dy > 1e-10 (theta = 1/2 smoothing). */
double ora_primal_weight(double omega, double dx, double dy) {
  if (dx > 1e-10 && dy > 1e-10) return sqrt(omega * (dy / dx));
  return omega;
}

/* ------------------------------------------------------------ Step 5 ----- */

/* KKT residuals of a point in a given space (contract step 5):
 *   r_i = q_i - (Kx)_i on "=" rows, max(q_i - (Kx)_i, 0) on ">=" rows, pres = ||r||;
 *   lambda = c - K'y; dres = || lambda+ [l=-inf] + lambda- [u=+inf] ||;
 *   pobj = <c,x>; dobj = <q,y> + sum_{l>-inf} l lambda+ - sum_{u<inf} u lambda-;
 *   gap = |pobj - dobj|. */
static void kkt_residuals(int64_t n, int64_t m, int64_t m1,
                          const double *x, const double *y, const double *Kx, const double *KTy,
                          const double *c, const double *q, const double *l, const double *u,
                          ora_kkt *r) {
  double pres2 = 0.0, dres2 = 0.0, pobj = 0.0, dobj = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double ri = q[i] - Kx[i];
    if (i < m1) ri = dmax(ri, 0.0);
    pres2 += ri * ri;
    dobj += q[i] * y[i];
  }
  for (int64_t j = 0; j < n; ++j) {
    double lam = c[j] - KTy[j];
    double lp = dmax(lam, 0.0), lm = dmax(-lam, 0.0);
    double v = 0.0;
    if (l[j] == -ORA_INF) v += lp;
    if (u[j] == ORA_INF) v += lm;
    dres2 += v * v;
    pobj += c[j] * x[j];
    if (l[j] > -ORA_INF) dobj += l[j] * lp;
    if (u[j] < ORA_INF) dobj -= u[j] * lm;
  }
  r->pres = sqrt(pres2); r->dres = sqrt(dres2);
  r->pobj = pobj; r->dobj = dobj; r->gap = fabs(pobj - dobj);
}

/* Original-space KKT of a scaled candidate by unscaling its cached products:
 * x = Dc x~, y = Dr y~, Kx = Kx~ / Dr, K'y = K'y~ / Dc (contract step 5). */
static void kkt_original_from_scaled(const scaled_lp *S, const double *xs, const double *ys,
                                     const double *Kxs, const double *KTys, ora_kkt *r) {
  int64_t n = S->n, m = S->m;
  double *x = (double *)malloc((size_t)n * sizeof(double));
  double *KTy = (double *)malloc((size_t)n * sizeof(double));
  double *y = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *Kx = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  for (int64_t j = 0; j < n; ++j) { x[j] = S->Dc[j] * xs[j]; KTy[j] = KTys[j] / S->Dc[j]; }
  for (int64_t i = 0; i < m; ++i) { y[i] = S->Dr[i] * ys[i]; Kx[i] = Kxs[i] / S->Dr[i]; }
  kkt_residuals(n, m, S->m1, x, y, Kx, KTy, S->c0, S->q0, S->l0, S->u0, r);
  free(x); free(KTy); free(y); free(Kx);
}

/* Termination test ("relative KKT error ... satisfies the specified
 * termination tolerance"; contract step 5, reading c.3 #21). */
int32_t ora_termination(const ora_kkt *r, double norm_q, double norm_c, double eps_abs, double eps_rel) {
  return r->pres <= eps_abs + eps_rel * norm_q &&
         r->dres <= eps_abs + eps_rel * norm_c &&
         r->gap <= eps_abs + eps_rel * (fabs(r->pobj) + fabs(r->dobj));
}

/* rel_kkt reported in lp_result (contract step 6). */
double ora_rel_kkt(const ora_kkt *r, double norm_q, double norm_c) {
  double a = r->pres / (1.0 + norm_q);
  double b = r->dres / (1.0 + norm_c);
  double g = r->gap / (1.0 + fabs(r->pobj) + fabs(r->dobj));
  return dmax(a, dmax(b, g));
}

/* Weighted scaled-space KKT error used as raPDHG's restart metric ("KKT
 * error for raPDHG"; contract step 5):  sqrt(omega pres~^2 + dres~^2 omega^-1 + gap~^2),
 * omega^-1 = 1 / omega (reading 32). */
static double kkt_omega(const scaled_lp *S, double omega, const double *x, const double *y,
                        const double *Kx, const double *KTy) {
  ora_kkt r;
  kkt_residuals(S->n, S->m, S->m1, x, y, Kx, KTy, S->c, S->q, S->l, S->u, &r);
  double inv_omega = 1.0 / omega;
  return sqrt(omega * r.pres * r.pres + r.dres * r.dres * inv_omega + r.gap * r.gap);
}

/* Initial primal weight and step (contract step 2; readings c.3 #5 and #7):
 *   omega0 = ||c~|| / ||q~|| of the SCALED costs and right-hand side if both exceed 1e-10,
 *            else 1;
 *   eta0   = 1 / max_ij |K~_ij| (adaptive step; 1 if K~ = 0), or 0.998 / sigma_max(K~) for the
 *            constant-step variant (reading 34), so tau sigma ||K~||^2 = eta^2 sigma^2 < 1. */
static void initial_weight_and_step(const scaled_lp *S, const ora_options *o, double *omega, double *eta) {
  const int64_t n = S->n, m = S->m;
  *omega = 1.0;
  double nc = norm2(S->c, n), nq = m ? norm2(S->q, m) : 0.0;
  if (nc > 1e-10 && nq > 1e-10) *omega = nc / nq;
  *eta = 1.0;
  if (o->step_rule != 1) {
    double mx = 0.0;
    for (int64_t k = 0; k < S->K.nnz; ++k) mx = dmax(mx, fabs(S->K.v[k]));
    if (mx > 0.0) *eta = 1.0 / mx;
  } else {
    double sg = power_sigma(&S->K, &S->KT, o->power_iters);
    if (sg > 0.0) *eta = 0.998 / sg;
  }
}

/* raPDHG restart candidate (contract step 5, reading c.3 #10): the average if its
 * KKT_omega is STRICTLY smaller than the current iterate's, else the current iterate
 * (a tie keeps the current point).  Returns 1 for the average. */
int32_t ora_restart_candidate(double kkt_omega_avg, double kkt_omega_cur) {
  return kkt_omega_avg < kkt_omega_cur ? 1 : 0;
}

/* ---------------------------------------------------------- the solve ---- */

static void log_attempt(ora_log *g, int64_t j, int32_t acc, double eta, double eta_bar) {
  if (!g || g->att_len >= g->att_cap) return;
  double *r = g->att + 4 * g->att_len++;
  r[0] = (double)j; r[1] = acc; r[2] = eta; r[3] = eta_bar;
}
static void log_check(ora_log *g, int64_t k, double metric, double ref, double last, int32_t rs, int32_t ps) {
  if (!g || g->chk_len >= g->chk_cap) return;
  double *r = g->chk + 6 * g->chk_len++;
  r[0] = (double)k; r[1] = metric; r[2] = ref; r[3] = last; r[4] = rs; r[5] = ps;
}

static void cpy(double *d, const double *s, int64_t n) { if (n) memcpy(d, s, (size_t)n * sizeof(double)); }

static void fill_result(const scaled_lp *S, const double *xs, const double *ys, const double *Kxs,
                        const double *KTys, int32_t status, int64_t k, int64_t j, int64_t restarts,
                        double omega, double eta, double *x_out, double *y_out, double *lam_out,
                        ora_result *res) {
  ora_kkt r;
  kkt_original_from_scaled(S, xs, ys, Kxs, KTys, &r);
  res->status = status; res->iterations = k; res->attempts = j; res->restarts = restarts;
  res->primal_objective = r.pobj; res->dual_objective = r.dobj;
  res->primal_residual = r.pres; res->dual_residual = r.dres; res->gap = r.gap;
  res->rel_kkt = ora_rel_kkt(&r, S->nq0, S->nc0);
  res->omega = omega; res->eta = eta;
  /* Step 6: x = Dc x~, y = Dr y~, lambda = c - K'y (from the cached product). */
  for (int64_t jj = 0; jj < S->n; ++jj) {
    if (x_out) x_out[jj] = S->Dc[jj] * xs[jj];
    if (lam_out) lam_out[jj] = S->c0[jj] - KTys[jj] / S->Dc[jj];
  }
  if (y_out) for (int64_t i = 0; i < S->m; ++i) y_out[i] = S->Dr[i] * ys[i];
}

/* The certificate test of reading 35 on original-space rays (see ora_certificate).
 * dx (n), Kdx = K dx (m), dy (m), KTdy = K'dy (n); bounds / costs are original. */
static void certificate_test(int64_t n, int64_t m, int64_t m1, const double *c, const double *q,
                             const double *l, const double *u, const double *dx, const double *Kdx,
                             const double *dy, const double *KTdy, double eps_p, double eps_d,
                             ora_certificate *r) {
  double sy = 0.0, sx = 0.0;
  for (int64_t i = 0; i < m; ++i) sy += dy[i] * dy[i];
  for (int64_t j = 0; j < n; ++j) sx += dx[j] * dx[j];
  r->norm_dy = sqrt(sy);
  r->norm_dx = sqrt(sx);
  /* dual ray (primal infeasibility) */
  double obj = 0.0, viol = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    obj += q[i] * dy[i];
    if (i < m1) viol = dmax(viol, dmax(-dy[i], 0.0));
  }
  for (int64_t j = 0; j < n; ++j) {
    double lam = -KTdy[j], lp = dmax(lam, 0.0), lm = dmax(-lam, 0.0);
    if (l[j] > -ORA_INF) obj += l[j] * lp; else viol = dmax(viol, lp);
    if (u[j] < ORA_INF) obj -= u[j] * lm; else viol = dmax(viol, lm);
  }
  r->dual_ray_objective = r->norm_dy > 0.0 ? obj / r->norm_dy : 0.0;
  r->dual_ray_violation = r->norm_dy > 0.0 ? viol / r->norm_dy : 0.0;
  r->primal_infeasible = eps_p >= 0.0 && r->norm_dy > 0.0 && r->dual_ray_objective > eps_p &&
                         r->dual_ray_violation <= eps_p;
  /* primal ray (dual infeasibility) */
  obj = 0.0; viol = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    obj += c[j] * dx[j];
    if (u[j] < ORA_INF) viol = dmax(viol, dmax(dx[j], 0.0));
    if (l[j] > -ORA_INF) viol = dmax(viol, dmax(-dx[j], 0.0));
  }
  for (int64_t i = 0; i < m; ++i) viol = dmax(viol, i < m1 ? dmax(-Kdx[i], 0.0) : fabs(Kdx[i]));
  r->primal_ray_objective = r->norm_dx > 0.0 ? obj / r->norm_dx : 0.0;
  r->primal_ray_violation = r->norm_dx > 0.0 ? viol / r->norm_dx : 0.0;
  r->dual_infeasible = eps_d >= 0.0 && r->norm_dx > 0.0 && r->primal_ray_objective < -eps_d &&
                       r->primal_ray_violation <= eps_d;
}

/* The candidate rays in original space (reading 35): d = z - z_b for the current
 * iterate z = (x, y) and a base point z_b -- for r2HPDHG the epoch's Halpern anchor
 * (= its restart point), for raPDHG the iterate before the last accepted step --
 * unscaled (x = Dc x~, y = Dr y~), with the products from the cached ones:
 * K d_x = (K~x~ - K~x~_b) / Dr, K'd_y = (K~'y~ - K~'y~_b) / Dc. */
static void epoch_rays(const scaled_lp *S, const double *x, const double *y, const double *Kx,
                       const double *KTy, const double *xr, const double *yr, const double *Kxr,
                       const double *KTyr, double *dx, double *Kdx, double *dy, double *KTdy) {
  for (int64_t j = 0; j < S->n; ++j) {
    dx[j] = S->Dc[j] * (x[j] - xr[j]);
    KTdy[j] = (KTy[j] - KTyr[j]) / S->Dc[j];
  }
  for (int64_t i = 0; i < S->m; ++i) {
    dy[i] = S->Dr[i] * (y[i] - yr[i]);
    Kdx[i] = (Kx[i] - Kxr[i]) / S->Dr[i];
  }
}

/* Output for an infeasible status: the result fields describe the current
 * iterate; x_out / y_out / lam_out hold the unit certificate rays d_x/|d_x|,
 * d_y/|d_y| and -K'd_y/|d_y| (zero where a ray is zero). */
static void fill_infeasible(const scaled_lp *S, const double *x, const double *y, const double *Kx,
                            const double *KTy, const double *dx, const double *dy, const double *KTdy,
                            const ora_certificate *cert, int32_t status, int64_t k, int64_t j,
                            int64_t restarts, double omega, double eta, double *x_out, double *y_out,
                            double *lam_out, ora_result *res) {
  fill_result(S, x, y, Kx, KTy, status, k, j, restarts, omega, eta, NULL, NULL, NULL, res);
  const double sx = cert->norm_dx > 0.0 ? cert->norm_dx : 1.0, sy = cert->norm_dy > 0.0 ? cert->norm_dy : 1.0;
  for (int64_t jj = 0; jj < S->n; ++jj) {
    if (x_out) x_out[jj] = dx[jj] / sx;
    if (lam_out) lam_out[jj] = -KTdy[jj] / sy;
  }
  if (y_out) for (int64_t i = 0; i < S->m; ++i) y_out[i] = dy[i] / sy;
}

/* The check's pass test: the relative KKT termination (contract step 5), or for the
 * feasibility-polishing sub-solves (reading 36) the primal (mode 1) or dual (mode 2)
 * residual alone against eps_feas_polish in the same relative form. */
static int32_t check_pass(const ora_kkt *r, const scaled_lp *S, const ora_options *o) {
  const double e = o->eps_feas_polish;
  if (o->polish_mode == 1) return r->pres <= e + e * S->nq0;
  if (o->polish_mode == 2) return r->dres <= e + e * S->nc0;
  return ora_termination(r, S->nq0, S->nc0, o->eps_abs, o->eps_rel);
}

/* One solve on the scaled problem: contract steps 2-6. */
static void solve_scaled(const scaled_lp *S, const ora_options *o, const double *x0, const double *y0,
                         double *x_out, double *y_out, double *lam_out, ora_result *res, ora_log *g) {
  const int64_t n = S->n, m = S->m, m1 = S->m1;
  const int r2 = (o->algorithm == ORA_R2HPDHG);
  const size_t bn = (size_t)n * sizeof(double), bm = (size_t)(m ? m : 1) * sizeof(double);
  /* current z = (x, y) with cached products Kx = K~x, KTy = K~'y */
  double *x = malloc(bn), *KTy = malloc(bn), *y = malloc(bm), *Kx = malloc(bm);
  /* candidate z' = PDHG(z) */
  double *xp = malloc(bn), *KTyp = malloc(bn), *yp = malloc(bm), *Kxp = malloc(bm);
  /* raPDHG average (xa = x-bar) or r2HPDHG anchor z^0, with products */
  double *xa = malloc(bn), *KTya = malloc(bn), *ya = malloc(bm), *Kxa = malloc(bm);
  /* last restart point (for the primal weight) and scratch */
  double *xr = malloc(bn), *yr = malloc(bm), *tn = malloc(bn), *tm = malloc(bm);
  /* infeasibility detection (reading 35): the rays, and for raPDHG the iterate
     before the last accepted step with its products */
  double *rdx = malloc(bn), *rKTdy = malloc(bn), *rdy = malloc(bm), *rKdx = malloc(bm);
  double *xo = malloc(bn), *KTyo = malloc(bn), *yo = malloc(bm), *Kxo = malloc(bm);

  /* ---- Step 2: initialise (P:251 zero start; warm start P:249-267) ---- */
  double omega, eta;
  const int const_step = (o->step_rule == 1);
  initial_weight_and_step(S, o, &omega, &eta);
  for (int64_t jj = 0; jj < n; ++jj) x[jj] = median3(S->l[jj], x0 ? x0[jj] / S->Dc[jj] : 0.0, S->u[jj]);
  for (int64_t i = 0; i < m; ++i) y[i] = y0 ? y0[i] / S->Dr[i] : 0.0;
  project_dual(y, m1);
  csr_spmv(&S->K, x, Kx);
  csr_spmv(&S->KT, y, KTy);
  int64_t j = 0, k = 0, k_in = 0, restarts = 0;
  cpy(xr, x, n); cpy(yr, y, m);
  double last = ORA_INF, ref = 0.0, W = 0.0;
  int ref_set = 0;
  cpy(xa, x, n); cpy(ya, y, m); cpy(Kxa, Kx, m); cpy(KTya, KTy, n);
  if (!r2) { ref = kkt_omega(S, omega, x, y, Kx, KTy); ref_set = 1; }
  int32_t status = 0;
  double metric = 0.0;

  for (;;) {
    /* ---- Step 3: attempts until one is accepted (Eq. pdhg) ---- */
    int32_t acc = 0, rejects = 0;
    double eta_used = eta, M = 0.0, I = 0.0;
    while (!acc) {
      j += 1;
      double tau = eta * (1.0 / omega), sigma = eta * omega;   /* reading 32: x / omega as x * omega^-1 */
      for (int64_t jj = 0; jj < n; ++jj)
        xp[jj] = median3(S->l[jj], x[jj] - tau * (S->c[jj] - KTy[jj]), S->u[jj]);
      csr_spmv(&S->K, xp, Kxp);                                   /* SpMV #1 */
      for (int64_t i = 0; i < m; ++i) yp[i] = y[i] + sigma * (S->q[i] - 2.0 * Kxp[i] + Kx[i]);
      project_dual(yp, m1);
      double dx2 = 0.0, dy2 = 0.0;
      I = 0.0;
      for (int64_t jj = 0; jj < n; ++jj) { double d = xp[jj] - x[jj]; dx2 += d * d; }
      for (int64_t i = 0; i < m; ++i) {
        double d = yp[i] - y[i];
        dy2 += d * d;
        I += d * (Kxp[i] - Kx[i]);
      }
      M = omega * dx2 + dy2 * (1.0 / omega);
      double eta_bar, eta_next;
      eta_used = eta;
      ora_step_size(eta, omega, dx2, dy2, I, j, &eta_bar, &acc, &eta_next);
      if (const_step) { acc = 1; eta_next = eta; }   /* no line search: every step accepted */
      log_attempt(g, j, acc, eta_used, eta_bar);
      eta = eta_next;
      if (!acc && ++rejects >= 100) {
        fill_result(S, x, y, Kx, KTy, ORA_NUMERICAL_ERROR, k, j, restarts, omega, eta,
                    x_out, y_out, lam_out, res);
        goto done;
      }
    }

    /* ---- Step 4: commit the accepted step ---- */
    csr_spmv(&S->KT, yp, KTyp);                                   /* SpMV #2 */
    if (!r2 && ((k + 1) % o->check_frequency == 0 || k + 1 == o->iteration_limit)) {
      /* raPDHG's ray is the step about to be committed: keep its start point */
      cpy(xo, x, n); cpy(yo, y, m); cpy(Kxo, Kx, m); cpy(KTyo, KTy, n);
    }
    k += 1;
    double rP = 0.0;
    if (!r2) {
      cpy(x, xp, n); cpy(y, yp, m); cpy(Kx, Kxp, m); cpy(KTy, KTyp, n);
      double W1 = ora_average_update(n, xa, xp, W, eta_used);
      ora_average_update(m, ya, yp, W, eta_used);
      W = W1;
    } else {
      /* fixed-point residual ||z - PDHG(z)||_P, P = [[I/tau, -K'], [-K, I/sigma]] */
      rP = sqrt(dmax(0.0, M / eta_used - 2.0 * I));
      if (k_in == 0) { ref = rP; ref_set = 1; }
      ora_halpern_rho(n, k_in, o->reflection, x, xp, xa, x);
      ora_halpern_rho(m, k_in, o->reflection, y, yp, ya, y);
      ora_halpern_rho(m, k_in, o->reflection, Kx, Kxp, Kxa, Kx);
      ora_halpern_rho(n, k_in, o->reflection, KTy, KTyp, KTya, KTy);
    }
    k_in += 1;

    /* ---- Step 5: periodic check (every 64 iterations) ---- */
    if (k % o->check_frequency != 0 && k != o->iteration_limit) continue;
    /* infeasibility ("termination, restart, and infeasibility detection";
       reading 35): after the optimality tests, before the iteration limit */
#define INFEASIBILITY_CHECK()                                                                        \
    do {                                                                                             \
      ora_certificate cert;                                                                          \
      if (r2) epoch_rays(S, x, y, Kx, KTy, xa, ya, Kxa, KTya, rdx, rKdx, rdy, rKTdy);                \
      else epoch_rays(S, x, y, Kx, KTy, xo, yo, Kxo, KTyo, rdx, rKdx, rdy, rKTdy);                   \
      certificate_test(n, m, m1, S->c0, S->q0, S->l0, S->u0, rdx, rKdx, rdy, rKTdy,                  \
                       o->eps_primal_infeasible, o->eps_dual_infeasible, &cert);                     \
      if (cert.primal_infeasible || cert.dual_infeasible) {                                          \
        log_check(g, k, 0.0, ref, last, 0, 3);                                                       \
        fill_infeasible(S, x, y, Kx, KTy, rdx, rdy, rKTdy, &cert,                                    \
                        cert.primal_infeasible ? ORA_PRIMAL_INFEASIBLE : ORA_DUAL_INFEASIBLE, k, j,  \
                        restarts, omega, eta, x_out, y_out, lam_out, res);                           \
        goto done;                                                                                   \
      }                                                                                              \
    } while (0)
    const double *cx, *cy, *cKx, *cKTy;   /* the restart candidate */
    int32_t pass = 0;
    if (!r2) {
      csr_spmv(&S->K, xa, Kxa);           /* the average's products: 2 extra SpMVs */
      csr_spmv(&S->KT, ya, KTya);
      ora_kkt ka, kc;
      kkt_original_from_scaled(S, xa, ya, Kxa, KTya, &ka);
      kkt_original_from_scaled(S, x, y, Kx, KTy, &kc);
      if (check_pass(&ka, S, o)) {
        log_check(g, k, 0.0, ref, last, 0, 1);
        fill_result(S, xa, ya, Kxa, KTya, ORA_OPTIMAL, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        goto done;
      }
      if (check_pass(&kc, S, o)) {
        log_check(g, k, 0.0, ref, last, 0, 2);
        fill_result(S, x, y, Kx, KTy, ORA_OPTIMAL, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        goto done;
      }
      INFEASIBILITY_CHECK();
      if (k == o->iteration_limit) {
        int use_avg = ora_rel_kkt(&ka, S->nq0, S->nc0) < ora_rel_kkt(&kc, S->nq0, S->nc0);
        log_check(g, k, 0.0, ref, last, 0, 0);
        if (use_avg) fill_result(S, xa, ya, Kxa, KTya, ORA_ITERATION_LIMIT, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        else fill_result(S, x, y, Kx, KTy, ORA_ITERATION_LIMIT, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        goto done;
      }
      double e_c = kkt_omega(S, omega, x, y, Kx, KTy);
      double e_a = kkt_omega(S, omega, xa, ya, Kxa, KTya);
      if (ora_restart_candidate(e_a, e_c)) { cx = xa; cy = ya; cKx = Kxa; cKTy = KTya; metric = e_a; }
      else { cx = x; cy = y; cKx = Kx; cKTy = KTy; metric = e_c; }
    } else {
      ora_kkt kw;
      kkt_original_from_scaled(S, xp, yp, Kxp, KTyp, &kw);
      if (check_pass(&kw, S, o)) {
        log_check(g, k, rP, ref, last, 0, 1);
        fill_result(S, xp, yp, Kxp, KTyp, ORA_OPTIMAL, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        goto done;
      }
      INFEASIBILITY_CHECK();
      if (k == o->iteration_limit) {
        log_check(g, k, rP, ref, last, 0, 0);
        fill_result(S, xp, yp, Kxp, KTyp, ORA_ITERATION_LIMIT, k, j, restarts, omega, eta, x_out, y_out, lam_out, res);
        goto done;
      }
      cx = xp; cy = yp; cKx = Kxp; cKTy = KTyp; metric = rP;
    }
    int32_t rs = ora_restart_test(k_in, k, metric, ref, last);
    log_check(g, k, metric, ref, last, rs, 0);
    last = metric;
    if (rs) {
      restarts += 1;
      /* copy through scratch: the candidate may alias the current point */
      cpy(tn, cx, n); cpy(x, tn, n); cpy(tn, cKTy, n); cpy(KTy, tn, n);
      cpy(tm, cy, m); cpy(y, tm, m); cpy(tm, cKx, m); cpy(Kx, tm, m);
      double dxn = dist2(x, xr, n), dyn = dist2(y, yr, m);
      omega = ora_primal_weight(omega, dxn, dyn);
      cpy(xr, x, n); cpy(yr, y, m);
      k_in = 0;
      cpy(xa, x, n); cpy(ya, y, m); cpy(Kxa, Kx, m); cpy(KTya, KTy, n);
      if (!r2) { W = 0.0; ref = metric; }
      else ref_set = 0;
    }
  }
done:
  (void)ref_set;
  free(x); free(KTy); free(y); free(Kx); free(xp); free(KTyp); free(yp); free(Kxp);
  free(xa); free(KTya); free(ya); free(Kxa); free(xr); free(yr); free(tn); free(tm);
  free(rdx); free(rKTdy); free(rdy); free(rKdx); free(xo); free(KTyo); free(yo); free(Kxo);
}

/* Feasibility polishing ("as a final step, feasibility polishing is applied
 * ... to further enhance the feasibility of the solution"; SPEC
 * S:439-447; reading 36).  After an OPTIMAL main solve:
 *   primal polish: the same LP with c = 0, started at (x*, 0), until the primal residual
 *     alone passes eps_feas_polish (relative form, mode 1);
 *   dual polish:   the same LP with q = 0, started at (proj(0), y*), until the dual residual
 *     alone passes (mode 2);
 * both with the main algorithm and options, infeasibility detection off, each limited to
 * min(iteration_limit, ORA_POLISH_LIMIT) accepted steps (the q = 0 problem need not be
 * solvable even when the LP is, so an unbounded polish is never started).  The result is
 * (x from the primal polish, y and lambda from the dual polish); its KKT fields are
 * recomputed on the original data with the unscaled K; counts are summed over the three
 * solves; `polish` = 1 if both polish solves passed, 2 if one reached the iteration limit. */
int ora_spmv_pair(const ora_problem *p, const double *x, double *Kx, const double *w, double *KTw);

static void solve_polished(const ora_problem *p, const scaled_lp *S, const ora_options *o, const double *x0,
                           const double *y0, double *x_out, double *y_out, double *lam_out, ora_result *res,
                           ora_log *g) {
  const int64_t n = S->n, m = S->m;
  if (!o->feasibility_polishing) {
    solve_scaled(S, o, x0, y0, x_out, y_out, lam_out, res, g);
    return;
  }
  const size_t bn = (size_t)n * sizeof(double), bm = (size_t)(m ? m : 1) * sizeof(double);
  double *xm = malloc(bn), *ym = malloc(bm), *lm = malloc(bn), *xp = malloc(bn), *yd = malloc(bm), *ld = malloc(bn);
  double *zn = calloc((size_t)n, sizeof(double)), *zm = calloc((size_t)(m ? m : 1), sizeof(double));
  double *Kx = malloc(bm), *KTy = malloc(bn);
  solve_scaled(S, o, x0, y0, xm, ym, lm, res, g);
  if (res->status != ORA_OPTIMAL) {
    if (x_out) cpy(x_out, xm, n);
    if (y_out) cpy(y_out, ym, m);
    if (lam_out) cpy(lam_out, lm, n);
  } else {
    ora_options op = *o;
    op.feasibility_polishing = 0;
    if (op.iteration_limit > ORA_POLISH_LIMIT) op.iteration_limit = ORA_POLISH_LIMIT;
    op.eps_primal_infeasible = -1.0;
    op.eps_dual_infeasible = -1.0;
    ora_result r1, r2;
    memset(&r1, 0, sizeof(r1)); memset(&r2, 0, sizeof(r2));
    scaled_lp S1 = *S;                    /* c = 0 (scaled and original) */
    S1.c = zn; S1.c0 = zn; S1.nc0 = 0.0;
    op.polish_mode = 1;
    solve_scaled(&S1, &op, xm, NULL, xp, NULL, NULL, &r1, NULL);
    scaled_lp S2 = *S;                    /* q = 0 */
    S2.q = zm; S2.q0 = zm; S2.nq0 = 0.0;
    op.polish_mode = 2;
    solve_scaled(&S2, &op, NULL, ym, NULL, yd, ld, &r2, NULL);
    /* the polished pair on the original data */
    ora_kkt r;
    ora_spmv_pair(p, xp, Kx, yd, KTy);
    kkt_residuals(n, m, p->m1, xp, yd, Kx, KTy, p->c, p->q, p->l, p->u, &r);
    res->iterations += r1.iterations + r2.iterations;
    res->attempts += r1.attempts + r2.attempts;
    res->restarts += r1.restarts + r2.restarts;
    res->primal_objective = r.pobj; res->dual_objective = r.dobj;
    res->primal_residual = r.pres; res->dual_residual = r.dres; res->gap = r.gap;
    res->rel_kkt = ora_rel_kkt(&r, S->nq0, S->nc0);
    res->polish = (r1.status == ORA_OPTIMAL && r2.status == ORA_OPTIMAL) ? 1 : 2;
    if (x_out) cpy(x_out, xp, n);
    if (y_out) cpy(y_out, yd, m);
    if (lam_out) cpy(lam_out, ld, n);
  }
  free(xm); free(ym); free(lm); free(xp); free(yd); free(ld); free(zn); free(zm); free(Kx); free(KTy);
}

/* ------------------------------------------------------------ exports ---- */

void ora_default_options(ora_options *o) {
  o->eps_abs = 1e-4; o->eps_rel = 1e-4;          /* Appendix */
  o->iteration_limit = INT64_MAX;                /* Appendix */
  o->check_frequency = 64;
  o->algorithm = ORA_R2HPDHG;
  o->ruiz_iters = 10; o->pock_chambolle = 1;     /* contract c.3 #3 */
  o->step_rule = 0; o->power_iters = 200;
  o->eps_primal_infeasible = 1e-8;               /* Appendix */
  o->eps_dual_infeasible = 1e-8;                 /* Appendix */
  o->eps_feas_polish = 1e-6;                     /* Appendix */
  o->feasibility_polishing = 0;                  /* Appendix */
  o->polish_mode = 0;
  o->reflection = 1.0;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void ora_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

static int check_options(const ora_options *o) {
  if (!o || !(o->eps_abs >= 0.0) || !(o->eps_rel >= 0.0) || o->iteration_limit < 1 ||
      o->check_frequency < 1 || (o->algorithm != ORA_RAPDHG && o->algorithm != ORA_R2HPDHG) ||
      o->step_rule < 0 || o->step_rule > 1 || o->power_iters < 1 || !(o->eps_feas_polish >= 0.0) ||
      o->polish_mode < 0 || o->polish_mode > 2 || !(o->reflection >= 0.0 && o->reflection <= 1.0))
    return ORA_ERR_INVALID;
  return ORA_OK;
}

/* Wall-clock split of the calling thread's last ora_solve (bench.py's CPU baseline beside C5):
 * setup = validation + preconditioning + scaled copies, solve = steps 2-6.  Timing only. */
static _Thread_local ora_time_t g_t_setup = 0, g_t_solve = 0;
static ora_time_t wall(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (ora_time_t)t.tv_sec + (ora_time_t)t.tv_nsec / (ora_time_t)1000000000;
}
void ora_last_timing(ora_time_t *setup_s, ora_time_t *solve_s) {
  if (setup_s) *setup_s = g_t_setup;
  if (solve_s) *solve_s = g_t_solve;
}

/* Full single solve (contract steps 0-6).  x0/y0 (original space) may be NULL;
 * x_out (n), y_out (m), lam_out (n) may be NULL; log may be NULL. */
int ora_solve(const ora_problem *p, const ora_options *o, const double *x0, const double *y0,
              double *x_out, double *y_out, double *lam_out, ora_result *res, ora_log *g) {
  const ora_time_t t0 = wall();
  int e = ora_validate(p);
  if (e) return e;
  if ((e = check_options(o))) return e;
  int64_t m = p->m1 + p->m2;
  double *Dr = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *Dc = (double *)malloc((size_t)p->n * sizeof(double));
  if (!Dr || !Dc) { free(Dr); free(Dc); return ORA_ERR_OOM; }
  ora_precondition(p, o->ruiz_iters, o->pock_chambolle, Dr, Dc);
  scaled_lp S;
  if ((e = build_scaled(p, Dr, Dc, NULL, NULL, &S))) { free(Dr); free(Dc); return e; }
  if (g) { g->att_len = 0; g->chk_len = 0; }
  memset(res, 0, sizeof(*res));
  const ora_time_t t1 = wall();
  solve_polished(p, &S, o, x0, y0, x_out, y_out, lam_out, res, g);
  g_t_setup = t1 - t0;
  g_t_solve = wall() - t1;
  scaled_free(&S, 1);
  free(Dr); free(Dc);
  return ORA_OK;
}

/* Batch of instances sharing K, l, u (contract step 6 "Batch": the
 * instances share step 1, all other state is per instance).  C is batch x n
 * (NULL: use p->c for all), Q is batch x m (NULL: use p->q).  X0/Y0 optional
 * (batch x n / batch x m).  Instances run in parallel, one per thread. */
int ora_solve_batch(const ora_problem *p, int64_t batch, const double *C, const double *Q,
                    const ora_options *o, const double *X0, const double *Y0,
                    double *X_out, double *Y_out, ora_result *res) {
  int e = ora_validate(p);
  if (e) return e;
  if ((e = check_options(o))) return e;
  if (batch < 0) return ORA_ERR_INVALID;
  int64_t n = p->n, m = p->m1 + p->m2;
  for (int64_t b = 0; b < batch; ++b) {
    if (C) for (int64_t j = 0; j < n; ++j) if (!isfinite(C[b * n + j])) return ORA_ERR_NAN;
    if (Q) for (int64_t i = 0; i < m; ++i) if (!isfinite(Q[b * m + i])) return ORA_ERR_NAN;
  }
  double *Dr = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *Dc = (double *)malloc((size_t)n * sizeof(double));
  csr K, KT;
  ora_precondition(p, o->ruiz_iters, o->pock_chambolle, Dr, Dc);
  if ((e = scale_matrix(p, Dr, Dc, &K, &KT))) return e;
  int64_t b;
#pragma omp parallel for schedule(dynamic, 1)
  for (b = 0; b < batch; ++b) {
    ora_problem pb = *p;
    if (C) pb.c = C + b * n;
    if (Q) pb.q = Q + b * m;
    scaled_lp S;
    if (build_scaled(&pb, Dr, Dc, &K, &KT, &S) == ORA_OK) {
      memset(&res[b], 0, sizeof(res[b]));
      solve_polished(&pb, &S, o, X0 ? X0 + b * n : NULL, Y0 ? Y0 + b * m : NULL,
                     X_out ? X_out + b * n : NULL, Y_out ? Y_out + b * m : NULL, NULL, &res[b], NULL);
    }
    scaled_free(&S, 0);
  }
  csr_free(&K); csr_free(&KT);
  free(Dr); free(Dc);
  return ORA_OK;
}

/* ---- step-level entry points used by the pins (tests/test_oracle_*.py) ---- */

/* The scaled data of step 1: K~ (CSR values in K's pattern), K~' (CSR), c~, q~, l~, u~. */
int ora_scaled_problem(const ora_problem *p, int32_t ruiz_iters, int32_t pc, double *Dr, double *Dc,
                       double *Kv, int64_t *KTrp, int32_t *KTci, double *KTv,
                       double *cs, double *qs, double *ls, double *us) {
  int e = ora_validate(p);
  if (e) return e;
  ora_precondition(p, ruiz_iters, pc, Dr, Dc);
  scaled_lp S;
  if ((e = build_scaled(p, Dr, Dc, NULL, NULL, &S))) return e;
  int64_t n = p->n, m = S.m;
  if (Kv) cpy(Kv, S.K.v, p->nnz);
  if (KTrp) memcpy(KTrp, S.KT.rp, (size_t)(n + 1) * sizeof(int64_t));
  if (KTci && p->nnz) memcpy(KTci, S.KT.ci, (size_t)p->nnz * sizeof(int32_t));
  if (KTv) cpy(KTv, S.KT.v, p->nnz);
  if (cs) cpy(cs, S.c, n);
  if (qs) cpy(qs, S.q, m);
  if (ls) cpy(ls, S.l, n);
  if (us) cpy(us, S.u, n);
  scaled_free(&S, 1);
  return ORA_OK;
}

/* y = K x and t = K' w with the (unscaled) problem matrix. */
int ora_spmv_pair(const ora_problem *p, const double *x, double *Kx, const double *w, double *KTw) {
  csr K = { p->m1 + p->m2, p->n, p->nnz, (int64_t *)p->row_ptr, (int32_t *)p->col_idx, (double *)p->val };
  csr KT;
  if (csr_transpose(&K, &KT)) return ORA_ERR_OOM;
  if (x && Kx) csr_spmv(&K, x, Kx);
  if (w && KTw) csr_spmv(&KT, w, KTw);
  csr_free(&KT);
  return ORA_OK;
}

/* One literal PDHG step, Eq. (pdhg), on the problem as given (no scaling):
 * x+ = proj_X(x - tau (c - K'y)); y+ = proj_Y(y + sigma (q - K(2x+ - x))). */
int ora_pdhg_step(const ora_problem *p, const double *x, const double *y, double tau, double sigma,
                  double *x_out, double *y_out) {
  int64_t n = p->n, m = p->m1 + p->m2;
  double *KTy = malloc((size_t)n * sizeof(double)), *ex = malloc((size_t)n * sizeof(double));
  double *Kex = malloc((size_t)(m ? m : 1) * sizeof(double));
  int e = ora_spmv_pair(p, NULL, NULL, y, KTy);
  for (int64_t j = 0; j < n; ++j) x_out[j] = median3(p->l[j], x[j] - tau * (p->c[j] - KTy[j]), p->u[j]);
  for (int64_t j = 0; j < n; ++j) ex[j] = 2.0 * x_out[j] - x[j];
  e = e ? e : ora_spmv_pair(p, ex, Kex, NULL, NULL);
  for (int64_t i = 0; i < m; ++i) y_out[i] = y[i] + sigma * (p->q[i] - Kex[i]);
  project_dual(y_out, p->m1);
  free(KTy); free(ex); free(Kex);
  return e;
}

/* The projections of Eq. (pdhg) as standalone calls. */
void ora_project_box(int64_t n, const double *l, const double *u, double *x) {
  for (int64_t j = 0; j < n; ++j) x[j] = median3(l[j], x[j], u[j]);
}
void ora_project_dual(int64_t m1, double *y) { project_dual(y, m1); }

/* Independent original-space KKT of (x, y): products with the UNSCALED K
 * ("recomputed from scratch on original data"). */
int ora_kkt_original(const ora_problem *p, const double *x, const double *y, ora_kkt *out) {
  int64_t n = p->n, m = p->m1 + p->m2;
  double *Kx = malloc((size_t)(m ? m : 1) * sizeof(double)), *KTy = malloc((size_t)n * sizeof(double));
  int e = ora_spmv_pair(p, x, Kx, y, KTy);
  kkt_residuals(n, m, p->m1, x, y, Kx, KTy, p->c, p->q, p->l, p->u, out);
  free(Kx); free(KTy);
  return e;
}

/* sigma_max of the problem's K (as given) by the same power iteration (pins: SPEC S:144-146). */
int ora_spectral_norm(const ora_problem *p, int32_t iters, double *sigma) {
  csr K = { p->m1 + p->m2, p->n, p->nnz, (int64_t *)p->row_ptr, (int32_t *)p->col_idx, (double *)p->val };
  csr KT;
  if (csr_transpose(&K, &KT)) return ORA_ERR_OOM;
  *sigma = power_sigma(&K, &KT, iters);
  csr_free(&KT);
  return ORA_OK;
}

/* The certificate test of reading 35 on user-given original-space rays (d_x, d_y),
 * with products from the unscaled K (pins: SPEC S:425-426 Farkas examples). */
int ora_certificate_test(const ora_problem *p, const double *dx, const double *dy, double eps_p, double eps_d,
                         ora_certificate *out) {
  int64_t n = p->n, m = p->m1 + p->m2;
  double *Kdx = malloc((size_t)(m ? m : 1) * sizeof(double)), *KTdy = malloc((size_t)n * sizeof(double));
  int e = ora_spmv_pair(p, dx, Kdx, dy, KTdy);
  if (!e) certificate_test(n, m, p->m1, p->c, p->q, p->l, p->u, dx, Kdx, dy, KTdy, eps_p, eps_d, out);
  free(Kdx); free(KTdy);
  return e;
}

/* Weighted KKT error of (x, y) on the problem AS GIVEN (no scaling; products with K):
 * the raPDHG restart metric sqrt(omega pres^2 + dres^2 / omega + gap^2) of contract step 5,
 * evaluated by the same routine the solve applies to the scaled problem (pins). */
int ora_kkt_omega(const ora_problem *p, double omega, const double *x, const double *y, double *out) {
  int64_t n = p->n, m = p->m1 + p->m2;
  double *Kx = malloc((size_t)(m ? m : 1) * sizeof(double)), *KTy = malloc((size_t)n * sizeof(double));
  int e = ora_spmv_pair(p, x, Kx, y, KTy);
  scaled_lp S;
  memset(&S, 0, sizeof(S));
  S.n = n; S.m = m; S.m1 = p->m1;
  S.c = (double *)p->c; S.q = (double *)p->q; S.l = (double *)p->l; S.u = (double *)p->u;
  if (!e) *out = kkt_omega(&S, omega, x, y, Kx, KTy);
  free(Kx); free(KTy);
  return e;
}

/* omega0 and eta0 of contract step 2 for the problem scaled with the options'
 * ruiz_iters / pock_chambolle (pins of readings c.3 #5, #7 and 34). */
int ora_initial_steps(const ora_problem *p, const ora_options *o, double *omega0, double *eta0) {
  int e = ora_validate(p);
  if (e) return e;
  if ((e = check_options(o))) return e;
  int64_t m = p->m1 + p->m2;
  double *Dr = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
  double *Dc = (double *)malloc((size_t)p->n * sizeof(double));
  ora_precondition(p, o->ruiz_iters, o->pock_chambolle, Dr, Dc);
  scaled_lp S;
  if ((e = build_scaled(p, Dr, Dc, NULL, NULL, &S)) == ORA_OK) initial_weight_and_step(&S, o, omega0, eta0);
  scaled_free(&S, 1);
  free(Dr); free(Dc);
  return e;
}

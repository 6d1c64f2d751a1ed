// tiny_solver.cu -- register-resident per-instance PDHG for very small LPs
// (the paper's batched shortest-path LPs, P:334,
// P:156-157; and C1-sized single LPs).  NT threads own one instance (NT = 32: one warp, the
// C2 batches; NT = 64..256: a CTA, for LPs up to NT*RPT rows / NT*CPT columns); thread l
// owns rows i = l + NT t (t < RPT) and columns j = l + NT t (t < CPT) together with their
// ELL rows of K~ (width W) and K~' (width WT).  Every per-row / per-column quantity of the
// iteration (x, K~'y, x', average / anchor, restart point, c~, l~, u~ and the
// m-side analogues) lives in registers; only the two vectors that are
// gathered by the SpMVs (x' and y', and the average at checks) go through
// shared memory.  The contract's arithmetic (common.cuh helpers) in
// the oracle's order; sums run in lane / butterfly order (reading 27).
#include <cstdlib>

#include "common.cuh"

namespace mpax {

namespace {

struct TinyParams {
  int32_t n, m, m1;
  const int32_t *rp, *ci, *trp, *tci;
  const double *kv, *tkv, *Dr, *Dc, *ls, *us, *l0, *u0;
  const double *C0, *Q0, *X0, *Y0;
  int64_t cstride, qstride;
  const double *kmax, *sigma, *tab;
  double eps_abs, eps_rel, eps_pi, eps_di, eps_fp, rho;
  int64_t iter_limit;
  int32_t check_freq, polish_mode, verbose, display_freq;
  const lp_result *active;
  int64_t batch;
  unsigned long long *queue, qbase;
  double *X, *Y, *L;
  lp_result *res, *res_host;
  // decision log of instance log_inst (LG instantiations only): per attempt (j, accepted, eta,
  // eta_bar), per check (k, metric, ref, last, restart, outcome) -- the oracle's ora_log records
  double *alog, *clog;
  int64_t acap, ccap, log_inst;
};

// Barrier of the instance's threads: the warp, or the CTA.
template <int NT>
__device__ __forceinline__ void isync() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

constexpr int kRedV = 24;  // the largest reduction (raPDHG check)

template <int V>
__device__ __forceinline__ void wsum(double (&v)[V]) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    v[k] = s;
  }
}

template <int V>
__device__ __forceinline__ void wmax(double (&v)[V]) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s = fmax(s, __shfl_xor_sync(FULL, s, off));
    v[k] = s;
  }
}

// Sum (MX = false) or max over the instance's NT threads, every thread getting the total: the
// warp butterfly, then (NT > 32) the warps' partials through shared memory in warp order --
// fixed order, deterministic.  `red` holds 2 x (NT / 32) x kRedV doubles; `rb` alternates
// between its halves, so a buffer is rewritten only after an intervening barrier.
template <int NT, bool MX, int V>
__device__ __forceinline__ void ired(double (&v)[V], double *red, int &rb) {
  if (MX) wmax<V>(v); else wsum<V>(v);
  if (NT == 32) return;
  double *buf = red + rb * (NT / 32) * kRedV;
  rb ^= 1;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) buf[w * kRedV + k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = buf[k];
    for (int ww = 1; ww < NT / 32; ++ww) s = MX ? fmax(s, buf[ww * kRedV + k]) : s + buf[ww * kRedV + k];
    v[k] = s;
  }
}


// CS: constant step rule (eta = 0.998 / sigma_max(K~), every attempt accepted; DESIGN.md
// reading 34) -- the line-search reductions are then needed only where r2HPDHG uses
// r_P (restart reference at k_in = 0 and the check), and never for raPDHG.
template <bool R2, bool CS, int NT, int RPT, int CPT, int W, int WT, bool LG = false>
__global__ void __launch_bounds__(NT) tiny_kernel(const TinyParams P) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x;   // the thread's index within its instance (0 .. NT-1)
  const int n = P.n, m = P.m, m1 = P.m1;
  double *sx = sm, *sy = sm + NT * CPT;  // gather buffers: x' (or average) and y' (or average)
  double *red = sy + NT * RPT;           // cross-warp reduction scratch (NT > 32)
  int rb = 0;
  // ---- static per-lane structure: ELL rows of K~ and K~' in registers ----
  int rcol[RPT][W], ccol[CPT][WT];
  double rval[RPT][W], cval[CPT][WT];
  bool rok[RPT], cok[CPT];
  double dr[RPT], lsv[CPT], usv[CPT], dc[CPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = lane + NT * t;
    rok[t] = i < m;
    const int a = rok[t] ? P.rp[i] : 0, e = rok[t] ? P.rp[i + 1] : 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const bool ok = a + w < e;
      rcol[t][w] = ok ? P.ci[a + w] : 0;
      rval[t][w] = ok ? P.kv[a + w] : 0.0;
    }
    dr[t] = rok[t] ? P.Dr[i] : 1.0;
  }
#pragma unroll
  for (int t = 0; t < CPT; ++t) {
    const int j = lane + NT * t;
    cok[t] = j < n;
    const int a = cok[t] ? P.trp[j] : 0, e = cok[t] ? P.trp[j + 1] : 0;
#pragma unroll
    for (int w = 0; w < WT; ++w) {
      const bool ok = a + w < e;
      ccol[t][w] = ok ? P.tci[a + w] : 0;
      cval[t][w] = ok ? P.tkv[a + w] : 0.0;
    }
    dc[t] = cok[t] ? P.Dc[j] : 1.0;
    lsv[t] = cok[t] ? P.ls[j] : 0.0;
    usv[t] = cok[t] ? P.us[j] : 0.0;
  }
  // padding entries point at element 0 with value 0; keep the gather buffers finite
  for (int t = lane; t < NT * CPT; t += NT) sx[t] = 0.0;
  for (int t = lane; t < NT * RPT; t += NT) sy[t] = 0.0;
  const double eta0 = initial_eta(P.kmax, P.sigma, CS);
  // r2HPDHG reflection z <- a((1 + rho) w - rho z) + b z0 (rho = 1: 2 PDHG(z) - z; reading 38)
  const double rf1 = 1.0 + P.rho, rf0 = P.rho;
  // the check's pass test: relative KKT, or a polishing sub-solve's single residual (reading 36)
  auto tpass = [&](const Kkt5 &k, double nq, double nc) {
    return P.polish_mode ? polish_pass(P.polish_mode, k.pres, k.dres, nq, nc, P.eps_fp)
                         : kkt5_pass(k, nq, nc, P.eps_abs, P.eps_rel);
  };
  __shared__ unsigned long long s_inst;

  for (;;) {
    isync<NT>();
    if (lane == 0) s_inst = atomicAdd(P.queue, 1ull) - P.qbase;
    isync<NT>();
    const int64_t b = (int64_t)s_inst;
    if (b >= P.batch) return;
    if (P.active && P.active[b].status != LP_OPTIMAL) continue;  // polishing: main solve not OPTIMAL
    const double *c0 = P.C0 + b * P.cstride, *q0 = P.Q0 + b * P.qstride;

    // ---- step 2 ----
    double x[CPT], KTy[CPT], xp[CPT], KTyp[CPT], xa[CPT], KTya[CPT], xr[CPT], cs[CPT];
    double y[RPT], Kx[RPT], yp[RPT], Kxp[RPT], ya[RPT], Kxa[RPT], yr[RPT], qs[RPT];
    double v4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < CPT; ++t) {
      const int j = lane + NT * t;
      const double c = cok[t] ? c0[j] : 0.0;
      cs[t] = c * dc[t];
      v4[0] += cs[t] * cs[t];
      v4[2] += c * c;
      const double x0 = (cok[t] && P.X0) ? P.X0[b * n + j] / dc[t] : 0.0;
      x[t] = cok[t] ? median3(lsv[t], x0, usv[t]) : 0.0;
      sx[j] = x[t];
    }
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = lane + NT * t;
      const double q = rok[t] ? q0[i] : 0.0;
      qs[t] = q * dr[t];
      v4[1] += qs[t] * qs[t];
      v4[3] += q * q;
      double yv = (rok[t] && P.Y0) ? P.Y0[b * m + i] / dr[t] : 0.0;
      if (i < m1) yv = fmax(yv, 0.0);
      y[t] = rok[t] ? yv : 0.0;
      sy[i] = y[t];
    }
    ired<NT, false>(v4, red, rb);
    isync<NT>();
    const double nc0 = sqrt(v4[2]), nq0 = sqrt(v4[3]);
    double omega = 1.0;
    if (sqrt(v4[0]) > 1e-10 && sqrt(v4[1]) > 1e-10) omega = sqrt(v4[0]) / sqrt(v4[1]);
    double eta = eta0, ref = 0.0;
    // omega^-1 = 1 / omega, recomputed whenever omega changes; every x / omega of the iteration
    // is x * omega^-1 (reading 32, the same in the oracle and every kernel)
    double inv_omega = 1.0 / omega;
    {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) s += rval[t][w] * sx[rcol[t][w]];
        Kx[t] = s; Kxa[t] = s; ya[t] = y[t]; yr[t] = y[t];
        if (rok[t]) kkt_row_acc(v, false, lane + NT * t < m1, 1.0, y[t], s, 0.0, qs[t]);
      }
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WT; ++w) s += cval[t][w] * sy[ccol[t][w]];
        KTy[t] = s; KTya[t] = s; xa[t] = x[t]; xr[t] = x[t];
        if (cok[t]) kkt_col_acc(v, false, 1.0, x[t], s, 0.0, cs[t], 0.0, lsv[t], 0.0, usv[t]);
      }
      ired<NT, false>(v, red, rb);
      if (!R2) {
        const Kkt5 ks = kkt5(v);
        ref = kkt_omega(ks, omega, inv_omega);
      }
    }
#pragma unroll
    for (int t = 0; t < CPT; ++t) { xp[t] = x[t]; KTyp[t] = KTy[t]; }
#pragma unroll
    for (int t = 0; t < RPT; ++t) { yp[t] = y[t]; Kxp[t] = Kx[t]; }
    int64_t k = 0, jatt = 0, k_in = 0, restarts = 0;
    int64_t next_check = P.check_freq < P.iter_limit ? P.check_freq : P.iter_limit;  // k % F == 0 || k == limit
    // K~'y' of the latest candidate, gathered at the end of each attempt (off the next attempt's
    // critical path): the n-side commit of an accepted step uses it
    double KTyn[CPT];
#pragma unroll
    for (int t = 0; t < CPT; ++t) KTyn[t] = KTy[t];
    // line-search factors of the NEXT attempt, loaded one attempt ahead
    double f1n = 0.0, f2n = 0.0;
    if (!CS) step_factors(P.tab, 1, f1n, f2n);
    const double *ftab = P.tab + 2 * 2;  // the table entry of attempt jatt + 2 (loop-carried pointer)
    double W_ = 0.0, last = INFINITY, theta = 0.0, ha = 0.0, hb = 0.0;
    int status = 0, rejects = 0;
    int64_t nchk = 0;   // checks logged (LG)
    auto log_check = [&](double metric_, int restart_, int outcome) {
      if (LG && b == P.log_inst && lane == 0 && nchk < P.ccap) {
        double *r = P.clog + 6 * nchk;
        r[0] = (double)k; r[1] = metric_; r[2] = ref; r[3] = last; r[4] = restart_; r[5] = outcome;
      }
      ++nchk;
    };
    bool pending = false;
    int outsel = 0;  // 0 current, 1 candidate w / average, as set at termination
    bool rays = false;  // infeasible: the certificate rays are already written (reading 35)
    // the unit rays d_x / |d_x|, d_y / |d_y|, -K'd_y / |d_y| against the base point (xb, KTyb, yb)
    auto write_rays = [&](int64_t bi, double ny, double nx, const double (&xb)[CPT], const double (&KTyb)[CPT],
                          const double (&yb)[RPT]) {
      double *X = P.X + bi * (int64_t)n, *L = P.L + bi * (int64_t)n, *Y = P.Y + bi * (int64_t)m;
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        const int j = lane + NT * t;
        if (cok[t]) {
          X[j] = dc[t] * (x[t] - xb[t]) / nx;
          L[j] = -((KTy[t] - KTyb[t]) / dc[t]) / ny;
        }
      }
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int i = lane + NT * t;
        if (rok[t]) Y[i] = dr[t] * (y[t] - yb[t]) / ny;
      }
    };

    // Shared-memory hazards of the attempt loop: every write of sx (phase A) / sy (phase B) is
    // separated from the previous reads of that buffer by one of the loop's two instance barriers (isync)
    // (after phase A, after phase B); the check path ends with its own.
    isync<NT>();
    for (;;) {
      // ================= phase A: [commit n-side] + primal step =================
      // Branch-free: the commit is computed every attempt and selected by `pending`
      // (theta_p = 0 leaves the average bit-identical), so the attempt is one basic block.
      const double tau = eta * inv_omega, sigma = eta * omega;
      // raPDHG's averaging weight eta / (W + eta) if this attempt is accepted: its division's fast
      // path is issued beside the (dy2, I) butterfly below, whose shuffle chain hides the Newton
      // chain (issued here, the in-order warp stalled on it before the primal step: 9% of the
      // attempt, ncu source page); its (rare) slow path only at acceptance (bit-identical to /)
      const double W1c = W_ + eta;
      const double theta_p = pending ? theta : 0.0;
      const double f1 = f1n, f2 = f2n;
      if (!CS) {
        // the table entry of attempt jatt + 2, without a branch: the pointer stops on the table's
        // last entry, and past the table the factors are replaced at the end of the previous
        // attempt (the out-of-line pow, in the loop's rarely taken tail)
        f1n = __ldg(ftab);
        f2n = __ldg(ftab + 1);
        ftab += (jatt + 3 < kStepTab) ? 2 : 0;
      }
      // r2HPDHG: the Halpern coefficients this attempt commits with if accepted (index k_in),
      // loaded now so the table latency overlaps the attempt instead of the next commit
      double ha_n = 0.0, hb_n = 0.0;
      if (R2) halpern_coeffs(P.tab, k_in, ha_n, hb_n);
      // warp-uniform: does this attempt need ||dx||, ||dy||, <dy, K dx>?
      const bool need = !CS || (R2 && (k_in == 0 || k + 1 == next_check));
      double dx2 = 0.0;
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        const double s = KTyn[t];
        if (!R2) {
          xa[t] += theta_p * (xp[t] - xa[t]);
          x[t] = pending ? xp[t] : x[t];
          KTy[t] = pending ? s : KTy[t];
        } else {
          const double xc = ha * (rf1 * xp[t] - rf0 * x[t]) + hb * xa[t];
          const double kc = ha * (rf1 * s - rf0 * KTy[t]) + hb * KTya[t];
          x[t] = pending ? xc : x[t];
          KTy[t] = pending ? kc : KTy[t];
        }
        const double xn = median3(lsv[t], x[t] - tau * (cs[t] - KTy[t]), usv[t]);
        xp[t] = cok[t] ? xn : 0.0;
        sx[lane + NT * t] = xp[t];
        const double d = xp[t] - x[t];
        dx2 += d * d;
      }
      double vdx[1] = {dx2};
      if (NT == 32 && need) wsum<1>(vdx);  // ||dx||^2: its butterfly overlaps phase B (one warp)
      isync<NT>();
      // ================= phase B: [commit m-side] + SpMV #1 + dual step =================
      double dy2 = 0.0, I = 0.0;
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) s += rval[t][w] * sx[rcol[t][w]];
        if (!R2) {
          ya[t] += theta_p * (yp[t] - ya[t]);
          y[t] = pending ? yp[t] : y[t];
          Kx[t] = pending ? Kxp[t] : Kx[t];
        } else {
          const double yc = ha * (rf1 * yp[t] - rf0 * y[t]) + hb * ya[t];
          const double kc = ha * (rf1 * Kxp[t] - rf0 * Kx[t]) + hb * Kxa[t];
          y[t] = pending ? yc : y[t];
          Kx[t] = pending ? kc : Kx[t];
        }
        // q~ - 2 K~x' as one fma: 2 s is exact, so this is the oracle's q~ - 2.0 * s, one op shorter
        double yn = y[t] + sigma * (fma(-2.0, s, qs[t]) + Kx[t]);
        if (lane + NT * t < m1) yn = pos_part(yn);
        yp[t] = rok[t] ? yn : 0.0;
        Kxp[t] = rok[t] ? s : 0.0;
        sy[lane + NT * t] = yp[t];
        const double d = yp[t] - y[t];
        dy2 += d * d;
        I += d * (Kxp[t] - Kx[t]);
      }
      pending = false;
      double v3[2] = {dy2, I};
      bool theta_ok = true;
      const double theta_f = R2 ? 0.0 : div_rn_fast(eta, W1c, theta_ok);
      if (need) {  // ||dy||^2, <dy, K dx> (and ||dx||^2 for a CTA instance)
        if (NT == 32) {
          wsum<2>(v3);
        } else {
          double v3x[3] = {vdx[0], v3[0], v3[1]};
          ired<NT, false>(v3x, red, rb);
          vdx[0] = v3x[0]; v3[0] = v3x[1]; v3[1] = v3x[2];
        }
      }
      // K~'y' for the next attempt's commit (and this one's check), overlapping the butterfly
      isync<NT>();
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WT; ++w) s += cval[t][w] * sy[ccol[t][w]];
        KTyn[t] = cok[t] ? s : 0.0;
      }
      if (!R2) pin(theta_f);   // complete before the decision's own chain starts
      ++jatt;
      const double M = omega * vdx[0] + v3[0] * inv_omega;
      const double Iv = v3[1];
      // eta_bar = M / 2|I| by the division's fast path, taken as exact here; its rare slow path
      // (operands near the exponent limits) is taken in the loop's tail, which redoes the
      // decision from the saved pre-decision state -- so no branch waits on the quotient
      bool eb_ok = true;
      double eb = div_rn_fast(M, 2.0 * fabs(Iv), eb_ok);
      eb_ok = eb_ok || Iv == 0.0;
      eb = Iv == 0.0 ? INFINITY : eb;
      const double eta_used = eta;
      const double theta0 = theta, W0 = W_, ref0 = ref, ha0 = ha, hb0 = hb;
      const int rej0 = rejects;
      bool acc = false;
      double rP = 0.0;
      // the attempt's bookkeeping without branches (selects on acc); one rarely taken branch
      // leaves the common path: 100 consecutive rejections, an accepted step that is due a check,
      // or a slow-path division
      auto decide = [&](double ebv) {
        acc = CS || (eta_used <= ebv);
        if (!CS) eta = fmin(f1 * ebv, f2 * eta_used);
        rejects = acc ? 0 : rej0 + 1;
        if (!R2) {
          theta = acc ? theta_f : theta0;
          W_ = acc ? W1c : W0;
        } else {
          // r_P is read only as the restart reference (k_in = 0) and as the check metric:
          // skip its division and square root on the other attempts (they sit on the
          // warp's in-order issue path)
          rP = 0.0;
          if (acc && (k_in == 0 || k + 1 == next_check)) rP = sqrt(fmax(0.0, M / eta_used - 2.0 * Iv));
          ref = (acc && k_in == 0) ? rP : ref0;
          ha = acc ? ha_n : ha0;
          hb = acc ? hb_n : hb0;
        }
      };
      decide(eb);
      if (__builtin_expect(!(acc && k + 1 == next_check) && rejects < 100 && (CS || jatt + 1 < kStepTab) && eb_ok &&
                               (R2 || theta_ok || !acc), 1)) {
        if (LG && b == P.log_inst && lane == 0 && jatt <= P.acap) {
          double *r = P.alog + 4 * (jatt - 1);
          r[0] = (double)jatt; r[1] = acc ? 1.0 : 0.0; r[2] = eta_used; r[3] = eb;
        }
        k += acc;
        k_in += acc;
        pending = acc;
        continue;
      }
      if (!eb_ok) {   // the exact quotient; the decision again from the saved state
        eb = div_rn_slow(M, 2.0 * fabs(Iv));
        decide(eb);
      }
      if (!R2 && acc && !theta_ok) theta = div_rn_slow(eta_used, W1c);
      if (LG && b == P.log_inst && lane == 0 && jatt <= P.acap) {
        double *r = P.alog + 4 * (jatt - 1);
        r[0] = (double)jatt; r[1] = acc ? 1.0 : 0.0; r[2] = eta_used; r[3] = eb;
      }
      k += acc;
      k_in += acc;
      pending = acc;
      if (!(acc && k == next_check) && rejects < 100 && (CS || jatt + 1 < kStepTab)) continue;
      if (!CS && jatt + 1 >= kStepTab) {   // past the factor table: the next attempt's factors
        const double2 f = step_factors_far(jatt + 1);
        f1n = f.x;
        f2n = f.y;
        if (!(acc && k == next_check) && rejects < 100) continue;
      }
      if (rejects >= 100) { status = LP_NUMERICAL_ERROR; outsel = 0; break; }
      pending = false;   // the check commits this step itself
      next_check = (next_check + P.check_freq < P.iter_limit) ? next_check + P.check_freq : P.iter_limit;

      // ================= step 5: check =================
      isync<NT>();
      // infeasibility rays (reading 35): raPDHG from the point before this step (xo ...),
      // r2HPDHG from the epoch's Halpern anchor (xa ...)
      CertAcc cacc;
      double xo[CPT], KTyo[CPT], yo[RPT], Kxo[RPT];
#pragma unroll
      for (int t = 0; t < CPT; ++t) {  // commit-only, n side (K~'y' into KTyp)
        KTyp[t] = KTyn[t];
        if (!R2) {
          xo[t] = x[t]; KTyo[t] = KTy[t];
          xa[t] += theta * (xp[t] - xa[t]);
          x[t] = xp[t];
          KTy[t] = KTyp[t];
        } else {
          x[t] = ha * (rf1 * xp[t] - rf0 * x[t]) + hb * xa[t];
          KTy[t] = ha * (rf1 * KTyp[t] - rf0 * KTy[t]) + hb * KTya[t];
        }
      }
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        if (!R2) {
          yo[t] = y[t]; Kxo[t] = Kx[t];
          ya[t] += theta * (yp[t] - ya[t]);
          y[t] = yp[t];
          Kx[t] = Kxp[t];
        } else {
          y[t] = ha * (rf1 * yp[t] - rf0 * y[t]) + hb * ya[t];
          Kx[t] = ha * (rf1 * Kxp[t] - rf0 * Kx[t]) + hb * Kxa[t];
        }
      }
      double metric, dx2c, dy2c;
      int csel;  // restart candidate: 0 = current (x, y), 1 = average (ra) / w (r2)
      if (R2) {
        double v[10];
#pragma unroll
        for (int q = 0; q < 10; ++q) v[q] = 0.0;
#pragma unroll
        for (int t = 0; t < CPT; ++t) {
          const int j = lane + NT * t;
          if (cok[t]) {
            const double l0j = P.l0[j], u0j = P.u0[j];
            kkt_col_acc(v, true, dc[t], xp[t], KTyp[t], c0[j], cs[t], l0j, lsv[t], u0j, usv[t]);
            const double d = xp[t] - xr[t];
            v[4] += d * d;
            cert_col(cacc, dc[t], x[t], xa[t], KTy[t], KTya[t], c0[j], l0j, u0j);
          }
        }
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          const int i = lane + NT * t;
          if (rok[t]) {
            kkt_row_acc(v, true, i < m1, dr[t], yp[t], Kxp[t], q0[i], qs[t]);
            const double d = yp[t] - yr[t];
            v[5] += d * d;
            cert_row(cacc, i < m1, dr[t], y[t], ya[t], Kx[t], Kxa[t], q0[i]);
          }
        }
        v[6] = cacc.sy; v[7] = cacc.sx; v[8] = cacc.oy; v[9] = cacc.ox;
        ired<NT, false>(v, red, rb);
        const Kkt5 kw = kkt5(v);
        if (lane == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
          verbose_line(b, k, kw.pobj, kw.dobj, kw.pres, kw.dres, kw.gap, omega, eta);
        if (tpass(kw, nq0, nc0)) { log_check(rP, 0, 1); status = LP_OPTIMAL; outsel = 1; break; }
        {
          double mv[2] = {cacc.vy, cacc.vx};
          ired<NT, true>(mv, red, rb);
          CertAcc tot;
          tot.sy = v[6]; tot.sx = v[7]; tot.oy = v[8]; tot.ox = v[9]; tot.vy = mv[0]; tot.vx = mv[1];
          double ny, nx;
          const int st = cert_decide(tot, P.eps_pi, P.eps_di, ny, nx);
          if (st) {
            write_rays(b, ny, nx, xa, KTya, ya);
            log_check(0.0, 0, 3);
            status = st; outsel = 0; rays = true; break;
          }
        }
        if (k == P.iter_limit) { log_check(rP, 0, 0); status = LP_ITERATION_LIMIT; outsel = 1; break; }
        metric = rP; dx2c = v[4]; dy2c = v[5]; csel = 1;
      } else {
        // the average's products: K~ x-bar and K~' y-bar through the gather buffers
        isync<NT>();
#pragma unroll
        for (int t = 0; t < CPT; ++t) sx[lane + NT * t] = cok[t] ? xa[t] : 0.0;
#pragma unroll
        for (int t = 0; t < RPT; ++t) sy[lane + NT * t] = rok[t] ? ya[t] : 0.0;
        isync<NT>();
        double v[24];
#pragma unroll
        for (int q = 0; q < 24; ++q) v[q] = 0.0;
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < W; ++w) s += rval[t][w] * sx[rcol[t][w]];
          Kxa[t] = rok[t] ? s : 0.0;
          const int i = lane + NT * t;
          if (rok[t]) {
            const bool ge = i < m1;
            const double q0i = q0[i];
            kkt_row_acc(v + 0, true, ge, dr[t], ya[t], s, q0i, qs[t]);
            kkt_row_acc(v + 4, true, ge, dr[t], y[t], Kx[t], q0i, qs[t]);
            kkt_row_acc(v + 8, false, ge, dr[t], ya[t], s, q0i, qs[t]);
            kkt_row_acc(v + 12, false, ge, dr[t], y[t], Kx[t], q0i, qs[t]);
            const double da = ya[t] - yr[t], dcur = y[t] - yr[t];
            v[17] += da * da;
            v[19] += dcur * dcur;
            cert_row(cacc, ge, dr[t], y[t], yo[t], Kx[t], Kxo[t], q0i);
          }
        }
#pragma unroll
        for (int t = 0; t < CPT; ++t) {
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < WT; ++w) s += cval[t][w] * sy[ccol[t][w]];
          KTya[t] = cok[t] ? s : 0.0;
          const int j = lane + NT * t;
          if (cok[t]) {
            const double c0j = c0[j], l0j = P.l0[j], u0j = P.u0[j];
            kkt_col_acc(v + 0, true, dc[t], xa[t], s, c0j, cs[t], l0j, lsv[t], u0j, usv[t]);
            kkt_col_acc(v + 4, true, dc[t], x[t], KTy[t], c0j, cs[t], l0j, lsv[t], u0j, usv[t]);
            kkt_col_acc(v + 8, false, dc[t], xa[t], s, c0j, cs[t], l0j, lsv[t], u0j, usv[t]);
            kkt_col_acc(v + 12, false, dc[t], x[t], KTy[t], c0j, cs[t], l0j, lsv[t], u0j, usv[t]);
            const double da = xa[t] - xr[t], dcur = x[t] - xr[t];
            v[16] += da * da;
            v[18] += dcur * dcur;
            cert_col(cacc, dc[t], x[t], xo[t], KTy[t], KTyo[t], c0j, l0j, u0j);
          }
        }
        v[20] = cacc.sy; v[21] = cacc.sx; v[22] = cacc.oy; v[23] = cacc.ox;
        ired<NT, false>(v, red, rb);
        const Kkt5 ka = kkt5(v + 0), kc = kkt5(v + 4);
        if (lane == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
          verbose_line(b, k, kc.pobj, kc.dobj, kc.pres, kc.dres, kc.gap, omega, eta);
        if (tpass(ka, nq0, nc0)) { log_check(0.0, 0, 1); status = LP_OPTIMAL; outsel = 1; break; }
        if (tpass(kc, nq0, nc0)) { log_check(0.0, 0, 2); status = LP_OPTIMAL; outsel = 0; break; }
        {
          double mv[2] = {cacc.vy, cacc.vx};
          ired<NT, true>(mv, red, rb);
          CertAcc tot;
          tot.sy = v[20]; tot.sx = v[21]; tot.oy = v[22]; tot.ox = v[23]; tot.vy = mv[0]; tot.vx = mv[1];
          double ny, nx;
          const int st = cert_decide(tot, P.eps_pi, P.eps_di, ny, nx);
          if (st) {
            write_rays(b, ny, nx, xo, KTyo, yo);
            log_check(0.0, 0, 3);
            status = st; outsel = 0; rays = true; break;
          }
        }
        if (k == P.iter_limit) {
          log_check(0.0, 0, 0);
          status = LP_ITERATION_LIMIT;
          outsel = kkt5_rel(ka, nq0, nc0) < kkt5_rel(kc, nq0, nc0) ? 1 : 0;
          break;
        }
        const Kkt5 sa = kkt5(v + 8), sc = kkt5(v + 12);
        const double e_a = kkt_omega(sa, omega, inv_omega);
        const double e_c = kkt_omega(sc, omega, inv_omega);
        if (restart_to_average(e_a, e_c)) { csel = 1; metric = e_a; dx2c = v[16]; dy2c = v[17]; }
        else { csel = 0; metric = e_c; dx2c = v[18]; dy2c = v[19]; }
      }
      const bool restart = restart_due(k_in, k, metric, ref, last);
      log_check(metric, restart ? 1 : 0, 0);
      last = metric;
      if (restart) {
        ++restarts;
        omega = primal_weight(omega, sqrt(dx2c), sqrt(dy2c));
        inv_omega = 1.0 / omega;
#pragma unroll
        for (int t = 0; t < CPT; ++t) {
          if (csel) { x[t] = R2 ? xp[t] : xa[t]; KTy[t] = R2 ? KTyp[t] : KTya[t]; }
          xr[t] = x[t]; xa[t] = x[t]; KTya[t] = KTy[t];
        }
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          if (csel) { y[t] = R2 ? yp[t] : ya[t]; Kx[t] = R2 ? Kxp[t] : Kxa[t]; }
          yr[t] = y[t]; ya[t] = y[t]; Kxa[t] = Kx[t];
        }
        k_in = 0;
        if (!R2) { W_ = 0.0; ref = metric; }
      }
      isync<NT>();  // the check's gathers of sx / sy before the next phase A writes sx
    }

    // ---- step 6: output (candidate selected by outsel) ----
    {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      double *X = P.X + b * (int64_t)n, *L = P.L + b * (int64_t)n, *Y = P.Y + b * (int64_t)m;
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        const int j = lane + NT * t;
        if (cok[t]) {
          const double xs = outsel ? (R2 ? xp[t] : xa[t]) : x[t];
          const double kt = outsel ? (R2 ? KTyp[t] : KTya[t]) : KTy[t];
          kkt_col_acc(v, true, dc[t], xs, kt, c0[j], cs[t], P.l0[j], lsv[t], P.u0[j], usv[t]);
          if (!rays) {
            X[j] = dc[t] * xs;
            L[j] = c0[j] - kt / dc[t];
          }
        }
      }
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int i = lane + NT * t;
        if (rok[t]) {
          const double ys = outsel ? (R2 ? yp[t] : ya[t]) : y[t];
          const double kx = outsel ? (R2 ? Kxp[t] : Kxa[t]) : Kx[t];
          kkt_row_acc(v, true, i < m1, dr[t], ys, kx, q0[i], qs[t]);
          if (!rays) Y[i] = dr[t] * ys;
        }
      }
      ired<NT, false>(v, red, rb);
      if (lane == 0) {
        const Kkt5 ko = kkt5(v);
        lp_result r;
        r.status = status; r.polish = 0;
        r.iterations = k; r.attempts = jatt; r.restarts = restarts;
        r.primal_objective = ko.pobj; r.dual_objective = ko.dobj;
        r.primal_residual = ko.pres; r.dual_residual = ko.dres; r.gap = ko.gap;
        r.rel_kkt = kkt5_rel(ko, nq0, nc0);
        r.omega = omega; r.eta = eta; r.solve_seconds = 0.0;
        P.res[b] = r;
        if (P.res_host) P.res_host[b] = r;   // pinned host memory, device-mapped (UVA): no copy-out
      }
    }
  }
}

template <bool R2, bool CS, int NT, int RPT, int CPT, int W, int WT, bool LG = false>
int launch_tiny(TinyParams P, cudaStream_t s, unsigned long long *qbase) {
  const size_t smem = (size_t)NT * (CPT + RPT) * sizeof(double) +
                      (NT > 32 ? (size_t)2 * (NT / 32) * kRedV * sizeof(double) : 0);
  // occupancy of this instantiation: queried once per process (a small batch's solve is short
  // enough for the driver queries to show)
  static int sms = 0, per_sm = 0;
  if (per_sm == 0) {
    int dev = 0, s_ = 0, p_ = 0;
    MPAX_CUDA(cudaGetDevice(&dev));
    MPAX_CUDA(cudaDeviceGetAttribute(&s_, cudaDevAttrMultiProcessorCount, dev));
    MPAX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p_, tiny_kernel<R2, CS, NT, RPT, CPT, W, WT, LG>, NT, smem));
    sms = s_;
    per_sm = p_ < 1 ? 1 : p_;
  }
  int64_t grid = (int64_t)per_sm * sms;
  if (grid > P.batch) grid = P.batch;
  if (!qbase || *qbase == kQueueUnknown) {
    MPAX_CUDA(cudaMemsetAsync(P.queue, 0, sizeof(unsigned long long), s));
    P.qbase = 0;
  } else {
    P.qbase = *qbase;
  }
  MPAX_LAUNCH((tiny_kernel<R2, CS, NT, RPT, CPT, W, WT, LG>), (int)grid, NT, smem, s, P);
  MPAX_CHECK_LAUNCH();
  // every CTA ends on one ticket past the batch: the launch consumes batch + grid tickets
  if (qbase) *qbase = P.qbase + (unsigned long long)P.batch + (unsigned long long)grid;
  return LP_OK;
}

template <int NT, int RPT, int CPT, int W, int WT, bool LG = false>
int launch_alg(const TinyParams &P, bool r2, bool cs, cudaStream_t s, unsigned long long *qb) {
  if (cs) return r2 ? launch_tiny<true, true, NT, RPT, CPT, W, WT, LG>(P, s, qb)
                    : launch_tiny<false, true, NT, RPT, CPT, W, WT, LG>(P, s, qb);
  return r2 ? launch_tiny<true, false, NT, RPT, CPT, W, WT, LG>(P, s, qb)
            : launch_tiny<false, false, NT, RPT, CPT, W, WT, LG>(P, s, qb);
}

}  // namespace

// Returns LP_ERR_UNSUPPORTED when the LP does not fit one of the register layouts.
int tiny_solve(const DevProblem &D, const lp_options &o, const InstanceLaunch &L, cudaStream_t s,
               unsigned long long *queue, unsigned long long *qbase) {
  if (D.max_row < 0 || D.max_col < 0) return LP_ERR_UNSUPPORTED;
  TinyParams P;
  P.n = (int32_t)D.n; P.m = (int32_t)D.m; P.m1 = (int32_t)D.m1;
  P.rp = D.rp; P.ci = D.ci; P.trp = D.trp; P.tci = D.tci;
  P.kv = D.kv; P.tkv = D.tkv; P.Dr = D.Dr; P.Dc = D.Dc; P.ls = D.ls; P.us = D.us; P.l0 = D.l0; P.u0 = D.u0;
  P.C0 = L.C0; P.cstride = L.cstride; P.Q0 = L.Q0; P.qstride = L.qstride; P.X0 = L.X0; P.Y0 = L.Y0;
  P.kmax = D.kmax; P.sigma = D.sigma; P.tab = D.tab;
  P.eps_abs = o.eps_abs; P.eps_rel = o.eps_rel; P.iter_limit = o.iteration_limit; P.check_freq = o.check_frequency;
  P.eps_pi = o.eps_primal_infeasible; P.eps_di = o.eps_dual_infeasible;
  P.eps_fp = o.eps_feas_polish; P.polish_mode = L.polish_mode; P.active = L.active; P.rho = o.reflection;
  P.verbose = o.verbose; P.display_freq = o.display_frequency;
  P.batch = L.batch; P.queue = queue;
  P.X = L.X; P.Y = L.Y; P.L = L.L; P.res = L.res; P.res_host = L.res_host;
  P.alog = L.alog; P.clog = L.clog; P.acap = L.acap; P.ccap = L.ccap; P.log_inst = L.log_inst;
  const bool lg = L.alog || L.clog;
  const bool r2 = o.algorithm == LP_R2HPDHG, cs = o.step_rule == LP_STEP_CONSTANT;
  const int64_t n = D.n, m = D.m;
  const int W = D.max_row, WT = D.max_col;
  // ELL widths as tight as the LP allows: a padded slot is a zero-valued FMA on the attempt's
  // dependent chain (C2, the 5x5 grid: every column of K has exactly two entries)
  // a decision log (one instance's records): the C2 shapes only
  if (lg) {
    if (m <= 32 && n <= 64 && W <= 4 && WT <= 2) return launch_alg<32, 1, 2, 4, 2, true>(P, r2, cs, s, qbase);
    if (m <= 32 && n <= 64 && W <= 4 && WT <= 4) return launch_alg<32, 1, 2, 4, 4, true>(P, r2, cs, s, qbase);
    return LP_ERR_UNSUPPORTED;
  }
  if (m <= 32 && n <= 64 && W <= 4 && WT <= 2) return launch_alg<32, 1, 2, 4, 2>(P, r2, cs, s, qbase);
  if (m <= 32 && n <= 64 && W <= 4 && WT <= 4) return launch_alg<32, 1, 2, 4, 4>(P, r2, cs, s, qbase);
  if (m <= 32 && n <= 64 && W <= 8 && WT <= 8) return launch_alg<32, 1, 2, 8, 8>(P, r2, cs, s, qbase);
  // a CTA per instance for larger small LPs (C1: 50 x 100, rows <= 11, columns <= 12 entries)
  if (m <= 128 && n <= 128 && W <= 12 && WT <= 12) return launch_alg<128, 1, 1, 12, 12>(P, r2, cs, s, qbase);
  if (m <= 128 && n <= 128 && W <= 16 && WT <= 16) return launch_alg<128, 1, 1, 16, 16>(P, r2, cs, s, qbase);
  // Warcraft-shaped SPO+ LPs (k = 12: 144 x 1012, rows <= 16, columns <= 2 entries)
  if (m <= 256 && n <= 1024 && W <= 16 && WT <= 2) return launch_alg<256, 1, 4, 16, 2>(P, r2, cs, s, qbase);
  return LP_ERR_UNSUPPORTED;
}

}  // namespace mpax

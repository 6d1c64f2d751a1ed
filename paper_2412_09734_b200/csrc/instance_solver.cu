// instance_solver.cu -- the per-instance restarted PDHG kernel (SURVEY §8(a)
// rows a4-a11): one CTA (1-8 warps) owns one LP instance at a time and runs
// the WHOLE solve loop in-kernel -- attempts, line search, commit, periodic
// KKT check, restart, primal-weight update, termination -- then pulls the next
// instance from a device queue (batch scheduler).  No host
// synchronisation happens until every instance is done.
//
// Iteration: DESIGN.md §3 (= SURVEY §8(c) c.2), steps 2-6, organised like the
// grid kernel into two fused phases per attempt:
//   phase A (columns): [if the previous attempt was accepted] K~'_j y' (SpMV #2)
//       and the n-side commit -- raPDHG: eta-weighted average and z <- z';
//       r2HPDHG: z <- (k+1)/(k+2)(2z' - z) + 1/(k+2) z0 on x and the cached K~'y
//       (Eq. (hrpdhg)) -- then the next primal step
//       x'_j = proj(x_j - tau (c~_j - (K~'y)_j)) (Eq. (pdhg));
//   phase B (rows): [accepted] m-side commit, then K~_i x' (SpMV #1) and the dual
//       step y'_i = proj(y_i + sigma (q~_i - 2 K~_i x' + (K~x)_i));
//   then one fixed-order block reduction of ||dx||^2, ||dy||^2, <dy, K~dx> and the
//   line-search decision, taken redundantly by every thread.
// Every check_frequency accepted steps: a commit-only phase, the
// average's two SpMVs fused with the original-space KKT partials (raPDHG), the
// restart test and the primal-weight update.
//
// Layout: when they fit, K~ and K~' (CSR) are copied once per CTA into shared
// memory and the instance's 16 vectors live there too (template SMEM = true:
// the compiler sees shared-space pointers and emits LDS/STS).  Otherwise the
// matrices are read through the read-only path and the vectors live in a
// per-CTA slice of global memory.  Each SpMV row is summed by G lanes with a
// butterfly shuffle; every reduction is a fixed-order warp butterfly plus a
// fixed-order sum over warps: results are bitwise deterministic.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace mpax {

namespace {

constexpr int kRedMax = 20;  // largest reduction (raPDHG check)

struct InstParams {
  int32_t n, m, m1, nnz, gk, gkt;
  const int32_t *rp, *ci, *trp, *tci;
  const double *kv, *tkv, *Dr, *Dc, *ls, *us, *l0, *u0;
  const double *C0, *Q0, *X0, *Y0;
  int64_t cstride, qstride;
  const double *kmax, *sigma, *tab;
  double eps_abs, eps_rel, eps_pi, eps_di, eps_fp, rho;
  int64_t iter_limit;
  int32_t check_freq, alg, const_step, polish_mode, verbose, display_freq;
  int32_t hyb;  // global-state mode with the SpMV gather vectors (x, x', y, y') in shared memory
  const lp_result *active;
  int64_t batch;
  unsigned long long *queue;
  double *X, *Y, *L;
  lp_result *res;
  double *work;
  int64_t work_stride;
};

template <int NW>
__device__ __forceinline__ void bsync() {
  if (NW == 1) __syncwarp(); else __syncthreads();
}

// Fixed-order block reduction of V partial sums: warp butterfly (identical on every
// lane), then every thread sums the per-warp values in warp order.  `red` must not
// be rewritten before every thread has passed the NEXT barrier (callers alternate
// two buffers).
template <int NW, int V>
__device__ __forceinline__ void breduce(double (&v)[V], double *red) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    v[k] = s;
  }
  if (NW > 1) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) red[w * V + k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double s = red[k];
#pragma unroll
      for (int ww = 1; ww < NW; ++ww) s += red[ww * V + k];
      v[k] = s;
    }
  } else {
    __syncwarp();
  }
}

// The same for maxima of non-negative values (infeasibility violations).
template <int NW, int V>
__device__ __forceinline__ void breduce_max(double (&v)[V], double *red) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s = fmax(s, __shfl_xor_sync(FULL, s, off));
    v[k] = s;
  }
  if (NW > 1) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) red[w * V + k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double s = red[k];
#pragma unroll
      for (int ww = 1; ww < NW; ++ww) s = fmax(s, red[ww * V + k]);
      v[k] = s;
    }
  } else {
    __syncwarp();
  }
}

// Rows [0, rows) of a CSR matrix times x; G lanes per row; f(row, sum) on the group leader.
template <int NW, class F>
__device__ __forceinline__ void spmv_rows(int rows, int G, const int32_t *rp, const int32_t *ci, const double *v,
                                          const double *x, F &&f) {
  constexpr int T = NW * 32;
  if (G == 1) {
    // four rows per thread and step, their entries interleaved so that four independent
    // load chains are in flight (each row's sum keeps its sequential order: same result)
    constexpr int U = 4;
    for (int r0 = threadIdx.x; r0 < rows; r0 += U * T) {
      int a[U], e[U];
      double s[U];
      int len = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u * T;
        a[u] = r < rows ? rp[r] : 0;      // (rp / ci / v may live in shared memory: plain loads)
        e[u] = r < rows ? rp[r + 1] : 0;
        s[u] = 0.0;
        len = max(len, e[u] - a[u]);
      }
      for (int q = 0; q < len; ++q) {
        double w[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = a[u] + q < e[u];
          const int p = ok ? a[u] + q : 0;
          w[u] = ok ? v[p] : 0.0;
          xv[u] = ok ? x[ci[p]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (a[u] + q < e[u]) s[u] += w[u] * xv[u];
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r0 + u * T < rows) f(r0 + u * T, s[u]);
    }
    return;
  }
  const int per = T / G, gi = threadIdx.x / G, gl = threadIdx.x % G;
  const int iters = (rows + per - 1) / per;
  for (int it = 0; it < iters; ++it) {
    const int r = it * per + gi;
    double s = 0.0;
    if (r < rows) {
      const int e = rp[r + 1];
      for (int p = rp[r] + gl; p < e; p += G) s += v[p] * x[ci[p]];
    }
    for (int off = G >> 1; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (r < rows && gl == 0) f(r, s);
  }
}





// KKT contributions of one row / one column (contract step 5); orig: unscale with Dr, Dc.

template <int NW, bool SMEM>
__global__ void __launch_bounds__(NW * 32) instance_kernel(const InstParams P) {
  extern __shared__ __align__(16) double sm[];
  constexpr int T = NW * 32;
  const int tid = threadIdx.x;
  const int n = P.n, m = P.m, m1 = P.m1, nnz = P.nnz;
  // ---- shared-memory carve-up: reductions | [K~ values | K~' values | vectors | int arrays] ----
  double *red0 = sm, *red1 = sm + NW * kRedMax;
  double *after_red = sm + 2 * NW * kRedMax;
  const double *kv, *tkv;
  const int32_t *rp, *ci, *trp, *tci;
  double *base;
  if (SMEM) {
    double *skv = after_red, *stkv = skv + nnz;
    base = stkv + nnz;
    int32_t *srp = (int32_t *)(base + 8 * (n + m));
    int32_t *sci = srp + (m + 1), *strp = sci + nnz, *stci = strp + (n + 1);
    for (int t = tid; t < nnz; t += T) {
      skv[t] = P.kv[t]; stkv[t] = P.tkv[t]; sci[t] = P.ci[t]; stci[t] = P.tci[t];
    }
    for (int t = tid; t <= m; t += T) srp[t] = P.rp[t];
    for (int t = tid; t <= n; t += T) strp[t] = P.trp[t];
    kv = skv; tkv = stkv; rp = srp; ci = sci; trp = strp; tci = stci;
  } else {
    kv = P.kv; tkv = P.tkv; rp = P.rp; ci = P.ci; trp = P.trp; tci = P.tci;
    base = P.work + (int64_t)blockIdx.x * P.work_stride;
  }
  const double *Dr = P.Dr, *Dc = P.Dc, *ls = P.ls, *us = P.us;
  __shared__ unsigned long long s_inst;
  const bool r2 = (P.alg == LP_R2HPDHG);
  const int G = P.gk, Gt = P.gkt;
  const bool cstep = P.const_step != 0;  // constant step rule (reading 34)
  const double eta0 = initial_eta(P.kmax, P.sigma, cstep);
  // r2HPDHG reflection z <- a((1 + rho) w - rho z) + b z0 (rho = 1: 2 PDHG(z) - z; reading 38)
  const double rf1 = 1.0 + P.rho, rf0 = P.rho;
  // the check's pass test: relative KKT, or a polishing sub-solve's single residual (reading 36)
  auto tpass = [&](const Kkt5 &k, double nq, double nc) {
    return P.polish_mode ? polish_pass(P.polish_mode, k.pres, k.dres, nq, nc, P.eps_fp)
                         : kkt5_pass(k, nq, nc, P.eps_abs, P.eps_rel);
  };
  int rbuf = 0;
  auto redbuf = [&]() { rbuf ^= 1; return rbuf ? red1 : red0; };

  for (;;) {
    __syncthreads();
    if (tid == 0) s_inst = atomicAdd(P.queue, 1ull);
    __syncthreads();
    const int64_t b = (int64_t)s_inst;
    if (b >= P.batch) return;
    if (P.active && P.active[b].status != LP_OPTIMAL) continue;  // polishing: main solve not OPTIMAL

    // vectors of this instance (pointers swap for raPDHG commits)
    double *x = base, *KTy = x + n, *xp = KTy + n, *KTyp = xp + n, *xa = KTyp + n, *KTya = xa + n,
           *xr = KTya + n, *cs = xr + n;
    double *y = cs + n, *Kx = y + m, *yp = Kx + m, *Kxp = yp + m, *ya = Kxp + m, *Kxa = ya + m, *yr = Kxa + m,
           *qs = yr + m;
    if (!SMEM && P.hyb) {  // the vectors the SpMVs gather from live on chip (random reads hit smem)
      x = after_red; xp = x + n; y = xp + n; yp = y + m;
    }
    const double *c0 = P.C0 + b * P.cstride;
    const double *q0 = P.Q0 + b * P.qstride;
    const double *X0 = P.X0 ? P.X0 + b * (int64_t)n : nullptr;
    const double *Y0 = P.Y0 ? P.Y0 + b * (int64_t)m : nullptr;

    // ---- step 2: scaled data, start point, omega0, eta0 ----
    double v4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = tid; j < n; j += T) {
      const double dc = Dc[j], c = c0[j];
      const double cj = c * dc;
      cs[j] = cj;
      v4[0] += cj * cj;
      v4[2] += c * c;
      x[j] = median3(ls[j], X0 ? X0[j] / dc : 0.0, us[j]);
    }
    for (int i = tid; i < m; i += T) {
      const double dr = Dr[i], q = q0[i];
      const double qi = q * dr;
      qs[i] = qi;
      v4[1] += qi * qi;
      v4[3] += q * q;
      double yv = Y0 ? Y0[i] / dr : 0.0;
      if (i < m1) yv = fmax(yv, 0.0);
      y[i] = yv;
    }
    breduce<NW, 4>(v4, redbuf());
    const double nc0 = sqrt(v4[2]), nq0 = sqrt(v4[3]);
    double omega = 1.0;
    {
      const double nc = sqrt(v4[0]), nq = sqrt(v4[1]);
      if (nc > 1e-10 && nq > 1e-10) omega = nc / nq;
    }
    double inv_omega = 1.0 / omega;  // every x / omega is x * omega^-1 (reading 32)
    double eta = eta0;
    bsync<NW>();
    double ref = 0.0;
    {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      spmv_rows<NW>(m, G, rp, ci, kv, x, [&](int i, double s) {
        Kx[i] = s; Kxa[i] = s;
        const double yv = y[i];
        yr[i] = yv; ya[i] = yv;
        kkt_row_acc(v, false, i < m1, 1.0, yv, s, 0.0, qs[i]);
      });
      spmv_rows<NW>(n, Gt, trp, tci, tkv, y, [&](int j, double s) {
        KTy[j] = s; KTya[j] = s;
        const double xv = x[j];
        xr[j] = xv; xa[j] = xv;
        kkt_col_acc(v, false, 1.0, xv, s, 0.0, cs[j], 0.0, ls[j], 0.0, us[j]);
      });
      breduce<NW, 4>(v, redbuf());
      if (!r2) {  // raPDHG reference metric KKT_omega(z0)
        const Kkt5 ks = kkt5(v);
        ref = kkt_omega(ks, omega, inv_omega);
      }
    }
    int64_t k = 0, jatt = 0, k_in = 0, restarts = 0;
    double W = 0.0, last = INFINITY;
    int status = 0, rejects = 0;
    bool pending = false;                    // accepted attempt whose commit is fused into the next phases
    double theta = 0.0, ha = 0.0, hb = 0.0;  // raPDHG average weight / r2HPDHG Halpern coefficients
    const double *ox = x, *oy = y, *oKx = Kx, *oKTy = KTy;  // the returned candidate
    const double *bx = nullptr, *by = nullptr, *bKTy = nullptr;  // ray base (infeasible status)
    double ray_ny = 1.0, ray_nx = 1.0;
    // infeasibility test (reading 35) of z = (x, y) against the base z_b; true: status set
    auto infeasible = [&](const double *xb, const double *yb, const double *Kxb, const double *KTyb) {
      CertAcc acc;
      for (int j = tid; j < n; j += T) cert_col(acc, Dc[j], x[j], xb[j], KTy[j], KTyb[j], c0[j], P.l0[j], P.u0[j]);
      for (int i = tid; i < m; i += T) cert_row(acc, i < m1, Dr[i], y[i], yb[i], Kx[i], Kxb[i], q0[i]);
      double s4[4] = {acc.sy, acc.sx, acc.oy, acc.ox}, m2v[2] = {acc.vy, acc.vx};
      breduce<NW, 4>(s4, redbuf());
      breduce_max<NW, 2>(m2v, redbuf());
      CertAcc tot;
      tot.sy = s4[0]; tot.sx = s4[1]; tot.oy = s4[2]; tot.ox = s4[3]; tot.vy = m2v[0]; tot.vx = m2v[1];
      const int st = cert_decide(tot, P.eps_pi, P.eps_di, ray_ny, ray_nx);
      if (!st) return false;
      status = st; ox = x; oy = y; oKx = Kx; oKTy = KTy;
      bx = xb; by = yb; bKTy = KTyb;
      return true;
    };

    for (;;) {
      // ================= phase A: [commit n-side] + primal step =================
      const double tau = eta * inv_omega, sigma = eta * omega;
      double f1, f2;
      step_factors(P.tab, jatt + 1, f1, f2);  // prefetch this attempt's growth factors
      double v3[3] = {0.0, 0.0, 0.0};
      if (pending) {
        spmv_rows<NW>(n, Gt, trp, tci, tkv, yp, [&](int j, double s) {
          double xn, kt;
          if (!r2) {
            const double xv = xp[j];
            xa[j] += theta * (xv - xa[j]);
            xn = xv; kt = s;
            KTyp[j] = s;           // becomes K~'y after the pointer swap
          } else {
            xn = ha * (rf1 * xp[j] - rf0 * x[j]) + hb * xa[j];
            kt = ha * (rf1 * s - rf0 * KTy[j]) + hb * KTya[j];
            x[j] = xn; KTy[j] = kt;
          }
          const double xnew = median3(ls[j], xn - tau * (cs[j] - kt), us[j]);
          if (!r2) x[j] = xnew;    // the old-x buffer becomes x' after the swap
          else xp[j] = xnew;
          const double d = xnew - xn;
          v3[0] += d * d;
        });
        if (!r2) {
          double *t = x; x = xp; xp = t;
          t = KTy; KTy = KTyp; KTyp = t;
        }
      } else {
        for (int j = tid; j < n; j += T) {
          const double xo = x[j];
          const double xn = median3(ls[j], xo - tau * (cs[j] - KTy[j]), us[j]);
          xp[j] = xn;
          const double d = xn - xo;
          v3[0] += d * d;
        }
      }
      bsync<NW>();
      // ================= phase B: [commit m-side] + SpMV #1 + dual step =================
      const bool pend = pending;
      spmv_rows<NW>(m, G, rp, ci, kv, xp, [&](int i, double s) {
        double yv, kxv;
        if (pend) {
          if (!r2) {
            yv = yp[i];
            ya[i] += theta * (yv - ya[i]);
            kxv = Kxp[i];
          } else {
            yv = ha * (rf1 * yp[i] - rf0 * y[i]) + hb * ya[i];
            kxv = ha * (rf1 * Kxp[i] - rf0 * Kx[i]) + hb * Kxa[i];
            y[i] = yv; Kx[i] = kxv;
          }
        } else {
          yv = y[i]; kxv = Kx[i];
        }
        double yn = yv + sigma * (qs[i] - 2.0 * s + kxv);
        if (i < m1) yn = pos_part(yn);
        if (pend && !r2) { y[i] = yn; Kx[i] = s; }   // old buffers become y', K~x' after the swap
        else { yp[i] = yn; Kxp[i] = s; }
        const double d = yn - yv;
        v3[1] += d * d;
        v3[2] += d * (s - kxv);
      });
      if (pend && !r2) {
        double *t = y; y = yp; yp = t;
        t = Kx; Kx = Kxp; Kxp = t;
      }
      pending = false;
      breduce<NW, 3>(v3, redbuf());
      ++jatt;
      const double I = v3[2];
      const double M = omega * v3[0] + v3[1] * inv_omega;
      const double eb = (I != 0.0) ? M / (2.0 * fabs(I)) : INFINITY;
      const bool acc = cstep || (eta <= eb);
      const double eta_used = eta;
      if (!cstep) eta = fmin(f1 * eb, f2 * eta);
      if (!acc) {
        if (++rejects >= 100) { status = LP_NUMERICAL_ERROR; ox = x; oy = y; oKx = Kx; oKTy = KTy; break; }
        continue;
      }
      rejects = 0;
      // ---- step 4: prepare the commit ----
      double rP = 0.0;
      if (!r2) {
        const double W1 = W + eta_used;
        theta = eta_used / W1;
        W = W1;
      } else {
        rP = sqrt(fmax(0.0, M / eta_used - 2.0 * I));
        if (k_in == 0) ref = rP;
        ha = (double)(k_in + 1) / (double)(k_in + 2);
        hb = 1.0 / (double)(k_in + 2);
      }
      ++k;
      ++k_in;
      if (k % P.check_freq != 0 && k != P.iter_limit) { pending = true; continue; }

      // ================= step 5: check -- commit-only phase first =================
      const double *cx, *cy, *cKx, *cKTy;
      double metric, dx2, dy2;
      {
        double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        spmv_rows<NW>(n, Gt, trp, tci, tkv, yp, [&](int j, double s) {
          KTyp[j] = s;
          if (!r2) {
            xa[j] += theta * (xp[j] - xa[j]);
          } else {
            const double xpj = xp[j];
            x[j] = ha * (rf1 * xpj - rf0 * x[j]) + hb * xa[j];
            KTy[j] = ha * (rf1 * s - rf0 * KTy[j]) + hb * KTya[j];
            kkt_col_acc(v, true, Dc[j], xpj, s, c0[j], cs[j], P.l0[j], ls[j], P.u0[j], us[j]);
            const double d = xpj - xr[j];
            v[4] += d * d;
          }
        });
        for (int i = tid; i < m; i += T) {
          if (!r2) {
            ya[i] += theta * (yp[i] - ya[i]);
          } else {
            const double ypi = yp[i], kxp = Kxp[i];
            y[i] = ha * (rf1 * ypi - rf0 * y[i]) + hb * ya[i];
            Kx[i] = ha * (rf1 * kxp - rf0 * Kx[i]) + hb * Kxa[i];
            kkt_row_acc(v, true, i < m1, Dr[i], ypi, kxp, q0[i], qs[i]);
            const double d = ypi - yr[i];
            v[5] += d * d;
          }
        }
        if (!r2) {
          double *t = x; x = xp; xp = t;
          t = KTy; KTy = KTyp; KTyp = t;
          t = y; y = yp; yp = t;
          t = Kx; Kx = Kxp; Kxp = t;
          bsync<NW>();
        } else {
          breduce<NW, 6>(v, redbuf());
          const Kkt5 kw = kkt5(v);
          if (tid == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
            verbose_line(b, k, kw.pobj, kw.dobj, kw.pres, kw.dres, kw.gap, omega, eta);
          if (tpass(kw, nq0, nc0)) {
            status = LP_OPTIMAL; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break;
          }
          if (infeasible(xa, ya, Kxa, KTya)) break;   // rays from the epoch's Halpern anchor
          if (k == P.iter_limit) { status = LP_ITERATION_LIMIT; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break; }
          cx = xp; cy = yp; cKx = Kxp; cKTy = KTyp; metric = rP; dx2 = v[4]; dy2 = v[5];
        }
      }
      if (!r2) {
        // the average's products (2 SpMVs) fused with every KKT / distance partial
        double v[kRedMax];
#pragma unroll
        for (int t = 0; t < kRedMax; ++t) v[t] = 0.0;
        spmv_rows<NW>(m, G, rp, ci, kv, xa, [&](int i, double s) {
          Kxa[i] = s;
          const double dr = Dr[i], yai = ya[i], yi = y[i], kxi = Kx[i], q0i = q0[i], qsi = qs[i];
          kkt_row_acc(v + 0, true, i < m1, dr, yai, s, q0i, qsi);
          kkt_row_acc(v + 4, true, i < m1, dr, yi, kxi, q0i, qsi);
          kkt_row_acc(v + 8, false, i < m1, dr, yai, s, q0i, qsi);
          kkt_row_acc(v + 12, false, i < m1, dr, yi, kxi, q0i, qsi);
          const double da = yai - yr[i], dcur = yi - yr[i];
          v[17] += da * da;
          v[19] += dcur * dcur;
        });
        spmv_rows<NW>(n, Gt, trp, tci, tkv, ya, [&](int j, double s) {
          KTya[j] = s;
          const double dc = Dc[j], xaj = xa[j], xj = x[j], ktj = KTy[j];
          const double c0j = c0[j], csj = cs[j], l0j = P.l0[j], lsj = ls[j], u0j = P.u0[j], usj = us[j];
          kkt_col_acc(v + 0, true, dc, xaj, s, c0j, csj, l0j, lsj, u0j, usj);
          kkt_col_acc(v + 4, true, dc, xj, ktj, c0j, csj, l0j, lsj, u0j, usj);
          kkt_col_acc(v + 8, false, dc, xaj, s, c0j, csj, l0j, lsj, u0j, usj);
          kkt_col_acc(v + 12, false, dc, xj, ktj, c0j, csj, l0j, lsj, u0j, usj);
          const double da = xaj - xr[j], dcur = xj - xr[j];
          v[16] += da * da;
          v[18] += dcur * dcur;
        });
        breduce<NW, kRedMax>(v, redbuf());
        const Kkt5 ka = kkt5(v + 0), kc = kkt5(v + 4);
        if (tid == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
          verbose_line(b, k, kc.pobj, kc.dobj, kc.pres, kc.dres, kc.gap, omega, eta);
        if (tpass(ka, nq0, nc0)) {
          status = LP_OPTIMAL; ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; break;
        }
        if (tpass(kc, nq0, nc0)) {
          status = LP_OPTIMAL; ox = x; oy = y; oKx = Kx; oKTy = KTy; break;
        }
        if (infeasible(xp, yp, Kxp, KTyp)) break;     // rays from the last step (pre-commit point)
        if (k == P.iter_limit) {
          status = LP_ITERATION_LIMIT;
          if (kkt5_rel(ka, nq0, nc0) < kkt5_rel(kc, nq0, nc0)) { ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; }
          else { ox = x; oy = y; oKx = Kx; oKTy = KTy; }
          break;
        }
        const Kkt5 sa = kkt5(v + 8), sc = kkt5(v + 12);
        const double e_a = kkt_omega(sa, omega, inv_omega);
        const double e_c = kkt_omega(sc, omega, inv_omega);
        if (restart_to_average(e_a, e_c)) { cx = xa; cy = ya; cKx = Kxa; cKTy = KTya; metric = e_a; dx2 = v[16]; dy2 = v[17]; }
        else { cx = x; cy = y; cKx = Kx; cKTy = KTy; metric = e_c; dx2 = v[18]; dy2 = v[19]; }
      }
      // restart test (contract step 5): artificial / sufficient / necessary + stall
      const bool restart = restart_due(k_in, k, metric, ref, last);
      last = metric;
      if (restart) {
        ++restarts;
        omega = primal_weight(omega, sqrt(dx2), sqrt(dy2));
        inv_omega = 1.0 / omega;
        for (int j = tid; j < n; j += T) {
          const double xv = cx[j], kt = cKTy[j];
          x[j] = xv; xr[j] = xv; xa[j] = xv;
          KTy[j] = kt; KTya[j] = kt;
        }
        for (int i = tid; i < m; i += T) {
          const double yv = cy[i], kx = cKx[i];
          y[i] = yv; yr[i] = yv; ya[i] = yv;
          Kx[i] = kx; Kxa[i] = kx;
        }
        k_in = 0;
        if (!r2) { W = 0.0; ref = metric; }
        bsync<NW>();
      }
    }

    // ---- step 6: output the candidate in original space ----
    {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      double *X = P.X + b * (int64_t)n, *L = P.L + b * (int64_t)n, *Y = P.Y + b * (int64_t)m;
      for (int j = tid; j < n; j += T) {
        const double dc = Dc[j], xs = ox[j], kt = oKTy[j];
        kkt_col_acc(v, true, dc, xs, kt, c0[j], cs[j], P.l0[j], ls[j], P.u0[j], us[j]);
        if (bx) {  // infeasible: the unit rays d_x, d_y and -K'd_y (reading 35)
          X[j] = dc * (xs - bx[j]) / ray_nx;
          L[j] = -((kt - bKTy[j]) / dc) / ray_ny;
        } else {
          X[j] = dc * xs;
          L[j] = c0[j] - kt / dc;
        }
      }
      for (int i = tid; i < m; i += T) {
        const double dr = Dr[i];
        kkt_row_acc(v, true, i < m1, dr, oy[i], oKx[i], q0[i], qs[i]);
        Y[i] = bx ? dr * (oy[i] - by[i]) / ray_ny : dr * oy[i];
      }
      breduce<NW, 4>(v, redbuf());
      if (tid == 0) {
        const Kkt5 ko = kkt5(v);
        lp_result r;
        r.status = status;
        r.polish = 0;
        r.iterations = k;
        r.attempts = jatt;
        r.restarts = restarts;
        r.primal_objective = ko.pobj;
        r.dual_objective = ko.dobj;
        r.primal_residual = ko.pres;
        r.dual_residual = ko.dres;
        r.gap = ko.gap;
        r.rel_kkt = kkt5_rel(ko, nq0, nc0);
        r.omega = omega;
        r.eta = eta;
        r.solve_seconds = 0.0;
        P.res[b] = r;
      }
    }
  }
}

inline int pow2_floor(double v) {
  int g = 1;
  while (g * 2 <= v && g < 32) g *= 2;
  return g;
}

template <int NW, bool SMEM>
int launch_cfg(const InstParams &P0, size_t smem, size_t vec_bytes, cudaStream_t s, double **work,
               size_t *work_bytes) {
  InstParams P = P0;
  int dev = 0, sms = 0;
  MPAX_CUDA(cudaGetDevice(&dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (!SMEM) {
    // hybrid: x, x', y, y' (the gather sources of the two SpMVs) in shared memory when they fit
    const size_t hyb_bytes = smem + (size_t)2 * (size_t)(P.n + P.m) * sizeof(double);
    P.hyb = hyb_bytes <= 200 * 1024;
    if (P.hyb) smem = hyb_bytes;
  }
  MPAX_CUDA(cudaFuncSetAttribute(instance_kernel<NW, SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MPAX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, instance_kernel<NW, SMEM>, NW * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sms;
  if (grid > P.batch) grid = P.batch;
  if (grid < 1) grid = 1;
  if (!SMEM) {
    size_t need = (size_t)grid * vec_bytes;
    if (*work_bytes < need) {
      if (*work) MPAX_CUDA(cudaFreeAsync(*work, s));
      *work = nullptr;
      MPAX_CUDA(cudaMallocAsync((void **)work, need, s));
      *work_bytes = need;
    }
    P.work = *work;
    P.work_stride = (int64_t)(vec_bytes / sizeof(double));
  }
  MPAX_CUDA(cudaMemsetAsync(P.queue, 0, sizeof(unsigned long long), s));
  MPAX_LAUNCH((instance_kernel<NW, SMEM>), (int)grid, NW * 32, smem, s, P);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

template <int NW>
int launch(const InstParams &P, size_t red_bytes, size_t vec_bytes, size_t mat_bytes, cudaStream_t s,
           double **work, size_t *work_bytes) {
  int dev = 0, max_optin = 0;
  MPAX_CUDA(cudaGetDevice(&dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t all = red_bytes + vec_bytes + mat_bytes;
  if (all + 1024 <= (size_t)max_optin && all <= 160 * 1024)
    return launch_cfg<NW, true>(P, all, vec_bytes, s, work, work_bytes);
  return launch_cfg<NW, false>(P, red_bytes, vec_bytes, s, work, work_bytes);
}

}  // namespace

int instance_solve(const DevProblem &D, const lp_options &o, const InstanceLaunch &L, cudaStream_t s,
                   unsigned long long *queue, double **work, size_t *work_bytes) {
  InstParams P;
  P.n = (int32_t)D.n; P.m = (int32_t)D.m; P.m1 = (int32_t)D.m1; P.nnz = (int32_t)D.nnz;
  P.rp = D.rp; P.ci = D.ci; P.trp = D.trp; P.tci = D.tci;
  P.kv = D.kv; P.tkv = D.tkv; P.Dr = D.Dr; P.Dc = D.Dc; P.ls = D.ls; P.us = D.us; P.l0 = D.l0; P.u0 = D.u0;
  P.C0 = L.C0; P.cstride = L.cstride; P.Q0 = L.Q0; P.qstride = L.qstride; P.X0 = L.X0; P.Y0 = L.Y0;
  P.kmax = D.kmax; P.sigma = D.sigma; P.tab = D.tab; P.const_step = o.step_rule == LP_STEP_CONSTANT;
  P.eps_abs = o.eps_abs; P.eps_rel = o.eps_rel; P.iter_limit = o.iteration_limit;
  P.check_freq = o.check_frequency; P.alg = o.algorithm;
  P.eps_pi = o.eps_primal_infeasible; P.eps_di = o.eps_dual_infeasible;
  P.eps_fp = o.eps_feas_polish; P.polish_mode = L.polish_mode; P.active = L.active; P.rho = o.reflection;
  P.verbose = o.verbose; P.display_freq = o.display_frequency;
  P.batch = L.batch; P.queue = queue;
  P.X = L.X; P.Y = L.Y; P.L = L.L; P.res = L.res;
  P.work = nullptr; P.work_stride = 0; P.hyb = 0;
  // CTA size from the work per SpMV; group size from the mean row length
  const double nnz = (double)D.nnz;
  int NW = 1;
  if (nnz > 2048 || D.n + D.m > 1024) NW = 4;
  if (nnz > 32768 || D.n + D.m > 8192) NW = 8;
  {
    // latency mode: a batch that leaves SMs idle gives each instance a bigger CTA (up to one
    // thread per ~4 rows / columns), since its solve time is one CTA's per-attempt latency
    int dev = 0, sms = 0;
    MPAX_CUDA(cudaGetDevice(&dev));
    MPAX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (L.batch <= 2 * (int64_t)sms) {
      const int64_t want = (std::max(D.n, D.m) + 4 * 32 - 1) / (4 * 32);
      while (NW < 32 && NW < want) NW *= 2;
    }
    if (const char *e = getenv("MPAX_INST_NW")) {   // experiments; anything but a CTA size is ignored
      const int v = atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) NW = v;
    }
    if (NW == 2) NW = 4;              // the instantiated CTA sizes: 1, 4, 8, 16, 32 warps
    if (NW > 16 && NW != 32) NW = 32;
  }
  P.gk = pow2_floor(D.avg_row / 4.0);
  P.gkt = pow2_floor(D.avg_col / 4.0);
  const size_t vec_bytes = (size_t)8 * (size_t)(D.n + D.m) * sizeof(double);
  const size_t mat_bytes = (size_t)D.nnz * (2 * sizeof(double) + 2 * sizeof(int32_t)) +
                           (size_t)(D.n + D.m + 2) * sizeof(int32_t);
  const size_t red_bytes = (size_t)2 * NW * kRedMax * sizeof(double);
  switch (NW) {
    case 1: return launch<1>(P, red_bytes, vec_bytes, mat_bytes, s, work, work_bytes);
    case 2:
    case 4: return launch<4>(P, red_bytes, vec_bytes, mat_bytes, s, work, work_bytes);
    case 8: return launch<8>(P, red_bytes, vec_bytes, mat_bytes, s, work, work_bytes);
    case 16: return launch<16>(P, red_bytes, vec_bytes, mat_bytes, s, work, work_bytes);
    default: return launch<32>(P, red_bytes, vec_bytes, mat_bytes, s, work, work_bytes);
  }
}

}  // namespace mpax

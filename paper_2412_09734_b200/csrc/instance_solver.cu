// instance_solver.cu -- the per-instance restarted PDHG kernel (SURVEY §8(a)
// rows a4-a11): one CTA (1-8 warps) owns one LP instance at a time and runs
// the WHOLE solve loop in-kernel -- attempts, line search, commit, periodic
// KKT check, restart, primal-weight update, termination -- then pulls the next
// instance from a device queue (batch scheduler).  No host
// synchronisation happens until every instance is done.
//
// Iteration: DESIGN.md §3 (= SURVEY §8(c) c.2), steps 2-6:
//   step 3: x' = proj_X(x - tau (c~ - K~'y)); K~x'; y' = proj_Y(y + sigma (q~ - 2K~x' + K~x))
//           (PAPER.md Eq. (pdhg)), eta_bar = M / (2|<dy, K~x' - K~x>|), accept iff
//           eta <= eta_bar, eta <- min((1-(j+1)^-.3) eta_bar, (1+(j+1)^-.6) eta)
//   step 4: K~'y'; raPDHG: z <- z', eta-weighted average;
//           r2HPDHG: z <- (k+1)/(k+2) (2z' - z) + 1/(k+2) z0 on x, y AND the cached
//           products (Eq. (hrpdhg))
//   step 5: every check_frequency accepted steps: original-space KKT
//           termination test, restart test on KKT_omega (ra) / fixed-point residual
//           (r2), restart + primal weight sqrt(omega dy/dx).
//
// Layout: the instance's 16 vectors (8 n-long, 8 m-long) live in shared memory
// when they fit (small LPs such as the paper's batched grid LPs), otherwise in
// a per-CTA slice of global memory (L1/L2 resident).  K~ and K~' are shared by
// every instance and read through the read-only path.  Each SpMV row is summed
// by a group of G lanes (G = 1..32 chosen from the mean row length) with a
// butterfly shuffle, and every reduction is a fixed-order warp butterfly plus a
// fixed-order sum over warps: results are bitwise deterministic.
#include "common.cuh"

namespace mpax {

namespace {

constexpr int kRedMax = 20;  // largest reduction (raPDHG check)

struct InstParams {
  int32_t n, m, m1, gk, gkt;
  const int32_t *rp, *ci, *trp, *tci;
  const double *kv, *tkv, *Dr, *Dc, *ls, *us, *l0, *u0;
  const double *C0, *Q0, *X0, *Y0;
  int64_t cstride, qstride;
  const double *kmax, *tab;
  double eps_abs, eps_rel;
  int64_t iter_limit;
  int32_t check_freq, alg;
  int64_t batch;
  unsigned long long *queue;
  double *X, *Y, *L;
  lp_result *res;
  double *work;
  int64_t work_stride;
  int32_t vec_in_smem;
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
      for (int ww = 1; ww < NW; ++ww) s += red[ww * V + k];
      v[k] = s;
    }
  } else {
    __syncwarp();
  }
}

// Rows [0, rows) of a CSR matrix times x; G lanes per row; f(row, sum) on the group leader.
template <int NW, class F>
__device__ __forceinline__ void spmv_rows(int rows, int G, const int32_t *__restrict__ rp,
                                          const int32_t *__restrict__ ci, const double *__restrict__ v,
                                          const double *x, F &&f) {
  constexpr int T = NW * 32;
  const int per = T / G, gi = threadIdx.x / G, gl = threadIdx.x % G;
  const int iters = (rows + per - 1) / per;
  for (int it = 0; it < iters; ++it) {
    const int r = it * per + gi;
    double s = 0.0;
    if (r < rows) {
      const int e = __ldg(rp + r + 1);
      for (int p = __ldg(rp + r) + gl; p < e; p += G) s += __ldg(v + p) * x[__ldg(ci + p)];
    }
    for (int off = G >> 1; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (r < rows && gl == 0) f(r, s);
  }
}

struct Kkt {
  double pres, dres, pobj, dobj, gap;
};

__device__ __forceinline__ Kkt make_kkt(const double *v) {
  Kkt k;
  k.pres = sqrt(v[0]);
  k.dres = sqrt(v[1]);
  k.pobj = v[2];
  k.dobj = v[3];
  k.gap = fabs(v[2] - v[3]);
  return k;
}

__device__ __forceinline__ bool kkt_pass(const Kkt &k, double nq, double nc, double ea, double er) {
  return k.pres <= ea + er * nq && k.dres <= ea + er * nc && k.gap <= ea + er * (fabs(k.pobj) + fabs(k.dobj));
}

__device__ __forceinline__ double rel_kkt(const Kkt &k, double nq, double nc) {
  return fmax(k.pres / (1.0 + nq), fmax(k.dres / (1.0 + nc), k.gap / (1.0 + fabs(k.pobj) + fabs(k.dobj))));
}

// Partial sums (pres^2, dres^2, pobj, dobj) of a candidate, contract step 5.  orig:
// unscale x = Dc x~, y = Dr y~, Kx = Kx~ / Dr, K'y = K'y~ / Dc and use the original data.
template <int NW>
__device__ __forceinline__ void kkt_partial(bool orig, const InstParams &P, const double *c0, const double *q0,
                                            const double *cs, const double *qs, const double *xs,
                                            const double *ys, const double *Kxs, const double *KTys,
                                            double *v) {
  constexpr int T = NW * 32;
  for (int i = threadIdx.x; i < P.m; i += T) {
    const double dr = P.Dr[i];
    const double Kx = orig ? Kxs[i] / dr : Kxs[i];
    const double q = orig ? q0[i] : qs[i];
    const double y = orig ? dr * ys[i] : ys[i];
    double r = q - Kx;
    if (i < P.m1) r = fmax(r, 0.0);
    v[0] += r * r;
    v[3] += q * y;
  }
  for (int j = threadIdx.x; j < P.n; j += T) {
    const double dc = P.Dc[j];
    const double x = orig ? dc * xs[j] : xs[j];
    const double KTy = orig ? KTys[j] / dc : KTys[j];
    const double c = orig ? c0[j] : cs[j];
    const double l = orig ? P.l0[j] : P.ls[j];
    const double u = orig ? P.u0[j] : P.us[j];
    const double lam = c - KTy;
    const double lp = fmax(lam, 0.0), lm = fmax(-lam, 0.0);
    double d = 0.0;
    if (l == -INFINITY) d += lp;
    if (u == INFINITY) d += lm;
    v[1] += d * d;
    v[2] += c * x;
    if (l > -INFINITY) v[3] += l * lp;
    if (u < INFINITY) v[3] -= u * lm;
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) instance_kernel(const InstParams P) {
  extern __shared__ __align__(16) double sm[];
  constexpr int T = NW * 32;
  const int tid = threadIdx.x;
  const int n = P.n, m = P.m, m1 = P.m1;
  double *red0 = sm, *red1 = sm + NW * kRedMax;
  double *base = P.vec_in_smem ? sm + 2 * NW * kRedMax : P.work + (int64_t)blockIdx.x * P.work_stride;
  __shared__ unsigned long long s_inst;
  const bool r2 = (P.alg == LP_R2HPDHG);
  const double kmx = *P.kmax;
  const double eta0 = kmx > 0.0 ? 1.0 / kmx : 1.0;
  int rbuf = 0;
  auto redbuf = [&]() { rbuf ^= 1; return rbuf ? red1 : red0; };

  for (;;) {
    __syncthreads();
    if (tid == 0) s_inst = atomicAdd(P.queue, 1ull);
    __syncthreads();
    const int64_t b = (int64_t)s_inst;
    if (b >= P.batch) return;

    // vectors of this instance (pointers swap for raPDHG commits)
    double *x = base, *KTy = x + n, *xp = KTy + n, *KTyp = xp + n, *xa = KTyp + n, *KTya = xa + n,
           *xr = KTya + n, *cs = xr + n;
    double *y = cs + n, *Kx = y + m, *yp = Kx + m, *Kxp = yp + m, *ya = Kxp + m, *Kxa = ya + m, *yr = Kxa + m,
           *qs = yr + m;
    const double *c0 = P.C0 + b * P.cstride;
    const double *q0 = P.Q0 + b * P.qstride;
    const double *X0 = P.X0 ? P.X0 + b * (int64_t)n : nullptr;
    const double *Y0 = P.Y0 ? P.Y0 + b * (int64_t)m : nullptr;

    // ---- step 2: scaled data, start point, omega0, eta0 ----
    double v4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = tid; j < n; j += T) {
      const double dc = P.Dc[j], c = c0[j];
      const double cj = c * dc;
      cs[j] = cj;
      v4[0] += cj * cj;
      v4[2] += c * c;
      x[j] = median3(P.ls[j], X0 ? X0[j] / dc : 0.0, P.us[j]);
    }
    for (int i = tid; i < m; i += T) {
      const double dr = P.Dr[i], q = q0[i];
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
    double eta = eta0;
    bsync<NW>();
    spmv_rows<NW>(m, P.gk, P.rp, P.ci, P.kv, x, [&](int i, double s) { Kx[i] = s; });
    spmv_rows<NW>(n, P.gkt, P.trp, P.tci, P.tkv, y, [&](int j, double s) { KTy[j] = s; });
    bsync<NW>();
    for (int j = tid; j < n; j += T) { xr[j] = x[j]; xa[j] = x[j]; KTya[j] = KTy[j]; }
    for (int i = tid; i < m; i += T) { yr[i] = y[i]; ya[i] = y[i]; Kxa[i] = Kx[i]; }
    int64_t k = 0, jatt = 0, k_in = 0, restarts = 0;
    double W = 0.0, last = INFINITY, ref = 0.0;
    if (!r2) {  // raPDHG reference metric KKT_omega(z0)
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      kkt_partial<NW>(false, P, c0, q0, cs, qs, x, y, Kx, KTy, v);
      breduce<NW, 4>(v, redbuf());
      const Kkt ks = make_kkt(v);
      ref = sqrt(omega * ks.pres * ks.pres + ks.dres * ks.dres / omega + ks.gap * ks.gap);
    }
    bsync<NW>();

    int status = 0;
    // the returned candidate
    const double *ox = x, *oy = y, *oKx = Kx, *oKTy = KTy;

    for (;;) {
      // ---- step 3: attempts until one is accepted ----
      double eta_used = eta, M = 0.0, I = 0.0;
      int rejects = 0;
      for (;;) {
        ++jatt;
        const double tau = eta / omega, sigma = eta * omega;
        double v3[3] = {0.0, 0.0, 0.0};
        for (int j = tid; j < n; j += T) {
          const double xo = x[j];
          const double xn = median3(P.ls[j], xo - tau * (cs[j] - KTy[j]), P.us[j]);
          xp[j] = xn;
          const double d = xn - xo;
          v3[0] += d * d;
        }
        bsync<NW>();
        spmv_rows<NW>(m, P.gk, P.rp, P.ci, P.kv, xp, [&](int i, double s) {
          const double yo = y[i], kxo = Kx[i];
          double yn = yo + sigma * (qs[i] - 2.0 * s + kxo);
          if (i < m1) yn = fmax(yn, 0.0);
          Kxp[i] = s;
          yp[i] = yn;
          const double d = yn - yo;
          v3[1] += d * d;
          v3[2] += d * (s - kxo);
        });
        breduce<NW, 3>(v3, redbuf());
        I = v3[2];
        M = omega * v3[0] + v3[1] / omega;
        const double eb = (I != 0.0) ? M / (2.0 * fabs(I)) : INFINITY;
        const bool acc = (eta <= eb);
        eta_used = eta;
        double f1, f2;
        step_factors(P.tab, jatt, f1, f2);
        eta = fmin(f1 * eb, f2 * eta);
        if (acc) break;
        if (++rejects >= 100) { status = LP_NUMERICAL_ERROR; break; }
      }
      if (status) { ox = x; oy = y; oKx = Kx; oKTy = KTy; break; }

      // ---- step 4: commit (SpMV #2 = K~'y' fused with the update) ----
      double rP = 0.0;
      if (!r2) {
        const double W1 = W + eta_used, theta = eta_used / W1;
        W = W1;
        spmv_rows<NW>(n, P.gkt, P.trp, P.tci, P.tkv, yp, [&](int j, double s) {
          KTyp[j] = s;
          xa[j] += theta * (xp[j] - xa[j]);
        });
        for (int i = tid; i < m; i += T) ya[i] += theta * (yp[i] - ya[i]);
        double *t;
        t = x; x = xp; xp = t;
        t = KTy; KTy = KTyp; KTyp = t;
        t = y; y = yp; yp = t;
        t = Kx; Kx = Kxp; Kxp = t;
      } else {
        rP = sqrt(fmax(0.0, M / eta_used - 2.0 * I));
        if (k_in == 0) ref = rP;
        const double a = (double)(k_in + 1) / (double)(k_in + 2), bb = 1.0 / (double)(k_in + 2);
        spmv_rows<NW>(n, P.gkt, P.trp, P.tci, P.tkv, yp, [&](int j, double s) {
          KTyp[j] = s;
          x[j] = a * (2.0 * xp[j] - x[j]) + bb * xa[j];
          KTy[j] = a * (2.0 * s - KTy[j]) + bb * KTya[j];
        });
        for (int i = tid; i < m; i += T) {
          y[i] = a * (2.0 * yp[i] - y[i]) + bb * ya[i];
          Kx[i] = a * (2.0 * Kxp[i] - Kx[i]) + bb * Kxa[i];
        }
      }
      ++k;
      ++k_in;
      bsync<NW>();

      // ---- step 5: periodic check ----
      if (k % P.check_freq != 0 && k != P.iter_limit) continue;
      const double *cx, *cy, *cKx, *cKTy;
      double metric;
      double dist_x2, dist_y2;
      if (!r2) {
        spmv_rows<NW>(m, P.gk, P.rp, P.ci, P.kv, xa, [&](int i, double s) { Kxa[i] = s; });
        spmv_rows<NW>(n, P.gkt, P.trp, P.tci, P.tkv, ya, [&](int j, double s) { KTya[j] = s; });
        bsync<NW>();
        double v[kRedMax];
#pragma unroll
        for (int t = 0; t < kRedMax; ++t) v[t] = 0.0;
        kkt_partial<NW>(true, P, c0, q0, cs, qs, xa, ya, Kxa, KTya, v + 0);
        kkt_partial<NW>(true, P, c0, q0, cs, qs, x, y, Kx, KTy, v + 4);
        kkt_partial<NW>(false, P, c0, q0, cs, qs, xa, ya, Kxa, KTya, v + 8);
        kkt_partial<NW>(false, P, c0, q0, cs, qs, x, y, Kx, KTy, v + 12);
        for (int j = tid; j < n; j += T) {
          const double da = xa[j] - xr[j], dc = x[j] - xr[j];
          v[16] += da * da;
          v[18] += dc * dc;
        }
        for (int i = tid; i < m; i += T) {
          const double da = ya[i] - yr[i], dc = y[i] - yr[i];
          v[17] += da * da;
          v[19] += dc * dc;
        }
        breduce<NW, kRedMax>(v, redbuf());
        const Kkt ka = make_kkt(v + 0), kc = make_kkt(v + 4);
        if (kkt_pass(ka, nq0, nc0, P.eps_abs, P.eps_rel)) {
          status = LP_OPTIMAL; ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; break;
        }
        if (kkt_pass(kc, nq0, nc0, P.eps_abs, P.eps_rel)) {
          status = LP_OPTIMAL; ox = x; oy = y; oKx = Kx; oKTy = KTy; break;
        }
        if (k == P.iter_limit) {
          status = LP_ITERATION_LIMIT;
          if (rel_kkt(ka, nq0, nc0) < rel_kkt(kc, nq0, nc0)) { ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; }
          else { ox = x; oy = y; oKx = Kx; oKTy = KTy; }
          break;
        }
        const Kkt sa = make_kkt(v + 8), sc = make_kkt(v + 12);
        const double e_a = sqrt(omega * sa.pres * sa.pres + sa.dres * sa.dres / omega + sa.gap * sa.gap);
        const double e_c = sqrt(omega * sc.pres * sc.pres + sc.dres * sc.dres / omega + sc.gap * sc.gap);
        if (e_a < e_c) { cx = xa; cy = ya; cKx = Kxa; cKTy = KTya; metric = e_a; dist_x2 = v[16]; dist_y2 = v[17]; }
        else { cx = x; cy = y; cKx = Kx; cKTy = KTy; metric = e_c; dist_x2 = v[18]; dist_y2 = v[19]; }
      } else {
        double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        kkt_partial<NW>(true, P, c0, q0, cs, qs, xp, yp, Kxp, KTyp, v);
        for (int j = tid; j < n; j += T) { const double d = xp[j] - xr[j]; v[4] += d * d; }
        for (int i = tid; i < m; i += T) { const double d = yp[i] - yr[i]; v[5] += d * d; }
        breduce<NW, 6>(v, redbuf());
        const Kkt kw = make_kkt(v);
        if (kkt_pass(kw, nq0, nc0, P.eps_abs, P.eps_rel)) {
          status = LP_OPTIMAL; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break;
        }
        if (k == P.iter_limit) {
          status = LP_ITERATION_LIMIT; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break;
        }
        cx = xp; cy = yp; cKx = Kxp; cKTy = KTyp; metric = rP; dist_x2 = v[4]; dist_y2 = v[5];
      }
      // restart test (contract step 5): artificial / sufficient / necessary + stall
      const bool restart = ((double)k_in >= 0.36 * (double)k) || (metric <= 0.2 * ref) ||
                           (metric <= 0.8 * ref && metric > last);
      last = metric;
      if (restart) {
        ++restarts;
        const double dxn = sqrt(dist_x2), dyn = sqrt(dist_y2);
        if (dxn > 1e-10 && dyn > 1e-10) omega = sqrt(omega * (dyn / dxn));
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
      kkt_partial<NW>(true, P, c0, q0, cs, qs, ox, oy, oKx, oKTy, v);
      breduce<NW, 4>(v, redbuf());
      const Kkt ko = make_kkt(v);
      double *X = P.X + b * (int64_t)n, *L = P.L + b * (int64_t)n, *Y = P.Y + b * (int64_t)m;
      for (int j = tid; j < n; j += T) {
        const double dc = P.Dc[j];
        X[j] = dc * ox[j];
        L[j] = c0[j] - oKTy[j] / dc;
      }
      for (int i = tid; i < m; i += T) Y[i] = P.Dr[i] * oy[i];
      if (tid == 0) {
        lp_result r;
        r.status = status;
        r.pad = 0;
        r.iterations = k;
        r.attempts = jatt;
        r.restarts = restarts;
        r.primal_objective = ko.pobj;
        r.dual_objective = ko.dobj;
        r.primal_residual = ko.pres;
        r.dual_residual = ko.dres;
        r.gap = ko.gap;
        r.rel_kkt = rel_kkt(ko, nq0, nc0);
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

template <int NW>
int launch(const InstParams &P0, size_t smem_red, size_t vec_bytes, cudaStream_t s, double **work,
           size_t *work_bytes) {
  InstParams P = P0;
  int dev = 0, sms = 0, max_optin = 0;
  MPAX_CUDA(cudaGetDevice(&dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  size_t smem = smem_red;
  P.vec_in_smem = (smem_red + vec_bytes + 1024 <= (size_t)max_optin && vec_bytes <= 96 * 1024) ? 1 : 0;
  if (P.vec_in_smem) smem += vec_bytes;
  MPAX_CUDA(cudaFuncSetAttribute(instance_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MPAX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, instance_kernel<NW>, NW * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sms;
  if (grid > P.batch) grid = P.batch;
  if (grid < 1) grid = 1;
  if (!P.vec_in_smem) {
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
  MPAX_LAUNCH(instance_kernel<NW>, (int)grid, NW * 32, smem, s, P);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

}  // namespace

int instance_solve(const DevProblem &D, const lp_options &o, const InstanceLaunch &L, cudaStream_t s,
                   unsigned long long *queue, double **work, size_t *work_bytes) {
  InstParams P;
  P.n = (int32_t)D.n; P.m = (int32_t)D.m; P.m1 = (int32_t)D.m1;
  P.rp = D.rp; P.ci = D.ci; P.trp = D.trp; P.tci = D.tci;
  P.kv = D.kv; P.tkv = D.tkv; P.Dr = D.Dr; P.Dc = D.Dc; P.ls = D.ls; P.us = D.us; P.l0 = D.l0; P.u0 = D.u0;
  P.C0 = L.C0; P.cstride = L.cstride; P.Q0 = L.Q0; P.qstride = L.qstride; P.X0 = L.X0; P.Y0 = L.Y0;
  P.kmax = D.kmax; P.tab = D.tab;
  P.eps_abs = o.eps_abs; P.eps_rel = o.eps_rel; P.iter_limit = o.iteration_limit;
  P.check_freq = o.check_frequency; P.alg = o.algorithm;
  P.batch = L.batch; P.queue = queue;
  P.X = L.X; P.Y = L.Y; P.L = L.L; P.res = L.res;
  P.work = nullptr; P.work_stride = 0; P.vec_in_smem = 0;
  // CTA size from the work per SpMV; group size from the mean row length
  const double nnz = (double)D.nnz;
  int NW = 1;
  if (nnz > 2048 || D.n + D.m > 1024) NW = 4;
  if (nnz > 32768 || D.n + D.m > 8192) NW = 8;
  P.gk = pow2_floor(D.avg_row / 4.0);
  P.gkt = pow2_floor(D.avg_col / 4.0);
  const size_t vec_bytes = (size_t)8 * (size_t)(D.n + D.m) * sizeof(double);
  const size_t red_bytes = (size_t)2 * NW * kRedMax * sizeof(double);
  switch (NW) {
    case 1: return launch<1>(P, red_bytes, vec_bytes, s, work, work_bytes);
    case 4: return launch<4>(P, red_bytes, vec_bytes, s, work, work_bytes);
    default: return launch<8>(P, red_bytes, vec_bytes, s, work, work_bytes);
  }
}

}  // namespace mpax

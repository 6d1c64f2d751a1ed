// dmma_solver.cu -- batches that share one DENSE K:
// the two products of every PDHG attempt become fp64 tensor-core contractions
// ("a vector-vector multiplication can be transformed into a matrix-vector
// multiplication"; here 8 instances form the N = 8 side of DMMA.8x8x4).
//
// Design (B200): a thread-block cluster of CL CTAs serves a group of 8 instances.
// CTA c keeps the column slice K~[:, slice_c] resident in shared memory for the
// whole solve (C3: 200 x 100 fp64 = 160 KB), so K~ is read from HBM/L2 once, not
// once per instance per attempt as in the per-instance path.  Per attempt:
//   GEMM1   K~'y'  = K~_c' Y'      (n_c x 8, K = m)  -> n-side commit + primal step
//   GEMM2   P_c    = K~_c X'_c     (m x 8, K = n_c)  partial of K~x'
//   cluster barrier; CTA c sums the CL partials of its own row slice in rank order
//   through distributed shared memory (DSMEM) -> m-side commit + dual step;
//   per-instance ||dx||^2, ||dy||^2, <dy, K~dx> partials; cluster barrier; every CTA
//   sums the partials in rank order and takes each instance's line-search decision;
//   the Y' rows of the peers are copied into the local full Y' for the next GEMM1.
// Instances keep their own step sizes, accept/reject, commits, checks,
// restarts and termination; a finished instance is frozen until all 8 are done,
// then the cluster pulls the next group from a device queue.
//
// Arithmetic: the same contract as the other solvers; only the
// summation order of the products differs (tensor-core k-order), so results agree
// with the oracle to rounding.  mma.sync f64 lowers to DMMA on sm_100a (there is
// no f64 kind of tcgen05.mma).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

#ifdef MPAX_DEBUG
#include <cstdio>
#define DCHK(c)                                                                         \
  do {                                                                                  \
    if (!(c)) {                                                                         \
      printf("DCHK failed %s:%d block %d thread %d\n", __FILE__, __LINE__, blockIdx.x, threadIdx.x); \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define DCHK(c) \
  do {          \
  } while (0)
#endif

namespace mpax {

namespace {

constexpr int kThreads = 256;  // 8 warps per CTA
constexpr int kS = 8;          // instances per group (= DMMA N)

struct DmmaParams {
  int32_t n, m, m1, nc, np, mp, mc;  // n, m, m1; column slice width, padded slice width, padded m, row slice
  const double *K;                   // scaled dense K~, row-major m x n
  const double *Dr, *Dc, *ls, *us, *l0, *u0;
  const double *C0, *Q0, *X0, *Y0;
  int64_t cstride, qstride;
  const double *kmax, *sigma, *tab;
  double eps_abs, eps_rel, eps_pi, eps_di, eps_fp, rho;
  int64_t iter_limit;
  int32_t check_freq, alg, const_step, polish_mode, verbose, display_freq;
  const lp_result *active;
  int64_t batch;
  unsigned long long *queue;
  // per-instance state, instance-major [B][n] / [B][m]
  double *x, *KTy, *xa, *KTya, *xr, *cs, *xp, *KTyp;
  double *y, *Kx, *ya, *Kxa, *yr, *qs, *yp, *Kxp;
  double *X, *Y, *L;
  lp_result *res;
};

// per-instance scalar state (identical copy in every CTA of the cluster)
struct Inst {
  double omega, inv_omega, eta, W, ref, last, theta, ha, hb, rP, nc0, nq0, metric, dx2c, dy2c, eta_used, M, I;
  double ray_ny, ray_nx;  // infeasibility rays' norms (reading 35)
  long long k, j, k_in, restarts;
  int rejects, status, pending, done, check, outsel, csel, valid, cert, rays, skip;
};

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}


// Shared-memory layout of one CTA.
struct Smem {
  double *Ks;    // mp x np  : K~[:, slice] (zero padded)
  double *Yf;    // mp x 8   : full Y' (or y-bar at raPDHG checks), instance fastest
  double *Xc;    // np x 8   : X'_c (or x-bar slice)
  double *Pc;    // mp x 8   : partial K~_c X'_c
  double *part;  // 8 x 24   : per-instance partial sums of this CTA (current of two buffers)
  double *part_a, *part_b;
  double *wpart; // 8 warps x 8 x 24
  Inst *inst;    // 8
  int *grp;
};

// GEMM1: D(j, s) = sum_i Ks[i][j] * Yf[i][s] for the CTA's np columns; calls f(j, s, value).
template <class F>
__device__ __forceinline__ void gemm1(const Smem &S, int np, int mp, F &&f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  for (int jt = w; jt * 8 < np; jt += kThreads / 32) {
    double d0 = 0.0, d1 = 0.0;
    const int j = jt * 8 + r;
    DCHK(j < np);
    int kt = 0;
    // four k-steps' operands in flight before their DMMAs (the accumulation order is unchanged)
    for (; kt + 16 <= mp; kt += 16) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = S.Ks[(kt + 4 * u + q) * np + j];     // A(j, i=kt+4u+q)
        b[u] = S.Yf[(kt + 4 * u + q) * kS + r];     // B(i=kt+4u+q, s=r)
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(d0, d1, a[u], b[u]);
    }
    for (; kt < mp; kt += 4) {
      DCHK(kt + q < mp);
      const double a = S.Ks[(kt + q) * np + j];        // A(j, i=kt+q)
      const double b = S.Yf[(kt + q) * kS + r];        // B(i=kt+q, s=r)
      dmma(d0, d1, a, b);
    }
    f(j, 2 * q, d0);
    f(j, 2 * q + 1, d1);
  }
}

// GEMM1 whose epilogue operands are loaded before the k-loop (in flight during the DMMA chain):
// pre(j, s) returns them, f(j, s, value, ops) consumes them.
template <class Pre, class F>
__device__ __forceinline__ void gemm1_pre(const Smem &S, int np, int mp, Pre &&pre, F &&f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  for (int jt = w; jt * 8 < np; jt += kThreads / 32) {
    double d0 = 0.0, d1 = 0.0;
    const int j = jt * 8 + r;
    auto o0 = pre(j, 2 * q);
    auto o1 = pre(j, 2 * q + 1);
    int kt = 0;
    for (; kt + 16 <= mp; kt += 16) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = S.Ks[(kt + 4 * u + q) * np + j];
        b[u] = S.Yf[(kt + 4 * u + q) * kS + r];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(d0, d1, a[u], b[u]);
    }
    for (; kt < mp; kt += 4) {
      const double a = S.Ks[(kt + q) * np + j];
      const double b = S.Yf[(kt + q) * kS + r];
      dmma(d0, d1, a, b);
    }
    f(j, 2 * q, d0, o0);
    f(j, 2 * q + 1, d1, o1);
  }
}

// GEMM2: Pc(i, s) = sum_j Ks[i][j] * Xc[j][s].
__device__ __forceinline__ void gemm2(const Smem &S, int np, int mp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  for (int it = w; it * 8 < mp; it += kThreads / 32) {
    double d0 = 0.0, d1 = 0.0;
    const int i = it * 8 + r;
    DCHK(i < mp);
    int kt = 0;
    for (; kt + 16 <= np; kt += 16) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = S.Ks[i * np + kt + 4 * u + q];       // A(i, j=kt+4u+q)
        b[u] = S.Xc[(kt + 4 * u + q) * kS + r];     // B(j=kt+4u+q, s=r)
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(d0, d1, a[u], b[u]);
    }
    for (; kt < np; kt += 4) {
      DCHK(kt + q < np);
      const double a = S.Ks[i * np + kt + q];          // A(i, j=kt+q)
      const double b = S.Xc[(kt + q) * kS + r];        // B(j=kt+q, s=r)
      dmma(d0, d1, a, b);
    }
    S.Pc[i * kS + 2 * q] = d0;
    S.Pc[i * kS + 2 * q + 1] = d1;
  }
}

// Per-instance partial sums: v[s][0..V) accumulated per thread -> S.part[s][0..V) (fixed order).
// MX: bit k set = value k is max-reduced (non-negative), else summed.
template <int V, unsigned MX = 0u>
__device__ __forceinline__ void cta_partials(double (&v)[kS][V], const Smem &S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < kS; ++s)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double t = v[s][k];
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const double o = __shfl_xor_sync(FULL, t, off);
        t = ((MX >> k) & 1u) ? fmax(t, o) : t + o;
      }
      if (lane == 0) S.wpart[(w * kS + s) * 24 + k] = t;
    }
  __syncthreads();
  for (int t = threadIdx.x; t < kS * V; t += kThreads) {
    const int s = t / V, k = t % V;
    const bool mx = (MX >> k) & 1u;
    double a = 0.0;
    for (int ww = 0; ww < kThreads / 32; ++ww) {
      const double o = S.wpart[(ww * kS + s) * 24 + k];
      a = mx ? fmax(a, o) : a + o;
    }
    S.part[s * 24 + k] = a;
  }
}

// The attempt's three per-instance sums with the fragment layouts in mind: lane l holds
// ||dx||^2 for instances 2(l%4), 2(l%4)+1 (GEMM1 C fragment) and ||dy||^2, <dy, K~dx> for
// instance l%8 (row loop), so 3- and 2-level butterflies suffice; warps are then summed in
// order.  Fixed order: deterministic.
__device__ __forceinline__ void attempt_partials(double dxe, double dxo, double dy, double Iv, const Smem &S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    dxe += __shfl_xor_sync(FULL, dxe, off);
    dxo += __shfl_xor_sync(FULL, dxo, off);
  }
#pragma unroll
  for (int off = 8; off < 32; off <<= 1) {
    dy += __shfl_xor_sync(FULL, dy, off);
    Iv += __shfl_xor_sync(FULL, Iv, off);
  }
  if (lane < 4) {
    S.wpart[(w * kS + 2 * lane) * 24 + 0] = dxe;
    S.wpart[(w * kS + 2 * lane + 1) * 24 + 0] = dxo;
  }
  if (lane < kS) {
    S.wpart[(w * kS + lane) * 24 + 1] = dy;
    S.wpart[(w * kS + lane) * 24 + 2] = Iv;
  }
  __syncthreads();
  if (threadIdx.x < kS * 3) {
    const int s = threadIdx.x / 3, k = threadIdx.x % 3;
    double a = 0.0;
    for (int ww = 0; ww < kThreads / 32; ++ww) a += S.wpart[(ww * kS + s) * 24 + k];
    S.part[s * 24 + k] = a;
  }
}

// Check-phase accumulators with the fragment layouts in mind (no per-instance arrays, which
// would live in local memory): the GEMM1 epilogue of lane l touches instances 2(l%4) and
// 2(l%4)+1 (ce, co), the row loops instance tid % 8 (r).  MX: bit k = max-reduced value.
template <int V>
struct FragAcc {
  double ce[V], co[V], r[V];
  __device__ FragAcc() {
#pragma unroll
    for (int k = 0; k < V; ++k) { ce[k] = 0.0; co[k] = 0.0; r[k] = 0.0; }
  }
};
template <int V, unsigned MX>
__device__ __forceinline__ void frag_col(FragAcc<V> &A, int s, const double (&t)[V]) {
  const bool odd = s & 1;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const bool mx = (MX >> k) & 1u;
    const double e = odd ? 0.0 : t[k], o = odd ? t[k] : 0.0;   // 0 is neutral for sums and for maxima of values >= 0
    A.ce[k] = mx ? fmax(A.ce[k], e) : A.ce[k] + e;
    A.co[k] = mx ? fmax(A.co[k], o) : A.co[k] + o;
  }
}
template <int V, unsigned MX>
__device__ __forceinline__ void frag_row(FragAcc<V> &A, const double (&t)[V]) {
#pragma unroll
  for (int k = 0; k < V; ++k) A.r[k] = ((MX >> k) & 1u) ? fmax(A.r[k], t[k]) : A.r[k] + t[k];
}
// FragAcc -> S.part[s][0..V) (fixed order): column parts reduced over lanes with equal l%4,
// row parts over lanes with equal l%8, combined per instance, then warps in order.
template <int V, unsigned MX = 0u>
__device__ __forceinline__ void frag_partials(FragAcc<V> &A, const Smem &S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const bool mx = (MX >> k) & 1u;
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      const double e = __shfl_xor_sync(FULL, A.ce[k], off), o = __shfl_xor_sync(FULL, A.co[k], off);
      A.ce[k] = mx ? fmax(A.ce[k], e) : A.ce[k] + e;
      A.co[k] = mx ? fmax(A.co[k], o) : A.co[k] + o;
    }
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) {
      const double r = __shfl_xor_sync(FULL, A.r[k], off);
      A.r[k] = mx ? fmax(A.r[k], r) : A.r[k] + r;
    }
  }
  if (lane < 4) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      S.wpart[(w * kS + 2 * lane) * 24 + k] = A.ce[k];
      S.wpart[(w * kS + 2 * lane + 1) * 24 + k] = A.co[k];
    }
  }
  __syncwarp();
  if (lane < kS) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double *d = &S.wpart[(w * kS + lane) * 24 + k];
      *d = ((MX >> k) & 1u) ? fmax(*d, A.r[k]) : *d + A.r[k];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kS * V; t += kThreads) {
    const int s = t / V, k = t % V;
    const bool mx = (MX >> k) & 1u;
    double acc = 0.0;
    for (int ww = 0; ww < kThreads / 32; ++ww) {
      const double o = S.wpart[(ww * kS + s) * 24 + k];
      acc = mx ? fmax(acc, o) : acc + o;
    }
    S.part[s * 24 + k] = acc;
  }
}

// After a cluster barrier: tot[s][k] = sum over cluster ranks (in rank order) of part.
template <int CL, int V, unsigned MX = 0u>
__device__ __forceinline__ void cluster_totals(cg::cluster_group &cl, const Smem &S, double *tot /* kS*24 */) {
  for (int t = threadIdx.x; t < kS * V; t += kThreads) {
    const int s = t / V, k = t % V;
    const bool mx = (MX >> k) & 1u;
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      const double o = cl.map_shared_rank(S.part, c)[s * 24 + k];
      a = mx ? fmax(a, o) : a + o;
    }
    tot[s * 24 + k] = a;
  }
  __syncthreads();
}

template <int CL>
__global__ void __launch_bounds__(kThreads, 1) dmma_kernel(const DmmaParams P) {
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  extern __shared__ __align__(16) double sm[];
  const int n = P.n, m = P.m, m1 = P.m1, np = P.np, mp = P.mp;
  Smem S;
  S.Ks = sm;
  S.Yf = S.Ks + (size_t)mp * np;
  S.Xc = S.Yf + (size_t)mp * kS;
  S.Pc = S.Xc + (size_t)np * kS;
  S.part_a = S.Pc + (size_t)mp * kS;
  S.part_b = S.part_a + kS * 24;
  S.part = S.part_b;
  S.wpart = S.part_b + kS * 24;
  double *tot = S.wpart + (kThreads / 32) * kS * 24;
  S.inst = (Inst *)(tot + kS * 24);
  S.grp = (int *)(S.inst + kS);
  const int tid = threadIdx.x;
#ifdef MPAX_DEBUG
  if (tid == 0) printf("dmma block %d rank %d n %d m %d nc %d np %d mp %d mc %d batch %lld\n", blockIdx.x, crank, n, m,
                       P.nc, np, mp, P.mc, (long long)P.batch);
#endif
  const int j0 = crank * P.nc, jn = min(n, j0 + P.nc) - j0;      // this CTA's columns [j0, j0 + jn)
  const int i0 = crank * P.mc, in_ = max(0, min(m, i0 + P.mc) - i0);  // this CTA's rows [i0, i0 + in_)
  const bool r2 = P.alg == LP_R2HPDHG;
  // ---- K~ column slice into shared memory once (zero padded) ----
  for (int t = tid; t < mp * np; t += kThreads) {
    const int i = t / np, jj = t % np;
    S.Ks[t] = (i < m && jj < jn) ? P.K[(size_t)i * n + j0 + jj] : 0.0;
  }
  for (int t = tid; t < mp * kS; t += kThreads) { S.Yf[t] = 0.0; S.Pc[t] = 0.0; }
  for (int t = tid; t < np * kS; t += kThreads) S.Xc[t] = 0.0;
  const bool cstep = P.const_step != 0;  // constant step rule (reading 34)
  const double eta0 = initial_eta(P.kmax, P.sigma, cstep);
  // r2HPDHG reflection z <- a((1 + rho) w - rho z) + b z0 (rho = 1: 2 PDHG(z) - z; reading 38)
  const double rf1 = 1.0 + P.rho, rf0 = P.rho;
  // the check's pass test: relative KKT, or a polishing sub-solve's single residual (reading 36)
  auto tpass = [&](const Kkt5 &k, double nq, double nc) {
    return P.polish_mode ? polish_pass(P.polish_mode, k.pres, k.dres, nq, nc, P.eps_fp)
                         : kkt5_pass(k, nq, nc, P.eps_abs, P.eps_rel);
  };

  for (;;) {
    // ---- next group of 8 instances (rank 0 pulls from the queue) ----
    cl.sync();
    if (crank == 0 && tid == 0) *S.grp = (int)atomicAdd(P.queue, 1ull);
    cl.sync();
    const int64_t g = *cl.map_shared_rank(S.grp, 0);
    cl.sync();  // nobody leaves (or reuses S.grp) while a peer still reads rank 0's S.grp
    if (g * kS >= P.batch) return;
    const int64_t b0 = g * kS;
    if (tid < kS) {
      Inst &I = S.inst[tid];
      I = Inst();
      I.valid = (b0 + tid) < P.batch;
      I.done = !I.valid;
      if (I.valid && P.active && P.active[b0 + tid].status != LP_OPTIMAL) { I.done = 1; I.skip = 1; }
    }
    __syncthreads();
    // ---- step 2: scaled data, start point, norms (partials: |c~|^2, |q~|^2, |c|^2, |q|^2) ----
    {
      double v[kS][4] = {};
      for (int t = tid; t < jn * kS; t += kThreads) {
        const int s = t / jn, jj = t % jn, j = j0 + jj;
        if (!S.inst[s].valid) continue;
        const int64_t b = b0 + s;
        const double dc = P.Dc[j], c = P.C0[b * P.cstride + j], cj = c * dc;
        P.cs[b * n + j] = cj;
        v[s][0] += cj * cj;
        v[s][2] += c * c;
        const double xv = median3(P.ls[j], P.X0 ? P.X0[b * n + j] / dc : 0.0, P.us[j]);
        P.x[b * n + j] = xv; P.xa[b * n + j] = xv; P.xr[b * n + j] = xv; P.xp[b * n + j] = xv;
        S.Xc[jj * kS + s] = xv;
      }
      for (int t = tid; t < in_ * kS; t += kThreads) {
        const int s = t / in_, ii = t % in_, i = i0 + ii;
        if (!S.inst[s].valid) continue;
        const int64_t b = b0 + s;
        const double dr = P.Dr[i], qv = P.Q0[b * P.qstride + i], qi = qv * dr;
        P.qs[b * m + i] = qi;
        v[s][1] += qi * qi;
        v[s][3] += qv * qv;
        double yv = P.Y0 ? P.Y0[b * m + i] / dr : 0.0;
        if (i < m1) yv = fmax(yv, 0.0);
        P.y[b * m + i] = yv; P.ya[b * m + i] = yv; P.yr[b * m + i] = yv; P.yp[b * m + i] = yv;
        S.Yf[i * kS + s] = yv;
      }
      S.part = (S.part == S.part_a) ? S.part_b : S.part_a;  // double-buffered (see grid_solver.cu)
      cta_partials<4>(v, S);
      cl.sync();
      cluster_totals<CL, 4>(cl, S, tot);
      if (tid < kS && S.inst[tid].valid) {
        Inst &I = S.inst[tid];
        const double* t4 = tot + tid * 24;
        I.nc0 = sqrt(t4[2]); I.nq0 = sqrt(t4[3]);
        I.omega = 1.0;
        if (sqrt(t4[0]) > 1e-10 && sqrt(t4[1]) > 1e-10) I.omega = sqrt(t4[0]) / sqrt(t4[1]);
        I.inv_omega = 1.0 / I.omega;  // every x / omega is x * omega^-1 (reading 32)
        I.eta = eta0; I.last = INFINITY;
      }
      // full y0 from the peers' row slices
      for (int c = 0; c < CL; ++c) {
        if (c == crank) continue;
        const int ci0 = c * P.mc, cin = max(0, min(m, ci0 + P.mc) - ci0);
        const double *rem = cl.map_shared_rank(S.Yf, c);
        for (int t = tid; t < cin * kS; t += kThreads) S.Yf[(ci0 + t / kS) * kS + t % kS] = rem[(ci0 + t / kS) * kS + t % kS];
      }
      __syncthreads();
    }
    // K~x0 (GEMM2 + cluster reduce) and K~'y0 (GEMM1); raPDHG reference KKT_omega(z0)
    gemm2(S, np, mp);
    cl.sync();
    {
      double v[kS][4] = {};
      for (int t = tid; t < in_ * kS; t += kThreads) {
        const int ii = t / kS, s = t % kS, i = i0 + ii;
        if (!S.inst[s].valid) continue;
        double a = 0.0;
        for (int c = 0; c < CL; ++c) a += cl.map_shared_rank(S.Pc, c)[i * kS + s];
        const int64_t b = b0 + s;
        P.Kx[b * m + i] = a; P.Kxa[b * m + i] = a; P.Kxp[b * m + i] = a;
        kkt_row_acc(v[s], false, i < m1, 1.0, P.y[b * m + i], a, 0.0, P.qs[b * m + i]);
      }
      gemm1(S, np, mp, [&](int jj, int s, double val) {
        if (jj >= jn || !S.inst[s].valid) return;
        const int64_t b = b0 + s;
        const int j = j0 + jj;
        P.KTy[b * n + j] = val; P.KTya[b * n + j] = val; P.KTyp[b * n + j] = val;
        kkt_col_acc(v[s], false, 1.0, P.x[b * n + j], val, 0.0, P.cs[b * n + j], 0.0, P.ls[j], 0.0, P.us[j]);
      });
      S.part = (S.part == S.part_a) ? S.part_b : S.part_a;  // double-buffered (see grid_solver.cu)
      cta_partials<4>(v, S);
      cl.sync();
      cluster_totals<CL, 4>(cl, S, tot);
      if (tid < kS && S.inst[tid].valid && !r2) {
        Inst &I = S.inst[tid];
        const Kkt5 ks = kkt5(tot + tid * 24);
        I.ref = kkt_omega(ks, I.omega, I.inv_omega);
      }
      __syncthreads();
    }

    // ====================== attempts (lock-step over the group) ======================
    for (;;) {
      bool all_done = true;
      for (int s = 0; s < kS; ++s) all_done &= (bool)S.inst[s].done;
      if (all_done) break;
      // ---- phase A: GEMM1 = K~_c' Y' ; [commit n-side] ; primal step ; X'_c ----
      double dx_even = 0.0, dx_odd = 0.0;  // this lane's instances 2q and 2q+1 (GEMM1 fragment layout)
      struct OpsA {
        double x, kt, xp, xa, cs, ls, us, kta;
      };
      gemm1_pre(S, np, mp, [&](int jj, int s) {
        OpsA o = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const Inst &I = S.inst[s];
        if (jj >= jn || I.done) return o;
        const int j = j0 + jj;
        const int64_t off = (b0 + s) * n + j;
        o.x = P.x[off]; o.kt = P.KTy[off]; o.cs = P.cs[off]; o.ls = P.ls[j]; o.us = P.us[j];
        if (I.pending) {
          o.xp = P.xp[off]; o.xa = P.xa[off];
          if (r2) o.kta = P.KTya[off];
        }
        return o;
      }, [&](int jj, int s, double kty, const OpsA &op) {
        const Inst &I = S.inst[s];
        if (jj >= jn || I.done) { if (jj < np) S.Xc[jj * kS + s] = 0.0; return; }
        const int64_t b = b0 + s;
        const int j = j0 + jj;
        const int64_t o = b * n + j;
        double xv = op.x, kt = op.kt;
        if (I.pending) {
          const double xpv = op.xp;
          if (!r2) {
            P.xa[o] = op.xa + I.theta * (xpv - op.xa);
            xv = xpv; kt = kty;
          } else {
            xv = I.ha * (rf1 * xpv - rf0 * xv) + I.hb * op.xa;
            kt = I.ha * (rf1 * kty - rf0 * kt) + I.hb * op.kta;
          }
          P.x[o] = xv; P.KTy[o] = kt;
        }
        const double tau = I.eta * I.inv_omega;
        const double xn = median3(op.ls, xv - tau * (op.cs - kt), op.us);
        P.xp[o] = xn;
        S.Xc[jj * kS + s] = xn;
        const double d = xn - xv;
        if (s & 1) dx_odd += d * d; else dx_even += d * d;
      });
      __syncthreads();
      // ---- phase B operands of this thread's first two row items, loaded before GEMM2 (in flight
      // during it and the cluster barrier) ----
      struct OpsB {
        double y, kx, yp, kxp, ya, kxa, qs;
      };
      OpsB pb[2];
      auto load_b = [&](int t) {
        OpsB o = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const int ii = t / kS, s = t % kS, i = i0 + ii;
        const Inst &I = S.inst[s];
        if (I.done) return o;
        const int64_t off = (b0 + s) * m + i;
        o.y = P.y[off]; o.kx = P.Kx[off]; o.qs = P.qs[off];
        if (I.pending) {
          o.yp = P.yp[off]; o.kxp = P.Kxp[off]; o.ya = P.ya[off];
          if (r2) o.kxa = P.Kxa[off];
        }
        return o;
      };
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = tid + u * kThreads;
        if (t < in_ * kS) pb[u] = load_b(t);
      }
      // ---- GEMM2: partial K~_c X'_c ----
      gemm2(S, np, mp);
      cl.sync();
      // ---- phase B: reduce K~x' for own rows; [commit m-side]; dual step ----
      double dy_own = 0.0, I_own = 0.0;  // instance tid % 8 (kThreads is a multiple of kS)
      auto row_b = [&](int t, const OpsB &op) {
        const int ii = t / kS, s = t % kS, i = i0 + ii;
        const Inst &I = S.inst[s];
        if (I.done) return;
        double kxp = 0.0;
        for (int c = 0; c < CL; ++c) kxp += cl.map_shared_rank(S.Pc, c)[i * kS + s];
        const int64_t b = b0 + s;
        const int64_t o = b * m + i;
        double yv = op.y, kxv = op.kx;
        if (I.pending) {
          const double ypv = op.yp, kxpo = op.kxp;
          if (!r2) {
            P.ya[o] = op.ya + I.theta * (ypv - op.ya);
            yv = ypv; kxv = kxpo;
          } else {
            yv = I.ha * (rf1 * ypv - rf0 * yv) + I.hb * op.ya;
            kxv = I.ha * (rf1 * kxpo - rf0 * kxv) + I.hb * op.kxa;
          }
          P.y[o] = yv; P.Kx[o] = kxv;
        }
        const double sigma = I.eta * I.omega;
        double yn = yv + sigma * (op.qs - 2.0 * kxp + kxv);
        if (i < m1) yn = pos_part(yn);
        P.yp[o] = yn; P.Kxp[o] = kxp;
        S.Yf[i * kS + s] = yn;
        const double d = yn - yv;
        dy_own += d * d;
        I_own += d * (kxp - kxv);
      };
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = tid + u * kThreads;
        if (t < in_ * kS) row_b(t, pb[u]);
      }
      for (int t = tid + 2 * kThreads; t < in_ * kS; t += kThreads) row_b(t, load_b(t));
      S.part = (S.part == S.part_a) ? S.part_b : S.part_a;
      attempt_partials(dx_even, dx_odd, dy_own, I_own, S);
      cl.sync();
      cluster_totals<CL, 3>(cl, S, tot);
      // peers' Y' rows for the next GEMM1
      for (int c = 0; c < CL; ++c) {
        if (c == crank) continue;
        const int ci0 = c * P.mc, cin = max(0, min(m, ci0 + P.mc) - ci0);
        const double *rem = cl.map_shared_rank(S.Yf, c);
        for (int t = tid; t < cin * kS; t += kThreads) S.Yf[ci0 * kS + t] = rem[ci0 * kS + t];
      }
      // ---- decisions (step 3 / 4 bookkeeping), one thread per instance ----
      if (tid < kS) {
        Inst &I = S.inst[tid];
        I.check = 0;
        if (!I.done) {
          const double *t3 = tot + tid * 24;
          I.pending = 0;
          I.j += 1;
          double f1, f2;
          step_factors(P.tab, I.j, f1, f2);
          const double Iv = t3[2];
          const double M = I.omega * t3[0] + t3[1] * I.inv_omega;
          const double eb = (Iv != 0.0) ? M / (2.0 * fabs(Iv)) : INFINITY;
          const bool acc = cstep || I.eta <= eb;
          const double eta_used = I.eta;
          if (!cstep) I.eta = fmin(f1 * eb, f2 * I.eta);
          if (!acc) {
            if (++I.rejects >= 100) { I.status = LP_NUMERICAL_ERROR; I.done = 1; I.outsel = 0; }
          } else {
            I.rejects = 0;
            if (!r2) {
              const double W1 = I.W + eta_used;
              I.theta = eta_used / W1;
              I.W = W1;
            } else {
              I.rP = sqrt(fmax(0.0, M / eta_used - 2.0 * Iv));
              if (I.k_in == 0) I.ref = I.rP;
              I.ha = (double)(I.k_in + 1) / (double)(I.k_in + 2);
              I.hb = 1.0 / (double)(I.k_in + 2);
            }
            I.k += 1;
            I.k_in += 1;
            I.pending = 1;
            if (I.k % P.check_freq == 0 || I.k == P.iter_limit) I.check = 1;
          }
        }
      }
      __syncthreads();
      bool any_check = false;
      for (int s = 0; s < kS; ++s) any_check |= (bool)S.inst[s].check;
      if (!any_check) continue;

      // ====================== check (step 5) for the flagged instances ======================
      // commit-only, both sides, for every pending instance; K~'y' from GEMM1.
      // Infeasibility rays (reading 35) of the checked instances: raPDHG z - (pre-step point),
      // whose pre-step values are parked in xp / KTyp / yp / Kxp (free until the next attempt),
      // r2HPDHG z - (Halpern anchor xa ...).
      FragAcc<6> vc;          // r2HPDHG KKT of w and distances (sums)
      FragAcc<6> vq;          // |dy|^2, |dx|^2, dual-ray obj, c'dx | viol_y, viol_x (max)
      gemm1(S, np, mp, [&](int jj, int s, double kty) {
        const Inst &I = S.inst[s];
        if (jj >= jn || I.done || !I.pending) return;
        const int64_t b = b0 + s;
        const int j = j0 + jj;
        const int64_t o = b * n + j;
        const double xpv = P.xp[o];
        if (!r2) {
          const double xo = P.x[o], kto = P.KTy[o];
          P.xa[o] += I.theta * (xpv - P.xa[o]);
          P.x[o] = xpv; P.KTy[o] = kty;
          P.xp[o] = xo; P.KTyp[o] = kto;
          if (I.check) {
            CertAcc acc;
            cert_col(acc, P.Dc[j], xpv, xo, kty, kto, P.C0[b * P.cstride + j], P.l0[j], P.u0[j]);
            const double t6[6] = {acc.sy, acc.sx, acc.oy, acc.ox, acc.vy, acc.vx};
            frag_col<6, (3u << 4)>(vq, s, t6);
          }
        } else {
          P.KTyp[o] = kty;
          P.x[o] = I.ha * (rf1 * xpv - rf0 * P.x[o]) + I.hb * P.xa[o];
          P.KTy[o] = I.ha * (rf1 * kty - rf0 * P.KTy[o]) + I.hb * P.KTya[o];
          if (I.check) {
            CertAcc acc;
            cert_col(acc, P.Dc[j], P.x[o], P.xa[o], P.KTy[o], P.KTya[o], P.C0[b * P.cstride + j], P.l0[j], P.u0[j]);
            const double t6[6] = {acc.sy, acc.sx, acc.oy, acc.ox, acc.vy, acc.vx};
            frag_col<6, (3u << 4)>(vq, s, t6);
            double tc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            kkt_col_acc(tc, true, P.Dc[j], xpv, kty, P.C0[b * P.cstride + j], P.cs[o], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
            const double d = xpv - P.xr[o];
            tc[4] = d * d;
            frag_col<6, 0u>(vc, s, tc);
          }
        }
      });
      for (int t = tid; t < in_ * kS; t += kThreads) {
        const int ii = t / kS, s = t % kS, i = i0 + ii;
        const Inst &I = S.inst[s];
        if (I.done || !I.pending) continue;
        const int64_t b = b0 + s;
        const int64_t o = b * m + i;
        const double ypv = P.yp[o], kxp = P.Kxp[o];
        const double q0i = P.Q0[b * P.qstride + i];
        if (!r2) {
          const double yo = P.y[o], kxo = P.Kx[o];
          P.ya[o] += I.theta * (ypv - P.ya[o]);
          P.y[o] = ypv; P.Kx[o] = kxp;
          P.yp[o] = yo; P.Kxp[o] = kxo;
          if (I.check) {   // s = tid % 8 in these row loops (kThreads is a multiple of 8)
            CertAcc acc;
            cert_row(acc, i < m1, P.Dr[i], ypv, yo, kxp, kxo, q0i);
            const double t6[6] = {acc.sy, 0.0, acc.oy, 0.0, acc.vy, acc.vx};
            frag_row<6, (3u << 4)>(vq, t6);
          }
        } else {
          P.y[o] = I.ha * (rf1 * ypv - rf0 * P.y[o]) + I.hb * P.ya[o];
          P.Kx[o] = I.ha * (rf1 * kxp - rf0 * P.Kx[o]) + I.hb * P.Kxa[o];
          if (I.check) {
            CertAcc acc;
            cert_row(acc, i < m1, P.Dr[i], P.y[o], P.ya[o], P.Kx[o], P.Kxa[o], q0i);
            const double t6[6] = {acc.sy, 0.0, acc.oy, 0.0, acc.vy, acc.vx};
            frag_row<6, (3u << 4)>(vq, t6);
            double tr[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            kkt_row_acc(tr, true, i < m1, P.Dr[i], ypv, kxp, P.Q0[b * P.qstride + i], P.qs[o]);
            const double d = ypv - P.yr[o];
            tr[5] = d * d;
            frag_row<6, 0u>(vc, tr);
          }
        }
      }
      __syncthreads();
      if (tid < kS) S.inst[tid].pending = 0;
      cl.sync();  // every rank's commits (global state) visible before they are read across slices
      // certificate totals -> per-instance verdict (applied after the optimality tests)
      S.part = (S.part == S.part_a) ? S.part_b : S.part_a;
      frag_partials<6, (3u << 4)>(vq, S);
      cl.sync();
      cluster_totals<CL, 6, (3u << 4)>(cl, S, tot);
      if (tid < kS) {
        Inst &I = S.inst[tid];
        if (I.check) {
          const double *t6 = tot + tid * 24;
          CertAcc t;
          t.sy = t6[0]; t.sx = t6[1]; t.oy = t6[2]; t.ox = t6[3]; t.vy = t6[4]; t.vx = t6[5];
          I.cert = cert_decide(t, P.eps_pi, P.eps_di, I.ray_ny, I.ray_nx);
        }
      }
      __syncthreads();
      if (r2) {
        S.part = (S.part == S.part_a) ? S.part_b : S.part_a;
        frag_partials<6>(vc, S);
        cl.sync();
        cluster_totals<CL, 6>(cl, S, tot);
        if (tid < kS) {
          Inst &I = S.inst[tid];
          if (I.check) {
            const double *t6 = tot + tid * 24;
            const Kkt5 kw = kkt5(t6);
            if (cl.block_rank() == 0 && verbose_due(P.verbose, P.display_freq, I.k, P.check_freq))
              verbose_line(b0 + tid, I.k, kw.pobj, kw.dobj, kw.pres, kw.dres, kw.gap, I.omega, I.eta);
            if (tpass(kw, I.nq0, I.nc0)) { I.status = LP_OPTIMAL; I.done = 1; I.outsel = 1; }
            else if (I.cert) { I.status = I.cert; I.done = 1; I.outsel = 0; I.rays = 1; }
            else if (I.k == P.iter_limit) { I.status = LP_ITERATION_LIMIT; I.done = 1; I.outsel = 1; }
            else { I.metric = I.rP; I.dx2c = t6[4]; I.dy2c = t6[5]; I.csel = 1; }
          }
        }
      } else {
        // average's products: X-bar slice -> GEMM2 -> reduce; full Y-bar -> GEMM1
        __syncthreads();
        for (int t = tid; t < np * kS; t += kThreads) {
          const int jj = t / kS, s = t % kS;
          S.Xc[t] = (jj < jn && S.inst[s].check) ? P.xa[(b0 + s) * n + j0 + jj] : 0.0;
        }
        for (int t = tid; t < mp * kS; t += kThreads) {
          const int i = t / kS, s = t % kS;
          S.Yf[t] = (i < m && S.inst[s].check) ? P.ya[(b0 + s) * m + i] : 0.0;
        }
        __syncthreads();
        gemm2(S, np, mp);
        cl.sync();
        FragAcc<20> v;
        for (int t = tid; t < in_ * kS; t += kThreads) {   // s = tid % 8
          const int ii = t / kS, s = t % kS, i = i0 + ii;
          if (!S.inst[s].check) continue;
          double kxa = 0.0;
          for (int c = 0; c < CL; ++c) kxa += cl.map_shared_rank(S.Pc, c)[i * kS + s];
          const int64_t b = b0 + s;
          const int64_t o = b * m + i;
          P.Kxa[o] = kxa;
          const double dr = P.Dr[i], yai = P.ya[o], yi = P.y[o], kxi = P.Kx[o], q0 = P.Q0[b * P.qstride + i],
                       qsi = P.qs[o];
          const bool ge = i < m1;
          double tr[20];
#pragma unroll
          for (int k = 0; k < 20; ++k) tr[k] = 0.0;
          kkt_row_acc(tr + 0, true, ge, dr, yai, kxa, q0, qsi);
          kkt_row_acc(tr + 4, true, ge, dr, yi, kxi, q0, qsi);
          kkt_row_acc(tr + 8, false, ge, dr, yai, kxa, q0, qsi);
          kkt_row_acc(tr + 12, false, ge, dr, yi, kxi, q0, qsi);
          const double da = yai - P.yr[o], dcur = yi - P.yr[o];
          tr[17] = da * da;
          tr[19] = dcur * dcur;
          frag_row<20, 0u>(v, tr);
        }
        gemm1(S, np, mp, [&](int jj, int s, double kta) {
          if (jj >= jn || !S.inst[s].check) return;
          const int64_t b = b0 + s;
          const int j = j0 + jj;
          const int64_t o = b * n + j;
          P.KTya[o] = kta;
          const double dc = P.Dc[j], xaj = P.xa[o], xj = P.x[o], ktj = P.KTy[o];
          const double c0 = P.C0[b * P.cstride + j], csj = P.cs[o], l0 = P.l0[j], lsj = P.ls[j], u0 = P.u0[j],
                       usj = P.us[j];
          double tc[20];
#pragma unroll
          for (int k = 0; k < 20; ++k) tc[k] = 0.0;
          kkt_col_acc(tc + 0, true, dc, xaj, kta, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(tc + 4, true, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(tc + 8, false, dc, xaj, kta, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(tc + 12, false, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
          const double da = xaj - P.xr[o], dcur = xj - P.xr[o];
          tc[16] = da * da;
          tc[18] = dcur * dcur;
          frag_col<20, 0u>(v, s, tc);
        });
        S.part = (S.part == S.part_a) ? S.part_b : S.part_a;
        frag_partials<20>(v, S);
        cl.sync();
        cluster_totals<CL, 20>(cl, S, tot);
        if (tid < kS) {
          Inst &I = S.inst[tid];
          if (I.check) {
            const double *t = tot + tid * 24;
            const Kkt5 ka = kkt5(t + 0), kc = kkt5(t + 4);
            if (cl.block_rank() == 0 && verbose_due(P.verbose, P.display_freq, I.k, P.check_freq))
              verbose_line(b0 + tid, I.k, kc.pobj, kc.dobj, kc.pres, kc.dres, kc.gap, I.omega, I.eta);
            if (tpass(ka, I.nq0, I.nc0)) { I.status = LP_OPTIMAL; I.done = 1; I.outsel = 1; }
            else if (tpass(kc, I.nq0, I.nc0)) { I.status = LP_OPTIMAL; I.done = 1; I.outsel = 0; }
            else if (I.cert) { I.status = I.cert; I.done = 1; I.outsel = 0; I.rays = 1; }
            else if (I.k == P.iter_limit) {
              I.status = LP_ITERATION_LIMIT; I.done = 1;
              I.outsel = kkt5_rel(ka, I.nq0, I.nc0) < kkt5_rel(kc, I.nq0, I.nc0) ? 1 : 0;
            } else {
              const Kkt5 sa = kkt5(t + 8), sc = kkt5(t + 12);
              const double e_a = kkt_omega(sa, I.omega, I.inv_omega);
              const double e_c = kkt_omega(sc, I.omega, I.inv_omega);
              if (restart_to_average(e_a, e_c)) { I.csel = 1; I.metric = e_a; I.dx2c = t[16]; I.dy2c = t[17]; }
              else { I.csel = 0; I.metric = e_c; I.dx2c = t[18]; I.dy2c = t[19]; }
            }
          }
        }
      }
      // restart test and primal weight (contract step 5), one thread per instance
      __syncthreads();
      if (tid < kS) {
        Inst &I = S.inst[tid];
        I.pending = 0;
        if (I.check && !I.done) {
          const bool restart = restart_due(I.k_in, I.k, I.metric, I.ref, I.last);
          I.last = I.metric;
          I.check = restart ? 2 : 0;
          if (restart) {
            I.restarts += 1;
            I.omega = primal_weight(I.omega, sqrt(I.dx2c), sqrt(I.dy2c));
            I.inv_omega = 1.0 / I.omega;
            I.k_in = 0;
            if (!r2) { I.W = 0.0; I.ref = I.metric; }
          }
        } else if (I.check) {
          I.check = 0;
        }
      }
      __syncthreads();
      // restart copies (check == 2): candidate -> current, anchor / average, restart point
      for (int t = tid; t < jn * kS; t += kThreads) {
        const int s = t / jn, jj = t % jn;
        const Inst &I = S.inst[s];
        if (I.check != 2) continue;
        const int64_t o = (b0 + s) * n + j0 + jj;
        double xv = P.x[o], kt = P.KTy[o];
        if (I.csel) { xv = r2 ? P.xp[o] : P.xa[o]; kt = r2 ? P.KTyp[o] : P.KTya[o]; }
        P.x[o] = xv; P.xr[o] = xv; P.xa[o] = xv; P.KTy[o] = kt; P.KTya[o] = kt;
      }
      for (int t = tid; t < in_ * kS; t += kThreads) {
        const int s = t / in_, ii = t % in_;
        const Inst &I = S.inst[s];
        if (I.check != 2) continue;
        const int64_t o = (b0 + s) * m + i0 + ii;
        double yv = P.y[o], kx = P.Kx[o];
        if (I.csel) { yv = r2 ? P.yp[o] : P.ya[o]; kx = r2 ? P.Kxp[o] : P.Kxa[o]; }
        P.y[o] = yv; P.yr[o] = yv; P.ya[o] = yv; P.Kx[o] = kx; P.Kxa[o] = kx;
      }
      // the next attempt restarts from committed state: refresh the full current y in Yf
      __syncthreads();
      cl.sync();
      for (int t = tid; t < mp * kS; t += kThreads) {
        const int i = t / kS, s = t % kS;
        S.Yf[t] = (i < m && !S.inst[s].done) ? P.y[(b0 + s) * m + i] : 0.0;
      }
      __syncthreads();
      if (tid < kS) S.inst[tid].check = 0;
      __syncthreads();
    }

    // ====================== step 6: output every instance of the group ======================
    {
      double v[kS][4] = {};
      for (int t = tid; t < jn * kS; t += kThreads) {
        const int s = t / jn, jj = t % jn, j = j0 + jj;
        const Inst &I = S.inst[s];
        if (!I.valid || I.skip) continue;
        const int64_t b = b0 + s;
        const int64_t o = b * n + j;
        const double xs = I.outsel ? (r2 ? P.xp[o] : P.xa[o]) : P.x[o];
        const double kt = I.outsel ? (r2 ? P.KTyp[o] : P.KTya[o]) : P.KTy[o];
        const double dc = P.Dc[j], c0 = P.C0[b * P.cstride + j];
        kkt_col_acc(v[s], true, dc, xs, kt, c0, P.cs[o], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
        if (I.rays) {  // infeasible: unit rays against the base (r2: anchor; ra: parked pre-step point)
          const double xb = r2 ? P.xa[o] : P.xp[o], ktb = r2 ? P.KTya[o] : P.KTyp[o];
          P.X[o] = dc * (xs - xb) / I.ray_nx;
          P.L[o] = -((kt - ktb) / dc) / I.ray_ny;
        } else {
          P.X[o] = dc * xs;
          P.L[o] = c0 - kt / dc;
        }
      }
      for (int t = tid; t < in_ * kS; t += kThreads) {
        const int s = t / in_, ii = t % in_, i = i0 + ii;
        const Inst &I = S.inst[s];
        if (!I.valid || I.skip) continue;
        const int64_t b = b0 + s;
        const int64_t o = b * m + i;
        const double ys = I.outsel ? (r2 ? P.yp[o] : P.ya[o]) : P.y[o];
        const double kx = I.outsel ? (r2 ? P.Kxp[o] : P.Kxa[o]) : P.Kx[o];
        const double dr = P.Dr[i];
        kkt_row_acc(v[s], true, i < m1, dr, ys, kx, P.Q0[b * P.qstride + i], P.qs[o]);
        if (I.rays) P.Y[o] = dr * (ys - (r2 ? P.ya[o] : P.yp[o])) / I.ray_ny;
        else P.Y[o] = dr * ys;
      }
      S.part = (S.part == S.part_a) ? S.part_b : S.part_a;  // double-buffered (see grid_solver.cu)
      cta_partials<4>(v, S);
      cl.sync();
      cluster_totals<CL, 4>(cl, S, tot);
      if (crank == 0 && tid < kS && S.inst[tid].valid && !S.inst[tid].skip) {
        const Inst &I = S.inst[tid];
        const Kkt5 ko = kkt5(tot + tid * 24);
        lp_result r;
        r.status = I.status; r.polish = 0;
        r.iterations = I.k; r.attempts = I.j; r.restarts = I.restarts;
        r.primal_objective = ko.pobj; r.dual_objective = ko.dobj;
        r.primal_residual = ko.pres; r.dual_residual = ko.dres; r.gap = ko.gap;
        r.rel_kkt = kkt5_rel(ko, I.nq0, I.nc0);
        r.omega = I.omega; r.eta = I.eta; r.solve_seconds = 0.0;
        P.res[b0 + tid] = r;
      }
    }
  }
}

template <int CL>
int launch_dmma(const DmmaParams &P, size_t smem, cudaStream_t s) {
  MPAX_CUDA(cudaFuncSetAttribute(dmma_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  MPAX_CUDA(cudaFuncSetAttribute(dmma_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(CL);
  MPAX_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, (void *)dmma_kernel<CL>, &cfg));
  if (max_clusters < 1) return LP_ERR_UNSUPPORTED;
  const int64_t groups = (P.batch + kS - 1) / kS;
  const int64_t clusters = groups < max_clusters ? groups : max_clusters;
  cfg.gridDim = dim3((unsigned)(clusters * CL));
  MPAX_CUDA(cudaMemsetAsync(P.queue, 0, sizeof(unsigned long long), s));
  MPAX_CUDA(cudaLaunchKernelEx(&cfg, dmma_kernel<CL>, P));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

}  // namespace

size_t dmma_workspace_doubles(int64_t n, int64_t m, int64_t batch) { return (size_t)batch * (size_t)(8 * n + 8 * m); }

int dmma_solve(const DevProblem &D, const lp_options &o, const InstanceLaunch &L, cudaStream_t s,
               unsigned long long *queue, double *work) {
  if (!D.dense) return LP_ERR_UNSUPPORTED;
  const int n = (int)D.n, m = (int)D.m;
  const int mp = (m + 7) / 8 * 8;
  int dev = 0, max_optin = 0;
  MPAX_CUDA(cudaGetDevice(&dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // smallest cluster whose column slice fits in shared memory
  for (int CL : {1, 2, 4, 8}) {
    const int nc = (n + CL - 1) / CL;
    const int np = (nc + 7) / 8 * 8;
    const size_t smem = sizeof(double) * ((size_t)mp * np + (size_t)mp * kS + (size_t)np * kS + (size_t)mp * kS +
                                          2 * kS * 24 + (kThreads / 32) * kS * 24 + kS * 24) +
                        sizeof(Inst) * kS + 64;
    if (smem + 1024 > (size_t)max_optin) continue;
    DmmaParams P;
    P.n = n; P.m = m; P.m1 = (int)D.m1; P.nc = nc; P.np = np; P.mp = mp; P.mc = (m + CL - 1) / CL;
    P.K = D.kv;
    P.Dr = D.Dr; P.Dc = D.Dc; P.ls = D.ls; P.us = D.us; P.l0 = D.l0; P.u0 = D.u0;
    P.C0 = L.C0; P.Q0 = L.Q0; P.X0 = L.X0; P.Y0 = L.Y0; P.cstride = L.cstride; P.qstride = L.qstride;
    P.kmax = D.kmax; P.sigma = D.sigma; P.tab = D.tab; P.const_step = o.step_rule == LP_STEP_CONSTANT;
    P.eps_abs = o.eps_abs; P.eps_rel = o.eps_rel; P.iter_limit = o.iteration_limit;
    P.check_freq = o.check_frequency; P.alg = o.algorithm;
    P.eps_pi = o.eps_primal_infeasible; P.eps_di = o.eps_dual_infeasible;
    P.eps_fp = o.eps_feas_polish; P.polish_mode = L.polish_mode; P.active = L.active; P.rho = o.reflection;
    P.verbose = o.verbose; P.display_freq = o.display_frequency;
    P.batch = L.batch; P.queue = queue;
    const size_t BN = (size_t)L.batch * n, BM = (size_t)L.batch * m;
    double *w = work;
    P.x = w; w += BN; P.KTy = w; w += BN; P.xa = w; w += BN; P.KTya = w; w += BN; P.xr = w; w += BN;
    P.cs = w; w += BN; P.xp = w; w += BN; P.KTyp = w; w += BN;
    P.y = w; w += BM; P.Kx = w; w += BM; P.ya = w; w += BM; P.Kxa = w; w += BM; P.yr = w; w += BM;
    P.qs = w; w += BM; P.yp = w; w += BM; P.Kxp = w; w += BM;
    P.X = L.X; P.Y = L.Y; P.L = L.L; P.res = L.res;
    switch (CL) {
      case 1: return launch_dmma<1>(P, smem, s);
      case 2: return launch_dmma<2>(P, smem, s);
      case 4: return launch_dmma<4>(P, smem, s);
      default: return launch_dmma<8>(P, smem, s);
    }
  }
  return LP_ERR_UNSUPPORTED;
}

}  // namespace mpax

// sharded.cu -- one LP whose constraint matrix is ROW-SHARDED across GPUs
// (§3.5 device parallelism: "the constraint
// matrix is ... the primary candidate for sharding", listing P:234-241 shards
// axis 0).  GPU g holds rows [r_g, r_g + m_g) of K = [G; A], the matching q and
// dual iterate, the CSR of its K~_g' (n x m_g), and a replicated copy of every
// n-long vector (x, K~'y, averages ...).  Per attempt (DESIGN.md §3 step 3/4):
//   K~_g' y'_g  (local partial, n)  --ncclAllReduce(sum)-->  K~'y'    [SpMV #2]
//   commit n-side + primal step x'   (replicated, identical on every GPU)
//   commit m-side + K~_g x' + dual step y'_g                            [SpMV #1]
//   ||dy||^2, <dy, K~dx> local partials --ncclAllReduce(sum)--> line-search decision
// The decision state lives in device memory; the host only enqueues work: since
// k grows by at most one per attempt, it enqueues (next_check - k) attempts and
// synchronises once per 64 accepted steps to run the check.
// Preconditioning reduces the column norms across GPUs (max for Ruiz, sum for
// Pock-Chambolle).  With one GPU this is a multi-kernel single-GPU path; the
// "virtual" mode runs p row shards on ONE GPU with a fixed-order device sum in
// place of NCCL, which is how the partitioned arithmetic is tested here.
//
// Column sharding (the axis chosen by min(m, n); reading 33):
// GPU g holds the columns [c_g, c_g + n_g) of K (K~_{:,g}, m x n_g, and its transpose), the
// matching c, l, u and primal iterate, and a replicated copy of every m-long vector.  Per attempt
//   K~'_g y'  (local: y' is replicated)             commit n-side + primal step x'_g  (local)
//   K~_{:,g} x'_g (partial, m) --ncclAllReduce(sum)--> K~x'                           [SpMV #1]
//   commit m-side + dual step y' (replicated), ||dx||^2 partials reduced across GPUs
// so the exchanged vector is the m-long one: with m < n (C5: 40 MB instead of 80 MB) the
// collective moves the shorter vector.  Row norms of the preconditioner are reduced instead of
// column norms.  The same kernels serve both modes; `cols` selects the data each reads.
//
// Exchange variant B of the row engine (lp_options.sharded_exchange = 1): the
// K~_g' y'_g partials are REDUCE-SCATTERED, so GPU g receives only its slice J_g of K~'y' (n/p
// columns) and runs the n-side commit and primal step on that slice alone; x' is then
// ALL-GATHERED for the rows step.  Same bytes on the wire as the all-reduce (which is a
// reduce-scatter + all-gather), but the n-side elementwise work is split p ways instead of
// replicated; the column-side scalar partials are then reduced like the row-side ones.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

#ifdef MPAX_HAVE_NCCL
#include <nccl.h>
#endif

namespace mpax {

namespace {

constexpr int kB = 256;  // threads per block
constexpr int kV = 24;   // partial-sum slots

struct ShState {
  double omega, inv_omega, eta, W, ref, last, theta, ha, hb, rP, M, Iv, eta_used, metric, nc0, nq0, eta0;
  long long k, j, k_in, restarts;
  int rejects, status, pending, halt, restart, outsel, csel, r2, cstep, rays;
  double colsum[kV];  // totals over this GPU's columns (replicated data: identical on every GPU)
  double rowsum[kV];  // totals over this GPU's rows; reduced across GPUs in place
  // infeasibility certificate partials (reading 35): |dy|^2, |dx|^2, dual-ray obj, c'dx (summed),
  // viol_y, viol_x (max); columns replicated, rows reduced across GPUs (sums, then maxima)
  double certc[6], certr[6];
  double ray_ny, ray_nx;
  double rho;  // r2HPDHG reflection parameter (reading 38)
  long long nchk;  // checks taken (the decision log's row index)
  unsigned int cnt_cols, cnt_rows;
};

struct Vecs {
  double *x, *KTy, *xp, *KTyp, *xa, *KTya, *xr, *cs, *red;  // n
  double *y, *Kx, *yp, *Kxp, *ya, *Kxa, *yr, *qs;           // m_local
  double *part;                                             // blocks x kV
  double *tmp;                                              // m_local: K~_L x' (two-pass rows step)
  const double *pre;                                        // column mode: K~x' summed across shards (m)
  const double *c0, *q0, *X0, *Y0;
};



// row r of a CSR matrix times x (all lanes of the row's group get the sum): G == 1 is the
// warp-tile CSR-stream of common.cuh (every lane of the warp calls it, r = tile row + lane;
// rows = the matrix's row count, buf = the warp's kTileBuf doubles); G >= 2 lanes per row
// with 4 entries in flight per lane otherwise
// LR: compile the full-chunk (long-row) path of tile_row_dot in (the matrix has a row of kTileCH
// entries or more; common.cuh)
template <bool LR>
__device__ __forceinline__ double row_dot(int64_t r, bool valid, int G, int gl, const int32_t *__restrict__ rp,
                                          const int32_t *__restrict__ ci, const double *__restrict__ v,
                                          const double *__restrict__ x, int64_t rows, double *buf) {
  if (G == 1) return tile_row_dot<double, double, LR>((int)r, valid, (int)rows, rp, ci, v, x, buf);
  double s0 = 0.0, s1 = 0.0;
  if (valid) {
    const int32_t e = __ldg(rp + r + 1);
    for (int32_t p = __ldg(rp + r) + gl; p < e; p += 4 * G) {
      int32_t c[4];
      double w[4], xv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t q = p + k * G;
        const bool ok = q < e;
        c[k] = ok ? __ldcs(ci + q) : 0;
        w[k] = ok ? __ldcs(v + q) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) xv[k] = (p + k * G < e) ? x[c[k]] : 0.0;
      s0 += w[0] * xv[0];
      s1 += w[1] * xv[1];
      s0 += w[2] * xv[2];
      s1 += w[3] * xv[3];
    }
  }
  double s = s0 + s1;
  for (int off = G >> 1; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
  return s;
}

// Block partials of V values into part[block][.]; the last block to finish sums
// them in block order (all 256 threads, fixed assignment + fixed tree) into out.
// MX: bit k set = value k is max-reduced (non-negative), else summed.
template <int V, unsigned MX = 0u>
__device__ __forceinline__ void last_block_sum(double (&v)[V], double *part, unsigned int *counter, double *out) {
  __shared__ double sred[kB / 32][kV];
  __shared__ double stree[kB];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double o = __shfl_xor_sync(FULL, s, off);
      s = ((MX >> k) & 1u) ? fmax(s, o) : s + o;
    }
    if (lane == 0) sred[w][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < V) {
    const bool mx = (MX >> threadIdx.x) & 1u;
    double a = 0.0;
    for (int ww = 0; ww < kB / 32; ++ww) a = mx ? fmax(a, sred[ww][threadIdx.x]) : a + sred[ww][threadIdx.x];
    part[(int64_t)blockIdx.x * kV + threadIdx.x] = a;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int k = 0; k < V; ++k) {
    const bool mx = (MX >> k) & 1u;
    double a = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kB) {
      const double o = __ldcg(part + (int64_t)b * kV + k);
      a = mx ? fmax(a, o) : a + o;
    }
    stree[threadIdx.x] = a;
    __syncthreads();
    for (int h = kB / 2; h; h >>= 1) {
      if (threadIdx.x < h)
        stree[threadIdx.x] = mx ? fmax(stree[threadIdx.x], stree[threadIdx.x + h]) : stree[threadIdx.x] + stree[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = stree[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) *counter = 0u;
}

inline int blocks_for(int64_t work) {
  int64_t g = (work + kB - 1) / kB;
  if (g < 1) g = 1;
  if (g > 148 * 8) g = 148 * 8;
  return (int)g;
}

// ------------------------------------------------------------------ kernels --

#ifdef MPAX_SH_SPMV_MINB   // experiments: resident CTAs per SM for the K~'y SpMV
#define SH_SPMV_BOUNDS __launch_bounds__(kB, MPAX_SH_SPMV_MINB)
#else
#define SH_SPMV_BOUNDS
#endif
template <bool LR>
__global__ void SH_SPMV_BOUNDS k_cols_spmv(const ShState *st, int64_t n, int G, const int32_t *trp, const int32_t *tci,
                            const double *tkv, const double *ysrc, double *out) {
  if (st->halt) return;
  __shared__ double s_tile[kB / 32][kTileBuf];
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x, ng = (int64_t)gridDim.x * kB / G;
  const int gl = (int)(gt % G);
  const int64_t iters = (n + ng - 1) / ng;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t j = it * ng + gt / G;
    const double s = row_dot<LR>(j, j < n, G, gl, trp, tci, tkv, ysrc, n, s_tile[threadIdx.x >> 5]);
    if (j < n && gl == 0) out[j] = s;
  }
}

enum { COLS_STEP = 0, COLS_COMMIT_ONLY = 1, COLS_AVG = 2, COLS_INIT = 3, COLS_INIT2 = 4, COLS_OUT = 5, COLS_CERT = 6 };
enum { ROWS_STEP = 0, ROWS_COMMIT_ONLY = 1, ROWS_AVG = 2, ROWS_INIT = 3, ROWS_INIT2 = 4, ROWS_OUT = 5, ROWS_CERT = 6 };

// MODE is a template parameter: each instantiation keeps only its own branch (fewer registers,
// no per-element mode tests), the per-element arithmetic is unchanged.
#ifdef MPAX_SH_COLS_MINB   // experiments: resident CTAs per SM for the column-side step kernels
#define SH_COLS_BOUNDS __launch_bounds__(kB, MPAX_SH_COLS_MINB)
#else
#define SH_COLS_BOUNDS
#endif
template <int MODE>
__global__ void SH_COLS_BOUNDS k_cols(ShState *st, int64_t j0, int64_t n, const DevProblem P, const Vecs V) {
  constexpr int mode = MODE;
  if (st->halt && mode != COLS_OUT) return;
  const bool r2 = st->r2, pend = st->pending;
  const double tau = st->eta * st->inv_omega, theta = st->theta, ha = st->ha, hb = st->hb;
  const double rf1 = 1.0 + st->rho, rf0 = st->rho;  // reflection (reading 38)
  double v[20] = {};
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x, st_ = (int64_t)gridDim.x * kB;
  for (int64_t j = j0 + gt; j < n; j += st_) {   // columns [j0, n): all, or this shard's slice (variant B)
    const double dc = P.Dc[j];
    if (mode == COLS_STEP || mode == COLS_COMMIT_ONLY) {
      double xv = V.x[j], kt = V.KTy[j];
      const double xold = xv, ktold = kt;
      const double kty = V.red[j];
      if (pend) {
        const double xpv = V.xp[j];
        if (!r2) {
          V.xa[j] += theta * (xpv - V.xa[j]);
          xv = xpv; kt = kty;
        } else {
          xv = ha * (rf1 * xpv - rf0 * xv) + hb * V.xa[j];
          kt = ha * (rf1 * kty - rf0 * kt) + hb * V.KTya[j];
        }
        V.x[j] = xv; V.KTy[j] = kt;
      }
      if (mode == COLS_STEP) {
        const double xn = median3(P.ls[j], xv - tau * (V.cs[j] - kt), P.us[j]);
        V.xp[j] = xn;
        const double d = xn - xv;
        v[0] += d * d;
      } else if (!r2) {
        // raPDHG: park the pre-step point in xp / KTyp (the infeasibility rays' base, reading 35)
        if (pend) { V.xp[j] = xold; V.KTyp[j] = ktold; }
      } else {
        V.KTyp[j] = kty;
        if (pend) {
          const double xpv = V.xp[j];
          kkt_col_acc(v, true, dc, xpv, kty, V.c0[j], V.cs[j], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
          const double d = xpv - V.xr[j];
          v[4] += d * d;
        }
      }
    } else if (mode == COLS_AVG) {
      const double kta = V.red[j];
      V.KTya[j] = kta;
      const double xaj = V.xa[j], xj = V.x[j], ktj = V.KTy[j], c0 = V.c0[j], csj = V.cs[j], l0 = P.l0[j],
                   lsj = P.ls[j], u0 = P.u0[j], usj = P.us[j];
      kkt_col_acc(v + 0, true, dc, xaj, kta, c0, csj, l0, lsj, u0, usj);
      kkt_col_acc(v + 4, true, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
      kkt_col_acc(v + 8, false, dc, xaj, kta, c0, csj, l0, lsj, u0, usj);
      kkt_col_acc(v + 12, false, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
      const double da = xaj - V.xr[j], dcur = xj - V.xr[j];
      v[16] += da * da;
      v[18] += dcur * dcur;
    } else if (mode == COLS_CERT) {
      const double *xb = r2 ? V.xa : V.xp, *ktb = r2 ? V.KTya : V.KTyp;
      CertAcc acc;
      cert_col(acc, dc, V.x[j], xb[j], V.KTy[j], ktb[j], V.c0[j], P.l0[j], P.u0[j]);
      v[0] += acc.sy; v[1] += acc.sx; v[2] += acc.oy; v[3] += acc.ox;
      v[4] = fmax(v[4], acc.vy); v[5] = fmax(v[5], acc.vx);
    } else if (mode == COLS_INIT) {
      const double c = V.c0[j], cj = c * dc;
      V.cs[j] = cj;
      v[0] += cj * cj;
      v[1] += c * c;
      const double xv = median3(P.ls[j], V.X0 ? V.X0[j] / dc : 0.0, P.us[j]);
      V.x[j] = xv; V.xa[j] = xv; V.xr[j] = xv; V.xp[j] = xv;
    } else if (mode == COLS_INIT2) {
      const double kty = V.red[j];
      V.KTy[j] = kty; V.KTya[j] = kty; V.KTyp[j] = kty;
      kkt_col_acc(v, false, dc, V.x[j], kty, 0.0, V.cs[j], 0.0, P.ls[j], 0.0, P.us[j]);
    } else {  // COLS_OUT
      const int sel = st->outsel;
      const double xs = sel ? (r2 ? V.xp[j] : V.xa[j]) : V.x[j];
      const double kt = sel ? (r2 ? V.KTyp[j] : V.KTya[j]) : V.KTy[j];
      kkt_col_acc(v, true, dc, xs, kt, V.c0[j], V.cs[j], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
      if (st->rays) {  // infeasible: unit rays against the base (reading 35)
        const double xb = r2 ? V.xa[j] : V.xp[j], ktb = r2 ? V.KTya[j] : V.KTyp[j];
        V.red[j] = dc * (xs - xb) / st->ray_nx;
        V.KTyp[j] = -((kt - ktb) / dc) / st->ray_ny;
      } else {
        V.red[j] = dc * xs;                    // unscaled x (output buffer)
        V.KTyp[j] = V.c0[j] - kt / dc;         // reduced costs (output buffer)
      }
    }
  }
  if (mode == COLS_CERT) {
    double c6[6] = {v[0], v[1], v[2], v[3], v[4], v[5]};
    last_block_sum<6, (3u << 4)>(c6, V.part, &st->cnt_cols, st->certc);
    return;
  }
  last_block_sum<20>(v, V.part, &st->cnt_cols, st->colsum);
}

// pass 1 of the two-pass rows step: V.tmp = K~_L x' (warp-tile mapping, same order as the grid kernel)
#ifdef MPAX_SH_LEFT_MINB   // experiments: resident CTAs per SM for pass 1 of the rows-side SpMV
#define SH_LEFT_BOUNDS __launch_bounds__(kB, MPAX_SH_LEFT_MINB)
#else
#define SH_LEFT_BOUNDS
#endif
template <bool LR>
__global__ void SH_LEFT_BOUNDS k_rows_left(const ShState *st, int64_t m, const DevProblem P, const double *x, double *tmp) {
  if (st->halt) return;
  __shared__ double s_tile[kB / 32][kTileBuf];
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x, nthr = (int64_t)gridDim.x * kB;
  for (int64_t base = gt - (threadIdx.x & 31); base < m; base += nthr) {
    const int64_t r = base + (threadIdx.x & 31);
    const double v = tile_row_dot<double, double, LR>((int)r, r < m, (int)m, P.rpL, P.ciL, P.kvL, x,
                                                       s_tile[threadIdx.x >> 5]);
    if (r < m) tmp[r] = v;
  }
}

// pass 2 in column mode: V.tmp += K~_R x' (the sum order of the rows step's pass 2: left + right)
template <bool LR>
__global__ void k_rows_right_add(const ShState *st, int64_t m, const DevProblem P, const double *x, double *tmp) {
  if (st->halt) return;
  __shared__ double s_tile[kB / 32][kTileBuf];
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x, nthr = (int64_t)gridDim.x * kB;
  for (int64_t base = gt - (threadIdx.x & 31); base < m; base += nthr) {
    const int64_t r = base + (threadIdx.x & 31);
    const double v = tile_row_dot<double, double, LR>((int)r, r < m, (int)m, P.rpR, P.ciR, P.kvR, x,
                                                       s_tile[threadIdx.x >> 5]);
    if (r < m) tmp[r] = tmp[r] + v;
  }
}

// four resident CTAs per SM (<= 64 registers; the gathers want the warps): C5 by rows at one
// rank 1.419 -> 1.377 ms per attempt, by columns 1.403 -> 1.384 (3 CTAs: 1.394 / 1.404;
// scripts/gpu_ab_sharded_rows.sh)
#ifndef MPAX_SH_ROWS_MINB
#define MPAX_SH_ROWS_MINB 4
#endif
#define SH_ROWS_BOUNDS __launch_bounds__(kB, MPAX_SH_ROWS_MINB)
template <int MODE, bool LR>
__global__ void SH_ROWS_BOUNDS k_rows(ShState *st, int64_t m, int64_t m1, int G, const DevProblem P, const Vecs V) {
  constexpr int mode = MODE;
  if (st->halt && mode != ROWS_OUT) return;
  const bool r2 = st->r2, pend = st->pending;
  const double sigma = st->eta * st->omega, theta = st->theta, ha = st->ha, hb = st->hb;
  const double rf1 = 1.0 + st->rho, rf0 = st->rho;  // reflection (reading 38)
  double v[20] = {};
  __shared__ double s_tile[kB / 32][kTileBuf];
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x;
  const bool spmv = (mode == ROWS_STEP || mode == ROWS_AVG || mode == ROWS_INIT2);
  const int g = spmv ? G : 1;
  const int64_t ng = (int64_t)gridDim.x * kB / g;
  const int gl = (int)(gt % g);
  const int64_t iters = (m + ng - 1) / ng;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = it * ng + gt / g;
    const bool ok = i < m;
    const bool lead = ok && gl == 0;
    const double *src = mode == ROWS_AVG ? V.xa : (mode == ROWS_INIT2 ? V.x : V.xp);
    // ROWS_STEP over split K~_g: pass 1 (k_rows_left) parked K~_L x' in V.tmp; add K~_R x'
    const bool two = mode == ROWS_STEP && P.split_h > 0 && g == 1;
    const double s = !spmv ? 0.0
                     : V.pre ? (ok ? V.pre[i] : 0.0)   // column mode: the cross-shard sum, computed before
                     : two ? (ok ? V.tmp[i] : 0.0) + row_dot<LR>(i, ok, 1, 0, P.rpR, P.ciR, P.kvR, src, m, s_tile[threadIdx.x >> 5])
                           : row_dot<LR>(i, ok, g, gl, P.rp, P.ci, P.kv, src, m, s_tile[threadIdx.x >> 5]);
    if (!lead) continue;
    const double dr = P.Dr[i];
    const bool ge = i < m1;
    if (mode == ROWS_STEP || mode == ROWS_COMMIT_ONLY) {
      double yv = V.y[i], kxv = V.Kx[i];
      const double yold = yv, kxold = kxv;
      if (pend) {
        const double ypv = V.yp[i], kxp = V.Kxp[i];
        if (!r2) {
          V.ya[i] += theta * (ypv - V.ya[i]);
          yv = ypv; kxv = kxp;
        } else {
          yv = ha * (rf1 * ypv - rf0 * yv) + hb * V.ya[i];
          kxv = ha * (rf1 * kxp - rf0 * kxv) + hb * V.Kxa[i];
        }
        V.y[i] = yv; V.Kx[i] = kxv;
      }
      if (mode == ROWS_STEP) {
        double yn = yv + sigma * (V.qs[i] - 2.0 * s + kxv);
        if (ge) yn = pos_part(yn);
        V.yp[i] = yn; V.Kxp[i] = s;
        const double d = yn - yv;
        v[0] += d * d;
        v[1] += d * (s - kxv);
      } else if (r2 && pend) {
        const double ypv = V.yp[i], kxp = V.Kxp[i];
        kkt_row_acc(v, true, ge, dr, ypv, kxp, V.q0[i], V.qs[i]);
        const double d = ypv - V.yr[i];
        v[5] += d * d;
      } else if (!r2 && pend) {
        V.yp[i] = yold; V.Kxp[i] = kxold;   // raPDHG: park the pre-step point (reading 35)
      }
    } else if (mode == ROWS_CERT) {
      const double *yb = r2 ? V.ya : V.yp, *kxb = r2 ? V.Kxa : V.Kxp;
      CertAcc acc;
      cert_row(acc, ge, dr, V.y[i], yb[i], V.Kx[i], kxb[i], V.q0[i]);
      v[0] += acc.sy; v[1] += acc.sx; v[2] += acc.oy; v[3] += acc.ox;
      v[4] = fmax(v[4], acc.vy); v[5] = fmax(v[5], acc.vx);
    } else if (mode == ROWS_AVG) {
      V.Kxa[i] = s;
      const double yai = V.ya[i], yi = V.y[i], kxi = V.Kx[i], q0 = V.q0[i], qsi = V.qs[i];
      kkt_row_acc(v + 0, true, ge, dr, yai, s, q0, qsi);
      kkt_row_acc(v + 4, true, ge, dr, yi, kxi, q0, qsi);
      kkt_row_acc(v + 8, false, ge, dr, yai, s, q0, qsi);
      kkt_row_acc(v + 12, false, ge, dr, yi, kxi, q0, qsi);
      const double da = yai - V.yr[i], dcur = yi - V.yr[i];
      v[17] += da * da;
      v[19] += dcur * dcur;
    } else if (mode == ROWS_INIT) {
      const double q = V.q0[i], qi = q * dr;
      V.qs[i] = qi;
      v[0] += qi * qi;
      v[1] += q * q;
      double yv = V.Y0 ? V.Y0[i] / dr : 0.0;
      if (ge) yv = fmax(yv, 0.0);
      V.y[i] = yv; V.ya[i] = yv; V.yr[i] = yv; V.yp[i] = yv;
    } else if (mode == ROWS_INIT2) {
      V.Kx[i] = s; V.Kxa[i] = s; V.Kxp[i] = s;
      kkt_row_acc(v, false, ge, dr, V.y[i], s, 0.0, V.qs[i]);
    } else {  // ROWS_OUT
      const int sel = st->outsel;
      const double ys = sel ? (r2 ? V.yp[i] : V.ya[i]) : V.y[i];
      const double kx = sel ? (r2 ? V.Kxp[i] : V.Kxa[i]) : V.Kx[i];
      kkt_row_acc(v, true, ge, dr, ys, kx, V.q0[i], V.qs[i]);
      if (st->rays) V.Kxp[i] = dr * (ys - (r2 ? V.ya[i] : V.yp[i])) / st->ray_ny;
      else V.Kxp[i] = dr * ys;  // unscaled y (output buffer)
    }
  }
  if (mode == ROWS_CERT) {
    double c6[6] = {v[0], v[1], v[2], v[3], v[4], v[5]};
    last_block_sum<6, (3u << 4)>(c6, V.part, &st->cnt_rows, st->certr);
    return;
  }
  last_block_sum<20>(v, V.part, &st->cnt_rows, st->rowsum);
}

// ---- single-thread decisions (identical inputs on every GPU) ----
__global__ void k_init_decide(ShState *st, int stage) {
  if (stage == 0) {  // norms: colsum = (|c~|^2, |c|^2) replicated; rowsum = (|q~|^2, |q|^2) reduced
    const double nc = sqrt(st->colsum[0]), nq = sqrt(st->rowsum[0]);
    st->nc0 = sqrt(st->colsum[1]);
    st->nq0 = sqrt(st->rowsum[1]);
    st->omega = (nc > 1e-10 && nq > 1e-10) ? nc / nq : 1.0;
    st->inv_omega = 1.0 / st->omega;  // every x / omega is x * omega^-1 (reading 32)
    st->eta = st->eta0;
  } else if (!st->r2) {  // raPDHG reference KKT_omega(z0): rows (reduced) + columns
    double t[4];
    for (int k = 0; k < 4; ++k) t[k] = st->rowsum[k] + st->colsum[k];
    const Kkt5 ks = kkt5(t);
    st->ref = kkt_omega(ks, st->omega, st->inv_omega);
  }
}

// alog (one shard, or null): the decision log's attempt rows (j, accepted, eta, eta_bar), lp.h
__global__ void k_decide(ShState *st, const double *tab, int64_t check_freq, int64_t iter_limit, double *alog,
                         int64_t acap) {
  if (st->halt) return;
  st->j += 1;
  double f1 = 0.0, f2 = 0.0;
  if (!st->cstep) step_factors(tab, st->j, f1, f2);
  const double dx2 = st->colsum[0], dy2 = st->rowsum[0], I = st->rowsum[1];
  const double M = st->omega * dx2 + dy2 * st->inv_omega;
  const double eb = (I != 0.0) ? M / (2.0 * fabs(I)) : INFINITY;
  const bool acc = st->cstep || st->eta <= eb;  // constant step rule: DESIGN.md reading 34
  const double eta_used = st->eta;
  if (alog && st->j <= acap) {
    double *r = alog + 4 * (st->j - 1);
    r[0] = (double)st->j; r[1] = acc ? 1.0 : 0.0; r[2] = eta_used; r[3] = eb;
  }
  if (!st->cstep) st->eta = fmin(f1 * eb, f2 * st->eta);
  if (!acc) {
    st->pending = 0;
    if (++st->rejects >= 100) { st->status = LP_NUMERICAL_ERROR; st->halt = 1; st->outsel = 0; }
    return;
  }
  st->rejects = 0;
  if (!st->r2) {
    const double W1 = st->W + eta_used;
    st->theta = eta_used / W1;
    st->W = W1;
  } else {
    st->rP = sqrt(fmax(0.0, M / eta_used - 2.0 * I));
    if (st->k_in == 0) st->ref = st->rP;
    st->ha = (double)(st->k_in + 1) / (double)(st->k_in + 2);
    st->hb = 1.0 / (double)(st->k_in + 2);
  }
  st->k += 1;
  st->k_in += 1;
  st->pending = 1;
}

__global__ void k_check_decide(ShState *st, double eps_abs, double eps_rel, double eps_pi, double eps_di,
                               int64_t iter_limit, int verbose, int display_freq, int64_t check_freq,
                               int polish_mode, double eps_fp, double *clog, int64_t ccap) {
  // the decision log's check rows (k, metric, ref, last, restart, outcome), lp.h
  auto log_check = [&](double metric_, int restart_, int outcome) {
    if (clog && st->nchk < ccap) {
      double *r = clog + 6 * st->nchk;
      r[0] = (double)st->k; r[1] = metric_; r[2] = st->ref; r[3] = st->last; r[4] = restart_; r[5] = outcome;
    }
    st->nchk += 1;
  };
  // the check's pass test: relative KKT, or a polishing sub-solve's single residual (reading 36)
  auto tpass = [&](const Kkt5 &k) {
    return polish_mode ? polish_pass(polish_mode, k.pres, k.dres, st->nq0, st->nc0, eps_fp)
                       : kkt5_pass(k, st->nq0, st->nc0, eps_abs, eps_rel);
  };
  double t[20];
  for (int k = 0; k < 20; ++k) t[k] = st->colsum[k] + st->rowsum[k];
  st->pending = 0;
  st->restart = 0;
  const double nq0 = st->nq0, nc0 = st->nc0;
  // infeasibility verdict (reading 35), applied after the optimality tests
  CertAcc ct;
  ct.sy = st->certc[0] + st->certr[0]; ct.sx = st->certc[1] + st->certr[1];
  ct.oy = st->certc[2] + st->certr[2]; ct.ox = st->certc[3] + st->certr[3];
  ct.vy = fmax(st->certc[4], st->certr[4]); ct.vx = fmax(st->certc[5], st->certr[5]);
  double ny = 1.0, nx = 1.0;
  const int cert = cert_decide(ct, eps_pi, eps_di, ny, nx);
  if (st->r2) {
    const Kkt5 kw = kkt5(t);
    if (verbose_due(verbose, display_freq, st->k, check_freq))
      verbose_line(0, st->k, kw.pobj, kw.dobj, kw.pres, kw.dres, kw.gap, st->omega, st->eta);
    if (tpass(kw)) { log_check(st->rP, 0, 1); st->status = LP_OPTIMAL; st->halt = 1; st->outsel = 1; return; }
    if (cert) {
      log_check(0.0, 0, 3);
      st->status = cert; st->halt = 1; st->outsel = 0; st->rays = 1; st->ray_ny = ny; st->ray_nx = nx;
      return;
    }
    if (st->k == iter_limit) {
      log_check(st->rP, 0, 0);
      st->status = LP_ITERATION_LIMIT; st->halt = 1; st->outsel = 1;
      return;
    }
    st->metric = st->rP;
    st->csel = 1;
    st->colsum[22] = t[4];
    st->colsum[23] = t[5];
  } else {
    const Kkt5 ka = kkt5(t + 0), kc = kkt5(t + 4);
    if (verbose_due(verbose, display_freq, st->k, check_freq))
      verbose_line(0, st->k, kc.pobj, kc.dobj, kc.pres, kc.dres, kc.gap, st->omega, st->eta);
    if (tpass(ka)) { log_check(0.0, 0, 1); st->status = LP_OPTIMAL; st->halt = 1; st->outsel = 1; return; }
    if (tpass(kc)) { log_check(0.0, 0, 2); st->status = LP_OPTIMAL; st->halt = 1; st->outsel = 0; return; }
    if (cert) {
      log_check(0.0, 0, 3);
      st->status = cert; st->halt = 1; st->outsel = 0; st->rays = 1; st->ray_ny = ny; st->ray_nx = nx;
      return;
    }
    if (st->k == iter_limit) {
      log_check(0.0, 0, 0);
      st->status = LP_ITERATION_LIMIT; st->halt = 1;
      st->outsel = kkt5_rel(ka, nq0, nc0) < kkt5_rel(kc, nq0, nc0) ? 1 : 0;
      return;
    }
    const Kkt5 sa = kkt5(t + 8), sc = kkt5(t + 12);
    const double e_a = kkt_omega(sa, st->omega, st->inv_omega);
    const double e_c = kkt_omega(sc, st->omega, st->inv_omega);
    if (restart_to_average(e_a, e_c)) { st->csel = 1; st->metric = e_a; st->colsum[22] = t[16]; st->colsum[23] = t[17]; }
    else { st->csel = 0; st->metric = e_c; st->colsum[22] = t[18]; st->colsum[23] = t[19]; }
  }
  const double metric = st->metric;
  const bool restart = restart_due(st->k_in, st->k, metric, st->ref, st->last);
  log_check(metric, restart ? 1 : 0, 0);
  st->last = metric;
  if (restart) {
    st->restart = 1;
    st->restarts += 1;
    st->omega = primal_weight(st->omega, sqrt(st->colsum[22]), sqrt(st->colsum[23]));
    st->inv_omega = 1.0 / st->omega;
    st->k_in = 0;
    if (!st->r2) { st->W = 0.0; st->ref = metric; }
  }
}

__global__ void k_restart(const ShState *st, int64_t j0, int64_t n, int64_t m, const Vecs V) {
  if (!st->restart) return;
  const bool r2 = st->r2, csel = st->csel;
  const int64_t gt = blockIdx.x * (int64_t)kB + threadIdx.x, s = (int64_t)gridDim.x * kB;
  for (int64_t j = j0 + gt; j < n; j += s) {
    double xv = V.x[j], kt = V.KTy[j];
    if (csel) { xv = r2 ? V.xp[j] : V.xa[j]; kt = r2 ? V.KTyp[j] : V.KTya[j]; }
    V.x[j] = xv; V.xr[j] = xv; V.xa[j] = xv; V.KTy[j] = kt; V.KTya[j] = kt;
  }
  for (int64_t i = gt; i < m; i += s) {
    double yv = V.y[i], kx = V.Kx[i];
    if (csel) { yv = r2 ? V.yp[i] : V.ya[i]; kx = r2 ? V.Kxp[i] : V.Kxa[i]; }
    V.y[i] = yv; V.yr[i] = yv; V.ya[i] = yv; V.Kx[i] = kx; V.Kxa[i] = kx;
  }
}

__global__ void k_final(const ShState *st, lp_result *res) {
  double t[4];
  for (int k = 0; k < 4; ++k) t[k] = st->colsum[k] + st->rowsum[k];
  const Kkt5 ko = kkt5(t);
  lp_result r;
  r.status = st->status; r.polish = 0;
  r.iterations = st->k; r.attempts = st->j; r.restarts = st->restarts;
  r.primal_objective = ko.pobj; r.dual_objective = ko.dobj;
  r.primal_residual = ko.pres; r.dual_residual = ko.dres; r.gap = ko.gap;
  r.rel_kkt = kkt5_rel(ko, st->nq0, st->nc0);
  r.omega = st->omega; r.eta = st->eta; r.solve_seconds = 0.0;
  *res = r;
}

// fixed-order reduction over p same-device shard buffers (virtual mode)
__global__ void k_vreduce(double *const *ptrs, int p, int64_t off, int64_t count, int op_max) {
  for (int64_t t = off + blockIdx.x * (int64_t)kB + threadIdx.x; t < off + count; t += (int64_t)gridDim.x * kB) {
    double a = ptrs[0][t];
    for (int s = 1; s < p; ++s) a = op_max ? fmax(a, ptrs[s][t]) : a + ptrs[s][t];
    for (int s = 0; s < p; ++s) ptrs[s][t] = a;
  }
}

__global__ void k_set_eta0(ShState *st, const double *kmax, const double *sigma, int r2, int cstep, double rho) {
  st->eta0 = initial_eta(kmax, sigma, cstep != 0);
  st->rho = rho;
  st->r2 = r2;
  st->cstep = cstep;
}

}  // namespace

// ------------------------------------------------------------------ engine --

struct ShardData {
  DevProblem P;
  int64_t row_offset = 0;   // row mode: first global row of the shard; column mode: first global column
  int64_t *rp64 = nullptr;
  Vecs V{};
  ShState *st = nullptr;
  double *X = nullptr, *Y = nullptr, *L = nullptr;
  void *arena = nullptr;
  void *vecs = nullptr;
  int nb = 0;
  double *pol = nullptr;   // feasibility polishing: x* (n), x_p (n), zeros (n), y* (m), zeros (m), 8 partials
  const double *c0 = nullptr, *q0 = nullptr;   // the shard's own costs (V.c0 / V.q0 swap to zeros while polishing)
  int64_t j0 = 0, j1 = 0;   // the n-side range this shard updates: all of [0, n) except under variant B
};

struct ShardedLP {
  cudaStream_t s = nullptr;
  int nranks = 1, rank = 0;
  bool virt = false;
  void *comm = nullptr;  // ncclComm_t (borrowed)
  int64_t n = 0, m_global = 0, m1_global = 0;
  std::vector<ShardData> sh;
  double **d_ptrs = nullptr;  // virtual mode: per-shard pointer tables (kSlots x 64)
  std::vector<std::vector<double *>> tab_cache;   // the pointers each slot's table holds (uploaded once)
  ShState *h_st = nullptr;
  lp_result *d_res = nullptr, *h_res = nullptr;
  int *d_flags = nullptr, *h_flags = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double *alog = nullptr, *clog = nullptr;   // decision log of the main solve (lp_set_decision_log)
  int64_t acap = 0, ccap = 0;
  bool solved = false;
  bool sigma_ready = false;  // sigma_max(K~) computed into every shard's P.sigma
  int polish_mode = 0;       // the running solve is a polishing sub-solve (reading 36): 1 primal, 2 dual
  bool cols = false;         // column-sharded (every m-long vector replicated) instead of row-sharded
  bool vb = false;           // this solve uses exchange variant B (row engine): n-side work on slices
  int64_t ns = 0;            // variant B: columns per slice, ceil(n / p) (p = shards or ranks)
  // chunked overlap of the K~_g'y partials with their all-reduce (variant A): chunk c's reduction
  // runs on the comm stream while the compute stream sums chunk c + 1
  int chunks = 1;
  cudaStream_t comm_s = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t join_ev = nullptr;
};

namespace {

int upload_table(ShardedLP &E, int slot, double *const *bufs_host) {
  double **tab = E.d_ptrs + slot * 64;
  std::vector<double *> want(bufs_host, bufs_host + E.sh.size());
  if (E.tab_cache.size() <= (size_t)slot) E.tab_cache.resize(slot + 1);
  if (E.tab_cache[slot] != want) {
    // never inside a graph capture: the copy would be recorded from this temporary host array
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    MPAX_CUDA(cudaStreamIsCapturing(E.s, &cap));
    if (cap != cudaStreamCaptureStatusNone) {
      set_error_detail("sharded pointer table uploaded during a graph capture");
      return LP_ERR_UNSUPPORTED;
    }
    MPAX_CUDA(cudaMemcpyAsync(tab, bufs_host, E.sh.size() * sizeof(double *), cudaMemcpyHostToDevice, E.s));
    E.tab_cache[slot] = want;
  }
  return LP_OK;
}

int reduce_across(ShardedLP &E, int slot, int64_t count, bool op_max, double *const *bufs_host, int64_t off = 0,
                  cudaStream_t st = nullptr) {
  if (!st) st = E.s;
  if (E.virt) {
    if (E.sh.size() < 2) return LP_OK;
    double **tab = E.d_ptrs + slot * 64;
    // the table is uploaded only when its pointers change: the attempt loop then issues no host
    // copies, so it can be captured into a CUDA graph (sharded_solve)
    if (int r = upload_table(E, slot, bufs_host)) return r;
    MPAX_LAUNCH(k_vreduce, blocks_for(count), kB, 0, st, tab, (int)E.sh.size(), off, count, op_max ? 1 : 0);
    MPAX_CHECK_LAUNCH();
    return LP_OK;
  }
  if (E.nranks <= 1) return LP_OK;
#ifdef MPAX_HAVE_NCCL
  ncclResult_t r = ncclAllReduce(bufs_host[0] + off, bufs_host[0] + off, (size_t)count, ncclDouble,
                                 op_max ? ncclMax : ncclSum, (ncclComm_t)E.comm, st);
  if (r != ncclSuccess) {
    set_error_detail(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    return LP_ERR_NCCL;
  }
  return LP_OK;
#else
  set_error_detail("built without NCCL");
  return LP_ERR_UNSUPPORTED;
#endif
}

#define STRY(x)              \
  do {                       \
    int r_ = (x);            \
    if (r_ != LP_OK) return r_; \
  } while (0)

int reduce_vec(ShardedLP &E, int slot, std::vector<double *> bufs, int64_t count, bool op_max) {
  return reduce_across(E, slot, count, op_max, bufs.data());
}

// the scalar partials of the sharded side: row sums (row mode) or column sums (column mode)
int reduce_rowsum(ShardedLP &E, int slot) {
  std::vector<double *> b;
  for (auto &d : E.sh) b.push_back(E.cols ? d.st->colsum : d.st->rowsum);
  STRY(reduce_vec(E, slot, b, 20, false));   // the 20 partials k_cols / k_rows write ([20..23]: decision scratch)
  if (!E.vb) return LP_OK;
  b.clear();   // variant B: the column side is sliced as well
  for (auto &d : E.sh) b.push_back(d.st->colsum);
  return reduce_vec(E, slot + 6, b, 20, false);
}

// Variant B collectives on n-long buffers padded to p x ns: the reduce-scatter leaves shard g
// the sum of its slice [g ns, (g + 1) ns) (virtual mode: the whole sum, of which only the slice
// is read); the all-gather copies every shard's slice into every other shard's buffer.
__global__ void k_vgather(double *const *ptrs, int p, int64_t ns) {
  for (int64_t t = blockIdx.x * (int64_t)kB + threadIdx.x; t < (int64_t)p * ns; t += (int64_t)gridDim.x * kB) {
    const int owner = (int)(t / ns);
    const double v = ptrs[owner][t];
    for (int q = 0; q < p; ++q)
      if (q != owner) ptrs[q][t] = v;
  }
}

int table_for(ShardedLP &E, int slot, std::vector<double *> &bufs) { return upload_table(E, slot, bufs.data()); }

int reduce_scatter_vec(ShardedLP &E, int slot, std::vector<double *> bufs) {
  if (E.virt) return reduce_vec(E, slot, bufs, (int64_t)E.sh.size() * E.ns, false);
  if (E.nranks <= 1) return LP_OK;
#ifdef MPAX_HAVE_NCCL
  ncclResult_t r = ncclReduceScatter(bufs[0], bufs[0] + (int64_t)E.rank * E.ns, (size_t)E.ns, ncclDouble, ncclSum,
                                     (ncclComm_t)E.comm, E.s);
  if (r != ncclSuccess) {
    set_error_detail(std::string("ncclReduceScatter: ") + ncclGetErrorString(r));
    return LP_ERR_NCCL;
  }
  return LP_OK;
#else
  return LP_ERR_UNSUPPORTED;
#endif
}

int allgather_vec(ShardedLP &E, int slot, std::vector<double *> bufs) {
  if (E.virt) {
    if (E.sh.size() < 2) return LP_OK;
    STRY(table_for(E, slot, bufs));
    MPAX_LAUNCH(k_vgather, blocks_for((int64_t)E.sh.size() * E.ns), kB, 0, E.s, E.d_ptrs + slot * 64,
                (int)E.sh.size(), E.ns);
    MPAX_CHECK_LAUNCH();
    return LP_OK;
  }
  if (E.nranks <= 1) return LP_OK;
#ifdef MPAX_HAVE_NCCL
  ncclResult_t r = ncclAllGather(bufs[0] + (int64_t)E.rank * E.ns, bufs[0], (size_t)E.ns, ncclDouble,
                                 (ncclComm_t)E.comm, E.s);
  if (r != ncclSuccess) {
    set_error_detail(std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return LP_ERR_NCCL;
  }
  return LP_OK;
#else
  return LP_ERR_UNSUPPORTED;
#endif
}

}  // namespace

// Build the shards: validate, transpose, cross-shard preconditioning, scaling.
int sharded_setup(ShardedLP &E, const std::vector<lp_problem_desc> &descs, const std::vector<int64_t> &offsets) {
  cudaStream_t s = E.s;
  const int p = (int)descs.size();
  E.sh.resize(p);
  MPAX_CUDA(cudaMallocAsync((void **)&E.d_ptrs, 32 * 64 * sizeof(double *), s));   // slots 0..31
  for (int g = 0; g < p; ++g) {
    const lp_problem_desc &d = descs[g];
    ShardData &S = E.sh[g];
    DevProblem &P = S.P;
    P.n = d.n; P.m1 = d.m1; P.m2 = d.m2; P.m = d.m1 + d.m2; P.nnz = d.nnz;
    S.row_offset = offsets[g];
    const int64_t n = P.n, m = P.m, nnz = P.nnz;
    size_t bytes = 0;
    auto al = [&](size_t b) { size_t o = bytes; bytes += (b + 255) & ~(size_t)255; return o; };
    const size_t o_rp64 = al((m + 1) * 8), o_rp = al((m + 1) * 4), o_ci = al(nnz * 4 + 4), o_kv0 = al(nnz * 8 + 8),
                 o_kv = al(nnz * 8 + 8), o_trp = al((n + 1) * 4), o_tci = al(nnz * 4 + 4), o_perm = al(nnz * 4 + 4),
                 o_tkv = al(nnz * 8 + 8), o_l0 = al(n * 8), o_u0 = al(n * 8), o_ls = al(n * 8), o_us = al(n * 8),
                 o_Dr = al(m * 8 + 8), o_Dc = al(n * 8), o_kmax = al(8), o_sigma = al(8), o_c0 = al(n * 8), o_q0 = al(m * 8 + 8),
                 o_st = al(sizeof(ShState)), o_flag = al(64);
    char *base = nullptr;
    MPAX_CUDA(cudaMallocAsync((void **)&base, bytes, s));
    S.arena = base;
    S.rp64 = (int64_t *)(base + o_rp64); P.rp = (int32_t *)(base + o_rp); P.ci = (int32_t *)(base + o_ci);
    P.kv0 = (double *)(base + o_kv0); P.kv = (double *)(base + o_kv); P.trp = (int32_t *)(base + o_trp);
    P.tci = (int32_t *)(base + o_tci); P.perm = (int32_t *)(base + o_perm); P.tkv = (double *)(base + o_tkv);
    P.l0 = (double *)(base + o_l0); P.u0 = (double *)(base + o_u0); P.ls = (double *)(base + o_ls);
    P.us = (double *)(base + o_us); P.Dr = (double *)(base + o_Dr); P.Dc = (double *)(base + o_Dc);
    P.kmax = (double *)(base + o_kmax);
    P.sigma = (double *)(base + o_sigma);
    double *c0 = (double *)(base + o_c0), *q0 = (double *)(base + o_q0);
    S.st = (ShState *)(base + o_st);
    int *flag = (int *)(base + o_flag);
    P.tab = const_cast<double *>(step_table(s));
    auto cp = [&](void *dst, const void *src, size_t b) -> int {
      if (b) MPAX_CUDA(cudaMemcpyAsync(dst, src, b, cudaMemcpyDefault, s));
      return LP_OK;
    };
    STRY(cp(S.rp64, d.row_ptr, (m + 1) * 8));
    STRY(cp(P.ci, d.col_idx, nnz * 4));
    STRY(cp(P.kv0, d.values, nnz * 8));
    STRY(cp(P.l0, d.l, n * 8));
    STRY(cp(P.u0, d.u, n * 8));
    STRY(cp(c0, d.c, n * 8));
    STRY(cp(q0, d.q, m * 8));
    MPAX_CUDA(cudaMemsetAsync(S.st, 0, sizeof(ShState), s));
    const int init[8] = {0, INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX, 0, 0, 0};
    memcpy(E.h_flags + 8 * g, init, sizeof(init));
    STRY(cp(flag, E.h_flags + 8 * g, sizeof(init)));
    STRY(setup_validate(P, S.rp64, c0, n, q0, m, s, flag));
    STRY(setup_transpose(P, S.rp64, s, flag));
    STRY(cp(E.h_flags + 8 * g, flag, 8 * sizeof(int)));
    // vectors
    double *vec = nullptr;
    S.nb = 148 * 8;
    // n-vectors padded by 64 (variant B slices of ceil(n / p) columns, p <= 64; pads stay zero) and
    // every vector on a 256-byte boundary
    const int64_t na = (n + 64 + 31) / 32 * 32, ma = ((m > 0 ? m : 1) + 31) / 32 * 32;
    const size_t nv = 12 * (size_t)na + 10 * (size_t)ma + (size_t)S.nb * kV;
    MPAX_CUDA(cudaMallocAsync((void **)&vec, nv * sizeof(double), s));
    MPAX_CUDA(cudaMemsetAsync(vec, 0, nv * sizeof(double), s));
    S.vecs = vec;
    Vecs &V = S.V;
    double *w = vec;
    V.x = w; w += na; V.KTy = w; w += na; V.xp = w; w += na; V.KTyp = w; w += na; V.xa = w; w += na;
    V.KTya = w; w += na; V.xr = w; w += na; V.cs = w; w += na; V.red = w; w += na;
    V.y = w; w += ma; V.Kx = w; w += ma; V.yp = w; w += ma; V.Kxp = w; w += ma; V.ya = w; w += ma;
    V.Kxa = w; w += ma; V.yr = w; w += ma; V.qs = w; w += ma;
    S.X = w; w += na; S.L = w; w += na; w += na; S.Y = w; w += ma;
    V.tmp = w; w += ma;
    V.part = w; w += (size_t)S.nb * kV;
    V.c0 = c0; V.q0 = q0;
    S.c0 = c0; S.q0 = q0;
    V.pre = E.cols ? V.tmp : nullptr;
  }
  MPAX_CUDA(cudaStreamSynchronize(s));
  for (int g = 0; g < p; ++g) {
    const int *f = E.h_flags + 8 * g;
    if (f[0] == 3) return LP_ERR_DIMENSION;
    if (f[0] == 2) return LP_ERR_NAN;
    if (f[0] == 1) return LP_ERR_CROSSED_BOUNDS;
    E.sh[g].P.max_row = f[5];   // longest row of K_g / of K_g' (setup_validate, setup_transpose)
    E.sh[g].P.max_col = f[6];
  }
  // preconditioning with column norms reduced across shards
  std::vector<double *> rho(p), gam(p);
  for (int g = 0; g < p; ++g) {
    MPAX_CUDA(cudaMallocAsync((void **)&rho[g], (size_t)(E.sh[g].P.m + 1) * sizeof(double), s));
    MPAX_CUDA(cudaMallocAsync((void **)&gam[g], (size_t)E.sh[g].P.n * sizeof(double), s));
    STRY(setup_precond_init(E.sh[g].P, s));
  }
  int *noflag = nullptr;
  MPAX_CUDA(cudaMallocAsync((void **)&noflag, sizeof(int), s));
  MPAX_CUDA(cudaMemsetAsync(noflag, 0, sizeof(int), s));
  for (int r = 0; r < 11; ++r) {
    for (int g = 0; g < p; ++g) STRY(setup_precond_norms(E.sh[g].P, rho[g], gam[g], r == 10, s, noflag));
    if (E.cols) STRY(reduce_vec(E, 1, rho, E.m_global, r < 10));   // row norms over every shard's columns
    else STRY(reduce_vec(E, 1, gam, E.n, r < 10));
    for (int g = 0; g < p; ++g) STRY(setup_precond_update(E.sh[g].P, rho[g], gam[g], s, noflag));
  }
  std::vector<double *> km(p);
  for (int g = 0; g < p; ++g) {
    STRY(setup_scale(E.sh[g].P, s, noflag));
    km[g] = E.sh[g].P.kmax;
  }
  STRY(reduce_vec(E, 2, km, 1, true));
  for (int g = 0; g < p; ++g) {
    MPAX_CUDA(cudaFreeAsync(rho[g], s));
    MPAX_CUDA(cudaFreeAsync(gam[g], s));
  }
  MPAX_CUDA(cudaFreeAsync(noflag, s));
  // column halves of each K~_g for the two-pass rows-side SpMV (grid_solver.cu grid_split_prepare):
  // the gather target is x' -- replicated in row mode (8n bytes at every p), this shard's
  // columns in column mode (8 n_local bytes: past the L2 knee only at small p)
  for (int g = 0; g < p; ++g) STRY(grid_split_prepare(E.sh[g].P, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  return LP_OK;
}

namespace {

// 1 = warp-tile mapping (short rows), else G lanes per row (G ~ mean length / 4)
inline int group_of(double avg, int mx) {
  if (tile_mapping_ok(avg, mx)) return 1;
  int g = 2;
  while (g * 2 <= avg / 4.0 && g < 32) g *= 2;
  return g;
}

// launch KERNEL<mode> (mode 0..6, the COLS_* / ROWS_* enums)
#define SH_MODE_LAUNCH(KERNEL, mode, ...)                                              \
  switch (mode) {                                                                      \
    case 0: MPAX_LAUNCH(KERNEL<0>, __VA_ARGS__); break;                                \
    case 1: MPAX_LAUNCH(KERNEL<1>, __VA_ARGS__); break;                                \
    case 2: MPAX_LAUNCH(KERNEL<2>, __VA_ARGS__); break;                                \
    case 3: MPAX_LAUNCH(KERNEL<3>, __VA_ARGS__); break;                                \
    case 4: MPAX_LAUNCH(KERNEL<4>, __VA_ARGS__); break;                                \
    case 5: MPAX_LAUNCH(KERNEL<5>, __VA_ARGS__); break;                                \
    default: MPAX_LAUNCH(KERNEL<6>, __VA_ARGS__); break;                               \
  }

// KERNEL<mode, lr> for the row-side kernels (lr: the matrix has long rows)
#define SH_ONE_LR(KERNEL, M, LRV, ...)                                                 \
  { auto kfn = KERNEL<M, LRV>; MPAX_LAUNCH(kfn, __VA_ARGS__); }
#define SH_MODE_LR(KERNEL, M, lr, ...)                                                 \
  if (lr) SH_ONE_LR(KERNEL, M, true, __VA_ARGS__) else SH_ONE_LR(KERNEL, M, false, __VA_ARGS__)
#define SH_MODE_LAUNCH_LR(KERNEL, mode, lr, ...)                                       \
  switch (mode) {                                                                      \
    case 0: SH_MODE_LR(KERNEL, 0, lr, __VA_ARGS__) break;                              \
    case 1: SH_MODE_LR(KERNEL, 1, lr, __VA_ARGS__) break;                              \
    case 2: SH_MODE_LR(KERNEL, 2, lr, __VA_ARGS__) break;                              \
    case 3: SH_MODE_LR(KERNEL, 3, lr, __VA_ARGS__) break;                              \
    case 4: SH_MODE_LR(KERNEL, 4, lr, __VA_ARGS__) break;                              \
    case 5: SH_MODE_LR(KERNEL, 5, lr, __VA_ARGS__) break;                              \
    default: SH_MODE_LR(KERNEL, 6, lr, __VA_ARGS__) break;                             \
  }
#define SH_LR(KERNEL, lr, ...)                                                         \
  if (lr) MPAX_LAUNCH(KERNEL<true>, __VA_ARGS__); else MPAX_LAUNCH(KERNEL<false>, __VA_ARGS__)
inline bool long_rows(int max_len) { return max_len < 0 || max_len >= kTileCH; }   // unknown: keep the path

int launch_cols(ShardedLP &E, int mode) {
  for (auto &S : E.sh) {
    SH_MODE_LAUNCH(k_cols, mode, blocks_for(S.j1 - S.j0), kB, 0, E.s, S.st, S.j0, S.j1, S.P, S.V);
  }
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}
int launch_rows(ShardedLP &E, int mode) {
  const bool spmv_mode = (mode == ROWS_STEP || mode == ROWS_AVG || mode == ROWS_INIT2);
  if (E.vb && spmv_mode) {   // variant B: the rows' SpMV gathers the full vector the slices updated
    std::vector<double *> bufs;
    for (auto &S : E.sh) bufs.push_back(mode == ROWS_AVG ? S.V.xa : (mode == ROWS_INIT2 ? S.V.x : S.V.xp));
    STRY(allgather_vec(E, mode == ROWS_AVG ? 10 : (mode == ROWS_INIT2 ? 11 : 12), bufs));
  }
  if (E.cols && spmv_mode) {
    // column mode: K~_{:,g} src_g (partial over this shard's columns) into V.pre, summed across
    // shards; k_rows then reads the sum (G = 1: one thread per row)
    std::vector<double *> bufs;
    for (auto &S : E.sh) {
      const int G = group_of(S.P.avg_row, S.P.max_row);
      const double *src = mode == ROWS_AVG ? S.V.xa : (mode == ROWS_INIT2 ? S.V.x : S.V.xp);
      const bool lr = long_rows(S.P.max_row);
      if (S.P.split_h > 0 && G == 1 && S.P.m > 0) {   // column halves (past the L2 knee): two passes
        SH_LR(k_rows_left, lr, blocks_for(S.P.m), kB, 0, E.s, S.st, S.P.m, S.P, src, S.V.tmp);
        SH_LR(k_rows_right_add, lr, blocks_for(S.P.m), kB, 0, E.s, S.st, S.P.m, S.P, src, S.V.tmp);
      } else {
        SH_LR(k_cols_spmv, lr, blocks_for(S.P.m * G), kB, 0, E.s, S.st, S.P.m, G, S.P.rp, S.P.ci, S.P.kv, src,
              S.V.tmp);
      }
      bufs.push_back(S.V.tmp);
    }
    MPAX_CHECK_LAUNCH();
    STRY(reduce_vec(E, 8, bufs, E.m_global, false));
    for (auto &S : E.sh)
      SH_MODE_LAUNCH_LR(k_rows, mode, long_rows(S.P.max_row), blocks_for(S.P.m), kB, 0, E.s, S.st, S.P.m, S.P.m1,
                        1, S.P, S.V);
    MPAX_CHECK_LAUNCH();
    return LP_OK;
  }
  for (auto &S : E.sh) {
    const int G = group_of(S.P.avg_row, S.P.max_row);
    const bool spmv = (mode == ROWS_STEP || mode == ROWS_AVG || mode == ROWS_INIT2);
    if (mode == ROWS_STEP && S.P.split_h > 0 && G == 1 && S.P.m > 0)
      SH_LR(k_rows_left, long_rows(S.P.max_row), blocks_for(S.P.m), kB, 0, E.s, S.st, S.P.m, S.P, S.V.xp,
            S.V.tmp);
    SH_MODE_LAUNCH_LR(k_rows, mode, long_rows(S.P.max_row), blocks_for(S.P.m * (spmv ? G : 1)), kB, 0, E.s, S.st,
                      S.P.m, S.P.m1, G, S.P, S.V);
  }
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}
// K~_g' src_g into red (every shard), then the cross-shard sum
int cols_spmv(ShardedLP &E, int which /*0: yp, 1: y, 2: ya*/) {
  const int pp = E.virt ? (int)E.sh.size() : E.nranks;
  if (E.chunks > 1 && !E.cols && !E.vb && pp > 1 && E.n >= 64 * E.chunks) {
    // chunked: rows [c0, c1) of every K~_g' summed on the compute stream, then all-reduced on the
    // comm stream while the next chunk is summed (same sums per element, in the same shard order)
    std::vector<double *> bufs;
    for (auto &S : E.sh) bufs.push_back(S.V.red);
    STRY(upload_table(E, 0, bufs.data()));
    const int64_t per = (E.n + E.chunks - 1) / E.chunks;
    for (int c = 0; c < E.chunks; ++c) {
      const int64_t c0 = c * per, c1 = std::min<int64_t>(E.n, c0 + per);
      if (c0 >= c1) break;
      for (auto &S : E.sh) {
        const int G = group_of(S.P.avg_col, S.P.max_col);
        const double *src = which == 0 ? S.V.yp : (which == 1 ? S.V.y : S.V.ya);
        SH_LR(k_cols_spmv, long_rows(S.P.max_col), blocks_for((c1 - c0) * G), kB, 0, E.s, S.st, c1 - c0, G,
              S.P.trp + c0, S.P.tci, S.P.tkv, src, S.V.red + c0);
      }
      MPAX_CHECK_LAUNCH();
      MPAX_CUDA(cudaEventRecord(E.chunk_ev[c], E.s));
      MPAX_CUDA(cudaStreamWaitEvent(E.comm_s, E.chunk_ev[c], 0));
      STRY(reduce_across(E, 0, c1 - c0, false, bufs.data(), c0, E.comm_s));
    }
    MPAX_CUDA(cudaEventRecord(E.join_ev, E.comm_s));
    MPAX_CUDA(cudaStreamWaitEvent(E.s, E.join_ev, 0));
    return LP_OK;
  }
  std::vector<double *> bufs;
  for (auto &S : E.sh) {
    const int G = group_of(S.P.avg_col, S.P.max_col);
    const double *src = which == 0 ? S.V.yp : (which == 1 ? S.V.y : S.V.ya);
    SH_LR(k_cols_spmv, long_rows(S.P.max_col), blocks_for(S.P.n * G), kB, 0, E.s, S.st, S.P.n, G, S.P.trp,
          S.P.tci, S.P.tkv, src, S.V.red);
    bufs.push_back(S.V.red);
  }
  MPAX_CHECK_LAUNCH();
  if (E.cols) return LP_OK;   // column mode: y' is replicated, the shard's K~'_g y' is complete
  if (E.vb) return reduce_scatter_vec(E, 0, bufs);   // variant B: each shard needs its slice only
  return reduce_vec(E, 0, bufs, E.n, false);
}

}  // namespace

namespace {

// sigma_max(K~) of the column-sharded K~ (power.cu): v_g holds this shard's columns of the
// unsharded start vector; u = sum_g K~_{:,g} v_g reduced across shards (m-long), w_g = K~_{:,g}' u
// local, ||w||^2 = sum_g ||w_g||^2 reduced across shards, v_g = w_g / ||w||.
int sharded_power_cols(ShardedLP &E) {
  cudaStream_t s = E.s;
  std::vector<PowerState> ps(E.sh.size());
  for (size_t g = 0; g < E.sh.size(); ++g)
    STRY(power_begin_cols(ps[g], E.sh[g].P.n, E.sh[g].P.m, E.sh[g].row_offset, s));
  auto normalise = [&](bool from_w, bool sigma) -> int {
    std::vector<double *> ss;
    for (size_t g = 0; g < E.sh.size(); ++g) {
      STRY(power_sumsq(ps[g], from_w ? ps[g].w : ps[g].v, s));
      ss.push_back(power_ss(ps[g]));
    }
    STRY(reduce_vec(E, 19, ss, 1, false));
    for (size_t g = 0; g < E.sh.size(); ++g)
      STRY(power_finish(ps[g], from_w ? ps[g].w : ps[g].v, sigma ? E.sh[g].P.sigma : nullptr, s));
    return LP_OK;
  };
  STRY(normalise(false, false));
  std::vector<double *> us;
  for (auto &p : ps) us.push_back(p.u);
  for (int t = 0; t < kPowerIters; ++t) {
    for (size_t g = 0; g < E.sh.size(); ++g) STRY(power_kv(E.sh[g].P, ps[g], s));
    STRY(reduce_vec(E, 18, us, E.sh[0].P.m, false));
    for (size_t g = 0; g < E.sh.size(); ++g) STRY(power_ktu(E.sh[g].P, ps[g], s));
    STRY(normalise(true, true));
  }
  for (auto &p : ps) STRY(power_end(p, s));
  E.sigma_ready = true;
  return LP_OK;
}

// sigma_max(K~) of the row-sharded K~ (power.cu): u_g = K~_g v on each shard's rows,
// w = sum_g K~_g' u_g reduced across shards, then the replicated normalisation.
int sharded_power(ShardedLP &E) {
  cudaStream_t s = E.s;
  if (E.cols) return sharded_power_cols(E);
  std::vector<PowerState> ps(E.sh.size());
  for (size_t g = 0; g < E.sh.size(); ++g) STRY(power_begin(ps[g], E.n, E.sh[g].P.m, s));
  std::vector<double *> ws;
  for (auto &p : ps) ws.push_back(p.w);
  for (int t = 0; t < kPowerIters; ++t) {
    for (size_t g = 0; g < E.sh.size(); ++g) STRY(power_products(E.sh[g].P, ps[g], s));
    STRY(reduce_vec(E, 4, ws, E.n, false));
    for (size_t g = 0; g < E.sh.size(); ++g) STRY(power_normalize(ps[g], E.sh[g].P.sigma, s));
  }
  for (auto &p : ps) STRY(power_end(p, s));
  E.sigma_ready = true;
  return LP_OK;
}

}  // namespace

int sharded_solve(ShardedLP &E, const lp_options &o, const double *X0, const double *Y0, lp_result *out) {
  cudaStream_t s = E.s;
  const bool r2 = o.algorithm == LP_R2HPDHG, cstep = o.step_rule == LP_STEP_CONSTANT;
  MPAX_CUDA(cudaEventRecord(E.ev0, s));
  if (cstep && !E.sigma_ready) STRY(sharded_power(E));
  // exchange variant (row engine): B slices the n-side work, A replicates it
  const int pp = E.virt ? (int)E.sh.size() : E.nranks;
  E.vb = !E.cols && o.sharded_exchange == 1 && pp > 1;
  E.ns = (E.n + pp - 1) / pp;
  for (size_t g = 0; g < E.sh.size(); ++g) {
    ShardData &S = E.sh[g];
    S.j0 = 0;
    S.j1 = S.P.n;
    if (E.vb) {
      const int64_t q = E.virt ? (int64_t)g : E.rank;
      S.j0 = std::min<int64_t>(E.n, q * E.ns);
      S.j1 = std::min<int64_t>(E.n, (q + 1) * E.ns);
    }
  }
  for (auto &S : E.sh) {
    MPAX_CUDA(cudaMemsetAsync(S.st, 0, sizeof(ShState), s));
    if (!E.cols) {
      S.V.X0 = X0;                                        // full n (replicated)
      S.V.Y0 = Y0 ? Y0 + S.row_offset : nullptr;          // virtual: the full m; a real rank: fixed below
    } else {
      S.V.X0 = X0 ? X0 + (E.virt ? S.row_offset : 0) : nullptr;   // this process's columns
      S.V.Y0 = Y0;                                        // full m (replicated)
    }
    MPAX_LAUNCH(k_set_eta0, 1, 1, 0, s, S.st, S.P.kmax, S.P.sigma, r2 ? 1 : 0, cstep ? 1 : 0, o.reflection);
  }
  if (!E.virt && !E.cols) for (auto &S : E.sh) S.V.Y0 = Y0;   // a real rank passes its own rows
  // ---- step 2 ----
  STRY(launch_cols(E, COLS_INIT));
  STRY(launch_rows(E, ROWS_INIT));
  STRY(reduce_rowsum(E, 3));
  for (auto &S : E.sh) MPAX_LAUNCH(k_init_decide, 1, 1, 0, s, S.st, 0);
  STRY(cols_spmv(E, 1));
  STRY(launch_cols(E, COLS_INIT2));
  STRY(launch_rows(E, ROWS_INIT2));
  STRY(reduce_rowsum(E, 3));
  for (auto &S : E.sh) MPAX_LAUNCH(k_init_decide, 1, 1, 0, s, S.st, 1);
  MPAX_CHECK_LAUNCH();
  // ---- attempts, checks ----
  const int64_t F = o.check_frequency, LIM = o.iteration_limit;
  auto attempts = [&](int64_t cnt) -> int {
    for (int64_t a = 0; a < cnt; ++a) {
      STRY(cols_spmv(E, 0));
      STRY(launch_cols(E, COLS_STEP));
      STRY(launch_rows(E, ROWS_STEP));
      STRY(reduce_rowsum(E, 3));
      for (size_t g = 0; g < E.sh.size(); ++g)
        MPAX_LAUNCH(k_decide, 1, 1, 0, s, E.sh[g].st, E.sh[g].P.tab, F, LIM, g == 0 ? E.alog : nullptr,
                    (int64_t)E.acap);
    }
    MPAX_CHECK_LAUNCH();
    return LP_OK;
  };
  if (E.vb && E.virt) {   // the x' all-gather's pointer table, before any capture of the attempt loop
    std::vector<double *> b;
    for (auto &S : E.sh) b.push_back(S.V.xp);
    STRY(table_for(E, 12, b));
  }
  // A chunk of F attempts that starts at a check boundary is replayed from a CUDA graph captured
  // once per solve (every kernel argument and collective buffer is fixed within a solve; the
  // virtual pointer tables were uploaded by step 2): one launch per F attempts instead of
  // F x (4 p + collectives).  Chunks after rejections (fewer than F attempts left) are enqueued
  // directly.  MPAX_SHARDED_GRAPH=0 switches the graph off; a failed capture falls back.
  const char *genv = getenv("MPAX_SHARDED_GRAPH");
  bool use_graph = !(genv && atoi(genv) == 0);
  struct GraphGuard {
    cudaGraphExec_t x = nullptr;
    ~GraphGuard() { if (x) cudaGraphExecDestroy(x); }
  } gexec;
  int64_t glaunches = 0;
  int64_t k = 0;
  for (;;) {
    int64_t next = ((k / F) + 1) * F;
    if (next > LIM) next = LIM;
    const int64_t chunk = next - k;
    if (use_graph && chunk == F) {
      if (!gexec.x) {
        // captured on a private stream (the handle's may be the legacy default stream, which
        // cannot capture); the graph is then launched on the handle's stream, in its order
        const int64_t c0 = g_launches.load();
        cudaGraph_t graph = nullptr;
        cudaStream_t cs = nullptr, s0 = s;
        int rc = LP_ERR_CUDA;
        cudaError_t ec = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        if (ec == cudaSuccess) ec = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (ec == cudaSuccess) {
          E.s = cs;
          s = cs;
          rc = attempts(F);
          ec = cudaStreamEndCapture(cs, &graph);
          E.s = s0;
          s = s0;
        }
        if (cs) cudaStreamDestroy(cs);
        glaunches = g_launches.load() - c0;   // launches recorded at capture: counted per replay
        g_launches.fetch_sub(glaunches);
        if (rc != LP_OK || ec != cudaSuccess || !graph || cudaGraphInstantiate(&gexec.x, graph, 0) != cudaSuccess) {
          gexec.x = nullptr;
          use_graph = false;
          (void)cudaGetLastError();
        }
        if (graph) cudaGraphDestroy(graph);
      }
      if (gexec.x) {
        MPAX_CUDA(cudaGraphLaunch(gexec.x, s));
        g_launches.fetch_add(glaunches);
      } else {
        STRY(attempts(chunk));
      }
    } else {
      STRY(attempts(chunk));
    }
    MPAX_CUDA(cudaMemcpyAsync(E.h_st, E.sh[0].st, sizeof(ShState), cudaMemcpyDeviceToHost, s));
    MPAX_CUDA(cudaStreamSynchronize(s));
    if (E.h_st->halt) break;
    k = E.h_st->k;
    if (k != next) continue;
    // check (step 5): commit-only; raPDHG: average products + every KKT partial
    STRY(cols_spmv(E, 0));
    STRY(launch_cols(E, COLS_COMMIT_ONLY));
    STRY(launch_rows(E, ROWS_COMMIT_ONLY));
    if (!r2) {
      STRY(launch_rows(E, ROWS_AVG));
      STRY(cols_spmv(E, 2));
      STRY(launch_cols(E, COLS_AVG));
    }
    STRY(reduce_rowsum(E, 3));
    // infeasibility certificate partials (reading 35): columns replicated, rows reduced
    STRY(launch_cols(E, COLS_CERT));
    STRY(launch_rows(E, ROWS_CERT));
    {
      std::vector<double *> sums, maxs;
      for (auto &S : E.sh) {
        double *c = E.cols ? S.st->certc : S.st->certr;   // the sharded side's certificate partials
        sums.push_back(c);
        maxs.push_back(c + 4);
      }
      STRY(reduce_vec(E, 5, sums, 4, false));
      STRY(reduce_vec(E, 6, maxs, 2, true));
      if (E.vb) {   // variant B: the column side is sliced too
        sums.clear();
        maxs.clear();
        for (auto &S : E.sh) { sums.push_back(S.st->certc); maxs.push_back(S.st->certc + 4); }
        STRY(reduce_vec(E, 16, sums, 4, false));
        STRY(reduce_vec(E, 17, maxs, 2, true));
      }
    }
    // verbose lines from one shard of rank 0 only (every shard takes the same decisions)
    for (size_t g = 0; g < E.sh.size(); ++g)
      MPAX_LAUNCH(k_check_decide, 1, 1, 0, s, E.sh[g].st, o.eps_abs, o.eps_rel, o.eps_primal_infeasible,
                  o.eps_dual_infeasible, LIM, (g == 0 && E.rank == 0) ? o.verbose : 0, o.display_frequency,
                  (int64_t)o.check_frequency, E.polish_mode, o.eps_feas_polish, g == 0 ? E.clog : nullptr,
                  (int64_t)E.ccap);
    for (auto &S : E.sh)
      MPAX_LAUNCH(k_restart, blocks_for(S.j1 - S.j0 > S.P.m ? S.j1 - S.j0 : S.P.m), kB, 0, s, S.st, S.j0, S.j1, S.P.m,
                  S.V);
    MPAX_CHECK_LAUNCH();
    MPAX_CUDA(cudaMemcpyAsync(E.h_st, E.sh[0].st, sizeof(ShState), cudaMemcpyDeviceToHost, s));
    MPAX_CUDA(cudaStreamSynchronize(s));
    if (E.h_st->halt) break;
  }
  // ---- step 6: output ----
  STRY(launch_cols(E, COLS_OUT));
  STRY(launch_rows(E, ROWS_OUT));
  STRY(reduce_rowsum(E, 3));
  if (E.vb) {   // variant B: the unscaled x and the reduced costs were written slice by slice
    std::vector<double *> xr, lr;
    for (auto &S : E.sh) { xr.push_back(S.V.red); lr.push_back(S.V.KTyp); }
    STRY(allgather_vec(E, 13, xr));
    STRY(allgather_vec(E, 14, lr));
  }
  MPAX_LAUNCH(k_final, 1, 1, 0, s, E.sh[0].st, E.d_res);
  MPAX_CHECK_LAUNCH();
  for (auto &S : E.sh) {
    MPAX_CUDA(cudaMemcpyAsync(S.X, S.V.red, S.P.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MPAX_CUDA(cudaMemcpyAsync(S.L, S.V.KTyp, S.P.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (S.P.m) MPAX_CUDA(cudaMemcpyAsync(S.Y, S.V.Kxp, S.P.m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  MPAX_CUDA(cudaEventRecord(E.ev1, s));
  MPAX_CUDA(cudaMemcpyAsync(E.h_res, E.d_res, sizeof(lp_result), cudaMemcpyDeviceToHost, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  float ms = 0.0f;
  MPAX_CUDA(cudaEventElapsedTime(&ms, E.ev0, E.ev1));
  *out = *E.h_res;
  out->solve_seconds = ms * 1e-3;
  E.solved = true;
  return LP_OK;
}

namespace {

// Feasibility polishing on a sharded LP (reading 36; the single-GPU path's polish_combine_kernel):
// per-shard partials of the combined point's objectives -- the n-side terms are replicated, so
// only the first shard of rank 0 contributes them; q'y and |q|^2 are summed across shards.
__global__ void k_polish_partials(int64_t n, int64_t m, const double *c0, const double *q0, const double *l0,
                                  const double *u0, const double *x, const double *lam, const double *y,
                                  int own_cols, int own_rows, double *out) {
  __shared__ double red[4][kB / 32];
  double v[4] = {0.0, 0.0, 0.0, 0.0};  // c'x + l/u dual terms split below: [c'x, dual obj, |c|^2, |q|^2]
  if (own_cols) {
    for (int64_t j = threadIdx.x; j < n; j += kB) {
      const double lm = lam[j], lp = fmax(lm, 0.0), ln = fmax(-lm, 0.0);
      v[0] += c0[j] * x[j];
      v[2] += c0[j] * c0[j];
      if (l0[j] > -INFINITY) v[1] += l0[j] * lp;
      if (u0[j] < INFINITY) v[1] -= u0[j] * ln;
    }
  }
  if (own_rows) {
    for (int64_t i = threadIdx.x; i < m; i += kB) {
      v[1] += q0[i] * y[i];
      v[3] += q0[i] * q0[i];
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < 4; ++k) {
    double t = v[k];
    for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(FULL, t, off);
    if (lane == 0) red[k][w] = t;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int ww = 0; ww < kB / 32; ++ww) t += red[threadIdx.x][ww];
    out[threadIdx.x] = t;
  }
}

__global__ void k_polish_final(const double *t, const lp_result *r1, const lp_result *r2, lp_result *res) {
  lp_result r = *res;
  const double pres = r1->primal_residual, dres = r2->dual_residual;
  const double nc = sqrt(t[2]), nq = sqrt(t[3]), gap = fabs(t[0] - t[1]);
  r.primal_objective = t[0]; r.dual_objective = t[1];
  r.primal_residual = pres; r.dual_residual = dres; r.gap = gap;
  r.rel_kkt = fmax(pres / (1.0 + nq), fmax(dres / (1.0 + nc), gap / (1.0 + fabs(t[0]) + fabs(t[1]))));
  r.iterations += r1->iterations + r2->iterations;
  r.attempts += r1->attempts + r2->attempts;
  r.restarts += r1->restarts + r2->restarts;
  r.polish = (r1->status == LP_OPTIMAL && r2->status == LP_OPTIMAL) ? 1 : 2;
  *res = r;
}

}  // namespace

// lp_solve on a sharded handle with feasibility polishing (reading 36): the main solve, then -- if
// it ended OPTIMAL -- a primal polish (c = 0 from (x*, 0)) and a dual polish (q = 0 from
// (proj 0, y*)) on the same sharded engine with residual-only tests, infeasibility detection off
// and at most min(iteration_limit, 100000) accepted steps each; x from the primal polish, y and
// the reduced costs from the dual polish, objectives recomputed on the original c, q, l, u.
int sharded_solve_polished(ShardedLP &E, const lp_options &o, const double *X0, const double *Y0, lp_result *out) {
  lp_options om = o;
  om.feasibility_polishing = 0;
  STRY(sharded_solve(E, om, X0, Y0, out));
  if (!o.feasibility_polishing || out->status != LP_OPTIMAL) return LP_OK;
  struct LogOff {   // the polishing sub-solves are not logged (lp.h)
    ShardedLP &E; double *a, *c;
    explicit LogOff(ShardedLP &e) : E(e), a(e.alog), c(e.clog) { E.alog = nullptr; E.clog = nullptr; }
    ~LogOff() { E.alog = a; E.clog = c; }
  } log_off(E);
  cudaStream_t s = E.s;
  const int64_t n = E.n;
  int64_t mtot = 0;
  for (auto &S : E.sh) mtot += S.P.m;
  for (auto &S : E.sh) {
    if (!S.pol) {
      const int64_t mm = S.P.m > 0 ? S.P.m : 1;
      MPAX_CUDA(cudaMallocAsync((void **)&S.pol, (size_t)(3 * n + 2 * mm + 8) * sizeof(double), s));
      MPAX_CUDA(cudaMemsetAsync(S.pol, 0, (size_t)(3 * n + 2 * mm + 8) * sizeof(double), s));
    }
  }
  // the main solve's (x*, y*) in sharded_solve's warm-start layout: the replicated side from the
  // first shard, the sharded side concatenated in this process's shard order
  int64_t ntot = 0;
  for (auto &S : E.sh) ntot += S.P.n;
  const int64_t nx = E.cols ? ntot : n, ny = E.cols ? E.sh[0].P.m : mtot;
  double *xstar = nullptr, *ystar = nullptr;
  lp_result *res_d = nullptr;
  MPAX_CUDA(cudaMallocAsync((void **)&xstar, (size_t)(nx > 0 ? nx : 1) * sizeof(double), s));
  MPAX_CUDA(cudaMallocAsync((void **)&ystar, (size_t)(ny > 0 ? ny : 1) * sizeof(double), s));
  MPAX_CUDA(cudaMallocAsync((void **)&res_d, 3 * sizeof(lp_result), s));
  MPAX_CUDA(cudaMemcpyAsync(res_d, E.d_res, sizeof(lp_result), cudaMemcpyDeviceToDevice, s));
  {
    int64_t ox = 0, oy = 0;
    for (size_t g = 0; g < E.sh.size(); ++g) {
      auto &S = E.sh[g];
      if (E.cols || g == 0) MPAX_CUDA(cudaMemcpyAsync(xstar + ox, S.X, S.P.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      if ((!E.cols || g == 0) && S.P.m)
        MPAX_CUDA(cudaMemcpyAsync(ystar + oy, S.Y, S.P.m * sizeof(double), cudaMemcpyDeviceToDevice, s));
      if (E.cols) ox += S.P.n; else oy += S.P.m;
    }
  }
  lp_options op = o;
  op.feasibility_polishing = 0;
  op.eps_primal_infeasible = -1.0;
  op.eps_dual_infeasible = -1.0;
  if (op.iteration_limit > 100000) op.iteration_limit = 100000;
  lp_result r1, r2;
  // primal polish: c = 0 (zeros at pol + 2n), from (x*, 0)
  for (auto &S : E.sh) S.V.c0 = S.pol + 2 * n;
  E.polish_mode = 1;
  int rc = sharded_solve(E, op, xstar, nullptr, &r1);
  for (auto &S : E.sh) S.V.c0 = S.c0;
  if (rc != LP_OK) { E.polish_mode = 0; return rc; }
  MPAX_CUDA(cudaMemcpyAsync(res_d + 1, E.d_res, sizeof(lp_result), cudaMemcpyDeviceToDevice, s));
  for (auto &S : E.sh) MPAX_CUDA(cudaMemcpyAsync(S.pol + n, S.X, S.P.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // dual polish: q = 0 (zeros at pol + 3n + m), from (proj 0, y*)
  for (auto &S : E.sh) S.V.q0 = S.pol + 3 * n + (S.P.m > 0 ? S.P.m : 1);
  E.polish_mode = 2;
  rc = sharded_solve(E, op, nullptr, ny > 0 ? ystar : nullptr, &r2);
  for (auto &S : E.sh) S.V.q0 = S.q0;
  E.polish_mode = 0;
  if (rc != LP_OK) return rc;
  MPAX_CUDA(cudaMemcpyAsync(res_d + 2, E.d_res, sizeof(lp_result), cudaMemcpyDeviceToDevice, s));
  // combine: X <- x_p; Y, L stay the dual polish's; objectives on the original data
  std::vector<double *> parts;
  for (size_t g = 0; g < E.sh.size(); ++g) {
    auto &S = E.sh[g];
    MPAX_CUDA(cudaMemcpyAsync(S.X, S.pol + n, S.P.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    double *pt = S.pol + 3 * n + 2 * (S.P.m > 0 ? S.P.m : 1);
    const int first = (g == 0 && E.rank == 0) ? 1 : 0;   // the replicated side is counted once
    if (E.vb)   // variant B: every shard sums its own slice of the n-side terms
      MPAX_LAUNCH(k_polish_partials, 1, kB, 0, s, S.j1 - S.j0, S.P.m, S.V.c0 + S.j0, S.V.q0, S.P.l0 + S.j0,
                  S.P.u0 + S.j0, S.X + S.j0, S.L + S.j0, S.Y, 1, 1, pt);
    else
      MPAX_LAUNCH(k_polish_partials, 1, kB, 0, s, S.P.n, S.P.m, S.V.c0, S.V.q0, S.P.l0, S.P.u0, S.X, S.L, S.Y,
                  E.cols ? 1 : first, E.cols ? first : 1, pt);
    parts.push_back(pt);
  }
  MPAX_CHECK_LAUNCH();
  STRY(reduce_vec(E, 7, parts, 4, false));
  MPAX_LAUNCH(k_polish_final, 1, 1, 0, s, parts[0], res_d + 1, res_d + 2, res_d);
  MPAX_CHECK_LAUNCH();
  MPAX_CUDA(cudaMemcpyAsync(E.d_res, res_d, sizeof(lp_result), cudaMemcpyDeviceToDevice, s));
  MPAX_CUDA(cudaMemcpyAsync(E.h_res, res_d, sizeof(lp_result), cudaMemcpyDeviceToHost, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  const double secs = out->solve_seconds + r1.solve_seconds + r2.solve_seconds;
  *out = *E.h_res;
  out->solve_seconds = secs;
  cudaFreeAsync(xstar, s);
  cudaFreeAsync(ystar, s);
  cudaFreeAsync(res_d, s);
  return LP_OK;
}

ShardedLP *sharded_new(cudaStream_t s) {
  ShardedLP *E = new ShardedLP();
  E->s = s;
  if (cudaMallocHost((void **)&E->h_st, sizeof(ShState)) != cudaSuccess ||
      cudaMallocHost((void **)&E->h_res, sizeof(lp_result)) != cudaSuccess ||
      cudaMallocHost((void **)&E->h_flags, 8 * 64 * sizeof(int)) != cudaSuccess ||
      cudaMallocAsync((void **)&E->d_res, sizeof(lp_result), s) != cudaSuccess ||
      cudaEventCreate(&E->ev0) != cudaSuccess || cudaEventCreate(&E->ev1) != cudaSuccess) {
    return E;  // caller checks h_st
  }
  // chunked exchange (variant A): MPAX_SHARDED_CHUNKS, default 4 chunks when ranks exchange
  if (const char *e = getenv("MPAX_SHARDED_CHUNKS")) E->chunks = std::max(1, std::min(16, atoi(e)));
  else E->chunks = -1;   // resolved at create: 4 with NCCL ranks, 1 otherwise
  if (cudaStreamCreateWithFlags(&E->comm_s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&E->join_ev, cudaEventDisableTiming) != cudaSuccess)
    return E;
  E->chunk_ev.resize(16);
  for (auto &ev : E->chunk_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  return E;
}

void sharded_free(ShardedLP *E) {
  if (!E) return;
  for (auto &S : E->sh) {
    if (S.arena) cudaFreeAsync(S.arena, E->s);
    if (S.vecs) cudaFreeAsync(S.vecs, E->s);
    if (S.P.split_mem) cudaFreeAsync(S.P.split_mem, E->s);
    if (S.pol) cudaFreeAsync(S.pol, E->s);
  }
  if (E->d_ptrs) cudaFreeAsync(E->d_ptrs, E->s);
  if (E->d_res) cudaFreeAsync(E->d_res, E->s);
  cudaStreamSynchronize(E->s);
  if (E->h_st) cudaFreeHost(E->h_st);
  if (E->h_res) cudaFreeHost(E->h_res);
  if (E->h_flags) cudaFreeHost(E->h_flags);
  if (E->ev0) cudaEventDestroy(E->ev0);
  if (E->ev1) cudaEventDestroy(E->ev1);
  for (auto ev : E->chunk_ev) if (ev) cudaEventDestroy(ev);
  if (E->join_ev) cudaEventDestroy(E->join_ev);
  if (E->comm_s) cudaStreamDestroy(E->comm_s);
  delete E;
}

int sharded_get(ShardedLP *E, double *x, double *y, double *rc) {
  if (!E->solved) return LP_ERR_NOT_SOLVED;
  cudaStream_t s = E->s;
  if (E->cols) {   // x, rc: this process's columns in shard order; y replicated
    int64_t off = 0;
    for (auto &S : E->sh) {
      if (x) MPAX_CUDA(cudaMemcpyAsync(x + off, S.X, S.P.n * sizeof(double), cudaMemcpyDefault, s));
      if (rc) MPAX_CUDA(cudaMemcpyAsync(rc + off, S.L, S.P.n * sizeof(double), cudaMemcpyDefault, s));
      off += S.P.n;
    }
    if (y && E->sh[0].P.m)
      MPAX_CUDA(cudaMemcpyAsync(y, E->sh[0].Y, E->sh[0].P.m * sizeof(double), cudaMemcpyDefault, s));
    MPAX_CUDA(cudaStreamSynchronize(s));
    return LP_OK;
  }
  if (x) MPAX_CUDA(cudaMemcpyAsync(x, E->sh[0].X, E->n * sizeof(double), cudaMemcpyDefault, s));
  if (rc) MPAX_CUDA(cudaMemcpyAsync(rc, E->sh[0].L, E->n * sizeof(double), cudaMemcpyDefault, s));
  if (y) {
    int64_t off = 0;
    for (auto &S : E->sh) {
      if (S.P.m) MPAX_CUDA(cudaMemcpyAsync(y + off, S.Y, S.P.m * sizeof(double), cudaMemcpyDefault, s));
      off += S.P.m;
    }
  }
  MPAX_CUDA(cudaStreamSynchronize(s));
  return LP_OK;
}

int64_t sharded_n(const ShardedLP *E) { return E->n; }
// this process's share: columns (column mode; all n in row mode) and rows (all m in column mode)
int64_t sharded_n_local(const ShardedLP *E) {
  if (!E->cols) return E->n;
  int64_t n = 0;
  for (auto &S : E->sh) n += S.P.n;
  return n;
}
int64_t sharded_m_local(const ShardedLP *E) {
  if (E->cols) return E->sh.empty() ? 0 : E->sh[0].P.m;
  int64_t m = 0;
  for (auto &S : E->sh) m += S.P.m;
  return m;
}

// Create: `descs` are this process's row shards (one per GPU rank, p for virtual mode).
void sharded_set_log(ShardedLP *E, double *alog, int64_t acap, double *clog, int64_t ccap) {
  E->alog = alog; E->acap = acap; E->clog = clog; E->ccap = ccap;
}

int sharded_create(ShardedLP *E, const std::vector<lp_problem_desc> &descs, const std::vector<int64_t> &offsets,
                   int64_t n, int64_t m1g, int64_t m2g, void *comm, int rank, int nranks, bool virt, bool cols) {
  E->n = n; E->m1_global = m1g; E->m_global = m1g + m2g;
  E->comm = comm; E->rank = rank; E->nranks = nranks; E->virt = virt; E->cols = cols;
  if (E->chunks < 0) E->chunks = (!virt && nranks > 1) ? 4 : 1;
  if (!E->h_st || !E->d_res) return LP_ERR_OUT_OF_MEMORY;
  return sharded_setup(*E, descs, offsets);
}

}  // namespace mpax

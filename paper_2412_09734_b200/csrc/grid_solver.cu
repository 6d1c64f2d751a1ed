// grid_solver.cu -- one LP spread over the whole GPU (SURVEY §8(a) rows a4-a10,
// configs C4/C5): a persistent cooperative kernel whose CTAs stay resident for
// the entire solve and meet at grid barriers, so no host round trip and no
// kernel launch happens per iteration ("the loop stays on device").
//
// One attempt = two fused phases and two grid barriers:
//   phase A (columns j of K~'):  [accepted last attempt]  K~'_j y'  (SpMV #2) and the
//       n-side commit (raPDHG: average + swap; r2HPDHG: Halpern reflection on x and
//       K~'y, Eq. (hrpdhg)), then the next primal step
//       x'_j = proj(x_j - tau (c~_j - (K~'y)_j)) (Eq. (pdhg)) and ||dx||^2.
//   phase B (rows i of K~):  [accepted] m-side commit, then K~_i x' (SpMV #1), the
//       dual step y'_i = proj(y_i + sigma (q~_i - 2 K~_i x' + (K~x)_i)), ||dy||^2 and
//       <dy, K~x' - K~x>.
//   Every CTA then sums the per-CTA partials in a fixed order and takes the
//   line-search decision redundantly: no extra barrier, no float atomics.
// Every check_frequency accepted steps a commit-only phase, the
// average's two SpMVs (raPDHG) fused with the original-space KKT partials, the
// restart test and primal-weight update, and an optional restart copy.
//
// Data layout: CSR of K~ and of K~' (int32 offsets/indices, fp64 values), all
// vectors fp64 SoA.  The matrices are streamed with evict-first loads; the
// gathered vector (x' in phase B, y' in phase A) uses the default policy so it
// can stay L2-resident.  Short rows (mean <= 48, as in C4/C5) use the warp-tile
// CSR-stream mapping (one warp per 32 consecutive rows, coalesced chunks, each lane
// sums and finishes its own row); long rows are summed by G lanes (butterfly), G from
// the mean row length.  Results are bitwise deterministic.
#include <cooperative_groups.h>

#include <stdlib.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mpax {

namespace {

constexpr int kNP = 26;      // max partial values per phase (raPDHG check: 20 KKT / distance + 6 certificate)
constexpr int kBS = 512;     // threads per CTA

// T: storage type of K~'s values and of every iterate vector (double; float for fp32 storage,
// DESIGN.md reading 39).  Arithmetic and reductions are fp64 in both: loads widen, stores round.
template <typename T>
struct GridParams {
  int64_t n, m, m1;
  const int32_t *rp, *ci, *trp, *tci;
  const T *kv, *tkv;
  const double *Dr, *Dc, *ls, *us, *l0, *u0, *c0, *q0, *X0, *Y0, *kmax, *sigma, *tab;
  T *lsw, *usw;                                   // float: l~, u~ rounded (the attempt's projection)
  T *cs, *qs;
  T *x, *KTy, *xp, *KTyp, *xa, *KTya, *xr;        // n-side
  T *y, *Kx, *yp, *Kxp, *ya, *Kxa, *yr;           // m-side
  double *part;                                   // gridDim.x x kNP
  double *tpart;                                  // 2 x blocks x ceil(tiles / blocks): per-tile partials
  // two-pass phase B over the column halves of K~ (split != 0): pass 1 parks K~_L x' in tmp
  const int32_t *rpL, *ciL, *rpR, *ciR;
  const T *kvL, *kvR;
  double *tmp;
  int32_t split;
  double *tpartA;                                 // ceil(n / 32): phase A's per-tile ||dx||^2 (global claims)
  unsigned long long *gctr;                       // global tile counter of phase A (monotonic)
  double eps_abs, eps_rel, eps_pi, eps_di, eps_fp, rho;
  int64_t iter_limit;
  int32_t check_freq, alg, gk, gkt, const_step, polish_mode, verbose, display_freq, vpol, tdist, dyn;
  int32_t lean;   // bit 0 / 1: phase A / B through the lean out-of-line sweeps (phase_tiles)
  int32_t lrA, lrB;   // K~' / K~ has a row of kTileCH entries or more (tile_row_dot's long-row test)
  double *X, *Y, *L;
  lp_result *res;
  // decision log (CTA 0, thread 0): per attempt (j, accepted, eta, eta_bar), per check
  // (k, metric, ref, last, restart, outcome) -- the oracle's ora_log records, same meaning
  double *alog, *clog;
  int64_t acap, ccap;
};


// KKT contributions of one row / one column (contract step 5), original or scaled space.

#ifdef MPAX_TRACE
// Phase timers (trace build only, MPAX_TRACE_BUILD=1): CTA 0 / the last CTA, thread 0.
__device__ __forceinline__ unsigned long long tnow() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TR(...) __VA_ARGS__
#else
#define TR(...)
#endif

__device__ __forceinline__ void st_evict_last(double *p, double v) {
  asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
               "st.global.L2::cache_hint.f64 [%0], %1, pol;\n\t}" :: "l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_evict_last(float *p, double v) {
  asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
               "st.global.L2::cache_hint.f32 [%0], %1, pol;\n\t}" :: "l"(p), "f"((float)v) : "memory");
}

// streamed (evict-first) loads of the matrices
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const float *p) { return (double)__ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t *p) { return __ldcs(p); }

// Sum of row r of a CSR matrix times x (all lanes of the row's group get the sum).
// G == 1: warp-tile CSR-stream (common.cuh tile_row_dot): the warp's 32 consecutive rows,
// one per lane, streamed coalesced; no idle lanes in the epilogue.
// G >= 2: G lanes per row, each taking its entries four at a time (index and value loads
// first, then the four gathers, then the FMAs) so that twelve loads are in flight per lane;
// two interleaved accumulators, butterfly over the group.  Fixed order: deterministic.
template <typename V, typename X>
__device__ __forceinline__ double row_dot(int64_t r, bool valid, int rows, int G, int gl,
                                          const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                          const V *__restrict__ v, const X *x, double *tbuf, bool lr = true) {
  // (the kernel body's own tile sweeps -- step 2, the checks, the experimental drivers -- keep the
  // serial per-lane sum: the full-chunk warp sum inlined here costs the whole kernel's register
  // allocation 7% at C4; the hot sweeps of long-row matrices run in phase_tiles<.., LR = true>)
  if (G == 1) return tile_row_dot<V, X, false>((int)r, valid, rows, rp, ci, v, x, tbuf, lr);
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
        c[k] = ok ? ld_stream(ci + q) : 0;
        w[k] = ok ? ld_stream(v + q) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) xv[k] = (p + k * G < e) ? (double)x[c[k]] : 0.0;
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

// MX: bit k set = value k is max-reduced (non-negative violations), else summed.
template <int V, unsigned MX = 0u>
__device__ __forceinline__ void block_partials(double (&v)[V], double *part, double (*s_red)[kNP]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    double s = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double o = __shfl_xor_sync(FULL, s, off);
      s = ((MX >> k) & 1u) ? fmax(s, o) : s + o;
    }
    if (lane == 0) s_red[wid][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < V) {
    const bool mx = (MX >> threadIdx.x) & 1u;
    double s = 0.0;
    for (int w = 0; w < kBS / 32; ++w) s = mx ? fmax(s, s_red[w][threadIdx.x]) : s + s_red[w][threadIdx.x];
    part[(int64_t)blockIdx.x * kNP + threadIdx.x] = s;
  }
}

// After a grid barrier: every CTA sums the per-CTA partials in the same fixed order
// (warp k reduces value k: lanes take CTAs b = lane + 32i into 4 interleaved
// accumulators, then a butterfly; identical code and data in every CTA).
template <int V, unsigned MX = 0u>
__device__ __forceinline__ void grid_totals(double (&t)[V], const double *part, double *s_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = (int)gridDim.x;
  for (int k = w; k < V; k += kBS / 32) {
    if ((MX >> k) & 1u) {  // max of non-negative partials
      double s = 0.0;
      for (int b = lane; b < nb; b += 32) s = fmax(s, __ldcg(part + (int64_t)b * kNP + k));
#pragma unroll
      for (int off = 16; off; off >>= 1) s = fmax(s, __shfl_xor_sync(FULL, s, off));
      if (lane == 0) s_tot[k] = s;
      continue;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = lane;
    for (; b + 96 < nb; b += 128) {
      a0 += __ldcg(part + (int64_t)b * kNP + k);
      a1 += __ldcg(part + (int64_t)(b + 32) * kNP + k);
      a2 += __ldcg(part + (int64_t)(b + 64) * kNP + k);
      a3 += __ldcg(part + (int64_t)(b + 96) * kNP + k);
    }
    for (; b < nb; b += 32) a0 += __ldcg(part + (int64_t)b * kNP + k);
    double s = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (lane == 0) s_tot[k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < V; ++k) t[k] = s_tot[k];
}

// ---- lean hot phases (warp-tile mapping) -------------------------------------------------
// The fused attempt's two SpMV sweeps run in out-of-line functions that read their pointers
// and scalars from a per-CTA context in shared memory right where they are used (volatile:
// not hoisted into registers).  Inlined into the kernel body, the sweeps shared the 64-register
// budget of 2 CTAs x 512 threads per SM with the whole solve's state and spilled in the tile
// loop (round 1: 648 B of stack per thread, ~1.2 GB of local-memory loads per C5 attempt,
// profiles/r01g_summary.md); here the tile loop owns the registers.
enum PhaseMode : int {
  kA_RA = 0,   // phase A, raPDHG, commit pending: average + swap, primal step
  kA_R2 = 1,   // phase A, r2HPDHG, commit pending: Halpern reflection, primal step
  kB_PARK = 2, // phase B pass 1: park K~_L x' (no epilogue)
  kB_RA = 3,   // phase B, raPDHG, commit pending: average + swap, dual step
  kB_R2 = 4,   // phase B, r2HPDHG, commit pending
  kB_NOP = 5,  // phase B, no pending commit (after a rejected attempt or a check)
};
template <typename T>
struct PhaseCtx {
  const int32_t *rp, *ci;
  const T *kv, *tgt;              // the sweep's matrix and gathered vector
  const double *add;              // + add[row] (two-pass phase B pass 2), or null
  double *park;                   // pass 1 output
  // epilogue vectors (meaning per mode, see phase_tiles)
  T *e0, *e1, *e2, *e3, *e4;
  const T *r0, *r1, *r2, *r3, *r4;
  double tau_sigma, theta, ha, hb, rf1, rf0;
  int rows, m1;
  double *tpart;                  // per-tile partials (2 per tile)
  int t0, kmax;                   // this CTA's tile range [t0, t0 + kmax) (contiguous slots)
  unsigned long long *gctr;       // non-null: claim tiles from this global counter (all CTAs)
  unsigned long long gbase;       //   counter value at the phase's start; tiles [0, kmax)
};

template <int MODE, typename T, bool LR>
__device__ __noinline__ void phase_tiles(const volatile PhaseCtx<T> *cx, int *s_ctr, double *tbuf) {
  const int lane = threadIdx.x & 31;
  const int rows = cx->rows, t0 = cx->t0, kmax = cx->kmax;
  unsigned long long *const gctr = cx->gctr;
  const unsigned long long gbase = cx->gbase;
  for (;;) {
    int kk = 0;
    if (lane == 0) kk = gctr ? (int)(atomicAdd(gctr, 1ull) - gbase) : atomicAdd(s_ctr, 1);
    kk = __shfl_sync(FULL, kk, 0);
    if (kk >= kmax) break;
    const int r = ((t0 + kk) << 5) + lane;
    const bool ok = r < rows;
    double c0 = 0.0, c1 = 0.0;
    if (MODE == kB_PARK) {
      const double sl = tile_row_dot<T, T, LR>(r, ok, rows, (const int32_t *)cx->rp, (const int32_t *)cx->ci,
                                               (const T *)cx->kv, (const T *)cx->tgt, tbuf);
      if (ok) cx->park[r] = sl;
      continue;
    }
    double s = tile_row_dot<T, T, LR>(r, ok, rows, (const int32_t *)cx->rp, (const int32_t *)cx->ci,
                                      (const T *)cx->kv, (const T *)cx->tgt, tbuf);
    if (ok) {
      if (MODE == kA_RA) {
        // r0 = xp, r1 = cs, r2 = ls, r3 = us; e0 = xa (rw), e1 = KTy' (w), e2 = the old x buffer (w: x')
        const double o_xp = cx->r0[r], o_xa = cx->e0[r];
        cx->e0[r] = o_xa + cx->theta * (o_xp - o_xa);
        cx->e1[r] = s;
        const double xnew = median3((double)cx->r2[r], o_xp - cx->tau_sigma * ((double)cx->r1[r] - s), (double)cx->r3[r]);
        cx->e2[r] = xnew;
        const double d = xnew - o_xp;
        c0 = d * d;
      } else if (MODE == kA_R2) {
        // r0 = xp, r1 = cs, r2 = ls, r3 = us, r4 = KTya, e0 = xa (r), e1 = x (rw), e2 = KTy (rw), e3 = x' (w)
        const double xn = cx->ha * (cx->rf1 * (double)cx->r0[r] - cx->rf0 * (double)cx->e1[r]) + cx->hb * (double)cx->e0[r];
        const double kt = cx->ha * (cx->rf1 * s - cx->rf0 * (double)cx->e2[r]) + cx->hb * (double)cx->r4[r];
        cx->e1[r] = xn;
        cx->e2[r] = kt;
        const double xnew = median3((double)cx->r2[r], xn - cx->tau_sigma * ((double)cx->r1[r] - kt), (double)cx->r3[r]);
        cx->e3[r] = xnew;
        const double d = xnew - xn;
        c0 = d * d;
      } else {
        if (cx->add) s += cx->add[r];
        double yv, kxv;
        if (MODE == kB_RA) {
          // r0 = qs, r1 = yp, r2 = Kxp; e0 = ya (rw), e1 = the old y buffer (w: y'), e2 = the old Kx buffer (w)
          yv = cx->r1[r];
          kxv = cx->r2[r];
          const double o_ya = cx->e0[r];
          cx->e0[r] = o_ya + cx->theta * (yv - o_ya);
        } else if (MODE == kB_R2) {
          // r0 = qs, r1 = yp, r2 = Kxp, r3 = ya, r4 = Kxa; e0 = y (rw), e1 = Kx (rw), e2 = y' (w), e3 = K~x' (w)
          yv = cx->ha * (cx->rf1 * (double)cx->r1[r] - cx->rf0 * (double)cx->e0[r]) + cx->hb * (double)cx->r3[r];
          kxv = cx->ha * (cx->rf1 * (double)cx->r2[r] - cx->rf0 * (double)cx->e1[r]) + cx->hb * (double)cx->r4[r];
          cx->e0[r] = yv;
          cx->e1[r] = kxv;
        } else {
          // r0 = qs, r1 = y, r2 = Kx; e2 = y' (w), e3 = K~x' (w)
          yv = cx->r1[r];
          kxv = cx->r2[r];
        }
        double yn = yv + cx->tau_sigma * ((double)cx->r0[r] - 2.0 * s + kxv);
        if (r < cx->m1) yn = pos_part(yn);
        if (MODE == kB_RA) { cx->e1[r] = yn; cx->e2[r] = s; }
        else { cx->e2[r] = yn; cx->e3[r] = s; }
        const double d = yn - yv;
        c0 = d * d;
        c1 = d * (s - kxv);
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      c0 += __shfl_xor_sync(FULL, c0, off);
      c1 += __shfl_xor_sync(FULL, c1, off);
    }
    if (lane == 0) {
      cx->tpart[(size_t)(t0 + kk) * 2] = c0;
      cx->tpart[(size_t)(t0 + kk) * 2 + 1] = c1;
    }
  }
}

template <int MINB, typename T>
__global__ void __launch_bounds__(kBS, MINB) grid_kernel(GridParams<T> P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_red[kBS / 32][kNP];
  __shared__ double s_tot[kNP];
  __shared__ double s_tile[kBS / 32][kTileBuf];   // per-warp product buffer of the G == 1 mapping
  __shared__ int s_ctr;                             // tile counter of tiles_dynamic
  __shared__ PhaseCtx<T> s_cx;                      // context of the lean hot phases (phase_tiles)
  double *const tbuf = s_tile[threadIdx.x >> 5];
  // L2 policy of the attempt's vector traffic (P.vpol): 0 = default; 1 = every
  // vector access except the stores of the next gather target (x', y') is evict-first, so the
  // target stays L2-resident for the next phase's SpMV; 2 = 1 + those stores evict-last.
  const int vpol = P.vpol, tdist = P.tdist, dyn = P.dyn;
  auto lv = [vpol](const auto *p) -> double { return vpol ? (double)__ldcs(p) : (double)*p; };
  auto sv = [vpol](T *p, double v) { if (vpol) __stcs(p, (T)v); else *p = (T)v; };
  auto st_tgt = [vpol](T *p, double v) { if (vpol == 2) st_evict_last(p, v); else *p = (T)v; };
  // Hot-loop driver of the warp-tile mapping (G == 1): CTA b owns the contiguous tiles
  // [b T, (b + 1) T) of 32 rows; its warps claim them dynamically from a shared counter, so
  // early warps take more tiles instead of idling at the CTA barrier (the static mapping
  // left 30% of phase B's warp samples waiting there, ncu C5).  Each tile's V contributions
  // are summed over its lanes (butterfly) into P.tpart[tile], and the CTA sums its tiles in
  // tile order: the result does not depend on which warp took which tile (deterministic).
  // On return, thread 0 holds the CTA totals in tot[] and every other thread zeros.
  auto tiles_dynamic = [&](int rows, auto &&body, auto &tot, bool reduce) {
    constexpr int V = sizeof(tot) / sizeof(double);
    const int ntiles = (rows + 31) >> 5;
    const int nb = (int)gridDim.x, per = (ntiles + nb - 1) / nb;
    // k-th tile of this CTA: contiguous range (tdist 0) or interleaved over the CTAs (tdist 1)
    const int kmax = tdist ? (ntiles - (int)blockIdx.x + nb - 1) / nb : max(0, min(ntiles, ((int)blockIdx.x + 1) * per) - (int)blockIdx.x * per);
    const int t0 = (int)blockIdx.x * per, t1 = t0 + kmax;   // this CTA's slots in P.tpart
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_ctr = 0;
    __syncthreads();
    for (;;) {
      int kk = 0;
      if (lane == 0) kk = atomicAdd(&s_ctr, 1);
      kk = __shfl_sync(FULL, kk, 0);
      if (kk >= kmax) break;
      const int t = tdist ? (int)blockIdx.x + kk * nb : t0 + kk;
      const int r = (t << 5) + lane;
      double c[V];
      body(r, r < rows, c);
      if (!reduce) continue;
#pragma unroll
      for (int k = 0; k < V; ++k) {
#pragma unroll
        for (int off = 16; off; off >>= 1) c[k] += __shfl_xor_sync(FULL, c[k], off);
        if (lane == 0) P.tpart[(size_t)(t0 + kk) * 2 + k] = c[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < V; ++k) tot[k] = 0.0;
    if (reduce && threadIdx.x < 32) {
      double a[V];
#pragma unroll
      for (int k = 0; k < V; ++k) a[k] = 0.0;
      for (int t = t0 + lane; t < t1; t += 32)
#pragma unroll
        for (int k = 0; k < V; ++k) a[k] += __ldcg(P.tpart + (size_t)t * 2 + k);
#pragma unroll
      for (int k = 0; k < V; ++k) {
#pragma unroll
        for (int off = 16; off; off >>= 1) a[k] += __shfl_xor_sync(FULL, a[k], off);
        if (threadIdx.x == 0) tot[k] = a[k];
      }
    }
  };
  // Lean phase driver: thread 0 writes the context (fill), the CTA runs phase_tiles<MODE> over its
  // contiguous tile range with dynamic claims, then (reduce) warp 0 sums the tile partials in tile
  // order: on return thread 0 holds the CTA totals in tot[0..1], every other thread zeros.
  auto lean_range = [&](int rows) {
    const int ntiles = (rows + 31) >> 5, nb = (int)gridDim.x, per = (ntiles + nb - 1) / nb;
    const int t0 = (int)blockIdx.x * per;
    s_cx.rows = rows;
    s_cx.t0 = t0;
    s_cx.kmax = max(0, min(ntiles, t0 + per) - t0);
    s_cx.tpart = P.tpart;
    s_ctr = 0;
  };
  auto lean_reduce = [&](double (&tot)[2]) {
    tot[0] = 0.0; tot[1] = 0.0;
    if (threadIdx.x < 32) {
      const int t0 = s_cx.t0, t1 = t0 + s_cx.kmax;
      double a0 = 0.0, a1 = 0.0;
      for (int t = t0 + (int)threadIdx.x; t < t1; t += 32) {
        a0 += __ldcg(P.tpart + (size_t)t * 2);
        a1 += __ldcg(P.tpart + (size_t)t * 2 + 1);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        a0 += __shfl_xor_sync(FULL, a0, off);
        a1 += __shfl_xor_sync(FULL, a1, off);
      }
      if (threadIdx.x == 0) { tot[0] = a0; tot[1] = a1; }
    }
  };
  const bool leanA = P.lean & 1, leanB = P.lean & 2;
  const int n = (int)P.n, m = (int)P.m, m1 = (int)P.m1;  // < 2^31 (lp_create checks)
  const int gtid = blockIdx.x * kBS + threadIdx.x, gthreads = gridDim.x * kBS;
  const bool r2 = (P.alg == LP_R2HPDHG);
  // SpMV group mapping (fixed for the whole solve, so every row / column has one owner group)
  const int G = P.gk, Gt = P.gkt;
  const int grp = gtid / G, ngrp = gthreads / G;
  const int gl = (int)(gtid % G);
  const int grpt = gtid / Gt, ngrpt = gthreads / Gt;
  const int glt = (int)(gtid % Gt);
  const int row_iters = (m + ngrp - 1) / ngrp, col_iters = (n + ngrpt - 1) / ngrpt;
  T *x = P.x, *KTy = P.KTy, *xp = P.xp, *KTyp = P.KTyp, *xa = P.xa, *KTya = P.KTya, *xr = P.xr;
  T *y = P.y, *Kx = P.Kx, *yp = P.yp, *Kxp = P.Kxp, *ya = P.ya, *Kxa = P.Kxa, *yr = P.yr;
  const T *cs = P.cs, *qs = P.qs;
  // the attempt's bounds: l~, u~ themselves (fp64), or their fp32 copies (written below)
  const T *lsT, *usT;
  if constexpr (sizeof(T) == sizeof(double)) { lsT = (const T *)P.ls; usT = (const T *)P.us; }
  else { lsT = P.lsw; usT = P.usw; }
  // Per-CTA partials are double-buffered: reduction r writes buffer r % 2, so a CTA that has
  // moved on can never overwrite partials a slower CTA is still summing (that would let CTAs
  // take different decisions and then wait at different grid barriers).
  int pbuf = 1;
  auto next_part = [&]() { pbuf ^= 1; return P.part + (size_t)pbuf * gridDim.x * kNP; };
  auto cur_part = [&]() { return (const double *)(P.part + (size_t)pbuf * gridDim.x * kNP); };

  // ---------------- step 2: initialise ----------------
  {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = gtid; j < n; j += gthreads) {
      const double dc = P.Dc[j], c = P.c0[j], cj = c * dc;
      P.cs[j] = (T)cj;
      v[0] += cj * cj;
      v[2] += c * c;
      x[j] = (T)median3(P.ls[j], P.X0 ? P.X0[j] / dc : 0.0, P.us[j]);
      if constexpr (sizeof(T) != sizeof(double)) { P.lsw[j] = (T)P.ls[j]; P.usw[j] = (T)P.us[j]; }
    }
    for (int i = gtid; i < m; i += gthreads) {
      const double dr = P.Dr[i], q = P.q0[i], qi = q * dr;
      P.qs[i] = (T)qi;
      v[1] += qi * qi;
      v[3] += q * q;
      double yv = P.Y0 ? P.Y0[i] / dr : 0.0;
      if (i < m1) yv = fmax(yv, 0.0);
      y[i] = (T)yv;
    }
    block_partials<4>(v, next_part(), s_red);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.gctr = 0ull;   // before the first grid barrier
  }
  grid.sync();
  double tot4[4];
  grid_totals<4>(tot4, cur_part(), s_tot);
  const double nc0 = sqrt(tot4[2]), nq0 = sqrt(tot4[3]);
  double omega = 1.0;
  if (sqrt(tot4[0]) > 1e-10 && sqrt(tot4[1]) > 1e-10) omega = sqrt(tot4[0]) / sqrt(tot4[1]);
  double inv_omega = 1.0 / omega;  // every x / omega is x * omega^-1 (reading 32)
  const bool cstep = P.const_step != 0;  // constant step rule (reading 34)
  double eta = initial_eta(P.kmax, P.sigma, cstep);
  // r2HPDHG reflection z <- a((1 + rho) w - rho z) + b z0 (rho = 1: 2 PDHG(z) - z; reading 38)
  const double rf1 = 1.0 + P.rho, rf0 = P.rho;
  // the check's pass test: relative KKT, or a polishing sub-solve's single residual (reading 36)
  auto tpass = [&](const Kkt5 &k, double nq, double nc) {
    return P.polish_mode ? polish_pass(P.polish_mode, k.pres, k.dres, nq, nc, P.eps_fp)
                         : kkt5_pass(k, nq, nc, P.eps_abs, P.eps_rel);
  };
  {
    // K~x0, K~'y0; anchors / restart point; KKT_omega(z0) partials (scaled space)
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int it = 0; it < row_iters; ++it) {
      const int i = it * ngrp + grp;
      const bool ok = i < m;
      const double s = row_dot(i, ok, m, G, gl, P.rp, P.ci, P.kv, x, tbuf, P.lrB);
      if (ok && gl == 0) {
        Kx[i] = (T)s; Kxa[i] = (T)s;
        const double yv = y[i];
        ya[i] = (T)yv; yr[i] = (T)yv;
        kkt_row_acc(v, false, i < m1, 1.0, yv, s, 0.0, qs[i]);
      }
    }
    for (int it = 0; it < col_iters; ++it) {
      const int j = it * ngrpt + grpt;
      const bool ok = j < n;
      const double s = row_dot(j, ok, n, Gt, glt, P.trp, P.tci, P.tkv, y, tbuf, P.lrA);
      if (ok && glt == 0) {
        KTy[j] = (T)s; KTya[j] = (T)s;
        const double xv = x[j];
        xa[j] = (T)xv; xr[j] = (T)xv;
        kkt_col_acc(v, false, 1.0, xv, s, 0.0, (double)cs[j], 0.0, (double)lsT[j], 0.0, (double)usT[j]);
      }
    }
    block_partials<4>(v, next_part(), s_red);
  }
  grid.sync();
  int64_t k = 0, jatt = 0, k_in = 0, restarts = 0;
  double W = 0.0, last = INFINITY, ref = 0.0;
  {
    double t[4];
    grid_totals<4>(t, cur_part(), s_tot);
    if (!r2) {
      const Kkt5 ks = kkt5(t);
      ref = kkt_omega(ks, omega, inv_omega);
    }
  }

  int status = 0;
  bool pending = false;        // an accepted attempt whose commit is fused into the next phases
  double theta = 0.0, ha = 0.0, hb = 0.0;  // raPDHG average weight / r2HPDHG Halpern coefficients
  int rejects = 0;
  // returned candidate (pointers)
  const T *ox = x, *oy = y, *oKx = Kx, *oKTy = KTy;
  bool done = false;
  // infeasibility (reading 35): t = reduced (|dy|^2, |dx|^2, dual-ray obj, c'dx, viol_y, viol_x);
  // on a certificate the status is set and the output writes the rays against (bx, by, bKTy)
  const T *bx = nullptr, *by = nullptr, *bKTy = nullptr;
  double ray_ny = 1.0, ray_nx = 1.0;
  auto certify = [&](const double *t, const T *xb, const T *yb, const T *KTyb) {
    CertAcc tot;
    tot.sy = t[0]; tot.sx = t[1]; tot.oy = t[2]; tot.ox = t[3]; tot.vy = t[4]; tot.vx = t[5];
    const int st = cert_decide(tot, P.eps_pi, P.eps_di, ray_ny, ray_nx);
    if (!st) return false;
    status = st; ox = x; oy = y; oKx = Kx; oKTy = KTy;
    bx = xb; by = yb; bKTy = KTyb;
    return true;
  };

  int64_t nchk = 0;   // checks logged
  auto log_check = [&](double metric_, int restart_, int outcome) {
    if (P.clog && blockIdx.x == 0 && threadIdx.x == 0 && nchk < P.ccap) {
      double *r = P.clog + 6 * nchk;
      r[0] = (double)k; r[1] = metric_; r[2] = ref; r[3] = last; r[4] = restart_; r[5] = outcome;
    }
    ++nchk;
  };
  unsigned long long gbase = 0;   // phase A's global tile counter value at this phase's start
  bool sliceA = false;            // phase A used global claims: reduce this CTA's slice in phase B
  bool sliceA2 = false;           // the same for the lean sweep (partials in P.tpart, stride 2)
  TR(unsigned long long tr_a = 0, tr_aw = 0, tr_b = 0, tr_bw = 0, tr_chk = 0, tr_n = 0, tr_t0 = 0, tr_t1 = 0);
  TR(const bool tr_on = threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1));
  while (!done) {
    TR(if (tr_on) tr_t0 = tnow());
    // ================= phase A: [commit n-side] + primal step =================
    const double tau = eta * inv_omega, sigma = eta * omega;
    double v3[3] = {0.0, 0.0, 0.0};
    if (pending) {
      // one column j of phase A; returns its ||dx||^2 term
      auto colA = [&](int j, bool ok, bool lead) -> double {
        // operands of the epilogue, loaded before the dot so they are in flight with it
        double o_xp = 0.0, o_xa = 0.0, o_x = 0.0, o_kt = 0.0, o_kta = 0.0, o_cs = 0.0, o_ls = 0.0, o_us = 0.0;
        if (lead) {
          o_xp = lv(xp + j); o_xa = lv(xa + j); o_cs = lv(cs + j); o_ls = lv(lsT + j); o_us = lv(usT + j);
          if (r2) { o_x = lv(x + j); o_kt = lv(KTy + j); o_kta = lv(KTya + j); }
        }
        const double s = row_dot(j, ok, n, Gt, glt, P.trp, P.tci, P.tkv, yp, tbuf, P.lrA);
        if (!lead) return 0.0;
        double xn, kt;
        if (!r2) {
          sv(xa + j, o_xa + theta * (o_xp - o_xa));
          xn = o_xp; kt = s;
          sv(KTyp + j, s);       // becomes KTy after the pointer swap
        } else {
          xn = ha * (rf1 * o_xp - rf0 * o_x) + hb * o_xa;
          kt = ha * (rf1 * s - rf0 * o_kt) + hb * o_kta;
          sv(x + j, xn); sv(KTy + j, kt);
        }
        const double xnew = median3(o_ls, xn - tau * (o_cs - kt), o_us);
        st_tgt(r2 ? xp + j : x + j, xnew);   // ra: the old-x buffer becomes x' after the swap
        const double d = xnew - xn;
        return d * d;
      };
      if (Gt == 1 && leanA) {
        const bool glob = P.lean & 4;   // claims from one global counter (no inter-CTA tail at the barrier)
        if (threadIdx.x == 0) {
          lean_range(n);
          s_cx.gctr = nullptr;
          if (glob) { s_cx.gctr = P.gctr; s_cx.gbase = gbase; s_cx.t0 = 0; s_cx.kmax = (n + 31) >> 5; s_cx.tpart = P.tpartA; }
          s_cx.rp = P.trp; s_cx.ci = P.tci; s_cx.kv = P.tkv; s_cx.tgt = yp; s_cx.add = nullptr;
          s_cx.r0 = xp; s_cx.r1 = cs; s_cx.r2 = lsT; s_cx.r3 = usT; s_cx.r4 = KTya;
          s_cx.e0 = xa;
          if (!r2) { s_cx.e1 = KTyp; s_cx.e2 = x; }
          else { s_cx.e1 = x; s_cx.e2 = KTy; s_cx.e3 = xp; }
          s_cx.tau_sigma = tau; s_cx.theta = theta; s_cx.ha = ha; s_cx.hb = hb; s_cx.rf1 = rf1; s_cx.rf0 = rf0;
        }
        __syncthreads();
        if (!r2) { if (P.lrA) phase_tiles<kA_RA, T, true>(&s_cx, &s_ctr, tbuf); else phase_tiles<kA_RA, T, false>(&s_cx, &s_ctr, tbuf); }
        else { if (P.lrA) phase_tiles<kA_R2, T, true>(&s_cx, &s_ctr, tbuf); else phase_tiles<kA_R2, T, false>(&s_cx, &s_ctr, tbuf); }
        __syncthreads();
        if (glob) {
          // every warp made exactly one failing claim: the phase consumed tiles + warps values;
          // this CTA's fixed slice of the tile partials is summed in tile order after the barrier
          gbase += (unsigned long long)((n + 31) >> 5) + (unsigned long long)gridDim.x * (kBS / 32);
          sliceA2 = true;
          v3[0] = 0.0;
        } else {
          double t2[2];
          lean_reduce(t2);
          v3[0] = t2[0];
        }
      } else if (Gt == 1 && (dyn & 4)) {
        // global dynamic claims: warps of every CTA take column tiles from one monotonic counter,
        // so CTAs that run ahead take more tiles (no inter-CTA tail at the barrier).  Every warp
        // makes exactly one failing claim per phase, so each phase consumes ntiles + all warps
        // counter values and every CTA advances gbase identically.  Tile partials go to
        // P.tpartA[tile]; CTA b sums its fixed slice in tile order after the barrier (phase B):
        // deterministic whichever warp took which tile.
        const int ntA = (n + 31) >> 5, lane = threadIdx.x & 31;
        for (;;) {
          unsigned long long c = 0;
          if (lane == 0) c = atomicAdd(P.gctr, 1ull);
          c = __shfl_sync(FULL, c, 0);
          const long long t = (long long)(c - gbase);
          if (t >= ntA) break;
          const int j = ((int)t << 5) + lane;
          double d = colA(j, j < n, j < n);
#pragma unroll
          for (int off = 16; off; off >>= 1) d += __shfl_xor_sync(FULL, d, off);
          if (lane == 0) P.tpartA[t] = d;
        }
        gbase += (unsigned long long)ntA + (unsigned long long)gridDim.x * (kBS / 32);
        sliceA = true;
      } else if (Gt == 1 && (dyn & 1)) {
        double t1[1];
        tiles_dynamic(n, [&](int j, bool ok, double (&c)[1]) { c[0] = colA(j, ok, ok); }, t1, true);
        v3[0] = t1[0];
      } else {
        for (int it = 0; it < col_iters; ++it) {
          const int j = it * ngrpt + grpt;
          const bool ok = j < n;
          v3[0] += colA(j, ok, ok && glt == 0);
        }
      }
      if (!r2) {  // swap: x <-> x', K~'y <-> K~'y'
        T *t = x; x = xp; xp = t;
        t = KTy; KTy = KTyp; KTyp = t;
      }
    } else {
      for (int j = gtid; j < n; j += gthreads) {
        const double xo = lv(x + j);
        const double xn = median3(lv(lsT + j), xo - tau * (lv(cs + j) - lv(KTy + j)), lv(usT + j));
        st_tgt(xp + j, xn);
        const double d = xn - xo;
        v3[0] += d * d;
      }
    }
    TR(if (tr_on) { tr_t1 = tnow(); tr_a += tr_t1 - tr_t0; });
    grid.sync();
    TR(if (tr_on) { tr_t0 = tnow(); tr_aw += tr_t0 - tr_t1; });
    // ================= phase B: [commit m-side] + SpMV #1 + dual step =================
    {
      // one row i of phase B; returns its ||dy||^2 and <dy, K~x' - K~x> terms
      auto rowB = [&](int i, bool ok, bool lead, double (&c)[2], const int32_t *rp_, const int32_t *ci_,
                      const T *kv_, const double *addp) {
        double o_y = 0.0, o_kx = 0.0, o_yp = 0.0, o_ya = 0.0, o_kxp = 0.0, o_kxa = 0.0, o_qs = 0.0, o_add = 0.0;
        if (lead) {
          o_qs = lv(qs + i);
          if (addp) o_add = addp[i];   // pass 1's K~_L x' (two-pass phase B)
          if (pending) {
            o_yp = lv(yp + i); o_ya = lv(ya + i); o_kxp = lv(Kxp + i);
            if (r2) { o_y = lv(y + i); o_kx = lv(Kx + i); o_kxa = lv(Kxa + i); }
          } else {
            o_y = lv(y + i); o_kx = lv(Kx + i);
          }
        }
        const double s = o_add + row_dot(i, ok, m, G, gl, rp_, ci_, kv_, xp, tbuf, P.lrB);
        c[0] = 0.0; c[1] = 0.0;
        if (!lead) return;
        double yv, kxv;
        if (pending) {
          if (!r2) {
            yv = o_yp;
            sv(ya + i, o_ya + theta * (o_yp - o_ya));
            kxv = o_kxp;
          } else {
            yv = ha * (rf1 * o_yp - rf0 * o_y) + hb * o_ya;
            kxv = ha * (rf1 * o_kxp - rf0 * o_kx) + hb * o_kxa;
            sv(y + i, yv); sv(Kx + i, kxv);
          }
        } else {
          yv = o_y; kxv = o_kx;
        }
        double yn = yv + sigma * (o_qs - 2.0 * s + kxv);
        if (i < m1) yn = pos_part(yn);
        if (pending && !r2) { st_tgt(y + i, yn); sv(Kx + i, s); }   // old buffers become y', K~x' after the swap
        else { st_tgt(yp + i, yn); sv(Kxp + i, s); }
        const double d = yn - yv;
        c[0] = d * d;
        c[1] = d * (s - kxv);
      };
      if (G == 1 && leanB) {
        // pass 1 (two-pass split): K~_L x' of this CTA's row tiles parked in tmp; pass 2 (or the
        // only pass): K~_R x' (+ tmp) or K~x' with the row epilogue
        if (P.split) {
          __syncthreads();
          if (threadIdx.x == 0) {
            lean_range(m);
            s_cx.gctr = nullptr;
            s_cx.rp = P.rpL; s_cx.ci = P.ciL; s_cx.kv = P.kvL; s_cx.tgt = xp; s_cx.park = P.tmp;
          }
          __syncthreads();
          if (P.lrB) phase_tiles<kB_PARK, T, true>(&s_cx, &s_ctr, tbuf);
          else phase_tiles<kB_PARK, T, false>(&s_cx, &s_ctr, tbuf);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          lean_range(m);
          s_cx.gctr = nullptr;
          if (P.split) { s_cx.rp = P.rpR; s_cx.ci = P.ciR; s_cx.kv = P.kvR; s_cx.add = P.tmp; }
          else { s_cx.rp = P.rp; s_cx.ci = P.ci; s_cx.kv = P.kv; s_cx.add = nullptr; }
          s_cx.tgt = xp; s_cx.m1 = m1; s_cx.r0 = qs;
          s_cx.tau_sigma = sigma; s_cx.theta = theta; s_cx.ha = ha; s_cx.hb = hb; s_cx.rf1 = rf1; s_cx.rf0 = rf0;
          if (pending && !r2) { s_cx.r1 = yp; s_cx.r2 = Kxp; s_cx.e0 = ya; s_cx.e1 = y; s_cx.e2 = Kx; }
          else if (pending) { s_cx.r1 = yp; s_cx.r2 = Kxp; s_cx.r3 = ya; s_cx.r4 = Kxa; s_cx.e0 = y; s_cx.e1 = Kx; s_cx.e2 = yp; s_cx.e3 = Kxp; }
          else { s_cx.r1 = y; s_cx.r2 = Kx; s_cx.e2 = yp; s_cx.e3 = Kxp; }
        }
        __syncthreads();
        if (P.lrB) {
          if (pending && !r2) phase_tiles<kB_RA, T, true>(&s_cx, &s_ctr, tbuf);
          else if (pending) phase_tiles<kB_R2, T, true>(&s_cx, &s_ctr, tbuf);
          else phase_tiles<kB_NOP, T, true>(&s_cx, &s_ctr, tbuf);
        } else {
          if (pending && !r2) phase_tiles<kB_RA, T, false>(&s_cx, &s_ctr, tbuf);
          else if (pending) phase_tiles<kB_R2, T, false>(&s_cx, &s_ctr, tbuf);
          else phase_tiles<kB_NOP, T, false>(&s_cx, &s_ctr, tbuf);
        }
        __syncthreads();
        double t2[2];
        lean_reduce(t2);
        v3[1] = t2[0]; v3[2] = t2[1];
      } else if (G == 1 && (dyn & 2)) {
        double t2[2];
        if (P.split) {
          // pass 1: K~_L x' of the CTA's tiles into tmp (gather target: the first column half of
          // x' only, L2-resident); pass 2: K~_R x' + tmp and the row epilogue
          double none[1];
          tiles_dynamic(m, [&](int i, bool ok, double (&c)[1]) {
            const double sl = tile_row_dot<T, T, false>(i, ok, m, P.rpL, P.ciL, P.kvL, xp, tbuf);
            if (ok) P.tmp[i] = sl;
            c[0] = 0.0;
          }, none, false);
          tiles_dynamic(m, [&](int i, bool ok, double (&c)[2]) { rowB(i, ok, ok, c, P.rpR, P.ciR, P.kvR, P.tmp); },
                        t2, true);
        } else {
          tiles_dynamic(m, [&](int i, bool ok, double (&c)[2]) { rowB(i, ok, ok, c, P.rp, P.ci, P.kv, nullptr); },
                        t2, true);
        }
        v3[1] = t2[0]; v3[2] = t2[1];
      } else {
        for (int it = 0; it < row_iters; ++it) {
          const int i = it * ngrp + grp;
          const bool ok = i < m;
          double c[2];
          rowB(i, ok, ok && gl == 0, c, P.rp, P.ci, P.kv, nullptr);
          v3[1] += c[0]; v3[2] += c[1];
        }
      }
      if (pending && !r2) {
        T *t = y; y = yp; yp = t;
        t = Kx; Kx = Kxp; Kxp = t;
      }
      pending = false;
      if (sliceA2) {  // the lean phase A's global-claim partials: this CTA's fixed slice, tile order
        sliceA2 = false;
        const int ntA = (n + 31) >> 5, nb = (int)gridDim.x, TA = (ntA + nb - 1) / nb;
        const int a0 = (int)blockIdx.x * TA, a1 = min(ntA, a0 + TA);
        if (threadIdx.x < 32) {
          double a = 0.0;
          for (int t = a0 + (int)threadIdx.x; t < a1; t += 32) a += __ldcg(P.tpartA + (size_t)t * 2);
#pragma unroll
          for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
          v3[0] = threadIdx.x == 0 ? a : 0.0;
        } else {
          v3[0] = 0.0;
        }
      }
      if (sliceA) {  // phase A's tile partials of this CTA's fixed slice, in tile order
        sliceA = false;
        const int ntA = (n + 31) >> 5, nb = (int)gridDim.x, TA = (ntA + nb - 1) / nb;
        const int a0 = (int)blockIdx.x * TA, a1 = min(ntA, a0 + TA);
        if (threadIdx.x < 32) {
          double a = 0.0;
          for (int t = a0 + (int)threadIdx.x; t < a1; t += 32) a += __ldcg(P.tpartA + t);
#pragma unroll
          for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
          v3[0] = threadIdx.x == 0 ? a : 0.0;
        } else {
          v3[0] = 0.0;
        }
      }
      block_partials<3>(v3, next_part(), s_red);
    }
    TR(if (tr_on) { tr_t1 = tnow(); tr_b += tr_t1 - tr_t0; });
    grid.sync();
    double t3[3];
    grid_totals<3>(t3, cur_part(), s_tot);
    TR(if (tr_on) { tr_t0 = tnow(); tr_bw += tr_t0 - tr_t1; ++tr_n; });
    ++jatt;
    const double I = t3[2];
    const double M = omega * t3[0] + t3[1] * inv_omega;
    const double eb = (I != 0.0) ? M / (2.0 * fabs(I)) : INFINITY;
    const bool acc = cstep || (eta <= eb);
    const double eta_used = eta;
    if (P.alog && blockIdx.x == 0 && threadIdx.x == 0 && jatt <= P.acap) {
      double *r = P.alog + 4 * (jatt - 1);
      r[0] = (double)jatt; r[1] = acc ? 1.0 : 0.0; r[2] = eta_used; r[3] = eb;
    }
    if (!cstep) {
      double f1, f2;
      step_factors(P.tab, jatt, f1, f2);
      eta = fmin(f1 * eb, f2 * eta);
    }
    if (!acc) {
      if (++rejects >= 100) { status = LP_NUMERICAL_ERROR; ox = x; oy = y; oKx = Kx; oKTy = KTy; break; }
      continue;
    }
    rejects = 0;
    // accepted: prepare the commit (step 4)
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
    TR(if (tr_on) tr_t1 = tnow());

    // ================= check: commit-only phase (both sides) =================
    // infeasibility rays (reading 35): r2HPDHG z - anchor here, raPDHG z - (pre-step point) below
    {
      double v[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) v[q] = 0.0;
      CertAcc acc;
      for (int it = 0; it < col_iters; ++it) {
        const int j = it * ngrpt + grpt;
        const bool ok = j < n;
        const double s = row_dot(j, ok, n, Gt, glt, P.trp, P.tci, P.tkv, yp, tbuf, P.lrA);
        if (ok && glt == 0) {
          KTyp[j] = (T)s;
          if (!r2) {
            xa[j] = (T)((double)xa[j] + theta * ((double)xp[j] - (double)xa[j]));
          } else {
            x[j] = (T)(ha * (rf1 * (double)xp[j] - rf0 * (double)x[j]) + hb * (double)xa[j]);
            KTy[j] = (T)(ha * (rf1 * s - rf0 * (double)KTy[j]) + hb * (double)KTya[j]);
            const double dc = P.Dc[j];
            kkt_col_acc(v, true, dc, xp[j], s, P.c0[j], cs[j], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
            const double d = xp[j] - xr[j];
            v[4] += d * d;
            cert_col(acc, dc, x[j], xa[j], KTy[j], KTya[j], P.c0[j], P.l0[j], P.u0[j]);
          }
        }
      }
      for (int i = gtid; i < m; i += gthreads) {
        if (!r2) {
          ya[i] = (T)((double)ya[i] + theta * ((double)yp[i] - (double)ya[i]));
        } else {
          const double ypi = yp[i], kxp = Kxp[i];
          y[i] = (T)(ha * (rf1 * ypi - rf0 * (double)y[i]) + hb * (double)ya[i]);
          Kx[i] = (T)(ha * (rf1 * kxp - rf0 * (double)Kx[i]) + hb * (double)Kxa[i]);
          kkt_row_acc(v, true, i < m1, P.Dr[i], ypi, kxp, P.q0[i], qs[i]);
          const double d = ypi - yr[i];
          v[5] += d * d;
          cert_row(acc, i < m1, P.Dr[i], y[i], ya[i], Kx[i], Kxa[i], P.q0[i]);
        }
      }
      if (!r2) {
        T *t = x; x = xp; xp = t;
        t = KTy; KTy = KTyp; KTyp = t;
        t = y; y = yp; yp = t;
        t = Kx; Kx = Kxp; Kxp = t;
      }
      v[6] = acc.sy; v[7] = acc.sx; v[8] = acc.oy; v[9] = acc.ox; v[10] = acc.vy; v[11] = acc.vx;
      if (r2) block_partials<12, (3u << 10)>(v, next_part(), s_red);
    }
    grid.sync();
    const T *cx, *cy, *cKx, *cKTy;
    double metric, dx2, dy2;
    if (!r2) {
      // average's products (2 SpMVs) fused with all KKT / distance partials
      double v[kNP];
#pragma unroll
      for (int q = 0; q < kNP; ++q) v[q] = 0.0;
      CertAcc acc;
      for (int it = 0; it < row_iters; ++it) {
        const int i = it * ngrp + grp;
        const bool ok = i < m;
        const double s = row_dot(i, ok, m, G, gl, P.rp, P.ci, P.kv, xa, tbuf, P.lrB);
        if (ok && gl == 0) {
          Kxa[i] = (T)s;
          const double dr = P.Dr[i], yai = ya[i], yi = y[i], kxi = Kx[i], q0 = P.q0[i], qsi = qs[i];
          kkt_row_acc(v + 0, true, i < m1, dr, yai, s, q0, qsi);
          kkt_row_acc(v + 4, true, i < m1, dr, yi, kxi, q0, qsi);
          kkt_row_acc(v + 8, false, i < m1, dr, yai, s, q0, qsi);
          kkt_row_acc(v + 12, false, i < m1, dr, yi, kxi, q0, qsi);
          const double da = yai - yr[i], dcur = yi - yr[i];
          v[17] += da * da;
          v[19] += dcur * dcur;
          cert_row(acc, i < m1, dr, yi, yp[i], kxi, Kxp[i], q0);   // yp, Kxp: the pre-step point
        }
      }
      for (int it = 0; it < col_iters; ++it) {
        const int j = it * ngrpt + grpt;
        const bool ok = j < n;
        const double s = row_dot(j, ok, n, Gt, glt, P.trp, P.tci, P.tkv, ya, tbuf, P.lrA);
        if (ok && glt == 0) {
          KTya[j] = (T)s;
          const double dc = P.Dc[j], xaj = xa[j], xj = x[j], ktj = KTy[j];
          const double c0 = P.c0[j], csj = cs[j], l0 = P.l0[j], lsj = P.ls[j], u0 = P.u0[j], usj = P.us[j];
          kkt_col_acc(v + 0, true, dc, xaj, s, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(v + 4, true, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(v + 8, false, dc, xaj, s, c0, csj, l0, lsj, u0, usj);
          kkt_col_acc(v + 12, false, dc, xj, ktj, c0, csj, l0, lsj, u0, usj);
          const double da = xaj - xr[j], dcur = xj - xr[j];
          v[16] += da * da;
          v[18] += dcur * dcur;
          cert_col(acc, dc, xj, xp[j], ktj, KTyp[j], c0, l0, u0);
        }
      }
      v[20] = acc.sy; v[21] = acc.sx; v[22] = acc.oy; v[23] = acc.ox; v[24] = acc.vy; v[25] = acc.vx;
      block_partials<kNP, (3u << 24)>(v, next_part(), s_red);
      grid.sync();
      double t[kNP];
      grid_totals<kNP, (3u << 24)>(t, cur_part(), s_tot);
      const Kkt5 ka = kkt5(t + 0), kc = kkt5(t + 4);
      if (blockIdx.x == 0 && threadIdx.x == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
        verbose_line(0, k, kc.pobj, kc.dobj, kc.pres, kc.dres, kc.gap, omega, eta);
      if (tpass(ka, nq0, nc0)) { log_check(0.0, 0, 1); status = LP_OPTIMAL; ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; break; }
      if (tpass(kc, nq0, nc0)) { log_check(0.0, 0, 2); status = LP_OPTIMAL; ox = x; oy = y; oKx = Kx; oKTy = KTy; break; }
      if (certify(t + 20, xp, yp, KTyp)) { log_check(0.0, 0, 3); break; }
      if (k == P.iter_limit) {
        log_check(0.0, 0, 0);
        status = LP_ITERATION_LIMIT;
        if (kkt5_rel(ka, nq0, nc0) < kkt5_rel(kc, nq0, nc0)) { ox = xa; oy = ya; oKx = Kxa; oKTy = KTya; }
        else { ox = x; oy = y; oKx = Kx; oKTy = KTy; }
        break;
      }
      const Kkt5 sa = kkt5(t + 8), sc = kkt5(t + 12);
      const double e_a = kkt_omega(sa, omega, inv_omega);
      const double e_c = kkt_omega(sc, omega, inv_omega);
      if (restart_to_average(e_a, e_c)) { cx = xa; cy = ya; cKx = Kxa; cKTy = KTya; metric = e_a; dx2 = t[16]; dy2 = t[17]; }
      else { cx = x; cy = y; cKx = Kx; cKTy = KTy; metric = e_c; dx2 = t[18]; dy2 = t[19]; }
    } else {
      double t[12];
      grid_totals<12, (3u << 10)>(t, cur_part(), s_tot);
      const Kkt5 kw = kkt5(t);
      if (blockIdx.x == 0 && threadIdx.x == 0 && verbose_due(P.verbose, P.display_freq, k, P.check_freq))
        verbose_line(0, k, kw.pobj, kw.dobj, kw.pres, kw.dres, kw.gap, omega, eta);
      if (tpass(kw, nq0, nc0)) { log_check(rP, 0, 1); status = LP_OPTIMAL; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break; }
      if (certify(t + 6, xa, ya, KTya)) { log_check(0.0, 0, 3); break; }
      if (k == P.iter_limit) { log_check(rP, 0, 0); status = LP_ITERATION_LIMIT; ox = xp; oy = yp; oKx = Kxp; oKTy = KTyp; break; }
      cx = xp; cy = yp; cKx = Kxp; cKTy = KTyp; metric = rP; dx2 = t[4]; dy2 = t[5];
    }
    const bool restart = restart_due(k_in, k, metric, ref, last);
    log_check(metric, restart ? 1 : 0, 0);
    last = metric;
    if (restart) {
      ++restarts;
      omega = primal_weight(omega, sqrt(dx2), sqrt(dy2));
      inv_omega = 1.0 / omega;
      for (int j = gtid; j < n; j += gthreads) {
        const T xv = cx[j], kt = cKTy[j];
        x[j] = xv; xr[j] = xv; xa[j] = xv; KTy[j] = kt; KTya[j] = kt;
      }
      for (int i = gtid; i < m; i += gthreads) {
        const T yv = cy[i], kx = cKx[i];
        y[i] = yv; yr[i] = yv; ya[i] = yv; Kx[i] = kx; Kxa[i] = kx;
      }
      k_in = 0;
      if (!r2) { W = 0.0; ref = metric; }
      grid.sync();
    }
    TR(if (tr_on) tr_chk += tnow() - tr_t1);
  }
  TR(if (tr_on && tr_n)
       printf("[trace] cta %d attempts %llu  per attempt (us): A work %.1f  A barrier %.1f  B work %.1f  "
              "B barrier+totals %.1f  | checks total %.1f us\n", blockIdx.x, tr_n, tr_a * 1e-3 / tr_n,
              tr_aw * 1e-3 / tr_n, tr_b * 1e-3 / tr_n, tr_bw * 1e-3 / tr_n, tr_chk * 1e-3));

  // ================= step 6: output the candidate =================
  {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = gtid; j < n; j += gthreads) {
      const double dc = P.Dc[j], xs = ox[j], kt = oKTy[j];
      kkt_col_acc(v, true, dc, xs, kt, P.c0[j], cs[j], P.l0[j], P.ls[j], P.u0[j], P.us[j]);
      if (bx) {  // infeasible: the unit rays (reading 35)
        P.X[j] = dc * (xs - bx[j]) / ray_nx;
        P.L[j] = -((kt - bKTy[j]) / dc) / ray_ny;
      } else {
        P.X[j] = dc * xs;
        P.L[j] = P.c0[j] - kt / dc;
      }
    }
    for (int i = gtid; i < m; i += gthreads) {
      const double dr = P.Dr[i];
      kkt_row_acc(v, true, i < m1, dr, oy[i], oKx[i], P.q0[i], qs[i]);
      P.Y[i] = bx ? dr * (oy[i] - by[i]) / ray_ny : dr * oy[i];
    }
    block_partials<4>(v, next_part(), s_red);
  }
  grid.sync();
  double t[4];
  grid_totals<4>(t, cur_part(), s_tot);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const Kkt5 ko = kkt5(t);
    lp_result r;
    r.status = status; r.polish = 0;
    r.iterations = k; r.attempts = jatt; r.restarts = restarts;
    r.primal_objective = ko.pobj; r.dual_objective = ko.dobj;
    r.primal_residual = ko.pres; r.dual_residual = ko.dres; r.gap = ko.gap;
    r.rel_kkt = kkt5_rel(ko, nq0, nc0);
    r.omega = omega; r.eta = eta; r.solve_seconds = 0.0;
    *P.res = r;
  }
}

// ---- column halves of K~ (grid_split_prepare) ----
__global__ void split_count(int m, int h, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            int32_t *cntL) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    int c = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) c += ci[p] < h;
    cntL[i] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cntL[m] = 0;
}
// stable partition of every row into its left (column < h) and right entries; rpL from the scan
__global__ void split_fill(int m, int h, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ kv, const int32_t *__restrict__ rpL, int32_t *rpR,
                           int32_t *ciL, double *kvL, int32_t *ciR, double *kvR) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += gridDim.x * blockDim.x) {
    rpR[i] = rp[i] - rpL[i];
    if (i == m) continue;
    int pl = rpL[i], pr = rp[i] - rpL[i];
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      if (ci[p] < h) { ciL[pl] = ci[p]; kvL[pl++] = kv[p]; }
      else { ciR[pr] = ci[p]; kvR[pr++] = kv[p]; }
    }
  }
}

// The two-pass phase B pays when x' (elem x n bytes: 8 fp64, 4 fp32 storage) is past the
// L2-resident knee of random gathers (~64-72 MB, profiles/gather_rates.json) and the rows use the
// warp-tile mapping.  MPAX_GRID_SPLIT=1 forces it (tests), =0 disables it.
bool split_wanted(const DevProblem &D, int elem) {
  const char *e = getenv("MPAX_GRID_SPLIT");
  if (e) return atoi(e) == 1 && tile_mapping_ok(D.avg_row, D.max_row) && D.n >= 2;
  return tile_mapping_ok(D.avg_row, D.max_row) && (double)elem * (double)D.n > 64e6;
}

__global__ void round_f32(int64_t n, const double *__restrict__ a, float *__restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __double2float_rn(a[i]);
}

inline int pow2_floor(double v) {
  int g = 1;
  while (g * 2 <= v && g < 32) g *= 2;
  return g;
}

}  // namespace

int grid_split_prepare(DevProblem &P, cudaStream_t s, int elem) {
  if (P.split_h > 0 || !split_wanted(P, elem) || P.nnz <= 0) return LP_OK;
  const int m = (int)P.m, h = (int)(P.n / 2);
  const int64_t nnz = P.nnz;
  // one allocation: rpL, rpR (m+1 each), ciL/ciR (nnz), kvL/kvR (nnz), scan scratch
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, (int32_t *)nullptr, (int32_t *)nullptr, m + 1, s);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t o_rpL = 0, o_rpR = o_rpL + al(4 * (size_t)(m + 1)), o_ci = o_rpR + al(4 * (size_t)(m + 1)),
               o_kv = o_ci + al(4 * (size_t)nnz), o_cnt = o_kv + al(8 * (size_t)nnz), o_tmp = o_cnt + al(4 * (size_t)(m + 1)),
               total = o_tmp + al(temp);
  char *base = nullptr;
  MPAX_CUDA(cudaMallocAsync((void **)&base, total, s));
  P.split_mem = base;
  P.rpL = (int32_t *)(base + o_rpL); P.rpR = (int32_t *)(base + o_rpR);
  int32_t *cnt = (int32_t *)(base + o_cnt);
  MPAX_LAUNCH(split_count, 148 * 8, 256, 0, s, m, h, P.rp, P.ci, cnt);
  MPAX_CUDA(cub::DeviceScan::ExclusiveSum(base + o_tmp, temp, cnt, P.rpL, m + 1, s));
  // left entries first, right entries after them, in one ci / kv block each
  int32_t nL = 0;
  MPAX_CUDA(cudaMemcpyAsync(&nL, P.rpL + m, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  P.ciL = (int32_t *)(base + o_ci); P.ciR = P.ciL + nL;
  P.kvL = (double *)(base + o_kv); P.kvR = P.kvL + nL;
  // the right half's row pointers index from the start of ciR / kvR
  MPAX_LAUNCH(split_fill, 148 * 8, 256, 0, s, m, h, P.rp, P.ci, P.kv, P.rpL, P.rpR, P.ciL, P.kvL, P.ciR, P.kvR);
  MPAX_CHECK_LAUNCH();
  P.split_h = h;
  return LP_OK;
}

int grid_f32_prepare(DevProblem &P, cudaStream_t s) {
  const int64_t nnz = P.nnz;
  if (nnz <= 0) return LP_OK;
  const bool halves = P.split_h > 0;
  if (P.f32_mem && P.f32_split_h == (halves ? P.split_h : 0)) return LP_OK;
  if (P.f32_mem) MPAX_CUDA(cudaFreeAsync(P.f32_mem, s));
  P.f32_mem = nullptr;
  float *b = nullptr;
  MPAX_CUDA(cudaMallocAsync((void **)&b, (size_t)(halves ? 3 : 2) * (size_t)nnz * sizeof(float), s));
  P.f32_mem = b;
  P.kv32 = b; P.tkv32 = b + nnz;
  MPAX_LAUNCH(round_f32, 148 * 8, 256, 0, s, nnz, P.kv, P.kv32);
  MPAX_LAUNCH(round_f32, 148 * 8, 256, 0, s, nnz, P.tkv, P.tkv32);
  if (halves) {   // kvL, kvR are one contiguous block of nnz values (grid_split_prepare)
    P.kvL32 = b + 2 * nnz;
    P.kvR32 = P.kvL32 + (P.kvR - P.kvL);
    MPAX_LAUNCH(round_f32, 148 * 8, 256, 0, s, nnz, P.kvL, P.kvL32);
  }
  MPAX_CHECK_LAUNCH();
  P.f32_split_h = halves ? P.split_h : 0;
  return LP_OK;
}

namespace {

template <typename T>
int grid_launch(const DevProblem &D, const lp_options &o, const GridLaunch &L, cudaStream_t s, double **work,
                size_t *work_bytes) {
  constexpr bool f32 = sizeof(T) == sizeof(float);
  int dev = 0, sms = 0, coop = 0;
  MPAX_CUDA(cudaGetDevice(&dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MPAX_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return LP_ERR_UNSUPPORTED;
  // register budget: 2 CTAs of 512 threads per SM (64 regs; the spills sit in the rare check
  // code) by default -- measured 12% faster than 1 CTA/SM at 128 regs on a 2e7-nnz LP, equal at C4;
  // MPAX_GRID_MINB=1 selects the 128-register build
  // CTAs per SM: 2 x 512 threads (64 registers) give the memory-level parallelism a large LP's
  // gathers need (C5: 1.4 ms per attempt, against 3.2 ms with 1); with fewer than ~4 row +
  // column tiles per warp the phases are latency chains and 1 CTA of 128 registers per SM
  // (fewer spills, half the CTAs at every grid barrier) is faster (C4: 51 -> 46 us per attempt)
  const char *env = getenv("MPAX_GRID_MINB");
  const int64_t tiles = (D.m + 31) / 32 + (D.n + 31) / 32;
  const int minb = env ? (atoi(env) == 1 ? 1 : 2) : (tiles < 4 * 2 * (int64_t)sms * (kBS / 32) ? 1 : 2);
  void *kfn = minb == 1 ? (void *)grid_kernel<1, T> : (void *)grid_kernel<2, T>;
  int per_sm = 0;
  MPAX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kBS, 0));
  if (per_sm < 1) return LP_ERR_UNSUPPORTED;
  const int64_t n = D.n, m = D.m;
  int blocks = per_sm * sms;
  // small problems do not need the whole GPU
  const int64_t work_items = (D.nnz + n + m);
  while (blocks > sms && (int64_t)blocks * kBS > 4 * work_items) blocks -= sms;
  const int64_t ntile = (std::max(n, m) + 31) / 32;
  const size_t ntp = 2 * (size_t)blocks * (size_t)((ntile + blocks - 1) / blocks);  // P.tpart slots
  const size_t ntpA = 2 * (size_t)((n + 31) / 32) + 1;   // + the counter (the lean sweep writes 2 per tile)
  // fp64 block: per-CTA / per-tile partials, tmp (m), the counter; then the T block: 8n + 8m
  // iterate vectors (+ l~, u~ copies for fp32 storage)
  // every vector starts on a 256-byte boundary (a warp's 32 consecutive fp64 elements = 8 sectors;
  // one element off and every warp access touches 9)
  auto up = [](size_t v, size_t a) { return (v + a - 1) / a * a; };
  const size_t dbl = up((size_t)m + 2 * (size_t)blocks * kNP + ntp + ntpA, 32);
  const size_t ne = up((size_t)n, 256 / sizeof(T)), me = up((size_t)m, 256 / sizeof(T));
  const size_t tvec = 8 * ne + 8 * me + (f32 ? 2 * ne : 0);
  const size_t need = dbl * sizeof(double) + tvec * sizeof(T);
  if (*work_bytes < need) {
    if (*work) MPAX_CUDA(cudaFreeAsync(*work, s));
    *work = nullptr;
    MPAX_CUDA(cudaMallocAsync((void **)work, need, s));
    *work_bytes = need;
  }
  double *w = *work;
  T *wt = (T *)(w + dbl);
  GridParams<T> P;
  P.n = n; P.m = m; P.m1 = D.m1;
  P.rp = D.rp; P.ci = D.ci; P.trp = D.trp; P.tci = D.tci;
  if constexpr (f32) { P.kv = D.kv32; P.tkv = D.tkv32; }
  else { P.kv = D.kv; P.tkv = D.tkv; }
  P.Dr = D.Dr; P.Dc = D.Dc; P.ls = D.ls; P.us = D.us; P.l0 = D.l0; P.u0 = D.u0;
  P.c0 = L.c0; P.q0 = L.q0; P.X0 = L.X0; P.Y0 = L.Y0; P.kmax = D.kmax; P.sigma = D.sigma; P.tab = D.tab;
  P.const_step = o.step_rule == LP_STEP_CONSTANT;
  P.cs = wt; wt += ne;
  P.x = wt; wt += ne; P.KTy = wt; wt += ne; P.xp = wt; wt += ne; P.KTyp = wt; wt += ne; P.xa = wt; wt += ne;
  P.KTya = wt; wt += ne; P.xr = wt; wt += ne;
  P.qs = wt; wt += me;
  P.y = wt; wt += me; P.Kx = wt; wt += me; P.yp = wt; wt += me; P.Kxp = wt; wt += me; P.ya = wt; wt += me;
  P.Kxa = wt; wt += me; P.yr = wt; wt += me;
  P.lsw = nullptr; P.usw = nullptr;
  if constexpr (f32) { P.lsw = wt; wt += ne; P.usw = wt; wt += ne; }
  P.part = w; w += 2 * (size_t)blocks * kNP;
  P.tpart = w; w += ntp;
  P.tmp = w; w += m;
  P.gctr = (unsigned long long *)w; w += 1;
  P.tpartA = w;
  P.eps_abs = o.eps_abs; P.eps_rel = o.eps_rel; P.iter_limit = o.iteration_limit;
  P.eps_pi = o.eps_primal_infeasible; P.eps_di = o.eps_dual_infeasible;
  P.eps_fp = o.eps_feas_polish; P.polish_mode = L.polish_mode; P.rho = o.reflection;
  P.verbose = o.verbose; P.display_freq = o.display_frequency;
  P.check_freq = o.check_frequency; P.alg = o.algorithm;
  // thread per row for short rows (all lanes do useful epilogue work), 8 or 32 lanes for long rows
  // G ~ mean row length / 4 (measured on B200 for this persistent kernel: 4 lanes per 20-entry
  // row beat 1 and 8; each group walks its rows sequentially, so shorter groups mean longer
  // dependent chains; scripts/micro/spmv_bench.cu has the standalone-SpMV comparison)
  // G = 1: warp-tile CSR-stream for short rows, else G lanes per row (G ~ mean length / 4)
  auto group = [](double avg, int mx) { return tile_mapping_ok(avg, mx) ? 1 : std::max(2, pow2_floor(avg / 4.0)); };
  P.gk = group(D.avg_row, D.max_row);
  P.gkt = group(D.avg_col, D.max_col);
  P.lrB = (D.max_row < 0 || D.max_row >= kTileCH) ? 1 : 0;   // unknown lengths: keep the test
  P.lrA = (D.max_col < 0 || D.max_col >= kTileCH) ? 1 : 0;
  // phase A keeps the static mapping: with fewer than ~4 column tiles per warp (C4: 1.3) the
  // tile chunks are a serial latency chain and G lanes per column are faster (C4 phase A
  // 21 -> 17 us per attempt, trace build); phase B's dynamic tile driver wins at any size
  if (P.gkt == 1 && (n + 31) / 32 < 4 * (int64_t)blocks * (kBS / 32)) P.gkt = std::max(2, pow2_floor(D.avg_col / 4.0));
  // tuning experiments only; anything but a power of two in [1, 32] is ignored
  auto gsize = [](const char *e, int d) { const int v = atoi(e); return (v >= 1 && v <= 32 && !(v & (v - 1))) ? v : d; };
  if (const char *e = getenv("MPAX_GRID_G")) P.gk = gsize(e, P.gk);
  if (const char *e = getenv("MPAX_GRID_GT")) P.gkt = gsize(e, P.gkt);
  P.vpol = 0;
  if (const char *e = getenv("MPAX_GRID_VPOL")) P.vpol = atoi(e);
  P.tdist = 0;
  if (const char *e = getenv("MPAX_GRID_TDIST")) P.tdist = atoi(e);
  // dynamic tile driver per hot phase (bit 0: phase A inside each CTA, bit 1: phase B inside
  // each CTA, bit 2: phase A from one global counter); measured on C5: phase B 1.2 -> 0.85 ms;
  // phase A 0.66 -> 0.73 ms (bit 0), barrier wait 60-75 -> 7 us but work +50-75 us (bit 2):
  // phase B only by default
  P.dyn = 2;
  if (const char *e = getenv("MPAX_GRID_DYN")) P.dyn = atoi(e);
  // lean out-of-line sweeps where the 64-register budget of 2 CTAs per SM needs them (C5); with
  // 1 CTA of 128 registers per SM the inlined sweeps are 1.5% faster (C4: 44.6 -> 44.0 us per
  // attempt, scripts/gpu_c4_knobs.sh)
  P.lean = minb == 1 ? 0 : 3;
  if (const char *e = getenv("MPAX_GRID_LEAN")) P.lean = atoi(e);   // experiments: 0 = the inlined sweeps
  P.split = (D.split_h > 0 && split_wanted(D, (int)sizeof(T)) && P.gk == 1 && (P.dyn & 2) &&
             (!f32 || D.f32_split_h == D.split_h)) ? 1 : 0;
  P.rpL = D.rpL; P.ciL = D.ciL; P.rpR = D.rpR; P.ciR = D.ciR;
  if constexpr (f32) { P.kvL = D.kvL32; P.kvR = D.kvR32; }
  else { P.kvL = D.kvL; P.kvR = D.kvR; }
  P.X = L.X; P.Y = L.Y; P.L = L.L; P.res = L.res;
  P.alog = L.alog; P.clog = L.clog; P.acap = L.acap; P.ccap = L.ccap;
  void *args[] = {&P};
  MPAX_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(blocks), dim3(kBS), args, 0, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

}  // namespace

int grid_solve(const DevProblem &D, const lp_options &o, const GridLaunch &L, cudaStream_t s, double **work,
               size_t *work_bytes) {
  if (o.precision == LP_FP32) {
    if (D.nnz > 0 && !D.f32_mem) return LP_ERR_INVALID_ARGUMENT;   // grid_f32_prepare first
    return grid_launch<float>(D, o, L, s, work, work_bytes);
  }
  return grid_launch<double>(D, o, L, s, work, work_bytes);
}

}  // namespace mpax

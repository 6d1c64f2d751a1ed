// setup.cu -- one-time device setup of an LP handle:
//   validate, CSR of K' by a stable radix sort on the
//   column index, Ruiz (10 rounds, inf-norm) + Pock-Chambolle (alpha = 1)
//   diagonal scaling (contract step 1 in DESIGN.md §3), the
//   scaled matrix / bounds, max|K~| for eta0, and the line-search factor table.
//
// Determinism: every reduction here is a per-row / per-column sequential loop
// in stored order (K' rows are in increasing row order, so column sums run in
// the same order as a row-major scan) or an order-free max, so the scalings are
// bitwise reproducible run to run.
#include <cub/cub.cuh>

#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace mpax {

namespace {

// ---- validation -------------------------------------------------------------
// flag[0] = worst severity (3 dimension, 2 NaN/inf, 1 crossed bounds), flag[1] = an index.
__device__ __forceinline__ void report(int *flag, int sev, int idx) {
  atomicMax(flag, sev);
  atomicMin(flag + 1 + sev, idx);
}

__global__ void validate_kernel(int64_t m, int64_t n, int64_t nnz, const int64_t *__restrict__ rp,
                                const int32_t *__restrict__ ci, const double *__restrict__ v,
                                const double *__restrict__ c, int64_t nc, const double *__restrict__ q,
                                int64_t nq, const double *__restrict__ l, const double *__restrict__ u,
                                int *flag) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < m; i += stride) {  // rows: offsets, ranges, sorted columns
    int64_t a = rp[i], b = rp[i + 1];
    if ((i == 0 && a != 0) || (i == m - 1 && b != nnz) || b < a || a < 0 || b > nnz) {
      report(flag, 3, (int)i);
      continue;
    }
    atomicMax(flag + 5, (int)(b - a));
    for (int64_t p = a; p < b; ++p) {
      int32_t j = ci[p];
      if (j < 0 || j >= n || (p > a && j <= ci[p - 1])) { report(flag, 3, (int)i); break; }
    }
  }
  for (int64_t p = tid; p < nnz; p += stride)
    if (!isfinite(v[p])) report(flag, 2, (int)p);
  for (int64_t j = tid; j < nc; j += stride)
    if (!isfinite(c[j])) report(flag, 2, (int)j);
  for (int64_t i = tid; i < nq; i += stride)
    if (!isfinite(q[i])) report(flag, 2, (int)i);
  for (int64_t j = tid; j < n; j += stride) {
    double lj = l[j], uj = u[j];
    if (isnan(lj) || isnan(uj)) report(flag, 2, (int)j);
    else if (lj == INFINITY || uj == -INFINITY || lj > uj) report(flag, 1, (int)j);
  }
}

// ---- transpose --------------------------------------------------------------
__global__ void rows_to_int32(int64_t m, const int64_t *__restrict__ rp64, int32_t *__restrict__ rp32,
                              int32_t *__restrict__ row_of, const int *flag) {
  if (*flag) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
    rp32[i] = (int32_t)rp64[i];
    if (i < m)
      for (int64_t p = rp64[i]; p < rp64[i + 1]; ++p) row_of[p] = (int32_t)i;
  }
}

__global__ void iota_kernel(int64_t nnz, int32_t *__restrict__ a, const int *flag) {
  if (*flag) return;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    a[p] = (int32_t)p;
}

// K' row pointer: trp[j] = first position of column j in the sorted keys (lower bound).
__global__ void transpose_finish(int64_t n, int64_t nnz, const int32_t *__restrict__ skeys,
                                 const int32_t *__restrict__ perm, const int32_t *__restrict__ row_of,
                                 int32_t *__restrict__ trp, int32_t *__restrict__ tci, int *flag) {
  if (*flag) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = tid; j <= n; j += st) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < j) lo = mid + 1; else hi = mid;
    }
    trp[j] = (int32_t)lo;
  }
  // longest column of K (= row of K'): flag[6]
  for (int64_t j = tid; j < n; j += st) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] <= j) lo = mid + 1; else hi = mid;
    }
    int64_t a = 0, h2 = nnz;
    while (a < h2) {
      int64_t mid = (a + h2) >> 1;
      if (skeys[mid] < j) a = mid + 1; else h2 = mid;
    }
    atomicMax(flag + 6, (int)(lo - a));
  }
  for (int64_t d = tid; d < nnz; d += st) tci[d] = row_of[perm[d]];
}

// ---- preconditioning (contract step 1) ---------------------------------------
// a_ij = (|K_ij| Dr_i) Dc_j.  use_sum = 0: inf-norm (Ruiz), 1: 1-norm (Pock-Chambolle alpha=1).
__global__ void precond_norms(int64_t m, int64_t n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                              const int32_t *__restrict__ trp, const int32_t *__restrict__ tci,
                              const int32_t *__restrict__ perm, const double *__restrict__ kv0,
                              const double *__restrict__ Dr, const double *__restrict__ Dc,
                              double *__restrict__ rho, double *__restrict__ gam, int use_sum, const int *flag) {
  if (*flag) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = tid; t < m + n; t += st) {
    double acc = 0.0;
    if (t < m) {
      int64_t i = t;
      double dr = Dr[i];
      for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
        double a = __dmul_rn(fabs(kv0[p]) * dr, Dc[ci[p]]);   // (never contracted with the sum)
        acc = use_sum ? acc + a : fmax(acc, a);
      }
      rho[i] = acc;
    } else {
      int64_t j = t - m;
      double dc = Dc[j];
      for (int32_t d = trp[j]; d < trp[j + 1]; ++d) {
        double a = __dmul_rn(fabs(kv0[perm[d]]) * Dr[tci[d]], dc);
        acc = use_sum ? acc + a : fmax(acc, a);
      }
      gam[j] = acc;
    }
  }
}

__global__ void precond_update(int64_t m, int64_t n, const double *__restrict__ rho, const double *__restrict__ gam,
                               double *__restrict__ Dr, double *__restrict__ Dc, const int *flag) {
  if (*flag) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = tid; t < m + n; t += st) {
    if (t < m) { double r = rho[t]; Dr[t] *= (r > 0.0 ? 1.0 / sqrt(r) : 1.0); }
    else { double g = gam[t - m]; Dc[t - m] *= (g > 0.0 ? 1.0 / sqrt(g) : 1.0); }
  }
}

__global__ void set_ones(int64_t len, double *__restrict__ a) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x)
    a[t] = 1.0;
}

// K~_ij = (K_ij Dr_i) Dc_j into both copies; l~ = l / Dc, u~ = u / Dc; max |K~| (order-free max on the bits).
__global__ void scale_kernel(int64_t m, int64_t n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                             const int32_t *__restrict__ trp, const int32_t *__restrict__ tci,
                             const int32_t *__restrict__ perm, const double *__restrict__ kv0,
                             const double *__restrict__ Dr, const double *__restrict__ Dc, double *__restrict__ kv,
                             double *__restrict__ tkv, const double *__restrict__ l0, const double *__restrict__ u0,
                             double *__restrict__ ls, double *__restrict__ us, unsigned long long *kmax_bits,
                             const int *flag) {
  if (*flag) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  double mx = 0.0;
  for (int64_t t = tid; t < m + n; t += st) {
    if (t < m) {
      double dr = Dr[t];
      for (int32_t p = rp[t]; p < rp[t + 1]; ++p) {
        double s = (kv0[p] * dr) * Dc[ci[p]];
        kv[p] = s;
        mx = fmax(mx, fabs(s));
      }
    } else {
      int64_t j = t - m;
      double dc = Dc[j];
      for (int32_t d = trp[j]; d < trp[j + 1]; ++d) tkv[d] = (kv0[perm[d]] * Dr[tci[d]]) * dc;
      ls[j] = l0[j] / dc;
      us[j] = u0[j] / dc;
    }
  }
  if (mx > 0.0) atomicMax(kmax_bits, (unsigned long long)__double_as_longlong(mx));
}

__global__ void step_table_kernel(double *tab) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < kStepTab; j += gridDim.x * blockDim.x) {
    double jp1 = (double)(j + 1);
    tab[2 * j] = 1.0 - pow(jp1, -0.3);
    tab[2 * j + 1] = 1.0 + pow(jp1, -0.6);
    tab[2 * kStepTab + 2 * j] = (double)(j + 1) / (double)(j + 2);
    tab[2 * kStepTab + 2 * j + 1] = 1.0 / (double)(j + 2);
  }
}

// Standalone SpMV with the solver's scaled matrices (lp_spmv_scaled: parity tests and the
// bench's SpMV-pair bandwidth), with the grid kernel's mappings: G == 1 is the warp-tile
// CSR-stream (common.cuh tile_row_dot) for short rows; G >= 2 lanes per row otherwise, each
// lane with four entries in flight (index and value streamed evict-first, then the four
// gathers), butterfly over the group.  Fixed order: deterministic.
// accumulate (G == 1 only): y = y + K x, the second pass over the right column half of K~ as
// in the grid kernel's two-pass phase B (same summation order: left half, then right).
__global__ void __launch_bounds__(256) spmv_kernel(int64_t rows, int G, const int32_t *__restrict__ rp,
                                                   const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                   const double *__restrict__ x, double *__restrict__ y,
                                                   int accumulate) {
  __shared__ double s_tile[256 / 32][kTileBuf];
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (G == 1) {
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = gt - (threadIdx.x & 31); base < rows; base += nthr) {
      const int64_t r = base + (threadIdx.x & 31);
      const double a = (accumulate && r < rows) ? y[r] : 0.0;
      const double s = a + tile_row_dot((int)r, r < rows, (int)rows, rp, ci, v, x, s_tile[threadIdx.x >> 5]);
      if (r < rows) y[r] = s;
    }
    return;
  }
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  const int gl = (int)(gt % G);
  const int64_t iters = (rows + ng - 1) / ng;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t r = it * ng + gt / G;
    double s0 = 0.0, s1 = 0.0;
    if (r < rows) {
      const int32_t e = __ldg(rp + r + 1);
      for (int32_t p = __ldg(rp + r) + gl; p < e; p += 4 * G) {
        int32_t c[4];
        double w[4], xv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int32_t q = p + k * G;
          c[k] = q < e ? __ldcs(ci + q) : 0;
          w[k] = q < e ? __ldcs(v + q) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[k] = p + k * G < e ? x[c[k]] : 0.0;
        s0 += w[0] * xv[0];
        s1 += w[1] * xv[1];
        s0 += w[2] * xv[2];
        s1 += w[3] * xv[3];
      }
    }
    double s = s0 + s1;
    for (int off = G >> 1; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (r < rows && gl == 0) y[r] = s;
  }
}

// ---- fused single-CTA setup for small LPs --------------------------------------
// Same checks and the same arithmetic, in the same order, as validate_kernel +
// transpose + precond_norms/update + scale_kernel, in ONE launch with block
// barriers between the phases (the multi-kernel path costs ~35 launches, which
// dominates the per-batch setup of the paper's small LPs).  The transpose places
// column j's entries by scanning K in row-major order, which is the stable order.
// T threads: 1024 in general, 256 when m + n <= 256 (the C2 LPs: a quarter of the warps to
// synchronise at each of the ~70 block barriers of the 11 scaling rounds)

template <int kSmallT>
__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(FULL, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < kSmallT / 32 ? warp_tot[lane] : 0;
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(FULL, t, off);
      if (lane >= off) t += u;
    }
    if (lane < kSmallT / 32) warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const int before = w ? warp_tot[w - 1] : 0;
  const int res = before + incl - v;
  __syncthreads();
  return res;
}

template <int kSmallT>
__global__ void __launch_bounds__(kSmallT) setup_small_kernel(
    int m, int n, int nnz, const int64_t *__restrict__ rp64, const int32_t *__restrict__ ci,
    const double *__restrict__ kv0, const double *__restrict__ c, int64_t nc, const double *__restrict__ q, int64_t nq,
    const double *__restrict__ l0, const double *__restrict__ u0, int32_t *__restrict__ rp, int32_t *__restrict__ trp,
    int32_t *__restrict__ tci, int32_t *__restrict__ perm, double *__restrict__ kv, double *__restrict__ tkv,
    double *__restrict__ ls, double *__restrict__ us, double *__restrict__ Dr, double *__restrict__ Dc,
    double *__restrict__ kmax, int *flag) {
  extern __shared__ double sh[];
  double *rho = sh, *gam = sh + m;
  __shared__ int warp_tot[kSmallT / 32];
  __shared__ unsigned long long s_kmax;
  const int tid = threadIdx.x;
  // phase 0: validation (validate_kernel's checks)
  for (int i = tid; i < m; i += kSmallT) {
    const int64_t a = rp64[i], b = rp64[i + 1];
    if ((i == 0 && a != 0) || (i == m - 1 && b != nnz) || b < a || a < 0 || b > nnz) { report(flag, 3, i); continue; }
    atomicMax(flag + 5, (int)(b - a));
    for (int64_t p = a; p < b; ++p) {
      const int32_t j = ci[p];
      if (j < 0 || j >= n || (p > a && j <= ci[p - 1])) { report(flag, 3, i); break; }
    }
  }
  for (int p = tid; p < nnz; p += kSmallT) if (!isfinite(kv0[p])) report(flag, 2, p);
  for (int64_t j = tid; j < nc; j += kSmallT) if (!isfinite(c[j])) report(flag, 2, (int)j);
  for (int64_t i = tid; i < nq; i += kSmallT) if (!isfinite(q[i])) report(flag, 2, (int)i);
  for (int j = tid; j < n; j += kSmallT) {
    const double lj = l0[j], uj = u0[j];
    if (isnan(lj) || isnan(uj)) report(flag, 2, j);
    else if (lj == INFINITY || uj == -INFINITY || lj > uj) report(flag, 1, j);
  }
  if (tid == 0) s_kmax = 0ull;
  __syncthreads();
  if (*(volatile int *)flag) return;
  // phase 1: row pointers, column counts, K' row pointers (block scan), stable placement
  for (int i = tid; i <= m; i += kSmallT) rp[i] = (int32_t)rp64[i];
  int running = 0;
  for (int j0 = 0; j0 < n; j0 += kSmallT) {
    const int j = j0 + tid;
    int cnt = 0;
    if (j < n)
      for (int p = 0; p < nnz; ++p) cnt += (ci[p] == j);
    if (j < n) atomicMax(flag + 6, cnt);
    const int off = block_exclusive_scan<kSmallT>(cnt, warp_tot);
    if (j < n) trp[j] = running + off;
    // block total for the next chunk
    if (tid == kSmallT - 1) warp_tot[0] = off + cnt;
    __syncthreads();
    running += warp_tot[0];
    __syncthreads();
  }
  if (tid == 0) trp[n] = nnz;
  __syncthreads();
  for (int j = tid; j < n; j += kSmallT) {
    int d = trp[j];
    int row = 0;
    for (int p = 0; p < nnz; ++p) {
      while (rp[row + 1] <= p) ++row;
      if (ci[p] == j) { tci[d] = row; perm[d] = p; ++d; }
    }
  }
  for (int i = tid; i < m; i += kSmallT) Dr[i] = 1.0;
  for (int j = tid; j < n; j += kSmallT) Dc[j] = 1.0;
  __syncthreads();
  // phase 2: Ruiz x10 + Pock-Chambolle (alpha = 1), as precond_norms / precond_update
  for (int r = 0; r < 11; ++r) {
    const bool use_sum = (r == 10);
    for (int t = tid; t < m + n; t += kSmallT) {
      double acc = 0.0;
      if (t < m) {
        const double dr = Dr[t];
        for (int p = rp[t]; p < rp[t + 1]; ++p) {
          const double a = __dmul_rn(fabs(kv0[p]) * dr, Dc[ci[p]]);   // (never contracted with the sum)
          acc = use_sum ? acc + a : fmax(acc, a);
        }
        rho[t] = acc;
      } else {
        const int j = t - m;
        const double dc = Dc[j];
        for (int d = trp[j]; d < trp[j + 1]; ++d) {
          const double a = __dmul_rn(fabs(kv0[perm[d]]) * Dr[tci[d]], dc);
          acc = use_sum ? acc + a : fmax(acc, a);
        }
        gam[j] = acc;
      }
    }
    __syncthreads();
    for (int t = tid; t < m + n; t += kSmallT) {
      if (t < m) { const double rr = rho[t]; Dr[t] *= (rr > 0.0 ? 1.0 / sqrt(rr) : 1.0); }
      else { const double g = gam[t - m]; Dc[t - m] *= (g > 0.0 ? 1.0 / sqrt(g) : 1.0); }
    }
    __syncthreads();
  }
  // phase 3: scaled values, bounds, max |K~|
  double mx = 0.0;
  for (int t = tid; t < m + n; t += kSmallT) {
    if (t < m) {
      const double dr = Dr[t];
      for (int p = rp[t]; p < rp[t + 1]; ++p) {
        const double sv = (kv0[p] * dr) * Dc[ci[p]];
        kv[p] = sv;
        mx = fmax(mx, fabs(sv));
      }
    } else {
      const int j = t - m;
      const double dc = Dc[j];
      for (int d = trp[j]; d < trp[j + 1]; ++d) tkv[d] = (kv0[perm[d]] * Dr[tci[d]]) * dc;
      ls[j] = l0[j] / dc;
      us[j] = u0[j] / dc;
    }
  }
  if (mx > 0.0) atomicMax(&s_kmax, (unsigned long long)__double_as_longlong(mx));
  __syncthreads();
  if (tid == 0) *kmax = __longlong_as_double((long long)s_kmax);
}

// ---- fused multi-CTA setup for LPs whose K fits in shared memory (the C2 batches) ----------
// One launch does the whole create of a small LP batch: CTA 0 copies the shared K, l, u into the
// handle, validates them, transposes K and runs the 11 scaling rounds with every array in shared
// memory (no L2 round trips on the rounds' dependent loads); CTAs 1.. copy and check the
// per-instance costs c / q in parallel.  Same checks, same arithmetic in the same order as
// validate_kernel + transpose + precond_norms/update + scale_kernel (Dr, Dc bitwise equal).
// Each CTA writes its own 8 validation ints (vflag[blockIdx.x * 8 ..]; the flag layout of
// `report`) so no initialisation launch is needed; the host combines them (max / min).
struct TinySetupArgs {
  int m, n, nnz;
  const int64_t *rp64_src;
  const int32_t *ci_src;
  const double *kv0_src, *l_src, *u_src, *c_src, *q_src;
  int64_t nc, nq;
  int32_t *rp, *ci, *trp, *tci, *perm;
  double *kv0, *l0, *u0, *c_dst, *q_dst, *kv, *tkv, *ls, *us, *Dr, *Dc, *kmax;
  int *vflag;
  unsigned long long *queue;  // the handle's work-queue counter, zeroed here
  int *tstamp;                // diagnostics (MPAX_HOST_TRACE): CTA 0's phase times in cycles, or null
};
constexpr int kTinySetupT = 256;
constexpr int kCostPer = 8;    // cost values per thread of the cost CTAs

__device__ __forceinline__ void sreport(int *f, int sev, int idx) {
  atomicMax(f, sev);
  atomicMin(f + 1 + sev, idx);
}

__global__ void __launch_bounds__(kTinySetupT) setup_tiny_kernel(const TinySetupArgs A) {
  long long t_start = clock64();
  auto stamp = [&](int k) {
    if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0) A.tstamp[k] = (int)(clock64() - t_start);
  };
  __shared__ int f[8];
  __shared__ int warp_tot[kTinySetupT / 32];
  __shared__ unsigned long long s_kmax;
  const int tid = threadIdx.x;
  if (tid < 8) f[tid] = (tid >= 1 && tid <= 4) ? INT32_MAX : 0;
  if (tid == 0) s_kmax = 0ull;
  if (tid == 0 && blockIdx.x == 0 && A.queue) *A.queue = 0ull;
  __syncthreads();
  if (blockIdx.x > 0) {  // per-instance costs: copy into the handle and check finiteness
    // kCostPer consecutive values per thread, every load issued before any use (one memory
    // round trip per CTA instead of one per grid-stride iteration)
    const int64_t total = A.nc + A.nq;
    const int64_t base = ((int64_t)(blockIdx.x - 1) * kTinySetupT + tid) * kCostPer;
    const int64_t stride = (int64_t)(gridDim.x - 1) * kTinySetupT * kCostPer;
    for (int64_t t0 = base; t0 < total; t0 += stride) {
      double v[kCostPer];
#pragma unroll
      for (int u = 0; u < kCostPer; ++u) {
        const int64_t t = t0 + u;
        v[u] = t < A.nc ? A.c_src[t] : (t < total ? A.q_src[t - A.nc] : 0.0);
      }
#pragma unroll
      for (int u = 0; u < kCostPer; ++u) {
        const int64_t t = t0 + u;
        if (t >= total) break;
        if (t < A.nc) {
          if (A.c_dst != A.c_src) A.c_dst[t] = v[u];
          if (!isfinite(v[u])) sreport(f, 2, (int)t);
        } else {
          if (A.q_dst != A.q_src) A.q_dst[t - A.nc] = v[u];
          if (!isfinite(v[u])) sreport(f, 2, (int)(t - A.nc));
        }
      }
    }
    __syncthreads();
    if (tid < 8) A.vflag[blockIdx.x * 8 + tid] = f[tid];
    return;
  }
  const int m = A.m, n = A.n, nnz = A.nnz;
  extern __shared__ double sh[];
  double *kvs = sh, *Dr = kvs + nnz, *Dc = Dr + m, *rho = Dc + n, *gam = rho + m, *ls = gam + n, *us = ls + n;
  int *rp = (int *)(us + n), *ci = rp + m + 1, *trp = ci + nnz, *tci = trp + n + 1, *perm = tci + nnz,
      *rowof = perm + nnz, *rank = rowof + nnz;
  // phase 0: every input load in flight at once (one memory round trip): K, l, u into shared
  // memory and the handle; value / bound checks (validate_kernel's)
  const int span = max(max(m + 1, nnz), n);
  for (int t = tid; t < span; t += kTinySetupT) {
    if (t <= m) {
      const int64_t a = A.rp64_src[t];
      rp[t] = (int32_t)a;
      A.rp[t] = (int32_t)a;
      if (t < m && a != (int32_t)a) sreport(f, 3, t);
    }
    if (t < nnz) {
      const int32_t j = A.ci_src[t];
      const double v = A.kv0_src[t];
      ci[t] = j; kvs[t] = v;
      A.ci[t] = j; A.kv0[t] = v;
      if (!isfinite(v)) sreport(f, 2, t);
    }
    if (t < n) {
      const double lj = A.l_src[t], uj = A.u_src[t];
      ls[t] = lj; us[t] = uj;
      if (A.l0 != A.l_src) A.l0[t] = lj;
      if (A.u0 != A.u_src) A.u0[t] = uj;
      if (isnan(lj) || isnan(uj)) sreport(f, 2, t);
      else if (lj == INFINITY || uj == -INFINITY || lj > uj) sreport(f, 1, t);
    }
  }
  for (int j = tid; j <= n; j += kTinySetupT) trp[j] = 0;
  __syncthreads();
  // row structure (offsets, ranges, sorted in-range columns) and each entry's row
  for (int i = tid; i < m; i += kTinySetupT) {
    const int a = rp[i], b = rp[i + 1];
    if ((i == 0 && a != 0) || (i == m - 1 && b != nnz) || b < a || a < 0 || b > nnz) { sreport(f, 3, i); continue; }
    atomicMax(f + 5, b - a);
    for (int p = a; p < b; ++p) {
      const int32_t j = ci[p];
      if (j < 0 || j >= n || (p > a && j <= ci[p - 1])) { sreport(f, 3, i); break; }
      rowof[p] = i;
    }
  }
  __syncthreads();
  if (f[0] != 0) {
    if (tid < 8) A.vflag[tid] = f[tid];
    return;
  }
  stamp(0);
  // phase 1: the stable transpose, every entry in parallel.  Entries are in row-major order, so
  // an entry's position within its column is the number of earlier entries in that column.
  for (int p = tid; p < nnz; p += kTinySetupT) {
    const int j = ci[p];
    atomicAdd(trp + j, 1);
    int r = 0;
#pragma unroll 8
    for (int q = 0; q < p; ++q) r += (ci[q] == j);
    rank[p] = r;
  }
  __syncthreads();
  int running = 0;
  for (int j0 = 0; j0 < n; j0 += kTinySetupT) {
    const int j = j0 + tid;
    const int cnt = j < n ? trp[j] : 0;
    if (j < n) atomicMax(f + 6, cnt);
    const int off = block_exclusive_scan<kTinySetupT>(cnt, warp_tot);  // (synchronises)
    if (j < n) trp[j] = running + off;
    if (tid == kTinySetupT - 1) warp_tot[0] = off + cnt;
    __syncthreads();
    running += warp_tot[0];
    __syncthreads();
  }
  if (tid == 0) trp[n] = nnz;
  for (int p = tid; p < nnz; p += kTinySetupT) {
    const int d = trp[ci[p]] + rank[p];
    tci[d] = rowof[p];
    perm[d] = p;
  }
  for (int i = tid; i < m; i += kTinySetupT) Dr[i] = 1.0;
  for (int j = tid; j < n; j += kTinySetupT) Dc[j] = 1.0;
  __syncthreads();
  stamp(1);
  // phase 2a: 10 Ruiz rounds.  Every entry's a_ij = (|K_ij| Dr_i) Dc_j in parallel; the row and
  // column maxima through integer atomicMax on the bit patterns of these non-negative doubles
  // (order-free, so exactly the sequential maxima); then 1 / sqrt per row / column.
  unsigned long long *rmax = (unsigned long long *)rho, *cmax = (unsigned long long *)gam;
  for (int t = tid; t < m + n; t += kTinySetupT) {
    if (t < m) rmax[t] = 0ull; else cmax[t - m] = 0ull;
  }
  __syncthreads();
  for (int r = 0; r < 10; ++r) {
    for (int p = tid; p < nnz; p += kTinySetupT) {
      const int i = rowof[p], j = ci[p];
      const unsigned long long a = (unsigned long long)__double_as_longlong((fabs(kvs[p]) * Dr[i]) * Dc[j]);
      atomicMax(rmax + i, a);
      atomicMax(cmax + j, a);
    }
    __syncthreads();
    for (int t = tid; t < m + n; t += kTinySetupT) {
      unsigned long long *slot = t < m ? rmax + t : cmax + (t - m);
      const double g = __longlong_as_double((long long)*slot);
      *slot = 0ull;   // ready for the next round
      double f = 1.0;
      if (g > 0.0) {
        const double sg = sqrt(g);
        bool ok;
        f = div_rn_fast(1.0, sg, ok);
        if (!ok) f = 1.0 / sg;
      }
      if (t < m) Dr[t] *= f; else Dc[t - m] *= f;
    }
    __syncthreads();
  }
  stamp(2);
  // phase 2b: Pock-Chambolle (alpha = 1): row / column sums in stored order (K' rows are in
  // increasing row order), sequential per row / column as the oracle's
  for (int t = tid; t < m + n; t += kTinySetupT) {
    double acc = 0.0;
    if (t < m) {
      const double dr = Dr[t];
      // __dmul_rn / __dadd_rn: never contracted into an FMA (the oracle rounds product and sum apart)
      for (int p = rp[t]; p < rp[t + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(fabs(kvs[p]) * dr, Dc[ci[p]]));
      rho[t] = acc;
    } else {
      const int j = t - m;
      const double dc = Dc[j];
      for (int d = trp[j]; d < trp[j + 1]; ++d) acc = __dadd_rn(acc, __dmul_rn(fabs(kvs[perm[d]]) * Dr[tci[d]], dc));
      gam[j] = acc;
    }
  }
  __syncthreads();
  for (int t = tid; t < m + n; t += kTinySetupT) {
    if (t < m) { const double rr = rho[t]; Dr[t] *= (rr > 0.0 ? 1.0 / sqrt(rr) : 1.0); }
    else { const double g = gam[t - m]; Dc[t - m] *= (g > 0.0 ? 1.0 / sqrt(g) : 1.0); }
  }
  __syncthreads();
  stamp(3);
  // phase 3: scaled values, K' structure, bounds, max |K~| into the handle
  double mx = 0.0;
  for (int t = tid; t < m + n; t += kTinySetupT) {
    if (t < m) {
      const double dr = Dr[t];
      A.Dr[t] = dr;
      for (int p = rp[t]; p < rp[t + 1]; ++p) {
        const double sv = (kvs[p] * dr) * Dc[ci[p]];
        A.kv[p] = sv;
        mx = fmax(mx, fabs(sv));
      }
    } else {
      const int j = t - m;
      const double dc = Dc[j];
      A.Dc[j] = dc;
      A.trp[j] = trp[j];
      for (int d = trp[j]; d < trp[j + 1]; ++d) {
        A.tci[d] = tci[d];
        A.perm[d] = perm[d];
        A.tkv[d] = (kvs[perm[d]] * Dr[tci[d]]) * dc;
      }
      A.ls[j] = ls[j] / dc;
      A.us[j] = us[j] / dc;
    }
  }
  if (mx > 0.0) atomicMax(&s_kmax, (unsigned long long)__double_as_longlong(mx));
  __syncthreads();
  if (tid == 0) {
    A.trp[n] = nnz;
    *A.kmax = __longlong_as_double((long long)s_kmax);
  }
  stamp(4);
  if (tid < 8) A.vflag[tid] = f[tid];
}

size_t tiny_setup_smem(int64_t m, int64_t n, int64_t nnz) {
  return (size_t)(nnz + 2 * (m + n) + 2 * n) * sizeof(double) + (size_t)(m + 1 + n + 1 + 5 * nnz) * sizeof(int);
}

inline int grid_for(int64_t work, int block = 256) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

}  // namespace

// Finiteness of replaced costs / right-hand sides (lp_update_batch): flags as validate_kernel's.
__global__ void validate_costs_kernel(const double *__restrict__ c, int64_t nc, const double *__restrict__ q,
                                      int64_t nq, int *flag) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc + nq; t += st) {
    if (t < nc) { if (!isfinite(c[t])) report(flag, 2, (int)t); }
    else if (!isfinite(q[t - nc])) report(flag, 2, (int)(t - nc));
  }
}

__global__ void flag_init_kernel(int *flag) {
  if (threadIdx.x < 8) flag[threadIdx.x] = (threadIdx.x >= 1 && threadIdx.x <= 4) ? INT32_MAX : 0;
}

int validate_costs(const double *c, int64_t nc, const double *q, int64_t nq, int *d_flag, cudaStream_t s) {
  MPAX_LAUNCH(flag_init_kernel, 1, 32, 0, s, d_flag);
  MPAX_LAUNCH(validate_costs_kernel, grid_for(nc + nq), 256, 0, s, c, nc, q, nq, d_flag);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int setup_validate(DevProblem &P, const int64_t *row_ptr64, const double *c, int64_t nc, const double *q, int64_t nq,
                   cudaStream_t s, int *d_flag) {
  int64_t work = P.m + P.nnz + nc + nq + P.n;
  MPAX_LAUNCH(validate_kernel, grid_for(work), 256, 0, s, P.m, P.n, P.nnz, row_ptr64, P.ci, P.kv0, c, nc, q, nq,
              P.l0, P.u0, d_flag);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

namespace {
double *g_tab[64] = {nullptr};
std::mutex g_tab_mu;
}  // namespace

const double *step_table(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (!g_tab[dev]) {
    double *t = nullptr;
    if (cudaMalloc(&t, 4 * kStepTab * sizeof(double)) != cudaSuccess) return nullptr;
    MPAX_LAUNCH(step_table_kernel, 64, 256, 0, s, t);
    if (cudaStreamSynchronize(s) != cudaSuccess) return nullptr;
    g_tab[dev] = t;
  }
  return g_tab[dev];
}

int setup_transpose(DevProblem &P, const int64_t *row_ptr64, cudaStream_t s, int *d_flag) {
  const int64_t m = P.m, n = P.n, nnz = P.nnz;
  int32_t *row_of = nullptr, *keys_out = nullptr, *idx_in = nullptr;
  size_t nz = (size_t)(nnz > 0 ? nnz : 1);
  MPAX_CUDA(cudaMallocAsync(&row_of, nz * sizeof(int32_t), s));
  MPAX_CUDA(cudaMallocAsync(&keys_out, nz * sizeof(int32_t), s));
  MPAX_CUDA(cudaMallocAsync(&idx_in, nz * sizeof(int32_t), s));
  MPAX_LAUNCH(rows_to_int32, grid_for(m + 1), 256, 0, s, m, row_ptr64, P.rp, row_of, d_flag);
  MPAX_LAUNCH(iota_kernel, grid_for(nnz), 256, 0, s, nnz, idx_in, d_flag);
  // stable LSD radix sort of (col, position) pairs: rows stay in increasing order within a column
  if (nnz > 0) {
    int end_bit = 1;
    while (end_bit < 31 && (1ll << end_bit) <= n) ++end_bit;
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, P.ci, keys_out, idx_in, P.perm, (int)nnz, 0, end_bit, s);
    void *temp = nullptr;
    MPAX_CUDA(cudaMallocAsync(&temp, temp_bytes, s));
    MPAX_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, P.ci, keys_out, idx_in, P.perm, (int)nnz, 0,
                                              end_bit, s));
    g_launches.fetch_add(4, std::memory_order_relaxed);  // CUB's onesweep/histogram kernels (approx.)
    MPAX_CUDA(cudaFreeAsync(temp, s));
  }
  MPAX_LAUNCH(transpose_finish, grid_for(n + 1 + nnz), 256, 0, s, n, nnz, keys_out, P.perm, row_of, P.trp, P.tci,
              d_flag);
  MPAX_CHECK_LAUNCH();
  MPAX_CUDA(cudaFreeAsync(row_of, s));
  MPAX_CUDA(cudaFreeAsync(keys_out, s));
  MPAX_CUDA(cudaFreeAsync(idx_in, s));
  P.avg_row = m > 0 ? (double)nnz / (double)m : 0.0;
  P.avg_col = (double)nnz / (double)n;
  return LP_OK;
}

int setup_precond_init(DevProblem &P, cudaStream_t s) {
  MPAX_LAUNCH(set_ones, grid_for(P.m), 256, 0, s, P.m, P.Dr);
  MPAX_LAUNCH(set_ones, grid_for(P.n), 256, 0, s, P.n, P.Dc);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int setup_precond_norms(DevProblem &P, double *rho, double *gam, int use_sum, cudaStream_t s, int *d_flag) {
  MPAX_LAUNCH(precond_norms, grid_for(P.m + P.n, 128), 128, 0, s, P.m, P.n, P.rp, P.ci, P.trp, P.tci, P.perm, P.kv0,
              P.Dr, P.Dc, rho, gam, use_sum, d_flag);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int setup_precond_update(DevProblem &P, const double *rho, const double *gam, cudaStream_t s, int *d_flag) {
  MPAX_LAUNCH(precond_update, grid_for(P.m + P.n), 256, 0, s, P.m, P.n, rho, gam, P.Dr, P.Dc, d_flag);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int setup_scale(DevProblem &P, cudaStream_t s, int *d_flag) {
  MPAX_CUDA(cudaMemsetAsync(P.kmax, 0, sizeof(double), s));
  MPAX_LAUNCH(scale_kernel, grid_for(P.m + P.n, 128), 128, 0, s, P.m, P.n, P.rp, P.ci, P.trp, P.tci, P.perm, P.kv0,
              P.Dr, P.Dc, P.kv, P.tkv, P.l0, P.u0, P.ls, P.us, (unsigned long long *)P.kmax, d_flag);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int setup_build(DevProblem &P, const int64_t *row_ptr64, cudaStream_t s, int *d_flag) {
  int rc = setup_transpose(P, row_ptr64, s, d_flag);
  if (rc) return rc;
  // Ruiz x10 then Pock-Chambolle alpha=1 (contract step 1)
  double *rho = nullptr, *gam = nullptr;
  MPAX_CUDA(cudaMallocAsync(&rho, (size_t)(P.m > 0 ? P.m : 1) * sizeof(double), s));
  MPAX_CUDA(cudaMallocAsync(&gam, (size_t)P.n * sizeof(double), s));
  if ((rc = setup_precond_init(P, s))) return rc;
  for (int r = 0; r < 11; ++r) {
    if ((rc = setup_precond_norms(P, rho, gam, r == 10, s, d_flag))) return rc;
    if ((rc = setup_precond_update(P, rho, gam, s, d_flag))) return rc;
  }
  if ((rc = setup_scale(P, s, d_flag))) return rc;
  MPAX_CUDA(cudaFreeAsync(rho, s));
  MPAX_CUDA(cudaFreeAsync(gam, s));
  return LP_OK;
}

// The fused multi-CTA launch applies when K, the scalings and the transpose fit in shared memory.
constexpr size_t kTinySetupSmem = 160 * 1024;
bool setup_tiny_ok(const DevProblem &P) {
  // the per-entry rank scan of the transpose is O(nnz^2 / threads): small K only
  return P.m + P.n <= 8192 && P.nnz <= 2048 && tiny_setup_smem(P.m, P.n, P.nnz) <= kTinySetupSmem;
}

int setup_tiny_blocks(int64_t nc, int64_t nq) {
  const int64_t per = (int64_t)kTinySetupT * kCostPer;
  int64_t g = (nc + nq + per - 1) / per;
  if (g > 147) g = 147;
  if (g < 1) g = 1;
  return (int)(1 + g);
}

int setup_tiny(DevProblem &P, const TinySetupSources &S, int64_t *rp64_dst, double *c_dst, int64_t nc,
               double *q_dst, int64_t nq, int *vflag, int blocks, cudaStream_t s, unsigned long long *queue) {
  const size_t need = tiny_setup_smem(P.m, P.n, P.nnz);
  static bool attr_set = false;  // opt in to large dynamic shared memory once, only when needed
  if (need > 48 * 1024 && !attr_set) {
    MPAX_CUDA(cudaFuncSetAttribute(setup_tiny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kTinySetupSmem));
    attr_set = true;
  }
  (void)rp64_dst;
  TinySetupArgs A;
  A.m = (int)P.m; A.n = (int)P.n; A.nnz = (int)P.nnz;
  A.rp64_src = S.rp64; A.ci_src = S.ci; A.kv0_src = S.kv0; A.l_src = S.l; A.u_src = S.u;
  A.c_src = S.c; A.q_src = S.q; A.nc = nc; A.nq = nq;
  A.rp = P.rp; A.ci = P.ci; A.trp = P.trp; A.tci = P.tci; A.perm = P.perm;
  A.kv0 = P.kv0; A.l0 = P.l0; A.u0 = P.u0; A.c_dst = c_dst; A.q_dst = q_dst;
  A.kv = P.kv; A.tkv = P.tkv; A.ls = P.ls; A.us = P.us; A.Dr = P.Dr; A.Dc = P.Dc; A.kmax = P.kmax;
  A.vflag = vflag;
  A.queue = queue;
  // diagnostics: phase stamps into the tail of the (pinned, mapped) flag buffer
  A.tstamp = getenv("MPAX_HOST_TRACE") ? vflag + 8 * kMaxSetupBlocks - 8 : nullptr;
  const size_t smem = tiny_setup_smem(P.m, P.n, P.nnz);
  MPAX_LAUNCH(setup_tiny_kernel, blocks, kTinySetupT, smem, s, A);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

bool setup_small_ok(const DevProblem &P) {
  return P.m + P.n <= 4096 && (double)P.n * (double)P.nnz <= (double)(1 << 22);
}

int setup_small(DevProblem &P, const int64_t *row_ptr64, const double *c, int64_t nc, const double *q, int64_t nq,
                cudaStream_t s, int *d_flag) {
  const size_t smem = (size_t)(P.m + P.n) * sizeof(double);
  if (P.m + P.n <= 256) {
    MPAX_LAUNCH(setup_small_kernel<256>, 1, 256, smem, s, (int)P.m, (int)P.n, (int)P.nnz, row_ptr64, P.ci, P.kv0, c,
                nc, q, nq, P.l0, P.u0, P.rp, P.trp, P.tci, P.perm, P.kv, P.tkv, P.ls, P.us, P.Dr, P.Dc, P.kmax, d_flag);
  } else {
    MPAX_LAUNCH(setup_small_kernel<1024>, 1, 1024, smem, s, (int)P.m, (int)P.n, (int)P.nnz, row_ptr64, P.ci, P.kv0,
                c, nc, q, nq, P.l0, P.u0, P.rp, P.trp, P.tci, P.perm, P.kv, P.tkv, P.ls, P.us, P.Dr, P.Dc, P.kmax, d_flag);
  }
  MPAX_CHECK_LAUNCH();
  P.avg_row = P.m > 0 ? (double)P.nnz / (double)P.m : 0.0;
  P.avg_col = (double)P.nnz / (double)P.n;
  return LP_OK;
}

int spmv_scaled(const DevProblem &P, const double *v, double *Kv, const double *w, double *KTw, cudaStream_t s) {
  auto group = [](double avg, int mx) {  // as grid_solver.cu: 1 = warp-tile mapping
    if (tile_mapping_ok(avg, mx)) return 1;
    int g = 2;
    while (g * 2 <= avg / 4.0 && g < 32) g *= 2;
    return g;
  };
  const int G = group(P.avg_row, P.max_row), GT = group(P.avg_col, P.max_col);
  const int blocks = 148 * 8;  // grid-stride over row groups: 8 CTAs of 256 threads per SM
  if (v && Kv && P.m > 0) {
    if (G == 1 && P.split_h > 0) {  // the column halves built for the grid kernel (grid_split_prepare)
      MPAX_LAUNCH(spmv_kernel, blocks, 256, 0, s, P.m, 1, P.rpL, P.ciL, P.kvL, v, Kv, 0);
      MPAX_LAUNCH(spmv_kernel, blocks, 256, 0, s, P.m, 1, P.rpR, P.ciR, P.kvR, v, Kv, 1);
    } else {
      MPAX_LAUNCH(spmv_kernel, blocks, 256, 0, s, P.m, G, P.rp, P.ci, P.kv, v, Kv, 0);
    }
  }
  if (w && KTw) MPAX_LAUNCH(spmv_kernel, blocks, 256, 0, s, P.n, GT, P.trp, P.tci, P.tkv, w, KTw, 0);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

}  // namespace mpax

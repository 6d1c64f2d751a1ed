// power.cu -- sigma_max(K~) for the constant step rule (
// DESIGN.md §3 reading 34): the step eta = 0.998 / sigma_max(K~) makes
// tau * sigma * ||K~||^2 = eta^2 ||K~||^2 < 1, the classical PDHG condition
// (P:57 with the step of Chambolle-Pock), so every attempt is accepted.
//
// Power iteration on K~'K~ with the deterministic start vector
//   v_j = frac(j * 2654435761 / 2^32) + 0.5, normalised,
// then kPowerIters times: u = K~ v, w = K~' u, s = ||w||, v = w / s,
// sigma = sqrt(s); a zero w ends the iteration with sigma = 0 (eta = 1).
// The reductions run in a fixed order (block trees / last-block sums), so the
// result is reproducible run to run; it differs from a sequential sum by ulps.
#include "common.cuh"

namespace mpax {

namespace {

constexpr int kPT = 256;      // threads of the multi-kernel path
constexpr int kPBlocks = 296; // 2 x 148 SMs, fixed so the partial order is fixed

__device__ __forceinline__ double start_entry(int64_t j) {
  return (double)((uint32_t)((uint64_t)j * 2654435761ull)) / 4294967296.0 + 0.5;
}

// Deterministic block sum (warp butterflies, then warp 0 over the warp totals).
__device__ double block_sum(double v, double *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  __syncthreads();  // red may still be read from the previous call
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? red[lane] : 0.0;
    for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(FULL, t, off);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Single CTA: the whole iteration in one launch (small LPs; vectors in smem
// when they fit, else in the scratch the host passes).
__global__ void __launch_bounds__(1024) power_small_kernel(int m, int n, const int32_t *__restrict__ rp,
                                                           const int32_t *__restrict__ ci,
                                                           const double *__restrict__ kv,
                                                           const int32_t *__restrict__ trp,
                                                           const int32_t *__restrict__ tci,
                                                           const double *__restrict__ tkv, double *scratch,
                                                           int use_smem, int iters, double *sigma_out) {
  extern __shared__ double sh[];
  __shared__ double red[33];
  double *v = use_smem ? sh : scratch;
  double *w = v + n, *u = w + n;
  const int tid = threadIdx.x, T = blockDim.x;
  double ss = 0.0;
  for (int j = tid; j < n; j += T) {
    const double e = start_entry(j);
    v[j] = e;
    ss += e * e;
  }
  const double nv = sqrt(block_sum(ss, red));
  for (int j = tid; j < n; j += T) v[j] /= nv;
  __syncthreads();
  double sigma = 0.0;
  for (int t = 0; t < iters; ++t) {
    for (int i = tid; i < m; i += T) {
      double a = 0.0;
      for (int32_t p = rp[i]; p < rp[i + 1]; ++p) a += kv[p] * v[ci[p]];
      u[i] = a;
    }
    __syncthreads();
    ss = 0.0;
    for (int j = tid; j < n; j += T) {
      double a = 0.0;
      for (int32_t p = trp[j]; p < trp[j + 1]; ++p) a += tkv[p] * u[tci[p]];
      w[j] = a;
      ss += a * a;
    }
    const double sw = sqrt(block_sum(ss, red));  // barrier inside: w complete
    if (!(sw > 0.0)) { sigma = 0.0; break; }
    for (int j = tid; j < n; j += T) v[j] = w[j] / sw;
    sigma = sqrt(sw);
    __syncthreads();
  }
  if (tid == 0) *sigma_out = sigma;
}

// One warp, K~ and K~' as zero-padded ELL (widths W, WT) in shared memory: the
// whole iteration is a latency chain, so the small LPs of a batch (C2) run it
// with no block barriers and with every gather of a row issued at once.
constexpr int kWarpMaxDim = 256, kWarpMaxW = 16;

__global__ void __launch_bounds__(32) power_warp_kernel(int m, int n, int W, int WT, const int32_t *__restrict__ rp,
                                                        const int32_t *__restrict__ ci,
                                                        const double *__restrict__ kv,
                                                        const int32_t *__restrict__ trp,
                                                        const int32_t *__restrict__ tci,
                                                        const double *__restrict__ tkv, int iters,
                                                        double *sigma_out) {
  extern __shared__ double sh[];
  double *v = sh, *u = v + n, *rv = u + m, *cv = rv + (size_t)m * W;
  int *rc = (int *)(cv + (size_t)n * WT), *cc = rc + m * W;
  const int lane = threadIdx.x;
  for (int i = lane; i < m; i += 32) {
    const int a = rp[i], e = rp[i + 1];
    for (int w = 0; w < W; ++w) {
      const bool ok = a + w < e;
      rc[i * W + w] = ok ? ci[a + w] : 0;
      rv[i * W + w] = ok ? kv[a + w] : 0.0;
    }
  }
  for (int j = lane; j < n; j += 32) {
    const int a = trp[j], e = trp[j + 1];
    for (int w = 0; w < WT; ++w) {
      const bool ok = a + w < e;
      cc[j * WT + w] = ok ? tci[a + w] : 0;
      cv[j * WT + w] = ok ? tkv[a + w] : 0.0;
    }
  }
  // Normalisation: the direction of v is all the iteration carries, so between the
  // first and the last step v is rescaled by an exact power of two (no rounding,
  // no division or square root on the chain); sigma = sqrt(||K~'K~ v|| / ||v||) at
  // the end equals the oracle's sqrt(||w||) for unit v up to rounding.
  double ss = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double e = start_entry(j);
    v[j] = e;
    ss += e * e;
  }
  for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(FULL, ss, off);
  const double nv = sqrt(ss);
  for (int j = lane; j < n; j += 32) v[j] /= nv;
  __syncwarp();
  double vv = 1.0, ww = 0.0;  // ||v||^2 of the current iterate, ||w||^2 of the last product
  bool zero = false;
  for (int t = 0; t < iters; ++t) {
    for (int i = lane; i < m; i += 32) {
      double s = 0.0;
#pragma unroll 4
      for (int w = 0; w < W; ++w) s += rv[i * W + w] * v[rc[i * W + w]];
      u[i] = s;
    }
    __syncwarp();
    double wl[kWarpMaxDim / 32];
    ss = 0.0;
#pragma unroll
    for (int q = 0; q < kWarpMaxDim / 32; ++q) {
      const int j = lane + 32 * q;
      if (j >= n) break;
      double s = 0.0;
#pragma unroll 4
      for (int w = 0; w < WT; ++w) s += cv[j * WT + w] * u[cc[j * WT + w]];
      wl[q] = s;
      ss += s * s;
    }
    for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(FULL, ss, off);
    if (!(ss > 0.0)) { zero = true; break; }
    ww = ss;
    if (t + 1 == iters) break;  // v (with ||v||^2 = vv) produced the last w
    // v = w * 2^-e with 2^e ~ ||w||: exact, keeps the iterate near unit length
    const int e = (int)((__double_as_longlong(ss) >> 52) & 0x7ff) - 1023;
    const double sc = __longlong_as_double((long long)(1023 - (e >> 1)) << 52);  // 2^-(e/2), normal
    double vl = 0.0;
#pragma unroll
    for (int q = 0; q < kWarpMaxDim / 32; ++q) {
      const int j = lane + 32 * q;
      if (j >= n) break;
      v[j] = wl[q] * sc;
      vl += (wl[q] * sc) * (wl[q] * sc);
    }
    __syncwarp();
    if (t + 2 == iters) {  // the next product is the last: its v's norm is needed
      for (int off = 16; off; off >>= 1) vl += __shfl_xor_sync(FULL, vl, off);
      vv = vl;
    }
  }
  const double sigma = zero ? 0.0 : sqrt(sqrt(ww) / sqrt(vv));
  if (lane == 0) *sigma_out = sigma;
}

// The same iteration with the ELL rows in registers (the tiny solver's layouts:
// lane l owns rows l + 32t, t < RPT, and columns l + 32t, t < CPT): ~70
// instructions per iteration instead of ~210, for the C2-sized LPs.
template <int RPT, int CPT, int W, int WT>
__global__ void __launch_bounds__(32) power_reg_kernel(int m, int n, const int32_t *__restrict__ rp,
                                                       const int32_t *__restrict__ ci, const double *__restrict__ kv,
                                                       const int32_t *__restrict__ trp,
                                                       const int32_t *__restrict__ tci,
                                                       const double *__restrict__ tkv, int iters,
                                                       double *sigma_out) {
  __shared__ double v[32 * CPT], u[32 * RPT];
  const int lane = threadIdx.x;
  int rcol[RPT][W], ccol[CPT][WT];
  double rval[RPT][W], cval[CPT][WT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = lane + 32 * t;
    const int a = i < m ? rp[i] : 0, e = i < m ? rp[i + 1] : 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      rcol[t][w] = a + w < e ? ci[a + w] : 0;
      rval[t][w] = a + w < e ? kv[a + w] : 0.0;
    }
  }
#pragma unroll
  for (int t = 0; t < CPT; ++t) {
    const int j = lane + 32 * t;
    const int a = j < n ? trp[j] : 0, e = j < n ? trp[j + 1] : 0;
#pragma unroll
    for (int w = 0; w < WT; ++w) {
      ccol[t][w] = a + w < e ? tci[a + w] : 0;
      cval[t][w] = a + w < e ? tkv[a + w] : 0.0;
    }
  }
  double vl[CPT], ss = 0.0;
#pragma unroll
  for (int t = 0; t < CPT; ++t) {
    const int j = lane + 32 * t;
    vl[t] = j < n ? start_entry(j) : 0.0;
    ss += vl[t] * vl[t];
  }
  for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(FULL, ss, off);
  const double nv = sqrt(ss);
#pragma unroll
  for (int t = 0; t < CPT; ++t) v[lane + 32 * t] = vl[t] / nv;
  for (int t = lane; t < 32 * RPT; t += 32) u[t] = 0.0;
  __syncwarp();
  double vv = 1.0, ww = 0.0;
  bool zero = false;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) s += rval[r][w] * v[rcol[r][w]];
      u[lane + 32 * r] = s;
    }
    __syncwarp();
    double wl[CPT];
    ss = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < WT; ++w) s += cval[c][w] * u[ccol[c][w]];
      wl[c] = s;
      ss += s * s;
    }
    for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(FULL, ss, off);
    if (!(ss > 0.0)) { zero = true; break; }
    ww = ss;
    if (t + 1 == iters) break;
    const int e = (int)((__double_as_longlong(ss) >> 52) & 0x7ff) - 1023;
    const double sc = __longlong_as_double((long long)(1023 - (e >> 1)) << 52);
    double q = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const double x = wl[c] * sc;
      v[lane + 32 * c] = x;
      q += x * x;
    }
    __syncwarp();
    if (t + 2 == iters) {
      for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(FULL, q, off);
      vv = q;
    }
  }
  if (lane == 0) *sigma_out = zero ? 0.0 : sqrt(sqrt(ww) / sqrt(vv));
}

template <int RPT, int CPT, int W, int WT>
int launch_power_reg(const DevProblem &P, cudaStream_t s) {
  MPAX_LAUNCH((power_reg_kernel<RPT, CPT, W, WT>), 1, 32, 0, s, (int)P.m, (int)P.n, P.rp, P.ci, P.kv, P.trp, P.tci,
              P.tkv, kPowerIters, P.sigma);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

// ---- multi-kernel path (large LPs) ----
struct PowerWs {
  double part[kPBlocks];
  double norm;      // ||.|| of the last reduced vector
  double ss;        // column shards: this shard's sum of squares, then (reduced) the total
  int done;         // a zero w was met: sigma fixed at 0
  unsigned count;   // last-block counter
};

__global__ void pw_start(int64_t n, double *__restrict__ v) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    v[j] = start_entry(j);
}

// ws->norm = ||a||_2; with sigma_out: the iteration step (sigma = sqrt(norm), or done).
__global__ void __launch_bounds__(kPT) pw_norm(int64_t n, const double *__restrict__ a, PowerWs *ws,
                                               double *sigma_out) {
  __shared__ double red[33];
  __shared__ bool last;
  if (ws->done) return;
  double ss = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)kPT + threadIdx.x; j < n; j += (int64_t)kPBlocks * kPT) ss += a[j] * a[j];
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) {
    ws->part[blockIdx.x] = ss;
    __threadfence();
    last = atomicInc(&ws->count, kPBlocks - 1) == kPBlocks - 1;  // wraps to 0 for the next use
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < kPBlocks; ++b) t += ((volatile double *)ws->part)[b];
    const double nrm = sqrt(t);
    ws->norm = nrm;
    if (sigma_out) {
      if (nrm > 0.0) *sigma_out = sqrt(nrm);
      else { *sigma_out = 0.0; ws->done = 1; }
    }
  }
}

// ---- column shards (sharded.cu): v_g = columns [off, off + n) of v, u = sum_g K~_{:,g} v_g is
// reduced across shards, w_g = K~_{:,g}' u, and ||w||^2 = sum_g ||w_g||^2 ----
__global__ void pw_start_off(int64_t n, int64_t off, double *__restrict__ v) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    v[j] = start_entry(off + j);   // the unsharded start vector's entries
}

// ws->ss = sum_j a_j^2 over this shard (per block, then the blocks in order: fixed order)
__global__ void __launch_bounds__(kPT) pw_sumsq(int64_t n, const double *__restrict__ a, PowerWs *ws) {
  __shared__ double red[33];
  __shared__ bool last;
  if (ws->done) return;
  double ss = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)kPT + threadIdx.x; j < n; j += (int64_t)kPBlocks * kPT) ss += a[j] * a[j];
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) {
    ws->part[blockIdx.x] = ss;
    __threadfence();
    last = atomicInc(&ws->count, kPBlocks - 1) == kPBlocks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < kPBlocks; ++b) t += ((volatile double *)ws->part)[b];
    ws->ss = t;
  }
}

// after the cross-shard sum of ws->ss: ||.|| and, with sigma_out, the iteration step (as pw_norm)
__global__ void pw_finish(PowerWs *ws, double *sigma_out) {
  if (ws->done) return;
  const double nrm = sqrt(ws->ss);
  ws->norm = nrm;
  if (sigma_out) {
    if (nrm > 0.0) *sigma_out = sqrt(nrm);
    else { *sigma_out = 0.0; ws->done = 1; }
  }
}

__global__ void pw_scale(int64_t n, double *__restrict__ v, const double *__restrict__ a, const PowerWs *ws) {
  if (ws->done) return;
  const double s = ws->norm;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    v[j] = a[j] / s;
}

__global__ void pw_spmv(int64_t rows, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                        const double *__restrict__ kv, const double *__restrict__ x, double *__restrict__ y,
                        const PowerWs *ws) {
  if (ws->done) return;
  // warp per row, lanes stride the row, butterfly sum (fixed order)
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    double s = 0.0;
    for (int32_t p = rp[r] + lane; p < rp[r + 1]; p += 32) s += kv[p] * x[ci[p]];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (lane == 0) y[r] = s;
  }
}

inline int blocks_for(int64_t work, int block = 256) {
  int64_t b = (work + block - 1) / block;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

int power_begin(PowerState &S, int64_t n, int64_t m, cudaStream_t s) {
  S.n = n; S.m = m;
  const size_t vb = (size_t)(2 * n + (m > 0 ? m : 1)) * sizeof(double);
  MPAX_CUDA(cudaMallocAsync((void **)&S.buf, vb + sizeof(PowerWs), s));
  S.v = (double *)S.buf; S.w = S.v + n; S.u = S.w + n;
  S.ws = S.buf + vb;
  PowerWs *ws = (PowerWs *)S.ws;
  MPAX_CUDA(cudaMemsetAsync(ws, 0, sizeof(PowerWs), s));
  MPAX_LAUNCH(pw_start, blocks_for(n), 256, 0, s, n, S.v);
  MPAX_LAUNCH(pw_norm, kPBlocks, kPT, 0, s, n, S.v, ws, (double *)nullptr);
  MPAX_LAUNCH(pw_scale, blocks_for(n), 256, 0, s, n, S.v, S.v, ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_products(const DevProblem &P, PowerState &S, cudaStream_t s) {
  const PowerWs *ws = (const PowerWs *)S.ws;
  MPAX_LAUNCH(pw_spmv, blocks_for(S.m * 32), 256, 0, s, S.m, P.rp, P.ci, P.kv, S.v, S.u, ws);
  MPAX_LAUNCH(pw_spmv, blocks_for(S.n * 32), 256, 0, s, S.n, P.trp, P.tci, P.tkv, S.u, S.w, ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_normalize(PowerState &S, double *sigma_out, cudaStream_t s) {
  PowerWs *ws = (PowerWs *)S.ws;
  MPAX_LAUNCH(pw_norm, kPBlocks, kPT, 0, s, S.n, S.w, ws, sigma_out);
  MPAX_LAUNCH(pw_scale, blocks_for(S.n), 256, 0, s, S.n, S.v, S.w, ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_begin_cols(PowerState &S, int64_t n, int64_t m, int64_t off, cudaStream_t s) {
  S.n = n; S.m = m;
  const size_t vb = (size_t)(2 * n + (m > 0 ? m : 1)) * sizeof(double);
  MPAX_CUDA(cudaMallocAsync((void **)&S.buf, vb + sizeof(PowerWs), s));
  S.v = (double *)S.buf; S.w = S.v + n; S.u = S.w + n;
  S.ws = S.buf + vb;
  MPAX_CUDA(cudaMemsetAsync(S.ws, 0, sizeof(PowerWs), s));
  MPAX_LAUNCH(pw_start_off, blocks_for(n), 256, 0, s, n, off, S.v);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_kv(const DevProblem &P, PowerState &S, cudaStream_t s) {
  MPAX_LAUNCH(pw_spmv, blocks_for(S.m * 32), 256, 0, s, S.m, P.rp, P.ci, P.kv, S.v, S.u, (const PowerWs *)S.ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_ktu(const DevProblem &P, PowerState &S, cudaStream_t s) {
  MPAX_LAUNCH(pw_spmv, blocks_for(S.n * 32), 256, 0, s, S.n, P.trp, P.tci, P.tkv, S.u, S.w, (const PowerWs *)S.ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_sumsq(PowerState &S, const double *a, cudaStream_t s) {
  MPAX_LAUNCH(pw_sumsq, kPBlocks, kPT, 0, s, S.n, a, (PowerWs *)S.ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

double *power_ss(PowerState &S) { return &((PowerWs *)S.ws)->ss; }

int power_finish(PowerState &S, const double *a, double *sigma_out, cudaStream_t s) {
  PowerWs *ws = (PowerWs *)S.ws;
  MPAX_LAUNCH(pw_finish, 1, 1, 0, s, ws, sigma_out);
  MPAX_LAUNCH(pw_scale, blocks_for(S.n), 256, 0, s, S.n, S.v, a, ws);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int power_end(PowerState &S, cudaStream_t s) {
  if (S.buf) MPAX_CUDA(cudaFreeAsync(S.buf, s));
  S.buf = nullptr;
  return LP_OK;
}

int power_sigma(DevProblem &P, cudaStream_t s) {
  const int64_t m = P.m, n = P.n;
  const int iters = kPowerIters;
  if (m == 0 || P.nnz == 0) {  // K~ = 0: sigma = 0, eta = 1 (as the oracle)
    MPAX_CUDA(cudaMemsetAsync(P.sigma, 0, sizeof(double), s));
    P.sigma_ready = true;
    return LP_OK;
  }
  // register layouts of the tiny solver (same bounds as tiny_solve)
  if (P.max_row >= 0 && P.max_col >= 0 && m <= 32 && n <= 64) {
    int rc = LP_ERR_UNSUPPORTED;
    if (P.max_row <= 4 && P.max_col <= 4) rc = launch_power_reg<1, 2, 4, 4>(P, s);
    else if (P.max_row <= 8 && P.max_col <= 8) rc = launch_power_reg<1, 2, 8, 8>(P, s);
    if (rc == LP_OK) { P.sigma_ready = true; return LP_OK; }
    if (rc != LP_ERR_UNSUPPORTED) return rc;
  }
  const size_t wbytes = (size_t)(n + m) * 8 + (size_t)(m * P.max_row + n * P.max_col) * 12;
  if (m <= kWarpMaxDim && n <= kWarpMaxDim && P.max_row >= 0 && P.max_row <= kWarpMaxW && P.max_col <= kWarpMaxW &&
      wbytes <= 96 * 1024) {
    if (wbytes > 48 * 1024)
      MPAX_CUDA(cudaFuncSetAttribute(power_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wbytes));
    MPAX_LAUNCH(power_warp_kernel, 1, 32, wbytes, s, (int)m, (int)n, P.max_row, P.max_col, P.rp, P.ci, P.kv, P.trp,
                P.tci, P.tkv, iters, P.sigma);
    MPAX_CHECK_LAUNCH();
    P.sigma_ready = true;
    return LP_OK;
  }
  if (m + n <= 16384 && P.nnz <= (1 << 20)) {
    const size_t bytes = (size_t)(2 * n + m) * sizeof(double);
    const bool smem = bytes <= 160 * 1024;
    double *scratch = nullptr;
    if (!smem) MPAX_CUDA(cudaMallocAsync(&scratch, bytes, s));
    if (smem && bytes > 48 * 1024)
      MPAX_CUDA(cudaFuncSetAttribute(power_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    int64_t T = ((m > n ? m : n) + 31) / 32 * 32;
    if (T > 1024) T = 1024;
    MPAX_LAUNCH(power_small_kernel, 1, (int)T, smem ? bytes : 0, s, (int)m, (int)n, P.rp, P.ci, P.kv, P.trp, P.tci,
                P.tkv, scratch, smem ? 1 : 0, iters, P.sigma);
    MPAX_CHECK_LAUNCH();
    if (scratch) MPAX_CUDA(cudaFreeAsync(scratch, s));
    P.sigma_ready = true;
    return LP_OK;
  }
  PowerState S;
  int rc = power_begin(S, n, m, s);
  for (int t = 0; rc == LP_OK && t < iters; ++t) {
    rc = power_products(P, S, s);
    if (rc == LP_OK) rc = power_normalize(S, P.sigma, s);
  }
  const int rc2 = power_end(S, s);
  if (rc != LP_OK) return rc;
  if (rc2 != LP_OK) return rc2;
  P.sigma_ready = true;
  return LP_OK;
}

}  // namespace mpax

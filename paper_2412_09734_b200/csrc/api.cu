// api.cu -- the C ABI of include/lp.h: argument checks, uploads, dispatch to the
// device setup (setup.cu) and solver kernels (instance_solver.cu), copies out.
// Host code here only marshals; every step of the method runs in kernels.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

#ifdef MPAX_HAVE_NCCL
#include <nccl.h>
#endif

namespace mpax {
std::atomic<int64_t> g_launches{0};
static thread_local std::string t_detail;
void set_error_detail(const std::string &s) { t_detail = s; }
}  // namespace mpax

using namespace mpax;

struct lp_handle_s {
  cudaStream_t stream = nullptr;
  DevProblem P;
  int64_t batch = 1;
  bool is_batch = false;
  double *C0 = nullptr, *Q0 = nullptr;  // batch x n / batch x m (or n / m when shared)
  int64_t cstride = 0, qstride = 0;
  double *X = nullptr, *Y = nullptr, *L = nullptr;
  double *X0 = nullptr, *Y0 = nullptr;  // warm-start staging
  double *pol = nullptr;                // feasibility-polishing buffers (lazily allocated)
  double *spo = nullptr;                // SPO+ staging for host inputs / outputs (lazily allocated)
  lp_result *d_res = nullptr, *h_res = nullptr;
  unsigned long long *queue = nullptr;
  unsigned long long qbase = kQueueUnknown;  // the queue counter's value when known (tiny_solve)
  double *work = nullptr;
  size_t work_bytes = 0;
  int64_t *rp64 = nullptr;
  int *d_flag = nullptr, *h_flag = nullptr;  // validation flags (8 ints; the fused small setup: 8 per CTA)
  void *arena = nullptr;  // one allocation holding every per-handle array
  ShardedLP *sharded = nullptr;  // row-sharded handle (lp_create_sharded / _virtual)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool solved = false;
  // decision log of the grid path (lp_set_decision_log): device-visible buffers, or null
  double *alog = nullptr, *clog = nullptr;
  int64_t acap = 0, ccap = 0;
  int64_t log_inst = 0;   // the batch instance the register kernel logs
};

namespace {

// Host-side phase timer of the API calls (MPAX_HOST_TRACE=1: one stderr line per call with the
// microseconds since the call started at each mark; diagnostics only, off by default).
struct HostTrace {
  bool on;
  const char *what;
  std::chrono::steady_clock::time_point t0;
  char buf[512];
  int len = 0;
  explicit HostTrace(const char *w) : on(getenv("MPAX_HOST_TRACE") != nullptr), what(w) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  void mark(const char *label) {
    if (!on || len > 400) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    len += snprintf(buf + len, sizeof(buf) - len, " %s %.1f", label, us);
  }
  ~HostTrace() {
    if (on) fprintf(stderr, "[host] %s:%s\n", what, buf);
  }
};

std::once_flag g_pool_once;

// Pinned host buffers (result / flag staging) are recycled across handles:
// cudaMallocHost costs far more than a whole small-batch solve.
std::mutex g_pin_mu;
std::multimap<size_t, void *> g_pin_free;

size_t pin_class(size_t bytes) {
  size_t c = 256;
  while (c < bytes) c <<= 1;
  return c;
}
void *pin_get(size_t bytes) {
  const size_t c = pin_class(bytes);
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.find(c);
    if (it != g_pin_free.end()) {
      void *p = it->second;
      g_pin_free.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  if (cudaMallocHost(&p, c) != cudaSuccess) return nullptr;
  return p;
}
void pin_put(void *p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace(pin_class(bytes), p);
}

// Timing events are recycled across handles too (creating two per handle is a measurable part
// of a small batch's setup).
std::mutex g_ev_mu;
std::vector<cudaEvent_t> g_ev_free;
cudaEvent_t ev_get() {
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    if (!g_ev_free.empty()) {
      cudaEvent_t e = g_ev_free.back();
      g_ev_free.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  return cudaEventCreate(&e) == cudaSuccess ? e : nullptr;
}
void ev_put(cudaEvent_t e) {
  if (!e) return;
  std::lock_guard<std::mutex> lk(g_ev_mu);
  g_ev_free.push_back(e);
}

void init_pool() {
  std::call_once(g_pool_once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

int fail(int code, const std::string &msg) {
  set_error_detail(msg);
  return code;
}

template <class T>
int dalloc(T **p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  MPAX_CUDA(cudaMallocAsync((void **)p, count * sizeof(T), s));
  return LP_OK;
}

#define TRY(x)            \
  do {                    \
    int r_ = (x);         \
    if (r_ != LP_OK) {    \
      return r_;          \
    }                     \
  } while (0)

void free_handle(lp_handle h) {
  if (!h) return;
  if (h->sharded) {
    sharded_free(h->sharded);
    delete h;
    return;
  }
  cudaStream_t s = h->stream;
  for (void *p : {(void *)h->arena, (void *)h->X0, (void *)h->Y0, (void *)h->work, (void *)h->pol, (void *)h->spo,
                 h->P.split_mem, h->P.f32_mem})
    if (p) cudaFreeAsync(p, s);
  // every D2H into the pinned buffers was followed by a stream sync, so they can be recycled now
  pin_put(h->h_res, (size_t)h->batch * sizeof(lp_result));
  pin_put(h->h_flag, 8 * kMaxSetupBlocks * sizeof(int));
  ev_put(h->ev0);
  ev_put(h->ev1);
  delete h;
}

// Carves typed, 256-byte aligned arrays out of one device allocation.
struct Arena {
  size_t off = 0;
  char *base = nullptr;
  template <class T>
  void take(T **p, size_t count) {
    if (count == 0) count = 1;
    off = (off + 255) & ~(size_t)255;
    *p = base ? (T *)(base + off) : nullptr;
    off += count * sizeof(T);
  }
};

// Device-to-device uploads of one create in one launch: entry e copies bytes[e] (a multiple of
// 4) from src[e] to dst[e]; block 0 also writes the validation flags' initial values.
struct UploadList {
  static constexpr int kMax = 8;
  void *dst[kMax];
  const void *src[kMax];
  size_t bytes[kMax];
  int count = 0;
  int flag_init[8];
  int *flag = nullptr;
  void add(void *d, const void *s_, size_t b) {
    if (b == 0) return;
    dst[count] = d; src[count] = s_; bytes[count] = b; ++count;
  }
};
__global__ void upload_gather_kernel(const UploadList U) {
  if (blockIdx.x == 0 && threadIdx.x < 8 && U.flag) U.flag[threadIdx.x] = U.flag_init[threadIdx.x];
  for (int e = 0; e < U.count; ++e) {
    const size_t words = U.bytes[e] / 4;
    const uint32_t *src = (const uint32_t *)U.src[e];
    uint32_t *dst = (uint32_t *)U.dst[e];
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = src[i];
  }
}
int upload_gather(const UploadList &U, cudaStream_t s) {
  size_t words = 0;
  for (int e = 0; e < U.count; ++e) words = std::max(words, U.bytes[e] / 4);
  const int blocks = (int)std::min<size_t>(148 * 4, std::max<size_t>(1, (words + 255) / 256));
  MPAX_LAUNCH(upload_gather_kernel, blocks, 256, 0, s, U);
  MPAX_CHECK_LAUNCH();
  return LP_OK;
}

int check_desc(const lp_problem_desc *p) {
  if (!p) return fail(LP_ERR_INVALID_ARGUMENT, "problem descriptor is NULL");
  if (p->memory != LP_HOST && p->memory != LP_DEVICE) return fail(LP_ERR_INVALID_ARGUMENT, "bad memory kind");
  if (p->n < 1 || p->m1 < 0 || p->m2 < 0 || p->nnz < 0)
    return fail(LP_ERR_DIMENSION, "need n >= 1, m1, m2, nnz >= 0");
  const int64_t m = p->m1 + p->m2;
  if (p->nnz >= (int64_t)INT32_MAX || p->n >= (int64_t)INT32_MAX || m >= (int64_t)INT32_MAX)
    return fail(LP_ERR_UNSUPPORTED, "nnz, n and m must be < 2^31");
  if (m == 0 && p->nnz != 0) return fail(LP_ERR_DIMENSION, "nnz > 0 with no rows");
  if (p->dense && p->nnz != p->n * m) return fail(LP_ERR_DIMENSION, "dense K needs nnz = m*n");
  if (!p->row_ptr || (p->nnz > 0 && (!p->col_idx || !p->values)) || !p->c || !p->l || !p->u ||
      (m > 0 && !p->q))
    return fail(LP_ERR_INVALID_ARGUMENT, "a required array is NULL");
  return LP_OK;
}

int create_common(const lp_problem_desc *p, int64_t batch, const double *C, const double *Q, int32_t memory,
                  void *stream, lp_handle *out, bool is_batch) {
  HostTrace tr("create");
  TRY(check_desc(p));
  if (!out) return fail(LP_ERR_INVALID_ARGUMENT, "out is NULL");
  if (batch < 1) return fail(LP_ERR_BATCH_SHAPE, "batch must be >= 1");
  if (memory != LP_HOST && memory != LP_DEVICE) return fail(LP_ERR_INVALID_ARGUMENT, "bad memory kind");
  init_pool();
  lp_handle h = new lp_handle_s();
  h->stream = (cudaStream_t)stream;
  h->batch = batch;
  h->is_batch = is_batch;
  cudaStream_t s = h->stream;
  DevProblem &P = h->P;
  P.n = p->n; P.m1 = p->m1; P.m2 = p->m2; P.m = p->m1 + p->m2; P.nnz = p->nnz; P.dense = p->dense;
  const int64_t n = P.n, m = P.m, nnz = P.nnz;
  int rc = LP_OK;
  auto cleanup = [&](int code) { free_handle(h); return code; };
#define CK(x)                       \
  do {                              \
    rc = (x);                       \
    if (rc != LP_OK) return cleanup(rc); \
  } while (0)
  const bool perC = is_batch && C != nullptr, perQ = is_batch && Q != nullptr;
  h->cstride = perC ? n : 0;
  h->qstride = perQ ? m : 0;
  auto carve = [&](Arena &A) {
    A.take(&h->rp64, m + 1); A.take(&P.rp, m + 1); A.take(&P.ci, nnz); A.take(&P.kv0, nnz); A.take(&P.kv, nnz);
    A.take(&P.trp, n + 1); A.take(&P.tci, nnz); A.take(&P.perm, nnz); A.take(&P.tkv, nnz);
    A.take(&P.l0, n); A.take(&P.u0, n); A.take(&P.ls, n); A.take(&P.us, n); A.take(&P.Dr, m); A.take(&P.Dc, n);
    A.take(&P.kmax, 1); A.take(&P.sigma, 1); A.take(&h->C0, perC ? batch * n : n); A.take(&h->Q0, perQ ? batch * m : m);
    A.take(&h->X, batch * n); A.take(&h->Y, batch * m); A.take(&h->L, batch * n);
    A.take(&h->d_res, batch); A.take(&h->queue, 1); A.take(&h->d_flag, 8 * kMaxSetupBlocks);
  };
  {
    Arena sizing;
    carve(sizing);
    CK(dalloc((char **)&h->arena, sizing.off, s));
    tr.mark("arena");
    Arena real;
    real.base = (char *)h->arena;
    carve(real);
  }
  P.tab = const_cast<double *>(step_table(s));
  if (!P.tab) return cleanup(fail(LP_ERR_CUDA, "line-search table"));
  h->h_res = (lp_result *)pin_get((size_t)batch * sizeof(lp_result));
  h->h_flag = (int *)pin_get(8 * kMaxSetupBlocks * sizeof(int));
  if (!h->h_res || !h->h_flag) return cleanup(fail(LP_ERR_OUT_OF_MEMORY, "pinned host buffers"));
  if (!(h->ev0 = ev_get()) || !(h->ev1 = ev_get()))
    return cleanup(fail(LP_ERR_CUDA, "event create"));
  tr.mark("bufs");
  auto cp = [&](void *dst, const void *src, size_t bytes) -> int {
    if (bytes == 0) return LP_OK;
    MPAX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    return LP_OK;
  };
  const int64_t nC = perC ? batch * n : n, nQ = m > 0 ? (perQ ? batch * m : m) : 0;
  const double *srcC = perC ? C : p->c, *srcQ = perQ ? Q : p->q;
  if (setup_tiny_ok(P)) {
    // one launch: K, l, u, c / q copied into the handle, validated, transposed and scaled
    // (device inputs are read in place; host inputs are copied in first)
    const int blocks = setup_tiny_blocks(nC, nQ);
    TinySetupSources S;
    if (p->memory == LP_DEVICE && memory == LP_DEVICE) {
      S.rp64 = p->row_ptr; S.ci = p->col_idx; S.kv0 = p->values; S.l = p->l; S.u = p->u; S.c = srcC; S.q = srcQ;
    } else {
      CK(cp(P.ci, p->col_idx, (size_t)nnz * sizeof(int32_t)));
      CK(cp(P.kv0, p->values, (size_t)nnz * sizeof(double)));
      CK(cp(h->rp64, p->row_ptr, (size_t)(m + 1) * sizeof(int64_t)));
      CK(cp(P.l0, p->l, (size_t)n * sizeof(double)));
      CK(cp(P.u0, p->u, (size_t)n * sizeof(double)));
      CK(cp(h->C0, srcC, (size_t)nC * sizeof(double)));
      if (nQ) CK(cp(h->Q0, srcQ, (size_t)nQ * sizeof(double)));
      S.rp64 = h->rp64; S.ci = P.ci; S.kv0 = P.kv0; S.l = P.l0; S.u = P.u0; S.c = h->C0; S.q = h->Q0;
    }
    cudaEvent_t te[3] = {nullptr, nullptr, nullptr};
    if (tr.on) for (auto &e : te) { cudaEventCreate(&e); }
    if (tr.on) cudaEventRecord(te[0], s);
    // the per-CTA validation records go straight into the pinned host buffer (device-mapped, UVA)
    CK(setup_tiny(P, S, h->rp64, h->C0, nC, h->Q0, nQ, h->h_flag, blocks, s, h->queue));
    if (tr.on) cudaEventRecord(te[1], s);
    h->qbase = 0;  // zeroed by the setup kernel
    tr.mark("launch");
    if (tr.on) cudaEventRecord(te[2], s);
    tr.mark("d2h");
    if (cudaStreamSynchronize(s) != cudaSuccess) return cleanup(fail(LP_ERR_CUDA, "setup"));
    tr.mark("sync");
    if (tr.on) {
      float k_ms = 0.f, c_ms = 0.f;
      cudaEventElapsedTime(&k_ms, te[0], te[1]);
      cudaEventElapsedTime(&c_ms, te[1], te[2]);
      tr.mark(k_ms * 1e3f > 0 ? "gpu_kernel" : "gpu_kernel");
      const int *ts = h->h_flag + 8 * kMaxSetupBlocks - 8;
      fprintf(stderr, "[host] create device: setup kernel %.1f us, flag copy %.1f us; CTA 0 cycles: validated %d "
              "transposed %d ruiz %d pc %d done %d\n", k_ms * 1e3, c_ms * 1e3, ts[0], ts[1], ts[2], ts[3], ts[4]);
      for (auto &e : te) cudaEventDestroy(e);
    }
    // combine the per-CTA validation records (severity max, first index min, lengths max)
    int f[8] = {0, INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX, 0, 0, 0};
    for (int b = 0; b < blocks; ++b) {
      const int *r = h->h_flag + 8 * b;
      f[0] = std::max(f[0], r[0]);
      for (int k = 1; k <= 4; ++k) f[k] = std::min(f[k], r[k]);
      f[5] = std::max(f[5], r[5]);
      f[6] = std::max(f[6], r[6]);
    }
    memcpy(h->h_flag, f, sizeof(f));
  } else {
    const int init[8] = {0, INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX, 0, 0, 0};
    memcpy(h->h_flag, init, sizeof(init));
    UploadList U;
    U.add(h->rp64, p->row_ptr, (size_t)(m + 1) * sizeof(int64_t));
    U.add(P.ci, p->col_idx, (size_t)nnz * sizeof(int32_t));
    U.add(P.kv0, p->values, (size_t)nnz * sizeof(double));
    U.add(P.l0, p->l, (size_t)n * sizeof(double));
    U.add(P.u0, p->u, (size_t)n * sizeof(double));
    U.add(h->C0, perC ? (const void *)C : (const void *)p->c, (size_t)(perC ? batch * n : n) * sizeof(double));
    if (m > 0) U.add(h->Q0, perQ ? (const void *)Q : (const void *)p->q, (size_t)(perQ ? batch * m : m) * sizeof(double));
    if (p->memory == LP_DEVICE && memory == LP_DEVICE) {
      // device inputs: every copy and the flags' initial values in ONE gather kernel (a small
      // LP's create is bound by per-call overhead, not bytes: C2 8 copy calls -> 1 launch)
      for (int k = 0; k < 8; ++k) U.flag_init[k] = init[k];
      U.flag = h->d_flag;
      CK(upload_gather(U, s));
    } else {
      for (int k = 0; k < U.count; ++k) CK(cp(U.dst[k], U.src[k], U.bytes[k]));
      CK(cp(h->d_flag, h->h_flag, sizeof(init)));
    }
    if (setup_small_ok(P)) {
      CK(setup_small(P, h->rp64, h->C0, perC ? batch * n : n, h->Q0, perQ ? batch * m : m, s, h->d_flag));
    } else {
      CK(setup_validate(P, h->rp64, h->C0, perC ? batch * n : n, h->Q0, perQ ? batch * m : m, s, h->d_flag));
      CK(setup_build(P, h->rp64, s, h->d_flag));
    }
    CK(cp(h->h_flag, h->d_flag, 8 * sizeof(int)));
    if (cudaStreamSynchronize(s) != cudaSuccess) return cleanup(fail(LP_ERR_CUDA, "setup"));
  }
  const int *flag = h->h_flag;
  if (flag[0] == 3) return cleanup(fail(LP_ERR_DIMENSION, "CSR structure invalid at row " + std::to_string(flag[4])));
  if (flag[0] == 2) return cleanup(fail(LP_ERR_NAN, "NaN or infinity in K, c or q (or NaN in l/u) near index " + std::to_string(flag[3])));
  if (flag[0] == 1) return cleanup(fail(LP_ERR_CROSSED_BOUNDS, "crossed bounds at index " + std::to_string(flag[2])));
  P.max_row = flag[5];
  P.max_col = flag[6];
  tr.mark("done");
  *out = h;
  return LP_OK;
#undef CK
}

int check_options(const lp_options *o) {
  if (!o) return fail(LP_ERR_INVALID_ARGUMENT, "options NULL");
  if (!(o->eps_abs >= 0.0) || !(o->eps_rel >= 0.0) || o->iteration_limit < 1 || o->check_frequency < 1 ||
      (o->algorithm != LP_RAPDHG && o->algorithm != LP_R2HPDHG))
    return fail(LP_ERR_INVALID_ARGUMENT, "bad option value");
  if (o->feasibility_polishing && !(o->eps_feas_polish >= 0.0))
    return fail(LP_ERR_INVALID_ARGUMENT, "bad eps_feas_polish");
  if (o->path < LP_PATH_AUTO || o->path > LP_PATH_DMMA) return fail(LP_ERR_INVALID_ARGUMENT, "bad path");
  if (o->step_rule != LP_STEP_ADAPTIVE && o->step_rule != LP_STEP_CONSTANT)
    return fail(LP_ERR_INVALID_ARGUMENT, "bad step_rule");
  if (!(o->reflection >= 0.0 && o->reflection <= 1.0)) return fail(LP_ERR_INVALID_ARGUMENT, "reflection not in [0, 1]");
  if (o->precision != LP_FP64 && o->precision != LP_FP32) return fail(LP_ERR_INVALID_ARGUMENT, "bad precision");
  if (o->sharded_exchange != 0 && o->sharded_exchange != 1) return fail(LP_ERR_INVALID_ARGUMENT, "bad sharded_exchange");
  return LP_OK;
}

int run_sharded(lp_handle h, const lp_options *o, const double *X0, const double *Y0, lp_result *out) {
  cudaStream_t s = h->stream;
  const int64_t n = sharded_n_local(h->sharded), ml = sharded_m_local(h->sharded);
  const double *dX0 = nullptr, *dY0 = nullptr;
  if (X0) {
    if (!h->X0) TRY(dalloc(&h->X0, n, s));
    MPAX_CUDA(cudaMemcpyAsync(h->X0, X0, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
    dX0 = h->X0;
  }
  if (Y0 && ml > 0) {
    if (!h->Y0) TRY(dalloc(&h->Y0, ml, s));
    MPAX_CUDA(cudaMemcpyAsync(h->Y0, Y0, (size_t)ml * sizeof(double), cudaMemcpyDefault, s));
    dY0 = h->Y0;
  }
  const int rc = sharded_solve_polished(*h->sharded, *o, dX0, dY0, out);
  if (rc == LP_OK) h->solved = true;
  return rc;
}

// ---- feasibility polishing (reading 36): combine the two sub-solves per instance ----
// Instances whose main status is OPTIMAL take x from the primal polish and y, lambda
// from the dual polish; the result's residuals are those sub-solves' (computed on the
// original q / c they kept), the objectives are recomputed on the original data.
__global__ void polish_combine_kernel(int64_t n, int64_t m, int64_t m1, const double *C0, int64_t cstride,
                                      const double *Q0, int64_t qstride, const double *l0, const double *u0,
                                      const double *X1, const lp_result *res1, const double *Y2, const double *L2,
                                      const lp_result *res2, double *X, double *Y, double *L, lp_result *res) {
  const int64_t b = blockIdx.x;
  if (res[b].status != LP_OPTIMAL) return;
  __shared__ double red[4][8];
  const double *c = C0 + b * cstride, *q = Q0 + b * qstride;
  double v[4] = {0.0, 0.0, 0.0, 0.0};  // c'x, dual objective, |c|^2, |q|^2
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double xj = X1[b * n + j], lam = L2[b * n + j];
    X[b * n + j] = xj;
    L[b * n + j] = lam;
    v[0] += c[j] * xj;
    v[2] += c[j] * c[j];
    const double lp = fmax(lam, 0.0), lm = fmax(-lam, 0.0);
    if (l0[j] > -INFINITY) v[1] += l0[j] * lp;
    if (u0[j] < INFINITY) v[1] -= u0[j] * lm;
  }
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double yi = Y2[b * m + i];
    Y[b * m + i] = yi;
    v[1] += q[i] * yi;
    v[3] += q[i] * q[i];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < 4; ++k) {
    double s = v[k];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (lane == 0) red[k][w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[4];
    for (int k = 0; k < 4; ++k) {
      t[k] = 0.0;
      for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) t[k] += red[k][ww];
    }
    lp_result r = res[b];
    const double pres = res1[b].primal_residual, dres = res2[b].dual_residual;
    const double nc = sqrt(t[2]), nq = sqrt(t[3]), gap = fabs(t[0] - t[1]);
    r.primal_objective = t[0]; r.dual_objective = t[1];
    r.primal_residual = pres; r.dual_residual = dres; r.gap = gap;
    r.rel_kkt = fmax(pres / (1.0 + nq), fmax(dres / (1.0 + nc), gap / (1.0 + fabs(t[0]) + fabs(t[1]))));
    r.iterations += res1[b].iterations + res2[b].iterations;
    r.attempts += res1[b].attempts + res2[b].attempts;
    r.restarts += res1[b].restarts + res2[b].restarts;
    r.polish = (res1[b].status == LP_OPTIMAL && res2[b].status == LP_OPTIMAL) ? 1 : 2;
    res[b] = r;
  }
}

// ---- SPO+ (Eq. spo+ loss P:76-78, Eq. spo+ gradient P:80-82) ----
__global__ void spo_costs_kernel(int64_t count, const double *__restrict__ Cp, const double *__restrict__ Ct,
                                 double *__restrict__ C0) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    C0[t] = 2.0 * Cp[t] - Ct[t];
}

// one CTA per instance: loss[b] = -obj_b + 2 c^_b'x*_b - obj*_b, grad[b] = 2 (x*_b - x_b)
__global__ void spo_loss_kernel(int64_t n, const double *__restrict__ Cp, const double *__restrict__ Xt,
                                const double *__restrict__ ot, const double *__restrict__ X,
                                const lp_result *__restrict__ res, double *__restrict__ loss,
                                double *__restrict__ grad) {
  const int64_t b = blockIdx.x;
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double xt = Xt[b * n + j];
    s += Cp[b * n + j] * xt;
    grad[b * n + j] = 2.0 * (xt - X[b * n + j]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) t += red[ww];
    loss[b] = -res[b].primal_objective + 2.0 * t - ot[b];
  }
}

int run_solve(lp_handle h, const lp_options *o, const double *X0, const double *Y0, int32_t memory,
              lp_result *out) {
  if (!h || !out) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle or result");
  HostTrace tr("solve");
  TRY(check_options(o));
  if (memory != LP_HOST && memory != LP_DEVICE) return fail(LP_ERR_INVALID_ARGUMENT, "bad memory kind");
  if (h->sharded) {
    if (o->precision == LP_FP32) return fail(LP_ERR_UNSUPPORTED, "fp32 storage is a grid-path option");
    return run_sharded(h, o, X0, Y0, out);
  }
  cudaStream_t s = h->stream;
  const int64_t n = h->P.n, m = h->P.m, B = h->batch;
  // warm starts: staged into library memory (original space; scaled in-kernel)
  const double *dX0 = nullptr, *dY0 = nullptr;
  if (X0) {
    if (!h->X0) TRY(dalloc(&h->X0, B * n, s));
    MPAX_CUDA(cudaMemcpyAsync(h->X0, X0, (size_t)(B * n) * sizeof(double), cudaMemcpyDefault, s));
    dX0 = h->X0;
  }
  if (Y0 && m > 0) {
    if (!h->Y0) TRY(dalloc(&h->Y0, B * m, s));
    MPAX_CUDA(cudaMemcpyAsync(h->Y0, Y0, (size_t)(B * m) * sizeof(double), cudaMemcpyDefault, s));
    dY0 = h->Y0;
  }
  if (o->path == LP_PATH_DMMA && !h->P.dense) return fail(LP_ERR_UNSUPPORTED, "the DMMA path needs a dense K");
  const bool big = h->P.nnz >= 32768 || h->P.n + h->P.m >= 4096;
  const bool use_grid = (B == 1) && (o->path == LP_PATH_GRID || (o->path == LP_PATH_AUTO && big));
  if (o->path == LP_PATH_GRID && B != 1) return fail(LP_ERR_UNSUPPORTED, "the grid path solves one LP");
  if (o->precision == LP_FP32 && !use_grid)
    return fail(LP_ERR_UNSUPPORTED, "fp32 storage is a grid-path option (one large LP; DESIGN.md reading 39)");
  const bool want_log = h->alog || h->clog;
  if (want_log && !use_grid && o->path != LP_PATH_AUTO)
    return fail(LP_ERR_UNSUPPORTED, "the decision log is recorded by the grid path and the register kernel only");
  // a batch sharing a dense K: fp64 tensor-core path (auto from 8 instances on)
  const bool dmma = !use_grid && h->P.dense && (o->path == LP_PATH_DMMA || (o->path == LP_PATH_AUTO && B >= 8));
  if (dmma) {
    const size_t need = dmma_workspace_doubles(n, m, B) * sizeof(double);
    if (h->work_bytes < need) {
      if (h->work) MPAX_CUDA(cudaFreeAsync(h->work, s));
      h->work = nullptr;
      TRY(dalloc((char **)&h->work, need, s));
      h->work_bytes = need;
    }
  }
  bool host_written = false;   // the register kernel wrote the results into h_res itself
  // one solve of the batch (main, or a polishing sub-solve) on the chosen path
  auto dispatch = [&](const lp_options &oo, InstanceLaunch L) -> int {
    if (use_grid) {
      GridLaunch G;
      G.c0 = L.C0; G.q0 = L.Q0; G.X0 = L.X0; G.Y0 = L.Y0; G.X = L.X; G.Y = L.Y; G.L = L.L; G.res = L.res;
      G.polish_mode = L.polish_mode;
      if (L.polish_mode == 0) { G.alog = h->alog; G.clog = h->clog; G.acap = h->acap; G.ccap = h->ccap; }
      if (int rs = grid_split_prepare(h->P, s, oo.precision == LP_FP32 ? 4 : 8)) return rs;
      if (oo.precision == LP_FP32)
        if (int rs = grid_f32_prepare(h->P, s)) return rs;
      int rc = grid_solve(h->P, oo, G, s, &h->work, &h->work_bytes);
      if (rc == LP_ERR_UNSUPPORTED) return fail(rc, "cooperative launch unavailable");
      return rc;
    }
    int rc = LP_ERR_UNSUPPORTED;
    if (dmma) {
      rc = dmma_solve(h->P, oo, L, s, h->queue, h->work);
      h->qbase = kQueueUnknown;
      if (rc == LP_ERR_UNSUPPORTED && oo.path == LP_PATH_DMMA) return fail(rc, "dense K too large for the DMMA path");
    }
    if (rc == LP_ERR_UNSUPPORTED && oo.path == LP_PATH_AUTO) {
      rc = tiny_solve(h->P, oo, L, s, h->queue, &h->qbase);
      if (rc == LP_OK && L.res_host) host_written = true;
      if (rc == LP_ERR_UNSUPPORTED && (L.alog || L.clog))
        return fail(rc, "the register kernel logs decisions for the C2 shapes only");
    }
    if (rc == LP_ERR_UNSUPPORTED) {
      rc = instance_solve(h->P, oo, L, s, h->queue, &h->work, &h->work_bytes);
      h->qbase = kQueueUnknown;  // (the generic kernels reset the counter themselves)
    }
    return rc;
  };
  MPAX_CUDA(cudaEventRecord(h->ev0, s));
  // constant step rule: sigma_max(K~) once per handle (K is fixed for its lifetime)
  if (o->step_rule == LP_STEP_CONSTANT && !h->P.sigma_ready) TRY(power_sigma(h->P, s));
  InstanceLaunch L;
  L.C0 = h->C0; L.cstride = h->cstride; L.Q0 = h->Q0; L.qstride = h->qstride;
  L.X0 = dX0; L.Y0 = dY0; L.batch = B; L.X = h->X; L.Y = h->Y; L.L = h->L; L.res = h->d_res;
  // the main solve's results straight into the pinned host buffer (device-mapped through UVA) when
  // they are final: no polishing pass rewrites them afterwards
  L.res_host = o->feasibility_polishing ? nullptr : h->h_res;
  if (want_log && !use_grid) {   // the register kernel's one-instance log (main solve only)
    if (dmma) return fail(LP_ERR_UNSUPPORTED, "the DMMA path does not log decisions");
    L.alog = h->alog; L.clog = h->clog; L.acap = h->acap; L.ccap = h->ccap; L.log_inst = h->log_inst;
  }
  TRY(dispatch(*o, L));
  if (o->feasibility_polishing) {
    // (reading 36) primal polish: c = 0 from (x*, 0); dual polish: q = 0 from (proj 0, y*);
    // residual-only tests, infeasibility detection off, min(limit, kPolishLimit) steps
    bool run = true;
    if (use_grid) {  // one LP: run the sub-solves only after an OPTIMAL main solve
      MPAX_CUDA(cudaMemcpyAsync(h->h_res, h->d_res, sizeof(lp_result), cudaMemcpyDeviceToHost, s));
      MPAX_CUDA(cudaStreamSynchronize(s));
      run = h->h_res[0].status == LP_OPTIMAL;
    }
    if (run) {
      if (!h->pol) {
        const int64_t mm = m > 0 ? m : 1;
        const size_t dbl = (size_t)(4 * B * n + 3 * B * mm + n + mm);
        TRY(dalloc((char **)&h->pol, dbl * sizeof(double) + 2 * (size_t)B * sizeof(lp_result), s));
        MPAX_CUDA(cudaMemsetAsync(h->pol, 0, dbl * sizeof(double), s));
      }
      const int64_t mm = m > 0 ? m : 1;
      double *X1 = h->pol, *L1 = X1 + B * n, *X2 = L1 + B * n, *L2 = X2 + B * n, *Y1 = L2 + B * n,
             *Y2 = Y1 + B * mm, *zn = Y2 + B * mm, *zm = zn + n;
      lp_result *res1 = (lp_result *)(zm + mm), *res2 = res1 + B;
      lp_options op = *o;
      op.feasibility_polishing = 0;
      op.eps_primal_infeasible = -1.0;
      op.eps_dual_infeasible = -1.0;
      if (op.iteration_limit > kPolishLimit) op.iteration_limit = kPolishLimit;
      InstanceLaunch L1l = L;
      L1l.C0 = zn; L1l.cstride = 0; L1l.X0 = h->X; L1l.Y0 = nullptr;
      L1l.X = X1; L1l.Y = Y1; L1l.L = L1; L1l.res = res1; L1l.polish_mode = 1; L1l.active = h->d_res;
      TRY(dispatch(op, L1l));
      InstanceLaunch L2l = L;
      L2l.Q0 = zm; L2l.qstride = 0; L2l.X0 = nullptr; L2l.Y0 = m > 0 ? h->Y : nullptr;
      L2l.X = X2; L2l.Y = Y2; L2l.L = L2; L2l.res = res2; L2l.polish_mode = 2; L2l.active = h->d_res;
      TRY(dispatch(op, L2l));
      MPAX_LAUNCH(polish_combine_kernel, (int)B, 256, 0, s, n, m, h->P.m1, h->C0, h->cstride, h->Q0, h->qstride,
                  h->P.l0, h->P.u0, X1, res1, Y2, L2, res2, h->X, h->Y, h->L, h->d_res);
      MPAX_CHECK_LAUNCH();
    }
  }
  MPAX_CUDA(cudaEventRecord(h->ev1, s));
  tr.mark("launched");
  if (!host_written)
    MPAX_CUDA(cudaMemcpyAsync(h->h_res, h->d_res, (size_t)B * sizeof(lp_result), cudaMemcpyDeviceToHost, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  tr.mark("sync");
  float ms = 0.0f;
  MPAX_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  for (int64_t b = 0; b < B; ++b) {
    out[b] = h->h_res[b];
    out[b].solve_seconds = ms * 1e-3;
  }
  tr.mark("copied");
  h->solved = true;
  return LP_OK;
}

}  // namespace

extern "C" {

void lp_default_options(lp_options *o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->eps_abs = 1e-4;
  o->eps_rel = 1e-4;
  o->eps_primal_infeasible = 1e-8;
  o->eps_dual_infeasible = 1e-8;
  o->eps_feas_polish = 1e-6;
  o->iteration_limit = INT64_MAX;
  o->check_frequency = 64;
  o->algorithm = LP_R2HPDHG;
  o->warm_start = 0;
  o->feasibility_polishing = 0;
  o->verbose = 0;
  o->display_frequency = 10;
  o->path = LP_PATH_AUTO;
  o->step_rule = LP_STEP_ADAPTIVE;
  o->reflection = 1.0;
  o->precision = LP_FP64;
  o->sharded_exchange = 0;
}

int lp_create(const lp_problem_desc *p, void *cuda_stream, lp_handle *out) {
  return create_common(p, 1, nullptr, nullptr, p ? p->memory : LP_HOST, cuda_stream, out, false);
}

int lp_create_batch(const lp_problem_desc *shared, int64_t batch, const double *C, const double *Q,
                    int32_t memory, void *cuda_stream, lp_handle *out) {
  return create_common(shared, batch, C, Q, memory, cuda_stream, out, true);
}

int lp_update_batch(lp_handle h, const double *C, const double *Q, int32_t memory) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (h->sharded) return fail(LP_ERR_UNSUPPORTED, "lp_update_batch on a sharded handle");
  if (memory != LP_HOST && memory != LP_DEVICE) return fail(LP_ERR_INVALID_ARGUMENT, "bad memory kind");
  cudaStream_t s = h->stream;
  const int64_t n = h->P.n, m = h->P.m, B = h->batch;
  if (C && h->cstride == 0 && B > 1) return fail(LP_ERR_BATCH_SHAPE, "handle was created with a shared c");
  if (Q && m > 0 && h->qstride == 0 && B > 1) return fail(LP_ERR_BATCH_SHAPE, "handle was created with a shared q");
  const int64_t nc = C ? (h->cstride ? B * n : n) : 0, nq = (Q && m > 0) ? (h->qstride ? B * m : m) : 0;
  if (C) MPAX_CUDA(cudaMemcpyAsync(h->C0, C, (size_t)nc * sizeof(double), cudaMemcpyDefault, s));
  if (nq) MPAX_CUDA(cudaMemcpyAsync(h->Q0, Q, (size_t)nq * sizeof(double), cudaMemcpyDefault, s));
  // the new costs are validated like lp_create's (NaN / infinity -> LP_ERR_NAN, the handle keeps
  // no solution); synchronous, so the caller's (possibly temporary) buffers are free on return
  h->solved = false;
  if (nc + nq > 0) {
    TRY(validate_costs(h->C0, nc, h->Q0, nq, h->d_flag, s));
    MPAX_CUDA(cudaMemcpyAsync(h->h_flag, h->d_flag, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  MPAX_CUDA(cudaStreamSynchronize(s));
  if (nc + nq > 0 && h->h_flag[0] == 2)
    return fail(LP_ERR_NAN, "NaN or infinity in the updated c or q near index " + std::to_string(h->h_flag[3]));
  return LP_OK;
}

int lp_solve(lp_handle h, const lp_options *o, const double *x0, const double *y0, int32_t memory,
             lp_result *out) {
  if (h && h->batch != 1) return fail(LP_ERR_BATCH_SHAPE, "lp_solve on a batch handle; use lp_solve_batch");
  return run_solve(h, o, x0, y0, memory, out);
}

int lp_solve_batch(lp_handle h, const lp_options *o, const double *X0, const double *Y0, int32_t memory,
                   lp_result *out) {
  return run_solve(h, o, X0, Y0, memory, out);
}

int lp_spo_plus(lp_handle h, const lp_options *o, const double *C_pred, const double *C_true,
                const double *X_true, const double *obj_true, int32_t warm, int32_t memory, double *loss,
                double *grad, lp_result *out) {
  if (!h || !o || !C_pred || !C_true || !X_true || !obj_true || !loss || !grad || !out)
    return fail(LP_ERR_INVALID_ARGUMENT, "NULL argument");
  if (memory != LP_HOST && memory != LP_DEVICE) return fail(LP_ERR_INVALID_ARGUMENT, "bad memory kind");
  if (h->sharded) return fail(LP_ERR_UNSUPPORTED, "SPO+ on a sharded handle");
  const int64_t n = h->P.n, m = h->P.m, B = h->batch;
  if (B > 1 && h->cstride != n) return fail(LP_ERR_BATCH_SHAPE, "the handle shares one c; SPO+ needs per-instance costs");
  if (warm && !h->solved) return fail(LP_ERR_NOT_SOLVED, "warm start requested before any solve");
  cudaStream_t s = h->stream;
  // device views of the inputs / outputs (staged when they live on the host)
  const double *Cp = C_pred, *Ct = C_true, *Xt = X_true, *ot = obj_true;
  double *dl = loss, *dg = grad;
  if (memory == LP_HOST) {
    if (!h->spo) TRY(dalloc(&h->spo, (size_t)(4 * B * n + 2 * B), s));
    double *w = h->spo;
    double *cp = w, *ct = cp + B * n, *xt = ct + B * n, *otd = xt + B * n;
    dg = otd + B; dl = dg + B * n;
    MPAX_CUDA(cudaMemcpyAsync(cp, C_pred, (size_t)(B * n) * sizeof(double), cudaMemcpyHostToDevice, s));
    MPAX_CUDA(cudaMemcpyAsync(ct, C_true, (size_t)(B * n) * sizeof(double), cudaMemcpyHostToDevice, s));
    MPAX_CUDA(cudaMemcpyAsync(xt, X_true, (size_t)(B * n) * sizeof(double), cudaMemcpyHostToDevice, s));
    MPAX_CUDA(cudaMemcpyAsync(otd, obj_true, (size_t)B * sizeof(double), cudaMemcpyHostToDevice, s));
    Cp = cp; Ct = ct; Xt = xt; ot = otd;
  }
  const int64_t cnt = B * n;
  MPAX_LAUNCH(spo_costs_kernel, (int)std::min<int64_t>((cnt + 255) / 256, 148 * 16), 256, 0, s, cnt, Cp, Ct, h->C0);
  MPAX_CHECK_LAUNCH();
  // warm start from the previous inner solutions (copied by run_solve into its staging buffers)
  TRY(run_solve(h, o, warm ? h->X : nullptr, (warm && m > 0) ? h->Y : nullptr, LP_DEVICE, out));
  MPAX_LAUNCH(spo_loss_kernel, (int)B, 256, 0, s, n, Cp, Xt, ot, h->X, h->d_res, dl, dg);
  MPAX_CHECK_LAUNCH();
  if (memory == LP_HOST) {
    MPAX_CUDA(cudaMemcpyAsync(loss, dl, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost, s));
    MPAX_CUDA(cudaMemcpyAsync(grad, dg, (size_t)(B * n) * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  MPAX_CUDA(cudaStreamSynchronize(s));
  return LP_OK;
}

int lp_get_solution(lp_handle h, int64_t instance, double *x, double *y, double *rc, int32_t memory) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (!h->solved) return fail(LP_ERR_NOT_SOLVED, "no solve yet");
  if (h->sharded) {
    if (instance != 0) return fail(LP_ERR_BATCH_SHAPE, "instance out of range");
    const int r = sharded_get(h->sharded, x, y, rc);
    return r == LP_OK ? r : fail(r, "sharded get");
  }
  if (instance < 0 || instance >= h->batch) return fail(LP_ERR_BATCH_SHAPE, "instance out of range");
  cudaStream_t s = h->stream;
  const int64_t n = h->P.n, m = h->P.m;
  if (x) MPAX_CUDA(cudaMemcpyAsync(x, h->X + instance * n, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
  if (y && m) MPAX_CUDA(cudaMemcpyAsync(y, h->Y + instance * m, (size_t)m * sizeof(double), cudaMemcpyDefault, s));
  if (rc) MPAX_CUDA(cudaMemcpyAsync(rc, h->L + instance * n, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
  if (memory != LP_DEVICE) MPAX_CUDA(cudaStreamSynchronize(s));  // device destinations: stream-ordered
  return LP_OK;
}

int lp_get_solutions(lp_handle h, double *X, double *Y, int32_t memory) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (h->sharded) return fail(LP_ERR_UNSUPPORTED, "lp_get_solutions on a sharded handle (use lp_get_solution)");
  if (!h->solved) return fail(LP_ERR_NOT_SOLVED, "no solve yet");
  cudaStream_t s = h->stream;
  const int64_t n = h->P.n, m = h->P.m, B = h->batch;
  if (X) MPAX_CUDA(cudaMemcpyAsync(X, h->X, (size_t)(B * n) * sizeof(double), cudaMemcpyDefault, s));
  if (Y && m) MPAX_CUDA(cudaMemcpyAsync(Y, h->Y, (size_t)(B * m) * sizeof(double), cudaMemcpyDefault, s));
  if (memory != LP_DEVICE) MPAX_CUDA(cudaStreamSynchronize(s));  // device destinations: stream-ordered
  return LP_OK;
}

int lp_get_shape(lp_handle h, int64_t *n, int64_t *m1, int64_t *m2, int64_t *batch) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (h->sharded) {
    if (n) *n = sharded_n_local(h->sharded);
    if (m1) *m1 = 0;
    if (m2) *m2 = sharded_m_local(h->sharded);
    if (batch) *batch = 1;
    return LP_OK;
  }
  if (n) *n = h->P.n;
  if (m1) *m1 = h->P.m1;
  if (m2) *m2 = h->P.m2;
  if (batch) *batch = h->batch;
  return LP_OK;
}

int lp_set_decision_log_instance(lp_handle h, int64_t instance) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (instance < 0 || instance >= h->batch) return fail(LP_ERR_BATCH_SHAPE, "instance out of range");
  h->log_inst = instance;
  return LP_OK;
}

int lp_set_decision_log(lp_handle h, double *att, int64_t att_cap, double *chk, int64_t chk_cap) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if ((att && att_cap < 0) || (chk && chk_cap < 0)) return fail(LP_ERR_INVALID_ARGUMENT, "negative capacity");
  h->alog = att_cap > 0 ? att : nullptr;
  h->acap = att_cap > 0 ? att_cap : 0;
  h->clog = chk_cap > 0 ? chk : nullptr;
  h->ccap = chk_cap > 0 ? chk_cap : 0;
  if (h->sharded) sharded_set_log(h->sharded, h->alog, h->acap, h->clog, h->ccap);
  return LP_OK;
}

int lp_get_scaling(lp_handle h, double *Dr, double *Dc, int32_t memory) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (h->sharded) return fail(LP_ERR_UNSUPPORTED, "lp_get_scaling on a sharded handle");
  cudaStream_t s = h->stream;
  if (Dr && h->P.m) MPAX_CUDA(cudaMemcpyAsync(Dr, h->P.Dr, (size_t)h->P.m * sizeof(double), cudaMemcpyDefault, s));
  if (Dc) MPAX_CUDA(cudaMemcpyAsync(Dc, h->P.Dc, (size_t)h->P.n * sizeof(double), cudaMemcpyDefault, s));
  MPAX_CUDA(cudaStreamSynchronize(s));
  return LP_OK;
}

int lp_spmv_scaled(lp_handle h, const double *v, double *Kv, const double *w, double *KTw, int32_t memory) {
  if (!h) return fail(LP_ERR_INVALID_ARGUMENT, "NULL handle");
  if (h->sharded) return fail(LP_ERR_UNSUPPORTED, "lp_spmv_scaled on a sharded handle");
  cudaStream_t s = h->stream;
  const int64_t n = h->P.n, m = h->P.m;
  double *dv = nullptr, *dKv = nullptr, *dw = nullptr, *dKTw = nullptr;
  if (memory == LP_DEVICE) {  // device buffers are used in place: no staging copies
    if (!h->is_batch) TRY(grid_split_prepare(h->P, s));
    TRY(spmv_scaled(h->P, v && Kv ? v : nullptr, v && Kv ? Kv : nullptr, w && KTw ? w : nullptr,
                    w && KTw ? KTw : nullptr, s));
    MPAX_CUDA(cudaStreamSynchronize(s));
    return LP_OK;
  }
  if (v && Kv) {
    TRY(dalloc(&dv, n, s)); TRY(dalloc(&dKv, m, s));
    MPAX_CUDA(cudaMemcpyAsync(dv, v, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
  }
  if (w && KTw) {
    TRY(dalloc(&dw, m, s)); TRY(dalloc(&dKTw, n, s));
    if (m) MPAX_CUDA(cudaMemcpyAsync(dw, w, (size_t)m * sizeof(double), cudaMemcpyDefault, s));
  }
  if (!h->is_batch) TRY(grid_split_prepare(h->P, s));   // the layout the grid kernel's K~x' uses
  TRY(spmv_scaled(h->P, dv, dKv, dw, dKTw, s));
  if (dKv && m) MPAX_CUDA(cudaMemcpyAsync(Kv, dKv, (size_t)m * sizeof(double), cudaMemcpyDefault, s));
  if (dKTw) MPAX_CUDA(cudaMemcpyAsync(KTw, dKTw, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
  for (double *p : {dv, dKv, dw, dKTw})
    if (p) cudaFreeAsync(p, s);
  MPAX_CUDA(cudaStreamSynchronize(s));
  return LP_OK;
}

int lp_create_sharded(const lp_problem_desc *local_rows, int64_t global_row_offset, int64_t m1_global,
                      int64_t m2_global, void *nccl_comm, int rank, int nranks, void *cuda_stream, lp_handle *out) {
  TRY(check_desc(local_rows));
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || global_row_offset < 0 || m1_global < 0 || m2_global < 0)
    return fail(LP_ERR_INVALID_ARGUMENT, "bad sharding arguments");
  const int64_t ml = local_rows->m1 + local_rows->m2;
  const int64_t want_m1 = std::max<int64_t>(0, std::min<int64_t>(m1_global - global_row_offset, ml));
  if (local_rows->m1 != want_m1 || global_row_offset + ml > m1_global + m2_global)
    return fail(LP_ERR_DIMENSION, "local m1/m2 inconsistent with the global row split");
  if (nranks > 1 && !nccl_comm) return fail(LP_ERR_INVALID_ARGUMENT, "nccl_comm needed for nranks > 1");
  init_pool();
  lp_handle h = new lp_handle_s();
  h->stream = (cudaStream_t)cuda_stream;
  h->sharded = sharded_new(h->stream);
  std::vector<lp_problem_desc> d{*local_rows};
  std::vector<int64_t> off{global_row_offset};
  const int rc = sharded_create(h->sharded, d, off, local_rows->n, m1_global, m2_global, nccl_comm, rank, nranks,
                                false);
  if (rc != LP_OK) {
    free_handle(h);
    return fail(rc, "sharded setup failed");
  }
  *out = h;
  return LP_OK;
}

// Column split of an LP into `shards` blocks balanced by nnz (host-side CSR extraction: setup only).
static int create_virtual_cols(const lp_problem_desc *p, int32_t shards, void *cuda_stream, lp_handle *out) {
  const int64_t m = p->m1 + p->m2, n = p->n, nnz = p->nnz;
  std::vector<int64_t> rp(m + 1);
  std::vector<int32_t> ci(nnz > 0 ? nnz : 1);
  std::vector<double> v(nnz > 0 ? nnz : 1);
  if (cudaMemcpy(rp.data(), p->row_ptr, (m + 1) * sizeof(int64_t), cudaMemcpyDefault) != cudaSuccess ||
      (nnz && cudaMemcpy(ci.data(), p->col_idx, nnz * sizeof(int32_t), cudaMemcpyDefault) != cudaSuccess) ||
      (nnz && cudaMemcpy(v.data(), p->values, nnz * sizeof(double), cudaMemcpyDefault) != cudaSuccess))
    return fail(LP_ERR_CUDA, "CSR read");
  // column cut balanced by nnz: prefix of the column counts
  std::vector<int64_t> cc(n + 1, 0);
  for (int64_t k = 0; k < nnz; ++k) {
    if (ci[k] < 0 || ci[k] >= n) return fail(LP_ERR_DIMENSION, "column index out of range");
    cc[ci[k] + 1] += 1;
  }
  for (int64_t j = 0; j < n; ++j) cc[j + 1] += cc[j];
  std::vector<int64_t> cut(shards + 1, 0);
  cut[shards] = n;
  for (int g = 1; g < shards; ++g) {
    cut[g] = std::lower_bound(cc.begin(), cc.end(), nnz * g / shards) - cc.begin();
    cut[g] = std::min<int64_t>(std::max<int64_t>(cut[g], cut[g - 1]), n);
  }
  std::vector<std::vector<int64_t>> lrp(shards);
  std::vector<std::vector<int32_t>> lci(shards);
  std::vector<std::vector<double>> lv(shards);
  std::vector<lp_problem_desc> d(shards);
  std::vector<int64_t> off(shards);
  for (int g = 0; g < shards; ++g) {
    const int64_t c0 = cut[g], c1 = cut[g + 1];
    lrp[g].assign(m + 1, 0);
    for (int64_t i = 0; i < m; ++i) {
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] >= c0 && ci[k] < c1) { lci[g].push_back((int32_t)(ci[k] - c0)); lv[g].push_back(v[k]); }
      lrp[g][i + 1] = (int64_t)lci[g].size();
    }
    d[g] = *p;
    d[g].n = c1 - c0;
    d[g].nnz = (int64_t)lci[g].size();
    d[g].row_ptr = lrp[g].data();
    d[g].col_idx = lci[g].empty() ? nullptr : lci[g].data();
    d[g].values = lv[g].empty() ? nullptr : lv[g].data();
    d[g].c = p->c + c0;
    d[g].l = p->l + c0;
    d[g].u = p->u + c0;
    d[g].dense = 0;
    d[g].memory = LP_HOST;   // (sharded setup copies every array with cudaMemcpyDefault)
    off[g] = c0;
  }
  init_pool();
  lp_handle h = new lp_handle_s();
  h->stream = (cudaStream_t)cuda_stream;
  h->sharded = sharded_new(h->stream);
  const int rc = sharded_create(h->sharded, d, off, n, p->m1, p->m2, nullptr, 0, 1, true, true);
  if (rc != LP_OK) {
    free_handle(h);
    return fail(rc, "sharded setup failed");
  }
  *out = h;
  return LP_OK;
}

int lp_shard_axis(int64_t m, int64_t n) { return m < n ? LP_SHARD_COLS : LP_SHARD_ROWS; }

int lp_create_sharded_virtual_axis(const lp_problem_desc *p, int32_t shards, int32_t axis, void *cuda_stream,
                                   lp_handle *out) {
  TRY(check_desc(p));
  if (!out || shards < 1 || shards > 64) return fail(LP_ERR_INVALID_ARGUMENT, "shards must be in [1, 64]");
  if (axis == LP_SHARD_AUTO) axis = lp_shard_axis(p->m1 + p->m2, p->n);
  if (axis == LP_SHARD_COLS) {
    if (shards > p->n) return fail(LP_ERR_INVALID_ARGUMENT, "more shards than columns");
    return create_virtual_cols(p, shards, cuda_stream, out);
  }
  if (axis != LP_SHARD_ROWS) return fail(LP_ERR_INVALID_ARGUMENT, "bad axis");
  return lp_create_sharded_virtual(p, shards, cuda_stream, out);
}

int lp_create_sharded_cols(const lp_problem_desc *local_cols, int64_t global_col_offset, int64_t n_global,
                           void *nccl_comm, int rank, int nranks, void *cuda_stream, lp_handle *out) {
  TRY(check_desc(local_cols));
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || global_col_offset < 0 ||
      global_col_offset + local_cols->n > n_global)
    return fail(LP_ERR_INVALID_ARGUMENT, "bad sharding arguments");
  if (nranks > 1 && !nccl_comm) return fail(LP_ERR_INVALID_ARGUMENT, "nccl_comm needed for nranks > 1");
  init_pool();
  lp_handle h = new lp_handle_s();
  h->stream = (cudaStream_t)cuda_stream;
  h->sharded = sharded_new(h->stream);
  std::vector<lp_problem_desc> d{*local_cols};
  std::vector<int64_t> off{global_col_offset};
  const int rc = sharded_create(h->sharded, d, off, n_global, local_cols->m1, local_cols->m2, nccl_comm, rank,
                                nranks, false, true);
  if (rc != LP_OK) {
    free_handle(h);
    return fail(rc, "sharded setup failed");
  }
  *out = h;
  return LP_OK;
}

int lp_create_sharded_virtual(const lp_problem_desc *p, int32_t shards, void *cuda_stream, lp_handle *out) {
  TRY(check_desc(p));
  if (!out || shards < 1 || shards > 64) return fail(LP_ERR_INVALID_ARGUMENT, "shards must be in [1, 64]");
  const int64_t m = p->m1 + p->m2;
  // row split balanced by nnz: a cut on the row_ptr prefix
  std::vector<int64_t> rp(m + 1);
  if (cudaMemcpy(rp.data(), p->row_ptr, (m + 1) * sizeof(int64_t), cudaMemcpyDefault) != cudaSuccess)
    return fail(LP_ERR_CUDA, "row_ptr read");
  std::vector<int64_t> cut(shards + 1, 0);
  cut[shards] = m;
  for (int g = 1; g < shards; ++g) {
    const int64_t target = rp[m] * g / shards;
    cut[g] = std::lower_bound(rp.begin(), rp.end(), target) - rp.begin();
    if (cut[g] < cut[g - 1]) cut[g] = cut[g - 1];
    if (cut[g] > m) cut[g] = m;
  }
  std::vector<std::vector<int64_t>> lrp(shards);
  std::vector<lp_problem_desc> d(shards);
  std::vector<int64_t> off(shards);
  for (int g = 0; g < shards; ++g) {
    const int64_t r0 = cut[g], r1 = cut[g + 1];
    lrp[g].resize(r1 - r0 + 1);
    for (int64_t i = r0; i <= r1; ++i) lrp[g][i - r0] = rp[i] - rp[r0];
    d[g] = *p;
    d[g].m1 = std::max<int64_t>(0, std::min<int64_t>(p->m1 - r0, r1 - r0));
    d[g].m2 = (r1 - r0) - d[g].m1;
    d[g].nnz = rp[r1] - rp[r0];
    d[g].row_ptr = lrp[g].data();
    d[g].col_idx = p->col_idx + rp[r0];
    d[g].values = p->values + rp[r0];
    d[g].q = p->q + r0;
    d[g].dense = 0;
    off[g] = r0;
  }
  init_pool();
  lp_handle h = new lp_handle_s();
  h->stream = (cudaStream_t)cuda_stream;
  h->sharded = sharded_new(h->stream);
  const int rc = sharded_create(h->sharded, d, off, p->n, p->m1, p->m2, nullptr, 0, 1, true);
  if (rc != LP_OK) {
    free_handle(h);
    return fail(rc, "sharded setup failed");
  }
  *out = h;
  return LP_OK;
}

int lp_nccl_unique_id(void *out_id128) {
#ifdef MPAX_HAVE_NCCL
  if (!out_id128) return fail(LP_ERR_INVALID_ARGUMENT, "NULL id buffer");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(LP_ERR_NCCL, "ncclGetUniqueId");
  memcpy(out_id128, &id, sizeof(id));
  return LP_OK;
#else
  return fail(LP_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

int lp_nccl_comm_init(void **comm, int nranks, const void *id128, int rank) {
#ifdef MPAX_HAVE_NCCL
  if (!comm || !id128) return fail(LP_ERR_INVALID_ARGUMENT, "NULL argument");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  const ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return fail(LP_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  *comm = (void *)c;
  return LP_OK;
#else
  return fail(LP_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

int lp_nccl_comm_destroy(void *comm) {
#ifdef MPAX_HAVE_NCCL
  if (comm) ncclCommDestroy((ncclComm_t)comm);
  return LP_OK;
#else
  return fail(LP_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

int64_t lp_kernel_launch_count(void) { return g_launches.load(); }

const char *lp_error_string(int code) {
  switch (code) {
    case LP_OK: return "ok";
    case LP_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LP_ERR_DIMENSION: return "dimension / structure error";
    case LP_ERR_NAN: return "NaN or misplaced infinity";
    case LP_ERR_CROSSED_BOUNDS: return "crossed bounds";
    case LP_ERR_BATCH_SHAPE: return "batch shape error";
    case LP_ERR_OUT_OF_MEMORY: return "out of device memory";
    case LP_ERR_CUDA: return "CUDA error";
    case LP_ERR_NCCL: return "NCCL error";
    case LP_ERR_NOT_SOLVED: return "not solved";
    case LP_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown error";
  }
}

const char *lp_last_error_detail(void) { return t_detail.c_str(); }

void lp_destroy(lp_handle h) { free_handle(h); }

}  // extern "C"

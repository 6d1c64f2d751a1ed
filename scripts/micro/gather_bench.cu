// Microbenchmark (not product code): throughput of random 8-byte gathers on B200.
//
// The SpMV pair of the grid kernel reads one fp64 of x' (or y') per nonzero at a uniformly random
// column (G-RAND).  This measures how many such gathers per second the chip sustains, by load
// path and by the size of the gathered array (L1-, L2- and DRAM-resident), so that the C5 SpMV
// can be placed against the right ceiling.  Indices come from a counter hash in
// registers (no index stream) unless stated, each thread keeps U independent gathers in flight.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16; return v;
}
__device__ __forceinline__ double ld_nc_noalloc(const double *p) {
  double r; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p)); return r;
}
__device__ __forceinline__ double ld_evict_last(const double *p) {
  double r;
  asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
               "ld.global.nc.L2::cache_hint.f64 %0, [%1], pol;\n\t}" : "=d"(r) : "l"(p));
  return r;
}

enum { M_PLAIN = 0, M_LDG, M_CG, M_NOALLOC, M_TEX, M_BCAST, M_SMEM, M_STREAMIDX, M_SORTED16, M_EVLAST, M_SPMV, M_SPMV_EL, M_NMODES };
static const char *kName[M_NMODES] = {"ld.global", "ld.global.nc (__ldg)", "ld.global.cg (L2 only)",
  "ld.nc.L1::no_allocate", "tex1Dfetch<int2>", "1 line per LDG (shfl-broadcast addr)",
  "shared memory", "__ldg + streamed int32 index (SpMV-like)", "16 lanes share a 128-B line",
  "ld.nc.L2::evict_last", "SpMV-like: streamed idx+val (.cs), gather __ldg",
  "SpMV-like: streamed idx+val (.cs), gather L2::evict_last"};

template <int MODE, int U>
__global__ void __launch_bounds__(512) gather(const double *__restrict__ x, uint32_t mask, int64_t per_thread,
                                              const int32_t *__restrict__ idx, cudaTextureObject_t tex,
                                              double *out, const double *__restrict__ val) {
  extern __shared__ double sx[];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  if (MODE == M_SMEM) {
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sx[i] = x[i];
    __syncthreads();
  }
  double acc = 0;
  for (int64_t it = 0; it < per_thread; it += U) {
    uint32_t c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ctr = (uint32_t)((it + u) * nthr + tid);
      if (MODE == M_STREAMIDX || MODE == M_SPMV || MODE == M_SPMV_EL) c[u] = (uint32_t)__ldcs(idx + (it + u) * nthr + tid);
      else if (MODE == M_SORTED16) c[u] = ((mix(ctr >> 4) << 4) | (lane & 15)) & mask;
      else c[u] = (uint32_t)(((uint64_t)mix(ctr * 0x9e3779b9U + 12345U) * (mask + 1ull)) >> 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == M_PLAIN) v[u] = x[c[u]];
      else if (MODE == M_LDG || MODE == M_STREAMIDX || MODE == M_SORTED16) v[u] = __ldg(x + c[u]);
      else if (MODE == M_CG) v[u] = __ldcg(x + c[u]);
      else if (MODE == M_NOALLOC) v[u] = ld_nc_noalloc(x + c[u]);
      else if (MODE == M_EVLAST || MODE == M_SPMV_EL) v[u] = ld_evict_last(x + c[u]);
      else if (MODE == M_SPMV) v[u] = __ldg(x + c[u]);
      else if (MODE == M_TEX) { int2 t = tex1Dfetch<int2>(tex, (int)c[u]); v[u] = __hiloint2double(t.y, t.x); }
      else if (MODE == M_SMEM) v[u] = sx[c[u]];
    }
    if (MODE == M_BCAST) {
      // every LDG touches one line: lane k's address is broadcast to the warp, lane k keeps the value
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double mine = 0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const uint32_t a = __shfl_sync(0xffffffffu, c[u], k);
          const double t = __ldg(x + a);
          if (k == lane) mine = t;
        }
        v[u] = mine;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == M_SPMV || MODE == M_SPMV_EL) acc += __ldcs(val + (it + u) * nthr + tid) * v[u];
      else acc += v[u];
    }
  }
  if (acc == 12345.678) out[0] = acc;  // keep the loads alive
}

static const double *g_val = nullptr;
template <int MODE>
static int run(const double *x, uint32_t mask, const int32_t *idx, int64_t nidx, cudaTextureObject_t tex,
               double *out, int sms, float clock_ghz) {
  constexpr int U = 8;
  const int threads = 512;
  int blocks_per_sm = 2;
  size_t smem = MODE == M_SMEM ? (size_t)(mask + 1) * sizeof(double) : 0;
  if (MODE == M_SMEM) {
    CK(cudaFuncSetAttribute(gather<MODE, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    blocks_per_sm = 1;
  }
  const int blocks = sms * blocks_per_sm;
  const int64_t nthr = (int64_t)blocks * threads;
  int64_t per_thread = (nidx / nthr) / U * U;
  const double total = (double)per_thread * nthr;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaEventRecord(a));
    gather<MODE, U><<<blocks, threads, smem>>>(x, mask, per_thread, idx, tex, out, g_val);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0 && ms < best) best = ms;
  }
  const double gps = total / (best * 1e-3);
  const double cyc_per_gather_sm = sms * clock_ghz * 1e9 / gps;
  printf("{\"mode\": \"%s\", \"array_mb\": %.2f, \"gathers\": %.0f, \"ms\": %.4f, \"G_gathers_per_s\": %.2f, "
         "\"cycles_per_gather_per_sm\": %.3f, \"sector_GBps\": %.1f}\n",
         kName[MODE], (mask + 1) * 8.0 / 1e6, total, best, gps / 1e9, cyc_per_gather_sm, gps * 32 / 1e9);
  fflush(stdout);
  CK(cudaEventDestroy(a)); CK(cudaEventDestroy(b));
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const float ghz = clk_khz / 1e6f;
  const int sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_mb\": %.1f, \"clock_ghz\": %.3f}\n", prop.name, sms,
         prop.l2CacheSize / 1e6, ghz);
  const uint32_t max_elems = 1u << 26;  // 512 MB
  double *x; int32_t *idx; double *out;
  const int64_t nidx = 100000000;       // the C5 SpMV's gathers per matvec
  CK(cudaMalloc(&x, (size_t)max_elems * 8));
  CK(cudaMalloc(&idx, (size_t)nidx * 4));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, (size_t)max_elems * 8));
  double *val;
  CK(cudaMalloc(&val, (size_t)nidx * 8));
  CK(cudaMemset(val, 0, (size_t)nidx * 8));
  g_val = val;
  const bool sweep = getenv("SWEEP") != nullptr;
  const uint32_t sizes_mb_sweep[] = {32, 48, 64, 72, 80, 88, 96, 112};
  const uint32_t sizes_log2[] = {14u, 22u, 23u, 24u, 26u};
  const int nsz = sweep ? 8 : 5;
  for (int zi = 0; zi < nsz; ++zi) {
    // mask + 1 = number of elements (a power of two in the default run; any size in the sweep)
    const uint32_t mask = sweep ? (uint32_t)((uint64_t)sizes_mb_sweep[zi] * 1000000ull / 8) - 1
                                : (1u << sizes_log2[zi]) - 1;
    const uint32_t log2 = sweep ? 0u : sizes_log2[zi];
    // streamed indices for the SpMV-like mode: host-side LCG, uniform over the array
    {
      int32_t *h = (int32_t *)malloc((size_t)nidx * 4);
      uint64_t s = 88172645463325252ull;
      for (int64_t i = 0; i < nidx; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int32_t)(s % (mask + 1ull)); }
      CK(cudaMemcpy(idx, h, (size_t)nidx * 4, cudaMemcpyHostToDevice));
      free(h);
    }
    if (sweep) {
      if (run<M_LDG>(x, mask, idx, nidx, 0, out, sms, ghz)) return 1;
      if (run<M_SPMV>(x, mask, idx, nidx, 0, out, sms, ghz)) return 1;
      if (run<M_SPMV_EL>(x, mask, idx, nidx, 0, out, sms, ghz)) return 1;
      continue;
    }
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = x;
    rd.res.linear.desc = cudaCreateChannelDesc<int2>();
    rd.res.linear.sizeInBytes = (size_t)(mask + 1) * 8;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    const bool tex_ok = cudaCreateTextureObject(&tex, &rd, &td, nullptr) == cudaSuccess;
    cudaGetLastError();
    if (run<M_PLAIN>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_LDG>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_CG>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_NOALLOC>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_EVLAST>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (tex_ok && run<M_TEX>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_BCAST>(x, mask, idx, nidx / 4, tex, out, sms, ghz)) return 1;
    if (run<M_STREAMIDX>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (run<M_SORTED16>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (log2 == 14 && run<M_SMEM>(x, mask, idx, nidx, tex, out, sms, ghz)) return 1;
    if (tex_ok) cudaDestroyTextureObject(tex);
  }
  return 0;
}

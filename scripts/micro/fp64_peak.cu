// fp64 peak microbenchmarks for the roofline denominators ("fp64 DFMA and DMMA
// peaks are measured by the build on the box"):
//   dfma: every thread runs 8 independent DFMA chains (a = a * b + c), all SMs, 8 warps/SMSP;
//   dmma: every warp runs 8 independent mma.sync.m8n8k4.f64 accumulator chains (512 flop each).
// Prints one JSON line: TFLOP/s best of 10 (CUDA events), SM clock read via nvml is not needed:
// the driver's clocks are recorded by bench.py's sampler in the same run.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double *out, int iters, double a, double b) {
  double d0[8], d1[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { d0[k] = 0.0; d1[k] = 0.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d0[k], d1[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d0[k] + d1[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks_per_sm = 8, iters = 20000;
  const int blocks = sms * blocks_per_sm;
  double best_dfma = 0.0, best_dmma = 0.0;
  for (int rep = 0; rep < 11; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
    if (rep) best_dfma = fmax(best_dfma, flops / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4, 0.5, 0.25);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dflops = 512.0 * 8.0 * (iters / 4) * (double)(threads / 32) * blocks;
    if (rep) best_dmma = fmax(best_dmma, dflops / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"error\": \"%s\", "
         "\"how\": \"dfma: 8 independent chains/thread, %d CTAs x %d threads; dmma: mma.sync.m8n8k4.f64, 8 "
         "accumulator chains/warp; best of 10, CUDA events\"}\n",
         best_dfma, best_dmma, sms, cudaGetErrorString(err), blocks, threads);
  return err == cudaSuccess ? 0 : 1;
}

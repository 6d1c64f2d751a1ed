// Microbenchmark (not product code): cost of a cooperative-groups grid barrier on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, double *out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}
int main() {
  double *out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bs : {256, 512, 1024}) for (int per : {1, 2}) {
    if (bs * per > 2048) continue;
    int iters = 2000; void *args[] = {&iters, &out};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)k_sync, sms * per, bs, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, sms * per, bs, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("blocks=%d x %d threads: %.3f us per grid.sync (%s)\n", sms * per, bs, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// selftest.cu -- lp_selftest_division (include/lp.h): bitwise check of div_rn_fast against the
// compiler's IEEE `a / b` on device-generated operands.
#include "common.cuh"

namespace mpax {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ double operand(uint64_t h) {
  const unsigned kind = (unsigned)(h >> 59);  // 32 kinds
  if (kind == 0) return 0.0;
  if (kind == 1) return -0.0;
  if (kind == 2) return INFINITY;
  if (kind == 3) return -INFINITY;
  if (kind == 4) return NAN;
  if (kind == 5) return __longlong_as_double((long long)(h & 0x000fffffffffffffull));  // subnormal
  uint64_t bits = h & 0x800fffffffffffffull;                                             // sign + mantissa
  uint64_t e;
  if (kind < 20) e = 1 + (mix64(h) % 2046);        // any finite exponent
  else e = 1023 - 40 + (mix64(h) % 80);             // the solver's range, about 2^-40 .. 2^40
  return __longlong_as_double((long long)(bits | (e << 52)));
}

__global__ void div_selftest_kernel(int64_t count, uint64_t seed, unsigned long long *mism,
                                    unsigned long long *slow) {
  unsigned long long my_m = 0, my_s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    // every fourth pair divides 1.0 (the reciprocals of the scaling rounds)
    const double a = (i & 3) == 0 ? 1.0 : operand(mix64(seed ^ (2 * (uint64_t)i)));
    const double b = operand(mix64(seed ^ (2 * (uint64_t)i + 1) ^ 0x9e3779b97f4a7c15ull));
    bool ok;
    const double q = div_rn_fast(a, b, ok);
    const double r = a / b;
    if (!ok) ++my_s;
    else if (__double_as_longlong(q) != __double_as_longlong(r) && !(isnan(q) && isnan(r))) ++my_m;
  }
  atomicAdd(mism, my_m);
  atomicAdd(slow, my_s);
}

}  // namespace
}  // namespace mpax

using namespace mpax;

extern "C" int lp_selftest_division(int64_t count, uint64_t seed, int64_t *mismatches, int64_t *slow) {
  if (!mismatches || !slow || count < 0) return LP_ERR_INVALID_ARGUMENT;
  unsigned long long *d = nullptr;
  MPAX_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
  MPAX_CUDA(cudaMemset(d, 0, 2 * sizeof(unsigned long long)));
  MPAX_LAUNCH(div_selftest_kernel, 148 * 8, 256, 0, (cudaStream_t)0, count, seed, d, d + 1);
  MPAX_CHECK_LAUNCH();
  unsigned long long h[2];
  MPAX_CUDA(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  MPAX_CUDA(cudaFree(d));
  *mismatches = (int64_t)h[0];
  *slow = (int64_t)h[1];
  return LP_OK;
}

// Microbenchmark (not product code): CSR SpMV mappings on B200 for G-RAND-like matrices.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

__global__ void k_g1(int m, const int *rp, const int *ci, const double *v, const double *x, double *y) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    int p = rp[r], e = rp[r + 1];
    double s0 = 0, s1 = 0;
    for (; p + 3 < e; p += 4) {
      int c0 = __ldcs(ci + p), c1 = __ldcs(ci + p + 1), c2 = __ldcs(ci + p + 2), c3 = __ldcs(ci + p + 3);
      double w0 = __ldcs(v + p), w1 = __ldcs(v + p + 1), w2 = __ldcs(v + p + 2), w3 = __ldcs(v + p + 3);
      s0 += w0 * x[c0]; s1 += w1 * x[c1]; s0 += w2 * x[c2]; s1 += w3 * x[c3];
    }
    for (; p < e; ++p) s0 += __ldcs(v + p) * x[__ldcs(ci + p)];
    y[r] = s0 + s1;
  }
}
template <int G>
__global__ void k_g(int m, const int *rp, const int *ci, const double *v, const double *x, double *y) {
  int gt = blockIdx.x * blockDim.x + threadIdx.x, ng = gridDim.x * blockDim.x / G, g = gt / G, l = gt % G;
  int iters = (m + ng - 1) / ng;
  for (int it = 0; it < iters; ++it) {
    int r = it * ng + g;
    double s = 0;
    if (r < m) { int e = rp[r + 1]; for (int p = rp[r] + l; p < e; p += G) s += __ldcs(v + p) * x[__ldcs(ci + p)]; }
    for (int off = G / 2; off; off >>= 1) s += __shfl_xor_sync(0xffffffff, s, off);
    if (r < m && l == 0) y[r] = s;
  }
}
// warp per 32 rows, cooperative: the warp streams the contiguous nnz range of its rows (coalesced), segmented sum via smem
template <int RPW>
__global__ void k_seg(int m, const int *rp, const int *ci, const double *v, const double *x, double *y) {
  // each warp takes RPW consecutive rows; lanes stride over the contiguous nnz range; per-entry row via search
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31, nw = gridDim.x * blockDim.x >> 5;
  for (int r0 = warp * RPW; r0 < m; r0 += nw * RPW) {
    int r1 = min(r0 + RPW, m);
    int a = rp[r0], b = rp[r1];
    // each lane owns rows r0+lane (RPW==32): compute its own sum from the coalesced pass
    double acc = 0;
    int myrow = r0 + lane, ms = myrow < r1 ? rp[myrow] : b, me = myrow < r1 ? rp[myrow + 1] : b;
    for (int base = a; base < b; base += 32) {
      int p = base + lane;
      double prod = 0; 
      if (p < b) prod = __ldcs(v + p) * x[__ldcs(ci + p)];
      // distribute: every lane sums the products that fall in its row range
      for (int t = 0; t < 32; ++t) {
        double pv = __shfl_sync(0xffffffff, prod, t);
        int pp = base + t;
        if (pp >= ms && pp < me) acc += pv;
      }
    }
    if (myrow < r1) y[myrow] = acc;
  }
}

int main(int argc, char **argv) {
  for (int m : {100000, 1000000}) {
    int n = 2 * m, r = 20;
    std::mt19937 gen(1);
    std::vector<int> rp(m + 1), ci((size_t)m * r);
    for (int i = 0; i <= m; ++i) rp[i] = i * r;
    for (int i = 0; i < m; ++i) {
      for (int k = 0; k < r; ++k) ci[(size_t)i * r + k] = gen() % n;
      std::sort(ci.begin() + (size_t)i * r, ci.begin() + (size_t)(i + 1) * r);
    }
    std::vector<double> v((size_t)m * r, 1.0), x(n, 1.0);
    int *drp, *dci; double *dv, *dx, *dy;
    cudaMalloc(&drp, (m + 1) * 4); cudaMalloc(&dci, (size_t)m * r * 4); cudaMalloc(&dv, (size_t)m * r * 8);
    cudaMalloc(&dx, n * 8); cudaMalloc(&dy, m * 8);
    cudaMemcpy(drp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dci, ci.data(), (size_t)m * r * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), (size_t)m * r * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
    double bytes = (double)m * r * 12 + (m + 1) * 4 + m * 8 + n * 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
      for (int w = 0; w < 3; ++w) launch();
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) launch();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double us = ms * 1e3 / 20;
      printf("m=%d %-22s %8.2f us  %7.1f GB/s (%s)\n", m, name, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    int sms = 148;
    run("g1 148x4x256", [&] { k_g1<<<sms * 4, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g1 148x8x256", [&] { k_g1<<<sms * 8, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g1 full grid", [&] { k_g1<<<(m + 255) / 256, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g4 148x4x256", [&] { k_g<4><<<sms * 4, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g4 full grid", [&] { k_g<4><<<(m * 4 + 255) / 256, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g8 full grid", [&] { k_g<8><<<(m * 8 + 255) / 256, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g32 full grid", [&] { k_g<32><<<(m * 32 + 255) / 256, 256>>>(m, drp, dci, dv, dx, dy); });
    run("g8 148x8x256", [&] { k_g<8><<<sms * 8, 256>>>(m, drp, dci, dv, dx, dy); });
    run("seg32 148x8x256", [&] { k_seg<32><<<sms * 8, 256>>>(m, drp, dci, dv, dx, dy); });
    cudaFree(drp); cudaFree(dci); cudaFree(dv); cudaFree(dx); cudaFree(dy);
  }
  return 0;
}

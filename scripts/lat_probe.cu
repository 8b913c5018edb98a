// Dependent-chain latencies on one warp (cycles per op): DFMA, DADD, DMUL, rsqrt(double),
// 64-bit shuffle, shared-memory load, L2 load (ld.global.cg).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, const double* gmem, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane; sm[lane + 32] = lane;
  __syncwarp();
  double x = 1.0 + lane * 1e-9, y = 0.999999;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); if (lane == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + y;
  t1 = clock64(); if (lane == 0) cyc[1] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64(); if (lane == 0) cyc[2] = t1 - t0;
  // 64-bit shuffle chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64(); if (lane == 0) cyc[3] = t1 - t0;
  // shared load chain
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x += sm[idx]; idx = ((int)x & 31); }
  t1 = clock64(); if (lane == 0) cyc[4] = t1 - t0;
  // L2 load chain (pointer chase through gmem with .cg)
  long long p = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double v = __ldcg(gmem + p); p = (long long)v; }
  t1 = clock64(); if (lane == 0) cyc[5] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * y;
  t1 = clock64(); if (lane == 0) cyc[6] = t1 - t0;
  // double division chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 2.0);
  t1 = clock64(); if (lane == 0) cyc[7] = t1 - t0;
  out[lane] = x + (double)p;
}

int main() {
  double *out, *g;
  long long* cyc;
  cudaMalloc(&out, 256 * 8);
  cudaMalloc(&cyc, 16 * 8);
  const int N = 1 << 20;
  cudaMalloc(&g, N * 8);
  double* h = new double[N];
  for (long long i = 0; i < N; ++i) h[i] = (double)((i * 7919LL + 4099LL) % N);
  cudaMemcpy(g, h, N * 8, cudaMemcpyHostToDevice);
  const int iters = 1000;
  lat<<<1, 32>>>(out, cyc, g, 10);
  lat<<<1, 32>>>(out, cyc, g, iters);
  long long c[8];
  cudaMemcpy(c, cyc, 64, cudaMemcpyDeviceToHost);
  const char* names[8] = {"dfma", "dadd", "rsqrt+add", "shfl64", "lds+dadd", "ldg.cg (L2/HBM chase)", "dmul", "div+add"};
  for (int k = 0; k < 8; ++k) printf("%-24s %8.1f cycles/op\n", names[k], (double)c[k] / iters);
  return 0;
}

// FP64 tensor-pipe (DMMA m8n8k4) peak microbenchmark for the roofline denominator of
// the q-space Gram.  Every warp runs a long chain of independent mma.sync f64 ops on
// register operands (no memory traffic); grid = SMs x blocks_per_sm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
// Also times plain FP64 FMA (DFMA) throughput the same way.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_loop(int iters, double* out) {
  double c[CHAINS][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(int iters, double* out) {
  double c[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma(a, c[k], b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best = 0.0;
  int best_cfg = 0;
  for (int bps : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      dmma_loop<8><<<sms * bps, threads>>>(100, out);
      cudaEventRecord(e0);
      dmma_loop<8><<<sms * bps, threads>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)sms * bps * threads / 32.0;
      const double flops = warps * iters * 8 * 512.0;
      const double tf = flops / (ms * 1e-3) / 1e12;
      std::printf("dmma blocks/SM=%d threads=%d: %.3f ms  %.2f TFLOP/s\n", bps, threads, ms, tf);
      if (tf > best) { best = tf; best_cfg = bps * 1000 + threads; }
    }
  }
  double best_fma = 0.0;
  for (int bps : {2, 4, 8}) {
    dfma_loop<<<sms * bps, 256>>>(100, out);
    cudaEventRecord(e0);
    dfma_loop<<<sms * bps, 256>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)sms * bps * 256 * iters * 8 * 2.0;
    const double tf = flops / (ms * 1e-3) / 1e12;
    std::printf("dfma blocks/SM=%d: %.3f ms  %.2f TFLOP/s\n", bps, ms, tf);
    if (tf > best_fma) best_fma = tf;
  }
  std::printf("{\"dmma_f64_tflops\": %.3f, \"dfma_f64_tflops\": %.3f, \"sms\": %d, \"cfg\": %d}\n",
              best, best_fma, sms, best_cfg);
  return 0;
}

// Cost of factoring one 32 x 32 SPD diagonal block by one warp (lane = row, registers):
//   A: bg_diag_step (column broadcast by 64-bit shuffles, csrc/linalg.cu)
//   B: column broadcast through shared memory (one STS + broadcast LDS per column)
#include <cstdio>
#include <cstdlib>

namespace ssnal {
void note_launch() {}
}
#include "../paper_1910_01312_b200/csrc/linalg.cu"

template <int J>
__device__ __forceinline__ void sm_diag_step(double (&r)[32], int lane, double* rd, double (*colbuf)[32]) {
  double d = __shfl_sync(0xffffffffu, r[J], J);
  if (!(d > 0.0)) d = 1.0;
  const double inv = rsqrt(d);
  if (lane == J) { r[J] = d * inv; rd[J] = inv; }
  else if (lane > J) r[J] *= inv;
  colbuf[J & 1][lane] = r[J];
  __syncwarp();
#pragma unroll
  for (int c = J + 1; c < 32; ++c) {
    const double lcj = colbuf[J & 1][c];
    if (lane >= c) r[c] = fma(-r[J], lcj, r[c]);
  }
  if constexpr (J + 1 < 32) sm_diag_step<J + 1>(r, lane, rd, colbuf);
}

__global__ void probe(const double* A, double* out, long long* cyc, int reps, int variant) {
  __shared__ double rd[32];
  __shared__ double colbuf[2][32];
  __shared__ int fail;
  const int lane = threadIdx.x;
  if (lane == 0) fail = 0;
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    double r[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = c <= lane ? A[lane * 32 + c] + it * 1e-30 : 0.0;
    if (variant == 0) ssnal::bg_diag_step<0>(r, lane, rd, 0, &fail, __shfl_sync(0xffffffffu, r[0], 0), colbuf);
    else sm_diag_step<0>(r, lane, rd, colbuf);
#pragma unroll
    for (int c = 0; c < 32; ++c) acc += r[c];
  }
  long long t1 = clock64();
  out[lane] = acc;
  if (lane == 0) *cyc = t1 - t0;
}

int main() {
  double h[32 * 32];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *dA, *dout;
  long long* dc;
  cudaMalloc(&dA, sizeof(h));
  cudaMalloc(&dout, 256);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int v = 0; v < 2; ++v) {
    probe<<<1, 32>>>(dA, dout, dc, 2, v);
    probe<<<1, 32>>>(dA, dout, dc, 50, v);
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("variant %s: %.0f cycles per 32x32 block (%.2f us at 1.965 GHz)\n",
           v ? "smem-broadcast" : "shuffle (bg_diag_step)", c / 50.0, c / 50.0 / 1965.0);
  }
  return 0;
}

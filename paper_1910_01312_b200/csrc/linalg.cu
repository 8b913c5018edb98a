// Dense SPD solve for the reduced Newton system: blocked right-looking Cholesky
// (32-column panels; diagonal block by one warp with shuffles, panel TRSM one row
// per thread, trailing SYRK update from a shared-memory copy of the panel),
// followed by blocked forward / backward substitution -- all inside ONE CTA so
// the factor never leaves L2 and no host round trip is needed.
// Replaces scipy.linalg.solve(..., assume_a="sym") of ref solver.py:175-191.
#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

static constexpr int NB = 32;
static constexpr int CH_NT = 1024;
static constexpr int PANEL_ROWS = 768;  // panel rows kept in shared memory (stride NB+1)

__global__ void __launch_bounds__(CH_NT, 1) chol_solve_kernel(double* __restrict__ M, long long m,
                                                                const double* __restrict__ b,
                                                                double scale, double* __restrict__ x,
                                                                int* __restrict__ info) {
  extern __shared__ double smem[];
  double* D = smem;                       // NB x (NB+1) diagonal block
  double* P = smem + NB * (NB + 1);       // panel rows x (NB+1)
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) fail = 0;
  __syncthreads();
  for (long long k0 = 0; k0 < m; k0 += NB) {
    const int kb = (int)min((long long)NB, m - k0);
    // 1. diagonal block -> D, factor with warp 0
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      int i = idx / kb, j = idx % kb;
      D[i * (NB + 1) + j] = M[(k0 + i) * m + k0 + j];
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = 0; j < kb; ++j) {
        // lane i (>= j) owns row i of the current column
        double dj = D[j * (NB + 1) + j];
        if (dj <= 0.0 || !(dj == dj)) {
          if (lane == 0 && fail == 0) fail = (int)(k0 + j + 1);
          dj = 1.0;
        }
        double ljj = sqrt(dj);
        __syncwarp();
        if (lane == j) D[j * (NB + 1) + j] = ljj;
        if (lane > j && lane < kb) D[lane * (NB + 1) + j] /= ljj;
        __syncwarp();
        // rank-1 update of the remaining lower block: rows lane, cols j+1..lane
        if (lane > j && lane < kb) {
          double lij = D[lane * (NB + 1) + j];
          for (int c = j + 1; c <= lane; ++c) D[lane * (NB + 1) + c] -= lij * D[c * (NB + 1) + j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      int i = idx / kb, j = idx % kb;
      if (j <= i) M[(k0 + i) * m + k0 + j] = D[i * (NB + 1) + j];
    }
    // 2. panel solve: rows below, L21 = A21 L11^{-T}; one thread per row
    const long long r0 = k0 + kb;
    const long long nr = m - r0;
    const bool in_smem = nr <= PANEL_ROWS;
    for (long long i = tid; i < nr; i += blockDim.x) {
      double row[NB];
      const long long gi = r0 + i;
      for (int j = 0; j < kb; ++j) row[j] = M[gi * m + k0 + j];
      for (int j = 0; j < kb; ++j) {
        double s = row[j];
        for (int t = 0; t < j; ++t) s -= row[t] * D[j * (NB + 1) + t];
        row[j] = s / D[j * (NB + 1) + j];
      }
      for (int j = 0; j < kb; ++j) {
        M[gi * m + k0 + j] = row[j];
        if (in_smem) P[i * (NB + 1) + j] = row[j];
      }
    }
    __syncthreads();
    // 3. trailing update (lower triangle): A22 -= L21 L21^T
    const double* Lp = in_smem ? P : nullptr;
    for (long long i = warp; i < nr; i += (CH_NT / 32)) {
      for (long long j = lane; j <= i; j += 32) {
        double s = 0.0;
        if (in_smem) {
          for (int t = 0; t < kb; ++t) s += Lp[i * (NB + 1) + t] * Lp[j * (NB + 1) + t];
        } else {
          for (int t = 0; t < kb; ++t) s += M[(r0 + i) * m + k0 + t] * M[(r0 + j) * m + k0 + t];
        }
        M[(r0 + i) * m + r0 + j] -= s;
      }
    }
    __syncthreads();
  }
  // forward substitution  L y = scale * b   (y kept in x)
  for (long long i = tid; i < m; i += blockDim.x) x[i] = scale * b[i];
  __syncthreads();
  for (long long k0 = 0; k0 < m; k0 += NB) {
    const int kb = (int)min((long long)NB, m - k0);
    // stage the diagonal block of L in shared memory: the warp-serial solve below
    // then waits on smem (~30 cycles) instead of L2 (~600) per step
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      int i = idx / kb, j = idx % kb;
      D[i * (NB + 1) + j] = j <= i ? M[(k0 + i) * m + k0 + j] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      double yv = lane < kb ? x[k0 + lane] : 0.0;
      for (int j = 0; j < kb; ++j) {
        if (lane == j) yv = yv / D[j * (NB + 1) + j];
        const double yj = __shfl_sync(0xffffffffu, yv, j);
        if (lane > j && lane < kb) yv -= D[lane * (NB + 1) + j] * yj;
      }
      if (lane < kb) x[k0 + lane] = yv;
    }
    __syncthreads();
    for (long long i = k0 + kb + tid; i < m; i += blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < kb; ++t) s += M[i * m + k0 + t] * x[k0 + t];
      x[i] -= s;
    }
    __syncthreads();
  }
  // backward substitution  L^T x = y
  const long long nblk = ceil_div(m, NB);
  for (long long bk = nblk - 1; bk >= 0; --bk) {
    const long long k0 = bk * NB;
    const int kb = (int)min((long long)NB, m - k0);
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      int i = idx / kb, j = idx % kb;
      D[i * (NB + 1) + j] = j <= i ? M[(k0 + i) * m + k0 + j] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      double xv = lane < kb ? x[k0 + lane] : 0.0;
      for (int j = kb - 1; j >= 0; --j) {
        if (lane == j) xv = xv / D[j * (NB + 1) + j];
        const double xj = __shfl_sync(0xffffffffu, xv, j);
        if (lane < j) xv -= D[j * (NB + 1) + lane] * xj;
      }
      if (lane < kb) x[k0 + lane] = xv;
    }
    __syncthreads();
    for (long long i = tid; i < k0; i += blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < kb; ++t) s += M[(k0 + t) * m + i] * x[k0 + t];
      x[i] -= s;
    }
    __syncthreads();
  }
  if (tid == 0) *info = fail;
}

// Small systems (m <= SMALL_M): the whole lower triangle lives in shared memory
// (odd row stride: conflict-free column access), right-looking column Cholesky
// with all 1024 threads on the trailing update, then column-sweep substitutions.
static constexpr int SMALL_M = 160;

static constexpr int SM_NT = 512;  // 128 registers/thread: the 32-double row of warp 0 stays in RF

__global__ void __launch_bounds__(SM_NT, 1) chol_small_kernel(const double* __restrict__ M, int m,
                                                                const double* __restrict__ b,
                                                                double scale,
                                                                double* __restrict__ x,
                                                                int* __restrict__ info) {
  extern __shared__ double S[];
  const int ld = m | 1;
  double* y = S + (size_t)m * ld;
  __shared__ int fail;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  if (tid == 0) fail = 0;
  for (int idx = tid; idx < m * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    if (j <= i) S[i * ld + j] = M[(long long)i * m + j];
  }
  for (int i = tid; i < m; i += blockDim.x) y[i] = scale * b[i];
  __syncthreads();
  const int lane = tx, warp = ty;
  __shared__ double rdiag[32];
  for (int k0 = 0; k0 < m; k0 += 32) {
    const int kb = min(32, m - k0);
    // (1) diagonal block, 2-D parallel over its (i, c) pairs: per column one barrier
    //     for the scaled column, one for the rank-1 update (every thread recomputes
    //     the pivot sqrt itself instead of waiting on a broadcast)
    for (int j = 0; j < kb; ++j) {
      double d = S[(k0 + j) * ld + k0 + j];
      if (!(d > 0.0)) {
        if (tid == 0 && fail == 0) fail = k0 + j + 1;
        d = 1.0;
      }
      const double ljj = sqrt(d);
      __syncthreads();  // everyone has read the pivot before it is overwritten
      if (tid == 0) {
        S[(k0 + j) * ld + k0 + j] = ljj;
        rdiag[j] = 1.0 / ljj;
      }
      for (int i = k0 + j + 1 + tid; i < k0 + kb; i += blockDim.x) S[i * ld + k0 + j] /= ljj;
      __syncthreads();
      const int r = kb - j - 1;  // trailing rows inside the block
      for (int idx = tid; idx < r * r; idx += blockDim.x) {
        const int ii = idx / r, cc = idx % r;
        if (cc <= ii) {
          const int i = k0 + j + 1 + ii, c = k0 + j + 1 + cc;
          S[i * ld + c] = fma(-S[i * ld + k0 + j], S[c * ld + k0 + j], S[i * ld + c]);
        }
      }
    }
    (void)lane;
    (void)warp;
    __syncthreads();
    // (2) panel: L21 = A21 L11^{-T}, one thread per row (reciprocal diagonal)
    for (int i = k0 + kb + tid; i < m; i += blockDim.x) {
      double* row = S + i * ld + k0;
      for (int j = 0; j < kb; ++j) {
        double s = row[j];
        const double* lj = S + (k0 + j) * ld + k0;
        for (int t = 0; t < j; ++t) s = fma(-row[t], lj[t], s);
        row[j] = s * rdiag[j];
      }
    }
    __syncthreads();
    // (3) trailing update A22 -= L21 L21^T (lower triangle)
    for (int i = k0 + kb + ty; i < m; i += SM_NT / 32) {
      const double* li = S + i * ld + k0;
      for (int c = k0 + kb + tx; c <= i; c += 32) {
        const double* lc = S + c * ld + k0;
        double s = 0.0;
        for (int t = 0; t < kb; ++t) s = fma(li[t], lc[t], s);
        S[i * ld + c] -= s;
      }
    }
    __syncthreads();
  }
  // forward L z = y and backward L^T x = z: diagonal block by warp 0 with shuffles,
  // off-diagonal updates by all threads
  for (int k0 = 0; k0 < m; k0 += 32) {
    const int kb = min(32, m - k0);
    if (warp == 0) {
      double yv = lane < kb ? y[k0 + lane] : 0.0;
      for (int j = 0; j < kb; ++j) {
        if (lane == j) yv = yv / S[(k0 + j) * ld + k0 + j];
        const double yj = __shfl_sync(0xffffffffu, yv, j);
        if (lane > j && lane < kb) yv = fma(-S[(k0 + lane) * ld + k0 + j], yj, yv);
      }
      if (lane < kb) y[k0 + lane] = yv;
    }
    __syncthreads();
    for (int i = k0 + kb + tid; i < m; i += blockDim.x) {
      double s = y[i];
      for (int t = 0; t < kb; ++t) s = fma(-S[i * ld + k0 + t], y[k0 + t], s);
      y[i] = s;
    }
    __syncthreads();
  }
  for (int k0 = ((m - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
    const int kb = min(32, m - k0);
    if (warp == 0) {
      double xv = lane < kb ? y[k0 + lane] : 0.0;
      for (int j = kb - 1; j >= 0; --j) {
        if (lane == j) xv = xv / S[(k0 + j) * ld + k0 + j];
        const double xj = __shfl_sync(0xffffffffu, xv, j);
        if (lane < j) xv = fma(-S[(k0 + j) * ld + k0 + lane], xj, xv);
      }
      if (lane < kb) y[k0 + lane] = xv;
    }
    __syncthreads();
    for (int i = tid; i < k0; i += blockDim.x) {
      double s = y[i];
      for (int t = 0; t < kb; ++t) s = fma(-S[(k0 + t) * ld + i], y[k0 + t], s);
      y[i] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < m; i += blockDim.x) x[i] = y[i];
  if (tid == 0) *info = fail;
}

// Blocked (NB = 16) shared-memory Cholesky + solves for m <= SMALL_M.
//  - 16 x 16 diagonal blocks: warp 0, lane i holds row i in registers; pivots by
//    shuffle, rsqrt, no block barrier inside the block;
//  - panel: one thread per row below, the 16-wide row in registers, reciprocal
//    pivots (16-step dependent chain);
//  - trailing update: each thread keeps one L row (16 values) in registers and
//    sweeps columns, one shared load per FMA;
//  - substitutions: 16-row diagonal blocks by warp 0 with shuffles, off-diagonal
//    updates by all threads.  Three block barriers per 16 columns.
constexpr int NB16 = 16;

__device__ __forceinline__ void warp_chol16(double* S, int ld, int k0, int kb, int lane,
                                            double* rdiag, int* fail) {
  double r[NB16];
#pragma unroll
  for (int c = 0; c < NB16; ++c)
    r[c] = (lane < kb && c <= lane) ? S[(k0 + lane) * ld + k0 + c] : (c == lane ? 1.0 : 0.0);
  double mydiag = 1.0;
#pragma unroll
  for (int j = 0; j < NB16; ++j) {
    double d = __shfl_sync(0xffffffffu, r[j], j);
    if (j < kb && !(d > 0.0)) {
      if (lane == 0 && *fail == 0) *fail = k0 + j + 1;
      d = 1.0;
    }
    const double inv = rsqrt(d);
    const double ljj = d * inv;
    if (lane == j) mydiag = ljj;
    r[j] = (lane == j) ? ljj : r[j] * inv;
#pragma unroll
    for (int c = j + 1; c < NB16; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, r[j], c);
      if (lane >= c) r[c] = fma(-r[j], lcj, r[c]);
    }
  }
  if (lane < kb) {
#pragma unroll
    for (int c = 0; c < NB16; ++c)
      if (c <= lane) S[(k0 + lane) * ld + k0 + c] = r[c];
    rdiag[lane] = 1.0 / mydiag;
  }
}

__global__ void __launch_bounds__(SM_NT, 1) chol_small16_kernel(const double* __restrict__ M, int m,
                                                                  const double* __restrict__ b,
                                                                  double scale,
                                                                  double* __restrict__ x,
                                                                  int* __restrict__ info) {
  extern __shared__ double S[];
  const int ld = m | 1;
  double* y = S + (size_t)m * ld;
  __shared__ int fail;
  __shared__ double rdiag[NB16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) fail = 0;
  for (int idx = tid; idx < m * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    if (j <= i) S[i * ld + j] = M[(long long)i * m + j];
  }
  for (int i = tid; i < m; i += blockDim.x) y[i] = scale * b[i];
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += NB16) {
    const int kb = min(NB16, m - k0);
    if (warp == 0) warp_chol16(S, ld, k0, kb, lane, rdiag, &fail);
    __syncthreads();
    // panel rows below: L21 = A21 L11^{-T}
    for (int i = k0 + kb + tid; i < m; i += blockDim.x) {
      double row[NB16];
#pragma unroll
      for (int j = 0; j < NB16; ++j) row[j] = j < kb ? S[i * ld + k0 + j] : 0.0;
#pragma unroll
      for (int j = 0; j < NB16; ++j) {
        if (j < kb) {
          double s = row[j];
#pragma unroll
          for (int t = 0; t < j; ++t) s = fma(-row[t], S[(k0 + j) * ld + k0 + t], s);
          row[j] = s * rdiag[j];
        }
      }
#pragma unroll
      for (int j = 0; j < NB16; ++j)
        if (j < kb) S[i * ld + k0 + j] = row[j];
    }
    __syncthreads();
    // trailing update A22 -= L21 L21^T: thread (rows by warp, columns by lane)
    const int r0 = k0 + kb;
    for (int i = r0 + warp; i < m; i += SM_NT / 32) {
      double li[NB16];
#pragma unroll
      for (int t = 0; t < NB16; ++t) li[t] = t < kb ? S[i * ld + k0 + t] : 0.0;
      for (int c = r0 + lane; c <= i; c += 32) {
        const double* lc = S + c * ld + k0;
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < NB16; ++t)
          if (t < kb) s = fma(li[t], lc[t], s);
        S[i * ld + c] -= s;
      }
    }
    __syncthreads();
  }
  // forward L z = y
  for (int k0 = 0; k0 < m; k0 += NB16) {
    const int kb = min(NB16, m - k0);
    if (warp == 0) {
      double yv = lane < kb ? y[k0 + lane] : 0.0;
      const double lrow_diag = lane < kb ? S[(k0 + lane) * ld + k0 + lane] : 1.0;
#pragma unroll
      for (int j = 0; j < NB16; ++j) {
        if (j < kb) {
          if (lane == j) yv = yv / lrow_diag;
          const double yj = __shfl_sync(0xffffffffu, yv, j);
          if (lane > j && lane < kb) yv = fma(-S[(k0 + lane) * ld + k0 + j], yj, yv);
        }
      }
      if (lane < kb) y[k0 + lane] = yv;
    }
    __syncthreads();
    for (int i = k0 + kb + tid; i < m; i += blockDim.x) {
      double s = y[i];
#pragma unroll
      for (int t = 0; t < NB16; ++t)
        if (t < kb) s = fma(-S[i * ld + k0 + t], y[k0 + t], s);
      y[i] = s;
    }
    __syncthreads();
  }
  // backward L^T x = z
  for (int k0 = ((m - 1) / NB16) * NB16; k0 >= 0; k0 -= NB16) {
    const int kb = min(NB16, m - k0);
    if (warp == 0) {
      double xv = lane < kb ? y[k0 + lane] : 0.0;
      const double ldiag = lane < kb ? S[(k0 + lane) * ld + k0 + lane] : 1.0;
#pragma unroll
      for (int j = NB16 - 1; j >= 0; --j) {
        if (j < kb) {
          if (lane == j) xv = xv / ldiag;
          const double xj = __shfl_sync(0xffffffffu, xv, j);
          if (lane < j) xv = fma(-S[(k0 + j) * ld + k0 + lane], xj, xv);
        }
      }
      if (lane < kb) y[k0 + lane] = xv;
    }
    __syncthreads();
    for (int i = tid; i < k0; i += blockDim.x) {
      double s = y[i];
#pragma unroll
      for (int t = 0; t < NB16; ++t)
        if (t < kb) s = fma(-S[(k0 + t) * ld + i], y[k0 + t], s);
      y[i] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < m; i += blockDim.x) x[i] = y[i];
  if (tid == 0) *info = fail;
}

cudaError_t launch_chol_solve(double* M, long long m, const double* b, double scale, double* x,
                              int* info, cudaStream_t stream) {
  if (m <= SMALL_M) {
    const int mi = (int)m;
    const size_t smem = ((size_t)mi * (mi | 1) + mi) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(chol_small16_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    { note_launch(); chol_small16_kernel<<<1, SM_NT, smem, stream>>>(M, mi, b, scale, x, info); }
    return cudaGetLastError();
  }
  if (m <= 0) {
    const int mi = (int)m;
    const size_t smem = ((size_t)mi * (mi | 1) + mi) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(chol_small_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    { note_launch(); chol_small_kernel<<<1, SM_NT, smem, stream>>>(M, mi, b, scale, x, info); }
    return cudaGetLastError();
  }
  size_t smem = (size_t)(NB * (NB + 1) + PANEL_ROWS * (NB + 1)) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  { note_launch(); chol_solve_kernel<<<1, CH_NT, smem, stream>>>(M, m, b, scale, x, info); }
  return cudaGetLastError();
}

}  // namespace ssnal

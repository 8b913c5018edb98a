// Dense SPD solve for the reduced Newton system: blocked right-looking Cholesky
// (32-column panels; diagonal block by one warp with shuffles, panel TRSM one row
// per thread, trailing SYRK update from a shared-memory copy of the panel),
// followed by blocked forward / backward substitution -- all inside ONE CTA so
// the factor never leaves L2 and no host round trip is needed.
// Replaces scipy.linalg.solve(..., assume_a="sym") of ref solver.py:175-191.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "ssnal_internal.h"

namespace cg = cooperative_groups;

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

// ---------------------------------------------------------------------------
// Latency-first small SPD solve (m <= 160): the matrix is padded to m16 = 16k with
// an identity tail and (scale b)^T appended as row m16, so the forward substitution
// L z = b falls out of the factorisation itself (row m16 is just one more row below
// every panel).  Per 16-column panel:
//   (1) diagonal block: warp 0, lane i holds row i in registers (compile-time
//       indices only), pivots by shuffle;
//   (2) panel TRSM: one thread per row below (row in registers, diagonal-block
//       entries broadcast from shared memory);
//   (3) trailing SYRK on the fp64 tensor cores: 8x8 output tiles, four
//       mma.m8n8k4 per tile for the 16-wide panel, C loaded / stored in place,
//       the A operand negated so D = S - L21 L21^T in one pass.
// Back substitution L^T x = z by 16-blocks: warp-0 shuffle solve + one block-wide
// column update.  Three barriers per panel, two per back-substitution block.
// Shared row stride ld = m16 + 4 (= 4 mod 16): the m8n8k4 A/B fragments
// (rows lane/4, k = lane%4) hit 16 distinct bank pairs per phase.
static constexpr int TC_NB = 16;
static constexpr int TC_MAX = 160;
static constexpr int TC_NT = 512;

__device__ __forceinline__ void tc_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// column J of the 16x16 diagonal block; template recursion keeps every register
// index a compile-time constant (no local-memory arrays)
template <int J>
__device__ __forceinline__ void tc_diag_step(double (&r)[TC_NB], int lane, int k0, double* rdg,
                                             int* fail, double d, double (*colbuf)[TC_NB]) {
  if (!(d > 0.0)) {
    if (lane == 0 && *fail == 0) *fail = k0 + J + 1;
    d = 1.0;
  }
  const double inv = rsqrt(d);
  const double sq = d * inv;
  if (lane == J) {
    r[J] = sq;
    rdg[k0 + J] = inv;
  } else if (lane > J) {
    r[J] *= inv;
  }
  // column J broadcast through shared memory (one store + broadcast loads; the 64-bit
  // shuffles per column were throughput-bound, scripts/diag_probe.cu), buffer by parity
  if (lane < TC_NB) colbuf[J & 1][lane] = r[J];
  __syncwarp();
#pragma unroll
  for (int c = J + 1; c < TC_NB; ++c) {
    const double lcj = colbuf[J & 1][c];
    if (lane >= c) r[c] = fma(-r[J], lcj, r[c]);
  }
  if constexpr (J + 1 < TC_NB)
    tc_diag_step<J + 1>(r, lane, k0, rdg, fail, __shfl_sync(0xffffffffu, r[J + 1], J + 1), colbuf);
}

// factor the 16x16 diagonal block at (k0, k0) in place (warp-wide call)
__device__ __forceinline__ void tc_factor_diag(double* S, int ld, int k0, int lane, double* rdg,
                                               int* fail) {
  __shared__ double colbuf[2][TC_NB];
  double r[TC_NB];
#pragma unroll
  for (int c = 0; c < TC_NB; ++c)
    r[c] = (lane < TC_NB && c <= lane) ? S[(k0 + lane) * ld + k0 + c] : 0.0;
  tc_diag_step<0>(r, lane, k0, rdg, fail, __shfl_sync(0xffffffffu, r[0], 0), colbuf);
  if (lane < TC_NB) {
#pragma unroll
    for (int c = 0; c < TC_NB; ++c)
      if (c <= lane) S[(k0 + lane) * ld + k0 + c] = r[c];
  }
}

// S[ri..ri+8)[ci..ci+8) -= L[ri..][k0..k0+16) L[ci..][k0..k0+16)^T  (4 x m8n8k4)
__device__ __forceinline__ void tc_syrk_tile(double* S, int ld, int k0, int ri, int ci, int lane) {
  double* cp = S + (ri + (lane >> 2)) * ld + ci + 2 * (lane & 3);
  double c0 = cp[0], c1 = cp[1];
  const double* ap = S + (ri + (lane >> 2)) * ld + k0 + (lane & 3);
  const double* bp = S + (ci + (lane >> 2)) * ld + k0 + (lane & 3);
#pragma unroll
  for (int q = 0; q < TC_NB; q += 4) tc_dmma(c0, c1, -ap[q], bp[q]);
  cp[0] = c0;
  cp[1] = c1;
}

// p-space mode: the kernel also assembles the Woodbury system from the raw Gram
// (M = Q_JJ) and projects the solution -- the work of pspace_assemble_kernel and
// pspace_project_kernel (newton.cu), same expressions and reduction trees
struct TcPspace {
  const int32_t* J;
  const double* grad;
  const double* a;
  double sigma, asa;
};

template <bool PS>
__global__ void __launch_bounds__(TC_NT, 1) chol_tc_kernel(const double* __restrict__ M, int m,
                                                           const double* __restrict__ b,
                                                           double scale,
                                                           double* __restrict__ x,
                                                           int* __restrict__ info, TcPspace ps) {
  extern __shared__ double S[];
  const int m16 = (m + TC_NB - 1) / TC_NB * TC_NB;
  const int ld = m16 + 4;
  double* rdg = S + (size_t)(m16 + 8) * ld;  // reciprocal pivots, m16
  double* aJ = rdg + m16;                     // p-space mode: a_J, grad_J, Q a_J
  double* gJ = aJ + m16;
  double* qa = gJ + m16;
  __shared__ int fail;
  __shared__ double red2[2 * 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) fail = 0;
  if (PS) {
    for (int r = tid; r < m; r += TC_NT) {
      const int j = ps.J[r];
      aJ[r] = ps.a[j];
      gJ[r] = ps.grad[j];
    }
  }
  // lower triangle of M by asynchronous 8-byte copies (every load in flight at
  // once: M sits in L2 from the assembling kernel); identity tail, b row and zero
  // padding by plain stores
  for (int i = warp; i < m16 + 8; i += TC_NT / 32) {
    for (int j = lane; j < m16; j += 32) {
      if (i < m && j <= i) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(S + i * ld + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                     "l"(M + (long long)i * m + j));
      } else {
        double v = 0.0;
        if (i >= m && i < m16) v = (i == j) ? 1.0 : 0.0;
        else if (i == m16 && !PS) v = j < m ? scale * b[j] : 0.0;
        S[i * ld + j] = v;
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (PS) {
    // qa = Q a_J (warp per row, lanes stride the row, warp_sum: pspace_assemble's order)
    for (int r = warp; r < m; r += TC_NT / 32) {
      double sacc = 0.0;
      for (int c = lane; c < m; c += 32) sacc += (c <= r ? S[r * ld + c] : S[c * ld + r]) * aJ[c];
      sacc = warp_sum(sacc);
      if (lane == 0) qa[r] = sacc;
    }
    __syncthreads();
    double v2[2] = {0.0, 0.0};  // a'Qa, a'g
    for (int r = tid; r < m; r += TC_NT) {
      v2[0] += aJ[r] * qa[r];
      v2[1] += aJ[r] * gJ[r];
    }
    const int ops2[2] = {0, 0};
    block_reduce<2>(v2, ops2, red2);
    if (tid == 0) { red2[0] = v2[0]; red2[1] = v2[1]; }
    __syncthreads();
    const double aqa = red2[0], ag = red2[1];
    const bool proj = ps.asa != 0.0;
    const double inv = proj ? 1.0 / ps.asa : 0.0;
    for (int i = warp; i < m; i += TC_NT / 32) {
      for (int c = lane; c <= i; c += 32) {
        double mm = S[i * ld + c];
        if (proj) mm = mm - (aJ[i] * qa[c] + qa[i] * aJ[c]) * inv + aqa * inv * inv * aJ[i] * aJ[c];
        S[i * ld + c] = (i == c ? 1.0 : 0.0) + ps.sigma * mm;
      }
    }
    for (int j = tid; j < m; j += TC_NT) S[m16 * ld + j] = proj ? gJ[j] - aJ[j] * (ag * inv) : gJ[j];
    __syncthreads();
  }
  // diagonal block 0; afterwards every diagonal block is factored by warp 0 right
  // after it has applied the previous panel's update to that block, overlapping the
  // other warps' trailing update (one-panel look-ahead)
  if (warp == 0) tc_factor_diag(S, ld, 0, lane, rdg, &fail);
  __syncthreads();
  for (int k0 = 0; k0 < m16; k0 += TC_NB) {
    // (2) panel TRSM for rows k0+16 .. m16 (the b row included)
    const int r0 = k0 + TC_NB;
    for (int i = r0 + tid; i <= m16; i += blockDim.x) {
      double row[TC_NB];
#pragma unroll
      for (int t = 0; t < TC_NB; ++t) row[t] = S[i * ld + k0 + t];
      // right-looking inside the row: short dependent chain (mul, fma) per column
#pragma unroll
      for (int j = 0; j < TC_NB; ++j) {
        row[j] *= rdg[k0 + j];
#pragma unroll
        for (int t = j + 1; t < TC_NB; ++t) row[t] = fma(-row[j], S[(k0 + t) * ld + k0 + j], row[t]);
      }
#pragma unroll
      for (int t = 0; t < TC_NB; ++t) S[i * ld + k0 + t] = row[t];
    }
    __syncthreads();
    // (3) SYRK: rows [r0, m16 + 8) x cols [r0, m16), lower tiles (I >= C).  The three
    // tiles of the next diagonal block (I, C < 2) go to warp 0, which then factors
    // that block; the other warps take the remaining tiles round-robin.
    const int nr = (m16 + 8 - r0) / 8, nc = (m16 - r0) / 8;
    if (nc > 0) {
      if (warp == 0) {
        tc_syrk_tile(S, ld, k0, r0, r0, lane);
        tc_syrk_tile(S, ld, k0, r0 + 8, r0, lane);
        tc_syrk_tile(S, ld, k0, r0 + 8, r0 + 8, lane);
        __syncwarp();
        tc_factor_diag(S, ld, r0, lane, rdg, &fail);
      } else {
        // tiles after the first three, in (I, C) order; warp w takes every 15th
        // starting at w - 1: walk (I, C) forward without divisions
        int I = 2, C = 0, skip = warp - 1;
        while (I < nr) {
          const int rowlen = min(I, nc - 1) + 1;
          if (C + skip < rowlen) {
            C += skip;
            tc_syrk_tile(S, ld, k0, r0 + 8 * I, r0 + 8 * C, lane);
            skip = TC_NT / 32 - 1;
          } else {
            skip -= rowlen - C;
            C = 0;
            ++I;
          }
        }
      }
    }
    __syncthreads();
  }
  // back substitution L^T x = z (z in row m16, overwritten by x)
  double* z = S + (size_t)m16 * ld;
  for (int k0 = m16 - TC_NB; k0 >= 0; k0 -= TC_NB) {
    if (warp == 0) {
      double zv = lane < TC_NB ? z[k0 + lane] : 0.0;
#pragma unroll
      for (int j = TC_NB - 1; j >= 0; --j) {
        if (lane == j) zv *= rdg[k0 + j];
        const double xj = __shfl_sync(0xffffffffu, zv, j);
        if (lane < j) zv = fma(-S[(k0 + j) * ld + k0 + lane], xj, zv);
      }
      if (lane < TC_NB) z[k0 + lane] = zv;
    }
    __syncthreads();
    for (int j = tid; j < k0; j += blockDim.x) {
      double s = z[j];
#pragma unroll
      for (int t = 0; t < TC_NB; ++t) s = fma(-S[(k0 + t) * ld + j], z[k0 + t], s);
      z[j] = s;
    }
    __syncthreads();
  }
  if (PS) {  // y <- P_J y = y - (a_J'y / a'a) a_J  (pspace_project_kernel's order)
    double v1[1] = {0.0};
    if (ps.asa != 0.0)
      for (int r = tid; r < m; r += TC_NT) v1[0] += aJ[r] * z[r];
    const int ops1[1] = {0};
    block_reduce<1>(v1, ops1, red2);
    if (tid == 0) red2[0] = v1[0];
    __syncthreads();
    const double coef = ps.asa != 0.0 ? red2[0] / ps.asa : 0.0;
    for (int i = tid; i < m; i += TC_NT) x[i] = ps.asa != 0.0 ? z[i] - coef * aJ[i] : z[i];
  } else {
    for (int i = tid; i < m; i += blockDim.x) x[i] = z[i];
  }
  if (tid == 0) *info = fail;
}


// ---------------------------------------------------------------------------
// Grid-wide SPD solve for 160 < m <= 2048 (q-space systems of configs 1/4, p-space
// systems up to direct_solve_threshold): M (row-major, lower triangle used) stays in
// L2; one cooperative launch over all SMs, three grid barriers per 32-column panel:
//   (1) CTA 0: 32x32 diagonal block (warp 0, registers + shuffles; identity-padded
//       past m) and the forward-substitution block z_k = L_kk^{-1} z_k;
//   (2) all CTAs: panel TRSM, one thread per row below (row in registers, L_kk and
//       its reciprocal pivots staged in each CTA's shared memory);
//   (3) all warps: trailing SYRK as 8x8 DMMA tiles (k = 32: eight m8n8k4 per tile)
//       plus the forward update of z below the panel.
// Back substitution L^T x = z by CTA 0 (32-blocks: warp shuffle solve + column
// update).  Replaces the single-CTA blocked kernel, which was latency-bound on one
// SM for these sizes.
static constexpr int BG_NB = 32;
static constexpr int BG_NT = 256;

template <int J>
__device__ __forceinline__ void bg_diag_step(double (&r)[BG_NB], int lane, double* rd, int k0,
                                             int* fail, double d, double (*colbuf)[BG_NB]) {
  if (!(d > 0.0)) {
    if (lane == 0 && *fail == 0) *fail = k0 + J + 1;
    d = 1.0;
  }
  const double inv = rsqrt(d);
  const double sq = d * inv;
  if (lane == J) {
    r[J] = sq;
    rd[J] = inv;
  } else if (lane > J) {
    r[J] *= inv;
  }
  // column J broadcast through shared memory (one store, then broadcast loads): 64-bit
  // shuffles per column were throughput-bound (scripts/diag_probe.cu: 11.5 -> 6.8 us per
  // 32 x 32 block); the buffer alternates by J parity, so one __syncwarp per column
  colbuf[J & 1][lane] = r[J];
  __syncwarp();
  if constexpr (J + 1 < BG_NB) {
    // column J+1 first and the next pivot fetched right away: the pivot chain (shuffle ->
    // rsqrt -> scale -> store -> broadcast) is the critical path, the updates of the
    // columns past J+1 are independent of it and fill its latency
    {
      const double lcj = colbuf[J & 1][J + 1];
      if (lane >= J + 1) r[J + 1] = fma(-r[J], lcj, r[J + 1]);
    }
    const double dnext = __shfl_sync(0xffffffffu, r[J + 1], J + 1);
#pragma unroll
    for (int c = J + 2; c < BG_NB; ++c) {
      const double lcj = colbuf[J & 1][c];
      if (lane >= c) r[c] = fma(-r[J], lcj, r[c]);
    }
    bg_diag_step<J + 1>(r, lane, rd, k0, fail, dnext, colbuf);
  }
}

// scripts/chol_probe.cu: per-phase globaltimer stamps of CTA 0 thread 0
#ifdef SSNAL_CHOL_TIMING
__device__ unsigned long long g_chol_marks[12][64];
#define CHOL_MARK(k)                                                                 \
  do {                                                                               \
    if (rank == 0 && threadIdx.x == 0) {                                             \
      unsigned long long t_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_chol_marks[k][min(k0_mark, 63)] = t_;                                        \
    }                                                                                \
  } while (0)
#else
#define CHOL_MARK(k) \
  do {               \
  } while (0)
#endif

__global__ void __launch_bounds__(BG_NT) chol_big_kernel(double* __restrict__ M, int m,
                                                         const double* __restrict__ b,
                                                         double scale, double* __restrict__ x,
                                                         int* __restrict__ info) {
  // z = scale b is built and solved in place in x
  double* z = x;
  cg::grid_group grid = cg::this_grid();
  __shared__ double D[BG_NB][BG_NB + 1];
  __shared__ double rd[BG_NB];
  __shared__ double colbuf[2][BG_NB];
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long gtid = (long long)blockIdx.x * BG_NT + tid;
  const long long gthreads = (long long)gridDim.x * BG_NT;
  const int gwarp = blockIdx.x * (BG_NT / 32) + warp, nwarps = gridDim.x * (BG_NT / 32);
  if (tid == 0) fail = 0;
  const unsigned rank = blockIdx.x;
  int k0_mark = 0;
  (void)rank;
  (void)k0_mark;
  for (long long i = gtid; i < m; i += gthreads) z[i] = scale * b[i];
  grid.sync();
  CHOL_MARK(0);
  // (1) diagonal block + forward block of panel k0 (CTA 0, warp 0): factor, inverse,
  // z_k = Linv z_k.  Panel 0 runs before the loop; every later one as the look-ahead of
  // the previous panel's update phase (it only needs that panel's update of its own
  // block, done first by the same warp), so it overlaps the other warps' SYRK tiles
  __shared__ double zs[BG_NB];
  auto diag_phase = [&](int k0, int kb) {
      double r[BG_NB];
#pragma unroll
      for (int c = 0; c < BG_NB; ++c)
        r[c] = (lane < kb && c < kb && c <= lane) ? M[(long long)(k0 + lane) * m + k0 + c]
                                                  : (lane == c ? 1.0 : 0.0);
      CHOL_MARK(6);
      bg_diag_step<0>(r, lane, rd, k0, &fail, __shfl_sync(0xffffffffu, r[0], 0), colbuf);
      __syncwarp();
      CHOL_MARK(7);
#pragma unroll
      for (int c = 0; c < BG_NB; ++c) D[lane][c] = c <= lane ? r[c] : 0.0;
      if (lane < kb) {
#pragma unroll
        for (int c = 0; c < BG_NB; ++c)
          if (c <= lane && c < kb) M[(long long)(k0 + lane) * m + k0 + c] = r[c];
      }
      __syncwarp();
      // Linv = L_kk^{-1}, column `lane` by forward substitution on e_lane (unrolled:
      // col[t] = 0 for t < lane, so the sums need no predicate).  Linv^T goes to the
      // block's (unused) strict upper triangle of M: the panel TRSM becomes a DMMA
      // product and both substitutions become matrix-vector products -- no 32-step
      // shuffle chains outside the factorization itself
      // right-looking order: as soon as col[t] is known every later partial sum takes its
      // term (independent FMAs), so the dependent chain is one FMA + one multiply per row
      // instead of the whole row sum; each sum still adds its terms in ascending t
      double col[BG_NB];
#pragma unroll
      for (int i = 0; i < BG_NB; ++i) col[i] = 0.0;
#pragma unroll
      for (int t = 0; t < BG_NB; ++t) {
        col[t] = t < lane ? 0.0 : (t == lane ? rd[t] : -col[t] * rd[t]);
#pragma unroll
        for (int i = t + 1; i < BG_NB; ++i) col[i] = fma(D[i][t], col[t], col[i]);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < BG_NB; ++i) {
        D[i][lane] = col[i];  // D now holds Linv (row i, column lane)
        if (i > lane && i < kb && lane < kb) M[(long long)(k0 + lane) * m + k0 + i] = col[i];
      }
      __syncwarp();
      CHOL_MARK(8);
      // z_k = Linv z_k
      zs[lane] = lane < kb ? z[k0 + lane] : 0.0;
      __syncwarp();
      double zv = 0.0;
#pragma unroll
      for (int t = 0; t < BG_NB; ++t) zv = fma(D[lane][t], zs[t], zv);
      if (lane < kb) z[k0 + lane] = zv;
      };
  if (blockIdx.x == 0 && warp == 0) diag_phase(0, min(BG_NB, m));
  grid.sync();
  for (int k0 = 0; k0 < m; k0 += BG_NB) {
    const int kb = min(BG_NB, m - k0);
    k0_mark = k0 / BG_NB;
    CHOL_MARK(1);
    const int r0 = k0 + kb;
    if (r0 >= m) break;
    // (2) panel TRSM rows [r0, m) as a DMMA product: L_rk = A_rk Linv^T (Linv of the
    // diagonal block from the strict upper triangle + reciprocal pivots), one 8-row tile
    // per warp, 4 column tiles x 8 k-steps of m8n8k4
    for (int idx = tid; idx < BG_NB * BG_NB; idx += BG_NT) {
      const int j = idx / BG_NB, t = idx % BG_NB;  // Linv[j][t], t <= j
      double v = 0.0;
      if (j < kb && t < kb) {
        if (t < j) v = M[(long long)(k0 + t) * m + k0 + j];
        else if (t == j) v = 1.0 / M[(long long)(k0 + j) * m + k0 + j];
      }
      D[j][t] = v;
    }
    __syncthreads();
    {
      const int ntile_r = (m - r0 + 7) / 8;
      for (int T = gwarp; T < ntile_r; T += nwarps) {
        const int row = r0 + 8 * T + (lane >> 2);
        double af[BG_NB / 4];
#pragma unroll
        for (int q = 0; q < BG_NB / 4; ++q) {
          const int k = 4 * q + (lane & 3);
          af[q] = (row < m && k < kb) ? M[(long long)row * m + k0 + k] : 0.0;
        }
        double c[4][2];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          c[nb][0] = c[nb][1] = 0.0;
#pragma unroll
          for (int q = 0; q < BG_NB / 4; ++q) {
            const double bv = D[nb * 8 + (lane >> 2)][4 * q + (lane & 3)];  // B[k][n] = Linv[n][k]
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(c[nb][0]), "+d"(c[nb][1])
                : "d"(af[q]), "d"(bv));
          }
        }
        // C fragment: row 8T + lane/4, columns nb*8 + 2 (lane%4) + {0, 1}
        if (row < m) {
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) {
            const int col = nb * 8 + 2 * (lane & 3);
            if (col < kb) M[(long long)row * m + k0 + col] = c[nb][0];
            if (col + 1 < kb) M[(long long)row * m + k0 + col + 1] = c[nb][1];
          }
        }
      }
    }
    grid.sync();
    CHOL_MARK(2);
    // (3) SYRK tiles over [r0, m) and the forward update of z.  The next diagonal block
    // (tile rows/columns I, C < 4) and its z rows belong to CTA 0's warp 0, which then
    // factors that block right away (look-ahead); every other warp takes the rest.
    {
      const int kb2 = min(BG_NB, m - r0);
      auto syrk_tile = [&](int I, int C) {
        const int ri = r0 + 8 * I + (lane >> 2), ci = r0 + 8 * C + (lane >> 2);
        const int cc = r0 + 8 * C + 2 * (lane & 3);
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int q = 0; q < BG_NB; q += 4) {
          const int kk = q + (lane & 3);
          const double av = (ri < m && kk < kb) ? -M[(long long)ri * m + k0 + kk] : 0.0;
          const double bv = (ci < m && kk < kb) ? M[(long long)ci * m + k0 + kk] : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c0), "+d"(c1)
                       : "d"(av), "d"(bv));
        }
        if (ri < m) {
          if (cc < m && cc <= ri) M[(long long)ri * m + cc] += c0;
          if (cc + 1 < m && cc + 1 <= ri) M[(long long)ri * m + cc + 1] += c1;
        }
      };
      auto z_row = [&](long long c) {
        double mv[BG_NB];  // the row's panel entries, all loads in flight at once
#pragma unroll
        for (int t = 0; t < BG_NB; ++t) mv[t] = t < kb ? M[c * m + k0 + t] : 0.0;
        double sacc = z[c];
#pragma unroll
        for (int t = 0; t < BG_NB; ++t)
          if (t < kb) sacc = fma(-mv[t], z[k0 + t], sacc);
        z[c] = sacc;
      };
      if (blockIdx.x == 0) {
        // CTA 0: the next diagonal block's tiles (<= 10) spread over its warps, its z rows,
        // then warp 0 factors the block while warps 1-7 join the general update below
        const int ntd = (kb2 + 7) / 8;
        for (int tix = warp; tix < ntd * (ntd + 1) / 2; tix += BG_NT / 32) {
          int I = 0;
          while ((I + 1) * (I + 2) / 2 <= tix) ++I;
          syrk_tile(I, tix - I * (I + 1) / 2);
        }
        if (tid < kb2) z_row(r0 + tid);
        __syncthreads();
        if (warp == 0) diag_phase(r0, kb2);
      }
      if (!(blockIdx.x == 0 && warp == 0)) {
        const int gw = gwarp - 1, ngw = nwarps - 1;  // warp 0 of CTA 0 excluded
        const int nt = (m - r0 + 7) / 8;
        const long long ntiles = (long long)nt * (nt + 1) / 2;
        for (long long tix = gw; tix < ntiles; tix += ngw) {
          int I = (int)((sqrt(8.0 * (double)tix + 1.0) - 1.0) * 0.5);
          while ((long long)(I + 1) * (I + 2) / 2 <= tix) ++I;
          while ((long long)I * (I + 1) / 2 > tix) --I;
          const int C = (int)(tix - (long long)I * (I + 1) / 2);
          if (I < 4) continue;  // the next diagonal block: warp 0 of CTA 0
          syrk_tile(I, C);
        }
        const long long gt = gtid - 32, ngt = gthreads - 32;
        for (long long c = r0 + BG_NB + gt; c < m; c += ngt) z_row(c);
      }
    }
    grid.sync();
    CHOL_MARK(3);
  }
  CHOL_MARK(4);
  if (blockIdx.x != 0) return;
  // back substitution L^T x = z in CTA 0, block by block: x_k = Linv_k^T z_k (a
  // matrix-vector product from the stored Linv^T, no shuffle chain), then the
  // column update of z above the block
  __shared__ double xk[BG_NB];
  for (int k0 = ((m - 1) / BG_NB) * BG_NB; k0 >= 0; k0 -= BG_NB) {
    const int kb = min(BG_NB, m - k0);
    if (warp == 0) {
      // lane j: x_j = sum_{t >= j} Linv[t][j] z_t; Linv[t][j] (t > j) at M[(k0+j) m + k0+t]
      double lv[BG_NB];
#pragma unroll
      for (int t = 0; t < BG_NB; ++t)
        lv[t] = (lane < kb && t < kb && t > lane) ? M[(long long)(k0 + lane) * m + k0 + t] : 0.0;
      const double dj = lane < kb ? 1.0 / M[(long long)(k0 + lane) * m + k0 + lane] : 0.0;
      const double zl = lane < kb ? z[k0 + lane] : 0.0;
      double xv = dj * zl;
#pragma unroll
      for (int t = 0; t < BG_NB; ++t) {
        const double zt = __shfl_sync(0xffffffffu, zl, t);
        xv = fma(lv[t], zt, xv);
      }
      if (lane < kb) z[k0 + lane] = xv;
      xk[lane] = lane < kb ? xv : 0.0;
    }
    __syncthreads();
    for (int j = tid; j < k0; j += BG_NT) {
      double mv[BG_NB];  // all column loads in flight at once
#pragma unroll
      for (int t = 0; t < BG_NB; ++t) mv[t] = t < kb ? M[(long long)(k0 + t) * m + j] : 0.0;
      double s = z[j];
#pragma unroll
      for (int t = 0; t < BG_NB; ++t)
        if (t < kb) s = fma(-mv[t], xk[t], s);
      z[j] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < m; i += BG_NT) x[i] = z[i];
  CHOL_MARK(5);
  if (tid == 0) *info = fail;
}


static int big_grid() {
  static DeviceCache cache;
  return per_device(cache, [](int dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, chol_big_kernel, BG_NT, 0);
    return sms * (per < 1 ? 1 : (per > 2 ? 2 : per));
  });
}


size_t chol_tc_smem(int m, bool ps = false) {
  const int m16 = (m + TC_NB - 1) / TC_NB * TC_NB;
  return ((size_t)(m16 + 8) * (m16 + 4) + (ps ? 4 : 1) * m16) * sizeof(double);
}

// p-space Woodbury solve for p <= 160 in one launch: Q (p x p Gram, overwritten
// only in shared memory), y = P_J (I + sigma P_J Q P_J)^{-1} P_J grad_J
cudaError_t launch_chol_pspace(const double* Q, long long p, const int32_t* J, const double* grad,
                               const double* a, double sigma, double asa, double* y, int* info,
                               cudaStream_t stream) {
  if (p > TC_MAX) return cudaErrorInvalidValue;
  static DeviceCache attr;
  const int err = per_device(attr, [](int) {
    return (int)cudaFuncSetAttribute(chol_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)chol_tc_smem(TC_MAX, true));
  });
  if (err != cudaSuccess) return (cudaError_t)err;
  TcPspace ps{J, grad, a, sigma, asa};
  const int pi = (int)p;
  { note_launch(); chol_tc_kernel<true><<<1, TC_NT, chol_tc_smem(pi, true), stream>>>(Q, pi, nullptr, 1.0, y, info, ps); }
  return cudaGetLastError();
}

cudaError_t launch_chol_solve(double* M, long long m, const double* b, double scale, double* x,
                              int* info, cudaStream_t stream) {
  if (m <= TC_MAX) {
    const int mi = (int)m;
    const size_t smem = chol_tc_smem(mi);
    static DeviceCache attr;
    const int err = per_device(attr, [](int) {
      return (int)cudaFuncSetAttribute(chol_tc_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)chol_tc_smem(TC_MAX));
    });
    if (err != cudaSuccess) return (cudaError_t)err;
    (void)smem;
    { note_launch(); chol_tc_kernel<false><<<1, TC_NT, smem, stream>>>(M, mi, b, scale, x, info, TcPspace{}); }
    return cudaGetLastError();
  }
  if (m <= 2048) {
    int mi = (int)m;
    void* args[] = {&M, &mi, (void*)&b, &scale, &x, &info};
    note_launch();
    return cudaLaunchCooperativeKernel((void*)chol_big_kernel, dim3(big_grid()), dim3(BG_NT), args,
                                       0, stream);
  }
  size_t smem = (size_t)(NB * (NB + 1) + PANEL_ROWS * (NB + 1)) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  { note_launch(); chol_solve_kernel<<<1, CH_NT, smem, stream>>>(M, m, b, scale, x, info); }
  return cudaGetLastError();
}

}  // namespace ssnal

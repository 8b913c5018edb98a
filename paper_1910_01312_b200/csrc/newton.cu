// Reduced Newton system in SAMPLE space (p = |J| < q): the Woodbury dual of the
// factor-space system.  With Z = X_J (p x q) and P_J = I - a_J a_J^T / a_J^T a_J,
//
//   (I_q + sigma Z^T P_J Z)^{-1} = I - sigma Z^T P_J (I_p + sigma P_J Z Z^T P_J)^{-1} P_J Z
//
// so t = -X^T s solves the q x q system via one p x p SPD solve:
//   y = (I_p + sigma P_J Q_JJ P_J)^{-1} P_J grad_J,   t = -g_r + sigma Z^T (P_J y).
// Q_JJ = Z Z^T is formed on the fp64 tensor cores (DMMA) from gathered rows.
// This is the p x p route of ref solver.py:224-258 (Q_JJ, a rank-one correction,
// a dense symmetric solve) in an always-SPD form.
#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

cudaError_t launch_chol_pspace(const double* Q, long long p, const int32_t* J, const double* grad,
                               const double* a, double sigma, double asa, double* y, int* info,
                               cudaStream_t stream);
cudaError_t launch_chol_solve(double* M, long long m, const double* b, double scale, double* x,
                              int* info, cudaStream_t stream);

static constexpr int RT = 64;      // output tile edge
static constexpr int RK = 32;      // k (feature) chunk staged per step
static constexpr int RLD = RK + 4; // padded smem row for conflict-free fragments

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct RowsArgs {
  const double* A;
  long long n, q, lda;
  const double* rs;
  int svr;
  const int32_t* J;
  long long p;
};

__device__ __forceinline__ const double* logical_row(const RowsArgs& g, long long li, double& sg) {
  long long pr = li;
  sg = 1.0;
  if (g.svr && li >= g.n) { pr = li - g.n; sg = -1.0; }
  if (g.rs) sg *= g.rs[pr];
  return g.A + pr * g.lda;
}

// Q_JJ = Z Z^T (p x p, full symmetric), tile pair (ti <= tj) per block; 8 warps x
// (8 rows x 64 cols) of DMMA 8x8x4 accumulators per 64x64 tile.
__global__ void __launch_bounds__(256) rows_gram_kernel(RowsArgs g, double* __restrict__ Qjj,
                                                        int ntile) {
  __shared__ double sA[RT][RLD];
  __shared__ double sB[RT][RLD];
  int pair = blockIdx.x, ti = 0;
  while (pair >= ntile - ti) { pair -= ntile - ti; ++ti; }
  const int tj = ti + pair;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ri = (long long)ti * RT, rj = (long long)tj * RT;
  // split-K over the feature dimension (blockIdx.y), partial tiles folded later
  const long long kchunk = ceil_div(ceil_div(g.q, (long long)gridDim.y), RK) * RK;
  const long long kbeg = blockIdx.y * kchunk, kend = min(g.q, kbeg + kchunk);
  Qjj += (long long)blockIdx.y * g.p * g.p;
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (long long k0 = kbeg; k0 < kend; k0 += RK) {
    for (int idx = threadIdx.x; idx < RT * RK; idx += blockDim.x) {
      int r = idx / RK, kk = idx % RK;
      long long col = k0 + kk;
      double va = 0.0, vb = 0.0;
      if (col < kend) {
        if (ri + r < g.p) {
          double sg;
          const double* row = logical_row(g, g.J[ri + r], sg);
          va = sg * __ldg(row + col);
        }
        if (rj + r < g.p) {
          double sg;
          const double* row = logical_row(g, g.J[rj + r], sg);
          vb = sg * __ldg(row + col);
        }
      }
      sA[r][kk] = va;
      sB[r][kk] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RK; kk += 4) {
      // A fragment (m = lane/4, k = lane%4) = Z[ri + 8w + m][k]
      const double a = sA[warp * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        // B fragment (k = lane%4, n = lane/4) = Z[rj + 8t + n][k]
        const double b = sB[t * 8 + (lane >> 2)][kk + (lane & 3)];
        dmma(acc[t][0], acc[t][1], a, b);
      }
    }
    __syncthreads();
  }
  const long long row = ri + warp * 8 + (lane >> 2);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      long long col = rj + t * 8 + 2 * (lane & 3) + h;
      if (row < g.p && col < g.p) {
        Qjj[row * g.p + col] = acc[t][h];
        if (ti != tj) Qjj[col * g.p + row] = acc[t][h];  // diagonal tiles hold both halves
      }
    }
  }
}

// Q = sum over the split-K partial Grams (fixed order)
__global__ void rows_gram_fold_kernel(const double* __restrict__ part, long long pp, int nsplit,
                                      double* __restrict__ Q) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= pp) return;
  double s = part[idx];
  for (int b = 1; b < nsplit; ++b) s += part[(long long)b * pp + idx];
  Q[idx] = s;
}

// Single-CTA O(p^2) assembly: gJ, aJ gathered; qa = Q a; scalars; M = I + sigma P Q P,
// b = P gJ (case a'Sa = 0: M = I + sigma Q, b = gJ).
__global__ void __launch_bounds__(1024) pspace_assemble_kernel(
    const int32_t* __restrict__ J, long long p, const double* __restrict__ grad,
    const double* __restrict__ a, double sigma, double asa, double* __restrict__ Q,
    double* __restrict__ aJ, double* __restrict__ qa, double* __restrict__ b) {
  __shared__ double red[2 * 32];
  for (long long r = threadIdx.x; r < p; r += blockDim.x) aJ[r] = a[J[r]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long r = warp; r < p; r += nw) {
    double s = 0.0;
    for (long long c = lane; c < p; c += 32) s += Q[r * p + c] * aJ[c];
    s = warp_sum(s);
    if (lane == 0) qa[r] = s;
  }
  __syncthreads();
  double v[2] = {0.0, 0.0};  // a'Qa, a'g
  for (long long r = threadIdx.x; r < p; r += blockDim.x) {
    v[0] += aJ[r] * qa[r];
    v[1] += aJ[r] * grad[J[r]];
  }
  const int ops[2] = {0, 0};
  block_reduce<2>(v, ops, red);
  __shared__ double aqa_s, ag_s;
  if (threadIdx.x == 0) { aqa_s = v[0]; ag_s = v[1]; }
  __syncthreads();
  const double aqa = aqa_s, ag = ag_s;
  const bool proj = asa != 0.0;
  const double inv = proj ? 1.0 / asa : 0.0;
  for (long long idx = threadIdx.x; idx < p * p; idx += blockDim.x) {
    long long r = idx / p, c = idx % p;
    double m = Q[idx];
    if (proj) m = m - (aJ[r] * qa[c] + qa[r] * aJ[c]) * inv + aqa * inv * inv * aJ[r] * aJ[c];
    Q[idx] = (r == c ? 1.0 : 0.0) + sigma * m;
  }
  for (long long r = threadIdx.x; r < p; r += blockDim.x) {
    double g = grad[J[r]];
    b[r] = proj ? g - aJ[r] * (ag * inv) : g;
  }
}

// w = P_J y (in place), single CTA.
__global__ void __launch_bounds__(1024) pspace_project_kernel(long long p, const double* aJ,
                                                               double asa, double* y) {
  __shared__ double red[32];
  if (asa == 0.0) return;
  double v[1] = {0.0};
  for (long long r = threadIdx.x; r < p; r += blockDim.x) v[0] += aJ[r] * y[r];
  const int ops[1] = {0};
  block_reduce<1>(v, ops, red);
  __shared__ double ay;
  if (threadIdx.x == 0) ay = v[0];
  __syncthreads();
  const double coef = ay / asa;
  for (long long r = threadIdx.x; r < p; r += blockDim.x) y[r] = y[r] - coef * aJ[r];
}

// part[split][q] = sum_{r in split} w_r X_{J_r}   (gathered transposed product)
static constexpr int GX_SPLIT = 16;
__global__ void __launch_bounds__(256) gather_xt_kernel(RowsArgs g, const double* __restrict__ w,
                                                        double* __restrict__ part) {
  const long long chunk = ceil_div(g.p, GX_SPLIT);
  const long long k0 = blockIdx.y * chunk, k1 = min(g.p, k0 + chunk);
  const long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= g.q) return;
  double s = 0.0;
  for (long long r = k0; r < k1; ++r) {
    double sg;
    const double* row = logical_row(g, g.J[r], sg);
    s = fma(w[r] * sg, __ldg(row + col), s);
  }
  part[blockIdx.y * g.q + col] = s;
}

// t = -g_r + sigma * sum_splits part
__global__ void pspace_finish_kernel(const double* __restrict__ part, long long q, double sigma,
                                     const double* __restrict__ g_r, double* __restrict__ t) {
  const long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= q) return;
  double s = 0.0;
  for (int b = 0; b < GX_SPLIT; ++b) s += part[b * q + col];
  t[col] = -g_r[col] + sigma * s;
}

static int gram_ksplit(long long p, long long q) {
  const long long nt = ceil_div(p, RT);
  const long long pairs = nt * (nt + 1) / 2;
  long long s = ceil_div(2 * 148, pairs);
  s = min(s, ceil_div(q, RK));
  s = min(s, 16LL);
  return (int)max(s, 1LL);
}

size_t pspace_ws_bytes(long long p, long long q) {
  return (size_t)((gram_ksplit(p, q) + 1) * p * p + 4 * p + GX_SPLIT * q + 64) * sizeof(double);
}

// Given Q_JJ (p x p, overwritten): y = P_J (I + sigma P_J Q_JJ P_J)^{-1} P_J grad_J.
// vecs: 4p doubles (aJ, qa, b, scratch).  Used by the sparse operator's direct route.
cudaError_t launch_pspace_solve(const int32_t* J, long long p, const double* grad, const double* a,
                                double sigma, double asa, double* Q, double* vecs, double* y,
                                int* info, cudaStream_t stream) {
  double* aJ = vecs;
  double* qa = aJ + p;
  double* b = qa + p;
  if (p <= 160) return launch_chol_pspace(Q, p, J, grad, a, sigma, asa, y, info, stream);
  { note_launch(); pspace_assemble_kernel<<<1, 1024, 0, stream>>>(J, p, grad, a, sigma, asa, Q, aJ, qa, b); }
  cudaError_t e = launch_chol_solve(Q, p, b, 1.0, y, info, stream);
  if (e != cudaSuccess) return e;
  { note_launch(); pspace_project_kernel<<<1, 1024, 0, stream>>>(p, aJ, asa, y); }
  return cudaGetLastError();
}

cudaError_t launch_pspace_direction(const double* A, long long n, long long q, long long lda,
                                    const double* rs, int svr, const int32_t* J, long long p,
                                    const double* grad, const double* a, double sigma, double asa,
                                    const double* g_r, double* t, int* info, void* ws,
                                    cudaStream_t stream) {
  double* Q = (double*)ws;
  double* aJ = Q + p * p;
  double* qa = aJ + p;
  double* b = qa + p;
  double* y = b + p;
  double* part = y + p;
  double* gpart = part + GX_SPLIT * q;
  RowsArgs g{A, n, q, lda, rs, svr, J, p};
  const int ntile = (int)ceil_div(p, RT);
  const int ks = gram_ksplit(p, q);
  { note_launch(); rows_gram_kernel<<<dim3(ntile * (ntile + 1) / 2, ks), 256, 0, stream>>>(g, gpart, ntile); }
  { note_launch(); rows_gram_fold_kernel<<<(unsigned)ceil_div(p * p, 256), 256, 0, stream>>>(gpart, p * p, ks, Q); }
  if (p <= 160) {  // assemble + Cholesky + projection in one single-CTA launch
    cudaError_t e = launch_chol_pspace(Q, p, J, grad, a, sigma, asa, y, info, stream);
    if (e != cudaSuccess) return e;
  } else {
    { note_launch(); pspace_assemble_kernel<<<1, 1024, 0, stream>>>(J, p, grad, a, sigma, asa, Q, aJ, qa, b); }
    cudaError_t e = launch_chol_solve(Q, p, b, 1.0, y, info, stream);
    if (e != cudaSuccess) return e;
    { note_launch(); pspace_project_kernel<<<1, 1024, 0, stream>>>(p, aJ, asa, y); }
  }
  { note_launch(); gather_xt_kernel<<<dim3((unsigned)ceil_div(q, 256), GX_SPLIT), 256, 0, stream>>>(g, y, part); }
  { note_launch(); pspace_finish_kernel<<<(unsigned)ceil_div(q, 256), 256, 0, stream>>>(part, q, sigma, g_r, t); }
  return cudaGetLastError();
}

}  // namespace ssnal

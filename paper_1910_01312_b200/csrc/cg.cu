// Conjugate gradients for the sample-space reduced Newton system with a sparse
// operator (configs 2, 3):  (I_p + sigma P_J Q_JJ P_J) y = P_J grad_J,
// Q_JJ y = X_J (X_J^T y) applied matrix-free (scatter -> CSC X^T -> CSR row gather).
// The iteration runs without host round trips: alpha, beta, the residual norm and
// a convergence flag live in device memory (cgs[]), every step kernel reads them;
// the host looks at the flag once per batch of iterations.  Iterates stay in
// range(P_J) (b and the operator's image do), so P_J is applied to Q_JJ p only.
// Replaces the CG branch of ref solver.py:151-172, 253-258.
#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

int stream_blocks(long long n, int per_thread);

enum { CG_RZ = 0, CG_PAP = 1, CG_BETA = 2, CG_RR = 3, CG_TOL2 = 4, CG_DONE = 5, CG_IT = 6,
       CG_DOT = 7, CG_TICKET = 8 };

// out = x - (aJ.x / asa) aJ  with aJ.x read from *dot (asa == 0: out = x)
__global__ void cg_project_kernel(long long p, const double* __restrict__ x,
                                  const double* __restrict__ aJ, const double* dot, double asa,
                                  double* __restrict__ out) {
  const double c = asa != 0.0 ? *dot / asa : 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = x[i] - c * aJ[i];
}

// Ap = pv + sigma (zq - (aJ.zq / asa) aJ);  cgs[PAP] = pv . Ap   (fixed-order fold)
__global__ void __launch_bounds__(SSNAL_NT) cg_ap_kernel(long long p,
                                                         const double* __restrict__ pv,
                                                         const double* __restrict__ zq,
                                                         const double* __restrict__ aJ,
                                                         double asa, double sigma,
                                                         double* __restrict__ Ap, double* cgs,
                                                         double* part) {
  __shared__ double red[32];
  if (cgs[CG_DONE] != 0.0) return;
  const double c = asa != 0.0 ? cgs[CG_DOT] / asa : 0.0;
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = pv[i] + sigma * (zq[i] - c * aJ[i]);
    Ap[i] = a;
    acc[0] = fma(pv[i], a, acc[0]);
  }
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) cgs[CG_PAP] = acc[0];
}

// alpha = rz / pAp; y += alpha pv; r -= alpha Ap; rr = r.r; beta = rr / rz; rz = rr
__global__ void __launch_bounds__(SSNAL_NT) cg_step_kernel(long long p, double* __restrict__ y,
                                                           double* __restrict__ r,
                                                           const double* __restrict__ pv,
                                                           const double* __restrict__ Ap,
                                                           double* cgs, double* part) {
  __shared__ double red[32];
  if (cgs[CG_DONE] != 0.0) return;
  const double pap = cgs[CG_PAP];
  const double alpha = pap > 0.0 ? cgs[CG_RZ] / pap : 0.0;
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x) {
    y[i] = fma(alpha, pv[i], y[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    acc[0] = fma(ri, ri, acc[0]);
  }
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) {
    const double rr = acc[0];
    cgs[CG_BETA] = cgs[CG_RZ] > 0.0 ? rr / cgs[CG_RZ] : 0.0;
    cgs[CG_RZ] = rr;
    cgs[CG_RR] = rr;
    cgs[CG_IT] += 1.0;
    if (rr <= cgs[CG_TOL2] || !(pap > 0.0)) cgs[CG_DONE] = 1.0;
  }
}

// pv = r + beta pv (skipped once converged)
__global__ void cg_dir_kernel(long long p, const double* __restrict__ r, double* __restrict__ pv,
                              const double* cgs) {
  if (cgs[CG_DONE] != 0.0) return;
  const double beta = cgs[CG_BETA];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x)
    pv[i] = fma(beta, pv[i], r[i]);
}

// y = 0, r = pv = b, rz = b.b, done = (rz <= tol^2) with the reference's CG target
// tol = min(eta, ||grad||^(1+tau)) / sigma computed from the device ||grad||^2
__global__ void __launch_bounds__(SSNAL_NT) cg_init_kernel(long long p, const double* __restrict__ b,
                                                           double* __restrict__ y,
                                                           double* __restrict__ r,
                                                           double* __restrict__ pv,
                                                           const double* g2, double eta,
                                                           double tau, double sigma,
                                                           double* cgs, double* part) {
  const double tol = fmin(eta, pow(sqrt(*g2), 1.0 + tau)) / sigma;
  const double tol2 = tol * tol;
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x) {
    y[i] = 0.0;
    r[i] = b[i];
    pv[i] = b[i];
    acc[0] = fma(b[i], b[i], acc[0]);
  }
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) {
    cgs[CG_RZ] = acc[0];
    cgs[CG_RR] = acc[0];
    cgs[CG_TOL2] = tol2;
    cgs[CG_IT] = 0.0;
    cgs[CG_DONE] = acc[0] <= tol2 ? 1.0 : 0.0;
  }
}

__global__ void scatter_zero_kernel(const int32_t* __restrict__ rows, long long p,
                                    double* __restrict__ dst) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p) dst[rows[i]] = 0.0;
}

static int cg_blocks(long long p) { return stream_blocks(p, 4); }

cudaError_t launch_cg_init(long long p, const double* b, double* y, double* r, double* pv,
                           const double* g2, double eta, double tau, double sigma, double* cgs,
                           double* part, cudaStream_t s) {
  note_launch();
  cg_init_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, b, y, r, pv, g2, eta, tau, sigma, cgs, part);
  return cudaGetLastError();
}

cudaError_t launch_cg_project(long long p, const double* x, const double* aJ, const double* dot,
                              double asa, double* out, cudaStream_t s) {
  note_launch();
  cg_project_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, x, aJ, dot, asa, out);
  return cudaGetLastError();
}

cudaError_t launch_cg_ap(long long p, const double* pv, const double* zq, const double* aJ,
                         double asa, double sigma, double* Ap, double* cgs, double* part,
                         cudaStream_t s) {
  note_launch();
  cg_ap_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, pv, zq, aJ, asa, sigma, Ap, cgs, part);
  return cudaGetLastError();
}

cudaError_t launch_cg_step(long long p, double* y, double* r, const double* pv, const double* Ap,
                           double* cgs, double* part, cudaStream_t s) {
  note_launch();
  cg_step_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, y, r, pv, Ap, cgs, part);
  return cudaGetLastError();
}

cudaError_t launch_cg_dir(long long p, const double* r, double* pv, const double* cgs,
                          cudaStream_t s) {
  note_launch();
  cg_dir_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, r, pv, cgs);
  return cudaGetLastError();
}

cudaError_t launch_scatter_zero(const int32_t* rows, long long p, double* dst, cudaStream_t s) {
  note_launch();
  scatter_zero_kernel<<<(unsigned)ceil_div(p, 256LL), 256, 0, s>>>(rows, p, dst);
  return cudaGetLastError();
}

}  // namespace ssnal

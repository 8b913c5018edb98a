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

#include <cooperative_groups.h>

#include <algorithm>

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

// alpha = rz / pAp; y += alpha pv; r -= alpha Ap; z = Dinv r (dinv NULL: z = r);
// rz' = r.z; beta = rz' / rz; rz = rz'; rr = r.r
__global__ void __launch_bounds__(SSNAL_NT) cg_step_kernel(long long p, double* __restrict__ y,
                                                           double* __restrict__ r,
                                                           const double* __restrict__ pv,
                                                           const double* __restrict__ Ap,
                                                           const double* __restrict__ dinv,
                                                           double* __restrict__ z,
                                                           double* cgs, double* part) {
  __shared__ double red[2 * 32];
  if (cgs[CG_DONE] != 0.0) return;
  const double pap = cgs[CG_PAP];
  const double alpha = pap > 0.0 ? cgs[CG_RZ] / pap : 0.0;
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x) {
    y[i] = fma(alpha, pv[i], y[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
    if (dinv) z[i] = zi;
    acc[0] = fma(ri, zi, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  const int ops[2] = {0, 0};
  block_reduce<2>(acc, ops, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<2>(part, gridDim.x, 2, ops, acc, red);
  if (threadIdx.x == 0) {
    const double rz = acc[0];
    cgs[CG_BETA] = cgs[CG_RZ] > 0.0 ? rz / cgs[CG_RZ] : 0.0;
    cgs[CG_RZ] = rz;
    cgs[CG_RR] = acc[1];
    cgs[CG_IT] += 1.0;
    if (!(pap > 0.0) || !(rz > 0.0)) cgs[CG_DONE] = 1.0;  // exact solve / breakdown
  }
}

// Stopping test of Algorithm 3 Step 1 on the TRUE Newton residual: with
// t = -X^T s + sigma X_J^T P_J y and d = -s - sigma P~ X t, the residual is
// (Q + sigma Q P~ Q) d + Q s = sigma^2 X X_J^T P Q_JJ P r_y; the caller passes
// zn = X X_J^T P Q_JJ P r and scale = sigma^2: done when scale^2 ||zn||^2 <= cgs[TOL2].
__global__ void __launch_bounds__(SSNAL_NT) cg_check_kernel(long long n, const double* __restrict__ zn,
                                                            double sigma, double* cgs,
                                                            double* part) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc[0] = fma(zn[i], zn[i], acc[0]);
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) {
    cgs[CG_RR] = sigma * sigma * acc[0];
    if (cgs[CG_RR] <= cgs[CG_TOL2]) cgs[CG_DONE] = 1.0;
  }
}

cudaError_t launch_cg_check(long long n, const double* zn, double sigma, double* cgs, double* part,
                            cudaStream_t s) {
  note_launch();
  cg_check_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, s>>>(n, zn, sigma, cgs, part);
  return cudaGetLastError();
}

// sharded stopping test: *sq = ||zn||^2 already all-reduced over the ranks
__global__ void cg_check_final_kernel(const double* sq, double scale, double* cgs) {
  cgs[CG_RR] = scale * scale * *sq;
  if (cgs[CG_RR] <= cgs[CG_TOL2]) cgs[CG_DONE] = 1.0;
}

cudaError_t launch_cg_check_final(const double* sq, double scale, double* cgs, cudaStream_t s) {
  note_launch();
  cg_check_final_kernel<<<1, 1, 0, s>>>(sq, scale, cgs);
  return cudaGetLastError();
}

// pv = z + beta pv (z = r unpreconditioned; skipped once converged)
__global__ void cg_dir_kernel(long long p, const double* __restrict__ r, double* __restrict__ pv,
                              const double* cgs) {
  if (cgs[CG_DONE] != 0.0) return;
  const double beta = cgs[CG_BETA];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x)
    pv[i] = fma(beta, pv[i], r[i]);
}

// y = 0, r = b, pv = z = Dinv b (dinv NULL: z = b), rz = b.z, done = (b == 0); the
// target tol = min(eta, ||grad||^(1+tau)) is computed from the device ||grad||^2
__global__ void __launch_bounds__(SSNAL_NT) cg_init_kernel(long long p, const double* __restrict__ b,
                                                           double* __restrict__ y,
                                                           double* __restrict__ r,
                                                           double* __restrict__ pv,
                                                           const double* __restrict__ dinv,
                                                           const double* g2, double eta,
                                                           double tau, double* cgs, double* part) {
  const double tol = fmin(eta, pow(sqrt(*g2), 1.0 + tau));
  const double tol2 = tol * tol;
  __shared__ double red[2 * 32];
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (long long)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double zi = dinv ? bi * dinv[i] : bi;
    y[i] = 0.0;
    r[i] = bi;
    pv[i] = zi;
    acc[0] = fma(bi, zi, acc[0]);
    acc[1] = fma(bi, bi, acc[1]);
  }
  const int ops[2] = {0, 0};
  block_reduce<2>(acc, ops, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
  if (!last_block_arrive(reinterpret_cast<unsigned int*>(cgs + CG_TICKET), gridDim.x)) return;
  block_fold_partials<2>(part, gridDim.x, 2, ops, acc, red);
  if (threadIdx.x == 0) {
    cgs[CG_RZ] = acc[0];
    cgs[CG_RR] = acc[1];
    cgs[CG_TOL2] = tol2;
    cgs[CG_IT] = 0.0;
    cgs[CG_DONE] = acc[1] > 0.0 ? 0.0 : 1.0;  // b = 0: y = 0 is exact
  }
}

// Jacobi preconditioner of the factor-space system I + sigma X_J^T P X_J:
// dinv_k = 1 / (1 + sigma (sum_{i in J} x_ik^2 - u_k^2 / a'a)),  u = X_J^T a_J
__global__ void cg_jacobi_kernel(long long q, const double* __restrict__ colsq,
                                 const double* __restrict__ u, double asa, double sigma,
                                 double* __restrict__ dinv) {
  const double inv = asa != 0.0 ? 1.0 / asa : 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < q;
       k += (long long)gridDim.x * blockDim.x) {
    const double d = 1.0 + sigma * fmax(colsq[k] - inv * u[k] * u[k], 0.0);
    dinv[k] = 1.0 / d;
  }
}

cudaError_t launch_cg_jacobi(long long q, const double* colsq, const double* u, double asa,
                             double sigma, double* dinv, cudaStream_t s) {
  note_launch();
  cg_jacobi_kernel<<<stream_blocks(q, 4), SSNAL_NT, 0, s>>>(q, colsq, u, asa, sigma, dinv);
  return cudaGetLastError();
}

__global__ void scatter_zero_kernel(const int32_t* __restrict__ rows, long long p,
                                    double* __restrict__ dst) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p) dst[rows[i]] = 0.0;
}

static int cg_blocks(long long p) { return stream_blocks(p, 4); }

cudaError_t launch_cg_init(long long p, const double* b, double* y, double* r, double* pv,
                           const double* dinv, const double* g2, double eta, double tau,
                           double* cgs, double* part, cudaStream_t s) {
  note_launch();
  cg_init_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, b, y, r, pv, dinv, g2, eta, tau, cgs, part);
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
                           const double* dinv, double* z, double* cgs, double* part,
                           cudaStream_t s) {
  note_launch();
  cg_step_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, y, r, pv, Ap, dinv, z, cgs, part);
  return cudaGetLastError();
}

cudaError_t launch_cg_dir(long long p, const double* r, double* pv, const double* cgs,
                          cudaStream_t s) {
  note_launch();
  cg_dir_kernel<<<cg_blocks(p), SSNAL_NT, 0, s>>>(p, r, pv, cgs);
  return cudaGetLastError();
}

// One CG iteration's vector work in ONE cooperative launch (replaces cg_ap + cg_step +
// cg_dir: three launches and two device-wide reductions per iteration):
//   A: Ap = pv + sigma (zq - c aJ), c = cgs[DOT] / asa;  pAp          -> grid sync
//   B: alpha = rz / pAp; y += alpha pv; r -= alpha Ap; z = Dinv r; rz', rr -> grid sync
//   C: beta = rz' / rz;  pv = z + beta pv
// Every block folds the same per-block partials in block order, so alpha and beta are
// identical in every block and the sums are the unfused kernels' (same grid, same order).
namespace cgrp = cooperative_groups;
static constexpr int CGU_NT = 512;
static constexpr int CGU_MAX_GRID = 512;  // 3 * CGU_MAX_GRID partial doubles (cg_part_doubles)
__global__ void __launch_bounds__(CGU_NT) cg_update_kernel(
    long long p, double* __restrict__ y, double* __restrict__ r, double* __restrict__ pv,
    const double* __restrict__ zq, const double* __restrict__ aJ, double asa, double sigma,
    const double* __restrict__ dinv, double* __restrict__ Ap, double* __restrict__ z, double* cgs,
    double* part) {
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double red[2 * 32];
  if (cgs[CG_DONE] != 0.0) return;  // uniform over the grid: set only by a finished launch
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double c = asa != 0.0 ? cgs[CG_DOT] / asa : 0.0;
  const double rz_old = cgs[CG_RZ];
  double a1[1] = {0.0};
  for (long long i = i0; i < p; i += stride) {
    const double a = pv[i] + sigma * (zq[i] - c * aJ[i]);
    Ap[i] = a;
    a1[0] = fma(pv[i], a, a1[0]);
  }
  const int o1[1] = {0};
  const int ops[2] = {0, 0};
  block_reduce<1>(a1, o1, red);
  if (threadIdx.x == 0) part[blockIdx.x] = a1[0];
  grid.sync();
  block_fold_partials<1>(part, gridDim.x, 1, o1, a1, red);
  __shared__ double bc[2];
  if (threadIdx.x == 0) bc[0] = a1[0];
  __syncthreads();
  const double pap = bc[0];
  const double alpha = pap > 0.0 ? rz_old / pap : 0.0;
  double acc[2] = {0.0, 0.0};
  for (long long i = i0; i < p; i += stride) {
    y[i] = fma(alpha, pv[i], y[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    const double zi = dinv ? ri * dinv[i] : ri;
    if (dinv) z[i] = zi;
    acc[0] = fma(ri, zi, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  block_reduce<2>(acc, ops, red);
  double* part2 = part + gridDim.x;
  if (threadIdx.x == 0) {
    part2[2 * blockIdx.x] = acc[0];
    part2[2 * blockIdx.x + 1] = acc[1];
  }
  grid.sync();
  block_fold_partials<2>(part2, gridDim.x, 2, ops, acc, red);
  if (threadIdx.x == 0) {
    bc[0] = acc[0];
    bc[1] = acc[1];
  }
  __syncthreads();
  const double rz = bc[0];
  const bool stop = !(pap > 0.0) || !(rz > 0.0);  // exact solve / breakdown
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cgs[CG_PAP] = pap;
    cgs[CG_BETA] = rz_old > 0.0 ? rz / rz_old : 0.0;
    cgs[CG_RZ] = rz;
    cgs[CG_RR] = bc[1];
    cgs[CG_IT] += 1.0;
    if (stop) cgs[CG_DONE] = 1.0;
  }
  if (stop) return;
  const double beta = rz_old > 0.0 ? rz / rz_old : 0.0;
  const double* zz = dinv ? z : r;
  for (long long i = i0; i < p; i += stride) pv[i] = fma(beta, pv[i], zz[i]);
}

static int cg_update_grid(long long p) {
  static DeviceCache cache;
  const int cap = per_device(cache, [](int dev) {
    int sms = 148, per = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cg_update_kernel, CGU_NT, 0);
    return std::min(CGU_MAX_GRID, sms * std::max(1, std::min(per, 2)));
  });
  return (int)std::max(1LL, std::min((long long)cap, ceil_div(p, (long long)CGU_NT)));
}

// part: 3 * grid doubles (cg_part_doubles covers it)
cudaError_t launch_cg_update(long long p, double* y, double* r, double* pv, const double* zq,
                             const double* aJ, double asa, double sigma, const double* dinv,
                             double* Ap, double* z, double* cgs, double* part, cudaStream_t s) {
  note_launch();
  void* args[] = {&p, &y, &r, &pv, &zq, &aJ, &asa, &sigma, &dinv, &Ap, &z, &cgs, &part};
  return cudaLaunchCooperativeKernel((void*)cg_update_kernel, dim3(cg_update_grid(p)),
                                     dim3(CGU_NT), args, 0, s);
}

cudaError_t launch_scatter_zero(const int32_t* rows, long long p, double* dst, cudaStream_t s) {
  note_launch();
  scatter_zero_kernel<<<(unsigned)ceil_div(p, 256LL), 256, 0, s>>>(rows, p, dst);
  return cudaGetLastError();
}

}  // namespace ssnal

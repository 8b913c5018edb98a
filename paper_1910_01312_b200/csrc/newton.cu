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

// Workspace for any system order p' <= p: the split-K factor grows as p' shrinks (fewer
// tile pairs), so the bound is the max over tile counts, each at its largest p'.
// (Sizing with the split of p itself under-allocated p' < p: e.g. q = 400 sized at
// p = 400 -> 11 splits, but p' = 380 takes 13 and its partial tiles ran past the end.)
size_t pspace_ws_bytes(long long p, long long q) {
  long long worst = 0;
  for (long long nt = 1; nt <= ceil_div(max(p, 1LL), (long long)RT); ++nt) {
    const long long pp = min(p, nt * RT);
    worst = max(worst, (gram_ksplit(pp, q) + 1) * pp * pp);
  }
  return (size_t)(worst + 4 * p + GX_SPLIT * q + 64) * sizeof(double);
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

// ---------------------------------------------------------------- factor-space gradient
// The SsN gradient grad = Q s = X r with r = X^T s, s = w - Pi(u), kept in factor space
// across Newton steps:
//   X^T w  moves by alpha t per accepted step (t = X^T d, the Newton system's solution;
//          Qw moves by alpha X t = alpha Qd, so the pair stays consistent),
//   X^T Pi moves by X^T (Pi_new - Pi_old), whose support is the slots whose projection
//          changed -- about the free set, O(p) rows -- gathered in the accept pass.
// So a Newton step sweeps A once (X [t, r] in the epilogue) instead of three times.

// grad[J[k]] = x_{J_k} . r  (warp per row; the p-space system's right-hand side)
__global__ void __launch_bounds__(256) rows_grad_kernel(RowsArgs g, const double* __restrict__ r,
                                                        double* __restrict__ grad) {
  const long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= g.p) return;
  double sg;
  const double* row = logical_row(g, g.J[k], sg);
  double acc = 0.0;
  for (long long c = lane; c < g.q; c += 32) acc = fma(__ldg(row + c), r[c], acc);
  acc = warp_sum(acc);
  if (lane == 0) grad[g.J[k]] = sg * acc;
}

cudaError_t launch_rows_grad(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, const int32_t* J, long long p,
                             const double* r, double* grad, cudaStream_t stream) {
  if (p < 1) return cudaSuccess;
  RowsArgs g{A, n, q, lda, rs, svr, J, p};
  note_launch();
  rows_grad_kernel<<<(unsigned)ceil_div(p * 32, 256LL), 256, 0, stream>>>(g, r, grad);
  return cudaGetLastError();
}

// Accepted Armijo step (as accept_kernel, same numpy-ordered arithmetic) plus
//   s = w_new - Pi_new  and  part[block][c] = sum over changed slots i of this block's
//   contiguous chunk (ascending i) of (Pi_new - Pi_old)_i x_i[c]
// (changed slots collected per 256-slot tile by ballot + warp prefix into smem).
static constexpr int AQ_NT = 256;
static constexpr int AQ_MAXC = 8;  // q <= 2048
struct AcceptQArgs {
  RowsArgs g;  // logical rows of X (J unused)
  long long n;
  double alpha, cu;
  double *w, *qw, *u, *xp, *s;
  const double *d, *qd, *txj;
  uint8_t* fr;
  const uint8_t* tfj;
  double* part;  // [grid][q]
  unsigned int* ticket;
  int* touched;  // [grid]: this CTA saw a changed slot (its partial is nonzero)
  // last-CTA fold: xpi += sum_b part[b] (block order), xw += alpha t, r = xw - xpi
  const double* t;
  double *xw, *xpi, *r;
  double* dsum;  // sharded driver: the fold goes here (all-reduced, then launch_factor_update)
  // accepted trial's projection record -> current record (replaces a D2D memcpy)
  const ProjState* st_src;
  ProjState* st_dst;
  // linear update over the slots free before AND after the step:
  // there Pi_new - Pi_old = cu (Qd)_i - dlam a_i exactly, and their rows sum to
  // cu G t - dlam m1 minus the leaving rows' share -- no row gathers for them.
  // gt = G t (kept q-space Gram of the CURRENT free set times t), m1 = X_J^T a_J; NULL: off
  const double* gt;
  const double* m1;
  const double* avec;
};

template <int NC>
__global__ void __launch_bounds__(AQ_NT) accept_q_kernel(AcceptQArgs a) {
  // changed slots of the CTA's chunk are collected over several 256-slot tiles (ascending
  // slot order) and their rows gathered in one batch of 4-row rounds: one barrier per
  // tile in the streaming part, and few single-row rounds when a tile has 1-3 changes
  constexpr int LCAP = 1024;
  __shared__ int list[LCAP];
  __shared__ double dval[LCAP];
  __shared__ int wcnt[2][AQ_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // multiplier change of the accepted trial (st_dst still holds the old record: it is
  // overwritten by the last CTA, after every CTA has read it)
  const bool lin = a.gt != nullptr;
  const double dlam = lin ? a.st_src->lam - a.st_dst->lam : 0.0;
  const long long chunk = ceil_div(ceil_div(a.n, (long long)gridDim.x), (long long)AQ_NT) * AQ_NT;
  const long long b0 = (long long)blockIdx.x * chunk, b1 = min(a.n, b0 + chunk);
  double acc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  int any = 0, cnt = 0, par = 0;
  // rows of list[0, cnt) added to acc in list order (the order of the sums is the slot
  // order whatever the batching: results do not depend on LCAP)
  auto flush = [&]() {
    __syncthreads();
    int k = 0;
    for (; k + 4 <= cnt; k += 4) {
      double sg[4], f[4], v[4][NC];
      const double* row[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        row[u] = logical_row(a.g, b0 + list[k + u], sg[u]);
        f[u] = dval[k + u] * sg[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const long long col = tid + (long long)c * AQ_NT;
          v[u][c] = col < a.g.q ? __ldg(row[u] + col) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(f[u], v[u][c], acc[c]);
    }
    for (; k < cnt; ++k) {
      double sg;
      const double* row = logical_row(a.g, b0 + list[k], sg);
      const double f = dval[k] * sg;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const long long col = tid + (long long)c * AQ_NT;
        if (col < a.g.q) acc[c] = fma(f, __ldg(row + col), acc[c]);
      }
    }
    __syncthreads();
    cnt = 0;
  };
  for (long long base = b0; base < b1; base += AQ_NT) {
    const long long i = base + tid;
    double dpi = 0.0;
    if (i < b1) {
      const double qdi = a.qd[i];
      const double wn = __dadd_rn(a.w[i], __dmul_rn(a.alpha, a.d[i]));
      a.w[i] = wn;
      a.qw[i] = __dadd_rn(a.qw[i], __dmul_rn(a.alpha, qdi));
      a.u[i] = __dadd_rn(a.u[i], __dmul_rn(a.cu, qdi));
      const double xn = a.txj[i];
      dpi = xn - a.xp[i];
      a.xp[i] = xn;
      const uint8_t f_old = a.fr[i], f_new = a.tfj[i];
      a.fr[i] = f_new;
      a.s[i] = __dsub_rn(wn, xn);
      if (lin && f_old) {
        // free before: its linear share is inside cu G t - dlam m1; free after too:
        // nothing left to gather, leaving: the difference to the actual change
        dpi = f_new ? 0.0 : dpi - (a.cu * qdi - dlam * a.avec[i]);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, dpi != 0.0);
    if (lane == 0) wcnt[par][warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < AQ_NT / 32; ++w) {
      off += w < warp ? wcnt[par][w] : 0;
      tot += wcnt[par][w];
    }
    if (dpi != 0.0) {
      const int o = cnt + off + __popc(bal & ((1u << lane) - 1u));
      list[o] = (int)(i - b0);
      dval[o] = dpi;
    }
    cnt += tot;
    any |= tot;
    par ^= 1;
    if (cnt + AQ_NT > LCAP) flush();
  }
  if (__syncthreads_or(cnt)) flush();
  if (any) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long col = tid + (long long)c * AQ_NT;
      if (col < a.g.q) a.part[(long long)blockIdx.x * a.g.q + col] = acc[c];
    }
  }
  if (tid == 0) a.touched[blockIdx.x] = any ? 1 : 0;
  if (!last_block_arrive(a.ticket, gridDim.x)) return;
  if (a.st_dst && tid < (int)(sizeof(ProjState) / sizeof(unsigned int)))
    reinterpret_cast<unsigned int*>(a.st_dst)[tid] =
        reinterpret_cast<const unsigned int*>(a.st_src)[tid];
  // fold only the CTAs that saw a change (typically a handful), in block order
  // touched CTAs listed in block order: all flags loaded at once, ballot + warp prefix
  __shared__ int blist[148 * 8];
  int m = 0;
  for (unsigned c0 = 0; c0 < gridDim.x; c0 += AQ_NT) {
    const unsigned b = c0 + tid;
    const bool f = b < gridDim.x && __ldcg(a.touched + b) != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[0][warp] = __popc(bal);
    __syncthreads();
    int off = m, tot = 0;
#pragma unroll
    for (int w = 0; w < AQ_NT / 32; ++w) {
      off += w < warp ? wcnt[0][w] : 0;
      tot += wcnt[0][w];
    }
    if (f) blist[off + __popc(bal & ((1u << lane) - 1u))] = (int)b;
    m += tot;
    __syncthreads();
  }
  // columns in chunks of 256: warp w sums the touched CTAs k = w, w + 8, ... (k order),
  // lane l columns c0 + l + 32 i (i < 8; coalesced), two k at a time so 16 loads are in
  // flight per lane; the 8 warp partials are then added in warp order (deterministic)
  __shared__ double wsum[AQ_NT / 32][AQ_NT];
  for (long long c0 = 0; c0 < a.g.q; c0 += AQ_NT) {
    double acc8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc8[i] = 0.0;
    int k = warp;
    for (; k + AQ_NT / 32 < m; k += 2 * (AQ_NT / 32)) {
      const double* p0 = a.part + (long long)blist[k] * a.g.q + c0 + lane;
      const double* p1 = a.part + (long long)blist[k + AQ_NT / 32] * a.g.q + c0 + lane;
      double v0[8], v1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool in = c0 + lane + 32 * i < a.g.q;
        v0[i] = in ? __ldcg(p0 + 32 * i) : 0.0;
        v1[i] = in ? __ldcg(p1 + 32 * i) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc8[i] = (acc8[i] + v0[i]) + v1[i];
    }
    if (k < m) {
      const double* p0 = a.part + (long long)blist[k] * a.g.q + c0 + lane;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c0 + lane + 32 * i < a.g.q) acc8[i] += __ldcg(p0 + 32 * i);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) wsum[warp][lane + 32 * i] = acc8[i];
    __syncthreads();
    const long long c = c0 + tid;
    if (c < a.g.q) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < AQ_NT / 32; ++w) sum += wsum[w][tid];
      if (lin) sum += a.cu * a.gt[c] - dlam * a.m1[c];
      if (a.dsum) {
        a.dsum[c] = sum;
      } else {
        const double pi = a.xpi[c] + sum;
        const double ww = __dadd_rn(a.xw[c], __dmul_rn(a.alpha, a.t[c]));
        a.xpi[c] = pi;
        a.xw[c] = ww;
        a.r[c] = ww - pi;
      }
    }
    __syncthreads();
  }
}

// out = G t for the kept q-space Gram (tile-symmetric storage of gram_kernel: the tile
// (I, J) with I > J is stored transposed at (J, I); GT = 128), a warp per row, lanes stride
// the columns, fixed shuffle tree
static constexpr int GTV_TILE = 128;
__global__ void __launch_bounds__(256) gram_tvec_kernel(const double* __restrict__ G, long long q,
                                                        const double* __restrict__ t,
                                                        double* __restrict__ out) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= q) return;
  const long long ti = i / GTV_TILE;
  double acc = 0.0;
  for (long long j = lane; j < q; j += 32) {
    const double g = (ti > j / GTV_TILE) ? __ldg(G + j * q + i) : __ldg(G + i * q + j);
    acc = fma(g, __ldg(t + j), acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[i] = acc;
}

cudaError_t launch_gram_tvec(const double* G, long long q, const double* t, double* out,
                             cudaStream_t stream) {
  note_launch();
  gram_tvec_kernel<<<(unsigned)ceil_div(q * 32, 256LL), 256, 0, stream>>>(G, q, t, out);
  return cudaGetLastError();
}

int accept_q_grid(long long n) {
  long long g = ceil_div(n, (long long)AQ_NT);
  return (int)max(1LL, min(g, 148LL * 8));
}

size_t accept_q_ws_bytes(long long n, long long q) {
  return 256 + 148 * 8 * sizeof(int) + (size_t)accept_q_grid(n) * q * sizeof(double);
}

cudaError_t launch_accept_q(const double* A, long long n_phys, long long q, long long lda,
                            const double* rs, int svr, long long n, double alpha, double cu,
                            double* w, const double* d, double* qw, const double* qd, double* u,
                            double* xp, const double* txj, uint8_t* fr, const uint8_t* tfj,
                            double* s, const double* t, double* xw, double* xpi, double* r,
                            double* part, const ProjState* st_src, ProjState* st_dst,
                            cudaStream_t stream, double* dsum, const double* gt,
                            const double* m1, const double* avec) {
  if (q > (long long)AQ_NT * AQ_MAXC) return cudaErrorInvalidValue;
  AcceptQArgs a;
  a.g = RowsArgs{A, n_phys, q, lda, rs, svr, nullptr, 0};
  a.n = n; a.alpha = alpha; a.cu = cu;
  a.w = w; a.qw = qw; a.u = u; a.xp = xp; a.s = s; a.d = d; a.qd = qd; a.txj = txj;
  a.fr = fr; a.tfj = tfj;
  a.ticket = (unsigned int*)part;  // zeroed workspace; reset by the last CTA
  a.touched = (int*)((char*)part + 256);
  a.part = (double*)((char*)part + 256 + 148 * 8 * sizeof(int));
  a.t = t; a.xw = xw; a.xpi = xpi; a.r = r; a.dsum = dsum;
  a.st_src = st_src; a.st_dst = st_dst;
  a.gt = (gt && m1 && avec && st_src && st_dst) ? gt : nullptr;
  a.m1 = m1; a.avec = avec;
  const int grid = accept_q_grid(n);
  const int nc = (int)ceil_div(q, (long long)AQ_NT);
  note_launch();
  if (nc <= 1) accept_q_kernel<1><<<grid, AQ_NT, 0, stream>>>(a);
  else if (nc <= 2) accept_q_kernel<2><<<grid, AQ_NT, 0, stream>>>(a);
  else if (nc <= 4) accept_q_kernel<4><<<grid, AQ_NT, 0, stream>>>(a);
  else accept_q_kernel<8><<<grid, AQ_NT, 0, stream>>>(a);
  return cudaGetLastError();
}

// sharded: xpi += dsum (the all-reduced X^T (Pi_new - Pi_old)), xw += alpha t, r = xw - xpi
__global__ void factor_update_kernel(long long q, double alpha, const double* __restrict__ t,
                                     const double* __restrict__ dsum, double* __restrict__ xw,
                                     double* __restrict__ xpi, double* __restrict__ r) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= q) return;
  const double pi = xpi[c] + dsum[c];
  const double ww = __dadd_rn(xw[c], __dmul_rn(alpha, t[c]));
  xpi[c] = pi;
  xw[c] = ww;
  r[c] = ww - pi;
}

cudaError_t launch_factor_update(long long q, double alpha, const double* t, const double* dsum,
                                 double* xw, double* xpi, double* r, cudaStream_t s) {
  note_launch();
  factor_update_kernel<<<(unsigned)ceil_div(q, 256LL), 256, 0, s>>>(q, alpha, t, dsum, xw, xpi, r);
  return cudaGetLastError();
}

}  // namespace ssnal

// Shard-local kernels of the row-sharded solver (one process per GPU, each rank
// owns a contiguous slice of the samples / dual slots).  Everything coupling the
// ranks reduces to tiny fixed-size records that the host all-gathers and folds in
// rank order, so every rank holds bit-identical scalars and takes the same branch:
//
//   proj_local  : the multiplier search of the projection onto {a'x = d, l<=x<=u}
//                 split into "evaluate at lambda" (f, one-sided slopes, nearest
//                 breakpoints: 5 doubles per trial) and "apply at lambda" (x, free
//                 mask and the 6 fused sums of proj.cu's apply phase) -- the
//                 safeguarded Newton of proj.cu driven one pass per all-gather;
//   sum_slices  : ordered sum of the world's all-gathered partials (X^T v,
//                 Gram blocks, dot records) -- deterministic, no atomics;
//   hs_apply_coef / qspace_assemble : the Newton-direction pieces whose global
//                 scalars (a_J'y, a_J'a_J, the summed Gram) come from the host.
// Replaces, for the sharded path, the cross-slot reductions inside ref
// projection.py:152-211 and solver.py:238-269.
#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

int stream_blocks(long long n, int per_thread);

static constexpr int DREC = 8;   // doubles per (trial, block) partial record

struct LocalArgs {
  const double* A;
  const double* B;
  double coef[SSNAL_MAX_TRIALS];
  double lam[SSNAL_MAX_TRIALS];
  const double* a;
  const double* l;
  const double* u;
  double lc, uc;
  long long n;
  double* x_out;
  unsigned char* free_out;
  const double* ref;
  const double* base;  // line-search base Pi (slot 0 becomes the Bregman term, proj.cu)
  double base_lam;
  double* part;  // [T][nblk][DREC]
  const SProj* sp = nullptr;  // native sharded driver: lam[t] from the device search state;
                              // eval skips trials no longer searching
};

__device__ __forceinline__ void local_elem(const LocalArgs& p, int t, long long i, double& v,
                                           double& a, double& l, double& u) {
  v = p.A[i];
  if (p.B) v = __dsub_rn(v, __dmul_rn(p.coef[t], p.B[i]));
  a = p.a[i];
  l = p.l ? p.l[i] : p.lc;
  u = p.u ? p.u[i] : p.uc;
}

// f = sum a clip(v - lam a, l, u); sR / sL = sum a^2 over slots free immediately
// right / left of lam; bR = min breakpoint > lam; bL = max breakpoint < lam; the
// breakpoint range tmin / tmax (a bracket of the root whenever the set is feasible)
__global__ void __launch_bounds__(SSNAL_NT) proj_local_eval_kernel(LocalArgs p) {
  __shared__ double red[7 * 32];
  const int t = blockIdx.y;
  if (p.sp && p.sp[t].status != SP_SEARCH) return;  // uniform per block
  const double lam = p.sp ? p.sp[t].lam : p.lam[t];
  double f = 0.0, sR = 0.0, sL = 0.0, bR = INFINITY, bL = -INFINITY;
  double tmin = INFINITY, tmax = -INFINITY;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    local_elem(p, t, i, v, a, l, u);
    const double y = __dsub_rn(v, __dmul_rn(lam, a));
    f += a * fmin(fmax(y, l), u);
    if (a != 0.0) {
      const double t1 = (v - u) / a, t2 = (v - l) / a;  // lam where y hits u, l
      const double b0 = fmin(t1, t2), b1 = fmax(t1, t2);  // free on (b0, b1)
      tmin = fmin(tmin, b0);
      tmax = fmax(tmax, b1);
      if (b0 <= lam && lam < b1) sR += a * a;
      if (b0 < lam && lam <= b1) sL += a * a;
      if (b0 > lam) bR = fmin(bR, b0);
      else if (b1 > lam) bR = fmin(bR, b1);
      if (b1 < lam) bL = fmax(bL, b1);
      else if (b0 < lam) bL = fmax(bL, b0);
    }
  }
  double vals[7] = {f, sR, sL, bR, bL, tmin, tmax};
  const int ops[7] = {0, 0, 0, 1, 2, 1, 2};
  block_reduce<7>(vals, ops, red);
  if (threadIdx.x == 0) {
    double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * DREC;
    for (int k = 0; k < 7; ++k) mine[k] = vals[k];
  }
}

// x = clip(v - lam a, l, u), free mask (ref projection.py:134-149 tolerance, as in
// proj.cu's apply) and {sum v^2 (with a base: the Bregman term), sum (v-x)^2, sum (x-ref)^2, sum_free a^2, nfree,
// sum x(2v - x)}
__global__ void __launch_bounds__(SSNAL_NT) proj_local_apply_kernel(LocalArgs p) {
  __shared__ double red[6 * 32];
  const int t = blockIdx.y;
  const double lam = p.sp ? p.sp[t].lam : p.lam[t];
  double sv2 = 0.0, sr2 = 0.0, sd2 = 0.0, sa2 = 0.0, nfree = 0.0, sxv = 0.0;
  double* xo = p.x_out ? p.x_out + (long long)t * p.n : nullptr;
  unsigned char* fo = p.free_out ? p.free_out + (long long)t * p.n : nullptr;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    local_elem(p, t, i, v, a, l, u);
    const double y = __dsub_rn(v, __dmul_rn(lam, a));
    const double x = fmin(fmax(y, l), u);
    const bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
    const bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
    const bool fr = !(lower || upper);
    if (xo) xo[i] = x;
    if (fo) fo[i] = fr ? 1 : 0;
    const double r = v - x;
    if (p.base) {
      const double xb = p.base[i];
      sv2 += (x - xb) * (v - 0.5 * (x + xb) - 0.5 * (lam + p.base_lam) * a);
    } else {
      sv2 += v * v;
    }
    sr2 += r * r;
    sxv += x * (2.0 * v - x);
    if (p.ref) { const double dd = x - p.ref[i]; sd2 += dd * dd; }
    if (fr) { sa2 += a * a; nfree += 1.0; }
  }
  double vals[6] = {sv2, sr2, sd2, sa2, nfree, sxv};
  const int ops[6] = {0, 0, 0, 0, 0, 0};
  block_reduce<6>(vals, ops, red);
  if (threadIdx.x == 0) {
    double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * DREC;
    for (int k = 0; k < 6; ++k) mine[k] = vals[k];
  }
}

// one block per trial: fold the block partials in block order -> rec[t][0..nv)
template <int NV>
__global__ void __launch_bounds__(SSNAL_NT) proj_local_fold_kernel(const double* part, int nblk,
                                                                   int mode, double* rec) {
  __shared__ double red[NV * 32];
  const int t = blockIdx.x;
  int ops[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) ops[k] = 0;
  if (mode == 0) {
    ops[3] = 1; ops[4] = 2;
    if (NV > 6) { ops[5] = 1; ops[6] = 2; }
  }
  double vals[NV];
  block_fold_partials<NV>(part + (long long)t * nblk * DREC, nblk, DREC, ops, vals, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) rec[t * DREC + k] = vals[k];
}

size_t proj_local_ws_bytes(long long n, int T) {
  return (size_t)stream_blocks(n, 4) * T * DREC * sizeof(double) + 256;
}

cudaError_t launch_proj_local(const double* A, const double* B, const double* coef,
                              const double* lam, const double* a, const double* l,
                              const double* u, double lc, double uc, long long n, int T, int mode,
                              double* x_out, uint8_t* free_out, const double* ref,
                              const double* base, double base_lam, double* rec, void* ws,
                              cudaStream_t s) {
  LocalArgs p;
  p.A = A; p.B = B; p.a = a; p.l = l; p.u = u; p.lc = lc; p.uc = uc; p.n = n;
  p.x_out = x_out; p.free_out = free_out; p.ref = ref; p.part = (double*)ws;
  p.base = base; p.base_lam = base_lam;
  for (int t = 0; t < T; ++t) {
    p.coef[t] = B ? coef[t] : 0.0;
    p.lam[t] = lam[t];
  }
  const int nblk = stream_blocks(n, 4);
  const dim3 grid(nblk, T);
  note_launch();
  if (mode == 0) proj_local_eval_kernel<<<grid, SSNAL_NT, 0, s>>>(p);
  else proj_local_apply_kernel<<<grid, SSNAL_NT, 0, s>>>(p);
  note_launch();
  if (mode == 0) proj_local_fold_kernel<7><<<T, SSNAL_NT, 0, s>>>(p.part, nblk, 0, rec);
  else proj_local_fold_kernel<6><<<T, SSNAL_NT, 0, s>>>(p.part, nblk, 1, rec);
  return cudaGetLastError();
}

// out[i] = sum_{r < k} src[r * len + i]   (r ascending)
__global__ void sum_slices_kernel(int k, long long len, const double* __restrict__ src,
                                  double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    double s = src[i];
    for (int r = 1; r < k; ++r) s += src[(long long)r * len + i];
    out[i] = s;
  }
}

cudaError_t launch_sum_slices(int k, long long len, const double* src, double* out,
                              cudaStream_t s) {
  note_launch();
  sum_slices_kernel<<<stream_blocks(len, 4), SSNAL_NT, 0, s>>>(k, len, src, out);
  return cudaGetLastError();
}

// out = alpha add + beta free (y - coef a)   (the HS-Jacobian product of ref
// projection.py:214-225 with the global coef = a_J'y_J / a_J'a_J supplied)
__global__ void hs_apply_coef_kernel(const uint8_t* __restrict__ fm, const double* __restrict__ a,
                                     const double* __restrict__ y, long long n, double beta,
                                     const double* __restrict__ add, double alpha, double coef,
                                     double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double h = fm[i] ? y[i] - coef * a[i] : 0.0;
    out[i] = (add ? alpha * add[i] : 0.0) + beta * h;
  }
}

cudaError_t launch_hs_apply_coef(const uint8_t* fm, const double* a, const double* y, long long n,
                                 double beta, const double* add, double alpha, double coef,
                                 double* out, cudaStream_t s) {
  note_launch();
  hs_apply_coef_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, s>>>(fm, a, y, n, beta, add, alpha,
                                                                 coef, out);
  return cudaGetLastError();
}

// M = I + sigma (S - shift I - u u^T / asa)   (asa == 0: no rank-one term), in place
__global__ void qspace_shift_assemble_kernel(long long m, const double* __restrict__ u, double asa,
                                             double sigma, double shift, double* __restrict__ M) {
  const double inv = asa != 0.0 ? 1.0 / asa : 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m * m;
       k += (long long)gridDim.x * blockDim.x) {
    const long long r = k / m, c = k % m;
    const double g = M[k] - (r == c ? shift : 0.0) - (u ? inv * u[r] * u[c] : 0.0);
    M[k] = (r == c ? 1.0 : 0.0) + sigma * g;
  }
}

cudaError_t launch_qspace_shift_assemble(long long m, const double* u, double asa, double sigma,
                                         double shift, double* M, cudaStream_t s) {
  note_launch();
  qspace_shift_assemble_kernel<<<(unsigned)min(ceil_div(m * m, 256LL), 4096LL), 256, 0, s>>>(
      m, u, asa, sigma, shift, M);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- native sharded driver
// The sharded projection of ssnal_alm_solve_sharded (driver.cu project_sharded): the
// multiplier search of sharded.py ShardedBackend.project run on the device.  Each pass
// evaluates every searching trial's 5-double record at its lam (proj_local_eval), the
// records are all-gathered, and sproj_update folds them in rank order and moves lam
// (safeguarded Newton on the piecewise-linear phi', exact on the affine piece that
// holds the root, ref projection.py:204-208); the apply pass writes x / the free mask
// rank-locally and sproj_finish folds the 6 sums into the global ProjState records.
static LocalArgs local_args(const ShardProj& P, const SProj* sp, double* part) {
  LocalArgs p;
  p.A = P.A; p.B = P.B; p.a = P.a; p.l = P.l; p.u = P.u; p.lc = P.lc; p.uc = P.uc; p.n = P.n;
  p.x_out = P.x_out; p.free_out = P.free_out; p.ref = P.ref; p.part = part;
  p.base = P.base; p.base_lam = P.base_lam; p.sp = sp;
  for (int t = 0; t < SSNAL_MAX_TRIALS; ++t) {
    p.coef[t] = (P.B && t < P.T) ? P.coef[t] : 0.0;
    p.lam[t] = 0.0;
  }
  return p;
}

struct SInit {
  double hints[SSNAL_MAX_TRIALS];
  double coef[SSNAL_MAX_TRIALS];
  int has_hints, T;
  double hint;
  const double *num, *den;
};

// warm starts as proj.cu: explicit per-trial hints, else the first-order start along
// the ray hint - coef * (a_J'B_J / a_J'a_J) when the slope scalars are given, else hint
__global__ void sproj_init_kernel(SInit a, SProj* sp) {
  const int t = threadIdx.x;
  if (t >= a.T) return;
  double c = a.hint;
  if (a.has_hints) c = a.hints[t];
  else if (a.num && a.den && *a.den != 0.0) c = a.hint - a.coef[t] * (*a.num / *a.den);
  sp[t] = SProj{c, -INFINITY, INFINITY, SP_SEARCH, 0};
}

cudaError_t launch_sproj_init(const ShardProj& P, SProj* sp, cudaStream_t s) {
  SInit a;
  for (int t = 0; t < SSNAL_MAX_TRIALS; ++t) {
    a.hints[t] = t < P.T ? P.hints[t] : 0.0;
    a.coef[t] = (P.B && t < P.T) ? P.coef[t] : 0.0;
  }
  a.has_hints = P.has_hints;
  a.T = P.T;
  a.hint = P.hint;
  a.num = P.B ? P.slope_num : nullptr;
  a.den = P.B ? P.slope_den : nullptr;
  note_launch();
  sproj_init_kernel<<<1, 32, 0, s>>>(a, sp);
  return cudaGetLastError();
}

cudaError_t launch_sproj_eval(const ShardProj& P, const SProj* sp, double* part, double* rec,
                              cudaStream_t s) {
  const LocalArgs p = local_args(P, sp, part);
  const int nblk = stream_blocks(P.n, 4);
  note_launch();
  proj_local_eval_kernel<<<dim3(nblk, P.T), SSNAL_NT, 0, s>>>(p);
  note_launch();
  proj_local_fold_kernel<7><<<P.T, SSNAL_NT, 0, s>>>(part, nblk, 0, rec);
  return cudaGetLastError();
}

cudaError_t launch_sproj_apply(const ShardProj& P, const SProj* sp, double* part, double* rec,
                               cudaStream_t s) {
  const LocalArgs p = local_args(P, sp, part);
  const int nblk = stream_blocks(P.n, 4);
  note_launch();
  proj_local_apply_kernel<<<dim3(nblk, P.T), SSNAL_NT, 0, s>>>(p);
  note_launch();
  proj_local_fold_kernel<6><<<P.T, SSNAL_NT, 0, s>>>(part, nblk, 1, rec);
  return cudaGetLastError();
}

// one thread per trial: fold the world's records in rank order (sum f, slopes; min of
// the breakpoints above, max below -- sharded.py ShardedBackend._fold) and take one
// step of the search (sharded.py ShardedBackend.project, the same branches)
__global__ void sproj_update_kernel(int world, int T, const double* __restrict__ rec_all,
                                    double d, SProj* sp) {
  const int t = threadIdx.x;
  if (t >= T) return;
  SProj s = sp[t];
  if (s.status != SP_SEARCH) return;
  double f = 0.0, sr = 0.0, sl = 0.0, br = INFINITY, bl = -INFINITY;
  double tmin = INFINITY, tmax = -INFINITY;
  for (int r = 0; r < world; ++r) {
    const double* x = rec_all + ((long long)r * T + t) * DREC;
    f += x[0]; sr += x[1]; sl += x[2];
    br = fmin(br, x[3]);
    bl = fmax(bl, x[4]);
    tmin = fmin(tmin, x[5]);
    tmax = fmax(tmax, x[6]);
  }
  // phi' is constant below tmin and above tmax, so [tmin, tmax] brackets the root of
  // a feasible set (the Newton / flat steps below never leave it)
  if (isfinite(tmin) && tmin > s.lo) s.lo = tmin;
  if (isfinite(tmax) && tmax < s.hi) s.hi = tmax;
  ++s.passes;
  const double g = d - f, c = s.lam;
  double ln;
  if (g < 0.0) {  // root to the right (phi' = d - f is non-decreasing)
    s.lo = fmax(s.lo, c);
    if (sr > 0.0) {
      ln = c - g / sr;
      if (ln <= br) { s.lam = ln; s.status = SP_DONE; sp[t] = s; return; }
    } else {
      if (!isfinite(br)) { s.status = SP_INFEAS_HIGH; sp[t] = s; return; }
      ln = br;
    }
  } else {  // root at or left of c
    // g == 0: c is a root.  Where phi' is flat left of c no slot is free there, so every
    // root of the flat piece gives the same x and free mask: stop (walking left one
    // breakpoint per pass to the leftmost root would cost a pass per breakpoint)
    if (g == 0.0) { s.status = SP_DONE; sp[t] = s; return; }
    s.hi = fmin(s.hi, c);
    if (sl > 0.0) {
      ln = c - g / sl;
      if (ln >= bl) { s.lam = ln; s.status = SP_DONE; sp[t] = s; return; }
    } else {
      if (!isfinite(bl)) { s.status = SP_INFEAS_LOW; sp[t] = s; return; }
      ln = bl;
    }
  }
  // safeguard: outside the bracket, or every other pass once the warm-started Newton has
  // had 3 (a walk through breakpoints of flat pieces then halves the bracket at least
  // every second pass)
  if (isfinite(s.lo) && isfinite(s.hi) && (!(s.lo < ln && ln < s.hi) || (s.passes > 3 && (s.passes & 1))))
    ln = 0.5 * (s.lo + s.hi);
  s.lam = ln;
  sp[t] = s;
}

cudaError_t launch_sproj_update(int world, int T, const double* rec_all, double d, SProj* sp,
                                cudaStream_t s) {
  note_launch();
  sproj_update_kernel<<<1, 32, 0, s>>>(world, T, rec_all, d, sp);
  return cudaGetLastError();
}

// global records from the apply pass: sums folded in rank order; the search state's
// lam / bracket / status; in_count = THIS rank's free slots (the row count of its J)
__global__ void sproj_finish_kernel(int world, int T, const double* __restrict__ rec_all,
                                    const double* __restrict__ rec_loc, const SProj* sp,
                                    int base_mode, ProjState* st) {
  const int t = threadIdx.x;
  if (t >= T) return;
  double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < world; ++r) {
    const double* x = rec_all + ((long long)r * T + t) * DREC;
    for (int k = 0; k < 6; ++k) v[k] += x[k];
  }
  const SProj s = sp[t];
  ProjState o;
  memset(&o, 0, sizeof o);
  o.lo = s.lo;
  o.hi = s.hi;
  o.lam = s.lam;
  o.tmin = o.tmax = s.lam;
  if (base_mode) { o.sum_bh = v[0]; o.sum_v2 = 0.0; } else { o.sum_v2 = v[0]; }
  o.sum_r2 = v[1];
  o.sum_dref2 = v[2];
  o.sum_a2_free = v[3];
  o.nfree = llround(v[4]);
  o.sum_xv = v[5];
  o.in_count = llround(rec_loc[t * DREC + 4]);
  o.status = s.status == SP_DONE ? PROJ_APPLIED
             : s.status == SP_INFEAS_LOW ? PROJ_INFEASIBLE_LOW
             : s.status == SP_INFEAS_HIGH ? PROJ_INFEASIBLE_HIGH
                                          : PROJ_NEWTON;
  o.passes = s.passes;
  st[t] = o;
}

cudaError_t launch_sproj_finish(int world, int T, const double* rec_all, const double* rec_loc,
                                const SProj* sp, int base_mode, ProjState* st, cudaStream_t s) {
  note_launch();
  sproj_finish_kernel<<<1, 32, 0, s>>>(world, T, rec_all, rec_loc, sp, base_mode, st);
  return cudaGetLastError();
}

}  // namespace ssnal

// Projection onto K cap L = {x : a'x = d, l <= x <= u} on sm_100a.
//
// Replaces ref projection.py:152-211 (project_box_line) and :134-149 (_classify).
// The reference sorts all 2n breakpoints and binary-searches them with one
// O(n) grad_phi evaluation per probe.  Here the root of the non-decreasing
// piecewise-linear phi'(lambda) = d - a'clip(v - lambda a, l, u) is bracketed by
// a K-ary search in lambda (K = 32 sub-intervals per pass, all 31 probes summed in
// registers in ONE streaming pass), then the bracket is closed onto the two
// ADJACENT breakpoints t_l < t_u of the reference's sorted array and lambda is
// the reference's interpolation  t_l - f_l (t_u - t_l) / (f_u - f_l)  with f_l,
// f_u direct deterministic sums.  No sort, no atomics on floating-point data;
// every reduction is a fixed-order two-stage tree, so results are bit-
// reproducible run to run.
//
// Batching: blockIdx.y = trial t evaluates v_t = A - coef[t] * B, which is how
// the Armijo line search evaluates several step lengths in one launch sequence.
//
// Phases (one launch each, every phase closes with a last-block-done finalize):
//   range  : tmin / tmax over breakpoints, f(-inf), f(+inf)          (status 0|2|<0)
//   pass   : 31 probe sums + in-bracket breakpoint stats -> narrower bracket (x P)
//   exact  : direct sums at <= 4 candidate breakpoints -> lambda      (status 2)
//   apply  : x = clip(v - lambda a), free mask, fused reductions
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>

#include "common.cuh"
#include "ssnal_internal.h"

namespace cg = cooperative_groups;

namespace ssnal {

static constexpr int KSUB = 32;          // sub-intervals per pass
static constexpr int NPROBE = KSUB - 1;  // interior probes per pass
static constexpr int PSTRIDE = 40;       // doubles per block partial record

struct ProjArgs {
  const double* A;
  const double* B;
  double coef[SSNAL_MAX_TRIALS];
  double hints[SSNAL_MAX_TRIALS];  // per-trial warm starts (multi-trial kernel), has_hints
  int has_hints;
  // first-order warm start along the ray v = A - coef B: lambda(coef) ~ hint - coef *
  // (*slope_num / *slope_den) (the free-set sums a_J'B_J and a_J'a_J of the base point,
  // device scalars), when set and no explicit hints
  const double* slope_num;
  const double* slope_den;
  const double* a;
  const double* l;
  const double* u;
  double lc, uc, d;
  long long n;
  ProjState* st;
  double* part;  // [T][nblk][PSTRIDE]
  double* x_out;             // [T][n] or null
  unsigned char* free_out;   // [T][n] or null
  const double* ref;         // reference vector for sum (x - ref)^2, or null
  const double* base;        // Pi at the line-search base point, or null (see bregman_term)
  double base_lam;           // its multiplier
};

// Line-search trial from the base point u (projection Pi, multiplier lam_b) to
// v = u - coef*Qd (projection x, multiplier lam): the i-th term of the Bregman
// divergence of h(v) = 1/2 ||v||^2 - 1/2 dist(v, K)^2 (grad h = Pi),
//   B_h = sum_i (x_i - Pi_i)(v_i - (x_i + Pi_i)/2 - lam_bar a_i),  lam_bar = (lam + lam_b)/2
// (the lam_bar a shift is exact since a'x = a'Pi = d and removes the large part of
// every free-slot term).  psi(w + alpha d) - psi(w) = alpha g'd + alpha^2 d'Qd / 2 + B_h / sigma
// then needs no difference of O(||u||^2) sums.
__device__ __forceinline__ double bregman_term(double x, double xb, double v, double a,
                                               double lam_bar) {
  return (x - xb) * (v - 0.5 * (x + xb) - lam_bar * a);
}

// (v - bound) / a with numpy's rounding; division by +-1 is exact in IEEE arithmetic,
// so the SVM duals (a = labels or (e; -e)) skip the DP division bit-identically
__device__ __forceinline__ double bp_div(double x, double a) {
  return a == 1.0 ? x : (a == -1.0 ? -x : __ddiv_rn(x, a));
}

__device__ __forceinline__ void load_elem(const ProjArgs& p, int t, long long i, double& v,
                                          double& a, double& l, double& u) {
  v = p.A[i];
  if (p.B) v = __dsub_rn(v, __dmul_rn(p.coef[t], p.B[i]));
  a = p.a[i];
  l = p.l ? p.l[i] : p.lc;
  u = p.u ? p.u[i] : p.uc;
}

// a * clip(v - lam a, l, u) with numpy's rounding for v - lam*a (no fma contraction)
__device__ __forceinline__ double contrib(double v, double a, double l, double u, double lam) {
  double y = __dsub_rn(v, __dmul_rn(lam, a));
  return a * fmin(fmax(y, l), u);
}

__device__ __forceinline__ double probe_at(const ProjState& s, int k) {
  // k in [0, KSUB]; k = 0 -> lo, k = KSUB -> hi exactly
  if (k <= 0) return s.lo;
  if (k >= KSUB) return s.hi;
  double h = (s.hi - s.lo) / KSUB;
  return s.lo + (double)k * h;
}

// ------------------------------------------------------------------ range
__global__ void __launch_bounds__(SSNAL_NT) proj_range_kernel(ProjArgs p) {
  __shared__ double red[5 * 32];
  const int t = blockIdx.y;
  ProjState* st = p.st + t;
  double tmin = INFINITY, tmax = -INFINITY, s_left = 0.0, s_right = 0.0, nnz = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    load_elem(p, t, i, v, a, l, u);
    if (a != 0.0) {
      double t1 = bp_div(__dsub_rn(v, u), a), t2 = bp_div(__dsub_rn(v, l), a);
      tmin = fmin(tmin, fmin(t1, t2));
      tmax = fmax(tmax, fmax(t1, t2));
      nnz += 1.0;
      // saturation values: lambda -> -inf puts a>0 slots at u, a<0 slots at l
      s_left += a > 0.0 ? a * u : a * l;
      s_right += a > 0.0 ? a * l : a * u;
    }
  }
  double vals[5] = {tmin, tmax, s_left, s_right, nnz};
  const int ops[5] = {1, 2, 0, 0, 0};
  block_reduce<5>(vals, ops, red);
  double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * PSTRIDE;
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) mine[k] = vals[k];
  if (!last_block_arrive(&st->ticket, gridDim.x)) return;
  block_fold_partials<5>(p.part + (long long)t * gridDim.x * PSTRIDE, gridDim.x, PSTRIDE, ops,
                         vals, red);
  if (threadIdx.x != 0) return;
  const double r0 = vals[0], r1 = vals[1], r2 = vals[2], r3 = vals[3], r4 = vals[4];
  st->tmin = r0;
  st->tmax = r1;
  st->passes = 0;
  st->in_count = -1;
  if (r4 == 0.0) {  // a == 0: equality constraint is 0 = d, project by clipping
    st->lam = 0.0;
    st->status = PROJ_DONE;
    return;
  }
  double f_neg = p.d - r2, f_pos = p.d - r3;
  if (f_neg >= 0.0) {  // ref projection.py:186-191
    st->lam = r0;
    st->status = f_neg > 1e-9 * (1.0 + fabs(p.d)) ? PROJ_INFEASIBLE_LOW : PROJ_DONE;
    return;
  }
  if (f_pos < 0.0) {  // ref projection.py:192-193
    st->status = PROJ_INFEASIBLE_HIGH;
    return;
  }
  st->lo = r0;
  st->hi = r1;
  st->flo = f_neg;
  st->fhi = f_pos;
  st->below_max = r0;
  st->above_min = INFINITY;
  st->status = PROJ_SEARCH;
}

// ------------------------------------------------------------------ pass
__global__ void __launch_bounds__(SSNAL_NT) proj_pass_kernel(ProjArgs p) {
  __shared__ double red[(NPROBE + 8) * 32];
  const int t = blockIdx.y;
  ProjState* st = p.st + t;
  if (st->status != PROJ_SEARCH && st->status != PROJ_NEWTON) return;  // uniform across grid
  ProjState s = *st;
  if (s.status == PROJ_NEWTON) {  // fallback after the Newton passes: finite bracket
    if (!(s.lo > -INFINITY)) s.lo = s.tmin;
    if (!(s.hi < INFINITY)) s.hi = s.tmax;
    s.below_max = -INFINITY;
    s.above_min = INFINITY;
  }
  const double lo = s.lo, hi = s.hi;
  double acc[NPROBE];
#pragma unroll
  for (int k = 0; k < NPROBE; ++k) acc[k] = 0.0;
  double s_const = 0.0, s_slope = 0.0;  // settled slots: sum of (alpha + beta lambda)
  double bmax = -INFINITY, amin = INFINITY, imin = INFINITY, imax = -INFINITY, icnt = 0.0;
  double probes[NPROBE];
#pragma unroll
  for (int k = 0; k < NPROBE; ++k) probes[k] = probe_at(s, k + 1);

  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    load_elem(p, t, i, v, a, l, u);
    if (a == 0.0) continue;
    double t1 = bp_div(__dsub_rn(v, u), a), t2 = bp_div(__dsub_rn(v, l), a);
    double ta = fmin(t1, t2), tb = fmax(t1, t2);
    bool in_a = ta > lo && ta <= hi, in_b = tb > lo && tb <= hi;
    if (ta <= lo) bmax = fmax(bmax, ta); else if (ta > hi) amin = fmin(amin, ta);
    if (tb <= lo) bmax = fmax(bmax, tb); else if (tb > hi) amin = fmin(amin, tb);
    if (in_a) { icnt += 1.0; imin = fmin(imin, ta); imax = fmax(imax, ta); }
    if (in_b) { icnt += 1.0; imin = fmin(imin, tb); imax = fmax(imax, tb); }
    if (in_a || in_b) {
#pragma unroll
      for (int k = 0; k < NPROBE; ++k) acc[k] += contrib(v, a, l, u, probes[k]);
    } else if (tb <= lo) {  // saturated on the right side over the whole bracket
      s_const += a > 0.0 ? a * l : a * u;
    } else if (ta > hi) {   // saturated on the left side
      s_const += a > 0.0 ? a * u : a * l;
    } else {                // linear over the whole bracket: a v - a^2 lambda
      s_const += a * v;
      s_slope -= a * a;
    }
  }
  // reduce: probes (sum), s_const, s_slope (sum), bmax (max), amin, imin (min), imax, icnt
  double vals[NPROBE + 7];
  int ops[NPROBE + 7];
#pragma unroll
  for (int k = 0; k < NPROBE; ++k) { vals[k] = acc[k]; ops[k] = 0; }
  vals[NPROBE + 0] = s_const; ops[NPROBE + 0] = 0;
  vals[NPROBE + 1] = s_slope; ops[NPROBE + 1] = 0;
  vals[NPROBE + 2] = bmax;    ops[NPROBE + 2] = 2;
  vals[NPROBE + 3] = amin;    ops[NPROBE + 3] = 1;
  vals[NPROBE + 4] = imin;    ops[NPROBE + 4] = 1;
  vals[NPROBE + 5] = imax;    ops[NPROBE + 5] = 2;
  vals[NPROBE + 6] = icnt;    ops[NPROBE + 6] = 0;
  block_reduce<NPROBE + 7>(vals, ops, red);
  double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * PSTRIDE;
  if (threadIdx.x == 0)
    for (int k = 0; k < NPROBE + 7; ++k) mine[k] = vals[k];
  if (!last_block_arrive(&st->ticket, gridDim.x)) return;
  double tot[NPROBE + 7];
  block_fold_partials<NPROBE + 7>(p.part + (long long)t * gridDim.x * PSTRIDE, gridDim.x,
                                  PSTRIDE, ops, tot, red);
  if (threadIdx.x != 0) return;
  const double below = fmax(s.below_max, tot[NPROBE + 2]);
  const double above = fmin(s.above_min, tot[NPROBE + 3]);
  const double in_min = tot[NPROBE + 4], in_max = tot[NPROBE + 5];
  const long long in_cnt = (long long)tot[NPROBE + 6];
  st->passes = s.passes + 1;
  st->status = PROJ_SEARCH;
  st->below_max = below;
  st->above_min = above;
  st->in_count = in_cnt;
  st->in_min = in_min;
  st->in_max = in_max;
  const double width = hi - lo;
  const bool tiny = !(width > 4.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)));
  if (in_cnt == 0 || in_min == in_max || tiny) {
    st->status = PROJ_BRACKETED;  // the exact phase closes onto adjacent breakpoints
    return;
  }
  // f(probe_k) = d - (sum over unsettled + s_const + s_slope * probe_k); pick the first
  // sub-interval whose right end has f >= 0.
  int k_hit = KSUB;
  for (int k = 1; k < KSUB; ++k) {
    double fk = p.d - (tot[k - 1] + tot[NPROBE] + tot[NPROBE + 1] * probe_at(s, k));
    if (fk >= 0.0) { k_hit = k; break; }
  }
  double new_lo = probe_at(s, k_hit - 1), new_hi = probe_at(s, k_hit);
  st->lo = new_lo;
  st->hi = new_hi;
}

// ------------------------------------------------------------------ newton
// Safeguarded Newton on the piecewise-affine phi'(lambda), O(1) work per slot per
// pass: at the current point c one pass sums f(c), the slopes of the segments left
// and right of c (sum of a_i^2 over slots free there) and the nearest breakpoints
// on either side.  If the affine root of the segment the sign of f(c) points into
// lies inside that segment it IS the multiplier (same affine piece the reference
// interpolates on, ref projection.py:204-208); otherwise c moves to the Newton
// point (or the next breakpoint on a flat piece, or the bracket midpoint) and the
// bracket [lo, hi] with f(lo) < 0 <= f(hi) shrinks.  Warm-started from the
// previous multiplier, one or two passes suffice in the line search.
__global__ void __launch_bounds__(SSNAL_NT) proj_newton_kernel(ProjArgs p, int fresh,
                                                               double hint) {
  __shared__ double red[8 * 32];
  const int t = blockIdx.y;
  ProjState* st = p.st + t;
  if (!fresh && st->status != PROJ_NEWTON) return;
  const double c = fresh ? hint : st->lam;
  double fsum = 0.0, sp = 0.0, sm = 0.0, amin = INFINITY, bmax = -INFINITY;
  double tmin = INFINITY, tmax = -INFINITY, nnz = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    load_elem(p, t, i, v, a, l, u);
    if (a == 0.0) continue;
    double t1 = bp_div(__dsub_rn(v, u), a), t2 = bp_div(__dsub_rn(v, l), a);
    double ta = fmin(t1, t2), tb = fmax(t1, t2);
    fsum += contrib(v, a, l, u, c);
    const double a2 = a * a;
    if (ta <= c && c < tb) sp += a2;  // free just right of c
    if (ta < c && c <= tb) sm += a2;  // free just left of c
    if (ta > c) amin = fmin(amin, ta); else if (ta < c) bmax = fmax(bmax, ta);
    if (tb > c) amin = fmin(amin, tb); else if (tb < c) bmax = fmax(bmax, tb);
    tmin = fmin(tmin, ta);
    tmax = fmax(tmax, tb);
    nnz += 1.0;
  }
  double vals[8] = {fsum, sp, sm, amin, bmax, tmin, tmax, nnz};
  const int ops[8] = {0, 0, 0, 1, 2, 1, 2, 0};
  block_reduce<8>(vals, ops, red);
  double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * PSTRIDE;
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) mine[k] = vals[k];
  if (!last_block_arrive(&st->ticket, gridDim.x)) return;
  block_fold_partials<8>(p.part + (long long)t * gridDim.x * PSTRIDE, gridDim.x, PSTRIDE, ops,
                         vals, red);
  if (threadIdx.x != 0) return;
  const double f = p.d - vals[0], slope_r = vals[1], slope_l = vals[2];
  const double above = vals[3], below = vals[4];
  double lo, hi;
  int passes;
  if (fresh) {
    lo = -INFINITY;
    hi = INFINITY;
    passes = 0;
    st->tmin = vals[5];
    st->tmax = vals[6];
    st->in_count = -1;
    if (vals[7] == 0.0) {  // a == 0: constraint 0 = d, project by clipping
      st->lam = 0.0;
      st->status = PROJ_DONE;
      st->passes = 1;
      return;
    }
  } else {
    lo = st->lo;
    hi = st->hi;
    passes = st->passes;
  }
  ++passes;
  st->passes = passes;
  double next;
  // f >= 0 branch also covers f == 0: the reference returns the LEFTMOST root (first
  // sorted breakpoint with f >= 0, interpolated against its predecessor), so a zero
  // on a flat piece keeps stepping left to where the flat zero piece starts.
  if (f < 0.0) {
    lo = c;
    if (!(above < INFINITY)) {  // right of every breakpoint: phi'(+inf) < 0
      st->status = PROJ_INFEASIBLE_HIGH;
      return;
    }
    if (slope_r > 0.0) {
      const double r = c - f / slope_r;
      if (r <= above) {
        st->lam = r;
        st->status = PROJ_DONE;
        return;
      }
      lo = above;  // phi'(above) = f + slope (above - c) < 0
      next = r;
    } else {
      next = above;  // flat piece: step to the next breakpoint
    }
  } else {
    hi = c;
    if (!(below > -INFINITY)) {  // left of every breakpoint: phi'(-inf) >= 0
      // ref projection.py:186-191: lambda = smallest breakpoint (or infeasible)
      st->lam = st->tmin;
      st->status = f > 1e-9 * (1.0 + fabs(p.d)) ? PROJ_INFEASIBLE_LOW : PROJ_DONE;
      return;
    }
    if (slope_l > 0.0) {
      const double r = c - f / slope_l;
      if (r >= below) {
        st->lam = r;
        st->status = PROJ_DONE;
        return;
      }
      hi = below;  // phi'(below) = f - slope (c - below) > 0
      next = r;
    } else {
      next = below;
    }
  }
  // safeguard: stay strictly inside the bracket, bisect when Newton leaves it
  const bool flat_step = (f < 0.0 && !(slope_r > 0.0)) || (f >= 0.0 && !(slope_l > 0.0));
  if (!flat_step && !(next > lo && next < hi)) {
    if (lo > -INFINITY && hi < INFINITY) next = 0.5 * (lo + hi);
    else if (lo > -INFINITY) next = f < 0.0 ? above : lo + 2.0 * (c - lo) + 1.0;
    else next = below;
  }
  st->lo = lo;
  st->hi = hi;
  st->lam = next;
  st->status = PROJ_NEWTON;
}

// ------------------------------------------------------------------ exact
// Candidates are sorted breakpoint values; f is evaluated by direct sums.
__global__ void __launch_bounds__(SSNAL_NT) proj_exact_kernel(ProjArgs p) {
  __shared__ double red[4 * 32];
  __shared__ double cand_s[4];
  __shared__ int ncand_s;
  const int t = blockIdx.y;
  ProjState* st = p.st + t;
  if (st->status != PROJ_BRACKETED) return;
  if (threadIdx.x == 0) {
    const ProjState s = *st;
    int nc = 0;
    cand_s[nc++] = s.below_max;
    if (s.in_count > 0) {
      cand_s[nc++] = s.in_min;
      if (s.in_max != s.in_min) cand_s[nc++] = s.in_max;
    }
    if (s.above_min < INFINITY) cand_s[nc++] = s.above_min;
    ncand_s = nc;
  }
  __syncthreads();
  const int nc = ncand_s;
  double cand[4];
  for (int k = 0; k < 4; ++k) cand[k] = k < nc ? cand_s[k] : 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    load_elem(p, t, i, v, a, l, u);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < nc) acc[k] += contrib(v, a, l, u, cand[k]);
  }
  const int ops[4] = {0, 0, 0, 0};
  block_reduce<4>(acc, ops, red);
  double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * PSTRIDE;
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) mine[k] = acc[k];
  if (!last_block_arrive(&st->ticket, gridDim.x)) return;
  double f[4];
  block_fold_partials<4>(p.part + (long long)t * gridDim.x * PSTRIDE, gridDim.x, PSTRIDE, ops, f,
                         red);
  if (threadIdx.x != 0) return;
  for (int k = 0; k < nc; ++k) f[k] = p.d - f[k];
  // first candidate with f >= 0 is t_u; its predecessor is t_l (ref projection.py:195-208)
  int iu = nc - 1;
  for (int k = 0; k < nc; ++k)
    if (f[k] >= 0.0) { iu = k; break; }
  double lam;
  if (iu == 0) {
    lam = cand[0];  // rounding put the root at/below t_l: flat zero segment
  } else {
    const double tl = cand[iu - 1], tu = cand[iu], fl = f[iu - 1], fu = f[iu];
    if (fu == fl || tu == tl) lam = tl;
    else lam = tl - fl * (tu - tl) / (fu - fl);
  }
  st->lam = lam;
  st->status = PROJ_DONE;
}

// ------------------------------------------------------------------ apply
__global__ void __launch_bounds__(SSNAL_NT) proj_apply_kernel(ProjArgs p) {
  __shared__ double red[6 * 32];
  const int t = blockIdx.y;
  ProjState* st = p.st + t;
  if (st->status != PROJ_DONE) return;
  const double lam = st->lam;
  double sv2 = 0.0, sr2 = 0.0, sd2 = 0.0, sa2 = 0.0, nfree = 0.0, sxv = 0.0;
  double* xo = p.x_out ? p.x_out + (long long)t * p.n : nullptr;
  unsigned char* fo = p.free_out ? p.free_out + (long long)t * p.n : nullptr;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v, a, l, u;
    load_elem(p, t, i, v, a, l, u);
    double y = __dsub_rn(v, __dmul_rn(lam, a));
    double x = fmin(fmax(y, l), u);
    // ref projection.py:134-149: bound slots within 1e-12 (1 + |bound|)
    bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
    bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
    bool fr = !(lower || upper);
    if (xo) xo[i] = x;
    if (fo) fo[i] = fr ? 1 : 0;
    double r = v - x;
    sv2 += p.base ? bregman_term(x, p.base[i], v, a, 0.5 * (lam + p.base_lam)) : v * v;
    sr2 += r * r;
    sxv += x * (2.0 * v - x);
    if (p.ref) { double dd = x - p.ref[i]; sd2 += dd * dd; }
    if (fr) { sa2 += a * a; nfree += 1.0; }
  }
  double vals[6] = {sv2, sr2, sd2, sa2, nfree, sxv};
  const int ops[6] = {0, 0, 0, 0, 0, 0};
  block_reduce<6>(vals, ops, red);
  double* mine = p.part + ((long long)t * gridDim.x + blockIdx.x) * PSTRIDE;
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) mine[k] = vals[k];
  if (!last_block_arrive(&st->ticket, gridDim.x)) return;
  double r[6];
  block_fold_partials<6>(p.part + (long long)t * gridDim.x * PSTRIDE, gridDim.x, PSTRIDE, ops, r,
                         red);
  if (threadIdx.x != 0) return;
  st->sum_v2 = p.base ? 0.0 : r[0];
  st->sum_bh = p.base ? r[0] : 0.0;
  st->sum_r2 = r[1];
  st->sum_dref2 = r[2];
  st->sum_a2_free = r[3];
  st->nfree = (long long)r[4];
  st->sum_xv = r[5];
  st->status = PROJ_APPLIED;
}

// ------------------------------------------------------------------ fused
// The whole default search (warm-started Newton passes, then apply) as ONE
// cooperative launch: passes are separated by grid-wide barriers instead of
// kernel boundaries, every block folds the (tiny) per-block partials of its
// trial itself -- in the same fixed order, so all blocks hold bit-identical
// state and branch uniformly -- and the apply pass follows without a return to
// the host.  A trial still searching after max_newton passes is written back with
// status NEWTON for the multi-launch K-ary fallback.
__device__ __forceinline__ void newton_update(double f, double slope_r, double slope_l,
                                              double above, double below, double tmin, double d,
                                              double& c, double& lo, double& hi, double& lam,
                                              int& status) {
  double next;
  if (f < 0.0) {
    lo = c;
    if (!(above < INFINITY)) { status = PROJ_INFEASIBLE_HIGH; return; }
    if (slope_r > 0.0) {
      const double r = c - f / slope_r;
      if (r <= above) { lam = r; status = PROJ_DONE; return; }
      lo = above;
      next = r;
    } else {
      next = above;
    }
  } else {
    hi = c;
    if (!(below > -INFINITY)) {
      lam = tmin;
      status = f > 1e-9 * (1.0 + fabs(d)) ? PROJ_INFEASIBLE_LOW : PROJ_DONE;
      return;
    }
    if (slope_l > 0.0) {
      const double r = c - f / slope_l;
      if (r >= below) { lam = r; status = PROJ_DONE; return; }
      hi = below;
      next = r;
    } else {
      next = below;
    }
  }
  const bool flat_step = (f < 0.0 && !(slope_r > 0.0)) || (f >= 0.0 && !(slope_l > 0.0));
  if (!flat_step && !(next > lo && next < hi)) {
    if (lo > -INFINITY && hi < INFINITY) next = 0.5 * (lo + hi);
    else if (lo > -INFINITY) next = f < 0.0 ? above : lo + 2.0 * (c - lo) + 1.0;
    else next = below;
  }
  c = next;
  status = PROJ_NEWTON;
}

__global__ void __launch_bounds__(SSNAL_NT) proj_fused_kernel(ProjArgs p, double hint,
                                                              int max_newton, int* active) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[8 * 32];
  __shared__ double sh[8];
  __shared__ int sh_status;
  const int t = blockIdx.y;
  const unsigned nb = gridDim.x;
  const long long region = (long long)gridDim.y * nb * PSTRIDE;
  double c = hint, lo = -INFINITY, hi = INFINITY, lam = 0.0, tmin = INFINITY, tmax = -INFINITY;
  int status = PROJ_NEWTON, passes = 0;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *active = (int)gridDim.y;
  for (int pass = 0;; ++pass) {
    double* part = p.part + (pass & 1) * region + (long long)t * nb * PSTRIDE;
    const int ops[8] = {0, 0, 0, 1, 2, 1, 2, 0};
    double vals[8] = {0.0, 0.0, 0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0};
    if (status == PROJ_NEWTON) {
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
           i += (long long)nb * blockDim.x) {
        double v, a, l, u;
        load_elem(p, t, i, v, a, l, u);
        if (a == 0.0) continue;
        const double t1 = bp_div(__dsub_rn(v, u), a), t2 = bp_div(__dsub_rn(v, l), a);
        const double ta = fmin(t1, t2), tb = fmax(t1, t2);
        vals[0] += contrib(v, a, l, u, c);
        const double a2 = a * a;
        if (ta <= c && c < tb) vals[1] += a2;
        if (ta < c && c <= tb) vals[2] += a2;
        if (ta > c) vals[3] = fmin(vals[3], ta); else if (ta < c) vals[4] = fmax(vals[4], ta);
        if (tb > c) vals[3] = fmin(vals[3], tb); else if (tb < c) vals[4] = fmax(vals[4], tb);
        vals[5] = fmin(vals[5], ta);
        vals[6] = fmax(vals[6], tb);
        vals[7] += 1.0;
      }
      block_reduce<8>(vals, ops, red);
      if (threadIdx.x == 0)
        for (int k = 0; k < 8; ++k) part[(long long)blockIdx.x * PSTRIDE + k] = vals[k];
    }
    grid.sync();
    bool finished_now = false;
    if (status == PROJ_NEWTON) {
      block_fold_partials<8>(part, nb, PSTRIDE, ops, vals, red);
      if (threadIdx.x == 0) {
        ++passes;
        if (pass == 0) { tmin = vals[5]; tmax = vals[6]; }
        if (vals[7] == 0.0) {
          lam = 0.0;
          status = PROJ_DONE;
        } else {
          newton_update(p.d - vals[0], vals[1], vals[2], vals[3], vals[4], tmin, p.d, c, lo, hi,
                        lam, status);
        }
        sh[0] = c; sh[1] = lo; sh[2] = hi; sh[3] = lam; sh[4] = tmin; sh[5] = tmax;
        sh[6] = (double)passes;
        sh_status = status;
      }
      __syncthreads();
      c = sh[0]; lo = sh[1]; hi = sh[2]; lam = sh[3]; tmin = sh[4]; tmax = sh[5];
      passes = (int)sh[6];
      status = sh_status;
      finished_now = status != PROJ_NEWTON;
      __syncthreads();
    }
    if (gridDim.y == 1) {  // single trial: every block knows the status
      if (status != PROJ_NEWTON || pass + 1 >= max_newton) break;
    } else {
      if (finished_now && blockIdx.x == 0 && threadIdx.x == 0) atomicSub(active, 1);
      grid.sync();
      const int left = *(volatile int*)active;
      if (left == 0 || pass + 1 >= max_newton) break;
    }
  }
  // apply (region 2)
  double* part = p.part + 2 * region + (long long)t * nb * PSTRIDE;
  if (status == PROJ_DONE) {
    double s6[6] = {0, 0, 0, 0, 0, 0};
    double* xo = p.x_out ? p.x_out + (long long)t * p.n : nullptr;
    unsigned char* fo = p.free_out ? p.free_out + (long long)t * p.n : nullptr;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
         i += (long long)nb * blockDim.x) {
      double v, a, l, u;
      load_elem(p, t, i, v, a, l, u);
      const double y = __dsub_rn(v, __dmul_rn(lam, a));
      const double x = fmin(fmax(y, l), u);
      const bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
      const bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
      const bool fr = !(lower || upper);
      if (xo) xo[i] = x;
      if (fo) fo[i] = fr ? 1 : 0;
      const double r = v - x;
      s6[0] += p.base ? bregman_term(x, p.base[i], v, a, 0.5 * (lam + p.base_lam)) : v * v;
      s6[1] += r * r;
      if (p.ref) { const double dd = x - p.ref[i]; s6[2] += dd * dd; }
      if (fr) { s6[3] += a * a; s6[4] += 1.0; }
      s6[5] += x * (2.0 * v - x);
    }
    const int ops6[6] = {0, 0, 0, 0, 0, 0};
    block_reduce<6>(s6, ops6, red);
    if (threadIdx.x == 0)
      for (int k = 0; k < 6; ++k) part[(long long)blockIdx.x * PSTRIDE + k] = s6[k];
  }
  grid.sync();
  if (blockIdx.x != 0) return;
  ProjState* st = p.st + t;
  if (status == PROJ_DONE) {
    double r[6];
    const int ops6[6] = {0, 0, 0, 0, 0, 0};
    block_fold_partials<6>(part, nb, PSTRIDE, ops6, r, red);
    if (threadIdx.x != 0) return;
    st->sum_v2 = p.base ? 0.0 : r[0];
    st->sum_bh = p.base ? r[0] : 0.0;
    st->sum_r2 = r[1];
    st->sum_dref2 = r[2];
    st->sum_a2_free = r[3];
    st->nfree = (long long)r[4];
    st->sum_xv = r[5];
    st->lam = lam;
    st->status = PROJ_APPLIED;
  } else {
    if (threadIdx.x != 0) return;
    st->lam = c;  // Newton iterate for the fallback (or tmin for infeasible-low)
    st->lo = lo;
    st->hi = hi;
    st->status = status;
  }
  st->tmin = tmin;
  st->tmax = tmax;
  st->passes = passes;
  st->in_count = -1;
}

// ------------------------------------------------------------------ cluster
// Small-n variant (n <= CL_CTAS * CL_NT * CL_EPT, e.g. the 50,000-slot config-1
// dual): one thread-block CLUSTER of 16 CTAs per trial, every slot's (v, a) held in
// registers across all passes (read from HBM/L2 once), and the per-pass reduction
// exchanged through distributed shared memory: each CTA publishes its 8-value
// partial, one cluster barrier, every CTA folds the 16 partials in rank order (so
// all hold identical state) and takes the Newton step itself.  No grid-wide
// barrier, no second launch, and the T line-search trials run as T independent
// clusters side by side.  Partials are double-buffered by pass parity: a CTA can
// only overwrite a buffer after every CTA has passed the following barrier.
#ifndef SSNAL_CL_CTAS
#define SSNAL_CL_CTAS 16
#define SSNAL_CL_EPT 8
#endif
static constexpr int CL_CTAS = SSNAL_CL_CTAS;
static constexpr int CL_NT = 512;
static constexpr int CL_EPT = SSNAL_CL_EPT;
static constexpr int CL_MAX_PASSES = 12;
static constexpr int CL_SMEM = 2 * CL_EPT * CL_NT * (int)sizeof(double);

__global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_NT, 1)
    proj_cluster_kernel(ProjArgs p, double hint) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double red[8 * 32];
  __shared__ double gath[2][CL_CTAS][8];  // [pass parity][source rank][slot], filled by pushes
  __shared__ double sh[8];
  __shared__ int sh_status;
  // breakpoints do not depend on lambda: computed once (two divisions per slot),
  // kept in shared memory beside the registers holding v and a
  extern __shared__ double bp_dyn[];  // [2][CL_EPT][CL_NT]
  double (*bpa)[CL_NT] = reinterpret_cast<double (*)[CL_NT]>(bp_dyn);
  double (*bpb)[CL_NT] = reinterpret_cast<double (*)[CL_NT]>(bp_dyn + CL_EPT * CL_NT);
  const unsigned rank = cluster.block_rank();
  const int t = blockIdx.y;
  const int tid = threadIdx.x;
  const long long stride = (long long)CL_CTAS * CL_NT;
  const long long base = (long long)rank * CL_NT + tid;
  double v[CL_EPT], a[CL_EPT];
  // all loads first (every element's request in flight at once), then the math
#pragma unroll
  for (int k = 0; k < CL_EPT; ++k) {
    const long long i = min(base + k * stride, p.n - 1);
    v[k] = __ldg(p.A + i);
    a[k] = __ldg(p.a + i);
  }
  if (p.B) {
    double bv[CL_EPT];
#pragma unroll
    for (int k = 0; k < CL_EPT; ++k) bv[k] = __ldg(p.B + min(base + k * stride, p.n - 1));
#pragma unroll
    for (int k = 0; k < CL_EPT; ++k) v[k] = __dsub_rn(v[k], __dmul_rn(p.coef[t], bv[k]));
  }
#pragma unroll
  for (int k = 0; k < CL_EPT; ++k) {
    const long long i = base + k * stride;
    if (i >= p.n) { v[k] = 0.0; a[k] = 0.0; }
    double ta = 0.0, tb = 0.0;
    if (a[k] != 0.0) {
      const double l = p.l ? p.l[i] : p.lc, u = p.u ? p.u[i] : p.uc;
      const double t1 = bp_div(__dsub_rn(v[k], u), a[k]);
      const double t2 = bp_div(__dsub_rn(v[k], l), a[k]);
      ta = fmin(t1, t2);
      tb = fmax(t1, t2);
    }
    bpa[k][tid] = ta;
    bpb[k][tid] = tb;
  }
  double c = hint, lo = -INFINITY, hi = INFINITY, lam = 0.0, tmin = INFINITY, tmax = -INFINITY;
  if (p.slope_num && p.slope_den && *p.slope_den != 0.0)  // first-order start along the ray
    c = hint - p.coef[t] * (*p.slope_num / *p.slope_den);
  int status = PROJ_NEWTON, passes = 0;
  const int ops[8] = {0, 0, 0, 1, 2, 1, 2, 0};
  bool empty = false;
  for (int pass = 0; status == PROJ_NEWTON && pass < CL_MAX_PASSES; ++pass) {
    // slots 5-7 (breakpoint range, active-slot count) do not depend on c: reduced and
    // exchanged on pass 0 only; later passes carry the five Newton quantities
    const int nv = pass == 0 ? 8 : 5;
    double vals[8] = {0.0, 0.0, 0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0};
#pragma unroll
    for (int k = 0; k < CL_EPT; ++k) {
      const long long i = base + k * stride;
      if (i >= p.n || a[k] == 0.0) continue;
      const double l = p.l ? p.l[i] : p.lc, u = p.u ? p.u[i] : p.uc;
      const double ta = bpa[k][tid], tb = bpb[k][tid];
      vals[0] += contrib(v[k], a[k], l, u, c);
      const double a2 = a[k] * a[k];
      if (ta <= c && c < tb) vals[1] += a2;
      if (ta < c && c <= tb) vals[2] += a2;
      if (ta > c) vals[3] = fmin(vals[3], ta); else if (ta < c) vals[4] = fmax(vals[4], ta);
      if (tb > c) vals[3] = fmin(vals[3], tb); else if (tb < c) vals[4] = fmax(vals[4], tb);
      if (pass == 0) {
        vals[5] = fmin(vals[5], ta);
        vals[6] = fmax(vals[6], tb);
        vals[7] += 1.0;
      }
    }
    // warp trees, then slot k folded across warps by thread k (block_reduce's order) and
    // pushed straight into slot [rank] of every CTA of the cluster; after the cluster
    // barrier EVERY thread folds the 16 rank partials and runs the (deterministic) Newton
    // update itself: two barriers per pass instead of six
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= nv) break;
      const double w = ops[k] == 0 ? warp_sum(vals[k]) : (ops[k] == 1 ? warp_min(vals[k]) : warp_max(vals[k]));
      if (lane == 0) red[k * 32 + warp] = w;
    }
    __syncthreads();
    const int buf = pass & 1;
    if (tid < nv) {
      const int op = (tid == 3 || tid == 5) ? 1 : ((tid == 4 || tid == 6) ? 2 : 0);  // = ops[tid]
      double r = red[tid * 32];
      for (int w = 1; w < CL_NT / 32; ++w) {
        const double x = red[tid * 32 + w];
        r = op == 0 ? r + x : (op == 1 ? fmin(r, x) : fmax(r, x));
      }
#pragma unroll 4
      for (int q = 0; q < CL_CTAS; ++q) *cluster.map_shared_rank(&gath[buf][rank][tid], q) = r;
    }
    cluster.sync();  // arrive.release / wait.acquire: every push of this pass is visible
    if (warp == 0) {
      // lane k < 8 folds slot k over the ranks (fixed order), lane 0 runs the update
      double r = 0.0;
      if (lane < nv) {
        const int op = (lane == 3 || lane == 5) ? 1 : ((lane == 4 || lane == 6) ? 2 : 0);
        r = gath[buf][0][lane];
        for (int q = 1; q < CL_CTAS; ++q) {
          const double x = gath[buf][q][lane];
          r = op == 0 ? r + x : (op == 1 ? fmin(r, x) : fmax(r, x));
        }
      }
      double res_[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) res_[k] = __shfl_sync(0xffffffffu, r, k);
      if (lane == 0) {
        if (pass == 0) { tmin = res_[5]; tmax = res_[6]; empty = res_[7] == 0.0; }
        if (empty) {
          lam = 0.0;
          status = PROJ_DONE;
        } else {
          newton_update(p.d - res_[0], res_[1], res_[2], res_[3], res_[4], tmin, p.d, c, lo, hi,
                        lam, status);
        }
        sh[0] = c; sh[1] = lo; sh[2] = hi; sh[3] = lam; sh[4] = tmin; sh[5] = tmax;
        sh_status = status;
      }
    }
    __syncthreads();
    c = sh[0]; lo = sh[1]; hi = sh[2]; lam = sh[3]; tmin = sh[4]; tmax = sh[5];
    status = sh_status;
    passes = pass + 1;
  }
  // apply at lambda: x, free mask, the six fused sums
  double s6[6] = {0, 0, 0, 0, 0, 0};
  if (status == PROJ_DONE) {
    double* xo = p.x_out ? p.x_out + (long long)t * p.n : nullptr;
    unsigned char* fo = p.free_out ? p.free_out + (long long)t * p.n : nullptr;
#pragma unroll
    for (int k = 0; k < CL_EPT; ++k) {
      const long long i = base + k * stride;
      if (i >= p.n) continue;
      const double l = p.l ? p.l[i] : p.lc, u = p.u ? p.u[i] : p.uc;
      const double y = __dsub_rn(v[k], __dmul_rn(lam, a[k]));
      const double x = fmin(fmax(y, l), u);
      const bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
      const bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
      const bool fr = !(lower || upper);
      if (xo) xo[i] = x;
      if (fo) fo[i] = fr ? 1 : 0;
      const double r = v[k] - x;
      s6[0] += p.base ? bregman_term(x, p.base[i], v[k], a[k], 0.5 * (lam + p.base_lam))
                      : v[k] * v[k];
      s6[1] += r * r;
      if (p.ref) { const double dd = x - p.ref[i]; s6[2] += dd * dd; }
      if (fr) { s6[3] += a[k] * a[k]; s6[4] += 1.0; }
      s6[5] += x * (2.0 * v[k] - x);
    }
  }
  const int ops6[6] = {0, 0, 0, 0, 0, 0};
  block_reduce<6>(s6, ops6, red);
  const int buf = passes & 1;  // the buffer no CTA can still be reading
  if (tid == 0)
    for (int k = 0; k < 6; ++k) red[k] = s6[k];
  __syncthreads();
  if (tid < 6) {
    double* dst = cluster.map_shared_rank(&gath[buf][rank][0], 0);
    dst[tid] = red[tid];
  }
  // every CTA arrives (release); only rank 0 waits and folds, the others may exit:
  // after the last pass barrier nothing else is written into their shared memory
  cluster.barrier_arrive();
  if (rank != 0) return;
  cluster.barrier_wait();
  if (tid == 0) {
    ProjState* st = p.st + t;
    if (status == PROJ_DONE) {
      double r[6];
      for (int k = 0; k < 6; ++k) {
        r[k] = gath[buf][0][k];
        for (int q = 1; q < CL_CTAS; ++q) r[k] += gath[buf][q][k];
      }
      st->sum_v2 = p.base ? 0.0 : r[0];
      st->sum_bh = p.base ? r[0] : 0.0;
      st->sum_r2 = r[1];
      st->sum_dref2 = r[2];
      st->sum_a2_free = r[3];
      st->nfree = (long long)r[4];
      st->sum_xv = r[5];
      st->lam = lam;
      st->status = PROJ_APPLIED;
    } else {
      st->lam = c;
      st->lo = lo;
      st->hi = hi;
      st->status = status;
    }
    st->tmin = tmin;
    st->tmax = tmax;
    st->passes = passes;
    st->in_count = -1;
  }
}


// ------------------------------------------------------------------ multi-trial
// Large-n projection (n above the cluster path's register capacity, e.g. the
// 2,000,000-slot config-4 dual): ALL T line-search trials of a batch in ONE
// cooperative launch that reads each slot's (u, Qd, a) ONCE per pass.  The 8 warps of
// a block are split into T trial groups of 8/T warps; the groups walk the same slots
// (the repeats hit L1), so a pass costs one read of the inputs whatever T is, where
// the trial-per-blockIdx.y kernels read them T times.  Per pass: per-warp Newton sums
// -> per-trial block partial -> grid barrier -> every block folds the partials of every
// trial in block order (identical state everywhere, uniform branching) and takes the
// safeguarded Newton step (newton_update).  Up to PM_MAX_PASSES passes (cheap once
// the inputs sit in L2), then the apply pass: the six fused sums per trial, and x /
// the free mask written only when asked (a batch defers them: the driver materialises
// the ONE accepted trial, proj_materialize_kernel).
static constexpr int PM_NT = 256;
static constexpr int PM_WARPS = PM_NT / 32;
static constexpr int PM_MAX_PASSES = 16;
static constexpr int PM_UNROLL = 4;
static constexpr int PM_INACTIVE = 99;

// scripts/proj_probe.cu: per-phase globaltimer stamps of block 0 thread 0
#ifdef SSNAL_PROJ_TIMING
__device__ unsigned long long g_proj_marks[64];
__device__ int g_proj_nmarks;
#define PROJ_MARK()                                                      \
  do {                                                                   \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                           \
      unsigned long long t_;                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      const int k_ = g_proj_nmarks;                                      \
      if (k_ < 64) g_proj_marks[k_] = t_;                                \
      g_proj_nmarks = k_ + 1;                                            \
    }                                                                    \
  } while (0)
#else
#define PROJ_MARK() \
  do {              \
  } while (0)
#endif

// one slot's Newton-pass terms at c (contrib, one-sided slopes, nearest breakpoints,
// and on pass 0 the breakpoint range and count)
__device__ __forceinline__ void pm_slot(double uu, double bb, double a, double l, double u,
                                        double coef, bool hasB, double c, bool first,
                                        double (&vals)[8]) {
  if (a == 0.0) return;
  const double v = hasB ? __dsub_rn(uu, __dmul_rn(coef, bb)) : uu;
  const double t1 = bp_div(__dsub_rn(v, u), a), t2 = bp_div(__dsub_rn(v, l), a);
  const double ta = fmin(t1, t2), tb = fmax(t1, t2);
  vals[0] += contrib(v, a, l, u, c);
  const double a2 = a * a;
  if (ta <= c && c < tb) vals[1] += a2;
  if (ta < c && c <= tb) vals[2] += a2;
  if (ta > c) vals[3] = fmin(vals[3], ta); else if (ta < c) vals[4] = fmax(vals[4], ta);
  if (tb > c) vals[3] = fmin(vals[3], tb); else if (tb < c) vals[4] = fmax(vals[4], tb);
  if (first) {
    vals[5] = fmin(vals[5], ta);
    vals[6] = fmax(vals[6], tb);
    vals[7] += 1.0;
  }
}

// The Newton pass over this warp's slots: 32-bit indices, the argument pointers hoisted
// into registers, constant bounds specialised (CB), full chunks of PM_UNROLL slots loaded
// together without per-slot guards, a guarded tail.  (The generic loop spent most of
// its issue slots on 64-bit index arithmetic, bounds predicates and reloads of kernel
// parameters.)
template <bool CB>
__device__ __forceinline__ void pm_pass(const ProjArgs& p, double coef, double c, bool first,
                                        int start, int stride, double (&vals)[8]) {
  const double* __restrict__ A = p.A;
  const double* __restrict__ B = p.B;
  const double* __restrict__ av = p.a;
  const double* __restrict__ lv = p.l;
  const double* __restrict__ uv = p.u;
  const double lc = p.lc, uc = p.uc;
  const bool hasB = B != nullptr;
  const int n = (int)p.n;
  int i = start;
  const int full_end = n - (PM_UNROLL - 1) * stride;
  for (; i < full_end; i += PM_UNROLL * stride) {
    double uu[PM_UNROLL], bb[PM_UNROLL], aa[PM_UNROLL], ll[PM_UNROLL], ul[PM_UNROLL];
#pragma unroll
    for (int k = 0; k < PM_UNROLL; ++k) {
      const int ik = i + k * stride;
      uu[k] = __ldg(A + ik);
      bb[k] = hasB ? __ldg(B + ik) : 0.0;
      aa[k] = __ldg(av + ik);
      ll[k] = CB ? lc : (lv ? __ldg(lv + ik) : lc);
      ul[k] = CB ? uc : (uv ? __ldg(uv + ik) : uc);
    }
#pragma unroll
    for (int k = 0; k < PM_UNROLL; ++k) pm_slot(uu[k], bb[k], aa[k], ll[k], ul[k], coef, hasB, c, first, vals);
  }
  for (; i < n; i += stride) {
    const double uu = __ldg(A + i), bb = hasB ? __ldg(B + i) : 0.0, a = __ldg(av + i);
    const double l = CB ? lc : (lv ? __ldg(lv + i) : lc), u = CB ? uc : (uv ? __ldg(uv + i) : uc);
    pm_slot(uu, bb, a, l, u, coef, hasB, c, first, vals);
  }
}

template <int T>
__global__ void __launch_bounds__(PM_NT, 2) proj_multi_kernel(ProjArgs p, double hint,
                                                           int max_newton, int nt, int write_x) {
  cg::grid_group grid = cg::this_grid();
  constexpr int G = PM_WARPS / T;  // warps per trial group
  __shared__ double wred[PM_WARPS][8];
  __shared__ double wfold[PM_WARPS][8];
  __shared__ double s_c[T], s_lo[T], s_hi[T], s_lam[T], s_tmin[T], s_tmax[T], s_coef[T];
  __shared__ int s_status[T], s_passes[T];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = warp % T, g = warp / T;
  const unsigned nb = gridDim.x;
  const long long region = (long long)T * nb * PSTRIDE;
  if (threadIdx.x < T) {
    s_c[threadIdx.x] = hint;
#pragma unroll
    for (int k = 0; k < T; ++k) {  // static indices (see s_coef)
      if ((int)threadIdx.x != k) continue;
      if (p.has_hints) {
        s_c[k] = p.hints[k];
      } else if (p.slope_num && p.slope_den && *p.slope_den != 0.0) {
        s_c[k] = hint - p.coef[k] * (*p.slope_num / *p.slope_den);
      }
    }
    s_lo[threadIdx.x] = -INFINITY;
    s_hi[threadIdx.x] = INFINITY;
    s_lam[threadIdx.x] = 0.0;
    s_tmin[threadIdx.x] = INFINITY;
    s_tmax[threadIdx.x] = -INFINITY;
    s_status[threadIdx.x] = (int)threadIdx.x < nt ? PROJ_NEWTON : PM_INACTIVE;
    s_passes[threadIdx.x] = 0;
#pragma unroll
    for (int k = 0; k < T; ++k)  // static indices: no local copy of the param array
      if ((int)threadIdx.x == k) s_coef[k] = p.coef[k];
  }
  __syncthreads();
  PROJ_MARK();
  const double coef = s_coef[t];
  const long long stride = (long long)nb * G * 32;
  const long long start = ((long long)blockIdx.x * G + g) * 32 + lane;
  const int ops[8] = {0, 0, 0, 1, 2, 1, 2, 0};
  for (int pass = 0;; ++pass) {
    const int status = s_status[t];
    const double c = s_c[t];
    double vals[8] = {0.0, 0.0, 0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0};
    if (status == PROJ_NEWTON) {
      if (p.l || p.u) pm_pass<false>(p, coef, c, pass == 0, (int)start, (int)stride, vals);
      else pm_pass<true>(p, coef, c, pass == 0, (int)start, (int)stride, vals);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double w = ops[k] == 0 ? warp_sum(vals[k]) : (ops[k] == 1 ? warp_min(vals[k]) : warp_max(vals[k]));
        if (lane == 0) wred[warp][k] = w;
      }
    }
    __syncthreads();
    PROJ_MARK();
    double* part = p.part + (pass & 1) * region;
    if (status == PROJ_NEWTON && g == 0 && lane < 8) {  // the trial's G warps, in order
      const int op = (lane == 3 || lane == 5) ? 1 : ((lane == 4 || lane == 6) ? 2 : 0);  // ops[lane]
      double r = wred[t][lane];
      for (int gg = 1; gg < G; ++gg) {
        const double x = wred[gg * T + t][lane];
        r = op == 0 ? r + x : (op == 1 ? fmin(r, x) : fmax(r, x));
      }
      part[((long long)t * nb + blockIdx.x) * PSTRIDE + lane] = r;
    }
    grid.sync();
    PROJ_MARK();
    double r[8] = {0.0, 0.0, 0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0};
    if (status == PROJ_NEWTON) {
      // the trial's G warps fold the block partials (warp g: blocks g*32 + lane +
      // k*32G, two at a time with their loads in flight), fixed warp trees, then warp 0
      // combines the G results in g order: every block gets bit-identical totals
      const double* base = part + (long long)t * nb * PSTRIDE;
      for (unsigned b = g * 32 + lane; b < nb; b += 64 * G) {
        const unsigned b2 = b + 32 * G;
        double x1[8], x2[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          x1[k] = __ldcg(base + (long long)b * PSTRIDE + k);
          x2[k] = b2 < nb ? __ldcg(base + (long long)b2 * PSTRIDE + k)
                          : (ops[k] == 0 ? 0.0 : (ops[k] == 1 ? INFINITY : -INFINITY));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          r[k] = ops[k] == 0 ? r[k] + x1[k] : (ops[k] == 1 ? fmin(r[k], x1[k]) : fmax(r[k], x1[k]));
          r[k] = ops[k] == 0 ? r[k] + x2[k] : (ops[k] == 1 ? fmin(r[k], x2[k]) : fmax(r[k], x2[k]));
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        r[k] = ops[k] == 0 ? warp_sum(r[k]) : (ops[k] == 1 ? warp_min(r[k]) : warp_max(r[k]));
      if (G > 1) {
        __syncwarp();
        if (lane == 0)
#pragma unroll
          for (int k = 0; k < 8; ++k) wfold[warp][k] = r[k];
      }
    }
    if (G > 1) __syncthreads();
    if (status == PROJ_NEWTON && g == 0) {
      if (G > 1 && lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double v = wfold[t][k];
          for (int gg = 1; gg < G; ++gg) {
            const double x = wfold[gg * T + t][k];
            v = ops[k] == 0 ? v + x : (ops[k] == 1 ? fmin(v, x) : fmax(v, x));
          }
          r[k] = v;
        }
      }
      if (lane == 0) {
        double cc = s_c[t], lo = s_lo[t], hi = s_hi[t], lam = s_lam[t], tmin = s_tmin[t];
        int stt = status;
        if (pass == 0) {
          tmin = r[5];
          s_tmin[t] = r[5];
          s_tmax[t] = r[6];
        }
        if (pass == 0 && r[7] == 0.0) {  // a == 0: the constraint is 0 = d, clip only
          lam = 0.0;
          stt = PROJ_DONE;
        } else {
          newton_update(p.d - r[0], r[1], r[2], r[3], r[4], tmin, p.d, cc, lo, hi, lam, stt);
        }
        s_c[t] = cc; s_lo[t] = lo; s_hi[t] = hi; s_lam[t] = lam; s_status[t] = stt;
        s_passes[t] = pass + 1;
      }
    }
    __syncthreads();
    PROJ_MARK();
    bool any = false;
#pragma unroll
    for (int k = 0; k < T; ++k) any |= s_status[k] == PROJ_NEWTON;
    if (!any || pass + 1 >= max_newton) break;
  }
  // apply: the six fused sums per trial (+ x and the mask when written)
  const int status = s_status[t];
  const double lam = s_lam[t];
  double s6[6] = {0, 0, 0, 0, 0, 0};
  if (status == PROJ_DONE) {
    double* xo = (write_x && p.x_out) ? p.x_out + (long long)t * p.n : nullptr;
    unsigned char* fo = (write_x && p.free_out) ? p.free_out + (long long)t * p.n : nullptr;
    const double lam_bar = 0.5 * (lam + p.base_lam);
    const double* __restrict__ A = p.A;
    const double* __restrict__ B = p.B;
    const double* __restrict__ av = p.a;
    const double* __restrict__ base = p.base;
    const double* __restrict__ ref = p.ref;
    const int n = (int)p.n, istride = (int)stride;
#pragma unroll 4
    for (int i = (int)start; i < n; i += istride) {
      double v = __ldg(A + i);
      if (B) v = __dsub_rn(v, __dmul_rn(coef, __ldg(B + i)));
      const double a = __ldg(av + i);
      const double l = p.l ? p.l[i] : p.lc, u = p.u ? p.u[i] : p.uc;
      const double y = __dsub_rn(v, __dmul_rn(lam, a));
      const double x = fmin(fmax(y, l), u);
      const bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
      const bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
      const bool fr = !(lower || upper);
      if (xo) xo[i] = x;
      if (fo) fo[i] = fr ? 1 : 0;
      const double r = v - x;
      s6[0] += base ? bregman_term(x, __ldg(base + i), v, a, lam_bar) : v * v;
      s6[1] += r * r;
      if (ref) { const double dd = x - __ldg(ref + i); s6[2] += dd * dd; }
      if (fr) { s6[3] += a * a; s6[4] += 1.0; }
      s6[5] += x * (2.0 * v - x);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double w = warp_sum(s6[k]);
      if (lane == 0) wred[warp][k] = w;
    }
  }
  __syncthreads();
  PROJ_MARK();
  double* part = p.part + 2 * region;
  if (status == PROJ_DONE && g == 0 && lane < 6) {
    double r = wred[t][lane];
    for (int gg = 1; gg < G; ++gg) r += wred[gg * T + t][lane];
    part[((long long)t * nb + blockIdx.x) * PSTRIDE + lane] = r;
  }
  grid.sync();
  PROJ_MARK();
  if (blockIdx.x != 0 || g != 0 || status == PM_INACTIVE) return;
  ProjState* st = p.st + t;
  if (status == PROJ_DONE) {
    double r[6] = {0, 0, 0, 0, 0, 0};
    const double* base = part + (long long)t * nb * PSTRIDE;
    for (unsigned b = lane; b < nb; b += 32) {
#pragma unroll
      for (int k = 0; k < 6; ++k) r[k] += __ldcg(base + (long long)b * PSTRIDE + k);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) r[k] = warp_sum(r[k]);
    if (lane != 0) return;
    st->sum_v2 = p.base ? 0.0 : r[0];
    st->sum_bh = p.base ? r[0] : 0.0;
    st->sum_r2 = r[1];
    st->sum_dref2 = r[2];
    st->sum_a2_free = r[3];
    st->nfree = (long long)r[4];
    st->sum_xv = r[5];
    st->lam = lam;
    st->status = PROJ_APPLIED;
  } else {
    if (lane != 0) return;
    st->lam = s_c[t];  // Newton iterate for the K-ary fallback (tmin for infeasible-low)
    st->lo = s_lo[t];
    st->hi = s_hi[t];
    st->status = status;
  }
  st->tmin = s_tmin[t];
  st->tmax = s_tmax[t];
  st->passes = s_passes[t];
  st->in_count = -1;
}

// x and the free mask of ONE trial of a deferred batch: v = A - coef B at the trial's
// multiplier (read from its device state), the apply pass's arithmetic bit for bit
__global__ void __launch_bounds__(SSNAL_NT) proj_materialize_kernel(ProjArgs p, double coef,
                                                                    const ProjState* st,
                                                                    double* __restrict__ x_out,
                                                                    unsigned char* __restrict__ f_out) {
  const double lam = st->lam;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = __ldg(p.A + i);
    if (p.B) v = __dsub_rn(v, __dmul_rn(coef, __ldg(p.B + i)));
    const double a = __ldg(p.a + i);
    const double l = p.l ? p.l[i] : p.lc, u = p.u ? p.u[i] : p.uc;
    const double y = __dsub_rn(v, __dmul_rn(lam, a));
    const bool lower = y <= __dadd_rn(l, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(l))));
    const bool upper = !lower && (y >= __dsub_rn(u, __dmul_rn(1e-12, __dadd_rn(1.0, fabs(u)))));
    x_out[i] = fmin(fmax(y, l), u);
    f_out[i] = (lower || upper) ? 0 : 1;
  }
}

static bool cluster_ok(long long n, int T) {
  static DeviceCache cache;
  const int ok = per_device(cache, [](int dev) {
    int sup = 0;
    cudaDeviceGetAttribute(&sup, cudaDevAttrClusterLaunch, dev);
    if (!sup) return 0;
    if (cudaFuncSetAttribute(proj_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess)
      return 0;
    if (cudaFuncSetAttribute(proj_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             CL_SMEM) != cudaSuccess)
      return 0;
    return 1;
  });
  // in the solve (L2 cold after every sweep of A) the register-resident cluster
  // kernel wins for single trials too (bench op profile: -9 % projection time)
  return ok == 1 && n <= (long long)CL_CTAS * CL_NT * CL_EPT && T >= 1;
}

static bool multi_ok(long long n, int T) {
  return T >= 1 && T <= PM_WARPS && n < (1LL << 31) - (1LL << 24) && !cluster_ok(n, T);
}

// Line-search trials one cluster-projection launch runs in a single wave: a 16-CTA
// cluster needs 16 SMs of one GPC, so only ~7 fit on a B200 at once -- an 8-trial
// batch ran as two waves (2x the latency of 7).  Not limited without the cluster path.
int proj_wave_trials(long long n, bool first) {
  // multi-trial kernel: every trial costs a full set of per-slot FP64 work per pass (the
  // inputs are read once): the speculative batch is the unit step alone (config 4: batch
  // sizes 1 / 2 / 3 / 4 -> 183 / 184 / 191 / 190 ms per solve), a backtracking batch, 4
  // step lengths (SSNAL_FIRST_BATCH overrides the first)
  if (multi_ok(n, 1)) {
    static const int fb = std::getenv("SSNAL_FIRST_BATCH") ? std::atoi(std::getenv("SSNAL_FIRST_BATCH")) : 1;
    return first ? std::max(1, std::min(fb, PM_WARPS)) : 4;
  }
  if (!cluster_ok(n, 1)) return SSNAL_MAX_TRIALS;
  static DeviceCache cache;
  return per_device(cache, [](int) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL_CTAS, 1, 1);
    cfg.blockDim = dim3(CL_NT, 1, 1);
    cfg.dynamicSmemBytes = CL_SMEM;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, (void*)proj_cluster_kernel, &cfg) != cudaSuccess || c < 1)
      c = SSNAL_MAX_TRIALS;
    return c;
  });
}

int proj_blocks(long long n) {
  long long b = ceil_div(n, (long long)SSNAL_NT * 4);
  if (b < 1) b = 1;
  if (b > SSNAL_MAX_BLOCKS / 2) b = SSNAL_MAX_BLOCKS / 2;
  return (int)b;
}

size_t proj_ws_bytes(long long n, int T) {
  // 3 partial regions (two ping-pong search regions + apply) + the active-trial counter
  return (size_t)3 * T * proj_blocks(n) * PSTRIDE * sizeof(double) + 64;
}

static int fused_capacity() {
  static DeviceCache cache;
  return per_device(cache, [](int dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, proj_fused_kernel, SSNAL_NT, 0);
    return sms * per;
  });
}

template <int T>
static int multi_capacity() {
  static DeviceCache cache;
  return per_device(cache, [](int dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, proj_multi_kernel<T>, PM_NT, 0);
    return sms * std::min(per, 2);
  });
}


// whether a batched projection of T trials leaves x / the mask unwritten (the driver
// then materialises the accepted trial with launch_proj_materialize)
bool proj_defers(long long n, int T) { return T > 1 && multi_ok(n, T); }

template <int T>
static cudaError_t launch_multi(ProjArgs& p, const ProjLaunch& L, cudaStream_t stream) {
  if (L.n >= (1LL << 31) - (1LL << 24)) return cudaErrorInvalidValue;  // 32-bit slot indices
  constexpr int G = PM_WARPS / T;
  long long nb = ceil_div(L.n, (long long)G * 32 * PM_UNROLL);
  nb = std::min<long long>(nb, std::min(multi_capacity<T>(), proj_blocks(L.n)));
  if (nb < 1) nb = 1;
  double hint = L.hint;
  int maxn = std::max(L.newton, PM_MAX_PASSES);
  int nt = L.T;
  int write_x = (L.T == 1 || !L.defer) ? 1 : 0;
  void* args[] = {&p, &hint, &maxn, &nt, &write_x};
  note_launch();
  return cudaLaunchCooperativeKernel((void*)proj_multi_kernel<T>, dim3((unsigned)nb), dim3(PM_NT),
                                     args, 0, stream);
}

cudaError_t launch_proj_materialize(const ProjLaunch& L, double coef, const ProjState* st,
                                    double* x_out, unsigned char* f_out, cudaStream_t stream) {
  ProjArgs p{};
  p.A = L.A; p.B = L.B; p.a = L.a; p.l = L.l; p.u = L.u; p.lc = L.lc; p.uc = L.uc; p.n = L.n;
  const int nblk = (int)std::min<long long>(ceil_div(L.n, (long long)SSNAL_NT * 4), SSNAL_MAX_BLOCKS);
  note_launch();
  proj_materialize_kernel<<<nblk, SSNAL_NT, 0, stream>>>(p, coef, st, x_out, f_out);
  return cudaGetLastError();
}

cudaError_t launch_project(const ProjLaunch& L, cudaStream_t stream) {
  ProjArgs p;
  p.A = L.A; p.B = L.B;
  for (int t = 0; t < SSNAL_MAX_TRIALS; ++t) p.coef[t] = (L.coef && t < L.T) ? L.coef[t] : 0.0; p.a = L.a; p.l = L.l; p.u = L.u;
  p.has_hints = L.hints != nullptr;
  p.slope_num = L.B ? L.slope_num : nullptr;
  p.slope_den = L.B ? L.slope_den : nullptr;
  for (int t = 0; t < SSNAL_MAX_TRIALS; ++t) p.hints[t] = (L.hints && t < L.T) ? L.hints[t] : L.hint;
  p.lc = L.lc; p.uc = L.uc; p.d = L.d; p.n = L.n; p.st = L.st; p.part = L.part;
  p.x_out = L.x_out; p.free_out = L.free_out; p.ref = L.ref;
  p.base = L.base; p.base_lam = L.base_lam;
  const int nblk = proj_blocks(L.n);
  if (L.newton > 0 && L.passes == 0 && L.phases == PHASE_APPLY && cluster_ok(L.n, L.T)) {
    note_launch();
    proj_cluster_kernel<<<dim3(CL_CTAS, L.T), CL_NT, CL_SMEM, stream>>>(p, L.hint);
    return cudaGetLastError();
  }
  if (L.newton > 0 && L.passes == 0 && L.phases == PHASE_APPLY && multi_ok(L.n, L.T)) {
    if (L.T == 1) return launch_multi<1>(p, L, stream);
    if (L.T == 2) return launch_multi<2>(p, L, stream);
    if (L.T <= 4) return launch_multi<4>(p, L, stream);
    return launch_multi<8>(p, L, stream);
  }
  const int nbf = std::min(nblk, fused_capacity() / L.T);  // co-resident grid for grid.sync
  if (L.newton > 0 && L.passes == 0 && L.phases == PHASE_APPLY && nbf >= 1) {
    int* active = (int*)((char*)L.part + (size_t)3 * L.T * nblk * PSTRIDE * sizeof(double));
    double hint = L.hint;
    int maxn = L.newton;
    void* args[] = {&p, &hint, &maxn, &active};
    note_launch();
    return cudaLaunchCooperativeKernel((void*)proj_fused_kernel, dim3(nbf, L.T), dim3(SSNAL_NT),
                                       args, 0, stream);
  }
  dim3 grid(nblk, L.T);
  if (L.newton > 0) {
    for (int k = 0; k < L.newton; ++k) {
      note_launch();
      proj_newton_kernel<<<grid, SSNAL_NT, 0, stream>>>(p, k == 0 ? 1 : 0, L.hint);
    }
  } else if (L.phases & PHASE_RANGE) {
    note_launch();
    proj_range_kernel<<<grid, SSNAL_NT, 0, stream>>>(p);
  }
  for (int k = 0; k < L.passes; ++k) { note_launch(); proj_pass_kernel<<<grid, SSNAL_NT, 0, stream>>>(p); }
  if (L.phases & PHASE_EXACT) { note_launch(); proj_exact_kernel<<<grid, SSNAL_NT, 0, stream>>>(p); }
  if (L.phases & PHASE_APPLY) { note_launch(); proj_apply_kernel<<<grid, SSNAL_NT, 0, stream>>>(p); }
  return cudaGetLastError();
}

}  // namespace ssnal

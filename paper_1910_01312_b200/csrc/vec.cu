// Vector kernels: fused dot products, numpy-ordered elementwise ops, the
// HS-Jacobian product and free-set compaction (ballot/prefix-sum).
#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

static constexpr int MAXDOT = 8;
static constexpr int TICKET_BYTES = 256;

struct DotArgs {
  const double* x[MAXDOT];
  const double* y[MAXDOT];
  const uint8_t* mask;
  long long n;
  int k;
  double* out;
  unsigned int* ticket;
  double* part;  // [nblk][MAXDOT]
};

int stream_blocks(long long n, int per_thread) {
  long long b = ceil_div(n, (long long)SSNAL_NT * per_thread);
  if (b < 1) b = 1;
  if (b > SSNAL_MAX_BLOCKS) b = SSNAL_MAX_BLOCKS;
  return (int)b;
}

__global__ void __launch_bounds__(SSNAL_NT) dots_kernel(DotArgs p) {
  __shared__ double red[MAXDOT * 32];
  double acc[MAXDOT];
#pragma unroll
  for (int j = 0; j < MAXDOT; ++j) acc[j] = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    if (p.mask && !p.mask[i]) continue;
#pragma unroll
    for (int j = 0; j < MAXDOT; ++j) {
      if (j < p.k) {
        double xv = p.x[j][i];
        acc[j] += xv * (p.y[j] ? p.y[j][i] : xv);
      }
    }
  }
  const int ops[MAXDOT] = {0, 0, 0, 0, 0, 0, 0, 0};
  block_reduce<MAXDOT>(acc, ops, red);
  if (threadIdx.x == 0)
    for (int j = 0; j < MAXDOT; ++j) p.part[blockIdx.x * MAXDOT + j] = acc[j];
  if (!last_block_arrive(p.ticket, gridDim.x)) return;
  block_fold_partials<MAXDOT>(p.part, gridDim.x, MAXDOT, ops, acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < MAXDOT; ++j)
      if (j < p.k) p.out[j] = acc[j];
  }
}

size_t reduce_ws_bytes(long long n) {
  // capacity for the one-element-per-thread grids of the latency-bound passes
  return TICKET_BYTES + (size_t)stream_blocks(n, 1) * MAXDOT * sizeof(double);
}

cudaError_t launch_dots(int k, const double* const* xs, const double* const* ys,
                        const uint8_t* mask, long long n, double* out, void* ws,
                        cudaStream_t stream) {
  DotArgs p;
  for (int j = 0; j < MAXDOT; ++j) {
    p.x[j] = j < k ? xs[j] : nullptr;
    p.y[j] = (j < k && ys) ? ys[j] : nullptr;
  }
  p.mask = mask;
  p.n = n;
  p.k = k;
  p.out = out;
  p.ticket = (unsigned int*)ws;
  p.part = (double*)((char*)ws + TICKET_BYTES);
  { note_launch(); dots_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(p); }
  return cudaGetLastError();
}

__global__ void vec_kernel(int op, long long n, double alpha, const double* __restrict__ x,
                           const double* __restrict__ y, const double* __restrict__ z,
                           double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double r;
    switch (op) {
      case 0: {
        double yz = z ? __dadd_rn(y[i], z[i]) : y[i];
        r = __dadd_rn(x[i], __dmul_rn(alpha, yz));
        break;
      }
      case 1: r = __dsub_rn(__dsub_rn(x[i], y[i]), z[i]); break;
      case 2: r = __dadd_rn(x[i], __dmul_rn(alpha, y[i])); break;
      case 3: r = __dsub_rn(x[i], y[i]); break;
      case 5: r = __dmul_rn(x[i], y[i]); break;
      case 6: r = 1.0 / (1.0 + alpha * fmax(x[i] - y[i], 0.0)); break;
      default: r = __dmul_rn(alpha, x[i]); break;
    }
    out[i] = r;
  }
}

cudaError_t launch_vec(int op, long long n, double alpha, const double* x, const double* y,
                       const double* z, double* out, cudaStream_t stream) {
  { note_launch(); vec_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(op, n, alpha, x, y, z, out); }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- HS-Jacobian
// out = alpha*add + beta * P y with P = S(I - aa'/(a'Sa))S; ref projection.py:214-225.
__global__ void hs_finish_kernel(const uint8_t* __restrict__ fm, const double* __restrict__ a,
                                 const double* __restrict__ y, long long n, double beta,
                                 const double* __restrict__ add, double alpha,
                                 double* __restrict__ out, const double* sums) {
  const double ay = sums[0], aa = sums[1];
  const double coef = aa != 0.0 ? ay / aa : 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double py = fm[i] ? __dsub_rn(y[i], __dmul_rn(coef, a[i])) : 0.0;
    double r = beta * py;
    if (add) r = alpha * add[i] + r;
    out[i] = r;
  }
}

// out = alpha*add + beta*P y with the sums {a_J'y_J, a_J'a_J} supplied (DEVICE): the
// sharded driver all-reduces them between the dots and this pass
cudaError_t launch_hs_finish(const uint8_t* fm, const double* a, const double* y, long long n,
                             double beta, const double* add, double alpha, double* out,
                             const double* sums, cudaStream_t stream) {
  note_launch();
  hs_finish_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(fm, a, y, n, beta, add, alpha,
                                                                  out, sums);
  return cudaGetLastError();
}

cudaError_t launch_hs_apply(const uint8_t* fm, const double* a, const double* y, long long n,
                            double beta, const double* add, double alpha, double* out,
                            void* ws, cudaStream_t stream) {
  // sums[0] = a_J'y_J, sums[1] = a_J'a_J, computed into the tail of ws
  double* sums = (double*)((char*)ws + reduce_ws_bytes(n));
  const double* xs[2] = {a, a};
  const double* ys[2] = {y, nullptr};
  cudaError_t e = launch_dots(2, xs, ys, fm, n, sums, ws, stream);
  if (e != cudaSuccess) return e;
  { note_launch(); hs_finish_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(fm, a, y, n, beta, add, alpha,
                                                                  out, sums); }
  return cudaGetLastError();
}

// Newton direction epilogue, one pass: out = alpha*add + beta*P y (as hs_finish) and
// the three line-search inner products {g'out, w'qw, w'y} of the new direction,
// folded in fixed order into dots_out[0..2] (replaces hs_finish + a dots launch).
struct HsDotArgs {
  const uint8_t* fm;
  const double* a;
  const double* y;
  long long n;
  double beta, alpha;
  const double* add;
  double* out;
  const double* ay_p;  // a_J'y_J
  const double* aa_p;  // a_J'a_J
  const double* g;
  const double* w;
  const double* qw;
  double* dots_out;
  unsigned int* ticket;
  double* part;
  const double* t;     // optional: dots_out[3] = t't (length q), by block 0
  long long q;
};

__global__ void __launch_bounds__(SSNAL_NT) hs_finish_dots_kernel(HsDotArgs p) {
  __shared__ double red[3 * 32];
  if (p.t && blockIdx.x == 0) {
    double tt[1] = {0.0};
    for (long long i = threadIdx.x; i < p.q; i += blockDim.x) tt[0] += p.t[i] * p.t[i];
    const int ops1[1] = {0};
    block_reduce<1>(tt, ops1, red);
    if (threadIdx.x == 0) p.dots_out[3] = tt[0];
  }
  const double ay = *p.ay_p, aa = *p.aa_p;
  const double coef = aa != 0.0 ? ay / aa : 0.0;
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    const double yi = p.y[i];
    double py = p.fm[i] ? __dsub_rn(yi, __dmul_rn(coef, p.a[i])) : 0.0;
    double r = p.beta * py;
    if (p.add) r = p.alpha * p.add[i] + r;
    p.out[i] = r;
    const double wi = p.w[i];
    acc[0] += p.g[i] * r;
    acc[1] += wi * p.qw[i];
    acc[2] += wi * yi;
  }
  const int ops[3] = {0, 0, 0};
  block_reduce<3>(acc, ops, red);
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) p.part[blockIdx.x * 3 + j] = acc[j];
  if (!last_block_arrive(p.ticket, gridDim.x)) return;
  block_fold_partials<3>(p.part, gridDim.x, 3, ops, acc, red);
  if (threadIdx.x == 0)
    for (int j = 0; j < 3; ++j) p.dots_out[j] = acc[j];
}

cudaError_t launch_hs_apply_dots(const uint8_t* fm, const double* a, const double* y, long long n,
                                 double beta, const double* add, double alpha, double* out,
                                 const double* g, const double* w, const double* qw,
                                 double* dots_out, void* ws, cudaStream_t stream) {
  double* sums = (double*)((char*)ws + reduce_ws_bytes(n));
  const double* xs[2] = {a, a};
  const double* ys[2] = {y, nullptr};
  cudaError_t e = launch_dots(2, xs, ys, fm, n, sums, ws, stream);
  if (e != cudaSuccess) return e;
  HsDotArgs p{fm, a, y, n, beta, alpha, add, out, sums, sums + 1, g, w, qw, dots_out,
              (unsigned int*)ws, (double*)((char*)ws + TICKET_BYTES), nullptr, 0};
  { note_launch(); hs_finish_dots_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(p); }
  return cudaGetLastError();
}

cudaError_t launch_hs_finish_dots(const uint8_t* fm, const double* a, const double* y, long long n,
                                  double beta, const double* add, double alpha, double* out,
                                  const double* ay, const double* aa, const double* g,
                                  const double* w, const double* qw, const double* t, long long q,
                                  double* dots_out, void* ws, cudaStream_t stream) {
  HsDotArgs p{fm, a, y, n, beta, alpha, add, out, ay, aa, g, w, qw, dots_out,
              (unsigned int*)ws, (double*)((char*)ws + TICKET_BYTES), t, q};
  // one slot per thread (n = 5e4: 196 CTAs): no serial grid-stride chain of loads
  { note_launch(); hs_finish_dots_kernel<<<stream_blocks(n, 1), SSNAL_NT, 0, stream>>>(p); }
  return cudaGetLastError();
}

// Accepted Armijo step, one pass: w += alpha d, Qw += alpha Qd, u += cu Qd (cu =
// -sigma alpha), Pi(u) and the free mask from trial j (replaces 3 vec launches + 2 copies;
// same numpy-ordered arithmetic as vec op 2)
__global__ void accept_kernel(long long n, double alpha, double cu, double* __restrict__ w,
                              const double* __restrict__ d, double* __restrict__ qw,
                              const double* __restrict__ qd, double* __restrict__ u,
                              double* __restrict__ xp, const double* __restrict__ txj,
                              uint8_t* __restrict__ fr, const uint8_t* __restrict__ tfj) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double qdi = qd[i];
    w[i] = __dadd_rn(w[i], __dmul_rn(alpha, d[i]));
    qw[i] = __dadd_rn(qw[i], __dmul_rn(alpha, qdi));
    u[i] = __dadd_rn(u[i], __dmul_rn(cu, qdi));
    xp[i] = txj[i];
    fr[i] = tfj[i];
  }
}

cudaError_t launch_accept(long long n, double alpha, double cu, double* w, const double* d,
                          double* qw, const double* qd, double* u, double* xp, const double* txj,
                          uint8_t* fr, const uint8_t* tfj, cudaStream_t stream) {
  { note_launch(); accept_kernel<<<stream_blocks(n, 4), SSNAL_NT, 0, stream>>>(n, alpha, cu, w, d, qw, qd, u, xp, txj, fr, tfj); }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- compaction
// Tile = SSNAL_NT threads x CPT contiguous elements; pass 1 counts per tile and
// the last block scans tile counts; pass 2 writes ascending indices.
static constexpr int CPT = 16;
static constexpr int TILE = SSNAL_NT * CPT;

__device__ __forceinline__ int block_exclusive_scan(int v, int* sm /* >= 33 */, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int s = lane < nw ? sm[lane] : 0;
    int si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    if (lane < nw) sm[lane] = si - s;
    if (lane == nw - 1) sm[32] = si;
  }
  __syncthreads();
  int r = sm[warp] + incl - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SSNAL_NT) compact_count_kernel(const uint8_t* __restrict__ m,
                                                                 long long n, int* tile_cnt,
                                                                 long long* count,
                                                                 unsigned int* ticket, int ntiles) {
  __shared__ int sm[33];
  long long base = (long long)blockIdx.x * TILE + (long long)threadIdx.x * CPT;
  int c = 0;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    long long i = base + j;
    if (i < n && m[i]) ++c;
  }
  int tot;
  block_exclusive_scan(c, sm, &tot);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
  if (!last_block_arrive(ticket, gridDim.x)) return;
  // exclusive scan of tile counts in place (tile_cnt -> offsets), chunked by the block
  int carry = 0;
  for (int start = 0; start < ntiles; start += SSNAL_NT) {
    int idx = start + threadIdx.x;
    int v = idx < ntiles ? __ldcg(tile_cnt + idx) : 0;
    int chunk_tot;
    int ex = block_exclusive_scan(v, sm, &chunk_tot);
    if (idx < ntiles) tile_cnt[idx] = carry + ex;
    carry += chunk_tot;
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(SSNAL_NT) compact_write_kernel(const uint8_t* __restrict__ m,
                                                                 long long n,
                                                                 const int* __restrict__ tile_off,
                                                                 int32_t* __restrict__ idx) {
  __shared__ int sm[33];
  long long base = (long long)blockIdx.x * TILE + (long long)threadIdx.x * CPT;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    long long i = base + j;
    if (i < n && m[i]) bits |= 1u << j;
  }
  int tot;
  int off = block_exclusive_scan(__popc(bits), sm, &tot) + tile_off[blockIdx.x];
  while (bits) {
    int j = __ffs(bits) - 1;
    bits &= bits - 1;
    idx[off++] = (int32_t)(base + j);
  }
}

size_t compact_ws_bytes(long long n) {
  return TICKET_BYTES + (size_t)ceil_div(n, TILE) * sizeof(int) + 64;
}

cudaError_t launch_compact(const uint8_t* m, long long n, int32_t* idx, long long* count,
                           void* ws, cudaStream_t stream) {
  int ntiles = (int)ceil_div(n, TILE);
  if (ntiles < 1) ntiles = 1;
  unsigned int* ticket = (unsigned int*)ws;
  int* tile = (int*)((char*)ws + TICKET_BYTES);
  { note_launch(); compact_count_kernel<<<ntiles, SSNAL_NT, 0, stream>>>(m, n, tile, count, ticket, ntiles); }
  { note_launch(); compact_write_kernel<<<ntiles, SSNAL_NT, 0, stream>>>(m, n, tile, idx); }
  return cudaGetLastError();
}

}  // namespace ssnal

// Dense data-operator kernels for Q = X X^T, X = S diag(row_sign) A (row-major A).
//
//   X^T V : column panels x row splits; each warp streams whole rows (coalesced,
//           lanes over columns), per-lane register accumulators, warps folded
//           in fixed order, splits folded by a second deterministic pass.
//   X D   : one warp per row, D staged in shared memory, shuffle-reduced dots.
//   Gram  : G = X_J^T X_J on the fp64 tensor cores (DMMA 8x8x4) over gathered
//           free rows J, split-K over J with fixed-order fold, then assembled
//           into the Prop. 3.5 Newton matrix I + sigma (G - m1 m1^T / a'Sa).
// ref: kernels.py:97-106,144-154 (column-wise Q), solver.py:224-262 (Q_JJ, cols@v).
#include <algorithm>

#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

int stream_blocks(long long n, int per_thread);

// ------------------------------------------------------------------ X^T V
static constexpr int XT_MAXC = 10;  // scalar columns per lane per panel (320-wide panels)
static constexpr int XT_PANEL = 32 * XT_MAXC;
static constexpr int XT_WARPS = 8;

struct XtArgs {
  const double* A;
  long long n, q, lda;
  const double* rs;
  int svr;
  const double* v[4];
  int k;
  double* part;  // [nsplit][k][q]
  double* out;   // [k][q]
};

template <int KV>
__global__ void __launch_bounds__(XT_WARPS * 32) dense_xt_kernel(XtArgs p, int kofs) {
  __shared__ double red[XT_WARPS][KV][XT_PANEL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long col0 = (long long)blockIdx.y * XT_PANEL;
  const long long nsplit = gridDim.x;
  const long long rows_per = ceil_div(p.n, nsplit);
  const long long r0 = blockIdx.x * rows_per;
  const long long r1 = min(p.n, r0 + rows_per);
  double acc[KV][XT_MAXC];
#pragma unroll
  for (int j = 0; j < KV; ++j)
#pragma unroll
    for (int c = 0; c < XT_MAXC; ++c) acc[j][c] = 0.0;
  const double* vp[KV];
#pragma unroll
  for (int j = 0; j < KV; ++j) vp[j] = kofs == 0 ? p.v[j] : p.v[j + 2];  // kofs in {0, 2}
  for (long long r = r0 + warp; r < r1; r += XT_WARPS) {
    double coef[KV];
    const double sg = p.rs ? p.rs[r] : 1.0;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      double cv = vp[j][r];
      if (p.svr) cv = __dsub_rn(cv, vp[j][r + p.n]);
      coef[j] = sg * cv;
    }
    const double* row = p.A + r * p.lda + col0;
    double av[XT_MAXC];
#pragma unroll
    for (int c = 0; c < XT_MAXC; ++c) {
      long long col = col0 + lane + 32 * c;
      av[c] = col < p.q ? __ldg(row + lane + 32 * c) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < KV; ++j)
#pragma unroll
      for (int c = 0; c < XT_MAXC; ++c) acc[j][c] = fma(coef[j], av[c], acc[j][c]);
  }
#pragma unroll
  for (int j = 0; j < KV; ++j)
#pragma unroll
    for (int c = 0; c < XT_MAXC; ++c) red[warp][j][lane + 32 * c] = acc[j][c];
  __syncthreads();
  for (int idx = threadIdx.x; idx < KV * XT_PANEL; idx += blockDim.x) {
    int j = idx / XT_PANEL, c = idx % XT_PANEL;
    long long col = col0 + c;
    if (col >= p.q) continue;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < XT_WARPS; ++w) s += red[w][j][c];
    p.part[((long long)blockIdx.x * p.k + kofs + j) * p.q + col] = s;
  }
}

// one warp per output entry: lanes fold splits lane, lane+32, ..., then a fixed
// shuffle tree -- deterministic and ~32x shorter dependency chains than a thread fold
// Vectorised X^T V (even lda, 16B-aligned A): thread t owns the column pair
// (2t, 2t+1) of a panel; the block streams its contiguous row range UNR rows at a
// time, i.e. UNR independent 16-byte loads in flight per thread, with the row
// coefficients (labels x vector entries) loaded alongside.  Partials per row split.
template <int KV, int UNR>
__global__ void __launch_bounds__(512) dense_xt2_kernel(XtArgs p, int kofs) {
  const long long col = (long long)blockIdx.y * (2 * blockDim.x) + 2 * threadIdx.x;
  const bool active = col < p.q;
  const long long nsplit = gridDim.x;
  const long long rows_per = ceil_div(p.n, nsplit);
  const long long r0 = blockIdx.x * rows_per;
  const long long r1 = min(p.n, r0 + rows_per);
  const double* vp[KV];
#pragma unroll
  for (int j = 0; j < KV; ++j) vp[j] = kofs == 0 ? p.v[j] : p.v[j + 2];
  double ax[KV], ay[KV];
#pragma unroll
  for (int j = 0; j < KV; ++j) ax[j] = ay[j] = 0.0;
  const double* base = p.A + col;
  for (long long r = r0; r < r1; r += UNR) {
    double2 av[UNR];
    double cf[UNR][KV];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long rr = r + u;
      const bool ok = rr < r1;
      av[u] = (ok && active) ? __ldg(reinterpret_cast<const double2*>(base + rr * p.lda))
                             : make_double2(0.0, 0.0);
      const double sg = (ok && p.rs) ? p.rs[rr] : 1.0;
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        double cv = ok ? vp[j][rr] : 0.0;
        if (ok && p.svr) cv = __dsub_rn(cv, vp[j][rr + p.n]);
        cf[u][j] = sg * cv;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        ax[j] = fma(cf[u][j], av[u].x, ax[j]);
        ay[j] = fma(cf[u][j], av[u].y, ay[j]);
      }
  }
  if (!active) return;
#pragma unroll
  for (int j = 0; j < KV; ++j) {
    double* dst = p.part + ((long long)blockIdx.x * p.k + kofs + j) * p.q + col;
    dst[0] = ax[j];
    dst[1] = ay[j];
  }
}

__global__ void dense_xt_fold_kernel(const double* __restrict__ part, long long nsplit, int k,
                                     long long q, double* __restrict__ out) {
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= (long long)k * q) return;
  double s = 0.0;
  for (long long b = lane; b < nsplit; b += 32) s += __ldcg(part + b * k * q + idx);
  s = warp_sum(s);
  if (lane == 0) out[idx] = s;
}

static int xt_splits(long long n) {
  long long s = ceil_div(n, 64);  // at least 64 rows per split
  if (s > 4 * 148) s = 4 * 148;
  if (s < 1) s = 1;
  return (int)s;
}

bool stream_ok(const double* A, long long lda, long long q);
int stream_grid(long long n);
cudaError_t launch_stream_xt(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, int k, const double* const* vs, int kofs,
                             int ktot, double* part, cudaStream_t stream,
                             const double* vsub = nullptr, double* vout = nullptr);
cudaError_t launch_stream_xd(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, int k, const double* d, double* out,
                             long long nlog, cudaStream_t stream, double* sq_part = nullptr,
                             double* sq_out = nullptr, unsigned int* sq_ticket = nullptr,
                             int epi = 0, const uint8_t* fm = nullptr, const double* av = nullptr,
                             double* sq_out2 = nullptr);
cudaError_t launch_hs_finish_dots(const uint8_t* fm, const double* a, const double* y, long long n,
                                  double beta, const double* add, double alpha, double* out,
                                  const double* ay, const double* aa, const double* g,
                                  const double* w, const double* qw, const double* t, long long q,
                                  double* dots_out, void* ws, cudaStream_t stream);
cudaError_t launch_vec(int op, long long n, double alpha, const double* x, const double* y,
                       const double* z, double* out, cudaStream_t s);
cudaError_t launch_dots(int k, const double* const* xs, const double* const* ys,
                        const uint8_t* mask, long long n, double* out, void* ws, cudaStream_t s);
size_t reduce_ws_bytes(long long n);

size_t dense_xt_ws_bytes(long long n_phys, long long q, int k) {
  const long long splits = max((long long)xt_splits(n_phys), (long long)stream_grid(n_phys));
  return (size_t)splits * k * q * sizeof(double);
}

// layout: [0, 256) tickets at FIXED offsets (a workspace reused across problem sizes
// must never see a ticket where another size wrote partial sums), then the dots
// fallback's workspace (its own ticket at byte 256), the per-CTA squared-norm
// partials, the X^T partials
static size_t grad_red_bytes(long long n_phys) {
  return (reduce_ws_bytes(2 * n_phys) + 255) / 256 * 256;
}
size_t gradient_ws_bytes(long long n_phys, long long q) {
  return 256 + grad_red_bytes(n_phys) + (size_t)(2 * stream_grid(n_phys) + 32) * sizeof(double) +
         dense_xt_ws_bytes(n_phys, q, 1);
}

static bool vec2_ok(const double* A, long long lda, long long q) {
  return (lda % 2 == 0) && (q % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
}

cudaError_t launch_dense_xt(const double* A, long long n, long long q, long long lda,
                            const double* rs, int svr, int k, const double* const* vs,
                            double* out, void* ws, cudaStream_t stream) {
  XtArgs p;
  p.A = A; p.n = n; p.q = q; p.lda = lda; p.rs = rs; p.svr = svr; p.k = k;
  for (int j = 0; j < 4; ++j) p.v[j] = j < k ? vs[j] : nullptr;
  p.part = (double*)ws;
  p.out = out;
  int nsplit = xt_splits(n);
  if (stream_ok(A, lda, q)) {  // TMA-staged streaming (csrc/stream.cu)
    const int grid = stream_grid(n);
    for (int j = 0; j < k;) {
      const int kk = (k - j >= 2) ? 2 : 1;
      cudaError_t e = launch_stream_xt(A, n, q, lda, rs, svr, kk, vs, j, k, p.part, stream);
      if (e != cudaSuccess) return e;
      j += kk;
    }
    long long tot = (long long)k * q;
    { note_launch(); dense_xt_fold_kernel<<<(unsigned)ceil_div(tot * 32, 256), 256, 0, stream>>>(p.part, grid, k, q, out); }
    return cudaGetLastError();
  }
  if (vec2_ok(A, lda, q)) {
    long long pairs = q / 2;
    int threads = (int)min(512LL, ceil_div(pairs, 32) * 32);
    dim3 grid2(nsplit, (unsigned)ceil_div(pairs, threads));
    for (int j = 0; j < k;) {
      if (k - j >= 2) {
        { note_launch(); dense_xt2_kernel<2, 8><<<grid2, threads, 0, stream>>>(p, j); }
        j += 2;
      } else {
        { note_launch(); dense_xt2_kernel<1, 8><<<grid2, threads, 0, stream>>>(p, j); }
        j += 1;
      }
    }
    long long tot = (long long)k * q;
    { note_launch(); dense_xt_fold_kernel<<<(unsigned)ceil_div(tot * 32, 256), 256, 0, stream>>>(p.part, nsplit, k, q, out); }
    return cudaGetLastError();
  }
  nsplit = min(nsplit, 296);
  dim3 grid(nsplit, (unsigned)ceil_div(q, XT_PANEL));
  for (int j = 0; j < k;) {
    if (k - j >= 2) {
      { note_launch(); dense_xt_kernel<2><<<grid, XT_WARPS * 32, 0, stream>>>(p, j); }
      j += 2;
    } else {
      { note_launch(); dense_xt_kernel<1><<<grid, XT_WARPS * 32, 0, stream>>>(p, j); }
      j += 1;
    }
  }
  long long tot = (long long)k * q;
  { note_launch(); dense_xt_fold_kernel<<<(unsigned)ceil_div(tot * 32, 256), 256, 0, stream>>>(p.part, nsplit, k, q, out); }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ X D
static constexpr int X_WARPS = 8;
static constexpr int X_ROWS = 2;  // rows in flight per warp

template <int KV>
__global__ void __launch_bounds__(X_WARPS * 32) dense_x_kernel(const double* __restrict__ A,
                                                               long long n, long long q,
                                                               long long lda,
                                                               const double* __restrict__ rs,
                                                               int svr, const double* __restrict__ d,
                                                               int k, int kofs,
                                                               double* __restrict__ out,
                                                               long long nlog) {
  extern __shared__ double sd[];  // [KV][q]
  for (long long i = threadIdx.x; i < (long long)KV * q; i += blockDim.x)
    sd[i] = d[(long long)kofs * q + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * X_WARPS + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * X_WARPS;
  for (long long r0 = gw * X_ROWS; r0 < n; r0 += nw * X_ROWS) {
    double acc[X_ROWS][KV];
#pragma unroll
    for (int rr = 0; rr < X_ROWS; ++rr)
#pragma unroll
      for (int j = 0; j < KV; ++j) acc[rr][j] = 0.0;
    for (long long c = lane; c < q; c += 32) {
#pragma unroll
      for (int rr = 0; rr < X_ROWS; ++rr) {
        long long r = r0 + rr;
        if (r < n) {
          double a = __ldg(A + r * lda + c);
#pragma unroll
          for (int j = 0; j < KV; ++j) acc[rr][j] = fma(a, sd[j * q + c], acc[rr][j]);
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < X_ROWS; ++rr) {
      long long r = r0 + rr;
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        double s = warp_sum(acc[rr][j]);
        if (lane == 0 && r < n) {
          double v = rs ? rs[r] * s : s;
          out[(long long)(kofs + j) * nlog + r] = v;
          if (svr) out[(long long)(kofs + j) * nlog + r + n] = -v;
        }
      }
    }
  }
}

// Vectorised X D: one warp per R rows, lanes stride the row in 16-byte column
// pairs with all CP x R loads of a warp-task issued before the FMAs (D staged in
// shared memory as double2), shuffle-tree dot products.
template <int KV, int R, int CP>
__global__ void __launch_bounds__(256, 2) dense_x2_kernel(const double* __restrict__ A, long long n,
                                                      long long q, long long lda,
                                                      const double* __restrict__ rs, int svr,
                                                      const double* __restrict__ d, int kofs,
                                                      double* __restrict__ out, long long nlog) {
  extern __shared__ double2 sd2[];  // [KV][q/2]
  const long long pairs = q / 2;
  for (long long i = threadIdx.x; i < (long long)KV * pairs; i += blockDim.x) {
    const long long j = i / pairs, c = i % pairs;
    sd2[i] = make_double2(d[(kofs + j) * q + 2 * c], d[(kofs + j) * q + 2 * c + 1]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r0 = gw * R; r0 < n; r0 += nw * R) {
    double2 av[R][CP];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int cp = 0; cp < CP; ++cp) {
        const long long c = lane + 32 * cp, r = r0 + rr;
        av[rr][cp] = (c < pairs && r < n)
                         ? __ldg(reinterpret_cast<const double2*>(A + r * lda) + c)
                         : make_double2(0.0, 0.0);
      }
    double acc[R][KV];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int j = 0; j < KV; ++j) acc[rr][j] = 0.0;
#pragma unroll
    for (int cp = 0; cp < CP; ++cp) {
      const long long c = lane + 32 * cp;
      if (c < pairs) {
#pragma unroll
        for (int j = 0; j < KV; ++j) {
          const double2 dv = sd2[j * pairs + c];
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            acc[rr][j] = fma(av[rr][cp].y, dv.y, fma(av[rr][cp].x, dv.x, acc[rr][j]));
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const long long r = r0 + rr;
#pragma unroll
      for (int j = 0; j < KV; ++j) {
        const double s = warp_sum(acc[rr][j]);
        if (lane == 0 && r < n) {
          const double v = rs ? rs[r] * s : s;
          out[(long long)(kofs + j) * nlog + r] = v;
          if (svr) out[(long long)(kofs + j) * nlog + r + n] = -v;
        }
      }
    }
  }
}

template <int KV, int CP>
static void launch_x2(const double* A, long long n, long long q, long long lda, const double* rs,
                      int svr, const double* d, int kofs, double* out, long long nlog,
                      cudaStream_t stream) {
  constexpr int R = 2;
  const size_t smem = (size_t)KV * (q / 2) * sizeof(double2);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(dense_x2_kernel<KV, R, CP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  long long blocks = ceil_div(n, 8LL * R);
  if (blocks > 8 * 148) blocks = 8 * 148;
  note_launch();
  dense_x2_kernel<KV, R, CP><<<(unsigned)blocks, 256, smem, stream>>>(A, n, q, lda, rs, svr, d, kofs,
                                                                      out, nlog);
}

template <int KV>
static bool dispatch_x2(const double* A, long long n, long long q, long long lda, const double* rs,
                        int svr, const double* d, int kofs, double* out, long long nlog,
                        cudaStream_t stream) {
  const long long cps = ceil_div(q / 2, 32);
  if (cps <= 1) launch_x2<KV, 1>(A, n, q, lda, rs, svr, d, kofs, out, nlog, stream);
  else if (cps <= 2) launch_x2<KV, 2>(A, n, q, lda, rs, svr, d, kofs, out, nlog, stream);
  else if (cps <= 4) launch_x2<KV, 4>(A, n, q, lda, rs, svr, d, kofs, out, nlog, stream);
  else if (cps <= 8) launch_x2<KV, 8>(A, n, q, lda, rs, svr, d, kofs, out, nlog, stream);
  else return false;
  return true;
}

cudaError_t launch_dense_x(const double* A, long long n, long long q, long long lda,
                           const double* rs, int svr, int k, const double* d, double* out,
                           cudaStream_t stream) {
  long long nlog = svr ? 2 * n : n;
  if (stream_ok(A, lda, q) && q <= 512) {  // TMA-staged streaming (csrc/stream.cu)
    for (int j = 0; j < k;) {
      const int kk = (k - j >= 2) ? 2 : 1;
      cudaError_t e = launch_stream_xd(A, n, q, lda, rs, svr, kk, d + (long long)j * q,
                                       out + (long long)j * nlog, nlog, stream);
      if (e != cudaSuccess) return e;
      j += kk;
    }
    return cudaGetLastError();
  }
  if (vec2_ok(A, lda, q) && q <= 512) {
    for (int j = 0; j < k;) {
      if (k - j >= 2) {
        dispatch_x2<2>(A, n, q, lda, rs, svr, d, j, out, nlog, stream);
        j += 2;
      } else {
        dispatch_x2<1>(A, n, q, lda, rs, svr, d, j, out, nlog, stream);
        j += 1;
      }
    }
    return cudaGetLastError();
  }
  long long blocks = ceil_div(n, (long long)X_WARPS * X_ROWS);
  if (blocks > 4 * 148) blocks = 4 * 148;
  if (blocks < 1) blocks = 1;
  for (int j = 0; j < k;) {
    int kv = (k - j >= 2) ? 2 : 1;
    size_t smem = (size_t)kv * q * sizeof(double);
    if (kv == 2) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(dense_x_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      { note_launch(); dense_x_kernel<2><<<(unsigned)blocks, X_WARPS * 32, smem, stream>>>(A, n, q, lda, rs, svr, d, k, j, out, nlog); }
    } else {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(dense_x_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      { note_launch(); dense_x_kernel<1><<<(unsigned)blocks, X_WARPS * 32, smem, stream>>>(A, n, q, lda, rs, svr, d, k, j, out, nlog); }
    }
    j += kv;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Gram (DMMA)
// G = sum_r x_r x_r^T over gathered rows r of X (the free set J, or the slots whose
// free flag changed, signed), FP64 tensor cores (DMMA m8n8k4; tcgen05 has no f64 kind).
//   * CTA = one 128 x 128 tile pair (ti <= tj) of G x one split of the row list; 8 warps
//     as 2 x 4, each warp a 64 x 32 block = 8 x 4 DMMA tiles (64 accumulators), so one
//     k-step of 4 rows issues 32 DMMAs from 12 shared-memory fragment loads;
//   * rows staged 32 at a time by cp.async (16-byte LDGSTS, zero-filled past q) into a
//     two-stage ring: the gather of stage k+1 overlaps the DMMAs of stage k; diagonal
//     pairs stage one slice and read both operands from it;
//   * split-K over the row list into `split` fixed chunks (one wave: pairs x split <=
//     SMs), partials folded in split order by gram_fold_kernel -> deterministic.
static constexpr int GT = 128;             // output tile edge
static constexpr int GK = 32;              // gathered rows per stage
static constexpr int GLD = GT + 4;         // padded smem row: conflict-free 64-bit fragments
static constexpr int GSPLIT = 32;          // max split-K chunks (partials buffer)
static constexpr int GNT = 256;
static constexpr size_t GSTAGE = (size_t)GK * GLD;  // doubles per operand per stage
static constexpr size_t GSMEM = 4 * GSTAGE * sizeof(double) + 2 * GK * sizeof(double);

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(double* dst, const double* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes));
}

struct GramArgs {
  const double* A;
  long long n, q, lda;
  const int32_t* J;
  const long long* p_dev;
  double* part;  // [split][q][q] (upper tile pairs + full diagonal tiles)
  int ntile, split;
  // m1 = X_J^T a_J rides on the diagonal tiles' staged rows: weights w_r = a_{J_r} times
  // the row sign, part_m1[split][q]
  const double* a;
  const double* rs;
  int svr;
  double* part_m1;
  // incremental mode: J lists the slots whose free flag CHANGED; the slot enters with
  // weight +1 if now free (mask[slot] = 1), -1 if it left the free set
  const uint8_t* sign_mask;
  int aligned;  // rows 16-byte aligned (cp.async staging) else scalar staging
  // device-side choice (driver): ctl->mode 1 = incremental over Jd (ctl->count rows,
  // signed by sign_mask), 0 = rebuild over J (ctl->count = p rows)
  const GramCtl* ctl;
  const int32_t* Jd;
};

// one staged block of GK rows: 8 k-steps x (8 A + 4 B fragments, 32 DMMAs) per warp
template <bool SIGNED>
__device__ __forceinline__ void gram_kstage(double (&acc)[8][4][2], const double* __restrict__ cA,
                                            const double* __restrict__ cB,
                                            const double* __restrict__ sgn, int lane, int wm,
                                            int wn) {
#pragma unroll
  for (int kk = 0; kk < GK; kk += 4) {
    const int kr = kk + (lane & 3);
    double af[8], bf[4];
#pragma unroll
    for (int a = 0; a < 8; ++a) af[a] = cA[kr * GLD + wm * 64 + a * 8 + (lane >> 2)];
    if (SIGNED) {
      const double sg = sgn[kr];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] *= sg;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = cB[kr * GLD + wn * 32 + b * 8 + (lane >> 2)];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
}

// grid.x = tile pair index (ti <= tj), grid.y = split
__global__ void __launch_bounds__(GNT, 1) gram_kernel(GramArgs g) {
  extern __shared__ double gsm[];
  double* sA = gsm;                    // [2][GK][GLD]
  double* sB = gsm + 2 * GSTAGE;       // [2][GK][GLD]
  double* sw = gsm + 4 * GSTAGE;       // [2][GK] m1 weights (incl. sign)
  __shared__ double ssg[2][GK];        // row signs (incremental mode)
  const bool incr = g.ctl ? g.ctl->mode == 1 : g.sign_mask != nullptr;
  const long long p = g.ctl ? g.ctl->count : *g.p_dev;
  const int32_t* __restrict__ Jl = (g.ctl && incr) ? g.Jd : g.J;
  const uint8_t* __restrict__ smask = incr ? g.sign_mask : nullptr;
  int pair = blockIdx.x, ti = 0;
  while (pair >= g.ntile - ti) { pair -= g.ntile - ti; ++ti; }
  const int tj = ti + pair;
  const long long chunk = ceil_div(p, (long long)g.split);
  const long long k0 = blockIdx.y * chunk;
  const long long k1 = min(p, k0 + chunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp block: rows wm*64.., cols wn*32..
  const long long ci = (long long)ti * GT, cj = (long long)tj * GT;
  const bool diag = ti == tj;
  const bool signed_rows = smask != nullptr;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double m1acc = 0.0;

  // Staging, software-pipelined over THREE stages of row indices: the J entries (and
  // the m1 weights / signs, which chain J -> a, sign_mask) of stage k+2 are loaded into
  // registers while stage k computes; stage k+1's cp.async copies are issued from the
  // registers loaded one iteration earlier.  (With the J loads at the head of each stage
  // every stage began with a dependent L2 round trip: ncu showed the warps stalled on
  // the sign extension of the loaded index.)
  static_assert(GK == 32 && GNT == 256, "staging map assumes 32 rows x 256 threads");
  const int ch = tid & 63, kr0 = tid >> 6;
  struct Pre {
    long long rowoff[8];
    double w, sg;
  };
  auto pre = [&](long long kb, Pre& R) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long r = kb + kr0 + 4 * i;
      long long off = -1;
      if (r < k1) {
        const long long li = Jl[r];
        off = (li >= g.n ? li - g.n : li) * g.lda;  // SVR block: x x^T is sign-free
      }
      R.rowoff[i] = off;
    }
    R.w = 0.0;
    R.sg = 1.0;
    if (tid < GK) {
      const long long r = kb + tid;
      if (r < k1) {
        const long long li = Jl[r];
        const long long pr = li >= g.n ? li - g.n : li;
        if (signed_rows && !smask[li]) R.sg = -1.0;  // a leaving row: -x x^T
        if (diag) {  // m1 weight (gram_m1's order of operations)
          double w = g.a[li];
          if (g.rs) w *= g.rs[pr];
          if (g.svr && li >= g.n) w = -w;
          R.w = w * R.sg;
        }
      }
    }
  };
  // stage rows [kb, kb + GK) into buffer s from prefetched row offsets
  auto issue = [&](long long kb, int s, const Pre& R) {
    double* dA = sA + s * GSTAGE;
    double* dB = sB + s * GSTAGE;
    if (g.aligned) {
      // 64 16-byte chunks per 128-column slice: thread tid copies chunk (tid & 63) of rows
      // (tid >> 6) + 4i, i < 8, on both sides
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (side == 1 && diag) break;
        const long long c0 = (side ? cj : ci) + 2 * ch;
        const int bytes_full = c0 < g.q ? (c0 + 1 < g.q ? 16 : 8) : 0;
        double* dbase = (side ? dB : dA) + 2 * ch;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int kr = kr0 + 4 * i;
          const bool ok = R.rowoff[i] >= 0 && bytes_full > 0;
          cp_async16(dbase + kr * GLD, ok ? g.A + R.rowoff[i] + c0 : g.A, ok ? bytes_full : 0);
        }
      }
    } else {
      const int nsides = diag ? 1 : 2;
      for (int idx = tid; idx < GK * GT * nsides; idx += GNT) {
        const int side = idx / (GK * GT), rem = idx % (GK * GT);
        const int kr = rem / GT, c = rem % GT;
        const long long r = kb + kr;
        const long long col = (side ? cj : ci) + c;
        double v = 0.0;
        if (r < k1 && col < g.q) {
          const long long li = Jl[r];
          const long long pr = li >= g.n ? li - g.n : li;
          v = __ldg(g.A + pr * g.lda + col);
        }
        (side ? dB : dA)[kr * GLD + c] = v;
      }
    }
    if (tid < GK) {
      sw[s * GK + tid] = R.w;
      ssg[s][tid] = R.sg;
    }
  };

  int buf = 0;
  Pre R;
  if (k0 < k1) {
    pre(k0, R);
    issue(k0, 0, R);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (k0 + GK < k1) pre(k0 + GK, R);
  for (long long kb = k0; kb < k1; kb += GK) {
    if (kb + GK < k1) issue(kb + GK, buf ^ 1, R);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (kb + 2 * GK < k1) pre(kb + 2 * GK, R);  // in flight during this stage's DMMAs
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const double* cA = sA + buf * GSTAGE;
    const double* cB = diag ? cA : sB + buf * GSTAGE;
    if (diag && tid < GT) {  // m1 column ci + tid from the unsigned staged rows
      const int nk = (int)min((long long)GK, k1 - kb);
      for (int kr = 0; kr < nk; ++kr) m1acc = fma(sw[buf * GK + kr], cA[kr * GLD + tid], m1acc);
    }
    // (block-uniform branch: the rebuild's k-loop carries no sign multiplies)
    if (signed_rows) {
      gram_kstage<true>(acc, cA, cB, ssg[buf], lane, wm, wn);
    } else {
      gram_kstage<false>(acc, cA, cB, ssg[buf], lane, wm, wn);
    }
    __syncthreads();  // buffer `buf` free for the stage after next
    buf ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (diag && tid < GT && ci + tid < g.q) g.part_m1[blockIdx.y * g.q + ci + tid] = m1acc;
  // C fragment: row = lane/4, cols = 2*(lane%4) + {0,1}
  double* dst = g.part + (long long)blockIdx.y * g.q * g.q;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const long long row = ci + wm * 64 + a * 8 + (lane >> 2);
    if (row >= g.q) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const long long col = cj + wn * 32 + b * 8 + 2 * (lane & 3);
      if (col < g.q) dst[row * g.q + col] = acc[a][b][0];
      if (col + 1 < g.q) dst[row * g.q + col + 1] = acc[a][b][1];
    }
  }
}

// G (= X_J^T X_J in the partials' tile layout: upper tile pairs, lower tiles stored
// transposed) and m1 from the GSPLIT split-K partials, in split order; accumulate = 1
// adds them to the kept G / m1 (incremental update over the changed slots)
__global__ void gram_fold_kernel(const double* __restrict__ part, const double* __restrict__ part_m1,
                                 long long q, int split, double* __restrict__ G,
                                 double* __restrict__ m1, int accumulate,
                                 const GramCtl* __restrict__ ctl) {
  if (ctl) accumulate = ctl->mode == 1;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < q * q) {
    const long long i = idx / q, j = idx % q;
    if (i / GT <= j / GT) {  // stored positions only
      double s = accumulate ? G[idx] : 0.0;
      double d = 0.0;
      for (int b = 0; b < split; ++b) d += part[(long long)b * q * q + idx];
      G[idx] = s + d;
    }
  }
  if (idx < q) {
    double d = 0.0;
    for (int b = 0; b < split; ++b) d += part_m1[b * q + idx];
    m1[idx] = (accumulate ? m1[idx] : 0.0) + d;
  }
}

// M = I + sigma (G - m1 m1^T / asa)   (asa == 0: I + sigma G)
__global__ void gram_assemble_kernel(const double* __restrict__ G, long long q,
                                     const double* __restrict__ m1, double sigma,
                                     const double* __restrict__ asa_dev,
                                     double* __restrict__ M) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= q * q) return;
  long long i = idx / q, j = idx % q;
  long long si = i, sj = j;
  if (i / GT > j / GT) { si = j; sj = i; }  // lower tiles are stored transposed
  double g = G[si * q + sj];
  const double asa = *asa_dev;
  if (asa != 0.0) g = g - m1[i] * m1[j] / asa;
  M[idx] = (i == j ? 1.0 : 0.0) + sigma * g;
}

// chg = (fr != kept), kept = fr: the slots whose free flag changed since the kept Gram
__global__ void mask_diff_kernel(const uint8_t* __restrict__ fr, uint8_t* __restrict__ kept,
                                 uint8_t* __restrict__ chg, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint8_t f = fr[i];
    chg[i] = f != kept[i];
    kept[i] = f;
  }
}

// split-K chunks the partials buffer holds: one wave of tile pairs on up to 192 SMs
static int gram_split_cap(long long q) {
  const long long nt = ceil_div(q, GT);
  const long long npairs = nt * (nt + 1) / 2;
  return (int)std::max(1LL, std::min((long long)GSPLIT, 192 / npairs));
}

size_t gram_ws_bytes(long long q) {
  const size_t sp = (size_t)gram_split_cap(q);
  return sp * q * q * sizeof(double) + sp * q * sizeof(double);
}

// G (+)= sum over the listed slots of (+-) x x^T, m1 (+)= sum (+-) a_j x_j
// driver: rebuild over J (p rows) or update over the changed slots Jd (count d) --
// whichever gathers fewer rows, with the updates since the last rebuild capped at 2p
// (bounds the rounding drift of +-x x^T sums); decided on the device, no host sync
__global__ void gram_select_kernel(GramCtl* c, const long long* __restrict__ p_dev,
                                   const long long* __restrict__ d_dev, int force_full) {
  const long long p = *p_dev, d = *d_dev;
  const bool incr = !force_full && c->valid && 2 * d < p && c->accum + d <= 2 * p;
  if (incr) {
    c->mode = 1;
    c->count = d;
    c->accum += d;
    ++c->updates;
    c->rows += d;
  } else {
    c->mode = 0;
    c->count = p;
    c->accum = 0;
    ++c->builds;
    c->rows += p;
  }
  c->valid = 1;
}

cudaError_t launch_gram_select(GramCtl* ctl, const long long* p_dev, const long long* d_dev,
                               int force_full, cudaStream_t stream) {
  note_launch();
  gram_select_kernel<<<1, 1, 0, stream>>>(ctl, p_dev, d_dev, force_full);
  return cudaGetLastError();
}

cudaError_t launch_gram_update(const double* A, long long n, long long q, long long lda,
                               const double* rs, int svr, const int32_t* J, const long long* p_dev,
                               const uint8_t* sign_mask, const double* a, double* G, double* m1,
                               int accumulate, void* ws, cudaStream_t stream,
                               const GramCtl* ctl, const int32_t* Jd) {
  static DeviceCache cache;  // SM count (0 = the smem opt-in failed)
  const int nsm = per_device(cache, [](int dev) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)GSMEM) != cudaSuccess)
      return 0;
    return v > 0 ? v : 148;
  });
  if (nsm == 0) return cudaErrorInvalidValue;
  GramArgs g;
  g.A = A; g.n = n; g.q = q; g.lda = lda; g.J = J; g.p_dev = p_dev;
  g.part = (double*)ws;
  g.ntile = (int)ceil_div(q, GT);
  const int npairs = g.ntile * (g.ntile + 1) / 2;
  g.split = std::max(1, std::min(gram_split_cap(q), nsm / npairs));  // one wave
  double* part_m1 = g.part + (long long)gram_split_cap(q) * q * q;
  g.a = a; g.rs = rs; g.svr = svr; g.part_m1 = part_m1; g.sign_mask = sign_mask;
  g.aligned = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  g.ctl = ctl;
  g.Jd = Jd;
  { note_launch(); gram_kernel<<<dim3(npairs, g.split), GNT, GSMEM, stream>>>(g); }
  { note_launch(); gram_fold_kernel<<<(unsigned)ceil_div(q * q, 256), 256, 0, stream>>>(g.part, part_m1, q, g.split, G, m1, accumulate, ctl); }
  return cudaGetLastError();
}

cudaError_t launch_gram_assemble(const double* G, long long q, const double* m1, double sigma,
                                 const double* asa_dev, double* M, cudaStream_t stream) {
  note_launch();
  gram_assemble_kernel<<<(unsigned)ceil_div(q * q, 256), 256, 0, stream>>>(G, q, m1, sigma, asa_dev, M);
  return cudaGetLastError();
}

cudaError_t launch_mask_diff(const uint8_t* fr, uint8_t* kept, uint8_t* chg, long long n,
                             cudaStream_t stream) {
  const int blocks = (int)std::min<long long>(ceil_div(n, 256LL * 8), SSNAL_MAX_BLOCKS);
  note_launch();
  mask_diff_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, stream>>>(fr, kept, chg, n);
  return cudaGetLastError();
}

// one-shot M = I + sigma (X_J^T P X_J) (C-ABI ssnal_dense_gram); G is built in M itself
cudaError_t launch_dense_gram(const double* A, long long n, long long q, long long lda,
                              const double* rs, int svr, const int32_t* J, const long long* p_dev,
                              long long p_max, const double* a, double sigma,
                              const double* asa_dev, double* M, double* m1, void* ws,
                              cudaStream_t stream) {
  (void)p_max;
  double* G = (double*)((char*)ws + gram_ws_bytes(q));  // see gram_ws_bytes_full
  cudaError_t e = launch_gram_update(A, n, q, lda, rs, svr, J, p_dev, nullptr, a, G, m1, 0, ws,
                                     stream, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  return launch_gram_assemble(G, q, m1, sigma, asa_dev, M, stream);
}

size_t gram_ws_bytes_full(long long q) { return gram_ws_bytes(q) + (size_t)q * q * sizeof(double); }

// Fused SsN gradient (ref solver.py:143-148 with the linear-kernel operator):
//   s = w - Pi(u);  g_r = X^T s;  grad = X g_r;  *g2 = ||grad||^2
// streaming route: the X^T pass stages s on the fly (and writes it), the X pass
// accumulates ||grad||^2 -- two sweeps of A, no separate elementwise or dot launch.
cudaError_t launch_dense_gradient(const double* A, long long n, long long q, long long lda,
                                  const double* rs, int svr, const double* w, const double* xp,
                                  double* s_out, double* g_r, double* grad, double* g2, void* ws,
                                  cudaStream_t stream) {
  const long long nlog = svr ? 2 * n : n;
  char* base = (char*)ws;
  unsigned int* ticket = (unsigned int*)base;
  void* red_ws = (void*)(base + 256);
  double* sq_part = (double*)(base + 256 + grad_red_bytes(n));
  double* part = sq_part + 2 * stream_grid(n) + 32;
  if (stream_ok(A, lda, q) && q <= 512) {
    const double* vs[1] = {w};
    cudaError_t e = launch_stream_xt(A, n, q, lda, rs, svr, 1, vs, 0, 1, part, stream, xp, s_out);
    if (e != cudaSuccess) return e;
    { note_launch(); dense_xt_fold_kernel<<<(unsigned)ceil_div(q * 32, 256LL), 256, 0, stream>>>(part, stream_grid(n), 1, q, g_r); }
    return launch_stream_xd(A, n, q, lda, rs, svr, 1, g_r, grad, nlog, stream, sq_part, g2, ticket);
  }
  cudaError_t e = launch_vec(3, nlog, 0.0, w, xp, nullptr, s_out, stream);
  if (e != cudaSuccess) return e;
  const double* vs[1] = {s_out};
  e = launch_dense_xt(A, n, q, lda, rs, svr, 1, vs, g_r, part, stream);
  if (e != cudaSuccess) return e;
  e = launch_dense_x(A, n, q, lda, rs, svr, 1, g_r, grad, stream);
  if (e != cudaSuccess) return e;
  const double* xs[1] = {grad};
  const double* ys[1] = {nullptr};
  return launch_dots(1, xs, ys, nullptr, nlog, g2, red_ws, stream);
}

// Dense Newton-direction epilogue (ref solver.py:259-269): from t = X^T d
//   Qd = X t;  d = -s - sigma P_J(Qd)  with a_J'(Qd)_J folded in the X sweep and
//   a_J'a_J = the projection record's sum_a2_free;  dots = {g'd, w'Qw, w'Qd, t't}
// two launches (streaming X sweep + one elementwise/dot pass)
cudaError_t launch_direction_epilogue(const double* A, long long n, long long q, long long lda,
                                      const double* rs, int svr, const double* t, double* qdir,
                                      const uint8_t* fm, const double* a, const double* asa_dev,
                                      const double* s, double sigma, const double* grad,
                                      const double* w, const double* qw, double* dir,
                                      double* dots4, void* ws, cudaStream_t stream) {
  const long long nlog = svr ? 2 * n : n;
  char* base = (char*)ws;
  unsigned int* ticket = (unsigned int*)base;
  void* red_ws = (void*)(base + 256);
  double* ad = (double*)(base + 128);  // a_J'(Qd)_J slot (inside the ticket page)
  double* sq_part = (double*)(base + 256 + grad_red_bytes(n));
  if (stream_ok(A, lda, q) && q <= 512) {
    cudaError_t e = launch_stream_xd(A, n, q, lda, rs, svr, 1, t, qdir, nlog, stream, sq_part, ad,
                                     ticket, 2, fm, a);
    if (e != cudaSuccess) return e;
  } else {
    cudaError_t e = launch_dense_x(A, n, q, lda, rs, svr, 1, t, qdir, stream);
    if (e != cudaSuccess) return e;
    const double* xs[1] = {a};
    const double* ys[1] = {qdir};
    e = launch_dots(1, xs, ys, fm, nlog, ad, red_ws, stream);
    if (e != cudaSuccess) return e;
  }
  return launch_hs_finish_dots(fm, a, qdir, nlog, -sigma, s, -1.0, dir, ad, asa_dev, grad, w, qw,
                               t, q, dots4, red_ws, stream);
}

// Start of an inner solve in factor space: s = w - Pi(u) staged in one X^T sweep,
// r = X^T s (the gradient's factor; grad = X r is formed later by the direction
// epilogue).
cudaError_t launch_gradient_factor(const double* A, long long n, long long q, long long lda,
                                   const double* rs, int svr, const double* w, const double* xp,
                                   double* s_out, double* r, void* ws, cudaStream_t stream) {
  const long long nlog = svr ? 2 * n : n;
  char* base = (char*)ws;
  double* sq_part = (double*)(base + 256 + grad_red_bytes(n));
  double* part = sq_part + 2 * stream_grid(n) + 32;
  if (stream_ok(A, lda, q) && q <= 512) {
    const double* vs[1] = {w};
    cudaError_t e = launch_stream_xt(A, n, q, lda, rs, svr, 1, vs, 0, 1, part, stream, xp, s_out);
    if (e != cudaSuccess) return e;
    note_launch();
    dense_xt_fold_kernel<<<(unsigned)ceil_div(q * 32, 256LL), 256, 0, stream>>>(
        part, stream_grid(n), 1, q, r);
    return cudaGetLastError();
  }
  cudaError_t e = launch_vec(3, nlog, 0.0, w, xp, nullptr, s_out, stream);
  if (e != cudaSuccess) return e;
  const double* vs[1] = {s_out};
  return launch_dense_xt(A, n, q, lda, rs, svr, 1, vs, r, part, stream);
}

// grad = X r with ||grad||^2 folded into *g2 (one sweep; the Sigma = 0 steps)
cudaError_t launch_grad_from_factor(const double* A, long long n, long long q, long long lda,
                                    const double* rs, int svr, const double* r, double* grad,
                                    double* g2, void* ws, cudaStream_t stream) {
  const long long nlog = svr ? 2 * n : n;
  char* base = (char*)ws;
  unsigned int* ticket = (unsigned int*)base;
  void* red_ws = (void*)(base + 256);
  double* sq_part = (double*)(base + 256 + grad_red_bytes(n));
  if (stream_ok(A, lda, q) && q <= 512)
    return launch_stream_xd(A, n, q, lda, rs, svr, 1, r, grad, nlog, stream, sq_part, g2, ticket);
  cudaError_t e = launch_dense_x(A, n, q, lda, rs, svr, 1, r, grad, stream);
  if (e != cudaSuccess) return e;
  const double* xs[1] = {grad};
  const double* ys[1] = {nullptr};
  return launch_dots(1, xs, ys, nullptr, nlog, g2, red_ws, stream);
}

// Factor-space Newton epilogue: ONE sweep X [t, r] gives Qd and the gradient
// grad = X r of the current point (a_J'(Qd)_J and ||grad||^2 folded in the sweep), then
// d = -s - sigma P_J(Qd) and {g'd, w'Qw, w'Qd, t't} as launch_direction_epilogue.
// t2 = [t ; r] (2q), qg = [Qd ; grad] (2 nlog).
cudaError_t launch_direction_epilogue_q(const double* A, long long n, long long q, long long lda,
                                        const double* rs, int svr, const double* t2, double* qg,
                                        const uint8_t* fm, const double* a,
                                        const double* asa_dev, const double* s, double sigma,
                                        const double* w, const double* qw, double* dir,
                                        double* dots4, double* g2, void* ws,
                                        cudaStream_t stream, int parts) {
  const long long nlog = svr ? 2 * n : n;
  char* base = (char*)ws;
  unsigned int* ticket = (unsigned int*)base;
  void* red_ws = (void*)(base + 256);
  double* ad = (double*)(base + 128);
  double* sq_part = (double*)(base + 256 + grad_red_bytes(n));
  double* qdir = qg;
  double* grad = qg + nlog;
  if (!(parts & 1)) {
  } else if (stream_ok(A, lda, q) && q <= 512) {
    cudaError_t e = launch_stream_xd(A, n, q, lda, rs, svr, 2, t2, qg, nlog, stream, sq_part, ad,
                                     ticket, 3, fm, a, g2);
    if (e != cudaSuccess) return e;
  } else {
    cudaError_t e = launch_dense_x(A, n, q, lda, rs, svr, 2, t2, qg, stream);
    if (e != cudaSuccess) return e;
    const double* xs[1] = {a};
    const double* ys[1] = {qdir};
    e = launch_dots(1, xs, ys, fm, nlog, ad, red_ws, stream);
    if (e != cudaSuccess) return e;
    const double* gx[1] = {grad};
    const double* gy[1] = {nullptr};
    e = launch_dots(1, gx, gy, nullptr, nlog, g2, red_ws, stream);
    if (e != cudaSuccess) return e;
  }
  if (!(parts & 2)) return cudaGetLastError();
  return launch_hs_finish_dots(fm, a, qdir, nlog, -sigma, s, -1.0, dir, ad, asa_dev, grad, w, qw,
                               t2, q, dots4, red_ws, stream);
}

size_t direction_ws_bytes(long long n_phys, long long q) { return gradient_ws_bytes(n_phys, q); }

}  // namespace ssnal

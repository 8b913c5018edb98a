// CSR data operator (configs 2, 3): Q = X X^T with X = diag(y) A, A sparse n x q.
//
//   X d    : warp per row group -- each 8-lane sub-warp owns a row, lanes stride the
//            row's nonzeros (coalesced index/value loads), gather d[col] through the
//            read-only path, sub-warp shuffle tree.  Optional row list (X_J d).
//   X^T v  : on the CSC copy (built once per problem).  Columns are cut into
//            segments of <= SEG nonzeros (Zipf-hot columns span many segments), one
//            warp per segment; whole-column segments write the output directly,
//            split columns write partials folded in segment order.  Balanced and
//            deterministic: no atomics, fixed summation order.
//   scatter/gather helpers for the sample-space CG of the reduced Newton system.
#include <cstdlib>

#include "common.cuh"
#include "ssnal_internal.h"

#include <algorithm>
#include <cstdint>

namespace ssnal {

static constexpr int SUB = 8;  // lanes per row in X d

// out[r] = rs[i] * sum_k val[k] d[col[k]],  i = rows ? rows[r] : r  (r < nrows)
// Each lane sums entries sl, sl + SUB, sl + 2 SUB, ... of its row in order; the index /
// value loads of XD_UNROLL such entries are issued before their gathers (predicated),
// so a 30-50 nnz row is one or two rounds of independent loads instead of a chain.
static constexpr int XD_UNROLL = 4;
__global__ void __launch_bounds__(256) csr_xd_kernel(const int64_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ indices,
                                                     const double* __restrict__ values,
                                                     const double* __restrict__ rs,
                                                     const int32_t* __restrict__ rows, long long nrows,
                                                     const double* __restrict__ d,
                                                     double* __restrict__ out) {
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / SUB;
  const int sl = threadIdx.x & (SUB - 1);
  if (g >= nrows) return;
  const long long i = rows ? (long long)__ldg(rows + g) : g;
  const long long k0 = __ldg(indptr + i), k1 = __ldg(indptr + i + 1);
  double s = 0.0;
  for (long long kb = k0 + sl; kb < k1; kb += XD_UNROLL * SUB) {
    int idx[XD_UNROLL];
    double v[XD_UNROLL];
#pragma unroll
    for (int u = 0; u < XD_UNROLL; ++u) {
      const long long k = kb + u * SUB;
      const bool ok = k < k1;
      idx[u] = ok ? __ldg(indices + k) : 0;
      v[u] = ok ? __ldg(values + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < XD_UNROLL; ++u)
      if (kb + u * SUB < k1) s = fma(v[u], __ldg(d + idx[u]), s);
  }
#pragma unroll
  for (int o = SUB / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, SUB);
  if (sl == 0) out[g] = rs ? rs[i] * s : s;
}

// segment s covers CSC entries [seg_beg[s], seg_end[s]) of column seg_col[s];
// seg_slot[s] < 0: whole column (write out directly), else partial slot index.
__global__ void __launch_bounds__(256) csc_xt_kernel(const int64_t* __restrict__ seg_beg,
                                                     const int64_t* __restrict__ seg_end,
                                                     const int32_t* __restrict__ seg_col,
                                                     const int32_t* __restrict__ seg_slot,
                                                     long long nseg,
                                                     const int32_t* __restrict__ rowidx,
                                                     const double* __restrict__ valt,
                                                     const double* __restrict__ rs,
                                                     const double* __restrict__ v,
                                                     double* __restrict__ out,
                                                     double* __restrict__ part) {
  const long long s = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  const long long k0 = seg_beg[s], k1 = seg_end[s];
  double acc = 0.0;
  for (long long k = k0 + lane; k < k1; k += 32) {
    const int r = rowidx[k];
    const double cv = rs ? rs[r] * v[r] : v[r];
    acc = fma(valt[k], cv, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    const int slot = seg_slot[s];
    if (slot < 0) out[seg_col[s]] = acc;
    else part[slot] = acc;
  }
}

// masked column sums of squares on the same segment plan:
//   out[k] = sum_{i : keep[i]} A_ik^2  (the Jacobi diagonal of X_J^T X_J)
__global__ void __launch_bounds__(256) csc_colsq_kernel(const int64_t* __restrict__ seg_beg,
                                                        const int64_t* __restrict__ seg_end,
                                                        const int32_t* __restrict__ seg_col,
                                                        const int32_t* __restrict__ seg_slot,
                                                        long long nseg,
                                                        const int32_t* __restrict__ rowidx,
                                                        const double* __restrict__ valt,
                                                        const uint8_t* __restrict__ keep,
                                                        double* __restrict__ out,
                                                        double* __restrict__ part) {
  const long long s = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  const long long k0 = seg_beg[s], k1 = seg_end[s];
  double acc = 0.0;
  for (long long k = k0 + lane; k < k1; k += 32) {
    const double v = valt[k];
    if (keep[rowidx[k]]) acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    const int slot = seg_slot[s];
    if (slot < 0) out[seg_col[s]] = acc;
    else part[slot] = acc;
  }
}

// split columns: out[col] = sum of its partial slots [pbeg, pend), a warp per column
// (lanes stride the slots, fixed shuffle tree: deterministic).  Zipf-hot columns have
// up to ~2000 slots; a thread walking them serially sat on the critical path.
__global__ void csc_fold_kernel(const int32_t* __restrict__ fold_col,
                                const int32_t* __restrict__ fold_beg, long long nfold,
                                const double* __restrict__ part, double* __restrict__ out) {
  const long long f = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= nfold) return;
  double s = 0.0;
  for (int k = fold_beg[f] + lane; k < fold_beg[f + 1]; k += 32) s += part[k];
  s = warp_sum(s);
  if (lane == 0) out[fold_col[f]] = s;
}

// dst[i] = 0 for all i in [0, n) that are not overwritten later: zero fill
__global__ void fill_kernel(double* __restrict__ dst, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = v;
}

// dst[rows[r]] = src[r]  (r < p)
__global__ void scatter_kernel(const int32_t* __restrict__ rows, long long p,
                               const double* __restrict__ src, double* __restrict__ dst) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < p) dst[rows[r]] = src[r];
}

// dst[r] = src[rows[r]]
__global__ void gather_kernel(const int32_t* __restrict__ rows, long long p,
                              const double* __restrict__ src, double* __restrict__ dst) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < p) dst[r] = src[rows[r]];
}

// Gram of m selected sparse vectors (CSR rows or CSC columns, sorted indices):
//   G[r][c] = s_r s_c sum_{k in idx_r cap idx_c, keep[k]} val_r[k] val_c[k]
// one thread per (r, c >= r) pair merging the two sorted index lists (fixed order,
// deterministic), mirrored into the lower triangle.  Used for the direct reduced
// Newton systems of the sparse operator when min(p, q) is small (the p x p Q_JJ
// of ref solver.py:224-246, or the q x q X_J^T X_J factor-space Gram).
static constexpr int GT = 16;
__global__ void __launch_bounds__(GT * GT) sparse_gram_kernel(
    const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
    const double* __restrict__ val, const int32_t* __restrict__ sel, long long m,
    const uint8_t* __restrict__ keep, const double* __restrict__ sign, double* __restrict__ G) {
  const long long r = (long long)blockIdx.y * GT + threadIdx.y;
  const long long c = (long long)blockIdx.x * GT + threadIdx.x;
  if (blockIdx.x < blockIdx.y || r >= m || c >= m || c < r) return;
  const long long vr = sel ? (long long)sel[r] : r, vc = sel ? (long long)sel[c] : c;
  long long i = ptr[vr], j = ptr[vc];
  const long long ie = ptr[vr + 1], je = ptr[vc + 1];
  double s = 0.0;
  while (i < ie && j < je) {
    const int a = idx[i], b = idx[j];
    if (a == b) {
      if (!keep || keep[a]) s = fma(val[i], val[j], s);
      ++i;
      ++j;
    } else if (a < b) {
      ++i;
    } else {
      ++j;
    }
  }
  if (sign) s *= sign[vr] * sign[vc];
  G[r * m + c] = s;
  G[c * m + r] = s;
}

cudaError_t launch_sparse_gram_rows(const CsrOp& op, const int32_t* rows, long long p, double* G,
                                    cudaStream_t stream) {
  const unsigned nt = (unsigned)ceil_div(p, (long long)GT);
  note_launch();
  sparse_gram_kernel<<<dim3(nt, nt), dim3(GT, GT), 0, stream>>>(
      op.indptr, op.indices, op.values, rows, p, nullptr, op.row_sign, G);
  return cudaGetLastError();
}

// X_J^T X_J over the CSC columns keeping rows with free[row] != 0 (row signs square away)
cudaError_t launch_sparse_gram_cols(const CsrOp& op, const uint8_t* free_rows, double* G,
                                    cudaStream_t stream) {
  const unsigned nt = (unsigned)ceil_div(op.q, (long long)GT);
  note_launch();
  sparse_gram_kernel<<<dim3(nt, nt), dim3(GT, GT), 0, stream>>>(
      op.colptr, op.rowidx, op.valt, nullptr, op.q, free_rows, nullptr, G);
  return cudaGetLastError();
}

// M = I + sigma (G - u u^T / asa)  in place  (asa == 0: M = I + sigma G)
__global__ void qspace_assemble_kernel(long long m, const double* __restrict__ u, double asa,
                                       double sigma, double* __restrict__ G) {
  const double inv = asa != 0.0 ? 1.0 / asa : 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m * m;
       k += (long long)gridDim.x * blockDim.x) {
    const long long r = k / m, c = k % m;
    G[k] = (r == c ? 1.0 : 0.0) + sigma * (G[k] - inv * u[r] * u[c]);
  }
}

cudaError_t launch_qspace_assemble(long long m, const double* u, double asa, double sigma,
                                   double* G, cudaStream_t stream) {
  note_launch();
  qspace_assemble_kernel<<<(unsigned)min(ceil_div(m * m, 256LL), 4096LL), 256, 0, stream>>>(
      m, u, asa, sigma, G);
  return cudaGetLastError();
}

cudaError_t launch_csr_xd(const CsrOp& op, const int32_t* rows, long long nrows, const double* d,
                          double* out, cudaStream_t stream) {
  const long long threads = nrows * SUB;
  note_launch();
  csr_xd_kernel<<<(unsigned)ceil_div(threads, 256LL), 256, 0, stream>>>(
      op.indptr, op.indices, op.values, op.row_sign, rows, nrows, d, out);
  return cudaGetLastError();
}

cudaError_t launch_csc_xt(const CsrOp& op, const double* v, double* out, double* part,
                          cudaStream_t stream) {
  note_launch();
  csc_xt_kernel<<<(unsigned)ceil_div(op.nseg * 32, 256LL), 256, 0, stream>>>(
      op.seg_beg, op.seg_end, op.seg_col, op.seg_slot, op.nseg, op.rowidx, op.valt, op.row_sign,
      v, out, part);
  if (op.nfold > 0) {
    note_launch();
    csc_fold_kernel<<<(unsigned)ceil_div(op.nfold * 32, 256LL), 256, 0, stream>>>(
        op.fold_col, op.fold_beg, op.nfold, part, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_csc_colsq(const CsrOp& op, const uint8_t* keep, double* out, double* part,
                             cudaStream_t stream) {
  note_launch();
  csc_colsq_kernel<<<(unsigned)ceil_div(op.nseg * 32, 256LL), 256, 0, stream>>>(
      op.seg_beg, op.seg_end, op.seg_col, op.seg_slot, op.nseg, op.rowidx, op.valt, keep, out,
      part);
  if (op.nfold > 0) {
    note_launch();
    csc_fold_kernel<<<(unsigned)ceil_div(op.nfold * 32, 256LL), 256, 0, stream>>>(
        op.fold_col, op.fold_beg, op.nfold, part, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_fill(double* dst, long long n, double v, cudaStream_t stream) {
  note_launch();
  fill_kernel<<<(unsigned)min(ceil_div(n, 1024LL), 1184LL), 256, 0, stream>>>(dst, n, v);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const int32_t* rows, long long p, const double* src, double* dst,
                           cudaStream_t stream) {
  note_launch();
  scatter_kernel<<<(unsigned)ceil_div(p, 256LL), 256, 0, stream>>>(rows, p, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather(const int32_t* rows, long long p, const double* src, double* dst,
                          cudaStream_t stream) {
  note_launch();
  gather_kernel<<<(unsigned)ceil_div(p, 256LL), 256, 0, stream>>>(rows, p, src, dst);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- J-restricted CSC
// X_J^T w for the matrix-free reduced Newton systems: the CSC entries of the free
// rows J, built once per Newton step (one pass over the CSC) and reused by every CG
// iteration of that step, so a product reads nnz(X_J) instead of nnz(X) and gathers
// from the p-vector w (row slot = position in J) instead of a scattered n-vector.
// Segments keep the operator's plan (same columns, same fold slots, entries in CSC
// order), so the product stays deterministic.  Row signs are folded into the values.
static constexpr int CJ_WARPS = 8;  // segments per block

__device__ __forceinline__ long long block_exclusive_scan_ll(long long v, long long* sm,
                                                             long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const long long x = lane < nw ? sm[lane] : 0;
    long long xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < nw) sm[lane] = xi - x;
    if (lane == nw - 1) sm[32] = xi;
  }
  __syncthreads();
  const long long r = sm[warp] + incl - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

// pass 1: kept entries per segment (warp per segment) and per block; the last block
// turns the block counts into exclusive offsets
__global__ void __launch_bounds__(CJ_WARPS * 32) cscj_count_kernel(
    const int64_t* __restrict__ seg_beg, const int64_t* __restrict__ seg_end, long long nseg,
    const int32_t* __restrict__ rowidx, const uint8_t* __restrict__ keep, int* __restrict__ cnt,
    long long* __restrict__ blk, unsigned int* ticket, int nblk, int32_t* __restrict__ empty,
    unsigned int* nempty) {
  __shared__ long long sm[33];
  __shared__ int wc[CJ_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long s = (long long)blockIdx.x * CJ_WARPS + warp;
  int c = 0;
  if (s < nseg) {
    for (long long k = seg_beg[s] + lane; k < seg_end[s]; k += 32) c += keep[rowidx[k]] ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
      cnt[s] = c;
      if (c == 0) empty[atomicAdd(nempty, 1u)] = (int32_t)s;  // order irrelevant: zero writes
    }
  }
  if (lane == 0) wc[warp] = s < nseg ? c : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < CJ_WARPS; ++w) t += wc[w];
    blk[blockIdx.x] = t;
  }
  if (!last_block_arrive(ticket, gridDim.x)) return;
  long long carry = 0;
  for (int start = 0; start < nblk; start += blockDim.x) {
    const int idx = start + threadIdx.x;
    const long long v = idx < nblk ? __ldcg(blk + idx) : 0;
    long long tot;
    const long long ex = block_exclusive_scan_ll(v, sm, &tot);
    if (idx < nblk) blk[idx] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) blk[nblk] = carry;
}

// pass 2: compact the kept entries of each segment (ballot + popc keeps CSC order)
__global__ void __launch_bounds__(CJ_WARPS * 32) cscj_fill_kernel(
    const int64_t* __restrict__ seg_beg, const int64_t* __restrict__ seg_end, long long nseg,
    const int32_t* __restrict__ rowidx, const double* __restrict__ valt,
    const double* __restrict__ rs, const uint8_t* __restrict__ keep,
    const int32_t* __restrict__ posJ, const int* __restrict__ cnt,
    const long long* __restrict__ blk, int64_t* __restrict__ jbeg, int64_t* __restrict__ jend,
    int32_t* __restrict__ jpos, double* __restrict__ jval, int32_t* __restrict__ jseg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long s = (long long)blockIdx.x * CJ_WARPS + warp;
  if (s >= nseg) return;
  long long off = blk[blockIdx.x];
  for (int w = 0; w < warp; ++w) off += cnt[(long long)blockIdx.x * CJ_WARPS + w];
  if (lane == 0) {
    jbeg[s] = off;
    jend[s] = off + cnt[s];
  }
  const long long k1 = seg_end[s];
  for (long long k0 = seg_beg[s]; k0 < k1; k0 += 32) {
    const long long k = k0 + lane;
    int r = 0;
    bool kp = false;
    if (k < k1) {
      r = rowidx[k];
      kp = keep[r] != 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, kp);
    if (kp) {
      const long long o = off + __popc(bal & ((1u << lane) - 1u));
      jpos[o] = posJ[r];
      jval[o] = rs ? valt[k] * rs[r] : valt[k];
      jseg[o] = (int32_t)s;
    }
    off += __popc(bal);
  }
}

// pos[J[r]] = r
__global__ void index_map_kernel(const int32_t* __restrict__ J, long long p,
                                 int32_t* __restrict__ pos) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < p) pos[J[r]] = (int32_t)r;
}

// out = X_J^T w on the J-restricted CSC (w indexed by position in J), nnz-balanced:
// the kept entries are cut into CH-entry chunks, one warp per chunk, CH_E consecutive
// entries per lane.  Each lane runs a sequential segmented sum over its entries
// (segment ids from cscj_fill), the lanes' open partials are joined by a warp
// segmented scan, and a segment that crosses a chunk boundary leaves its chunk
// partials in cval / ctail for cscj_fix_kernel, which adds them in chunk order.
// Zipf data leave most of the ~1e6 column segments with 0-3 kept entries, where a
// warp per segment ran at ~1/10 of the HBM rate; here every lane streams CH_E entries.
// Fixed chunking => fixed summation order: deterministic run to run.
static constexpr int CH_E = 4;           // smallest entries-per-lane instantiation:
static constexpr int CH = 32 * CH_E;     // sizes the per-chunk workspace arrays

__device__ __forceinline__ void seg_write(int s, double v, const int32_t* __restrict__ seg_col,
                                          const int32_t* __restrict__ seg_slot,
                                          double* __restrict__ out, double* __restrict__ part) {
  const int slot = seg_slot[s];
  if (slot < 0) out[seg_col[s]] = v;
  else part[slot] = v;
}

// TR (CHE = 8): the chunk is loaded INTERLEAVED (lane l takes entries 32 u + l: every index /
// value load is one fully coalesced 128/256-byte request, and the 32 gathers of one
// instruction are 32 consecutive CSC entries -- ascending row slots of one column, so a
// column present in a fraction f of the J rows touches ~2/f lines instead of 16/f), then
// transposed through shared memory (index i stored at i + i/8: conflict-free both ways)
// into the 8-consecutive-entries-per-lane layout of the segmented sum below.  The kernel
// is bound by L1 tag lookups (one per distinct 128-byte line per gather instruction).
template <int CHE, bool TR>
__global__ void __launch_bounds__(256, CHE <= 8 ? 4 : 1) cscj_xt_kernel(
    const long long* __restrict__ total, const int32_t* __restrict__ jseg,
    const int32_t* __restrict__ jpos, const double* __restrict__ jval,
    const int32_t* __restrict__ seg_col, const int32_t* __restrict__ seg_slot,
    const double* __restrict__ w, double* __restrict__ out, double* __restrict__ part,
    double* __restrict__ cval, double* __restrict__ ctail, uint8_t* __restrict__ cflag) {
  const long long nnz = *total;
  const long long nch = (nnz + (32 * CHE) - 1) / (32 * CHE);
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr int NONE = 0x7fffffff;
  for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nch; c += nw) {
    const long long c0 = c * (32 * CHE), e0 = c0 + lane * CHE;
    // the chunk's first segment F continues from the previous chunk?
    const int F = jseg[c0];
    const bool chunk_in = c0 > 0 && jseg[c0 - 1] == F;
    const int next = c0 + (32 * CHE) < nnz ? jseg[c0 + (32 * CHE)] : NONE;
    int sg[CHE];
    double pr[CHE];
    {
      double wg[CHE];
      if constexpr (TR) {
        static_assert(!TR || CHE == 8, "transposed load is written for 8 entries per lane");
        __shared__ int t_seg[8][288];
        __shared__ double t_val[8][288], t_w[8][288];
        const int wp = threadIdx.x >> 5;
        int ps[CHE];
#pragma unroll
        for (int u = 0; u < CHE; ++u) {
          const long long e = c0 + 32 * u + lane;
          const bool ok = e < nnz;
          sg[u] = ok ? __ldg(jseg + e) : NONE;
          ps[u] = ok ? __ldg(jpos + e) : 0;
          pr[u] = ok ? __ldg(jval + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CHE; ++u) wg[u] = sg[u] != NONE ? __ldg(w + ps[u]) : 0.0;
        __syncwarp();  // the previous chunk's reads of this warp's tile are done
#pragma unroll
        for (int u = 0; u < CHE; ++u) {
          const int i = 32 * u + lane, ip = i + (i >> 3);
          t_seg[wp][ip] = sg[u];
          t_val[wp][ip] = pr[u];
          t_w[wp][ip] = wg[u];
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < CHE; ++u) {
          const int ip = 9 * lane + u;  // (8 lane + u) + lane
          sg[u] = t_seg[wp][ip];
          pr[u] = t_val[wp][ip];
          wg[u] = t_w[wp][ip];
        }
      } else {
        const int4* s4 = reinterpret_cast<const int4*>(jseg + e0);
        const int4* p4 = reinterpret_cast<const int4*>(jpos + e0);
        const double2* v2 = reinterpret_cast<const double2*>(jval + e0);
        int ps[CHE];
        double vv[CHE];
#pragma unroll
        for (int h = 0; h < CHE / 4; ++h) {
          const int4 a = __ldg(s4 + h), b = __ldg(p4 + h);
          sg[4 * h] = a.x; sg[4 * h + 1] = a.y; sg[4 * h + 2] = a.z; sg[4 * h + 3] = a.w;
          ps[4 * h] = b.x; ps[4 * h + 1] = b.y; ps[4 * h + 2] = b.z; ps[4 * h + 3] = b.w;
        }
#pragma unroll
        for (int h = 0; h < CHE / 2; ++h) {
          const double2 v = __ldg(v2 + h);
          vv[2 * h] = v.x; vv[2 * h + 1] = v.y;
        }
        // gathers of w after all index loads are in flight
#pragma unroll
        for (int u = 0; u < CHE; ++u) {
          const bool ok = e0 + u < nnz;
          if (!ok) sg[u] = NONE;
          pr[u] = ok ? vv[u] : 0.0;
          wg[u] = ok ? __ldg(w + ps[u]) : 0.0;
        }
      }
      // sequential segmented sums over the lane's entries
      const int head = sg[0];
      int cur = sg[0];
      double run = 0.0, hsum = 0.0;
      bool single = true;
#pragma unroll
      for (int u = 0; u < CHE; ++u) {
        if (sg[u] != cur) {
          if (single) {
            hsum = run;
            single = false;
          } else if (cur != NONE) {
            seg_write(cur, run, seg_col, seg_slot, out, part);  // started and ended in lane
          }
          cur = sg[u];
          run = 0.0;
        }
        run = fma(pr[u], wg[u], run);
      }
      // warp segmented inclusive scan of the open tails (cur, run)
      const int prevK = __shfl_up_sync(0xffffffffu, cur, 1);
      bool reset = lane == 0 || !single || prevK != cur;
      double S = run;
      {
        bool r = reset;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double vs = __shfl_up_sync(0xffffffffu, S, o);
          const bool rs_ = __shfl_up_sync(0xffffffffu, r, o);
          if (lane >= o && !r) {
            S += vs;
            r = rs_;
          }
        }
      }
      const double prevS = __shfl_up_sync(0xffffffffu, S, 1);
      const int nextHead = __shfl_down_sync(0xffffffffu, head, 1);
      bool wrote_close = false;
      // (a) a head segment that closes inside this lane (lane holds >= 2 segments)
      if (!single && head != NONE) {
        const double tot = (lane > 0 && prevK == head) ? prevS + hsum : hsum;
        if (chunk_in && head == F) {
          cval[c] = tot;
          wrote_close = true;
        } else {
          seg_write(head, tot, seg_col, seg_slot, out, part);
        }
      }
      // (b) the lane's tail segment: closes at the lane end unless the next lane (or the
      // next chunk) continues it
      bool owns_tail = false;
      if (cur != NONE) {
        const bool cont = lane < 31 ? (nextHead == cur) : (next == cur);
        if (!cont) {
          if (chunk_in && cur == F) {
            cval[c] = S;
            wrote_close = true;
          } else {
            seg_write(cur, S, seg_col, seg_slot, out, part);
          }
        } else if (lane == 31) {
          if (chunk_in && cur == F) {
            cval[c] = S;  // F spans the whole chunk and continues
          } else {
            ctail[c] = S;
            owns_tail = true;
          }
        }
      }
      const unsigned cl = __ballot_sync(0xffffffffu, wrote_close);
      const unsigned ot = __ballot_sync(0xffffffffu, owns_tail);
      if (lane == 0) cflag[c] = (uint8_t)((cl ? 1 : 0) | (ot ? 2 : 0));
    }
  }
}

// segments that cross chunk boundaries: tail partial + the following chunks' first-
// segment partials, in chunk order, up to the chunk where the segment closes
template <int CHE>
__global__ void __launch_bounds__(256) cscj_fix_kernel(
    const long long* __restrict__ total, const int32_t* __restrict__ jseg,
    const int32_t* __restrict__ seg_col, const int32_t* __restrict__ seg_slot,
    const double* __restrict__ cval, const double* __restrict__ ctail,
    const uint8_t* __restrict__ cflag, double* __restrict__ out, double* __restrict__ part,
    const int32_t* __restrict__ empty, const unsigned int* __restrict__ nempty) {
  const long long nnz = *total;
  const long long nch = (nnz + (32 * CHE) - 1) / (32 * CHE);
  const long long ne = *nempty;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (long long)gridDim.x * blockDim.x)
    seg_write(empty[e], 0.0, seg_col, seg_slot, out, part);
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nch;
       c += (long long)gridDim.x * blockDim.x) {
    if (!(cflag[c] & 2)) continue;
    double t = ctail[c];
    for (long long d = c + 1; d < nch; ++d) {
      t += cval[d];
      if (cflag[d] & 1) break;
    }
    seg_write(jseg[c * (32 * CHE) + (32 * CHE) - 1], t, seg_col, seg_slot, out, part);
  }
}

// J-restricted CSR (once per Newton step of the CG route): row lengths of J's rows,
// block sums + last-block exclusive scan, then per block the row offsets and a warp per
// row copying (index, sign * value).  The CG's X_J d then reads p contiguous rows.
static constexpr int RJ_NT = 256;
__global__ void __launch_bounds__(RJ_NT) csrj_count_kernel(const int64_t* __restrict__ indptr,
                                                           const int32_t* __restrict__ J,
                                                           long long p, long long* __restrict__ rblk,
                                                           unsigned int* ticket, int nblk) {
  __shared__ long long sm[33];
  const long long r = (long long)blockIdx.x * RJ_NT + threadIdx.x;
  long long len = 0;
  if (r < p) {
    const int i = J[r];
    len = indptr[i + 1] - indptr[i];
  }
  long long tot;
  block_exclusive_scan_ll(len, sm, &tot);
  if (threadIdx.x == 0) rblk[blockIdx.x] = tot;
  if (!last_block_arrive(ticket, gridDim.x)) return;
  long long carry = 0;
  for (int start = 0; start < nblk; start += RJ_NT) {
    const int idx = start + threadIdx.x;
    const long long v = idx < nblk ? __ldcg(rblk + idx) : 0;
    long long t;
    const long long ex = block_exclusive_scan_ll(v, sm, &t);
    if (idx < nblk) rblk[idx] = carry + ex;
    carry += t;
  }
  if (threadIdx.x == 0) rblk[nblk] = carry;
}

__global__ void __launch_bounds__(RJ_NT) csrj_fill_kernel(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
    const double* __restrict__ values, const double* __restrict__ rs,
    const int32_t* __restrict__ J, long long p, const long long* __restrict__ rblk, int nblk,
    const int32_t* __restrict__ hot_rank, int64_t* __restrict__ rptr, int32_t* __restrict__ ridx,
    double* __restrict__ rval) {
  __shared__ long long sm[33];
  __shared__ long long off[RJ_NT];
  const long long r0 = (long long)blockIdx.x * RJ_NT;
  const long long r = r0 + threadIdx.x;
  long long len = 0;
  if (r < p) {
    const int i = J[r];
    len = indptr[i + 1] - indptr[i];
  }
  long long tot;
  const long long ex = block_exclusive_scan_ll(len, sm, &tot);
  off[threadIdx.x] = rblk[blockIdx.x] + ex;
  if (r < p) rptr[r] = off[threadIdx.x];
  if (blockIdx.x == nblk - 1 && threadIdx.x == 0) rptr[p] = rblk[nblk];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = warp; t < RJ_NT && r0 + t < p; t += RJ_NT / 32) {
    const int i = J[r0 + t];
    const long long k0 = indptr[i], k1 = indptr[i + 1], o = off[t];
    const double sg = rs ? rs[i] : 1.0;
    for (long long k = k0 + lane; k < k1; k += 32) {
      // hot columns (operator's popularity table) are stored as ~rank < 0: the product
      // reads their d entries from its shared-memory copy
      const int32_t col = indices[k];
      const int32_t hr = hot_rank ? __ldg(hot_rank + col) : -1;
      ridx[o + (k - k0)] = hr >= 0 ? ~hr : col;
      rval[o + (k - k0)] = sg * values[k];
    }
  }
}

// X_J d on the packed rows with the CG's a_J . (X_J d) folded in (replaces a dots
// launch per CG iteration): grid-stride over 32-row groups on a fixed grid, per-block
// partial, last-block fold in block order (deterministic)
__global__ void __launch_bounds__(256) csrj_xd_dot_kernel(
    const int64_t* __restrict__ rptr, const int32_t* __restrict__ ridx,
    const double* __restrict__ rval, long long p, const double* __restrict__ d,
    double* __restrict__ out, const double* __restrict__ wdot, double* dot_out,
    double* __restrict__ part, unsigned int* ticket) {
  __shared__ double red[32];
  const int sl = threadIdx.x & (SUB - 1);
  double acc[1] = {0.0};
  // warp-uniform trip count: every lane reaches every full-mask shuffle (a sub-warp past
  // the last row runs an empty row instead of leaving the loop)
  const long long wstride = (long long)gridDim.x * blockDim.x / SUB;
  for (long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / SUB; g0 < p;
       g0 += wstride) {
    const long long g = g0 + ((threadIdx.x & 31) / SUB);
    const bool valid = g < p;
    const long long k0 = valid ? __ldg(rptr + g) : 0, k1 = valid ? __ldg(rptr + g + 1) : 0;
    double s = 0.0;
    for (long long kb = k0 + sl; kb < k1; kb += XD_UNROLL * SUB) {
      int idx[XD_UNROLL];
      double v[XD_UNROLL];
#pragma unroll
      for (int u = 0; u < XD_UNROLL; ++u) {
        const long long k = kb + u * SUB;
        const bool ok = k < k1;
        idx[u] = ok ? __ldg(ridx + k) : 0;
        v[u] = ok ? __ldg(rval + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < XD_UNROLL; ++u)
        if (kb + u * SUB < k1) s = fma(v[u], __ldg(d + idx[u]), s);
    }
#pragma unroll
    for (int o = SUB / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, SUB);
    if (sl == 0 && valid) {
      out[g] = s;
      acc[0] = fma(wdot[g], s, acc[0]);
    }
  }
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(ticket, gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) *dot_out = acc[0];
}

// The same product with shared-memory staging of the d entries of the operator's hot
// columns (Zipf popularity: the 4096 most populated columns hold ~2/3 of the entries):
// each 512-thread CTA (two per SM) copies d[hot_cols[0..nhot)] into shared memory once and then
// grid-strides over the packed rows, whose hot entries carry ~rank instead of the
// column.  The plain kernel is bound by L1/TEX gather wavefronts (one per scattered
// 8-byte load, 96 % L1 throughput at 0.50 of HBM); shared-memory lookups take the hot
// share off that path.  Per-row summation order is the plain kernel's: bit-identical out.
static constexpr int HOT_NT = 512;
__global__ void __launch_bounds__(HOT_NT, 2) csrj_xd_dot_hot_kernel(
    const int64_t* __restrict__ rptr, const int32_t* __restrict__ ridx,
    const double* __restrict__ rval, long long p, const double* __restrict__ d,
    const int32_t* __restrict__ hot_cols, int nhot, double* __restrict__ out,
    const double* __restrict__ wdot, double* dot_out, double* __restrict__ part,
    unsigned int* ticket) {
  extern __shared__ double hot[];
  __shared__ double red[32];
  for (int k = threadIdx.x; k < nhot; k += HOT_NT) hot[k] = __ldg(d + __ldg(hot_cols + k));
  __syncthreads();
  const int sl = threadIdx.x & (SUB - 1), sub = (threadIdx.x & 31) / SUB;
  double acc[1] = {0.0};
  const long long wstride = (long long)gridDim.x * blockDim.x / SUB;
  // Software pipeline over the warp's row groups (the chain row pointer -> entries ->
  // gather is three dependent loads): iteration i gathers for group i while the entry
  // loads of group i+1 and the row pointers of group i+2 are in flight.
  auto ptrs = [&](long long g0, long long& a, long long& b) {
    const long long g = g0 + sub;
    const bool ok = g < p;
    a = ok ? __ldg(rptr + g) : 0;
    b = ok ? __ldg(rptr + g + 1) : 0;
  };
  auto ents = [&](long long a, long long b, int (&ix)[XD_UNROLL], double (&vv)[XD_UNROLL]) {
#pragma unroll
    for (int u = 0; u < XD_UNROLL; ++u) {
      const long long k = a + sl + u * SUB;
      const bool ok = k < b;
      ix[u] = ok ? __ldg(ridx + k) : 0;
      vv[u] = ok ? __ldg(rval + k) : 0.0;
    }
  };
  long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / SUB;
  long long k0, k1, nk0, nk1;
  int idx[XD_UNROLL];
  double v[XD_UNROLL];
  ptrs(g0, k0, k1);
  ents(k0, k1, idx, v);
  ptrs(g0 + wstride, nk0, nk1);
  for (; g0 < p; g0 += wstride) {
    int nidx[XD_UNROLL];
    double nv[XD_UNROLL];
    long long nnk0, nnk1;
    ents(nk0, nk1, nidx, nv);
    ptrs(g0 + 2 * wstride, nnk0, nnk1);
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < XD_UNROLL; ++u)
      if (k0 + sl + u * SUB < k1) s = fma(v[u], idx[u] < 0 ? hot[~idx[u]] : __ldg(d + idx[u]), s);
    // rows longer than one round (XD_UNROLL * SUB entries): the plain loop
    for (long long kb = k0 + sl + XD_UNROLL * SUB; kb < k1; kb += XD_UNROLL * SUB) {
      int ix[XD_UNROLL];
      double vv[XD_UNROLL];
      ents(kb - sl, k1, ix, vv);
#pragma unroll
      for (int u = 0; u < XD_UNROLL; ++u)
        if (kb + u * SUB < k1) s = fma(vv[u], ix[u] < 0 ? hot[~ix[u]] : __ldg(d + ix[u]), s);
    }
#pragma unroll
    for (int o = SUB / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, SUB);
    const long long g = g0 + sub;
    if (sl == 0 && g < p) {
      out[g] = s;
      if (wdot) acc[0] = fma(wdot[g], s, acc[0]);
    }
#pragma unroll
    for (int u = 0; u < XD_UNROLL; ++u) {
      idx[u] = nidx[u];
      v[u] = nv[u];
    }
    k0 = nk0; k1 = nk1; nk0 = nnk0; nk1 = nnk1;
  }
  if (!wdot) return;
  const int ops[1] = {0};
  block_reduce<1>(acc, ops, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (!last_block_arrive(ticket, gridDim.x)) return;
  block_fold_partials<1>(part, gridDim.x, 1, ops, acc, red);
  if (threadIdx.x == 0) *dot_out = acc[0];
}

static int hot_grid(long long p, int max_blocks) {
  static DeviceCache cache;
  const int sms = per_device(cache, [](int dev) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(csrj_xd_dot_hot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(SSNAL_CSR_HOT_MAX * sizeof(double)));
    return n;
  });
  return (int)std::max(1LL, std::min({ceil_div(p * SUB, (long long)HOT_NT), 2LL * sms,
                                      (long long)max_blocks}));
}

cudaError_t launch_csrj_xd_dot(const CscJ& c, long long p, const double* d, double* out,
                               const double* wdot, double* dot_out, double* part,
                               int max_blocks, unsigned int* ticket, cudaStream_t stream) {
  if (p < 1) return cudaMemsetAsync(dot_out, 0, sizeof(double), stream);
  note_launch();
  if (c.nhot > 0) {
    csrj_xd_dot_hot_kernel<<<hot_grid(p, max_blocks), HOT_NT, c.nhot * sizeof(double), stream>>>(
        c.rptr, c.ridx, c.rval, p, d, c.hot_cols, c.nhot, out, wdot, dot_out, part, ticket);
    return cudaGetLastError();
  }
  // one resident wave (8 CTAs of 256 threads per SM at 32 registers), grid-stride over the
  // rows: a grid capped only by the partial buffer (2720 CTAs = 2.3 waves on 148 SMs) left
  // the last wave 30 % full (115 us against 81 us for the same rows without the dot)
  static DeviceCache wave_cache;
  const int wave = per_device(wave_cache, [](int dev) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 8 * sms;
  });
  const int grid = (int)std::max(1LL, std::min({ceil_div(p * SUB, 256LL), (long long)max_blocks,
                                                (long long)wave}));
  csrj_xd_dot_kernel<<<grid, 256, 0, stream>>>(c.rptr, c.ridx, c.rval, p, d, out, wdot, dot_out,
                                                part, ticket);
  return cudaGetLastError();
}

cudaError_t launch_csrj_xd(const CscJ& c, long long p, const double* d, double* out,
                           cudaStream_t stream) {
  if (p < 1) return cudaSuccess;
  note_launch();
  if (c.nhot > 0) {
    csrj_xd_dot_hot_kernel<<<hot_grid(p, 1 << 30), HOT_NT, c.nhot * sizeof(double), stream>>>(
        c.rptr, c.ridx, c.rval, p, d, c.hot_cols, c.nhot, out, nullptr, nullptr, nullptr, nullptr);
    return cudaGetLastError();
  }
  csr_xd_kernel<<<(unsigned)ceil_div(p * SUB, 256LL), 256, 0, stream>>>(
      c.rptr, c.ridx, c.rval, nullptr, nullptr, p, d, out);
  return cudaGetLastError();
}

size_t cscj_ws_bytes(const CsrOp& op) {
  const long long nblk = ceil_div(op.nseg, (long long)CJ_WARPS);
  const long long cap = op.nnz + 32 * 32;  // vector loads of the last chunk (CHE <= 32) stay inside
  const long long nch = ceil_div(cap, (long long)CH);
  const long long rb = ceil_div(op.n, (long long)RJ_NT) + 1;
  return 256 + sizeof(int32_t) * (size_t)op.n + sizeof(int) * (size_t)op.nseg +
         sizeof(long long) * (size_t)(nblk + 1) + 2 * sizeof(int64_t) * (size_t)op.nseg +
         (2 * sizeof(int32_t) + sizeof(double)) * (size_t)cap + (2 * sizeof(double) + 1) * nch +
         sizeof(int64_t) * (size_t)(op.n + 1) + (sizeof(int32_t) + sizeof(double)) * (size_t)op.nnz +
         sizeof(long long) * (size_t)rb + sizeof(int32_t) * (size_t)op.nseg + 18 * 256;
}

static char* al256(char* p) { return (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255); }

CscJ cscj_layout(const CsrOp& op, void* ws) {
  const long long nblk = ceil_div(op.nseg, (long long)CJ_WARPS);
  const long long cap = op.nnz + 32 * 32;
  const long long nch = ceil_div(cap, (long long)CH);
  CscJ c;
  char* p = al256((char*)ws);
  c.ticket = (unsigned int*)p; p = al256(p + 256);
  c.posJ = (int32_t*)p; p = al256(p + sizeof(int32_t) * op.n);
  c.cnt = (int*)p; p = al256(p + sizeof(int) * op.nseg);
  c.blk = (long long*)p; p = al256(p + sizeof(long long) * (nblk + 1));
  c.beg = (int64_t*)p; p = al256(p + sizeof(int64_t) * op.nseg);
  c.end = (int64_t*)p; p = al256(p + sizeof(int64_t) * op.nseg);
  c.pos = (int32_t*)p; p = al256(p + sizeof(int32_t) * cap);
  c.seg = (int32_t*)p; p = al256(p + sizeof(int32_t) * cap);
  c.val = (double*)p; p = al256(p + sizeof(double) * cap);
  c.cval = (double*)p; p = al256(p + sizeof(double) * nch);
  c.ctail = (double*)p; p = al256(p + sizeof(double) * nch);
  c.cflag = (uint8_t*)p; p = al256(p + nch);
  c.rptr = (int64_t*)p; p = al256(p + sizeof(int64_t) * (op.n + 1));
  c.ridx = (int32_t*)p; p = al256(p + sizeof(int32_t) * op.nnz);
  c.rval = (double*)p; p = al256(p + sizeof(double) * op.nnz);
  c.rblk = (long long*)p; p = al256(p + sizeof(long long) * (ceil_div(op.n, (long long)RJ_NT) + 1));
  c.empty = (int32_t*)p; p = al256(p + sizeof(int32_t) * op.nseg);
  c.nempty = (unsigned int*)p;
  // measured on config-3 data (|J| = 700k, 69 % of the entries in the 4096 hot columns):
  // 84 us against 81 us for the plain gather kernel -- random 8-byte shared-memory
  // lookups still cost ~5 bank-conflict wavefronts each and the longer kernel runs at
  // lower occupancy, so the staging is off unless SSNAL_CSR_HOT=1 (study knob)
  static const bool hot_on = std::getenv("SSNAL_CSR_HOT") && std::atoi(std::getenv("SSNAL_CSR_HOT")) != 0;
  c.nhot = (hot_on && op.hot_cols && op.hot_rank && op.nhot > 0 && op.nhot <= SSNAL_CSR_HOT_MAX)
               ? (int)op.nhot : 0;
  c.hot_cols = op.hot_cols;
  return c;
}

cudaError_t launch_cscj_build(const CsrOp& op, const uint8_t* keep, const int32_t* J, long long p,
                              const CscJ& c, cudaStream_t stream) {
  const long long nblk = ceil_div(op.nseg, (long long)CJ_WARPS);
  cudaError_t e0 = cudaMemsetAsync(c.nempty, 0, sizeof(unsigned int), stream);
  if (e0 != cudaSuccess) return e0;
  note_launch();
  index_map_kernel<<<(unsigned)ceil_div(std::max(p, 1LL), 256LL), 256, 0, stream>>>(J, p, c.posJ);
  note_launch();
  cscj_count_kernel<<<(unsigned)nblk, CJ_WARPS * 32, 0, stream>>>(
      op.seg_beg, op.seg_end, op.nseg, op.rowidx, keep, c.cnt, c.blk, c.ticket, (int)nblk,
      c.empty, c.nempty);
  note_launch();
  cscj_fill_kernel<<<(unsigned)nblk, CJ_WARPS * 32, 0, stream>>>(
      op.seg_beg, op.seg_end, op.nseg, op.rowidx, op.valt, op.row_sign, keep, c.posJ, c.cnt,
      c.blk, c.beg, c.end, c.pos, c.val, c.seg);
  if (p > 0) {
    const int rb = (int)ceil_div(p, (long long)RJ_NT);
    note_launch();
    csrj_count_kernel<<<rb, RJ_NT, 0, stream>>>(op.indptr, J, p, c.rblk, c.ticket, rb);
    note_launch();
    csrj_fill_kernel<<<rb, RJ_NT, 0, stream>>>(op.indptr, op.indices, op.values, op.row_sign, J,
                                               p, c.rblk, rb, c.nhot > 0 ? op.hot_rank : nullptr,
                                               c.rptr, c.ridx, c.rval);
  }
  return cudaGetLastError();
}

template <int CHE, bool TR = false>
static void launch_cscj_xt_che(const CsrOp& op, const CscJ& c, const double* w, double* out,
                               double* part, cudaStream_t stream) {
  const long long nblk = ceil_div(op.nseg, (long long)CJ_WARPS);
  const long long* total = c.blk + nblk;  // kept entries (cscj_count_kernel)
  // segments without kept entries are never visited by the chunks: the fix kernel
  // writes their zeros from the build's list
  const long long nch_max = ceil_div(op.nnz, (long long)(32 * CHE));
  const unsigned grid = (unsigned)std::max(1LL, std::min(ceil_div(nch_max, 8LL), 148LL * 8));
  note_launch();
  cscj_xt_kernel<CHE, TR><<<grid, 256, 0, stream>>>(total, c.seg, c.pos, c.val, op.seg_col,
                                                 op.seg_slot, w, out, part, c.cval, c.ctail,
                                                 c.cflag);
  note_launch();
  cscj_fix_kernel<CHE><<<(unsigned)std::max(1LL, std::min(ceil_div(std::max(nch_max, (long long)op.nseg), 256LL),
                                                           148LL * 4)), 256,
                         0, stream>>>(total, c.seg, op.seg_col, op.seg_slot, c.cval, c.ctail, c.cflag,
                                      out, part, c.empty, c.nempty);
}

cudaError_t launch_cscj_xt(const CsrOp& op, const CscJ& c, const double* w, double* out,
                           double* part, cudaStream_t stream) {
  // entries per lane of the nnz-balanced product (SSNAL_CSCJ_CHE = 4 | 8 | 16 | 32; the
  // workspace is sized for the smallest chunk, larger chunks fit)
  static const int che = std::getenv("SSNAL_CSCJ_CHE") ? std::atoi(std::getenv("SSNAL_CSCJ_CHE")) : 8;
  // measured slower than the per-lane vector loads (175 vs 120 us, config-3 data): study knob
  static const bool tr = std::getenv("SSNAL_CSCJ_T") && std::atoi(std::getenv("SSNAL_CSCJ_T")) != 0;
  if (che == 8 && tr) launch_cscj_xt_che<8, true>(op, c, w, out, part, stream);
  else if (che == 32) launch_cscj_xt_che<32>(op, c, w, out, part, stream);
  else if (che == 16) launch_cscj_xt_che<16>(op, c, w, out, part, stream);
  else if (che == 4) launch_cscj_xt_che<4>(op, c, w, out, part, stream);
  else launch_cscj_xt_che<8>(op, c, w, out, part, stream);
  if (op.nfold > 0) {
    note_launch();
    csc_fold_kernel<<<(unsigned)ceil_div(op.nfold * 32, 256LL), 256, 0, stream>>>(
        op.fold_col, op.fold_beg, op.nfold, part, out);
  }
  return cudaGetLastError();
}

}  // namespace ssnal

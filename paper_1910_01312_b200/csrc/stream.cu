// TMA-staged streaming of the sample matrix A for the two data-operator products.
//
// Every product of the SSsNAL step that touches A (X^T v for the gradient and the
// KKT map, X d for Q-images) reads A exactly once, so it is HBM bound.  One CTA
// per SM owns a contiguous slab of rows; a producer warp streams the slab into a
// 4-stage shared-memory ring with 1-D bulk copies (cp.async.bulk, TMA engine,
// mbarrier complete_tx), eight consumer warps compute from shared memory and
// release stages through "empty" mbarriers.  192 KB in flight per SM keeps HBM
// saturated without relying on occupancy.
//   XT : consumers own column pairs, accumulate coef_r * A[r, :] in registers;
//        per-CTA partials are folded deterministically afterwards.
//   XD : each consumer warp takes whole rows of a stage, d is held in registers,
//        shuffle-tree dot products.
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "ssnal_internal.h"

#include <cstdlib>

namespace ssnal {

namespace {

#ifndef SSNAL_NSTAGE
#define SSNAL_NSTAGE 4
#define SSNAL_STAGE_KB 48
#endif
constexpr int NSTAGE = SSNAL_NSTAGE;
constexpr int STAGE_BYTES = SSNAL_STAGE_KB * 1024;
constexpr int NCONS = 8;                      // consumer warps
constexpr int NTHREADS = (NCONS + 1) * 32;    // + one producer warp
constexpr int ROWS_CTA = 512;
constexpr int XD_WARPS1 = 8;                  // X d consumer warps, one right-hand side
constexpr int XD_WARPS2 = 8;                  // ... two right-hand sides (16: -7 % on config 1)                 // rows per CTA slab (coefficients fit in smem)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait suspends in hardware between probes; the bounded loop turns a protocol
// bug into a trapped kernel (an error the host sees) instead of a hung GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (long long spin = 0; spin < (1LL << 26); ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct StreamArgs {
  const double* A;
  long long n, q, lda;
  const double* rs;
  int svr;
  int rows_per_stage;
  // XT
  const double* v[2];
  int k;
  double* part;  // [grid][k][q]
  // XD
  const double* d;  // [k][q]
  double* out;      // [k][nlog]
  long long nlog;
  // fused gradient: XT stages coef = v - vsub and writes the difference to vout;
  // XD accumulates sum out^2 (per-CTA partials, last-CTA fold into *sq_out)
  const double* vsub;
  double* vout;
  // XD epilogue reduction (last-CTA fold into *sq_out): epi 1 = sum out^2 (gradient
  // norm), epi 2 = sum over free slots of a_i out_i (the HS product's a_J'(Qd)_J)
  int epi;
  const uint8_t* fm;
  const double* av;
  double* sq_part;
  double* sq_out;
  unsigned int* sq_ticket;
  // epi 3 (k = 2, the factor-space Newton epilogue X [t, r]): output 0 folds as epi 2,
  // output 1 (the gradient X r) as epi 1 into *sq_out2 (partials at sq_part + grid)
  double* sq_out2;
};

// Producer: stream rows [r0, r1) of A through the ring.  Returns after the last issue.
__device__ __forceinline__ void produce(const StreamArgs& p, long long r0, long long r1,
                                       char* ring, uint64_t* full, uint64_t* empty) {
  const long long rows = r1 - r0;
  const long long nchunk = ceil_div(rows, (long long)p.rows_per_stage);
  for (long long c = 0; c < nchunk; ++c) {
    const int s = (int)(c % NSTAGE);
    if (c >= NSTAGE) mbar_wait(&empty[s], (uint32_t)(((c / NSTAGE) - 1) & 1));
    const long long rb = r0 + c * p.rows_per_stage;
    const long long nr = min((long long)p.rows_per_stage, r1 - rb);
    const uint32_t bytes = (uint32_t)(nr * p.lda * sizeof(double));
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(ring + (size_t)s * STAGE_BYTES, p.A + rb * p.lda, bytes, &full[s]);
  }
}

template <int KV, int CP>
__global__ void __launch_bounds__(NTHREADS, 1) stream_xt_kernel(StreamArgs p) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
  __shared__ double coef_s[ROWS_CTA][KV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rows_per = ceil_div(p.n, (long long)gridDim.x);
  const long long r0 = blockIdx.x * rows_per, r1 = min(p.n, r0 + rows_per);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCONS) {
    if (lane == 0 && r1 > r0) produce(p, r0, r1, ring, full, empty);
    return;
  }
  const int t = threadIdx.x;  // consumer thread 0..255, owns pairs t, t+256, ...
  // row coefficients (labels x vector entries) of the whole slab, loaded once while the
  // first stages are in flight
  for (long long r = t; r < r1 - r0; r += NCONS * 32) {
    const long long gr = r0 + r;
    const double sg = p.rs ? p.rs[gr] : 1.0;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      double cv = p.v[j][gr];
      if (p.vsub && j == 0) {  // s = w - Pi(u) (numpy order, as vec op 3), written out
        cv = __dsub_rn(cv, p.vsub[gr]);
        p.vout[gr] = cv;
      }
      if (p.svr) {
        double c2 = p.v[j][gr + p.n];
        if (p.vsub && j == 0) {
          c2 = __dsub_rn(c2, p.vsub[gr + p.n]);
          p.vout[gr + p.n] = c2;
        }
        cv = __dsub_rn(cv, c2);
      }
      coef_s[r][j] = sg * cv;
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCONS * 32) : "memory");
  const long long pairs = p.q / 2;
  double ax[KV][CP], ay[KV][CP];
#pragma unroll
  for (int j = 0; j < KV; ++j)
#pragma unroll
    for (int c = 0; c < CP; ++c) ax[j][c] = ay[j][c] = 0.0;
  const long long rows = r1 - r0;
  const long long nchunk = rows > 0 ? ceil_div(rows, (long long)p.rows_per_stage) : 0;
  for (long long ch = 0; ch < nchunk; ++ch) {
    const int s = (int)(ch % NSTAGE);
    const long long rb = r0 + ch * p.rows_per_stage;
    const int nr = (int)min((long long)p.rows_per_stage, r1 - rb);
    mbar_wait(&full[s], (uint32_t)((ch / NSTAGE) & 1));
    const double* st = reinterpret_cast<const double*>(ring + (size_t)s * STAGE_BYTES);
    const int rl0 = (int)(rb - r0);
    for (int r = 0; r < nr; ++r) {
      double cf[KV];
#pragma unroll
      for (int j = 0; j < KV; ++j) cf[j] = coef_s[rl0 + r][j];
      const double2* row = reinterpret_cast<const double2*>(st + (size_t)r * p.lda);
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        const long long pc = t + 256LL * c;
        if (pc < pairs) {
          const double2 a = row[pc];
#pragma unroll
          for (int j = 0; j < KV; ++j) {
            ax[j][c] = fma(cf[j], a.x, ax[j][c]);
            ay[j][c] = fma(cf[j], a.y, ay[j][c]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    const long long pc = t + 256LL * c;
    if (pc >= pairs) continue;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      double* dst = p.part + ((long long)blockIdx.x * p.k + j) * p.q + 2 * pc;
      dst[0] = ax[j][c];
      dst[1] = ay[j][c];
    }
  }
}

// per-row contribution of the XD epilogue reduction (logical rows gr and, for the
// SVR block, gr + n holding -val)
__device__ __forceinline__ double epi_term(const StreamArgs& p, long long gr, double val,
                                           double acc) {
  if (p.epi == 1) return fma(val, val, p.svr ? fma(val, val, acc) : acc);
  if (p.epi >= 2) {  // 2, and output 0 of 3
    if (p.fm[gr]) acc = fma(p.av[gr], val, acc);
    if (p.svr && p.fm[gr + p.n]) acc = fma(p.av[gr + p.n], -val, acc);
  }
  return acc;
}

// epi_term with the epi >= 2 coefficients read from the staged slab copy (row rl)
__device__ __forceinline__ double epi_term_s(const StreamArgs& p, const double (*ec)[ROWS_CTA],
                                             int rl, double val, double acc) {
  if (p.epi == 1) return fma(val, val, p.svr ? fma(val, val, acc) : acc);
  if (p.epi >= 2) {
    acc = fma(ec[0][rl], val, acc);
    if (p.svr) acc = fma(ec[1][rl], -val, acc);
  }
  return acc;
}

template <int KV, int CP, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) stream_xd_kernel(StreamArgs p) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rows_per = ceil_div(p.n, (long long)gridDim.x);
  const long long r0 = blockIdx.x * rows_per, r1 = min(p.n, r0 + rows_per);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0 && r1 > r0) produce(p, r0, r1, ring, full, empty);
    return;
  }
  // row signs of the slab staged once (a global load per row sat on the critical path
  // of every row's reduction)
  __shared__ double rs_s[ROWS_CTA];
  // epi >= 2: the fold coefficients free_i ? a_i : 0 of the slab's logical rows (and of
  // their SVR mirrors), staged likewise -- lane 0 read them per row from global memory,
  // a dependent load on every row of the epilogue sweep
  __shared__ double ec_s[2][ROWS_CTA];
  for (long long r = threadIdx.x; r < r1 - r0; r += NCW * 32) {
    rs_s[r] = p.rs ? p.rs[r0 + r] : 1.0;
    if (p.epi >= 2) {
      const long long g = r0 + r;
      ec_s[0][r] = p.fm[g] ? p.av[g] : 0.0;
      if (p.svr) ec_s[1][r] = p.fm[g + p.n] ? p.av[g + p.n] : 0.0;
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
  const long long pairs = p.q / 2;
  // this lane's slice of d: pairs lane, lane+32, ... (CP*... <= 8 per lane for q <= 512)
  double2 dv[KV][CP * 2];
#pragma unroll
  for (int j = 0; j < KV; ++j)
#pragma unroll
    for (int c = 0; c < CP * 2; ++c) {
      const long long pc = lane + 32LL * c;
      dv[j][c] = pc < pairs ? make_double2(p.d[j * p.q + 2 * pc], p.d[j * p.q + 2 * pc + 1])
                            : make_double2(0.0, 0.0);
    }
  const long long rows = r1 - r0;
  const long long nchunk = rows > 0 ? ceil_div(rows, (long long)p.rows_per_stage) : 0;
  double sq = 0.0;  // lane 0: sum of squares of this warp's outputs (fused gradient norm)
  double sq2 = 0.0;  // epi 3: sum of squares of output 1
  for (long long ch = 0; ch < nchunk; ++ch) {
    const int s = (int)(ch % NSTAGE);
    const long long rb = r0 + ch * p.rows_per_stage;
    const int nr = (int)min((long long)p.rows_per_stage, r1 - rb);
    mbar_wait(&full[s], (uint32_t)((ch / NSTAGE) & 1));
    const double* st = reinterpret_cast<const double*>(ring + (size_t)s * STAGE_BYTES);
    // two rows per warp iteration: their shuffle trees interleave
    for (int r = warp; r < nr; r += 2 * NCW) {
      const int r2 = r + NCW;
      const bool two = r2 < nr;
      const double2* row = reinterpret_cast<const double2*>(st + (size_t)r * p.lda);
      const double2* row2 = reinterpret_cast<const double2*>(st + (size_t)(two ? r2 : r) * p.lda);
      double acc[KV], acc2[KV];
#pragma unroll
      for (int j = 0; j < KV; ++j) acc[j] = acc2[j] = 0.0;
#pragma unroll
      for (int c = 0; c < CP * 2; ++c) {
        const long long pc = lane + 32LL * c;
        if (pc < pairs) {
          const double2 a = row[pc];
          const double2 b2 = row2[pc];
#pragma unroll
          for (int j = 0; j < KV; ++j) {
            acc[j] = fma(a.y, dv[j][c].y, fma(a.x, dv[j][c].x, acc[j]));
            acc2[j] = fma(b2.y, dv[j][c].y, fma(b2.x, dv[j][c].x, acc2[j]));
          }
        }
      }
      // reduce-scatter butterfly over the 2 KV row sums: each level halves the values a
      // lane keeps, so the 2 KV totals land in different lane groups (KV = 2: 6 shuffles
      // instead of 20) and their epilogues run in parallel, one writer lane per output:
      //   value index v = 2*bit4 (+ bit3 for KV = 2): row = bit4, right-hand side j = bit3
      const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
      double z;
      if constexpr (KV == 2) {
        const double s0 = b4 ? acc[0] : acc2[0], s1 = b4 ? acc[1] : acc2[1];
        const double k0 = b4 ? acc2[0] : acc[0], k1 = b4 ? acc2[1] : acc[1];
        const double w0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
        const double w1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
        z = (b3 ? w1 : w0) + __shfl_xor_sync(0xffffffffu, b3 ? w0 : w1, 8);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
      } else {
        z = (b4 ? acc2[0] : acc[0]) + __shfl_xor_sync(0xffffffffu, b4 ? acc[0] : acc2[0], 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
      }
      const int jo = KV == 2 ? b3 : 0;
      const bool writer = (lane & (KV == 2 ? 7 : 15)) == 0 && (b4 == 0 || two);
      if (writer) {
        const int rr = b4 ? r2 : r;
        const int rl = (int)(rb - r0) + rr;
        const double val = rs_s[rl] * z;
        p.out[(long long)jo * p.nlog + rb + rr] = val;
        if (p.svr) p.out[(long long)jo * p.nlog + rb + rr + p.n] = -val;
        if (jo == 0) sq = epi_term_s(p, ec_s, rl, val, sq);
        if (KV == 2 && jo == 1 && p.epi == 3) sq2 = fma(val, val, p.svr ? fma(val, val, sq2) : sq2);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (p.epi) {  // consumer warps only (the producer warp has returned)
    __shared__ double wsq[NCW], wsq2[NCW];
    __shared__ bool last;
    sq = warp_sum(sq);  // writer lanes hold the per-lane partials
    sq2 = warp_sum(sq2);
    if (lane == 0) {
      wsq[warp] = sq;
      wsq2[warp] = sq2;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    if (threadIdx.x == 0) {
      double c = 0.0, c2 = 0.0;
      for (int w = 0; w < NCW; ++w) {
        c += wsq[w];
        c2 += wsq2[w];
      }
      p.sq_part[blockIdx.x] = c;
      if (p.epi == 3) p.sq_part[gridDim.x + blockIdx.x] = c2;
      __threadfence();
      last = atomicAdd(p.sq_ticket, 1u) == gridDim.x - 1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    if (last && warp == 0) {
      double c = 0.0, c2 = 0.0;
      for (unsigned b = lane; b < gridDim.x; b += 32) {
        c += __ldcg(p.sq_part + b);
        if (p.epi == 3) c2 += __ldcg(p.sq_part + gridDim.x + b);
      }
      c = warp_sum(c);
      c2 = warp_sum(c2);
      if (lane == 0) {
        *p.sq_out = c;
        if (p.epi == 3) *p.sq_out2 = c2;
        *p.sq_ticket = 0u;
      }
    }
  }
}

int rows_per_stage(long long lda) {
  long long r = STAGE_BYTES / (lda * (long long)sizeof(double));
  return (int)(r < 1 ? 1 : r);
}

template <class K>
cudaError_t launch_stream(K kernel, const StreamArgs& p, int grid, cudaStream_t stream,
                          int threads = NTHREADS) {
  const int smem = NSTAGE * STAGE_BYTES;
  // the smem opt-in once per kernel (a host API call per launch sat on the critical path
  // right after every host decision)
  // (per kernel pointer and device; kernels of one signature share K, so the key is the
  // pointer, not the template instance)
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> opted;
  {
    const std::pair<int, const void*> key(current_device(), (const void*)kernel);
    std::lock_guard<std::mutex> lock(mu);
    if (!opted.count(key)) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      opted.insert(key);
    }
  }
  note_launch();
  kernel<<<grid, threads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool stream_ok(const double* A, long long lda, long long q) {
  return (lda % 2 == 0) && (q % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
         lda * (long long)sizeof(double) <= STAGE_BYTES && q <= 2048;
}

int stream_grid(long long n) {
  // one slab of <= ROWS_CTA rows per CTA, at least one CTA per SM when n allows
  long long g = ceil_div(n, (long long)ROWS_CTA);
  if (g < 148) g = min(148LL, ceil_div(n, 8LL));
  return (int)(g < 1 ? 1 : g);
}

// X^T [v0 (, v1)] into part[grid][k][q]; caller folds.  k <= 2.
cudaError_t launch_stream_xt(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, int k, const double* const* vs, int kofs,
                             int ktot, double* part, cudaStream_t stream, const double* vsub,
                             double* vout) {
  StreamArgs p{};
  p.vsub = vsub;
  p.vout = vout;
  p.A = A; p.n = n; p.q = q; p.lda = lda; p.rs = rs; p.svr = svr;
  p.rows_per_stage = rows_per_stage(lda);
  p.v[0] = vs[kofs];
  p.v[1] = k > 1 ? vs[kofs + 1] : nullptr;
  p.k = ktot;
  p.part = part + (long long)kofs * q;  // slot kofs of each CTA record (record stride ktot*q)
  const int grid = stream_grid(n);
  const long long pairs = q / 2;
  const int cp = (int)ceil_div(pairs, 256LL);
  if (k == 2) {
    if (cp <= 1) return launch_stream(stream_xt_kernel<2, 1>, p, grid, stream);
    if (cp <= 2) return launch_stream(stream_xt_kernel<2, 2>, p, grid, stream);
    return launch_stream(stream_xt_kernel<2, 4>, p, grid, stream);
  }
  if (cp <= 1) return launch_stream(stream_xt_kernel<1, 1>, p, grid, stream);
  if (cp <= 2) return launch_stream(stream_xt_kernel<1, 2>, p, grid, stream);
  return launch_stream(stream_xt_kernel<1, 4>, p, grid, stream);
}

cudaError_t launch_stream_xd(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, int k, const double* d, double* out,
                             long long nlog, cudaStream_t stream, double* sq_part, double* sq_out,
                             unsigned int* sq_ticket, int epi, const uint8_t* fm,
                             const double* av, double* sq_out2) {
  StreamArgs p{};
  p.sq_out2 = sq_out2;
  p.epi = sq_out ? (epi ? epi : 1) : 0;
  p.fm = fm;
  p.av = av;
  p.sq_part = sq_part;
  p.sq_out = sq_out;
  p.sq_ticket = sq_ticket;
  p.A = A; p.n = n; p.q = q; p.lda = lda; p.rs = rs; p.svr = svr;
  // whole rounds of 2 rows x XD warps per stage (q = 300: 16 rows of 2.4 KB instead of
  // 20, whose 4-row second round left 3/4 of the warps idle)
  {
    const int wmax = 16;  // the larger consumer count either instantiation may use
    const int r = rows_per_stage(lda);
    p.rows_per_stage = r >= 2 * wmax ? r / (2 * wmax) * (2 * wmax) : (r >= 16 ? r / 16 * 16 : r);
  }
  p.d = d;
  p.out = out;
  p.nlog = nlog;
  const int grid = stream_grid(n);
  const long long pairs = q / 2;
  const int cp = (int)ceil_div(pairs, 64LL);  // lanes hold 2*CP pairs each
  // 8 consumer warps for one or two right-hand sides (the 16-warp variants measured no
  // better and spilled at <2, 4, 16>: pruned in round 2)
  static_assert(XD_WARPS1 == 8 && XD_WARPS2 == 8, "instantiated for 8 consumer warps");
  if (k == 2) {
    if (cp <= 1) return launch_stream(stream_xd_kernel<2, 1, 8>, p, grid, stream);
    if (cp <= 2) return launch_stream(stream_xd_kernel<2, 2, 8>, p, grid, stream);
    return launch_stream(stream_xd_kernel<2, 4, 8>, p, grid, stream);
  }
  if (cp <= 1) return launch_stream(stream_xd_kernel<1, 1, 8>, p, grid, stream);
  if (cp <= 2) return launch_stream(stream_xd_kernel<1, 2, 8>, p, grid, stream);
  return launch_stream(stream_xd_kernel<1, 4, 8>, p, grid, stream);
}

}  // namespace ssnal

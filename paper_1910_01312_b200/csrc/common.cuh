// Shared device helpers for the SSsNAL sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define SSNAL_NT 256          // threads per block for streaming kernels
#define SSNAL_MAX_BLOCKS 592  // 4 x 148 SMs: cap for grid-stride streaming grids
#define SSNAL_MAX_TRIALS 16   // batched projections per launch (line-search step lengths)

namespace ssnal {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reduction of NV values per thread (sum / min / max selected per slot
// by `ops`: 0 = sum, 1 = min, 2 = max).  Result valid in thread 0 (vals[]).
// Deterministic: fixed shuffle tree, then warps combined in index order.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&vals)[NV], const int (&ops)[NV],
                                             double* smem /* >= NV * 32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double v = vals[k];
    v = ops[k] == 0 ? warp_sum(v) : (ops[k] == 1 ? warp_min(v) : warp_max(v));
    if (lane == 0) smem[k * 32 + warp] = v;
  }
  __syncthreads();
  // slot k is combined across warps by thread k (fixed order), then broadcast to thread 0
  // threads 0..NV-1 fold one slot each in lockstep; the per-slot op is read from a
  // bit mask built at compile time (a dynamic ops[k] would copy ops[] to local memory)
  static_assert(NV <= 64, "block_reduce: at most 64 slots");
  unsigned long long is_sum = 0ull, is_min = 0ull;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (ops[k] == 0) is_sum |= 1ull << k;
    if (ops[k] == 1) is_min |= 1ull << k;
  }
  for (int k = threadIdx.x; k < NV; k += blockDim.x) {
    const unsigned op = ((is_sum >> k) & 1ull) ? 0u : (((is_min >> k) & 1ull) ? 1u : 2u);
    double v = smem[k * 32];
    for (int w = 1; w < nwarps; ++w) {
      double x = smem[k * 32 + w];
      v = op == 0 ? v + x : (op == 1 ? fmin(v, x) : fmax(v, x));
    }
    smem[k * 32] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) vals[k] = smem[k * 32];
  }
  __syncthreads();
}

// Fold the per-block partial records of a grid (record b at base + b*stride, NV
// values each) inside ONE block: thread t folds records t, t+blockDim, ... in
// order, then a fixed shuffle/warp tree combines threads.  Result in thread 0.
template <int NV>
__device__ __forceinline__ void block_fold_partials(const double* base, unsigned nrec,
                                                    long long stride, const int (&ops)[NV],
                                                    double (&vals)[NV], double* smem) {
#pragma unroll
  for (int k = 0; k < NV; ++k)
    vals[k] = ops[k] == 0 ? 0.0 : (ops[k] == 1 ? INFINITY : -INFINITY);
  for (unsigned b = threadIdx.x; b < nrec; b += blockDim.x) {
    const double* q = base + (long long)b * stride;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double x = __ldcg(q + k);
      vals[k] = ops[k] == 0 ? vals[k] + x : (ops[k] == 1 ? fmin(vals[k], x) : fmax(vals[k], x));
    }
  }
  block_reduce<NV>(vals, ops, smem);
}

// "Last block done" ticket: returns true in exactly one block (the last to arrive),
// after a device-scope fence so that every block's partials are visible to it.
__device__ __forceinline__ bool last_block_arrive(unsigned int* ticket, unsigned int nblocks) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(ticket, 1u);
    is_last = (prev == nblocks - 1);
    if (is_last) *ticket = 0u;  // reset for the next launch
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

__host__ __device__ inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace ssnal

namespace ssnal {
// host-side count of kernel launches issued by this library (ssnal_launch_count)
void note_launch();

// A launch setting computed once PER DEVICE ORDINAL (occupancy-derived grid sizes,
// cudaFuncSetAttribute opt-ins): slot d holds value + 1 (0 = not yet computed).
// Thread-safe: concurrent first calls compute the same value and store it atomically.
struct DeviceCache {
  std::atomic<int> slot[64];
};

inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  return dev;
}

template <class F>
inline int per_device(DeviceCache& c, F compute) {
  const int dev = current_device();
  int v = c.slot[dev].load(std::memory_order_acquire);
  if (v == 0) {
    v = compute(dev) + 1;
    c.slot[dev].store(v, std::memory_order_release);
  }
  return v - 1;
}
}  // namespace ssnal

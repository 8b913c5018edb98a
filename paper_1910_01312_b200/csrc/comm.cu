// Collectives of the row-sharded native driver (driver.cu, ssnal_alm_solve_sharded).
//
// The driver only needs two operations, both enqueued on its stream:
//   allreduce_sum(buf, count)  -- every rank ends with the same sum of all ranks' bufs
//   allgather(in, out, count)  -- out[r * count + i] = rank r's in[i]
// (q-vectors, the q x q Gram, scalar records; ref kernels.py:144-154 X^T v and the
// inner products of solver.py:151-172 / projection.py:152-211 are what they reduce).
//
// Two transports implement ssnal_comm_t:
//  * NCCL (one process per GPU over NVLink / NVSwitch): libnccl.so.2 is opened with
//    dlopen -- the copy torch already loaded when it is in the process -- so the
//    library itself has no link-time NCCL dependency.  NCCL all-reduce hands every
//    rank the same reduced buffer (ring: reduce-scatter then all-gather of the reduced
//    chunks; NVLS: one switch reduction multicast back), so replicated scalars stay
//    bit-identical across ranks and every rank takes the same branch.
//  * loopback (tests): world ranks as host threads of ONE process on ONE GPU, each
//    with its own stream.  A collective drains the caller's stream, meets the other
//    ranks at a host barrier and sums their buffers in rank order with a kernel; no
//    kernel ever waits on another rank (the ranks' kernels only serialise on the GPU),
//    so the multi-rank control flow runs on a one-GPU box.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {

struct NcclApi {
  bool ok = false;
  const char* why = "libnccl.so.2 not loaded";
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.all_gather &&
           a.comm_destroy && a.error_string;
    if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    return a;
  }();
  return api;
}

int nccl_allreduce(void* ctx, double* buf, int64_t count, void* stream) {
  if (count <= 0) return 0;
  const ncclResult_t r = nccl().all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                                           (ncclComm_t)ctx, (cudaStream_t)stream);
  return r == ncclSuccess ? 0 : SSNAL_E_DEVICE;
}

int nccl_allgather(void* ctx, const double* in, double* out, int64_t count, void* stream) {
  if (count <= 0) return 0;
  const ncclResult_t r = nccl().all_gather(in, out, (size_t)count, ncclFloat64, (ncclComm_t)ctx,
                                           (cudaStream_t)stream);
  return r == ncclSuccess ? 0 : SSNAL_E_DEVICE;
}

// ---------------------------------------------------------------- loopback
constexpr int LOOP_MAX = 16;

struct LoopGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;  // a rank timed out: every later collective fails fast
  const double* ptr[LOOP_MAX] = {};
};

struct LoopComm {
  LoopGroup* g;
  int rank;
  double* tmp = nullptr;
  size_t cap = 0;
};

// host barrier of the group's ranks (generation counted; 600 s timeout breaks the group)
bool loop_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  if (g->broken) return false;
  const unsigned long long my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return true;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g->gen != my || g->broken; }) ||
      g->broken) {
    g->broken = true;
    g->cv.notify_all();
    return false;
  }
  return true;
}

struct PtrSet {
  const double* p[LOOP_MAX];
};

// out[i] = sum_{r < world} src_r[i], r ascending
__global__ void loop_sum_kernel(PtrSet s, int world, long long len, double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    double v = s.p[0][i];
    for (int r = 1; r < world; ++r) v += s.p[r][i];
    out[i] = v;
  }
}

int loop_allreduce(void* ctx, double* buf, int64_t count, void* stream) {
  auto* c = static_cast<LoopComm*>(ctx);
  LoopGroup* g = c->g;
  cudaStream_t s = (cudaStream_t)stream;
  if (count <= 0) return 0;
  if (cudaStreamSynchronize(s) != cudaSuccess) return SSNAL_E_DEVICE;
  if ((size_t)count > c->cap) {
    if (c->tmp) cudaFree(c->tmp);
    c->tmp = nullptr;
    if (cudaMalloc(&c->tmp, sizeof(double) * (size_t)count) != cudaSuccess) return SSNAL_E_DEVICE;
    c->cap = (size_t)count;
  }
  g->ptr[c->rank] = buf;
  if (!loop_barrier(g)) return SSNAL_E_DEVICE;
  PtrSet ps{};
  for (int r = 0; r < g->world; ++r) ps.p[r] = g->ptr[r];
  note_launch();
  loop_sum_kernel<<<(unsigned)std::min<long long>(ceil_div(count, 256LL), 1184LL), 256, 0, s>>>(
      ps, g->world, (long long)count, c->tmp);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return SSNAL_E_DEVICE;
  if (!loop_barrier(g)) return SSNAL_E_DEVICE;  // every rank has read every buffer
  return cudaMemcpyAsync(buf, c->tmp, sizeof(double) * (size_t)count, cudaMemcpyDeviceToDevice,
                         s) == cudaSuccess
             ? 0
             : SSNAL_E_DEVICE;
}

int loop_allgather(void* ctx, const double* in, double* out, int64_t count, void* stream) {
  auto* c = static_cast<LoopComm*>(ctx);
  LoopGroup* g = c->g;
  cudaStream_t s = (cudaStream_t)stream;
  if (count <= 0) return 0;
  if (cudaStreamSynchronize(s) != cudaSuccess) return SSNAL_E_DEVICE;
  g->ptr[c->rank] = in;
  if (!loop_barrier(g)) return SSNAL_E_DEVICE;
  for (int r = 0; r < g->world; ++r)
    if (cudaMemcpyAsync(out + (size_t)r * count, g->ptr[r], sizeof(double) * (size_t)count,
                        cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return SSNAL_E_DEVICE;
  if (cudaStreamSynchronize(s) != cudaSuccess) return SSNAL_E_DEVICE;
  return loop_barrier(g) ? 0 : SSNAL_E_DEVICE;
}

}  // namespace

int nccl_unique_id(unsigned char* id, const char** err) {
  const NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.why;
    return SSNAL_E_DEVICE;
  }
  ncclUniqueId uid;
  const ncclResult_t r = a.get_unique_id(&uid);
  if (r != ncclSuccess) {
    *err = a.error_string(r);
    return SSNAL_E_DEVICE;
  }
  static_assert(sizeof(ncclUniqueId) == SSNAL_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &uid, sizeof uid);
  return SSNAL_OK;
}

int nccl_comm_create(int world, int rank, const unsigned char* id, ssnal_comm_t* out,
                     const char** err) {
  const NcclApi& a = nccl();
  if (!a.ok) {
    *err = a.why;
    return SSNAL_E_DEVICE;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = a.comm_init_rank(&comm, world, uid, rank);
  if (r != ncclSuccess) {
    *err = a.error_string(r);
    return SSNAL_E_DEVICE;
  }
  out->world = world;
  out->rank = rank;
  out->allreduce_sum = nccl_allreduce;
  out->allgather = nccl_allgather;
  out->ctx = comm;
  out->kind = SSNAL_COMM_NCCL;
  return SSNAL_OK;
}

int loop_group_create(int world, void** group) {
  if (world < 1 || world > LOOP_MAX) return SSNAL_E_ARG;
  auto* g = new LoopGroup;
  g->world = world;
  *group = g;
  return SSNAL_OK;
}

int loop_comm_create(void* group, int rank, ssnal_comm_t* out) {
  auto* g = static_cast<LoopGroup*>(group);
  if (!g || rank < 0 || rank >= g->world) return SSNAL_E_ARG;
  auto* c = new LoopComm{g, rank};
  out->world = g->world;
  out->rank = rank;
  out->allreduce_sum = loop_allreduce;
  out->allgather = loop_allgather;
  out->ctx = c;
  out->kind = SSNAL_COMM_LOOPBACK;
  return SSNAL_OK;
}

int comm_destroy(ssnal_comm_t* c) {
  if (!c || !c->ctx) return SSNAL_OK;
  if (c->kind == SSNAL_COMM_NCCL) {
    const NcclApi& a = nccl();
    if (a.ok) a.comm_destroy((ncclComm_t)c->ctx);
  } else if (c->kind == SSNAL_COMM_LOOPBACK) {
    auto* lc = static_cast<LoopComm*>(c->ctx);
    if (lc->tmp) cudaFree(lc->tmp);
    delete lc;
  }
  c->ctx = nullptr;
  return SSNAL_OK;
}

int loop_group_destroy(void* group) {
  delete static_cast<LoopGroup*>(group);
  return SSNAL_OK;
}

}  // namespace ssnal

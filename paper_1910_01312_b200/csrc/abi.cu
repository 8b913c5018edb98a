// extern "C" entry points of include/ssnal_b200.h: argument checks, launch, error text.
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {
int stream_blocks(long long n, int per_thread);
size_t reduce_ws_bytes(long long n);
size_t compact_ws_bytes(long long n);
size_t dense_xt_ws_bytes(long long n_phys, long long q, int k);
size_t gram_ws_bytes_full(long long q);
cudaError_t launch_dots(int k, const double* const* xs, const double* const* ys,
                        const uint8_t* mask, long long n, double* out, void* ws, cudaStream_t s);
cudaError_t launch_vec(int op, long long n, double alpha, const double* x, const double* y,
                       const double* z, double* out, cudaStream_t s);
cudaError_t launch_hs_apply(const uint8_t* fm, const double* a, const double* y, long long n,
                            double beta, const double* add, double alpha, double* out, void* ws,
                            cudaStream_t s);
cudaError_t launch_compact(const uint8_t* m, long long n, int32_t* idx, long long* count, void* ws,
                           cudaStream_t s);
cudaError_t launch_dense_xt(const double* A, long long n, long long q, long long lda,
                            const double* rs, int svr, int k, const double* const* vs, double* out,
                            void* ws, cudaStream_t s);
cudaError_t launch_dense_x(const double* A, long long n, long long q, long long lda,
                           const double* rs, int svr, int k, const double* d, double* out,
                           cudaStream_t s);
cudaError_t launch_dense_gram(const double* A, long long n, long long q, long long lda,
                              const double* rs, int svr, const int32_t* J, const long long* p_dev,
                              long long p_max, const double* a, double sigma, const double* asa_dev,
                              double* M, double* m1, void* ws, cudaStream_t s);
cudaError_t launch_chol_solve(double* M, long long m, const double* b, double scale, double* x,
                              int* info, cudaStream_t s);
size_t pspace_ws_bytes(long long p, long long q);
size_t alm_ws_bytes(long long n_phys, long long q, int svr, int world);
size_t alm_ws_bytes_csr(const ssnal_csr_operator_t* op, int world);
int alm_solve_dense(const ssnal_dense_problem_t* pb, const ssnal_options_t* opt, const double* x0,
                    const double* w0, double* x_out, ssnal_report_t* rep, void* ws,
                    size_t ws_bytes, ssnal_progress_fn cb, void* ctx, cudaStream_t stream,
                    const char** err, const ssnal_comm_t* comm);
cudaError_t launch_pspace_direction(const double* A, long long n, long long q, long long lda,
                                    const double* rs, int svr, const int32_t* J, long long p,
                                    const double* grad, const double* a, double sigma, double asa,
                                    const double* g_r, double* t, int* info, void* ws,
                                    cudaStream_t stream);
size_t proj_local_ws_bytes(long long n, int T);
size_t gradient_ws_bytes(long long n_phys, long long q);
cudaError_t launch_direction_epilogue(const double* A, long long n, long long q, long long lda,
                                      const double* rs, int svr, const double* t, double* qdir,
                                      const uint8_t* fm, const double* a, const double* asa_dev,
                                      const double* s, double sigma, const double* grad,
                                      const double* w, const double* qw, double* dir,
                                      double* dots4, void* ws, cudaStream_t stream);
cudaError_t launch_dense_gradient(const double* A, long long n, long long q, long long lda,
                                  const double* rs, int svr, const double* w, const double* xp,
                                  double* s_out, double* g_r, double* grad, double* g2, void* ws,
                                  cudaStream_t stream);
cudaError_t launch_proj_local(const double* A, const double* B, const double* coef,
                              const double* lam, const double* a, const double* l,
                              const double* u, double lc, double uc, long long n, int T, int mode,
                              double* x_out, uint8_t* free_out, const double* ref,
                              const double* base, double base_lam, double* rec, void* ws,
                              cudaStream_t s);
cudaError_t launch_sum_slices(int k, long long len, const double* src, double* out,
                              cudaStream_t s);
cudaError_t launch_hs_apply_coef(const uint8_t* fm, const double* a, const double* y, long long n,
                                 double beta, const double* add, double alpha, double coef,
                                 double* out, cudaStream_t s);
cudaError_t launch_qspace_shift_assemble(long long m, const double* u, double asa, double sigma,
                                         double shift, double* M, cudaStream_t s);
}  // namespace ssnal

#include <atomic>

namespace ssnal {
static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace ssnal

using namespace ssnal;

static thread_local char g_err[512] = "";

static int fail_arg(const char* fn, const char* what) {
  snprintf(g_err, sizeof g_err, "%s: invalid argument: %s", fn, what);
  return SSNAL_E_ARG;
}

static int check(const char* fn, cudaError_t e) {
  if (e == cudaSuccess) return SSNAL_OK;
  snprintf(g_err, sizeof g_err, "%s: CUDA error %d (%s)", fn, (int)e, cudaGetErrorString(e));
  return (int)e;
}

#define S(stream) ((cudaStream_t)(stream))

extern "C" {

const char* ssnal_version(void) { return "ssnal_b200 0.1.0 (sm_100a)"; }

const char* ssnal_last_error(void) { return g_err; }

unsigned long long ssnal_launch_count(void) { return g_launches.load(); }

int ssnal_device_check(int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return check("ssnal_device_check", e);
  if (prop.major != 10 || prop.minor != 0) {
    snprintf(g_err, sizeof g_err, "ssnal_device_check: device %d is sm_%d%d, library is sm_100a",
             device, prop.major, prop.minor);
    return SSNAL_E_DEVICE;
  }
  return SSNAL_OK;
}

size_t ssnal_proj_state_bytes(void) { return sizeof(ssnal_proj_state_t); }
size_t ssnal_report_bytes(void) { return sizeof(ssnal_report_t); }
size_t ssnal_project_ws_bytes(int64_t n, int T) { return proj_ws_bytes(n, T); }
size_t ssnal_reduce_ws_bytes(int64_t n, int k) { (void)k; return reduce_ws_bytes(n) + 64; }
size_t ssnal_dense_xt_ws_bytes(int64_t n_phys, int64_t q, int k) {
  return dense_xt_ws_bytes(n_phys, q, k);
}
size_t ssnal_gram_ws_bytes(int64_t q) { return gram_ws_bytes_full(q); }
size_t ssnal_compact_ws_bytes(int64_t n) { return compact_ws_bytes(n); }

int ssnal_project_ex(const double* A, const double* B, const double* coef, const double* a,
                     const double* l, const double* u, double l_const, double u_const, double d,
                     int64_t n, int T, ssnal_proj_state_t* state, void* ws, double* x_out,
                     uint8_t* free_out, const double* ref, const double* base, double base_lam,
                     double lam_hint, int newton_passes, int phases, int passes, void* stream) {
  if (n < 1) return fail_arg("ssnal_project", "n < 1");
  if (T < 1 || T > SSNAL_MAX_TRIALS) return fail_arg("ssnal_project", "T must be in [1, 16]");
  if (!A || !a || !state || !ws) return fail_arg("ssnal_project", "null A/a/state/ws");
  if (B && !coef) return fail_arg("ssnal_project", "B given without coef");
  if (passes < 0) return fail_arg("ssnal_project", "passes < 0");
  ProjLaunch L;
  L.A = A; L.B = B; L.coef = coef; L.a = a; L.l = l; L.u = u;
  L.lc = l_const; L.uc = u_const; L.d = d; L.n = n; L.T = T;
  L.st = state; L.part = (double*)ws; L.x_out = x_out; L.free_out = free_out; L.ref = ref;
  L.base = base; L.base_lam = base_lam;
  L.phases = phases; L.passes = passes;
  L.hint = lam_hint; L.newton = newton_passes < 0 ? 0 : newton_passes;
  return check("ssnal_project", launch_project(L, S(stream)));
}

int ssnal_project(const double* A, const double* B, const double* coef, const double* a,
                  const double* l, const double* u, double l_const, double u_const, double d,
                  int64_t n, int T, ssnal_proj_state_t* state, void* ws, double* x_out,
                  uint8_t* free_out, const double* ref, double lam_hint, int newton_passes,
                  int phases, int passes, void* stream) {
  return ssnal_project_ex(A, B, coef, a, l, u, l_const, u_const, d, n, T, state, ws, x_out,
                          free_out, ref, nullptr, 0.0, lam_hint, newton_passes, phases, passes,
                          stream);
}

int ssnal_hs_apply(const uint8_t* free_mask, const double* a, const double* y, int64_t n,
                   double beta, const double* add, double alpha, double* out, void* ws,
                   void* stream) {
  if (n < 1 || !free_mask || !a || !y || !out || !ws) return fail_arg("ssnal_hs_apply", "null/size");
  return check("ssnal_hs_apply",
               launch_hs_apply(free_mask, a, y, n, beta, add, alpha, out, ws, S(stream)));
}

int ssnal_dots(int k, const double* const* xs, const double* const* ys, const uint8_t* mask,
               int64_t n, double* out, void* ws, void* stream) {
  if (k < 1 || k > 8) return fail_arg("ssnal_dots", "k must be in [1, 8]");
  if (n < 1 || !xs || !out || !ws) return fail_arg("ssnal_dots", "null/size");
  return check("ssnal_dots", launch_dots(k, xs, ys, mask, n, out, ws, S(stream)));
}

int ssnal_vec(int op, int64_t n, double alpha, const double* x, const double* y, const double* z,
              double* out, void* stream) {
  if (op < 0 || op > 6 || n < 1 || !x || !out) return fail_arg("ssnal_vec", "op/size/null");
  if ((op == 1 || op == 2 || op == 3 || op == 0 || op >= 5) && !y) return fail_arg("ssnal_vec", "y required");
  if (op == 1 && !z) return fail_arg("ssnal_vec", "z required for op 1");
  return check("ssnal_vec", launch_vec(op, n, alpha, x, y, z, out, S(stream)));
}

int ssnal_dense_xt(const double* A, int64_t n_phys, int64_t q, int64_t lda, const double* row_sign,
                   int svr_block, int k, const double* const* vs, double* out, void* ws,
                   void* stream) {
  if (n_phys < 1 || q < 1 || lda < q || k < 1 || k > 4 || !A || !vs || !out || !ws)
    return fail_arg("ssnal_dense_xt", "size/null");
  return check("ssnal_dense_xt", launch_dense_xt(A, n_phys, q, lda, row_sign, svr_block, k, vs, out,
                                                 ws, S(stream)));
}

int ssnal_dense_x(const double* A, int64_t n_phys, int64_t q, int64_t lda, const double* row_sign,
                  int svr_block, int k, const double* d, double* out, void* stream) {
  if (n_phys < 1 || q < 1 || lda < q || k < 1 || k > 4 || !A || !d || !out)
    return fail_arg("ssnal_dense_x", "size/null");
  if ((long long)2 * q * sizeof(double) > 200 * 1024) return fail_arg("ssnal_dense_x", "q too large");
  return check("ssnal_dense_x", launch_dense_x(A, n_phys, q, lda, row_sign, svr_block, k, d, out,
                                               S(stream)));
}

int ssnal_compact(const uint8_t* mask, int64_t n, int32_t* idx, int64_t* count, void* ws,
                  void* stream) {
  if (n < 1 || !mask || !idx || !count || !ws) return fail_arg("ssnal_compact", "size/null");
  if (n > 0x7fffffffLL) return fail_arg("ssnal_compact", "n exceeds int32 index range");
  return check("ssnal_compact", launch_compact(mask, n, idx, (long long*)count, ws, S(stream)));
}

int ssnal_dense_gram(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                     const double* row_sign, int svr_block, const int32_t* J,
                     const int64_t* p_dev, int64_t p_max, const double* a, double sigma,
                     const double* asa_dev, double* M, double* m1, void* ws, void* stream) {
  if (n_phys < 1 || q < 1 || lda < q || !A || !J || !p_dev || !a || !asa_dev || !M || !m1 || !ws)
    return fail_arg("ssnal_dense_gram", "size/null");
  return check("ssnal_dense_gram",
               launch_dense_gram(A, n_phys, q, lda, row_sign, svr_block, J, (const long long*)p_dev,
                                 p_max, a, sigma, asa_dev, M, m1, ws, S(stream)));
}

size_t ssnal_pspace_ws_bytes(int64_t p, int64_t q) { return pspace_ws_bytes(p, q); }

size_t ssnal_alm_ws_bytes(int64_t n_phys, int64_t q, int svr_block) {
  return alm_ws_bytes(n_phys, q, svr_block, 0);
}

size_t ssnal_alm_ws_bytes_csr(const ssnal_csr_operator_t* op) {
  return op ? alm_ws_bytes_csr(op, 0) : 0;
}

size_t ssnal_alm_ws_bytes_sharded(int64_t n_phys, int64_t q, int svr_block, int world) {
  return world >= 1 ? alm_ws_bytes(n_phys, q, svr_block, world) : 0;
}

size_t ssnal_alm_ws_bytes_csr_sharded(const ssnal_csr_operator_t* op, int world) {
  return (op && world >= 1) ? alm_ws_bytes_csr(op, world) : 0;
}

static bool csr_ok(const ssnal_csr_operator_t* op) {
  return op && op->n >= 1 && op->q >= 1 && op->indptr && op->indices && op->values &&
         op->colptr && op->rowidx && op->valt && op->seg_beg && op->seg_end && op->seg_col &&
         op->seg_slot && (op->nfold == 0 || (op->fold_col && op->fold_beg));
}

int ssnal_csr_xd(const ssnal_csr_operator_t* op, const int32_t* rows, int64_t nrows,
                 const double* d, double* out, void* stream) {
  if (!csr_ok(op) || !d || !out || nrows < 0) return fail_arg("ssnal_csr_xd", "operator/null");
  if (nrows == 0) return SSNAL_OK;
  return check("ssnal_csr_xd", launch_csr_xd(*op, rows, nrows, d, out, S(stream)));
}

int ssnal_csr_xt(const ssnal_csr_operator_t* op, const double* v, double* out, void* ws,
                 void* stream) {
  if (!csr_ok(op) || !v || !out || (op->nslots > 0 && !ws))
    return fail_arg("ssnal_csr_xt", "operator/null");
  return check("ssnal_csr_xt", launch_csc_xt(*op, v, out, (double*)ws, S(stream)));
}

size_t ssnal_csr_restricted_ws_bytes(const ssnal_csr_operator_t* op) {
  if (!csr_ok(op)) return 0;
  return cscj_ws_bytes(*op) + 256 + sizeof(double) * (size_t)(op->nslots + 1);
}

int ssnal_csr_xt_restricted(const ssnal_csr_operator_t* op, const uint8_t* keep,
                            const int32_t* J, int64_t p, const double* w, double* out, void* ws,
                            void* stream) {
  if (!csr_ok(op) || !keep || !out || !ws || p < 0 || p > op->n || (p > 0 && (!J || !w)))
    return fail_arg("ssnal_csr_xt_restricted", "operator/null/size");
  const CscJ c = cscj_layout(*op, ws);
  double* part = (double*)(((uintptr_t)ws + cscj_ws_bytes(*op) + 255) & ~(uintptr_t)255);
  cudaError_t e = launch_cscj_build(*op, keep, J, p, c, S(stream));
  if (e == cudaSuccess) e = launch_cscj_xt(*op, c, w, out, part, S(stream));
  return check("ssnal_csr_xt_restricted", e);
}

int ssnal_csr_xd_restricted(const ssnal_csr_operator_t* op, const uint8_t* keep,
                            const int32_t* J, int64_t p, const double* d, double* out, void* ws,
                            void* stream) {
  if (!csr_ok(op) || !keep || !ws || p < 0 || p > op->n || (p > 0 && (!J || !d || !out)))
    return fail_arg("ssnal_csr_xd_restricted", "operator/null/size");
  const CscJ c = cscj_layout(*op, ws);
  cudaError_t e = launch_cscj_build(*op, keep, J, p, c, S(stream));
  if (e == cudaSuccess) e = launch_csrj_xd(c, p, d, out, S(stream));
  return check("ssnal_csr_xd_restricted", e);
}

int ssnal_csr_colsq(const ssnal_csr_operator_t* op, const uint8_t* keep, double* out, void* ws,
                    void* stream) {
  if (!csr_ok(op) || !keep || !out || (op->nslots > 0 && !ws))
    return fail_arg("ssnal_csr_colsq", "operator/null");
  return check("ssnal_csr_colsq", launch_csc_colsq(*op, keep, out, (double*)ws, S(stream)));
}

static int alm_solve_common(const char* name, const ssnal_dense_problem_t* problem,
                            const ssnal_options_t* options, const double* x0, const double* w0,
                            double* x_out, ssnal_report_t* report, void* ws, size_t ws_bytes,
                            ssnal_progress_fn progress, void* progress_ctx, void* stream,
                            const ssnal_comm_t* comm);

int ssnal_alm_solve_dense(const ssnal_dense_problem_t* problem, const ssnal_options_t* options,
                          const double* x0, const double* w0, double* x_out,
                          ssnal_report_t* report, void* ws, size_t ws_bytes,
                          ssnal_progress_fn progress, void* progress_ctx, void* stream) {
  return alm_solve_common("ssnal_alm_solve_dense", problem, options, x0, w0, x_out, report, ws,
                          ws_bytes, progress, progress_ctx, stream, nullptr);
}

int ssnal_alm_solve_sharded(const ssnal_dense_problem_t* problem, const ssnal_options_t* options,
                            const ssnal_comm_t* comm, const double* x0, const double* w0,
                            double* x_out, ssnal_report_t* report, void* ws, size_t ws_bytes,
                            ssnal_progress_fn progress, void* progress_ctx, void* stream) {
  if (!comm || comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world ||
      !comm->allreduce_sum || !comm->allgather)
    return fail_arg("ssnal_alm_solve_sharded", "invalid communicator");
  return alm_solve_common("ssnal_alm_solve_sharded", problem, options, x0, w0, x_out, report, ws,
                          ws_bytes, progress, progress_ctx, stream, comm);
}

int ssnal_nccl_unique_id(unsigned char* id) {
  if (!id) return fail_arg("ssnal_nccl_unique_id", "null id");
  const char* err = nullptr;
  const int rc = nccl_unique_id(id, &err);
  if (rc != SSNAL_OK) snprintf(g_err, sizeof g_err, "ssnal_nccl_unique_id: %s", err ? err : "failed");
  return rc;
}

int ssnal_nccl_comm_create(int world, int rank, const unsigned char* id, ssnal_comm_t* out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world)
    return fail_arg("ssnal_nccl_comm_create", "world/rank/null");
  const char* err = nullptr;
  const int rc = nccl_comm_create(world, rank, id, out, &err);
  if (rc != SSNAL_OK)
    snprintf(g_err, sizeof g_err, "ssnal_nccl_comm_create: %s", err ? err : "failed");
  return rc;
}

int ssnal_loopback_group_create(int world, void** group) {
  if (!group) return fail_arg("ssnal_loopback_group_create", "null group");
  const int rc = loop_group_create(world, group);
  if (rc != SSNAL_OK) return fail_arg("ssnal_loopback_group_create", "world outside 1..16");
  return rc;
}

int ssnal_loopback_comm_create(void* group, int rank, ssnal_comm_t* out) {
  if (!group || !out) return fail_arg("ssnal_loopback_comm_create", "null group/out");
  const int rc = loop_comm_create(group, rank, out);
  if (rc != SSNAL_OK) return fail_arg("ssnal_loopback_comm_create", "rank outside the group");
  return rc;
}

int ssnal_loopback_group_destroy(void* group) { return loop_group_destroy(group); }

int ssnal_comm_destroy(ssnal_comm_t* comm) { return comm_destroy(comm); }

static int alm_solve_common(const char* name, const ssnal_dense_problem_t* problem,
                            const ssnal_options_t* options, const double* x0, const double* w0,
                            double* x_out, ssnal_report_t* report, void* ws, size_t ws_bytes,
                            ssnal_progress_fn progress, void* progress_ctx, void* stream,
                            const ssnal_comm_t* comm) {
  if (!problem || !options || !x_out || !report || !ws)
    return fail_arg(name, "null problem/options/x_out/report/ws");
  const ssnal_dense_problem_t& p = *problem;
  if (p.csr) {
    if (!csr_ok(p.csr) || p.svr_block || p.n != p.csr->n || p.n_phys != p.csr->n ||
        p.q != p.csr->q || !p.c || !p.a)
      return fail_arg(name, "inconsistent sparse problem");
  } else if (p.n_phys < 1 || p.q < 1 || p.lda < p.q || !p.A || !p.c || !p.a ||
             p.n != (p.svr_block ? 2 * p.n_phys : p.n_phys)) {
    return fail_arg(name, "inconsistent problem sizes");
  }
  const char* err = nullptr;
  int rc = alm_solve_dense(problem, options, x0, w0, x_out, report, ws, ws_bytes, progress,
                           progress_ctx, S(stream), &err, comm);
  if (rc != SSNAL_OK) snprintf(g_err, sizeof g_err, "%s: %s", name, err ? err : "failed");
  return rc;
}

int ssnal_dense_newton_pspace(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                              const double* row_sign, int svr_block, const int32_t* J, int64_t p,
                              const double* grad, const double* a, double sigma, double asa,
                              const double* g_r, double* t, int* info, void* ws, void* stream) {
  if (n_phys < 1 || q < 1 || lda < q || p < 1 || !A || !J || !grad || !a || !g_r || !t || !info ||
      !ws)
    return fail_arg("ssnal_dense_newton_pspace", "size/null");
  return check("ssnal_dense_newton_pspace",
               launch_pspace_direction(A, n_phys, q, lda, row_sign, svr_block, J, p, grad, a, sigma,
                                       asa, g_r, t, info, ws, S(stream)));
}

int ssnal_chol_solve(double* M, int64_t m, const double* b, double scale, double* x, int* info,
                     void* stream) {
  if (m < 1 || !M || !b || !x || !info) return fail_arg("ssnal_chol_solve", "size/null");
  return check("ssnal_chol_solve", launch_chol_solve(M, m, b, scale, x, info, S(stream)));
}

/* ---- row-sharded path (csrc/dist.cu) ---- */
size_t ssnal_proj_local_ws_bytes(int64_t n, int T) { return proj_local_ws_bytes(n, T); }

int ssnal_proj_local(const double* A, const double* B, const double* coef, const double* lam,
                     const double* a, const double* l, const double* u, double l_const,
                     double u_const, int64_t n, int T, int mode, double* x_out, uint8_t* free_out,
                     const double* ref, const double* base, double base_lam, double* rec,
                     void* ws, void* stream) {
  if (n < 1) return fail_arg("ssnal_proj_local", "n < 1");
  if (T < 1 || T > SSNAL_MAX_TRIALS) return fail_arg("ssnal_proj_local", "T must be in [1, 16]");
  if (!A || !a || !lam || !rec || !ws) return fail_arg("ssnal_proj_local", "null A/a/lam/rec/ws");
  if (B && !coef) return fail_arg("ssnal_proj_local", "B given without coef");
  if (mode != 0 && mode != 1) return fail_arg("ssnal_proj_local", "mode must be 0 or 1");
  return check("ssnal_proj_local", launch_proj_local(A, B, coef, lam, a, l, u, l_const, u_const,
                                                     n, T, mode, x_out, free_out, ref, base,
                                                     base_lam, rec, ws, S(stream)));
}

int ssnal_sum_slices(int k, int64_t len, const double* src, double* out, void* stream) {
  if (k < 1 || len < 1 || !src || !out) return fail_arg("ssnal_sum_slices", "size/null");
  return check("ssnal_sum_slices", launch_sum_slices(k, len, src, out, S(stream)));
}

int ssnal_hs_apply_coef(const uint8_t* free_mask, const double* a, const double* y, int64_t n,
                        double beta, const double* add, double alpha, double coef, double* out,
                        void* stream) {
  if (n < 1 || !free_mask || !a || !y || !out) return fail_arg("ssnal_hs_apply_coef", "null/size");
  return check("ssnal_hs_apply_coef", launch_hs_apply_coef(free_mask, a, y, n, beta, add, alpha,
                                                           coef, out, S(stream)));
}

int ssnal_qspace_assemble(int64_t m, const double* u, double asa, double sigma, double shift,
                          double* M, void* stream) {
  if (m < 1 || !M) return fail_arg("ssnal_qspace_assemble", "size/null");
  return check("ssnal_qspace_assemble",
               launch_qspace_shift_assemble(m, u, asa, sigma, shift, M, S(stream)));
}

/* ---- fused SsN gradient ---- */
size_t ssnal_gradient_ws_bytes(int64_t n_phys, int64_t q) { return gradient_ws_bytes(n_phys, q); }

int ssnal_dense_gradient(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                         const double* row_sign, int svr_block, const double* w, const double* xp,
                         double* s_out, double* g_r, double* grad, double* g2, void* ws,
                         void* stream) {
  if (n_phys < 1 || q < 1 || lda < q) return fail_arg("ssnal_dense_gradient", "bad shape");
  if (!A || !w || !xp || !s_out || !g_r || !grad || !g2 || !ws)
    return fail_arg("ssnal_dense_gradient", "null pointer");
  return check("ssnal_dense_gradient",
               launch_dense_gradient(A, n_phys, q, lda, row_sign, svr_block, w, xp, s_out, g_r,
                                     grad, g2, ws, S(stream)));
}

int ssnal_dense_direction_epilogue(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                                   const double* row_sign, int svr_block, const double* t,
                                   double* qdir, const uint8_t* free_mask, const double* a,
                                   const double* asa_dev, const double* s, double sigma,
                                   const double* grad, const double* w, const double* qw,
                                   double* dir, double* dots4, void* ws, void* stream) {
  if (n_phys < 1 || q < 1 || lda < q) return fail_arg("ssnal_dense_direction_epilogue", "bad shape");
  if (!A || !t || !qdir || !free_mask || !a || !asa_dev || !s || !grad || !w || !qw || !dir ||
      !dots4 || !ws)
    return fail_arg("ssnal_dense_direction_epilogue", "null pointer");
  return check("ssnal_dense_direction_epilogue",
               launch_direction_epilogue(A, n_phys, q, lda, row_sign, svr_block, t, qdir, free_mask,
                                         a, asa_dev, s, sigma, grad, w, qw, dir, dots4, ws,
                                         S(stream)));
}

}  // extern "C"

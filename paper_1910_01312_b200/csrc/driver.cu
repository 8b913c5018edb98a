// Native SSsNAL driver: Algorithm 1 (ALM outer loop) + Algorithm 3 (semismooth
// Newton inner loop) for Q = X X^T on one CUDA stream.
//
// Control flow mirrors ref solver.py:331-530 branch for branch (and
// paper_1910_01312_b200/solver.py, the Python mirror of the same loop): criteria
// (A')/(B'), grad floor, steepest-descent rescue, Armijo batches, best-iterate
// safeguard, sigma cap stagnation.  The host only synchronises at the
// decision points: the KKT residual per outer step, the start of every inner
// solve, and one pinned read per Newton step (gradient norm + Newton
// direction inner products + the unit-step Armijo trial, enqueued together).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ssnal_internal.h"

namespace ssnal {

int stream_blocks(long long n, int per_thread);
size_t reduce_ws_bytes(long long n);
size_t compact_ws_bytes(long long n);
size_t dense_xt_ws_bytes(long long n_phys, long long q, int k);
size_t gram_ws_bytes(long long q);
size_t pspace_ws_bytes(long long p, long long q);
cudaError_t launch_dots(int k, const double* const* xs, const double* const* ys,
                        const uint8_t* mask, long long n, double* out, void* ws, cudaStream_t s);
cudaError_t launch_vec(int op, long long n, double alpha, const double* x, const double* y,
                       const double* z, double* out, cudaStream_t s);
size_t gradient_ws_bytes(long long n_phys, long long q);
cudaError_t launch_dense_gradient(const double* A, long long n, long long q, long long lda,
                                  const double* rs, int svr, const double* w, const double* xp,
                                  double* s_out, double* g_r, double* grad, double* g2, void* ws,
                                  cudaStream_t stream);
cudaError_t launch_direction_epilogue(const double* A, long long n, long long q, long long lda,
                                      const double* rs, int svr, const double* t, double* qdir,
                                      const uint8_t* fm, const double* a, const double* asa_dev,
                                      const double* s, double sigma, const double* grad,
                                      const double* w, const double* qw, double* dir,
                                      double* dots4, void* ws, cudaStream_t stream);
cudaError_t launch_hs_apply_dots(const uint8_t* fm, const double* a, const double* y, long long n,
                                 double beta, const double* add, double alpha, double* out,
                                 const double* g, const double* w, const double* qw,
                                 double* dots_out, void* ws, cudaStream_t stream);
cudaError_t launch_accept(long long n, double alpha, double cu, double* w, const double* d,
                          double* qw, const double* qd, double* u, double* xp, const double* txj,
                          uint8_t* fr, const uint8_t* tfj, cudaStream_t stream);
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
cudaError_t launch_gram_update(const double* A, long long n, long long q, long long lda,
                               const double* rs, int svr, const int32_t* J, const long long* p_dev,
                               const uint8_t* sign_mask, const double* a, double* G, double* m1,
                               int accumulate, void* ws, cudaStream_t stream,
                               const GramCtl* ctl, const int32_t* Jd);
cudaError_t launch_gram_select(GramCtl* ctl, const long long* p_dev, const long long* d_dev,
                               int force_full, cudaStream_t stream);
cudaError_t launch_gram_assemble(const double* G, long long q, const double* m1, double sigma,
                                 const double* asa_dev, double* M, cudaStream_t stream);
cudaError_t launch_mask_diff(const uint8_t* fr, uint8_t* kept, uint8_t* chg, long long n,
                             cudaStream_t stream);
cudaError_t launch_pspace_direction(const double* A, long long n, long long q, long long lda,
                                    const double* rs, int svr, const int32_t* J, long long p,
                                    const double* grad, const double* a, double sigma, double asa,
                                    const double* g_r, double* t, int* info, void* ws,
                                    cudaStream_t stream);

cudaError_t launch_cg_init(long long p, const double* b, double* y, double* r, double* pv,
                           const double* dinv, const double* g2, double eta, double tau,
                           double* cgs, double* part, cudaStream_t s);
cudaError_t launch_cg_jacobi(long long q, const double* colsq, const double* u, double asa,
                             double sigma, double* dinv, cudaStream_t s);
cudaError_t launch_cg_project(long long p, const double* x, const double* aJ, const double* dot,
                              double asa, double* out, cudaStream_t s);
cudaError_t launch_cg_ap(long long p, const double* pv, const double* zq, const double* aJ,
                         double asa, double sigma, double* Ap, double* cgs, double* part,
                         cudaStream_t s);
cudaError_t launch_cg_step(long long p, double* y, double* r, const double* pv, const double* Ap,
                           const double* dinv, double* z, double* cgs, double* part,
                           cudaStream_t s);
cudaError_t launch_cg_dir(long long p, const double* r, double* pv, const double* cgs,
                          cudaStream_t s);
cudaError_t launch_scatter_zero(const int32_t* rows, long long p, double* dst, cudaStream_t s);
cudaError_t launch_cg_check(long long n, const double* zn, double sigma, double* cgs, double* part,
                            cudaStream_t s);
cudaError_t launch_sparse_gram_rows(const CsrOp& op, const int32_t* rows, long long p, double* G,
                                    cudaStream_t s);
cudaError_t launch_sparse_gram_cols(const CsrOp& op, const uint8_t* free_rows, double* G,
                                    cudaStream_t s);
cudaError_t launch_qspace_assemble(long long m, const double* u, double asa, double sigma,
                                   double* G, cudaStream_t s);
cudaError_t launch_pspace_solve(const int32_t* J, long long p, const double* grad, const double* a,
                                double sigma, double asa, double* Q, double* vecs, double* y,
                                int* info, cudaStream_t s);

cudaError_t launch_gradient_factor(const double* A, long long n, long long q, long long lda,
                                   const double* rs, int svr, const double* w, const double* xp,
                                   double* s_out, double* r, void* ws, cudaStream_t stream);
cudaError_t launch_direction_epilogue_q(const double* A, long long n, long long q, long long lda,
                                        const double* rs, int svr, const double* t2, double* qg,
                                        const uint8_t* fm, const double* a,
                                        const double* asa_dev, const double* s, double sigma,
                                        const double* w, const double* qw, double* dir,
                                        double* dots4, double* g2, void* ws, cudaStream_t stream,
                                        int parts);
cudaError_t launch_grad_from_factor(const double* A, long long n, long long q, long long lda,
                                    const double* rs, int svr, const double* r, double* grad,
                                    double* g2, void* ws, cudaStream_t stream);
cudaError_t launch_rows_grad(const double* A, long long n, long long q, long long lda,
                             const double* rs, int svr, const int32_t* J, long long p,
                             const double* r, double* grad, cudaStream_t stream);
size_t accept_q_ws_bytes(long long n, long long q);
cudaError_t launch_accept_q(const double* A, long long n_phys, long long q, long long lda,
                            const double* rs, int svr, long long n, double alpha, double cu,
                            double* w, const double* d, double* qw, const double* qd, double* u,
                            double* xp, const double* txj, uint8_t* fr, const uint8_t* tfj,
                            double* s, const double* t, double* xw, double* xpi, double* r,
                            double* part, const ProjState* st_src, ProjState* st_dst,
                            cudaStream_t stream, double* dsum = nullptr, const double* gt = nullptr,
                            const double* m1 = nullptr, const double* avec = nullptr);
cudaError_t launch_gram_tvec(const double* G, long long q, const double* t, double* out,
                             cudaStream_t stream);

// direct reduced systems of the sparse operator: min(p, q) up to this size (M buffer)
constexpr long long SPARSE_DIRECT_MAX = 2048;
// dense operator: the factor-space gradient (accept_q) handles q <= ACCEPT_Q_MAX; larger q
// run the full-gradient path.  Direct systems: q x q up to DENSE_QSYS_MAX (workspace M,
// G), p x p up to DENSE_PSYS_MAX.
constexpr long long ACCEPT_Q_MAX = 2048;
constexpr long long DENSE_QSYS_MAX = 4096;
constexpr long long DENSE_PSYS_MAX = 4096;
// forcing-term cap of the matrix-free CG route (see cg_direction)
// (1e-4 in round 1; the reference's own eta = 1e-2 converges configs 2 and 3 at full size
// -- 3.0 s / 113 s, objectives equal to the oracle's to 1e-12 -- so no cap below it)
constexpr double SPARSE_CG_ETA = 1e-2;
// study knobs (scripts/cg_study.py): SSNAL_CG_ETA_CAP overrides the cap, SSNAL_CG_BATCH
// the iterations between true-residual checks
static double cg_eta_cap() {
  static const double v = std::getenv("SSNAL_CG_ETA_CAP") ? std::atof(std::getenv("SSNAL_CG_ETA_CAP"))
                                                          : SPARSE_CG_ETA;
  return v;
}
// CG stopping rule.  0: the TRUE Newton residual of Algorithm 3 Step 1 (an n-row product
// per check).  1: the reference's rule (solver.py:151-172, 253: absolute residual of its
// (I/sigma + Q_JJ + ..) v = g_J system <= target), which in factor space is
// ||P_J X_J r_t|| <= target -- the true residual is sigma X X_J^T of that vector.
cudaError_t launch_cg_update(long long p, double* y, double* r, double* pv, const double* zq,
                             const double* aJ, double asa, double sigma, const double* dinv,
                             double* Ap, double* z, double* cgs, double* part, cudaStream_t s);
// SSNAL_ACCEPT_LIN=0: the accept pass gathers the rows of every changed slot (A/B knob)
static bool accept_lin() {
  static const bool v = !(std::getenv("SSNAL_ACCEPT_LIN") && std::atoi(std::getenv("SSNAL_ACCEPT_LIN")) == 0);
  return v;
}
// SSNAL_CG_FUSED=0: the unfused cg_ap / cg_step / cg_dir launches (A/B knob)
static bool cg_fused() {
  static const bool v = !(std::getenv("SSNAL_CG_FUSED") && std::atoi(std::getenv("SSNAL_CG_FUSED")) == 0);
  return v;
}
// SSNAL_CG_ADAPT=0: run the true-residual test after every batch.  Default: after the
// first test, a batch is followed by the test only when the recurrence residual predicts
// it may pass (||r||^2 rho^2 <= 4 tol^2 with rho^2 = true^2 / ||r||^2 from the last test),
// or after 3 skipped batches -- the test costs a full Gram product plus an n-row X
// product, ~15 % of a 16-iteration batch.
static bool cg_adapt() {
  static const bool v = !(std::getenv("SSNAL_CG_ADAPT") && std::atoi(std::getenv("SSNAL_CG_ADAPT")) == 0);
  return v;
}
static int cg_rule() {
  static const int v = std::getenv("SSNAL_CG_RULE") ? std::atoi(std::getenv("SSNAL_CG_RULE")) : 0;
  return v;
}
// max / mean column sum of squares above which the factor-space Jacobi PCG is used
constexpr double HOT_COLUMN_SPREAD = 50.0;

namespace {

constexpr int TMAX = 8;  // batched Armijo trials per launch
constexpr int CG_BATCH_DEFAULT = 16;  // CG iterations between host checks of the device flag
static int cg_batch() {
  static const int v = std::getenv("SSNAL_CG_BATCH") ? std::atoi(std::getenv("SSNAL_CG_BATCH"))
                                                     : CG_BATCH_DEFAULT;
  return v > 0 ? v : CG_BATCH_DEFAULT;
}
constexpr int NSCAL = 16;

struct DriverError {
  int code;
  const char* what;
};

// bump allocator over the caller's workspace (256-byte aligned slices)
struct Carver {
  char* base;
  size_t off = 0, cap;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
};

// Device "blob" read back by every host decision in ONE copy: scalars at 0, the
// Cholesky info at 128, then st_trial[TMAX], st_cur, st_kkt (carve keeps them contiguous)
constexpr size_t BLOB_ST = 256;
constexpr size_t BLOB_BYTES = BLOB_ST + (TMAX + 2) * sizeof(ProjState);

struct Pinned {
  double scal[NSCAL];
  double cg[8];
  int info;
  int pad;
  ProjState st[TMAX];
  alignas(256) char blob[BLOB_BYTES];
  alignas(64) volatile unsigned int seq;  // written by publish_kernel after the blob
};

// Host decision read-back without a copy-engine round trip: one CTA stores the blob
// prefix straight into the mapped pinned buffer, fences system-wide, then bumps the
// sequence word the host spins on.
__global__ void publish_kernel(const unsigned int* __restrict__ src, unsigned int nwords,
                               unsigned int* dst, volatile unsigned int* seq_word,
                               unsigned int seq) {
  for (unsigned int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *seq_word = seq;
}

Pinned* pinned_buffer() {
  static thread_local Pinned* buf = nullptr;
  if (!buf) {
    if (cudaHostAlloc(&buf, sizeof(Pinned), cudaHostAllocMapped) != cudaSuccess) buf = nullptr;
    else buf->seq = 0u;
  }
  return buf;
}

struct Layout {
  double *x, *w, *qw, *u, *xp, *s, *grad, *qdir, *dir, *tmp, *qx, *qwx, *best_x, *tx;
  double *gr, *t, *M, *m1, *scal;
  // dense operator, factor-space gradient: r = t + q (t2 = [t ; r]), X^T w, X^T Pi(u),
  // accept partials; qdir and grad are adjacent ([Qd ; grad] from one X sweep)
  double *r, *xw, *xpi, *qpart, *gt;
  uint8_t *fr, *tfree;
  int32_t* J;
  long long* pcount;
  // kept q-space Gram (dense, p >= q): G = X_J^T X_J and m1 = X_J^T a_J of the free set
  // frg, updated over the slots whose flag changed (chg -> Jd, dcount in the blob)
  double* G;
  uint8_t *frg, *chg;
  int32_t* Jd;
  long long* dcount;
  GramCtl* gctl;
  int* info;
  ProjState *st_cur, *st_trial, *st_kkt;
  void *ws_proj, *ws_red, *ws_xt, *ws_gram, *ws_cmp, *ws_ps, *ws_grad;
  // sparse operator: sample-space CG buffers, scattered vector, CSC partial slots
  double *ys, *tq, *cg_gJ, *cg_aJ, *cg_b, *cg_y, *cg_r, *cg_pv, *cg_Ap, *cg_zq, *cg_w, *cgs,
      *cg_part, *csc_part, *cg_d, *cg_u, *cg_z;
  CscJ cj;  // J-restricted CSC (matrix-free Newton systems)
  // row-sharded driver: the all-reduced Gram [G ; m1] (q x q + q), the all-reduced
  // X^T dPi of an accepted step, the projection search state and records (local T x 8,
  // all-gathered world x T x 8), the shard-local projection partials, HS sums
  double *Gg, *dsum, *rec_loc, *rec_all, *hsum;
  SProj* sp;
  void* ws_plocal;
};

// per-block partials of the CG kernels: the step kernels' 2 per block, the fused update's
// 3 per block on at most 512 blocks (cg.cu CGU_MAX_GRID)
size_t cg_part_doubles(long long n) { return 2 * (size_t)stream_blocks(n, 4) + 8 + 3 * 512; }

Layout carve(char* base, long long n, long long n_phys, long long q, size_t* total,
             const ssnal_csr_operator_t* csr = nullptr, int world = 0) {
  Carver cv{base, 0, 0};
  Layout L{};
  const bool sparse = csr != nullptr;
  L.x = cv.take<double>(n);
  L.w = cv.take<double>(n);
  L.qw = cv.take<double>(n);
  L.u = cv.take<double>(n);
  L.xp = cv.take<double>(n);
  L.s = cv.take<double>(n);
  L.qdir = cv.take<double>(2 * (size_t)n);
  L.dir = cv.take<double>(n);
  L.tmp = cv.take<double>(n);
  L.qx = cv.take<double>(n);
  L.qwx = cv.take<double>(2 * n);
  L.best_x = cv.take<double>(n);
  L.tx = cv.take<double>((size_t)TMAX * n);
  L.gr = cv.take<double>(2 * q);
  L.grad = L.qdir ? L.qdir + n : nullptr;
  L.t = cv.take<double>(2 * (size_t)q);
  L.r = L.t ? L.t + q : nullptr;
  L.xw = cv.take<double>(q);
  L.xpi = cv.take<double>(q);
  const bool qsys = !sparse && q <= DENSE_QSYS_MAX;
  L.qpart = (sparse || q > ACCEPT_Q_MAX)
                ? nullptr
                : cv.take<double>(accept_q_ws_bytes(n, q) / sizeof(double) + 1);
  L.M = qsys ? cv.take<double>((size_t)q * q) : nullptr;
  if (qsys) {
    L.G = cv.take<double>((size_t)q * q);
    L.frg = cv.take<uint8_t>(n);
    L.chg = cv.take<uint8_t>(n);
    L.Jd = cv.take<int32_t>(n);
    L.dcount = cv.take<long long>(1);
    L.gctl = cv.take<GramCtl>(1);
  }
  L.m1 = cv.take<double>(q);
  L.gt = cv.take<double>(q);
  {  // contiguous read-back blob (see BLOB_ST)
    char* blob = cv.take<char>(BLOB_BYTES);
    L.scal = reinterpret_cast<double*>(blob);
    L.info = reinterpret_cast<int*>(blob ? blob + 128 : nullptr);
    L.st_trial = reinterpret_cast<ProjState*>(blob ? blob + BLOB_ST : nullptr);
    L.st_cur = L.st_trial ? L.st_trial + TMAX : nullptr;
    L.st_kkt = L.st_trial ? L.st_trial + TMAX + 1 : nullptr;
  }
  L.fr = cv.take<uint8_t>(n);
  L.tfree = cv.take<uint8_t>((size_t)TMAX * n);
  L.J = cv.take<int32_t>(n);
  L.pcount = cv.take<long long>(1);

  L.ws_proj = cv.take<char>(proj_ws_bytes(n, TMAX));
  L.ws_red = cv.take<char>(reduce_ws_bytes(n) + 64);
  L.ws_cmp = cv.take<char>(compact_ws_bytes(n));
  if (!sparse) {
    L.ws_xt = cv.take<char>(dense_xt_ws_bytes(n_phys, q, 2));
    L.ws_grad = cv.take<char>(gradient_ws_bytes(n_phys, q));
    L.ws_gram = qsys ? cv.take<char>(gram_ws_bytes(q)) : nullptr;
    L.ws_ps = cv.take<char>(pspace_ws_bytes(std::min(q - 1, DENSE_PSYS_MAX), q));
  } else {
    L.ys = cv.take<double>(n);
    L.tq = cv.take<double>(q);
    L.cg_gJ = cv.take<double>(n);
    L.cg_aJ = cv.take<double>(n);
    L.cg_b = cv.take<double>(n);
    L.cg_y = cv.take<double>(n);
    L.cg_r = cv.take<double>(n);
    L.cg_pv = cv.take<double>(n);
    L.cg_Ap = cv.take<double>(n);
    L.cg_zq = cv.take<double>(n);
    L.cg_w = cv.take<double>(n);
    L.cg_d = cv.take<double>(q);
    L.cg_u = cv.take<double>(q);
    L.cg_z = cv.take<double>(q);
    L.cgs = cv.take<double>(16);
    L.cg_part = cv.take<double>(cg_part_doubles(n));
    L.csc_part = cv.take<double>(csr->nslots > 0 ? csr->nslots : 1);
    const long long md = std::min<long long>(SPARSE_DIRECT_MAX, std::max(q, n));
    L.M = cv.take<double>((size_t)md * md);
    L.ws_ps = cv.take<double>(4 * (size_t)md);
    char* cj = cv.take<char>(cscj_ws_bytes(*csr));
    if (base) L.cj = cscj_layout(*csr, cj);
  }
  if (world > 0) {
    const bool qs = sparse ? q <= SPARSE_DIRECT_MAX : qsys;
    L.Gg = qs ? cv.take<double>((size_t)q * q + q) : nullptr;
    L.dsum = cv.take<double>(q);
    L.rec_loc = cv.take<double>(8 * TMAX);
    L.rec_all = cv.take<double>(8 * (size_t)TMAX * world);
    L.hsum = cv.take<double>(8);
    L.sp = cv.take<SProj>(TMAX);
    L.ws_plocal = cv.take<char>(proj_local_ws_bytes(n, TMAX));
  }
  *total = cv.off + 256;
  return L;
}

// SSNAL_SYNC_CHECK=1: synchronise after every checked call and name the driver line of
// the first failure (a fault is otherwise reported at the next host decision)
void ck_at(cudaError_t e, int line) {
  static const int sync_check = std::getenv("SSNAL_SYNC_CHECK") ? 1 : 0;
  if (e == cudaSuccess && sync_check) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (sync_check) std::fprintf(stderr, "ssnal driver: %s at driver.cu:%d\n", cudaGetErrorString(e), line);
    throw DriverError{(int)e, cudaGetErrorString(e)};
  }
}
#define ck(e) ck_at((e), __LINE__)

// CUDA-event timing per op class (ssnal_options_t.profile); events are pooled
struct Prof {
  struct Rec {
    int op;
    cudaEvent_t e0, e1;
  };
  std::vector<Rec> recs;
  size_t used = 0;
  static std::vector<cudaEvent_t>& pool() {
    static thread_local std::vector<cudaEvent_t> p;
    return p;
  }
  cudaEvent_t get() {
    auto& p = pool();
    if (used == p.size()) {
      cudaEvent_t e;
      ck(cudaEventCreate(&e));
      p.push_back(e);
    }
    return p[used++];
  }
};

struct Driver {
  const ssnal_dense_problem_t& P;
  const ssnal_options_t& O;
  cudaStream_t S;
  Layout L;
  Pinned* H;
  long long syncs = 0, newton = 0, projections = 0, cg_iters = 0, cg_fallbacks = 0;
  long long proj_fallbacks = 0;
  double lam_kkt = 0.0, lam_cur = 0.0;
  double sigma = 1.0;
  double c_norm = 0.0;
  Prof prof;
  double op_bytes[SSNAL_NOPS] = {};
  double op_flops[SSNAL_NOPS] = {};
  long long op_calls[SSNAL_NOPS] = {};

  // row-sharded driver (ssnal_alm_solve_sharded): this rank's slice of the dual slots;
  // every cross-slot sum goes through C (null: one GPU, no collectives)
  const ssnal_comm_t* C = nullptr;
  long long collectives = 0;
  long long cur_local = 0;  // sharded: this rank's free slots of the current record

  Driver(const ssnal_dense_problem_t& p, const ssnal_options_t& o, cudaStream_t s, Layout l,
         Pinned* h, const ssnal_comm_t* c = nullptr)
      : P(p), O(o), S(s), L(l), H(h), C(c) {}

  bool sh() const { return C != nullptr; }

  // in-place sum over the ranks (enqueued on S; every rank receives the same buffer)
  void allsum(double* buf, long long count) {
    if (!C || count <= 0) return;
    ++collectives;
    if (C->allreduce_sum(C->ctx, buf, (int64_t)count, S) != 0)
      throw DriverError{SSNAL_E_DEVICE, "sharded all-reduce failed"};
  }
  void allgather(const double* in, double* out, long long count) {
    ++collectives;
    if (C->allgather(C->ctx, in, out, (int64_t)count, S) != 0)
      throw DriverError{SSNAL_E_DEVICE, "sharded all-gather failed"};
  }

  template <class F>
  void timed(int op, double bytes, F&& f) {
    op_bytes[op] += bytes;
    ++op_calls[op];
    if (!O.profile) {
      f();
      return;
    }
    cudaEvent_t e0 = prof.get(), e1 = prof.get();
    ck(cudaEventRecord(e0, S));
    f();
    ck(cudaEventRecord(e1, S));
    prof.recs.push_back({op, e0, e1});
  }

  double a_bytes() const {
    if (P.csr)  // values + column indices + row pointers (+ labels)
      return 12.0 * P.csr->nnz + 8.0 * P.n_phys + (P.row_sign ? 8.0 * P.n_phys : 0.0);
    return 8.0 * P.n_phys * P.q + (P.row_sign ? 8.0 * P.n_phys : 0.0);
  }

  void cg_report(long long p) {
    cg_iters += (long long)H->cg[6];
    if (std::getenv("SSNAL_DEBUG_CG"))
      std::fprintf(stderr, "cg p=%lld sigma=%.3g it=%d |r|=%.3e |res|=%.3e tol=%.3e done=%g\n", p,
                   sigma, (int)H->cg[6], std::sqrt(H->cg[0]), std::sqrt(H->cg[3]),
                   std::sqrt(H->cg[4]), H->cg[5]);
  }

  // zq = X_J v on the packed J rows with cgs[7] = a_J . zq folded in
  void xd_dot(long long p, const double* v) {
    ck(launch_csrj_xd_dot(L.cj, p, v, L.cg_zq, L.cg_aJ, L.cgs + 7, L.cg_part,
                          (int)cg_part_doubles(P.n) - 8, reinterpret_cast<unsigned int*>(L.cgs + 8),
                          S));
    allsum(L.cgs + 7, 1);
  }

  // X_J^T w over the J-restricted CSC (all-reduced when sharded)
  void cscj_xt(const double* w, double* out) {
    ck(launch_cscj_xt(*P.csr, L.cj, w, out, L.csc_part, S));
    allsum(out, P.q);
  }

  // Gate of the CG's true-residual test (cg_adapt): rho2 = (true residual)^2 / ||r||^2 at
  // the last test, rr0 the recurrence ||r||^2 read just before it.
  struct CheckGate {
    double rho2 = -1.0, rr0 = 0.0;
    int skipped = 0;
  };
  // after a batch: 1 = run the test now, 0 = skip it (next batch), -1 = the CG flagged
  // done (breakdown / exact solve).  Reads the device scalars (one small sync).
  int gate_peek(CheckGate& g, bool more) {
    if (!cg_adapt()) return 1;
    ck(cudaMemcpyAsync(H->cg, L.cgs, sizeof(double) * 8, cudaMemcpyDeviceToHost, S));
    ck(cudaStreamSynchronize(S));
    ++syncs;
    if (H->cg[5] != 0.0) return -1;
    g.rr0 = H->cg[3];
    if (g.rho2 > 0.0 && more && g.skipped < 3 && g.rr0 * g.rho2 > 4.0 * H->cg[4]) {
      ++g.skipped;
      return 0;
    }
    return 1;
  }
  // after a test that did not pass: H->cg[3] holds the true residual squared
  void gate_update(CheckGate& g) {
    g.rho2 = g.rr0 > 0.0 ? H->cg[3] / g.rr0 : -1.0;
    g.skipped = 0;
  }

  // Factor-space Jacobi-preconditioned CG for p >= q (Zipf-hot columns make the
  // sample-space spectrum spread; column scaling flattens it):
  //   (I_q + sigma X_J^T P_J X_J) t = -X^T s,  D = diag(.)  (ref solver.py:151-172 role)
  // Newton residual of d = -s - sigma P~ X t:  sigma X X_J^T P_J X_J r_t.
  bool cg_direction_q(long long p, double asa, const double* g2_dev, int max_it) {
    const CsrOp& op = *P.csr;
    const long long q = P.q;
    ck(launch_gather(L.J, p, P.a, L.cg_aJ, S));
    cscj_xt(L.cg_aJ, L.cg_u);  // u = X_J^T a_J
    ck(launch_csc_colsq(op, L.fr, L.cg_d, L.csc_part, S));
    allsum(L.cg_d, q);
    ck(launch_cg_jacobi(q, L.cg_d, L.cg_u, asa, sigma, L.cg_d, S));
    ck(launch_vec(4, q, -1.0, L.gr, nullptr, nullptr, L.cg_b, S));
    ck(launch_cg_init(q, L.cg_b, L.cg_y, L.cg_r, L.cg_pv, L.cg_d, g2_dev,
                      std::min(O.eta, cg_eta_cap()), O.tau, L.cgs, L.cg_part, S));
    // v (q) -> out (q) = sigma-free part X_J^T P X_J v, via zq (p) and ys (n)
    auto gram_apply = [&](const double* v, double* out) {
      xd_dot(p, v);
      ck(launch_cg_project(p, L.cg_zq, L.cg_aJ, L.cgs + 7, asa, L.cg_w, S));
      cscj_xt(L.cg_w, out);
    };
    CheckGate gate;
    for (int it = 0; it < max_it;) {
      for (int b = 0; b < cg_batch() && it < max_it; ++b, ++it) {
        if (cg_fused()) {
          // X_J^T P zq = X_J^T zq - (a_J.zq / a'a) u with u = X_J^T a_J (the Jacobi setup's):
          // no projection pass, and the vector updates of the iteration in one launch
          xd_dot(p, L.cg_pv);
          cscj_xt(L.cg_zq, L.tq);
          ck(launch_cg_update(q, L.cg_y, L.cg_r, L.cg_pv, L.tq, L.cg_u, asa, sigma, L.cg_d,
                              L.cg_Ap, L.cg_z, L.cgs, L.cg_part, S));
          continue;
        }
        gram_apply(L.cg_pv, L.tq);
        ck(launch_cg_ap(q, L.cg_pv, L.tq, L.tq, 0.0, sigma, L.cg_Ap, L.cgs, L.cg_part, S));
        ck(launch_cg_step(q, L.cg_y, L.cg_r, L.cg_pv, L.cg_Ap, L.cg_d, L.cg_z, L.cgs, L.cg_part,
                          S));
        ck(launch_cg_dir(q, L.cg_z, L.cg_pv, L.cgs, S));
      }
      if (cg_rule() == 0) {
        const int g = gate_peek(gate, it < max_it);
        if (g < 0) break;
        if (g == 0) continue;
      }
      if (cg_rule() == 1) {
        xd_dot(p, L.cg_r);
        ck(launch_cg_project(p, L.cg_zq, L.cg_aJ, L.cgs + 7, asa, L.cg_w, S));
        dots({{L.cg_w, L.cg_w}}, L.cgs + 10, p);
        ck(launch_cg_check_final(L.cgs + 10, 1.0, L.cgs, S));
      } else {
        gram_apply(L.cg_r, L.tq);
        ck(launch_csr_xd(op, nullptr, P.n_phys, L.tq, L.tmp, S));
        if (sh()) {  // ||X (.)||^2 is a sum over the slots: all-reduced before the test
          dots({{L.tmp, nullptr}}, L.cgs + 10, P.n);
          ck(launch_cg_check_final(L.cgs + 10, sigma, L.cgs, S));
        } else {
          ck(launch_cg_check(P.n, L.tmp, sigma, L.cgs, L.cg_part, S));
        }
      }
      ck(cudaMemcpyAsync(H->cg, L.cgs, sizeof(double) * 8, cudaMemcpyDeviceToHost, S));
      ck(cudaStreamSynchronize(S));
      ++syncs;
      if (H->cg[5] != 0.0) break;
      gate_update(gate);
    }
    cg_report(p);
    ck(cudaMemcpyAsync(L.t, L.cg_y, sizeof(double) * q, cudaMemcpyDeviceToDevice, S));
    return H->cg[5] != 0.0;
  }

  // sample-space CG for the sparse operator: t = -X^T s + sigma X_J^T P_J y
  bool cg_direction(long long p, double asa, const double* g2_dev, int max_it) {
    const CsrOp& op = *P.csr;
    ck(launch_gather(L.J, p, L.grad, L.cg_gJ, S));
    ck(launch_gather(L.J, p, P.a, L.cg_aJ, S));
    dots({{L.cg_aJ, L.cg_gJ}}, L.cgs + 7, p);
    ck(launch_cg_project(p, L.cg_gJ, L.cg_aJ, L.cgs + 7, asa, L.cg_b, S));
    // target min(eta, ||grad||^(1+tau)) (ref solver.py:229) on the TRUE Newton residual,
    // eta capped at SPARSE_CG_ETA: the reference falls back to an exact solve when its CG
    // stalls; the matrix-free path instead solves tighter from the start
    ck(launch_cg_init(p, L.cg_b, L.cg_y, L.cg_r, L.cg_pv, nullptr, g2_dev,
                      std::min(O.eta, cg_eta_cap()), O.tau, L.cgs, L.cg_part, S));
    CheckGate gate;
    for (int it = 0; it < max_it;) {
      for (int b = 0; b < cg_batch() && it < max_it; ++b, ++it) {
        ck(launch_cscj_xt(op, L.cj, L.cg_pv, L.tq, L.csc_part, S));
        xd_dot(p, L.tq);
        if (cg_fused()) {
          ck(launch_cg_update(p, L.cg_y, L.cg_r, L.cg_pv, L.cg_zq, L.cg_aJ, asa, sigma, nullptr,
                              L.cg_Ap, nullptr, L.cgs, L.cg_part, S));
          continue;
        }
        ck(launch_cg_ap(p, L.cg_pv, L.cg_zq, L.cg_aJ, asa, sigma, L.cg_Ap, L.cgs, L.cg_part, S));
        ck(launch_cg_step(p, L.cg_y, L.cg_r, L.cg_pv, L.cg_Ap, nullptr, nullptr, L.cgs, L.cg_part,
                          S));
        ck(launch_cg_dir(p, L.cg_r, L.cg_pv, L.cgs, S));
      }
      // Newton residual of the direction built from y (Algorithm 3 Step 1 test):
      // (Q + sigma Q P~ Q) d + Q s = sigma^2 X X_J^T P Q_JJ P r
      if (cg_rule() == 1) {
        ck(launch_cg_check_final(L.cgs + 3, 1.0, L.cgs, S));
        ck(cudaMemcpyAsync(H->cg, L.cgs, sizeof(double) * 8, cudaMemcpyDeviceToHost, S));
        ck(cudaStreamSynchronize(S));
        ++syncs;
        if (H->cg[5] != 0.0) break;
        continue;
      }
      {
        const int g = gate_peek(gate, it < max_it);
        if (g < 0) break;
        if (g == 0) continue;
      }
      dots({{L.cg_aJ, L.cg_r}}, L.cgs + 7, p);
      ck(launch_cg_project(p, L.cg_r, L.cg_aJ, L.cgs + 7, asa, L.cg_w, S));
      ck(launch_cscj_xt(op, L.cj, L.cg_w, L.tq, L.csc_part, S));
      xd_dot(p, L.tq);
      ck(launch_cg_project(p, L.cg_zq, L.cg_aJ, L.cgs + 7, asa, L.cg_w, S));
      ck(launch_cscj_xt(op, L.cj, L.cg_w, L.tq, L.csc_part, S));
      ck(launch_csr_xd(op, nullptr, P.n_phys, L.tq, L.tmp, S));
      ck(launch_cg_check(P.n, L.tmp, sigma * sigma, L.cgs, L.cg_part, S));
      ck(cudaMemcpyAsync(H->cg, L.cgs, sizeof(double) * 8, cudaMemcpyDeviceToHost, S));
      ck(cudaStreamSynchronize(S));
      ++syncs;
      if (H->cg[5] != 0.0) break;
      gate_update(gate);
    }
    cg_report(p);
    // w = P_J y, t = -g_r + sigma X^T scatter(w)
    dots({{L.cg_aJ, L.cg_y}}, L.cgs + 7, p);
    ck(launch_cg_project(p, L.cg_y, L.cg_aJ, L.cgs + 7, asa, L.cg_w, S));
    sparse_t_from_sample(L.cg_w, p, true);
    return H->cg[5] != 0.0;
  }

  // Column-popularity spread of A (max / mean column sum of squares), once per solve:
  // a large spread (Zipf-hot columns) selects the Jacobi-preconditioned factor-space
  // CG even when p < q.
  bool hot_columns() {
    if (col_spread < 0.0) {
      ck(cudaMemsetAsync(L.tfree, 1, P.n, S));
      ck(launch_csc_colsq(*P.csr, L.tfree, L.cg_d, L.csc_part, S));
      allsum(L.cg_d, P.q);
      std::vector<double> cs(P.q);
      ck(cudaMemcpyAsync(cs.data(), L.cg_d, sizeof(double) * P.q, cudaMemcpyDeviceToHost, S));
      ck(cudaStreamSynchronize(S));
      double mx = 0.0, sum = 0.0;
      for (double v : cs) { mx = std::max(mx, v); sum += v; }
      col_spread = sum > 0.0 ? mx / (sum / P.q) : 1.0;
    }
    return col_spread > HOT_COLUMN_SPREAD;
  }
  double col_spread = -1.0;

  // matrix-free reduced Newton solve; on CG failure fall back to the direct system
  // when it fits (ref solver.py:251-255), else keep iterating up to 4x the budget
  // (p: global free count for the routing; pl: this rank's, the size of its J)
  // sharded: always the factor-space CG (the sample-space system couples the ranks' J)
  void sparse_iterative(long long p, long long pl, double asa, const double* g2_dev) {
    const bool can_direct = sh() ? P.q <= SPARSE_DIRECT_MAX
                                 : std::min<long long>(p, P.q) <= SPARSE_DIRECT_MAX;
    const int max_it = can_direct ? O.cg_max_iters : 4 * O.cg_max_iters;
    ck(launch_cscj_build(*P.csr, L.fr, L.J, pl, L.cj, S));  // X_J's CSC for every CG product
    const bool ok = (!sh() && p < P.q && !hot_columns()) ? cg_direction(p, asa, g2_dev, max_it)
                                                         : cg_direction_q(pl, asa, g2_dev, max_it);
    if (O.profile) {
      // algorithmic bytes of the CG phase (profiled solves only: one extra 8-byte read):
      // per iteration the two products stream nnz(X_J) (value, index) pairs each, 12 B,
      // and the vector updates make ~9 passes over the system vectors
      int64_t nnzj = 0;
      ck(cudaMemcpyAsync(&nnzj, L.cj.rptr + pl, sizeof nnzj, cudaMemcpyDeviceToHost, S));
      ck(cudaStreamSynchronize(S));
      op_bytes[SSNAL_OP_NEWTON] += H->cg[6] * (24.0 * (double)nnzj + 72.0 * (double)std::min<long long>(p, P.q));
    }
    if (!ok && can_direct) {
      ++cg_fallbacks;
      sparse_direct(p, pl, asa);
    }
  }

  // t = -g_r + sigma X_J^T w  for a sample-space w (p, already in range(P_J))
  void sparse_t_from_sample(const double* w, long long p, bool cj = false) {
    if (cj) {
      ck(launch_cscj_xt(*P.csr, L.cj, w, L.tq, L.csc_part, S));
    } else {
      ck(launch_scatter(L.J, p, w, L.ys, S));
      ck(launch_csc_xt(*P.csr, L.ys, L.tq, L.csc_part, S));
      ck(launch_scatter_zero(L.J, p, L.ys, S));
    }
    ck(launch_vec(4, P.q, sigma, L.tq, nullptr, nullptr, L.t, S));  // sigma X^T P_J y
    ck(launch_vec(3, P.q, 0.0, L.t, L.gr, nullptr, L.t, S));       // - X^T s
  }

  // direct reduced systems for the sparse operator (ref solver.py:238-246):
  //   p < q : Q_JJ by sparse row merges, (I + sigma P Q_JJ P) y = P g_J, t from y;
  //   p >= q: X_J^T X_J by masked column merges, (I + sigma X_J^T P X_J) t = -X^T s.
  void sparse_direct(long long p, long long pl, double asa) {
    const CsrOp& op = *P.csr;
    if (p < P.q && !sh()) {
      ck(launch_sparse_gram_rows(op, L.J, p, L.M, S));
      double* y = (double*)L.ws_ps + 3 * p;
      ck(launch_pspace_solve(L.J, p, L.grad, P.a, sigma, asa, L.M, (double*)L.ws_ps, y, L.info,
                             S));
      sparse_t_from_sample(y, p);
      return;
    }
    ck(launch_sparse_gram_cols(op, L.fr, L.M, S));
    allsum(L.M, P.q * P.q);
    // u = X_J^T a_J (the rank-one correction's factor vector)
    ck(launch_gather(L.J, pl, P.a, L.cg_aJ, S));
    ck(launch_scatter(L.J, pl, L.cg_aJ, L.ys, S));
    ck(launch_csc_xt(op, L.ys, L.tq, L.csc_part, S));
    ck(launch_scatter_zero(L.J, pl, L.ys, S));
    allsum(L.tq, P.q);
    ck(launch_qspace_assemble(P.q, L.tq, asa, sigma, L.M, S));
    ck(launch_chol_solve(L.M, P.q, L.gr, -1.0, L.t, L.info, S));
  }

  // ---------------------------------------------------------------- plumbing
  // one D2H copy of the blob prefix that holds the scalars, info and the T states
  // SSNAL_TRACE_SYNC: GPU idle across each host decision = (event recorded right
  // after the host resumes) - (event recorded before the sync), summed and printed
  cudaEvent_t tr_a = nullptr, tr_b = nullptr;
  double tr_idle = 0.0;
  long long tr_n = 0;
  bool tr_on = std::getenv("SSNAL_TRACE_SYNC") != nullptr;
  void trace_resume() {
    if (!tr_on || !tr_a) return;
    ck(cudaEventRecord(tr_b, S));
    ck(cudaEventSynchronize(tr_b));
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, tr_a, tr_b));
    tr_idle += ms;
    ++tr_n;
  }

  void fetch(const ProjState* states, int T, bool info) {
    if (tr_on) {
      if (!tr_a) {
        cudaEventCreate(&tr_a);
        cudaEventCreate(&tr_b);
      }
      ck(cudaEventRecord(tr_a, S));
    }
    const char* base = reinterpret_cast<const char*>(L.scal);
    size_t st_off = 0, bytes = 128 + sizeof(int);
    if (states) {
      st_off = (size_t)(reinterpret_cast<const char*>(states) - base);
      bytes = st_off + sizeof(ProjState) * T;
    }
    const unsigned int seq = H->seq + 1u;
    note_launch();
    publish_kernel<<<1, 256, 0, S>>>(reinterpret_cast<const unsigned int*>(base),
                                     (unsigned int)((bytes + 3) / 4),
                                     reinterpret_cast<unsigned int*>(H->blob), &H->seq, seq);
    ck(cudaGetLastError());
    // spin on the sequence word; every 4096 polls ask the stream whether it failed or
    // drained without publishing (then fall back to a plain synchronize)
    for (unsigned long long spin = 1;; ++spin) {
      if (H->seq == seq) break;
      if ((spin & 4095u) == 0u) {
        const cudaError_t q = cudaStreamQuery(S);
        if (q != cudaSuccess && q != cudaErrorNotReady) ck(q);
        if (q == cudaSuccess && H->seq != seq) {
          ck(cudaStreamSynchronize(S));
          if (H->seq != seq) throw DriverError{SSNAL_E_DEVICE, "read-back did not publish"};
        }
      }
    }
    ++syncs;
    std::memcpy(H->scal, H->blob, sizeof(double) * NSCAL);
    if (info) std::memcpy(&H->info, H->blob + 128, sizeof(int));
    if (states) std::memcpy(H->st, H->blob + st_off, sizeof(ProjState) * T);
  }

  void project(const double* A, ProjState* st, int T, const double* B, const double* coefs,
               double* xo, uint8_t* fo, const double* ref, double hint, int newton_passes = 3,
               int passes = 0, int phases = 4, const double* hints = nullptr) {
    if (sh()) {  // continuation (finish) when called without Newton passes
      project_sharded(A, st, T, B, coefs, xo, fo, ref, hint, hints, newton_passes == 0,
                      newton_passes == 0 ? 8 : std::max(newton_passes, 1));
      return;
    }
    ProjLaunch pl;
    pl.hints = hints;
    pl.A = A; pl.B = B; pl.coef = coefs; pl.a = P.a; pl.l = P.l; pl.u = P.u;
    pl.lc = P.l_const; pl.uc = P.u_const; pl.d = P.d; pl.n = P.n; pl.T = T;
    pl.st = st; pl.part = (double*)L.ws_proj; pl.x_out = xo; pl.free_out = fo; pl.ref = ref;
    pl.phases = phases; pl.passes = passes; pl.hint = hint; pl.newton = newton_passes;
    if (B && O.psi_stable == 2) {  // line-search trials: psi differences from the base point
      pl.base = L.xp;
      pl.base_lam = lam_cur;
    }
    if (B && xo == L.tx) {  // a line-search batch: x / mask of the accepted trial only
      pl.defer = 1;
      trial_deferred = proj_defers(P.n, T);
      if (qgrad() && slope_ok && !hints) {
        // lambda(alpha) ~ lam_cur - sigma alpha a_J'(Qd)_J / a_J'a_J: the direction
        // epilogue's fold (ws_grad + 128) and the base point's a_J'a_J
        pl.slope_num = reinterpret_cast<const double*>(static_cast<const char*>(L.ws_grad) + 128);
        pl.slope_den = &L.st_cur->sum_a2_free;
      }
    }
    // algorithmic bytes: each streaming launch reads v (+B), a (+l, u vectors); apply
    // also writes x and the mask
    const double per = 8.0 * P.n * (2 + (B != nullptr) + (P.l != nullptr) + (P.u != nullptr));
    const double bytes = T * (per * (newton_passes + passes + 1) +
                              (xo ? 8.0 * P.n : 0.0) + (fo ? 1.0 * P.n : 0.0));
    timed(SSNAL_OP_PROJ, bytes, [&] { ck(launch_project(pl, S)); });
    ++projections;
  }

  // Row-sharded projection (dist.cu): unless continuing, the search state starts at the
  // warm start; `passes` passes of eval -> all-gather of the 5-double records ->
  // rank-ordered fold + Newton step, then apply (x / mask rank-locally) -> all-gather ->
  // global records.  A trial still searching comes back with status != APPLIED and
  // finish() continues it.
  void project_sharded(const double* A, ProjState* st, int T, const double* B,
                       const double* coefs, double* xo, uint8_t* fo, const double* ref,
                       double hint, const double* hints, bool cont, int passes) {
    ShardProj sp{};
    sp.A = A; sp.B = B; sp.a = P.a; sp.l = P.l; sp.u = P.u;
    sp.lc = P.l_const; sp.uc = P.u_const; sp.d = P.d; sp.n = P.n; sp.T = T;
    for (int t = 0; t < T; ++t) {
      sp.coef[t] = B ? coefs[t] : 0.0;
      sp.hints[t] = hints ? hints[t] : hint;
    }
    sp.has_hints = hints != nullptr;
    sp.hint = hint;
    if (B && xo == L.tx && qgrad() && slope_ok && !hints) {
      sp.slope_num = reinterpret_cast<const double*>(static_cast<const char*>(L.ws_grad) + 128);
      sp.slope_den = &L.st_cur->sum_a2_free;
    }
    sp.x_out = xo; sp.free_out = fo; sp.ref = ref;
    if (B && O.psi_stable == 2) {
      sp.base = L.xp;
      sp.base_lam = lam_cur;
    }
    trial_deferred = false;
    const double per = 8.0 * P.n * (2 + (B != nullptr) + (P.l != nullptr) + (P.u != nullptr));
    const double bytes = T * (per * (passes + 1) + (xo ? 8.0 * P.n : 0.0) + (fo ? 1.0 * P.n : 0.0));
    timed(SSNAL_OP_PROJ, bytes, [&] {
      if (!cont) ck(launch_sproj_init(sp, L.sp, S));
      for (int k = 0; k < passes; ++k) {
        ck(launch_sproj_eval(sp, L.sp, (double*)L.ws_plocal, L.rec_loc, S));
        allgather(L.rec_loc, L.rec_all, 8LL * T);
        ck(launch_sproj_update(C->world, T, L.rec_all, P.d, L.sp, S));
      }
      ck(launch_sproj_apply(sp, L.sp, (double*)L.ws_plocal, L.rec_loc, S));
      allgather(L.rec_loc, L.rec_all, 8LL * T);
      ck(launch_sproj_finish(C->world, T, L.rec_all, L.rec_loc, L.sp, sp.base != nullptr, st, S));
    });
    ++projections;
  }

  static void raise_status(int s) {
    if (s == PROJ_INFEASIBLE_LOW || s == PROJ_INFEASIBLE_HIGH)
      throw DriverError{SSNAL_E_ARG, "projection bracket failed: constraint set infeasible"};
  }

  // rare: a trial needed more bracketing than the default launch
  bool finish(ProjState* st_dev, int T, const double* A, const double* B, const double* coefs,
              double* xo, uint8_t* fo, const double* ref) {
    static const bool dbg_proj = std::getenv("SSNAL_DEBUG_PROJ") != nullptr;
    if (dbg_proj)
      for (int t = 0; t < T; ++t)
        std::fprintf(stderr, "proj T=%d t=%d passes=%d status=%d nfree=%lld lam=%.17g lo=%.17g hi=%.17g\n",
                     T, t, H->st[t].passes, H->st[t].status, (long long)H->st[t].nfree,
                     H->st[t].lam, H->st[t].lo, H->st[t].hi);
    bool extra = false;
    for (int round = 0;; ++round) {
      bool pending = false;
      for (int t = 0; t < T; ++t) {
        raise_status(H->st[t].status);
        if (H->st[t].status != PROJ_APPLIED) pending = true;
      }
      if (!pending) return extra;
      if (round > 20) throw DriverError{SSNAL_E_ARG, "projection failed to bracket the multiplier"};
      if (!extra) ++proj_fallbacks;
      extra = true;
      if (dbg_proj)
        for (int t = 0; t < T; ++t)
          std::fprintf(stderr, "  round %d t=%d passes=%d status=%d lam=%.17g lo=%.17g hi=%.17g\n",
                       round, t, H->st[t].passes, H->st[t].status, H->st[t].lam, H->st[t].lo,
                       H->st[t].hi);
      project(A, st_dev, T, B, coefs, xo, fo, ref, 0.0, 0, 8, PHASE_EXACT | PHASE_APPLY);
      fetch(st_dev, T, false);
    }
  }

  // sums over the dual slots are rank-local partials until all-reduced; sums over
  // q-vectors (replicated on every rank) are not
  void dots(std::initializer_list<std::pair<const double*, const double*>> pairs, double* out,
            long long len, bool replicated = false) {
    const double* xs[8];
    const double* ys[8];
    int k = 0;
    for (auto& pr : pairs) {
      xs[k] = pr.first;
      ys[k] = pr.second;
      ++k;
    }
    timed(SSNAL_OP_VEC, 8.0 * len * 2 * k,
          [&] { ck(launch_dots(k, xs, ys, nullptr, len, out, L.ws_red, S)); });
    if (!replicated) allsum(out, k);
  }

  void vec(int op, double alpha, const double* x, const double* y, const double* z, double* out) {
    const int nin = 1 + (y != nullptr) + (z != nullptr);
    timed(SSNAL_OP_VEC, 8.0 * P.n * (nin + 1),
          [&] { ck(launch_vec(op, P.n, alpha, x, y, z, out, S)); });
  }

  void xt(std::initializer_list<const double*> vs, double* out) {
    const double* arr[4];
    int k = 0;
    for (auto v : vs) arr[k++] = v;
    timed(SSNAL_OP_XT, a_bytes() + 8.0 * k * (P.n + P.q), [&] {
      if (P.csr) {
        for (int j = 0; j < k; ++j) ck(launch_csc_xt(*P.csr, arr[j], out + (size_t)j * P.q,
                                                     L.csc_part, S));
      } else {
        ck(launch_dense_xt(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, k, arr, out,
                           L.ws_xt, S));
      }
    });
    allsum(out, (long long)k * P.q);
  }

  void xd(const double* d, double* out, int k) {
    timed(SSNAL_OP_XD, a_bytes() + 8.0 * k * (P.n + P.q), [&] {
      if (P.csr) {
        for (int j = 0; j < k; ++j)
          ck(launch_csr_xd(*P.csr, nullptr, P.n_phys, d + (size_t)j * P.q, out + (size_t)j * P.n, S));
      } else {
        ck(launch_dense_x(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, k, d, out, S));
      }
    });
  }

  double psi(double wqw, const ProjState& r, double x_sq) const {
    const double diff = O.psi_stable ? r.sum_xv : (r.sum_v2 - r.sum_r2);
    return 0.5 * wqw + diff / (2.0 * sigma) - x_sq / (2.0 * sigma);
  }

  // ---------------------------------------------------------------- outer pieces
  // returns residual; p and objective through refs; refreshes Qw when w given
  bool cold_zero = false;  // x = w = 0 (cold start, first outer iteration)

  double kkt_and_refresh(double* x, double* w, double* qw_out, long long& p, double& obj) {
    if (w && cold_zero) {
      // X^T [x, w] = 0 and Q x = Q w = 0: no sweep of A needed
      ck(cudaMemsetAsync(L.gr, 0, sizeof(double) * 2 * P.q, S));
      ck(cudaMemsetAsync(L.qx, 0, sizeof(double) * P.n, S));
      ck(cudaMemsetAsync(qw_out, 0, sizeof(double) * P.n, S));
      cold_zero = false;
    } else if (w) {
      xt({x, w}, L.gr);
      xd(L.gr, L.qwx, 2);
      ck(cudaMemcpyAsync(L.qx, L.qwx, sizeof(double) * P.n, cudaMemcpyDeviceToDevice, S));
      ck(cudaMemcpyAsync(qw_out, L.qwx + P.n, sizeof(double) * P.n, cudaMemcpyDeviceToDevice, S));
    } else {
      xt({x}, L.gr);
      xd(L.gr, L.qx, 1);
    }
    vec(1, 0.0, x, L.qx, P.c, L.tmp);
    project(L.tmp, L.st_kkt, 1, nullptr, nullptr, nullptr, nullptr, x, lam_kkt);
    dots({{x, nullptr}, {x, L.qx}, {P.c, x}}, L.scal, P.n);
    fetch(L.st_kkt, 1, false);
    const double xx = H->scal[0], xqx = H->scal[1], cx = H->scal[2];
    finish(L.st_kkt, 1, L.tmp, nullptr, nullptr, nullptr, nullptr, x);
    lam_kkt = H->st[0].lam;
    p = H->st[0].nfree;
    obj = 0.5 * xqx + cx;
    return std::sqrt(H->st[0].sum_dref2) / (1.0 + std::sqrt(xx));
  }

  // ---------------------------------------------------------------- inner pieces
  // s = w - Pi(u), g_r = X^T s, grad = X g_r; with g2: ||grad||^2 into that device slot
  // (dense: one fused call, csrc/dense.cu launch_dense_gradient)
  void gradient(double* g2 = nullptr) {
    if (!P.csr) {
      // both sweeps of A (X^T then X) are accounted to the X^T class
      timed(SSNAL_OP_XT, 2.0 * a_bytes() + 8.0 * (4 * P.n + 2 * P.q), [&] {
        ck(launch_dense_gradient(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.w, L.xp,
                                 L.s, L.gr, L.grad, g2 ? g2 : L.scal + NSCAL - 1, L.ws_grad, S));
      });
      return;
    }
    vec(3, 0.0, L.w, L.xp, nullptr, L.s);
    xt({L.s}, L.gr);
    xd(L.gr, L.grad, 1);
    if (g2) dots({{L.grad, nullptr}}, g2, P.n);
  }

  // start of an inner solve (dense): s = w - Pi(u), r = X^T s (one sweep), X^T Pi = X^T w - r
  void start_factor() {
    timed(SSNAL_OP_XT, a_bytes() + 8.0 * (3 * P.n + P.q), [&] {
      ck(launch_gradient_factor(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.w, L.xp,
                                L.s, L.r, L.ws_grad, S));
    });
    allsum(L.r, P.q);
    ck(launch_vec(3, P.q, 0.0, L.xw, L.r, nullptr, L.xpi, S));
  }

  bool slope_ok = false;  // ws_grad + 128 holds a_J'(Qd)_J of the current direction
  // the kept Gram G / m1 describe the CURRENT free set and the direction is the Newton
  // one (Qd = X t): the accept pass may use the linear update over the staying free slots
  bool lin_ok = false;

  void direction(long long p, double asa, const double* g2_dev) {
    tdir = L.t;
    slope_ok = false;
    lin_ok = false;
    if (p == 0) {  // Sigma = 0: d = -s, Qd = -grad (ref solver.py:221-222)
      if (qgrad()) {  // grad = X r (one sweep, ||grad||^2 folded); t = X^T d = -r
        timed(SSNAL_OP_XD, a_bytes() + 8.0 * (P.n + P.q), [&] {
          ck(launch_grad_from_factor(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.r,
                                     L.grad, L.scal + 4, L.ws_grad, S));
        });
        allsum(L.scal + 4, 1);
        ck(launch_vec(4, P.q, -1.0, L.r, nullptr, nullptr, L.t, S));
      }
      vec(4, -1.0, L.s, nullptr, nullptr, L.dir);
      vec(4, -1.0, L.grad, nullptr, nullptr, L.qdir);
      dots({{L.grad, L.dir}, {L.w, L.qw}, {L.w, L.qdir}, {L.s, L.grad}}, L.scal, P.n);
      return;
    }
    if (P.csr) {  // direct when min(p, q) is small, else matrix-free sample-space CG
      const long long lim = std::min<long long>(O.direct_solve_threshold, SPARSE_DIRECT_MAX);
      // sharded: only the q x q direct system (the p x p one couples the ranks' J)
      const bool direct = sh() ? P.q <= lim : std::min<long long>(p, P.q) <= lim;
      const long long pl = sh() ? cur_local : p;
      timed(SSNAL_OP_NEWTON, 0.0, [&] {
        ck(launch_compact(L.fr, P.n, L.J, L.pcount, L.ws_cmp, S));
        if (direct) sparse_direct(p, pl, asa);
        else sparse_iterative(p, pl, asa, g2_dev);
      });
      xd(L.t, L.qdir, 1);
      timed(SSNAL_OP_VEC, 8.0 * P.n * 5, [&] {
        if (sh()) {  // {a_J'(Qd)_J, a_J'a_J} summed over the ranks first
          const double* xs[2] = {P.a, P.a};
          const double* ys[2] = {L.qdir, nullptr};
          ck(launch_dots(2, xs, ys, L.fr, P.n, L.hsum, L.ws_red, S));
          allsum(L.hsum, 2);
          ck(launch_hs_finish(L.fr, P.a, L.qdir, P.n, -sigma, L.s, -1.0, L.dir, L.hsum, S));
        } else {
          ck(launch_hs_apply(L.fr, P.a, L.qdir, P.n, -sigma, L.s, -1.0, L.dir, L.ws_red, S));
        }
      });
      if (!direct) {
        // inexact y: X t is not Q d.  Recompute the exact image (t = X^T d, Qd = X t)
        // so Qw stays Q w along the iterates and psi / the Armijo test are exact.
        xt({L.dir}, L.t);
        xd(L.t, L.qdir, 1);
      }
      dots({{L.grad, L.dir}, {L.w, L.qw}, {L.w, L.qdir}}, L.scal, P.n);
      dots({{L.t, nullptr}}, L.scal + 3, P.q, true);
      return;
    }
    // sharded: always the q x q system (the p x p one couples the ranks' free rows)
    const bool qroute = p >= P.q || sh();
    if (sh() && (P.q > O.direct_solve_threshold || P.q > DENSE_QSYS_MAX))
      throw DriverError{SSNAL_E_ARG, "sharded dense solve: q x q system above the direct limit"};
    if (!qroute && p > O.direct_solve_threshold)
      throw DriverError{SSNAL_E_ARG, "p x p system above direct_solve_threshold (no CG path)"};
    if (p >= P.q && P.q > O.direct_solve_threshold)
      throw DriverError{SSNAL_E_ARG, "q x q system above direct_solve_threshold (no CG path)"};
    if (!qroute && p > DENSE_PSYS_MAX)
      throw DriverError{SSNAL_E_ARG, "p x p system above the dense workspace cap (4096)"};
    if (p >= P.q && P.q > DENSE_QSYS_MAX)
      throw DriverError{SSNAL_E_ARG, "q x q system above the dense workspace cap (4096)"};
    // gathered rows of A (p x q) once + the system matrix written and factored
    const double m = (double)std::min<long long>(p, P.q);
    const double* g_r = qgrad() ? L.r : L.gr;
    timed(SSNAL_OP_NEWTON, p < P.q ? 8.0 * p * P.q + 16.0 * m * m : 1.0 * P.n + 4.0 * p, [&] {
      ck(launch_compact(L.fr, P.n, L.J, L.pcount, L.ws_cmp, S));
      if (!qroute) {
        // factor-space gradient: the right-hand side needs grad_J = X_J r only
        if (qgrad())
          ck(launch_rows_grad(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.J, p, L.r,
                              L.grad, S));
        ck(launch_pspace_direction(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.J, p,
                                   L.grad, P.a, sigma, asa, g_r, L.t, L.info, L.ws_ps, S));
      }
    });
    if (qroute) {
      const double* asa_dev = &L.st_cur->sum_a2_free;
      // gathered rows: bytes and flops added once the row count is known (gram_rows)
      timed(SSNAL_OP_GRAM, 0.0, [&] { gram(); });
      lin_ok = accept_lin();
      const double* G = L.G;
      const double* m1 = L.m1;
      if (sh()) {  // the kept Gram is this rank's rows; [G ; m1] summed over the ranks
        const size_t qq = (size_t)P.q * P.q;
        ck(cudaMemcpyAsync(L.Gg, L.G, sizeof(double) * qq, cudaMemcpyDeviceToDevice, S));
        ck(cudaMemcpyAsync(L.Gg + qq, L.m1, sizeof(double) * P.q, cudaMemcpyDeviceToDevice, S));
        allsum(L.Gg, (long long)qq + P.q);
        G = L.Gg;
        m1 = L.Gg + qq;
      }
      const double qd = (double)P.q;
      op_flops[SSNAL_OP_CHOL] += qd * qd * qd / 3.0 + 2.0 * qd * qd;
      timed(SSNAL_OP_CHOL, 24.0 * qd * qd, [&] {
        ck(launch_gram_assemble(G, P.q, m1, sigma, asa_dev, L.M, S));
        ck(launch_chol_solve(L.M, P.q, g_r, -1.0, L.t, L.info, S));
      });
    }
    if (qgrad()) {
      slope_ok = true;
      // ONE sweep X [t, r]: Qd and this point's gradient (a_J'(Qd)_J and ||grad||^2
      // folded), then d = -s - sigma P(Qd) and {g'd, w'Qw, w'Qd, t't}
      // sweep: A + labels, [Qd ; grad] written, mask + a read for the a_J'(Qd)_J fold
      timed(SSNAL_OP_XD, a_bytes() + 16.0 * P.n + 9.0 * P.n + 16.0 * P.q, [&] {
        ck(launch_direction_epilogue_q(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.t,
                                       L.qdir, L.fr, P.a, &L.st_cur->sum_a2_free, L.s, sigma,
                                       L.w, L.qw, L.dir, L.scal, L.scal + 4, L.ws_grad, S, 1));
      });
      if (sh()) {  // a_J'(Qd)_J (P_J's coefficient, the ray slope) and ||grad||^2
        allsum(reinterpret_cast<double*>(static_cast<char*>(L.ws_grad) + 128), 1);
        allsum(L.scal + 4, 1);
      }
      timed(SSNAL_OP_VEC, 8.0 * P.n * 7 + 1.0 * P.n, [&] {
        ck(launch_direction_epilogue_q(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.t,
                                       L.qdir, L.fr, P.a, &L.st_cur->sum_a2_free, L.s, sigma,
                                       L.w, L.qw, L.dir, L.scal, L.scal + 4, L.ws_grad, S, 2));
      });
      allsum(L.scal, 3);  // {g'd, w'Qw, w'Qd}; t't is a q-space (replicated) sum
      return;
    }
    // Qd = X t (a_J'(Qd)_J folded in the sweep), d = -s - sigma P(Qd), and
    // {g'd, w'Qw, w'Qd, t't}: two launches
    timed(SSNAL_OP_XD, a_bytes() + 8.0 * (P.n + P.q) + 8.0 * P.n * 8, [&] {
      ck(launch_direction_epilogue(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.t,
                                   L.qdir, L.fr, P.a, &L.st_cur->sum_a2_free, L.s, sigma, L.grad,
                                   L.w, L.qw, L.dir, L.scal, L.ws_grad, S));
    });
  }

  // Kept q-space Gram G = X_J^T X_J, m1 = X_J^T a_J (sigma-free, valid across outer
  // iterations): each Newton step of the q-space route either rebuilds it from all p
  // free rows or updates it over the slots whose free flag changed since (+x x^T
  // entering, -x x^T leaving) -- whichever gathers fewer rows, decided on the device
  // (gram_select_kernel; SSNAL_GRAM_FULL=1 always rebuilds).  Jd ascending and the
  // fixed split-K order keep it deterministic.
  void gram() {
    static const int force_full = std::getenv("SSNAL_GRAM_FULL") != nullptr ? 1 : 0;
    ck(launch_mask_diff(L.fr, L.frg, L.chg, P.n, S));
    ck(launch_compact(L.chg, P.n, L.Jd, L.dcount, L.ws_cmp, S));
    ck(launch_gram_select(L.gctl, L.pcount, L.dcount, force_full, S));
    ck(launch_gram_update(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, L.J, L.pcount,
                          L.fr, P.a, L.G, L.m1, 0, L.ws_gram, S, L.gctl, L.Jd));
  }

  // dense operator: the SsN gradient is kept in factor space
  bool qgrad() const { return P.csr == nullptr && P.q <= ACCEPT_Q_MAX; }
  const double* tdir = nullptr;  // X^T d of the current direction (factor-space update)

  void steepest(double out[4]) {
    slope_ok = false;
    lin_ok = false;
    vec(4, -1.0, L.grad, nullptr, nullptr, L.dir);
    tdir = L.gr + P.q;
    xt({L.dir}, L.gr + P.q);
    xd(L.gr + P.q, L.qdir, 1);
    dots({{L.grad, L.dir}, {L.w, L.qw}, {L.w, L.qdir}, {L.dir, L.qdir}}, L.scal, P.n);
    fetch(nullptr, 0, false);
    for (int k = 0; k < 4; ++k) out[k] = H->scal[k];
  }

  // [gradient, ||grad||^2] + direction + unit trial, one sync
  void advance(long long p, double asa, bool with_gradient, double& gnorm2, double dotsv[4],
               ProjState& trial0) {
    // dense: the accept pass already produced r = X^T s; grad = X r comes with the
    // direction's sweep
    if (with_gradient && !qgrad()) gradient(L.scal + 4);
    // ||grad||^2 of this point on the device: scal[4] after a gradient, scal[0] at the start
    direction(p, asa, with_gradient ? L.scal + 4 : L.scal + 0);
    // the first Armijo batch (alpha = 1, beta, ..., beta^(T0-1)) is projected
    // speculatively with the direction: most steps then need no further host round trip
    const int T0 = std::min(std::min(TMAX, std::max(1, O.line_search_batch)),
                            proj_wave_trials(P.n, true));
    double coefs[TMAX];
    double alpha = 1.0;
    for (int k = 0; k < T0; ++k) {
      coefs[k] = sigma * alpha;
      alpha *= O.backtrack;
    }
    project(L.u, L.st_trial, T0, L.qdir, coefs, L.tx, L.tfree, L.x, lam_cur);
    fetch(L.st_trial, T0, p > 0);
    if (p > 0 && H->info != 0) throw DriverError{SSNAL_E_ARG, "reduced Newton matrix not SPD"};
    gnorm2 = H->scal[4];
    for (int k = 0; k < 4; ++k) dotsv[k] = H->scal[k];
    finish(L.st_trial, T0, L.u, L.qdir, coefs, L.tx, L.tfree, L.x);
    first_T = T0;
    for (int k = 0; k < T0; ++k) first_batch[k] = H->st[k];
    trial0 = H->st[0];
  }
  ProjState first_batch[TMAX];
  int first_T = 0;

  // Armijo (ref solver.py:292-319); returns false on failure (LineSearchError)
  bool line_search(double gd, double psi0, double wqw, double wqdir, double dqd, double x_sq,
                   const ProjState* first, double& alpha_out, int& j_out, ProjState& rec) {
    if (gd >= 0.0) return false;
    double alpha = 1.0;
    int tried = 0;
    bool have_last = false;
    double lam_last = 0.0, alpha_last = 1.0;
    while (tried < 61) {
      const int T = (tried == 0 && first) ? first_T
                    : tried == 0 ? 1
                                 : std::min(std::min(std::min(TMAX, std::max(1, O.line_search_batch)),
                                                     proj_wave_trials(P.n)),
                                            61 - tried);
      double alphas[TMAX], coefs[TMAX];
      for (int k = 0; k < T; ++k) {
        alphas[k] = alpha;
        coefs[k] = sigma * alpha;
        alpha *= O.backtrack;
      }
      if (tried == 0 && first) {
        for (int k = 0; k < T; ++k) H->st[k] = first[k];
      } else {
        // warm starts along the ray: lambda(alpha) interpolated linearly between the base
        // point (alpha = 0, lam_cur) and the smallest step length already projected
        double hints[TMAX];
        const double* hp = nullptr;
        if (tried > 0 && have_last) {
          for (int k = 0; k < T; ++k)
            hints[k] = lam_cur + (lam_last - lam_cur) * (alphas[k] / alpha_last);
          hp = hints;
        }
        project(L.u, L.st_trial, T, L.qdir, coefs, L.tx, L.tfree, L.x, lam_cur, 3, 0, 4, hp);
        fetch(L.st_trial, T, false);
        finish(L.st_trial, T, L.u, L.qdir, coefs, L.tx, L.tfree, L.x);
      }
      if (T > 0 && H->st[T - 1].status == PROJ_APPLIED) {
        have_last = true;
        lam_last = H->st[T - 1].lam;
        alpha_last = alphas[T - 1];
      }
      for (int k = 0; k < T; ++k) {
        const double a = alphas[k];
        const double quad = wqw + 2.0 * a * wqdir + a * a * dqd;
        // delta mode: psi(w + a d) - psi(w) = a g'd + a^2 d'Qd / 2 + B_h / sigma
        const bool ok = O.psi_stable == 2
                            ? a * gd + 0.5 * a * a * dqd + H->st[k].sum_bh / sigma <= O.mu * a * gd
                            : psi(quad, H->st[k], x_sq) <= psi0 + O.mu * a * gd;
        if (ok) {
          lam_cur = H->st[k].lam;
          alpha_out = a;
          j_out = k;
          rec = H->st[k];
          return true;
        }
      }
      tried += T;
    }
    return false;
  }

  bool trial_deferred = false;  // the last trial batch left x / mask unwritten

  void materialize(double alpha, int j) {
    if (!trial_deferred) return;
    ProjLaunch pl;
    pl.A = L.u; pl.B = L.qdir; pl.a = P.a; pl.l = P.l; pl.u = P.u;
    pl.lc = P.l_const; pl.uc = P.u_const; pl.n = P.n;
    timed(SSNAL_OP_PROJ, 8.0 * P.n * 4 + 1.0 * P.n, [&] {
      ck(launch_proj_materialize(pl, sigma * alpha, L.st_trial + j, L.tx + (size_t)j * P.n,
                                 L.tfree + (size_t)j * P.n, S));
    });
  }

  void accept(double alpha, int j) {
    trace_resume();
    materialize(alpha, j);
    if (qgrad()) {  // + s, and X^T w, X^T Pi(u), r = X^T s updated from the changed slots
      const bool lin = lin_ok && tdir == L.t && L.G != nullptr;
      timed(SSNAL_OP_VEC, 8.0 * P.n * 9 + 2.0 * P.n, [&] {
        if (lin) ck(launch_gram_tvec(L.G, P.q, L.t, L.gt, S));
        ck(launch_accept_q(P.A, P.n_phys, P.q, P.lda, P.row_sign, P.svr_block, P.n, alpha,
                           -(sigma * alpha), L.w, L.dir, L.qw, L.qdir, L.u, L.xp,
                           L.tx + (size_t)j * P.n, L.fr, L.tfree + (size_t)j * P.n, L.s, tdir,
                           L.xw, L.xpi, L.r, L.qpart, L.st_trial + j, L.st_cur, S,
                           sh() ? L.dsum : nullptr, lin ? L.gt : nullptr, L.m1, P.a));
      });
      lin_ok = false;
      if (sh()) {  // X^T (Pi_new - Pi_old) summed over the ranks, then the factor update
        allsum(L.dsum, P.q);
        ck(launch_factor_update(P.q, alpha, tdir, L.dsum, L.xw, L.xpi, L.r, S));
      }
      return;
    }
    timed(SSNAL_OP_VEC, 8.0 * P.n * 8 + 2.0 * P.n, [&] {
      ck(launch_accept(P.n, alpha, -(sigma * alpha), L.w, L.dir, L.qw, L.qdir, L.u, L.xp,
                       L.tx + (size_t)j * P.n, L.fr, L.tfree + (size_t)j * P.n, S));
    });
    ck(cudaMemcpyAsync(L.st_cur, L.st_trial + j, sizeof(ProjState), cudaMemcpyDeviceToDevice, S));
  }

  // ---------------------------------------------------------------- ssn_solve
  // returns inner iterations; sets flags; leaves Pi(u) in L.xp and its record in cur
  int ssn_solve(double eps_k, double delta_k, bool& converged, bool& hit_max, ProjState& cur) {
    const double coeff = std::sqrt(O.lambda_min_surrogate / sigma);
    const bool dbg = std::getenv("SSNAL_DEBUG_CG") != nullptr;
    const double floor_ = 1e-12 * (1.0 + c_norm);
    // start: u = x - sigma (Qw + c), Pi(u), s, grad
    vec(0, -sigma, L.x, L.qw, P.c, L.u);
    project(L.u, L.st_cur, 1, nullptr, nullptr, L.xp, L.fr, L.x, lam_cur);
    if (qgrad()) {
      // X^T w from the outer refresh (kkt_and_refresh), r = X^T s in one sweep,
      // X^T Pi = X^T w - r; the gradient norm comes with the first direction
      ck(cudaMemcpyAsync(L.xw, L.gr + P.q, sizeof(double) * P.q, cudaMemcpyDeviceToDevice, S));
      start_factor();
      dots({{L.x, nullptr}}, L.scal + 1, P.n);
    } else {
      gradient();
      dots({{L.grad, nullptr}, {L.x, nullptr}}, L.scal, P.n);
    }
    fetch(L.st_cur, 1, false);
    double gnorm2 = H->scal[0];
    const double x_sq = H->scal[1];
    if (H->st[0].status != PROJ_APPLIED) {
      finish(L.st_cur, 1, L.u, nullptr, nullptr, L.xp, L.fr, L.x);
      if (qgrad()) {
        start_factor();
      } else {
        gradient();
        dots({{L.grad, nullptr}, {L.x, nullptr}}, L.scal, P.n);
      }
      fetch(nullptr, 0, false);
      gnorm2 = H->scal[0];
    }
    cur = H->st[0];
    cur_local = cur.in_count;
    lam_cur = cur.lam;
    double dv[4];
    ProjState trial0;
    double unused;
    advance(cur.nfree, cur.sum_a2_free, false, unused, dv, trial0);
    if (qgrad()) gnorm2 = unused;  // ||X r||^2 from the direction's sweep
    converged = false;
    bool exhausted = true;
    int its = 0;
    for (int it = 0; it < O.max_inner; ++it) {
      const double gnorm = std::sqrt(gnorm2);
      const double dist = std::sqrt(cur.sum_dref2);
      if (gnorm <= coeff * eps_k && gnorm <= coeff * delta_k * dist) {
        if (dbg) std::fprintf(stderr, "ssn stop it=%d criteria |g|=%.3e\n", it, gnorm);
        converged = true;
        exhausted = false;
        break;
      }
      if (gnorm <= floor_) {
        if (dbg) std::fprintf(stderr, "ssn stop it=%d floor |g|=%.3e\n", it, gnorm);
        converged = true;
        exhausted = false;
        break;
      }
      double gd = dv[0], wqw = dv[1], wqdir = dv[2], dqd = dv[3];
      ++newton;
      bool steepest_dir = false;
      const ProjState* first = first_batch;
      if (gd >= 0.0) {
        double sv[4];
        steepest(sv);
        gd = sv[0]; wqw = sv[1]; wqdir = sv[2]; dqd = sv[3];
        steepest_dir = true;
        first = nullptr;
      }
      const double psi0 = psi(wqw, cur, x_sq);
      // predicted decrease below the resolution of psi (ref solver.py:369-371); the
      // delta mode forms psi differences directly and has no such floor
      if (O.psi_stable != 2 && O.mu * std::fabs(gd) <= 1e-16 * (1.0 + std::fabs(psi0))) {
        if (dbg)
          std::fprintf(stderr, "ssn stop it=%d resolution |g|=%.3e gd=%.3e psi0=%.6e crit=%.3e\n",
                       it, gnorm, gd, psi0, coeff * eps_k);
        converged = true;
        exhausted = false;
        break;
      }
      double alpha;
      int j;
      ProjState rec;
      if (!line_search(gd, psi0, wqw, wqdir, dqd, x_sq, first, alpha, j, rec)) {
        if (steepest_dir) {
          exhausted = false;
          break;
        }
        double sv[4];
        steepest(sv);
        gd = sv[0]; wqw = sv[1]; wqdir = sv[2]; dqd = sv[3];
        if (O.psi_stable != 2 && O.mu * (-gd) <= 1e-16 * (1.0 + std::fabs(psi0))) {
          exhausted = false;
          break;
        }
        if (!line_search(gd, psi0, wqw, wqdir, dqd, x_sq, nullptr, alpha, j, rec)) {
          exhausted = false;
          break;
        }
      }
      if (dbg)
        std::fprintf(stderr, "ssn it=%d |g|=%.3e eps=%.3e dist=%.3e alpha=%.3g steep=%d p=%lld\n",
                     it, gnorm, coeff * eps_k, coeff * delta_k * dist, alpha, (int)steepest_dir,
                     (long long)cur.nfree);
      accept(alpha, j);
      cur = rec;
      cur_local = rec.in_count;
      ++its;
      advance(cur.nfree, cur.sum_a2_free, true, gnorm2, dv, trial0);
    }
    hit_max = exhausted;
    return its;
  }

  // ---------------------------------------------------------------- alm_solve
  void alm_solve(const double* x0, const double* w0, double* x_out, ssnal_report_t* rep,
                 ssnal_progress_fn cb, void* ctx) {
    const auto t0 = std::chrono::steady_clock::now();
    const size_t nb = sizeof(double) * P.n;
    if (x0) ck(cudaMemcpyAsync(L.x, x0, nb, cudaMemcpyDeviceToDevice, S));
    else ck(cudaMemsetAsync(L.x, 0, nb, S));
    if (w0) ck(cudaMemcpyAsync(L.w, w0, nb, cudaMemcpyDeviceToDevice, S));
    else ck(cudaMemsetAsync(L.w, 0, nb, S));
    cold_zero = x0 == nullptr && w0 == nullptr;
    if (sh() && !P.csr && !qgrad())
      throw DriverError{SSNAL_E_ARG, "sharded dense solve needs q <= 2048 (factor-space gradient)"};
    if (P.csr) ck(cudaMemsetAsync(L.cj.ticket, 0, sizeof(unsigned int), S));
    else {
      if (L.qpart) ck(cudaMemsetAsync(L.qpart, 0, 256, S));  // accept_q ticket
      if (L.gctl) ck(cudaMemsetAsync(L.gctl, 0, sizeof(GramCtl), S));  // no kept Gram yet
    }
    ck(cudaMemsetAsync(L.qw, 0, nb, S));
    dots({{P.c, nullptr}}, L.scal, P.n);
    fetch(nullptr, 0, false);
    c_norm = std::sqrt(H->scal[0]);
    sigma = O.sigma0;
    lam_kkt = lam_cur = 0.0;
    int outer = 0, inner_total = 0, inner_last = 0, stalled = 0;
    long long p_last = -1;
    bool converged = false, stagnated = false, max_outer = false;
    int hit_mask = 0, hit_count = 0;
    unsigned long long hit_mask64 = 0ull;
    double res = INFINITY, obj_last = 0.0;
    double best_res = INFINITY, best_obj = 0.0;
    long long best_p = 0;
    bool have_best = false;
    for (int k = 0; k <= O.max_outer; ++k) {
      long long p_kkt;
      res = kkt_and_refresh(L.x, L.w, L.qw, p_kkt, obj_last);
      if (p_last < 0) p_last = p_kkt;
      if (cb) cb(k, res, sigma, p_last, inner_last, ctx);
      if (!have_best || res < best_res) {
        have_best = true;
        best_res = res;
        best_obj = obj_last;
        best_p = p_last;
        ck(cudaMemcpyAsync(L.best_x, L.x, nb, cudaMemcpyDeviceToDevice, S));
        stalled = 0;
      } else if (sigma >= O.sigma_max) {
        if (++stalled >= 3) {
          stagnated = true;
          break;
        }
      }
      if (res < O.tol_kkt) {
        converged = true;
        break;
      }
      if (k == O.max_outer) {
        max_outer = true;
        break;
      }
      bool conv_in, hit;
      ProjState cur;
      const double e = std::pow(0.5, k);
      inner_last = ssn_solve(e, e, conv_in, hit, cur);
      if (hit && k < 31) hit_mask |= 1 << k;
      if (hit && k < 64) hit_mask64 |= 1ull << k;
      if (hit) ++hit_count;
      inner_total += inner_last;
      ck(cudaMemcpyAsync(L.x, L.xp, nb, cudaMemcpyDeviceToDevice, S));
      p_last = cur.nfree;
      sigma = std::min(sigma * O.sigma_growth, O.sigma_max);
      ++outer;
    }
    const bool use_best = have_best && best_res < res;
    ck(cudaMemcpyAsync(x_out, use_best ? L.best_x : L.x, nb, cudaMemcpyDeviceToDevice, S));
    ck(cudaStreamSynchronize(S));
    rep->kkt_residual = use_best ? best_res : res;
    rep->objective = use_best ? best_obj : obj_last;
    rep->unbounded_support_count = (int)(use_best ? best_p : p_last);
    rep->outer_iters = outer;
    rep->total_inner_iters = inner_total;
    rep->converged = converged ? 1 : 0;
    rep->hit_max_inner_mask = hit_mask;
    rep->stagnated = stagnated ? 1 : 0;
    rep->max_outer_reached = max_outer ? 1 : 0;
    rep->syncs = syncs;
    rep->newton_steps = newton;
    rep->projections = projections;
    rep->cg_iters = cg_iters;
    rep->cg_fallbacks = cg_fallbacks;
    GramCtl gc{};
    if (L.gctl) {
      ck(cudaMemcpyAsync(&gc, L.gctl, sizeof(GramCtl), cudaMemcpyDeviceToHost, S));
      ck(cudaStreamSynchronize(S));
    }
    rep->gram_builds = gc.builds;
    rep->gram_updates = gc.updates;
    const long long gram_rows = gc.rows;
    rep->gram_rows = gram_rows;
    op_bytes[SSNAL_OP_GRAM] = 8.0 * (double)gram_rows * P.q;
    op_flops[SSNAL_OP_GRAM] = (double)gram_rows * P.q * (P.q + 1.0);
    rep->proj_fallbacks = proj_fallbacks;
    rep->hit_max_inner_mask64 = hit_mask64;
    rep->hit_max_inner_count = hit_count;
    for (int k = 0; k < SSNAL_NOPS; ++k) {
      rep->op_calls[k] = op_calls[k];
      rep->op_bytes[k] = op_bytes[k];
      rep->op_flops[k] = op_flops[k];
      rep->op_seconds[k] = 0.0;
    }
    for (auto& r : prof.recs) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, r.e0, r.e1));
      rep->op_seconds[r.op] += 1e-3 * ms;
    }
    rep->wall_time =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (tr_on)
      std::fprintf(stderr, "trace: %lld host decisions before accept, GPU idle %.3f ms total\n",
                   tr_n, tr_idle);
  }
};

}  // namespace

size_t alm_ws_bytes(long long n_phys, long long q, int svr, int world) {
  size_t total = 0;
  const long long n = svr ? 2 * n_phys : n_phys;
  carve(nullptr, n, n_phys, q, &total, nullptr, world);
  return total;
}

size_t alm_ws_bytes_csr(const ssnal_csr_operator_t* op, int world) {
  size_t total = 0;
  carve(nullptr, op->n, op->n, op->q, &total, op, world);
  return total;
}

// comm == nullptr: one GPU; else the row-sharded driver over comm's ranks (the problem is
// this rank's slice, d the global right-hand side)
int alm_solve_dense(const ssnal_dense_problem_t* pb, const ssnal_options_t* opt, const double* x0,
                    const double* w0, double* x_out, ssnal_report_t* rep, void* ws,
                    size_t ws_bytes, ssnal_progress_fn cb, void* ctx, cudaStream_t stream,
                    const char** err, const ssnal_comm_t* comm) {
  size_t need = 0;
  const int world = comm ? comm->world : 0;
  Layout L = carve((char*)ws, pb->n, pb->n_phys, pb->q, &need, pb->csr, world);
  if (ws_bytes < need) {
    *err = "workspace smaller than ssnal_alm_ws_bytes()";
    return SSNAL_E_ARG;
  }
  Pinned* H = pinned_buffer();
  if (!H) {
    *err = "cudaHostAlloc of the pinned scalar buffer failed";
    return SSNAL_E_DEVICE;
  }
  std::memset(rep, 0, sizeof(*rep));
  // every last-block ticket, projection record and kept-Gram control word in the
  // workspace starts at zero, whatever the caller allocated it with
  if (cudaMemsetAsync(ws, 0, need, stream) != cudaSuccess) {
    *err = "cudaMemsetAsync of the workspace failed";
    return SSNAL_E_DEVICE;
  }
  Driver d(*pb, *opt, stream, L, H, comm);
  try {
    d.alm_solve(x0, w0, x_out, rep, cb, ctx);
  } catch (const DriverError& e) {
    *err = e.what;
    return e.code;
  }
  return SSNAL_OK;
}

}  // namespace ssnal

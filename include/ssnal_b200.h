/*
 * ssnal_b200.h -- C-ABI of the B200 (sm_100a) SSsNAL hot path.
 *
 * Drop-in boundary for the reference package ``ssnal`` (arXiv 1910.01312,
 * /root/reference/pkg/src/ssnal).  Every entry point names the reference
 * interface it replaces.  Conventions:
 *   - all array arguments are DEVICE pointers (fp64 unless stated), sizes are
 *     int64_t, `stream` is a cudaStream_t passed as void*;
 *   - every call is asynchronous on `stream` and returns 0 on success or a
 *     nonzero code (cudaError_t or SSNAL_E_*); ssnal_last_error() describes it;
 *   - "logical rows": the data operator is X = S (diag(row_sign) A) with A the
 *     row-major n_phys x q sample matrix (leading dimension lda), row_sign an
 *     optional +-1 label vector (C-SVC: X = diag(y) A) and S = [I] or, with
 *     svr_block = 1, S = [I; -I] (eps-SVR: X = [A; -A], 2 n_phys logical rows).
 *     Q = X X^T is never formed (ref kernels.py:68-154 forms its columns).
 *   - every reduction is a fixed-order tree: results are bit-reproducible.
 * No entry point has a CPU fallback.
 */
#ifndef SSNAL_B200_H
#define SSNAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSNAL_OK 0
#define SSNAL_E_ARG 1001      /* invalid argument */
#define SSNAL_E_DEVICE 1002   /* no sm_100 device / wrong architecture */

/* Device-resident record of one projection (one per batched trial). */
typedef struct ssnal_proj_state_t {
  double lo, hi, flo, fhi;        /* current bracket in lambda and phi' values there   */
  double below_max, above_min;    /* nearest breakpoints outside the bracket           */
  double in_min, in_max;          /* extreme breakpoints inside (lo, hi]               */
  long long in_count;             /* breakpoints inside (lo, hi]                       */
  double lam;                     /* equality multiplier lambda-hat (ref lambda_hat)   */
  double tmin, tmax;              /* breakpoint range                                   */
  double sum_v2;                  /* sum v_i^2                                          */
  double sum_r2;                  /* sum (v_i - x_i)^2                                  */
  double sum_dref2;               /* sum (x_i - ref_i)^2 (ref optional)                 */
  double sum_a2_free;             /* a_J' a_J over the free set (a' Sigma a)            */
  double sum_xv;                  /* sum x_i (2 v_i - x_i) = ||v||^2 - ||v - x||^2 without
                                     cancellation (the psi term of ref solver.py:130-133) */
  double sum_bh;                  /* trials with a base point only (sum_v2 is 0 then):
                                     Bregman divergence of h = |.|^2/2 - dist(., K)^2/2
                                     between the trial and the base, psi differences  */
  long long nfree;                /* p = |J|                                            */
  int status;                     /* 3 applied, 2 lambda known, <0 infeasible, else searching */
  int passes;                     /* K-ary bracketing passes used                       */
  unsigned int ticket;            /* internal: last-block-done counter (keep zeroed)    */
  unsigned int pad_;
} ssnal_proj_state_t;

/* ---- library / device ------------------------------------------------- */
const char* ssnal_version(void);
const char* ssnal_last_error(void);
unsigned long long ssnal_launch_count(void);        /* kernels launched by this library */
int ssnal_device_check(int device);                 /* SSNAL_E_DEVICE unless sm_100 */
size_t ssnal_proj_state_bytes(void);
size_t ssnal_report_bytes(void);                   /* sizeof(ssnal_report_t): layout check */
size_t ssnal_project_ws_bytes(int64_t n, int T);
size_t ssnal_reduce_ws_bytes(int64_t n, int k);
size_t ssnal_dense_xt_ws_bytes(int64_t n_phys, int64_t q, int k);
size_t ssnal_gram_ws_bytes(int64_t q);
size_t ssnal_compact_ws_bytes(int64_t n);

/* ---- projection onto {x : a'x = d, l <= x <= u} ------------------------
 * Replaces ref projection.py:152-211 project_box_line (+ :134-149 _classify).
 * Projects T <= 16 vectors v_t = A - coef[t] * B (B may be NULL; coef is a HOST
 * array of T doubles, passed by value to the kernels), each trial t writing
 * state[t] and, when non-NULL, x_out[t*n..] (projection), free_out[t*n..] (uint8
 * free-set mask Sigma) and the fused sums of ssnal_proj_state_t.  l or u NULL =>
 * the scalar l_const / u_const bound for every slot.
 * Root search for lambda: `newton_passes` > 0 runs that many safeguarded Newton
 * passes warm-started at lam_hint (O(1) work per slot per pass, exact on the
 * final affine piece); otherwise phases bit0 starts a K-ary search over the full
 * breakpoint range.  `passes` K-ary passes follow (they take over any unfinished
 * Newton search), then bit1 exact (closes a K-ary bracket onto adjacent
 * breakpoints) and bit2 apply.  Passes after convergence are no-ops.
 * state[t].status == 3 on completion; 0, 1 or 4 means more passes are needed
 * (call again with newton_passes = 0, phases = 6). */
int ssnal_project(const double* A, const double* B, const double* coef,
                  const double* a, const double* l, const double* u,
                  double l_const, double u_const, double d, int64_t n, int T,
                  ssnal_proj_state_t* state, void* ws,
                  double* x_out, uint8_t* free_out, const double* ref,
                  double lam_hint, int newton_passes, int phases, int passes, void* stream);

/* Line-search trials: as ssnal_project, plus the projection base = Pi(u) (multiplier
 * base_lam) of the base point the trials A - coef[t] B start from.  Each record then
 * carries sum_bh = the Bregman divergence of h = |.|^2/2 - dist(., K)^2/2 between
 * trial and base (sum_v2 = 0), from which psi(w + alpha d) - psi(w) is formed without
 * cancellation (ref solver.py:292-319 evaluates psi_t and psi_0 separately). */
int ssnal_project_ex(const double* A, const double* B, const double* coef,
                     const double* a, const double* l, const double* u,
                     double l_const, double u_const, double d, int64_t n, int T,
                     ssnal_proj_state_t* state, void* ws,
                     double* x_out, uint8_t* free_out, const double* ref,
                     const double* base, double base_lam,
                     double lam_hint, int newton_passes, int phases, int passes, void* stream);

/* ---- HS-Jacobian -------------------------------------------------------
 * Replaces ref projection.py:214-225 hs_jacobian_apply.
 * out = alpha * add + beta * P y,  P = S (I - a a'/(a'Sa)) S (or S if a'Sa = 0),
 * S = diag(free).  add may be NULL.  ws: ssnal_reduce_ws_bytes(n, 2). */
int ssnal_hs_apply(const uint8_t* free_mask, const double* a, const double* y, int64_t n,
                   double beta, const double* add, double alpha, double* out,
                   void* ws, void* stream);

/* ---- fused dot products ------------------------------------------------
 * out[j] = sum_i m_i x_j[i] y_j[i], j < k <= 8 (y_j NULL => x_j^2; mask NULL =>
 * all ones).  xs / ys are HOST arrays of k device pointers.  Used for the
 * norms and inner products of ref solver.py:130-148, 303-309, 353-358. */
int ssnal_dots(int k, const double* const* xs, const double* const* ys,
               const uint8_t* mask, int64_t n, double* out, void* ws, void* stream);

/* ---- elementwise vector ops (numpy rounding order) ----------------------
 * op 0: out = x + alpha * (y + z)   (z may be NULL)  -- u(w) = x - sigma (Qw + c)
 * op 1: out = (x - y) - z                            -- x - Qx - c (KKT map)
 * op 2: out = x + alpha * y                          -- w + alpha d, Qw + alpha Qd
 * op 3: out = x - y                                  -- s(w) = w - Pi(u(w))
 * op 4: out = alpha * x
 * op 5: out = x * y (elementwise)                    -- Jacobi preconditioner apply
 * op 6: out = 1 / (1 + alpha * max(x - y, 0))        -- Jacobi inverse diagonal */
int ssnal_vec(int op, int64_t n, double alpha, const double* x, const double* y,
              const double* z, double* out, void* stream);

/* ---- dense data operator (Q = X X^T) -----------------------------------
 * ssnal_dense_xt: out[:, j] = X^T v_j for the k <= 4 logical-length vectors
 *   vs[j] (HOST array of device pointers); out is q x k column-major.
 *   Replaces the X^T half of ref kernels.py:144-154 KernelOperator.matvec.
 * ssnal_dense_x: out[:, j] = X d_j, d q x k column-major, out n_log x k.
 *   The X half of the same matvec, and the Q-image products of
 *   ref solver.py:260-262 (cols @ v).                                       */
int ssnal_dense_xt(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                   const double* row_sign, int svr_block, int k, const double* const* vs,
                   double* out, void* ws, void* stream);
int ssnal_dense_x(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                  const double* row_sign, int svr_block, int k, const double* d,
                  double* out, void* stream);

/* ---- reduced Newton system (Prop. 3.5 in factor space) ------------------
 * ssnal_compact: ascending indices of nonzero mask entries (the free set J)
 *   into idx (int32), count into *count (DEVICE int64).  ref: np.flatnonzero
 *   in projection.py:144-148.
 * ssnal_dense_gram: M = I + sigma (G - m1 m1'/asa) (or I + sigma G when asa = 0)
 *   with G = X_J^T X_J (fp64 tensor cores, DMMA) and m1 = X_J^T a_J over the
 *   *p_dev (DEVICE count, <= p_max) logical rows J; *asa_dev is a'Sigma a (DEVICE
 *   scalar, e.g. state.sum_a2_free).  No host synchronisation is needed.
 *   This is the q x q matrix I_r + sigma L^T Sigma (I - aa'/(a'Sa)) Sigma L of
 *   the paper's Prop. 3.5 proof, which replaces the p x p system assembled in
 *   ref solver.py:232-258.  M is q x q row-major (symmetric).
 * ssnal_chol_solve: in-place Cholesky of the SPD m x m matrix M (lower factor)
 *   and x = scale * M^{-1} b; *info (DEVICE int) = 0 or the failing column+1. */
int ssnal_compact(const uint8_t* mask, int64_t n, int32_t* idx, int64_t* count,
                  void* ws, void* stream);
int ssnal_dense_gram(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                     const double* row_sign, int svr_block,
                     const int32_t* J, const int64_t* p_dev, int64_t p_max, const double* a,
                     double sigma, const double* asa_dev, double* M, double* m1,
                     void* ws, void* stream);
int ssnal_chol_solve(double* M, int64_t m, const double* b, double scale, double* x,
                     int* info, void* stream);

/* ssnal_dense_newton_pspace: the same Newton image through the p x p SPD system
 *   (I_p + sigma P_J Q_JJ P_J) y = P_J grad_J,   t = -g_r + sigma X_J^T (P_J y),
 * (Woodbury dual of ssnal_dense_gram's q x q system; chosen when p < q).  J holds
 * the p logical free rows (host-known p), grad = Q s (n_log), g_r = X^T s (q),
 * asa = a_J'a_J (host scalar).  Writes t (q) and *info (DEVICE int).  This is the
 * p x p route of ref solver.py:224-258 (Q_JJ + rank-one term, dense symmetric
 * solve).  ws: ssnal_pspace_ws_bytes(p, q). */
size_t ssnal_pspace_ws_bytes(int64_t p, int64_t q);
int ssnal_dense_newton_pspace(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                              const double* row_sign, int svr_block, const int32_t* J, int64_t p,
                              const double* grad, const double* a, double sigma, double asa,
                              const double* g_r, double* t, int* info, void* ws, void* stream);

/* ---- sparse (CSR) data operator ------------------------------------------
 * X = diag(row_sign) A with A n x q in CSR (DEVICE arrays) plus its CSC copy and a
 * segment plan for the transposed product (columns cut into segments of <= SEG
 * nonzeros; split columns fold partial slots in order), built once per problem
 * (the Python host builds it with numpy).  Replaces the sparse-sample use of ref
 * kernels.py:68-154 for the linear kernel. */
typedef struct ssnal_csr_operator_t {
  int64_t n, q, nnz;
  const int64_t* indptr;   const int32_t* indices; const double* values;   /* CSR */
  const int64_t* colptr;   const int32_t* rowidx;  const double* valt;     /* CSC */
  const double* row_sign;                                                  /* or NULL */
  int64_t nseg;            /* segments of the CSC product                           */
  const int64_t* seg_beg;  const int64_t* seg_end; const int32_t* seg_col; const int32_t* seg_slot;
  int64_t nfold;           /* split columns                                         */
  const int32_t* fold_col; const int32_t* fold_beg;   /* fold_beg: nfold + 1 entries  */
  int64_t nslots;          /* partial slots (workspace doubles for ssnal_csr_xt)    */
  /* hot-column staging of the CG's X_J d (optional study path, used only with
   * SSNAL_CSR_HOT=1 in the environment; nhot = 0 disables it): the nhot
   * (<= SSNAL_CSR_HOT_MAX) most populated columns, hot_cols[k] = column of rank k,
   * hot_rank[col] = rank or -1.  The packed J rows store ~rank for hot columns and the
   * product reads their d entries from a shared-memory copy instead of gathering.    */
  int64_t nhot;
  const int32_t* hot_cols; const int32_t* hot_rank;   /* nhot / q entries (DEVICE)   */
} ssnal_csr_operator_t;
#define SSNAL_CSR_HOT_MAX 4096

/* out[r] = row_sign[i] * A[i,:] . d for i = rows[r] (rows NULL: i = r), r < nrows */
int ssnal_csr_xd(const ssnal_csr_operator_t* op, const int32_t* rows, int64_t nrows,
                 const double* d, double* out, void* stream);
/* out = X^T v (q), v of length n; ws >= nslots doubles */
int ssnal_csr_xt(const ssnal_csr_operator_t* op, const double* v, double* out, void* ws,
                 void* stream);
/* out = X_J^T w for a p-vector w indexed by position in J (J = ascending rows with
 * keep != 0, p = |J|): builds the J-restricted CSC once (count + ballot compaction)
 * and runs the nnz-balanced segmented product on it.  The CG products of the reduced
 * Newton system (ref solver.py:151-172) use the same two steps.  ws >=
 * ssnal_csr_restricted_ws_bytes(op), zeroed once before first use. */
size_t ssnal_csr_restricted_ws_bytes(const ssnal_csr_operator_t* op);
int ssnal_csr_xt_restricted(const ssnal_csr_operator_t* op, const uint8_t* keep,
                            const int32_t* J, int64_t p, const double* w, double* out, void* ws,
                            void* stream);
/* out[r] = row_sign[J[r]] * A[J[r],:] . d (r < p) through the same build's packed
 * J-restricted CSR (the CG's X_J d).  Same workspace as ssnal_csr_xt_restricted. */
int ssnal_csr_xd_restricted(const ssnal_csr_operator_t* op, const uint8_t* keep,
                            const int32_t* J, int64_t p, const double* d, double* out, void* ws,
                            void* stream);
/* out[k] = sum_{i : keep[i] != 0} A[i,k]^2 (q): the Jacobi diagonal of X_J^T X_J for the
 * factor-space CG (row signs square away); ws >= nslots doubles.  Replaces the diagonal
 * the reference's CG branch would read off Q_JJ (ref solver.py:151-172, 253-258). */
int ssnal_csr_colsq(const ssnal_csr_operator_t* op, const uint8_t* keep, double* out, void* ws,
                    void* stream);

/* ---- native SSsNAL driver ------------------------------------------------
 * The whole Algorithm 1 / Algorithm 3 loop of ref solver.py:331-530 (alm_solve,
 * ssn_solve, line_search, newton_direction, kkt_residual) run from C++ on one
 * stream: kernels are enqueued back to back and the host synchronises only at
 * the reference's decision points (one pinned read per Newton step in the
 * common case).  Same constants, criteria, safeguards and report fields as the
 * reference; eps_k = delta_k = 0.5^k (the reference defaults). */
typedef struct ssnal_dense_problem_t {
  const double* A;          /* n_phys x q row-major samples (DEVICE)                 */
  int64_t n_phys, q, lda;
  const double* row_sign;   /* labels for C-SVC or NULL                              */
  int svr_block;            /* 1: X = [A; -A] (eps-SVR)                              */
  int64_t n;                /* logical variables (2 n_phys for SVR)                  */
  const double* c;          /* linear term (DEVICE, n)                               */
  const double* a;          /* equality row (DEVICE, n)                              */
  const double* l;          /* lower bounds (DEVICE, n) or NULL => l_const           */
  const double* u;          /* upper bounds (DEVICE, n) or NULL => u_const           */
  double l_const, u_const, d;
  const ssnal_csr_operator_t* csr;  /* non-NULL: sparse operator (A, lda unused); the
                                       reduced Newton system is then solved by CG in
                                       sample space (matrix-free)                      */
} ssnal_dense_problem_t;

typedef struct ssnal_options_t {
  double sigma0, sigma_growth, sigma_max, tol_kkt, lambda_min_surrogate;  /* AlmOptions */
  int max_outer;
  double mu, backtrack, tau, eta;                                         /* SsnOptions */
  int max_inner, direct_solve_threshold, cg_max_iters, line_search_batch;
  int psi_stable;           /* 0: reference formula; 1: psi via sum Pi(u)(2u - Pi(u));
                               2: Armijo on psi differences (Bregman form, ssnal_project_ex) */
  int profile;              /* 1: CUDA-event timing per op class into the report      */
} ssnal_options_t;

/* op classes of ssnal_report_t.op_seconds / op_calls */
#define SSNAL_OP_XT 0       /* X^T V products (streams A)                             */
#define SSNAL_OP_XD 1       /* X D products (streams A)                               */
#define SSNAL_OP_PROJ 2     /* projections (Newton/K-ary passes + apply)              */
#define SSNAL_OP_NEWTON 3   /* reduced Newton system: compaction, p-space solve, CG   */
#define SSNAL_OP_VEC 4      /* elementwise ops, fused dots, HS-Jacobian               */
#define SSNAL_OP_GRAM 5     /* q-space Gram X_J^T X_J (rebuild or changed-slot update) */
#define SSNAL_OP_CHOL 6     /* assembly + Cholesky solve of the q x q Newton system   */
#define SSNAL_NOPS 7

typedef struct ssnal_report_t {
  double kkt_residual, objective, wall_time;
  int outer_iters, total_inner_iters, unbounded_support_count, converged;
  int hit_max_inner_mask;   /* bit k: inner solver hit max_inner at outer k (k < 31);
                               see hit_max_inner_mask64 / _count for the rest          */
  int stagnated, max_outer_reached;
  long long syncs, newton_steps, projections, launches;
  double op_seconds[SSNAL_NOPS];   /* device time per op class (profile = 1)         */
  long long op_calls[SSNAL_NOPS];
  double op_bytes[SSNAL_NOPS];     /* algorithmic HBM bytes per op class             */
  double op_flops[SSNAL_NOPS];     /* algorithmic flops (GRAM: rows q (q+1); CHOL: m^3/3) */
  long long cg_iters;              /* sparse operator: CG iterations, all Newton steps */
  long long cg_fallbacks;          /* CG solves that fell back to the direct system     */
  long long gram_builds;           /* dense q-space Gram rebuilt from all p free rows   */
  long long gram_updates;          /* ... updated over the changed slots only           */
  long long gram_rows;             /* rows gathered by both                             */
  long long proj_fallbacks;        /* projections finished by the K-ary fallback        */
  unsigned long long hit_max_inner_mask64; /* bit k: max_inner hit at outer k (k < 64)  */
  int hit_max_inner_count;         /* all outer iterations that hit max_inner           */
  int pad_;
} ssnal_report_t;

/* per outer iteration: (k, R_KKT, sigma, p, inner iterations) as ref solver.py:474-475 */
typedef void (*ssnal_progress_fn)(int k, double kkt, double sigma, long long p, int inner,
                                  void* ctx);

size_t ssnal_alm_ws_bytes(int64_t n_phys, int64_t q, int svr_block);
size_t ssnal_alm_ws_bytes_csr(const ssnal_csr_operator_t* op);
int ssnal_alm_solve_dense(const ssnal_dense_problem_t* problem, const ssnal_options_t* options,
                          const double* x0, const double* w0, double* x_out,
                          ssnal_report_t* report, void* ws, size_t ws_bytes,
                          ssnal_progress_fn progress, void* progress_ctx, void* stream);

/* ---- row-sharded path ------------------------------------------------------
 * One process per GPU, rank r owning a slice of the n dual slots (rows of X).
 * The cross-slot reductions of the projection (ref projection.py:152-211) are
 * split into shard-local records the host all-gathers and folds in rank order:
 *   mode 0 (eval at lam[t]):  rec[t*8 + 0..6] = { sum a clip(v - lam a, l, u),
 *     sum a^2 over slots free just right of lam, ... just left, nearest breakpoint
 *     > lam (+inf), nearest breakpoint < lam (-inf), smallest breakpoint, largest }
 *   mode 1 (apply at lam[t]): x_out / free_out (T x n) and rec[t*8 + 0..5] =
 *     { sum v^2, sum (v-x)^2, sum (x-ref)^2, sum_free a^2, nfree, sum x(2v-x) }
 *     (base != NULL: slot 0 is the Bregman term of ssnal_project_ex instead of sum v^2)
 * with v = A - coef[t] B.  coef and lam are HOST arrays of T <= 16; rec is a
 * DEVICE array of 8 T doubles.  ws: ssnal_proj_local_ws_bytes(n, T). */
size_t ssnal_proj_local_ws_bytes(int64_t n, int T);
int ssnal_proj_local(const double* A, const double* B, const double* coef, const double* lam,
                     const double* a, const double* l, const double* u, double l_const,
                     double u_const, int64_t n, int T, int mode, double* x_out, uint8_t* free_out,
                     const double* ref, const double* base, double base_lam, double* rec,
                     void* ws, void* stream);
/* out[i] = sum_{r<k} src[r*len + i] in rank order (the all-gathered partials of
 * X^T v, Gram blocks and dot records; deterministic). */
int ssnal_sum_slices(int k, int64_t len, const double* src, double* out, void* stream);
/* out = alpha*add + beta*free(y - coef*a): ssnal_hs_apply with the global
 * coef = a_J'y_J / a_J'a_J supplied (ref projection.py:214-225). */
int ssnal_hs_apply_coef(const uint8_t* free_mask, const double* a, const double* y, int64_t n,
                        double beta, const double* add, double alpha, double coef, double* out,
                        void* stream);
/* M = I + sigma (M - shift I - u u'/asa) in place (u NULL or asa == 0: no rank-one
 * term): the factor-space Newton matrix from the rank-summed Gram of
 * ssnal_dense_gram(sigma = 1, a'a = 0) blocks (shift = world size). */
int ssnal_qspace_assemble(int64_t m, const double* u, double asa, double sigma, double shift,
                          double* M, void* stream);

/* ---- row-sharded native driver ------------------------------------------------
 * The whole loop of ssnal_alm_solve_dense over world ranks, rank r holding a slice of
 * the dual slots (rows of X: C-SVC rows, or [x+ ; x-] of its SVR rows) -- the problem
 * passed is that slice, with d the GLOBAL right-hand side of a'x = d.  Replaces ref
 * solver.py:429-530 alm_solve for a partitioned sample set: the reference's
 * cross-slot sums (kernels.py:144-154 X^T v, solver.py:151-172 / 238-269 the Newton
 * system and its inner products, projection.py:152-211 the multiplier search) become
 *   allreduce_sum: q-vectors (X^T v, X^T dPi), the kept q x q Gram, dot partials;
 *   allgather:     the projection search's 8-double records (folded in rank order).
 * Every rank receives the same reduced buffers, so the host decisions agree.  The
 * reduced Newton system is always the q x q one (dense: q <= 2048; sparse: q x q direct
 * for q <= 2048, else the factor-space Jacobi CG).  Both collectives are enqueued on
 * `stream`; a transport must order them with the solver's kernels on that stream. */
#define SSNAL_COMM_ID_BYTES 128
#define SSNAL_COMM_NCCL 1          /* ssnal_nccl_comm_create                              */
#define SSNAL_COMM_LOOPBACK 2      /* ssnal_loopback_comm_create (tests: ranks = threads) */
typedef struct ssnal_comm_t {
  int world, rank;
  int (*allreduce_sum)(void* ctx, double* buf, int64_t count, void* stream);  /* in place */
  int (*allgather)(void* ctx, const double* in, double* out, int64_t count, void* stream);
  void* ctx;
  int kind;                /* SSNAL_COMM_*, 0 for a caller-provided transport          */
  int pad_;
} ssnal_comm_t;

/* NCCL transport (libnccl.so.2 opened at run time): rank 0 makes the id, every rank
 * calls create with it after selecting its device (one process per GPU). */
int ssnal_nccl_unique_id(unsigned char* id /* SSNAL_COMM_ID_BYTES */);
int ssnal_nccl_comm_create(int world, int rank, const unsigned char* id, ssnal_comm_t* out);
/* Loopback transport: world ranks as host threads of one process on one GPU (each with
 * its own stream); a collective drains the caller's stream, meets the other ranks at a
 * host barrier and sums their buffers in rank order -- no kernel waits on a rank. */
int ssnal_loopback_group_create(int world, void** group);
int ssnal_loopback_comm_create(void* group, int rank, ssnal_comm_t* out);
int ssnal_loopback_group_destroy(void* group);
int ssnal_comm_destroy(ssnal_comm_t* comm);

size_t ssnal_alm_ws_bytes_sharded(int64_t n_phys, int64_t q, int svr_block, int world);
size_t ssnal_alm_ws_bytes_csr_sharded(const ssnal_csr_operator_t* op, int world);
int ssnal_alm_solve_sharded(const ssnal_dense_problem_t* problem, const ssnal_options_t* options,
                            const ssnal_comm_t* comm, const double* x0, const double* w0,
                            double* x_out, ssnal_report_t* report, void* ws, size_t ws_bytes,
                            ssnal_progress_fn progress, void* progress_ctx, void* stream);

/* Fused SsN gradient of the dense operator (ref solver.py:143-148):
 *   s = w - x_p (written), g_r = X^T s (q), grad = X g_r (n_log), *g2 = ||grad||^2
 * with *g2 a DEVICE double; two streaming sweeps of A.  ws: ssnal_gradient_ws_bytes
 * (zero-initialised once; the kernels leave their tickets at zero). */
size_t ssnal_gradient_ws_bytes(int64_t n_phys, int64_t q);
int ssnal_dense_gradient(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                         const double* row_sign, int svr_block, const double* w, const double* xp,
                         double* s_out, double* g_r, double* grad, double* g2, void* ws,
                         void* stream);

/* Dense Newton-direction epilogue (ref solver.py:259-269), from t = X^T d:
 *   qdir = X t;  dir = -s - sigma P_J(qdir)  (P_J from the free mask, a_J'a_J read from
 *   *asa_dev -- the projection record's sum_a2_free); dots4 (DEVICE, 4 doubles) =
 *   {grad'dir, w'qw, w'qdir, t't}.  ws: ssnal_gradient_ws_bytes (shared with the
 *   gradient call; stream-ordered use). */
int ssnal_dense_direction_epilogue(const double* A, int64_t n_phys, int64_t q, int64_t lda,
                                   const double* row_sign, int svr_block, const double* t,
                                   double* qdir, const uint8_t* free_mask, const double* a,
                                   const double* asa_dev, const double* s, double sigma,
                                   const double* grad, const double* w, const double* qw,
                                   double* dir, double* dots4, void* ws, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SSNAL_B200_H */

// Internal declarations shared by the .cu translation units (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/ssnal_b200.h"

namespace ssnal {

enum ProjStatus {
  PROJ_SEARCH = 0,
  PROJ_BRACKETED = 1,
  PROJ_DONE = 2,
  PROJ_APPLIED = 3,
  PROJ_NEWTON = 4,
  PROJ_INFEASIBLE_LOW = -1,
  PROJ_INFEASIBLE_HIGH = -2,
};

enum ProjPhase { PHASE_RANGE = 1, PHASE_EXACT = 2, PHASE_APPLY = 4 };

// ProjState is the device record ssnal_proj_state_t of the public header.
using ProjState = ssnal_proj_state_t;
using CsrOp = ssnal_csr_operator_t;

// device-side control of the kept q-space Gram (dense.cu gram_select_kernel)
struct GramCtl {
  long long count, accum, builds, updates, rows;
  int mode, valid;
};

cudaError_t launch_csr_xd(const CsrOp& op, const int32_t* rows, long long nrows, const double* d,
                          double* out, cudaStream_t stream);
cudaError_t launch_csc_xt(const CsrOp& op, const double* v, double* out, double* part,
                          cudaStream_t stream);
cudaError_t launch_csc_colsq(const CsrOp& op, const uint8_t* keep, double* out, double* part,
                             cudaStream_t s);
cudaError_t launch_fill(double* dst, long long n, double v, cudaStream_t stream);
cudaError_t launch_scatter(const int32_t* rows, long long p, const double* src, double* dst,
                           cudaStream_t stream);
cudaError_t launch_gather(const int32_t* rows, long long p, const double* src, double* dst,
                          cudaStream_t stream);

// J-restricted CSC of the free rows (sparse.cu): rebuilt per Newton step
struct CscJ {
  unsigned int* ticket;
  int32_t* posJ;   // position in J of each kept row (n)
  int* cnt;        // kept entries per segment
  long long* blk;  // per-block offsets
  int64_t *beg, *end;
  int32_t* pos;    // row slot in J per kept entry
  double* val;     // signed values
  int32_t* seg;    // segment id per kept entry (nnz-balanced product)
  double *cval, *ctail;  // per 256-entry chunk: first-segment / open-tail partial sums
  uint8_t* cflag;        // bit 0: first segment closes in the chunk; bit 1: owns an open tail
  // J-restricted CSR: the free rows' entries packed contiguously (row signs folded), so
  // every CG product X_J d streams them without the J -> indptr indirection
  int64_t* rptr;   // p + 1
  int32_t* ridx;
  double* rval;
  long long* rblk; // per-block row-length offsets
  int32_t* empty;  // segments without kept entries (written as zeros by every product)
  unsigned int* nempty;
  // hot-column staging of X_J d (operator's popularity table; 0: off): ridx holds ~rank
  int nhot;
  const int32_t* hot_cols;
};
size_t cscj_ws_bytes(const CsrOp& op);
CscJ cscj_layout(const CsrOp& op, void* ws);
cudaError_t launch_cscj_build(const CsrOp& op, const uint8_t* keep, const int32_t* J, long long p,
                              const CscJ& c, cudaStream_t stream);
cudaError_t launch_cscj_xt(const CsrOp& op, const CscJ& c, const double* w, double* out,
                           double* part, cudaStream_t stream);
cudaError_t launch_csrj_xd(const CscJ& c, long long p, const double* d, double* out,
                           cudaStream_t stream);
cudaError_t launch_csrj_xd_dot(const CscJ& c, long long p, const double* d, double* out,
                               const double* wdot, double* dot_out, double* part,
                               int max_blocks, unsigned int* ticket, cudaStream_t stream);

struct ProjLaunch {
  const double *A, *B, *coef, *a, *l, *u;
  double lc, uc, d;
  long long n;
  int T;
  ProjState* st;
  double* part;
  double* x_out;
  unsigned char* free_out;
  const double* ref;
  const double* base = nullptr;  // line-search base Pi: sum_bh instead of sum_v2
  double base_lam = 0.0;
  int phases;
  int passes;
  double hint;  // warm-start multiplier for the Newton passes
  int newton;   // Newton passes (0: start from the full breakpoint range instead)
  int defer = 0;  // batched trials may leave x / the mask unwritten (see proj_defers)
  const double* hints = nullptr;  // per-trial warm starts (host array of T), else `hint`
  const double* slope_num = nullptr;  // device scalars: first-order start along the ray
  const double* slope_den = nullptr;
};

// ---- row-sharded native driver (dist.cu, comm.cu) -----------------------------------
// Device state of one trial's multiplier search (the safeguarded Newton of the sharded
// projection, one all-gather of 5-double records per pass)
enum { SP_SEARCH = 0, SP_DONE = 1, SP_INFEAS_LOW = -1, SP_INFEAS_HIGH = -2 };
struct SProj {
  double lam, lo, hi;
  int status, passes;
};
struct ShardProj {  // one sharded projection call (driver.cu project_sharded)
  const double *A, *B, *a, *l, *u;
  double lc, uc, d;
  long long n;
  int T;
  double coef[SSNAL_MAX_TRIALS];
  double hints[SSNAL_MAX_TRIALS];
  int has_hints;
  double hint;
  const double* slope_num;  // device scalars: first-order start along the ray (or null)
  const double* slope_den;
  double* x_out;
  unsigned char* free_out;
  const double* ref;
  const double* base;
  double base_lam;
};
size_t proj_local_ws_bytes(long long n, int T);
cudaError_t launch_sproj_init(const ShardProj& P, SProj* sp, cudaStream_t s);
cudaError_t launch_sproj_eval(const ShardProj& P, const SProj* sp, double* part, double* rec,
                              cudaStream_t s);
cudaError_t launch_sproj_update(int world, int T, const double* rec_all, double d, SProj* sp,
                                cudaStream_t s);
cudaError_t launch_sproj_apply(const ShardProj& P, const SProj* sp, double* part, double* rec,
                               cudaStream_t s);
cudaError_t launch_sproj_finish(int world, int T, const double* rec_all, const double* rec_loc,
                                const SProj* sp, int base_mode, ProjState* st, cudaStream_t s);
cudaError_t launch_hs_finish(const uint8_t* fm, const double* a, const double* y, long long n,
                             double beta, const double* add, double alpha, double* out,
                             const double* sums, cudaStream_t s);
cudaError_t launch_factor_update(long long q, double alpha, const double* t, const double* dsum,
                                 double* xw, double* xpi, double* r, cudaStream_t s);
cudaError_t launch_cg_check_final(const double* sq, double scale, double* cgs, cudaStream_t s);
int nccl_unique_id(unsigned char* id, const char** err);
int nccl_comm_create(int world, int rank, const unsigned char* id, ssnal_comm_t* out,
                     const char** err);
int loop_group_create(int world, void** group);
int loop_comm_create(void* group, int rank, ssnal_comm_t* out);
int loop_group_destroy(void* group);
int comm_destroy(ssnal_comm_t* c);

int proj_blocks(long long n);
int proj_wave_trials(long long n, bool first = false);
size_t proj_ws_bytes(long long n, int T);
cudaError_t launch_project(const ProjLaunch& L, cudaStream_t stream);
bool proj_defers(long long n, int T);
cudaError_t launch_proj_materialize(const ProjLaunch& L, double coef, const ProjState* st,
                                    double* x_out, unsigned char* f_out, cudaStream_t stream);

}  // namespace ssnal

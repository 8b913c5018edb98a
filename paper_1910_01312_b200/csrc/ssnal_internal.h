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

cudaError_t launch_csr_xd(const CsrOp& op, const int32_t* rows, long long nrows, const double* d,
                          double* out, cudaStream_t stream);
cudaError_t launch_csc_xt(const CsrOp& op, const double* v, double* out, double* part,
                          cudaStream_t stream);
cudaError_t launch_fill(double* dst, long long n, double v, cudaStream_t stream);
cudaError_t launch_scatter(const int32_t* rows, long long p, const double* src, double* dst,
                           cudaStream_t stream);
cudaError_t launch_gather(const int32_t* rows, long long p, const double* src, double* dst,
                          cudaStream_t stream);

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
  int phases;
  int passes;
  double hint;  // warm-start multiplier for the Newton passes
  int newton;   // Newton passes (0: start from the full breakpoint range instead)
};

int proj_blocks(long long n);
size_t proj_ws_bytes(long long n, int T);
cudaError_t launch_project(const ProjLaunch& L, cudaStream_t stream);

}  // namespace ssnal

// Per-phase timing of proj_multi_kernel (globaltimer stamps of block 0 thread 0) on an
// eps-SVR-shaped 2,000,000-slot problem.  Built on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSSNAL_PROJ_TIMING -o /tmp/proj_probe \
//        scripts/proj_probe.cu && /tmp/proj_probe
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace ssnal {
void note_launch() {}
}
#include "../paper_1910_01312_b200/csrc/proj.cu"

int main() {
  const long long m = 1000000, n = 2 * m;
  std::vector<double> u(n), qd(n), a(n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> N(0.0, 1.0);
  for (long long i = 0; i < n; ++i) {
    u[i] = 50.0 * N(rng);
    qd[i] = 0.01 * N(rng);
    a[i] = i < m ? 1.0 : -1.0;
  }
  for (int k = 0; k < 20000; ++k) u[(k * 104729LL) % n] = 1.2 * (k % 100) / 100.0 - 0.1;
  double *du, *dq, *da, *dx, *dpart;
  unsigned char* df;
  ssnal::ProjState* dst;
  cudaMalloc(&du, n * 8);
  cudaMalloc(&dq, n * 8);
  cudaMalloc(&da, n * 8);
  cudaMalloc(&dx, 8 * n * 8);
  cudaMalloc(&df, 8 * n);
  cudaMalloc(&dst, 16 * sizeof(ssnal::ProjState));
  cudaMemset(dst, 0, 16 * sizeof(ssnal::ProjState));
  const size_t wsb = ssnal::proj_ws_bytes(n, 8);
  cudaMalloc(&dpart, wsb);
  cudaMemset(dpart, 0, wsb);
  cudaMemcpy(du, u.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, qd.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(da, a.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int T : {1, 2, 4}) {
    double coefs[16];
    for (int t = 0; t < 16; ++t) coefs[t] = 1.0 / (1 << t);
    ssnal::ProjLaunch L;
    L.A = du; L.B = dq; L.coef = coefs; L.a = da; L.l = nullptr; L.u = nullptr;
    L.lc = 0.0; L.uc = 1.0; L.d = 0.0; L.n = n; L.T = T; L.st = dst; L.part = dpart;
    L.x_out = dx; L.free_out = df; L.ref = nullptr; L.phases = ssnal::PHASE_APPLY; L.passes = 0;
    L.hint = 0.0; L.newton = 3; L.defer = 1;
    for (int rep = 0; rep < 6; ++rep) {
      int zero = 0;
      cudaMemcpyToSymbol(ssnal::g_proj_nmarks, &zero, sizeof(int));
      cudaEventRecord(e0);
      cudaError_t e = ssnal::launch_project(L, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      int nm = 0;
      unsigned long long mk[64];
      cudaMemcpyFromSymbol(&nm, ssnal::g_proj_nmarks, sizeof(int));
      cudaMemcpyFromSymbol(mk, ssnal::g_proj_marks, sizeof(mk));
      ssnal::ProjState st[8];
      cudaMemcpy(st, dst, sizeof(st), cudaMemcpyDeviceToHost);
      if (rep < 4) continue;
      printf("T=%d %s %.1f us (passes %d, status %d) marks:", T, cudaGetErrorString(e), ms * 1e3,
             st[0].passes, st[0].status);
      for (int k = 1; k < nm && k < 64; ++k) printf(" %.1f", (mk[k] - mk[k - 1]) * 1e-3);
      printf("\n");
    }
    L.hint = 0.0;
  }
  return 0;
}

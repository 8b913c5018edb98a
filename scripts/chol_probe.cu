// Per-phase timing of chol_big_kernel (globaltimer stamps of CTA 0 thread 0 at every
// cluster barrier).  Built on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSSNAL_CHOL_TIMING -o /tmp/chol_probe \
//        scripts/chol_probe.cu && /tmp/chol_probe 500
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace ssnal {
void note_launch() {}
}
#include "../paper_1910_01312_b200/csrc/linalg.cu"

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 500;
  std::vector<double> h((size_t)m * m), b(m, 1.0);
  srand(1);
  // SPD: I + G G^T / m with G random
  std::vector<double> G((size_t)m * m);
  for (auto& v : G) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < m; ++k) s += G[(size_t)i * m + k] * G[(size_t)j * m + k] / m;
      h[(size_t)i * m + j] = s;
    }
  double *dM, *dM0, *db, *dx;
  int* dinfo;
  cudaMalloc(&dM, sizeof(double) * m * m);
  cudaMalloc(&dM0, sizeof(double) * m * m);
  cudaMalloc(&db, sizeof(double) * m);
  cudaMalloc(&dx, sizeof(double) * m);
  cudaMalloc(&dinfo, sizeof(int));
  cudaMemcpy(dM0, h.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemcpy(dM, dM0, sizeof(double) * m * m, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    cudaError_t e = ssnal::launch_chol_solve(dM, m, db, 1.0, dx, dinfo, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    int info = -1;
    cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
    printf("rep %d: %s, %.1f us, info %d\n", rep, cudaGetErrorString(e), ms * 1e3, info);
  }
  unsigned long long marks[12][64];
  cudaMemcpyFromSymbol(marks, ssnal::g_chol_marks, sizeof(marks));
  const unsigned long long t0 = marks[0][0];
  const int np = (m + 31) / 32;
  for (int k = 0; k < np; ++k)
    printf("panel %2d: diag %7.2f (load %6.2f fact %6.2f inv+store %6.2f fwd+sync %6.2f)  "
           "trsm+sync %7.2f  syrk+sync %7.2f us\n", k,
           (marks[1][k] - (k ? marks[3][k - 1] : t0)) * 1e-3,
           (marks[6][k] - (k ? marks[3][k - 1] : t0)) * 1e-3, (marks[7][k] - marks[6][k]) * 1e-3,
           (marks[8][k] - marks[7][k]) * 1e-3, (marks[1][k] - marks[8][k]) * 1e-3,
           (marks[2][k] - marks[1][k]) * 1e-3, (marks[3][k] - marks[2][k]) * 1e-3);
  printf("start->loop %.2f us, back substitution %.2f us, total %.2f us\n",
         (marks[0][0] - t0) * 1e-3, (marks[5][np - 1] - marks[4][np - 1]) * 1e-3,
         (marks[5][np - 1] - t0) * 1e-3);
  return 0;
}

// Standalone check + timing of launch_syev_topk (Alg. 3 commit eigen-solver: RR tridiagonalisation with
// saved reflectors, multisection, inverse iteration, back-transformation) against the QL path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include [-DCMSVD_INV_PROF] -o invbench invbench.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/k_eig.cu"
using namespace cmsvd;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 160;
  const int kw = argc > 2 ? atoi(argv[2]) : 32;
  const double gap = argc > 3 ? atof(argv[3]) : 0.0;  // >0: force pairs of eigenvalues this close (relative)
  std::vector<double> X((size_t)n * n), h((size_t)n * n), spec(n);
  srand(3);
  for (auto& x : X) x = rand() / (double)RAND_MAX - 0.5;
  // orthonormalise X (Gram-Schmidt) so the spectrum is exactly spec
  for (int j = 0; j < n; ++j) {
    for (int q = 0; q < j; ++q) {
      double t = 0;
      for (int i = 0; i < n; ++i) t += X[q * n + i] * X[j * n + i];
      for (int i = 0; i < n; ++i) X[j * n + i] -= t * X[q * n + i];
    }
    double s = 0;
    for (int i = 0; i < n; ++i) s += X[j * n + i] * X[j * n + i];
    for (int i = 0; i < n; ++i) X[j * n + i] /= sqrt(s);
  }
  for (int k = 0; k < n; ++k) spec[k] = pow(0.93, k) * (1.0 + 0.01 * (k % 3));
  if (gap > 0)
    for (int k = 1; k < n; k += 2) spec[k] = spec[k - 1] * (1.0 - gap);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += X[k * n + i] * spec[k] * X[k * n + j];
      h[(size_t)j * n + i] = s;
    }
  double *dG, *Z, *ev, *scr, *V, *VH, *evq;
  int *dn, *perm, *st;
  cudaMalloc(&dG, 8 * n * n); cudaMalloc(&Z, 8 * n * kw); cudaMalloc(&ev, 8 * kw);
  cudaMalloc(&scr, syev_topk_scratch_bytes(n, kw)); cudaMalloc(&V, 8 * n * n); cudaMalloc(&VH, 8 * n * n);
  cudaMalloc(&evq, 8 * n); cudaMalloc(&dn, 4); cudaMalloc(&perm, 4 * n); cudaMalloc(&st, 4);
  cudaMemcpy(dG, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dn, &n, 4, cudaMemcpyHostToDevice);
  Ctx c; c.stream = 0;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    cudaError_t e = launch_syev_topk(c, dG, n, dn, kw, Z, ev, scr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("launch error\n"); return 1; }
    printf("topk  rep %d: %.3f ms\n", rep, ms);
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    launch_syev(c, dG, n, (int64_t)n * n, dn, 1, n, V, (int64_t)n * n, VH, evq, perm, n, st);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("QL    rep %d: %.3f ms\n", rep, ms);
  }
  std::vector<double> hz((size_t)n * kw), hev(kw);
  cudaMemcpy(hz.data(), Z, 8 * n * kw, cudaMemcpyDeviceToHost);
  cudaMemcpy(hev.data(), ev, 8 * kw, cudaMemcpyDeviceToHost);
  double maxres = 0, maxorth = 0, maxev = 0;
  for (int j = 0; j < kw; ++j) {
    maxev = fmax(maxev, fabs(hev[j] - spec[j]) / spec[0]);
    for (int i = 0; i < n; ++i) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += h[(size_t)k * n + i] * hz[(size_t)j * n + k];
      maxres = fmax(maxres, fabs(s - hev[j] * hz[(size_t)j * n + i]) / spec[0]);
    }
    for (int q = 0; q <= j; ++q) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += hz[(size_t)j * n + i] * hz[(size_t)q * n + i];
      maxorth = fmax(maxorth, fabs(s - (q == j ? 1.0 : 0.0)));
    }
  }
  printf("n=%d kw=%d gap=%g: max|ev-spec|/l0 %.2e  max|Gz-lz|/l0 %.2e  max|ZtZ-I| %.2e\n", n, kw, gap, maxev, maxres,
         maxorth);
  return 0;
}

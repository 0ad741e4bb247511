// Standalone timing of the batched eigenvalue kernel (k_tridiag_topk) on
// random symmetric PSD Grams; -DCMSVD_EIG_PROFILE prints per-phase cycles.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/k_eig.cu"
using namespace cmsvd;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 160;
  int P = argc > 2 ? atoi(argv[2]) : 8128;
  int kw = argc > 3 ? atoi(argv[3]) : 32;
  std::vector<double> h((size_t)n * n);
  srand(1);
  std::vector<double> X((size_t)n * n);
  for (auto& x : X) x = (rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += X[i * n + k] * X[j * n + k] * (k < 24 ? 1000.0 / (k + 1) : 0.01);
      h[(size_t)j * n + i] = s;
    }
  double* dG; cudaMalloc(&dG, sizeof(double) * n * n * (size_t)P);
  for (int p = 0; p < P; ++p) cudaMemcpy(dG + (size_t)p * n * n, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  std::vector<int> ns(P, n);
  int* dn; cudaMalloc(&dn, 4 * P); cudaMemcpy(dn, ns.data(), 4 * P, cudaMemcpyHostToDevice);
  double *ev, *tr; int* cnt;
  cudaMalloc(&ev, 8 * (size_t)P * kw); cudaMalloc(&tr, 8 * P); cudaMalloc(&cnt, 4 * P);
  Ctx c; c.stream = 0;
  double* scr; cudaMalloc(&scr, tridiag_scratch_bytes(P, n));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    launch_tridiag_topk(c, dG, n, (int64_t)n * n, dn, P, n, nullptr, kw, ev, cnt, tr, scr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("n=%d P=%d kw=%d: %.3f ms  (%.2f us/problem/SM)  err=%s\n", n, P, kw, ms, ms * 1e3 * 148 / P,
           cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> hev(kw);
  cudaMemcpy(hev.data(), ev, 8 * kw, cudaMemcpyDeviceToHost);
  printf("top eig: %.6e %.6e ... %.6e\n", hev[0], hev[1], hev[kw - 1]);
  return 0;
}

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
  if (getenv("GLMB")) c.gl_batch_mb = atoi(getenv("GLMB"));
  double* scr; cudaMalloc(&scr, tridiag_scratch_bytes(P, n));
  std::vector<double> evs[3];
  std::vector<double> trs[3];
  const char* vname[3] = {"smem", "rr  ", "duo "};
  for (int variant = 0; variant < 3; ++variant) {
  c.eig_rr = variant >= 1;
  c.eig_duo = variant == 2;
  c.eig_duo160 = variant == 2;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    launch_tridiag_topk(c, dG, n, (int64_t)n * n, dn, P, n, nullptr, kw, ev, cnt, tr, scr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s n=%d P=%d kw=%d: %.3f ms  (%.2f us/problem/SM)  err=%s\n", vname[variant], n, P, kw, ms,
           ms * 1e3 * 148 / P, cudaGetErrorString(cudaGetLastError()));
  }
  evs[variant].resize((size_t)P * kw);
  trs[variant].resize(P);
  cudaMemcpy(evs[variant].data(), ev, 8 * (size_t)P * kw, cudaMemcpyDeviceToHost);
  cudaMemcpy(trs[variant].data(), tr, 8 * (size_t)P, cudaMemcpyDeviceToHost);
  }
#ifdef CMSVD_RR_PROF
  unsigned long long hp[8];
  cudaMemcpyFromSymbol(hp, g_rr_prof, sizeof(hp));
  const char* nm[8] = {"elem wait B3_0", "elem F0", "elem wait B3_1", "elem F1", "row wait B2_0", "row R0", "row wait B2_1", "row R1"};
  for (int q = 0; q < 8; ++q) printf("  %-18s %10.1f cycles/step\n", nm[q], hp[q] / 3.0 / (n - 2));
#endif
  double md = 0, mx = 0, md2 = 0;
  for (size_t q = 0; q < evs[0].size(); ++q) { md = fmax(md, fabs(evs[0][q] - evs[1][q])); md2 = fmax(md2, fabs(evs[1][q] - evs[2][q])); mx = fmax(mx, fabs(evs[0][q])); }
  printf("max |ev_rr - ev_duo| = %.3e\n", md2);
  double sd = 0;
  for (int q = 0; q < P; ++q) {
    double s0 = trs[0][q], s1 = trs[1][q];
    for (int l = 0; l < kw; ++l) { s0 -= evs[0][(size_t)q * kw + l]; s1 -= evs[1][(size_t)q * kw + l]; }
    sd = fmax(sd, fabs(s0 - s1) / fmax(fabs(s0), 1e-300));
  }
  printf("max |ev_smem - ev_rr| = %.3e (max ev %.3e); max rel diff of trace - top = %.3e\n", md, mx, sd);
  std::vector<double> hev(kw);
  cudaMemcpy(hev.data(), ev, 8 * kw, cudaMemcpyDeviceToHost);
  printf("top eig: %.6e %.6e ... %.6e\n", hev[0], hev[1], hev[kw - 1]);
  return 0;
}

// Phase timing of k_pair_tc (built with -DCMSVD_TC_PROF): P identical pairs of a random orthonormal
// Q (m x q) and F (m x w); prints average cycles per pair (CTAs 0..147) in each phase.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/k_pair_tc.cu"
using namespace cmsvd;
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 512, q = 128, w = 128;
  const int P = argc > 2 ? atoi(argv[2]) : 8128;
  std::vector<float> Q((size_t)m * q), F((size_t)m * w);
  srand(3);
  for (auto& x : Q) x = (rand() / (float)RAND_MAX - 0.5f) * 0.1f;
  for (auto& x : F) x = rand() / (float)RAND_MAX - 0.5f;
  float *dQ, *dF, *dZ; double* dW;
  cudaMalloc(&dQ, 4 * Q.size()); cudaMalloc(&dF, 4 * F.size());
  cudaMalloc(&dZ, 4 * (size_t)q * w * P); cudaMalloc(&dW, 8 * (size_t)w * w * P);
  cudaMemcpy(dQ, Q.data(), 4 * Q.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dF, F.data(), 4 * F.size(), cudaMemcpyHostToDevice);
  BaseDesc bdh{}; bdh.basis = dQ; bdh.q = q; bdh.rr = q;
  AppDesc adh{}; adh.F = dF; adh.w = w;
  BaseDesc* dbd; AppDesc* dad; int2* dp;
  cudaMalloc(&dbd, sizeof(BaseDesc)); cudaMalloc(&dad, sizeof(AppDesc)); cudaMalloc(&dp, 8 * (size_t)P);
  cudaMemcpy(dbd, &bdh, sizeof(bdh), cudaMemcpyHostToDevice); cudaMemcpy(dad, &adh, sizeof(adh), cudaMemcpyHostToDevice);
  cudaMemset(dp, 0, 8 * (size_t)P);
  Ctx c; c.stream = 0;
  for (int rep = 0; rep < 3; ++rep) {
#ifdef CMSVD_TC_PROF
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
#endif
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    launch_pair_tc(c, dp, P, dbd, dad, m, 1, q, w, dZ, dW);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[8] = {};
#ifdef CMSVD_TC_PROF
    cudaMemcpyFromSymbol(h, g_tc_prof, sizeof(h));
#endif
    const int tiles = (m + 127) / 128;
    printf("P=%d m=%d: %.3f ms (%.1f us/pair/SM)  err=%s\n", P, m, ms, ms * 1e3 * 148 / P, cudaGetErrorString(cudaGetLastError()));
    const char* nm[6] = {"phase1 (Z)", "stage+R' issue", "R' wait", "epilogue", "W' MMA", "drain"};
    for (int k = 0; k < 6; ++k) printf("   %-16s %9.0f cycles/pair\n", nm[k], (double)h[k] / 148);
    (void)tiles;
  }
  return 0;
}

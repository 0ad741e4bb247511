// Standalone accuracy check of k_pair_tc: Z = Q^T F and W' = (F - QZ)^T (F - QZ)
// for one pair with random orthonormal-ish Q (m x q) and F = Q C + noise.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/k_pair_tc.cu"
using namespace cmsvd;
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 2048, q = argc > 2 ? atoi(argv[2]) : 64, w = argc > 3 ? atoi(argv[3]) : 64;
  double noise = argc > 4 ? atof(argv[4]) : 0.05;
  srand(7);
  auto rn = []() { double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0); return sqrt(-2 * log(u)) * cos(6.283185307 * v); };
  std::vector<double> Qd((size_t)m * q), Fd((size_t)m * w);
  for (auto& x : Qd) x = rn();
  // Gram-Schmidt
  for (int j = 0; j < q; ++j) {
    for (int i = 0; i < j; ++i) { double d = 0; for (int k = 0; k < m; ++k) d += Qd[(size_t)i * m + k] * Qd[(size_t)j * m + k]; for (int k = 0; k < m; ++k) Qd[(size_t)j * m + k] -= d * Qd[(size_t)i * m + k]; }
    double n = 0; for (int k = 0; k < m; ++k) n += Qd[(size_t)j * m + k] * Qd[(size_t)j * m + k]; n = sqrt(n);
    for (int k = 0; k < m; ++k) Qd[(size_t)j * m + k] /= n;
  }
  for (int b = 0; b < w; ++b)
    for (int k = 0; k < m; ++k) {
      double s = 0; for (int a = 0; a < q; ++a) s += Qd[(size_t)a * m + k] * (a < 16 ? 40.0 * rn() : 0.0);
      Fd[(size_t)b * m + k] = s + noise * rn();
    }
  std::vector<float> Q(Qd.begin(), Qd.end()), F(Fd.begin(), Fd.end());
  // references from the fp32-rounded inputs
  std::vector<double> Zr((size_t)q * w), Rr((size_t)m * w), Wr((size_t)w * w);
  for (int b = 0; b < w; ++b) for (int a = 0; a < q; ++a) { double s = 0; for (int k = 0; k < m; ++k) s += (double)Q[(size_t)a * m + k] * F[(size_t)b * m + k]; Zr[(size_t)b * q + a] = s; }
  for (int b = 0; b < w; ++b) for (int k = 0; k < m; ++k) { double s = F[(size_t)b * m + k]; for (int a = 0; a < q; ++a) s -= (double)Q[(size_t)a * m + k] * Zr[(size_t)b * q + a]; Rr[(size_t)b * m + k] = s; }
  for (int b = 0; b < w; ++b) for (int c = 0; c < w; ++c) { double s = 0; for (int k = 0; k < m; ++k) s += Rr[(size_t)b * m + k] * Rr[(size_t)c * m + k]; Wr[(size_t)c * w + b] = s; }
  float *dQ, *dF, *dZ; double* dW;
  cudaMalloc(&dQ, 4 * Q.size()); cudaMalloc(&dF, 4 * F.size()); cudaMalloc(&dZ, 4 * (size_t)q * w); cudaMalloc(&dW, 8 * (size_t)w * w);
  cudaMemcpy(dQ, Q.data(), 4 * Q.size(), cudaMemcpyHostToDevice); cudaMemcpy(dF, F.data(), 4 * F.size(), cudaMemcpyHostToDevice);
  BaseDesc bdh{}; bdh.basis = dQ; bdh.q = q; bdh.rr = q;
  AppDesc adh{}; adh.F = dF; adh.w = w;
  BaseDesc* dbd; AppDesc* dad; int2* dp; int2 hp = make_int2(0, 0);
  cudaMalloc(&dbd, sizeof(BaseDesc)); cudaMalloc(&dad, sizeof(AppDesc)); cudaMalloc(&dp, 8);
  cudaMemcpy(dbd, &bdh, sizeof(bdh), cudaMemcpyHostToDevice); cudaMemcpy(dad, &adh, sizeof(adh), cudaMemcpyHostToDevice); cudaMemcpy(dp, &hp, 8, cudaMemcpyHostToDevice);
  Ctx c; c.stream = 0;
  cudaError_t e = launch_pair_tc(c, dp, 1, dbd, dad, m, 1, q, w, dZ, dW);
  cudaError_t e2 = cudaDeviceSynchronize();
  std::vector<float> Z((size_t)q * w); std::vector<double> W((size_t)w * w);
  cudaMemcpy(Z.data(), dZ, 4 * Z.size(), cudaMemcpyDeviceToHost); cudaMemcpy(W.data(), dW, 8 * W.size(), cudaMemcpyDeviceToHost);
  double ez = 0, zmax = 0, ew = 0, wmax = 0, ewd = 0;
  for (size_t i = 0; i < Z.size(); ++i) { ez = fmax(ez, fabs(Z[i] - Zr[i])); zmax = fmax(zmax, fabs(Zr[i])); }
  for (int b = 0; b < w; ++b) for (int cc = 0; cc < w; ++cc) { size_t i = (size_t)cc * w + b; ew = fmax(ew, fabs(W[i] - Wr[i])); wmax = fmax(wmax, fabs(Wr[i])); if (b == cc) ewd = fmax(ewd, fabs(W[i] - Wr[i]) / Wr[i]); }
  printf("m=%d q=%d w=%d noise=%g: %s/%s  Z: max err %.3e (max |Z| %.3e, rel %.2e)   W': max err %.3e (max |W'| %.3e, rel %.2e, diag rel %.2e)\n",
         m, q, w, noise, cudaGetErrorString(e), cudaGetErrorString(e2), ez, zmax, ez / zmax, ew, wmax, ew / wmax, ewd);
  return 0;
}

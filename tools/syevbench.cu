// Standalone check + timing of k_syev_ql: residual ||G V - V diag(l)|| and
// orthogonality ||V^T V - I|| on random symmetric matrices (incl. degenerate).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/k_eig.cu"
using namespace cmsvd;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 128;
  int P = argc > 2 ? atoi(argv[2]) : 128;
  std::vector<double> h((size_t)n * n * P);
  srand(2);
  for (int p = 0; p < P; ++p) {
    std::vector<double> X((size_t)n * n);
    for (auto& x : X) x = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < n; ++k) {
          double sc = (p % 3 == 0) ? (k < 24 ? 1000.0 / (k + 1) : 0.01) : (p % 3 == 1 ? 1.0 : (k < n / 2 ? 1.0 : 0.0));
          s += X[i * n + k] * X[j * n + k] * sc;
        }
        h[(size_t)p * n * n + (size_t)j * n + i] = s;
      }
  }
  double *dG, *dV, *dVH, *dev;
  int *dn, *dperm, *dst;
  cudaMalloc(&dG, 8 * h.size()); cudaMemcpy(dG, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&dV, 8 * h.size()); cudaMalloc(&dVH, 8 * h.size()); cudaMalloc(&dev, 8 * (size_t)n * P);
  cudaMalloc(&dperm, 4 * (size_t)n * P); cudaMalloc(&dst, 4 * P);
  std::vector<int> ns(P, n);
  cudaMalloc(&dn, 4 * P); cudaMemcpy(dn, ns.data(), 4 * P, cudaMemcpyHostToDevice);
  Ctx c; c.stream = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(dG, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);  // the n > 160 path works in place
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = launch_syev(c, dG, n, (int64_t)n * n, dn, P, n, dV, (int64_t)n * n, dVH, dev, dperm, n, dst);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("syev n=%d P=%d: %.3f ms launch=%s sync=%s\n", n, P, ms, cudaGetErrorString(e), cudaGetErrorString(cudaDeviceSynchronize()));
  }
  std::vector<double> V(h.size()), ev((size_t)n * P);
  std::vector<int> perm((size_t)n * P), st(P);
  cudaMemcpy(V.data(), dV, 8 * V.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(ev.data(), dev, 8 * ev.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(perm.data(), dperm, 4 * perm.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(st.data(), dst, 4 * P, cudaMemcpyDeviceToHost);
  for (int p = 0; p < 3 && p < P; ++p) {
    const double* G = &h[(size_t)p * n * n];
    const double* Vp = &V[(size_t)p * n * n];
    double res = 0, orth = 0, gn = 0;
    for (int l = 0; l < n; ++l) {
      const double* v = Vp + (size_t)perm[(size_t)p * n + l] * n;
      double lam = ev[(size_t)p * n + l];
      for (int i = 0; i < n; ++i) {
        double s = 0;
        for (int k = 0; k < n; ++k) s += G[(size_t)k * n + i] * v[k];
        res = fmax(res, fabs(s - lam * v[i]));
      }
      for (int l2 = 0; l2 < n; ++l2) {
        const double* u = Vp + (size_t)perm[(size_t)p * n + l2] * n;
        double s = 0;
        for (int k = 0; k < n; ++k) s += u[k] * v[k];
        orth = fmax(orth, fabs(s - (l == l2 ? 1.0 : 0.0)));
      }
    }
    for (size_t i = 0; i < (size_t)n * n; ++i) gn = fmax(gn, fabs(G[i]));
    printf("p=%d iters=%d  max|GV-VL|/max|G| = %.3e  max|VtV-I| = %.3e  l0=%.6e l_last=%.6e\n", p, st[p], res / gn,
           orth, ev[(size_t)p * n], ev[(size_t)p * n + n - 1]);
  }
  return 0;
}

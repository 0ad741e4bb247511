// Standalone check of k_gemm_ws.cu (the warp-specialised TMA-fed 3xTF32 kernel): each mode against a
// double-precision host product of ITS OWN inputs (Z from Q, F; R' from Q, the GPU's Z, F; W' from the GPU's
// R' planes), on a small collection with ragged tiles.  Build: tools/build_ws_test.sh; run on a B200.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2601_11626_b200/csrc/k_gemm_ws.cu"

namespace cmsvd {
cudaError_t ensure(DevMem& b, size_t bytes) {
  if (b.bytes >= bytes) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.bytes = bytes;
  return cudaMalloc(&b.p, bytes);
}
}  // namespace cmsvd
using namespace cmsvd;

#define CKC(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoi(argv[1]) : 256;
  const int kc = argc > 2 ? atoi(argv[2]) : 256;
  const int P = argc > 4 ? atoi(argv[4]) : 3;      // P > 3: timing only (uniform q = w = kc)
  const int N = P > 3 ? 8 : 3;
  Ctx c;
  c.m = m; c.count = N;
  cudaStreamCreate(&c.stream);
  cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, 0);
  std::vector<float> U((size_t)N * kc * m), F((size_t)N * kc * m);
  srand(1);
  for (auto& x : U) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : F) x = (float)rand() / RAND_MAX - 0.5f;
  float *dU, *dF;
  CKC(cudaMalloc(&dU, U.size() * 4)); CKC(cudaMalloc(&dF, F.size() * 4));
  CKC(cudaMemcpy(dU, U.data(), U.size() * 4, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(dF, F.data(), F.size() * 4, cudaMemcpyHostToDevice));
  CKC(ensure(c.d_Qp, U.size() * 8)); CKC(ensure(c.d_Fp, U.size() * 8)); CKC(ensure(c.d_QTp, U.size() * 8));
  CKC(launch_split_planes_t(c, dU, (int64_t)kc * m, m, kc, N, (float*)c.d_QTp.p));
  CKC(launch_split_planes(c, dU, (int64_t)kc * m, m, kc, kc, N, (float*)c.d_Qp.p));
  CKC(launch_split_planes(c, dF, (int64_t)kc * m, m, kc, kc, N, (float*)c.d_Fp.p));
  c.planes_cols = kc; c.planes_ok = true; c.planes_F = dF; c.planes_fstride = (int64_t)kc * m;
  std::vector<BaseDesc> bd(N); std::vector<AppDesc> ad(N);
  const int qs[3] = {kc, kc - 5, kc - 64}, wsz[3] = {kc, kc - 3, kc - 40};
  for (int i = 0; i < N; ++i) {
    bd[i] = BaseDesc{}; bd[i].basis = dU + (size_t)i * kc * m; bd[i].q = P > 3 ? kc : qs[i]; bd[i].rr = bd[i].q;
    ad[i] = AppDesc{}; ad[i].F = dF + (size_t)i * kc * m; ad[i].w = P > 3 ? kc : wsz[i];
  }
  BaseDesc* dbd; AppDesc* dad; int2* dpr;
  CKC(cudaMalloc(&dbd, N * sizeof(BaseDesc))); CKC(cudaMalloc(&dad, N * sizeof(AppDesc))); CKC(cudaMalloc(&dpr, P * 8));
  CKC(cudaMemcpy(dbd, bd.data(), N * sizeof(BaseDesc), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(dad, ad.data(), N * sizeof(AppDesc), cudaMemcpyHostToDevice));
  std::vector<int2> hp(P);
  for (int p = 0; p < P; ++p) hp[p] = P > 3 ? make_int2((p / 7) % N, ((p / 7) % N + 1 + p % 7) % N) : make_int2(p, (p + 1) % 3);
  CKC(cudaMemcpy(dpr, hp.data(), P * 8, cudaMemcpyHostToDevice));
  const int QMAX = kc, WMAX = kc;
  float *Z, *Zp, *Rp; double* W;
  CKC(cudaMalloc(&Z, (size_t)P * QMAX * WMAX * 4)); CKC(cudaMalloc(&Zp, (size_t)P * QMAX * WMAX * 8));
  CKC(cudaMalloc(&Rp, (size_t)P * m * WMAX * 8)); CKC(cudaMalloc(&W, (size_t)P * WMAX * WMAX * 8));
  CKC(cudaMemset(Z, 0xff, (size_t)P * QMAX * WMAX * 4)); CKC(cudaMemset(Zp, 0xff, (size_t)P * QMAX * WMAX * 8));
  CKC(cudaMemset(Rp, 0xff, (size_t)P * m * WMAX * 8)); CKC(cudaMemset(W, 0, (size_t)P * WMAX * WMAX * 8));
  const int upto = argc > 3 ? atoi(argv[3]) : 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < (P > 3 ? 3 : 1); ++rep)
    for (int mode = 0; mode <= upto; ++mode) {
      cudaEventRecord(e0, c.stream);
      CKC(launch_gemm_ws(c, mode, dpr, P, dbd, dad, 1, QMAX, WMAX, Z, Zp, Rp, W));
      cudaEventRecord(e1, c.stream);
      CKC(cudaStreamSynchronize(c.stream));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * m * kc * kc * P;
      printf("mode %d: %.3f ms, %.1f TF/s fp32-equivalent\n", mode, ms, fl / ms * 1e-9);
    }
  if (P > 3) return 0;
  std::vector<float> hZ((size_t)P * QMAX * WMAX), hZp((size_t)P * QMAX * WMAX * 2), hRp((size_t)P * m * WMAX * 2);
  std::vector<double> hW((size_t)P * WMAX * WMAX);
  CKC(cudaMemcpy(hZ.data(), Z, hZ.size() * 4, cudaMemcpyDeviceToHost));
  CKC(cudaMemcpy(hZp.data(), Zp, hZp.size() * 4, cudaMemcpyDeviceToHost));
  CKC(cudaMemcpy(hRp.data(), Rp, hRp.size() * 4, cudaMemcpyDeviceToHost));
  CKC(cudaMemcpy(hW.data(), W, hW.size() * 8, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int p = 0; p < P; ++p) {
    const int bi = hp[p].x, aj = hp[p].y, q = qs[bi], w = wsz[aj];
    const float* Q = &U[(size_t)bi * kc * m]; const float* Fj = &F[(size_t)aj * kc * m];
    double ez = 0, er = 0, ew = 0, ep = 0, zmax = 0, rmax = 0, wmax = 0;
    for (int j = 0; j < WMAX; ++j)
      for (int i = 0; i < QMAX; ++i) {
        double s = 0;
        if (i < q && j < w) for (int64_t k = 0; k < m; ++k) s += (double)Q[(size_t)i * m + k] * Fj[(size_t)j * m + k];
        const size_t o = (size_t)p * QMAX * WMAX + (size_t)j * QMAX + i;
        ez = fmax(ez, fabs(hZ[o] - s)); zmax = fmax(zmax, fabs(s));
        const double hl = (double)hZp[((size_t)p * 2) * QMAX * WMAX + (size_t)j * QMAX + i] +
                          (double)hZp[((size_t)p * 2 + 1) * QMAX * WMAX + (size_t)j * QMAX + i];
        ep = fmax(ep, fabs(hl - hZ[o]));
      }
    if (upto >= 1)
      for (int j = 0; j < WMAX; ++j)
        for (int64_t i = 0; i < m; ++i) {
          double s = 0;
          if (j < w) {
            s = Fj[(size_t)j * m + i];
            for (int k = 0; k < q; ++k) s -= (double)Q[(size_t)k * m + i] * hZ[(size_t)p * QMAX * WMAX + (size_t)j * QMAX + k];
          }
          const double g = (double)hRp[((size_t)p * 2) * m * WMAX + (size_t)j * m + i] +
                           (double)hRp[((size_t)p * 2 + 1) * m * WMAX + (size_t)j * m + i];
          er = fmax(er, fabs(g - s)); rmax = fmax(rmax, fabs(s));
        }
    if (upto >= 2)
      for (int j = 0; j < w; ++j)
        for (int i = 0; i < w; ++i) {
          double s = 0;
          for (int64_t k = 0; k < m; ++k) {
            const double a = (double)hRp[((size_t)p * 2) * m * WMAX + (size_t)i * m + k] + (double)hRp[((size_t)p * 2 + 1) * m * WMAX + (size_t)i * m + k];
            const double b = (double)hRp[((size_t)p * 2) * m * WMAX + (size_t)j * m + k] + (double)hRp[((size_t)p * 2 + 1) * m * WMAX + (size_t)j * m + k];
            s += a * b;
          }
          ew = fmax(ew, fabs(hW[(size_t)p * WMAX * WMAX + (size_t)j * WMAX + i] - s)); wmax = fmax(wmax, fabs(s));
        }
    printf("pair %d (q=%d w=%d): Z err %.3e (max %.3e) planes %.3e | R err %.3e (max %.3e) | W err %.3e (max %.3e)\n",
           p, q, w, ez, zmax, ep, er, rmax, ew, wmax);
    if (!(ez <= 2e-6 * zmax + 1e-6) || !(er <= 1e-5 * (rmax + 1)) || !(ew <= 1e-5 * (wmax + 1)) || !(ep <= 1e-7 * zmax)) ++bad;
  }
  printf(bad ? "FAILED\n" : "ws_test ok\n");
  return bad != 0;
}

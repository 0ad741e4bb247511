// k_pair.cu -- per-candidate assembly and finalisation kernels of the
// merge-error pipeline (S3, S7, S8, S9) and the small block-spectra helpers.
//
// Incremental estimate (Lemma 1 + Cor. 3 + Cor. 2, PAPER.md:1297-1468,
// 490-540).  With the base state (U_r, D = diag(sigma_r)) and the appended
// operand F, F = Q Z + R' (Q = projection basis whose first rr columns are
// U_r, Z = Q^T F, R' = (I - Q Q^T) F), the Gram of the core
// K = [[D, Z_r], [0, B]] (Lemma 1's S_{t+1} in the basis [Q_t, Q_res]) is
//     G = K^T K = [[D^2, D Z_r], [Z_r^T D, Z^T Z + R'^T R']]      (rr + w)^2
// so sigma~^2 = top-r eigenvalues of G and, since trace(G) = ||[U_r D, F]||_F^2,
//     err^2_I = tail_inc(base) + extra(app) + (trace(G) - sum_{l<r} lambda_l(G))
// which equals E_base + E_app - sum_{l<=r} sigma~_l^2 (Cor. 2) with the
// dropped energy summed directly instead of by cancellation.
//
// Residual bound (Thm 2 + Cor. 1):
// mu = top-r of spec(base) u sigma(R'), sigma(R')^2 = eig(R'^T R'),
//     err^2_R = rest(base) + sum_{unselected} spec^2 + (tr(W') - sum_{sel} eig W')
//               + ||Z||_F^2 + extra(app)
// = E_base + E_app - sum_{l<=r} mu_l^2.
//
// Weyl bound (Thm 1 / Eq. 5) for K = 2:
//     err^2_W = min(tailw_i + E_j, tailw_j + E_i) = E_i + E_j - max_k top_r(A_k).
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cmsvd {

// Build the per-pair GEMM descriptors and eigen-problem sizes on the device.
__global__ void k_make_descs(const int2* __restrict__ pairs, int64_t P, const BaseDesc* __restrict__ bd,
                             const AppDesc* __restrict__ ad, int64_t m, int use_full_basis, int QMAX, int WMAX,
                             int GMAX, float* Zws, float* Rws, double* Wws, double* ZZws, GemmDesc* dZ,
                             GemmDesc* dR, GemmDesc* dW, GemmDesc* dZZ, int* nG, int* nW, double* thrW, int r) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const AppDesc a = ad[pr.y];
  const int q = use_full_basis ? b.q : b.rr;
  float* Z = Zws + p * (int64_t)QMAX * WMAX;
  float* R = Rws + p * (int64_t)m * WMAX;
  double* W = Wws + p * (int64_t)WMAX * WMAX;
  double* ZZ = ZZws + p * (int64_t)WMAX * WMAX;
  GemmDesc g;
  // Z = Q^T F  (q x w)
  g.A = b.basis; g.lda = m; g.B = a.F; g.ldb = m; g.C0 = nullptr; g.ldc0 = 0;
  g.C = Z; g.ldc = QMAX; g.M = q; g.N = a.w; g.K = (int)m; g.sym = 0;
  dZ[p] = g;
  // R' = F - Q Z  (m x w)
  g.A = b.basis; g.lda = m; g.B = Z; g.ldb = QMAX; g.C0 = a.F; g.ldc0 = m;
  g.C = R; g.ldc = m; g.M = (int)m; g.N = a.w; g.K = q; g.sym = 0;
  dR[p] = g;
  // W' = R'^T R'  (w x w, fp64 accumulation)
  g.A = R; g.lda = m; g.B = R; g.ldb = m; g.C0 = nullptr; g.ldc0 = 0;
  g.C = W; g.ldc = WMAX; g.M = a.w; g.N = a.w; g.K = (int)m; g.sym = 1;
  dW[p] = g;
  // Z^T Z (w x w, fp64 accumulation)
  g.A = Z; g.lda = QMAX; g.B = Z; g.ldb = QMAX; g.C0 = nullptr; g.ldc0 = 0;
  g.C = ZZ; g.ldc = WMAX; g.M = a.w; g.N = a.w; g.K = q; g.sym = 1;
  dZZ[p] = g;
  nG[p] = b.rr + a.w;
  nW[p] = a.w;
  thrW[p] = (b.ns >= r) ? b.spec[r - 1] * b.spec[r - 1] : 0.0;
  (void)GMAX;
}

// G = [[D^2, D Z_r], [Z_r^T D, ZZ + W]] (fp64, ld GMAX) and ||Z||_F^2.
__global__ void __launch_bounds__(kThreads) k_build_G(const int2* __restrict__ pairs, const BaseDesc* __restrict__ bd,
                                                      const AppDesc* __restrict__ ad, int QMAX, int WMAX, int GMAX,
                                                      const float* __restrict__ Zws, const double* __restrict__ Wws,
                                                      const double* __restrict__ ZZws, double* __restrict__ Gws,
                                                      double* __restrict__ zn2) {
  const int64_t p = blockIdx.x;
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const int w = ad[pr.y].w;
  const int rr = b.rr;
  const int n = rr + w;
  const float* Z = Zws + p * (int64_t)QMAX * WMAX;
  const double* W = Wws + p * (int64_t)WMAX * WMAX;
  const double* ZZ = ZZws + p * (int64_t)WMAX * WMAX;
  double* G = Gws + p * (int64_t)GMAX * GMAX;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e % n, j = e / n;
    double v;
    if (i < rr && j < rr) v = (i == j) ? b.spec[i] * b.spec[i] : 0.0;
    else if (i < rr) v = b.spec[i] * (double)Z[(int64_t)(j - rr) * QMAX + i];
    else if (j < rr) v = b.spec[j] * (double)Z[(int64_t)(i - rr) * QMAX + j];
    else v = ZZ[(int64_t)(j - rr) * WMAX + (i - rr)] + W[(int64_t)(j - rr) * WMAX + (i - rr)];
    G[(int64_t)j * GMAX + i] = v;
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < w; ++i) s += ZZ[(int64_t)i * WMAX + i];
    if (b.full)  // A22: ||F||^2 = ||U_r^T F||^2 + ||(I - U_r U_r^T) F||^2 (whole operand is "residual-free")
      for (int i = 0; i < w; ++i) s += W[(int64_t)i * WMAX + i];
    zn2[p] = s;
  }
}

// Final per-pair combination (S3, S7, S8, S9): one thread per pair.
__global__ void k_finalize(const int2* __restrict__ pairs, int64_t P, const BaseDesc* __restrict__ bd,
                           const AppDesc* __restrict__ ad, int r, unsigned kinds, const double* __restrict__ evG,
                           const int* __restrict__ cntG, const double* __restrict__ trG,
                           const double* __restrict__ evW, const int* __restrict__ cntW,
                           const double* __restrict__ trW, const double* __restrict__ zn2, double* __restrict__ err2,
                           double* __restrict__ total, float* __restrict__ sigma_tilde, float* __restrict__ mu) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const AppDesc a = ad[pr.y];
  const double tot = b.E + a.E;
  total[p] = tot;
  double ew = nan(""), er = nan(""), ei = nan("");
  if (kinds & CMSVD_WEYL) {
    ew = fmin(b.tailw + a.E, a.tailw + b.E);
  }
  if (kinds & CMSVD_INCREMENTAL) {
    const double* ev = evG + p * r;
    int c = cntG[p];
    double top = 0.0;
    for (int l = 0; l < r; ++l) {
      double lam = (l < c) ? fmax(ev[l], 0.0) : 0.0;
      top += lam;
      if (sigma_tilde) sigma_tilde[p * r + l] = (float)sqrt(lam);
    }
    ei = b.tail_inc + a.extra + fmax(trG[p] - top, 0.0);
  } else if (sigma_tilde) {
    for (int l = 0; l < r; ++l) sigma_tilde[p * r + l] = nanf("");
  }
  if (kinds & CMSVD_RESIDUAL) {
    const double* ev = b.full ? nullptr : evW + p * r;
    int c = b.full ? 0 : cntW[p];
    int ib = 0, iw = 0;
    double sel_w = 0.0;
    for (int l = 0; l < r; ++l) {
      double sb = (ib < b.ns) ? b.spec[ib] : -1.0;
      double sw = (iw < c) ? sqrt(fmax(ev[iw], 0.0)) : -1.0;
      double v;
      if (sb < 0.0 && sw < 0.0) v = 0.0;
      else if (sb >= sw) { v = sb; ++ib; }
      else { v = sw; sel_w += fmax(ev[iw], 0.0); ++iw; }
      if (mu) mu[p * r + l] = (float)v;
    }
    double unsel = 0.0;
    for (int l = ib; l < b.ns; ++l) unsel += b.spec[l] * b.spec[l];
    // A22 (full-range base): R = 0, mu = top-r sigma(A_i), err^2 = E_i - sum_sel sigma^2 + ||F||^2 + extra
    er = b.rest_res + unsel + (b.full ? 0.0 : fmax(trW[p] - sel_w, 0.0)) + zn2[p] + a.extra;
  } else if (mu) {
    for (int l = 0; l < r; ++l) mu[p * r + l] = nanf("");
  }
  auto clampv = [&](double v) { return isnan(v) ? v : fmin(fmax(v, 0.0), tot); };
  err2[3 * p + 0] = clampv(ew);
  err2[3 * p + 1] = clampv(er);
  err2[3 * p + 2] = clampv(ei);
}

// Tighter certified variants beyond the paper, one thread per pair:
//   err2x[2p]   = residual bound with the tracked basis U_r (A4): mu = top-r of sigma(A_i) U sigma(R_r),
//                 R_r = (I - U_r U_r^T) F, summed as the dropped part like k_finalize;
//   err2x[2p+1] = per-index Weyl bound E_i + E_j - sum_{l<r} max(sigma_l(A_i), sigma_l(A_j))^2 (A8; the
//                 inequality sigma_l(M) >= sigma_l(A_k) of the proof line PAPER.md:1530-1533).
// zn2[p] = ||U_r^T F||_F^2; evW/cntW/trW = eigenvalues of R_r^T R_r above sigma_r(A_i)^2.
__global__ void k_finalize_tight(const int2* __restrict__ pairs, int64_t P, const BaseDesc* __restrict__ bd,
                                 const AppDesc* __restrict__ ad, int r, const double* __restrict__ evW,
                                 const int* __restrict__ cntW, const double* __restrict__ trW,
                                 const double* __restrict__ zn2, double* __restrict__ err2x,
                                 double* __restrict__ total) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const AppDesc a = ad[pr.y];
  const double tot = b.E + a.E;
  total[p] = tot;
  // residual with U_r
  const double* ev = evW + p * r;
  const int c = cntW[p];
  int ib = 0, iw = 0;
  double sel_w = 0.0;
  for (int l = 0; l < r; ++l) {
    const double sb = (ib < b.ns) ? b.spec[ib] : -1.0;
    const double sw = (iw < c) ? sqrt(fmax(ev[iw], 0.0)) : -1.0;
    if (sb < 0.0 && sw < 0.0) break;
    if (sb >= sw) ++ib;
    else { sel_w += fmax(ev[iw], 0.0); ++iw; }
  }
  double unsel = 0.0;
  for (int l = ib; l < b.ns; ++l) unsel += b.spec[l] * b.spec[l];
  const double er = b.rest_res + unsel + fmax(trW[p] - sel_w, 0.0) + zn2[p] + a.extra;
  // per-index Weyl: sum of the dropped part, E_i + E_j - sum_{l<r} max^2 =
  //   (E_i - sum_{l<r} s_il^2) + (E_j - sum_{l<r} s_jl^2) + sum_{l<r} min(s_il, s_jl)^2
  double mn = 0.0;
  for (int l = 0; l < r; ++l) {
    const double si = (l < b.ns) ? b.spec[l] : 0.0, sj = (l < a.ns) ? a.spec[l] : 0.0;
    const double lo = fmin(si, sj);
    mn += lo * lo;
  }
  const double ew = b.tailw + a.tailw + mn;
  auto clampv = [&](double v) { return fmin(fmax(v, 0.0), tot); };
  err2x[2 * p + 0] = clampv(er);
  err2x[2 * p + 1] = clampv(ew);
}

// ||Z||_F^2 per pair (rows < QMAX of a q x w fp32 block, ld QMAX), fp64 accumulation; one CTA per pair.
__global__ void __launch_bounds__(kThreads) k_znorm(const int2* __restrict__ pairs, const BaseDesc* __restrict__ bd,
                                                    const AppDesc* __restrict__ ad, const float* __restrict__ Zws,
                                                    int QMAX, int WMAX, double* __restrict__ zn2) {
  __shared__ double red[kThreads / 32];
  const int64_t p = blockIdx.x;
  const int2 pr = pairs[p];
  const int q = bd[pr.x].rr, w = ad[pr.y].w;
  const float* Z = Zws + p * (int64_t)QMAX * WMAX;
  double acc = 0.0;
  for (int e = threadIdx.x; e < q * w; e += blockDim.x) {
    const double z = Z[(int64_t)(e / q) * QMAX + (e % q)];
    acc = fma(z, z, acc);
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) zn2[p] = s;
}

// Single-problem G builder for cluster commits (same layout as k_build_G).
__global__ void k_build_G1(int rr, int w, const double* __restrict__ spec, const float* __restrict__ Z, int ldz,
                           const double* __restrict__ ZZ, const double* __restrict__ WW, double* __restrict__ G) {
  const int n = rr + w;
  const int ldw = w > 0 ? w : 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    int i = e % n, j = e / n;
    double v;
    if (i < rr && j < rr) v = (i == j) ? spec[i] * spec[i] : 0.0;
    else if (i < rr) v = spec[i] * (double)Z[(int64_t)(j - rr) * ldz + i];
    else if (j < rr) v = spec[j] * (double)Z[(int64_t)(i - rr) * ldz + j];
    else v = ZZ[(int64_t)(j - rr) * ldw + (i - rr)] + WW[(int64_t)(j - rr) * ldw + (i - rr)];
    G[(int64_t)j * n + i] = v;
  }
}

cudaError_t launch_build_G1(Ctx& c, int rr, int w, const double* spec, const float* Z, int ldz, const double* ZZ,
                            const double* WW, double* G) {
  int n = rr + w;
  int blocks = (n * n + 255) / 256;
  if (blocks < 1) blocks = 1;
  k_build_G1<<<blocks, 256, 0, c.stream>>>(rr, w, spec, Z, ldz, ZZ, WW, G);
  c.launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Block-spectra helpers (S2)
// ---------------------------------------------------------------------------
// Per block: sigma_l = sqrt(max(lambda_l, 0)) (fp64, non-increasing), rank,
// rr = min(r, rank), tail sums, fp32 sigma output, BaseDesc/AppDesc.
__global__ void k_spec_stats(int count, int nmax, int r, const double* __restrict__ evals,
                             const int* __restrict__ kcols, const double* __restrict__ E, double* __restrict__ sig,
                             float* __restrict__ sig32, int* __restrict__ rank, const int64_t* __restrict__ uoff,
                             const float* __restrict__ Ubase, const int64_t* __restrict__ boff,
                             const int* __restrict__ ncols, const float* __restrict__ arena,
                             const int64_t* __restrict__ foff, const float* __restrict__ Fbase,
                             BaseDesc* __restrict__ bd, AppDesc* __restrict__ ad_raw, AppDesc* __restrict__ ad_trunc,
                             double tau) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int k = kcols[i];
  const double* ev = evals + (int64_t)i * nmax;
  double* s = sig + (int64_t)i * nmax;
  double all = 0.0;
  for (int l = 0; l < k; ++l) {
    s[l] = sqrt(fmax(ev[l], 0.0));
    all += fmax(ev[l], 0.0);
  }
  for (int l = k; l < nmax; ++l) s[l] = 0.0;
  int rk = 0;
  if (k > 0 && s[0] > 0.0)
    for (int l = 0; l < k; ++l) rk += (s[l] > tau * s[0]);
  rank[i] = rk;
  const int rr = rk < r ? rk : r;
  double tail_inc = 0.0, tailw = 0.0;
  for (int l = k - 1; l >= rr; --l) tail_inc += fmax(ev[l], 0.0);
  for (int l = k - 1; l >= r; --l) tailw += fmax(ev[l], 0.0);
  for (int l = 0; l < r; ++l) sig32[(int64_t)i * r + l] = (l < k) ? (float)s[l] : 0.f;
  const double Ei = E[i];
  BaseDesc b;
  b.basis = Ubase + uoff[i];
  b.spec = s;
  b.q = rk;
  b.rr = rr;
  b.ns = k;
  b.full = 0;
  b.E = Ei;
  b.tail_inc = tail_inc;
  b.rest_res = fmax(Ei - all, 0.0);
  b.tailw = tailw;
  bd[i] = b;
  AppDesc a;
  a.F = arena + boff[i];
  a.w = ncols[i];
  a.ns = k;
  a.spec = s;
  a.E = Ei;
  a.extra = 0.0;
  a.tailw = tailw;
  ad_raw[i] = a;
  a.F = Fbase + foff[i];
  a.w = rr;
  a.extra = tail_inc + fmax(Ei - all, 0.0);
  ad_trunc[i] = a;
}

// U[:, l] = A V[:, perm[l]] / sigma_l for l < rank (else 0); fp64 accumulation.
__global__ void __launch_bounds__(kThreads) k_leftvec(int64_t m, const float* __restrict__ arena,
                                                      const int64_t* __restrict__ boff, const int* __restrict__ kcols,
                                                      const double* __restrict__ V, int64_t strideV,
                                                      const int* __restrict__ perm, int nmax,
                                                      const double* __restrict__ sig, const int* __restrict__ rank,
                                                      float* __restrict__ U, const int64_t* __restrict__ uoff) {
  const int blk = blockIdx.z;
  const int l = blockIdx.y;
  const int k = kcols[blk];
  if (l >= k) return;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  float* u = U + uoff[blk] + (int64_t)l * m;
  if (l >= rank[blk]) { u[row] = 0.f; return; }
  const double* v = V + (int64_t)blk * strideV + (int64_t)perm[(int64_t)blk * nmax + l] * k;
  const float* A = arena + boff[blk];
  double acc = 0.0;
  for (int c = 0; c < k; ++c) acc = fma((double)A[(int64_t)c * m + row], v[c], acc);
  u[row] = (float)(acc / sig[(int64_t)blk * nmax + l]);
}

// TRUNC operand F_i = U_i[:, :rr] diag(sigma_i[:rr]) (fp32).
__global__ void k_trunc_operand(int64_t m, const BaseDesc* __restrict__ bd, const AppDesc* __restrict__ ad_trunc,
                                float* Fbase) {
  const int blk = blockIdx.z, l = blockIdx.y;
  const BaseDesc b = bd[blk];
  if (l >= b.rr) return;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  float* F = const_cast<float*>(ad_trunc[blk].F);
  F[(int64_t)l * m + row] = (float)((double)b.basis[(int64_t)l * m + row] * b.spec[l]);
}

}  // namespace cmsvd

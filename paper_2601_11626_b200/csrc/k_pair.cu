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

// G = [[D^2, D Z_r], [Z_r^T D, ZZ + W]] (fp64, ld GMAX) and ||Z||_F^2.  Only the lower triangles of W and ZZ
// are read (their producers may leave the strict upper triangle uncomputed).  upper: 0 = G written in full,
// 1 = the strict upper triangle of G is not written (the band reduction reads the lower storage only),
// 2 = it is poisoned with NaN (test knob CMSVD_G_POISON=1: proves that nothing downstream reads it).
__global__ void __launch_bounds__(kThreads) k_build_G(const int2* __restrict__ pairs, const BaseDesc* __restrict__ bd,
                                                      const AppDesc* __restrict__ ad, int QMAX, int WMAX, int GMAX,
                                                      const float* __restrict__ Zws, const double* __restrict__ Wws,
                                                      const double* __restrict__ ZZws, double* __restrict__ Gws,
                                                      double* __restrict__ zn2, int upper) {
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
    if (i < j && upper) {
      if (upper == 2) G[(int64_t)j * GMAX + i] = __longlong_as_double(0x7ff8000000000000ll);
      continue;
    }
    double v;
    if (i < rr && j < rr) v = (i == j) ? b.spec[i] * b.spec[i] : 0.0;
    else if (i < rr) v = b.spec[i] * (double)Z[(int64_t)(j - rr) * QMAX + i];
    else if (j < rr) v = b.spec[j] * (double)Z[(int64_t)(i - rr) * QMAX + j];
    else {
      const int a = max(i, j) - rr, c = min(i, j) - rr;   // (row a, column c) of the lower triangle
      v = (ZZws ? ZZ[(int64_t)c * WMAX + a] : 0.0) + W[(int64_t)c * WMAX + a];
    }
    G[(int64_t)j * GMAX + i] = v;
  }
  if (threadIdx.x == 0) {
    // ZZws == nullptr: W already holds Z^T Z + R'^T R' (fused by k_gemm_ws; full bases only)
    double s = 0.0;
    if (ZZws)
      for (int i = 0; i < w; ++i) s += ZZ[(int64_t)i * WMAX + i];
    if (b.full || !ZZws)  // A22: ||F||^2 = ||U_r^T F||^2 + ||(I - U_r U_r^T) F||^2 (whole operand is "residual-free")
      for (int i = 0; i < w; ++i) s += W[(int64_t)i * WMAX + i];
    zn2[p] = s;
  }
}

// Z^T Z (fp64 accumulation) for w <= 128, replacing k_gemm_tn<double> on Z: one CTA per pair; the 136
// lower-triangular 8x8 tiles of the 128 x 128 product are owned by threads 0..135.  Rows of Z arrive 32
// at a time by cp.async into a double-buffered fp32 staging area (no registers held across the
// products), are widened once into the fp64 operand rows, and each thread accumulates its tile; the
// tile and its mirror are stored (store-only epilogue).  The accumulation is the sequential fma over k of
// k_gemm_tn (fp32 products are exact in fp64): bitwise the same ZZ.
constexpr int kZZThreads = 160;
constexpr int kZZBK = 32;
constexpr int kZZLD = 162;  // doubles per operand row (tile t at 10 t: 8 + 2 pad; +2 spreads the widening stores)
constexpr size_t kZZSmem = (size_t)kZZBK * kZZLD * 8 + 2 * (size_t)kZZBK * 128 * 4;

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}

__global__ void __launch_bounds__(kZZThreads, 2) k_syrk_zz(const int2* __restrict__ pairs,
                                                           const BaseDesc* __restrict__ bd,
                                                           const AppDesc* __restrict__ ad, int use_full_basis,
                                                           int QMAX, int WMAX, const float* __restrict__ Zws,
                                                           double* __restrict__ ZZws) {
  extern __shared__ __align__(16) unsigned char zz_smem[];
  double* Zs = reinterpret_cast<double*>(zz_smem);
  float* Zst = reinterpret_cast<float*>(zz_smem + (size_t)kZZBK * kZZLD * 8);   // [2][128 cols][32 rows]
  const int64_t p = blockIdx.x;
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const int w = ad[pr.y].w;
  const int q = use_full_basis ? b.q : b.rr;
  const float* Z = Zws + p * (int64_t)QMAX * WMAX;
  double* ZZ = ZZws + p * (int64_t)WMAX * WMAX;
  const int tid = threadIdx.x;
  int ti = 0, tj = tid;
  while (tj > ti) { ++ti; tj -= ti; }                        // tid = ti (ti + 1) / 2 + tj, tj <= ti
  const bool active = tid < 136 && 8 * tj < w;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  auto fetch = [&](int l0, float* dst) {
    for (int e = tid; e < kZZBK * 128; e += kZZThreads) {
      const int l = e & (kZZBK - 1), j = e >> 5;
      const bool v = l0 + l < q && j < w;
      cp_async4(dst + e, v ? Z + (int64_t)j * QMAX + l0 + l : Z, v);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nch = (q + kZZBK - 1) / kZZBK;
  if (nch > 0) fetch(0, Zst);
  for (int c = 0; c < nch; ++c) {
    const int l0 = c * kZZBK;
    if (c + 1 < nch) {
      fetch(l0 + kZZBK, Zst + ((c + 1) & 1) * kZZBK * 128);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // chunk c staged by every thread; the previous products are done with Zs
    const float* src = Zst + (c & 1) * kZZBK * 128;
    for (int e = tid; e < kZZBK * 128; e += kZZThreads) {
      const int l = e & (kZZBK - 1), j = e >> 5;
      Zs[l * kZZLD + j + 2 * (j >> 3)] = (double)src[e];
    }
    __syncthreads();
    if (active) {
      const int lmax = min(kZZBK, q - l0);
      for (int l = 0; l < lmax; ++l) {
        const double* row = Zs + l * kZZLD;
        double a[8], bb[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 x = *reinterpret_cast<const double2*>(row + 10 * ti + 2 * u);
          const double2 y = *reinterpret_cast<const double2*>(row + 10 * tj + 2 * u);
          a[2 * u] = x.x; a[2 * u + 1] = x.y;
          bb[2 * u] = y.x; bb[2 * u + 1] = y.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gj = 8 * tj + j;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gi = 8 * ti + i;
        if (gi < w && gj < w) {
          ZZ[(int64_t)gj * WMAX + gi] = acc[i][j];
          if (ti != tj) ZZ[(int64_t)gi * WMAX + gj] = acc[i][j];
        }
      }
    }
  }
}

cudaError_t launch_syrk_zz(Ctx& c, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad,
                           int use_full_basis, int QMAX, int WMAX, const float* Zws, double* ZZws) {
  if (P <= 0) return cudaSuccess;
  if (WMAX > 128) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_syrk_zz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZZSmem);
  if (e != cudaSuccess) return e;
  k_syrk_zz<<<(unsigned)P, kZZThreads, kZZSmem, c.stream>>>(pairs, bd, ad, use_full_basis, QMAX, WMAX, Zws, ZZws);
  c.launches += 1;
  return cudaGetLastError();
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
    // zn2 == nullptr: no projection was computed (A22 base, residual without the incremental estimator);
    // then ||F||^2 = E_app - extra by the appended block's spectrum
    er = b.rest_res + unsel + (b.full ? 0.0 : fmax(trW[p] - sel_w, 0.0)) + (zn2 ? zn2[p] : a.E - a.extra) + a.extra;
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

// U[:, l] = A V[:, perm[l]] / sigma_l for l < rank (else 0); fp64 accumulation, sequential over the
// columns of A.  A thread computes kLvCols columns l of one row (A read once per kLvCols products), the
// CTA's V columns are staged in shared memory.  Grid: (ceil(m / kThreads), ceil(nmax / kLvCols), count).
constexpr int kLvCols = 8;
__global__ void __launch_bounds__(kThreads) k_leftvec(int64_t m, const float* __restrict__ arena,
                                                      const int64_t* __restrict__ boff, const int* __restrict__ kcols,
                                                      const double* __restrict__ V, int64_t strideV,
                                                      const int* __restrict__ perm, int nmax,
                                                      const double* __restrict__ sig, const int* __restrict__ rank,
                                                      float* __restrict__ U, const int64_t* __restrict__ uoff) {
  extern __shared__ double lv_smem[];                     // kLvCols x k
  const int blk = blockIdx.z;
  const int l0 = blockIdx.y * kLvCols;
  const int k = kcols[blk];
  if (l0 >= k) return;
  const int rk = rank[blk];
  const int nl = min(kLvCols, k - l0);
  for (int e = threadIdx.x; e < kLvCols * k; e += blockDim.x) {
    const int t = e / k, c = e % k;
    lv_smem[e] = (t < nl && l0 + t < rk)
                     ? V[(int64_t)blk * strideV + (int64_t)perm[(int64_t)blk * nmax + l0 + t] * k + c]
                     : 0.0;
  }
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  const float* A = arena + boff[blk];
  double acc[kLvCols];
#pragma unroll
  for (int t = 0; t < kLvCols; ++t) acc[t] = 0.0;
#pragma unroll 4
  for (int c = 0; c < k; ++c) {
    const double a = (double)A[(int64_t)c * m + row];
#pragma unroll
    for (int t = 0; t < kLvCols; ++t) acc[t] = fma(a, lv_smem[t * k + c], acc[t]);
  }
  float* Ub = U + uoff[blk];
#pragma unroll
  for (int t = 0; t < kLvCols; ++t) {
    const int l = l0 + t;
    if (t < nl) Ub[(int64_t)l * m + row] = (l < rk) ? (float)(acc[t] / sig[(int64_t)blk * nmax + l]) : 0.f;
  }
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

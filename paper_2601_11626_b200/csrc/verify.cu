// verify.cu -- cluster verification and compression accounting (SURVEY.md
// §8(f) N1; PAPER.md:142-173 per-cluster truncated SVD M_c ~ U_c S_c V_c^T,
// Ũ_c = U_c S_c, mem_c = r_c (m + N_c); PAPER.md:579-597 relative
// reconstruction error and compression ratio).
//
// For each cluster c of a partition, the exact rank-r error of the explicit
// concatenation M_c (Thm EYM: the error of the rank-r
// truncated SVD, i.e. of the reconstruction Ũ_c V_c^T) is
//   err2_c = sum_{j>r} sigma_j^2(M_c) = tr(Gram) - sum_{j<=r} lambda_j(Gram),
// with Gram = M_c^T M_c (N_c <= m) or M_c M_c^T (m < N_c), both fp64
// accumulated from the fp32 blocks; the eigenvalues come from the batched
// tridiagonalisation + bisection (k_eig.cu), so min(m, N_c) <= 512.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "kernels.cuh"

namespace cmsvd {

// C (n x n, fp64, ld n) = X^T X for X (m x n fp32, column-major, ld m) if !ROWS,
// or X X^T (m x m) if ROWS; 64x64 output tiles, fp64 accumulation, one batch
// entry per cluster (blockIdx.z) with its own X pointer / n.
template <bool ROWS>
__global__ void __launch_bounds__(256) k_gram(const float* const* __restrict__ Xs, const int* __restrict__ ncols,
                                              int64_t m, double* const* __restrict__ Cs, int64_t ldc) {
  constexpr int BT = 64, BK = 16;
  __shared__ double As[BK][BT + 1];
  __shared__ double Bs[BK][BT + 1];
  const float* X = Xs[blockIdx.z];
  if (!X) return;  // this cluster takes the other orientation
  const int n = ncols[blockIdx.z];
  const int64_t N = ROWS ? m : n;   // output dimension
  const int64_t K = ROWS ? n : m;   // contraction length
  const int64_t i0 = (int64_t)blockIdx.x * BT, j0 = (int64_t)blockIdx.y * BT;
  if (i0 >= N || j0 >= N) return;
  double* C = Cs[blockIdx.z];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = tid + 256 * t;
      // operand element (row i of the output, k): ROWS -> X[k*m + i]; else X[i*m + k]
      if (ROWS) {
        const int i = e & 63, k = e >> 6;
        const int64_t gi = i0 + i, gj = j0 + i, gk = k0 + k;
        As[k][i] = (gi < N && gk < K) ? (double)X[gk * m + gi] : 0.0;
        Bs[k][i] = (gj < N && gk < K) ? (double)X[gk * m + gj] : 0.0;
      } else {
        const int k = e & 15, i = e >> 4;
        const int64_t gi = i0 + i, gj = j0 + i, gk = k0 + k;
        As[k][i] = (gi < N && gk < K) ? (double)X[gi * m + gk] : 0.0;
        Bs[k][i] = (gj < N && gk < K) ? (double)X[gj * m + gk] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[k][tx + 16 * q]; b[q] = Bs[k][ty + 16 * q]; }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + tx + 16 * p, j = j0 + ty + 16 * q;
      if (i < N && j < N) C[j * ldc + i] = acc[p][q];
    }
}

#define CKV(expr, where)                                   \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return cuda_fail(c, _e, where); \
  } while (0)

constexpr int64_t kVerifyMax = 4096;

Status do_cluster_verify(Ctx& c, int32_t r, const int32_t* assign, int32_t n_clusters, double* exact_err2,
                         double* total, int64_t* mem) {
  if (c.count <= 0) return fail(c, CMSVD_E_STATE, "cluster_verify: no collection registered");
  if (r < 1 || n_clusters < 0 || !assign) return fail(c, CMSVD_E_ARG, "cluster_verify: need r >= 1, assign");
  if (n_clusters == 0) return CMSVD_OK;
  if (!exact_err2 || !total || !mem) return fail(c, CMSVD_E_ARG, "cluster_verify: outputs are required");
  const int N = c.count;
  const int64_t m = c.m;
  std::vector<std::vector<int>> members(n_clusters);
  for (int i = 0; i < N; ++i) {
    if (assign[i] < 0 || assign[i] >= n_clusters)
      return fail(c, CMSVD_E_ARG, "cluster_verify: assign[" + std::to_string(i) + "] out of range");
    members[assign[i]].push_back(i);
  }
  std::vector<int64_t> ncol(n_clusters, 0), dim(n_clusters, 0), xoff(n_clusters + 1, 0);
  int dmax = 1;
  for (int g = 0; g < n_clusters; ++g) {
    if (members[g].empty()) return fail(c, CMSVD_E_ARG, "cluster_verify: empty cluster " + std::to_string(g));
    for (int i : members[g]) ncol[g] += c.n[i];
    dim[g] = std::min<int64_t>(m, ncol[g]);
    // the Gram's eigenvalues: n <= 512 by the pair path's solvers, up to kVerifyMax by the two-stage
    // reduction with the panel and the band in global memory (k_sbr.cu)
    if (dim[g] > kVerifyMax)
      return fail(c, CMSVD_E_SHAPE, "cluster_verify: min(m, N_c) = " + std::to_string(dim[g]) + " > " +
                                        std::to_string(kVerifyMax) + " for cluster " + std::to_string(g));
    dmax = std::max<int>(dmax, (int)dim[g]);
    xoff[g + 1] = xoff[g] + ((m * ncol[g] + 31) / 32) * 32;
  }
  // one fp64 Gram slot of dmax^2 per cluster, same stride for the eigen-solver
  const int64_t gs = (int64_t)dmax * dmax;
  CKV(ensure(c.ws[WS_A], (size_t)xoff[n_clusters] * 4), "cluster_verify: concatenations");
  CKV(ensure(c.ws[WS_G], (size_t)n_clusters * gs * 8), "cluster_verify: Grams");
  CKV(ensure(c.ws[WS_EV], (size_t)n_clusters * r * 8 + (size_t)n_clusters * 16 + 256), "cluster_verify: ev");
  CKV(ensure(c.ws[WS_PAIR], tridiag_scratch_bytes(n_clusters, dmax)), "cluster_verify: scratch");
  CKV(ensure(c.ws[WS_META], (size_t)n_clusters * 24 + 256), "cluster_verify: meta");
  float* X = (float*)c.ws[WS_A].p;
  double* G = (double*)c.ws[WS_G].p;
  // gather each cluster's blocks into a contiguous m x N_c concatenation (column order = member order)
  for (int g = 0; g < n_clusters; ++g) {
    int64_t col = 0;
    for (int i : members[g]) {
      CKV(cudaMemcpyAsync(X + xoff[g] + col * m, (const float*)c.arena.p + c.boff[i], (size_t)m * c.n[i] * 4,
                          cudaMemcpyDeviceToDevice, c.stream),
          "cluster_verify: gather");
      col += c.n[i];
    }
  }
  // Grams, split by orientation (two launches at most)
  std::vector<const float*> hx(n_clusters);
  std::vector<double*> hg(n_clusters);
  std::vector<int> hn(n_clusters), hd(n_clusters);
  for (int g = 0; g < n_clusters; ++g) {
    hx[g] = X + xoff[g];
    hg[g] = G + g * gs;
    hn[g] = (int)ncol[g];
    hd[g] = (int)dim[g];
  }
  char* mb = (char*)c.ws[WS_META].p;
  const float** dX = (const float**)mb;
  double** dG = (double**)(dX + n_clusters);
  int* dN = (int*)(dG + n_clusters);
  int* dD = dN + n_clusters;
  CKV(cudaMemcpyAsync(dX, hx.data(), (size_t)n_clusters * 8, cudaMemcpyHostToDevice, c.stream), "cluster_verify: h2d");
  CKV(cudaMemcpyAsync(dG, hg.data(), (size_t)n_clusters * 8, cudaMemcpyHostToDevice, c.stream), "cluster_verify: h2d");
  CKV(cudaMemcpyAsync(dN, hn.data(), (size_t)n_clusters * 4, cudaMemcpyHostToDevice, c.stream), "cluster_verify: h2d");
  CKV(cudaMemcpyAsync(dD, hd.data(), (size_t)n_clusters * 4, cudaMemcpyHostToDevice, c.stream), "cluster_verify: h2d");
  // the Gram kernel reads the orientation per launch: launch all clusters with the column Gram where
  // N_c <= m and the row Gram where N_c > m (each launch skips the other kind through a null pointer)
  std::vector<const float*> hx_col(n_clusters, nullptr), hx_row(n_clusters, nullptr);
  bool any_col = false, any_row = false;
  for (int g = 0; g < n_clusters; ++g) {
    if (ncol[g] <= m) { hx_col[g] = hx[g]; any_col = true; }
    else { hx_row[g] = hx[g]; any_row = true; }
  }
  CKV(ensure(c.ws[WS_B], (size_t)n_clusters * 16 + 64), "cluster_verify: ptrs");
  const float** dXr = (const float**)c.ws[WS_B].p;
  const float** dXc = dXr + n_clusters;
  CKV(cudaMemcpyAsync(dXr, hx_row.data(), (size_t)n_clusters * 8, cudaMemcpyHostToDevice, c.stream),
      "cluster_verify: h2d");
  CKV(cudaMemcpyAsync(dXc, hx_col.data(), (size_t)n_clusters * 8, cudaMemcpyHostToDevice, c.stream),
      "cluster_verify: h2d");
  const unsigned tiles = (unsigned)((dmax + 63) / 64);
  if (any_col) {
    k_gram<false><<<dim3(tiles, tiles, n_clusters), 256, 0, c.stream>>>(dXc, dN, m, dG, dmax);
    c.launches += 1;
    CKV(cudaGetLastError(), "cluster_verify: column Grams");
  }
  if (any_row) {
    k_gram<true><<<dim3(tiles, tiles, n_clusters), 256, 0, c.stream>>>(dXr, dN, m, dG, dmax);
    c.launches += 1;
    CKV(cudaGetLastError(), "cluster_verify: row Grams");
  }
  double* ev = (double*)c.ws[WS_EV].p;
  int* cnt = (int*)(ev + (size_t)n_clusters * r);
  double* tr = (double*)(cnt + 2 * n_clusters);
  CKV(launch_tridiag_topk(c, G, dmax, gs, dD, n_clusters, dmax, nullptr, r, ev, cnt, tr,
                          (double*)c.ws[WS_PAIR].p),
      "cluster_verify: eigenvalues");
  std::vector<double> hev((size_t)n_clusters * r), htr(n_clusters);
  std::vector<int> hcnt(n_clusters);
  CKV(cudaMemcpyAsync(hev.data(), ev, hev.size() * 8, cudaMemcpyDeviceToHost, c.stream), "cluster_verify: d2h");
  CKV(cudaMemcpyAsync(hcnt.data(), cnt, (size_t)n_clusters * 4, cudaMemcpyDeviceToHost, c.stream),
      "cluster_verify: d2h");
  CKV(cudaMemcpyAsync(htr.data(), tr, (size_t)n_clusters * 8, cudaMemcpyDeviceToHost, c.stream),
      "cluster_verify: d2h");
  CKV(cudaStreamSynchronize(c.stream), "cluster_verify: sync");
  for (int g = 0; g < n_clusters; ++g) {
    double top = 0.0, E = 0.0;
    for (int l = 0; l < std::min(r, hcnt[g]); ++l) top += std::max(hev[(size_t)g * r + l], 0.0);
    for (int i : members[g]) E += c.E[i];
    total[g] = E;
    exact_err2[g] = std::min(std::max(htr[g] - top, 0.0), E);
    const int64_t rc = std::min<int64_t>(r, std::min<int64_t>(m, ncol[g]));
    mem[g] = std::min<int64_t>(m * ncol[g], rc * (m + ncol[g]));  // reading A23: store the smaller form
  }
  return CMSVD_OK;
}

// Factors of each cluster's rank-r truncated SVD M_c ~ U_c S_c V_c^T: Ũ_c = U_c S_c
// (m x r_c) and V_c (N_c x r_c), from the Gram eigenvectors.  Column Gram (N_c <= m): V = eigenvectors,
// Ũ = M V.  Row Gram (m < N_c): U = eigenvectors, Ũ = U S, V = M^T U S^-1.  fp64 accumulation.
// One thread per output element; the eigenvector of the l-th largest eigenvalue is column perm[l] of Ev.
__global__ void k_cluster_factors(int64_t m, int ncol, int dim, int rc, bool rows, const float* __restrict__ X,
                                  const double* __restrict__ Ev, const int* __restrict__ perm,
                                  const double* __restrict__ lam, float* __restrict__ Ut, float* __restrict__ V) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nU = m * rc, nV = (int64_t)ncol * rc;
  if (e >= nU + nV) return;
  const double s1 = sqrt(fmax(lam[0], 0.0));
  if (e < nU) {                                  // Ũ[i, l]
    const int l = (int)(e / m);
    const int64_t i = e % m;
    const double sl = sqrt(fmax(lam[l], 0.0));
    const double* ev = Ev + (int64_t)perm[l] * dim;
    double acc = 0.0;
    if (rows) acc = ev[i] * sl;                  // U S
    else
      for (int k = 0; k < ncol; ++k) acc = fma((double)X[(int64_t)k * m + i], ev[k], acc);   // M V
    Ut[(int64_t)l * m + i] = (sl > 1e-5 * s1) ? (float)acc : 0.f;
  } else {                                       // V[k, l]
    const int64_t f = e - nU;
    const int l = (int)(f / ncol);
    const int k = (int)(f % ncol);
    const double sl = sqrt(fmax(lam[l], 0.0));
    const double* ev = Ev + (int64_t)perm[l] * dim;
    double acc = 0.0;
    if (rows) {
      for (int64_t i = 0; i < m; ++i) acc = fma((double)X[(int64_t)k * m + i], ev[i], acc);   // (M^T U)[k, l]
      acc = (sl > 1e-5 * s1) ? acc / sl : 0.0;
    } else {
      acc = (sl > 1e-5 * s1) ? ev[k] : 0.0;
    }
    V[(int64_t)l * ncol + k] = (float)acc;
  }
}

Status do_cluster_factors(Ctx& c, int32_t r, const int32_t* assign, int32_t n_clusters, float* Ut, float* Vout,
                          int32_t* rc_out) {
  if (c.count <= 0) return fail(c, CMSVD_E_STATE, "cluster_factors: no collection registered");
  if (r < 1 || n_clusters < 0 || !assign) return fail(c, CMSVD_E_ARG, "cluster_factors: need r >= 1, assign");
  if (n_clusters == 0) return CMSVD_OK;
  if (!Ut || !Vout || !rc_out) return fail(c, CMSVD_E_ARG, "cluster_factors: outputs are required");
  const int N = c.count;
  const int64_t m = c.m;
  std::vector<std::vector<int>> members(n_clusters);
  for (int i = 0; i < N; ++i) {
    if (assign[i] < 0 || assign[i] >= n_clusters)
      return fail(c, CMSVD_E_ARG, "cluster_factors: assign[" + std::to_string(i) + "] out of range");
    members[assign[i]].push_back(i);
  }
  size_t uo = 0, vo = 0;
  for (int g = 0; g < n_clusters; ++g) {
    if (members[g].empty()) return fail(c, CMSVD_E_ARG, "cluster_factors: empty cluster " + std::to_string(g));
    int64_t nc = 0;
    for (int i : members[g]) nc += c.n[i];
    const int64_t dim = std::min<int64_t>(m, nc);
    if (dim > kEigMax)
      return fail(c, CMSVD_E_SHAPE, "cluster_factors: min(m, N_c) > " + std::to_string(kEigMax));
    const int rc = (int)std::min<int64_t>(r, dim);
    // one cluster at a time: gather, Gram, eigenvectors, factors
    CKV(ensure(c.ws[WS_A], (size_t)m * nc * 4), "cluster_factors: concatenation");
    CKV(ensure(c.ws[WS_G], (size_t)dim * dim * 8), "cluster_factors: Gram");
    CKV(ensure(c.ws[WS_V], (size_t)dim * dim * 8 * 2), "cluster_factors: vectors");
    CKV(ensure(c.ws[WS_EV], (size_t)dim * 8 + 64), "cluster_factors: eigenvalues");
    CKV(ensure(c.ws[WS_PERM], (size_t)dim * 4 + 64), "cluster_factors: perm");
    CKV(ensure(c.ws[WS_STAT], 64), "cluster_factors: status");
    CKV(ensure(c.ws[WS_META], 64), "cluster_factors: meta");
    CKV(ensure(c.ws[WS_OUT], (size_t)(m + nc) * rc * 4 + 64), "cluster_factors: out");
    float* X = (float*)c.ws[WS_A].p;
    int64_t col = 0;
    for (int i : members[g]) {
      CKV(cudaMemcpyAsync(X + col * m, (const float*)c.arena.p + c.boff[i], (size_t)m * c.n[i] * 4,
                          cudaMemcpyDeviceToDevice, c.stream),
          "cluster_factors: gather");
      col += c.n[i];
    }
    const bool rows = nc > m;
    const float* hx[1] = {X};
    double* hg[1] = {(double*)c.ws[WS_G].p};
    const int hn[1] = {(int)nc};
    const int hd[1] = {(int)dim};
    char* mb = (char*)c.ws[WS_META].p;
    CKV(cudaMemcpyAsync(mb, hx, 8, cudaMemcpyHostToDevice, c.stream), "cluster_factors: h2d");
    CKV(cudaMemcpyAsync(mb + 8, hg, 8, cudaMemcpyHostToDevice, c.stream), "cluster_factors: h2d");
    CKV(cudaMemcpyAsync(mb + 16, hn, 4, cudaMemcpyHostToDevice, c.stream), "cluster_factors: h2d");
    CKV(cudaMemcpyAsync(mb + 20, hd, 4, cudaMemcpyHostToDevice, c.stream), "cluster_factors: h2d");
    const unsigned tiles = (unsigned)((dim + 63) / 64);
    if (rows) k_gram<true><<<dim3(tiles, tiles, 1), 256, 0, c.stream>>>((const float* const*)mb, (const int*)(mb + 16), m,
                                                                   (double* const*)(mb + 8), dim);
    else k_gram<false><<<dim3(tiles, tiles, 1), 256, 0, c.stream>>>((const float* const*)mb, (const int*)(mb + 16), m,
                                                                (double* const*)(mb + 8), dim);
    c.launches += 1;
    CKV(cudaGetLastError(), "cluster_factors: Gram");
    double* Ev = (double*)c.ws[WS_V].p;
    CKV(launch_syev(c, (const double*)c.ws[WS_G].p, dim, dim * dim, (const int*)(mb + 20), 1, (int)dim, Ev, dim * dim,
                    Ev + dim * dim, (double*)c.ws[WS_EV].p, (int*)c.ws[WS_PERM].p, dim, (int*)c.ws[WS_STAT].p),
        "cluster_factors: eigenvectors");
    float* dU = (float*)c.ws[WS_OUT].p;
    float* dVo = dU + (size_t)m * rc;
    const int64_t tot = (m + nc) * rc;
    k_cluster_factors<<<(unsigned)((tot + 255) / 256), 256, 0, c.stream>>>(
        m, (int)nc, (int)dim, rc, rows, X, Ev, (const int*)c.ws[WS_PERM].p, (const double*)c.ws[WS_EV].p, dU, dVo);
    c.launches += 1;
    CKV(cudaGetLastError(), "cluster_factors: factors");
    int st = 0;
    CKV(cudaMemcpyAsync(&st, c.ws[WS_STAT].p, 4, cudaMemcpyDeviceToHost, c.stream), "cluster_factors: d2h");
    CKV(cudaMemcpyAsync(Ut + uo, dU, (size_t)m * rc * 4, cudaMemcpyDeviceToHost, c.stream), "cluster_factors: d2h");
    CKV(cudaMemcpyAsync(Vout + vo, dVo, (size_t)nc * rc * 4, cudaMemcpyDeviceToHost, c.stream), "cluster_factors: d2h");
    CKV(cudaStreamSynchronize(c.stream), "cluster_factors: sync");
    if (st < 0) return fail(c, CMSVD_E_NOCONV, "cluster_factors: eigensolver did not converge for cluster " +
                                                   std::to_string(g));
    rc_out[g] = rc;
    uo += (size_t)m * rc;
    vo += (size_t)nc * rc;
  }
  return CMSVD_OK;
}

}  // namespace cmsvd

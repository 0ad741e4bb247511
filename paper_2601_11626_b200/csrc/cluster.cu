// cluster.cu -- S10: the three greedy clustering drivers of Appendix E
// (Algorithms 1-3) run on the host; the GPU is called only
// for (a) residual-mode sort keys ||(I - B B^T) F_j||_F^2 of all remaining
// candidates against the current state basis B, (b) tentative merge
// evaluations through the pair pipeline (pair_eval_dev) with the cluster
// state as the base, and (c) state commits:
//   Alg. 3 (incremental): U <- top-r left singular vectors of [U diag(s), F]
//          = [U diag(s), F] v_l / sigma~_l from the eigenvectors of the core
//          Gram (Cor. 3; truncate after every append);
//   Alg. 2 (residual):    Q <- [Q, orth(R)], mu <- top_r(mu u sigma(R))
//          (Thm 2 construction; proof Step 5).
// Readings (A9-A11): anchor = largest remaining ||A||_F (ties ->
// smaller id); frobenius order ascending ||A||_F; residual order ascending key
// re-ranked after each accept; inclusive certificate err^2 <= eps^2 E; a
// window of `knn` candidates per step, first passing one accepted, none
// passing closes the cluster; zero-energy blocks merge unconditionally.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "engine.h"
#include "kernels.cuh"

namespace cmsvd {

#define CK(expr, where)                                    \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return cuda_fail(c, _e, where); \
  } while (0)

// ||R||_F^2 per problem (R: m x w at R + p*strideR), fp64, deterministic.
__global__ void __launch_bounds__(kThreads) k_rnorm(const float* __restrict__ R, int64_t strideR, int64_t m,
                                                    const int* __restrict__ ws, double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  const int p = blockIdx.x;
  const int64_t len = m * ws[p];
  const float* r = R + p * strideR;
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) acc = fma((double)r[e], (double)r[e], acc);
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) out[p] = s;
}

// Alg. 3 commit: Unew[:, l] = (U diag(s) v[0:rr] + F v[rr:]) / sqrt(lambda_l), v = V[:, perm[l]].
__global__ void k_commit_inc(int64_t m, const float* __restrict__ U, const double* __restrict__ s, int rr,
                             const float* __restrict__ F, int w, const double* __restrict__ V,
                             const int* __restrict__ perm, const double* __restrict__ lam, float* __restrict__ Unew) {
  const int l = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int n = rr + w;
  const double* v = V + (int64_t)perm[l] * n;
  double acc = 0.0;
  for (int a = 0; a < rr; ++a) acc = fma((double)U[(int64_t)a * m + i] * s[a], v[a], acc);
  for (int b = 0; b < w; ++b) acc = fma((double)F[(int64_t)b * m + i], v[rr + b], acc);
  Unew[(int64_t)l * m + i] = (float)(acc / sqrt(lam[l]));
}

// Alg. 2 commit: Q[:, q0 + l] = R v_{perm[l]} / sqrt(lambda_l).
__global__ void k_commit_res(int64_t m, const float* __restrict__ R, int w, const double* __restrict__ V,
                             const int* __restrict__ perm, const double* __restrict__ lam, float* __restrict__ Qnew) {
  const int l = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double* v = V + (int64_t)perm[l] * w;
  double acc = 0.0;
  for (int b = 0; b < w; ++b) acc = fma((double)R[(int64_t)b * m + i], v[b], acc);
  Qnew[(int64_t)l * m + i] = (float)(acc / sqrt(lam[l]));
}

namespace {

enum { CW_BASIS0 = 0, CW_BASIS1, CW_SPEC, CW_KEYS, CW_PAIRS, CW_OUT, CW_Z, CW_R, CW_G, CW_V, CW_EV, CW_PERM,
       CW_STAT, CW_DESC, CW_NS, CW_SAVE };

size_t au(size_t x) { return (x + 255) / 256 * 256; }

struct Driver {
  Ctx& c;
  const cmsvd_cluster_opts& o;
  int N;
  int64_t m;
  const AppDesc* d_ad;
  std::vector<AppDesc> h_ad;  // host copy of the operand descriptors
  int wmax = 1;
  // state
  BaseDesc st{};
  int cur = 0;                // which basis buffer is live
  std::vector<double> spec;   // host copy of the state spectrum
  int cap = 0;                // basis capacity (columns)
  EigKeep keep;               // reflectors of the last evaluation's Grams (Alg. 3 commits reuse them)
  std::vector<int> last_win;

  Driver(Ctx& cc, const cmsvd_cluster_opts& oo) : c(cc), o(oo), N(cc.count), m(cc.m) {}

  float* basis(int which) { return (float*)c.cws[CW_BASIS0 + which].p; }

  Status setup() {
    d_ad = (const AppDesc*)(o.operand == CMSVD_OPERAND_TRUNC ? c.d_adesc_trunc.p : c.d_adesc_raw.p);
    h_ad.resize(N);
    CK(cudaMemcpyAsync(h_ad.data(), d_ad, (size_t)N * sizeof(AppDesc), cudaMemcpyDeviceToHost, c.stream), "cluster");
    CK(cudaStreamSynchronize(c.stream), "cluster");
    for (auto& a : h_ad) wmax = std::max(wmax, a.w);
    cap = (int)std::min<int64_t>(m, (int64_t)o.r + wmax);
    if (o.algorithm == CMSVD_ALG_RESIDUAL) cap = (int)m;
    cap = std::max(cap, std::max(c.nmax, 1));
    CK(ensure(c.cws[CW_BASIS0], (size_t)m * cap * 4), "cluster: basis");
    CK(ensure(c.cws[CW_BASIS1], (size_t)m * cap * 4), "cluster: basis");
    CK(ensure(c.cws[CW_SPEC], (size_t)std::max(cap, o.r) * 8 + 64), "cluster: spec");
    CK(ensure(c.cws[CW_KEYS], (size_t)N * 8), "cluster: keys");
    CK(ensure(c.cws[CW_PAIRS], (size_t)N * 8), "cluster: pairs");
    CK(ensure(c.cws[CW_OUT], au((size_t)N * 24) + au((size_t)N * 8)), "cluster: out");
    return CMSVD_OK;
  }

  Status upload_state() {
    st.spec = (const double*)c.cws[CW_SPEC].p;
    st.basis = basis(cur);
    if (!spec.empty())
      CK(cudaMemcpyAsync(c.cws[CW_SPEC].p, spec.data(), spec.size() * 8, cudaMemcpyHostToDevice, c.stream), "cluster");
    CK(cudaMemcpyAsync((BaseDesc*)c.d_bdesc.p + N, &st, sizeof(BaseDesc), cudaMemcpyHostToDevice, c.stream),
       "cluster");
    return CMSVD_OK;
  }

  // initial state from the anchor block
  Status init_state(int anchor) {
    const int rank = c.rank[anchor], k = c.kcols[anchor];
    const double* sg = &c.sig[(size_t)anchor * c.nmax];
    const float* Ub = (const float*)c.d_U.p + c.uoff[anchor];
    cur = 0;
    st = BaseDesc{};
    st.E = c.E[anchor];
    if (o.algorithm == CMSVD_ALG_APPROX) {
      const int rr = std::min(o.r, rank);
      CK(cudaMemcpyAsync(basis(cur), Ub, (size_t)m * rr * 4, cudaMemcpyDeviceToDevice, c.stream), "cluster: init");
      spec.assign(sg, sg + rr);
      st.q = rr; st.rr = rr; st.ns = rr;
      double tail = 0.0;
      for (int l = k - 1; l >= rr; --l) tail += sg[l] * sg[l];
      st.tail_inc = tail + std::max(0.0, c.E[anchor] - std::accumulate(sg, sg + k, 0.0,
                                                                       [](double a, double b) { return a + b * b; }));
    } else {
      CK(cudaMemcpyAsync(basis(cur), Ub, (size_t)m * rank * 4, cudaMemcpyDeviceToDevice, c.stream), "cluster: init");
      const int kk = std::min(o.r, k);
      spec.assign(sg, sg + kk);
      st.q = rank; st.rr = 0; st.ns = kk;
      double rest = 0.0;
      for (int l = k - 1; l >= kk; --l) rest += sg[l] * sg[l];
      st.rest_res = rest;
    }
    return upload_state();
  }

  // residual keys ||(I - B B^T) F_j||^2 for the given candidates
  Status keys(const std::vector<int>& cand, std::vector<double>& out) {
    const int P = (int)cand.size();
    out.assign(P, 0.0);
    if (P == 0) return CMSVD_OK;
    std::vector<int2> pr(P);
    for (int t = 0; t < P; ++t) pr[t] = make_int2(N, cand[t]);
    int2* d_pr = (int2*)c.cws[CW_PAIRS].p;
    CK(cudaMemcpyAsync(d_pr, pr.data(), (size_t)P * 8, cudaMemcpyHostToDevice, c.stream), "cluster: keys");
    const int q = std::max(st.q, 1);
    CK(ensure(c.cws[CW_Z], (size_t)P * q * wmax * 4), "cluster: Z");
    CK(ensure(c.cws[CW_R], (size_t)P * m * wmax * 4), "cluster: R");
    CK(ensure(c.cws[CW_DESC], au((size_t)P * 4 * sizeof(GemmDesc)) + au((size_t)P * 16) + au((size_t)P * 8)),
       "cluster: desc");
    char* db = (char*)c.cws[CW_DESC].p;
    GemmDesc* dZ = (GemmDesc*)db;
    GemmDesc* dR = dZ + P;
    GemmDesc* dW = dR + P;
    GemmDesc* dZZ = dW + P;
    int* nG = (int*)(db + au((size_t)P * 4 * sizeof(GemmDesc)));
    int* nW = nG + P;
    double* thr = (double*)(db + au((size_t)P * 4 * sizeof(GemmDesc)) + au((size_t)P * 16));
    const bool full = o.algorithm == CMSVD_ALG_RESIDUAL;
    k_make_descs<<<(P + 255) / 256, 256, 0, c.stream>>>(d_pr, P, (const BaseDesc*)c.d_bdesc.p, d_ad, m, full ? 1 : 0,
                                                        q, wmax, q + wmax, (float*)c.cws[CW_Z].p,
                                                        (float*)c.cws[CW_R].p, nullptr, nullptr, dZ, dR, dW, dZZ, nG,
                                                        nW, thr, o.r);
    c.launches += 1;
    CK(cudaGetLastError(), "cluster: keys descs");
    CK(launch_gemm_tn(c, dZ, P, q, wmax, false), "cluster: keys Z");
    CK(launch_gemm_nn_sub(c, dR, P, (int)m, wmax), "cluster: keys R");
    double* d_keys = (double*)c.cws[CW_KEYS].p;
    k_rnorm<<<P, kThreads, 0, c.stream>>>((const float*)c.cws[CW_R].p, m * wmax, m, nW, d_keys);
    c.launches += 1;
    CK(cudaGetLastError(), "cluster: keys norm");
    CK(cudaMemcpyAsync(out.data(), d_keys, (size_t)P * 8, cudaMemcpyDeviceToHost, c.stream), "cluster: keys d2h");
    CK(cudaStreamSynchronize(c.stream), "cluster: keys sync");
    return CMSVD_OK;
  }

  // tentative evaluations of the state against a window of candidates
  Status evaluate(const std::vector<int>& win, std::vector<double>& err2, std::vector<double>& tot) {
    const int P = (int)win.size();
    std::vector<int2> pr(P);
    for (int t = 0; t < P; ++t) pr[t] = make_int2(N, win[t]);
    int2* d_pr = (int2*)c.cws[CW_PAIRS].p;
    CK(cudaMemcpyAsync(d_pr, pr.data(), (size_t)P * 8, cudaMemcpyHostToDevice, c.stream), "cluster: eval");
    Dims d;
    d.qmax = st.q;
    d.rrmax = st.rr;
    d.wmax = wmax;
    const unsigned kinds = o.algorithm == CMSVD_ALG_RESIDUAL ? CMSVD_RESIDUAL : CMSVD_INCREMENTAL;
    double* d_e = (double*)c.cws[CW_OUT].p;
    double* d_t = (double*)((char*)c.cws[CW_OUT].p + au((size_t)N * 24));
    // Alg. 3: keep the Grams' tridiagonal reductions, so that the commit of the accepted candidate only
    // computes its top-r eigenvectors (inverse iteration + back-transformation) instead of rebuilding G
    keep = EigKeep{};
    last_win = win;
    if (o.algorithm == CMSVD_ALG_APPROX && c.commit_topk) {
      const int64_t gm = std::max(1, st.rr + wmax);
      keep.save_stride = gm * gm + 2 * gm;
      CK(ensure(c.cws[CW_SAVE], (size_t)P * keep.save_stride * 8), "cluster: save");
      keep.save = (double*)c.cws[CW_SAVE].p;
    }
    Status s = pair_eval_dev(c, d_pr, P, o.r, kinds, (const BaseDesc*)c.d_bdesc.p, d_ad, d, d_e, d_t, nullptr,
                             nullptr, false, &keep);
    if (s != CMSVD_OK) return s;
    std::vector<double> e3(3 * P);
    tot.resize(P);
    CK(cudaMemcpyAsync(e3.data(), d_e, (size_t)P * 24, cudaMemcpyDeviceToHost, c.stream), "cluster: eval d2h");
    CK(cudaMemcpyAsync(tot.data(), d_t, (size_t)P * 8, cudaMemcpyDeviceToHost, c.stream), "cluster: eval d2h");
    CK(cudaStreamSynchronize(c.stream), "cluster: eval sync");
    err2.resize(P);
    for (int t = 0; t < P; ++t) err2[t] = e3[3 * t + (kinds == CMSVD_RESIDUAL ? 1 : 2)];
    return CMSVD_OK;
  }

  // Alg. 3 state update from the top eigenpairs of G (lam on the host, ev on the device, vectors in CW_V)
  Status finish_inc(int j, double e2, const AppDesc& a, int n, const std::vector<double>& lam, const int* perm,
                    const double* ev) {
    (void)j;
    const int rr = st.rr, w = a.w;
    const double s0 = lam.empty() ? 0.0 : std::sqrt(std::max(lam[0], 0.0));
    int kp = 0;
    for (int l = 0; l < std::min(o.r, n); ++l)
      if (s0 > 0.0 && std::sqrt(std::max(lam[l], 0.0)) > kTau * s0) ++kp;
    if (kp > 0) {
      dim3 g((unsigned)((m + 255) / 256), kp);
      k_commit_inc<<<g, 256, 0, c.stream>>>(m, basis(cur), st.spec, rr, a.F, w, (const double*)c.cws[CW_V].p, perm,
                                            ev, basis(1 - cur));
      c.launches += 1;
      CK(cudaGetLastError(), "cluster: commit inc");
    }
    cur = 1 - cur;
    spec.resize(kp);
    for (int l = 0; l < kp; ++l) spec[l] = std::sqrt(std::max(lam[l], 0.0));
    st.q = kp; st.rr = kp; st.ns = kp;
    st.E += a.E;
    st.tail_inc = e2;
    return upload_state();
  }

  // commit candidate j (its accepted certificate value e2)
  Status commit(int j, double e2) {
    const AppDesc& a = h_ad[j];
    const int w = a.w;
    const int rr = st.rr, q = st.q;
    int2 pr = make_int2(N, j);
    int2* d_pr = (int2*)c.cws[CW_PAIRS].p;
    CK(cudaMemcpyAsync(d_pr, &pr, 8, cudaMemcpyHostToDevice, c.stream), "cluster: commit");
    const int qz = std::max(q, 1);
    CK(ensure(c.cws[CW_Z], (size_t)qz * std::max(w, 1) * 4 * 2), "cluster: Z");
    CK(ensure(c.cws[CW_R], (size_t)m * std::max(w, 1) * 4 * 2), "cluster: R");
    const int n = (o.algorithm == CMSVD_ALG_APPROX) ? rr + w : w;
    const int nn = std::max(n, 1);
    // Alg. 3 keeps only the top-r eigenpairs of G: tridiagonal reduction + bisection + inverse iteration
    // (k_eig.cu launch_syev_topk) instead of the full QL with vectors
    const int kw = std::min(o.r, n);
    const bool topk = o.algorithm == CMSVD_ALG_APPROX && c.commit_topk && n <= 160 && kw >= 1 && kw <= 64;
    // the accepted candidate's G was reduced by the last evaluation (same state, same operand)
    const int t_win = (int)(std::find(last_win.begin(), last_win.end(), j) - last_win.begin());
    const bool reuse = topk && keep.kept && t_win < (int)last_win.size();
    if (reuse) {
      CK(ensure(c.cws[CW_V], (size_t)nn * nn * 8 * 2), "cluster: V");
      CK(ensure(c.cws[CW_PERM], (size_t)nn * 4 + 64), "cluster: perm");
      int* perm = (int*)c.cws[CW_PERM].p;
      std::vector<int> id(kw);
      for (int l = 0; l < kw; ++l) id[l] = l;
      CK(cudaMemcpyAsync(perm, id.data(), (size_t)kw * 4, cudaMemcpyHostToDevice, c.stream), "cluster: commit");
      const double* ev_t = keep.evG + (size_t)t_win * o.r;
      CK(launch_topk_vectors(c, n, kw, keep.dd + (size_t)t_win * keep.nstride,
                             keep.save + (size_t)t_win * keep.save_stride, ev_t, keep.gsh + 4 * (size_t)t_win,
                             (double*)c.cws[CW_V].p),
         "cluster: commit vectors");
      std::vector<double> lam(kw);
      CK(cudaMemcpyAsync(lam.data(), ev_t, (size_t)kw * 8, cudaMemcpyDeviceToHost, c.stream), "cluster: commit d2h");
      CK(cudaStreamSynchronize(c.stream), "cluster: commit sync");
      return finish_inc(j, e2, a, n, lam, perm, ev_t);
    }
    CK(ensure(c.cws[CW_G], (size_t)nn * nn * 8 * 3 + (topk ? syev_topk_scratch_bytes(n, kw) : 0)), "cluster: G");
    CK(ensure(c.cws[CW_V], (size_t)nn * nn * 8 * 2), "cluster: V");
    CK(ensure(c.cws[CW_EV], (size_t)nn * 8 + (size_t)nn * 8), "cluster: ev");
    CK(ensure(c.cws[CW_PERM], (size_t)nn * 4 + 64), "cluster: perm");
    CK(ensure(c.cws[CW_NS], 64), "cluster: ns");
    CK(ensure(c.cws[CW_DESC], 8 * sizeof(GemmDesc) + 256), "cluster: desc");
    float* Z = (float*)c.cws[CW_Z].p;
    float* R = (float*)c.cws[CW_R].p;
    float* Z2 = Z + (size_t)qz * std::max(w, 1);
    float* R2 = R + (size_t)m * std::max(w, 1);
    double* G = (double*)c.cws[CW_G].p;
    GemmDesc hd[4];
    std::memset(hd, 0, sizeof(hd));
    // Z = B^T F, R = F - B Z
    hd[0].A = basis(cur); hd[0].lda = m; hd[0].B = a.F; hd[0].ldb = m; hd[0].C = Z; hd[0].ldc = qz;
    hd[0].M = q; hd[0].N = w; hd[0].K = (int)m;
    hd[1].A = basis(cur); hd[1].lda = m; hd[1].B = Z; hd[1].ldb = qz; hd[1].C0 = a.F; hd[1].ldc0 = m;
    hd[1].C = R; hd[1].ldc = m; hd[1].M = (int)m; hd[1].N = w; hd[1].K = q;
    // re-orthogonalisation pass (Alg. 2 basis growth): Z2 = B^T R, R2 = R - B Z2
    hd[2] = hd[0]; hd[2].B = R; hd[2].C = Z2;
    hd[3] = hd[1]; hd[3].B = Z2; hd[3].C0 = R; hd[3].C = R2;
    GemmDesc* d_hd = (GemmDesc*)c.cws[CW_DESC].p;
    CK(cudaMemcpyAsync(d_hd, hd, sizeof(hd), cudaMemcpyHostToDevice, c.stream), "cluster: commit");
    int* d_ns = (int*)c.cws[CW_NS].p;
    CK(cudaMemcpyAsync(d_ns, &n, 4, cudaMemcpyHostToDevice, c.stream), "cluster: commit");
    double* ev = (double*)c.cws[CW_EV].p;
    int* perm = (int*)c.cws[CW_PERM].p;
    int* stat = perm + nn;
    std::vector<double> lam(nn);
    int status = 0;
    const float* Rf = R;
    if (q > 0) {
      CK(launch_gemm_tn(c, d_hd + 0, 1, q, w, false), "cluster: commit Z");
      CK(launch_gemm_nn_sub(c, d_hd + 1, 1, (int)m, w), "cluster: commit R");
    } else {
      CK(cudaMemcpyAsync(R, a.F, (size_t)m * w * 4, cudaMemcpyDeviceToDevice, c.stream), "cluster: commit");
    }
    if (o.algorithm == CMSVD_ALG_RESIDUAL) {
      if (q > 0) {
        CK(launch_gemm_tn(c, d_hd + 2, 1, q, w, false), "cluster: commit Z2");
        CK(launch_gemm_nn_sub(c, d_hd + 3, 1, (int)m, w), "cluster: commit R2");
        Rf = R2;
      }
      GemmDesc gw{};
      gw.A = Rf; gw.lda = m; gw.B = Rf; gw.ldb = m; gw.C = G; gw.ldc = n; gw.M = w; gw.N = w; gw.K = (int)m; gw.sym = 1;
      CK(cudaMemcpyAsync(d_hd, &gw, sizeof(gw), cudaMemcpyHostToDevice, c.stream), "cluster: commit");
      CK(launch_gemm_tn(c, d_hd, 1, w, w, true), "cluster: commit W");
    } else {
      // G = [[D^2, D Z_r], [Z_r^T D, Z^T Z + R^T R]]: reuse the pair kernels on a single pair
      GemmDesc g2[2] = {};
      double* ZZ = G + (size_t)nn * nn;
      double* WW = ZZ + (size_t)nn * nn;
      g2[0].A = Z; g2[0].lda = qz; g2[0].B = Z; g2[0].ldb = qz; g2[0].C = ZZ; g2[0].ldc = std::max(w, 1);
      g2[0].M = w; g2[0].N = w; g2[0].K = q; g2[0].sym = 1;
      g2[1].A = R; g2[1].lda = m; g2[1].B = R; g2[1].ldb = m; g2[1].C = WW; g2[1].ldc = std::max(w, 1);
      g2[1].M = w; g2[1].N = w; g2[1].K = (int)m; g2[1].sym = 1;
      CK(cudaMemcpyAsync(d_hd, g2, sizeof(g2), cudaMemcpyHostToDevice, c.stream), "cluster: commit");
      CK(launch_gemm_tn(c, d_hd, 2, w, w, true), "cluster: commit grams");
      CK(launch_build_G1(c, rr, w, st.spec, Z, qz, ZZ, WW, G), "cluster: commit G");
    }
    if (topk) {
      std::vector<int> id(kw);
      for (int l = 0; l < kw; ++l) id[l] = l;
      CK(cudaMemcpyAsync(perm, id.data(), (size_t)kw * 4, cudaMemcpyHostToDevice, c.stream), "cluster: commit");
      CK(launch_syev_topk(c, G, n, d_ns, kw, (double*)c.cws[CW_V].p, ev, G + (size_t)nn * nn * 3),
         "cluster: commit eig");
      std::fill(lam.begin(), lam.end(), 0.0);
      CK(cudaMemcpyAsync(lam.data(), ev, (size_t)kw * 8, cudaMemcpyDeviceToHost, c.stream), "cluster: commit d2h");
    } else {
      CK(launch_syev(c, G, n, (int64_t)n * n, d_ns, 1, n, (double*)c.cws[CW_V].p, (int64_t)n * n,
                     (double*)c.cws[CW_V].p + (size_t)nn * nn, ev, perm, n, stat),
         "cluster: commit eig");
      CK(cudaMemcpyAsync(lam.data(), ev, (size_t)n * 8, cudaMemcpyDeviceToHost, c.stream), "cluster: commit d2h");
      CK(cudaMemcpyAsync(&status, stat, 4, cudaMemcpyDeviceToHost, c.stream), "cluster: commit d2h");
    }
    CK(cudaStreamSynchronize(c.stream), "cluster: commit sync");
    if (status < 0) return fail(c, CMSVD_E_NOCONV, "cluster: commit eigensolver did not converge");
    const double l0 = lam.empty() ? 0.0 : std::max(lam[0], 0.0);
    const double s0 = std::sqrt(l0);
    if (o.algorithm == CMSVD_ALG_APPROX) {
      return finish_inc(j, e2, a, n, lam, perm, ev);
    } else {
      int keep = 0;
      for (int l = 0; l < n; ++l)
        if (s0 > 0.0 && std::sqrt(std::max(lam[l], 0.0)) > kTau * s0) ++keep;
      keep = std::min(keep, (int)m - q);
      if (keep > 0) {
        dim3 g((unsigned)((m + 255) / 256), keep);
        k_commit_res<<<g, 256, 0, c.stream>>>(m, Rf, w, (const double*)c.cws[CW_V].p, perm, ev,
                                              basis(cur) + (size_t)q * m);
        c.launches += 1;
        CK(cudaGetLastError(), "cluster: commit res");
      }
      // mu pool <- top_r(mu u sigma(R))
      std::vector<double> pool(spec);
      for (int l = 0; l < n; ++l) pool.push_back(std::sqrt(std::max(lam[l], 0.0)));
      std::sort(pool.begin(), pool.end(), std::greater<double>());
      if ((int)pool.size() > o.r) pool.resize(o.r);
      spec = pool;
      st.q = q + keep;
      st.ns = (int)spec.size();
      st.E += a.E;
      st.rest_res = e2;  // E_new - sum mu_new^2 = the accepted certificate value
    }
    return upload_state();
  }
};

}  // namespace

// Predicted errors of given block sequences (clusters in append order), the estimates of the
// slack diagnostic: Weyl = Eq. 5 over the K blocks; residual /
// incremental = the Alg. 2 / Alg. 3 state after appending blocks 2..K to block 1 in order, each append
// one tentative evaluation + commit on the GPU (the drivers' own machinery).  A single block gives its
// own truncation error for every kind.
Status do_sequence_errors(Ctx& c, const int32_t* offs, const int32_t* ids, int32_t nseq, int32_t r, uint32_t kinds,
                          int operand, double* err2, double* total) {
  if (nseq < 0 || !offs || (nseq > 0 && (!ids || !err2 || !total)))
    return fail(c, CMSVD_E_ARG, "sequence_errors: bad arguments");
  if (c.count <= 0 || c.spectra_r <= 0) return fail(c, CMSVD_E_STATE, "sequence_errors: call block_spectra first");
  if (r != c.spectra_r) return fail(c, CMSVD_E_STATE, "sequence_errors: r differs from the block_spectra r");
  if ((kinds & ~7u) != 0 || kinds == 0) return fail(c, CMSVD_E_ARG, "sequence_errors: bad kinds mask");
  if (operand != CMSVD_OPERAND_RAW && operand != CMSVD_OPERAND_TRUNC)
    return fail(c, CMSVD_E_ARG, "sequence_errors: bad operand");
  if (c.big && (kinds & CMSVD_RESIDUAL))
    return fail(c, CMSVD_E_SHAPE, "sequence_errors: the residual state needs an explicit range basis (A22)");
  for (int32_t s = 0; s < nseq; ++s) {
    if (offs[s + 1] <= offs[s]) return fail(c, CMSVD_E_ARG, "sequence_errors: empty sequence " + std::to_string(s));
    for (int32_t t = offs[s]; t < offs[s + 1]; ++t)
      if (ids[t] < 0 || ids[t] >= c.count)
        return fail(c, CMSVD_E_SHAPE, "sequence_errors: block id out of range in sequence " + std::to_string(s));
  }
  const int nmax = c.nmax;
  auto top_r = [&](int b) {
    const double* sg = &c.sig[(size_t)b * nmax];
    double t = 0.0;
    for (int l = 0; l < std::min(r, c.kcols[b]); ++l) t += sg[l] * sg[l];
    return t;
  };
  for (int32_t s = 0; s < nseq; ++s) {
    const int32_t* seq = ids + offs[s];
    const int K = offs[s + 1] - offs[s];
    double tot = 0.0, top = 0.0;
    for (int t = 0; t < K; ++t) { tot += c.E[seq[t]]; top = std::max(top, top_r(seq[t])); }
    total[s] = tot;
    auto clampv = [&](double v) { return std::min(std::max(v, 0.0), tot); };
    err2[3 * s + 0] = (kinds & CMSVD_WEYL) ? clampv(tot - top) : std::nan("");
    for (int kk = 1; kk <= 2; ++kk) {
      const unsigned bit = kk == 1 ? CMSVD_RESIDUAL : CMSVD_INCREMENTAL;
      if (!(kinds & bit)) { err2[3 * s + kk] = std::nan(""); continue; }
      if (K == 1) { err2[3 * s + kk] = clampv(c.E[seq[0]] - top_r(seq[0])); continue; }
      cmsvd_cluster_opts o{};
      o.algorithm = kk == 1 ? CMSVD_ALG_RESIDUAL : CMSVD_ALG_APPROX;
      o.sort = CMSVD_SORT_FROBENIUS;
      o.knn = 1;
      o.operand = operand;
      o.r = r;
      o.eps = 0.5;
      Driver d(c, o);
      Status st = d.setup();
      if (st != CMSVD_OK) return st;
      st = d.init_state(seq[0]);
      if (st != CMSVD_OK) return st;
      double e = 0.0;
      for (int t = 1; t < K; ++t) {
        std::vector<double> e2v, totv;
        st = d.evaluate(std::vector<int>{seq[t]}, e2v, totv);
        if (st != CMSVD_OK) return st;
        e = e2v[0];
        st = d.commit(seq[t], e);
        if (st != CMSVD_OK) return st;
      }
      err2[3 * s + kk] = clampv(e);
    }
  }
  return CMSVD_OK;
}

Status do_cluster(Ctx& c, const cmsvd_cluster_opts* o, int32_t* assign, int32_t* order, int32_t* n_clusters,
                  double* cluster_err2, double* cluster_total, int64_t* n_evals) {
  if (!o) return fail(c, CMSVD_E_ARG, "cluster: opts is NULL");
  if (!(o->eps > 0.0 && o->eps < 1.0) || o->r < 1 || o->knn < 1)
    return fail(c, CMSVD_E_ARG, "cluster: need 0 < eps < 1, r >= 1, knn >= 1");
  if (o->algorithm < 0 || o->algorithm > 2 || o->sort < 0 || o->sort > 1 || o->operand < 0 || o->operand > 1)
    return fail(c, CMSVD_E_ARG, "cluster: bad algorithm/sort/operand");
  if (c.count <= 0 || c.spectra_r <= 0) return fail(c, CMSVD_E_STATE, "cluster: call block_spectra first");
  if (o->r != c.spectra_r) return fail(c, CMSVD_E_STATE, "cluster: r differs from the block_spectra r");
  if (c.big && o->algorithm == CMSVD_ALG_RESIDUAL)
    return fail(c, CMSVD_E_SHAPE, "cluster: Alg. 2 needs an explicit range basis; blocks wider than 512 columns "
                                  "keep only U_r (A22)");
  const int N = c.count;
  const double eps2 = o->eps * o->eps;
  std::vector<int> rem(N);
  std::iota(rem.begin(), rem.end(), 0);
  std::stable_sort(rem.begin(), rem.end(), [&](int a, int b) { return c.E[a] > c.E[b] || (c.E[a] == c.E[b] && a < b); });
  std::vector<int32_t> asg(N, -1), ord(N, -1);
  std::vector<double> ce2, ctot;
  int64_t evals = 0;
  auto finish = [&](const std::vector<int>& members, double e2, double tot) {
    const int cid = (int)ce2.size();
    for (size_t t = 0; t < members.size(); ++t) { asg[members[t]] = cid; ord[members[t]] = (int)t; }
    ce2.push_back(std::min(std::max(e2, 0.0), tot));
    ctot.push_back(tot);
  };
  if (o->algorithm == CMSVD_ALG_MAX_NORM) {
    // Algorithm 1: norms and the anchor's top-r energy only.
    while (!rem.empty()) {
      const int anchor = rem.front();
      rem.erase(rem.begin());
      std::vector<int> members{anchor};
      int width = c.n[anchor];
      double e_head;
      if (width > o->r) {
        const double* sg = &c.sig[(size_t)anchor * c.nmax];
        e_head = 0.0;
        for (int l = 0; l < std::min(o->r, c.kcols[anchor]); ++l) e_head += sg[l] * sg[l];
      } else {
        while (!rem.empty() && width + c.n[rem.front()] <= o->r) {
          width += c.n[rem.front()];
          members.push_back(rem.front());
          rem.erase(rem.begin());
        }
        e_head = 0.0;
        for (int b : members) e_head += c.E[b];
      }
      double tot = 0.0;
      for (int b : members) tot += c.E[b];
      while (!rem.empty()) {
        const int b = rem.back();
        const double t2 = tot + c.E[b];
        const double e2 = t2 - e_head;
        ++evals;
        if (!(c.E[b] == 0.0 || e2 <= eps2 * t2)) break;
        rem.pop_back();
        members.push_back(b);
        tot = t2;
      }
      finish(members, tot - e_head, tot);
    }
  } else {
    Driver d(c, *o);
    Status s = d.setup();
    if (s != CMSVD_OK) return s;
    while (!rem.empty()) {
      const int anchor = rem.front();
      rem.erase(rem.begin());
      s = d.init_state(anchor);
      if (s != CMSVD_OK) return s;
      std::vector<int> members{anchor};
      double cert = (o->algorithm == CMSVD_ALG_APPROX) ? d.st.tail_inc : d.st.rest_res;
      while (!rem.empty()) {
        std::vector<int> cand(rem);
        if (o->sort == CMSVD_SORT_FROBENIUS) {
          std::stable_sort(cand.begin(), cand.end(),
                           [&](int a, int b) { return c.E[a] < c.E[b] || (c.E[a] == c.E[b] && a < b); });
        } else {
          std::vector<double> k;
          s = d.keys(cand, k);
          if (s != CMSVD_OK) return s;
          std::vector<int> idx(cand.size());
          std::iota(idx.begin(), idx.end(), 0);
          std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
            return k[a] < k[b] || (k[a] == k[b] && cand[a] < cand[b]);
          });
          std::vector<int> sorted(cand.size());
          for (size_t t = 0; t < idx.size(); ++t) sorted[t] = cand[idx[t]];
          cand.swap(sorted);
        }
        const int W = std::min<int>(o->knn, (int)cand.size());
        std::vector<int> win(cand.begin(), cand.begin() + W);
        std::vector<double> e2, tot;
        s = d.evaluate(win, e2, tot);
        if (s != CMSVD_OK) return s;
        int acc = -1;
        for (int t = 0; t < W; ++t) {
          ++evals;
          if (c.E[win[t]] == 0.0 || e2[t] <= eps2 * tot[t]) { acc = t; break; }
        }
        if (acc < 0) break;
        const int b = win[acc];
        s = d.commit(b, e2[acc]);
        if (s != CMSVD_OK) return s;
        cert = e2[acc];
        rem.erase(std::find(rem.begin(), rem.end(), b));
        members.push_back(b);
      }
      finish(members, cert, d.st.E);
    }
  }
  const int K = (int)ce2.size();
  if (assign) std::memcpy(assign, asg.data(), (size_t)N * 4);
  if (order) std::memcpy(order, ord.data(), (size_t)N * 4);
  if (n_clusters) *n_clusters = K;
  if (cluster_err2) std::memcpy(cluster_err2, ce2.data(), (size_t)K * 8);
  if (cluster_total) std::memcpy(cluster_total, ctot.data(), (size_t)K * 8);
  if (n_evals) *n_evals = evals;
  return CMSVD_OK;
}

}  // namespace cmsvd

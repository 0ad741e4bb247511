// engine.cu -- host orchestration of libcmsvd: collection registration (S1),
// block spectra (S2) and the batched pair-evaluation pipeline (S3-S9).
// Everything runs on the context stream; host syncs only where a result must
// be read back (status flags, host outputs).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "engine.h"
#include "kernels.cuh"

namespace cmsvd {

cudaError_t ensure(DevMem& b, size_t bytes) {
  if (bytes <= b.bytes && b.p) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  size_t want = bytes < 256 ? 256 : bytes;
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) { b.p = nullptr; return e; }
  b.bytes = want;
  return cudaSuccess;
}

void release(DevMem& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static cudaEvent_t prof_event(Ctx& c) {
  if (!c.prof.pool.empty()) {
    cudaEvent_t e = c.prof.pool.back();
    c.prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int prof_begin(Ctx& c, int cat) {
  if (!c.prof.on) return -1;
  Prof::Rec r;
  r.cat = cat;
  r.a = prof_event(c);
  r.b = prof_event(c);
  r.work = 0;
  cudaEventRecord(r.a, c.stream);
  c.prof.recs.push_back(r);
  return (int)c.prof.recs.size() - 1;
}

void prof_end(Ctx& c, int rec, int64_t work) {
  if (rec < 0) return;
  cudaEventRecord(c.prof.recs[rec].b, c.stream);
  c.prof.recs[rec].work = work;
}

void prof_collect(Ctx& c) {
  if (c.prof.recs.empty()) return;
  cudaStreamSynchronize(c.stream);
  for (auto& r : c.prof.recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      c.prof.ms[r.cat] += ms;
      c.prof.launches[r.cat] += 1;
      c.prof.work[r.cat] += r.work;
    }
    c.prof.pool.push_back(r.a);
    c.prof.pool.push_back(r.b);
  }
  c.prof.recs.clear();
}

Status fail(Ctx& c, cmsvd_status s, const std::string& msg) {
  c.err = msg;
  return s;
}

Status cuda_fail(Ctx& c, cudaError_t e, const char* where) {
  c.err = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? CMSVD_E_NOMEM : CMSVD_E_CUDA;
}

#define CK(expr, where)                                  \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(c, _e, where); \
  } while (0)

// Workspace slots

// ---------------------------------------------------------------------------
// S1: register
// ---------------------------------------------------------------------------
Status do_register(Ctx& c, int64_t m, int32_t count, const int32_t* n, const float* const* blocks, const int64_t* ld,
                   int where) {
  if (!n || !blocks) return fail(c, CMSVD_E_ARG, "register: n and blocks must be non-NULL");
  if (where != CMSVD_HOST && where != CMSVD_DEVICE) return fail(c, CMSVD_E_ARG, "register: bad `where`");
  if (m <= 0 || count <= 0) return fail(c, CMSVD_E_SHAPE, "register: m and count must be >= 1");
  for (int32_t i = 0; i < count; ++i) {
    if (n[i] <= 0) return fail(c, CMSVD_E_SHAPE, "register: n[" + std::to_string(i) + "] must be >= 1");
    if (ld && ld[i] < m) return fail(c, CMSVD_E_SHAPE, "register: ld[" + std::to_string(i) + "] < m");
    if (!blocks[i]) return fail(c, CMSVD_E_ARG, "register: blocks[" + std::to_string(i) + "] is NULL");
  }
  c.spectra_r = 0;
  c.planes_ok = false;
  c.trunc_ready = false;
  c.m = m;
  c.count = count;
  c.n.assign(n, n + count);
  c.boff.resize(count + 1);
  int64_t off = 0, maxlen = 0;
  c.nmax = 0;
  for (int32_t i = 0; i < count; ++i) {
    c.boff[i] = off;
    off += align_up((size_t)n[i] * m, kArenaAlign);
    maxlen = std::max<int64_t>(maxlen, (int64_t)n[i] * m);
    c.nmax = std::max(c.nmax, n[i]);
  }
  c.boff[count] = off;
  CK(ensure(c.arena, (size_t)off * 4), "register: arena");
  const cudaMemcpyKind kind = where == CMSVD_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  float* arena = (float*)c.arena.p;
  for (int32_t i = 0; i < count; ++i) {
    int64_t ldi = ld ? ld[i] : m;
    if (ldi == m) {
      CK(cudaMemcpyAsync(arena + c.boff[i], blocks[i], (size_t)n[i] * m * 4, kind, c.stream), "register: copy");
    } else {
      CK(cudaMemcpy2DAsync(arena + c.boff[i], (size_t)m * 4, blocks[i], (size_t)ldi * 4, (size_t)m * 4, n[i], kind,
                           c.stream),
         "register: copy2d");
    }
  }
  // energies
  const int mc = energy_max_chunks(maxlen);
  std::vector<int64_t> meta(2 * count);
  for (int32_t i = 0; i < count; ++i) {
    meta[i] = c.boff[i];
    meta[count + i] = (int64_t)n[i] * m;
  }
  CK(ensure(c.ws[WS_META], meta.size() * 8), "register: meta");
  CK(ensure(c.ws[WS_PARTIAL], (size_t)count * mc * 8), "register: partial");
  CK(ensure(c.ws[WS_BAD], 16), "register: flag");
  CK(ensure(c.d_E, (size_t)count * 8), "register: E");
  int64_t* d_meta = (int64_t*)c.ws[WS_META].p;
  CK(cudaMemcpyAsync(d_meta, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, c.stream), "register: meta h2d");
  CK(cudaMemsetAsync(c.ws[WS_BAD].p, 0, 4, c.stream), "register: memset");
  {
    int pr = prof_begin(c, PC_ENERGY);
    CK(launch_energy(c, d_meta, d_meta + count, maxlen, (double*)c.ws[WS_PARTIAL].p, (int*)c.ws[WS_BAD].p,
                     (double*)c.d_E.p),
       "register: energy kernel");
    int64_t bytes = 0;
    for (int32_t i = 0; i < count; ++i) bytes += (int64_t)n[i] * m * 4;
    prof_end(c, pr, bytes);
  }
  c.E.resize(count);
  int bad = 0;
  CK(cudaMemcpyAsync(c.E.data(), c.d_E.p, (size_t)count * 8, cudaMemcpyDeviceToHost, c.stream), "register: E d2h");
  CK(cudaMemcpyAsync(&bad, c.ws[WS_BAD].p, 4, cudaMemcpyDeviceToHost, c.stream), "register: flag d2h");
  CK(cudaStreamSynchronize(c.stream), "register: sync");
  if (bad) {
    c.count = 0;
    return fail(c, CMSVD_E_NONFINITE, "register: a block contains NaN or Inf");
  }
  return CMSVD_OK;
}

// ---------------------------------------------------------------------------
// S2: block spectra (tall-thin / square blocks with n_i <= min(m, 160))
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// S2 for blocks wider than kEigMax columns (configs 3, 4: square weight-like
// blocks).  Reading A22: the per-block Gram is too large for the
// batched eigensolver, so the top-s singular triplets (s = min(m, 2r, 512))
// come from randomized subspace iteration with fp64 accumulation and CholQR2
// orthonormalisation, followed by a Rayleigh-Ritz step:
//   Y = A Omega; repeat q: Z = orth(A^T orth(Y)), Y = A Z;  Q = orth(Y)
//   Bt = A^T Q;  H = Bt^T Bt = W diag(lambda) W^T;  sigma = sqrt(lambda), U_r = Q W_r
// The block's range is taken as R^m (n_i >= m required), so the paper-literal
// residual R = (I - QQ^T)F vanishes and rank_i = min(m, n_i).
// ---------------------------------------------------------------------------
Status do_block_spectra_big(Ctx& c, int32_t r, double* energy, float* sigma, int32_t* rank_out) {
  const int64_t m = c.m;
  const int N = c.count;
  for (int i = 0; i < N; ++i)
    if (c.n[i] < m)
      return fail(c, CMSVD_E_SHAPE, "block_spectra: blocks wider than " + std::to_string(kEigMax) +
                                        " columns must have n_i >= m (A22)");
  const int s = (int)std::min<int64_t>(std::min<int64_t>(m, 2 * (int64_t)r), kEigMax);
  const int kc = (int)std::min<int64_t>(r, m);
  c.spectra_resid = 0.0;
  c.spectra_iters = 0;
  if (kc > s)  // the subspace holds s columns: more than s = min(m, 2r, 512) top vectors cannot be returned
    return fail(c, CMSVD_E_SHAPE, "block_spectra: r > " + std::to_string(kEigMax) + " on blocks wider than " +
                                      std::to_string(kEigMax) + " columns");
  const int nmax = c.nmax;
  c.big = true;
  c.kcols.assign(N, kc);
  c.uoff.resize(N + 1);
  c.foff.resize(N + 1);
  int64_t uo = 0;
  for (int i = 0; i < N; ++i) {
    c.uoff[i] = uo;
    uo += align_up((size_t)kc * m, kArenaAlign);
  }
  c.uoff[N] = uo;
  for (int i = 0; i <= N; ++i) c.foff[i] = c.uoff[i];
  CK(ensure(c.d_U, (size_t)uo * 4), "spectra: U");
  CK(ensure(c.d_Ftrunc, (size_t)uo * 4), "spectra: Ftrunc");
  CK(ensure(c.d_sig, (size_t)N * nmax * 8), "spectra: sig");
  CK(ensure(c.d_sig32, (size_t)N * r * 4), "spectra: sig32");
  CK(ensure(c.d_rank, (size_t)N * 4), "spectra: rank");
  CK(ensure(c.d_bdesc, (size_t)(N + 1) * sizeof(BaseDesc)), "spectra: bdesc");
  CK(ensure(c.d_adesc_raw, (size_t)(N + 1) * sizeof(AppDesc)), "spectra: adesc");
  CK(ensure(c.d_adesc_trunc, (size_t)(N + 1) * sizeof(AppDesc)), "spectra: adesc");
  CK(ensure(c.d_meta32, (size_t)N * 4), "spectra: meta");
  CK(cudaMemcpyAsync(c.d_meta32.p, c.n.data(), (size_t)N * 4, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
  const int* d_ncols = (const int*)c.d_meta32.p;
  // group blocks by width (Omega is shared inside a group), batch under the workspace budget
  std::vector<int> order(N);
  for (int i = 0; i < N; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return c.n[a] < c.n[b]; });
  const int pr_all = prof_begin(c, PC_SPEC_EIG);
  for (int g0 = 0; g0 < N;) {
    const int n = c.n[order[g0]];
    int g1 = g0;
    while (g1 < N && c.n[order[g1]] == n) ++g1;
    const size_t per = 8 * ((size_t)m * s + (size_t)n * s + (size_t)std::max<int64_t>(m, n) * s + 5 * (size_t)s * s +
                            2 * (size_t)s) + 64;
    const int nbmax = (int)std::max<size_t>(1, std::min<size_t>((size_t)(g1 - g0), c.ws_budget / per));
    CK(ensure(c.ws[WS_C], (size_t)n * s * 8), "spectra: Omega");
    double* Om = (double*)c.ws[WS_C].p;
    CK(launch_randn(c, Om, (int64_t)n * s, 0x243F6A8885A308D3ull ^ (uint64_t)n), "spectra: Omega");
    for (int b0 = g0; b0 < g1; b0 += nbmax) {
      const int nb = std::min(nbmax, g1 - b0);
      CK(ensure(c.ws[WS_A], (size_t)nb * m * s * 8), "spectra: Y");
      CK(ensure(c.ws[WS_PAIR], (size_t)nb * n * s * 8), "spectra: Z");
      CK(ensure(c.ws[WS_OUT], (size_t)nb * std::max<int64_t>(m, n) * s * 8), "spectra: tmp");
      CK(ensure(c.ws[WS_G], (size_t)nb * s * s * 8 * 2), "spectra: H");
      CK(ensure(c.ws[WS_V], (size_t)nb * s * s * 8), "spectra: V");
      CK(ensure(c.ws[WS_B], (size_t)nb * s * s * 8), "spectra: VH");
      CK(ensure(c.ws[WS_EV], (size_t)nb * s * 8), "spectra: ev");
      CK(ensure(c.ws[WS_PERM], (size_t)nb * s * 4), "spectra: perm");
      CK(ensure(c.ws[WS_STAT], (size_t)nb * 4 * 2 + (size_t)nb * 8 + 64), "spectra: stat");
      double* Y = (double*)c.ws[WS_A].p;
      double* Z = (double*)c.ws[WS_PAIR].p;
      double* Tmp = (double*)c.ws[WS_OUT].p;
      double* H = (double*)c.ws[WS_G].p;
      double* T = H + (size_t)nb * s * s;
      int* st = (int*)c.ws[WS_STAT].p;
      // pointer tables: A (arena), U, Ftrunc, ids, ns
      std::vector<const float*> hA(nb), hU(nb), hF(nb);
      std::vector<int> hid(nb), hns(nb, s);
      for (int t = 0; t < nb; ++t) {
        const int i = order[b0 + t];
        hid[t] = i;
        hA[t] = (const float*)c.arena.p + c.boff[i];
        hU[t] = (const float*)c.d_U.p + c.uoff[i];
        hF[t] = (const float*)c.d_Ftrunc.p + c.foff[i];
      }
      CK(ensure(c.ws[WS_META], (size_t)nb * 8 * 3 + (size_t)nb * 8 + 64), "spectra: ptrs");
      char* mb = (char*)c.ws[WS_META].p;
      const float** dA = (const float**)mb;
      const float** dU = dA + nb;
      const float** dF = dU + nb;
      int* dids = (int*)(dF + nb);
      int* dns = dids + nb;
      CK(cudaMemcpyAsync(dA, hA.data(), (size_t)nb * 8, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
      CK(cudaMemcpyAsync(dU, hU.data(), (size_t)nb * 8, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
      CK(cudaMemcpyAsync(dF, hF.data(), (size_t)nb * 8, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
      CK(cudaMemcpyAsync(dids, hid.data(), (size_t)nb * 4, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
      CK(cudaMemcpyAsync(dns, hns.data(), (size_t)nb * 4, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
      const int64_t ms = m * s, ns_ = (int64_t)n * s;
      const bool tcp = c.big_tc && c.use_tc;
      // ... through the TMA-fed warp-specialised kernel on pre-split tf32 planes of A and A^T (k_gemm_ws MODE 3)
      const bool wsp = tcp && c.tc_ws && gemm_ws_available() && (m & 3) == 0 && (n & 3) == 0 && (s & 3) == 0;
      float *Y32 = nullptr, *Z32 = nullptr;
      float *Ap = nullptr, *ATp = nullptr, *Yp = nullptr, *Zp = nullptr, *Omp = nullptr;
      GemmDesc *dAtY = nullptr, *dAZ = nullptr;
      if (wsp) {
        const size_t pa = (size_t)nb * 2 * m * n * 4;
        CK(ensure(c.d_Ap, pa), "spectra: A planes");
        CK(ensure(c.d_ATp, pa), "spectra: A^T planes");
        CK(ensure(c.ws[WS_D], ((size_t)nb * 2 * (m + n) * s + (size_t)2 * n * s) * 4), "spectra: basis planes");
        Ap = (float*)c.d_Ap.p;
        ATp = (float*)c.d_ATp.p;
        Yp = (float*)c.ws[WS_D].p;
        Zp = Yp + (size_t)nb * 2 * m * s;
        Omp = Zp + (size_t)nb * 2 * n * s;
        CK(launch_split_planes_ptr(c, (const float* const*)dA, m, n, nb, Ap, ATp), "spectra: split A");
        CK(launch_split_planes64(c, Om, (int64_t)n * s, 1, Omp), "spectra: split Omega");
        CK(launch_gemm_ws_tn64(c, nb, (int)m, s, n, ATp, Omp, true, Y, m, ms), "spectra: AO (ws)");
        CK(cholqr(c, nb, m, s, Y, Tmp, H, T, st, 1), "spectra: cholqr");
      } else if (tcp) {
        // the products with A on tcgen05 (3xTF32 tiles, fp64 outputs for the fp64 CholQR2); the
        // orthonormal bases enter them rounded to fp32 (a 6e-8 relative perturbation of the basis,
        // which the next power iteration and CholQR absorb; the Rayleigh-Ritz values move by O(u32))
        CK(ensure(c.ws[WS_D], (size_t)nb * (m + n) * s * 4 + (size_t)n * s * 4), "spectra: fp32 bases");
        CK(ensure(c.ws[WS_E], (size_t)3 * nb * sizeof(GemmDesc)), "spectra: descs");
        Y32 = (float*)c.ws[WS_D].p;
        Z32 = Y32 + (size_t)nb * m * s;
        float* Om32 = Z32 + (size_t)nb * n * s;
        GemmDesc* dAO = (GemmDesc*)c.ws[WS_E].p;
        dAtY = dAO + nb;
        dAZ = dAtY + nb;
        std::vector<GemmDesc> hd(3 * (size_t)nb);
        for (int t = 0; t < nb; ++t) {
          GemmDesc g{};
          g.A = hA[t]; g.lda = m; g.C0 = nullptr; g.ldc0 = 0; g.sym = 0;
          g.B = Om32; g.ldb = n; g.C = Y + (size_t)t * ms; g.ldc = m; g.M = (int)m; g.N = s; g.K = n;   // Y = A Om
          hd[t] = g;
          g.B = Y32 + (size_t)t * ms; g.ldb = m; g.C = Z + (size_t)t * ns_; g.ldc = n; g.M = n; g.K = (int)m;  // Z = A^T Y
          hd[nb + t] = g;
          g.B = Z32 + (size_t)t * ns_; g.ldb = n; g.C = Y + (size_t)t * ms; g.ldc = m; g.M = (int)m; g.K = n;  // Y = A Z
          hd[2 * nb + t] = g;
        }
        CK(cudaMemcpyAsync(dAO, hd.data(), hd.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice, c.stream),
           "spectra: h2d");
        CK(launch_to_f32(c, Om, Om32, (int64_t)n * s), "spectra: Omega32");
        CK(launch_gemm_tc_nn64(c, dAO, nb, (int)m, s), "spectra: AO (tc)");
        CK(cholqr(c, nb, m, s, Y, Tmp, H, T, st, 1), "spectra: cholqr");
      } else {
        CK((gemm_mixed<float, false>(c, nb, (int)m, s, n, nullptr, m, 0, Om, n, 0, Y, m, ms, 1.0, dA)), "spectra: AO");
        CK(cholqr(c, nb, m, s, Y, Tmp, H, T, st), "spectra: cholqr");
      }
      // power steps A A^T (orthonormalised once per step; the intermediate Z = A^T Y is used as is on the
      // tcgen05 path: the step's condition number (sigma_1 / sigma_s)^2 stays far inside CholQR's fp64
      // range), CholQR2 for the final basis of each Rayleigh-Ritz step
      auto power = [&](int iters) -> Status {
        for (int it = 0; it < iters; ++it) {
          const int passes = it + 1 == iters ? 2 : 1;
          if (wsp) {
            CK(launch_split_planes64(c, Y, ms, nb, Yp), "spectra: Y planes");
            CK(launch_gemm_ws_tn64(c, nb, n, s, (int)m, Ap, Yp, false, Z, n, ns_), "spectra: AtY (ws)");
            CK(launch_split_planes64(c, Z, ns_, nb, Zp), "spectra: Z planes");
            CK(launch_gemm_ws_tn64(c, nb, (int)m, s, n, ATp, Zp, false, Y, m, ms), "spectra: AZ (ws)");
          } else if (tcp) {
            CK(launch_to_f32(c, Y, Y32, (int64_t)nb * ms), "spectra: Y32");
            CK(launch_gemm_tc(c, dAtY, nb, n, s, false, true), "spectra: AtY (tc)");
            CK(launch_to_f32(c, Z, Z32, (int64_t)nb * ns_), "spectra: Z32");
            CK(launch_gemm_tc_nn64(c, dAZ, nb, (int)m, s), "spectra: AZ (tc)");
          } else {
            CK((gemm_mixed<float, true>(c, nb, n, s, (int)m, nullptr, m, 0, Y, m, ms, Z, n, ns_, 1.0, dA)),
               "spectra: AtY");
            CK(cholqr(c, nb, n, s, Z, Tmp, H, T, st), "spectra: cholqr");
            CK((gemm_mixed<float, false>(c, nb, (int)m, s, n, nullptr, m, 0, Z, n, ns_, Y, m, ms, 1.0, dA)),
               "spectra: AZ");
          }
          CK(cholqr(c, nb, m, s, Y, Tmp, H, T, st, passes), "spectra: cholqr");
        }
        return CMSVD_OK;
      };
      // Rayleigh-Ritz: Bt = A^T Q, H = Bt^T Bt = W diag(lambda) W^T, U_r = Q W_r, descriptors
      auto rayleigh_ritz = [&]() -> Status {
        if (wsp) {
          CK(launch_split_planes64(c, Y, ms, nb, Yp), "spectra: Y planes");
          CK(launch_gemm_ws_tn64(c, nb, n, s, (int)m, Ap, Yp, false, Z, n, ns_), "spectra: Bt (ws)");
        } else if (tcp) {
          CK(launch_to_f32(c, Y, Y32, (int64_t)nb * ms), "spectra: Y32");
          CK(launch_gemm_tc(c, dAtY, nb, n, s, false, true), "spectra: Bt (tc)");
        } else {
          CK((gemm_mixed<float, true>(c, nb, n, s, (int)m, nullptr, m, 0, Y, m, ms, Z, n, ns_, 1.0, dA)), "spectra: Bt");
        }
        CK((gemm_mixed<double, true>(c, nb, s, s, n, Z, n, ns_, Z, n, ns_, H, s, (int64_t)s * s, 1.0, nullptr, 1)),
           "spectra: H");
        CK(launch_syev(c, H, s, (int64_t)s * s, dns, nb, s, (double*)c.ws[WS_V].p, (int64_t)s * s,
                       (double*)c.ws[WS_B].p, (double*)c.ws[WS_EV].p, (int*)c.ws[WS_PERM].p, s, st + nb),
           "spectra: eig(H)");
        dim3 g((unsigned)((m + 255) / 256), (unsigned)((kc + 7) / 8), nb);   // kLvCols = 8 Ritz vectors per CTA
        k_big_leftvec<<<g, 256, 0, c.stream>>>(m, s, kc, Y, (const double*)c.ws[WS_V].p, (const int*)c.ws[WS_PERM].p,
                                               (float* const*)dU);
        c.launches += 1;
        CK(cudaGetLastError(), "spectra: U_r");
        k_big_stats<<<(nb + 127) / 128, 128, 0, c.stream>>>(
            nb, dids, s, r, m, nmax, (const double*)c.ws[WS_EV].p, (const double*)c.d_E.p, d_ncols,
            (double*)c.d_sig.p, (float*)c.d_sig32.p, (int*)c.d_rank.p, (const float* const*)dU,
            (const float* const*)dA, (const float* const*)dF, (BaseDesc*)c.d_bdesc.p, (AppDesc*)c.d_adesc_raw.p,
            (AppDesc*)c.d_adesc_trunc.p);
        c.launches += 1;
        CK(cudaGetLastError(), "spectra: stats");
        return CMSVD_OK;
      };
      // a-posteriori accuracy guard: the Ritz residuals rho_l = ||A A^T u_l - lambda_l u_l|| / lambda_l for
      // l < kc (A A^T u_l = A (Bt w_l), Bt = A^T Q); an eigenvalue of A A^T lies within rho_l lambda_l of
      // lambda_l, so rho_l <= tol bounds the relative error of sigma_l by tol / 2.  Returns the largest
      // rho per block in `resid` (host).
      std::vector<double> resid(nb);
      auto ritz_check = [&]() -> Status {
        CK(ensure(c.ws[WS_SBR], (size_t)nb * ((size_t)s * kc + (size_t)n * kc + (size_t)m * kc) * 8 + 64),
           "spectra: guard");
        double* Wg = (double*)c.ws[WS_SBR].p;
        double* BW = Wg + (size_t)nb * s * kc;
        double* Pm = BW + (size_t)nb * n * kc;
        CK(launch_ritz_gather(c, nb, s, kc, (const double*)c.ws[WS_V].p, (const int*)c.ws[WS_PERM].p, Wg),
           "spectra: guard gather");
        CK((gemm_mixed<double, false>(c, nb, n, kc, s, Z, n, ns_, Wg, s, (int64_t)s * kc, BW, n, (int64_t)n * kc)),
           "spectra: guard A^T U");
        if (wsp && (kc & 3) == 0) {
          // on the TMA-fed tcgen05 kernel like the power steps (3xTF32: ~1e-7 relative, the guard resolves 1e-4)
          CK(launch_split_planes64(c, BW, (int64_t)n * kc, nb, Zp), "spectra: guard planes");
          CK(launch_gemm_ws_tn64(c, nb, (int)m, kc, n, ATp, Zp, false, Pm, m, (int64_t)m * kc),
             "spectra: guard A A^T U (ws)");
        } else {
          CK((gemm_mixed<float, false>(c, nb, (int)m, kc, n, nullptr, m, 0, BW, n, (int64_t)n * kc, Pm, m,
                                       (int64_t)m * kc, 1.0, dA)),
             "spectra: guard A A^T U");
        }
        CK(launch_ritz_resid(c, nb, m, s, kc, Pm, (const double*)c.ws[WS_EV].p, (const float* const*)dU,
                             (double*)(st + 2 * nb)),
           "spectra: guard residual");
        CK(cudaMemcpyAsync(resid.data(), st + 2 * nb, (size_t)nb * 8, cudaMemcpyDeviceToHost, c.stream),
           "spectra: d2h");
        return CMSVD_OK;
      };
      int done = 0, todo = c.subspace_iters;
      const int cap = std::max(c.subspace_iters, c.subspace_max);
      for (;;) {
        Status sp = power(todo);
        if (sp != CMSVD_OK) return sp;
        done += todo;
        sp = rayleigh_ritz();
        if (sp != CMSVD_OK) return sp;
        sp = ritz_check();
        if (sp != CMSVD_OK) return sp;
        std::vector<int> stat(nb);
        CK(cudaMemcpyAsync(stat.data(), st + nb, (size_t)nb * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
        CK(cudaStreamSynchronize(c.stream), "spectra: sync");
        for (int t = 0; t < nb; ++t)
          if (stat[t] < 0)
            return fail(c, CMSVD_E_NOCONV, "block_spectra: QL did not converge on the Rayleigh-Ritz matrix of block " +
                                               std::to_string(hid[t]) + " (" + std::to_string(s) + "x" +
                                               std::to_string(s) + ")");
        int worst = 0;
        for (int t = 1; t < nb; ++t)
          if (!(resid[t] <= resid[worst])) worst = t;
        c.spectra_iters = std::max(c.spectra_iters, done);
        if (resid[worst] <= kRitzTol) {
          c.spectra_resid = std::max(c.spectra_resid, resid[worst]);   // the accepted (final) residuals
          break;
        }
        if (done >= cap) {
          char buf[160];
          snprintf(buf, sizeof(buf), " after %d power iterations: Ritz residual %.3g > %.1g (block %d, %dx%d)", done,
                   resid[worst], kRitzTol, hid[worst], (int)m, n);
          return fail(c, CMSVD_E_NOCONV, std::string("block_spectra: subspace iteration not converged") + buf);
        }
        todo = std::min(cap - done, std::max(4, c.subspace_iters / 2));
      }
    }
    g0 = g1;
  }
  prof_end(c, pr_all);
  {
    dim3 g2((unsigned)((m + kThreads - 1) / kThreads), kc, N);
    k_trunc_operand<<<g2, kThreads, 0, c.stream>>>(m, (const BaseDesc*)c.d_bdesc.p, (const AppDesc*)c.d_adesc_trunc.p,
                                                   (float*)c.d_Ftrunc.p);
    c.launches += 1;
    CK(cudaGetLastError(), "spectra: trunc");
  }
  // tf32 hi/lo planes of U_r and of the TRUNC operands, split once per block (survey K2): the operands of the
  // TMA-fed contraction kernel k_gemm_ws (bases wider than one 128-column tile only)
  c.planes_ok = false;
  if (c.use_tc && c.tc_big && c.tc_ws && kc > 128 && (m & 3) == 0 && (kc & 3) == 0 && N > 0) {
    const size_t pb = (size_t)N * 2 * kc * m * 4;
    CK(ensure(c.d_Qp, pb), "spectra: Q planes");
    CK(ensure(c.d_Fp, pb), "spectra: F planes");
    CK(ensure(c.d_QTp, pb), "spectra: Q^T planes");
    const int64_t ustride = c.uoff[1] - c.uoff[0];
    CK(launch_split_planes(c, (const float*)c.d_U.p, ustride, m, kc, kc, N, (float*)c.d_Qp.p), "spectra: Q planes");
    CK(launch_split_planes(c, (const float*)c.d_Ftrunc.p, ustride, m, kc, kc, N, (float*)c.d_Fp.p),
       "spectra: F planes");
    CK(launch_split_planes_t(c, (const float*)c.d_U.p, ustride, m, kc, N, (float*)c.d_QTp.p), "spectra: Q^T planes");
    c.planes_cols = kc;
    c.planes_F = (const float*)c.d_Ftrunc.p;
    c.planes_fstride = ustride;
    c.planes_ok = true;
  }
  c.sig.resize((size_t)N * nmax);
  c.rank.resize(N);
  CK(cudaMemcpyAsync(c.sig.data(), c.d_sig.p, (size_t)N * nmax * 8, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  CK(cudaMemcpyAsync(c.rank.data(), c.d_rank.p, (size_t)N * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  if (sigma)
    CK(cudaMemcpyAsync(sigma, c.d_sig32.p, (size_t)N * r * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  CK(cudaStreamSynchronize(c.stream), "spectra: sync");
  c.rr.resize(N);
  c.tc_ok = true;
  for (int i = 0; i < N; ++i) c.rr[i] = std::min(kc, c.rank[i]);
  if (energy) std::memcpy(energy, c.E.data(), (size_t)N * 8);
  if (rank_out) std::memcpy(rank_out, c.rank.data(), (size_t)N * 4);
  c.spectra_r = r;
  return CMSVD_OK;
}

Status do_block_spectra(Ctx& c, int32_t r, double* energy, float* sigma, int32_t* rank_out) {
  if (c.count <= 0) return fail(c, CMSVD_E_STATE, "block_spectra: no collection registered");
  if (r < 1) return fail(c, CMSVD_E_ARG, "block_spectra: r must be >= 1");
  const int64_t m = c.m;
  const int N = c.count;
  int nbig = 0;
  for (int i = 0; i < N; ++i) nbig += c.n[i] > kEigMax;
  if (nbig > 0) {
    if (nbig < N)
      return fail(c, CMSVD_E_SHAPE, "block_spectra: collections mixing blocks wider than " +
                                        std::to_string(kEigMax) + " columns with narrower ones are not supported");
    return do_block_spectra_big(c, r, energy, sigma, rank_out);
  }
  c.big = false;
  c.planes_ok = false;
  for (int i = 0; i < N; ++i)
    if (c.n[i] > m) return fail(c, CMSVD_E_SHAPE, "block_spectra: wide blocks (m < n_i <= 512) are not supported");
  const int nmax = c.nmax;
  c.kcols.assign(c.n.begin(), c.n.end());
  c.uoff.resize(N + 1);
  c.foff.resize(N + 1);
  int64_t uo = 0, fo = 0;
  for (int i = 0; i < N; ++i) {
    c.uoff[i] = uo;
    uo += align_up((size_t)c.kcols[i] * m, kArenaAlign);
    c.foff[i] = fo;
    fo += align_up((size_t)std::min(r, c.kcols[i]) * m, kArenaAlign);
  }
  c.uoff[N] = uo;
  c.foff[N] = fo;
  CK(ensure(c.d_U, (size_t)uo * 4), "spectra: U");
  CK(ensure(c.d_Ftrunc, (size_t)fo * 4), "spectra: Ftrunc");
  CK(ensure(c.d_sig, (size_t)N * nmax * 8), "spectra: sig");
  CK(ensure(c.d_sig32, (size_t)N * r * 4), "spectra: sig32");
  CK(ensure(c.d_rank, (size_t)N * 4), "spectra: rank");
  CK(ensure(c.d_bdesc, (size_t)(N + 1) * sizeof(BaseDesc)), "spectra: bdesc");
  CK(ensure(c.d_adesc_raw, (size_t)(N + 1) * sizeof(AppDesc)), "spectra: adesc");
  CK(ensure(c.d_adesc_trunc, (size_t)(N + 1) * sizeof(AppDesc)), "spectra: adesc");
  // metadata: boff, uoff, foff (int64), kcols, n (int32)
  std::vector<int64_t> m64(3 * N);
  std::vector<int32_t> m32(2 * N);
  for (int i = 0; i < N; ++i) {
    m64[i] = c.boff[i];
    m64[N + i] = c.uoff[i];
    m64[2 * N + i] = c.foff[i];
    m32[i] = c.kcols[i];
    m32[N + i] = c.n[i];
  }
  CK(ensure(c.d_meta64, m64.size() * 8), "spectra: meta");
  CK(ensure(c.d_meta32, m32.size() * 4), "spectra: meta");
  CK(cudaMemcpyAsync(c.d_meta64.p, m64.data(), m64.size() * 8, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
  CK(cudaMemcpyAsync(c.d_meta32.p, m32.data(), m32.size() * 4, cudaMemcpyHostToDevice, c.stream), "spectra: h2d");
  const int64_t* d_boff = (const int64_t*)c.d_meta64.p;
  const int64_t* d_uoff = d_boff + N;
  const int64_t* d_foff = d_boff + 2 * N;
  const int* d_kcols = (const int*)c.d_meta32.p;
  const int* d_ncols = d_kcols + N;
  // Gram A_i^T A_i in fp64 (exact products of fp32 data)
  const int64_t gstride = (int64_t)nmax * nmax;
  CK(ensure(c.ws[WS_G], (size_t)N * gstride * 8), "spectra: G");
  CK(ensure(c.ws[WS_V], (size_t)N * gstride * 8), "spectra: V");
  CK(ensure(c.ws[WS_EV], (size_t)N * nmax * 8), "spectra: ev");
  CK(ensure(c.ws[WS_PERM], (size_t)N * nmax * 4), "spectra: perm");
  CK(ensure(c.ws[WS_STAT], (size_t)N * 4), "spectra: stat");
  std::vector<GemmDesc> gd(N);
  const float* arena = (const float*)c.arena.p;
  double* G = (double*)c.ws[WS_G].p;
  for (int i = 0; i < N; ++i) {
    GemmDesc g{};
    g.A = arena + c.boff[i]; g.lda = m; g.B = arena + c.boff[i]; g.ldb = m;
    g.C = G + (int64_t)i * gstride; g.ldc = nmax; g.M = c.kcols[i]; g.N = c.kcols[i]; g.K = (int)m; g.sym = 1;
    gd[i] = g;
  }
  CK(ensure(c.ws[WS_A], gd.size() * sizeof(GemmDesc)), "spectra: gd");
  CK(cudaMemcpyAsync(c.ws[WS_A].p, gd.data(), gd.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice, c.stream),
     "spectra: gd h2d");
  {
    int pr = prof_begin(c, PC_SPEC_GRAM);
    CK(launch_gemm_tn(c, (const GemmDesc*)c.ws[WS_A].p, N, nmax, nmax, true), "spectra: gram");
    prof_end(c, pr);
  }
  // eigen-decomposition A_i^T A_i = V diag(lambda) V^T (values + vectors)
  {
    int pr = prof_begin(c, PC_SPEC_EIG);
    CK(ensure(c.ws[WS_B], (size_t)N * gstride * 8), "spectra: VH");
    CK(launch_syev(c, G, nmax, gstride, d_kcols, N, nmax, (double*)c.ws[WS_V].p, gstride, (double*)c.ws[WS_B].p,
                   (double*)c.ws[WS_EV].p, (int*)c.ws[WS_PERM].p, nmax, (int*)c.ws[WS_STAT].p),
       "spectra: eig");
    prof_end(c, pr);
  }
  std::vector<int> stat(N);
  CK(cudaMemcpyAsync(stat.data(), c.ws[WS_STAT].p, (size_t)N * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  CK(cudaStreamSynchronize(c.stream), "spectra: sync");
  for (int i = 0; i < N; ++i)
    if (stat[i] < 0) return fail(c, CMSVD_E_NOCONV, "block_spectra: QL did not converge for block " +
                                                        std::to_string(i) + " (" + std::to_string(c.kcols[i]) + "x" +
                                                        std::to_string(c.kcols[i]) + " Gram)");
  const int pr_misc = prof_begin(c, PC_SPEC_MISC);
  k_spec_stats<<<(N + 127) / 128, 128, 0, c.stream>>>(
      N, nmax, r, (const double*)c.ws[WS_EV].p, d_kcols, (const double*)c.d_E.p, (double*)c.d_sig.p,
      (float*)c.d_sig32.p, (int*)c.d_rank.p, d_uoff, (const float*)c.d_U.p, d_boff, d_ncols, arena, d_foff,
      (const float*)c.d_Ftrunc.p, (BaseDesc*)c.d_bdesc.p, (AppDesc*)c.d_adesc_raw.p, (AppDesc*)c.d_adesc_trunc.p,
      kTau);
  c.launches += 1;
  CK(cudaGetLastError(), "spectra: stats");
  {
    dim3 g((unsigned)((m + kThreads - 1) / kThreads), (unsigned)((nmax + 7) / 8), N);
    const size_t lv_smem = (size_t)8 * nmax * sizeof(double);
    CK(cudaFuncSetAttribute(k_leftvec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lv_smem), "spectra: leftvec");
    k_leftvec<<<g, kThreads, lv_smem, c.stream>>>(m, arena, d_boff, d_kcols, (const double*)c.ws[WS_V].p, gstride,
                                            (const int*)c.ws[WS_PERM].p, nmax, (const double*)c.d_sig.p,
                                            (const int*)c.d_rank.p, (float*)c.d_U.p, d_uoff);
    c.launches += 1;
    CK(cudaGetLastError(), "spectra: leftvec");
    dim3 g2((unsigned)((m + kThreads - 1) / kThreads), std::min(r, nmax), N);
    k_trunc_operand<<<g2, kThreads, 0, c.stream>>>(m, (const BaseDesc*)c.d_bdesc.p, (const AppDesc*)c.d_adesc_trunc.p,
                                                   (float*)c.d_Ftrunc.p);
    c.launches += 1;
    CK(cudaGetLastError(), "spectra: trunc");
  }
  prof_end(c, pr_misc);
  // host copies
  c.sig.resize((size_t)N * nmax);
  c.rank.resize(N);
  CK(cudaMemcpyAsync(c.sig.data(), c.d_sig.p, (size_t)N * nmax * 8, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  CK(cudaMemcpyAsync(c.rank.data(), c.d_rank.p, (size_t)N * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  if (sigma)
    CK(cudaMemcpyAsync(sigma, c.d_sig32.p, (size_t)N * r * 4, cudaMemcpyDeviceToHost, c.stream), "spectra: d2h");
  CK(cudaStreamSynchronize(c.stream), "spectra: sync");
  c.rr.resize(N);
  c.tc_ok = true;
  for (int i = 0; i < N; ++i) {
    c.rr[i] = std::min(r, c.rank[i]);
    if (c.rank[i] < c.kcols[i]) c.tc_ok = false;
  }
  if (energy) std::memcpy(energy, c.E.data(), (size_t)N * 8);
  if (rank_out) std::memcpy(rank_out, c.rank.data(), (size_t)N * 4);
  c.spectra_r = r;
  return CMSVD_OK;
}

// ---------------------------------------------------------------------------
// S3-S9: batched pair evaluation on device-resident pairs and outputs.
// ---------------------------------------------------------------------------
Status pair_eval_dev(Ctx& c, const int2* d_pairs, int64_t P, int r, unsigned kinds, const BaseDesc* d_bd,
                     const AppDesc* d_ad, const Dims& dims, double* d_err2, double* d_total, float* d_st,
                     float* d_mu, bool tight, EigKeep* keep) {
  if (keep) keep->kept = false;
  if (P <= 0) return CMSVD_OK;
  const int64_t m = c.m;
  // tight (N3): residual with the U_r basis + per-index Weyl; d_err2 is then P x 2
  if (tight) kinds = CMSVD_RESIDUAL;
  // A22 bases (c.big): the paper-literal residual needs no projection (R = (I - QQ^T)F = 0), so Weyl- and
  // residual-only evaluations run on the spectra alone
  const bool need_mat = (kinds & CMSVD_INCREMENTAL) != 0 || tight || ((kinds & CMSVD_RESIDUAL) != 0 && !c.big);
  const bool full = (kinds & CMSVD_RESIDUAL) != 0 && !tight;
  const int QMAX = std::max(1, full ? dims.qmax : dims.rrmax);
  // tcgen05 path (fp32 accumulation) unless the collection has numerically rank-deficient blocks: an
  // fp32-accumulated Gram resolves exactly-zero singular values only to ~sqrt(u32)*sigma_1, the
  // fp64-accumulated SIMT path to ~1e-8*sigma_1 ("precision dispatch")
  const bool use_tc = c.use_tc && c.tc_ok && (full ? dims.qmax : dims.rrmax) <= 128 && dims.wmax <= 128;
  const bool use_tc_big = !use_tc && c.use_tc && c.tc_ok && c.tc_big;  // same precision class, tiled
  const int WMAX = std::max(1, dims.wmax);
  // ... by the warp-specialised TMA-fed kernel when every operand is a registered block's pre-split planes
  const bool use_ws = use_tc_big && c.tc_ws && dims.planes && gemm_ws_supported(c, m) && (QMAX & 3) == 0 &&
                      QMAX <= c.planes_cols && WMAX <= c.planes_cols;
  // ... and Z^T Z folded into the W' contraction (Z planes as leading K stages): the lower-right block of the
  // core Gram from one tensor-core pass; the fp32 accumulation matches the precision class of Z itself.
  // Full-range (A22) bases only: their ||F||^2 split needs only tr(Z^T Z + W')
  const bool zz_fused = use_ws && c.big && c.zz_fused && WMAX <= 256 && !tight;
  const int GMAX = std::max(1, dims.rrmax + dims.wmax);
  if (need_mat && ((!tight && GMAX > kEigMax) || WMAX > kEigMax))
    return fail(c, CMSVD_E_SHAPE, "pair_errors: core size r'+w = " + std::to_string(GMAX) + " exceeds " +
                                      std::to_string(kEigMax) + " (large-core path not built yet)");
  size_t per_pair = 0;
  if (need_mat) {
    per_pair = align_up((size_t)QMAX * WMAX * 4, 256) * (use_ws ? 3 : 1) +
               (use_tc ? 0 : align_up((size_t)m * WMAX * 4, 256) * (use_ws ? 2 : 1)) +
               2 * align_up((size_t)WMAX * WMAX * 8, 256) + align_up((size_t)GMAX * GMAX * 8, 256) +
               4 * sizeof(GemmDesc) + 2 * (size_t)r * 8 + (size_t)(2 * GMAX + 4) * 8 + 64;
  }
  size_t budget = c.ws_budget;
  int64_t chunk = P;
  if (need_mat) chunk = std::max<int64_t>(1, std::min<int64_t>(P, (int64_t)(budget / per_pair)));
  chunk = std::min<int64_t>(chunk, 65535);
  for (int64_t p0 = 0; p0 < P; p0 += chunk) {
    const int64_t Pc = std::min(chunk, P - p0);
    const int2* pr = d_pairs + p0;
    double *evG = nullptr, *evW = nullptr, *trG = nullptr, *trW = nullptr, *zn2 = nullptr;
    int *cntG = nullptr, *cntW = nullptr;
    if (need_mat) {
      // carve the workspace
      size_t off = 0;
      auto carve = [&](size_t bytes) { size_t o = off; off += align_up(bytes, 256); return o; };
      size_t oZ = carve((size_t)Pc * QMAX * WMAX * 4);
      size_t oR = carve(use_tc ? 256 : (size_t)Pc * m * WMAX * 4 * (use_ws ? 2 : 1));   // ws: hi/lo planes of R'
      size_t oZp = carve(use_ws ? (size_t)Pc * QMAX * WMAX * 8 : 256);                   // ws: hi/lo planes of Z
      size_t oW = carve((size_t)Pc * WMAX * WMAX * 8), oZZ = carve((size_t)Pc * WMAX * WMAX * 8);
      size_t oG = carve((size_t)Pc * GMAX * GMAX * 8);
      size_t oD = carve((size_t)Pc * 4 * sizeof(GemmDesc));
      size_t onG = carve((size_t)Pc * 4), onW = carve((size_t)Pc * 4), othr = carve((size_t)Pc * 8);
      size_t oevG = carve((size_t)Pc * r * 8), oevW = carve((size_t)Pc * r * 8);
      size_t ocG = carve((size_t)Pc * 4), ocW = carve((size_t)Pc * 4);
      size_t otG = carve((size_t)Pc * 8), otW = carve((size_t)Pc * 8), ozn = carve((size_t)Pc * 8);
      size_t oscr = carve(tridiag_scratch_bytes((int)Pc, GMAX));
      CK(ensure(c.ws[WS_PAIR], off), "pairs: workspace");
      char* base = (char*)c.ws[WS_PAIR].p;
      float* Z = (float*)(base + oZ);
      float* R = (float*)(base + oR);
      double* W = (double*)(base + oW);
      double* ZZ = (double*)(base + oZZ);
      double* Gm = (double*)(base + oG);
      GemmDesc* dZ = (GemmDesc*)(base + oD);
      GemmDesc* dR = dZ + Pc;
      GemmDesc* dW = dR + Pc;
      GemmDesc* dZZ = dW + Pc;
      int* nG = (int*)(base + onG);
      int* nW = (int*)(base + onW);
      double* thrW = (double*)(base + othr);
      evG = (double*)(base + oevG);
      evW = (double*)(base + oevW);
      cntG = (int*)(base + ocG);
      cntW = (int*)(base + ocW);
      trG = (double*)(base + otG);
      trW = (double*)(base + otW);
      zn2 = (double*)(base + ozn);
      double* scr = (double*)(base + oscr);
      int pf = prof_begin(c, PC_DESCS);
      k_make_descs<<<(unsigned)((Pc + 255) / 256), 256, 0, c.stream>>>(pr, Pc, d_bd, d_ad, m, full ? 1 : 0, QMAX,
                                                                       WMAX, GMAX, Z, R, W, ZZ, dZ, dR, dW, dZZ, nG,
                                                                       nW, thrW, r);
      c.launches += 1;
      CK(cudaGetLastError(), "pairs: descs");
      prof_end(c, pf);
      if (use_ws) {
        float* Zp = (float*)(base + oZp);
        pf = prof_begin(c, PC_PROJ);
        CK(launch_gemm_ws(c, 0, pr, Pc, d_bd, d_ad, full ? 1 : 0, QMAX, WMAX, Z, Zp, R, W), "pairs: Z = Q^T F (ws)");
        prof_end(c, pf);
        pf = prof_begin(c, PC_RESID);
        CK(launch_gemm_ws(c, 1, pr, Pc, d_bd, d_ad, full ? 1 : 0, QMAX, WMAX, Z, Zp, R, W), "pairs: R = F - Q Z (ws)");
        prof_end(c, pf);
        pf = prof_begin(c, PC_GRAM_W);
        CK(launch_gemm_ws(c, 2, pr, Pc, d_bd, d_ad, full ? 1 : 0, QMAX, WMAX, Z, Zp, R, W, zz_fused),
           "pairs: W = R^T R (ws)");
        prof_end(c, pf);
      } else if (use_tc) {
        // fused tcgen05 3xTF32: Z = Q^T F, R' = F - Q Z (on chip), W' = R'^T R'
        // (tight: Q = U_r, the same projection as the incremental estimator)
        pf = prof_begin(c, PC_PAIR_TC);
        CK(launch_pair_tc(c, pr, Pc, d_bd, d_ad, m, full ? 1 : 0, QMAX, WMAX, Z, W), "pairs: tcgen05 Z/R/W");
        prof_end(c, pf);
      } else if (use_tc_big) {
        // operands wider than one 128-column tile: the same 3xTF32 contractions as tcgen05 GEMM tiles,
        // R' materialised (m x w per pair)
        pf = prof_begin(c, PC_PROJ);
        CK(launch_gemm_tc(c, dZ, (int)Pc, QMAX, WMAX, false, false), "pairs: Z = Q^T F (tc)");
        prof_end(c, pf);
        pf = prof_begin(c, PC_RESID);
        CK(launch_gemm_tc(c, dR, (int)Pc, (int)m, WMAX, true, false), "pairs: R = F - Q Z (tc)");
        prof_end(c, pf);
        pf = prof_begin(c, PC_GRAM_W);
        CK(launch_gemm_tc(c, dW, (int)Pc, WMAX, WMAX, false, true), "pairs: W = R^T R (tc)");
        prof_end(c, pf);
      } else {
        pf = prof_begin(c, PC_PROJ);
        CK(launch_gemm_tn(c, dZ, (int)Pc, QMAX, WMAX, false), "pairs: Z = Q^T F");
        prof_end(c, pf);
        pf = prof_begin(c, PC_RESID);
        CK(launch_gemm_nn_sub(c, dR, (int)Pc, (int)m, WMAX), "pairs: R = F - Q Z");
        prof_end(c, pf);
        pf = prof_begin(c, PC_GRAM_W);
        CK(launch_gemm_tn(c, dW, (int)Pc, WMAX, WMAX, true), "pairs: W = R^T R");
        prof_end(c, pf);
      }
      if (tight) {
        pf = prof_begin(c, PC_BUILD_G);
        k_znorm<<<(unsigned)Pc, kThreads, 0, c.stream>>>(pr, d_bd, d_ad, Z, QMAX, WMAX, zn2);
        c.launches += 1;
        CK(cudaGetLastError(), "pairs: ||U_r^T F||");
        prof_end(c, pf);
      } else {
        pf = prof_begin(c, PC_GRAM_ZZ);
        if (zz_fused) {
        } else if (c.zz_syrk && WMAX <= 128)
          CK(launch_syrk_zz(c, pr, Pc, d_bd, d_ad, full ? 1 : 0, QMAX, WMAX, Z, ZZ), "pairs: Z^T Z");
        else
          CK(launch_gemm_tn(c, dZZ, (int)Pc, WMAX, WMAX, true), "pairs: Z^T Z");
        prof_end(c, pf);
        pf = prof_begin(c, PC_BUILD_G);
        k_build_G<<<(unsigned)Pc, kThreads, 0, c.stream>>>(pr, d_bd, d_ad, QMAX, WMAX, GMAX, Z, W,
                                                           zz_fused ? nullptr : ZZ, Gm, zn2,
                                                           (GMAX > 160 && c.eig_sbr) ? c.g_upper : 0);
        c.launches += 1;
        CK(cudaGetLastError(), "pairs: build G");
        prof_end(c, pf);
      }
      if (kinds & CMSVD_INCREMENTAL) {
        const bool save = keep && keep->save && Pc == P && tridiag_can_save(c, GMAX) &&
                          keep->save_stride >= (int64_t)GMAX * GMAX + 2 * GMAX;
        pf = prof_begin(c, PC_EIG_G);
        CK(launch_tridiag_topk(c, Gm, GMAX, (int64_t)GMAX * GMAX, nG, (int)Pc, GMAX, nullptr, r, evG, cntG, trG, scr,
                               save ? keep->save : nullptr, save ? keep->save_stride : 0),
           "pairs: eig(G)");
        prof_end(c, pf);
        if (save) {  // launch_tridiag_topk's scratch: dd (Pc x GMAX), e2 (Pc x GMAX), gsh (4 per pair)
          keep->kept = true;
          keep->dd = scr;
          keep->gsh = scr + 2 * (size_t)Pc * GMAX;
          keep->evG = evG;
          keep->nstride = GMAX;
        }
      }
      if ((kinds & CMSVD_RESIDUAL) && (!c.big || tight)) {  // A22 bases: R = (I - QQ^T)F = 0, sigma(W') unused
        pf = prof_begin(c, PC_EIG_W);
        CK(launch_tridiag_topk(c, W, WMAX, (int64_t)WMAX * WMAX, nW, (int)Pc, WMAX, thrW, r, evW, cntW, trW, scr),
           "pairs: eig(W)");
        prof_end(c, pf);
      }
    }
    int prf = prof_begin(c, PC_FINALIZE);
    if (tight) {
      k_finalize_tight<<<(unsigned)((Pc + 127) / 128), 128, 0, c.stream>>>(pr, Pc, d_bd, d_ad, r, evW, cntW, trW,
                                                                         zn2, d_err2 + 2 * p0, d_total + p0);
      c.launches += 1;
      CK(cudaGetLastError(), "pairs: finalize (tight)");
      prof_end(c, prf);
      continue;
    }
    k_finalize<<<(unsigned)((Pc + 127) / 128), 128, 0, c.stream>>>(
        pr, Pc, d_bd, d_ad, r, kinds, evG, cntG, trG, evW, cntW, trW, zn2, d_err2 + 3 * p0, d_total + p0,
        d_st ? d_st + p0 * r : nullptr, d_mu ? d_mu + p0 * r : nullptr);
    c.launches += 1;
    CK(cudaGetLastError(), "pairs: finalize");
    prof_end(c, prf);
  }
  return CMSVD_OK;
}

Dims block_dims(const Ctx& c, int operand) {
  Dims d;
  for (int i = 0; i < c.count; ++i) {
    d.qmax = std::max(d.qmax, c.big ? c.rr[i] : c.rank[i]);  // A22: full-range bases keep only U_r
    d.rrmax = std::max(d.rrmax, c.rr[i]);
    d.wmax = std::max(d.wmax, operand == CMSVD_OPERAND_TRUNC ? c.rr[i] : c.n[i]);
  }
  return d;
}

Status do_pair_errors(Ctx& c, const int32_t* pairs, int64_t P, int32_t r, uint32_t kinds, int operand, int where,
                      double* err2, double* total, float* sigma_tilde, float* mu) {
  if (P < 0) return fail(c, CMSVD_E_ARG, "pair_errors: P < 0");
  if (P == 0) return CMSVD_OK;
  if (!pairs || !err2 || !total) return fail(c, CMSVD_E_ARG, "pair_errors: pairs, err2 and total are required");
  if (c.count <= 0 || c.spectra_r <= 0) return fail(c, CMSVD_E_STATE, "pair_errors: call block_spectra first");
  if (r != c.spectra_r) return fail(c, CMSVD_E_STATE, "pair_errors: r differs from the block_spectra r");
  if ((kinds & ~7u) != 0 || kinds == 0) return fail(c, CMSVD_E_ARG, "pair_errors: bad kinds mask");
  if (operand != CMSVD_OPERAND_RAW && operand != CMSVD_OPERAND_TRUNC)
    return fail(c, CMSVD_E_ARG, "pair_errors: bad operand");
  if (where != CMSVD_HOST && where != CMSVD_DEVICE) return fail(c, CMSVD_E_ARG, "pair_errors: bad `where`");
  const AppDesc* d_ad = (const AppDesc*)(operand == CMSVD_OPERAND_TRUNC ? c.d_adesc_trunc.p : c.d_adesc_raw.p);
  Dims dims = block_dims(c, operand);
  dims.planes = c.planes_ok && operand == CMSVD_OPERAND_TRUNC;
  if (where == CMSVD_HOST) {
    for (int64_t p = 0; p < 2 * P; ++p)
      if (pairs[p] < 0 || pairs[p] >= c.count)
        return fail(c, CMSVD_E_SHAPE, "pair_errors: pair index out of range at entry " + std::to_string(p));
    size_t off = 0;
    size_t oP = off; off += align_up((size_t)P * 8, 256);
    size_t oE = off; off += align_up((size_t)P * 24, 256);
    size_t oT = off; off += align_up((size_t)P * 8, 256);
    size_t oS = off; off += sigma_tilde ? align_up((size_t)P * r * 4, 256) : 0;
    size_t oM = off; off += mu ? align_up((size_t)P * r * 4, 256) : 0;
    CK(ensure(c.ws[WS_OUT], off), "pair_errors: io buffers");
    char* b = (char*)c.ws[WS_OUT].p;
    CK(cudaMemcpyAsync(b + oP, pairs, (size_t)P * 8, cudaMemcpyHostToDevice, c.stream), "pair_errors: h2d");
    Status s = pair_eval_dev(c, (const int2*)(b + oP), P, r, kinds, (const BaseDesc*)c.d_bdesc.p, d_ad, dims,
                             (double*)(b + oE), (double*)(b + oT), sigma_tilde ? (float*)(b + oS) : nullptr,
                             mu ? (float*)(b + oM) : nullptr);
    if (s != CMSVD_OK) return s;
    CK(cudaMemcpyAsync(err2, b + oE, (size_t)P * 24, cudaMemcpyDeviceToHost, c.stream), "pair_errors: d2h");
    CK(cudaMemcpyAsync(total, b + oT, (size_t)P * 8, cudaMemcpyDeviceToHost, c.stream), "pair_errors: d2h");
    if (sigma_tilde)
      CK(cudaMemcpyAsync(sigma_tilde, b + oS, (size_t)P * r * 4, cudaMemcpyDeviceToHost, c.stream), "pair_errors: d2h");
    if (mu) CK(cudaMemcpyAsync(mu, b + oM, (size_t)P * r * 4, cudaMemcpyDeviceToHost, c.stream), "pair_errors: d2h");
    CK(cudaStreamSynchronize(c.stream), "pair_errors: sync");
    return CMSVD_OK;
  }
  // device-resident pairs / outputs: validate indices on device
  CK(ensure(c.ws[WS_BAD], 16), "pair_errors: flag");
  CK(cudaMemsetAsync(c.ws[WS_BAD].p, 0, 4, c.stream), "pair_errors: memset");
  CK(launch_check_pairs(c, (const int2*)pairs, P, c.count, (int*)c.ws[WS_BAD].p), "pair_errors: check");
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c.ws[WS_BAD].p, 4, cudaMemcpyDeviceToHost, c.stream), "pair_errors: flag d2h");
  CK(cudaStreamSynchronize(c.stream), "pair_errors: sync");
  if (bad) return fail(c, CMSVD_E_SHAPE, "pair_errors: a device pair index is out of range");
  return pair_eval_dev(c, (const int2*)pairs, P, r, kinds, (const BaseDesc*)c.d_bdesc.p, d_ad, dims, err2, total,
                       sigma_tilde, mu);
}

// N3 (beyond the paper): residual bound with the tracked basis U_r and the per-index Weyl bound for the
// candidate pairs; err2x[2p + {0,1}], total[p].  Same validation and host/device conventions as
// do_pair_errors.
Status do_pair_errors_tight(Ctx& c, const int32_t* pairs, int64_t P, int32_t r, int operand, int where,
                            double* err2x, double* total) {
  if (P < 0) return fail(c, CMSVD_E_ARG, "pair_errors_tight: P < 0");
  if (P == 0) return CMSVD_OK;
  if (!pairs || !err2x || !total) return fail(c, CMSVD_E_ARG, "pair_errors_tight: pairs, err2x and total are required");
  if (c.count <= 0 || c.spectra_r <= 0) return fail(c, CMSVD_E_STATE, "pair_errors_tight: call block_spectra first");
  if (r != c.spectra_r) return fail(c, CMSVD_E_STATE, "pair_errors_tight: r differs from the block_spectra r");
  if (operand != CMSVD_OPERAND_RAW && operand != CMSVD_OPERAND_TRUNC)
    return fail(c, CMSVD_E_ARG, "pair_errors_tight: bad operand");
  if (where != CMSVD_HOST && where != CMSVD_DEVICE) return fail(c, CMSVD_E_ARG, "pair_errors_tight: bad `where`");
  const AppDesc* d_ad = (const AppDesc*)(operand == CMSVD_OPERAND_TRUNC ? c.d_adesc_trunc.p : c.d_adesc_raw.p);
  const Dims dims = block_dims(c, operand);
  if (where == CMSVD_HOST) {
    for (int64_t p = 0; p < 2 * P; ++p)
      if (pairs[p] < 0 || pairs[p] >= c.count)
        return fail(c, CMSVD_E_SHAPE, "pair_errors_tight: pair index out of range at entry " + std::to_string(p));
    size_t off = 0;
    size_t oP = off; off += align_up((size_t)P * 8, 256);
    size_t oE = off; off += align_up((size_t)P * 16, 256);
    size_t oT = off; off += align_up((size_t)P * 8, 256);
    CK(ensure(c.ws[WS_OUT], off), "pair_errors_tight: io buffers");
    char* b = (char*)c.ws[WS_OUT].p;
    CK(cudaMemcpyAsync(b + oP, pairs, (size_t)P * 8, cudaMemcpyHostToDevice, c.stream), "pair_errors_tight: h2d");
    Status s = pair_eval_dev(c, (const int2*)(b + oP), P, r, CMSVD_RESIDUAL, (const BaseDesc*)c.d_bdesc.p, d_ad, dims,
                             (double*)(b + oE), (double*)(b + oT), nullptr, nullptr, true);
    if (s != CMSVD_OK) return s;
    CK(cudaMemcpyAsync(err2x, b + oE, (size_t)P * 16, cudaMemcpyDeviceToHost, c.stream), "pair_errors_tight: d2h");
    CK(cudaMemcpyAsync(total, b + oT, (size_t)P * 8, cudaMemcpyDeviceToHost, c.stream), "pair_errors_tight: d2h");
    CK(cudaStreamSynchronize(c.stream), "pair_errors_tight: sync");
    return CMSVD_OK;
  }
  CK(ensure(c.ws[WS_BAD], 16), "pair_errors_tight: flag");
  CK(cudaMemsetAsync(c.ws[WS_BAD].p, 0, 4, c.stream), "pair_errors_tight: memset");
  CK(launch_check_pairs(c, (const int2*)pairs, P, c.count, (int*)c.ws[WS_BAD].p), "pair_errors_tight: check");
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c.ws[WS_BAD].p, 4, cudaMemcpyDeviceToHost, c.stream), "pair_errors_tight: flag d2h");
  CK(cudaStreamSynchronize(c.stream), "pair_errors_tight: sync");
  if (bad) return fail(c, CMSVD_E_SHAPE, "pair_errors_tight: a device pair index is out of range");
  return pair_eval_dev(c, (const int2*)pairs, P, r, CMSVD_RESIDUAL, (const BaseDesc*)c.d_bdesc.p, d_ad, dims, err2x,
                       total, nullptr, nullptr, true);
}

// Diagnostic entry: the pair path's batched eigensolver on caller matrices (include/cmsvd.h).
Status do_sym_eigvals(Ctx& c, int32_t count, int32_t nmax, const int32_t* n, const double* G, int32_t kw,
                      double* ev, double* trace) {
  if (!n || !G || !ev || count < 1) return fail(c, CMSVD_E_ARG, "sym_eigvals: NULL pointer or count < 1");
  if (nmax < 1 || nmax > 4096) return fail(c, CMSVD_E_SHAPE, "sym_eigvals: nmax must be in 1..4096");
  if (kw < 1 || kw > nmax) return fail(c, CMSVD_E_ARG, "sym_eigvals: kw must be in 1..nmax");
  for (int32_t p = 0; p < count; ++p)
    if (n[p] < 0 || n[p] > nmax) return fail(c, CMSVD_E_SHAPE, "sym_eigvals: n[p] outside 0..nmax");
  const size_t mat = (size_t)count * nmax * nmax * 8;
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t o = off; off += align_up(bytes, 256); return o; };
  const size_t oG = carve(mat), oN = carve((size_t)count * 4), oE = carve((size_t)count * kw * 8),
               oC = carve((size_t)count * 4), oT = carve((size_t)count * 8),
               oS = carve(tridiag_scratch_bytes(count, nmax));
  CK(ensure(c.ws[WS_PAIR], off), "sym_eigvals: workspace");
  char* b = (char*)c.ws[WS_PAIR].p;
  CK(cudaMemcpyAsync(b + oG, G, mat, cudaMemcpyHostToDevice, c.stream), "sym_eigvals: h2d");
  CK(cudaMemcpyAsync(b + oN, n, (size_t)count * 4, cudaMemcpyHostToDevice, c.stream), "sym_eigvals: h2d");
  CK(launch_tridiag_topk(c, (const double*)(b + oG), nmax, (int64_t)nmax * nmax, (const int*)(b + oN), count, nmax,
                         nullptr, kw, (double*)(b + oE), (int*)(b + oC), (double*)(b + oT), (double*)(b + oS)),
     "sym_eigvals: eigensolver");
  CK(cudaMemcpyAsync(ev, b + oE, (size_t)count * kw * 8, cudaMemcpyDeviceToHost, c.stream), "sym_eigvals: d2h");
  if (trace) CK(cudaMemcpyAsync(trace, b + oT, (size_t)count * 8, cudaMemcpyDeviceToHost, c.stream), "sym_eigvals: d2h");
  CK(cudaStreamSynchronize(c.stream), "sym_eigvals: sync");
  return CMSVD_OK;
}

}  // namespace cmsvd

// kernels.cuh -- launch wrappers of the libcmsvd kernels (host-callable).
#pragma once
#include "common.cuh"

namespace cmsvd {

// S1 energies
cudaError_t launch_energy(Ctx& c, const int64_t* d_boff, const int64_t* d_blen, int64_t maxlen, double* d_partial,
                          int* d_bad, double* d_E);
int energy_max_chunks(int64_t maxlen);

// SIMT batched GEMMs
cudaError_t launch_gemm_tn(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN, bool fp64acc);
cudaError_t launch_gemm_nn_sub(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN);

// eigensolvers
size_t syev_smem(int nmax);
// eigen-decomposition with vectors; VHws: scratch of nprob x stride_v doubles (Householder vectors)
cudaError_t launch_syev(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns, int nprob,
                        int nmax, double* Vws, int64_t stride_v, double* VHws, double* evals, int* perm,
                        int64_t stride_out, int* status);
size_t tridiag_smem(int nmax, int kw);
cudaError_t launch_tridiag_topk(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns,
                                int nprob, int nmax, const double* d_thr, int kw, double* ev, int* cnt,
                                double* trace, double* scratch, double* save = nullptr, int64_t save_stride = 0);
// whether launch_tridiag_topk can save the reflectors (register-resident kernel) at this size
bool tridiag_can_save(const Ctx& c, int nmax);
// top-kw eigenvectors (n x kw, ld n) of the matrix whose tridiagonal reduction is saved at `save` (layout of
// k_tridiag_rr), d = its diagonal, ev = its top-kw eigenvalues, gsh its Gershgorin data
cudaError_t launch_topk_vectors(Ctx& c, int n, int kw, const double* d, const double* save, const double* ev,
                                const double* gsh, double* Z);
size_t tridiag_scratch_bytes(int nprob, int nmax);
// two-stage (dense -> band -> tridiagonal) reduction for 160 < n <= 4096 (k_sbr.cu); outputs as k_tridiag
size_t sbr_ws_bytes(int nprob, int nmax);
cudaError_t launch_tridiag_sbr(Ctx& c, double* G, int64_t ld, int64_t stride, const int* d_ns, int nprob, int nmax,
                               const double* d_thr, int kw, int nstride, double* dd, double* ee, double* gsh,
                               int* cnt, double* trace, double* ws, int phase = 3);
int64_t sbr_ws_per(int nmax);   // doubles of band-reduction workspace per problem
// top-kw eigenpairs of one n x n symmetric matrix (n <= 160, kw <= 64): Z (n x kw, ld n), evals[kw]
// non-increasing; G is read only.  d_n: device int holding n.
size_t syev_topk_scratch_bytes(int n, int kw);
cudaError_t launch_syev_topk(Ctx& c, const double* G, int n, const int* d_n, int kw, double* Z, double* evals,
                             double* scratch);

// pair pipeline kernels (k_pair.cu)
__global__ void k_make_descs(const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad, int64_t m,
                             int use_full_basis, int QMAX, int WMAX, int GMAX, float* Zws, float* Rws, double* Wws,
                             double* ZZws, GemmDesc* dZ, GemmDesc* dR, GemmDesc* dW, GemmDesc* dZZ, int* nG, int* nW,
                             double* thrW, int r);
__global__ void k_build_G(const int2* pairs, const BaseDesc* bd, const AppDesc* ad, int QMAX, int WMAX, int GMAX,
                          const float* Zws, const double* Wws, const double* ZZws, double* Gws, double* zn2,
                          int upper);
__global__ void k_finalize_tight(const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad, int r,
                                 const double* evW, const int* cntW, const double* trW, const double* zn2,
                                 double* err2x, double* total);
__global__ void k_znorm(const int2* pairs, const BaseDesc* bd, const AppDesc* ad, const float* Zws, int QMAX,
                        int WMAX, double* zn2);
__global__ void k_finalize(const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad, int r, unsigned kinds,
                           const double* evG, const int* cntG, const double* trG, const double* evW, const int* cntW,
                           const double* trW, const double* zn2, double* err2, double* total, float* sigma_tilde,
                           float* mu);
__global__ void k_spec_stats(int count, int nmax, int r, const double* evals, const int* kcols, const double* E,
                             double* sig, float* sig32, int* rank, const int64_t* uoff, const float* Ubase,
                             const int64_t* boff, const int* ncols, const float* arena, const int64_t* foff,
                             const float* Fbase, BaseDesc* bd, AppDesc* ad_raw, AppDesc* ad_trunc, double tau);
__global__ void k_leftvec(int64_t m, const float* arena, const int64_t* boff, const int* kcols, const double* V,
                          int64_t strideV, const int* perm, int nmax, const double* sig, const int* rank, float* U,
                          const int64_t* uoff);
cudaError_t launch_pair_tc(Ctx& c, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad, int64_t m,
                           int use_full_basis, int QMAX, int WMAX, float* Zws, double* Wws);
// batched 3xTF32 tcgen05 GEMM tiles (C = A^T B, or C = C0 - A B with nnsub); out64: fp64 C
cudaError_t launch_gemm_tc(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN, bool nnsub, bool out64);
// warp-specialised TMA-fed 3xTF32 contractions on pre-split tf32 planes (k_gemm_ws.cu).  mode 0: Z = Q^T F
// (fp32 Z + its planes), 1: planes of R' = F - Q Z, 2: W' = R'^T R' (fp64)
bool gemm_ws_supported(const Ctx& c, int64_t m);
cudaError_t launch_split_planes(Ctx& c, const float* src, int64_t sstride, int64_t rows, int cols, int cols_dst,
                                int count, float* dst);
cudaError_t launch_split_planes_t(Ctx& c, const float* src, int64_t sstride, int64_t rows, int cols, int count,
                                  float* dst);
cudaError_t launch_split_planes_ptr(Ctx& c, const float* const* d_srcp, int64_t rows, int cols, int count, float* dst,
                                    float* dst_t);
cudaError_t launch_split_planes64(Ctx& c, const double* src, int64_t n, int count, float* dst);
cudaError_t launch_gemm_ws_tn64(Ctx& c, int batch, int M, int N, int K, const float* Ap, const float* Bp, bool b_shared,
                                double* C, int64_t ldc, int64_t sC);
bool gemm_ws_available();
cudaError_t launch_gemm_ws(Ctx& c, int mode, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad,
                           int use_full, int QMAX, int WMAX, float* Zws, float* Zp, float* Rp, double* Wws,
                           bool add_zz = false);   // mode 2 with add_zz: Wws = Z^T Z + R'^T R' (WMAX <= 256)
// C (fp64) = A B, A: M x K, B: K x N column-major fp32 (3xTF32 tiles)
cudaError_t launch_gemm_tc_nn64(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN);
// Y[i] = (float) X[i] for n doubles
cudaError_t launch_to_f32(Ctx& c, const double* X, float* Y, int64_t n);
cudaError_t launch_syrk_zz(Ctx& c, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad,
                           int use_full_basis, int QMAX, int WMAX, const float* Zws, double* ZZws);
cudaError_t launch_build_G1(Ctx& c, int rr, int w, const double* spec, const float* Z, int ldz, const double* ZZ,
                            const double* WW, double* G);
// k_big.cu: large-block spectra helpers
template <typename TAe, bool TA>
cudaError_t gemm_mixed(Ctx& c, int batch, int M, int N, int K, const TAe* A, int64_t lda, int64_t sA,
                       const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
                       double alpha = 1.0, const TAe* const* Ap = nullptr, int shape = 0);
__global__ void k_big_leftvec(int64_t m, int s, int kc, const double* Y, const double* V, const int* perm,
                              float* const* Uout);
__global__ void k_big_stats(int nb, const int* ids, int s, int r, int64_t m, int nmax_sig, const double* ev,
                            const double* E, const int* ncols, double* sig, float* sig32, int* rank,
                            const float* const* Uptr, const float* const* Aptr, const float* const* Fptr,
                            BaseDesc* bd, AppDesc* ad_raw, AppDesc* ad_trunc);
cudaError_t launch_randn(Ctx& c, double* X, int64_t n, uint64_t seed);
// Ritz-residual guard of the big-block spectra: Wg[b] = V[b][:, perm[b][0..kc)] (s x kc), and
// resid[b] = max_{l<kc} ||P[b][:, l] - lambda_l U[b][:, l]|| / lambda_l
constexpr double kRitzTol = 1e-4;
cudaError_t launch_ritz_gather(Ctx& c, int nb, int s, int kc, const double* V, const int* perm, double* Wg);
cudaError_t launch_ritz_resid(Ctx& c, int nb, int64_t m, int s, int kc, const double* P, const double* ev,
                              const float* const* U, double* resid);
cudaError_t cholqr(Ctx& c, int batch, int64_t rows, int s, double* Y, double* Ytmp, double* H, double* T,
                   int* status, int passes = 2);
__global__ void k_trunc_operand(int64_t m, const BaseDesc* bd, const AppDesc* ad_trunc, float* Fbase);

}  // namespace cmsvd

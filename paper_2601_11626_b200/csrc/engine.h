// engine.h -- host-side entry points of the libcmsvd engine (used by abi.cu
// and cluster.cu).
#pragma once
#include "common.cuh"

namespace cmsvd {

typedef cmsvd_status Status;

constexpr int kEigMax = 512;  // largest Gram handled by the eigensolvers (> 160: in place in global memory)

// context workspace slots (Ctx::ws)
enum { WS_PARTIAL = 0, WS_BAD, WS_META, WS_G, WS_V, WS_EV, WS_PERM, WS_STAT, WS_PAIR, WS_OUT, WS_A, WS_B, WS_C, WS_D, WS_E, WS_SBR };

struct Dims {
  int qmax = 0;   // projection-basis columns (full range)
  int rrmax = 0;  // tracked top-r columns
  int wmax = 0;   // appended-operand columns
  bool planes = false;  // every base / appended operand is a registered block's U_r / TRUNC factor (their tf32
                        // planes exist: k_gemm_ws may be used)
};

Status fail(Ctx& c, cmsvd_status s, const std::string& msg);

// profiling helpers: prof_begin returns the index of an open record (or -1)
int prof_begin(Ctx& c, int cat);
void prof_end(Ctx& c, int rec, int64_t work = 0);
void prof_collect(Ctx& c);
Status cuda_fail(Ctx& c, cudaError_t e, const char* where);

Status do_register(Ctx& c, int64_t m, int32_t count, const int32_t* n, const float* const* blocks, const int64_t* ld,
                   int where);
Status do_block_spectra_big(Ctx& c, int32_t r, double* energy, float* sigma, int32_t* rank_out);
Status do_block_spectra(Ctx& c, int32_t r, double* energy, float* sigma, int32_t* rank_out);
Status do_pair_errors(Ctx& c, const int32_t* pairs, int64_t P, int32_t r, uint32_t kinds, int operand, int where,
                      double* err2, double* total, float* sigma_tilde, float* mu);
// Reflectors of the incremental Grams kept by an evaluation (the greedy driver commits the accepted
// candidate from them instead of reducing G again).  In: save (P x save_stride doubles) or nullptr.
// Out: kept, and device pointers to the diagonals (ld nstride), Gershgorin data (4 per pair) and top-r
// eigenvalues (r per pair) of the evaluated Grams.
struct EigKeep {
  double* save = nullptr;
  int64_t save_stride = 0;
  bool kept = false;
  const double* dd = nullptr;
  const double* gsh = nullptr;
  const double* evG = nullptr;
  int nstride = 0;
};
Status pair_eval_dev(Ctx& c, const int2* d_pairs, int64_t P, int r, unsigned kinds, const BaseDesc* d_bd,
                     const AppDesc* d_ad, const Dims& dims, double* d_err2, double* d_total, float* d_st, float* d_mu,
                     bool tight = false, EigKeep* keep = nullptr);
Status do_pair_errors_tight(Ctx& c, const int32_t* pairs, int64_t P, int32_t r, int operand, int where,
                            double* err2x, double* total);
Dims block_dims(const Ctx& c, int operand);
cudaError_t launch_check_pairs(Ctx& c, const int2* d_pairs, int64_t P, int count, int* d_bad);
Status do_cluster_factors(Ctx& c, int32_t r, const int32_t* assign, int32_t n_clusters, float* Ut, float* V,
                          int32_t* rc_out);
Status do_cluster_verify(Ctx& c, int32_t r, const int32_t* assign, int32_t n_clusters, double* exact_err2,
                         double* total, int64_t* mem);
Status do_sequence_errors(Ctx& c, const int32_t* offs, const int32_t* ids, int32_t nseq, int32_t r, uint32_t kinds,
                          int operand, double* err2, double* total);
Status do_sym_eigvals(Ctx& c, int32_t count, int32_t nmax, const int32_t* n, const double* G, int32_t kw,
                      double* ev, double* trace);
Status do_cluster(Ctx& c, const cmsvd_cluster_opts* o, int32_t* assign, int32_t* order, int32_t* n_clusters,
                  double* cluster_err2, double* cluster_total, int64_t* n_evals);

}  // namespace cmsvd

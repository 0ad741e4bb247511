// common.cuh -- shared device helpers and the internal context of libcmsvd.
// B200 (sm_100a) only.  Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/cmsvd.h"


namespace cmsvd {

// Numerical-rank rule (reading A5): keep sigma_l > kTau * sigma_1.
constexpr double kTau = 1e-5;
constexpr int kThreads = 256;
constexpr int kArenaAlign = 32;  // floats (128 B) between block starts

// ---------------------------------------------------------------------------
// Device-side descriptors
// ---------------------------------------------------------------------------
// A "base" of a candidate merge: a block (its left singular basis and
// spectrum) or a cluster state of Alg. 2 / Alg. 3.
struct BaseDesc {
  const float* basis;   // m x q column-major (ld = m); first rr columns = tracked top-r basis
  const double* spec;   // spectrum, non-increasing, ns entries (sigma(A_i) all / mu pool / sigma~)
  int q;                // columns of the projection basis used by this evaluation
  int rr;               // size of the tracked top-r part (incremental)
  int ns;               // length of spec
  int full;             // 1: the base's range is all of R^m (A22, blocks wider than kEigMax): the
                        //    paper-literal residual (I - QQ^T)F is identically 0
  double E;             // energy ||.||_F^2 of the base
  double tail_inc;      // E - sum_{l<rr} spec_l^2, computed as a sum of the dropped part (>= 0)
  double rest_res;      // E - sum_{all l} spec_l^2 (energy not represented in spec, >= 0)
  double tailw;         // E - sum_{l<r} spec_l^2 (Weyl), summed from the dropped part
};

// An appended operand F (RAW block or TRUNC factor).
struct AppDesc {
  const float* F;       // m x w column-major (ld = m)
  int w;
  int ns;               // length of spec
  double E;             // full energy of the appended block
  double extra;         // E - ||F||_F^2 for TRUNC (the dropped tail), 0 for RAW
  double tailw;         // E - sum_{l<r} sigma_l^2 of the appended block (Weyl)
  const double* spec;   // sigma of the appended block, non-increasing (per-index Weyl, N3)
};

// One batched-GEMM problem for the SIMT kernels.
struct GemmDesc {
  const float* A; const float* B; const float* C0;  // C0: optional minuend (R = C0 - A B)
  void* C;
  int64_t lda, ldb, ldc, ldc0;
  int M, N, K;
  int sym;  // 1: C symmetric, only lower tiles computed and mirrored
};

// ---------------------------------------------------------------------------
// Host-side context
// ---------------------------------------------------------------------------
struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
};

// Per-kernel-category CUDA-event timing (cmsvd_profile_enable/read).
enum ProfCat {
  PC_ENERGY = 0, PC_SPEC_GRAM, PC_SPEC_EIG, PC_SPEC_MISC, PC_DESCS, PC_PROJ, PC_RESID, PC_GRAM_W, PC_GRAM_ZZ,
  PC_BUILD_G, PC_EIG_G, PC_EIG_W, PC_FINALIZE, PC_CLUSTER, PC_PAIR_TC, PC_SBR_PANEL, PC_SBR_SYMM, PC_SBR_SYR2K,
  PC_SBR_CHASE, PC_BISECT, PC_COUNT
};
static const char* const kProfNames[PC_COUNT] = {
  "energy", "spectra_gram", "spectra_eig", "spectra_misc", "pair_descs", "proj_Z", "resid_R", "gram_W",
  "gram_ZZ", "build_G", "eig_G", "eig_W", "finalize", "cluster_misc", "pair_tc", "sbr_panel", "sbr_symm",
  "sbr_syr2k", "sbr_chase", "bisect"};

struct Prof {
  bool on = false;
  struct Rec { int cat; cudaEvent_t a, b; int64_t work; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double ms[PC_COUNT] = {};
  int64_t launches[PC_COUNT] = {};
  int64_t work[PC_COUNT] = {};
};

struct Ctx {
  int device = 0;
  Prof prof;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t launches = 0;
  int sm_count = 148;

  // collection
  int64_t m = 0;
  int32_t count = 0;
  std::vector<int32_t> n;        // host copy
  std::vector<int64_t> boff;     // arena offsets (floats)
  int nmax = 0;
  DevMem arena;                  // packed fp32 blocks
  DevMem d_E;                    // fp64 energies
  std::vector<double> E;         // host copy

  // spectra (valid when spectra_r > 0)
  int spectra_r = 0;
  std::vector<int64_t> uoff;     // basis offsets (floats), block i basis m x k_i
  std::vector<int32_t> kcols;    // k_i = min(m, n_i)
  DevMem d_U;                    // fp32 left singular vectors
  DevMem d_sig;                  // fp64 all singular values, count x nmax
  std::vector<double> sig;       // host copy
  std::vector<int32_t> rank, rr;
  DevMem d_Ftrunc;               // fp32 TRUNC operands, m x min(r, k_i) each at foff
  std::vector<int64_t> foff;
  bool trunc_ready = false;
  // tf32 hi/lo planes of the bases and TRUNC operands (A22 collections with operands wider than 128 columns):
  // count x 2 x planes_cols x m fp32 each, fed to k_gemm_ws by TMA
  DevMem d_Ap, d_ATp;          // S2 (A22): tf32 planes of the blocks and of their transposes (k_gemm_ws MODE 3)
  DevMem d_Qp, d_Fp, d_QTp;   // QTp: the Q planes transposed (count x 2 x m x planes_cols), A operand of R' = F - Q Z
  int planes_cols = 0;
  const float* planes_F = nullptr;   // the fp32 TRUNC operands the F planes were split from (block i at i * planes_fstride)
  int64_t planes_fstride = 0;
  bool planes_ok = false;
  DevMem d_sig32, d_rank, d_bdesc, d_adesc_raw, d_adesc_trunc, d_meta64, d_meta32;

  // workspaces (grow-only)
  DevMem ws[16];
  DevMem cws[16];  // cluster-driver state and scratch
  size_t ws_budget = (size_t)24 << 30; // bytes of pair workspace per chunk (config 4: all 2016 pairs in one chunk)
  bool use_tc = true;                  // tcgen05 contraction kernel (CMSVD_NO_TC=1 selects the SIMT path)
  bool tc_ok = true;                   // every block numerically full column rank (set by block_spectra)
  int gl_batch_mb = 1024;              // in-place global-memory eigen batches (n > 160), MB of matrices per launch
  int syev_flags = 3;                  // k_syev_ql<true>: bit 0 column-resident back-transformation (CMSVD_SYEV_COLBT=0 clears), bit 1 fused QL sweeps (CMSVD_SYEV_QLF=0 clears)
  bool sbr_fused = false;              // band reduction: look-ahead fused update + product pass (CMSVD_SBR_FUSED=1;
                                       // measured 24.8 vs 23.0 ms unfused at n = 512: the partials' traffic)
  bool sbr_tma = true;                 // band reduction: TMA tile loads/stores in the rank-32 update (CMSVD_SBR_TMA=0)
  bool symm_dmma = true;               // band reduction: Y = A22 V T on the fp64 tensor cores (CMSVD_SYMM_DMMA=0: scalar kernel)
  bool syr2k_dmma = true;              // band reduction: rank-32 update on the fp64 tensor cores (CMSVD_SYR2K_DMMA=0: scalar kernel)
  bool syr2k_row = true;               // band reduction: row-persistent two-stage pipelined rank-32 update (CMSVD_SYR2K_ROW=0: one tile
                                       // per CTA); with the DMMA update 15.3 vs 16.8 ms, with the scalar update equal (17.2 vs 17.3)
  bool chase2 = false;                 // band chase: two problems in flight per persistent CTA (CMSVD_CHASE2=1).  Measured 25.6 vs
                                       // 22.8 ms: the chase is bound by task throughput (~4.7 tasks/us/SM in both), not by latency
  bool chase_small = true;             // band chase, n <= 256: 6-warp CTAs with half the band, two per SM (CMSVD_CHASE_SMALL=0: off)
  bool chase_split = true;             // band chase, n <= 512: phases on ever smaller bands as the active part shrinks (512 / 384 /
                                       // 256 / 128 rows: 1 / 2 / 2 / 4 CTAs per SM; CMSVD_CHASE_SPLIT=0: one kernel)
  bool chase_flags = false;            // band chase: per-sweep progress flags instead of time-step barriers
  int g_upper = 1;                     // core Grams of the band reduction: 1 = strict upper triangle not written, 0 = written,
                                       // 2 = poisoned with NaN (CMSVD_G_UPPER; the band reduction reads the lower storage only)
  int sbr_groups = 1;                  // band reduction, n <= 512: the band chase runs in this many groups of whole CTA waves, the
                                       // bisection of a finished group on a second stream under the next group's chase
                                       // (CMSVD_SBR_GROUPS; 1: one stream)
  cudaStream_t aux_stream = nullptr;   // second stream of the pipelined band reduction (created on first use)
  cudaEvent_t aux_ev[17] = {};         // group hand-over events + the join
  bool bisect_p = true;                // bisection on the division-free polynomial Sturm recurrence (CMSVD_BISECT_P=0: pivot form
                                       // with the fp32 coarse phase)
  bool sbr_panel_rr = true;            // band reduction, n <= 512: register-resident panel QR (CMSVD_SBR_PANEL_RR=0: shared-memory kernel)
  bool eig_sbr = true;                 // n > 160: two-stage (band) reduction instead of the one-stage in-place kernel
  bool eig_rr = true;                  // register-resident tridiagonalisation for n <= 160 (CMSVD_EIG_RR=0: smem kernel)
  bool zz_syrk = true;                 // w <= 128: Z^T Z by k_syrk_zz instead of k_gemm_tn (CMSVD_ZZ_SYRK=0: off)
  bool tc_big = true;                  // q or w > 128: tcgen05 GEMM tiles instead of SIMT (CMSVD_TC_BIG=0: off)
  bool tc_ws = true;                   // ... by the warp-specialised TMA-fed kernel on pre-split planes (CMSVD_TC_WS=0: off)
  bool zz_fused = true;                // k_gemm_ws: Z^T Z folded into the W' contraction (CMSVD_ZZ_FUSED=0: separate fp64 Gram)
  bool chol_blocked = true;            // CholQR: blocked Cholesky + inverse kernel (CMSVD_CHOL_BLOCKED=0: unblocked)
  bool big_tc = true;                  // A22 subspace-iteration products on tcgen05 tiles (CMSVD_BIG_TC=0: SIMT fp64)
  bool tc_wide = true;                 // ... with 256-column tiles for Z = Q^T F (CMSVD_TC_WIDE=0: 128)
  bool eig_duo = true;                 // n <= 128: two problems per CTA with dedicated row warps (CMSVD_EIG_DUO=0: off)
  bool eig_duo160 = true;              // ... and for 128 < n <= 160 (CMSVD_EIG_DUO160=0: off)
  bool commit_topk = true;             // Alg. 3 commits: top-r eigenpairs by inverse iteration (CMSVD_COMMIT_TOPK=0: QL)
  bool big = false;                    // collection of blocks wider than kEigMax (A22 spectra, full-range bases)
  int subspace_iters = 12;             // power iterations of the big-block spectra (CMSVD_SUBSPACE_ITERS)
  int subspace_max = 48;               // ... at most, while the Ritz-residual guard fails (CMSVD_SUBSPACE_MAX)
  double spectra_resid = 0.0;          // largest Ritz residual of the last big-block spectra (diagnostic)
  int spectra_iters = 0;               // power iterations the last big-block spectra needed
};

// grow-only device buffer
cudaError_t ensure(DevMem& b, size_t bytes);
void release(DevMem& b);

}  // namespace cmsvd

struct cmsvd_ctx_s {
  cmsvd::Ctx c;
};

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
namespace cmsvd {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree); red must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

}  // namespace cmsvd

#include <algorithm>
// abi.cu -- the extern "C" boundary of libcmsvd (declared in include/cmsvd.h).
// Every entry point converts C++/CUDA failures into a cmsvd_status plus a
// per-context message; no exception crosses the ABI.
#include <cmath>
#include <cstring>
#include <new>

#include "common.cuh"
#include "engine.h"

using namespace cmsvd;

namespace cmsvd {
__global__ void k_check_pairs(const int2* __restrict__ pairs, int64_t P, int count, int* bad) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int2 v = pairs[p];
  if (v.x < 0 || v.x >= count || v.y < 0 || v.y >= count) atomicOr(bad, 1);
}

cudaError_t launch_check_pairs(Ctx& c, const int2* d_pairs, int64_t P, int count, int* d_bad) {
  k_check_pairs<<<(unsigned)((P + 255) / 256), 256, 0, c.stream>>>(d_pairs, P, count, d_bad);
  c.launches += 1;
  return cudaGetLastError();
}
}  // namespace cmsvd

#define GUARD_CTX(ctx)                       \
  if (!(ctx)) return CMSVD_E_ARG;            \
  Ctx& c = (ctx)->c;                         \
  c.err.clear();                             \
  {                                          \
    cudaError_t _e = cudaSetDevice(c.device); \
    if (_e != cudaSuccess) return cuda_fail(c, _e, "cudaSetDevice"); \
  }

extern "C" {

const char* cmsvd_status_string(cmsvd_status s) {
  switch (s) {
    case CMSVD_OK: return "CMSVD_OK";
    case CMSVD_E_ARG: return "CMSVD_E_ARG";
    case CMSVD_E_SHAPE: return "CMSVD_E_SHAPE";
    case CMSVD_E_NONFINITE: return "CMSVD_E_NONFINITE";
    case CMSVD_E_STATE: return "CMSVD_E_STATE";
    case CMSVD_E_NOCONV: return "CMSVD_E_NOCONV";
    case CMSVD_E_CUDA: return "CMSVD_E_CUDA";
    case CMSVD_E_NOMEM: return "CMSVD_E_NOMEM";
  }
  return "CMSVD_E_UNKNOWN";
}

const char* cmsvd_last_error(cmsvd_ctx ctx) { return ctx ? ctx->c.err.c_str() : "NULL context"; }

const char* cmsvd_version(void) { return "cmsvd 0.1 (sm_100a)"; }

cmsvd_status cmsvd_create(int device, void* cuda_stream, cmsvd_ctx* out) {
  if (!out) return CMSVD_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return CMSVD_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return CMSVD_E_CUDA;
  cmsvd_ctx h = new (std::nothrow) cmsvd_ctx_s();
  if (!h) return CMSVD_E_NOMEM;
  h->c.device = device;
  if (cuda_stream) {
    h->c.stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete h;
      return CMSVD_E_CUDA;
    }
    h->c.own_stream = true;
  }
  cudaDeviceGetAttribute(&h->c.sm_count, cudaDevAttrMultiProcessorCount, device);
  if (const char* env = getenv("CMSVD_WS_BYTES")) h->c.ws_budget = (size_t)atoll(env);
  if (const char* env = getenv("CMSVD_NO_TC")) h->c.use_tc = !(env[0] == '1');
  if (const char* env = getenv("CMSVD_GL_BATCH_MB")) h->c.gl_batch_mb = std::max(1, atoi(env));
  if (const char* env = getenv("CMSVD_SYEV_COLBT")) if (env[0] == '0') h->c.syev_flags &= ~1;
  if (const char* env = getenv("CMSVD_SYEV_QLF")) if (env[0] == '0') h->c.syev_flags &= ~2;
  if (const char* env = getenv("CMSVD_ZZ_SYRK")) h->c.zz_syrk = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_BIG_TC")) h->c.big_tc = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_TC_WIDE")) h->c.tc_wide = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_TC_BIG")) h->c.tc_big = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_TC_WS")) h->c.tc_ws = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_ZZ_FUSED")) h->c.zz_fused = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_G_UPPER")) h->c.g_upper = atoi(env);
  if (const char* env = getenv("CMSVD_SBR_GROUPS")) h->c.sbr_groups = std::max(1, std::min(16, atoi(env)));
  if (const char* env = getenv("CMSVD_CHASE_SPLIT")) h->c.chase_split = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_BISECT_P")) h->c.bisect_p = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SBR_PANEL_RR")) h->c.sbr_panel_rr = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_CHOL_BLOCKED")) h->c.chol_blocked = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_EIG_DUO")) h->c.eig_duo = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_EIG_DUO160")) h->c.eig_duo160 = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_COMMIT_TOPK")) h->c.commit_topk = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SBR_FUSED")) h->c.sbr_fused = (env[0] == '1');
  if (const char* env = getenv("CMSVD_SBR_TMA")) h->c.sbr_tma = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SYMM_DMMA")) h->c.symm_dmma = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SYR2K_DMMA")) h->c.syr2k_dmma = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SYR2K_ROW")) h->c.syr2k_row = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_CHASE2")) h->c.chase2 = (env[0] == '1');
  if (const char* env = getenv("CMSVD_CHASE_SMALL")) h->c.chase_small = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_CHASE_FLAGS")) h->c.chase_flags = (env[0] == '1');
  if (const char* env = getenv("CMSVD_EIG_SBR")) h->c.eig_sbr = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_EIG_RR")) h->c.eig_rr = !(env[0] == '0');
  if (const char* env = getenv("CMSVD_SUBSPACE_MAX")) h->c.subspace_max = std::max(0, atoi(env));
  if (const char* env = getenv("CMSVD_SUBSPACE_ITERS")) h->c.subspace_iters = std::max(0, atoi(env));
  *out = h;
  return CMSVD_OK;
}

cmsvd_status cmsvd_destroy(cmsvd_ctx ctx) {
  if (!ctx) return CMSVD_OK;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  DevMem* bufs[] = {&c.arena, &c.d_E, &c.d_U, &c.d_sig, &c.d_Ftrunc, &c.d_sig32, &c.d_rank,
                    &c.d_bdesc, &c.d_adesc_raw, &c.d_adesc_trunc, &c.d_meta64, &c.d_meta32, &c.d_Qp, &c.d_Fp, &c.d_QTp, &c.d_Ap, &c.d_ATp};
  for (DevMem* b : bufs) release(*b);
  for (auto& b : c.ws) release(b);
  for (auto& b : c.cws) release(b);
  prof_collect(c);
  for (auto e : c.prof.pool) cudaEventDestroy(e);
  if (c.aux_stream) cudaStreamDestroy(c.aux_stream);
  for (auto& ev : c.aux_ev)
    if (ev) cudaEventDestroy(ev);
  if (c.own_stream) cudaStreamDestroy(c.stream);
  delete ctx;
  return CMSVD_OK;
}

cmsvd_status cmsvd_register(cmsvd_ctx ctx, int64_t m, int32_t count, const int32_t* n, const float* const* blocks,
                            const int64_t* ld, int where) {
  GUARD_CTX(ctx);
  try {
    return do_register(c, m, count, n, blocks, ld, where);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "register: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "register: unexpected exception");
  }
}

cmsvd_status cmsvd_block_spectra(cmsvd_ctx ctx, int32_t r, double* energy, float* sigma, int32_t* rank_out) {
  GUARD_CTX(ctx);
  try {
    return do_block_spectra(c, r, energy, sigma, rank_out);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "block_spectra: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "block_spectra: unexpected exception");
  }
}

cmsvd_status cmsvd_pair_errors(cmsvd_ctx ctx, const int32_t* pairs, int64_t P, int32_t r, uint32_t kinds, int operand,
                               int where, double* err2, double* total, float* sigma_tilde, float* mu) {
  GUARD_CTX(ctx);
  try {
    return do_pair_errors(c, pairs, P, r, kinds, operand, where, err2, total, sigma_tilde, mu);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "pair_errors: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "pair_errors: unexpected exception");
  }
}

cmsvd_status cmsvd_pair_errors_tight(cmsvd_ctx ctx, const int32_t* pairs, int64_t P, int32_t r, int operand,
                                     int where, double* err2x, double* total) {
  GUARD_CTX(ctx);
  try {
    return do_pair_errors_tight(c, pairs, P, r, operand, where, err2x, total);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "pair_errors_tight: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "pair_errors_tight: unexpected exception");
  }
}

cmsvd_status cmsvd_cluster_verify(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters,
                                  double* exact_err2, double* total, int64_t* mem) {
  GUARD_CTX(ctx);
  try {
    return do_cluster_verify(c, r, assign, n_clusters, exact_err2, total, mem);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "cluster_verify: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "cluster_verify: unexpected exception");
  }
}

cmsvd_status cmsvd_cluster_verify_ex(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters,
                                     double* exact_err2, double* total, int64_t* mem, double* rel, double* ratio) {
  GUARD_CTX(ctx);
  try {
    Status st = do_cluster_verify(c, r, assign, n_clusters, exact_err2, total, mem);
    if (st != CMSVD_OK) return st;
    double raw = 0.0, stored = 0.0;
    for (int32_t i = 0; i < c.count; ++i) raw += (double)c.m * (double)c.n[i];
    for (int32_t g = 0; g < n_clusters; ++g) {
      stored += (double)mem[g];
      if (rel) rel[g] = total[g] > 0.0 ? std::sqrt(std::max(exact_err2[g], 0.0) / total[g]) : 0.0;
    }
    if (ratio) *ratio = stored > 0.0 ? raw / stored : 0.0;
    return CMSVD_OK;
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "cluster_verify: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "cluster_verify: unexpected exception");
  }
}

cmsvd_status cmsvd_sequence_errors(cmsvd_ctx ctx, const int32_t* offs, const int32_t* ids, int32_t nseq, int32_t r,
                                   uint32_t kinds, int operand, double* err2, double* total) {
  GUARD_CTX(ctx);
  try {
    return do_sequence_errors(c, offs, ids, nseq, r, kinds, operand, err2, total);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "sequence_errors: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "sequence_errors: unexpected exception");
  }
}

cmsvd_status cmsvd_cluster_factors(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters, float* Ut,
                                   float* V, int32_t* rc) {
  GUARD_CTX(ctx);
  try {
    return do_cluster_factors(c, r, assign, n_clusters, Ut, V, rc);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "cluster_factors: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "cluster_factors: unexpected exception");
  }
}

cmsvd_status cmsvd_cluster(cmsvd_ctx ctx, const cmsvd_cluster_opts* opts, int32_t* assign, int32_t* order,
                           int32_t* n_clusters, double* cluster_err2, double* cluster_total, int64_t* n_evals) {
  GUARD_CTX(ctx);
  try {
    return do_cluster(c, opts, assign, order, n_clusters, cluster_err2, cluster_total, n_evals);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "cluster: host allocation failed");
  } catch (...) {
    return fail(c, CMSVD_E_ARG, "cluster: unexpected exception");
  }
}

cmsvd_status cmsvd_sym_eigvals(cmsvd_ctx ctx, int32_t count, int32_t nmax, const int32_t* n, const double* G,
                               int32_t kw, double* ev, double* trace) {
  GUARD_CTX(ctx);
  try {
    return do_sym_eigvals(c, count, nmax, n, G, kw, ev, trace);
  } catch (const std::bad_alloc&) {
    return fail(c, CMSVD_E_NOMEM, "sym_eigvals: host allocation failed");
  }
}

cmsvd_status cmsvd_spectra_diagnostics(cmsvd_ctx ctx, double* max_ritz_residual, int32_t* power_iterations) {
  if (!ctx) return CMSVD_E_ARG;
  if (max_ritz_residual) *max_ritz_residual = ctx->c.big ? ctx->c.spectra_resid : 0.0;
  if (power_iterations) *power_iterations = ctx->c.big ? ctx->c.spectra_iters : 0;
  return CMSVD_OK;
}

int64_t cmsvd_launch_count(cmsvd_ctx ctx) { return ctx ? ctx->c.launches : 0; }

cmsvd_status cmsvd_profile_enable(cmsvd_ctx ctx, int enable) {
  GUARD_CTX(ctx);
  prof_collect(c);
  c.prof.on = enable != 0;
  for (int k = 0; k < PC_COUNT; ++k) { c.prof.ms[k] = 0.0; c.prof.launches[k] = 0; c.prof.work[k] = 0; }
  return CMSVD_OK;
}

int32_t cmsvd_profile_read(cmsvd_ctx ctx, int32_t max, const char** names, double* ms, int64_t* launches) {
  if (!ctx) return 0;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  prof_collect(c);
  int32_t k = 0;
  for (; k < PC_COUNT && k < max; ++k) {
    if (names) names[k] = kProfNames[k];
    if (ms) ms[k] = c.prof.ms[k];
    if (launches) launches[k] = c.prof.launches[k];
  }
  return k;
}

}  // extern "C"

/*
 * cmsvd.h -- C ABI of the B200-native merge-error evaluation library
 * (arXiv 2601.11626, "compression-aware clustering of matrices under SVD
 * constraints").  Implemented in paper_2601_11626_b200/csrc (CUDA, sm_100a);
 * built as paper_2601_11626_b200/libcmsvd.so.
 *
 * The calls follow the paper's problem statement:
 *   cmsvd_register       register the collection A = {A_i in R^{m x n_i}}
 *                        (Eq. matrix_set) and compute the
 *                        Frobenius energies ||A_i||_F^2.
 *   cmsvd_block_spectra  per-block leading singular values and bases; the
 *                        Weyl bound "relies only on the Frobenius norms and
 *                        the leading singular values of the blocks"
 *                        (PAPER.md:247-249); Alg. 3 starts from the anchor's
 *                        top-r SVD.
 *   cmsvd_pair_errors    merge certificates (Definition 1)
 *                        for candidate (base, appended) pairs: Weyl bound
 *                        (Thm 1 / Eq. 5), residual bound
 *                        (Thm 2 + Cor 1 / Eq. 6) and the
 *                        incremental plug-in estimate (Lemma 1 + Cor 3 +
 *                        Cor 2).
 *   cmsvd_cluster        greedy clustering under (eps, r): Algorithms 1-3 of
 *                        Appendix E; the drivers run on
 *                        the host and call the GPU only for error evaluation
 *                        and state commits.
 *
 * Conventions (all entry points):
 *  - Errors: every call returns a cmsvd_status; on failure the outputs are
 *    unspecified and cmsvd_last_error(ctx) holds a one-line detail (valid
 *    until the next call on that context).  No C++ exception crosses the ABI.
 *  - Synchronisation: calls are synchronous with respect to their outputs
 *    (host outputs are written when the call returns; device outputs are
 *    complete on the context stream when the call returns).
 *  - Concurrency: a context is single-writer; distinct contexts may be used
 *    from different threads.
 *  - Determinism: identical inputs give bit-identical outputs on the same GPU
 *    (fixed reduction orders, no floating-point atomics).
 *  - Layout: matrices are column-major fp32; energies and squared errors are
 *    fp64; singular values are fp32.
 *  - Memory: the library owns its device memory (cudaMalloc on the context's
 *    device); caller pointers are borrowed for the duration of the call only.
 *  - Readings of ambiguous paper passages (rank tolerance tau = 1e-5, the
 *    TRUNC operand, pair orientation, inclusive thresholds, ...) are listed
 *    in DESIGN.md ("Readings").
 */
#ifndef CMSVD_H
#define CMSVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cmsvd_ctx_s* cmsvd_ctx;

typedef enum {
  CMSVD_OK = 0,
  CMSVD_E_ARG = 1,        /* invalid argument (NULL where required, r < 1, eps not in (0,1), ...) */
  CMSVD_E_SHAPE = 2,      /* m, n_i or count <= 0, ld < m, index out of range, unsupported shape */
  CMSVD_E_NONFINITE = 3,  /* NaN/Inf in a registered block */
  CMSVD_E_STATE = 4,      /* call order violated (e.g. pair_errors before block_spectra(r)) */
  CMSVD_E_NOCONV = 5,     /* an iterative eigensolver did not converge; detail names the problem */
  CMSVD_E_CUDA = 6,       /* CUDA runtime error (detail carries cudaGetErrorString) */
  CMSVD_E_NOMEM = 7       /* device or host allocation failed */
} cmsvd_status;

/* Where caller buffers live. */
enum { CMSVD_HOST = 0, CMSVD_DEVICE = 1 };

/* Estimator bitmask ("bound kind"). */
enum { CMSVD_WEYL = 1u, CMSVD_RESIDUAL = 2u, CMSVD_INCREMENTAL = 4u, CMSVD_ALL = 7u };

/* Appended operand (reading A6): RAW = the appended block A_j itself
 * (paper-faithful, Alg. 3 appends raw blocks); TRUNC = its
 * rank-r factor U_{j,r} diag(sigma_{j,1..r}) (used for square blocks with
 * n >> r; still an upper bound because F F^T <= A_j A_j^T). */
enum { CMSVD_OPERAND_RAW = 0, CMSVD_OPERAND_TRUNC = 1 };

/* Human-readable name of a status code (static storage). */
const char* cmsvd_status_string(cmsvd_status s);

/* Detail of the last failure on ctx ("" if none); valid until the next call. */
const char* cmsvd_last_error(cmsvd_ctx ctx);

/* Version string of the library build (static storage). */
const char* cmsvd_version(void);

/* Create a context on CUDA device `device`.  `cuda_stream` is a cudaStream_t
 * borrowed from the caller (e.g. torch.cuda.current_stream().cuda_stream) on
 * which all work is enqueued; NULL makes the library create its own
 * non-blocking stream.  *out receives the handle.
 * Errors: CMSVD_E_ARG (out == NULL), CMSVD_E_CUDA (bad device). */
cmsvd_status cmsvd_create(int device, void* cuda_stream, cmsvd_ctx* out);

/* Release every device buffer owned by ctx and the context itself
 * (a library-created stream is destroyed; a borrowed one is not). NULL is a no-op. */
cmsvd_status cmsvd_destroy(cmsvd_ctx ctx);

/* Register (replace) the collection: `count` >= 1 blocks with a common row
 * count m >= 1; block i is n[i] >= 1 columns of fp32, column-major with
 * leading dimension ld[i] >= m (ld may be NULL: all ld[i] = m), at
 * blocks[i].  `where` says whether the block pointers are host or device
 * memory (n, ld and the blocks[] array itself are always host memory).  The
 * library COPIES the data into one packed column-major arena and computes the
 * energies ||A_i||_F^2 in fp64 (S1), rejecting NaN/Inf.  Any previous
 * spectra/cluster state is discarded.
 * Errors: CMSVD_E_ARG, CMSVD_E_SHAPE, CMSVD_E_NONFINITE, CMSVD_E_NOMEM, CMSVD_E_CUDA. */
cmsvd_status cmsvd_register(cmsvd_ctx ctx, int64_t m, int32_t count, const int32_t* n,
                            const float* const* blocks, const int64_t* ld, int where);

/* Per-block spectra for target rank r >= 1 (S2): computes and caches on the
 * device each block's singular values (fp64 internally), left singular
 * vectors, numerical rank (sigma_l > tau * sigma_1, tau = 1e-5, reading A5),
 * the rank-r basis U_r, the full numerical-range basis (residual bound) and
 * the TRUNC operand U_r diag(sigma_r).
 * Host outputs (each may be NULL):
 *   energy[count]   fp64 ||A_i||_F^2
 *   sigma[count*r]  fp32 sigma_1..r(A_i), non-increasing, zero-padded past min(m, n_i)
 *   rank_out[count] numerical rank under tau.
 * Blocks with n_i <= 512 columns (n_i <= m) take the exact fp64 Gram
 * eigendecomposition.  Blocks wider than 512 columns (square/wide weight-like
 * blocks, n_i >= m) follow reading A22: top min(m, 2r, 512)
 * triplets by subspace iteration, range taken as R^m, rank_out = min(m, n_i).
 * Errors: CMSVD_E_STATE (no collection), CMSVD_E_ARG (r < 1), CMSVD_E_SHAPE
 * (unsupported shapes: m < n_i <= 512; 512 < n_i < m; a collection mixing
 * blocks wider than 512 columns with narrower ones; r > 512 on wide blocks),
 * CMSVD_E_NOCONV, CMSVD_E_CUDA, CMSVD_E_NOMEM. */
cmsvd_status cmsvd_block_spectra(cmsvd_ctx ctx, int32_t r, double* energy, float* sigma, int32_t* rank_out);

/* Evaluate P >= 0 candidate merges M = [A_base, F_app] (S3-S9).
 *   pairs[2p] = base block, pairs[2p+1] = appended block (0-based, < count;
 *   base == app is allowed and means [A, A]).  Orientation matters for the
 *   residual and incremental estimates (reading A7).
 *   r must equal the r of the last cmsvd_block_spectra call (else CMSVD_E_STATE).
 *   kinds: bitmask of CMSVD_WEYL | CMSVD_RESIDUAL | CMSVD_INCREMENTAL.
 *   operand: CMSVD_OPERAND_RAW or CMSVD_OPERAND_TRUNC.
 *   where: CMSVD_HOST or CMSVD_DEVICE -- applies to `pairs` and to all outputs.
 * Outputs (caller-allocated; sigma_tilde and mu may be NULL):
 *   err2[3p + {0,1,2}] fp64 predicted squared rank-r error {weyl, residual,
 *                      incremental}, clamped to [0, total[p]]; NaN for kinds
 *                      not requested.  Relative error = sqrt(err2/total).
 *   total[p]           fp64 E_base + E_app.
 *   sigma_tilde[p*r+l] fp32 incremental top-r singular values sigma~ (Cor. 3).
 *   mu[p*r+l]          fp32 residual-bound top-r mu (Thm 2, union of sigma(A_base)
 *                      and sigma((I - Q Q^T) F_app)).
 * P = 0 is a no-op.  Errors: CMSVD_E_ARG, CMSVD_E_SHAPE (pair index out of
 * range), CMSVD_E_STATE, CMSVD_E_NOCONV, CMSVD_E_CUDA, CMSVD_E_NOMEM. */
cmsvd_status cmsvd_pair_errors(cmsvd_ctx ctx, const int32_t* pairs, int64_t P, int32_t r, uint32_t kinds,
                               int operand, int where, double* err2, double* total, float* sigma_tilde,
                               float* mu);

/* Tighter certified variants BEYOND THE PAPER, for the
 * same candidate pairs / operand / where conventions as cmsvd_pair_errors:
 *   err2x[2p + 0] residual bound with the tracked top-r basis U_r of the base
 *                 instead of its full numerical range (reading A4: the
 *                 projector U_r U_r^T + W, W inside range(I - U_r U_r^T),
 *                 carries Thm 2's partial-sum argument);
 *                 mu = top-r of sigma(A_base) U sigma((I - U_r U_r^T) F_app);
 *   err2x[2p + 1] per-index Weyl bound E_i + E_j - sum_{l<=r} max(sigma_l(A_i),
 *                 sigma_l(F_j))^2 (reading A8, from sigma_l(M) >= sigma_l(A_k),
 *                 PAPER.md:1530-1533);
 *   total[p]      E_base + E_app.
 * Both are >= the exact error and <= the paper's residual / Weyl values
 * (chain exact <= incremental <= residual(U_r) <= residual(full) <= Weyl).
 * Errors as cmsvd_pair_errors. */
cmsvd_status cmsvd_pair_errors_tight(cmsvd_ctx ctx, const int32_t* pairs, int64_t P, int32_t r, int operand,
                                     int where, double* err2x, double* total);

/* Cluster verification and compression accounting (
 * PAPER.md:142-173, 579-597).  For the partition assign[count] (cluster ids
 * 0..n_clusters-1, every cluster non-empty; host arrays) and target rank r >= 1:
 *   exact_err2[c] = sum_{j>r} sigma_j^2(M_c) of the explicit concatenation M_c
 *                   of cluster c's blocks in ascending block order (Thm EYM,
 *                   the error of the rank-r truncated SVD
 *                   M_c ~ U_c S_c V_c^T and of the reconstruction Ũ_c V_c,i^T);
 *                   fp64 Gram (min(m, N_c) square) + eigenvalues;
 *   total[c]      = ||M_c||_F^2   (eps_rel = sqrt(exact_err2 / total));
 *   mem[c]        = min(m N_c, r_c (m + N_c)) stored parameters, r_c =
 *                   min(r, m, N_c) (reading A23: a cluster
 *                   is stored raw when that is smaller, cf. Table 2's 1.000*).
 * The compression ratio is sum_i m n_i / sum_c mem[c].
 * Errors: CMSVD_E_STATE (no collection), CMSVD_E_ARG (bad assign / r),
 * CMSVD_E_SHAPE (min(m, N_c) > 4096), CMSVD_E_NOCONV, CMSVD_E_CUDA, CMSVD_E_NOMEM. */
cmsvd_status cmsvd_cluster_verify(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters,
                                  double* exact_err2, double* total, int64_t* mem);

/* cmsvd_cluster_verify plus the derived quantities (any may be NULL): rel[c] = sqrt(exact_err2[c] /
 * total[c]) (0 for a zero-energy cluster; the certificate compares it with eps) and
 * *ratio = sum_i m n_i / sum_c mem[c].  Errors as cmsvd_cluster_verify. */
cmsvd_status cmsvd_cluster_verify_ex(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters,
                                     double* exact_err2, double* total, int64_t* mem, double* rel, double* ratio);

/* The compressed representation of a partition: for each
 * cluster c (ids 0..n_clusters-1 of assign[count], host arrays) the rank-r_c truncated SVD of the
 * concatenation M_c of its blocks in ascending block order, r_c = min(r, m, N_c), stored as
 *   Ũ_c = U_c S_c  (m x r_c, fp32, column-major) at Ut + sum_{c'<c} m r_c', and
 *   V_c            (N_c x r_c, fp32, column-major; rows follow the member blocks' columns)
 *                  at V + sum_{c'<c} N_c' r_c',
 * so that block i of cluster c is reconstructed as Ũ_c V_{c,i}^T; rc[c] = r_c.
 * Directions with sigma <= 1e-5 sigma_1 are returned as zero columns.  The caller allocates
 * Ut (sum_c m r_c floats), V (sum_c N_c r_c floats) and rc (n_clusters); host memory.
 * Errors: as cmsvd_cluster_verify. */
cmsvd_status cmsvd_cluster_factors(cmsvd_ctx ctx, int32_t r, const int32_t* assign, int32_t n_clusters, float* Ut,
                                   float* V, int32_t* rc);

/* Predicted errors of given block sequences -- the estimates of the paper's estimator
 * conservativeness diagnostic (slack Delta = predicted - exact; SURVEY.md
 * §8(f) N2).  Sequence s is ids[offs[s] .. offs[s+1]) (host arrays, non-empty, block ids
 * < count), the blocks in append order.  For each sequence:
 *   err2[3s + 0] Weyl bound, Eq. 5 over its K blocks;
 *   err2[3s + 1] residual bound: Alg. 2's state after appending blocks 2..K to block 1
 *                (Thm 2 / Cor 1);
 *   err2[3s + 2] incremental estimate: Alg. 3's state after the same appends (Lemma 1,
 *                Cor 3, Cor 2);
 *   total[s]     sum of the members' energies.
 * A single block gives its own truncation error for every kind; kinds not requested give
 * NaN.  The exact error of the concatenation comes from cmsvd_cluster_verify.
 * Errors as cmsvd_cluster (CMSVD_E_SHAPE for the residual kind on blocks wider than 512). */
cmsvd_status cmsvd_sequence_errors(cmsvd_ctx ctx, const int32_t* offs, const int32_t* ids, int32_t nseq, int32_t r,
                                   uint32_t kinds, int operand, double* err2, double* total);

/* Greedy clustering (Appendix E). */
enum { CMSVD_ALG_MAX_NORM = 0, CMSVD_ALG_RESIDUAL = 1, CMSVD_ALG_APPROX = 2 };
enum { CMSVD_SORT_FROBENIUS = 0, CMSVD_SORT_RESIDUAL = 1 };

typedef struct {
  int32_t algorithm; /* CMSVD_ALG_* */
  int32_t sort;      /* CMSVD_SORT_* (ignored by MAX_NORM) */
  int32_t knn;       /* candidate window per greedy step, >= 1; 1 = the paper's stop-on-first-rejection */
  int32_t operand;   /* CMSVD_OPERAND_* for appended blocks */
  int32_t r;         /* target rank, >= 1; must equal the last cmsvd_block_spectra r */
  double eps;        /* relative Frobenius tolerance, 0 < eps < 1; accept iff err^2 <= eps^2 * E (inclusive) */
} cmsvd_cluster_opts;

/* Run one greedy clustering on the registered collection.  Host outputs
 * (caller-allocated, count entries each unless stated; any may be NULL):
 *   assign[i]       cluster id of block i (clusters numbered in creation order)
 *   order[i]        position of block i in its cluster's append order
 *   n_clusters      number of clusters K
 *   cluster_err2[c] certificate err^2 of cluster c at close (first K used)
 *   cluster_total[c] energy of cluster c (first K used)
 *   n_evals         tentative merge evaluations performed.
 * Anchors: largest remaining ||A||_F (ties -> smaller id).  Candidates:
 * SORT_FROBENIUS ascending ||A||_F; SORT_RESIDUAL ascending ||(I-QQ^T)A_j||_F
 * against the current state, re-ranked after every accept.  Zero-energy
 * blocks merge unconditionally.
 * Errors: CMSVD_E_ARG, CMSVD_E_STATE, CMSVD_E_NOCONV, CMSVD_E_CUDA, CMSVD_E_NOMEM. */
cmsvd_status cmsvd_cluster(cmsvd_ctx ctx, const cmsvd_cluster_opts* opts, int32_t* assign, int32_t* order,
                           int32_t* n_clusters, double* cluster_err2, double* cluster_total, int64_t* n_evals);

/* Diagnostic: the batched fp64 symmetric eigensolver that yields sigma~^2 from the core Grams (Lemma 1 /
 * Cor. 3), on caller matrices, for parity tests.
 *   count >= 1 problems; problem p is n[p] x n[p] (0 <= n[p] <= nmax <= 4096) at G + p * nmax * nmax,
 *   column-major with leading dimension nmax, symmetric (only the lower triangle is read), host memory;
 *   ev[p * kw + l] = the l-th largest eigenvalue (l < min(kw, n[p])), non-increasing; entries l >= n[p]
 *   are unspecified; trace[p] = sum of the diagonal (may be NULL).  1 <= kw <= nmax.  The dispatch by
 *   size is the pair path's (n <= 160 register/shared-memory kernels, 160 < n <= 512 the two-stage band
 *   reduction; CMSVD_EIG_SBR=0 selects the one-stage in-place kernel) and, for 512 < n <= 4096, the
 *   cluster verification's (the two-stage reduction with the panel and the band in global memory).
 * Errors: CMSVD_E_ARG (NULL pointers, kw out of range), CMSVD_E_SHAPE (n[p] < 0, n[p] > nmax or
 * nmax > 4096), CMSVD_E_CUDA, CMSVD_E_NOMEM. */
cmsvd_status cmsvd_sym_eigvals(cmsvd_ctx ctx, int32_t count, int32_t nmax, const int32_t* n, const double* G,
                               int32_t kw, double* ev, double* trace);

/* Diagnostic: accuracy record of the last cmsvd_block_spectra on blocks wider than 512 columns (reading
 * A22, subspace iteration): the largest Ritz residual ||A A^T u_l - lambda_l u_l|| / lambda_l over the
 * returned l < r (guarded: the call iterates further while it exceeds 1e-4 and fails with CMSVD_E_NOCONV
 * after CMSVD_SUBSPACE_MAX power iterations) and the number of power iterations used.  Both 0 for
 * collections of narrower blocks (exact eigendecompositions).  Either output may be NULL. */
cmsvd_status cmsvd_spectra_diagnostics(cmsvd_ctx ctx, double* max_ritz_residual, int32_t* power_iterations);

/* Number of kernel launches this context has issued since creation (for the
 * bench's gpu_launches accounting). */
int64_t cmsvd_launch_count(cmsvd_ctx ctx);

/* Per-kernel-category timing with CUDA events recorded on the context stream
 * around each launch group (for bench.py's live roofline).  enable != 0
 * resets the accumulators and turns recording on; 0 turns it off. */
cmsvd_status cmsvd_profile_enable(cmsvd_ctx ctx, int enable);

/* Synchronises the context stream, then fills up to `max` categories:
 * names[k] (static strings), ms[k] (summed event time), launches[k] (number
 * of timed launch groups).  Any output may be NULL.  Returns the number of
 * categories written (0 for a NULL context). */
int32_t cmsvd_profile_read(cmsvd_ctx ctx, int32_t max, const char** names, double* ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* CMSVD_H */

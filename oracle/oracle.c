/*
 * oracle.c -- float64 CPU oracle for the merge-error evaluation of
 * arXiv 2601.11626 ("compression-aware clustering of matrices under SVD
 * constraints").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, helper or constant generator with the CUDA
 * path (paper_2601_11626_b200/csrc) and never imports it.
 *
 * Plain, slow, obviously correct: float64 throughout, textbook loops, no
 * blocking.  Each function cites the passage of PAPER.md it follows
 * (PAPER.md:<line>, section / equation).  Readings of ambiguous passages are
 * the SURVEY.md §8(c) readings A1..A21, listed in DESIGN.md.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"):
 *   or_svd          : vs LAPACK (numpy) on random inputs, closed forms
 *                     (identity, rank one, diag), U diag(s) V^T = A.
 *   or_pair_*       : brute-force SVD of the explicit concatenation (exact
 *                     error), Example D.1, Proposition 1 (corrected, A2),
 *                     [A, A] closed forms, untruncated exactness (Cor. 2),
 *                     soundness chain exact <= inc <= res <= weyl (F3, F4),
 *                     the hand-computed TRUNC merge (A6, n > r).
 *   or_sym_eig_topk : 1-D Laplacian closed form under a Haar similarity,
 *                     repeated eigenvalues, diagonal (tests/test_oracle_big_pins.py).
 *   or_block_spectra_big : block built from a known SVD (sigma, U_r), energy
 *                     split P1, LAPACK cross-check, A22 pair closed forms.
 *   or_exact_groups : LAPACK on random groups, union-spectrum closed form.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ENOCONV 5
#define OR_EARG 1

/* ------------------------------------------------------------------ */
/* Frobenius energy, PAPER.md:116-119 (fidelity in Frobenius norm) and   */
/* PAPER.md:1484-1488 (||M||_F^2 = sum_j ||A_j||_F^2).                   */
/* ------------------------------------------------------------------ */
double or_energy_f32(const float* a, int64_t len) {
  double s = 0.0;
  for (int64_t k = 0; k < len; ++k) s += (double)a[k] * (double)a[k];
  return s;
}

double or_energy(const double* a, int64_t len) {
  double s = 0.0;
  for (int64_t k = 0; k < len; ++k) s += a[k] * a[k];
  return s;
}

/* ------------------------------------------------------------------ */
/* Householder QR (textbook, no pivoting; A20).  A is m x n column-major */
/* with m >= n, overwritten: R in the upper triangle, the reflector      */
/* vectors v_k (v_k[k] = 1 implicit) below the diagonal, tau[k].         */
/* ------------------------------------------------------------------ */
static void hh_qr(int64_t m, int64_t n, double* A, int64_t lda, double* tau) {
  for (int64_t k = 0; k < n; ++k) {
    double* col = A + k * lda;
    double norm2 = 0.0;
    for (int64_t i = k; i < m; ++i) norm2 += col[i] * col[i];
    double alpha = col[k];
    double xnorm = sqrt(norm2);
    if (xnorm == 0.0) { tau[k] = 0.0; continue; }
    double beta = (alpha >= 0.0) ? -xnorm : xnorm;   /* new diagonal */
    double v0 = alpha - beta;
    for (int64_t i = k + 1; i < m; ++i) col[i] /= v0;  /* v = x - beta e1, scaled v[k] = 1 */
    tau[k] = (beta - alpha) / beta;
    col[k] = beta;
    /* apply H = I - tau v v^T to the trailing columns */
    for (int64_t j = k + 1; j < n; ++j) {
      double* cj = A + j * lda;
      double d = cj[k];
      for (int64_t i = k + 1; i < m; ++i) d += col[i] * cj[i];
      d *= tau[k];
      cj[k] -= d;
      for (int64_t i = k + 1; i < m; ++i) cj[i] -= d * col[i];
    }
  }
}

/* Thin Q (m x n) from the reflectors stored by hh_qr. */
static void hh_form_q(int64_t m, int64_t n, const double* A, int64_t lda, const double* tau,
                      double* Q, int64_t ldq) {
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  }
  for (int64_t k = n - 1; k >= 0; --k) {
    const double* v = A + k * lda;
    for (int64_t j = 0; j < n; ++j) {
      double* qj = Q + j * ldq;
      double d = qj[k];
      for (int64_t i = k + 1; i < m; ++i) d += v[i] * qj[i];
      d *= tau[k];
      qj[k] -= d;
      for (int64_t i = k + 1; i < m; ++i) qj[i] -= d * v[i];
    }
  }
}

/* ------------------------------------------------------------------ */
/* Cyclic one-sided (Hestenes) Jacobi on the columns of X (p x n).       */
/* Rotate pair (a,b) iff |gamma| > tol * sqrt(alpha*beta) (A19, fp64 tol =  */
/* max(p,8)*eps) and neither column is negligible (norm^2 <= tol^2 ||X||_F^2),*/
/* until a whole sweep rotates nothing.  On exit the columns of X are mutually   */
/* orthogonal: X = U diag(s), and V (n x n, may be NULL) accumulates the */
/* rotations so that X_in V = X_out.                                     */
/* ------------------------------------------------------------------ */
static int jacobi_onesided(int64_t p, int64_t n, double* X, int64_t ldx, double* V, int64_t ldv) {
  /* rounding noise in gamma is ~ p * eps * sqrt(alpha*beta): a fixed 1e-15
     would never be met for p >~ 10, so the threshold is p * DBL_EPSILON. */
  const double tol = (double)(p > 8 ? p : 8) * 2.220446049250313e-16;
  const int max_sweeps = 60;
  if (V) {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) V[i + j * ldv] = (i == j) ? 1.0 : 0.0;
  }
  /* A column whose norm is below tol * ||X||_F is at the rounding level of
     the matrix: its direction is meaningless and rotating it against the
     others never meets the relative criterion (A19).  Such pairs are skipped. */
  double fro2 = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < p; ++i) fro2 += X[i + j * ldx] * X[i + j * ldx];
  const double negligible = tol * tol * fro2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int64_t rotated = 0;
    for (int64_t a = 0; a + 1 < n; ++a) {
      for (int64_t b = a + 1; b < n; ++b) {
        double* xa = X + a * ldx;
        double* xb = X + b * ldx;
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < p; ++i) {
          alpha += xa[i] * xa[i];
          beta += xb[i] * xb[i];
          gamma += xa[i] * xb[i];
        }
        if (gamma == 0.0 || !(fabs(gamma) > tol * sqrt(alpha * beta))) continue;
        if (alpha <= negligible || beta <= negligible) continue;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = c * t;
        for (int64_t i = 0; i < p; ++i) {
          double u = xa[i], w = xb[i];
          xa[i] = c * u - s * w;
          xb[i] = s * u + c * w;
        }
        if (V) {
          double* va = V + a * ldv;
          double* vb = V + b * ldv;
          for (int64_t i = 0; i < n; ++i) {
            double u = va[i], w = vb[i];
            va[i] = c * u - s * w;
            vb[i] = s * u + c * w;
          }
        }
        ++rotated;
      }
    }
    if (rotated == 0) return OR_OK;
  }
  return OR_ENOCONV;
}

/* ------------------------------------------------------------------ */
/* Thin SVD A = U diag(s) V^T of an m x n matrix (any shape), k=min(m,n).*/
/* The truncated SVD whose optimality is Eckart-Young-Mirsky,            */
/* PAPER.md:1211-1238 (Thm 3).  For m > n: Householder QR, then one-sided*/
/* Jacobi on R (n x n), U = Q U_R.  For m < n: SVD of A^T.               */
/* s is sorted non-increasing; U (m x k, ldu) and V (n x k, ldv) may be  */
/* NULL.  A is not modified.                                             */
/* ------------------------------------------------------------------ */
int or_svd(int64_t m, int64_t n, const double* A, int64_t lda, double* s,
           double* U, int64_t ldu, double* V, int64_t ldv) {
  if (m <= 0 || n <= 0) return OR_EARG;
  if (m < n) {
    /* A^T = V diag(s) U^T */
    double* At = (double*)malloc(sizeof(double) * n * m);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) At[j + i * n] = A[i + j * lda];
    int st = or_svd(n, m, At, n, s, V, ldv, U, ldu);
    free(At);
    return st;
  }
  int64_t k = n;
  double* W = (double*)malloc(sizeof(double) * m * n);
  for (int64_t j = 0; j < n; ++j) memcpy(W + j * m, A + j * lda, sizeof(double) * m);
  double* R = (double*)calloc((size_t)(n * n), sizeof(double));
  double* tau = (double*)malloc(sizeof(double) * n);
  double* Q = NULL;
  if (m > n) {
    hh_qr(m, n, W, m, tau);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i <= j; ++i) R[i + j * n] = W[i + j * m];
    if (U) {
      Q = (double*)malloc(sizeof(double) * m * n);
      hh_form_q(m, n, W, m, tau, Q, m);
    }
  } else {
    for (int64_t j = 0; j < n; ++j) memcpy(R + j * n, W + j * m, sizeof(double) * n);
  }
  double* Vl = (double*)malloc(sizeof(double) * n * n);
  int st = jacobi_onesided(n, n, R, n, Vl, n);
  /* singular values = column norms; sort descending (stable on ties). */
  double* nrm = (double*)malloc(sizeof(double) * n);
  int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t j = 0; j < n; ++j) {
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i) t += R[i + j * n] * R[i + j * n];
    nrm[j] = sqrt(t);
    ord[j] = j;
  }
  for (int64_t a = 1; a < n; ++a) {           /* insertion sort, descending */
    int64_t x = ord[a];
    int64_t b = a - 1;
    while (b >= 0 && nrm[ord[b]] < nrm[x]) { ord[b + 1] = ord[b]; --b; }
    ord[b + 1] = x;
  }
  for (int64_t l = 0; l < k; ++l) s[l] = nrm[ord[l]];
  if (V) {
    for (int64_t l = 0; l < k; ++l)
      for (int64_t i = 0; i < n; ++i) V[i + l * ldv] = Vl[i + ord[l] * n];
  }
  if (U) {
    /* U_R column l = R(:,ord[l]) / s_l ; zero singular value -> zero column
       (its direction is arbitrary and carries no energy). */
    for (int64_t l = 0; l < k; ++l) {
      int64_t c = ord[l];
      double inv = (s[l] > 0.0) ? 1.0 / s[l] : 0.0;
      if (m > n) {
        for (int64_t i = 0; i < m; ++i) {
          double t = 0.0;
          for (int64_t q = 0; q < n; ++q) t += Q[i + q * m] * R[q + c * n];
          U[i + l * ldu] = t * inv;
        }
      } else {
        for (int64_t i = 0; i < m; ++i) U[i + l * ldu] = R[i + c * n] * inv;
      }
    }
  }
  free(W); free(R); free(tau); free(Q); free(Vl); free(nrm); free(ord);
  return st;
}

/* Exact optimal rank-r error of an explicit matrix, E_r^2 = sum_{j>r}     */
/* sigma_j^2, PAPER.md:262-265 (Thm 1 statement) / Thm EYM PAPER.md:1232. */
int or_exact_err2(int64_t m, int64_t ncols, const double* M, int64_t ldm, int32_t r, double* out) {
  int64_t k = m < ncols ? m : ncols;
  double* s = (double*)malloc(sizeof(double) * k);
  int st = or_svd(m, ncols, M, ldm, s, NULL, 0, NULL, 0);
  double t = 0.0;
  for (int64_t j = r; j < k; ++j) t += s[j] * s[j];
  *out = t;
  free(s);
  return st;
}

/* ------------------------------------------------------------------ */
/* Pair evaluation: the three merge estimators for M = [A_i, F_j].       */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t m;
  int32_t count;
  const int32_t* n;            /* columns of each block */
  const double* const* A;      /* block i, m x n[i] column-major */
  const double* E;             /* ||A_i||_F^2 */
  const double* const* sig;    /* all min(m,n_i) singular values, non-increasing */
  const double* const* U;      /* left singular vectors, m x min(m,n_i) */
  const int32_t* rank;         /* numerical rank under tau (A5) */
} or_collection;

static double sum_sq_top(const double* s, int64_t len, int64_t r) {
  double t = 0.0;
  for (int64_t l = 0; l < len && l < r; ++l) t += s[l] * s[l];
  return t;
}

static double clamp_err2(double e2, double total) {
  if (e2 < 0.0) return 0.0;
  if (e2 > total) return total;
  return e2;
}

/* Appended operand F_j (A6): RAW = A_j itself (m x n_j); TRUNC = the rank-r
 * factor U_{j,r'} diag(sigma_{j,1..r'}) (m x r'), r' = min(r, rank_j). */
static double* make_operand(const or_collection* c, int32_t j, int32_t r, int operand, int64_t* w) {
  int64_t m = c->m;
  if (operand == 0) {
    *w = c->n[j];
    double* F = (double*)malloc(sizeof(double) * m * (*w));
    memcpy(F, c->A[j], sizeof(double) * m * (*w));
    return F;
  }
  int64_t rr = c->rank[j] < r ? c->rank[j] : r;
  *w = rr;
  double* F = (double*)malloc(sizeof(double) * m * (rr > 0 ? rr : 1));
  for (int64_t l = 0; l < rr; ++l)
    for (int64_t i = 0; i < m; ++i) F[i + l * m] = c->U[j][i + l * m] * c->sig[j][l];
  return F;
}

/* Weyl bound, Thm 1 / Eq. 5 for K = 2 blocks:
 * E_r^2 <= ||A_i||^2 + ||A_j||^2 - max_k sum_{l<=r} sigma_l^2(A_k). */
static double pair_weyl(const or_collection* c, int32_t i, int32_t j, int32_t r) {
  int64_t ki = c->m < c->n[i] ? c->m : c->n[i];
  int64_t kj = c->m < c->n[j] ? c->m : c->n[j];
  double ti = sum_sq_top(c->sig[i], ki, r);
  double tj = sum_sq_top(c->sig[j], kj, r);
  double mx = ti > tj ? ti : tj;
  return c->E[i] + c->E[j] - mx;
}

/* Residual bound, Thm 2 + Cor 1 / Eq. 6 for the
 * 2-block sequence (A_i, F_j): Q = full numerical range basis of A_i (A4/A5),
 * R = (I - Q Q^T) F_j with one re-orthogonalisation pass,
 * mu = top-r of the multiset sigma(A_i) U sigma(R) (proof Step 5,
 * PAPER.md:1694-1706), err^2 = E_i + E_j - sum_{l<=r} mu_l^2.  Only the
 * partial-sum form of Thm 2 is used (A1). */
static int pair_residual_q(const or_collection* c, int32_t i, const double* F, int64_t w,
                           double Ej, int32_t r, int64_t q, double* err2, double* mu_out);
static int pair_residual(const or_collection* c, int32_t i, const double* F, int64_t w,
                         double Ej, int32_t r, double* err2, double* mu_out) {
  return pair_residual_q(c, i, F, w, Ej, r, c->rank[i], err2, mu_out);
}

/* Thm 2 residual with the first q left singular vectors of the base as the
 * projection basis: q = rank (paper-literal, A4) or q = min(r, rank) (the
 * tracked-basis variant beyond the paper, N3). */
static int pair_residual_q(const or_collection* c, int32_t i, const double* F, int64_t w,
                           double Ej, int32_t r, int64_t q, double* err2, double* mu_out) {
  int64_t m = c->m;
  const double* Q = c->U[i];
  double* R = (double*)malloc(sizeof(double) * m * w);
  memcpy(R, F, sizeof(double) * m * w);
  double* Z = (double*)malloc(sizeof(double) * (q > 0 ? q : 1) * w);
  /* q >= m: Q spans R^m (A22 blocks), Q Q^T = I and R = 0 exactly */
  if (q >= m) memset(R, 0, sizeof(double) * m * w);
  for (int pass = 0; pass < 2 && q < m; ++pass) {
    for (int64_t b = 0; b < w; ++b)
      for (int64_t a = 0; a < q; ++a) {
        double t = 0.0;
        for (int64_t k = 0; k < m; ++k) t += Q[k + a * m] * R[k + b * m];
        Z[a + b * q] = t;
      }
    for (int64_t b = 0; b < w; ++b)
      for (int64_t k = 0; k < m; ++k) {
        double t = 0.0;
        for (int64_t a = 0; a < q; ++a) t += Q[k + a * m] * Z[a + b * q];
        R[k + b * m] -= t;
      }
  }
  int64_t kr = q >= m ? 0 : (m < w ? m : w);
  double* sr = (double*)malloc(sizeof(double) * (kr > 0 ? kr : 1));
  int st = OR_OK;
  if (kr > 0) st = or_svd(m, w, R, m, sr, NULL, 0, NULL, 0);
  /* merge the two non-increasing lists, keep the top r */
  int64_t ki = m < c->n[i] ? m : c->n[i];
  const double* si = c->sig[i];
  int64_t a = 0, b = 0;
  double top = 0.0;
  for (int32_t l = 0; l < r; ++l) {
    double v;
    if (a < ki && (b >= kr || si[a] >= sr[b])) v = si[a++];
    else if (b < kr) v = sr[b++];
    else v = 0.0;
    if (mu_out) mu_out[l] = v;
    top += v * v;
  }
  *err2 = c->E[i] + Ej - top;
  free(R); free(Z); free(sr);
  return st;
}

/* Incremental plug-in estimate, Lemma 1 + Cor 3 + Cor 2 (PAPER.md:1297-1338,
 * 1395-1436, 522-531), written as its plain definition: the tracked state of
 * the base block after truncation to rank r is U_r diag(sigma_r) (Cor 3:
 * Q~ = Q U_r, S~ = Lambda_r), and appending F_j gives the Gram
 * [U_r S_r, F_j][U_r S_r, F_j]^T (Lemma 1, exact), so
 * sigma~ = top-r singular values of the explicit m x (r'+w) matrix
 * [U_r diag(sigma_r), F_j], and err^2 = E_i + E_j - sum_{l<=r} sigma~_l^2. */
static int pair_incremental(const or_collection* c, int32_t i, const double* F, int64_t w,
                            double Ej, int32_t r, double* err2, double* st_out) {
  int64_t m = c->m;
  int64_t ri = c->rank[i] < r ? c->rank[i] : r;
  int64_t nc = ri + w;
  double* X = (double*)malloc(sizeof(double) * m * nc);
  for (int64_t l = 0; l < ri; ++l)
    for (int64_t k = 0; k < m; ++k) X[k + l * m] = c->U[i][k + l * m] * c->sig[i][l];
  memcpy(X + ri * m, F, sizeof(double) * m * w);
  int64_t kk = m < nc ? m : nc;
  double* s = (double*)malloc(sizeof(double) * kk);
  int st = or_svd(m, nc, X, m, s, NULL, 0, NULL, 0);
  double top = 0.0;
  for (int32_t l = 0; l < r; ++l) {
    double v = (l < kk) ? s[l] : 0.0;
    if (st_out) st_out[l] = v;
    top += v * v;
  }
  *err2 = c->E[i] + Ej - top;
  free(X); free(s);
  return st;
}

/* Batched pair evaluation (OpenMP over independent pairs).
 * kinds bitmask: 1 weyl, 2 residual, 4 incremental; not requested -> NaN.
 * err2[3p + {0,1,2}], total[p], sigma_tilde[p*r + l], mu[p*r + l] (may be NULL).
 * Final clamp to [0, total] (A9, S9). */
int or_pair_errors(int64_t m, int32_t count, const int32_t* n, const double* const* A,
                   const double* E, const double* const* sig, const double* const* U,
                   const int32_t* rank, const int32_t* pairs, int64_t P, int32_t r,
                   uint32_t kinds, int operand, double* err2, double* total,
                   double* sigma_tilde, double* mu) {
  or_collection c = {m, count, n, A, E, sig, U, rank};
  int status = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t p = 0; p < P; ++p) {
    int32_t i = pairs[2 * p], j = pairs[2 * p + 1];
    int64_t w = 0;
    double* F = make_operand(&c, j, r, operand, &w);
    double Ej = E[j];
    double tot = E[i] + Ej;
    total[p] = tot;
    double e;
    err2[3 * p + 0] = NAN;
    err2[3 * p + 1] = NAN;
    err2[3 * p + 2] = NAN;
    if (kinds & 1u) err2[3 * p + 0] = clamp_err2(pair_weyl(&c, i, j, r), tot);
    if (kinds & 2u) {
      int st = pair_residual(&c, i, F, w, Ej, r, &e, mu ? mu + p * r : NULL);
      err2[3 * p + 1] = clamp_err2(e, tot);
      if (st) status = st;
    }
    if (kinds & 4u) {
      int st = pair_incremental(&c, i, F, w, Ej, r, &e, sigma_tilde ? sigma_tilde + p * r : NULL);
      err2[3 * p + 2] = clamp_err2(e, tot);
      if (st) status = st;
    }
    free(F);
  }
  return status;
}

/* Beyond the paper: err2x[2p] = residual bound with the tracked
 * basis U_r (q = min(r, rank_i), reading A4), err2x[2p+1] = per-index Weyl
 * bound E_i + E_j - sum_{l<=r} max(sigma_l(A_i), sigma_l(F_j))^2 (reading A8,
 * from sigma_l(M) >= sigma_l(A_k)), both clamped. */
int or_pair_errors_tight(int64_t m, int32_t count, const int32_t* n, const double* const* A,
                         const double* E, const double* const* sig, const double* const* U,
                         const int32_t* rank, const int32_t* pairs, int64_t P, int32_t r,
                         int operand, double* err2x, double* total) {
  or_collection c = {m, count, n, A, E, sig, U, rank};
  int status = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t p = 0; p < P; ++p) {
    int32_t i = pairs[2 * p], j = pairs[2 * p + 1];
    int64_t w = 0;
    double* F = make_operand(&c, j, r, operand, &w);
    double Ej = E[j];
    double tot = E[i] + Ej;
    total[p] = tot;
    int64_t q = rank[i] < r ? rank[i] : r;
    double e;
    int st = pair_residual_q(&c, i, F, w, Ej, r, q, &e, NULL);
    err2x[2 * p] = clamp_err2(e, tot);
    if (st) status = st;
    /* per-index Weyl on the two blocks' spectra (as Eq. 5's implementation, pair_weyl, for either operand) */
    int64_t ki = m < n[i] ? m : n[i];
    int64_t kj = m < n[j] ? m : n[j];
    double top = 0.0;
    for (int32_t l = 0; l < r; ++l) {
      double si = l < ki ? sig[i][l] : 0.0;
      double sj = l < kj ? sig[j][l] : 0.0;
      double mx = si > sj ? si : sj;
      top += mx * mx;
    }
    err2x[2 * p + 1] = clamp_err2(E[i] + Ej - top, tot);
    free(F);
  }
  return status;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Batched block spectra: or_svd per block (OpenMP over blocks). sig_k gets
 * min(m,n_i) values, U_k gets m x min(m,n_i) (caller-allocated). */
int or_block_svds(int64_t m, int32_t count, const int32_t* n, const double* const* A,
                  double* const* sig, double* const* U) {
  int status = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t i = 0; i < count; ++i) {
    int64_t k = m < n[i] ? m : n[i];
    int st = or_svd(m, n[i], A[i], m, sig[i], U ? U[i] : NULL, m, NULL, 0);
    (void)k;
    if (st) status = st;
  }
  return status;
}

/* ------------------------------------------------------------------ */
/* Spectra of blocks wider than 512 columns (configs 3 and 4, reading A15 */
/* / A22): the exact route of A15, written as the textbook algorithms.    */
/*   1. Gram G = A A^T (m x m, fp64 sums of exact fp32 products);          */
/*   2. Householder tridiagonalisation Q^T G Q = T (Golub & Van Loan,       */
/*      "Householder tridiagonalization": p = beta G22 v,                   */
/*      w = p - (beta p^T v / 2) v, G22 <- G22 - v w^T - w v^T), reflectors  */
/*      kept;                                                              */
/*   3. every eigenvalue of T by bisection on Sturm counts (the number of   */
/*      negative pivots of T - x I);                                        */
/*   4. the top-k eigenvectors by inverse iteration on T - lambda I         */
/*      (Gaussian elimination with partial pivoting, 3 iterations) with     */
/*      full Gram-Schmidt re-orthogonalisation against the vectors already */
/*      found, then back-transformed by the reflectors (u = Q y).           */
/* sigma_l = sqrt(max(lambda_l, 0)): A A^T = U diag(sigma^2) U^T, so the    */
/* left singular vectors of A are the eigenvectors of G (Thm EYM's SVD,     */
/* PAPER.md:1211-1238).  Squaring costs (sigma_1/sigma_l)^2 * 1e-16         */
/* relative accuracy only (A15).  OpenMP over rows / columns inside each    */
/* loop (the loop bodies are the textbook ones).                            */
/* ------------------------------------------------------------------ */

/* number of eigenvalues of the symmetric tridiagonal (d, e) below x */
static int64_t sturm_count(int64_t n, const double* d, const double* e, double x, double pivmin) {
  int64_t cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int64_t i = 1; i < n; ++i) {
    q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

/* Solve (T - x I) y = b in place (b -> y) by Gaussian elimination with
   partial pivoting on the tridiagonal (the eliminated matrix has two
   superdiagonals); zero pivots are replaced by pivmin. */
static void tri_solve_shifted(int64_t n, const double* d, const double* e, double x, double pivmin,
                              double* b, double* w /* 3n scratch */) {
  double* u0 = w;           /* diagonal of U */
  double* u1 = w + n;       /* first superdiagonal */
  double* u2 = w + 2 * n;   /* second superdiagonal (fill-in from row swaps) */
  /* working rows: row i = (a_i, b_i, c_i) at columns (i, i+1, i+2) */
  double a = d[0] - x, bb = n > 1 ? e[0] : 0.0, c = 0.0;
  for (int64_t i = 0; i < n - 1; ++i) {
    /* next row: (e_i, d_{i+1} - x, e_{i+1}) at columns (i, i+1, i+2) */
    double na = e[i], nb = d[i + 1] - x, nc = (i + 2 < n) ? e[i + 1] : 0.0;
    if (fabs(na) > fabs(a)) {       /* swap rows */
      double ta = a, tb = bb, tc = c;
      a = na; bb = nb; c = nc;
      na = ta; nb = tb; nc = tc;
      double tmp = b[i]; b[i] = b[i + 1]; b[i + 1] = tmp;
    }
    if (fabs(a) < pivmin) a = (a < 0.0 ? -pivmin : pivmin);
    double l = na / a;
    u0[i] = a; u1[i] = bb; u2[i] = c;
    b[i + 1] -= l * b[i];
    /* the remaining row after elimination starts at column i+1 */
    a = nb - l * bb;
    bb = nc - l * c;
    c = 0.0;
  }
  if (fabs(a) < pivmin) a = (a < 0.0 ? -pivmin : pivmin);
  u0[n - 1] = a; u1[n - 1] = 0.0; u2[n - 1] = 0.0;
  /* back substitution */
  for (int64_t i = n - 1; i >= 0; --i) {
    double t = b[i];
    if (i + 1 < n) t -= u1[i] * b[i + 1];
    if (i + 2 < n) t -= u2[i] * b[i + 2];
    b[i] = t / u0[i];
  }
}

/* Symmetric eigen-decomposition of the m x m matrix G (column-major, full
   storage; destroyed).  lam[m] = all eigenvalues, non-increasing;
   V (m x k, ldv) = eigenvectors of the top k (k <= m). */
int or_sym_eig_topk(int64_t m, double* G, int64_t ldg, int64_t k, double* lam, double* V, int64_t ldv) {
  if (m <= 0 || k < 0 || k > m) return OR_EARG;
  double* d = (double*)malloc(sizeof(double) * m);
  double* e = (double*)calloc((size_t)(m > 1 ? m : 1), sizeof(double));
  double* beta = (double*)calloc((size_t)(m > 1 ? m : 1), sizeof(double));
  double* p = (double*)malloc(sizeof(double) * m);
  /* 2. tridiagonalisation; reflector j (j = 0..m-3) acts on rows j+1..m-1 and
     is stored in G(j+1:m, j) with v[j+1] = 1 implicit */
  for (int64_t j = 0; j + 2 < m; ++j) {
    double* x = G + j * ldg;           /* column j, rows j+1..m-1 */
    const int64_t n2 = m - j - 1;
    double sig2 = 0.0;
    for (int64_t i = j + 2; i < m; ++i) sig2 += x[i] * x[i];
    double alpha = x[j + 1];
    if (sig2 == 0.0) {                  /* already tridiagonal in this column */
      beta[j] = 0.0;
      d[j] = G[j + j * ldg];
      e[j] = alpha;
      continue;
    }
    double mu = sqrt(alpha * alpha + sig2);
    double v0 = alpha <= 0.0 ? alpha - mu : -sig2 / (alpha + mu);   /* GVL Alg. 5.1.1 */
    double b = 2.0 * v0 * v0 / (sig2 + v0 * v0);
    for (int64_t i = j + 2; i < m; ++i) x[i] /= v0;
    x[j + 1] = 1.0;
    beta[j] = b;
    d[j] = G[j + j * ldg];
    e[j] = mu;                          /* (I - b v v^T) x = mu e_1 */
    const double* v = x + j + 1;        /* length n2 */
    /* p = b * G22 v  (G22 = G(j+1:m, j+1:m), symmetric: row i = column i) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n2; ++i) {
      const double* gi = G + (j + 1 + i) * ldg + j + 1;
      double t = 0.0;
      for (int64_t l = 0; l < n2; ++l) t += gi[l] * v[l];
      p[i] = b * t;
    }
    double pv = 0.0;
    for (int64_t i = 0; i < n2; ++i) pv += p[i] * v[i];
    const double half = 0.5 * b * pv;
    for (int64_t i = 0; i < n2; ++i) p[i] -= half * v[i];          /* p := w */
    /* G22 <- G22 - v w^T - w v^T */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n2; ++c) {
      double* gc = G + (j + 1 + c) * ldg + j + 1;
      const double vc = v[c], wc = p[c];
      for (int64_t i = 0; i < n2; ++i) gc[i] -= v[i] * wc + p[i] * vc;
    }
  }
  if (m >= 2) {
    d[m - 2] = G[(m - 2) + (m - 2) * ldg];
    e[m - 2] = G[(m - 1) + (m - 2) * ldg];
  }
  d[m - 1] = G[(m - 1) + (m - 1) * ldg];
  /* 3. bisection for every eigenvalue inside the Gershgorin interval */
  double lo = d[0], hi = d[0], tnorm = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
    if (d[i] - rad < lo) lo = d[i] - rad;
    if (d[i] + rad > hi) hi = d[i] + rad;
    if (fabs(d[i]) + rad > tnorm) tnorm = fabs(d[i]) + rad;
  }
  const double pivmin = 1e-300 + 2.2250738585072014e-308 * (tnorm > 1.0 ? tnorm : 1.0);
  const double eps = 2.220446049250313e-16;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t l = 0; l < m; ++l) {
    /* lam[l] = the (l+1)-th largest = the eigenvalue with m-1-l eigenvalues below it */
    const int64_t below = m - 1 - l;
    double a = lo - eps * tnorm, bnd = hi + eps * tnorm;
    /* to 2 ulps relative, or 1e-3 ulp of ||T|| absolute (the Gram route's own accuracy is ~ulp ||T||) */
    for (int it = 0;
         it < 200 && bnd - a > 2.0 * eps * (fabs(a) > fabs(bnd) ? fabs(a) : fabs(bnd)) + 1e-3 * eps * tnorm + pivmin;
         ++it) {
      double mid = 0.5 * (a + bnd);
      if (sturm_count(m, d, e, mid, pivmin) > below) bnd = mid;
      else a = mid;
    }
    lam[l] = 0.5 * (a + bnd);
  }
  /* 4. inverse iteration for the top k eigenvectors of T, re-orthogonalised */
  double* Y = (double*)calloc((size_t)(m * (k > 0 ? k : 1)), sizeof(double));
  double* scratch = (double*)malloc(sizeof(double) * 4 * m);
  for (int64_t l = 0; l < k; ++l) {
    double* y = Y + l * m;
    for (int64_t i = 0; i < m; ++i) y[i] = 1.0 + 0.5 * sin((double)(i + 1) * (double)(l + 7) * 0.7317);
    /* shift perturbed by a few ulps of ||T|| so that T - x I stays solvable */
    const double x = lam[l] + 4.0 * eps * tnorm;
    for (int it = 0; it < 3; ++it) {
      tri_solve_shifted(m, d, e, x, eps * tnorm, y, scratch);
      for (int64_t q = 0; q < l; ++q) {                 /* Gram-Schmidt against earlier vectors */
        const double* yq = Y + q * m;
        double t = 0.0;
        for (int64_t i = 0; i < m; ++i) t += yq[i] * y[i];
        for (int64_t i = 0; i < m; ++i) y[i] -= t * yq[i];
      }
      double nrm = 0.0;
      for (int64_t i = 0; i < m; ++i) nrm += y[i] * y[i];
      nrm = sqrt(nrm);
      for (int64_t i = 0; i < m; ++i) y[i] /= nrm;
    }
  }
  /* back-transformation u = H_0 H_1 ... H_{m-3} y, applied from the last reflector */
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t l = 0; l < k; ++l) {
    double* y = Y + l * m;
    for (int64_t j = m - 3; j >= 0; --j) {
      if (beta[j] == 0.0) continue;
      const double* v = G + j * ldg + j + 1;   /* v[0] = 1 stored */
      double t = 0.0;
      for (int64_t i = 0; i < m - j - 1; ++i) t += v[i] * y[j + 1 + i];
      t *= beta[j];
      for (int64_t i = 0; i < m - j - 1; ++i) y[j + 1 + i] -= t * v[i];
    }
    for (int64_t i = 0; i < m; ++i) V[i + l * ldv] = y[i];
  }
  free(d); free(e); free(beta); free(p); free(Y); free(scratch);
  return OR_OK;
}

/* Spectra of one block A (m x n, fp32 column-major, n >= m) by the Gram
   route above: sig[m] = sqrt(max(lambda, 0)) non-increasing, U (m x k) the
   left singular vectors of the top k. */
int or_block_spectra_big(int64_t m, int64_t n, const float* A, int64_t k, double* sig, double* U) {
  double* G = (double*)malloc(sizeof(double) * m * m);
  if (!G) return OR_EARG;
  /* 1. G = A A^T: G_ij = sum_c A_ic A_jc (A column-major: row i is strided), via A^T rows */
  double* At = (double*)malloc(sizeof(double) * m * n);     /* At[c + i*n] = A[i + c*m] */
  if (!At) { free(G); return OR_EARG; }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t c = 0; c < n; ++c) At[c + i * n] = (double)A[i + c * m];
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t j = 0; j < m; ++j) {
    const double* aj = At + j * n;
    for (int64_t i = j; i < m; ++i) {
      const double* ai = At + i * n;
      double t = 0.0;
      for (int64_t c = 0; c < n; ++c) t += ai[c] * aj[c];
      G[i + j * m] = t;
      G[j + i * m] = t;
    }
  }
  free(At);
  double* lam = (double*)malloc(sizeof(double) * m);
  int st = or_sym_eig_topk(m, G, m, k, lam, U, m);
  for (int64_t l = 0; l < m; ++l) sig[l] = sqrt(lam[l] > 0.0 ? lam[l] : 0.0);
  free(lam);
  free(G);
  return st;
}

/* Batched explicit-concatenation exact errors for tiny inputs:
 * groups given as CSR (offs[g]..offs[g+1]) of block ids. */
int or_exact_groups(int64_t m, const int32_t* n, const double* const* A, const int32_t* offs,
                    const int32_t* ids, int32_t G, int32_t r, double* out) {
  int status = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t g = 0; g < G; ++g) {
    int64_t nc = 0;
    for (int32_t t = offs[g]; t < offs[g + 1]; ++t) nc += n[ids[t]];
    double* M = (double*)malloc(sizeof(double) * m * nc);
    int64_t col = 0;
    for (int32_t t = offs[g]; t < offs[g + 1]; ++t) {
      memcpy(M + col * m, A[ids[t]], sizeof(double) * m * n[ids[t]]);
      col += n[ids[t]];
    }
    int st;
    const int64_t dim = m < nc ? m : nc;
    if (dim <= 512) {
      st = or_exact_err2(m, nc, M, m, r, out + g);
    } else {
      /* wide concatenations (reading A15): the smaller fp64 Gram, G = M M^T (m <= nc) or M^T M, and its
         eigenvalues by the tridiagonalisation + bisection of or_sym_eig_topk; E_r^2 = sum_{j>r} lambda_j */
      double* G = (double*)malloc(sizeof(double) * dim * dim);
      for (int64_t a = 0; a < dim; ++a)
        for (int64_t b = 0; b <= a; ++b) {
          double t = 0.0;
          if (m <= nc)
            for (int64_t c2 = 0; c2 < nc; ++c2) t += M[a + c2 * m] * M[b + c2 * m];
          else
            for (int64_t i = 0; i < m; ++i) t += M[i + a * m] * M[i + b * m];
          G[a + b * dim] = t;
          G[b + a * dim] = t;
        }
      double* lam = (double*)malloc(sizeof(double) * dim);
      st = or_sym_eig_topk(dim, G, dim, 0, lam, NULL, dim);
      double t = 0.0;
      for (int64_t j = dim - 1; j >= r; --j) t += lam[j] > 0.0 ? lam[j] : 0.0;
      out[g] = t;
      free(lam);
      free(G);
    }
    if (st) status = st;
    free(M);
  }
  return status;
}

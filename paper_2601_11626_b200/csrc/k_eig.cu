// k_eig.cu -- batched small symmetric eigensolvers in fp64, one CTA per
// problem, matrix staged in shared memory.
//
//  * k_syev_jacobi  : eigenvalues AND eigenvectors (cyclic two-sided Jacobi,
//                     parallel round-robin ordering).  Used where vectors are
//                     needed: block spectra (S2: A^T A = V diag(sigma^2) V^T,
//                     U = A V / sigma) and cluster-state commits (S10).
//  * k_tridiag_topk : values only -- Householder tridiagonalisation followed by
//                     Sturm-count multisection for the top-k eigenvalues
//                     (optionally only those above a threshold).  Used per
//                     candidate pair on the Gram of the incremental core
//                     (Lemma 1 / Cor. 3: sigma~^2 = eigenvalues of S_{t+1},
//                     PAPER.md:1325-1338, 1399-1436) and on the residual Gram
//                     R'^T R' (Thm 2: sigma(R) for the mu multiset).
// Both are fp64: the bounds subtract captured energy from total energy, so
// eigenvalue errors must be small relative to ||G|| * 1e-9.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "engine.h"

namespace cmsvd {

// fp64 reciprocal: MUFU.RCP64H approximation + 2 Newton steps (full precision
// for |q| >= pivmin, far cheaper than the IEEE division subroutine).
// (the approximation is good to ~1e-6; one cubic step y (1 + e + e^2), e = 1 - q y, reaches 1 ulp with
// three dependent operations instead of the four of two Newton steps -- measured: tools/rcp_prec.cu)
__device__ __forceinline__ double rcp_nr(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  const double e = fma(-q, y, 1.0);
  return fma(y * e, 1.0 + e, y);
}
// 1/sqrt(x): MUFU approximation (~1e-6) + one cubic step y (1 + e/2 + 3e^2/8), e = 1 - x y^2: full double
// precision in four dependent operations instead of six (tools/rsqrt_prec.cu)
__device__ __forceinline__ double rsqrt_cubic(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ double div_fast(double a, double b) { return a * rcp_nr(b); }
__device__ __forceinline__ float div_fast(float a, float b) { return __fdividef(a, b); }

// Sturm-count pivot clamp and sign test in the integer domain (the IEEE bit order of |q| is its
// magnitude order; after the clamp |q| >= pivmin > 0, so the sign bit is q < 0): the same results as
// fabs(q) < pivmin ? -pivmin : q and q < 0.0, off the fp64 pipe.
__device__ __forceinline__ double sturm_clamp(double q, unsigned long long pivbits, double negpiv) {
  unsigned hi = (unsigned)__double2hiint(q), lo = (unsigned)__double2loint(q);
  asm("lop3.b32 %0, %0, 0x7FFFFFFF, 0, 0xc0;" : "+r"(hi));  // |q| bits (a plain & becomes an fp64 abs)
  return (((unsigned long long)hi << 32) | lo) < pivbits ? negpiv : q;
}
// Reciprocal for the Sturm recurrences: the MUFU seed y, e = 1 - q y, 1/q = y (1 + e + e^2) in three
// dependent fp64 operations (the e^3 term is below the rounding of the result)
__device__ __forceinline__ double rcp_sturm(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  const double e = fma(-q, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ int sturm_neg(double q) { return (int)((unsigned)__double2hiint(q) >> 31); }

template <typename T>
__device__ __forceinline__ void sturm2(const T* __restrict__ d, const T* __restrict__ e2, int n, T x0, T x1,
                                       T pivmin, int& c0, int& c1) {
  T q0 = d[0] - x0, q1 = d[0] - x1;
  if (fabs(q0) < pivmin) q0 = -pivmin;
  if (fabs(q1) < pivmin) q1 = -pivmin;
  int a0 = q0 < T(0), a1 = q1 < T(0);
#pragma unroll 4
  for (int i = 1; i < n; ++i) {
    const T di = d[i], ei = e2[i - 1];
    q0 = (di - x0) - div_fast(ei, q0);
    q1 = (di - x1) - div_fast(ei, q1);
    if (fabs(q0) < pivmin) q0 = -pivmin;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    a0 += q0 < T(0);
    a1 += q1 < T(0);
  }
  c0 = a0;
  c1 = a1;
}

// ---------------------------------------------------------------------------
// Batched Householder tridiagonalisation (values path).
// Problem p: n = ns[p] (0 <= n <= 256), symmetric matrix at Gin + p*stride_in
// (ld_in, full storage).  Staged in shared memory (full storage, ld = n):
// 200 KB at n = 160, one CTA of 8 warps per SM.
// Step k applies reflector k's rank-2 update to the trailing matrix and, in
// the same pass, accumulates the product with reflector k+1 (which only needs
// the already-updated column k+1): warp per column, lanes over rows, a
// compile-time number of 32-row chunks per step (no predicated-off work
// except the last chunk), per-warp row partials combined in fixed order.
// Outputs per problem: d[n], e2[n-1] (squared sub-diagonal), trace, and
// Gershgorin data gsh[4] = {lo, hi, pivmin, norm}; cnt = min(kw, #eig > thr).
// ---------------------------------------------------------------------------
#ifndef CMSVD_TRI_WARPS
#define CMSVD_TRI_WARPS 8
#endif
constexpr int kTriWarps = CMSVD_TRI_WARPS;
#ifndef CMSVD_QL_BATCH
#define CMSVD_QL_BATCH 16   // columns of Z per load batch of the in-place QL rotation sweep (k_syev_ql<true>)
#endif
constexpr int kTriThreads = 32 * kTriWarps;
constexpr int kTriMax = 512;      // up to 16 row chunks of 32 lanes (n > 160: matrix in global memory)
constexpr int kEigSmemMax = 160;  // largest n staged entirely in shared memory

__device__ __forceinline__ double block_sum8(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < kTriWarps; ++k) t += red[k];  // fixed order, every thread
  return t;
}

// One fused pass over the LOWER triangle of the trailing block B (rows/cols 0..m-1, column-major, ld;
// the strictly upper part is never read or written), for the row segment [r0, r0 + 32 NT):
//   if UPD: B -= v w^T + w v^T   (v, w indexed with offset `off`)
//   part[wid][i] = sum_{j in this warp's columns, j <= i} B_new[i][j] u[j]      (row partials)
//   cpart[j]     = sum_{i > j} B_new[i][j] u[i]                                  (mirrored, one warp per column)
// so that (B_new u)_i = sum_wid part[wid][i] + cpart[i]; dpart[wid] = this warp's share of u^T B_new u.
// Segments after the first accumulate into cpart / dpart (same warp, fixed order).  NC columns of a
// warp are processed per iteration: all their loads are issued before any store so that they overlap
// (the compiler cannot reorder loads across stores itself); NC = 4 keeps more global loads in flight
// for the in-place (n > 160) reduction.
template <int NT, bool UPD, int NC = 2>
__device__ __forceinline__ void tri_pass(double* __restrict__ B, int ld, int m, const double* __restrict__ u,
                                         const double* __restrict__ vv, const double* __restrict__ ww, int off,
                                         double* __restrict__ part, int n, double* __restrict__ dpart,
                                         double* __restrict__ cpart, int r0, bool first) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[NT], vi[NT], wi[NT], ui[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int i = r0 + lane + 32 * t;
    const bool ok = i < m;
    acc[t] = 0.0;
    vi[t] = (UPD && ok) ? vv[off + i] : 0.0;
    wi[t] = (UPD && ok) ? ww[off + i] : 0.0;
    ui[t] = ok ? u[i] : 0.0;
  }
  const int jend = min(m, r0 + 32 * NT);  // columns with rows in this segment
  double cdot = 0.0;  // sum over this warp's columns of (this segment's) cpart[j] u[j]
  auto put = [&](int j, double c) {
    if (lane == 0) cpart[j] = first ? c : cpart[j] + c;
  };
  int j = wid;
  for (; j + (NC - 1) * kTriWarps < jend; j += NC * kTriWarps) {
    double uj[NC], vj[NC], wj[NC], x[NC][NT], c[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int jq = j + q * kTriWarps;
      uj[q] = u[jq];
      vj[q] = UPD ? vv[off + jq] : 0.0;
      wj[q] = UPD ? ww[off + jq] : 0.0;
      const double* __restrict__ col = B + jq * ld;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = r0 + lane + 32 * t;
        x[q][t] = (i < m && i >= jq) ? col[i] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int jq = j + q * kTriWarps;
      double* __restrict__ col = B + jq * ld;
      c[q] = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = r0 + lane + 32 * t;
        if (i < m && i >= jq) {
          if (UPD) {
            x[q][t] = fma(-vi[t], wj[q], x[q][t]);
            x[q][t] = fma(-wi[t], vj[q], x[q][t]);
            col[i] = x[q][t];
          }
          acc[t] = fma(x[q][t], uj[q], acc[t]);
          if (i > jq) c[q] = fma(x[q][t], ui[t], c[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      c[q] = warp_sum(c[q]);
      put(j + q * kTriWarps, c[q]);
      cdot = fma(c[q], uj[q], cdot);
    }
  }
  for (; j < jend; j += kTriWarps) {
    const double uj = u[j];
    double vj = 0.0, wj = 0.0;
    if (UPD) { vj = vv[off + j]; wj = ww[off + j]; }
    double* __restrict__ col = B + j * ld;
    double c0 = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = r0 + lane + 32 * t;
      if (i < m && i >= j) {
        double xx = col[i];
        if (UPD) {
          xx = fma(-vi[t], wj, xx);
          xx = fma(-wi[t], vj, xx);
          col[i] = xx;
        }
        acc[t] = fma(xx, uj, acc[t]);
        if (i > j) c0 = fma(xx, ui[t], c0);
      }
    }
    c0 = warp_sum(c0);
    put(j, c0);
    cdot = fma(c0, uj, cdot);
  }
  // columns of this warp beyond the segment have no rows here: the first segment still defines cpart
  if (first)
    for (int jj = j; jj < m; jj += kTriWarps)
      if (lane == 0) cpart[jj] = 0.0;
  double dw = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int i = r0 + lane + 32 * t;
    if (i < m) {
      part[wid * n + i] = acc[t];
      dw = fma(acc[t], ui[t], dw);
    }
  }
  dw = warp_sum(dw);
  if (lane == 0) dpart[wid] = first ? dw + cdot : dpart[wid] + dw + cdot;
}

#ifndef CMSVD_GL_NT
#define CMSVD_GL_NT 4
#endif
#ifndef CMSVD_GL_CTAS
#define CMSVD_GL_CTAS 2
#endif
#ifndef CMSVD_GL_NC
#define CMSVD_GL_NC 4
#endif
template <bool UPD>
__device__ __forceinline__ void tri_pass_dispatch(double* B, int ld, int m, const double* u, const double* vv,
                                                  const double* ww, int off, double* part, int n, double* dpart,
                                                  double* cpart) {
  switch ((m + 31) >> 5) {
    case 0: break;
    case 1: tri_pass<1, UPD>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, 0, true); break;
    case 2: tri_pass<2, UPD>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, 0, true); break;
    case 3: tri_pass<3, UPD>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, 0, true); break;
    case 4: tri_pass<4, UPD>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, 0, true); break;
    case 5: tri_pass<5, UPD>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, 0, true); break;
    default:  // n > 160 (in place in global memory): row segments of 32 GL_NT rows, GL_NC columns in flight per warp
      for (int r0 = 0; r0 < m; r0 += 32 * CMSVD_GL_NT)
        tri_pass<CMSVD_GL_NT, UPD, CMSVD_GL_NC>(B, ld, m, u, vv, ww, off, part, n, dpart, cpart, r0, r0 == 0);
      break;
  }
}

// Householder reduction of the n x n symmetric matrix A (shared memory, full
// storage, ld) to tridiagonal form; e2[k] = squared sub-diagonal.  With SAVE,
// reflector k (v_k, 1 at local 0, rows k+1..n-1) is written to column k of VH
// (n x n, global), tau_k to tauH[k] and the signed sub-diagonal beta_k to esg[k].
template <bool SAVE>
__device__ __forceinline__ void tri_reduce(double* __restrict__ A, int n, int ld, double* vA, double* vB,
                                           double* __restrict__ w, double* __restrict__ part,
                                           double* __restrict__ e2, double* __restrict__ esg,
                                           double* __restrict__ VH, double* __restrict__ tauH) {
  __shared__ double s_dot[kTriWarps], s_nrm[kTriWarps];
  __shared__ double cpart[kTriMax];  // mirrored column partials of the lower-triangle passes
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // Per step (3 barriers): [all warps] fused update + product pass, each warp
  // also reduces its partial dot p.v2 -> | [all threads, redundantly] K from the
  // 8 partial dots; per row p, w and the update of column k+1; per-warp partial
  // norms of the next column -> | [all threads, redundantly] next reflector
  // scalars from the 8 partial norms; per row v2 -> next pass.  No block-wide
  // serial reduction chain.
  auto rsqrt_nr = [](double x) { return rsqrt_cubic(x); };
  // next reflector from column kk (rows kk+1..), given the partial norms of rows kk+2.. in s_nrm
  auto reflector = [&](int kk, double* vec) -> double {
    const int s = n - 1 - kk;
    const double* x = A + kk * ld + (kk + 1);
    double sig2 = 0.0;
#pragma unroll
    for (int q = 0; q < kTriWarps; ++q) sig2 += s_nrm[q];
    const double alpha = x[0];
    double tau, scale, ee;
    if (sig2 == 0.0) {
      tau = 0.0; scale = 0.0; ee = alpha * alpha;
    } else {
      const double x2 = fma(alpha, alpha, sig2);
      const double xn = x2 * rsqrt_nr(x2);
      const double beta = alpha >= 0.0 ? -xn : xn;
      tau = (beta - alpha) * rcp_nr(beta);
      scale = rcp_nr(alpha - beta);
      ee = beta * beta;
    }
    if (tid == 0) {
      e2[kk] = ee;
      if (SAVE) { esg[kk] = (sig2 == 0.0) ? alpha : -copysign(1.0, alpha) * sqrt(ee); tauH[kk] = tau; }
    }
    for (int i = tid; i < s; i += kTriThreads) {
      const double vi = (i == 0) ? 1.0 : x[i] * scale;
      vec[i] = vi;
      if (SAVE) VH[(int64_t)kk * n + kk + 1 + i] = vi;
    }
    return tau;
  };
  auto partial_norm = [&](const double* x, int s) {  // sum_{i>=1} x[i]^2 over this thread's rows, warp-reduced
    double prt = 0.0;
    for (int i = 1 + tid; i < s; i += kTriThreads) prt = fma(x[i], x[i], prt);
    prt = warp_sum(prt);
    if (lane == 0) s_nrm[wid] = prt;
  };
  if (n >= 3) {
    double* v = vA;
    double* v2 = vB;
    partial_norm(A + 1, n - 1);
    __syncthreads();
    double tau = reflector(0, v);
    __syncthreads();
    tri_pass_dispatch<false>(A + 1 * ld + 1, ld, n - 1, v, nullptr, nullptr, 0, part, n, s_dot, cpart);
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
      const int s = n - 1 - k;  // trailing size of step k (rows/cols k+1..n-1)
      double dsum = 0.0;
#pragma unroll
      for (int q = 0; q < kTriWarps; ++q) dsum += s_dot[q];
      const double Kc = 0.5 * tau * tau * dsum;  // (tau/2) p.v with p = tau * sum(part)
      double p0 = cpart[0];
#pragma unroll
      for (int q = 0; q < kTriWarps; ++q) p0 += part[q * n];
      p0 *= tau;
      const double w0 = p0 - Kc;  // v[0] = 1
      double* c0 = A + (k + 1) * ld + (k + 1);
      double prt = 0.0;
      for (int i = tid; i < s; i += kTriThreads) {
        double pi = cpart[i];
#pragma unroll
        for (int q = 0; q < kTriWarps; ++q) pi += part[q * n + i];
        pi *= tau;
        const double wi = pi - Kc * v[i];
        w[i] = wi;
        double ci = c0[i];
        if (tau != 0.0) {
          ci = fma(-v[i], w0, ci - wi);
          c0[i] = ci;
        }
        if (i >= 2) prt = fma(ci, ci, prt);
      }
      prt = warp_sum(prt);
      if (lane == 0) s_nrm[wid] = prt;
      __syncthreads();
      const double tau2 = reflector(k + 1, v2);
      __syncthreads();
      // fused: update trailing (local 1..s-1) and partial products with v2
      if (tau != 0.0) tri_pass_dispatch<true>(c0 + ld + 1, ld, s - 1, v2, v, w, 1, part, n, s_dot, cpart);
      else tri_pass_dispatch<false>(c0 + ld + 1, ld, s - 1, v2, v, w, 1, part, n, s_dot, cpart);
      __syncthreads();
      double* tmp = v; v = v2; v2 = tmp;
      tau = tau2;
    }
  }
}

// GL = true: the matrix is reduced in place in global memory (L2-resident; n up to 512), only the
// vectors and partial sums live in shared memory.
template <bool GL>
__global__ void __launch_bounds__(kTriThreads, GL ? CMSVD_GL_CTAS : 1) k_tridiag(const double* __restrict__ Gin, int64_t ld_in,
                                                            int64_t stride_in, const int* __restrict__ ns,
                                                            const double* __restrict__ thr, int kw, int nstride,
                                                            double* __restrict__ dout, double* __restrict__ e2out,
                                                            double* __restrict__ gsh, int* __restrict__ cnt_out,
                                                            double* __restrict__ trace_out) {
  extern __shared__ double sm[];
  const int p = blockIdx.x;
  const int n = ns[p];
  const int ld = GL ? (int)ld_in : n;
  double* __restrict__ A = GL ? const_cast<double*>(Gin) + (int64_t)p * stride_in : sm;  // column-major
  double* vA = GL ? sm : A + n * ld;                    // reflector buffers (ping-pong)
  double* vB = vA + n;
  double* __restrict__ w = vB + n;
  double* __restrict__ pp = w + n;                      // tau * A v of the current reflector
  double* __restrict__ e2 = pp + n;
  double* __restrict__ part = e2 + n;                   // kTriWarps x n row-partials
  double* __restrict__ d = part;                        // aliases part at the end
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* Gp = Gin + (int64_t)p * stride_in;
  double* dO = dout + (int64_t)p * nstride;
  double* eO = e2out + (int64_t)p * nstride;
  if (n <= 0) {
    if (tid == 0) { cnt_out[p] = 0; trace_out[p] = 0.0; gsh[4 * p] = 0; gsh[4 * p + 1] = 0; gsh[4 * p + 2] = 1e-300; gsh[4 * p + 3] = 1e-300; }
    return;
  }
  if (!GL) {
    for (int j = wid; j < n; j += kTriWarps) {
      const double* src = Gp + (int64_t)j * ld_in;
      double* dst = A + j * ld;
      for (int i = lane; i < n; i += 32) dst[i] = src[i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += A[(int64_t)i * ld + i];
    trace_out[p] = s;
  }
  tri_reduce<false>(A, n, ld, vA, vB, w, part, e2, nullptr, nullptr, nullptr);
  if (tid == 0 && n >= 2 && n < 3) {
    const double t = A[(int64_t)(n - 2) * ld + (n - 1)];
    e2[n - 2] = t * t;
  }
  __syncthreads();
  for (int i = tid; i < n; i += kTriThreads) {
    const double di = A[(int64_t)i * ld + i];
    d[i] = di;
    dO[i] = di;
    if (i + 1 < n) eO[i] = e2[i];
  }
  __syncthreads();
  if (tid == 0) {
    double glo = 1e300, ghi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      double r = 0.0;
      if (i > 0) r += sqrt(e2[i - 1]);
      if (i + 1 < n) r += sqrt(e2[i]);
      glo = fmin(glo, d[i] - r);
      ghi = fmax(ghi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    const double nrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
    glo -= 2.2e-16 * nrm * n + pivmin;
    ghi += 2.2e-16 * nrm * n + pivmin;
    gsh[4 * p] = glo; gsh[4 * p + 1] = ghi; gsh[4 * p + 2] = pivmin; gsh[4 * p + 3] = nrm;
    int above = n;
    if (thr) {
      const double t = thr[p];
      if (t >= ghi) above = 0;
      else if (t > glo) {
        int c0, c1;
        sturm2<double>(d, e2, n, t, t, pivmin, c0, c1);
        above = n - c0;
      }
    }
    cnt_out[p] = min(kw, above);
  }
}

// ---------------------------------------------------------------------------
// Register-resident Householder tridiagonalisation (values path), n <= 32*S.
// The lower triangle of the matrix lives in the register file of one CTA of
// 16 warps: thread (lane, warp) holds A(i, j) for rows i = lane + 32 s and
// columns j = warp + 16 c, for the chunks (s, c) that meet the lower triangle
// (16 c <= 32 s + 31; 30 doubles per thread at n = 160).  The 32 x 32
// diagonal blocks (c = 2s, 2s+1) are stored in full, so every stored element
// contributes a_ij v_j to p_i and only the strictly-lower chunks (c < 2s) add
// the mirrored a_ij v_i to p_j: no per-element masks.  Per reflector k:
//   [B2] row partials of A v_k (shared memory), mirrored column partials
//        (lane butterfly) and v^T A v partials are in -> per row
//        p = tau A v, w = p - (tau/2)(p.v) v (zero for rows <= k)
//   the warp owning column k+1 waits (named barrier) for those rows only,
//        forms the updated column k+1 in temporaries and builds reflector
//        k+1 while the other warps head to
//   [B3] -> one fused pass over the registers: rank-2 update with (v_k, w_k)
//        and the products with v_{k+1} (-> B2).
// Passes are specialised at compile time on the first live column chunk
// k/16 (finished chunks cost nothing).  No matrix traffic through shared
// memory; same outputs as k_tridiag.
// ---------------------------------------------------------------------------
#ifdef CMSVD_RR_PROF
__device__ unsigned long long g_rr_prof[8];
#define RR_T(slot, cond) do { if ((cond) && blockIdx.x == 0) { unsigned long long _t = clock64(); if (lane == 0) atomicAdd(&g_rr_prof[slot], _t - t_last); } t_last = clock64(); } while (0)
#else
#define RR_T(slot, cond) do { } while (0)
#endif
constexpr int kRRWarps = 16;
constexpr int kRRThreads = 32 * kRRWarps;

__host__ __device__ constexpr bool rr_present(int s, int c) { return 16 * c <= 32 * s + 31; }
__host__ __device__ constexpr bool rr_lower(int s, int c) { return 16 * c + 15 < 32 * s; }  // strictly below
__host__ __device__ constexpr int rr_pow2(int x) { return x <= 1 ? 1 : x <= 2 ? 2 : x <= 4 ? 4 : x <= 8 ? 8 : 16; }

// One pass over the live chunks (column chunks c >= KC, row chunks s >= KC/2):
// UPD: a -= v w^T + w v^T;  MV: row partials of a u -> part[wid], mirrored
// column partials -> cs (butterfly over lanes), u^T a u partial -> red[wid].
// Matrix storage policies of the register-resident kernels: the chunks of one problem live either in
// the thread's registers (RegAcc) or, for a second problem sharing the CTA, in shared memory with the
// same ownership (SmemAcc: present chunk q of thread t at A[q * kRRThreads + t], conflict-free).
template <int S, int C>
struct RegAcc {
  double (&a)[S][C];
  __device__ __forceinline__ double ld(int s, int c) const { return a[s][c]; }
  __device__ __forceinline__ void st(int s, int c, double x) const { a[s][c] = x; }
};
template <int S, int C>
__host__ __device__ constexpr int rr_qidx(int s, int c) {  // ordinal of present chunk (s, c), row-major
  int q = 0;
  for (int s2 = 0; s2 < S; ++s2)
    for (int c2 = 0; c2 < C; ++c2) {
      if (s2 == s && c2 == c) return q;
      if (16 * c2 <= 32 * s2 + 31) ++q;
    }
  return q;
}
template <int S, int C>
__host__ __device__ constexpr int rr_nchunks() { return rr_qidx<S, C>(S, 0); }
template <int S, int C>
struct SmemAcc {
  double* A;   // this thread's column: A + tid
  __device__ __forceinline__ double ld(int s, int c) const { return A[rr_qidx<S, C>(s, c) * kRRThreads]; }
  __device__ __forceinline__ void st(int s, int c, double x) const { A[rr_qidx<S, C>(s, c) * kRRThreads] = x; }
};

// Split storage (two-problem kernel at n = 160): the last NQR present chunks (the longest-lived, row-major
// ordinals >= NQ - NQR) in registers, the others in shared memory like SmemAcc.
template <int S, int C, int NQR>
struct HybAcc {
  static constexpr int NQS = rr_nchunks<S, C>() - NQR;
  double (&a)[S][C];
  double* A;   // this thread's column of the shared-memory part: A + tid
  __device__ __forceinline__ double ld(int s, int c) const {
    return rr_qidx<S, C>(s, c) >= NQS ? a[s][c] : A[rr_qidx<S, C>(s, c) * kRRThreads];
  }
  __device__ __forceinline__ void st(int s, int c, double x) const {
    if (rr_qidx<S, C>(s, c) >= NQS) a[s][c] = x;
    else A[rr_qidx<S, C>(s, c) * kRRThreads] = x;
  }
};

template <int S, int C, int KC, bool UPD, bool MV, class ACC>
__device__ __forceinline__ void rr_pass(ACC a, const int lane, const int wid,
                                        const double* __restrict__ v, const double* __restrict__ w,
                                        const double* __restrict__ u, double* __restrict__ part,
                                        double* __restrict__ cs, double* __restrict__ red, const int pub_j,
                                        double* __restrict__ colbuf) {
  constexpr int NR = 32 * S;
  constexpr int CL = 2 * (S - 1);
  constexpr int C2 = rr_pow2(CL);
  constexpr int S0 = KC / 2;
  double vi[S], wi[S], ui[S], pr[S], pc[C2];
#pragma unroll
  for (int s = S0; s < S; ++s) {
    const int i = lane + 32 * s;
    if (UPD) { vi[s] = v[i]; wi[s] = w[i]; }
    if (MV) { ui[s] = u[i]; pr[s] = 0.0; }
  }
#pragma unroll
  for (int c = 0; c < C2; ++c) pc[c] = 0.0;
  double dd = 0.0;
#pragma unroll
  for (int c = KC; c < C; ++c) {
    const int j = wid + 16 * c;
    double vj = 0.0, wj = 0.0, uj = 0.0;
    if (UPD) { vj = v[j]; wj = w[j]; }
    if (MV) uj = u[j];
#pragma unroll
    for (int s = S0; s < S; ++s)
      if (rr_present(s, c)) {
        double x = a.ld(s, c);
        if (UPD) {
          x = fma(-vi[s], wj, fma(-wi[s], vj, x));
          a.st(s, c, x);
        }
        if (MV) {
          pr[s] = fma(x, uj, pr[s]);
          if (rr_lower(s, c)) pc[c] = fma(x, ui[s], pc[c]);
        }
      }
    if (j == pub_j) {  // this warp owns the column the next reflector is built from: publish it
#pragma unroll
      for (int s = S0; s < S; ++s)
        if (rr_present(s, c)) colbuf[lane + 32 * s] = a.ld(s, c);
    }
    if (MV && c < CL) dd = fma(uj, pc[c], dd);
  }
  if constexpr (MV) {
#pragma unroll
  for (int s = S0; s < S; ++s) dd = fma(ui[s], pr[s], dd);
  if (CL > 0) {  // recursive-halving butterfly: lane ends with the sum of chunk lane >> (5 - log2 C2)
    int cnt = C2;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      if (cnt > 1) {
        const int half = cnt >> 1;
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < C2 / 2; ++q)
          if (q < half) {
            const double send = hi ? pc[q] : pc[q + half];
            const double keep = hi ? pc[q + half] : pc[q];
            pc[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        cnt = half;
      } else {
        pc[0] += __shfl_xor_sync(0xffffffffu, pc[0], o);
      }
    }
    constexpr int sh = (C2 == 1) ? 5 : (C2 == 2) ? 4 : (C2 == 4) ? 3 : (C2 == 8) ? 2 : 1;
    const int c = lane >> sh;
    if ((lane & ((1 << sh) - 1)) == 0 && c < CL) cs[wid + 16 * c] = pc[0];
  }
#pragma unroll
  for (int s = S0; s < S; ++s) part[wid * NR + lane + 32 * s] = pr[s];
  dd = warp_sum(dd);
  if (lane == 0) red[wid] = dd;
  }
}

template <int S, int C, bool UPD, bool MV, class ACC>
__device__ __forceinline__ void rr_pass_kc(int kc, ACC a, const int lane, const int wid,
                                           const double* v, const double* w, const double* u, double* part,
                                           double* cs, double* red, int pub_j, double* colbuf) {
#define RR_CASE(K)                                                                                           \
  case K:                                                                                                    \
    if (K < C) rr_pass<S, C, (K < C ? K : 0), UPD, MV, ACC>(a, lane, wid, v, w, u, part, cs, red, pub_j, colbuf); \
    break;
  switch (kc) {
    RR_CASE(0) RR_CASE(1) RR_CASE(2) RR_CASE(3) RR_CASE(4) RR_CASE(5) RR_CASE(6) RR_CASE(7)
    RR_CASE(8) RR_CASE(9) RR_CASE(10) RR_CASE(11) RR_CASE(12) RR_CASE(13) RR_CASE(14) RR_CASE(15)
    default: break;
  }
#undef RR_CASE
}

// fixed-order pairwise sum of 16 values x[q * stride]
__device__ __forceinline__ double tree16(const double* x, int stride) {
  double t[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) t[q] = x[q * stride] + x[(q + 8) * stride];
#pragma unroll
  for (int q = 0; q < 4; ++q) t[q] += t[q + 4];
  t[0] += t[2];
  t[1] += t[3];
  return t[0] + t[1];
}

template <int S, int C, class ACC>
__device__ __forceinline__ void rr_column(int ck, ACC a, double* x) {
#pragma unroll
  for (int s = 0; s < S; ++s) x[s] = 0.0;
#define RR_COL(K)                                                      \
  case K:                                                              \
    _Pragma("unroll") for (int s = 0; s < S; ++s) if (K < C && rr_present(s, K)) x[s] = a.ld(s, K < C ? K : 0); \
    break;
  switch (ck) {
    RR_COL(0) RR_COL(1) RR_COL(2) RR_COL(3) RR_COL(4) RR_COL(5) RR_COL(6) RR_COL(7)
    RR_COL(8) RR_COL(9) RR_COL(10) RR_COL(11) RR_COL(12) RR_COL(13) RR_COL(14) RR_COL(15)
    default: break;
  }
#undef RR_COL
}

template <int S, int C>
__global__ void __launch_bounds__(kRRThreads, (S <= 3 ? 2 : 1)) k_tridiag_rr(const double* __restrict__ Gin, int64_t ld_in,
                                                              int64_t stride_in, const int* __restrict__ ns,
                                                              const double* __restrict__ thr, int kw, int nstride,
                                                              double* __restrict__ dout, double* __restrict__ e2out,
                                                              double* __restrict__ gsh, int* __restrict__ cnt_out,
                                                              double* __restrict__ trace_out,
                                                              double* __restrict__ save_base = nullptr,
                                                              int64_t save_stride = 0) {
  // save (optional; problem p at save_base + p * save_stride): [v_k as column k of an n x n array][tau_k]
  // [signed e_k], so that Q^T G Q = tridiag(d, e) with Q = H_0 ... H_{n-3}, H_k = I - tau_k v_k v_k^T
  double* const save = save_base ? save_base + (int64_t)blockIdx.x * save_stride : nullptr;
  constexpr int NR = 32 * S;
  constexpr int CL = 2 * (S - 1);
  static_assert(C == 2 * S && C <= 16, "column chunks");
  __shared__ double vb[2][NR], wb[NR], part[kRRWarps * NR], cs[NR], ds[NR], e2s[NR], colbuf[NR];
  __shared__ double red[kRRWarps], red2[S], s_tau[2], s_alpha, s_dk;
  const int p = blockIdx.x;
  const int n = ns[p];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* Gp = Gin + (int64_t)p * stride_in;
  double* dO = dout + (int64_t)p * nstride;
  double* eO = e2out + (int64_t)p * nstride;
  if (n <= 0) {
    if (tid == 0) { cnt_out[p] = 0; trace_out[p] = 0.0; gsh[4 * p] = 0; gsh[4 * p + 1] = 0; gsh[4 * p + 2] = 1e-300; gsh[4 * p + 3] = 1e-300; }
    return;
  }
  double a_[S][C];
  const RegAcc<S, C> a{a_};
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (rr_present(s, c)) {
        const int i = lane + 32 * s, j = wid + 16 * c;
        a_[s][c] = (i < n && j < n) ? Gp[(int64_t)j * ld_in + i] : 0.0;
      }
  if (wid == 0) {
    double t = 0.0;
    for (int i = lane; i < n; i += 32) t += Gp[(int64_t)i * ld_in + i];
    t = warp_sum(t);
    if (lane == 0) trace_out[p] = t;
  }
  auto rsqrt_nr = [](double x) { return rsqrt_cubic(x); };
  // reflector from the (updated) column kk held as x[s] = A(lane + 32 s, kk) by its owner warp:
  // e2[kk], d[kk], tau -> s_tau[kk & 1], v -> vb[kk & 1]
  auto reflector = [&](int kk, const double* x) {
    double sg = 0.0, al = 0.0, dk = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      if (i > kk + 1 && i < n) sg = fma(x[s], x[s], sg);
      if (i == kk + 1) al = x[s];
      if (i == kk) dk = x[s];
    }
    sg = warp_sum(sg);
    al = __shfl_sync(0xffffffffu, al, (kk + 1) & 31);
    dk = __shfl_sync(0xffffffffu, dk, kk & 31);
    double tau, scale, ee, es;
    if (sg == 0.0) {
      tau = 0.0; scale = 0.0; ee = al * al; es = al;
    } else {
      const double x2 = fma(al, al, sg);
      const double xn = x2 * rsqrt_nr(x2);
      const double beta = al >= 0.0 ? -xn : xn;
      tau = (beta - al) * rcp_nr(beta);
      scale = rcp_nr(al - beta);
      ee = beta * beta; es = beta;
    }
    if (lane == 0) { e2s[kk] = ee; ds[kk] = dk; s_tau[kk & 1] = tau; }
    if (save && lane == 0) { save[(int64_t)n * n + kk] = tau; save[(int64_t)n * n + n + kk] = es; }
    double* vv = vb[kk & 1];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      vv[i] = (i == kk + 1) ? 1.0 : ((i > kk + 1 && i < n) ? x[s] * scale : 0.0);
      if (save && i < n) save[(int64_t)kk * n + i] = vv[i];
    }
  };
  // columns without strictly-lower parts (the last two chunks) never get a mirrored sum
  for (int j = 16 * CL + tid; j < NR; j += kRRThreads) cs[j] = 0.0;
#ifdef CMSVD_RR_PROF
  unsigned long long t_last = clock64();
#endif
  if (n >= 3) {
    if (wid == 0) {
      double x[S];
      rr_column<S, C, RegAcc<S, C>>(0, a, x);
      reflector(0, x);
    }
    __syncthreads();
    // products with v_0; publish column 1 (reflector 1 is formed in the row phase of step 0)
    if (s_tau[0] != 0.0) rr_pass<S, C, 0, false, true, RegAcc<S, C>>(a, lane, wid, nullptr, nullptr, vb[0], part, cs, red, 1, colbuf);
    else rr_pass<S, C, 0, false, false, RegAcc<S, C>>(a, lane, wid, nullptr, nullptr, nullptr, part, cs, red, 1, colbuf);
    for (int k = 0; k + 2 < n; ++k) {
      const double* v = vb[k & 1];
      const double tau = s_tau[k & 1];
      const int k1 = k + 1;
      const bool more = k1 + 2 < n;  // reflector k+1 exists
      RR_T(0, wid == 1);
      __syncthreads();  // B2: part, cs, red of A v_k; colbuf = column k+1 (before step k's update)
      RR_T(1, wid == 1);
      // Row phase (warps 0..S-1, thread t = row t): w_t, and -- instead of a single owner warp -- the
      // updated column k+1 (same fma order as the register update), its norm and reflector k+1.
      if (tid < NR) {
        const double Kc = 0.5 * tau * tau * tree16(red, 1);
        const double pt = cs[tid] + tree16(&part[tid], NR);
        const double wt = (tid > k && tid < n && tau != 0.0) ? fma(tau, pt, -Kc * v[tid]) : 0.0;
        wb[tid] = wt;
        if (more) {
          double y = colbuf[tid];
          if (tau != 0.0) {
            const double pk1 = cs[k1] + tree16(&part[k1], NR);
            const double wk1 = fma(tau, pk1, -Kc * v[k1]);
            y = fma(-v[tid], wk1, fma(-wt, v[k1], y));
          }
          double sq = (tid > k1 + 1 && tid < n) ? y * y : 0.0;
          sq = warp_sum(sq);
          if (lane == 0) red2[wid] = sq;
          if (tid == k1 + 1) s_alpha = y;
          if (tid == k1) s_dk = y;
          asm volatile("bar.sync 1, %0;" ::"r"(NR) : "memory");  // row warps only
          double sg = 0.0;
#pragma unroll
          for (int q = 0; q < S; ++q) sg += red2[q];
          const double al = s_alpha;
          double tau1, scale, ee, es;
          if (sg == 0.0) {
            tau1 = 0.0; scale = 0.0; ee = al * al; es = al;
          } else {
            const double x2 = fma(al, al, sg);
            const double xn = x2 * rsqrt_nr(x2);
            const double beta = al >= 0.0 ? -xn : xn;
            tau1 = (beta - al) * rcp_nr(beta);
            scale = rcp_nr(al - beta);
            ee = beta * beta; es = beta;
          }
          if (tid == 0) { e2s[k1] = ee; ds[k1] = s_dk; s_tau[k1 & 1] = tau1; }
          const double vt = (tid == k1 + 1) ? 1.0 : ((tid > k1 + 1 && tid < n) ? y * scale : 0.0);
          vb[k1 & 1][tid] = vt;
          if (save) {
            if (tid < n) save[(int64_t)k1 * n + tid] = vt;
            if (tid == 0) { save[(int64_t)n * n + k1] = tau1; save[(int64_t)n * n + n + k1] = es; }
          }
        }
      }
      RR_T(6, wid == 1);
      __syncthreads();  // B3: w_k, v_{k+1}
      RR_T(7, wid == 1);
      const bool mv = more && s_tau[k1 & 1] != 0.0;
      const double* u = vb[k1 & 1];
      const int pub = (k + 3 < n) ? k + 2 : -1;  // column of reflector k+2
      if (tau != 0.0 && mv) rr_pass_kc<S, C, true, true, RegAcc<S, C>>(k >> 4, a, lane, wid, v, wb, u, part, cs, red, pub, colbuf);
      else if (tau != 0.0) rr_pass<S, C, 0, true, false, RegAcc<S, C>>(a, lane, wid, v, wb, nullptr, part, cs, red, pub, colbuf);
      else if (mv) rr_pass<S, C, 0, false, true, RegAcc<S, C>>(a, lane, wid, nullptr, nullptr, u, part, cs, red, pub, colbuf);
      else rr_pass<S, C, 0, false, false, RegAcc<S, C>>(a, lane, wid, nullptr, nullptr, nullptr, part, cs, red, pub, colbuf);
    }
  }
  __syncthreads();
  // trailing 2x2 (or n <= 2): d[n-2], d[n-1], e2[n-2]
  {
    const int lo = n >= 2 ? n - 2 : 0;
    for (int jj = lo; jj < n; ++jj) {
      if (wid == (jj & 15)) {
        double x[S];
        rr_column<S, C, RegAcc<S, C>>(jj >> 4, a, x);
        double dj = 0.0, ej = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const int i = lane + 32 * s;
          if (i == jj) dj = x[s];
          if (i == jj + 1) ej = x[s];
        }
        dj = __shfl_sync(0xffffffffu, dj, jj & 31);
        ej = __shfl_sync(0xffffffffu, ej, (jj + 1) & 31);
        if (lane == 0) {
          ds[jj] = dj;
          if (jj + 1 < n) e2s[jj] = ej * ej;
          if (save && jj + 1 < n) save[(int64_t)n * n + n + jj] = ej;
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += kRRThreads) {
    dO[i] = ds[i];
    if (i + 1 < n) eO[i] = e2s[i];
  }
  if (tid == 0) {
    const double* d = ds;
    const double* e2 = e2s;
    double glo = 1e300, ghi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      double r = 0.0;
      if (i > 0) r += sqrt(e2[i - 1]);
      if (i + 1 < n) r += sqrt(e2[i]);
      glo = fmin(glo, d[i] - r);
      ghi = fmax(ghi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    const double nrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
    glo -= 2.2e-16 * nrm * n + pivmin;
    ghi += 2.2e-16 * nrm * n + pivmin;
    gsh[4 * p] = glo; gsh[4 * p + 1] = ghi; gsh[4 * p + 2] = pivmin; gsh[4 * p + 3] = nrm;
    int above = n;
    if (thr) {
      const double t = thr[p];
      if (t >= ghi) above = 0;
      else if (t > glo) {
        int c0, c1;
        sturm2<double>(d, e2, n, t, t, pivmin, c0, c1);
        above = n - c0;
      }
    }
    cnt_out[p] = min(kw, above);
  }
}

template <int S>
struct RRProb {
  double vb[2][32 * S], wb[32 * S], part[kRRWarps * 32 * S], cs[32 * S], ds[32 * S], e2s[32 * S],
      colbuf[32 * S];
  double red[kRRWarps], red2[S], s_tau[2], s_alpha, s_dk;
  unsigned long long bar2, bar3;
};

__device__ __forceinline__ void rr_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void rr_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void rr_mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "RRW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra RRW_%=;\n\t"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ double rr_rsqrt_nr(double x) { return rsqrt_cubic(x); }

// reflector kk from the column held as x[s] = A(lane + 32 s, kk) by one warp (prologue, kk = 0)
template <int S>
__device__ __forceinline__ void rr_reflector_warp(RRProb<S>& P, int kk, const double* x, int n, int lane) {
  double sg = 0.0, al = 0.0, dk = 0.0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    if (i > kk + 1 && i < n) sg = fma(x[s], x[s], sg);
    if (i == kk + 1) al = x[s];
    if (i == kk) dk = x[s];
  }
  sg = warp_sum(sg);
  al = __shfl_sync(0xffffffffu, al, (kk + 1) & 31);
  dk = __shfl_sync(0xffffffffu, dk, kk & 31);
  double tau, scale, ee;
  if (sg == 0.0) {
    tau = 0.0; scale = 0.0; ee = al * al;
  } else {
    const double x2 = fma(al, al, sg);
    const double xn = x2 * rr_rsqrt_nr(x2);
    const double beta = al >= 0.0 ? -xn : xn;
    tau = (beta - al) * rcp_nr(beta);
    scale = rcp_nr(al - beta);
    ee = beta * beta;
  }
  if (lane == 0) { P.e2s[kk] = ee; P.ds[kk] = dk; P.s_tau[kk & 1] = tau; }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    P.vb[kk & 1][i] = (i == kk + 1) ? 1.0 : ((i > kk + 1 && i < n) ? x[s] * scale : 0.0);
  }
}

// row phase of step k on the row threads t0 = 0..32RW-1 (warps wr = 0..RW-1 of the group; thread t0 owns
// rows t0 + 32 RW j); bar_id = the group's named barrier for the norm.  RW = S: one row per thread.
template <int S, int RW = S>
__device__ __forceinline__ void rr_row_phase(RRProb<S>& P, int k, int n, int t0, int wr, int lane, int bar_id) {
  constexpr int NR = 32 * S;
  constexpr int RT = 32 * RW;
  constexpr int NRT = (NR + RT - 1) / RT;
  const double* v = P.vb[k & 1];
  const double tau = P.s_tau[k & 1];
  const int k1 = k + 1;
  const bool more = k1 + 2 < n;
  const double Kc = 0.5 * tau * tau * tree16(P.red, 1);
  double wk1 = 0.0;
  if (more && tau != 0.0) {
    const double pk1 = P.cs[k1] + tree16(&P.part[k1], NR);
    wk1 = fma(tau, pk1, -Kc * v[k1]);
  }
  double y[NRT];
  double sq = 0.0;
#pragma unroll
  for (int j = 0; j < NRT; ++j) {
    const int t = t0 + RT * j;
    y[j] = 0.0;
    if (NR % RT == 0 || t < NR) {
      const double pt = P.cs[t] + tree16(&P.part[t], NR);
      const double wt = (t > k && t < n && tau != 0.0) ? fma(tau, pt, -Kc * v[t]) : 0.0;
      P.wb[t] = wt;
      if (more) {
        double yy = P.colbuf[t];
        if (tau != 0.0) yy = fma(-v[t], wk1, fma(-wt, v[k1], yy));
        y[j] = yy;
        if (t > k1 + 1 && t < n) {
          if (j == 0) sq = yy * yy;
          else sq = fma(yy, yy, sq);
        }
        if (t == k1 + 1) P.s_alpha = yy;
        if (t == k1) P.s_dk = yy;
      }
    }
  }
  if (more) {
    sq = warp_sum(sq);
    if (lane == 0) P.red2[wr] = sq;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(RT) : "memory");
    double sg = 0.0;
#pragma unroll
    for (int q = 0; q < RW; ++q) sg += P.red2[q];
    const double al = P.s_alpha;
    double tau1, scale, ee;
    if (sg == 0.0) {
      tau1 = 0.0; scale = 0.0; ee = al * al;
    } else {
      const double x2 = fma(al, al, sg);
      const double xn = x2 * rr_rsqrt_nr(x2);
      const double beta = al >= 0.0 ? -xn : xn;
      tau1 = (beta - al) * rcp_nr(beta);
      scale = rcp_nr(al - beta);
      ee = beta * beta;
    }
    if (t0 == 0) { P.e2s[k1] = ee; P.ds[k1] = P.s_dk; P.s_tau[k1 & 1] = tau1; }
#pragma unroll
    for (int j = 0; j < NRT; ++j) {
      const int t = t0 + RT * j;
      if (NR % RT == 0 || t < NR)
        P.vb[k1 & 1][t] = (t == k1 + 1) ? 1.0 : ((t > k1 + 1 && t < n) ? y[j] * scale : 0.0);
    }
  }
}

// fused pass of step k (k = -1: prologue products with v_0 only), then arrive on B2
template <int S, int C, class ACC>
__device__ __forceinline__ void rr_fused_step(RRProb<S>& P, ACC a, int k, int n, int lane, int wid) {
  const int k1 = k + 1;
  if (k < 0) {
    if (P.s_tau[0] != 0.0) rr_pass<S, C, 0, false, true, ACC>(a, lane, wid, nullptr, nullptr, P.vb[0], P.part, P.cs, P.red, 1, P.colbuf);
    else rr_pass<S, C, 0, false, false, ACC>(a, lane, wid, nullptr, nullptr, nullptr, P.part, P.cs, P.red, 1, P.colbuf);
  } else {
    const double* v = P.vb[k & 1];
    const double tau = P.s_tau[k & 1];
    const bool more = k1 + 2 < n;
    const bool mv = more && P.s_tau[k1 & 1] != 0.0;
    const double* u = P.vb[k1 & 1];
    const int pub = (k + 3 < n) ? k + 2 : -1;
    if (tau != 0.0 && mv) rr_pass_kc<S, C, true, true, ACC>(k >> 4, a, lane, wid, v, P.wb, u, P.part, P.cs, P.red, pub, P.colbuf);
    else if (tau != 0.0) rr_pass<S, C, 0, true, false, ACC>(a, lane, wid, v, P.wb, nullptr, P.part, P.cs, P.red, pub, P.colbuf);
    else if (mv) rr_pass<S, C, 0, false, true, ACC>(a, lane, wid, nullptr, nullptr, u, P.part, P.cs, P.red, pub, P.colbuf);
    else rr_pass<S, C, 0, false, false, ACC>(a, lane, wid, nullptr, nullptr, nullptr, P.part, P.cs, P.red, pub, P.colbuf);
  }
  rr_mbar_arrive(&P.bar2);
}

// d, e^2 of the trailing 2x2 (or n <= 2) from the matrix chunks
template <int S, int C, class ACC>
__device__ __forceinline__ void rr_tail(RRProb<S>& P, ACC a, int n, int lane, int wid) {
  const int lo = n >= 2 ? n - 2 : 0;
  for (int jj = lo; jj < n; ++jj) {
    if (wid == (jj & 15)) {
      double x[S];
      rr_column<S, C, ACC>(jj >> 4, a, x);
      double dj = 0.0, ej = 0.0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        if (i == jj) dj = x[s];
        if (i == jj + 1) ej = x[s];
      }
      dj = __shfl_sync(0xffffffffu, dj, jj & 31);
      ej = __shfl_sync(0xffffffffu, ej, (jj + 1) & 31);
      if (lane == 0) {
        P.ds[jj] = dj;
        if (jj + 1 < n) P.e2s[jj] = ej * ej;
      }
    }
  }
}

// outputs of one problem (threads of one half of the CTA: h = 0..255)
template <int S>
__device__ __forceinline__ void rr_outputs(RRProb<S>& P, int n, int p, int h, int hstride, const double* thr, int kw,
                                           int nstride, double* dout, double* e2out, double* gsh, int* cnt_out) {
  double* dO = dout + (int64_t)p * nstride;
  double* eO = e2out + (int64_t)p * nstride;
  for (int i = h; i < n; i += hstride) {
    dO[i] = P.ds[i];
    if (i + 1 < n) eO[i] = P.e2s[i];
  }
  if (h == 0) {
    const double* d = P.ds;
    const double* e2 = P.e2s;
    double glo = 1e300, ghi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      double r = 0.0;
      if (i > 0) r += sqrt(e2[i - 1]);
      if (i + 1 < n) r += sqrt(e2[i]);
      glo = fmin(glo, d[i] - r);
      ghi = fmax(ghi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    if (n <= 0) { glo = 0.0; ghi = 0.0; }
    const double nrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
    glo -= 2.2e-16 * nrm * n + pivmin;
    ghi += 2.2e-16 * nrm * n + pivmin;
    gsh[4 * p] = glo; gsh[4 * p + 1] = ghi; gsh[4 * p + 2] = pivmin; gsh[4 * p + 3] = nrm;
    int above = n;
    if (thr && n > 0) {
      const double t = thr[p];
      if (t >= ghi) above = 0;
      else if (t > glo) {
        int c0, c1;
        sturm2<double>(d, e2, n, t, t, pivmin, c0, c1);
        above = n - c0;
      }
    }
    cnt_out[p] = n > 0 ? min(kw, above) : 0;
  }
}


// ---------------------------------------------------------------------------
// Two problems per CTA with dedicated row warps (k_tridiag_duo, n <= 160).
// Problem 0's lower-triangle chunks live in registers (n <= 128; at n = 160 only
// the last NQR chunks, the rest in shared memory: HybAcc), problem 1's in shared
// memory (SmemAcc), with the ownership of k_tridiag_rr; 16 element warps run the
// fused passes of both problems, RW dedicated row warps (thread t owns rows
// t + 32 RW j; RW = S for n <= 128: row t) run the row phases.  A row phase only waits for its own problem's partial
// products (mbarrier B2) and the element warps only for its results (mbarrier
// B3), so the latency-bound row phase of one problem overlaps the fused pass
// of the other:  element warps  F0(k) F1(k) F0(k+1) ...;  row warps  R0(k+1)
// R1(k+1) ...  (R_p(k+1) needs F_p(k); F_p(k+1) needs R_p(k+1)).
// ---------------------------------------------------------------------------
#ifndef CMSVD_DUO_GROUPS
#define CMSVD_DUO_GROUPS 1   // row-warp groups: 1 = shared by both problems, 2 = one per problem (measured: no gain at n = 128)
#endif
constexpr int kDuoGroups = CMSVD_DUO_GROUPS;
constexpr int kDuoThreads = kRRThreads + 32 * 4 * kDuoGroups;  // 16 element warps + 4 row warps per group
#ifndef CMSVD_DUO160_RW
#define CMSVD_DUO160_RW 3     // n = 160: row warps (measured: 2-4 within 2%)
#endif
#ifndef CMSVD_DUO160_NQR1
#define CMSVD_DUO160_NQR1 0   // n = 160: problem-1 chunks in registers (of 30; measured (NQR, NQR1) = (16, 4) / (14, 6): within 1%)
#endif
#ifndef CMSVD_DUO128_NQR
#define CMSVD_DUO128_NQR 20   // n <= 128: problem-0 chunks in registers (of 20)
#endif
#ifndef CMSVD_DUO128_NQR1
#define CMSVD_DUO128_NQR1 6   // n <= 128: problem-1 chunks in registers (of 20; measured 0/2/4/6/8/10: 6 best, -2%)
#endif
#ifndef CMSVD_DUO160_NQR
#define CMSVD_DUO160_NQR 18   // n = 160: problem-0 chunks in registers (of 30; >= 18 for shared memory)
#endif
__host__ __device__ constexpr int duo_threads(int S, int RW) { return S <= 4 ? kDuoThreads : kRRThreads + 32 * RW; }

template <int S, int C, int RW = S, int NQR = rr_nchunks<S, C>(), int NQR1 = 0>
__global__ void __launch_bounds__(duo_threads(S, RW), (S <= 2 ? 2 : 1)) k_tridiag_duo(const double* __restrict__ Gin, int64_t ld_in,
                                                                int64_t stride_in, const int* __restrict__ ns,
                                                                int nprob, const double* __restrict__ thr, int kw,
                                                                int nstride, double* __restrict__ dout,
                                                                double* __restrict__ e2out, double* __restrict__ gsh,
                                                                int* __restrict__ cnt_out,
                                                                double* __restrict__ trace_out) {
  constexpr int NR = 32 * S;
  constexpr int CL = 2 * (S - 1);
  constexpr int NQ = rr_nchunks<S, C>();
  constexpr int NT = duo_threads(S, RW);
  constexpr int NQS = NQ - NQR;  // problem-0 chunks in shared memory
  static_assert(C == 2 * S && S <= 5 && RW <= S && 32 * RW <= NT - kRRThreads, "duo kernel: n <= 160");
  extern __shared__ __align__(16) unsigned char duo_smem[];
  RRProb<S>* PP = reinterpret_cast<RRProb<S>*>(duo_smem);
  double* A0 = reinterpret_cast<double*>(duo_smem + 2 * sizeof(RRProb<S>));
  double* A1 = A0 + (size_t)NQS * kRRThreads;  // problem 1: its first NQ - NQR1 chunks (the rest in registers)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool elem = tid < kRRThreads;
  const int pa = 2 * blockIdx.x, pb = pa + 1;
  const int n0 = ns[pa], n1 = (pb < nprob) ? ns[pb] : 0;
  RRProb<S>& P0 = PP[0];
  RRProb<S>& P1 = PP[1];
  double a0_[S][C];
  using Acc0 = HybAcc<S, C, NQR>;
  const Acc0 a0{a0_, A0 + (elem ? tid : 0)};
  double a1_[S][C];
  using Acc1 = HybAcc<S, C, NQR1>;
  const Acc1 a1{a1_, A1 + (elem ? tid : 0)};
  if (elem) {
    const double* G0 = Gin + (int64_t)pa * stride_in;
    const double* G1 = Gin + (int64_t)pb * stride_in;
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (rr_present(s, c)) {
          const int i = lane + 32 * s, j = wid + 16 * c;
          a0.st(s, c, (i < n0 && j < n0) ? G0[(int64_t)j * ld_in + i] : 0.0);
          a1.st(s, c, (i < n1 && j < n1) ? G1[(int64_t)j * ld_in + i] : 0.0);
        }
    if (wid == 0 || wid == 8) {
      const double* G = wid == 0 ? G0 : G1;
      const int n = wid == 0 ? n0 : n1;
      double t = 0.0;
      for (int i = lane; i < n; i += 32) t += G[(int64_t)i * ld_in + i];
      t = warp_sum(t);
      if (lane == 0) {
        if (wid == 0) trace_out[pa] = t;
        else if (pb < nprob) trace_out[pb] = t;
      }
    }
  }
  for (int j = 16 * CL + tid; j < NR; j += NT) { P0.cs[j] = 0.0; P1.cs[j] = 0.0; }
  if (tid == 0) {
    rr_mbar_init(&P0.bar2, kRRThreads);
    rr_mbar_init(&P0.bar3, 32 * RW);
    rr_mbar_init(&P1.bar2, kRRThreads);
    rr_mbar_init(&P1.bar3, 32 * RW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == 0) {  // reflector 0 of each problem, by the owner warp of column 0
    double x[S];
    if (n0 >= 3) {
      rr_column<S, C, Acc0>(0, a0, x);
      rr_reflector_warp<S>(P0, 0, x, n0, lane);
    }
    if (n1 >= 3) {
      rr_column<S, C, Acc1>(0, a1, x);
      rr_reflector_warp<S>(P1, 0, x, n1, lane);
    }
  }
  __syncthreads();
  const int nsteps = max(n0, n1) - 2;
  if (elem) {
    if (n0 >= 3) rr_fused_step<S, C, Acc0>(P0, a0, -1, n0, lane, wid);
    if (n1 >= 3) rr_fused_step<S, C, Acc1>(P1, a1, -1, n1, lane, wid);
#ifdef CMSVD_RR_PROF
    unsigned long long t_last = clock64();
#endif
    for (int k = 0; k < nsteps; ++k) {
      if (k + 2 < n0) {
        rr_mbar_wait(&P0.bar3, k & 1);
        RR_T(0, wid == 1);
        rr_fused_step<S, C, Acc0>(P0, a0, k, n0, lane, wid);
        RR_T(1, wid == 1);
      }
      if (k + 2 < n1) {
        rr_mbar_wait(&P1.bar3, k & 1);
        RR_T(2, wid == 1);
        rr_fused_step<S, C, Acc1>(P1, a1, k, n1, lane, wid);
        RR_T(3, wid == 1);
      }
    }
  } else if (kDuoGroups == 2) {
    // one row-warp group per problem: the two row phases run concurrently
    const int g = (tid - kRRThreads) / 128, t = (tid - kRRThreads) % 128, wr = t >> 5;
    RRProb<S>& P = g == 0 ? P0 : P1;
    const int n = g == 0 ? n0 : n1;
    if (t < NR)
      for (int k = 0; k + 2 < n; ++k) {
        rr_mbar_wait(&P.bar2, k & 1);
        rr_row_phase<S>(P, k, n, t, wr, lane, 1 + g);
        rr_mbar_arrive(&P.bar3);
      }
  } else if (tid - kRRThreads < 32 * RW) {
    const int t = tid - kRRThreads, wr = wid - kRRWarps;
#ifdef CMSVD_RR_PROF
    unsigned long long t_last = clock64();
#endif
    for (int k = 0; k < nsteps; ++k) {
      if (k + 2 < n0) {
        rr_mbar_wait(&P0.bar2, k & 1);
        RR_T(4, wr == 0);
        rr_row_phase<S, RW>(P0, k, n0, t, wr, lane, 1);
        rr_mbar_arrive(&P0.bar3);
        RR_T(5, wr == 0);
      }
      if (k + 2 < n1) {
        rr_mbar_wait(&P1.bar2, k & 1);
        RR_T(6, wr == 0);
        rr_row_phase<S, RW>(P1, k, n1, t, wr, lane, 2);
        rr_mbar_arrive(&P1.bar3);
        RR_T(7, wr == 0);
      }
    }
  }
  __syncthreads();
  if (elem) {
    rr_tail<S, C, Acc0>(P0, a0, n0, lane, wid);
    rr_tail<S, C, Acc1>(P1, a1, n1, lane, wid);
  }
  __syncthreads();
  if (tid < NT / 2) rr_outputs<S>(P0, n0, pa, tid, NT / 2, thr, kw, nstride, dout, e2out, gsh, cnt_out);
  else if (pb < nprob) rr_outputs<S>(P1, n1, pb, tid - NT / 2, NT / 2, thr, kw, nstride, dout, e2out, gsh, cnt_out);
}

template <int S, int C, int NQR = rr_nchunks<S, C>(), int NQR1 = 0>
size_t duo_smem_bytes() {
  return 2 * sizeof(RRProb<S>) + (size_t)(2 * rr_nchunks<S, C>() - NQR - NQR1) * kRRThreads * sizeof(double);
}

// ---------------------------------------------------------------------------
// Plain bisection, one thread per wanted eigenvalue (high occupancy; the
// tridiagonals are read through L1).  fp32 coarse phase on the normalised
// matrix to ~4e-7 ||T||, widened by 1e-5 ||T||, then fp64 to max(1e-13 ||T||, 1e-11 lambda).
// ev[p*kw + l] = l-th largest eigenvalue for l < cnt[p], else 0.
// ---------------------------------------------------------------------------
// STAGE: the block's problems (at most kBisStage) are staged in shared memory, with the normalised fp32
// copies of the fp32 phase computed once (same fp32 operations as the per-step conversion of the
// unstaged variant, so the results are identical).
constexpr int kBisStage = 6;
template <bool STAGE>
__global__ void __launch_bounds__(128) k_bisect(int P, int kw, int nstride, const int* __restrict__ ns,
                                                const double* __restrict__ dd, const double* __restrict__ ee2,
                                                const double* __restrict__ gsh, const int* __restrict__ cnt,
                                                double* __restrict__ ev) {
  extern __shared__ double bis_sm[];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
  const int p0 = (int)(g0 / kw);
  if (STAGE) {  // problems p0 .. p0 + np - 1 of this block
    const int64_t glast = min((int64_t)P * kw, g0 + blockDim.x) - 1;
    const int np = glast >= g0 ? (int)(glast / kw) - p0 + 1 : 0;
    // problem q: (d_i, e2_{i-1}) pairs at bis_sm + 2 q nstride, their normalised fp32 copies after all
    // kBisStage fp64 problems (one vector load per Sturm step)
    double* de64 = bis_sm;
    float* de32 = reinterpret_cast<float*>(bis_sm + (size_t)2 * kBisStage * nstride);
    for (int q = 0; q < np; ++q) {
      const int pq = p0 + q;
      const int n = ns[pq];
      const float inv = (float)(1.0 / gsh[4 * pq + 3]);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double di = dd[(int64_t)pq * nstride + i];
        const double ei = i > 0 ? ee2[(int64_t)pq * nstride + i - 1] : 0.0;
        de64[(size_t)q * 2 * nstride + 2 * i] = di;
        de64[(size_t)q * 2 * nstride + 2 * i + 1] = ei;
        de32[(size_t)q * 2 * nstride + 2 * i] = (float)di * inv;
        de32[(size_t)q * 2 * nstride + 2 * i + 1] = (float)ei * inv * inv;
      }
    }
    __syncthreads();
  }
  if (g >= (int64_t)P * kw) return;
  const int p = (int)(g / kw), l = (int)(g % kw);
  double* out = ev + (int64_t)p * kw + l;
  if (l >= cnt[p]) { *out = 0.0; return; }
  const int n = ns[p];
  const double* d = dd + (int64_t)p * nstride;
  const double* e2 = ee2 + (int64_t)p * nstride;
  const double2* de64 = reinterpret_cast<const double2*>(bis_sm + (size_t)2 * (p - p0) * nstride);
  const float2* de32 = reinterpret_cast<const float2*>(
      reinterpret_cast<const float*>(bis_sm + (size_t)2 * kBisStage * nstride) + (size_t)2 * (p - p0) * nstride);
  // (d_i, e2_{i-1}), i >= 1
  auto ld64 = [&](int i) -> double2 { return STAGE ? de64[i] : make_double2(__ldg(d + i), __ldg(e2 + i - 1)); };
  const double d0 = STAGE ? de64[0].x : d[0];
  const double glo = gsh[4 * p], ghi = gsh[4 * p + 1], pivmin = gsh[4 * p + 2], nrm = gsh[4 * p + 3];
  const int target = n - 1 - l;
  double lo = glo, hi = ghi;
  // fp32 phase
  {
    const float inv = (float)(1.0 / nrm);
    float a = (float)(lo / nrm), b = (float)(hi / nrm);
    for (int it = 0; it < 40 && (b - a) > 4e-7f; ++it) {
      const float x = 0.5f * (a + b);
      float q = (float)(d0 * inv) - x;
      if (fabsf(q) < 1e-30f) q = -1e-30f;
      int c = q < 0.f;
      for (int i = 1; i < n; ++i) {
        const float2 de = STAGE ? de32[i] : make_float2((float)__ldg(d + i) * inv, (float)(__ldg(e2 + i - 1)) * inv * inv);
        q = (de.x - x) - __fdividef(de.y, q);
        if (fabsf(q) < 1e-30f) q = -1e-30f;
        c += q < 0.f;
      }
      if (c <= target) a = x; else b = x;
    }
    lo = fmax(glo, (double)a * nrm - 1e-5 * nrm);
    hi = fmin(ghi, (double)b * nrm + 1e-5 * nrm);
  }
  // stop at 1e-13 ||T|| absolute (the floor that resolves sigma = sqrt(lambda) near zero, A13) or
  // 1e-11 relative, whichever is looser: a large eigenvalue needs no more for sigma~ (1e-4) or for the
  // captured-energy sums (error <= 1e-11 E against the 1e-7 E floor)
  const double tol = 1e-13 * nrm;
  const unsigned long long pivbits = (unsigned long long)__double_as_longlong(pivmin);
  for (int it = 0; it < 80 && (hi - lo) > fmax(tol, 1e-11 * fmax(fabs(lo), fabs(hi))) + 4.4e-16 * fmax(fabs(lo), fabs(hi)); ++it) {
    const double x = 0.5 * (lo + hi);
    double q = sturm_clamp(d0 - x, pivbits, -pivmin);
    int c = sturm_neg(q);
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
      const double2 de = ld64(i);
      q = sturm_clamp((de.x - x) - de.y * rcp_sturm(q), pivbits, -pivmin);
      c += sturm_neg(q);
    }
    if (c <= target) lo = x; else hi = x;
  }
  *out = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------------------
// Division-free bisection (the default): Sturm counts from the polynomial recurrence
//   p_0 = 1, p_1 = d_0 - x, p_i = (d_{i-1} - x) p_{i-1} - e^2_{i-2} p_{i-2},  count(x) = sign changes of (p_i),
// on the matrix normalised by its Gershgorin norm (|d| <= 1, e^2 <= 1).  The pivot form above carries a
// reciprocal on its dependency chain (MUFU + 3 dependent DFMA + product + clamp per step: ncu shows the kernel
// waiting on fixed-latency dependencies at 54 % issue utilisation); here the chain is ONE DFMA per step (the
// product e^2 p_{i-2} and the shift d - x are off the chain) and a step is 3 fp64 instructions instead of 7, so
// the fp32 coarse phase is no longer worth its widening and all steps run in fp64.
//   * range: |p_i| grows by at most 2^1.3 per step; every 8 steps both running values are rescaled by the power
//     of two that brings the larger to [1, 2) (exponent arithmetic: exact, signs untouched);
//   * zeros: e^2 is floored at 2^-200 when staged (a relative perturbation of 2^-100 of an off-diagonal entry),
//     so p_{i+1} = -e^2 p_{i-1} != 0 after an exact zero p_i, and the sign-bit count over the two steps is 1
//     whichever sign bit the zero carries: no per-step test;
//   * Wilkinson's analysis of this recurrence (AEP ch. 5) gives the same backward stability as the pivot form.
// Stopping rule and output as k_bisect.
// ---------------------------------------------------------------------------
constexpr int kBisPStage = 6;
template <bool STAGE>
__global__ void __launch_bounds__(128) k_bisect_p(int P, int kw, int nstride, const int* __restrict__ ns,
                                                  const double* __restrict__ dd, const double* __restrict__ ee2,
                                                  const double* __restrict__ gsh, const int* __restrict__ cnt,
                                                  double* __restrict__ ev) {
  extern __shared__ double bis_sm[];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
  const int p0 = (int)(g0 / kw);
  constexpr double kE2Floor = 6.223015277861142e-61;   // 2^-200
  if (STAGE) {  // problems p0 .. p0 + np - 1 of this block: normalised (d_i, e2_{i-1}) pairs
    const int64_t glast = min((int64_t)P * kw, g0 + blockDim.x) - 1;
    const int np = glast >= g0 ? (int)(glast / kw) - p0 + 1 : 0;
    for (int q = 0; q < np; ++q) {
      const int pq = p0 + q;
      const int n = ns[pq];
      const double inv = 1.0 / gsh[4 * pq + 3];
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double di = dd[(int64_t)pq * nstride + i];
        const double ei = i > 0 ? ee2[(int64_t)pq * nstride + i - 1] : 0.0;
        bis_sm[(size_t)q * 2 * nstride + 2 * i] = di * inv;
        bis_sm[(size_t)q * 2 * nstride + 2 * i + 1] = fmax((ei * inv) * inv, kE2Floor);
      }
    }
    __syncthreads();
  }
  if (g >= (int64_t)P * kw) return;
  const int p = (int)(g / kw), l = (int)(g % kw);
  double* out = ev + (int64_t)p * kw + l;
  if (l >= cnt[p]) { *out = 0.0; return; }
  const int n = ns[p];
  const double* d = dd + (int64_t)p * nstride;
  const double* e2 = ee2 + (int64_t)p * nstride;
  const double nrm = gsh[4 * p + 3];
  const double inv = 1.0 / nrm;
  const double2* de = reinterpret_cast<const double2*>(bis_sm + (size_t)2 * (p - p0) * nstride);
  auto ld = [&](int i) -> double2 {   // (d_i, e2_{i-1}) normalised, i >= 1
    return STAGE ? de[i] : make_double2(__ldg(d + i) * inv, fmax((__ldg(e2 + i - 1) * inv) * inv, kE2Floor));
  };
  const double d0 = STAGE ? de[0].x : d[0] * inv;
  const int target = n - 1 - l;
  double lo = gsh[4 * p] * inv, hi = gsh[4 * p + 1] * inv;
  // stop at 1e-13 ||T|| absolute (the floor that resolves sigma = sqrt(lambda) near zero, A13) or 1e-11
  // relative, whichever is looser (as k_bisect); normalised: ||T|| = 1
  for (int it = 0; it < 120 && (hi - lo) > fmax(1e-13, 1e-11 * fmax(fabs(lo), fabs(hi))) + 4.4e-16 * fmax(fabs(lo), fabs(hi)); ++it) {
    const double x = 0.5 * (lo + hi);
    double pp = 1.0, pc = d0 - x;
    int c = (int)((unsigned)__double2hiint(pc) >> 31);
    auto step = [&](int i) {
      const double2 v = ld(i);
      const double t = v.y * pp;
      const double pn = fma(v.x - x, pc, -t);
      c += (int)((unsigned)(__double2hiint(pn) ^ __double2hiint(pc)) >> 31);
      pp = pc;
      pc = pn;
    };
    int i = 1;
    for (; i + 8 <= n; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step(i + u);
      const unsigned ha = (unsigned)__double2hiint(pc) & 0x7fffffffu, hb = (unsigned)__double2hiint(pp) & 0x7fffffffu;
      const unsigned ex = max(ha, hb) >> 20;                        // biased exponent of the larger
      const double f = __hiloint2double((int)((2046u - ex) << 20), 0);   // 2^(1023 - ex)
      pc *= f;
      pp *= f;
    }
    for (; i < n; ++i) step(i);
    if (c <= target) lo = x; else hi = x;
  }
  *out = 0.5 * (lo + hi) * nrm;
}

// Multisection for small batches (latency-bound: e.g. one greedy evaluation or
// commit): one warp per wanted eigenvalue, the 32 lanes evaluate Sturm counts
// at 32 interior points of the bracket, so each fp64 step narrows it 33x.
// Same stopping rule and output as k_bisect.
constexpr int64_t kMultisectMax = 1024;  // wanted eigenvalues in a launch below which multisection wins
__global__ void __launch_bounds__(128) k_multisect(int P, int kw, int nstride, const int* __restrict__ ns,
                                                   const double* __restrict__ dd, const double* __restrict__ ee2,
                                                   const double* __restrict__ gsh, const int* __restrict__ cnt,
                                                   double* __restrict__ ev) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= (int64_t)P * kw) return;
  const int p = (int)(g / kw), l = (int)(g % kw);
  double* out = ev + (int64_t)p * kw + l;
  if (l >= cnt[p]) { if (lane == 0) *out = 0.0; return; }
  const int n = ns[p];
  const double* d = dd + (int64_t)p * nstride;
  const double* e2 = ee2 + (int64_t)p * nstride;
  const double pivmin = gsh[4 * p + 2], nrm = gsh[4 * p + 3];
  double lo = gsh[4 * p], hi = gsh[4 * p + 1];
  const int target = n - 1 - l;
  const double tol = 1e-13 * nrm;
  for (int it = 0; it < 40 && (hi - lo) > tol + 4.4e-16 * fmax(fabs(lo), fabs(hi)); ++it) {
    const double h = (hi - lo) * (1.0 / 33.0);
    const double x = fma((double)(lane + 1), h, lo);
    const unsigned long long pivbits = (unsigned long long)__double_as_longlong(pivmin);
    double q = sturm_clamp(__ldg(d) - x, pivbits, -pivmin);
    int c = sturm_neg(q);
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
      q = sturm_clamp((__ldg(d + i) - x) - __ldg(e2 + i - 1) * rcp_sturm(q), pivbits, -pivmin);
      c += sturm_neg(q);
    }
    const unsigned below = __ballot_sync(0xffffffffu, c <= target);  // a prefix of the lanes
    const int k = __popc(below);
    const double xl = __shfl_sync(0xffffffffu, x, (k + 31) & 31);
    const double xh = __shfl_sync(0xffffffffu, x, k & 31);
    if (k > 0) lo = xl;
    if (k < 32) hi = xh;
  }
  if (lane == 0) *out = 0.5 * (lo + hi);
}

// One implicit QL sweep (tql2, Wilkinson-type shift) on the unreduced block l .. m of the tridiagonal (dd, ee):
// the rotations i = m-1 .. lo are left in rc[i], rs[i]; returns lo, the lowest rotation index generated (l, or
// the stop index + 1 after an underflow).  Sequential: one thread.
__device__ __forceinline__ int ql_sweep(double* __restrict__ dd, double* __restrict__ ee, int l, int m,
                                        double* __restrict__ rc, double* __restrict__ rs) {
  double g = (dd[l + 1] - dd[l]) / (2.0 * ee[l]);
  double r = hypot(g, 1.0);
  g = dd[m] - dd[l] + ee[l] / (g + copysign(r, g));
  double sn = 1.0, cs = 1.0, pp = 0.0;
  int i = m - 1;
  bool underflow = false;
  // every d/e value read below is an original one (the sweep writes ee[i+1], dd[i+1] behind the
  // read front), so the next iteration's operands are prefetched into registers
  double e_i = ee[i], d_i1 = dd[i + 1], d_i = dd[i];
  for (; i >= l; --i) {
    const double e_n = (i > l) ? ee[i - 1] : 0.0;
    const double d_n = (i > l) ? dd[i - 1] : 0.0;
    double f = sn * e_i;
    const double b = cs * e_i;
    // r = hypot(f, g), sn = f / r, cs = g / r: one MUFU.RSQ64H + a cubic step instead of the
    // IEEE hypot and two divisions on this sequential chain; scaled fallback near under/overflow
    const double x2 = fma(f, f, g * g);
    const double gq = d_i1 - pp;
    if (x2 > 1e-280 && x2 < 1e280) {
      // (d_i - gq) sn + 2 cs b = y ((d_i - gq) f + 2 g b): the bracket is formed while the
      // reciprocal square root is in flight, so one multiply follows it on the chain
      const double T = fma(d_i - gq, f, 2.0 * g * b);
      const double y = rsqrt_cubic(x2);
      ee[i + 1] = x2 * y;
      sn = f * y;
      cs = g * y;
      r = T * y;
    } else {
      r = hypot(f, g);
      ee[i + 1] = r;
      if (r == 0.0) {
        dd[i + 1] = gq;
        ee[m] = 0.0;
        underflow = true;
        break;
      }
      sn = f / r;
      cs = g / r;
      r = (d_i - gq) * sn + 2.0 * cs * b;
    }
    pp = sn * r;
    dd[i + 1] = gq + pp;
    g = cs * r - b;
    rc[i] = cs;
    rs[i] = sn;
    e_i = e_n;
    d_i1 = d_i;
    d_i = d_n;
  }
  // rotations actually generated: indices i_stop+1 .. m-1 (i_stop = i)
  if (!underflow) {
    dd[l] -= pp;
    ee[l] = g;
    ee[m] = 0.0;
  }
  return underflow ? i + 1 : l;
}

// ---------------------------------------------------------------------------
// Symmetric eigen-decomposition with vectors (block spectra S2, cluster-state
// commits S10): the tridiagonal reduction above with the reflectors saved,
// implicit QL with Wilkinson-type shift on the tridiagonal (rotations
// generated by one thread, applied to the rows of Z by all threads in
// parallel), back-transformation Z <- H_0 ... H_{n-3} Z.  One CTA per problem,
// fp64.  Outputs: evals[p*stride_out + l] non-increasing; the eigenvector of
// evals[l] is column perm[p*stride_out + l] of V_p (n x n, ld n, at
// Vws + p*stride_v); status[p] = QL iterations, or -1 on no convergence.
// ---------------------------------------------------------------------------
template <bool GL>
__global__ void __launch_bounds__(kTriThreads, 1) k_syev_ql(const double* __restrict__ Gin, int64_t ld_in,
                                                            int64_t stride_in, const int* __restrict__ ns,
                                                            double* __restrict__ Vws, int64_t stride_v,
                                                            double* __restrict__ VHws, double* __restrict__ evals,
                                                            int* __restrict__ perm, int64_t stride_out,
                                                            int* __restrict__ status, int max_iter, int flags) {
  extern __shared__ double sm[];
  const int p = blockIdx.x;
  const int n = ns[p];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ldz = GL ? (int)ld_in : (n | 1);
  double* __restrict__ A = GL ? const_cast<double*>(Gin) + (int64_t)p * stride_in : sm;  // later Z (n x ldz)
  const int64_t asz = GL ? 0 : (int64_t)n * ldz;
  double* vA = (GL ? sm : A) + asz;
  double* vB = vA + n;
  double* __restrict__ w = vB + n;
  double* __restrict__ part = w + n;                   // kTriWarps x n
  double* __restrict__ e2 = part + (int64_t)kTriWarps * n;
  double* __restrict__ dd = e2 + n;
  double* __restrict__ ee = dd + n;
  double* __restrict__ rc = ee + n;                    // rotation cosines of a sweep
  double* __restrict__ rs = rc + n;                    // rotation sines
  double* __restrict__ tauH = rs + n;
  __shared__ int s_l, s_m, s_iters, s_fail;
  double* VH = VHws + (int64_t)p * stride_v;
  double* V = Vws + (int64_t)p * stride_v;
  if (n <= 0) { if (tid == 0) status[p] = 0; return; }
  const int lda = GL ? (int)ld_in : n;
  if (!GL) {
    for (int j = wid; j < n; j += kTriWarps) {
      const double* src = Gin + (int64_t)p * stride_in + (int64_t)j * ld_in;
      for (int i = lane; i < n; i += 32) A[j * n + i] = src[i];
    }
  }
  __syncthreads();
#ifdef CMSVD_SYEV_PROF
  unsigned long long t0 = clock64();
#endif
  tri_reduce<true>(A, n, lda, vA, vB, w, part, e2, ee, VH, tauH);
#ifdef CMSVD_SYEV_PROF
  __syncthreads();
  unsigned long long t1 = clock64();
#endif
  __syncthreads();
  for (int i = tid; i < n; i += kTriThreads) dd[i] = A[(int64_t)i * lda + i];
  if (tid == 0) {
    if (n == 2) ee[0] = A[0 * lda + 1];
    ee[n - 1] = 0.0;
  }
  __syncthreads();
  // Z = I (overwrites A, which is dead), ld = ldz
  for (int64_t e = tid; e < (int64_t)n * ldz; e += kTriThreads) A[e] = 0.0;
  __syncthreads();
  for (int i = tid; i < n; i += kTriThreads) A[(int64_t)i * ldz + i] = 1.0;
  __shared__ double s_anorm;
  if (tid == 0) {
    s_iters = 0; s_fail = 0;
    double an = 0.0;
    for (int i = 0; i < n; ++i) an = fmax(an, fabs(dd[i]) + fabs(ee[i]) + (i > 0 ? fabs(ee[i - 1]) : 0.0));
    s_anorm = an;
  }
  __syncthreads();
  // ---- implicit QL (tql2) ----
  // deflate when |e_m| <= eps (|d_m| + |d_m+1|) or |e_m| <= 8 eps ||T|| (absolute accuracy ~ eps ||T||,
  // the same as the reduction's backward error; needed when both neighbours are ~0)
  const double defl_abs = 8.0 * 2.220446049250313e-16 * s_anorm;
  if (GL && (flags & 2)) {
    // Fused sweeps (in-place variant): warp 0 runs the QL iteration on (dd, ee) alone -- the rotations do not
    // depend on Z -- and leaves up to kQF consecutive sweeps in tables padded with identity rotations over
    // the union range [L, H]; every thread then passes its two rows of Z ONCE through the kQF rotation stages
    // (sweep k trails sweep k-1 by one column: the value leaving stage k-1 at column i+k is what stage k
    // rotates next; an identity stage is a one-column delay), so Z is read and written once per kQF sweeps.
    // Per element the same rotations in the same order as the sweep-by-sweep loop below.
    constexpr int kQF = 4, kQB = CMSVD_QL_BATCH;
    const int tl = n + 2 * kQF;                 // table row: index kQF + i for rotation i in [-kQF, n + kQF)
    double* __restrict__ tc = vA;               // kQF rows of cosines, then kQF rows of sines (vA .. e2 are dead)
    double* __restrict__ ts = vA + kQF * tl;
    __shared__ int s_cnt, s_L, s_H, s_lcur, s_itcur;
    if (tid == 0) { s_lcur = 0; s_itcur = 0; }
    for (;;) {
      for (int e = tid; e < kQF * tl; e += kTriThreads) { tc[e] = 1.0; ts[e] = 0.0; }
      __syncthreads();
      if (wid == 0) {
        int l = s_lcur, iter = s_itcur, cnt = 0, L = n, H = -1, fail = 0, its = 0;
        while (cnt < kQF && l < n) {
          int mq = n - 1;
          for (int base = l; base < n - 1; base += 32) {
            const int mm = base + lane;
            bool neg = false;
            if (mm < n - 1) {
              const double dsum = fabs(dd[mm]) + fabs(dd[mm + 1]);
              neg = fabs(ee[mm]) <= 2.220446049250313e-16 * dsum || fabs(ee[mm]) <= defl_abs;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, neg);
            if (bal) { mq = base + __ffs(bal) - 1; break; }
          }
          if (mq == l) { ++l; iter = 0; continue; }
          if (iter >= max_iter) { fail = 1; break; }
          int lo = 0;
          if (lane == 0) lo = ql_sweep(dd, ee, l, mq, tc + cnt * tl + kQF, ts + cnt * tl + kQF);
          lo = __shfl_sync(0xffffffffu, lo, 0);
          __syncwarp();
          L = min(L, lo);
          H = max(H, mq);
          ++cnt; ++iter; ++its;
        }
        if (lane == 0) {
          s_cnt = cnt; s_L = L; s_H = H; s_lcur = l; s_itcur = iter;
          s_iters += its;
          if (fail) s_fail = 1;
        }
      }
      __syncthreads();
      if (s_fail || s_cnt == 0) break;
      const int L = s_L, H = s_H;
      for (int row = tid; row < n; row += 2 * kTriThreads) {
        const bool two = row + kTriThreads < n;
        double* za = A + row;
        double* zb = A + (two ? row + kTriThreads : row);
        double fa[kQF], fb[kQF];
#pragma unroll
        for (int k = 0; k < kQF; ++k) fa[k] = fb[k] = 0.0;
        int i0 = H;
        while (i0 >= L - kQF) {
          const int nb = min(kQB, i0 - (L - kQF) + 1);
          double ca[kQB], cb[kQB];
#pragma unroll
          for (int t = 0; t < kQB; ++t) {
            const bool ld = t < nb && i0 - t >= L;
            ca[t] = ld ? za[(int64_t)(i0 - t) * ldz] : 0.0;
            cb[t] = ld ? zb[(int64_t)(i0 - t) * ldz] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < kQB; ++t)
            if (t < nb) {
              const int ii = i0 - t;
              double va = ca[t], vb = cb[t];
#pragma unroll
              for (int k = 0; k < kQF; ++k) {
                const double c_ = tc[k * tl + kQF + ii + k], s_ = ts[k * tl + kQF + ii + k];
                const double oa = s_ * va + c_ * fa[k];
                fa[k] = c_ * va - s_ * fa[k];
                va = oa;
                const double ob = s_ * vb + c_ * fb[k];
                fb[k] = c_ * vb - s_ * fb[k];
                vb = ob;
              }
              const int io = ii + kQF;
              if (io >= L && io <= H) {
                za[(int64_t)io * ldz] = va;
                if (two) zb[(int64_t)io * ldz] = vb;
              }
            }
          i0 -= nb;
        }
      }
      __syncthreads();
    }
  } else
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    while (true) {
      // deflation search by warp 0 (32 candidates per ballot), the sweep by its lane 0
      int mq = n - 1;
      if (wid == 0) {
        for (int base = l; base < n - 1; base += 32) {
          const int mm = base + lane;
          bool neg = false;
          if (mm < n - 1) {
            const double dsum = fabs(dd[mm]) + fabs(dd[mm + 1]);
            neg = fabs(ee[mm]) <= 2.220446049250313e-16 * dsum || fabs(ee[mm]) <= defl_abs;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, neg);
          if (bal) { mq = base + __ffs(bal) - 1; break; }
        }
      }
      if (tid == 0) {
        const int m = mq;
        s_m = m;
        if (m != l) {
          if (iter >= max_iter) { s_fail = 1; s_m = l; }
          else {
            s_l = ql_sweep(dd, ee, l, m, rc, rs);   // lowest rotation index applied
            s_iters += 1;
          }
        }
      }
      __syncthreads();
      const int m = s_m;
      if (m == l || s_fail) break;
      const int lo_i = s_l;
      // apply rotations i = m-1 .. lo_i to columns (i, i+1) of Z: each thread owns rows
      if (GL) {
        // a thread rotates two rows (tid, tid + kTriThreads) at once: the rotated column i of each row is
        // carried in a register to the next rotation; the original values of the next kQB columns of both rows
        // are loaded ahead in one batch (every load precedes the stores that follow it) -- 2 kQB loads in
        // flight per thread hide the global-memory latency of the in-place (n > 160) variant
        constexpr int kQB = CMSVD_QL_BATCH;
        for (int row = tid; row < n; row += 2 * kTriThreads) {
          const bool two = row + kTriThreads < n;
          double* za = A + row;
          double* zb = A + (two ? row + kTriThreads : row);
          double fa = za[(int64_t)m * ldz], fb = zb[(int64_t)m * ldz];
          int i = m - 1;
          while (i >= lo_i) {
            const int cnt = min(kQB, i - lo_i + 1);
            double ca[kQB], cb[kQB];
  #pragma unroll
            for (int t = 0; t < kQB; ++t) {
              ca[t] = (t < cnt) ? za[(int64_t)(i - t) * ldz] : 0.0;
              cb[t] = (t < cnt) ? zb[(int64_t)(i - t) * ldz] : 0.0;
            }
  #pragma unroll
            for (int t = 0; t < kQB; ++t)
              if (t < cnt) {
                const int ii = i - t;
                const double c_ = rc[ii], s_ = rs[ii];
                za[(int64_t)(ii + 1) * ldz] = s_ * ca[t] + c_ * fa;
                fa = c_ * ca[t] - s_ * fa;
                if (two) zb[(int64_t)(ii + 1) * ldz] = s_ * cb[t] + c_ * fb;
                fb = c_ * cb[t] - s_ * fb;
              }
            i -= cnt;
          }
          za[(int64_t)lo_i * ldz] = fa;
          if (two) zb[(int64_t)lo_i * ldz] = fb;
        }
      } else {
        for (int row = tid; row < n; row += kTriThreads) {
          double* z = A + row;
          // the rotated column i is carried in a register to the next rotation; loads run one ahead
          double f = z[(int64_t)m * ldz];
          double zi = z[(int64_t)(m - 1) * ldz];
          for (int i = m - 1; i >= lo_i; --i) {
            const double zn = (i > lo_i) ? z[(int64_t)(i - 1) * ldz] : 0.0;
            const double c_ = rc[i], s_ = rs[i];
            z[(int64_t)(i + 1) * ldz] = s_ * zi + c_ * f;
            f = c_ * zi - s_ * f;
            zi = zn;
          }
          z[(int64_t)lo_i * ldz] = f;
        }
      }
      __syncthreads();
      ++iter;
    }
    if (s_fail) break;
  }
  __syncthreads();
#ifdef CMSVD_SYEV_PROF
  unsigned long long t2 = clock64();
#endif
  // ---- back-transformation Z <- H_0 H_1 ... H_{n-3} Z ----
  // shared memory: thread per column; global memory (GL): a warp keeps two columns of Z in registers (row
  // 32 t + lane in slot t) and applies every reflector to them -- Z is read and written once instead of once
  // per reflector (2 GB of L2 / DRAM traffic per 512 x 512 problem), no barrier between reflectors; the
  // reflector vectors are shared by the CTA's warps through L1, the next one is loaded ahead
  if (GL && (flags & 1)) {
    for (int c0 = wid; c0 < n; c0 += 2 * kTriWarps) {
      const int c1 = c0 + kTriWarps;
      const bool two = c1 < n;
      double* za = A + (int64_t)c0 * ldz;
      double* zb = A + (int64_t)(two ? c1 : c0) * ldz;
      double z0[16], z1[16], vr[16], vn[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int j = 32 * t + lane;
        z0[t] = j < n ? za[j] : 0.0;
        z1[t] = j < n ? zb[j] : 0.0;
        vn[t] = 0.0;
      }
      auto loadv = [&](int k) {
        const double* v = VH + (int64_t)k * n;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = 32 * t + lane;
          vn[t] = (32 * t + 31 > k && j > k && j < n) ? v[j] : 0.0;
        }
      };
      if (n >= 3) loadv(n - 3);
      for (int k = n - 3; k >= 0; --k) {
#pragma unroll
        for (int t = 0; t < 16; ++t) vr[t] = vn[t];
        if (k > 0) loadv(k - 1);
        const double tk = tauH[k];
        if (tk == 0.0) continue;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          d0 = fma(vr[t], z0[t], d0);
          d1 = fma(vr[t], z1[t], d1);
        }
        d0 = warp_sum(d0) * tk;
        d1 = warp_sum(d1) * tk;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          z0[t] = fma(-d0, vr[t], z0[t]);
          z1[t] = fma(-d1, vr[t], z1[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int j = 32 * t + lane;
        if (j < n) {
          za[j] = z0[t];
          if (two) zb[j] = z1[t];
        }
      }
    }
    __syncthreads();
  } else
  for (int k = n - 3; k >= 0; --k) {
    const double tk = tauH[k];
    if (tk != 0.0) {
      const double* vk = VH + (int64_t)k * n + k + 1;  // length n-1-k, vk[0] = 1
      if (GL) {
        for (int c = wid; c < n; c += kTriWarps) {
          double* zc = A + (int64_t)c * ldz + k + 1;
          double dot = 0.0;
          for (int i = lane; i < n - 1 - k; i += 32) dot = fma(vk[i], zc[i], dot);
          dot = warp_sum(dot) * tk;
          for (int i = lane; i < n - 1 - k; i += 32) zc[i] = fma(-dot, vk[i], zc[i]);
        }
      } else {
        for (int c = tid; c < n; c += kTriThreads) {
          double* zc = A + (int64_t)c * ldz + k + 1;
          double dot = 0.0;
          for (int i = 0; i < n - 1 - k; ++i) dot = fma(vk[i], zc[i], dot);
          dot *= tk;
          for (int i = 0; i < n - 1 - k; ++i) zc[i] = fma(-dot, vk[i], zc[i]);
        }
      }
    }
    __syncthreads();
  }
#ifdef CMSVD_SYEV_PROF
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("syev n=%d: tridiag %llu  QL %llu  backtransform %llu cycles (iters %d)\n", n, t1 - t0, t2 - t1, clock64() - t2, s_iters);
#endif
  // ---- sort (non-increasing, ties by index) and write ----
  for (int i = tid; i < n; i += kTriThreads) {
    const double li = dd[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = dd[j];
      rank += (lj > li) || (lj == li && j < i);
    }
    evals[(int64_t)p * stride_out + rank] = li;
    perm[(int64_t)p * stride_out + rank] = i;
  }
  for (int j = wid; j < n; j += kTriWarps)
    for (int i = lane; i < n; i += 32) V[(int64_t)j * n + i] = A[(int64_t)j * ldz + i];
  if (tid == 0) status[p] = s_fail ? -1 : s_iters;
}

size_t syev_smem(int nmax) {
  const size_t vec = (size_t)(9 + kTriWarps) * nmax * 8 + 64;
  return nmax > kEigSmemMax ? vec : (size_t)nmax * (nmax | 1) * 8 + vec;
}

cudaError_t launch_syev(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns, int nprob,
                        int nmax, double* Vws, int64_t stride_v, double* VHws, double* evals, int* perm,
                        int64_t stride_out, int* status) {
  if (nprob <= 0) return cudaSuccess;
  if (nmax > kTriMax) return cudaErrorInvalidValue;
  const size_t smem = syev_smem(nmax);
  if (nmax <= kEigSmemMax) {
    cudaError_t e = cudaFuncSetAttribute(k_syev_ql<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_syev_ql<false><<<nprob, kTriThreads, smem, c.stream>>>(G, ld_in, stride_in, d_ns, Vws, stride_v, VHws, evals,
                                                             perm, stride_out, status, 60, 0);
    c.launches += 1;
    return cudaGetLastError();
  }
  // c.syev_flags: CMSVD_SYEV_COLBT=0 keeps the per-reflector back-transformation (one pass over Z per reflector),
  // CMSVD_SYEV_QLF=0 the sweep-by-sweep QL rotations instead of the fused pass (Z read and written once per 4 sweeps)
  const int col_bt = c.syev_flags;
  // in place in global memory (G is destroyed); batches sized to stay L2-resident
  cudaError_t e = cudaFuncSetAttribute(k_syev_ql<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int batch = (int)std::max<int64_t>(1, std::min<int64_t>(nprob, (int64_t)c.gl_batch_mb * (1 << 20) / ((int64_t)nmax * nmax * 8)));
  for (int p0 = 0; p0 < nprob; p0 += batch) {
    const int nb = std::min(batch, nprob - p0);
    k_syev_ql<true><<<nb, kTriThreads, smem, c.stream>>>(G + (int64_t)p0 * stride_in, ld_in, stride_in, d_ns + p0,
                                                         Vws + (int64_t)p0 * stride_v, stride_v,
                                                         VHws + (int64_t)p0 * stride_v, evals + (int64_t)p0 * stride_out,
                                                         perm + (int64_t)p0 * stride_out, stride_out, status + p0, 60,
                                                         col_bt);
    c.launches += 1;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

size_t tridiag_smem(int nmax, int kw) {
  (void)kw;
  const size_t vec = (size_t)(5 + kTriWarps) * nmax * 8 + 64;
  return nmax > kEigSmemMax ? vec : (size_t)nmax * nmax * 8 + vec;
}

// the two-problem kernel for n <= 128, except 64 < n <= 96 where two one-problem CTAs per SM of the
// register-resident kernel are 4% faster (measured, tools/eigbench.cu)
// (128 < n <= 160: problem 0 split between registers and shared memory, CMSVD_EIG_DUO160; the saving
// variant, for the greedy commits, stays on the one-problem kernel)
static bool uses_duo(const Ctx& c, int nmax) {
  return c.eig_rr && c.eig_duo && nmax <= 160 && !(nmax > 64 && nmax <= 96) && (nmax <= 128 || c.eig_duo160);
}
bool tridiag_can_save(const Ctx& c, int nmax) { return c.eig_rr && nmax <= 160 && !(nmax <= 128 && uses_duo(c, nmax)); }

// top-kw eigenvalues of nprob tridiagonals (dd, ee = e^2, Gershgorin data gsh) by bisection / multisection
static cudaError_t launch_bisect_topk(Ctx& c, int nprob, int kw, int nstride, const int* d_ns, const double* dd,
                                      const double* ee, const double* gsh, const int* cnt, double* ev) {
  cudaError_t e;
  const int64_t total = (int64_t)nprob * kw;
  const int prb = prof_begin(c, PC_BISECT);
  if (total <= kMultisectMax)
    k_multisect<<<(unsigned)((total + 3) / 4), 128, 0, c.stream>>>(nprob, kw, nstride, d_ns, dd, ee, gsh, cnt, ev);
  else
  {
    // stage the block's tridiagonals when a block spans at most kBisStage problems
    const size_t sm = (size_t)kBisStage * nstride * (2 * sizeof(double) + 2 * sizeof(float));
    const size_t smp = (size_t)kBisPStage * nstride * 2 * sizeof(double);
    if (c.bisect_p && 128 / kw + 2 <= kBisPStage && smp <= 96 * 1024) {
      e = cudaFuncSetAttribute(k_bisect_p<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp);
      if (e != cudaSuccess) return e;
      k_bisect_p<true><<<(unsigned)((total + 127) / 128), 128, smp, c.stream>>>(nprob, kw, nstride, d_ns, dd, ee, gsh,
                                                                                cnt, ev);
    } else if (c.bisect_p) {
      k_bisect_p<false><<<(unsigned)((total + 127) / 128), 128, 0, c.stream>>>(nprob, kw, nstride, d_ns, dd, ee, gsh,
                                                                                cnt, ev);
    } else if (128 / kw + 2 <= kBisStage && sm <= 96 * 1024) {
      e = cudaFuncSetAttribute(k_bisect<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      k_bisect<true><<<(unsigned)((total + 127) / 128), 128, sm, c.stream>>>(nprob, kw, nstride, d_ns, dd, ee, gsh,
                                                                             cnt, ev);
    } else {
      k_bisect<false><<<(unsigned)((total + 127) / 128), 128, 0, c.stream>>>(nprob, kw, nstride, d_ns, dd, ee, gsh,
                                                                              cnt, ev);
    }
  }
  c.launches += 1;
  prof_end(c, prb);
  return cudaGetLastError();
}

// Pipelined two-stage reduction (n <= 512, large batches).  Stage 1 (dense -> band: HBM / DMMA bound, several CTAs
// per SM) runs for the whole batch; the band chase (one CTA per SM: 139 KB of shared memory, latency bound at
// ~1.2 IPC) then runs in groups of whole CTA waves on the context's stream, and the bisection of a finished
// group (issue bound, little shared memory: co-resident with a chase CTA) on a second stream, i.e. under the
// next group's chase.  Same kernels, same per-problem arithmetic: the results are bitwise those of the
// one-stream path.  Measured on config 4 (2016 problems of n = 512): 85.2 / 84.3 / 85.0 ms per pass with 2 / 3 /
// 5 groups vs 86.0 with one stream -- the co-running bisection takes 2.2x as long and the chase is not
// faster, so the default stays one stream (CMSVD_SBR_GROUPS).  Cutting stage 1 into groups as well was
// measured slower (89.4 ms with 4 groups: a chase CTA leaves room for one stage-1 CTA per SM instead of four).
static cudaError_t launch_sbr_pipelined(Ctx& c, double* G, int64_t ld_in, int64_t stride_in, const int* d_ns,
                                        int nprob, int nmax, const double* d_thr, int kw, int nstride, double* dd,
                                        double* ee, double* gsh, int* cnt, double* trace, double* ev, int groups) {
  cudaError_t e;
  if (!c.aux_stream) {
    e = cudaStreamCreateWithFlags(&c.aux_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
  }
  for (int g = 0; g <= groups; ++g)
    if (!c.aux_ev[g]) {
      e = cudaEventCreateWithFlags(&c.aux_ev[g], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
  double* ws = (double*)c.ws[WS_SBR].p;
  const int64_t per = sbr_ws_per(nmax);
  e = launch_tridiag_sbr(c, G, ld_in, stride_in, d_ns, nprob, nmax, d_thr, kw, nstride, dd, ee, gsh, cnt, trace, ws, 1);
  if (e != cudaSuccess) return e;
  const int waves = (nprob + c.sm_count - 1) / c.sm_count;
  const int gs = (waves + groups - 1) / groups * c.sm_count;   // whole waves of one chase CTA per SM
  cudaStream_t main_stream = c.stream;
  for (int g = 0; g < groups; ++g) {
    const int p0 = g * gs, np = std::min(gs, nprob - p0);
    if (np <= 0) break;
    double* Gg = G + (int64_t)p0 * stride_in;
    const double* thr = d_thr ? d_thr + p0 : nullptr;
    double* ddg = dd + (int64_t)p0 * nstride;
    double* eeg = ee + (int64_t)p0 * nstride;
    e = launch_tridiag_sbr(c, Gg, ld_in, stride_in, d_ns + p0, np, nmax, thr, kw, nstride, ddg, eeg, gsh + 4 * (int64_t)p0,
                           cnt + p0, trace + p0, ws + (int64_t)p0 * per, 2);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(c.aux_ev[g], main_stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamWaitEvent(c.aux_stream, c.aux_ev[g], 0);
    if (e != cudaSuccess) return e;
    c.stream = c.aux_stream;
    e = launch_bisect_topk(c, np, kw, nstride, d_ns + p0, ddg, eeg, gsh + 4 * (int64_t)p0, cnt + p0,
                           ev + (int64_t)p0 * kw);
    c.stream = main_stream;
    if (e != cudaSuccess) return e;
  }
  e = cudaEventRecord(c.aux_ev[groups], c.aux_stream);
  if (e != cudaSuccess) return e;
  return cudaStreamWaitEvent(main_stream, c.aux_ev[groups], 0);
}

cudaError_t launch_tridiag_topk(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns,
                                int nprob, int nmax, const double* d_thr, int kw, double* ev, int* cnt,
                                double* trace, double* scratch, double* save, int64_t save_stride) {
  if (save && !tridiag_can_save(c, nmax)) return cudaErrorInvalidValue;
  if (nprob <= 0) return cudaSuccess;
  // n > 512 only through the two-stage reduction (cluster verification); the pair path stays <= 512
  if (nmax > kTriMax && (!c.eig_sbr || save)) return cudaErrorInvalidValue;
  const size_t smem = tridiag_smem(nmax, kw);
  const int nstride = nmax;
  double* dd = scratch;
  double* ee = dd + (size_t)nprob * nstride;
  double* gsh = ee + (size_t)nprob * nstride;
  cudaError_t e;
  const bool use_rr = c.eig_rr && nmax <= 160;
  if (!save && uses_duo(c, nmax)) {
#define DUO_LAUNCH(S_, C_, RW_, NQR_, NQR1_)                                                                        \
  do {                                                                                                              \
    const size_t sm2 = duo_smem_bytes<S_, C_, NQR_, NQR1_>();                                                       \
    e = cudaFuncSetAttribute(k_tridiag_duo<S_, C_, RW_, NQR_, NQR1_>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)sm2);                                                                             \
    if (e != cudaSuccess) return e;                                                                                 \
    k_tridiag_duo<S_, C_, RW_, NQR_, NQR1_><<<(nprob + 1) / 2, duo_threads(S_, RW_), sm2, c.stream>>>(              \
        G, ld_in, stride_in, d_ns, nprob, d_thr, kw, nstride, dd, ee, gsh, cnt, trace);                             \
  } while (0)
    if (nmax <= 32) DUO_LAUNCH(1, 2, 1, 2, 0);
    else if (nmax <= 64) DUO_LAUNCH(2, 4, 2, 6, 0);
    else if (nmax <= 96) DUO_LAUNCH(3, 6, 3, 12, 0);
    else if (nmax <= 128) DUO_LAUNCH(4, 8, 4, CMSVD_DUO128_NQR, CMSVD_DUO128_NQR1);
    else DUO_LAUNCH(5, 10, CMSVD_DUO160_RW, CMSVD_DUO160_NQR, CMSVD_DUO160_NQR1);
#undef DUO_LAUNCH
    c.launches += 1;
  } else if (use_rr) {
#define RR_LAUNCH(S_, C_)                                                                                          \
  k_tridiag_rr<S_, C_><<<nprob, kRRThreads, 0, c.stream>>>(G, ld_in, stride_in, d_ns, d_thr, kw, nstride, dd, ee, \
                                                          gsh, cnt, trace, save, save_stride)
    if (nmax <= 32) RR_LAUNCH(1, 2);
    else if (nmax <= 64) RR_LAUNCH(2, 4);
    else if (nmax <= 96) RR_LAUNCH(3, 6);
    else if (nmax <= 128) RR_LAUNCH(4, 8);
    else RR_LAUNCH(5, 10);
#undef RR_LAUNCH
    c.launches += 1;
  } else if (nmax <= kEigSmemMax) {
    e = cudaFuncSetAttribute(k_tridiag<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_tridiag<false><<<nprob, kTriThreads, smem, c.stream>>>(G, ld_in, stride_in, d_ns, d_thr, kw, nstride, dd, ee,
                                                             gsh, cnt, trace);
    c.launches += 1;
  } else if (c.eig_sbr) {
    // two-stage reduction (k_sbr.cu): dense -> band (BLAS3-shaped panels) -> tridiagonal (bulge chasing)
    e = ensure(c.ws[WS_SBR], sbr_ws_bytes(nprob, nmax));
    if (e != cudaSuccess) return e;
    // large batches of n <= 512 problems: groups of at least two CTA waves of the chase, pipelined on two streams
    const int groups = nmax <= 512 ? std::min(c.sbr_groups, nprob / (2 * c.sm_count)) : 1;
    if (groups >= 2)
      return launch_sbr_pipelined(c, const_cast<double*>(G), ld_in, stride_in, d_ns, nprob, nmax, d_thr, kw, nstride,
                                  dd, ee, gsh, cnt, trace, ev, groups);
    e = launch_tridiag_sbr(c, const_cast<double*>(G), ld_in, stride_in, d_ns, nprob, nmax, d_thr, kw, nstride, dd, ee,
                           gsh, cnt, trace, (double*)c.ws[WS_SBR].p);
    if (e != cudaSuccess) return e;
  } else {
    // in place in global memory (G is destroyed); batches sized to stay L2-resident
    e = cudaFuncSetAttribute(k_tridiag<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int batch = (int)std::max<int64_t>(1, std::min<int64_t>(nprob, (int64_t)c.gl_batch_mb * (1 << 20) / ((int64_t)nmax * nmax * 8)));
    for (int p0 = 0; p0 < nprob; p0 += batch) {
      const int nb = std::min(batch, nprob - p0);
      k_tridiag<true><<<nb, kTriThreads, smem, c.stream>>>(
          G + (int64_t)p0 * stride_in, ld_in, stride_in, d_ns + p0, d_thr ? d_thr + p0 : nullptr, kw, nstride,
          dd + (int64_t)p0 * nstride, ee + (int64_t)p0 * nstride, gsh + 4 * (int64_t)p0, cnt + p0, trace + p0);
      c.launches += 1;
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_bisect_topk(c, nprob, kw, nstride, d_ns, dd, ee, gsh, cnt, ev);
}

size_t tridiag_scratch_bytes(int nprob, int nmax) { return ((size_t)nprob * (2 * nmax + 4)) * 8; }

// ---------------------------------------------------------------------------
// Top-k eigenpairs of one symmetric n x n matrix (n <= 160), for the Alg. 3
// cluster-state commit ("incremental" update; only the top
// r eigenvectors of G are kept).  Replaces the full QL with vectors:
//   k_tridiag_rr (reflectors saved) -> k_bisect (top-k eigenvalues, 1e-13 ||T||)
//   -> k_tri_invit (inverse iteration on the tridiagonal, one warp per cluster
//      of close eigenvalues, Gram-Schmidt inside a cluster every iteration)
//   -> k_tri_backtrans (Z <- H_0 ... H_{n-3} Z, one warp per vector).
// ---------------------------------------------------------------------------
constexpr int kInvWarps = 16;
constexpr int kInvMaxK = 64;
constexpr int kInvIters = 3;  // 2 for an isolated eigenvalue
constexpr double kInvClusterTol = 1e-7;

__device__ __forceinline__ double inv_hash(unsigned j, unsigned i) {
  unsigned h = j * 0x9E3779B9u ^ (i + 0x7F4A7C15u) * 0x85EBCA6Bu;
  h ^= h >> 16; h *= 0x7FEB352Du; h ^= h >> 15; h *= 0x846CA68Bu; h ^= h >> 16;
  return (double)(h >> 8) * (2.0 / 16777216.0) - 1.0;
}

// d[n], e[n-1] signed off-diagonal; ev[kw] non-increasing; Z (n x kw, ld n) unit eigenvectors of the
// tridiagonal.  Per-warp LU factors and iterate live in shared memory (dynamic, kInvWarps * 6 * n doubles).
__global__ void __launch_bounds__(kInvWarps * 32) k_tri_invit(int n, int kw, const double* __restrict__ d,
                                                              const double* __restrict__ e,
                                                              const double* __restrict__ ev,
                                                              const double* __restrict__ gsh, double* __restrict__ Z) {
  extern __shared__ double inv_smem[];
  __shared__ int cl[kInvMaxK + 1];
  __shared__ int ncl;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double nrm = gsh[3];
  double* ds_ = inv_smem + (size_t)kInvWarps * 6 * n;  // the tridiagonal, staged once
  double* es_ = ds_ + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ds_[i] = d[i];
    es_[i] = i + 1 < n ? e[i] : 0.0;
  }
  if (threadIdx.x == 0) {
    // clusters: consecutive eigenvalues closer than kInvClusterTol ||T|| (LAPACK dstein uses 1e-3; the
    // commit stores the basis in fp32, and vectors of eigenvalues further apart than 1e-7 ||T|| come out
    // orthogonal to ~1e-13 / 1e-7 per iteration without Gram-Schmidt)
    int c = 0;
    cl[0] = 0;
    for (int j = 1; j < kw; ++j)
      if (ev[j - 1] - ev[j] > kInvClusterTol * nrm) cl[++c] = j;
    cl[++c] = kw;
    ncl = c;
  }
  __syncthreads();
  double* u0 = inv_smem + (size_t)wid * 6 * n;  // 1 / pivot
  double* u1 = u0 + n;
  double* u2 = u1 + n;
  double* ml = u2 + n;
  double* pv = ml + n;
  double* x = pv + n;
  const double tiny = 2.2204460492503131e-16 * nrm;
#ifdef CMSVD_INV_PROF
  const long long t_start = clock64();
#endif
  for (int c = blockIdx.x * kInvWarps + wid; c < ncl; c += gridDim.x * kInvWarps) {
    const int iters = cl[c + 1] - cl[c] > 1 ? kInvIters : kInvIters - 1;
    double xjm = 0.0;
    for (int j = cl[c]; j < cl[c + 1]; ++j) {
      double xj = ev[j];
      const double pertol = 10.0 * 2.2204460492503131e-16 * fmax(fabs(xj), nrm * 1e-3);
      if (j > cl[c] && xjm - xj < pertol) xj = xjm - pertol;
      xjm = xj;
      if (lane == 0) {
        // T - xj I = P L U, partial pivoting (rows k, k+1); U has up to two super-diagonals
        double w0 = ds_[0] - xj, w1 = es_[0];
#pragma unroll 4
        for (int k = 0; k + 1 < n; ++k) {
          const double ck = es_[k], ak1 = ds_[k + 1] - xj, bk1 = es_[k + 1];
          if (fabs(w0) >= fabs(ck)) {
            if (fabs(w0) < tiny) w0 = w0 >= 0.0 ? tiny : -tiny;
            const double r = rcp_nr(w0);
            const double mlt = ck * r;
            u0[k] = r; u1[k] = w1; u2[k] = 0.0; ml[k] = mlt; pv[k] = 0.0;
            w0 = fma(-mlt, w1, ak1);
            w1 = bk1;
          } else {
            const double r = rcp_nr(ck);
            const double mlt = w0 * r;
            u0[k] = r; u1[k] = ak1; u2[k] = bk1; ml[k] = mlt; pv[k] = 1.0;
            w0 = fma(-mlt, ak1, w1);
            w1 = -mlt * bk1;
          }
        }
        if (fabs(w0) < tiny) w0 = w0 >= 0.0 ? tiny : -tiny;
        u0[n - 1] = rcp_nr(w0);
      }
      for (int i = lane; i < n; i += 32) x[i] = inv_hash((unsigned)j, (unsigned)i);
      __syncwarp();
      for (int it = 0; it < iters; ++it) {
        if (lane == 0) {
          // forward: P, L
          double cur = x[0];
#pragma unroll 4
          for (int k = 0; k + 1 < n; ++k) {
            double nx = x[k + 1];
            if (pv[k] != 0.0) { const double t = cur; cur = nx; nx = t; }
            x[k] = cur;
            cur = fma(-ml[k], cur, nx);
          }
          // back substitution with U
          double x1 = cur * u0[n - 1], x2 = 0.0;
          x[n - 1] = x1;
#pragma unroll 4
          for (int k = n - 2; k >= 0; --k) {
            const double xk = fma(-u2[k], x2, fma(-u1[k], x1, x[k])) * u0[k];
            x[k] = xk;
            x2 = x1; x1 = xk;
          }
        }
        __syncwarp();
        // Gram-Schmidt against the cluster's earlier vectors, then normalise
        for (int q = cl[c]; q < j; ++q) {
          const double* zq = Z + (size_t)q * n;
          double t = 0.0;
          for (int i = lane; i < n; i += 32) t = fma(x[i], zq[i], t);
          t = warp_sum(t);
          for (int i = lane; i < n; i += 32) x[i] = fma(-t, zq[i], x[i]);
        }
        double ss = 0.0, mx = 0.0;
        for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(x[i]));
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
        for (int i = lane; i < n; i += 32) { x[i] *= sc; ss = fma(x[i], x[i], ss); }
        ss = warp_sum(ss);
        const double inv = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
        for (int i = lane; i < n; i += 32) x[i] *= inv;
        __syncwarp();
      }
      double* zj = Z + (size_t)j * n;
      for (int i = lane; i < n; i += 32) zj[i] = x[i];
#ifdef CMSVD_INV_PROF
      if (lane == 0) printf("invit: cluster %d/%d (size %d) vec %d: %lld cycles since start\n", c, ncl,
                            cl[c + 1] - cl[c], j, (long long)(clock64() - t_start));
#endif
      __threadfence_block();
      __syncwarp();
    }
  }
}

// Z (n x kw, ld n) <- H_0 H_1 ... H_{n-3} Z; VH column k = v_k, tau[k].  n <= 160.  Reflectors are
// staged into shared memory 32 at a time (dynamic: 32 * n doubles); one warp per column of Z.
__global__ void __launch_bounds__(kInvWarps * 32) k_tri_backtrans(int n, int kw, const double* __restrict__ VH,
                                                                  const double* __restrict__ tau,
                                                                  double* __restrict__ Z) {
  extern __shared__ double bt_smem[];
  __shared__ double st[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ncol = (kw + kInvWarps - 1) / kInvWarps;  // columns per warp (kw <= 64: at most 4)
  double z[4][5];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc)
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int j = wid + kInvWarps * cc, i = lane + 32 * s;
      z[cc][s] = (cc < ncol && j < kw && i < n) ? Z[(size_t)j * n + i] : 0.0;
    }
  for (int k1 = n - 3; k1 >= 0; k1 -= 32) {
    const int k0 = max(k1 - 31, 0);
    __syncthreads();
    for (int t = threadIdx.x; t < (k1 - k0 + 1) * n; t += blockDim.x) bt_smem[t] = VH[(size_t)k0 * n + t];
    if (threadIdx.x <= k1 - k0) st[threadIdx.x] = tau[k0 + threadIdx.x];
    __syncthreads();
    for (int k = k1; k >= k0; --k) {
      const double tk = st[k - k0];
      if (tk == 0.0) continue;
      const double* v = bt_smem + (size_t)(k - k0) * n;
      double vr[5];
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int i = lane + 32 * s;
        vr[s] = (i > k && i < n) ? v[i] : 0.0;
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        if (cc < ncol) {
          double t = 0.0;
#pragma unroll
          for (int s = 0; s < 5; ++s) t = fma(vr[s], z[cc][s], t);
          t = warp_sum(t) * tk;
#pragma unroll
          for (int s = 0; s < 5; ++s) z[cc][s] = fma(-t, vr[s], z[cc][s]);
        }
      }
    }
  }
#pragma unroll
  for (int cc = 0; cc < 4; ++cc)
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int j = wid + kInvWarps * cc, i = lane + 32 * s;
      if (cc < ncol && j < kw && i < n) Z[(size_t)j * n + i] = z[cc][s];
    }
}

cudaError_t launch_topk_vectors(Ctx& c, int n, int kw, const double* d, const double* save, const double* ev,
                                const double* gsh, double* Z) {
  if (n < 1 || n > 160 || kw < 1 || kw > kInvMaxK || kw > n) return cudaErrorInvalidValue;
  const int sm_inv = (kInvWarps * 6 + 2) * n * 8, sm_bt = 32 * n * 8;
  cudaError_t e = cudaFuncSetAttribute(k_tri_invit, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_inv);
  if (e != cudaSuccess) return e;
  k_tri_invit<<<(kw + kInvWarps - 1) / kInvWarps, kInvWarps * 32, sm_inv, c.stream>>>(n, kw, d, save + (size_t)n * n + n,
                                                                                     ev, gsh, Z);
  k_tri_backtrans<<<1, kInvWarps * 32, sm_bt, c.stream>>>(n, kw, save, save + (size_t)n * n, Z);
  c.launches += 2;
  return cudaGetLastError();
}

size_t syev_topk_scratch_bytes(int n, int kw) {
  (void)kw;
  return ((size_t)n * n + 2 * n + 2 * n + 4 + 8) * 8 + 64;
}

cudaError_t launch_syev_topk(Ctx& c, const double* G, int n, const int* d_n, int kw, double* Z, double* evals,
                             double* scratch) {
  if (n < 1 || n > 160 || kw < 1 || kw > kInvMaxK || kw > n) return cudaErrorInvalidValue;
  double* save = scratch;
  double* dd = save + (size_t)n * n + 2 * n;
  double* ee = dd + n;
  double* gsh = ee + n;
  double* trace = gsh + 4;
  int* cnt = (int*)(trace + 1);
#define RRS_LAUNCH(S_, C_)                                                                                           \
  k_tridiag_rr<S_, C_><<<1, kRRThreads, 0, c.stream>>>(G, n, (int64_t)n * n, d_n, nullptr, kw, n, dd, ee, gsh, cnt, \
                                                      trace, save)
  if (n <= 32) RRS_LAUNCH(1, 2);
  else if (n <= 64) RRS_LAUNCH(2, 4);
  else if (n <= 96) RRS_LAUNCH(3, 6);
  else if (n <= 128) RRS_LAUNCH(4, 8);
  else RRS_LAUNCH(5, 10);
#undef RRS_LAUNCH
  k_multisect<<<(unsigned)((kw + 3) / 4), 128, 0, c.stream>>>(1, kw, n, d_n, dd, ee, gsh, cnt, evals);
  const int sm_inv = (kInvWarps * 6 + 2) * n * 8, sm_bt = 32 * n * 8;
  cudaError_t e = cudaFuncSetAttribute(k_tri_invit, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_inv);
  if (e != cudaSuccess) return e;
  k_tri_invit<<<(kw + kInvWarps - 1) / kInvWarps, kInvWarps * 32, sm_inv, c.stream>>>(n, kw, dd, save + (size_t)n * n + n, evals, gsh, Z);
  k_tri_backtrans<<<1, kInvWarps * 32, sm_bt, c.stream>>>(n, kw, save, save + (size_t)n * n, Z);
  c.launches += 4;
  return cudaGetLastError();
}

}  // namespace cmsvd

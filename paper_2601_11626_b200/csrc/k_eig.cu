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
#include "common.cuh"
#include "kernels.cuh"

namespace cmsvd {

// ---------------------------------------------------------------------------
// Two-sided cyclic Jacobi with vectors.
// G: n x n fp64 (ld_in) per problem; V: n x n fp64 workspace per problem (ld n);
// outputs: evals[p*n + l] sorted non-increasing, perm[p*n + l] = column of V
// holding the l-th eigenvector.  status[p] = sweeps used, or -1 on no
// convergence.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_syev_jacobi(const double* __restrict__ Gin, int64_t ld_in,
                                                          int64_t stride_in, const int* __restrict__ ns,
                                                          double* __restrict__ Vws, int64_t stride_v,
                                                          double* __restrict__ evals, int* __restrict__ perm,
                                                          int64_t stride_out, int* __restrict__ status,
                                                          int max_sweeps) {
  extern __shared__ double sm[];
  const int p = blockIdx.x;
  const int n = ns[p];
  const int ld = n | 1;
  double* G = sm;                         // n x ld
  const int ne = n + (n & 1);             // even player count (dummy = n)
  double* rc = G + (int64_t)n * ld;       // cs per pair
  double* rs = rc + ne / 2;               // sn per pair
  double* ra = rs + ne / 2;               // new a
  double* rb = ra + ne / 2;               // new b
  int* rp = reinterpret_cast<int*>(rb + ne / 2);
  int* rq = rp + ne / 2;
  __shared__ int rotated;
  __shared__ double scale_s;
  double* V = Vws + (int64_t)p * stride_v;
  const double* Gp = Gin + (int64_t)p * stride_in;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e % n, j = e / n;
    G[(int64_t)j * ld + i] = Gp[(int64_t)j * ld_in + i];
    V[(int64_t)j * n + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fmax(s, fabs(G[(int64_t)i * ld + i]));
    scale_s = s;
  }
  __syncthreads();
  const double floor_abs = 64.0 * 2.220446049250313e-16 * scale_s;
  int sweep = 0;
  bool converged = (n <= 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int t = 0; t < ne - 1; ++t) {
      // pairs of this round (circle method)
      for (int k = threadIdx.x; k < ne / 2; k += blockDim.x) {
        int a, b;
        if (k == 0) { a = 0; b = (t % (ne - 1)) + 1; }
        else { a = ((k + t) % (ne - 1)) + 1; b = ((ne - 1 - k + t) % (ne - 1)) + 1; }
        if (a > b) { int x = a; a = b; b = x; }
        double cs = 1.0, sn = 0.0, na = 0.0, nb = 0.0;
        int pa = -1, pb = -1;
        if (b < n) {
          double ga = G[(int64_t)a * ld + a], gb = G[(int64_t)b * ld + b], gc = G[(int64_t)b * ld + a];
          double thr = fmax(1e-14 * sqrt(fabs(ga * gb)), floor_abs);
          if (fabs(gc) > thr) {
            double zeta = (gb - ga) / (2.0 * gc);
            double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            cs = 1.0 / sqrt(1.0 + tt * tt);
            sn = cs * tt;
            na = ga - tt * gc;
            nb = gb + tt * gc;
            pa = a; pb = b;
            rotated = 1;
          }
        }
        rc[k] = cs; rs[k] = sn; ra[k] = na; rb[k] = nb; rp[k] = pa; rq[k] = pb;
      }
      __syncthreads();
      // rows: G[a][j], G[b][j]
      const int np = ne / 2;
      for (int e = threadIdx.x; e < np * n; e += blockDim.x) {
        int k = e / n, j = e % n;
        int a = rp[k];
        if (a < 0) continue;
        int b = rq[k];
        double cs = rc[k], sn = rs[k];
        double ga = G[(int64_t)j * ld + a], gb = G[(int64_t)j * ld + b];
        G[(int64_t)j * ld + a] = cs * ga - sn * gb;
        G[(int64_t)j * ld + b] = sn * ga + cs * gb;
      }
      __syncthreads();
      // columns: G[i][a], G[i][b] and V[:, a], V[:, b]
      for (int e = threadIdx.x; e < np * n; e += blockDim.x) {
        int k = e / n, i = e % n;
        int a = rp[k];
        if (a < 0) continue;
        int b = rq[k];
        double cs = rc[k], sn = rs[k];
        double ga = G[(int64_t)a * ld + i], gb = G[(int64_t)b * ld + i];
        G[(int64_t)a * ld + i] = cs * ga - sn * gb;
        G[(int64_t)b * ld + i] = sn * ga + cs * gb;
        double va = V[(int64_t)a * n + i], vb = V[(int64_t)b * n + i];
        V[(int64_t)a * n + i] = cs * va - sn * vb;
        V[(int64_t)b * n + i] = sn * va + cs * vb;
      }
      __syncthreads();
      for (int k = threadIdx.x; k < np; k += blockDim.x) {
        int a = rp[k];
        if (a < 0) continue;
        int b = rq[k];
        G[(int64_t)a * ld + a] = ra[k];
        G[(int64_t)b * ld + b] = rb[k];
        G[(int64_t)b * ld + a] = 0.0;
        G[(int64_t)a * ld + b] = 0.0;
      }
      __syncthreads();
    }
    converged = (rotated == 0);
    __syncthreads();
  }
  // sort eigenvalues non-increasing (ties: smaller index first)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double li = G[(int64_t)i * ld + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      double lj = G[(int64_t)j * ld + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    evals[(int64_t)p * stride_out + rank] = li;
    perm[(int64_t)p * stride_out + rank] = i;
  }
  if (threadIdx.x == 0) status[p] = converged ? sweep : -1;
}

size_t syev_jacobi_smem(int nmax) {
  int ld = nmax | 1;
  int ne = nmax + (nmax & 1);
  return (size_t)nmax * ld * 8 + (size_t)(ne / 2) * (4 * 8 + 2 * 4) + 64;
}

cudaError_t launch_syev_jacobi(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns, int nprob,
                               int nmax, double* Vws, int64_t stride_v, double* evals, int* perm, int64_t stride_out,
                               int* status) {
  size_t smem = syev_jacobi_smem(nmax);
  cudaError_t e = cudaFuncSetAttribute(k_syev_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_syev_jacobi<<<nprob, kThreads, smem, c.stream>>>(G, ld_in, stride_in, d_ns, Vws, stride_v, evals, perm,
                                                      stride_out, status, 60);
  c.launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Householder tridiagonalisation + Sturm multisection, values only.
// Problem p: n = ns[p] (0 allowed), matrix at Gin + p*stride_in (ld_in),
// wants the kw largest eigenvalues that are > thr[p] (thr may be NULL: all).
// Outputs: ev[p*kw + l] (non-increasing; entries not computed are 0),
// cnt[p] = number of eigenvalues > thr (capped at kw), trace[p] = sum of the
// diagonal (fixed order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += (q < 0.0);
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
  }
  return cnt;
}

__global__ void __launch_bounds__(kThreads) k_tridiag_topk(const double* __restrict__ Gin, int64_t ld_in,
                                                           int64_t stride_in, const int* __restrict__ ns,
                                                           const double* __restrict__ thr, int kw,
                                                           double* __restrict__ ev, int* __restrict__ cnt_out,
                                                           double* __restrict__ trace_out) {
  extern __shared__ double sm[];
  const int p = blockIdx.x;
  const int n = ns[p];
  const int ld = n | 1;
  double* A = sm;                         // n x ld
  double* v = A + (int64_t)n * ld;        // n
  double* pw = v + n;                     // n
  double* d = pw + n;                     // n
  double* e2 = d + n;                     // n
  double* lo = e2 + n;                    // kw
  double* hi = lo + kw;                   // kw
  int* cnts = reinterpret_cast<int*>(hi + kw);  // blockDim.x
  __shared__ double red[kThreads / 32];
  __shared__ double s_tau, s_K;
  __shared__ int s_k, s_done;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Gp = Gin + (int64_t)p * stride_in;
  if (n <= 0) {
    if (threadIdx.x == 0) { cnt_out[p] = 0; trace_out[p] = 0.0; }
    for (int l = threadIdx.x; l < kw; l += blockDim.x) ev[(int64_t)p * kw + l] = 0.0;
    return;
  }
  for (int j = wid; j < n; j += nw)
    for (int i = lane; i < n; i += 32) A[(int64_t)j * ld + i] = Gp[(int64_t)j * ld_in + i];
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed-order trace (deterministic)
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += A[(int64_t)i * ld + i];
    trace_out[p] = s;
  }
  // ---- tridiagonalisation ----
  for (int k = 0; k + 2 < n; ++k) {
    const int s = n - 1 - k;
    const double* x = A + (int64_t)k * ld + (k + 1);   // column k, rows k+1..n-1
    if (wid == 0) {
      double t = 0.0;
      for (int i = 1 + lane; i < s; i += 32) t += x[i] * x[i];
      t = warp_sum(t);
      double alpha = x[0];
      if (lane == 0) {
        if (t == 0.0) {
          s_tau = 0.0;
          e2[k] = alpha * alpha;
        } else {
          double xn = sqrt(alpha * alpha + t);
          double beta = alpha >= 0.0 ? -xn : xn;
          s_tau = (beta - alpha) / beta;
          s_K = 1.0 / (alpha - beta);   // temporary: scale for v
          e2[k] = beta * beta;
        }
      }
      __syncwarp();
    }
    __syncthreads();
    const double tau = s_tau;
    if (tau == 0.0) continue;
    const double sc = s_K;
    for (int i = threadIdx.x; i < s; i += blockDim.x) v[i] = (i == 0) ? 1.0 : x[i] * sc;
    __syncthreads();
    // p = tau * A_trail v
    double* At = A + (int64_t)(k + 1) * ld + (k + 1);
    for (int j = wid; j < s; j += nw) {
      const double* col = At + (int64_t)j * ld;
      double t = 0.0;
      for (int i = lane; i < s; i += 32) t = fma(col[i], v[i], t);
      t = warp_sum(t);
      if (lane == 0) pw[j] = tau * t;
    }
    __syncthreads();
    if (wid == 0) {
      double t = 0.0;
      for (int i = lane; i < s; i += 32) t = fma(pw[i], v[i], t);
      t = warp_sum(t);
      if (lane == 0) s_K = 0.5 * tau * t;
      __syncwarp();
    }
    __syncthreads();
    const double Kc = s_K;
    for (int i = threadIdx.x; i < s; i += blockDim.x) pw[i] -= Kc * v[i];
    __syncthreads();
    for (int j = wid; j < s; j += nw) {
      double* col = At + (int64_t)j * ld;
      const double vj = v[j], wj = pw[j];
      for (int i = lane; i < s; i += 32) col[i] -= v[i] * wj + pw[i] * vj;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = A[(int64_t)i * ld + i];
  if (threadIdx.x == 0 && n >= 2) {
    double t = A[(int64_t)(n - 2) * ld + (n - 1)];
    e2[n - 2] = t * t;
  }
  __syncthreads();
  // ---- Gershgorin bounds, pivmin, count above threshold ----
  if (threadIdx.x == 0) {
    double glo = 1e300, ghi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      double r = 0.0;
      if (i > 0) r += sqrt(e2[i - 1]);
      if (i + 1 < n) r += sqrt(e2[i]);
      glo = fmin(glo, d[i] - r);
      ghi = fmax(ghi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    double nrm = fmax(fabs(glo), fabs(ghi));
    double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax);
    glo -= 2.2e-16 * nrm * n + pivmin;
    ghi += 2.2e-16 * nrm * n + pivmin;
    red[0] = glo; red[1] = ghi; red[2] = pivmin; red[3] = nrm;
    int above = n;
    if (thr) {
      double t = thr[p];
      if (t > glo) above = n - sturm_count(d, e2, n, t, pivmin);
      if (t >= ghi) above = 0;
    }
    s_k = min(kw, above);
  }
  __syncthreads();
  const double glo = red[0], ghi = red[1], pivmin = red[2], nrm = red[3];
  const int k = s_k;
  for (int l = threadIdx.x; l < kw; l += blockDim.x) {
    lo[l] = glo; hi[l] = ghi;
    if (l >= k) ev[(int64_t)p * kw + l] = 0.0;
  }
  if (threadIdx.x == 0) cnt_out[p] = k;
  __syncthreads();
  if (k == 0) return;
  // ---- multisection: T threads per eigenvalue, eigenvalues in batches ----
  const double tol_abs = 4.0 * 2.220446049250313e-16 * nrm;
  for (int base = 0; base < k; base += blockDim.x) {
    const int kk = min((int)blockDim.x, k - base);
    const int T = blockDim.x / kk;
    const int l = base + threadIdx.x / T, sidx = threadIdx.x % T;
    const bool active = (threadIdx.x / T) < kk;
    for (int it = 0; it < 200; ++it) {
      if (threadIdx.x == 0) s_done = 1;
      __syncthreads();
      int c = -1;
      if (active) {
        double a = lo[l], b = hi[l];
        if (b - a > tol_abs + 4.0 * 2.220446049250313e-16 * fmax(fabs(a), fabs(b))) {
          double x = a + (b - a) * (double)(sidx + 1) / (double)(T + 1);
          c = sturm_count(d, e2, n, x, pivmin);
          s_done = 0;
        }
      }
      cnts[threadIdx.x] = c;
      __syncthreads();
      if (s_done) break;
      if (active && sidx == 0 && c >= 0) {
        // target ascending index a = n-1-l: N(x) <= a  <=>  x <= lambda_a
        const int target = n - 1 - l;
        const double a = lo[l], b = hi[l];
        double na = a, nb = b;
        const int t0 = threadIdx.x;
        for (int s2 = 0; s2 < T; ++s2) {
          double xs = a + (b - a) * (double)(s2 + 1) / (double)(T + 1);
          if (cnts[t0 + s2] <= target) na = xs;
          else { nb = xs; break; }
        }
        lo[l] = na; hi[l] = nb;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < k; q += blockDim.x) ev[(int64_t)p * kw + q] = 0.5 * (lo[q] + hi[q]);
}

size_t tridiag_smem(int nmax, int kw) {
  int ld = nmax | 1;
  return (size_t)nmax * ld * 8 + (size_t)4 * nmax * 8 + (size_t)2 * kw * 8 + kThreads * 4 + 64;
}

cudaError_t launch_tridiag_topk(Ctx& c, const double* G, int64_t ld_in, int64_t stride_in, const int* d_ns,
                                int nprob, int nmax, const double* d_thr, int kw, double* ev, int* cnt,
                                double* trace) {
  if (nprob <= 0) return cudaSuccess;
  size_t smem = tridiag_smem(nmax, kw);
  cudaError_t e = cudaFuncSetAttribute(k_tridiag_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_tridiag_topk<<<nprob, kThreads, smem, c.stream>>>(G, ld_in, stride_in, d_ns, d_thr, kw, ev, cnt, trace);
  c.launches += 1;
  return cudaGetLastError();
}

}  // namespace cmsvd

// k_sbr.cu -- two-stage Householder tridiagonalisation of the large core Grams (160 < n <= 512:
// configs 3 and 4, n = r' + w = 256 / 512), the values path of Cor. 3's eigendecomposition
// (sigma~^2 = the top-r eigenvalues of the core Gram).
//
// The one-stage reduction applies a rank-2 update to the whole trailing matrix per column: at n = 512
// the 1 MB lower triangle of every problem is streamed from HBM 510 times (358 MB per problem).  Here:
//   stage 1 (dense -> band of half-bandwidth kSB = 16, "successive band reduction"), per panel t
//     (columns c0 = 16 t .. c0 + 15, trailing block A22 = rows/cols R0 = c0 + 16 .. n - 1):
//       k_sbr_panel  : Householder QR of the n_p x 16 panel below the band (n_p = n - R0), one CTA per
//                      problem in shared memory; V (unit lower trapezoidal), T of the compact WY form
//                      Q = I - V T V^T (LAPACK's larft recurrence), R written into the band;
//       k_sbr_symm   : Y = A22 V T (A22 read once per 128-row block as a symmetric row panel), per-block
//                      partials M_b = V_b^T Y_b;
//       k_sbr_syr2k  : A22 <- Q^T A22 Q = A22 - V W^T - W V^T with W = Y - 1/2 V (T^T sum_b M_b)
//                      (lower 64 x 64 tiles; W formed per tile from Y, V and the 16 x 16 partials);
//     so the trailing matrix is streamed ~2x per 16 columns instead of once per column, in BLAS3-shaped
//     register-tiled fp64 passes;
//   stage 2 (band -> tridiagonal by bulge chasing), k_sbr_chase: one CTA per problem, band (lower, with
//     room for the bulge: 2 kSB + 1 diagonals) in shared memory.  Sweep j annihilates column j below the
//     subdiagonal with a length-16 Householder H_0 (two-sided on the diagonal block, right-applied to the
//     block below, which fills it); step s >= 1 annihilates the first column of that fill with H_s
//     (left-applied to it, two-sided on the next diagonal block, right-applied to the next block).
//     One warp per sweep; sweep j may run step s once sweep j-1 has finished step s + 2 (the blocks the
//     two touch are then disjoint), tracked by per-sweep progress counters in shared memory.
// Outputs: those of k_tridiag (diagonal, squared sub-diagonal, Gershgorin data, count above the
// threshold, trace) so that the same bisection kernels follow.
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "engine.h"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace cmsvd {

#ifndef CMSVD_CHASE_SLEEP
#define CMSVD_CHASE_SLEEP 0
#endif

constexpr int kSB = 16;                 // band half-width of stage 1
constexpr int kSBMax = 512;             // largest n with the panel and the band in shared memory (pair path)
constexpr int kSBBig = 4096;            // largest n (cluster verification, global-memory panel and band)
constexpr int kSBLdb = 2 * kSB + 2;     // band storage: diagonals 0 .. 2 kSB (band + bulge), padded so that a
                                        // row walk (stride kSBLdb - 1 doubles) is free of bank conflicts
constexpr int kSymmRows = 128;          // rows of A22 per k_sbr_symm CTA
constexpr int kSymmJB = 32;             // columns staged per k_sbr_symm step
constexpr int kSymmThreads = 128;
constexpr int kSyrTile = 64;            // k_sbr_syr2k tile
constexpr int kSyrThreads = 256;
constexpr int kPanelThreads = 256;
constexpr int kChaseWarps = 12;

// workspace per problem (doubles): two sets (panel parity t & 1) of [V (ldv x kSB) | Y/W (ldv x kSB) | T
// (kSB x kSB)], the M partials (ceil(ldv/128) x kSB x kSB), the fused pass's product partials (one 2 x 64 x kSB
// slot per lower 64 x 64 tile), and for n > kSBMax the band of the chase (n x kSBLdb, global memory)
struct SbrWs {
  int ldv;            // rows of V and Y per problem (kSBMax for n <= kSBMax, else n rounded up to 128)
  int ntm;            // 64-row tiles per side
  int64_t per;        // doubles per problem
  int64_t set;        // doubles per V / W / T set
  int64_t moff;       // offset of the M partials
  int64_t poff;       // offset of the product partials
  int64_t band;       // offset of the global-memory band (0: band in shared memory)
  __host__ __device__ int64_t vsz() const { return (int64_t)ldv * kSB; }
  __host__ __device__ double* vp(double* ws, int p, int par) const { return ws + (int64_t)p * per + par * set; }
  __host__ __device__ double* mp(double* ws, int p) const { return ws + (int64_t)p * per + moff; }
};
static SbrWs sbr_layout(int nmax) {
  SbrWs L;
  L.ldv = nmax <= kSBMax ? kSBMax : (nmax + 127) / 128 * 128;
  L.ntm = (L.ldv + 63) / 64;
  const int64_t nmb = (L.ldv + kSymmRows - 1) / kSymmRows;
  L.set = (2 * L.vsz() + kSB * kSB + 15) / 16 * 16;
  L.moff = 2 * L.set;
  L.poff = L.moff + nmb * kSB * kSB;
  L.per = L.poff + (int64_t)L.ntm * (L.ntm + 1) / 2 * 2 * 64 * kSB;
  L.band = 0;
  if (nmax > kSBMax) {
    L.band = L.per;
    L.per += (int64_t)nmax * kSBLdb;
  }
  L.per = (L.per + 15) / 16 * 16;   // 128-byte problem stride (TMA alignment)
  return L;
}

__device__ __forceinline__ double sbr_rcp(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  double e = fma(-q, y, 1.0);
  y = fma(y, e, y);
  e = fma(-q, y, 1.0);
  return fma(y, e, y);
}

// number of stage-1 panels of an n x n problem: panel t exists while at least 2 rows lie below its band
__host__ __device__ __forceinline__ int sbr_panels(int n) { return n >= kSB + 2 ? (n - kSB - 2) / kSB + 1 : 0; }

// ---------------------------------------------------------------------------
// Stage 1a: panel QR.  Panel t of problem p: P = A[R0 .. n-1, c0 .. c0+15] (n_p x 16).
// ---------------------------------------------------------------------------
constexpr int kPanelLd = kSBMax + 1;   // column stride of the staged panel (odd: conflict-free columns)

template <bool SMEM>
__global__ void __launch_bounds__(kPanelThreads) k_sbr_panel(double* __restrict__ G, int64_t ld, int64_t stride,
                                                              const int* __restrict__ ns, int t,
                                                              double* __restrict__ ws, double* __restrict__ trace,
                                                              const SbrWs L, int par) {
  extern __shared__ __align__(16) double psm[];
  // SMEM: the panel is staged in shared memory ([kSB][kPanelLd]); else (n > kSBMax) it is factored in place
  // in global memory (its entries below the band hold the reflectors afterwards, which the band never reads)
  constexpr int kPld = SMEM ? kPanelLd : 0;
  double* red = psm + (SMEM ? kSB * kPanelLd : 0);   // [16][16] partial sums
  double* scal = red + 256;                          // beta, tau per column; S (16 x 16), T (16 x 16)
  double* S = scal + 2 * kSB;
  double* T = S + kSB * kSB;
  const int p = blockIdx.x;
  const int n = ns[p];
  const int tid = threadIdx.x;
  double* A = G + (int64_t)p * stride;
  if (t == 0 && tid == 0) {   // trace of the original matrix (invariant, kept for the finalisation)
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += A[(int64_t)i * ld + i];
    trace[p] = s;
  }
  if (t >= sbr_panels(n)) return;
  const int c0 = t * kSB, R0 = c0 + kSB, np = n - R0;
  double* P = SMEM ? psm : A + (int64_t)c0 * ld + R0;
  const int64_t ldp = SMEM ? (int64_t)kPld : ld;
  if (SMEM) {   // stage the panel
    for (int e = tid; e < kSB * np; e += kPanelThreads) {
      const int c = e / np, i = e - c * np;
      P[c * ldp + i] = A[(int64_t)(c0 + c) * ld + R0 + i];
    }
  }
  __syncthreads();
  const int g = tid >> 4, cc = tid & 15;   // 16 row groups x 16 columns
  const int kmax = min(kSB, np);
  for (int k = 0; k < kmax; ++k) {
    double* x = P + k * ldp;
    // squared norm below the diagonal element
    double part = 0.0;
    for (int i = k + 1 + tid; i < np; i += kPanelThreads) part = fma(x[i], x[i], part);
    part = warp_sum(part);
    if ((tid & 31) == 0) red[tid >> 5] = part;
    __syncthreads();
    double sig2 = 0.0;
#pragma unroll
    for (int q = 0; q < kPanelThreads / 32; ++q) sig2 += red[q];
    const double alpha = x[k];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (sig2 > 0.0) {
      const double xn = sqrt(fma(alpha, alpha, sig2));
      beta = alpha >= 0.0 ? -xn : xn;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();   // red reused below
    for (int i = k + 1 + tid; i < np; i += kPanelThreads) x[i] *= scale;
    if (tid == 0) { x[k] = beta; scal[k] = tau; }
    __syncthreads();
    // s_c = tau (P[k][c] + sum_{i>k} v_i P[i][c]) for c > k, then P[i][c] -= s_c v_i (v_k = 1)
    if (tau != 0.0) {
      double d = 0.0;
      if (cc > k) {
        const double* pc = P + cc * ldp;
        if (g == 0) d = pc[k];
        for (int i = k + 1 + g; i < np; i += 16) d = fma(x[i], pc[i], d);
      }
      red[g * 16 + cc] = d;
      __syncthreads();
      if (cc > k) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += red[q * 16 + cc];
        s *= tau;
        double* pc = P + cc * ldp;
        if (g == 0) pc[k] -= s;
        for (int i = k + 1 + g; i < np; i += 16) pc[i] = fma(-s, x[i], pc[i]);
      }
      __syncthreads();
    }
  }
  // V^T V (strictly upper part needed): S[j][k] = V[k][j] + sum_{i>k} V[i][j] V[i][k], j < k
  {
    const int j = tid >> 4, k = tid & 15;
    double s = 0.0;
    if (j < k && k < kmax) {
      const double* vj = P + j * ldp;
      const double* vk = P + k * ldp;
      s = vj[k];
      for (int i = k + 1; i < np; ++i) s = fma(vj[i], vk[i], s);
    }
    S[j * kSB + k] = s;
  }
  __syncthreads();
  // T (upper triangular): T[k][k] = tau_k, T[0:k][k] = -tau_k T[0:k][0:k] S[0:k][k]
  if (tid < 32) {
    const int i = tid;
    for (int k = 0; k < kSB; ++k) {
      const double tk = k < kmax ? scal[k] : 0.0;
      double s = 0.0;
      if (i < k)
        for (int l = i; l < k; ++l) s = fma(T[i * kSB + l], S[l * kSB + k], s);
      __syncwarp();
      if (i < kSB) T[i * kSB + k] = (i < k) ? -tk * s : (i == k ? tk : 0.0);
      __syncwarp();
    }
  }
  __syncthreads();
  // outputs: R into the band (rows R0 .. R0 + 15 of the panel columns, upper triangle), V, T
  double* Vw = L.vp(ws, p, par);
  double* Tw = Vw + 2 * L.vsz();
  for (int e = tid; e < kSB * kSB; e += kPanelThreads) {
    const int c = e >> 4, k = e & 15;   // R[k][c], k <= c
    if (SMEM && k <= c && k < np) A[(int64_t)(c0 + c) * ld + R0 + k] = P[c * ldp + k];
    Tw[e] = T[e];
  }
  for (int e = tid; e < kSB * L.ldv; e += kPanelThreads) {
    const int c = e / L.ldv, i = e - c * L.ldv;
    const double v = (i >= np || i < c) ? 0.0 : (i == c ? 1.0 : P[c * ldp + i]);
    Vw[(int64_t)c * L.ldv + i] = (c < kmax) ? v : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Stage 1a, register-resident variant (n <= kSBMax; the default).  The shared-memory kernel above spends its
// time in the load/store unit (two or three shared-memory wavefronts per DFMA: 16 % of the DFMA rate) and in
// five CTA barriers per column.  Here thread tid owns ROWS tid and tid + 256 of the panel, all 16 columns in
// registers (the column loop is fully unrolled, so every register index is static); shared memory carries
// only the 8 x 16 warp totals, double-buffered: ONE barrier per column.  Per column k:
//   1. every thread: partial dots of x = P[k+1:, k] (its rows below k) with all 16 columns -- columns c > k for
//      the update, c < k for the V^T V entries that larft needs, c = k for the norm; a transposing shuffle
//      reduction leaves the warp total of column c in lanes 2 c, 2 c + 1; the owner of row k publishes that row
//                                                                                                -> barrier
//   2. every warp, lane c (and c + 16): total of column c from the 8 warp totals; every lane forms beta, tau,
//      scale (rsqrt / rcp + Newton, as in the chase) and s_c = tau (P[k][c] + scale d_c); warp 0 also stores
//      tau, scale and S[c][k] (c < k)
//   3. every thread updates its rows in registers with s_c shuffled from lane c:
//      P[i][c] -= s_c scale x_i (i > k), P[k][c] -= s_c, P[k][k] = beta
// The Householder vectors stay unscaled in the registers (v = scale x below the diagonal) until V is written.
// ---------------------------------------------------------------------------
// NT threads own rows tid and tid + NT: 256 threads for panels of up to 512 rows, 128 for up to 256, 64 for up to
// 128 (half / a quarter of the warps and of the reduction's instructions, twice / four times the CTAs per SM)
constexpr int kP3Smem = (2 * (kPanelThreads / 32) * 16 + 2 * 16 + 2 * kSB + 2 * kSB * kSB) * (int)sizeof(double);

template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_sbr_panel3(double* __restrict__ G, int64_t ld, int64_t stride,
                                                                 const int* __restrict__ ns, int t,
                                                                 double* __restrict__ ws, double* __restrict__ trace,
                                                                 const SbrWs L, int par) {
  extern __shared__ __align__(16) double psm[];
  double* wtot = psm;                       // [2][8 warps][16]
  constexpr int kP3Warps = NT / 32;
  double* rowk = wtot + 2 * kP3Warps * 16;  // [2][16] row k of the panel (published by its owner)
  double* scal = rowk + 2 * 16;             // tau per column
  double* scl = scal + kSB;                 // scale per column
  double* S = scl + kSB;                    // 16 x 16
  double* T = S + kSB * kSB;                // 16 x 16
  const int p = blockIdx.x;
  const int n = ns[p];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* A = G + (int64_t)p * stride;
  if (t == 0 && tid < 32) {   // trace of the original matrix (invariant, kept for the finalisation)
    double s = 0.0;
    for (int i = tid; i < n; i += 32) s += A[(int64_t)i * ld + i];
    s = warp_sum(s);
    if (tid == 0) trace[p] = s;
  }
  if (t >= sbr_panels(n)) return;
  const int c0 = t * kSB, R0 = c0 + kSB, np = n - R0;
  const int kmax = min(kSB, np);
  const int r0 = tid, r1 = tid + NT;
  double p0[kSB], p1[kSB];
#pragma unroll
  for (int c = 0; c < kSB; ++c) {
    const double* col = A + (int64_t)(c0 + c) * ld + R0;
    p0[c] = r0 < np ? col[r0] : 0.0;
    p1[c] = r1 < np ? col[r1] : 0.0;
  }
  for (int i = tid; i < kSB * kSB; i += NT) S[i] = 0.0;
  if (tid < kSB) { scal[tid] = 0.0; scl[tid] = 0.0; }
  __syncthreads();
  const int lc = lane & 15;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int k = 0; k < kSB; ++k) {
    if (k < kmax) {   // CTA-uniform
      double* wt = wtot + (k & 1) * kP3Warps * 16;
      double* rk = rowk + (k & 1) * 16;
      // 1. partial dots of x (rows > k of column k) with every column, reduced over the warp
      const double x0 = r0 > k ? p0[k] : 0.0;
      const double x1 = p1[k];                 // r1 >= NT > k; zero beyond np
      double v[16];
#pragma unroll
      for (int c = 0; c < kSB; ++c) v[c] = fma(x1, p1[c], x0 * p0[c]);
      double w8[8], w4[4], w2[2], w1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double keep = b4 ? v[j + 8] : v[j], send = b4 ? v[j] : v[j + 8];
        w8[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double keep = b3 ? w8[j + 4] : w8[j], send = b3 ? w8[j] : w8[j + 4];
        w4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double keep = b2 ? w4[j + 2] : w4[j], send = b2 ? w4[j] : w4[j + 2];
        w2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      {
        const double keep = b1 ? w2[1] : w2[0], send = b1 ? w2[0] : w2[1];
        w1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      w1 += __shfl_xor_sync(0xffffffffu, w1, 1);   // warp total of column lane >> 1
      if ((lane & 1) == 0) wt[wid * 16 + (lane >> 1)] = w1;
      if (tid == k) {
#pragma unroll
        for (int c = 0; c < kSB; ++c) rk[c] = p0[c];
      }
      __syncthreads();
      // 2. totals and the reflector's scalars (every warp, redundantly)
      double d = 0.0;
#pragma unroll
      for (int w = 0; w < kP3Warps; ++w) d += wt[w * 16 + lc];
      const double sig2 = __shfl_sync(0xffffffffu, d, k);
      const double alpha = rk[k];
      const double pkc = rk[lc];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (sig2 > 0.0) {
        const double x2 = fma(alpha, alpha, sig2);
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x2));
        const double e = fma(-(x2 * y), y, 1.0);
        y = fma(y * e, fma(e, 0.375, 0.5), y);
        const double xn = x2 * y;
        beta = alpha >= 0.0 ? -xn : xn;
        tau = (beta - alpha) * sbr_rcp(beta);
        scale = sbr_rcp(alpha - beta);
      }
      const double sc = tau * fma(scale, d, pkc);   // lane c > k: tau (P[k][c] + v^T P[k+1:, c])
      if (wid == 0 && lane < kSB) {
        if (lane < k) S[lane * kSB + k] = scl[lane] * fma(scale, d, pkc);   // v_c^T v_k
        else if (lane == k) { scal[k] = tau; scl[k] = scale; }
      }
      // 3. update in registers
      const double f0 = r0 > k ? scale * p0[k] : (r0 == k ? 1.0 : 0.0);   // v_i of this thread's rows
      const double f1 = scale * p1[k];
#pragma unroll
      for (int c = k + 1; c < kSB; ++c) {
        const double scc = __shfl_sync(0xffffffffu, sc, c);
        p0[c] = fma(-scc, f0, p0[c]);
        p1[c] = fma(-scc, f1, p1[c]);
      }
      if (r0 == k) p0[k] = beta;
      // (column k + 1 writes the other halves of wtot / rowk; column k + 2 reuses these after the barrier of
      // column k + 1, which every warp reaches only after its reads above)
    }
  }
  __syncthreads();
  // T (upper triangular): T[k][k] = tau_k, T[0:k][k] = -tau_k T[0:k][0:k] S[0:k][k]
  if (tid < 32) {
    const int i = tid;
    for (int k = 0; k < kSB; ++k) {
      const double tk = k < kmax ? scal[k] : 0.0;
      double s = 0.0;
      if (i < k)
        for (int l = i; l < k; ++l) s = fma(T[i * kSB + l], S[l * kSB + k], s);
      __syncwarp();
      if (i < kSB) T[i * kSB + k] = (i < k) ? -tk * s : (i == k ? tk : 0.0);
      __syncwarp();
    }
  }
  __syncthreads();
  // outputs: R into the band (rows R0 .. R0 + 15 of the panel columns, upper triangle), T, V (unit lower
  // trapezoidal; zero rows from np on: the set was last written by panel t - 2, whose rows from np + 2 kSB on
  // are zero already; zero columns from kmax on)
  double* Vw = L.vp(ws, p, par);
  double* Tw = Vw + 2 * L.vsz();
  for (int i = tid; i < kSB * kSB; i += NT) Tw[i] = T[i];
  const int zend = t < 2 ? L.ldv : min(L.ldv, np + 2 * kSB);
#pragma unroll
  for (int c = 0; c < kSB; ++c) {
    if (r0 < kSB && r0 <= c && r0 < np) A[(int64_t)(c0 + c) * ld + R0 + r0] = p0[c];   // R[r0][c]
    const double sc = c < kmax ? scl[c] : 0.0;
    double* vw = Vw + (int64_t)c * L.ldv;
    if (r0 < zend) vw[r0] = (c < kmax && r0 < np) ? (r0 > c ? sc * p0[c] : (r0 == c ? 1.0 : 0.0)) : 0.0;
    if (r1 < zend) vw[r1] = (c < kmax && r1 < np) ? sc * p1[c] : 0.0;
    for (int i = 2 * NT + tid; i < zend; i += NT) vw[i] = 0.0;   // rows beyond this layout (np <= 2 NT): zero
  }
}

// ---------------------------------------------------------------------------
// Stage 1b: Y = A22 V T for rows [128 b, 128 b + 128) of A22 (n_p x n_p, symmetric, lower stored),
// M_b = V_b^T Y_b.  Thread t: rows i0 = t % 64 and i0 + 64, columns 8 (t / 64) .. + 7.  The 32-column
// slices of the symmetric row panel are staged by cp.async into two buffers (the next slice's copies in
// flight during the current slice's products); slices above the diagonal are read from the lower
// storage and transposed on the way into shared memory.
// ---------------------------------------------------------------------------
constexpr int kSymmLd = kSymmRows + 1;
constexpr int kSymmBuf = kSymmJB * kSymmLd + kSymmJB * kSB;   // doubles per stage buffer

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}

__global__ void __launch_bounds__(kSymmThreads, 3) k_sbr_symm(const double* __restrict__ G, int64_t ld,
                                                                int64_t stride, const int* __restrict__ ns, int t,
                                                                double* __restrict__ ws, const SbrWs L, int par) {
  extern __shared__ __align__(16) double ssm[];
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int I0 = blockIdx.y * kSymmRows;
  if (I0 >= np) return;
  const int tid = threadIdx.x;
  const double* A = G + (int64_t)p * stride + (int64_t)R0 * ld + R0;   // A22(i, j) at A[j * ld + i]
  const double* Vw = L.vp(ws, p, par);
  double* Yw = const_cast<double*>(Vw) + L.vsz();
  const int i0 = tid & 63, h = tid >> 6;
  const int imax = min(kSymmRows, np - I0);
  // stage the slice starting at column J0 into buffer `buf` (At[j][i] = A22(I0 + i, J0 + j), Vs[j][c])
  auto stage = [&](int J0, int buf) {
    double* At = ssm + buf * kSymmBuf;
    double* Vs = At + kSymmJB * kSymmLd;
    const int jmax = min(kSymmJB, np - J0);
    if (J0 + jmax - 1 <= I0) {            // all i >= j: lower storage, contiguous in i
      for (int e = tid; e < kSymmJB * kSymmRows; e += kSymmThreads) {
        const int jj = e >> 7, ii = e & 127;
        const bool ok = jj < jmax && ii < imax;
        cp_async8(At + jj * kSymmLd + ii, ok ? A + (int64_t)(J0 + jj) * ld + I0 + ii : A, ok);
      }
    } else if (I0 + imax - 1 < J0) {      // all i < j: A22(i, j) = A22(j, i) at A[i * ld + j], contiguous in j
      for (int e = tid; e < kSymmJB * kSymmRows; e += kSymmThreads) {
        const int ii = e >> 5, jj = e & 31;
        const bool ok = jj < jmax && ii < imax;
        cp_async8(At + jj * kSymmLd + ii, ok ? A + (int64_t)(I0 + ii) * ld + J0 + jj : A, ok);
      }
    } else {
      for (int e = tid; e < kSymmJB * kSymmRows; e += kSymmThreads) {
        const int jj = e >> 7, ii = e & 127;
        const bool ok = jj < jmax && ii < imax;
        const int gi = I0 + ii, gj = J0 + jj;
        const double* src = !ok ? A : (gi >= gj ? A + (int64_t)gj * ld + gi : A + (int64_t)gi * ld + gj);
        cp_async8(At + jj * kSymmLd + ii, src, ok);
      }
    }
    for (int e = tid; e < kSymmJB * kSB; e += kSymmThreads) {
      const int jj = e >> 4, c = e & 15;
      const bool ok = jj < jmax;
      cp_async8(Vs + e, ok ? Vw + (int64_t)c * L.ldv + J0 + jj : Vw, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[2][8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[a][c] = 0.0;
  const int nsl = (np + kSymmJB - 1) / kSymmJB;
  stage(0, 0);
  for (int k = 0; k < nsl; ++k) {
    if (k + 1 < nsl) {
      stage((k + 1) * kSymmJB, (k + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* At = ssm + (k & 1) * kSymmBuf;
    const double* Vs = At + kSymmJB * kSymmLd;
#pragma unroll 4
    for (int jj = 0; jj < kSymmJB; ++jj) {
      const double a0 = At[jj * kSymmLd + i0], a1 = At[jj * kSymmLd + i0 + 64];
      const double2* vr = reinterpret_cast<const double2*>(Vs + jj * kSB + 8 * h);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = vr[q];
        acc[0][2 * q] = fma(a0, v.x, acc[0][2 * q]);
        acc[0][2 * q + 1] = fma(a0, v.y, acc[0][2 * q + 1]);
        acc[1][2 * q] = fma(a1, v.x, acc[1][2 * q]);
        acc[1][2 * q + 1] = fma(a1, v.y, acc[1][2 * q + 1]);
      }
    }
    __syncthreads();   // this buffer is restaged at step k + 2
  }
  // X rows to shared memory (row stride 17: conflict-free column walks), then Y = X T and M_b = V_b^T Y_b
  constexpr int kX = kSB + 1;
  double* Xs = ssm;
  double* Ts = Xs + kSymmRows * kX;
  double* Ys = Ts + kSB * kSB;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) Xs[(i0 + 64 * a) * kX + 8 * h + c] = acc[a][c];
  const double* Tw = Vw + 2 * L.vsz();
  for (int e = tid; e < kSB * kSB; e += kSymmThreads) Ts[e] = Tw[e];
  __syncthreads();
  for (int e = tid; e < kSymmRows * kSB; e += kSymmThreads) {
    const int c = e >> 7, i = e & 127;
    double y = 0.0;
    for (int l = 0; l <= c; ++l) y = fma(Xs[i * kX + l], Ts[l * kSB + c], y);
    Ys[i * kX + c] = (i < imax) ? y : 0.0;
    if (i < imax) Yw[(int64_t)c * L.ldv + I0 + i] = y;
  }
  // the block's V rows in shared memory ([l][i], coalesced) for M_b = V_b^T Y_b
  double* Vb = Ys + kSymmRows * kX;
  for (int e = tid; e < kSymmRows * kSB; e += kSymmThreads) {
    const int l = e >> 7, i = e & 127;
    Vb[e] = i < imax ? Vw[(int64_t)l * L.ldv + I0 + i] : 0.0;
  }
  __syncthreads();
  double* Mw = L.mp(ws, p) + (int64_t)blockIdx.y * kSB * kSB;
  for (int e = tid; e < kSB * kSB; e += kSymmThreads) {
    const int a = e >> 4, c = e & 15;
    double s = 0.0;
    for (int i = 0; i < imax; ++i) s = fma(Vb[a * kSymmRows + i], Ys[i * kX + c], s);
    Mw[e] = s;
  }
}

// ---------------------------------------------------------------------------
// Stage 1c: W = Y - V Z in place of Y, Z = 1/2 T^T sum_b M_b (16 x 16), rows [128 b, 128 b + 128).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sbr_w(const int* __restrict__ ns, int t, double* __restrict__ ws,
                                                 const SbrWs L, int par) {
  __shared__ double Ms[kSB * kSB], Zs[kSB * kSB];
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int I0 = blockIdx.y * kSymmRows;
  if (I0 >= np) return;
  const int tid = threadIdx.x;
  double* Vw = L.vp(ws, p, par);
  double* Yw = Vw + L.vsz();
  const double* Tw = Vw + 2 * L.vsz();
  const double* Mw = L.mp(ws, p);
  const int nmb = (np + kSymmRows - 1) / kSymmRows;
  double s = 0.0;
  for (int b = 0; b < nmb; ++b) s += Mw[b * kSB * kSB + tid];
  Ms[tid] = s;
  __syncthreads();
  {
    const int a = tid >> 4, c = tid & 15;
    double z = 0.0;
    for (int l = 0; l <= a; ++l) z = fma(Tw[l * kSB + a], Ms[l * kSB + c], z);   // (T^T M)[a][c], T upper
    Zs[tid] = 0.5 * z;
  }
  __syncthreads();
  // thread (i, h): row I0 + i, columns 8 h .. 8 h + 7; the row of V is loaded once into registers
  const int imax = min(kSymmRows, np - I0);
  const int i = tid & 127, h = tid >> 7;
  if (i >= imax) return;
  const int64_t gi = I0 + i;
  double v[kSB], y[8];
#pragma unroll
  for (int l = 0; l < kSB; ++l) v[l] = Vw[(int64_t)l * L.ldv + gi];
#pragma unroll
  for (int c = 0; c < 8; ++c) y[c] = Yw[(int64_t)(8 * h + c) * L.ldv + gi];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double w = y[c];
#pragma unroll
    for (int l = 0; l < kSB; ++l) w = fma(-v[l], Zs[l * kSB + 8 * h + c], w);
    Yw[(int64_t)(8 * h + c) * L.ldv + gi] = w;
  }
}

// ---------------------------------------------------------------------------
// Stage 1d: A22 <- A22 - V W^T - W V^T on the lower 64 x 64 tiles.
// Thread t: rows tx = t % 32 (+32), columns 8 (t / 32) .. + 7 of the tile.  The tile's loads are issued
// first, the V / W rows of the tile are staged while they are in flight.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSyrThreads, 2) k_sbr_syr2k(double* __restrict__ G, int64_t ld, int64_t stride,
                                                                const int* __restrict__ ns, int t,
                                                                const double* __restrict__ ws, const SbrWs L,
                                                                int par) {
  __shared__ __align__(16) double VI[kSB * kSyrTile], WI[kSB * kSyrTile], VJ[kSB * kSyrTile], WJ[kSB * kSyrTile];
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  int q = blockIdx.y, ti = 0;
  while (q > ti) { ++ti; q -= ti; }      // blockIdx.y = ti (ti + 1) / 2 + tj, tj <= ti
  const int tj = q;
  if (ti >= nt) return;
  const int I0 = ti * kSyrTile, J0 = tj * kSyrTile;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  double* A = G + (int64_t)p * stride + (int64_t)R0 * ld + R0;
  const bool diag = ti == tj;
  double a[2][8];
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = tx + 32 * r2, j = 8 * ty + c;
      const bool ok = I0 + i < np && J0 + j < np && (!diag || i >= j);
      a[r2][c] = ok ? A[(int64_t)(J0 + j) * ld + I0 + i] : 0.0;
    }
  const double* Vw = L.vp(const_cast<double*>(ws), p, par);
  const double* Ww = Vw + L.vsz();
  // [l][i] layouts: column l of V / W for the tile rows (coalesced global loads)
  for (int e = tid; e < kSyrTile * kSB; e += kSyrThreads) {
    const int l = e >> 6, i = e & 63;
    const int gi = I0 + i, gj = J0 + i;
    VI[e] = gi < np ? Vw[(int64_t)l * L.ldv + gi] : 0.0;
    WI[e] = gi < np ? Ww[(int64_t)l * L.ldv + gi] : 0.0;
    VJ[e] = gj < np ? Vw[(int64_t)l * L.ldv + gj] : 0.0;
    WJ[e] = gj < np ? Ww[(int64_t)l * L.ldv + gj] : 0.0;
  }
  __syncthreads();
#pragma unroll 4
  for (int l = 0; l < kSB; ++l) {
    const double vi0 = VI[l * kSyrTile + tx], vi1 = VI[l * kSyrTile + tx + 32];
    const double wi0 = WI[l * kSyrTile + tx], wi1 = WI[l * kSyrTile + tx + 32];
    const double2* vj2 = reinterpret_cast<const double2*>(VJ + l * kSyrTile + 8 * ty);
    const double2* wj2 = reinterpret_cast<const double2*>(WJ + l * kSyrTile + 8 * ty);
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) {
      const double2 vj = vj2[c2], wj = wj2[c2];
      a[0][2 * c2] = fma(-vi0, wj.x, fma(-wi0, vj.x, a[0][2 * c2]));
      a[1][2 * c2] = fma(-vi1, wj.x, fma(-wi1, vj.x, a[1][2 * c2]));
      a[0][2 * c2 + 1] = fma(-vi0, wj.y, fma(-wi0, vj.y, a[0][2 * c2 + 1]));
      a[1][2 * c2 + 1] = fma(-vi1, wj.y, fma(-wi1, vj.y, a[1][2 * c2 + 1]));
    }
  }
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = tx + 32 * r2, j = 8 * ty + c;
      const bool ok = I0 + i < np && J0 + j < np && (!diag || i >= j);
      if (ok) A[(int64_t)(J0 + j) * ld + I0 + i] = a[r2][c];
    }
}

// ---------------------------------------------------------------------------
// Stage 1d (TMA variant): the 64 x 64 lower tile arrives by one cp.async.bulk.tensor (3-D tensor map over
// the batch of Grams: rows, columns, problem), is updated in shared memory, and leaves by a bulk tensor
// store -- no registers are held across the global latency, so more CTAs fit per SM.  Elements outside
// the problem's n (the box crosses n or the padded leading dimension) are zero-filled on load and land
// in the unused padding on store; in diagonal tiles only the lower triangle is updated.
// ---------------------------------------------------------------------------
using tc::smem_u32;
using tc::mbar_init;
using tc::fence_mbar_init;
using tc::mbar_wait;
using tc::fence_proxy_async;

// D = A B + D for one 8 x 8 x 4 fp64 tile (DMMA): a = A[g][t], b = B[t][g], (c0, c1) = C[g][2t .. 2t+1],
// g = lane / 4, t = lane % 4 (measured 37.1 TF/s on B200, tools/dmma_probe.cu)
__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}

__global__ void __launch_bounds__(kSyrThreads) k_sbr_syr2k_tma(const __grid_constant__ CUtensorMap tmap,
                                                                  const __grid_constant__ CUtensorMap tmv,
                                                                  const __grid_constant__ CUtensorMap tmw,
                                                                  const int* __restrict__ ns, int t) {
  extern __shared__ __align__(128) double tsm[];
  double* At = tsm;                                   // [64 cols][64 rows] (TMA box, dense)
  double* VI = At + kSyrTile * kSyrTile;
  double* WI = VI + kSB * kSyrTile;
  double* VJ = WI + kSB * kSyrTile;
  double* WJ = VJ + kSB * kSyrTile;
  uint64_t* bar = reinterpret_cast<uint64_t*>(WJ + kSB * kSyrTile);
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  int q = blockIdx.y, ti = 0;
  while (q > ti) { ++ti; q -= ti; }
  const int tj = q;
  if (ti >= nt) return;
  const int I0 = ti * kSyrTile, J0 = tj * kSyrTile;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"((unsigned)((kSyrTile * kSyrTile + 4 * kSB * kSyrTile) * sizeof(double)))
                 : "memory");
    tma_load_3d(At, &tmap, R0 + I0, R0 + J0, p, bar);
    // V / W rows of the tile ([l][i] boxes of the workspace; rows >= n_p hold zeros or stale values of the
    // unused padding, which only meet matrix entries outside the problem)
    tma_load_3d(VI, &tmv, I0, 0, p, bar);
    tma_load_3d(WI, &tmw, I0, 0, p, bar);
    tma_load_3d(VJ, &tmv, J0, 0, p, bar);
    tma_load_3d(WJ, &tmw, J0, 0, p, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  const int tx = tid & 31, ty = tid >> 5;
  const bool diag = ti == tj;
  double a[2][8];
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) a[r2][c] = At[(8 * ty + c) * kSyrTile + tx + 32 * r2];
#pragma unroll 4
  for (int l = 0; l < kSB; ++l) {
    const double vi0 = VI[l * kSyrTile + tx], vi1 = VI[l * kSyrTile + tx + 32];
    const double wi0 = WI[l * kSyrTile + tx], wi1 = WI[l * kSyrTile + tx + 32];
    const double2* vj2 = reinterpret_cast<const double2*>(VJ + l * kSyrTile + 8 * ty);
    const double2* wj2 = reinterpret_cast<const double2*>(WJ + l * kSyrTile + 8 * ty);
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) {
      const double2 vj = vj2[c2], wj = wj2[c2];
      a[0][2 * c2] = fma(-vi0, wj.x, fma(-wi0, vj.x, a[0][2 * c2]));
      a[1][2 * c2] = fma(-vi1, wj.x, fma(-wi1, vj.x, a[1][2 * c2]));
      a[0][2 * c2 + 1] = fma(-vi0, wj.y, fma(-wi0, vj.y, a[0][2 * c2 + 1]));
      a[1][2 * c2 + 1] = fma(-vi1, wj.y, fma(-wi1, vj.y, a[1][2 * c2 + 1]));
    }
  }
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = tx + 32 * r2, j = 8 * ty + c;
      if (!diag || i >= j) At[j * kSyrTile + i] = a[r2][c];
    }
  fence_proxy_async();     // generic-proxy smem writes visible to the bulk copy
  __syncthreads();
  if (tid == 0) {
    tma_store_3d(&tmap, R0 + I0, R0 + J0, p, At);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// ---------------------------------------------------------------------------
// Stage 1d on the fp64 tensor cores (DMMA m8n8k4), default: A22 tile (64 x 64) -= [V_I W_I] [W_J V_J]^T as a
// K = 32 product, a warp owning 32 rows x 16 columns as 4 x 2 accumulator fragments initialised from the
// tile.  The scalar kernel is bound by shared-memory wavefronts (73% of the SM rate); fragments cut them
// to ~60%, given conflict-free layouts: the tile and the V / W rows arrive through 4-D views (i % 16, j or
// l, i / 16, problem) as 16-row boxes with the 128-byte swizzle ([i / 16][j][16 i]), the tile leaves
// through the same map, and the k index of a step is mapped to l = s + 4t (see k_sbr_symm_dmma).
// ---------------------------------------------------------------------------
constexpr int kSyrDTile = kSyrTile * kSyrTile;       // doubles per tile (32 KB)
constexpr int kSyrDOp = kSB * kSyrTile;              // doubles per V / W operand (8 KB)
constexpr size_t kSyrDSmem = ((size_t)kSyrDTile + 4 * kSyrDOp + 2) * sizeof(double) + 1024;

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kSyrThreads, 3) k_sbr_syr2k_dmma(const __grid_constant__ CUtensorMap tm4,
                                                                   const __grid_constant__ CUtensorMap tv4,
                                                                   const __grid_constant__ CUtensorMap tw4,
                                                                   const int* __restrict__ ns, int t) {
  extern __shared__ uint8_t dsm_raw[];
  double* At = reinterpret_cast<double*>(dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u));
  double* VI = At + kSyrDTile;                        // [i / 16][l][16 i], swizzled
  double* WI = VI + kSyrDOp;
  double* VJ = WI + kSyrDOp;
  double* WJ = VJ + kSyrDOp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(WJ + kSyrDOp);
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  int q = blockIdx.y, ti = 0;
  while (q > ti) { ++ti; q -= ti; }
  const int tj = q;
  if (ti >= nt) return;
  const int I0 = ti * kSyrTile, J0 = tj * kSyrTile;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int fg = lane >> 2, ft = lane & 3;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"((unsigned)((kSyrDTile + 4 * kSyrDOp) * sizeof(double)))
                 : "memory");
    tma_load_4d(At, &tm4, 0, R0 + J0, (R0 + I0) >> 4, p, bar);
    tma_load_4d(VI, &tv4, 0, 0, I0 >> 4, p, bar);
    tma_load_4d(WI, &tw4, 0, 0, I0 >> 4, p, bar);
    tma_load_4d(VJ, &tv4, 0, 0, J0 >> 4, p, bar);
    tma_load_4d(WJ, &tw4, 0, 0, J0 >> 4, p, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // warp tile: rows 32 wr .. + 31, columns 16 wc .. + 15
  const int wr = wid & 1, wc = wid >> 1;
  const bool diag = ti == tj;
  // swizzled offsets: element (x, y) of a [x / 16][y][16 x] block with `pitch` y rows per 16-row group
  auto off = [](int x, int y, int pitch) {
    const int xb = x & 15;
    return (x >> 4) * (pitch * 16) + y * 16 + ((((xb >> 1) ^ (y & 7)) << 1) | (xb & 1));
  };
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const int i = 32 * wr + 8 * a + fg, j = 16 * wc + 8 * bb + 2 * ft;
      acc[a][bb][0] = At[off(i, j, kSyrTile)];
      acc[a][bb][1] = At[off(i, j + 1, kSyrTile)];
    }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const double* PI = half == 0 ? VI : WI;   // rows of the tile: V_I then W_I
    const double* QJ = half == 0 ? WJ : VJ;   // columns: W_J then V_J
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
      const int l = (s4 & 1) + 2 * ft + 8 * (s4 >> 1);   // k -> l: every half-warp covers the swizzle once
      double qb[2];
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) qb[bb] = QJ[off(16 * wc + 8 * bb + fg, l, kSB)];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double pa = -PI[off(32 * wr + 8 * a + fg, l, kSB)];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) dmma_f64(acc[a][bb][0], acc[a][bb][1], pa, qb[bb]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const int i = 32 * wr + 8 * a + fg, j = 16 * wc + 8 * bb + 2 * ft;
      if (!diag || i >= j) At[off(i, j, kSyrTile)] = acc[a][bb][0];
      if (!diag || i >= j + 1) At[off(i, j + 1, kSyrTile)] = acc[a][bb][1];
    }
  fence_proxy_async();     // generic-proxy smem writes visible to the bulk copy
  __syncthreads();
  if (tid == 0) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                 ::"l"(&tm4), "r"(0), "r"(R0 + J0), "r"((R0 + I0) >> 4), "r"(p), "r"(smem_u32(At))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// ---------------------------------------------------------------------------
// Stage 1d, row-persistent variant: one CTA per (problem, tile row I); it walks the tiles J = 0 .. I of the
// row through a two-stage ring (tile + V_J / W_J rows per stage; V_I / W_I stay resident), with a producer
// thread issuing the TMA loads, the bulk stores of finished tiles and the refills, so that the update of
// one tile overlaps the load of the next and the store of the previous one.  The one-tile-per-CTA kernel
// spends ~60% of its time waiting for its own loads (ncu: long scoreboard) and pays one CTA launch per
// 64 x 64 tile; here 21312 short CTAs per launch become <= 8 per problem.  Two CTAs per SM.
// ---------------------------------------------------------------------------
constexpr int kSyrRowThreads = kSyrThreads + 32;                       // 8 consumer warps + the producer warp
constexpr int kSyrRowStage = kSyrTile * kSyrTile + 2 * kSB * kSyrTile;  // doubles per stage (48 KB)
constexpr size_t kSyrRowSmem = ((size_t)2 * kSB * kSyrTile + 2 * kSyrRowStage + 8) * sizeof(double);

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kSyrRowThreads, 2) k_sbr_syr2k_row(const __grid_constant__ CUtensorMap tmap,
                                                                     const __grid_constant__ CUtensorMap tmv,
                                                                     const __grid_constant__ CUtensorMap tmw,
                                                                     const int* __restrict__ ns, int t) {
  extern __shared__ __align__(128) double rsm[];
  double* VI = rsm;
  double* WI = VI + kSB * kSyrTile;
  double* stage0 = WI + kSB * kSyrTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + 2 * kSyrRowStage);   // full[2], done[2], vw
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  const int ti = nt - 1 - (int)blockIdx.y;   // longest rows first
  if (ti < 0) return;
  const int I0 = ti * kSyrTile;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], kSyrThreads);
    mbar_init(&bars[3], kSyrThreads);
    mbar_init(&bars[4], 1);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr unsigned kStageTx = (unsigned)(kSyrRowStage * sizeof(double));
  if (tid >= kSyrThreads) {
    // ---------------- producer ----------------
    if (tid == kSyrThreads) {
      auto load_stage = [&](int tj) {
        const int s = tj & 1;
        double* At = stage0 + s * kSyrRowStage;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(kStageTx)
                     : "memory");
        tma_load_3d(At, &tmap, R0 + I0, R0 + tj * kSyrTile, p, &bars[s]);
        tma_load_3d(At + kSyrTile * kSyrTile, &tmv, tj * kSyrTile, 0, p, &bars[s]);
        tma_load_3d(At + kSyrTile * kSyrTile + kSB * kSyrTile, &tmw, tj * kSyrTile, 0, p, &bars[s]);
      };
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[4])),
                   "r"((unsigned)(2 * kSB * kSyrTile * sizeof(double)))
                   : "memory");
      tma_load_3d(VI, &tmv, I0, 0, p, &bars[4]);
      tma_load_3d(WI, &tmw, I0, 0, p, &bars[4]);
      load_stage(0);
      if (ti >= 1) load_stage(1);
      for (int tj = 0; tj <= ti; ++tj) {
        const int s = tj & 1;
        mbar_wait(&bars[2 + s], (tj >> 1) & 1u);                 // the consumers are done with tile tj
        tma_store_3d(&tmap, R0 + I0, R0 + tj * kSyrTile, p, stage0 + s * kSyrRowStage);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (tj + 2 <= ti) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the store has read the stage
          load_stage(tj + 2);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  // ---------------- consumers (8 warps) ----------------
  const int tx = tid & 31, ty = tid >> 5;
  mbar_wait(&bars[4], 0);
  for (int tj = 0; tj <= ti; ++tj) {
    const int s = tj & 1;
    double* At = stage0 + s * kSyrRowStage;
    const double* VJ = At + kSyrTile * kSyrTile;
    const double* WJ = VJ + kSB * kSyrTile;
    mbar_wait(&bars[s], (tj >> 1) & 1u);
    const bool diag = ti == tj;
    double a[2][8];
#pragma unroll
    for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
      for (int c = 0; c < 8; ++c) a[r2][c] = At[(8 * ty + c) * kSyrTile + tx + 32 * r2];
#pragma unroll 4
    for (int l = 0; l < kSB; ++l) {
      const double vi0 = VI[l * kSyrTile + tx], vi1 = VI[l * kSyrTile + tx + 32];
      const double wi0 = WI[l * kSyrTile + tx], wi1 = WI[l * kSyrTile + tx + 32];
      const double2* vj2 = reinterpret_cast<const double2*>(VJ + l * kSyrTile + 8 * ty);
      const double2* wj2 = reinterpret_cast<const double2*>(WJ + l * kSyrTile + 8 * ty);
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2) {
        const double2 vj = vj2[c2], wj = wj2[c2];
        a[0][2 * c2] = fma(-vi0, wj.x, fma(-wi0, vj.x, a[0][2 * c2]));
        a[1][2 * c2] = fma(-vi1, wj.x, fma(-wi1, vj.x, a[1][2 * c2]));
        a[0][2 * c2 + 1] = fma(-vi0, wj.y, fma(-wi0, vj.y, a[0][2 * c2 + 1]));
        a[1][2 * c2 + 1] = fma(-vi1, wj.y, fma(-wi1, vj.y, a[1][2 * c2 + 1]));
      }
    }
#pragma unroll
    for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int i = tx + 32 * r2, j = 8 * ty + c;
        if (!diag || i >= j) At[j * kSyrTile + i] = a[r2][c];
      }
    fence_proxy_async();          // generic-proxy smem writes visible to the bulk store
    mbar_arrive_cta(&bars[2 + s]);
  }
}

// the row-persistent pipeline with the DMMA update and the swizzled 4-D views (default)
__global__ void __launch_bounds__(kSyrRowThreads, 2) k_sbr_syr2k_rowd(const __grid_constant__ CUtensorMap tm4,
                                                                     const __grid_constant__ CUtensorMap tv4,
                                                                     const __grid_constant__ CUtensorMap tw4,
                                                                     const int* __restrict__ ns, int t) {
  extern __shared__ __align__(1024) double rsmd[];
  double* VI = rsmd;
  double* WI = VI + kSB * kSyrTile;
  double* stage0 = WI + kSB * kSyrTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + 2 * kSyrRowStage);   // full[2], done[2], vw
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  const int ti = nt - 1 - (int)blockIdx.y;   // longest rows first
  if (ti < 0) return;
  const int I0 = ti * kSyrTile;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], kSyrThreads);
    mbar_init(&bars[3], kSyrThreads);
    mbar_init(&bars[4], 1);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr unsigned kStageTx = (unsigned)(kSyrRowStage * sizeof(double));
  if (tid >= kSyrThreads) {
    // ---------------- producer ----------------
    if (tid == kSyrThreads) {
      auto load_stage = [&](int tj) {
        const int s = tj & 1;
        double* At = stage0 + s * kSyrRowStage;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(kStageTx)
                     : "memory");
        tma_load_4d(At, &tm4, 0, R0 + tj * kSyrTile, (R0 + I0) >> 4, p, &bars[s]);
        tma_load_4d(At + kSyrTile * kSyrTile, &tv4, 0, 0, (tj * kSyrTile) >> 4, p, &bars[s]);
        tma_load_4d(At + kSyrTile * kSyrTile + kSB * kSyrTile, &tw4, 0, 0, (tj * kSyrTile) >> 4, p, &bars[s]);
      };
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[4])),
                   "r"((unsigned)(2 * kSB * kSyrTile * sizeof(double)))
                   : "memory");
      tma_load_4d(VI, &tv4, 0, 0, I0 >> 4, p, &bars[4]);
      tma_load_4d(WI, &tw4, 0, 0, I0 >> 4, p, &bars[4]);
      load_stage(0);
      if (ti >= 1) load_stage(1);
      for (int tj = 0; tj <= ti; ++tj) {
        const int s = tj & 1;
        mbar_wait(&bars[2 + s], (tj >> 1) & 1u);                 // the consumers are done with tile tj
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                     ::"l"(&tm4), "r"(0), "r"(R0 + tj * kSyrTile), "r"((R0 + I0) >> 4), "r"(p),
                       "r"(smem_u32(stage0 + s * kSyrRowStage))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (tj + 2 <= ti) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the store has read the stage
          load_stage(tj + 2);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  // ---------------- consumers (8 warps) ----------------
  const int wid = tid >> 5, lane = tid & 31;
  const int fg = lane >> 2, ft = lane & 3;
  const int wr = wid & 1, wc = wid >> 1;
  auto off = [](int x, int y, int pitch) {
    const int xb = x & 15;
    return (x >> 4) * (pitch * 16) + y * 16 + ((((xb >> 1) ^ (y & 7)) << 1) | (xb & 1));
  };
  mbar_wait(&bars[4], 0);
  for (int tj = 0; tj <= ti; ++tj) {
    const int s = tj & 1;
    double* At = stage0 + s * kSyrRowStage;
    const double* VJ = At + kSyrTile * kSyrTile;
    const double* WJ = VJ + kSB * kSyrTile;
    mbar_wait(&bars[s], (tj >> 1) & 1u);
    const bool diag = ti == tj;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const int i = 32 * wr + 8 * a + fg, j = 16 * wc + 8 * bb + 2 * ft;
        acc[a][bb][0] = At[off(i, j, kSyrTile)];
        acc[a][bb][1] = At[off(i, j + 1, kSyrTile)];
      }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const double* PI = half == 0 ? VI : WI;
      const double* QJ = half == 0 ? WJ : VJ;
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int l = (s4 & 1) + 2 * ft + 8 * (s4 >> 1);
        double qb[2];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) qb[bb] = QJ[off(16 * wc + 8 * bb + fg, l, kSB)];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double pa = -PI[off(32 * wr + 8 * a + fg, l, kSB)];
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma_f64(acc[a][bb][0], acc[a][bb][1], pa, qb[bb]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const int i = 32 * wr + 8 * a + fg, j = 16 * wc + 8 * bb + 2 * ft;
        if (!diag || i >= j) At[off(i, j, kSyrTile)] = acc[a][bb][0];
        if (!diag || i >= j + 1) At[off(i, j + 1, kSyrTile)] = acc[a][bb][1];
      }
    fence_proxy_async();          // generic-proxy smem writes visible to the bulk store
    mbar_arrive_cta(&bars[2 + s]);
  }
}


// ---------------------------------------------------------------------------
// Stage 1b (TMA variant).  Slices below the diagonal block (all i >= j) arrive as one 128 x 32 box of the
// lower storage (dense [j][i] in shared memory); slices right of it (all i < j, A22(i, j) = G(j, i)) as two
// 16 x 128 boxes of the transposed region with the 128-byte swizzle, so that reading a row i of the slice
// (16-byte pairs (j, j+1)) is conflict-free; slices crossing the diagonal are copied element-wise by
// cp.async.  Two stages in flight; the V slices (32 x 16) follow by cp.async.
// ---------------------------------------------------------------------------
constexpr int kSymmJT = 16;                    // columns per TMA slice (one 16 x 128 swizzled box when transposed)
#ifndef CMSVD_SYMM_NS
#define CMSVD_SYMM_NS 2
#endif
constexpr int kSymmNS = CMSVD_SYMM_NS;         // stages in flight (2: 70 KB per CTA, three CTAs per SM)
constexpr int kSymmA = kSymmJT * kSymmRows;    // doubles per A slice (16 KB)
constexpr int kSymmStage = 2 * kSymmA + kSymmJT * kSB;   // lower box + transposed box + V slice (34 KB)
#ifndef CMSVD_SYMM_TT
#define CMSVD_SYMM_TT 128   // 256 (4 columns per thread, twice the warps) measured slower: 22.8 vs 21.4 ms per config-4 pass
#endif
constexpr int kSymmTT = CMSVD_SYMM_TT;          // threads: 64 row pairs x (kSymmTT / 64) column groups
constexpr int kSymmCW = kSB / (kSymmTT / 64);   // columns of Y per thread

__global__ void __launch_bounds__(kSymmTT, 2) k_sbr_symm_tma(const __grid_constant__ CUtensorMap tlo,
                                                                    const __grid_constant__ CUtensorMap tup,
                                                                    const double* __restrict__ G, int64_t ld,
                                                                    int64_t stride, const int* __restrict__ ns,
                                                                    int t, double* __restrict__ ws, const SbrWs L,
                                                                    int par) {
  extern __shared__ __align__(1024) double ysm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(ysm + kSymmNS * kSymmStage);
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int I0 = blockIdx.y * kSymmRows;
  if (I0 >= np) return;
  const int tid = threadIdx.x;
  const double* A = G + (int64_t)p * stride + (int64_t)R0 * ld + R0;   // A22(i, j) at A[j * ld + i]
  const double* Vw = L.vp(ws, p, par);
  double* Yw = const_cast<double*>(Vw) + L.vsz();
  const int i0 = tid & 63, h = tid >> 6;   // rows i0, i0 + 64; columns kSymmCW h .. + kSymmCW - 1
  const int imax = min(kSymmRows, np - I0);
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < kSymmNS; ++q) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto kind = [&](int J0) {
    const int jmax = min(kSymmJT, np - J0);
    return (J0 + jmax - 1 <= I0) ? 0 : ((I0 + imax - 1 < J0) ? 1 : 2);
  };
  auto issue = [&](int J0, int st) {
    double* As = ysm + st * kSymmStage;   // lower box [j][i] (dense), then the transposed box [i][j] (swizzled)
    double* Vs = As + 2 * kSymmA;
    const int jmax = min(kSymmJT, np - J0);
    const int kd = kind(J0);
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[st])),
                   "r"((unsigned)((kd == 2 ? 2 : 1) * kSymmA * sizeof(double)))
                   : "memory");
      if (kd != 1) tma_load_3d(As, &tlo, R0 + I0, R0 + J0, p, &bars[st]);
      if (kd != 0) tma_load_3d(As + kSymmA, &tup, R0 + J0, R0 + I0, p, &bars[st]);
    }
    for (int e = tid; e < kSymmJT * kSB; e += kSymmTT) {
      const int jj = e >> 4, c = e & 15;
      const bool ok = jj < jmax;
      cp_async8(Vs + e, ok ? Vw + (int64_t)c * L.ldv + J0 + jj : Vw, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[2][kSymmCW];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < kSymmCW; ++c) acc[a][c] = 0.0;
  const int nsl = (np + kSymmJT - 1) / kSymmJT;
  unsigned uses = 0;   // TMA completions consumed per stage (bit st: parity of the next wait)
  for (int q = 0; q < kSymmNS - 1 && q < nsl; ++q) issue(q * kSymmJT, q);
  for (int k = 0; k < nsl; ++k) {
    const int st = k % kSymmNS;
    const int J0 = k * kSymmJT;
    if (k + kSymmNS - 1 < nsl) issue((k + kSymmNS - 1) * kSymmJT, (k + kSymmNS - 1) % kSymmNS);
    const int pending = min(nsl, k + kSymmNS) - k - 1;   // groups committed after slice k's
    if (pending >= 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (pending == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    const int kd = kind(J0);
    mbar_wait(&bars[st], (uses >> st) & 1u);
    uses ^= 1u << st;
    __syncthreads();
    const double* As = ysm + st * kSymmStage;
    const double* Au = As + kSymmA;
    const double* Vs = As + 2 * kSymmA;
    const int jmax = min(kSymmJT, np - J0);
    if (kd == 2) {
      // slice crossing the diagonal block: A22(i, j) from the lower box if i >= j, else the transposed box
      const int sw = i0 & 7;
      for (int jj = 0; jj < jmax; ++jj) {
        const int gj = J0 + jj;
        const int cu = ((((jj >> 1) ^ sw) << 1) | (jj & 1));
        const double a0 = (I0 + i0 >= gj) ? As[jj * kSymmRows + i0] : Au[i0 * 16 + cu];
        const double a1 = (I0 + i0 + 64 >= gj) ? As[jj * kSymmRows + i0 + 64] : Au[(i0 + 64) * 16 + cu];
        const double2* vr = reinterpret_cast<const double2*>(Vs + jj * kSB + kSymmCW * h);
#pragma unroll
        for (int q = 0; q < kSymmCW / 2; ++q) {
          const double2 v = vr[q];
          acc[0][2 * q] = fma(a0, v.x, acc[0][2 * q]);
          acc[0][2 * q + 1] = fma(a0, v.y, acc[0][2 * q + 1]);
          acc[1][2 * q] = fma(a1, v.x, acc[1][2 * q]);
          acc[1][2 * q + 1] = fma(a1, v.y, acc[1][2 * q + 1]);
        }
      }
    } else if (kd == 0) {
#pragma unroll 4
      for (int jj = 0; jj < jmax; ++jj) {
        const double a0 = As[jj * kSymmRows + i0], a1 = As[jj * kSymmRows + i0 + 64];
        const double2* vr = reinterpret_cast<const double2*>(Vs + jj * kSB + kSymmCW * h);
#pragma unroll
        for (int q = 0; q < kSymmCW / 2; ++q) {
          const double2 v = vr[q];
          acc[0][2 * q] = fma(a0, v.x, acc[0][2 * q]);
          acc[0][2 * q + 1] = fma(a0, v.y, acc[0][2 * q + 1]);
          acc[1][2 * q] = fma(a1, v.x, acc[1][2 * q]);
          acc[1][2 * q + 1] = fma(a1, v.y, acc[1][2 * q + 1]);
        }
      }
    } else {
      // swizzled rows: A22(i, J0 + 2 kp .. + 1) at row i, 16-byte chunk kp ^ (i & 7)
      const int sw = i0 & 7;
#pragma unroll 2
      for (int kp = 0; 2 * kp < jmax; ++kp) {
        const int ch = (kp ^ sw) << 1;
        double2 a0 = *reinterpret_cast<const double2*>(Au + i0 * 16 + ch);
        double2 a1 = *reinterpret_cast<const double2*>(Au + (i0 + 64) * 16 + ch);
        if (2 * kp + 1 >= jmax) { a0.y = 0.0; a1.y = 0.0; }
        const double2* v0 = reinterpret_cast<const double2*>(Vs + (2 * kp) * kSB + kSymmCW * h);
        const double2* v1 = reinterpret_cast<const double2*>(Vs + (2 * kp + 1) * kSB + kSymmCW * h);
#pragma unroll
        for (int q = 0; q < kSymmCW / 2; ++q) {
          const double2 x = v0[q], y = v1[q];
          acc[0][2 * q] = fma(a0.y, y.x, fma(a0.x, x.x, acc[0][2 * q]));
          acc[0][2 * q + 1] = fma(a0.y, y.y, fma(a0.x, x.y, acc[0][2 * q + 1]));
          acc[1][2 * q] = fma(a1.y, y.x, fma(a1.x, x.x, acc[1][2 * q]));
          acc[1][2 * q + 1] = fma(a1.y, y.y, fma(a1.x, x.y, acc[1][2 * q + 1]));
        }
      }
    }
    __syncthreads();   // this stage is reissued kSymmNS - 1 steps later
  }
  // epilogue: X rows to shared memory (row stride 17); Y = X T by row (thread = row, X row in registers);
  // M_b = V_b^T Y_b = (V_b^T X_b) T with Q = V_b^T X_b as 8 row-group partials (16 independent
  // accumulators per thread, no long serial chains), then M = Q T
  constexpr int kX = kSB + 1;
  double* Xs = ysm;                          // [128][17]
  double* Ts = Xs + kSymmRows * kX;          // [16][16]
  double* Vb = Ts + kSB * kSB;               // [16][128]
  double* Qp = Vb + kSB * kSymmRows;         // [8][16][16] partials, then Q [16][16]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < kSymmCW; ++c) Xs[(i0 + 64 * a) * kX + kSymmCW * h + c] = acc[a][c];
  const double* Tw = Vw + 2 * L.vsz();
  for (int e = tid; e < kSB * kSB; e += kSymmTT) Ts[e] = Tw[e];
  for (int e = tid; e < kSymmRows * kSB; e += kSymmTT) {
    const int l = e >> 7, i = e & 127;
    Vb[e] = i < imax ? Vw[(int64_t)l * L.ldv + I0 + i] : 0.0;
  }
  __syncthreads();
  if (tid < kSymmRows) {
    const int i = tid;                       // one row per thread
    double x[kSB];
#pragma unroll
    for (int l = 0; l < kSB; ++l) x[l] = Xs[i * kX + l];
    if (i < imax) {
#pragma unroll
      for (int c = 0; c < kSB; ++c) {
        double y = 0.0;
#pragma unroll
        for (int l = 0; l <= c; ++l) y = fma(x[l], Ts[l * kSB + c], y);
        Yw[(int64_t)c * L.ldv + I0 + i] = y;
      }
    }
    // Q partial over rows 16 g .. 16 g + 15 for row a of V_b^T: thread (g = tid >> 4, a = tid & 15)
    const int g = tid >> 4, a = tid & 15;
    double q[kSB];
#pragma unroll
    for (int c = 0; c < kSB; ++c) q[c] = 0.0;
    for (int ii = 16 * g; ii < 16 * g + 16; ++ii) {
      const double v = Vb[a * kSymmRows + ii];
#pragma unroll
      for (int c = 0; c < kSB; ++c) q[c] = fma(v, Xs[ii * kX + c], q[c]);
    }
#pragma unroll
    for (int c = 0; c < kSB; ++c) Qp[(g * kSB + a) * kSB + c] = q[c];
  }
  __syncthreads();
  double* Mw = L.mp(ws, p) + (int64_t)blockIdx.y * kSB * kSB;
  for (int e = tid; e < kSB * kSB; e += kSymmTT) {     // Q = sum of the 8 partials (fixed order)
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += Qp[g * kSB * kSB + e];
    Vb[e] = t;                                               // Q [a][c] (V_b no longer needed)
  }
  __syncthreads();
  for (int e = tid; e < kSB * kSB; e += kSymmTT) {     // M = Q T  (T upper triangular)
    const int a = e >> 4, c = e & 15;
    double m = 0.0;
    for (int l = 0; l <= c; ++l) m = fma(Vb[a * kSB + l], Ts[l * kSB + c], m);
    Mw[e] = m;
  }
}

// ---------------------------------------------------------------------------
// Stage 1b on the fp64 tensor cores (DMMA m8n8k4), default.  The scalar kernel above is bound by
// shared-memory wavefronts (81% of the SM rate: every DFMA row operand is a 64-bit load of 32 lanes = 2
// wavefronts, 0.5 wavefronts per DFMA).  Here a warp owns 32 rows x 16 columns of Y as 4 x 2 accumulator
// fragments and reads the 16-column slice of A22 as 8 x 4 fragments, 16 + 8 loads for 32 DMMAs (8192 FMAs):
// 2.7x fewer wavefronts, provided every fragment load is free of bank conflicts:
//   * slices right of the diagonal block arrive as the transposed 16 x 128 box with the 128-byte swizzle
//     ([i][16 j], as before): fragment (rows 8a + g, k = j = 4s + t) touches 8 chunks x 2 halves exactly;
//   * slices below it arrive through a 4-D view of the lower storage (i % 16, j, i / 16, problem) as eight
//     16 x 16 boxes with the 128-byte swizzle ([i / 16][j][16 i]); with the k index mapped to j = s + 4t
//     (any bijection of k is allowed as long as the V fragment uses the same one) ... in both cases the k
//     index of a step is mapped to the column j so that each HALF-WARP (64-bit shared loads are served per
//     16 lanes: 4 values of g, all t) covers the 8 chunks x 2 halves of the swizzle once: j = (t & 1) + 2 s +
//     8 (t >> 1) for the transposed storage, j = (s & 1) + 2 t + 8 (s >> 1) for the lower storage;
//   * the V slice is staged with its own swizzle (symm_vswz), which serves both k mappings;
//   * slices crossing the diagonal run both passes with complementary masks.
// ---------------------------------------------------------------------------
// swizzle of the staged V slice: 2-bit value that differs between the four j of a k step under both mappings
__device__ __forceinline__ int symm_vswz(int jj) { return ((jj & 1) | ((jj >> 2) & 2)) ^ ((jj >> 1) & 3); }

constexpr int kSymmDNS = 3;                                // stages in flight
constexpr int kSymmDStage = kSymmA + kSymmJT * kSB;        // ONE box (lower or transposed) + the V slice (18 KB)
__global__ void __launch_bounds__(kSymmThreads, 4) k_sbr_symm_dmma(const __grid_constant__ CUtensorMap tlo4,
                                                                    const __grid_constant__ CUtensorMap tup,
                                                                    const double* __restrict__ G, int64_t ld,
                                                                    int64_t stride, const int* __restrict__ ns,
                                                                    int t, double* __restrict__ ws, const SbrWs L,
                                                                    int par) {
  extern __shared__ __align__(1024) double ysm[];
  __shared__ uint64_t bars[kSymmDNS];
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int I0 = blockIdx.y * kSymmRows;
  if (I0 >= np) return;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int fg = lane >> 2, ft = lane & 3;   // DMMA fragment coordinates
  const double* Vw = L.vp(ws, p, par);
  double* Yw = const_cast<double*>(Vw) + L.vsz();
  const int imax = min(kSymmRows, np - I0);
  (void)G; (void)ld; (void)stride;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < kSymmDNS; ++q) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int nsl = (np + kSymmJT - 1) / kSymmJT;
  // slices [kc0, kc1) cross the diagonal block: each is two work items (lower box masked to i >= j, then the
  // transposed box masked to i < j), so that a stage holds one 16 KB box and four CTAs fit per SM
  const int kc0 = min(nsl, I0 / kSymmJT);                              // first slice with a column > I0
  const int kc1 = min(nsl, (I0 + imax - 1) / kSymmJT + 1);             // first slice entirely right of the rows
  const int nc = kc1 - kc0;
  const int nitems = nsl + nc;
  // item -> (slice, box: 0 lower, 1 transposed, masked?)
  auto item_slice = [&](int it, int& box, bool& masked) {
    if (it < kc0) { box = 0; masked = false; return it; }
    if (it < kc0 + 2 * nc) { box = (it - kc0) & 1; masked = true; return kc0 + ((it - kc0) >> 1); }
    box = 1; masked = false;
    return it - nc;
  };
  auto issue = [&](int it, int st) {
    int box; bool masked;
    const int k = item_slice(it, box, masked);
    const int J0 = k * kSymmJT;
    double* As = ysm + st * kSymmDStage;   // lower boxes [i / 16][j][16 i] or the transposed box [i][16 j]
    double* Vs = As + kSymmA;
    const int jmax = min(kSymmJT, np - J0);
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[st])),
                   "r"((unsigned)(kSymmA * sizeof(double)))
                   : "memory");
      if (box == 0)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(smem_u32(As)), "l"(&tlo4), "r"(0), "r"(R0 + J0), "r"((R0 + I0) >> 4), "r"(p), "r"(smem_u32(&bars[st]))
            : "memory");
      else
        tma_load_3d(As, &tup, R0 + J0, R0 + I0, p, &bars[st]);
    }
    for (int e = tid; e < kSymmJT * kSB; e += kSymmThreads) {
      const int jj = e >> 4, c = e & 15;
      const bool ok = jj < jmax;
      cp_async8(Vs + jj * kSB + ((((c >> 1) ^ (symm_vswz(jj) << 1)) << 1) | (c & 1)),
                ok ? Vw + (int64_t)c * L.ldv + J0 + jj : Vw, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) acc[a][bb][0] = acc[a][bb][1] = 0.0;
  unsigned uses = 0;
  for (int q = 0; q < kSymmDNS - 1 && q < nitems; ++q) issue(q, q);
  for (int it = 0; it < nitems; ++it) {
    const int st = it % kSymmDNS;
    if (it + kSymmDNS - 1 < nitems) issue(it + kSymmDNS - 1, (it + kSymmDNS - 1) % kSymmDNS);
    const int pending = min(nitems, it + kSymmDNS) - it - 1;   // groups committed after this item's
    if (pending >= 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (pending == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    int box; bool masked;
    const int k = item_slice(it, box, masked);
    const int J0 = k * kSymmJT;
    mbar_wait(&bars[st], (uses >> st) & 1u);
    uses ^= 1u << st;
    __syncthreads();
    const double* Ab = ysm + st * kSymmDStage;
    const double* Vs = Ab + kSymmA;
    const int jmax = min(kSymmJT, np - J0);
    const bool full = jmax == kSymmJT && imax == kSymmRows;
    // one pass over the box; the k index t of a step is mapped to the column j of the slice so that every
    // half-warp covers the 8 chunks x 2 halves of the swizzle once (see the kernel comment)
    auto pass = [&](bool lower, bool msk) {
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int jj = lower ? (s4 & 1) + 2 * ft + 8 * (s4 >> 1) : (ft & 1) + 2 * s4 + 8 * (ft >> 1);
        const int vs = symm_vswz(jj) << 1;
        double vb[2];
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
          vb[bb] = Vs[jj * kSB + (((((8 * bb + fg) >> 1) ^ vs) << 1) | (fg & 1))];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = 32 * wid + 8 * a + fg;
          double av;
          if (lower) {
            const int ib = i & 15;
            av = Ab[(i >> 4) * 256 + jj * 16 + ((((ib >> 1) ^ (jj & 7)) << 1) | (ib & 1))];
          } else {
            av = Ab[i * 16 + ((((jj >> 1) ^ (i & 7)) << 1) | (jj & 1))];
          }
          if (msk) {
            const bool low = I0 + i >= J0 + jj;
            if (low != lower || jj >= jmax || i >= imax) av = 0.0;
          } else if (!full) {
            if (jj >= jmax || i >= imax) av = 0.0;
          }
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) dmma_f64(acc[a][bb][0], acc[a][bb][1], av, vb[bb]);
        }
      }
    };
    if (box == 0) {
      if (masked) pass(true, true); else pass(true, false);
    } else {
      if (masked) pass(false, true); else pass(false, false);
    }
    __syncthreads();   // this stage is reissued kSymmDNS - 1 items later
  }
  // epilogue: X rows to shared memory (row stride 17); Y = X T by row (thread = row, X row in registers);
  // M_b = V_b^T Y_b = (V_b^T X_b) T with Q = V_b^T X_b as 8 row-group partials (16 independent
  // accumulators per thread, no long serial chains), then M = Q T
  constexpr int kX = kSB + 1;
  double* Xs = ysm;                          // [128][17]
  double* Ts = Xs + kSymmRows * kX;          // [16][16]
  double* Vb = Ts + kSB * kSB;               // [16][128]
  double* Qp = Vb + kSB * kSymmRows;         // [8][16][16] partials, then Q [16][16]
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      Xs[(32 * wid + 8 * a + fg) * kX + 8 * bb + 2 * ft] = acc[a][bb][0];
      Xs[(32 * wid + 8 * a + fg) * kX + 8 * bb + 2 * ft + 1] = acc[a][bb][1];
    }
  const double* Tw = Vw + 2 * L.vsz();
  for (int e = tid; e < kSB * kSB; e += kSymmThreads) Ts[e] = Tw[e];
  for (int e = tid; e < kSymmRows * kSB; e += kSymmThreads) {
    const int l = e >> 7, i = e & 127;
    Vb[e] = i < imax ? Vw[(int64_t)l * L.ldv + I0 + i] : 0.0;
  }
  __syncthreads();
  if (tid < kSymmRows) {
    const int i = tid;                       // one row per thread
    double x[kSB];
#pragma unroll
    for (int l = 0; l < kSB; ++l) x[l] = Xs[i * kX + l];
    if (i < imax) {
#pragma unroll
      for (int c = 0; c < kSB; ++c) {
        double y = 0.0;
#pragma unroll
        for (int l = 0; l <= c; ++l) y = fma(x[l], Ts[l * kSB + c], y);
        Yw[(int64_t)c * L.ldv + I0 + i] = y;
      }
    }
    // Q partial over rows 16 g .. 16 g + 15 for row a of V_b^T: thread (g = tid >> 4, a = tid & 15)
    const int g = tid >> 4, a = tid & 15;
    double q[kSB];
#pragma unroll
    for (int c = 0; c < kSB; ++c) q[c] = 0.0;
    for (int ii = 16 * g; ii < 16 * g + 16; ++ii) {
      const double v = Vb[a * kSymmRows + ii];
#pragma unroll
      for (int c = 0; c < kSB; ++c) q[c] = fma(v, Xs[ii * kX + c], q[c]);
    }
#pragma unroll
    for (int c = 0; c < kSB; ++c) Qp[(g * kSB + a) * kSB + c] = q[c];
  }
  __syncthreads();
  double* Mw = L.mp(ws, p) + (int64_t)blockIdx.y * kSB * kSB;
  for (int e = tid; e < kSB * kSB; e += kSymmThreads) {     // Q = sum of the 8 partials (fixed order)
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += Qp[g * kSB * kSB + e];
    Vb[e] = t;                                               // Q [a][c] (V_b no longer needed)
  }
  __syncthreads();
  for (int e = tid; e < kSB * kSB; e += kSymmThreads) {     // M = Q T  (T upper triangular)
    const int a = e >> 4, c = e & 15;
    double m = 0.0;
    for (int l = 0; l <= c; ++l) m = fma(Vb[a * kSB + l], Ts[l * kSB + c], m);
    Mw[e] = m;
  }
}


// ---------------------------------------------------------------------------
// Fused stage 1 (look-ahead): one pass over the trailing matrix per panel.
//   k_sbr_strip(t)  : A22(t)[:, 0:16] -= V_t W_t[0:16]^T + W_t V_t[0:16]^T (the strip that holds panel t + 1),
//                     so that panel t + 1 can be factored before the rest of A22(t) is updated;
//   k_sbr_panel(t+1): its QR (V_{t+1}, T_{t+1}, R into the band);
//   k_sbr_fused(t)  : per lower 64 x 64 tile of A22(t) (TMA box of 66 rows: the padded pitch makes both
//                     product orientations conflict-free), the rank-32 update with (V_t, W_t) (strip columns
//                     excepted), then on fp64 tensor cores (DMMA) the products with V_{t+1} of the updated
//                     tile: X_I += A V'_J and X_J += A^T V'_I, where V' is V_{t+1} shifted by the 16 strip rows
//                     (TMA boxes starting at row -16: zero-filled), written as per-tile partials;
//   k_sbr_reduce(t+1): X = the partials in fixed order, Y_{t+1} = X T_{t+1}, M partials;  k_sbr_w(t+1).
// The trailing matrix is read and written once per panel (the separate symmetric product's full read is
// gone); V/W/T of panels t and t + 1 live in the two parity sets of the workspace.
// ---------------------------------------------------------------------------
constexpr int kFP = 66;   // row pitch of the fused tile (TMA box rows)

__global__ void __launch_bounds__(128) k_sbr_strip(double* __restrict__ G, int64_t ld, int64_t stride,
                                                   const int* __restrict__ ns, int t, double* __restrict__ ws,
                                                   const SbrWs L, int par) {
  __shared__ double VS[kSB * kSB], WS[kSB * kSB];
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const int i = blockIdx.y * 128 + threadIdx.x;
  const double* Vw = L.vp(ws, p, par);
  const double* Ww = Vw + L.vsz();
  for (int e = threadIdx.x; e < kSB * kSB; e += 128) {   // rows 0..15 of V_t, W_t: [j][l]
    const int j = e >> 4, l = e & 15;
    VS[e] = Vw[(int64_t)l * L.ldv + j];
    WS[e] = Ww[(int64_t)l * L.ldv + j];
  }
  __syncthreads();
  if (i >= np) return;
  double vi[kSB], wi[kSB];
#pragma unroll
  for (int l = 0; l < kSB; ++l) {
    vi[l] = Vw[(int64_t)l * L.ldv + i];
    wi[l] = Ww[(int64_t)l * L.ldv + i];
  }
  double* A = G + (int64_t)p * stride + (int64_t)R0 * ld + R0;
  const int jmax = min(kSB, i + 1);   // lower storage: j <= i
  for (int j = 0; j < jmax; ++j) {
    double a = A[(int64_t)j * ld + i];
#pragma unroll
    for (int l = 0; l < kSB; ++l) a = fma(-vi[l], WS[j * kSB + l], fma(-wi[l], VS[j * kSB + l], a));
    A[(int64_t)j * ld + i] = a;
  }
}

__global__ void __launch_bounds__(kSyrThreads, 2) k_sbr_fused(
    const __grid_constant__ CUtensorMap tmap66, const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmw,
    const __grid_constant__ CUtensorMap tvn, double* __restrict__ G, int64_t ld, int64_t stride,
    const int* __restrict__ ns, int t, double* __restrict__ ws, const SbrWs L) {
  extern __shared__ __align__(128) double fsm[];
  double* At = fsm;                          // [64 cols][kFP rows]
  double* VI = At + kSyrTile * kFP;          // V_t / W_t rows of the tile: [l][64]
  double* WI = VI + kSB * kSyrTile;
  double* VJ = WI + kSB * kSyrTile;
  double* WJ = VJ + kSB * kSyrTile;
  double* PI = WJ + kSB * kSyrTile;          // V_{t+1} rows (shifted by 16): [l][kFP]
  double* PJ = PI + kSB * kFP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(PJ + kSB * kFP);
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t >= sbr_panels(n)) return;
  const int R0 = (t + 1) * kSB, np = n - R0;
  const bool next = t + 1 < sbr_panels(n);
  const int nt = (np + kSyrTile - 1) / kSyrTile;
  int q = blockIdx.y, ti = 0;
  while (q > ti) { ++ti; q -= ti; }
  const int tj = q;
  if (ti >= nt) return;
  const int I0 = ti * kSyrTile, J0 = tj * kSyrTile;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const unsigned bytes = (unsigned)((kSyrTile * kFP + 4 * kSB * kSyrTile + (next ? 2 * kSB * kFP : 0)) *
                                      sizeof(double));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    tma_load_3d(At, &tmap66, R0 + I0, R0 + J0, p, bar);
    tma_load_3d(VI, &tmv, I0, 0, p, bar);
    tma_load_3d(WI, &tmw, I0, 0, p, bar);
    tma_load_3d(VJ, &tmv, J0, 0, p, bar);
    tma_load_3d(WJ, &tmw, J0, 0, p, bar);
    if (next) {
      tma_load_3d(PI, &tvn, I0 - kSB, 0, p, bar);
      tma_load_3d(PJ, &tvn, J0 - kSB, 0, p, bar);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  const int tx = tid & 31, ty = tid >> 5;
  const bool diag = ti == tj;
  double* A = G + (int64_t)p * stride + (int64_t)R0 * ld + R0;
  double a[2][8];
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) a[r2][c] = At[(8 * ty + c) * kFP + tx + 32 * r2];
#pragma unroll 4
  for (int l = 0; l < kSB; ++l) {
    const double vi0 = VI[l * kSyrTile + tx], vi1 = VI[l * kSyrTile + tx + 32];
    const double wi0 = WI[l * kSyrTile + tx], wi1 = WI[l * kSyrTile + tx + 32];
    const double2* vj2 = reinterpret_cast<const double2*>(VJ + l * kSyrTile + 8 * ty);
    const double2* wj2 = reinterpret_cast<const double2*>(WJ + l * kSyrTile + 8 * ty);
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) {
      const double2 vj = vj2[c2], wj = wj2[c2];
      a[0][2 * c2] = fma(-vi0, wj.x, fma(-wi0, vj.x, a[0][2 * c2]));
      a[1][2 * c2] = fma(-vi1, wj.x, fma(-wi1, vj.x, a[1][2 * c2]));
      a[0][2 * c2 + 1] = fma(-vi0, wj.y, fma(-wi0, vj.y, a[0][2 * c2 + 1]));
      a[1][2 * c2 + 1] = fma(-vi1, wj.y, fma(-wi1, vj.y, a[1][2 * c2 + 1]));
    }
  }
  __syncthreads();   // every thread's tile reads are done before the updated values are written back
#pragma unroll
  for (int r2 = 0; r2 < 2; ++r2)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = tx + 32 * r2, j = 8 * ty + c;
      const bool strip = tj == 0 && j < kSB;          // updated (and partly factored) by strip / panel t+1
      const bool ok = I0 + i < np && J0 + j < np && (!diag || i >= j) && !strip;
      if (ok) {
        A[(int64_t)(J0 + j) * ld + I0 + i] = a[r2][c];
        At[j * kFP + i] = a[r2][c];
        if (diag && i > j) At[i * kFP + j] = a[r2][c];   // full symmetric diagonal tile for the product
      }
    }
  if (!next) return;
  __syncthreads();
  // products on fp64 tensor cores: warps 0..3 X_I rows 16 w .. + 15 (A V'_J); warps 4..7 X_J rows
  // 16 (w - 4) .. + 15 (A^T V'_I), off-diagonal tiles only.  Fragments: a = M(g, t), b = V(t, g), c = X(g, 2t..)
  const int lane = tid & 31, wq = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const bool tr = wq >= 4;
  if (tr && diag) return;
  const int rb = 16 * (wq & 3);
  const double* Pb = tr ? PI : PJ;
  double cx[2][2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ntile = 0; ntile < 2; ++ntile) cx[mt][ntile][0] = cx[mt][ntile][1] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < kSyrTile / 4; ++ks) {
    const int k = 4 * ks + tq;
    double bf[2];
#pragma unroll
    for (int ntile = 0; ntile < 2; ++ntile) bf[ntile] = Pb[(8 * ntile + gq) * kFP + k];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = rb + 8 * mt + gq;
      double av = tr ? At[r * kFP + k] : At[k * kFP + r];   // A^T(r, k) = A(k, r) / A(r, k)
      av = ((tr ? I0 : J0) + k < np) ? av : 0.0;            // columns outside the problem (stale padding)
      dmma_f64(cx[mt][0][0], cx[mt][0][1], av, bf[0]);
      dmma_f64(cx[mt][1][0], cx[mt][1][1], av, bf[1]);
    }
  }
  double* part = ws + (int64_t)p * L.per + L.poff + ((int64_t)blockIdx.y * 2 + (tr ? 1 : 0)) * 64 * kSB;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ntile = 0; ntile < 2; ++ntile) {
      const int r = rb + 8 * mt + gq, c = 8 * ntile + 2 * tq;
      part[r * kSB + c] = cx[mt][ntile][0];
      part[r * kSB + c + 1] = cx[mt][ntile][1];
    }
}

// X_{t+1} rows [128 b, 128 b + 128) (A22(t+1) coordinates; A22(t) row i' + 16) from the partials of pass t in
// fixed order, then Y_{t+1} = X T_{t+1} and the M partial of the block (as the symmetric-product kernel).
__global__ void __launch_bounds__(kSymmRows) k_sbr_reduce(const int* __restrict__ ns, int t1,
                                                          double* __restrict__ ws, const SbrWs L, int par) {
  extern __shared__ __align__(16) double rsm[];
  constexpr int kX = kSB + 1;
  double* Xs = rsm;                          // [128][17]
  double* Ts = Xs + kSymmRows * kX;          // [16][16]
  double* Vb = Ts + kSB * kSB;               // [16][128]
  double* Qp = Vb + kSB * kSymmRows;         // [8][16][16]
  const int p = blockIdx.x;
  const int n = ns[p];
  if (t1 >= sbr_panels(n)) return;
  const int R0 = (t1 + 1) * kSB, np = n - R0;    // panel t1's trailing size; pass t1 - 1 had np + 16 rows
  const int I0 = blockIdx.y * kSymmRows;
  if (I0 >= np) return;
  const int tid = threadIdx.x;
  const int imax = min(kSymmRows, np - I0);
  const double* Vw = L.vp(ws, p, par);
  double* Yw = const_cast<double*>(Vw) + L.vsz();
  const double* Tw = Vw + 2 * L.vsz();
  const double* part = ws + (int64_t)p * L.per + L.poff;
  const int nt = (np + kSB + kSyrTile - 1) / kSyrTile;   // tiles per side of pass t1 - 1
  {
    const int ip = I0 + tid;                      // A22(t1) row
    double x[kSB];
#pragma unroll
    for (int c = 0; c < kSB; ++c) x[c] = 0.0;
    if (tid < imax) {
      const int i = ip + kSB;                     // A22(t1 - 1) row
      const int ti = i / kSyrTile, r = i % kSyrTile;
      for (int tj = 0; tj <= ti; ++tj) {          // X_I partials of tiles (ti, tj)
        const double* src = part + ((int64_t)(ti * (ti + 1) / 2 + tj) * 2) * 64 * kSB + r * kSB;
#pragma unroll
        for (int c = 0; c < kSB; ++c) x[c] += src[c];
      }
      for (int tk = ti + 1; tk < nt; ++tk) {      // X_J partials of tiles (tk, ti)
        const double* src = part + ((int64_t)(tk * (tk + 1) / 2 + ti) * 2 + 1) * 64 * kSB + r * kSB;
#pragma unroll
        for (int c = 0; c < kSB; ++c) x[c] += src[c];
      }
    }
#pragma unroll
    for (int c = 0; c < kSB; ++c) Xs[tid * kX + c] = x[c];
  }
  for (int e = tid; e < kSB * kSB; e += kSymmRows) Ts[e] = Tw[e];
  for (int e = tid; e < kSymmRows * kSB; e += kSymmRows) {
    const int l = e >> 7, i = e & 127;
    Vb[e] = i < imax ? Vw[(int64_t)l * L.ldv + I0 + i] : 0.0;
  }
  __syncthreads();
  {
    const int i = tid;
    double x[kSB];
#pragma unroll
    for (int l = 0; l < kSB; ++l) x[l] = Xs[i * kX + l];
    if (i < imax) {
#pragma unroll
      for (int c = 0; c < kSB; ++c) {
        double y = 0.0;
#pragma unroll
        for (int l = 0; l <= c; ++l) y = fma(x[l], Ts[l * kSB + c], y);
        Yw[(int64_t)c * L.ldv + I0 + i] = y;
      }
    }
    const int g = tid >> 4, a = tid & 15;
    double qv[kSB];
#pragma unroll
    for (int c = 0; c < kSB; ++c) qv[c] = 0.0;
    for (int ii = 16 * g; ii < 16 * g + 16; ++ii) {
      const double v = Vb[a * kSymmRows + ii];
#pragma unroll
      for (int c = 0; c < kSB; ++c) qv[c] = fma(v, Xs[ii * kX + c], qv[c]);
    }
#pragma unroll
    for (int c = 0; c < kSB; ++c) Qp[(g * kSB + a) * kSB + c] = qv[c];
  }
  __syncthreads();
  double* Mw = L.mp(ws, p) + (int64_t)blockIdx.y * kSB * kSB;
  for (int e = tid; e < kSB * kSB; e += kSymmRows) {
    double s2 = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) s2 += Qp[g * kSB * kSB + e];
    Vb[e] = s2;
  }
  __syncthreads();
  for (int e = tid; e < kSB * kSB; e += kSymmRows) {
    const int a = e >> 4, c = e & 15;
    double m = 0.0;
    for (int l = 0; l <= c; ++l) m = fma(Vb[a * kSB + l], Ts[l * kSB + c], m);
    Mw[e] = m;
  }
}

// ---------------------------------------------------------------------------
// Stage 2: bulge chasing on the band, one CTA per problem.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double& bat(double* Bd, int i, int j) { return Bd[j * kSBLdb + (i - j)]; }  // i >= j

// task (j, s) of sweep j on the band Bd (n x n), executed by one warp
// Band storage: element (i, j), i >= j, at Bd[j * kSBLdb + (i - j)] = Bd[j * (kSBLdb - 1) + i].
constexpr int kSBRow = kSBLdb - 1;   // stride between (i, j) and (i, j + 1)

// Task (j, s) of sweep j on the band Bd (n x n), executed by one warp; ps: 16 doubles of per-warp scratch.
// Lane (l16, hh) holds row / column l16 of the three 16 x 16 blocks the task updates (B: left-applied,
// s >= 1; D: two-sided; C: right-applied) at entries l = 8 hh + q.  The latency chain is kept short: the
// products with the Householder vector v = (1, x_1 .. x_{L-1}) * scale are formed from x before the
// reflector's scalars are known (v^T y = y_0 + scale * sum_{l>=1} x_l y_l), the squared norm from the two
// half-sums, and p = tau D v is broadcast through shared memory while K = tau/2 p.v is reduced.
// S0: the sweep's first step (s = 0: no block B; the annihilated column is column j itself)
template <bool FULL, bool S0>
__device__ __forceinline__ void chase_task_t(double* __restrict__ Bd, double* __restrict__ ps, int j, int s, int L,
                                             int L2) {
  const int lane = threadIdx.x & 31;
  const int r = j + 1 + s * kSB;
  const int cx = S0 ? j : r - kSB;    // column holding x (rows r .. r + L - 1)
  const int l16 = lane & 15, hh = lane >> 4;
  const int r2 = r + L;
  const double* px = Bd + cx * kSBRow + r;
  double* pB = Bd + (cx + l16) * kSBRow + r + 8 * hh;          // B[l][c = l16]   at pB[q]
  double* pDlo = Bd + (r + 8 * hh) * kSBRow + r + l16;          // D[a = l16][l], a >= l, at pDlo[q * kSBRow]
  double* pDup = Bd + (r + l16) * kSBRow + r + 8 * hh;          // D[l][a = l16], l > a,  at pDup[q]
  double* pC = Bd + (r + 8 * hh) * kSBRow + r2 + l16;           // C[a = l16][l]   at pC[q * kSBRow]
  double xl[8], b[8], dd[8], cr[8];
  const double alpha = px[0];
  const double xa = (l16 < L) ? px[l16] : 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int l = 8 * hh + q;
    if (FULL) {
      xl[q] = px[l];
      b[q] = S0 ? 0.0 : pB[q];
      dd[q] = *((l16 >= l) ? pDlo + q * kSBRow : pDup + q);   // one load through a selected address
      cr[q] = pC[q * kSBRow];
    } else {
      xl[q] = (l < L) ? px[l] : 0.0;
      b[q] = (!S0 && l < L) ? pB[q] : 0.0;
      dd[q] = (l16 < L && l < L) ? ((l16 >= l) ? pDlo[q * kSBRow] : pDup[q]) : 0.0;
      cr[q] = (l16 < L2 && l < L) ? pC[q * kSBRow] : 0.0;
    }
  }
  // half-sums over l >= 1 (entry l = 0 is q = 0 of the hh = 0 lanes) and the l = 0 terms
  double sq = 0.0, tb = 0.0, tp = 0.0, tq = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double xq = (hh == 0 && q == 0) ? 0.0 : xl[q];
    sq = fma(xq, xq, sq);
    tb = fma(xq, b[q], tb);
    tp = fma(xq, dd[q], tp);
    tq = fma(xq, cr[q], tq);
  }
  double b0 = hh == 0 ? b[0] : 0.0, d0 = hh == 0 ? dd[0] : 0.0, c0 = hh == 0 ? cr[0] : 0.0;
  sq += __shfl_xor_sync(0xffffffffu, sq, 16);
  tb += __shfl_xor_sync(0xffffffffu, tb, 16);
  tp += __shfl_xor_sync(0xffffffffu, tp, 16);
  tq += __shfl_xor_sync(0xffffffffu, tq, 16);
  b0 += __shfl_xor_sync(0xffffffffu, b0, 16);
  d0 += __shfl_xor_sync(0xffffffffu, d0, 16);
  c0 += __shfl_xor_sync(0xffffffffu, c0, 16);
  if (!(sq > 0.0)) return;   // x is already alpha e_0: H = I (warp-uniform)
  const double x2 = fma(alpha, alpha, sq);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x2));
  const double e = fma(-(x2 * y), y, 1.0);
  y = fma(y * e, fma(e, 0.375, 0.5), y);
  const double xn = x2 * y;
  const double beta = alpha >= 0.0 ? -xn : xn;
  const double tau = (beta - alpha) * sbr_rcp(beta);
  const double scale = sbr_rcp(alpha - beta);
  const double db = tau * fma(scale, tb, b0);   // tau v^T B[:, l16]
  const double pa = tau * fma(scale, tp, d0);   // p_a = tau (D v)_a, a = l16
  const double qd = tau * fma(scale, tq, c0);   // tau (C v)_a
  double vh[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) vh[q] = (hh == 0 && q == 0) ? 1.0 : xl[q] * scale;
  const double va = (l16 == 0) ? 1.0 : xa * scale;
  // broadcast p; meanwhile K = tau/2 p.v reduced over the 16 rows (lanes 0..15 and 16..31 hold the same p_a)
  if (lane < 16) ps[lane] = (l16 < L) ? pa : 0.0;
  double pv = (l16 < L) ? pa * va : 0.0;
  pv += __shfl_xor_sync(0xffffffffu, pv, 1);
  pv += __shfl_xor_sync(0xffffffffu, pv, 2);
  pv += __shfl_xor_sync(0xffffffffu, pv, 4);
  pv += __shfl_xor_sync(0xffffffffu, pv, 8);
  __syncwarp();
  double ph[8];
  {
    const double2* p2 = reinterpret_cast<const double2*>(ps + 8 * hh);
#pragma unroll
    for (int q = 0; q < 4; ++q) { const double2 t = p2[q]; ph[2 * q] = t.x; ph[2 * q + 1] = t.y; }
  }
  const double K = 0.5 * tau * pv;
  const double wa = fma(-K, va, pa);
  // stores (each lane writes only entries it loaded itself, or the lower entries of D it owns)
  if (S0) {
    if (lane < L) Bd[j * kSBRow + r + lane] = (lane == 0) ? beta : 0.0;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int l = 8 * hh + q;
      if (FULL || l < L) pB[q] = (l16 == 0) ? (l == 0 ? beta : 0.0) : fma(-db, vh[q], b[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int l = 8 * hh + q;
    const double wl = fma(-K, vh[q], ph[q]);
    if ((FULL || l16 < L) && l <= l16) pDlo[q * kSBRow] = fma(-va, wl, fma(-wa, vh[q], dd[q]));
    if (FULL || (l16 < L2 && l < L)) pC[q * kSBRow] = fma(-qd, vh[q], cr[q]);
  }
  __syncwarp();                       // p reads done before the scratch is reused by the next task
}

__device__ __forceinline__ void chase_task(double* __restrict__ Bd, double* __restrict__ ps, int n, int j, int s) {
  const int r = j + 1 + s * kSB;
  const int L = min(kSB, n - r);
  const int L2 = min(kSB, n - r - L);
  if (s == 0) {
    if (L == kSB && L2 == kSB) chase_task_t<true, true>(Bd, ps, j, s, L, L2);
    else chase_task_t<false, true>(Bd, ps, j, s, L, L2);
  } else {
    if (L == kSB && L2 == kSB) chase_task_t<true, false>(Bd, ps, j, s, L, L2);
    else chase_task_t<false, false>(Bd, ps, j, s, L, L2);
  }
}

// ---------------------------------------------------------------------------
// Stage 2, two problems in flight per CTA (CMSVD_CHASE2=1; an experiment kept for its negative result: the same
// 26 eigensolver tests pass, but a config-4 pass takes 25.6 ms against 22.8 ms for one CTA per problem -- both
// variants sustain ~4.7 tasks per microsecond and SM, so the chase is bound by task throughput, not by the
// per-step latency this design hides).  A bulge chase is one latency chain per
// time step (3 (n - 3) steps of ~1 us with at most n / 48 + 1 concurrent tasks): one problem per SM leaves
// the SM ~70% idle, and a second resident CTA does not fit (139 KB of band per problem, 52 K registers).
// But sweep j only touches columns >= j: once a problem has passed its middle, the first half of its band
// is dead.  A persistent CTA therefore keeps a circular band buffer of 1.5 x 512 columns and starts the
// next problem of its queue as soon as the previous one has freed enough columns (its finished diagonal /
// sub-diagonal entries are written out first): two problems, half a chase apart, share every time step and
// its barrier, and a problem completes every ~1.5 n steps instead of every 3 n.  Column c of a problem with
// offset `off` lives at physical column (off + c) mod kCh2Cap; a task whose 32 columns do not straddle the
// wrap point runs the plain pointer arithmetic on a shifted base, the rare straddling task goes element by
// element.
// ---------------------------------------------------------------------------
constexpr int kCh2Warps = 16;
constexpr int kCh2Cap = kSBMax + kSBMax / 2;

constexpr int kCh2WrapSz = kCh2Cap * kSBLdb;
template <bool WRAP>
struct ChAcc {
  double* base;   // Bd + off * kSBLdb: element (i, c) at base[c * kSBRow + i], minus kCh2WrapSz from column cw on
  int cw;         // first logical column stored before the start of the buffer (WRAP only)
  __device__ __forceinline__ double& at(int i, int c) const {
    return base[c * kSBRow + i - ((WRAP && c >= cw) ? kCh2WrapSz : 0)];
  }
};

template <bool FULL, bool WRAP>
__device__ __forceinline__ void chase2_task_t(const ChAcc<WRAP> A, double* __restrict__ ps, int j, int s, int L,
                                              int L2) {
  const int lane = threadIdx.x & 31;
  const int r = j + 1 + s * kSB;
  const int cx = (s == 0) ? j : r - kSB;    // column holding x (rows r .. r + L - 1)
  const int l16 = lane & 15, hh = lane >> 4;
  const int r2 = r + L;
  double xl[8], b[8], dd[8], cr[8];
  const double alpha = A.at(r, cx);
  const double xa = (l16 < L) ? A.at(r + l16, cx) : 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int l = 8 * hh + q;
    if (FULL) {
      xl[q] = A.at(r + l, cx);
      b[q] = s > 0 ? A.at(r + l, cx + l16) : 0.0;
      dd[q] = (l16 >= l) ? A.at(r + l16, r + l) : A.at(r + l, r + l16);
      cr[q] = A.at(r2 + l16, r + l);
    } else {
      xl[q] = (l < L) ? A.at(r + l, cx) : 0.0;
      b[q] = (s > 0 && l < L) ? A.at(r + l, cx + l16) : 0.0;
      dd[q] = (l16 < L && l < L) ? ((l16 >= l) ? A.at(r + l16, r + l) : A.at(r + l, r + l16)) : 0.0;
      cr[q] = (l16 < L2 && l < L) ? A.at(r2 + l16, r + l) : 0.0;
    }
  }
  double sq = 0.0, tb = 0.0, tp = 0.0, tq = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double xq = (hh == 0 && q == 0) ? 0.0 : xl[q];
    sq = fma(xq, xq, sq);
    tb = fma(xq, b[q], tb);
    tp = fma(xq, dd[q], tp);
    tq = fma(xq, cr[q], tq);
  }
  double b0 = hh == 0 ? b[0] : 0.0, d0 = hh == 0 ? dd[0] : 0.0, c0 = hh == 0 ? cr[0] : 0.0;
  sq += __shfl_xor_sync(0xffffffffu, sq, 16);
  tb += __shfl_xor_sync(0xffffffffu, tb, 16);
  tp += __shfl_xor_sync(0xffffffffu, tp, 16);
  tq += __shfl_xor_sync(0xffffffffu, tq, 16);
  b0 += __shfl_xor_sync(0xffffffffu, b0, 16);
  d0 += __shfl_xor_sync(0xffffffffu, d0, 16);
  c0 += __shfl_xor_sync(0xffffffffu, c0, 16);
  if (!(sq > 0.0)) return;   // x is already alpha e_0: H = I (warp-uniform)
  const double x2 = fma(alpha, alpha, sq);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x2));
  const double e = fma(-(x2 * y), y, 1.0);
  y = fma(y * e, fma(e, 0.375, 0.5), y);
  const double xn = x2 * y;
  const double beta = alpha >= 0.0 ? -xn : xn;
  const double tau = (beta - alpha) * sbr_rcp(beta);
  const double scale = sbr_rcp(alpha - beta);
  const double db = tau * fma(scale, tb, b0);
  const double pa = tau * fma(scale, tp, d0);
  const double qd = tau * fma(scale, tq, c0);
  double vh[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) vh[q] = (hh == 0 && q == 0) ? 1.0 : xl[q] * scale;
  const double va = (l16 == 0) ? 1.0 : xa * scale;
  if (lane < 16) ps[lane] = (l16 < L) ? pa : 0.0;
  double pv = (l16 < L) ? pa * va : 0.0;
  pv += __shfl_xor_sync(0xffffffffu, pv, 1);
  pv += __shfl_xor_sync(0xffffffffu, pv, 2);
  pv += __shfl_xor_sync(0xffffffffu, pv, 4);
  pv += __shfl_xor_sync(0xffffffffu, pv, 8);
  __syncwarp();
  double ph[8];
  {
    const double2* p2 = reinterpret_cast<const double2*>(ps + 8 * hh);
#pragma unroll
    for (int q = 0; q < 4; ++q) { const double2 t = p2[q]; ph[2 * q] = t.x; ph[2 * q + 1] = t.y; }
  }
  const double K = 0.5 * tau * pv;
  const double wa = fma(-K, va, pa);
  if (s == 0) {
    if (lane < L) A.at(r + lane, j) = (lane == 0) ? beta : 0.0;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int l = 8 * hh + q;
      if (FULL || l < L) A.at(r + l, cx + l16) = (l16 == 0) ? (l == 0 ? beta : 0.0) : fma(-db, vh[q], b[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int l = 8 * hh + q;
    const double wl = fma(-K, vh[q], ph[q]);
    if ((FULL || l16 < L) && l <= l16) A.at(r + l16, r + l) = fma(-va, wl, fma(-wa, vh[q], dd[q]));
    if (FULL || (l16 < L2 && l < L)) A.at(r2 + l16, r + l) = fma(-qd, vh[q], cr[q]);
  }
  __syncwarp();
}

__device__ __forceinline__ void chase2_task(double* __restrict__ Bd, double* __restrict__ ps, int n, int off, int j,
                                            int s) {
  const int r = j + 1 + s * kSB;
  const int L = min(kSB, n - r);
  const int L2 = min(kSB, n - r - L);
  const bool full = L == kSB && L2 == kSB;
  // columns touched: cx .. r + 15 with cx = j (s = 0) or r - 16
  const int cmin = off + ((s == 0) ? j : r - kSB), cmax = off + min(n - 1, r + kSB - 1);
  if (cmax < kCh2Cap || cmin >= kCh2Cap) {
    const ChAcc<false> A{Bd + (cmax < kCh2Cap ? off : off - kCh2Cap) * kSBLdb, 0};
    if (full) chase2_task_t<true, false>(A, ps, j, s, L, L2);
    else chase2_task_t<false, false>(A, ps, j, s, L, L2);
  } else {   // the task's columns straddle the end of the circular buffer
    const ChAcc<true> A{Bd + off * kSBLdb, kCh2Cap - off};
    if (full) chase2_task_t<true, true>(A, ps, j, s, L, L2);
    else chase2_task_t<false, true>(A, ps, j, s, L, L2);
  }
}

// d, e^2 are complete: Gershgorin data and the count above the threshold (as at the end of k_sbr_chase)
__global__ void __launch_bounds__(128) k_sbr_chase_fin(const int* __restrict__ ns, const double* __restrict__ thr,
                                                       int kw, int nstride, const double* __restrict__ dout,
                                                       const double* __restrict__ e2out, double* __restrict__ gsh,
                                                       int* __restrict__ cnt_out, int nprob) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nprob) return;
  const int n = ns[p];
  if (n <= 0) { cnt_out[p] = 0; gsh[4 * p] = 0; gsh[4 * p + 1] = 0; gsh[4 * p + 2] = 1e-300; gsh[4 * p + 3] = 1e-300; return; }
  const double* dO = dout + (int64_t)p * nstride;
  const double* eO = e2out + (int64_t)p * nstride;
  double glo = 1e300, ghi = -1e300, emax = 0.0;
  for (int i = 0; i < n; ++i) {
    double rr = 0.0;
    if (i > 0) rr += sqrt(eO[i - 1]);
    if (i + 1 < n) rr += sqrt(eO[i]);
    const double di = dO[i];
    glo = fmin(glo, di - rr);
    ghi = fmax(ghi, di + rr);
    if (i + 1 < n) emax = fmax(emax, eO[i]);
  }
  const double nrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
  glo -= 2.2e-16 * nrm * n + pivmin;
  ghi += 2.2e-16 * nrm * n + pivmin;
  gsh[4 * p] = glo; gsh[4 * p + 1] = ghi; gsh[4 * p + 2] = pivmin; gsh[4 * p + 3] = nrm;
  int above = n;
  if (thr) {
    const double tt = thr[p];
    if (tt >= ghi) above = 0;
    else if (tt > glo) {
      int c0 = 0;
      double qd = dO[0] - tt;
      if (fabs(qd) < pivmin) qd = -pivmin;
      c0 += qd < 0.0;
      for (int i = 1; i < n; ++i) {
        qd = (dO[i] - tt) - eO[i - 1] / qd;
        if (fabs(qd) < pivmin) qd = -pivmin;
        c0 += qd < 0.0;
      }
      above = n - c0;
    }
  }
  cnt_out[p] = min(kw, above);
}

// The scheduling state (two slots: problem, n, offset, start step, columns written out) is a function of
// uniform data only, so every thread carries it in registers: no shared-memory state, no elected thread.
__global__ void __launch_bounds__(kCh2Warps * 32, 1) k_sbr_chase2(const double* __restrict__ G, int64_t ld,
                                                                  int64_t stride, const int* __restrict__ ns,
                                                                  int nstride, double* __restrict__ dout,
                                                                  double* __restrict__ e2out, int nprob) {
  extern __shared__ __align__(16) double bsm2[];
  double* Bd = bsm2;                                             // [kCh2Cap][kSBLdb]
  double* vsc = bsm2 + (int64_t)kCh2Cap * kSBLdb + 32 * (threadIdx.x >> 5);   // per-warp p scratch
  const int tid = threadIdx.x, wid = tid >> 5;
  int act[2] = {0, 0}, sp[2] = {0, 0}, sn[2] = {0, 0}, so[2] = {0, 0}, st0[2] = {0, 0}, sx[2] = {0, 0};
  int next = blockIdx.x;
  int nnext = next < nprob ? ns[next] : 0;   // size of the next problem (loaded once, not once per time step)
  auto cell = [&](int off, int c, int d) -> double& {
    int pc = off + c;
    if (pc >= kCh2Cap) pc -= kCh2Cap;
    return Bd[pc * kSBLdb + d];
  };
  // write out the final diagonal / squared sub-diagonal entries of columns [from, upto) of slot q
  auto extract = [&](int q, int from, int upto) {
    double* dO = dout + (int64_t)sp[q] * nstride;
    double* eO = e2out + (int64_t)sp[q] * nstride;
    for (int i = from + tid; i < upto; i += blockDim.x) {
      dO[i] = cell(so[q], i, 0);
      if (i + 1 < sn[q]) { const double e1 = cell(so[q], i, 1); eO[i] = e1 * e1; }
    }
  };
  int tau_step = 0;
  for (;;) {
    // ---- retire finished problems (all sweeps done) ----
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (act[q] && tau_step - st0[q] > 3 * (sn[q] - 3)) {
        extract(q, sx[q], sn[q]);
        act[q] = 0;
      }
    // ---- start the next problem of this CTA's queue when a slot and enough dead columns are available ----
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      while (!act[q] && next < nprob) {
        const int o = 1 - q;
        const int p = next;
        const int n = nnext;
        if (n <= 0) { next += gridDim.x; nnext = next < nprob ? ns[next] : 0; continue; }
        int off = 0;
        if (act[o]) {
          const int To = tau_step - st0[o];
          const int fin = min(sn[o], max(0, (To - 1) / 3));   // its final columns (sweep j: step 0 at time 3 j)
          const int need = sn[o] + n - kCh2Cap;               // its leading columns this problem overwrites
          if (need > fin) break;
          if (need > sx[o]) { extract(o, sx[o], need); sx[o] = need; }
          off = so[o] + sn[o];
          if (off >= kCh2Cap) off -= kCh2Cap;
        }
        __syncthreads();   // the extract above (and the last time step) precede the overwrite
        const double* A = G + (int64_t)p * stride;
        for (int e = tid; e < n * kSBLdb; e += blockDim.x) {
          const int jj = e / kSBLdb, d = e - jj * kSBLdb;
          cell(off, jj, d) = (d <= kSB && jj + d < n) ? A[(int64_t)jj * ld + jj + d] : 0.0;
        }
        __syncthreads();
        act[q] = 1; sp[q] = p; sn[q] = n; so[q] = off; st0[q] = tau_step; sx[q] = 0;
        next += gridDim.x;
        nnext = next < nprob ? ns[next] : 0;
      }
    }
    if (!act[0] && !act[1]) break;
    // ---- one time step of every active problem: task (j, s = T - 3 j), both problems' tasks over the warps ----
    int cntq[2], jhiq[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      cntq[q] = 0; jhiq[q] = 0;
      const int n = sn[q], T = tau_step - st0[q];
      if (act[q] && n >= 3 && T <= 3 * (n - 3)) {
        const int jhi = min(T / 3, n - 3);
        const int num = 16 * T - n + 3;
        const int jlo = num > 0 ? (num + 46) / 47 : 0;
        jhiq[q] = jhi;
        cntq[q] = max(0, jhi - jlo + 1);
      }
    }
    for (int idx = wid; idx < cntq[0] + cntq[1]; idx += kCh2Warps) {
      const int q = idx < cntq[0] ? 0 : 1;
      const int j = jhiq[q] - (q == 0 ? idx : idx - cntq[0]);
      chase2_task(Bd, vsc, sn[q], so[q], j, tau_step - st0[q] - 3 * j);
    }
    __syncthreads();
    ++tau_step;
  }
}

// FLAGS: per-sweep progress flags (each warp owns whole sweeps and polls its predecessor's counter)
// instead of one CTA barrier per wavefront time step
// GB: n > kSBMax, the band lives in the problem's global workspace (L.band) instead of shared memory
// W: warps per CTA (12; 6 for n <= 256, where a time step has at most 6 tasks and the band takes half the
// shared memory: two CTAs per SM)
// W warps, band rows NB (shared memory): (12, 512) one CTA per SM, (8, 384) two, (6, 256) two, (3, 128) four
template <bool FLAGS, bool GB, int W = kChaseWarps, int NB = kSBMax>
__global__ void __launch_bounds__(W * 32, NB >= 512 ? 1 : (NB >= 384 ? 2 : (NB >= 256 ? 3 : 6))) k_sbr_chase(const double* __restrict__ G, int64_t ld,
                                                                    int64_t stride, const int* __restrict__ ns,
                                                                    const double* __restrict__ thr, int kw,
                                                                    int nstride, double* __restrict__ dout,
                                                                    double* __restrict__ e2out,
                                                                    double* __restrict__ gsh,
                                                                    int* __restrict__ cnt_out,
                                                                    double* __restrict__ ws, const SbrWs L, int nmax,
                                                                    int joff, int jstop, int fin) {
  // Two-phase use (256 < nmax <= 512, launch_tridiag_sbr): phase A (joff = 0, jstop = J = nmax - 256, fin = 0)
  // runs sweeps 0 .. J - 1 on the full band, writes d, e^2 of rows < J and the trailing band with the fill its
  // sweeps have left (rows >= J, diagonals 0 .. 2 kSB) back into the lower storage of G; phase B (joff = J, fin = 0) is the chase of that
  // trailing (n - J) x (n - J) band matrix, which fits the half-band variant (two CTAs per SM); k_sbr_chase_fin
  // follows.  One-phase use: joff = 0, jstop >= n, fin = 1.
  extern __shared__ __align__(16) double bsm[];
  const int nb = GB ? nmax : NB;
  double* Bd = GB ? ws + (int64_t)blockIdx.x * L.per + L.band : bsm;               // [n][kSBLdb]
  double* sbase = GB ? bsm : bsm + (int64_t)nb * kSBLdb;
  volatile int* prog = reinterpret_cast<volatile int*>(sbase);                     // steps done per sweep
  double* vsc = sbase + nb / 2 + 2 + 32 * (threadIdx.x >> 5);                      // per-warp p scratch
  const int p = blockIdx.x;
  int n = ns[p];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* A = G + (int64_t)p * stride;
  double* dO = dout + (int64_t)p * nstride;
  double* eO = e2out + (int64_t)p * nstride;
  if (n <= 0) {
    if (tid == 0 && fin) { cnt_out[p] = 0; gsh[4 * p] = 0; gsh[4 * p + 1] = 0; gsh[4 * p + 2] = 1e-300; gsh[4 * p + 3] = 1e-300; }
    return;
  }
  if (joff > 0) {   // phase B: the trailing band matrix (phase A has finished problems with n - joff <= 2 itself)
    if (n - joff <= 2) return;
    A += (int64_t)joff * ld + joff;
    dO += joff;
    eO += joff;
    n -= joff;
  }
  const int nsw = min(n - 2, jstop);   // sweeps run here (a complete reduction has n - 2)
  // a sweep annihilates only the first column of each fill block: between sweeps the matrix carries the rest of
  // the fill on diagonals kSB + 1 .. 2 kSB, so the hand-over between the phases is the band WITH its bulges
  const int dmax = joff > 0 ? 2 * kSB : kSB;
  for (int e = tid; e < n * kSBLdb; e += blockDim.x) {
    const int jj = e / kSBLdb, d = e - jj * kSBLdb;
    Bd[e] = (d <= dmax && jj + d < n) ? A[(int64_t)jj * ld + jj + d] : 0.0;
  }
  for (int e = tid; e < n; e += blockDim.x) prog[e] = 0;
  __syncthreads();
  if (FLAGS) {
  // sweeps j = wid, wid + W, ...; step s of sweep j waits until sweep j - 1 has completed step s + 2
  for (int j = wid; j < nsw; j += W) {
    const int nsteps = (n - 3 - j) / kSB + 1;   // steps with a window of >= 2 rows
    for (int s = 0; s < nsteps; ++s) {
      if (j > 0) {
        const int need = min(s + 3, (n - 3 - (j - 1)) / kSB + 1);
        if (lane == 0)
          while (prog[j - 1] < need) {
#if CMSVD_CHASE_SLEEP
            __nanosleep(CMSVD_CHASE_SLEEP);
#endif
          }
        __syncwarp();
        __threadfence_block();
      }
      chase_task(Bd, vsc, n, j, s);
      __threadfence_block();
      __syncwarp();
      if (lane == 0) prog[j] = s + 1;
    }
  }
  } else {
  // time-stepped wavefront: task (j, s) runs at time 3 j + s, so that step s of sweep j follows step s + 2
  // of sweep j - 1 (their blocks are then disjoint); the tasks of one time step are independent and
  // spread over the warps, one CTA barrier per time step (no polling)
  const int jlast = nsw - 1;
  const int tmax = jlast >= 0 ? 3 * jlast + (n - 3 - jlast) / kSB : -1;   // last step of the last sweep
#ifdef CMSVD_CHASE_PROF
  long long ct0 = clock64();
#endif
  for (int tt = 0; tt <= tmax; ++tt) {
    const int jhi = min(tt / 3, jlast);
    for (int idx = wid;; idx += W) {
      const int j = jhi - idx;
      const int s = tt - 3 * j;
      if (j < 0 || s >= (n - 3 - j) / kSB + 1) break;
      chase_task(Bd, vsc, n, j, s);
    }
    __syncthreads();
  }
#ifdef CMSVD_CHASE_PROF
  if (blockIdx.x == 0 && tid == 0) printf("chase: %d time steps, %lld cycles (%lld per step)\n", tmax + 1,
                                          clock64() - ct0, (clock64() - ct0) / (tmax + 1));
#endif
  }
  (void)prog;
  __syncthreads();
  // outputs (as k_tridiag): d, e^2, Gershgorin data, threshold count
  const bool partial = nsw < n - 2;
  const int nout = partial ? nsw : n;
  for (int i = tid; i < nout; i += blockDim.x) {
    dO[i] = Bd[i * kSBLdb];
    if (i + 1 < n) { const double e1 = Bd[i * kSBLdb + 1]; eO[i] = e1 * e1; }
  }
  if (partial) {   // the trailing band back into the lower storage of G (phase B reads it from there)
    double* Aw = const_cast<double*>(A);
    for (int e = nsw * kSBLdb + tid; e < n * kSBLdb; e += blockDim.x) {
      const int jj = e / kSBLdb, d = e - jj * kSBLdb;
      if (d <= 2 * kSB && jj + d < n) Aw[(int64_t)jj * ld + jj + d] = Bd[e];
    }
  }
  if (!fin) return;
  __syncthreads();
  if (tid == 0) {
    double glo = 1e300, ghi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      double rr = 0.0;
      if (i > 0) rr += fabs(Bd[(i - 1) * kSBLdb + 1]);
      if (i + 1 < n) rr += fabs(Bd[i * kSBLdb + 1]);
      const double di = Bd[i * kSBLdb];
      glo = fmin(glo, di - rr);
      ghi = fmax(ghi, di + rr);
      if (i + 1 < n) emax = fmax(emax, Bd[i * kSBLdb + 1] * Bd[i * kSBLdb + 1]);
    }
    const double nrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
    glo -= 2.2e-16 * nrm * n + pivmin;
    ghi += 2.2e-16 * nrm * n + pivmin;
    gsh[4 * p] = glo; gsh[4 * p + 1] = ghi; gsh[4 * p + 2] = pivmin; gsh[4 * p + 3] = nrm;
    int above = n;
    if (thr) {
      const double tt = thr[p];
      if (tt >= ghi) above = 0;
      else if (tt > glo) {
        // Sturm count of T - tt I
        int c0 = 0;
        double qd = Bd[0] - tt;
        if (fabs(qd) < pivmin) qd = -pivmin;
        c0 += qd < 0.0;
        for (int i = 1; i < n; ++i) {
          const double e1 = Bd[(i - 1) * kSBLdb + 1];
          qd = (Bd[i * kSBLdb] - tt) - e1 * e1 / qd;
          if (fabs(qd) < pivmin) qd = -pivmin;
          c0 += qd < 0.0;
        }
        above = n - c0;
      }
    }
    cnt_out[p] = min(kw, above);
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
static PFN_cuTensorMapEncodeTiled_v12000 sbr_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D map over the batch of n x n Grams: dims (rows = ld, cols = ld, problems), box0 x box1 x 1 boxes
static bool sbr_tensor_map(CUtensorMap* map, double* G, int64_t ld, int64_t stride, int nprob, int box0, int box1,
                           CUtensorMapSwizzle swz) {
  auto fn = sbr_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)ld, (cuuint64_t)nprob};
  cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(double), (cuuint64_t)stride * sizeof(double)};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, G, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D view of the lower storage (i % 16, j, i / 16, problem): eight 16 x 16 boxes with the 128-byte swizzle
// per 128 x 16 slice, shared-memory order [i / 16][j][16 i] (k_sbr_symm_dmma); ld must be a multiple of 16
static bool sbr_tensor_map_lo4(CUtensorMap* map, double* G, int64_t ld, int64_t stride, int nprob) {
  auto fn = sbr_encode_fn();
  if (!fn || (ld & 15) != 0) return false;
  cuuint64_t dims[4] = {16, (cuuint64_t)ld, (cuuint64_t)(ld / 16), (cuuint64_t)nprob};
  cuuint64_t strides[3] = {(cuuint64_t)ld * sizeof(double), 128, (cuuint64_t)stride * sizeof(double)};
  cuuint32_t box[4] = {16, (cuuint32_t)kSymmJT, (cuuint32_t)(kSymmRows / 16), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, G, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// the same view with 64-column boxes (the 64 x 64 tile of k_sbr_syr2k_dmma: four 16-row groups)
static bool sbr_tensor_map_tile4(CUtensorMap* map, double* G, int64_t ld, int64_t stride, int nprob) {
  auto fn = sbr_encode_fn();
  if (!fn || (ld & 15) != 0) return false;
  cuuint64_t dims[4] = {16, (cuuint64_t)ld, (cuuint64_t)(ld / 16), (cuuint64_t)nprob};
  cuuint64_t strides[3] = {(cuuint64_t)ld * sizeof(double), 128, (cuuint64_t)stride * sizeof(double)};
  cuuint32_t box[4] = {16, (cuuint32_t)kSyrTile, (cuuint32_t)(kSyrTile / 16), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, G, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// V / W rows of the workspace ([l][i], ld = L.ldv) as (i % 16, l, i / 16, problem): 64 rows x 16 l per box
static bool sbr_ws_map4(CUtensorMap* map, double* base, int nprob, const SbrWs& L) {
  auto fn = sbr_encode_fn();
  if (!fn || ((uintptr_t)base % 16) != 0 || (L.ldv & 15) != 0) return false;
  cuuint64_t dims[4] = {16, (cuuint64_t)kSB, (cuuint64_t)(L.ldv / 16), (cuuint64_t)nprob};
  cuuint64_t strides[3] = {(cuuint64_t)L.ldv * sizeof(double), 128, (cuuint64_t)L.per * sizeof(double)};
  cuuint32_t box[4] = {16, (cuuint32_t)kSB, (cuuint32_t)(kSyrTile / 16), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static bool sbr_ws_map(CUtensorMap* map, double* base, int nprob, const SbrWs& L, int rows) {
  auto fn = sbr_encode_fn();
  if (!fn || ((uintptr_t)base % 16) != 0) return false;
  cuuint64_t dims[3] = {(cuuint64_t)L.ldv, (cuuint64_t)kSB, (cuuint64_t)nprob};
  cuuint64_t strides[2] = {(cuuint64_t)L.ldv * sizeof(double), (cuuint64_t)L.per * sizeof(double)};
  cuuint32_t box[3] = {(cuuint32_t)rows, (cuuint32_t)kSB, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

size_t sbr_ws_bytes(int nprob, int nmax) { return (size_t)nprob * sbr_layout(nmax).per * sizeof(double); }
int64_t sbr_ws_per(int nmax) { return sbr_layout(nmax).per; }

// Stage 1 + stage 2 for nprob problems (n = ns[p] <= nmax <= kSBBig, G destroyed): writes dd, ee (e^2), gsh,
// cnt, trace like k_tridiag.  ws: sbr_ws_bytes(nprob, nmax) bytes.  n <= 512 (the pair path): panel and band
// in shared memory; larger n (N1 cluster verification): panel in place and band in global memory.
cudaError_t launch_tridiag_sbr(Ctx& c, double* G, int64_t ld, int64_t stride, const int* d_ns, int nprob, int nmax,
                               const double* d_thr, int kw, int nstride, double* dd, double* ee, double* gsh,
                               int* cnt, double* trace, double* ws, int phase) {
  // phase: bit 0 = stage 1 (dense -> band), bit 1 = stage 2 (band -> tridiagonal); the pipelined caller
  // (launch_tridiag_topk) issues the two stages of a group of problems on different streams
  if (nmax > kSBBig) return cudaErrorInvalidValue;
  const SbrWs L = sbr_layout(nmax);
  const bool big = nmax > kSBMax;
  const int npan = sbr_panels(nmax);
  const size_t psmem = ((size_t)kSB * kPanelLd + 256 + 2 * kSB + 2 * kSB * kSB) * sizeof(double);
  const size_t ssmem = (size_t)2 * kSymmBuf * sizeof(double);
  const size_t ssmem2 = ((size_t)kSymmRows * (kSB + 1) * 2 + kSB * kSB + kSymmRows * kSB) * sizeof(double);
  const size_t symm_smem = std::max(ssmem, ssmem2);
  CUtensorMap tmap, tlo, tup;
  const bool tma = c.sbr_tma && (stride * sizeof(double)) % 16 == 0 && (ld * sizeof(double)) % 16 == 0 &&
                   ((uintptr_t)G % 16) == 0 &&
                   sbr_tensor_map(&tmap, G, ld, stride, nprob, kSyrTile, kSyrTile, CU_TENSOR_MAP_SWIZZLE_NONE) &&
                   sbr_tensor_map(&tlo, G, ld, stride, nprob, kSymmRows, kSymmJT, CU_TENSOR_MAP_SWIZZLE_NONE) &&
                   sbr_tensor_map(&tup, G, ld, stride, nprob, 16, kSymmRows, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tlo4;
  const bool dmma = tma && c.symm_dmma && sbr_tensor_map_lo4(&tlo4, G, ld, stride, nprob);
  const size_t ydmem = std::max((size_t)kSymmDNS * kSymmDStage,
                                (size_t)kSymmRows * (kSB + 1) + kSB * kSB + 2 * kSymmRows * kSB + 4) * sizeof(double);
  const size_t ymem = std::max((size_t)kSymmNS * kSymmStage + 4,
                               (size_t)kSymmRows * (kSB + 1) + kSB * kSB + 2 * kSymmRows * kSB + 4) * sizeof(double);
  // V and W of both parity sets as 3-D maps (64 x 16 boxes; V of the next panel also as 66 x 16 boxes)
  CUtensorMap tmv[2], tmw[2], tvn[2], tm66;
  bool tma2 = tma;
  for (int q2 = 0; q2 < 2 && tma2; ++q2)
    tma2 = sbr_ws_map(&tmv[q2], ws + q2 * L.set, nprob, L, kSyrTile) &&
           sbr_ws_map(&tmw[q2], ws + q2 * L.set + L.vsz(), nprob, L, kSyrTile) &&
           sbr_ws_map(&tvn[q2], ws + q2 * L.set, nprob, L, kFP);
  CUtensorMap tm4, tv4[2], tw4[2];
  bool sdm = tma2 && c.syr2k_dmma && sbr_tensor_map_tile4(&tm4, G, ld, stride, nprob);
  for (int q2 = 0; q2 < 2 && sdm; ++q2)
    sdm = sbr_ws_map4(&tv4[q2], ws + q2 * L.set, nprob, L) && sbr_ws_map4(&tw4[q2], ws + q2 * L.set + L.vsz(), nprob, L);
  if (sdm) {
    cudaError_t e3 = cudaFuncSetAttribute(k_sbr_syr2k_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrDSmem);
    if (e3 != cudaSuccess) return e3;
    e3 = cudaFuncSetAttribute(k_sbr_syr2k_rowd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrRowSmem);
    if (e3 != cudaSuccess) return e3;
  }
  const bool fused = tma2 && c.sbr_fused &&
                     sbr_tensor_map(&tm66, G, ld, stride, nprob, kFP, kSyrTile, CU_TENSOR_MAP_SWIZZLE_NONE);
  const size_t tsmem = ((size_t)kSyrTile * kSyrTile + 4 * kSB * kSyrTile + 2) * sizeof(double);
  const size_t fsmem = ((size_t)kSyrTile * kFP + 4 * kSB * kSyrTile + 2 * kSB * kFP + 2) * sizeof(double);
  const size_t rsmem = ((size_t)kSymmRows * (kSB + 1) + kSB * kSB + 2 * kSB * kSymmRows) * sizeof(double);
  if (tma) {
    cudaError_t e2 = cudaFuncSetAttribute(k_sbr_syr2k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    if (e2 != cudaSuccess) return e2;
    e2 = cudaFuncSetAttribute(k_sbr_syr2k_row, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrRowSmem);
    if (e2 != cudaSuccess) return e2;
    e2 = cudaFuncSetAttribute(k_sbr_symm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ymem);
    if (e2 != cudaSuccess) return e2;
    e2 = cudaFuncSetAttribute(k_sbr_symm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ydmem);
    if (e2 != cudaSuccess) return e2;
    e2 = cudaFuncSetAttribute(k_sbr_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    if (e2 != cudaSuccess) return e2;
    e2 = cudaFuncSetAttribute(k_sbr_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
    if (e2 != cudaSuccess) return e2;
  }
  cudaError_t e = cudaFuncSetAttribute(k_sbr_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
  if (e != cudaSuccess) return e;

  e = cudaFuncSetAttribute(k_sbr_symm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)symm_smem);
  if (e != cudaSuccess) return e;
  auto panel = [&](int t) {
    const int pr = prof_begin(c, PC_SBR_PANEL);
    if (big)
      k_sbr_panel<false><<<nprob, kPanelThreads, (256 + 2 * kSB + 2 * kSB * kSB) * sizeof(double), c.stream>>>(
          G, ld, stride, d_ns, t, ws, trace, L, t & 1);
    else if (c.sbr_panel_rr) {
      const int np0 = nmax - (t + 1) * kSB;   // largest panel height of this launch
      if (np0 > 256) k_sbr_panel3<256><<<nprob, 256, kP3Smem, c.stream>>>(G, ld, stride, d_ns, t, ws, trace, L, t & 1);
      else if (np0 > 128) k_sbr_panel3<128><<<nprob, 128, kP3Smem, c.stream>>>(G, ld, stride, d_ns, t, ws, trace, L, t & 1);
      else k_sbr_panel3<64><<<nprob, 64, kP3Smem, c.stream>>>(G, ld, stride, d_ns, t, ws, trace, L, t & 1);
    }
    else
      k_sbr_panel<true><<<nprob, kPanelThreads, psmem, c.stream>>>(G, ld, stride, d_ns, t, ws, trace, L, t & 1);
    c.launches += 1;
    prof_end(c, pr);
  };
  auto symm_w = [&](int t) {
    const int np0 = nmax - (t + 1) * kSB;
    const int nrb = (np0 + kSymmRows - 1) / kSymmRows;
    int pr = prof_begin(c, PC_SBR_SYMM);
    if (dmma)
      k_sbr_symm_dmma<<<dim3(nprob, nrb), kSymmThreads, ydmem, c.stream>>>(tlo4, tup, G, ld, stride, d_ns, t, ws, L,
                                                                           t & 1);
    else if (tma)
      k_sbr_symm_tma<<<dim3(nprob, nrb), kSymmTT, ymem, c.stream>>>(tlo, tup, G, ld, stride, d_ns, t, ws, L,
                                                                         t & 1);
    else
      k_sbr_symm<<<dim3(nprob, nrb), kSymmThreads, symm_smem, c.stream>>>(G, ld, stride, d_ns, t, ws, L, t & 1);
    c.launches += 1;
    prof_end(c, pr);
    pr = prof_begin(c, PC_SBR_SYR2K);
    k_sbr_w<<<dim3(nprob, nrb), 256, 0, c.stream>>>(d_ns, t, ws, L, t & 1);
    c.launches += 1;
    prof_end(c, pr);
  };
  if (phase & 1) {
  // trace (panel 0 kernel) even when there are no panels
  panel(0);
  if (npan > 0) symm_w(0);
  for (int t = 0; t < npan; ++t) {
    const int np0 = nmax - (t + 1) * kSB;   // largest trailing size at this panel
    const int nt = (np0 + kSyrTile - 1) / kSyrTile;
    if (fused) {
      // look-ahead: strip of panel t + 1 first, its QR, then one pass over the rest with the product
      int pr = prof_begin(c, PC_SBR_SYR2K);
      k_sbr_strip<<<dim3(nprob, (np0 + 127) / 128), 128, 0, c.stream>>>(G, ld, stride, d_ns, t, ws, L, t & 1);
      c.launches += 1;
      prof_end(c, pr);
      if (t + 1 < npan) panel(t + 1);
      pr = prof_begin(c, PC_SBR_SYR2K);
      k_sbr_fused<<<dim3(nprob, nt * (nt + 1) / 2), kSyrThreads, fsmem, c.stream>>>(
          tm66, tmv[t & 1], tmw[t & 1], tvn[(t + 1) & 1], G, ld, stride, d_ns, t, ws, L);
      c.launches += 1;
      prof_end(c, pr);
      if (t + 1 < npan) {
        const int nrb1 = (np0 - kSB + kSymmRows - 1) / kSymmRows;
        pr = prof_begin(c, PC_SBR_SYMM);
        k_sbr_reduce<<<dim3(nprob, std::max(nrb1, 1)), kSymmRows, rsmem, c.stream>>>(d_ns, t + 1, ws, L,
                                                                                     (t + 1) & 1);
        c.launches += 1;
        prof_end(c, pr);
        pr = prof_begin(c, PC_SBR_SYR2K);
        k_sbr_w<<<dim3(nprob, std::max(nrb1, 1)), 256, 0, c.stream>>>(d_ns, t + 1, ws, L, (t + 1) & 1);
        c.launches += 1;
        prof_end(c, pr);
      }
    } else {
      const int pr = prof_begin(c, PC_SBR_SYR2K);
      if (sdm && c.syr2k_row)
        k_sbr_syr2k_rowd<<<dim3(nprob, nt), kSyrRowThreads, kSyrRowSmem, c.stream>>>(tm4, tv4[t & 1], tw4[t & 1],
                                                                                            d_ns, t);
      else if (sdm)
        k_sbr_syr2k_dmma<<<dim3(nprob, nt * (nt + 1) / 2), kSyrThreads, kSyrDSmem, c.stream>>>(tm4, tv4[t & 1],
                                                                                               tw4[t & 1], d_ns, t);
      else if (tma2 && c.syr2k_row)
        k_sbr_syr2k_row<<<dim3(nprob, nt), kSyrRowThreads, kSyrRowSmem, c.stream>>>(tmap, tmv[t & 1], tmw[t & 1],
                                                                                    d_ns, t);
      else if (tma2)
        k_sbr_syr2k_tma<<<dim3(nprob, nt * (nt + 1) / 2), kSyrThreads, tsmem, c.stream>>>(tmap, tmv[t & 1],
                                                                                          tmw[t & 1], d_ns, t);
      else
        k_sbr_syr2k<<<dim3(nprob, nt * (nt + 1) / 2), kSyrThreads, 0, c.stream>>>(G, ld, stride, d_ns, t, ws, L,
                                                                                 t & 1);
      c.launches += 1;
      prof_end(c, pr);
      if (t + 1 < npan) {
        panel(t + 1);
        symm_w(t + 1);
      }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  }
  if (!(phase & 2)) return cudaGetLastError();
  const size_t csmem = ((big ? 0 : (size_t)kSBMax * kSBLdb) + (size_t)(big ? nmax : kSBMax) / 2 + 2 +
                        32 * kChaseWarps) * sizeof(double);
  const int pr = prof_begin(c, PC_SBR_CHASE);
#define SBR_CHASE(F_, GB_)                                                                                        \
  do {                                                                                                            \
    e = cudaFuncSetAttribute(k_sbr_chase<F_, GB_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem);       \
    if (e != cudaSuccess) return e;                                                                               \
    k_sbr_chase<F_, GB_><<<nprob, kChaseWarps * 32, csmem, c.stream>>>(G, ld, stride, d_ns, d_thr, kw, nstride,  \
                                                                        dd, ee, gsh, cnt, ws, L, nmax, 0, 1 << 30, 1); \
  } while (0)
  if (big) SBR_CHASE(false, true);
  else if (c.chase_flags) SBR_CHASE(true, false);
  else if (!c.chase2 && (c.chase_split || (nmax <= kSBMax / 2 && c.chase_small))) {
    // The chase is latency bound (a time step lasts one task, ~1.1 us, whatever the number of tasks), and its
    // shared memory (the band with its fill, 34 diagonals) decides how many problems an SM holds.  The active
    // part of the matrix shrinks by one row per sweep, so the reduction is cut into phases that run on ever
    // smaller bands: active size <= 512 one CTA per SM, <= 384 two, <= 256 two (registers), <= 128 four; a
    // phase writes d, e^2 of its finished rows and hands the trailing band with its fill through the lower
    // storage of G to the next one; k_sbr_chase_fin (Gershgorin data, threshold count) follows.
    // CMSVD_CHASE_SPLIT=0: one kernel (the half-band one for n <= 256).
    int cur = 0, nph = 0;
#define SBR_PHASE(W_, NB_, JSTOP_, FIN_)                                                                           \
  do {                                                                                                             \
    const size_t sm_ = ((size_t)(NB_) * kSBLdb + (size_t)(NB_) / 2 + 2 + 32 * (W_)) * sizeof(double);              \
    e = cudaFuncSetAttribute(k_sbr_chase<false, false, W_, NB_>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                             (int)sm_);                                                                            \
    if (e != cudaSuccess) return e;                                                                                \
    k_sbr_chase<false, false, W_, NB_><<<nprob, (W_) * 32, sm_, c.stream>>>(G, ld, stride, d_ns, d_thr, kw,        \
                                                                            nstride, dd, ee, gsh, cnt, ws, L,      \
                                                                            nmax, cur, JSTOP_, FIN_);              \
    ++nph;                                                                                                         \
  } while (0)
    if (!c.chase_split) {
      SBR_PHASE(6, 256, 1 << 30, 1);
    } else {
      while (true) {
        const int a = nmax - cur;   // largest active size
        if (a > 384) { SBR_PHASE(12, 512, a - 384, 0); cur += a - 384; }
        else if (a > 256) { SBR_PHASE(8, 384, a - 256, 0); cur += a - 256; }
        else if (a > 128) { SBR_PHASE(6, 256, a - 128, 0); cur += a - 128; }
        else { SBR_PHASE(3, 128, 1 << 30, 0); break; }
      }
      k_sbr_chase_fin<<<(nprob + 127) / 128, 128, 0, c.stream>>>(d_ns, d_thr, kw, nstride, dd, ee, gsh, cnt, nprob);
    }
#undef SBR_PHASE
    c.launches += nph - (c.chase_split ? 0 : 1);
  } else if (c.chase2) {
    const size_t c2smem = ((size_t)kCh2Cap * kSBLdb + 32 * kCh2Warps) * sizeof(double);
    e = cudaFuncSetAttribute(k_sbr_chase2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2smem);
    if (e != cudaSuccess) return e;
    k_sbr_chase2<<<std::min(nprob, c.sm_count), kCh2Warps * 32, c2smem, c.stream>>>(G, ld, stride, d_ns, nstride, dd,
                                                                                   ee, nprob);
    k_sbr_chase_fin<<<(nprob + 127) / 128, 128, 0, c.stream>>>(d_ns, d_thr, kw, nstride, dd, ee, gsh, cnt, nprob);
    c.launches += 1;
  } else SBR_CHASE(false, false);
#undef SBR_CHASE
  c.launches += 1;
  prof_end(c, pr);
  return cudaGetLastError();
}

}  // namespace cmsvd

// k_gemm_simt.cu -- batched SIMT GEMMs used by the first (portable) pair
// pipeline and by the block-spectra / commit paths:
//   tn  : C = A^T B        (A: K x M, B: K x N, both column-major = K-major)
//         with fp32 or fp64 accumulation (S4 projection Z = Q^T F, the Grams
//         R'^T R' and Z^T Z of S5/S7, block Grams A^T A of S2);
//   nn  : C = C0 - A B     (A: M x K, B: K x N column-major) -- S5 residual
//         R' = F - Q Z (Lemma 1: R = A_{t+1} - Q_t Y).
// 64x64 output tiles, BK = 16, 256 threads x (4 x 4) register blocking,
// one problem per blockIdx.y.  The tcgen05 path (k_pair_tc.cu) replaces the
// fp32 contractions on the hot path.
#include "common.cuh"
#include "kernels.cuh"

namespace cmsvd {

constexpr int BM = 64, BN = 64, BK = 16, PADM = BM + 1, PADN = BN + 1;

template <typename AccT>
__global__ void __launch_bounds__(256) k_gemm_tn(const GemmDesc* __restrict__ descs, int tiles_n) {
  const GemmDesc d = descs[blockIdx.y];
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * BM, j0 = tn * BN;
  if (i0 >= d.M || j0 >= d.N) return;
  if (d.sym && tm < tn) return;
  // operands staged in the accumulation type (fp32 data converted once, not per use)
  __shared__ AccT As[BK][PADM];
  __shared__ AccT Bs[BK][PADN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  AccT acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = AccT(0);
  for (int k0 = 0; k0 < d.K; k0 += BK) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int e = tid + 256 * s;
      int k = e & 15, i = e >> 4;
      float va = 0.f, vb = 0.f;
      if (k0 + k < d.K) {
        if (i0 + i < d.M) va = d.A[(int64_t)(i0 + i) * d.lda + k0 + k];
        if (j0 + i < d.N) vb = d.B[(int64_t)(j0 + i) * d.ldb + k0 + k];
      }
      As[k][i] = (AccT)va;
      Bs[k][i] = (AccT)vb;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      AccT av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[k][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[k][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  AccT* C = reinterpret_cast<AccT*>(d.C);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      if (i < d.M && j < d.N) {
        C[(int64_t)j * d.ldc + i] = acc[a][b];
        if (d.sym && tm != tn) C[(int64_t)i * d.ldc + j] = acc[a][b];
      }
    }
}

__global__ void __launch_bounds__(256) k_gemm_nn_sub(const GemmDesc* __restrict__ descs, int tiles_n) {
  const GemmDesc d = descs[blockIdx.y];
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * BM, j0 = tn * BN;
  if (i0 >= d.M || j0 >= d.N) return;
  __shared__ float As[BK][PADM];
  __shared__ float Bs[BK][PADN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (int k0 = 0; k0 < d.K; k0 += BK) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int e = tid + 256 * s;
      int i = e & 63, k = e >> 6;          // A tile: 64 rows x 16 k, coalesced along rows
      float va = 0.f;
      if (k0 + k < d.K && i0 + i < d.M) va = d.A[(int64_t)(k0 + k) * d.lda + i0 + i];
      As[k][i] = va;
      int kb = e & 15, j = e >> 4;         // B tile: 16 k x 64 cols, coalesced along k
      float vb = 0.f;
      if (k0 + kb < d.K && j0 + j < d.N) vb = d.B[(int64_t)(j0 + j) * d.ldb + k0 + kb];
      Bs[kb][j] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[k][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[k][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  float* C = reinterpret_cast<float*>(d.C);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      if (i < d.M && j < d.N) {
        float c0 = d.C0 ? d.C0[(int64_t)j * d.ldc0 + i] : 0.f;
        C[(int64_t)j * d.ldc + i] = c0 - acc[a][b];
      }
    }
}

cudaError_t launch_gemm_tn(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN, bool fp64acc) {
  if (nprob <= 0) return cudaSuccess;
  int tm = (maxM + BM - 1) / BM, tn = (maxN + BN - 1) / BN;
  dim3 g(tm * tn, nprob);
  if (fp64acc) k_gemm_tn<double><<<g, 256, 0, c.stream>>>(d_descs, tn);
  else k_gemm_tn<float><<<g, 256, 0, c.stream>>>(d_descs, tn);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_gemm_nn_sub(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN) {
  if (nprob <= 0) return cudaSuccess;
  int tm = (maxM + BM - 1) / BM, tn = (maxN + BN - 1) / BN;
  dim3 g(tm * tn, nprob);
  k_gemm_nn_sub<<<g, 256, 0, c.stream>>>(d_descs, tn);
  c.launches += 1;
  return cudaGetLastError();
}

}  // namespace cmsvd

// Minimal tcgen05 kind::tf32 GEMM check: D(128 x N) = A(128 x K) * B(N x K)^T,
// K-major interleaved smem operands, TMEM accumulator, mbarrier completion.
// Also a 3xTF32 variant (hi*hi + hi*lo + lo*hi) compared with fp64.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2601_11626_b200/csrc/tc_common.cuh"
using namespace cmsvd::tc;

template <int N, int K, bool SPLIT3>
__global__ void k_test(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sAh = sm;                       // 128 x K
  uint8_t* sAl = sAh + 128 * K * 4;
  uint8_t* sBh = sAl + 128 * K * 4;        // N x K
  uint8_t* sBl = sBh + N * K * 4;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(A[r * K + k], h, l);
    *(float*)(sAh + il_off(r, k, 128)) = h;
    *(float*)(sAl + il_off(r, k, 128)) = l;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(B[r * K + k], h, l);
    *(float*)(sBh + il_off(r, k, N)) = h;
    *(float*)(sBl + il_off(r, k, N)) = l;
  }
  if (wid == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, N);
    const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), bh = smem_u32(sBh), bl = smem_u32(sBl);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t offA = s * 2 * 128 * 16, offB = s * 2 * N * 16;
      mma_tf32(tmem, make_desc(ah + offA, 128 * 16, 128), make_desc(bh + offB, N * 16, 128), idesc, s > 0);
      if (SPLIT3) {
        mma_tf32(tmem, make_desc(ah + offA, 128 * 16, 128), make_desc(bl + offB, N * 16, 128), idesc, 1);
        mma_tf32(tmem, make_desc(al + offA, 128 * 16, 128), make_desc(bh + offB, N * 16, 128), idesc, 1);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  // warp w reads lanes 32w..32w+31 (rows), N columns in chunks of 32
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * wid) << 16) + c0, v);
    wait_ld();
    const int row = 32 * wid + (tid & 31);
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem, 512);
}

template <int N, int K, bool S3>
void run() {
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  srand(3);
  for (auto& x : A) x = rand() / (float)RAND_MAX - 0.5f;
  for (auto& x : B) x = rand() / (float)RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * D.size());
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  size_t smem = 2 * (128 + N) * K * 4;
  cudaFuncSetAttribute(k_test<N, K, S3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_test<N, K, S3><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
  double maxerr = 0, maxv = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxv = fmax(maxv, fabs(s));
    }
  printf("N=%d K=%d split3=%d: %s  max|err|=%.3e  (max|D|=%.3e)  D[0]=%f D[1]=%f\n", N, K, (int)S3,
         cudaGetErrorString(e), maxerr, maxv, D[0], D[1]);
}

// MN-major variant: A (128 x K) and B (N x K) stored MN-major, 3xTF32
template <int N, int K>
__global__ void k_test_mn(const float* A, const float* B, float* D, int amn, int bmn, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sAh = sm;
  uint8_t* sAl = sAh + 128 * K * 4;
  uint8_t* sBh = sAl + 128 * K * 4;
  uint8_t* sBl = sBh + N * K * 4;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(A[r * K + k], h, l);
    uint32_t o = amn ? mn_off(r, k, 128) : il_off(r, k, 128);
    *(float*)(sAh + o) = h;
    *(float*)(sAl + o) = l;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(B[r * K + k], h, l);
    uint32_t o = bmn ? mn_off(r, k, N) : il_off(r, k, N);
    *(float*)(sBh + o) = h;
    *(float*)(sBl + o) = l;
  }
  if (wid == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, N, amn, bmn);
    const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), bh = smem_u32(sBh), bl = smem_u32(sBl);
    for (int s = 0; s < K / 8; ++s) {
      uint64_t da_h, da_l, db_h, db_l;
      if (amn) {
        uint32_t lbo = swap ? 128 : 128 * 32, sbo = swap ? 128 * 32 : 128;
        da_h = make_desc(ah + s * 128 * 32, lbo, sbo); da_l = make_desc(al + s * 128 * 32, lbo, sbo);
      } else { da_h = make_desc(ah + s * 2 * 128 * 16, 128 * 16, 128); da_l = make_desc(al + s * 2 * 128 * 16, 128 * 16, 128); }
      if (bmn) {
        uint32_t lbo = swap ? 128 : N * 32, sbo = swap ? N * 32 : 128;
        db_h = make_desc(bh + s * N * 32, lbo, sbo); db_l = make_desc(bl + s * N * 32, lbo, sbo);
      } else { db_h = make_desc(bh + s * 2 * N * 16, N * 16, 128); db_l = make_desc(bl + s * 2 * N * 16, N * 16, 128); }
      mma_tf32(tmem, da_h, db_h, idesc, s > 0);
      mma_tf32(tmem, da_h, db_l, idesc, 1);
      mma_tf32(tmem, da_l, db_h, idesc, 1);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * wid) << 16) + c0, v);
    wait_ld();
    const int row = 32 * wid + (tid & 31);
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem, 512);
}

template <int N, int K>
void run_mn(int amn, int bmn, int swap) {
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  srand(4);
  for (auto& x : A) x = rand() / (float)RAND_MAX - 0.5f;
  for (auto& x : B) x = rand() / (float)RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * D.size());
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  size_t smem = 2 * (128 + N) * K * 4;
  cudaFuncSetAttribute(k_test_mn<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_test_mn<N, K><<<1, 128, smem>>>(dA, dB, dD, amn, bmn, swap);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
  double maxerr = 0, maxv = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxv = fmax(maxv, fabs(s));
    }
  double s00 = 0; for (int k = 0; k < K; ++k) s00 += (double)A[k] * B[k];
  printf("amn=%d bmn=%d swap=%d N=%d K=%d: %s  max|err|=%.3e  (max|D|=%.3e) D00=%f ref=%f D01=%f\n", amn, bmn, swap, N, K,
         cudaGetErrorString(e), maxerr, maxv, D[0], s00, D[1]);
}

// padded K-major layout: byte(r,k) = (k/4)*LBO + (r/8)*SBO + (r%8)*16 + (k%4)*4
template <int N, int K>
__global__ void k_test_pad(const float* A, const float* B, float* D, int LBO, int SBO) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int szA = 16 * SBO, szB = (N / 8) * SBO;   // 128 rows / N rows
  uint8_t* sAh = sm;
  uint8_t* sAl = sAh + szA;
  uint8_t* sBh = sAl + szA;
  uint8_t* sBl = sBh + szB;
  const int tid = threadIdx.x, wid = tid >> 5;
  auto off = [&](int r, int k) { return (uint32_t)((k >> 2) * LBO + (r >> 3) * SBO + (r & 7) * 16 + (k & 3) * 4); };
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(A[r * K + k], h, l);
    *(float*)(sAh + off(r, k)) = h;
    *(float*)(sAl + off(r, k)) = l;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    float h, l;
    split_tf32(B[r * K + k], h, l);
    *(float*)(sBh + off(r, k)) = h;
    *(float*)(sBl + off(r, k)) = l;
  }
  if (wid == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(128, N);
    const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), bh = smem_u32(sBh), bl = smem_u32(sBl);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t o = 2 * s * LBO;
      mma_tf32(tmem, make_desc(ah + o, LBO, SBO), make_desc(bh + o, LBO, SBO), idesc, s > 0);
      mma_tf32(tmem, make_desc(ah + o, LBO, SBO), make_desc(bl + o, LBO, SBO), idesc, 1);
      mma_tf32(tmem, make_desc(al + o, LBO, SBO), make_desc(bh + o, LBO, SBO), idesc, 1);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * wid) << 16) + c0, v);
    wait_ld();
    const int row = 32 * wid + (tid & 31);
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tmem, 512);
}

template <int N, int K>
void run_pad(int LBO, int SBO) {
  std::vector<float> A(128 * K), B(N * K), D(128 * N);
  srand(5);
  for (auto& x : A) x = rand() / (float)RAND_MAX - 0.5f;
  for (auto& x : B) x = rand() / (float)RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * D.size());
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  size_t smem = 2 * (16 + N / 8) * SBO;
  cudaFuncSetAttribute(k_test_pad<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_test_pad<N, K><<<1, 128, smem>>>(dA, dB, dD, LBO, SBO);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
  double maxerr = 0, maxv = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxv = fmax(maxv, fabs(s));
    }
  printf("padded LBO=%d SBO=%d N=%d K=%d: %s  max|err|=%.3e  (max|D|=%.3e)\n", LBO, SBO, N, K, cudaGetErrorString(e),
         maxerr, maxv);
}

int main() {
  run_pad<128, 32>(144, 1152);
  run_pad<64, 32>(144, 1152);
  run_pad<128, 64>(144, 2304);
  run_pad<32, 32>(2048, 128);

  run<32, 32, false>();
  run<32, 32, true>();
  run<128, 64, true>();
  run<64, 32, true>();
  return 0;
}

// Which shared-memory word does tcgen05.mma kind::tf32 read for element (m, k) of an MN-major, 128-byte-swizzled
// A operand?  A region is filled with its own word index (two passes: index >> 2 and index & 3, both exact in
// tf32), B = [I_8; 0] (16 x 8, K-major, no swizzle), one M = 128, N = 16, K = 8 MMA: D[m][n] = A(m, k = n).
// Usage: mn_probe [LBO] [SBO]   (bytes)
#include <cstdio>
#include <cstdlib>
#include "../paper_2601_11626_b200/csrc/tc_common.cuh"
using namespace cmsvd;

__global__ void __launch_bounds__(128) probe(uint32_t lbo, uint32_t sbo, int pass, int amode, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (tc::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  float* A = reinterpret_cast<float*>(sm);            // 32 KB
  uint8_t* B = sm + 32768;                            // 16 rows x 8 k, interleaved no-swizzle (R = 16)
  for (int w = tid; w < 8192; w += 128) A[w] = pass == 0 ? (float)(w >> 2) : (float)(w & 3);
  for (int e = tid; e < 16 * 8; e += 128) {
    const int n = e / 8, k = e % 8;
    *reinterpret_cast<float*>(B + tc::il_off(n, k, 16)) = (n == k) ? 1.f : 0.f;
  }
  if (wid == 0) tc::tmem_alloc(&tbase, 32);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t sa = tc::smem_u32(A);
    // amode 0: control, K-major no swizzle; 1: MN-major 128B swizzle; 2: MN-major no swizzle; 3: K-major 128B swizzle
    const uint64_t lay = (amode == 1 || amode == 3) ? 2 : 0;
    const uint64_t da = (uint64_t)((sa >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                        ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | (lay << 61);
    const uint64_t db = tc::make_desc(tc::smem_u32(B), 16 * 16, 128);
    const uint32_t idesc = tc::make_idesc_tf32(128, 16, (amode == 1 || amode == 2) ? 1 : 0, 0);
    tc::mma_tf32(tmem, da, db, idesc, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  float v[16];
  tc::tmem_ld16(tmem + ((uint32_t)(32 * wid) << 16), v);
  tc::wait_ld();
  for (int j = 0; j < 8; ++j) out[(32 * wid + lane) * 8 + j] = v[j];
  tc::fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(tmem, 32);
}

int main(int argc, char** argv) {
  const uint32_t lbo = argc > 1 ? atoi(argv[1]) : 4096, sbo = argc > 2 ? atoi(argv[2]) : 1024;
  const int amode = argc > 3 ? atoi(argv[3]) : 1;
  float* d;
  cudaMalloc(&d, 2 * 1024 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  float h[2][1024];
  for (int pass = 0; pass < 2; ++pass) {
    probe<<<1, 128, 40000>>>(lbo, sbo, pass, amode, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    cudaMemcpy(h[pass], d, 4096, cudaMemcpyDeviceToHost);
  }
  printf("amode %d LBO %u SBO %u: word index read for (m, k), unswizzled byte = 4 * word\n", amode, lbo, sbo);
  for (int m = 0; m < 128; ++m) {
    if (!(m < 10 || (m % 32) < 2 || m == 127)) continue;
    printf("m %3d:", m);
    for (int k = 0; k < 8; ++k) {
      const int w = 4 * (int)h[0][m * 8 + k] + (int)h[1][m * 8 + k];
      // undo the 128-byte swizzle (16-byte chunk index ^= 128-byte row index % 8) for readability
      const int byte = 4 * w, row = byte >> 7, chunk = (byte >> 4) & 7, within = byte & 15;
      const int ub = (row << 7) | ((chunk ^ (row & 7)) << 4) | within;
      printf(" %5d(r%3d c%2d)", w, ub >> 7, (ub & 127) >> 2);
    }
    printf("\n");
  }
  return 0;
}

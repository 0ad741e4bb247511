// Microbenchmarks for roofline denominators not in MEASURED_PEAKS.json:
// FP32 FFMA, FP64 DFMA (SIMT), shared-memory bandwidth. Standalone binary.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void smem_loop(float* out, int iters) {
  __shared__ float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float4 v = buf[(idx + k * 32) & 1023];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    idx = (idx + 1) & 1023;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* of; double* od; cudaMalloc(&of, 1 << 26); cudaMalloc(&od, 1 << 27);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fma_loop<float><<<blocks, threads>>>(of, iters, 1.0000001f, 1e-7f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"ffma_tflops\": %.2f}\n", fl / ms / 1e9);
    cudaEventRecord(e0); fma_loop<double><<<blocks, threads>>>(od, iters / 4, 1.0000001, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 16 * (double)(iters / 4) * blocks * threads;
    printf("{\"dfma_tflops\": %.2f}\n", fl / ms / 1e9);
    cudaEventRecord(e0); smem_loop<<<blocks, threads>>>(of, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double by = 16.0 * 8 * (double)iters * blocks * threads;
    printf("{\"smem_tbps\": %.2f, \"smem_bytes_per_clk_per_sm_at_1965\": %.1f}\n", by / ms / 1e9, by / ms / 1e-3 / sms / 1.965e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  size_t l2; int l2i; cudaDeviceGetAttribute(&l2i, cudaDevAttrL2CacheSize, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d}\n", sms, clk, l2i);
  return 0;
}

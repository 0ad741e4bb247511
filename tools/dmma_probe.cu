#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// layout check: D = A (8x4) * B (4x8)
__global__ void kcheck(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];          // A[g][t] row-major 8x4
  double b = B[t * 8 + g];          // B[t][g] row-major 4x8
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  D[g * 8 + 2 * t] = c0; D[g * 8 + 2 * t + 1] = c1;
}
__global__ void kthru(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i * 0.5 + 1; hB[i] = (i % 7) - 2.5; }
  for (int g = 0; g < 8; ++g) for (int n = 0; n < 8; ++n) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[g*4+k]*hB[k*8+n]; ref[g*8+n] = s; }
  double *A, *B, *D; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&D, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  kcheck<<<1, 32>>>(A, B, D); cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
  printf("layout check max err %g\n", err);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kthru<<<148 * 2, 32 * warps>>>(out, iters); cudaDeviceSynchronize();
    cudaEventRecord(e0); kthru<<<148 * 2, 32 * warps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * 148 * 2 * warps;
    printf("warps/CTA %2d: %.2f TFLOP/s fp64 tensor\n", warps, flops / ms / 1e9);
  }
  return 0;
}

// Dependent-chain latencies on the device (cycles): DFMA, DADD, FFMA, SHFL (double), MUFU.RCP64H, LDS.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, int iters) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  float xf = (float)x;
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = x;
  __syncthreads();
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-12);
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + y;
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) xf = fmaf(xf, 1.0000001f, 1e-7f);
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-300;
  t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t1 = clock64(); cyc[4] = t1 - t0;
  int idx = threadIdx.x & 63;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = ((int)v & 1) + (threadIdx.x & 63); }
  t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64(); cyc[6] = t1 - t0;
  out[threadIdx.x] = x + xf + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 8);
  const int it = 1000;
  for (int nt : {32, 512}) {
    k<<<1, nt>>>(o, c, 1.0, it);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* nm[7] = {"DFMA", "DADD", "FFMA", "SHFL.f64+DADD", "MUFU.RCP64H", "LDS(dep)+cvt", "__syncthreads"};
    printf("threads=%d\n", nt);
    for (int q = 0; q < 7; ++q) printf("  %-16s %.1f cyc\n", nm[q], (double)h[q] / it);
  }
  return 0;
}

// Precision of rsqrt.approx.ftz.f64 and of its Newton / cubic corrections (max relative error vs 1/sqrt).
#include <cstdio>
#include <cmath>
__global__ void k(double* out, int n) {
  double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = exp(-30.0 + 60.0 * (i + 0.5) / n) * (1.0 + 0.37 * sin((double)i));
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    const double ref = 1.0 / sqrt(x);
    // one Newton
    double hh = 0.5 * x * y0, rr = fma(-hh, y0, 0.5), y1 = fma(y0, rr, y0);
    // two Newton
    hh = 0.5 * x * y1; rr = fma(-hh, y1, 0.5); double y2 = fma(y1, rr, y1);
    // cubic: e = 1 - x y0^2, y = y0 (1 + e/2 + 3 e^2 / 8)
    const double t = x * y0, e = fma(-t, y0, 1.0), p = fma(e, 0.375, 0.5), y3 = fma(y0 * e, p, y0);
    e0 = fmax(e0, fabs(y0 - ref) / ref); e1 = fmax(e1, fabs(y1 - ref) / ref);
    e2 = fmax(e2, fabs(y2 - ref) / ref); e3 = fmax(e3, fabs(y3 - ref) / ref);
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(e0));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(e1));
  atomicMax((unsigned long long*)&out[2], __double_as_longlong(e2));
  atomicMax((unsigned long long*)&out[3], __double_as_longlong(e3));
}
int main() {
  double* d; cudaMalloc(&d, 32); cudaMemset(d, 0, 32);
  k<<<148, 256>>>(d, 1 << 24);
  double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("rsqrt.approx.f64 max rel err %.3e | 1 Newton %.3e | 2 Newton %.3e | cubic %.3e\n", h[0], h[1], h[2], h[3]);
  return 0;
}

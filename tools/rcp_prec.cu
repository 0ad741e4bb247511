// Precision of rcp.approx.ftz.f64 and of its Newton / cubic corrections (max relative error vs 1/x).
#include <cstdio>
#include <cmath>
__global__ void k(double* out, int n) {
  double e0 = 0, e2 = 0, e3 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = (i & 1 ? -1.0 : 1.0) * exp(-200.0 + 400.0 * (i + 0.5) / n) * (1.0 + 0.37 * sin((double)i));
    double y0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    const double ref = 1.0 / x;
    double e = fma(-x, y0, 1.0), y = fma(y0, e, y0);
    e = fma(-x, y, 1.0); const double y2 = fma(y, e, y);
    const double ec = fma(-x, y0, 1.0), y3 = fma(y0 * ec, 1.0 + ec, y0);
    e0 = fmax(e0, fabs(y0 - ref) / fabs(ref)); e2 = fmax(e2, fabs(y2 - ref) / fabs(ref));
    e3 = fmax(e3, fabs(y3 - ref) / fabs(ref));
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(e0));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(e2));
  atomicMax((unsigned long long*)&out[2], __double_as_longlong(e3));
}
int main() {
  double* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
  k<<<148, 256>>>(d, 1 << 24);
  double h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("rcp.approx.f64 max rel err %.3e | 2 Newton %.3e | cubic %.3e\n", h[0], h[1], h[2]);
  return 0;
}

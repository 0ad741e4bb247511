// k_energy.cu -- S1: Frobenius energies E_i = ||A_i||_F^2 (
// ||M||_F^2 = sum_j ||A_j||_F^2) with fp64 accumulation and
// a NaN/Inf flag.  HBM-bound: 128-bit vectorised loads, warp-shuffle + fixed
// tree reductions (deterministic, no floating-point atomics).
#include "common.cuh"
#include "kernels.cuh"

namespace cmsvd {

constexpr int kChunk = 65536;  // floats per CTA (256 KB)

__device__ __forceinline__ double acc4(double a, float4 v, int& bad) {
  a = fma((double)v.x, (double)v.x, a);
  a = fma((double)v.y, (double)v.y, a);
  a = fma((double)v.z, (double)v.z, a);
  a = fma((double)v.w, (double)v.w, a);
  bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  return a;
}

__global__ void __launch_bounds__(kThreads) k_energy_partial(const float* __restrict__ arena,
                                                             const int64_t* __restrict__ boff,
                                                             const int64_t* __restrict__ blen,
                                                             int max_chunks, double* __restrict__ partial,
                                                             int* __restrict__ bad) {
  __shared__ double red[kThreads / 32];
  const int blk = blockIdx.y;
  const int64_t len = blen[blk];
  const int64_t start = (int64_t)blockIdx.x * kChunk;
  double acc = 0.0;
  int nonfinite = 0;
  if (start < len) {
    const float* p = arena + boff[blk] + start;
    const int64_t cnt = min((int64_t)kChunk, len - start);
    const int64_t nv = cnt >> 2;  // float4 count (block starts are 128-B aligned; kChunk % 4 == 0)
    const float4* p4 = reinterpret_cast<const float4*>(p);
    // 4 independent accumulators per thread (ILP), fixed order
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int64_t v = threadIdx.x;
    for (; v + 3 * kThreads < nv; v += 4 * kThreads) {
      float4 x0 = __ldcs(p4 + v);
      float4 x1 = __ldcs(p4 + v + kThreads);
      float4 x2 = __ldcs(p4 + v + 2 * kThreads);
      float4 x3 = __ldcs(p4 + v + 3 * kThreads);
      a0 = acc4(a0, x0, nonfinite); a1 = acc4(a1, x1, nonfinite);
      a2 = acc4(a2, x2, nonfinite); a3 = acc4(a3, x3, nonfinite);
    }
    for (; v < nv; v += kThreads) {
      float4 x0 = __ldcs(p4 + v);
      a0 = acc4(a0, x0, nonfinite);
    }
    for (int64_t e = nv * 4 + threadIdx.x; e < cnt; e += kThreads) {
      float x = p[e];
      a0 = fma((double)x, (double)x, a0);
      nonfinite |= !isfinite(x);
    }
    acc = (a0 + a1) + (a2 + a3);
  }
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)blk * max_chunks + blockIdx.x] = s;
  if (nonfinite) atomicOr(bad, 1);  // integer flag: order-independent
}

__global__ void __launch_bounds__(kThreads) k_energy_final(const double* __restrict__ partial, int max_chunks,
                                                           double* __restrict__ E) {
  __shared__ double red[kThreads / 32];
  const int blk = blockIdx.x;
  double acc = 0.0;
  for (int c = threadIdx.x; c < max_chunks; c += kThreads) acc += partial[(int64_t)blk * max_chunks + c];
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) E[blk] = s;
}

cudaError_t launch_energy(Ctx& c, const int64_t* d_boff, const int64_t* d_blen, int64_t maxlen, double* d_partial,
                          int* d_bad, double* d_E) {
  int max_chunks = (int)((maxlen + kChunk - 1) / kChunk);
  if (max_chunks < 1) max_chunks = 1;
  dim3 g1(max_chunks, c.count);
  k_energy_partial<<<g1, kThreads, 0, c.stream>>>((const float*)c.arena.p, d_boff, d_blen, max_chunks, d_partial,
                                                   d_bad);
  k_energy_final<<<c.count, kThreads, 0, c.stream>>>(d_partial, max_chunks, d_E);
  c.launches += 2;
  return cudaGetLastError();
}

int energy_max_chunks(int64_t maxlen) {
  int mc = (int)((maxlen + kChunk - 1) / kChunk);
  return mc < 1 ? 1 : mc;
}

}  // namespace cmsvd

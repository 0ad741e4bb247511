// k_gemm_ws.cu -- warp-specialised, TMA-fed 3xTF32 tcgen05 contractions of the pair path for operands
// wider than one 128-column tile (config 4: q = w = 256, m = 4096), survey K2 / K3:
//   MODE 0  Z  = Q^T F     (Lemma 1's projection Y = Q_t^T A)      K = m
//   MODE 1  R' = F - Q Z   (Thm 2's residual / Lemma 1's R)  K = q
//   MODE 2  W' = R'^T R'   (Gram of Lemma 1's R-factor)       K = m
//   MODE 3  C = A^T B (fp64 out) on K-major planes: the products with the block of the S2 subspace iteration
//           (Z = A^T Y, Y = A Z through the transposed planes; reading A22, block spectra PAPER.md:247-249)
// The fp32 operands are split ONCE into tf32 hi/lo planes (hi = RN_tf32(x), lo = x - hi): the bases Q and
// the TRUNC operands F per block after S2 (k_split_planes), Z and R' by the epilogues that produce them.
// Planes are fed to shared memory by cp.async.bulk.tensor (TMA, 128-byte swizzle) and consumed by
// tcgen05.mma kind::tf32 as hi*hi + hi*lo + lo*hi; no thread touches an operand.
//
// Persistent CTAs (one per SM), 12 warps: warp 0 = TMA producer, warp 1 = MMA issuer (one thread), warps
// 4..11 = epilogue (registers moved to them by setmaxnreg).  Output tile 128 x 256; per 32-long K stage the planes of A (128 x 32) and B (256 x 32);
// MODE 2 with w <= 256 reads its A operand out of the B tile (A = columns 128 tm .. of the same R'), so a
// stage is the B planes only and three stages fit.  Accumulation chains in TMEM are limited to one 128-long
// K block (the tensor core accumulates fp32 with truncation, k_pair_tc.cu): the two 256-column TMEM slots
// alternate per K block, the epilogue warps fold each finished block into fp32 registers with round-to-
// nearest adds while the next block's MMAs run, and write the tile while the next tile's MMAs run.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace cmsvd {
namespace {

using tc::smem_u32;

constexpr int kWsThreads = 384;   // warpgroup 0: TMA producer (warp 0) + MMA issuer (warp 1); warpgroups 1, 2: epilogue
constexpr int kWsKT = 32;                        // k elements per stage: one 128-byte swizzle row
constexpr int kWsBM = 128, kWsBN = 256;
constexpr uint32_t kWsATile = kWsBM * kWsKT * 4;  // bytes of one A plane per stage (16 KB)
constexpr uint32_t kWsBTile = kWsBN * kWsKT * 4;  // bytes of one B plane per stage (32 KB)
constexpr int kWsBlk = 128 / kWsKT;              // stages per TMEM accumulation chain (128-long K block)

// MODE 1 epilogue: the minuend F arrives by TMA in slices of kWsFC columns per column half (two slices in
// flight), so that no epilogue thread waits on a global load
constexpr int kWsFC = 16;
constexpr uint32_t kWsFHalf = kWsFC * kWsBM * 4;   // one half's slice: [col][row] fp32 (8 KB)
constexpr uint32_t kWsFBuf = 2 * kWsFHalf;         // both halves (16 KB)
constexpr int kWsFSteps = 128 / kWsFC;             // slices per tile

template <int MODE, bool SHARE_A>
struct WsCfg {
  static constexpr int kStages = SHARE_A ? 3 : 2;
  static constexpr uint32_t kStageBytes = SHARE_A ? 2 * kWsBTile : 2 * kWsATile + 2 * kWsBTile;
  static constexpr uint32_t kFOff = kStages * kStageBytes;
  static constexpr uint32_t kSmem = kFOff + (MODE == 1 ? 2 * kWsFBuf : 0) + 1024;
};

struct WsArgs {
  const int2* pairs;
  const BaseDesc* bd;
  const AppDesc* ad;
  int64_t P;
  int64_t m;
  int tiles_m, tiles_n;
  int QMAX, WMAX;
  int use_full;
  float* Zws;      // MODE 0 out: P x (QMAX x WMAX) fp32, ld QMAX
  float* Zp;       // MODE 0 out / MODE 1 in: P x 2 x (WMAX cols x QMAX rows) planes
  float* Rp;       // MODE 1 out / MODE 2 in: P x 2 x (WMAX cols x m rows) planes
  double* Wws;     // MODE 2 out: P x (WMAX x WMAX) fp64, ld WMAX
  // MODE 3 (plain batched product, S2): C[b] (Mg x Ng fp64, ld ldc, stride sC) = sum_k A[b](k, i) B[b](k, j)
  double* C64;
  int64_t ldc, sC;
  int Mg, Ng, Kg;
  int b_shared;    // 1: every problem uses B planes of batch entry 0
  int zzK;         // MODE 2 (shared-A variant): leading K elements taken from the Z planes (third map), so that
                   // the tile is Z^T Z + R'^T R' (the lower-right block of the core Gram); 0: W' alone
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_u(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// shared-memory matrix descriptors, 128-byte swizzle (layout type 2), version 1
// K-major tile (rows x 32 k, 128 B per row, 8-row atoms of 1024 B): SBO = 1024, LBO unused
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
}  // namespace

// hi/lo planes of `count` fp32 matrices (rows x cols, column-major, ld = rows, matrix i at src + i * sstride):
// dst[((i * 2 + h) * cols_dst + c) * rows + r]; columns cols .. cols_dst - 1 are zero-filled by the caller.
__global__ void __launch_bounds__(256) k_split_planes(const float* __restrict__ src, int64_t sstride, int64_t rows,
                                                      int cols, int cols_dst, float* __restrict__ dst) {
  const int i = blockIdx.z, cidx = blockIdx.y;
  const float* s = src + (int64_t)i * sstride + (int64_t)cidx * rows;
  float* dh = dst + (((int64_t)i * 2 + 0) * cols_dst + cidx) * rows;
  float* dl = dst + (((int64_t)i * 2 + 1) * cols_dst + cidx) * rows;
  (void)cols;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    float h, l;
    tc::split_tf32(s[r], h, l);
    dh[r] = h;
    dl[r] = l;
  }
}

// the same planes transposed (row-major: element (r, c) at r * cols + c), the K-major A operand of R' = F - Q Z
// (kind::tf32 takes K-major operands only: an MN-major descriptor reads zeros, tools/mn_probe.cu):
// dst[(i * 2 + h) * rows * cols + r * cols + c]
__global__ void __launch_bounds__(256) k_split_planes_t(const float* __restrict__ src, int64_t sstride, int64_t rows,
                                                        int cols, float* __restrict__ dst) {
  __shared__ float t[32][33];
  const int i = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const float* s = src + (int64_t)i * sstride;
  for (int cc = ty; cc < 32; cc += 8)
    t[cc][tx] = (r0 + tx < rows && c0 + cc < cols) ? s[(int64_t)(c0 + cc) * rows + r0 + tx] : 0.f;
  __syncthreads();
  float* dh = dst + ((int64_t)i * 2 + 0) * rows * cols;
  float* dl = dst + ((int64_t)i * 2 + 1) * rows * cols;
  for (int rr = ty; rr < 32; rr += 8) {
    if (r0 + rr < rows && c0 + tx < cols) {
      float h, l;
      tc::split_tf32(t[tx][rr], h, l);
      dh[(r0 + rr) * cols + c0 + tx] = h;
      dl[(r0 + rr) * cols + c0 + tx] = l;
    }
  }
}

// planes of fp32 matrices given by a pointer table (rows x cols each, ld = rows): normal [i][h][c][r] and
// transposed [i][h][r][c] in one pass over 32 x 32 tiles
__global__ void __launch_bounds__(256) k_split_planes_ptr(const float* const* __restrict__ srcp, int64_t rows, int cols,
                                                          float* __restrict__ dst, float* __restrict__ dst_t) {
  __shared__ float t[32][33];
  const int i = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const float* s = srcp[i];
  float* dh = dst + ((int64_t)i * 2 + 0) * rows * cols;
  float* dl = dst + ((int64_t)i * 2 + 1) * rows * cols;
  for (int cc = ty; cc < 32; cc += 8) {
    float x = 0.f;
    if (r0 + tx < rows && c0 + cc < cols) {
      x = s[(int64_t)(c0 + cc) * rows + r0 + tx];
      float h, l;
      tc::split_tf32(x, h, l);
      dh[(int64_t)(c0 + cc) * rows + r0 + tx] = h;
      dl[(int64_t)(c0 + cc) * rows + r0 + tx] = l;
    }
    t[cc][tx] = x;
  }
  __syncthreads();
  float* th = dst_t + ((int64_t)i * 2 + 0) * rows * cols;
  float* tl = dst_t + ((int64_t)i * 2 + 1) * rows * cols;
  for (int rr = ty; rr < 32; rr += 8) {
    if (r0 + rr < rows && c0 + tx < cols) {
      float h, l;
      tc::split_tf32(t[tx][rr], h, l);
      th[(r0 + rr) * cols + c0 + tx] = h;
      tl[(r0 + rr) * cols + c0 + tx] = l;
    }
  }
}

// planes of `count` fp64 matrices rounded to fp32 first (n elements each, matrix i at src + i * n):
// dst[(i * 2 + h) * n + e]
__global__ void __launch_bounds__(256) k_split_planes64(const double* __restrict__ src, int64_t n, int count,
                                                        float* __restrict__ dst) {
  const int i = blockIdx.y;
  const double* s = src + (int64_t)i * n;
  float* dh = dst + ((int64_t)i * 2 + 0) * n;
  float* dl = dst + ((int64_t)i * 2 + 1) * n;
  (void)count;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float h, l;
    tc::split_tf32((float)s[e], h, l);
    dh[e] = h;
    dl[e] = l;
  }
}

template <int MODE, bool SHARE_A>
__global__ void __launch_bounds__(kWsThreads, 1) k_gemm_ws(const __grid_constant__ CUtensorMap tmA,
                                                            const __grid_constant__ CUtensorMap tmB,
                                                            const __grid_constant__ CUtensorMap tmF,
                                                            const WsArgs a) {
  using Cfg = WsCfg<MODE, SHARE_A>;
  constexpr int kStages = Cfg::kStages;
  extern __shared__ uint8_t ws_smem_raw[];
  const uint32_t sm = (smem_u32(ws_smem_raw) + 1023u) & ~1023u;
  __shared__ uint64_t bar_full[3], bar_empty[3], bar_accf[2], bar_acce[2], bar_ff[2], bar_fe[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&bar_full[s], 1);
      tc::mbar_init(&bar_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&bar_accf[s], 1);
      tc::mbar_init(&bar_acce[s], 8);   // one arrival per epilogue warp
      tc::mbar_init(&bar_ff[s], 1);
      tc::mbar_init(&bar_fe[s], 8);
    }
    tc::fence_mbar_init();
  }
  if (wid == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  const int64_t tiles = (int64_t)a.tiles_m * a.tiles_n;
  const int64_t items = a.P * tiles;
  // K extent of an item (stages)
  auto item_k = [&](int64_t p) -> int {
    if (MODE == 1) {
      const BaseDesc b = a.bd[a.pairs[p].x];
      return (a.use_full ? b.q : b.rr);
    }
    if (MODE == 3) return a.Kg;
    if (MODE == 2) return (int)a.m + a.zzK;
    return (int)a.m;
  };

  if (wid < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (wid == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t p = item / tiles;
        const int t = (int)(item - p * tiles);
        const int tm = t / a.tiles_n, tn = t - tm * a.tiles_n;
        const int2 pr = MODE == 3 ? make_int2(0, 0) : a.pairs[p];
        const int K = item_k(p);
        const int nst = (K + kWsKT - 1) / kWsKT;
        for (int st = 0; st < nst; ++st, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1u;
          mbar_wait_u32(smem_u32(&bar_empty[s]), ph ^ 1u);
          const uint32_t full = smem_u32(&bar_full[s]);
          mbar_expect_tx(full, Cfg::kStageBytes);
          const uint32_t base = sm + s * Cfg::kStageBytes;
          const int k0 = st * kWsKT;
          if (SHARE_A) {
            if (k0 < a.zzK) {   // Z planes first (K = the projection index), then the rows of R'
              tma_load_4d(base, &tmF, k0, kWsBN * tn, 0, (int)p, full);
              tma_load_4d(base + kWsBTile, &tmF, k0, kWsBN * tn, 1, (int)p, full);
            } else {
              tma_load_4d(base, &tmB, k0 - a.zzK, kWsBN * tn, 0, (int)p, full);
              tma_load_4d(base + kWsBTile, &tmB, k0 - a.zzK, kWsBN * tn, 1, (int)p, full);
            }
          } else {
            const uint32_t bA = base, bB = base + 2 * kWsATile;
            if (MODE == 0) {
              tma_load_4d(bA, &tmA, k0, kWsBM * tm, 0, pr.x, full);
              tma_load_4d(bA + kWsATile, &tmA, k0, kWsBM * tm, 1, pr.x, full);
              tma_load_4d(bB, &tmB, k0, kWsBN * tn, 0, pr.y, full);
              tma_load_4d(bB + kWsBTile, &tmB, k0, kWsBN * tn, 1, pr.y, full);
            } else if (MODE == 3) {
              const int bb = a.b_shared ? 0 : (int)p;
              tma_load_4d(bA, &tmA, k0, kWsBM * tm, 0, (int)p, full);
              tma_load_4d(bA + kWsATile, &tmA, k0, kWsBM * tm, 1, (int)p, full);
              tma_load_4d(bB, &tmB, k0, kWsBN * tn, 0, bb, full);
              tma_load_4d(bB + kWsBTile, &tmB, k0, kWsBN * tn, 1, bb, full);
            } else if (MODE == 1) {
              tma_load_4d(bA, &tmA, k0, kWsBM * tm, 0, pr.x, full);
              tma_load_4d(bA + kWsATile, &tmA, k0, kWsBM * tm, 1, pr.x, full);
              tma_load_4d(bB, &tmB, k0, kWsBN * tn, 0, (int)p, full);
              tma_load_4d(bB + kWsBTile, &tmB, k0, kWsBN * tn, 1, (int)p, full);
            } else {
              tma_load_4d(bA, &tmA, k0, kWsBM * tm, 0, (int)p, full);
              tma_load_4d(bA + kWsATile, &tmA, k0, kWsBM * tm, 1, (int)p, full);
              tma_load_4d(bB, &tmB, k0, kWsBN * tn, 0, (int)p, full);
              tma_load_4d(bB + kWsBTile, &tmB, k0, kWsBN * tn, 1, (int)p, full);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (wid == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      const uint32_t idesc = tc::make_idesc_tf32(kWsBM, kWsBN);
      uint32_t it = 0, blk = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t p = item / tiles;
        const int t = (int)(item - p * tiles);
        const int tm = t / a.tiles_n;
        const int K = item_k(p);
        const int nst = (K + kWsKT - 1) / kWsKT;
        for (int st = 0; st < nst; ++st, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1u;
          const int slot = blk & 1;
          if ((st % kWsBlk) == 0) {   // new accumulation chain: its TMEM slot must have been drained
            mbar_wait_u32(smem_u32(&bar_acce[slot]), ((blk >> 1) & 1u) ^ 1u);
          }
          mbar_wait_u32(smem_u32(&bar_full[s]), ph);
          tc::fence_after();
          const uint32_t base = sm + s * Cfg::kStageBytes;
          uint32_t ah, al, bh, bl;
          if (SHARE_A) {
            bh = base;
            bl = base + kWsBTile;
            ah = bh + (uint32_t)tm * kWsBM * 128u;   // rows 128 tm .. of the B tile (128 B per row)
            al = bl + (uint32_t)tm * kWsBM * 128u;
          } else {
            ah = base;
            al = base + kWsATile;
            bh = base + 2 * kWsATile;
            bl = bh + kWsBTile;
          }
          const uint32_t d = tmem + 256u * slot;
#pragma unroll
          for (int ks = 0; ks < kWsKT / 8; ++ks) {
            const uint64_t dah = desc_k_sw128(ah + 32u * ks), dal = desc_k_sw128(al + 32u * ks);
            const uint64_t dbh = desc_k_sw128(bh + 32u * ks), dbl = desc_k_sw128(bl + 32u * ks);
            tc::mma_tf32(d, dah, dbh, idesc, ((st % kWsBlk) == 0 && ks == 0) ? 0u : 1u);
            tc::mma_tf32(d, dah, dbl, idesc, 1u);
            tc::mma_tf32(d, dal, dbh, idesc, 1u);
          }
          tc::mma_commit(&bar_empty[s]);
          if ((st % kWsBlk) == kWsBlk - 1 || st == nst - 1) {
            tc::mma_commit(&bar_accf[slot]);
            ++blk;
          }
        }
      }
    }
    __syncwarp();
  } else if (wid == 2 && MODE == 1) {
    // ------------------------------ minuend (F) loader ------------------------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t p = item / tiles;
        const int t = (int)(item - p * tiles);
        const int tm = t / a.tiles_n, tn = t - tm * a.tiles_n;
        const int app = a.pairs[p].y;
        for (int c = 0; c < kWsFSteps; ++c, ++it) {
          const int s = it & 1;
          mbar_wait_u32(smem_u32(&bar_fe[s]), ((it >> 1) & 1u) ^ 1u);
          const uint32_t full = smem_u32(&bar_ff[s]);
          mbar_expect_tx(full, kWsFBuf);
          const uint32_t dst = sm + Cfg::kFOff + s * kWsFBuf;
          tma_load_3d_u(dst, &tmF, kWsBM * tm, kWsBN * tn + kWsFC * c, app, full);
          tma_load_3d_u(dst + kWsFHalf, &tmF, kWsBM * tm, kWsBN * tn + 128 + kWsFC * c, app, full);
        }
      }
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ------------------------------ epilogue (8 warps) ------------------------------
    const int wq = wid & 3;                    // TMEM lane quarter this warp may read
    const int half = (wid - 4) >> 2;           // column half [128 half, 128 half + 128)
    const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
    const int row = 32 * wq + lane;
    uint32_t blk = 0, fit = 0;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      const int64_t p = item / tiles;
      const int t = (int)(item - p * tiles);
      const int tm = t / a.tiles_n, tn = t - tm * a.tiles_n;
      const int2 pr = MODE == 3 ? make_int2(0, 0) : a.pairs[p];
      const int K = item_k(p);
      const int nblk = (K + 127) / 128;
      float sum[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) sum[j] = 0.f;
      for (int b = 0; b < nblk; ++b, ++blk) {
        const int slot = blk & 1;
        mbar_wait_u32(smem_u32(&bar_accf[slot]), (blk >> 1) & 1u);
        tc::fence_after();
        const uint32_t tcol = tmem + 256u * slot + 128u * half + lane_off;
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          float v[32];
          tc::tmem_ld32(tcol + c, v);
          tc::wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c + j] += v[j];
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_acce[slot]));
      }
      // ---- write the tile: row `row` of the tile, columns 256 tn + 128 half + [0, 128) ----
      const int64_t gi = (int64_t)kWsBM * tm + row;
      const int j0 = kWsBN * tn + 128 * half;
      if (MODE == 0) {
        const BaseDesc bdesc = a.bd[pr.x];
        const int q = a.use_full ? bdesc.q : bdesc.rr;
        const int w = a.ad[pr.y].w;
        if (gi < a.QMAX) {
          float* Z = a.Zws + p * (int64_t)a.QMAX * a.WMAX;
          float* Zh = a.Zp + (p * 2 + 0) * (int64_t)a.QMAX * a.WMAX;
          float* Zl = a.Zp + (p * 2 + 1) * (int64_t)a.QMAX * a.WMAX;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            const int gj = j0 + j;
            if (gj < a.WMAX) {
              const float x = (gi < q && gj < w) ? sum[j] : 0.f;
              float h, l;
              tc::split_tf32(x, h, l);
              const int64_t o = (int64_t)gj * a.QMAX + gi;
              Z[o] = x;
              Zh[o] = h;
              Zl[o] = l;
            }
          }
        }
      } else if (MODE == 1) {
        const int w = a.ad[pr.y].w;
        float* Rh = a.Rp + (p * 2 + 0) * a.m * (int64_t)a.WMAX + gi;
        float* Rl = a.Rp + (p * 2 + 1) * a.m * (int64_t)a.WMAX + gi;
#pragma unroll
        for (int c = 0; c < kWsFSteps; ++c, ++fit) {
          const int s = fit & 1;
          mbar_wait_u32(smem_u32(&bar_ff[s]), (fit >> 1) & 1u);
          const uint32_t fb = sm + Cfg::kFOff + s * kWsFBuf + half * kWsFHalf + (uint32_t)row * 4u;
          float f[kWsFC];
#pragma unroll
          for (int j = 0; j < kWsFC; ++j)
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(f[j]) : "r"(fb + (uint32_t)j * (kWsBM * 4)));
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_fe[s]));
          if (gi < a.m) {
#pragma unroll
            for (int j = 0; j < kWsFC; ++j) {
              const int gj = j0 + kWsFC * c + j;
              if (gj < a.WMAX) {
                const float x = gj < w ? f[j] - sum[kWsFC * c + j] : 0.f;
                float h, l;
                tc::split_tf32(x, h, l);
                const int64_t o = (int64_t)gj * a.m;
                Rh[o] = h;
                Rl[o] = l;
              }
            }
          }
        }
      } else if (MODE == 3) {
        if (gi < a.Mg) {
          double* C = a.C64 + p * a.sC + gi;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            const int gj = j0 + j;
            if (gj < a.Ng) C[(int64_t)gj * a.ldc] = (double)sum[j];
          }
        }
      } else {
        const int w = a.ad[pr.y].w;
        if (gi < w) {
          double* W = a.Wws + p * (int64_t)a.WMAX * a.WMAX;
#pragma unroll
          for (int j = 0; j < 128; ++j) {
            const int gj = j0 + j;
            if (gj < w) W[(int64_t)gj * a.WMAX + gi] = (double)sum[j];
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (wid == 1) {
    __syncwarp();
    tc::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 ws_encode_fn() {
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

// K-major planes [batch][2][cols][rows] (rows contiguous = the contraction index): box 32 rows x box_cols
static bool ws_map_k(CUtensorMap* map, const float* base, int64_t rows, int cols, int64_t batch, int box_cols) {
  auto fn = ws_encode_fn();
  if (!fn || ((uintptr_t)base & 15) != 0 || (rows & 3) != 0) return false;
  cuuint64_t dims[4] = {(cuuint64_t)rows, (cuuint64_t)cols, 2, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)rows * 4, (cuuint64_t)rows * cols * 4, (cuuint64_t)rows * cols * 8};
  cuuint32_t box[4] = {(cuuint32_t)kWsKT, (cuuint32_t)box_cols, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
cudaError_t launch_split_planes(Ctx& c, const float* src, int64_t sstride, int64_t rows, int cols, int cols_dst,
                                int count, float* dst) {
  if (count <= 0 || cols <= 0) return cudaSuccess;
  dim3 g((unsigned)std::min<int64_t>((rows + 255) / 256, 64), cols, count);
  k_split_planes<<<g, 256, 0, c.stream>>>(src, sstride, rows, cols, cols_dst, dst);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_split_planes_t(Ctx& c, const float* src, int64_t sstride, int64_t rows, int cols, int count,
                                  float* dst) {
  if (count <= 0 || cols <= 0) return cudaSuccess;
  dim3 g((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32), count);
  k_split_planes_t<<<g, 256, 0, c.stream>>>(src, sstride, rows, cols, dst);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_split_planes_ptr(Ctx& c, const float* const* d_srcp, int64_t rows, int cols, int count, float* dst,
                                    float* dst_t) {
  if (count <= 0 || cols <= 0) return cudaSuccess;
  dim3 g((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32), count);
  k_split_planes_ptr<<<g, 256, 0, c.stream>>>(d_srcp, rows, cols, dst, dst_t);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_split_planes64(Ctx& c, const double* src, int64_t n, int count, float* dst) {
  if (count <= 0 || n <= 0) return cudaSuccess;
  dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 2048), count);
  k_split_planes64<<<g, 256, 0, c.stream>>>(src, n, count, dst);
  c.launches += 1;
  return cudaGetLastError();
}

bool gemm_ws_available() { return ws_encode_fn() != nullptr; }

bool gemm_ws_supported(const Ctx& c, int64_t m) { return ws_encode_fn() != nullptr && (m & 3) == 0 && c.planes_ok; }

template <int MODE, bool SHARE_A>
static cudaError_t launch_ws(Ctx& c, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tF,
                             const WsArgs& a) {
  using Cfg = WsCfg<MODE, SHARE_A>;
  cudaError_t e = cudaFuncSetAttribute(k_gemm_ws<MODE, SHARE_A>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const int64_t items = a.P * a.tiles_m * a.tiles_n;
  const unsigned grid = (unsigned)std::min<int64_t>(items, c.sm_count);
  k_gemm_ws<MODE, SHARE_A><<<grid, kWsThreads, Cfg::kSmem, c.stream>>>(tA, tB, tF, a);
  c.launches += 1;
  return cudaGetLastError();
}

// mode 0: Z = Q^T F (+ planes of Z); 1: R' planes = split(F - Q Z); 2: W' = R'^T R' (fp64 out).
// Qp / Fp: the per-block plane arenas of the context (c.d_Qp, c.d_Fp: count x 2 x planes_cols x m).
cudaError_t launch_gemm_ws(Ctx& c, int mode, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad,
                           int use_full, int QMAX, int WMAX, float* Zws, float* Zp, float* Rp, double* Wws,
                           bool add_zz) {
  if (P <= 0) return cudaSuccess;
  const int64_t m = c.m;
  WsArgs a{};
  a.pairs = pairs; a.bd = bd; a.ad = ad; a.P = P; a.m = m; a.QMAX = QMAX; a.WMAX = WMAX; a.use_full = use_full;
  a.Zws = Zws; a.Zp = Zp; a.Rp = Rp; a.Wws = Wws;
  a.tiles_n = (WMAX + kWsBN - 1) / kWsBN;
  CUtensorMap tA, tB;
  const float* Qp = (const float*)c.d_Qp.p;
  const float* Fp = (const float*)c.d_Fp.p;
  if (mode == 0) {
    a.tiles_m = (QMAX + kWsBM - 1) / kWsBM;
    if (!ws_map_k(&tA, Qp, m, c.planes_cols, c.count, kWsBM) || !ws_map_k(&tB, Fp, m, c.planes_cols, c.count, kWsBN))
      return cudaErrorInvalidValue;
    return launch_ws<0, false>(c, tA, tB, tB, a);
  }
  if (mode == 1) {
    a.tiles_m = (int)((m + kWsBM - 1) / kWsBM);
    // A = Q by rows: the transposed planes (k = column of Q contiguous)
    if (!ws_map_k(&tA, (const float*)c.d_QTp.p, c.planes_cols, (int)m, c.count, kWsBM) ||
        !ws_map_k(&tB, Zp, QMAX, WMAX, P, kWsBN))
      return cudaErrorInvalidValue;
    // the fp32 minuend F (TRUNC operands at a uniform stride): box 128 rows x kWsFC columns, no swizzle
    CUtensorMap tF;
    {
      auto fn = ws_encode_fn();
      cuuint64_t dims[3] = {(cuuint64_t)m, (cuuint64_t)c.planes_cols, (cuuint64_t)c.count};
      cuuint64_t strides[2] = {(cuuint64_t)m * 4, (cuuint64_t)c.planes_fstride * 4};
      cuuint32_t box[3] = {(cuuint32_t)kWsBM, (cuuint32_t)kWsFC, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      if (!fn || fn(&tF, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(c.planes_F), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    return launch_ws<1, false>(c, tA, tB, tF, a);
  }
  a.tiles_m = (WMAX + kWsBM - 1) / kWsBM;
  if (!ws_map_k(&tB, Rp, m, WMAX, P, kWsBN)) return cudaErrorInvalidValue;
  if (a.tiles_n == 1) {
    CUtensorMap tZ = tB;
    if (add_zz) {
      if (!ws_map_k(&tZ, Zp, QMAX, WMAX, P, kWsBN)) return cudaErrorInvalidValue;
      a.zzK = (QMAX + kWsKT - 1) / kWsKT * kWsKT;
    }
    return launch_ws<2, true>(c, tB, tB, tZ, a);
  }
  if (add_zz) return cudaErrorInvalidValue;
  if (!ws_map_k(&tA, Rp, m, WMAX, P, kWsBM)) return cudaErrorInvalidValue;
  return launch_ws<2, false>(c, tA, tB, tB, a);
}

// C[b] (M x N fp64, ld ldc, stride sC) = A[b]^T-planes . B[b]-planes: Ap [batch][2][M][K] (K contiguous),
// Bp [batch or 1][2][N][K]; 3xTF32 on k_gemm_ws (MODE 3)
cudaError_t launch_gemm_ws_tn64(Ctx& c, int batch, int M, int N, int K, const float* Ap, const float* Bp, bool b_shared,
                                double* C, int64_t ldc, int64_t sC) {
  if (batch <= 0 || M <= 0 || N <= 0) return cudaSuccess;
  WsArgs a{};
  a.P = batch; a.m = K; a.Mg = M; a.Ng = N; a.Kg = K; a.C64 = C; a.ldc = ldc; a.sC = sC; a.b_shared = b_shared ? 1 : 0;
  a.tiles_m = (M + kWsBM - 1) / kWsBM;
  a.tiles_n = (N + kWsBN - 1) / kWsBN;
  CUtensorMap tA, tB;
  if (!ws_map_k(&tA, Ap, K, M, batch, kWsBM) || !ws_map_k(&tB, Bp, K, N, b_shared ? 1 : batch, kWsBN))
    return cudaErrorInvalidValue;
  return launch_ws<3, false>(c, tA, tB, tB, a);
}

}  // namespace cmsvd

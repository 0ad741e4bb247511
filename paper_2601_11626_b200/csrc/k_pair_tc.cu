// k_pair_tc.cu -- fused per-candidate tensor-core contractions (S4, S5, S6
// Gram) on sm_100a: for the pair (base basis Q: m x q, appended F: m x w)
//   phase 1  Z  = Q^T F                      (K = m)       -> TMEM, then global (fp32)
//   phase 2  R' = F - Q Z   per 128-row tile (K = q)       -> TMEM -> registers (never HBM)
//            W' += R'^T R'  per tile         (K = 128)     -> TMEM, then global (fp64)
// i.e. Lemma 1's Y = Q_t^T A, R = A - Q_t Y and the Gram B^T B = R^T R of
// its R-factor, and Thm 2's residual.
// All products are 3xTF32 on tcgen05 (hi*hi + hi*lo + lo*hi with round-to-
// nearest splits, fp32 accumulation in TMEM, summed per 128-long K block with
// round-to-nearest adds, see below): fp32-equivalent accuracy, which the
// parity tolerances need (1xTF32 measured 1.3e-2 relative error).
// The cancellation R' = F - Q Z keeps an absolute error ~2^-22 ||Q|| ||Z|| per
// element, far below the tolerance floors (a 3-way split with six products is
// available with -DCMSVD_SPLIT3R=1).
//
// One CTA (8 warps) per pair; thread 0 issues the MMAs, all threads stage the
// operands (fp32 -> tf32 hi/lo split happens during the global -> smem copy,
// so the split operands never exist in HBM).  Operands are K-major in the
// no-swizzle canonical layout with padded strides LBO = 144 B, SBO = 1152 B
// (byte(r,k) = (k/4)*144 + (r/8)*1152 + (r%8)*16 + (k%4)*4), which makes every
// staging store pattern bank-conflict free.  Two smem stages; tcgen05.commit
// on per-stage mbarriers releases a stage.
// Limits of this kernel: q <= 128, w <= 128 (larger shapes use the SIMT path).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace cmsvd {
namespace {

#ifdef CMSVD_TC_PROF
__device__ unsigned long long g_tc_prof[8];
#define TC_T(slot) do { if (blockIdx.x < 148 && threadIdx.x == 0) { unsigned long long _t = clock64(); atomicAdd(&g_tc_prof[slot], _t - t_last); t_last = _t; } } while (0)
#else
#define TC_T(slot) do { } while (0)
#endif
constexpr int kTcThreads = 512;   // 16 warps: 4 per SM sub-partition (latency hiding for the staging)
constexpr int KT = 32;                  // k elements per stage
constexpr uint32_t LBO = 144, SBO = 1152;
constexpr uint32_t kTile = 128 * 144;   // bytes of a 128-row x 32-k operand tile (one of hi/lo)
constexpr uint32_t kStage = 6 * kTile;  // A hi/mid/lo, B hi/mid/lo (phase 1 and W' use hi/lo only)
constexpr uint32_t kSmemTc = 2 * kStage + 1024;
// R' = F - Q Z is a cancellation; with round-to-nearest splits the plain 3xTF32 products keep its error at
// ~2^-22 ||Q|| ||Z|| per element (set true for the 3-way split and six products)
#ifndef CMSVD_SPLIT3R
#define CMSVD_SPLIT3R 0
#endif
constexpr bool kSplit3R = CMSVD_SPLIT3R != 0;

__device__ __forceinline__ uint32_t poff(int r, int k) {
  return (uint32_t)((k >> 2) * LBO + (r >> 3) * SBO + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ void st_split4_3(uint8_t* hi, uint8_t* mi, uint8_t* lo, uint32_t off, float4 v) {
  float4 h, m, l;
  tc::split3_tf32(v.x, h.x, m.x, l.x);
  tc::split3_tf32(v.y, h.y, m.y, l.y);
  tc::split3_tf32(v.z, h.z, m.z, l.z);
  tc::split3_tf32(v.w, h.w, m.w, l.w);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(mi + off) = m;
  *reinterpret_cast<float4*>(lo + off) = l;
}

__device__ __forceinline__ void st_split4(uint8_t* hi, uint8_t* lo, uint32_t off, float4 v) {
  float4 h, l;
  tc::split_tf32(v.x, h.x, l.x);
  tc::split_tf32(v.y, h.y, l.y);
  tc::split_tf32(v.z, h.z, l.z);
  tc::split_tf32(v.w, h.w, l.w);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}

// Stage a (rows x 32) tile whose source is contiguous along k:
// element (r, k) = src[r*ld + k0 + k]  for r < nrows, k0 + k < kmax; else 0.
// Lanes: 8 k-chunks x 4 rows per warp -> coalesced 128 B per row in global,
// conflict-free 16 B stores in shared memory.
template <bool NC>
__device__ __forceinline__ float ldf(const float* p) { return NC ? __ldg(p) : __ldcg(p); }
template <bool NC>
__device__ __forceinline__ float4 ldf4(const float* p) {
  return NC ? __ldg(reinterpret_cast<const float4*>(p)) : __ldcg(reinterpret_cast<const float4*>(p));
}

// Split-phase staging (software pipelining): the global loads of stage i+1 are issued into registers
// before stage i's barrier and MMAs, and converted/stored one iteration later.
constexpr int kItK = 128 / (kTcThreads / 8);          // k-contiguous tile: row groups per thread
constexpr int kItR = KT / 4 / (kTcThreads / 128);      // row-contiguous tile: k quads per thread

template <bool NC>
__device__ __forceinline__ void load_kcontig(float4 (&v)[kItK], int rows, const float* __restrict__ src, int64_t ld,
                                             int nrows, int64_t k0, int64_t kmax) {
  const int tid = threadIdx.x;
  const int c = tid & 7;
  const bool vec = ((ld & 3) == 0) && ((k0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  const int64_t k = k0 + 4 * c;
#pragma unroll
  for (int i = 0; i < kItK; ++i) {
    const int r = (tid >> 3) + i * (kTcThreads / 8);
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < rows && r < nrows) {
      const float* p = src + (int64_t)r * ld + k;
      if (vec && k + 3 < kmax) {
        v[i] = ldf4<NC>(p);
      } else {
        if (k + 0 < kmax) v[i].x = ldf<NC>(p + 0);
        if (k + 1 < kmax) v[i].y = ldf<NC>(p + 1);
        if (k + 2 < kmax) v[i].z = ldf<NC>(p + 2);
        if (k + 3 < kmax) v[i].w = ldf<NC>(p + 3);
      }
    }
  }
}

// Two-source variant: rows r < nA come from srcA (row r), rows r >= nA from srcB (row r - nA) -- the operand
// of two grouped pairs with the same base (their appended blocks side by side).
template <bool NC>
__device__ __forceinline__ void load_kcontig2(float4 (&v)[kItK], int rows, const float* __restrict__ srcA, int nA,
                                              const float* __restrict__ srcB, int64_t ld, int nrows, int64_t k0,
                                              int64_t kmax) {
  const int tid = threadIdx.x;
  const int c = tid & 7;
  const bool vec = ((ld & 3) == 0) && ((k0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(srcA) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(srcB) & 15) == 0);
  const int64_t k = k0 + 4 * c;
#pragma unroll
  for (int i = 0; i < kItK; ++i) {
    const int r = (tid >> 3) + i * (kTcThreads / 8);
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < rows && r < nrows) {
      const float* p = (r < nA ? srcA + (int64_t)r * ld : srcB + (int64_t)(r - nA) * ld) + k;
      if (vec && k + 3 < kmax) {
        v[i] = ldf4<NC>(p);
      } else {
        if (k + 0 < kmax) v[i].x = ldf<NC>(p + 0);
        if (k + 1 < kmax) v[i].y = ldf<NC>(p + 1);
        if (k + 2 < kmax) v[i].z = ldf<NC>(p + 2);
        if (k + 3 < kmax) v[i].w = ldf<NC>(p + 3);
      }
    }
  }
}

__device__ __forceinline__ void store_kcontig(const float4 (&v)[kItK], uint8_t* hi, uint8_t* lo, int rows,
                                              uint8_t* mi) {
  const int tid = threadIdx.x;
  const int c = tid & 7;
#pragma unroll
  for (int i = 0; i < kItK; ++i) {
    const int r = (tid >> 3) + i * (kTcThreads / 8);
    if (r < rows) {
      if (mi) st_split4_3(hi, mi, lo, poff(r, 4 * c), v[i]);
      else st_split4(hi, lo, poff(r, 4 * c), v[i]);
    }
  }
}

__device__ __forceinline__ void load_rcontig(float4 (&v)[kItR], const float* __restrict__ src, int64_t ld, int64_t r0,
                                             int64_t rmax, int k0, int kmax) {
  const int r = threadIdx.x & 127;
  const int h = threadIdx.x >> 7;
  const bool rok = (r0 + r) < rmax;
#pragma unroll
  for (int t = 0; t < kItR; ++t) {
    const int kq = h + t * (kTcThreads / 128);
    v[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int k = k0 + 4 * kq;
    if (rok) {
      const float* p = src + (int64_t)k * ld + r0 + r;
      if (k + 0 < kmax) v[t].x = __ldg(p);
      if (k + 1 < kmax) v[t].y = __ldg(p + ld);
      if (k + 2 < kmax) v[t].z = __ldg(p + 2 * ld);
      if (k + 3 < kmax) v[t].w = __ldg(p + 3 * ld);
    }
  }
}

__device__ __forceinline__ void store_rcontig(const float4 (&v)[kItR], uint8_t* hi, uint8_t* mi, uint8_t* lo) {
  const int r = threadIdx.x & 127;
  const int h = threadIdx.x >> 7;
#pragma unroll
  for (int t = 0; t < kItR; ++t) {
    const uint32_t o = poff(r, 4 * (h + t * (kTcThreads / 128)));
    if (mi) st_split4_3(hi, mi, lo, o, v[t]);
    else st_split4(hi, lo, o, v[t]);
  }
}

// 6-product (3-way split) MMA sequence for one 32-k stage: hh, hm, mh, hl, mm, lh
__device__ __forceinline__ void issue_6x(uint32_t d_tmem, uint32_t ah, uint32_t am, uint32_t al, uint32_t bh,
                                         uint32_t bm, uint32_t bl, uint32_t idesc, bool first) {
#pragma unroll
  for (int s = 0; s < KT / 8; ++s) {
    const uint32_t o = 2 * s * LBO;
    const uint64_t dah = tc::make_desc(ah + o, LBO, SBO), dam = tc::make_desc(am + o, LBO, SBO),
                   dal = tc::make_desc(al + o, LBO, SBO);
    const uint64_t dbh = tc::make_desc(bh + o, LBO, SBO), dbm = tc::make_desc(bm + o, LBO, SBO),
                   dbl = tc::make_desc(bl + o, LBO, SBO);
    tc::mma_tf32(d_tmem, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
    tc::mma_tf32(d_tmem, dah, dbm, idesc, 1u);
    tc::mma_tf32(d_tmem, dam, dbh, idesc, 1u);
    tc::mma_tf32(d_tmem, dah, dbl, idesc, 1u);
    tc::mma_tf32(d_tmem, dam, dbm, idesc, 1u);
    tc::mma_tf32(d_tmem, dal, dbh, idesc, 1u);
  }
}

__device__ __forceinline__ void issue_3x(uint32_t d_tmem, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl,
                                         uint32_t idesc, bool first) {
#pragma unroll
  for (int s = 0; s < KT / 8; ++s) {
    const uint32_t o = 2 * s * LBO;
    const uint64_t dah = tc::make_desc(ah + o, LBO, SBO), dal = tc::make_desc(al + o, LBO, SBO);
    const uint64_t dbh = tc::make_desc(bh + o, LBO, SBO), dbl = tc::make_desc(bl + o, LBO, SBO);
    tc::mma_tf32(d_tmem, dah, dbh, idesc, (first && s == 0) ? 0u : 1u);
    tc::mma_tf32(d_tmem, dah, dbl, idesc, 1u);
    tc::mma_tf32(d_tmem, dal, dbh, idesc, 1u);
  }
}

}  // namespace

template <bool GROUP>
__global__ void __launch_bounds__(kTcThreads, 1) k_pair_tc(const int2* __restrict__ pairs,
                                                           const BaseDesc* __restrict__ bd,
                                                           const AppDesc* __restrict__ ad, int64_t m,
                                                           int use_full_basis, int QMAX, int WMAX,
                                                           float* __restrict__ Zws, double* __restrict__ Wws,
                                                           int64_t P) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned, derived by pointer arithmetic so that the compiler keeps the shared address space
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_stage[2];
  __shared__ uint64_t bar_done;
  __shared__ uint64_t bar_slot[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int wq = wid & 3;     // TMEM lane quarter of this warp (tcgen05.ld 32x32b: lanes 32*(warp%4)..)
  constexpr int kGroups = kTcThreads / 128;       // warps sharing a TMEM lane quarter
  constexpr int kColW = 128 / kGroups;            // columns per warp in the drains / epilogue
  const int half = wid >> 2;  // column group [kColW*half, kColW*half+kColW) handled by this warp in the drains
  const int64_t p = blockIdx.x;
  // Pairs 2g and 2g+1 with the same base and appended widths <= 64 are one CTA's work (their operands side
  // by side: one 128-wide MMA instead of two half-empty ones); the odd CTA of such a group exits.
  auto grouped_at = [&](int64_t x) {
    if (!GROUP || x < 0 || (x & 1) || x + 1 >= P) return false;
    const int2 p0 = pairs[x], p1 = pairs[x + 1];
    return p0.x == p1.x && ad[p0.y].w <= 64 && ad[p1.y].w <= 64;
  };
  if (grouped_at(p - 1)) return;
  const bool grouped = grouped_at(p);
  const int2 pr = pairs[p];
  const BaseDesc b = bd[pr.x];
  const AppDesc a = ad[pr.y];
  const AppDesc a2 = grouped ? ad[pairs[p + 1].y] : a;
  const int q = use_full_basis ? b.q : b.rr;
  const int w1 = a.w;                     // columns of the first pair (all columns when not grouped)
  const int w = grouped ? w1 + a2.w : w1;
  const int wp = ((w + 31) / 32) * 32;   // MMA N (multiple of 32 for the 32-column TMEM drains)
  float* Zg = Zws + p * (int64_t)QMAX * WMAX;
  double* Wg = Wws + p * (int64_t)WMAX * WMAX;
  float* Zg2 = grouped ? Zg + (int64_t)QMAX * WMAX : Zg;
  double* Wg2 = grouped ? Wg + (int64_t)WMAX * WMAX : Wg;
  const float* Q = b.basis;
  const float* F = a.F;
  const float* F2 = grouped ? a2.F : a.F;

  if (wid == 0) tc::tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_stage[0], 1);
    tc::mbar_init(&bar_stage[1], 1);
    tc::mbar_init(&bar_done, 1);
    tc::mbar_init(&bar_slot[0], 1);
    tc::mbar_init(&bar_slot[1], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  // TMEM columns: phase 1 Z block accumulators (two slots) at [0,128) and [128,256), running sum at
  // [256,384); phase 2 R' tile accumulator at [0,128), W' tile contribution at [128,256), sum at [256,384).
  const uint32_t t_z0 = tmem, t_r = tmem, t_w = tmem + 128, t_sum = tmem + 256;
  const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
  const int c_lo = kColW * half, c_hi = min(wp, kColW * half + kColW);
  // per-stage / per-slot mbarrier phases and "MMAs outstanding" flags as bit masks (bit s), so that the
  // runtime stage index never forces them into local memory
  uint32_t ph_stage = 0, ph_done = 0, ph_slot = 0, used = 0;
  auto stage_ptr = [&](int s, int which) { return sm + s * kStage + which * kTile; };
  auto acquire = [&](int s) {
    if ((used >> s) & 1u) {
      tc::mbar_wait(&bar_stage[s], (ph_stage >> s) & 1u);
      ph_stage ^= 1u << s;
      used &= ~(1u << s);
    }
  };
  // The tensor core accumulates fp32 with truncation: the bias grows linearly with the number of
  // accumulations (measured 1.3e-5 relative at K = 2048).  Accumulation chains in TMEM are therefore
  // limited to one 128-long K block; blocks are summed in fp32 registers with round-to-nearest.
  // running sum (fp32, round-to-nearest adds) kept in TMEM columns [256, 256+wp)
  bool sum_empty = true;
  auto drain_add = [&](uint32_t tcol) {
    for (int c = c_lo; c < c_hi; c += 32) {
      float v[32], acc[32];
      tc::tmem_ld32(tcol + lane_off + c, v);
      if (!sum_empty) tc::tmem_ld32(t_sum + lane_off + c, acc);
      tc::wait_ld();
      if (!sum_empty) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += acc[j];
      }
      tc::tmem_st32(t_sum + lane_off + c, v);
    }
    tc::wait_st();
    sum_empty = false;
  };
  // write the running sum (rows 32*wq + lane, this warp's column half) to global through a callback
  auto drain_sum = [&](auto&& store) {
    for (int c = c_lo; c < c_hi; c += 32) {
      float v[32];
      if (sum_empty) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      } else {
        tc::tmem_ld32(t_sum + lane_off + c, v);
        tc::wait_ld();
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) store(c + j, v[j]);
    }
  };
  const uint32_t idesc_z = tc::make_idesc_tf32(128, wp);
  constexpr int kBlk = 128 / KT;  // stages per K block

#ifdef CMSVD_TC_PROF
  unsigned long long t_last = clock64();
#endif
  // ---------------- phase 1: Z = Q^T F (K = m) ----------------
  if (w > 0) {
    int it = 0;
    const int nst = (int)((m + KT - 1) / KT);
    float4 qa[kItK], fb[kItK];
    load_kcontig<true>(qa, 128, Q, m, q, 0, m);
    if constexpr (GROUP) load_kcontig2<true>(fb, wp, F, w1, F2, m, w, 0, m);
    else load_kcontig<true>(fb, wp, F, m, w, 0, m);
    for (; it < nst; ++it) {
      const int s = it & 1;
      const int blk = it / kBlk, slot = blk & 1;
      acquire(s);
      store_kcontig(qa, stage_ptr(s, 0), stage_ptr(s, 1), 128, nullptr);
      store_kcontig(fb, stage_ptr(s, 2), stage_ptr(s, 3), wp, nullptr);
      if (it + 1 < nst) {  // next stage's loads fly during this stage's barrier and MMAs
        const int64_t k1 = (int64_t)(it + 1) * KT;
        load_kcontig<true>(qa, 128, Q, m, q, k1, m);
        if constexpr (GROUP) load_kcontig2<true>(fb, wp, F, w1, F2, m, w, k1, m);
        else load_kcontig<true>(fb, wp, F, m, w, k1, m);
      }
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        issue_3x(t_z0 + 128 * slot, tc::smem_u32(stage_ptr(s, 0)), tc::smem_u32(stage_ptr(s, 1)),
                 tc::smem_u32(stage_ptr(s, 2)), tc::smem_u32(stage_ptr(s, 3)), idesc_z, (it % kBlk) == 0);
        tc::mma_commit(&bar_stage[s]);
        if ((it % kBlk) == kBlk - 1 || it == nst - 1) tc::mma_commit(&bar_slot[slot]);
      }
      used |= 1u << s;
      // once block blk is issued, drain block blk-1 (its slot is reused by block blk+1)
      if (((it % kBlk) == kBlk - 1 || it == nst - 1) && blk >= 1) {
        const int ps = (blk - 1) & 1;
        tc::mbar_wait(&bar_slot[ps], (ph_slot >> ps) & 1u);
        ph_slot ^= 1u << ps;
        tc::fence_after();
        drain_add(t_z0 + 128 * ps);
        tc::fence_before();
      }
    }
    {  // last block
      const int lb = (nst - 1) / kBlk, ls = lb & 1;
      tc::mbar_wait(&bar_slot[ls], (ph_slot >> ls) & 1u);
      ph_slot ^= 1u << ls;
      tc::fence_after();
      drain_add(t_z0 + 128 * ls);
    }
    for (int s = 0; s < 2; ++s) acquire(s);
    const int ar = 32 * wq + lane;
    drain_sum([&](int j, float x) {
      if (ar < q && j < w) {
        if (!GROUP || j < w1) Zg[(int64_t)j * QMAX + ar] = x;
        else Zg2[(int64_t)(j - w1) * QMAX + ar] = x;
      }
    });
  }
  __threadfence_block();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  sum_empty = true;

  TC_T(0);  // phase 1 incl. Z drain
  // ---------------- phase 2: per 128-row tile, R' = F - Q Z, W' += R'^T R' ----------------
  const uint32_t idesc_r = tc::make_idesc_tf32(128, wp);
  const uint32_t idesc_w = tc::make_idesc_tf32(128, wp);
  int it = 0;
  float4 qv[kItR], zv[kItK];
  if (w > 0 && m > 0) {
    load_rcontig(qv, Q, m, 0, m, 0, q);
    if constexpr (GROUP) load_kcontig2<false>(zv, wp, Zg, w1, Zg2, QMAX, w, 0, q);
    else load_kcontig<false>(zv, wp, Zg, QMAX, w, 0, q);
  }
  for (int64_t m0 = 0; m0 < m && w > 0; m0 += 128) {
    // R accumulator over a-chunks of 32
    bool r_first = true;
    for (int a0 = 0; a0 < q; a0 += KT, ++it) {
      const int s = it & 1;
      acquire(s);
      store_rcontig(qv, stage_ptr(s, 0), kSplit3R ? stage_ptr(s, 4) : nullptr, stage_ptr(s, 1));
      store_kcontig(zv, stage_ptr(s, 2), stage_ptr(s, 3), wp, kSplit3R ? stage_ptr(s, 5) : nullptr);
      {  // next stage (possibly the first of the next tile): its loads also cover the epilogue
        int64_t nm0 = m0;
        int na0 = a0 + KT;
        if (na0 >= q) { na0 = 0; nm0 = m0 + 128; }
        if (nm0 < m) {
          load_rcontig(qv, Q, m, nm0, m, na0, q);
          if constexpr (GROUP) load_kcontig2<false>(zv, wp, Zg, w1, Zg2, QMAX, w, na0, q);
          else load_kcontig<false>(zv, wp, Zg, QMAX, w, na0, q);
        }
      }
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        if (kSplit3R)
          issue_6x(t_r, tc::smem_u32(stage_ptr(s, 0)), tc::smem_u32(stage_ptr(s, 4)), tc::smem_u32(stage_ptr(s, 1)),
                   tc::smem_u32(stage_ptr(s, 2)), tc::smem_u32(stage_ptr(s, 5)), tc::smem_u32(stage_ptr(s, 3)),
                   idesc_r, r_first);
        else
          issue_3x(t_r, tc::smem_u32(stage_ptr(s, 0)), tc::smem_u32(stage_ptr(s, 1)), tc::smem_u32(stage_ptr(s, 2)),
                   tc::smem_u32(stage_ptr(s, 3)), idesc_r, r_first);
        tc::mma_commit(&bar_stage[s]);
      }
      used |= 1u << s;
      r_first = false;
    }
    TC_T(1);  // staging + R' MMA issue
    if (tid == 0) tc::mma_commit(&bar_done);
    // the epilogue's F values (rows 32*wq + lane of this tile, this warp's 32 columns), loaded while
    // the tensor core finishes R'
    const int64_t grow_e = m0 + 32 * wq + lane;
    const int c0_e = kColW * half;
    float fpre[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int bcol = c0_e + j;
      if constexpr (GROUP)
        fpre[j] = (c0_e < wp && bcol < w && grow_e < m)
                      ? __ldg((bcol < w1 ? F + (int64_t)bcol * m : F2 + (int64_t)(bcol - w1) * m) + grow_e)
                      : 0.f;
      else
        fpre[j] = (c0_e < wp && bcol < w && grow_e < m) ? __ldg(F + (int64_t)bcol * m + grow_e) : 0.f;
    }
    tc::mbar_wait(&bar_done, ph_done);
    ph_done ^= 1;
    for (int s = 0; s < 2; ++s) acquire(s);
    tc::fence_after();
    TC_T(2);  // wait for R' MMAs
    // epilogue: rows r = 32*wq + lane of this tile -> R' into chunk buffer wq (columns of this warp's half)
    // chunk buffer (hi, lo) wq: operand with rows = b (128), k = r_local (32)
    uint8_t* chi = sm + (uint32_t)wq * 2 * kTile;
    uint8_t* clo = chi + kTile;
    const int64_t grow = m0 + 32 * wq + lane;
    for (int c0 = kColW * half; c0 < kColW * half + kColW; c0 += 32) {
      float v[32];
      if (c0 < wp) {
        if (q > 0) {
          tc::tmem_ld32(t_r + lane_off + c0, v);
          tc::wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int bcol = c0 + j;
        float rv = 0.f;
        if (c0 < wp && bcol < w && grow < m) rv = fpre[j] - v[j];
        float h, l;
        tc::split_tf32(rv, h, l);
        const uint32_t o = poff(bcol, lane);
        *reinterpret_cast<float*>(chi + o) = h;
        *reinterpret_cast<float*>(clo + o) = l;
      }
    }
    TC_T(3);  // epilogue (TMEM -> F - QZ -> split -> smem)
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      for (int cw = 0; cw < 4; ++cw) {
        const uint32_t h = tc::smem_u32(sm + cw * 2 * kTile), l = h + kTile;
        issue_3x(t_w, h, l, h, l, idesc_w, cw == 0);
      }
      tc::mma_commit(&bar_done);
    }
    tc::mbar_wait(&bar_done, ph_done);
    ph_done ^= 1;
    tc::fence_after();
    TC_T(4);  // W' MMAs
    drain_add(t_w);          // this tile's W' contribution -> fp32 registers (round-to-nearest)
    tc::fence_before();
    TC_T(5);  // drain
  }
  // ---------------- W' (rows b = 32*wq + lane) from the running sum ----------------
  if (w > 0) {
    const int br = 32 * wq + lane;
    drain_sum([&](int j, float x) {
      if constexpr (GROUP) {
        if (br < w1 && j < w1) Wg[(int64_t)j * WMAX + br] = (double)x;          // first pair's block
        else if (br >= w1 && j >= w1 && br < w && j < w)                         // second pair's block
          Wg2[(int64_t)(j - w1) * WMAX + (br - w1)] = (double)x;
      } else {
        if (br < w && j < w) Wg[(int64_t)j * WMAX + br] = (double)x;
      }
    });
  }
  tc::fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// Batched 3xTF32 GEMM tiles for operands wider than one 128-column tile (q or w > 128, e.g. config 4's
// 256-column bases and TRUNC operands), with the staging, MMA issue and per-128-K-block round-to-nearest
// summation of k_pair_tc's phase 1:
//   kTN    C (M x N) = A^T B       A: K x M, B: K x N column-major   (Z = Q^T F, W' = R'^T R')
//   kNNSub C (M x N) = C0 - A B    A: M x K, B: K x N column-major   (R' = F - Q Z)
// One CTA (16 warps) per 128 x 128 output tile: grid (tiles_m * tiles_n, batch); sym = 1 computes the
// lower tiles only and mirrors them.  OUT64 stores C as fp64 (W' for the fp64 Gram assembly).
// ---------------------------------------------------------------------------
enum { kTN = 0, kNNSub = 1, kNN = 2 };  // kNN: C = A B (A: M x K, B: K x N column-major)
// NT = output tile width (128, or 256 for the plain A^T B: the A tile is then staged once per 256 output
// columns, which brings the shared-memory traffic per MMA below the tensor core's operand rate; TMEM then
// holds one 256-column block slot + the running sum, so a block's drain is not overlapped with the next
// block's MMAs).
template <int MODE, bool OUT64, int NT>
__global__ void __launch_bounds__(kTcThreads, 1) k_gemm_tc(const GemmDesc* __restrict__ descs, int tiles_n) {
  static_assert(NT == 128 || (NT == 256 && MODE == kTN), "256-wide tiles: A^T B only");
  static_assert(MODE != kNNSub || !OUT64, "C0 - A B: fp32 output");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_stage[2];
  __shared__ uint64_t bar_slot[2];
  __shared__ uint32_t tmem_base;
  const GemmDesc d = descs[blockIdx.y];
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = 128 * tm, j0 = NT * tn;
  if (i0 >= d.M || j0 >= d.N) return;
  if (d.sym && NT == 128 && tm < tn) return;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int wq = wid & 3;
  constexpr int kGroups = kTcThreads / 128;
  constexpr int kColW = NT / kGroups;
  constexpr int kSlots = NT == 128 ? 2 : 1;
  const int half = wid >> 2;
  const int mr = min(128, d.M - i0), nc = min(NT, d.N - j0);
  const int wp = ((nc + 31) / 32) * 32;
  const int K = d.K;
  if (wid == 0) tc::tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_stage[0], 1);
    tc::mbar_init(&bar_stage[1], 1);
    tc::mbar_init(&bar_slot[0], 1);
    tc::mbar_init(&bar_slot[1], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t t_acc = tmem, t_sum = tmem + 256;   // block slots at [0, 256), running sum at [256, 256 + NT)
  const uint32_t lane_off = (uint32_t)(32 * wq) << 16;
  const int c_lo = kColW * half, c_hi = min(wp, kColW * half + kColW);
  uint32_t ph_stage = 0, ph_slot = 0, used = 0;
  auto stage_ptr = [&](int s, int which) { return sm + s * kStage + which * kTile; };
  auto acquire = [&](int s) {
    if ((used >> s) & 1u) {
      tc::mbar_wait(&bar_stage[s], (ph_stage >> s) & 1u);
      ph_stage ^= 1u << s;
      used &= ~(1u << s);
    }
  };
  bool sum_empty = true;
  auto drain_add = [&](uint32_t tcol) {  // 16-column chunks: the prefetched operands stay in registers
    for (int c = c_lo; c < c_hi; c += 16) {
      float v[16], acc[16];
      tc::tmem_ld16(tcol + lane_off + c, v);
      if (!sum_empty) tc::tmem_ld16(t_sum + lane_off + c, acc);
      tc::wait_ld();
      if (!sum_empty) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += acc[j];
      }
      tc::tmem_st16(t_sum + lane_off + c, v);
    }
    tc::wait_st();
    sum_empty = false;
  };
  const uint32_t idesc = tc::make_idesc_tf32(128, wp);
  constexpr int kBlk = 128 / KT;
  const int nst = (K + KT - 1) / KT;
  // B operand: NT rows (hi at stage tile 2 [.. 2 + NT/128), lo after it)
  constexpr int kBT = NT / 128;
  float4 av[kItK], ar[kItR], bv[kBT][kItK];
  auto load_a = [&](int64_t k0) {
    if (MODE == kTN) load_kcontig<true>(av, 128, d.A + (int64_t)i0 * d.lda, d.lda, mr, k0, K);
    else load_rcontig(ar, d.A, d.lda, i0, d.M, (int)k0, K);  // kNNSub, kNN
  };
  auto load_b = [&](int64_t k0) {
#pragma unroll
    for (int h = 0; h < kBT; ++h)
      load_kcontig<true>(bv[h], 128, d.B + (int64_t)(j0 + 128 * h) * d.ldb, d.ldb, nc - 128 * h, k0, K);
  };
  auto wait_block = [&](int pb) {  // MMAs of K block pb complete; fold it into the running sum
    const int ps = pb & 1;
    tc::mbar_wait(&bar_slot[ps], (ph_slot >> ps) & 1u);
    ph_slot ^= 1u << ps;
    tc::fence_after();
    drain_add(t_acc + 128 * (ps % kSlots));
  };
  if (nst > 0) {
    load_a(0);
    load_b(0);
  }
  for (int it = 0; it < nst; ++it) {
    const int s = it & 1;
    const int blk = it / kBlk, slot = blk % kSlots;
    acquire(s);
    if (MODE == kTN) store_kcontig(av, stage_ptr(s, 0), stage_ptr(s, 1), 128, nullptr);
    else store_rcontig(ar, stage_ptr(s, 0), nullptr, stage_ptr(s, 1));  // kNNSub, kNN
#pragma unroll
    for (int h = 0; h < kBT; ++h)
      store_kcontig(bv[h], stage_ptr(s, 2) + h * kTile, stage_ptr(s, 2 + kBT) + h * kTile, 128, nullptr);
    if (it + 1 < nst) {
      const int64_t k1 = (int64_t)(it + 1) * KT;
      load_a(k1);
      load_b(k1);
    }
    // one slot (NT = 256): the previous block must be drained before this block's first MMA
    if (kSlots == 1 && (it % kBlk) == 0 && blk >= 1) {
      wait_block(blk - 1);
      tc::fence_before();
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      issue_3x(t_acc + 128 * slot, tc::smem_u32(stage_ptr(s, 0)), tc::smem_u32(stage_ptr(s, 1)),
               tc::smem_u32(stage_ptr(s, 2)), tc::smem_u32(stage_ptr(s, 2 + kBT)), idesc, (it % kBlk) == 0);
      tc::mma_commit(&bar_stage[s]);
      if ((it % kBlk) == kBlk - 1 || it == nst - 1) tc::mma_commit(&bar_slot[blk & 1]);
    }
    used |= 1u << s;
    // two slots: once block blk is issued, drain block blk-1 (its slot is reused by block blk+1)
    if (kSlots == 2 && ((it % kBlk) == kBlk - 1 || it == nst - 1) && blk >= 1) {
      wait_block(blk - 1);
      tc::fence_before();
    }
  }
  // epilogue: row r = 32 wq + lane of the tile, this warp's columns [c_lo, c_hi);
  // the minuend C0 (one 32-column chunk) is loaded while the tensor core finishes the last block
  const int r = 32 * wq + lane;
  float c0v[32];
  if (MODE == kNNSub) {
    static_assert(MODE != kNNSub || kColW == 32, "one 32-column chunk per warp");
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int jj = c_lo + j;
      c0v[j] = (d.C0 && r < mr && jj < c_hi && jj < nc) ? __ldg(d.C0 + (int64_t)(j0 + jj) * d.ldc0 + i0 + r) : 0.f;
    }
  }
  if (nst > 0) wait_block((nst - 1) / kBlk);  // last block
  for (int s = 0; s < 2; ++s) acquire(s);
  for (int c = c_lo; c < c_hi; c += 32) {
    float v[32];
    if (sum_empty) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    } else {
      tc::tmem_ld32(t_sum + lane_off + c, v);
      tc::wait_ld();
    }
    if (r < mr) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int jj = c + j;
        if (jj < nc) {
          const int64_t gi = i0 + r, gj = j0 + jj;
          float x = v[j];
          if (MODE == kNNSub) x = c0v[j] - x;
          const bool mirror = d.sym && NT == 128 && tm != tn;
          if (OUT64) {
            double* C = reinterpret_cast<double*>(d.C);
            C[gj * d.ldc + gi] = (double)x;
            if (mirror) C[gi * d.ldc + gj] = (double)x;
          } else {
            float* C = reinterpret_cast<float*>(d.C);
            C[gj * d.ldc + gi] = x;
            if (mirror) C[gi * d.ldc + gj] = x;
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(tmem, 512);
}

cudaError_t launch_gemm_tc_nn64(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN) {
  if (nprob <= 0) return cudaSuccess;
  const int tm = (maxM + 127) / 128, tn = (maxN + 127) / 128;
  dim3 g(tm * tn, nprob);
  cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<kNN, true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemTc);
  if (e != cudaSuccess) return e;
  k_gemm_tc<kNN, true, 128><<<g, kTcThreads, kSmemTc, c.stream>>>(d_descs, tn);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_gemm_tc(Ctx& c, const GemmDesc* d_descs, int nprob, int maxM, int maxN, bool nnsub, bool out64) {
  if (nprob <= 0) return cudaSuccess;
  // 256-wide tiles for the plain fp32 A^T B when the operand is wider than one tile (Z = Q^T F)
  const bool wide = !nnsub && !out64 && maxN > 128 && c.tc_wide;
  const int ntile = wide ? 256 : 128;
  const int tm = (maxM + 127) / 128, tn = (maxN + ntile - 1) / ntile;
  dim3 g(tm * tn, nprob);
#define GTC(MODE_, O64_, NT_)                                                                                      \
  do {                                                                                                             \
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<MODE_, O64_, NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)kSmemTc);                                                            \
    if (e != cudaSuccess) return e;                                                                                \
    k_gemm_tc<MODE_, O64_, NT_><<<g, kTcThreads, kSmemTc, c.stream>>>(d_descs, tn);                               \
  } while (0)
  if (nnsub) {
    if (out64) return cudaErrorInvalidValue;
    GTC(kNNSub, false, 128);
  } else if (out64) {
    GTC(kTN, true, 128);
  } else if (wide) {
    GTC(kTN, false, 256);
  } else {
    GTC(kTN, false, 128);
  }
#undef GTC
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_pair_tc(Ctx& c, const int2* pairs, int64_t P, const BaseDesc* bd, const AppDesc* ad, int64_t m,
                           int use_full_basis, int QMAX, int WMAX, float* Zws, double* Wws) {
  if (P <= 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_pair_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTc);
  if (e != cudaSuccess) return e;
  // grouping of same-base pairs (operands <= 64 columns) only where it can happen: the general kernel keeps
  // its register budget
  if (WMAX <= 64) {
    e = cudaFuncSetAttribute(k_pair_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTc);
    if (e != cudaSuccess) return e;
    k_pair_tc<true><<<(unsigned)P, kTcThreads, kSmemTc, c.stream>>>(pairs, bd, ad, m, use_full_basis, QMAX, WMAX,
                                                                     Zws, Wws, P);
  } else {
    k_pair_tc<false><<<(unsigned)P, kTcThreads, kSmemTc, c.stream>>>(pairs, bd, ad, m, use_full_basis, QMAX, WMAX,
                                                                      Zws, Wws, P);
  }
  c.launches += 1;
  return cudaGetLastError();
}

}  // namespace cmsvd

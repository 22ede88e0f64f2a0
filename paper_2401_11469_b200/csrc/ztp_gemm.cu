// Resized GEMMs of one TP linear on sm_100a:
//   FWD  Y^T[j,t]  = sum_{k in S} W^T[k,j] X^T[k,t]
//   DX   dX^T[k,t] = sum_{j<n}   W^T[k,j] G^T[j,t], k in S
//   DW   dW^T[k,j] = sum_t       X^T[k,t] G^T[j,t], k in S
// with rows P of dX^T / dW^T imputed by Zero in the same kernel.
//
// Design: persistent, warp-specialised tcgen05
// kind::f16 GEMM accumulating in TMEM (2 x 256 fp32 columns, double-buffered so
// the epilogue of tile i overlaps the mainloop of tile i+1).
//   CG = 2 (default): a CTA pair (cluster of 2 on one TPC) computes a 256x256
//          tile with tcgen05.mma.cta_group::2 -- each CTA stages its 128 rows
//          of A and half (128 columns) of B, so L2->SM operand traffic per
//          FLOP is 2/3 of a 128x256 single-CTA tile.
//   CG = 1: a CTA computes a 128x256 tile (small-M problems).
//   warp 0      TMA producer (dense boxes from compact operands, or
//               tile::gather4 of the lineage rows in gather mode)
//   warp 1      MMA issuer (one thread of the even CTA), tcgen05.commit
//               multicast -> smem-slot release in both CTAs
//   warp 2      TMEM allocator
//   warps 4-11  epilogue (2 warpgroups: TMEM lane quarter x column half):
//               tcgen05.ld -> (GeLU | GeLU' | none) -> bf16 ->
//               swizzled smem staging -> 128-bit coalesced row stores at the
//               lineage row map (a6: scatter + Zero imputation), or fp32
//               split-K partials reduced by ztp_splitk_reduce.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "ztp_internal.h"
#include "ztp_ptx.cuh"

namespace ztp {

constexpr int BM = 128;   // rows per CTA
constexpr int BN = 256;   // tile columns (per CTA pair when CG = 2)
constexpr int BK = 64;
constexpr int EPI_WARPS = 8;                   // 2 warpgroups: TMEM lane quarter x column half
constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;           // 16 KB
constexpr int STAGING_PER_WARP = 32 * 128;     // one 32 x 64 bf16 plane (32 x 32 fp32)

template <int CG>
struct Cfg {
  static constexpr int BNL = BN / CG;                    // B columns staged by one CTA
  static constexpr int TM = BM * CG;                     // tile rows
#ifndef ZTP_STG3
#define ZTP_STG3 0
#endif
  // 2-CTA: a 4-stage operand ring and three epilogue staging buffers per warp
  // (stores of two chunks in flight while the third is filled); 1-CTA: 3 + 2
  static constexpr int STAGES = CG == 2 ? (ZTP_STG3 ? 4 : 5) : 3;
  static constexpr int STG_BUFS = (CG == 2 && ZTP_STG3) ? 3 : 2;
  static constexpr int B_BYTES = BNL * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // per CTA
  static constexpr int RING = STAGES * STAGE_BYTES;
  static constexpr int STAGING = EPI_WARPS * STG_BUFS * STAGING_PER_WARP;   // rotating per warp
  static constexpr int BARS = (2 * STAGES + 4) * 8 + 16;
  static constexpr int TOTAL = 1024 + RING + STAGING + BARS;
};

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// GeLU tanh approximation and its derivative, fp32.  tanh uses the
// SFU (tanh.approx.f32, max rel. error ~2^-11), below the 2^-8 resolution of
// the bf16 outputs these epilogues produce.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 8 bf16 (16 B) at p; a ragged last chunk (nv < 8 valid columns) is stored
// element-wise so nothing past the logical width is written.
__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* p, const uint4& w, int nv) {
  if (nv >= 8) {
    st_global_v4(p, w);
    return;
  }
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)(x[i >> 1] >> (16 * (i & 1)));
}

// Packed (f32x2, FFMA2 / FMUL2) GeLU of two values and, when want_d, its
// derivative, sharing one tanh:
//   u = c (x + a x^3),  t = tanh(u),  GeLU = x/2 (1 + t),
//   GeLU' = (1 + t)/2 + x/2 (1 - t^2) c (1 + 3 a x^2).
__device__ __forceinline__ void gelu2(float2 x, float2& h, float2& d, bool want_d) {
  constexpr float C = 0.7978845608028654f, CA = 0.7978845608028654f * 0.044715f;
  const float2 x2 = __fmul2_rn(x, x);
  const float2 s = __ffma2_rn(x2, make_float2(CA, CA), make_float2(C, C));
  const float2 u = __fmul2_rn(x, s);
  const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 hx = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  h = __ffma2_rn(hx, t, hx);
  if (want_d) {
    const float2 A = __ffma2_rn(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
    const float2 B = __ffma2_rn(make_float2(-t.x, -t.y), t, make_float2(1.0f, 1.0f));
    const float2 du = __ffma2_rn(x2, make_float2(3.0f * CA, 3.0f * CA), make_float2(C, C));
    d = __ffma2_rn(__fmul2_rn(hx, B), du, A);
  }
}
__device__ __forceinline__ uint32_t pack2(float2 v) { return pack_bf16(v.x, v.y); }
__device__ __forceinline__ float2 unpack2(uint32_t u) { return make_float2(bf16_lo(u), bf16_hi(u)); }


// Work units: computed tiles x K-splits first, then (unsplit launches only)
// the DX / DW tiles whose rows are all pruned -- they skip the MMA and write
// Zero.  Split launches leave pruned rows to the reduce kernel.
struct Work {
  int m0, n0, kb0, kb1, split;
  bool zero;
  int half;   // -1: the whole 256-column tile; 0 / 1: a 128-column half (2-CTA FWD tail, GemmParams::tail_r)
};

template <int KIND, int TM>
struct Sched {
  int m_tiles, n_tiles, mc, tiles_c, units_c, zero_m, num_units, num_kb, S, kbs;
  __device__ __forceinline__ Sched(const GemmParams& p) {
    m_tiles = (p.M + TM - 1) / TM;
    n_tiles = (p.N + BN - 1) / BN;
    num_kb = (p.kdim + BK - 1) / BK;
    mc = m_tiles;
    if (KIND != KIND_FWD) {
      const int mk = (p.n_kept + TM - 1) / TM;
      mc = mk < m_tiles ? mk : m_tiles;
    }
    tiles_c = mc * n_tiles;
    S = p.splits;
    kbs = p.kb_per_split;
    units_c = tiles_c * S;
    zero_m = m_tiles - mc;
    num_units = units_c + (S == 1 && !p.skip_zero ? zero_m * n_tiles : 0);
    tail_r = (KIND == KIND_FWD && S == 1) ? p.tail_r : 0;
    num_units += tail_r;   // the last tail_r tiles run as two 128-column halves each
  }
  int tail_r;
  // all-pruned (zero) units come FIRST: the epilogue warps write them while
  // the producer / MMA warps, which skip them, already stream the first tile.
  __device__ __forceinline__ Work get(int u0) const {
    Work w;
    const int nz = num_units - units_c - tail_r;   // all-pruned units (the tail halves are computed ones)
    w.half = -1;
    if (u0 >= nz) {
      const int u = u0 - nz;
      int s = u / tiles_c, t = u - s * tiles_c;
      if (tail_r > 0 && u >= tiles_c - tail_r) {   // FWD tail: last round's tiles as halves, one per pair
        const int v = u - (tiles_c - tail_r);
        s = 0;
        t = tiles_c - tail_r + (v >> 1);
        w.half = v & 1;
      }
      w.m0 = (t % mc) * TM;
      w.n0 = (t / mc) * BN;
      w.split = s;
      w.kb0 = s * kbs;
      w.kb1 = min(num_kb, w.kb0 + kbs);
      w.zero = false;
    } else {
      const int v = u0;
      w.m0 = (mc + v % zero_m) * TM;
      w.n0 = (v / zero_m) * BN;
      w.split = 0;
      w.kb0 = w.kb1 = 0;
      w.zero = true;
    }
    return w;
  }
};

// Pipeline state a CTA's roles carry from one work unit to the next.
struct Pipe {
  int stage = 0;       // smem ring slot (producer / MMA)
  uint32_t phase = 0;
  int acc = 0;         // TMEM accumulator buffer (MMA / epilogue)
  uint32_t aphase = 0;
  int sk = 0;          // epilogue staging buffers used so far (ping-pong)
};

// ---- TMA producer of one work unit (warp 0).
// A consumer's wait for a column block of its producer's output (ZTP_FLAGS):
// acquire the block's completion count, then order the TMA loads after it.
// A count that never arrives (a broken dependency) traps after 2 s instead
// of hanging the device.
__device__ __forceinline__ void flag_wait(const unsigned long long* f, unsigned long long tgt) {
  if (ld_acquire_u64(f) < tgt) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_u64(f) < tgt) {
      __nanosleep(64);
      if (globaltimer() - t0 > 2000000000ull) __trap();
    }
  }
  fence_proxy_async_global();
}

// AG / BG: operand A / B gathered row-by-row with TMA gather4 through the
// lineage list (true) or loaded as dense TMA boxes from a compact, already
// row-selected tensor (false; rows past the compact extent are zero-filled).
template <int KIND, int CG, bool AG, bool BG>
__device__ __forceinline__ void produce_unit(const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmParams& p,
                                             const Work& wk, int rank, bool leader, int lane, uint8_t* ring,
                                             uint64_t* full, uint64_t* empty, Pipe& ps,
                                             unsigned long long ftgt = 0) {
  using C = Cfg<CG>;
  constexpr int BNL = C::BNL;
  const int am0 = wk.m0 + BM * rank;   // this CTA's 128 rows of the tile (A)
  const int bn0 = wk.n0 + BNL * rank;  // this CTA's columns of B
  int ar0 = 0, ar1 = 0, ar2 = 0, ar3 = 0;
  if (KIND != KIND_FWD && AG) {
    const int mb = am0 + 4 * lane;
    ar0 = (mb + 0 < p.n_kept) ? __ldg(p.kept + mb + 0) : p.oob_row;
    ar1 = (mb + 1 < p.n_kept) ? __ldg(p.kept + mb + 1) : p.oob_row;
    ar2 = (mb + 2 < p.n_kept) ? __ldg(p.kept + mb + 2) : p.oob_row;
    ar3 = (mb + 3 < p.n_kept) ? __ldg(p.kept + mb + 3) : p.oob_row;
  }
  for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
    mbar_wait(&empty[ps.stage], ps.phase ^ 1);
    uint8_t* sa = ring + ps.stage * C::STAGE_BYTES;
    uint8_t* sb = sa + A_BYTES;
    uint64_t* fb = &full[ps.stage];
    if (leader && lane == 0) mbar_expect_tx(fb, CG * (wk.half < 0 ? C::STAGE_BYTES : A_BYTES + 8192));
    __syncwarp();
    auto load = [&](const CUtensorMap* tm, void* dst, int c0, int c1) {
      if (CG == 2)
        tma_load_2d_cg2(tm, fb, dst, c0, c1);
      else
        tma_load_2d(tm, fb, dst, c0, c1);
    };
    auto gather = [&](const CUtensorMap* tm, void* dst, int col, int r0, int r1, int r2, int r3) {
      if (CG == 2)
        tma_gather4_cg2(tm, fb, dst, col, r0, r1, r2, r3);
      else
        tma_gather4(tm, fb, dst, col, r0, r1, r2, r3);
    };
    if (KIND == KIND_FWD) {
      // both operands MN-major (contraction rows outer)
      if (AG || BG) {
        const int g = lane & 15, half = lane >> 4;
        const int kbase = kb * BK + 4 * g;
        int r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = kbase + i;
          r[i] = (k < p.n_kept) ? __ldg(p.kept + k) : p.oob_row;
        }
        if (AG) gather(tmA, sa + half * 8192 + g * 512, am0 + 64 * half, r[0], r[1], r[2], r[3]);
        if (BG) {
          constexpr int NB = BNL / 64, PER = NB / 2;
#pragma unroll
          for (int b = half * PER; b < (half + 1) * PER; ++b)
            gather(tmB, sb + b * 8192 + g * 512, bn0 + 64 * b, r[0], r[1], r[2], r[3]);
        }
      }
      if (lane == 0) {
        if (!AG) {
          load(tmA, sa, am0, kb * BK);
          load(tmA, sa + 8192, am0 + 64, kb * BK);
        }
        if (p.fi_flags && kb == wk.kb0) flag_wait(p.fi_flags + wk.n0 / BN, ftgt);
        if (!BG) {
          if (wk.half >= 0) {   // a 128-column half: this CTA's h-th 64-column box into block 0
            load(tmB, sb, bn0 + 64 * wk.half, kb * BK);
          } else {
#pragma unroll
            for (int b = 0; b < BNL / 64; ++b) load(tmB, sb + b * 8192, bn0 + 64 * b, kb * BK);
          }
        }
      }
    } else {
      // A: K-major rows (m) x 64 contraction columns
      if (AG) gather(tmA, sa + lane * 512, kb * BK, ar0, ar1, ar2, ar3);
      if (lane == 0) {
        if (!AG) load(tmA, sa, kb * BK, am0);
        if (p.fi_flags && kb == wk.kb0) flag_wait(p.fi_flags + wk.n0 / BN, ftgt);
        if (KIND == KIND_DX) {
          // B = G^T [n, N] MN-major dense: 64 contraction rows x BNL columns
#pragma unroll
          for (int b = 0; b < BNL / 64; ++b) load(tmB, sb + b * 8192, bn0 + 64 * b, kb * BK);
        } else {
          // B = G^T [n, N] K-major dense: BNL rows (output cols j) x 64 tokens
          load(tmB, sb, kb * BK, bn0);
        }
      }
    }
    if (++ps.stage == C::STAGES) {
      ps.stage = 0;
      ps.phase ^= 1;
    }
  }
}

// ---- The first unit's first stages with the A loads issued BEFORE the PDL
// wait (p.a_early: A -- weights, or FWD activations for dW -- is not written
// by the preceding kernel), the B loads after it; dense boxes only.  The ring
// is empty at kernel start, so the stages' empty barriers pass at once.
template <int KIND, int CG>
__device__ __forceinline__ void produce_unit_early(const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmParams& p,
                                                   Work wk, int rank, bool leader, int lane, uint8_t* ring,
                                                   uint64_t* full, uint64_t* empty, Pipe& ps) {
  using C = Cfg<CG>;
  constexpr int BNL = C::BNL;
  const int am0 = wk.m0 + BM * rank, bn0 = wk.n0 + BNL * rank;
  const int n = min(C::STAGES, wk.kb1 - wk.kb0);
  auto load = [&](const CUtensorMap* tm, uint64_t* fb, void* dst, int c0, int c1) {
    if (CG == 2)
      tma_load_2d_cg2(tm, fb, dst, c0, c1);
    else
      tma_load_2d(tm, fb, dst, c0, c1);
  };
  const int st0 = ps.stage;
  const uint32_t ph0 = ps.phase;
  for (int i = 0; i < n; ++i) {
    const int kb = wk.kb0 + i;
    mbar_wait(&empty[ps.stage], ps.phase ^ 1);
    uint8_t* sa = ring + ps.stage * C::STAGE_BYTES;
    uint64_t* fb = &full[ps.stage];
    if (leader && lane == 0) mbar_expect_tx(fb, CG * (wk.half < 0 ? C::STAGE_BYTES : A_BYTES + 8192));
    __syncwarp();
    if (lane == 0) {
      if (KIND == KIND_FWD) {
        load(tmA, fb, sa, am0, kb * BK);
        load(tmA, fb, sa + 8192, am0 + 64, kb * BK);
      } else {
        load(tmA, fb, sa, kb * BK, am0);
      }
    }
    if (++ps.stage == C::STAGES) {
      ps.stage = 0;
      ps.phase ^= 1;
    }
  }
  pdl_wait();   // B (the predecessor's output) from here on
  pdl_trigger();   // only after the wait: a dependent launched off this trigger may itself prefetch early
  int stg = st0;
  for (int i = 0; i < n; ++i) {
    const int kb = wk.kb0 + i;
    uint8_t* sb = ring + stg * C::STAGE_BYTES + A_BYTES;
    uint64_t* fb = &full[stg];
    if (lane == 0) {
      if (KIND == KIND_DW) {
        load(tmB, fb, sb, kb * BK, bn0);
      } else if (wk.half >= 0) {
        load(tmB, fb, sb, bn0 + 64 * wk.half, kb * BK);
      } else {
#pragma unroll
        for (int b = 0; b < BNL / 64; ++b) load(tmB, fb, sb + b * 8192, bn0 + 64 * b, kb * BK);
      }
    }
    if (++stg == C::STAGES) stg = 0;
  }
  (void)ph0;
  wk.kb0 += n;
  if (wk.kb0 < wk.kb1) produce_unit<KIND, CG, false, false>(tmA, tmB, p, wk, rank, leader, lane, ring, full, empty, ps);
}

// ---- MMA issuer of one work unit (warp 1 of the even CTA; lane 0 issues).
template <int KIND, int CG>
__device__ __forceinline__ void mma_unit(const Work& wk, int lane, uint16_t pmask, uint8_t* ring, uint64_t* full,
                                         uint64_t* empty, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                         Pipe& ps, unsigned long long** first = nullptr) {
  using C = Cfg<CG>;
  constexpr uint32_t IDESC_F = make_idesc_bf16(C::TM, BN, KIND == KIND_FWD ? 1 : 0, KIND == KIND_DW ? 0 : 1);
  constexpr uint32_t IDESC_H = make_idesc_bf16(C::TM, BN / 2, KIND == KIND_FWD ? 1 : 0, KIND == KIND_DW ? 0 : 1);
  const uint32_t IDESC = wk.half >= 0 ? IDESC_H : IDESC_F;
  mbar_wait(&tempty[ps.acc], ps.aphase ^ 1);
  tc_fence_after();
  const uint32_t d_tmem = tmem_base + ps.acc * BN;
  for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
    mbar_wait(&full[ps.stage], ps.phase);
    tc_fence_after();
    if (first && *first) {
      if (lane == 0) **first = globaltimer();
      *first = nullptr;
    }
    if (lane == 0) {
      const uint32_t sa = smem_u32(ring + ps.stage * C::STAGE_BYTES);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        uint64_t ad, bd;
        if (KIND == KIND_FWD)
          ad = make_sdesc_sw128(sa + kk * 2048, 8192, 1024);  // MN-major: LBO = 64-col block stride
        else
          ad = make_sdesc_sw128(sa + kk * 32, 16, 1024);      // K-major: SBO = 8-row group stride
        if (KIND == KIND_DW)
          bd = make_sdesc_sw128(sb + kk * 32, 16, 1024);
        else
          bd = make_sdesc_sw128(sb + kk * 2048, 8192, 1024);
        const uint32_t accum = (kb > wk.kb0 || kk > 0) ? 1u : 0u;
        if (CG == 2)
          umma_bf16_cg2(d_tmem, ad, bd, IDESC, accum);
        else
          umma_bf16(d_tmem, ad, bd, IDESC, accum);
      }
      if (CG == 2)
        umma_commit_mc(&empty[ps.stage], pmask);
      else
        umma_commit(&empty[ps.stage]);
    }
    __syncwarp();
    if (++ps.stage == C::STAGES) {
      ps.stage = 0;
      ps.phase ^= 1;
    }
  }
  if (lane == 0) {
    if (CG == 2)
      umma_commit_mc(&tfull[ps.acc], pmask);
    else
      umma_commit(&tfull[ps.acc]);
  }
  __syncwarp();
  if (++ps.acc == 2) {
    ps.acc = 0;
    ps.aphase ^= 1;
  }
}

// ---- Epilogue of one work unit (warps 4-11: TMEM lane quarter x column half).
template <int KIND, int CG>
__device__ __forceinline__ void epilogue_unit(const CUtensorMap* tmO, const CUtensorMap* tmO2, const CUtensorMap* tmW,
                                              const GemmParams& p, int S, const Work& wk, int rank, int ew, int lane,
                                              uint8_t* staging, uint64_t* tfull, uint64_t* tempty,
                                              uint32_t tmem_base, Pipe& ps, unsigned long long** first = nullptr) {
  const int lq = ew & 3;               // TMEM lane quarter == warp % 4 (rows lq*32 .. +31)
  const int ch = ew >> 2;              // column half of the 256-column accumulator
  constexpr int NBUF = Cfg<CG>::STG_BUFS;
  uint8_t* const stg_base = staging + ew * NBUF * STAGING_PER_WARP;
  uint8_t* stg = stg_base;
  auto release = [&]() {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (CG == 2)
        mbar_arrive_leader(&tempty[ps.acc]);
      else
        mbar_arrive(&tempty[ps.acc]);
    }
    if (++ps.acc == 2) {
      ps.acc = 0;
      ps.aphase ^= 1;
    }
  };
  const int m0 = wk.m0 + BM * rank, n0 = wk.n0;
  const bool zt = wk.zero;
  // a 128-column half unit (2-CTA FWD tail): accumulator columns [64 ch, +64)
  // hold the tile's columns [128 ch + 64 h, +64) -- each CTA staged its h-th box
  const bool hu = wk.half >= 0;
  const int nchunks = hu ? 1 : BN / 128;
  const uint32_t tbase = tmem_base + ((uint32_t)(lq * 32) << 16) + ps.acc * BN + ch * (hu ? BN / 4 : BN / 2);
  const int nc0 = n0 + ch * (BN / 2) + (hu ? 64 * wk.half : 0);   // first output column of this warp
  // Two staging buffers per warp alternate: before refilling one, the
  // lanes that issued TMA stores wait until at most the other buffer's
  // store is still reading (bulk wait_group.read 1).
  auto staging_free = [&]() {
    if (lane < 8) bulk_wait_read_n<NBUF - 1>();
    __syncwarp();
    stg = stg_base + (ps.sk % NBUF) * STAGING_PER_WARP;
    ++ps.sk;
  };
  if (S > 1) {
    // ---- split-K partial: fp32 tile -> ws[split] via TMA box stores
    //      (rows >= n_kept / cols >= N are outside the ws map: not written)
    mbar_wait(&tfull[ps.acc], ps.aphase);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tbase + c * 32, v);
      tmem_ld_wait();
      if (c == BN / 64 - 1) release();   // accumulator fully in registers: TMEM free
      staging_free();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_shared_v4(stg + lane * 128 + ((q ^ (lane & 7)) << 4),
                     make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(tmW, stg, nc0 + c * 32, m0 + lq * 32, wk.split);
        bulk_commit();
      }
    }
    return;
  }
  // this lane owns tile row m = m0 + lq*32 + lane; its output row index
  const int m = m0 + lq * 32 + lane;
  int orow = p.oob_out;                       // rows outside the output are not written
  int arow = 0;
  if (m < p.M) {
    int o;
    if (p.out_dense)
      o = m;                                      // compact output (row i <- unit i of the list)
    else if (KIND == KIND_FWD)
      o = p.out_pos ? __ldg(p.out_pos + m) : m;   // producer-side compaction for the next layer
    else
      o = (m < p.n_kept) ? __ldg(p.kept + m) : __ldg(p.pruned + (m - p.n_kept));
    if (o >= 0) orow = o;
    arow = p.aux_by_m ? m : o;
  }
  const bool dense_out = p.out_dense;
  // rows of the 4-row scatter group this lane issues (lanes 0..7)
  int sr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sr[j] = __shfl_sync(0xFFFFFFFFu, orow, (4 * lane + j) & 31);
  const bool has_aux = (p.epi == EPI_GELU_GRAD || p.epi == EPI_MUL) && !zt;
  // GeLU' operand (pre-activation, or GeLU'(pre) itself for EPI_MUL) of this
  // lane's row: the first chunk into registers and the rest of the row's
  // segment into L2 BEFORE waiting for the accumulator, so its HBM latency
  // hides behind this tile's mainloop
  uint4 pin[8];
  auto load_aux = [&](int col0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      pin[i] = make_uint4(0u, 0u, 0u, 0u);
      if (m < p.n_kept && col0 + 8 * i < p.N)
        pin[i] = __ldg(reinterpret_cast<const uint4*>(p.aux + (int64_t)arow * p.ld_aux + col0 + 8 * i));
    }
  };
  if (has_aux) {
    if (m < p.n_kept && nc0 + 72 <= p.N)
      prefetch_l2_bulk(p.aux + (int64_t)arow * p.ld_aux + nc0 + 64, (uint32_t)min(64, p.N - nc0 - 64) / 8 * 16);
    load_aux(nc0);
  }
  if (!zt) {
    mbar_wait(&tfull[ps.acc], ps.aphase);
    tc_fence_after();
    if (first && *first) {
      if (lane == 0) **first = globaltimer();
      *first = nullptr;
    }
  }
  if (p.dbg & 2) {
    if (!zt) release();
    return;
  }
  if (zt && !dense_out && !p.spread && p.zero_generic) {
    // All-pruned tile at a lineage row map (the Zero rows P): no data
    // to stage, so no TMA scatter4 (4 rows x 128 B per op) -- generic 16-byte
    // stores, eight lanes per 128-byte row segment, four rows per instruction.
    if (p.dbg & 1) return;
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 1
    for (int c = 0; c < BN / 128; ++c) {
      const int col = nc0 + c * 64 + 8 * (lane & 7);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int orr = __shfl_sync(0xFFFFFFFFu, orow, 4 * i + (lane >> 3));
        if (orr < 0 || orr >= p.out_rows || col >= p.N) continue;
        __nv_bfloat16* dst = p.out + (int64_t)orr * p.ld_out + col;
        if (col + 8 <= p.N)
          st_global_v4(dst, z4);
        else
          for (int e = 0; e < p.N - col; ++e) reinterpret_cast<uint16_t*>(dst)[e] = 0;
      }
    }
    return;
  }
  // one TMA store of a staged 32 x 64 bf16 plane (dense box or 4-row scatter)
  auto store_plane = [&](const CUtensorMap* tm, uint8_t* buf, int col0) {
    fence_proxy_async_smem();
    __syncwarp();
    if (p.dbg & 1) return;
    if (dense_out) {
      if (lane == 0) {
        tma_store_2d(tm, buf, col0, m0 + lq * 32);
        bulk_commit();
      }
    } else if (lane < 8) {
      tma_scatter4(tm, buf + lane * 512, col0, sr[0], sr[1], sr[2], sr[3]);
      bulk_commit();
    }
  };
  // Output-pruned dW written in full (p.spread).  The chunk's compact
  // columns [col0, col0 + 64) own the full columns [F0, F1) from their first
  // kept column up to the next chunk's (chunk 0 from column 0, the last one
  // to n_full), so every full column -- kept value or Zero unit --
  // is written by exactly one chunk.  Lane = row: each lane parks its packed
  // row in the warp's staging (8 KB, both ping-pong buffers: no TMA store is
  // in flight here) at a 136-byte pitch (2-way bank conflicts at most), the
  // span's col_pos entries go to shared memory once as byte offsets, then
  // every 8-column group is one uniform step: 8 shared loads from the lane's
  // own row, masked packing, one 16-byte store per row (a group shared with
  // the neighbouring chunk goes out element-wise).
  constexpr int SP_PITCH = 136, SP_POS = 32 * SP_PITCH, SP_PIECE = 64;   // pos staging: 64 groups (2 KB)
  auto spread_chunk = [&](const uint32_t (&pk)[32], int col0) {
    const uint32_t sb = smem_u32(stg_base);
    __syncwarp();   // previous chunk's reads of this buffer are done
    if (!zt) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(sb + lane * SP_PITCH + 8 * i), "r"(pk[2 * i]),
                     "r"(pk[2 * i + 1])
                     : "memory");
    }
    if ((p.dbg & 1) || col0 >= p.N) return;
    const int F0 = col0 == 0 ? 0 : __ldg(p.col_kept + col0);
    const int F1 = col0 + 64 >= p.N ? p.n_full : __ldg(p.col_kept + col0 + 64);
    const int V0 = F0 >> 3, nvec = ((F1 + 7) >> 3) - V0;
    const bool row_ok = orow >= 0 && orow < p.out_rows;
    __nv_bfloat16* const drow = p.full_out + (int64_t)(row_ok ? orow : 0) * p.ld_full;
    const uint32_t rb = sb + lane * SP_PITCH;
#pragma unroll 1
    for (int v0 = 0; v0 < nvec; v0 += SP_PIECE) {
      const int nv = min(SP_PIECE, nvec - v0);
      __syncwarp();   // the previous piece's offsets are consumed
      for (int k = lane; k < 8 * nv; k += 32) {
        const int j = 8 * (V0 + v0) + k;
        int o = -1;   // byte offset of the kept value in the lane's row, -1: Zero unit, -2: not owned
        if (j < F0 || j >= F1) {
          o = -2;
        } else if (!zt) {
          const int q = __ldg(p.col_pos + j) - col0;
          if ((unsigned)q < 64u) o = 2 * q;   // ascending lists: kept columns of the span are this chunk's
        }
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + SP_POS + 4 * k), "r"(o) : "memory");
      }
      __syncwarp();
#pragma unroll 1
      for (int g = 0; g < nv; ++g) {
        const uint4 qa = ld_shared_v4(sb + SP_POS + 32 * g);
        const uint4 qb = ld_shared_v4(sb + SP_POS + 32 * g + 16);
        const int q[8] = {(int)qa.x, (int)qa.y, (int)qa.z, (int)qa.w, (int)qb.x, (int)qb.y, (int)qb.z, (int)qb.w};
        uint32_t x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint16_t h = 0;
          if (q[e] >= 0) asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(rb + q[e]) : "memory");
          x[e] = h;
        }
        if (!row_ok) continue;
        __nv_bfloat16* dst = drow + 8 * (V0 + v0 + g);
        if (q[0] != -2 && q[7] != -2) {   // the whole group is this chunk's ([F0, F1) is contiguous)
          st_global_v4(dst, make_uint4(x[0] | (x[1] << 16), x[2] | (x[3] << 16), x[4] | (x[5] << 16),
                                       x[6] | (x[7] << 16)));
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (q[e] != -2) reinterpret_cast<uint16_t*>(dst)[e] = (uint16_t)x[e];
        }
      }
    }
  };
  const bool two_planes = p.epi == EPI_GELU || p.epi == EPI_GELU_D;
#pragma unroll 1
  for (int c = 0; c < nchunks; ++c) {
    const int col0 = nc0 + c * 64;
    uint32_t v[64];
    if (has_aux && c > 0) load_aux(col0);   // before the TMEM load so the two overlap (L2 hit)
    if (!zt) {
      tmem_ld_32x32b_x32(tbase + c * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld_32x32b_x32(tbase + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_ld_wait();
      if (c == nchunks - 1) release();   // accumulator fully in registers: TMEM free for tile i+2
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = 0u;
    }
    if (two_planes) {
      // out <- pre (EPI_GELU) or GeLU'(pre) (EPI_GELU_D); out2 <- GeLU(pre).
      // Both staging buffers are filled in one pass (tanh shared).
      if (lane < 8) bulk_wait_read0();
      __syncwarp();
      uint8_t* const b0 = stg_base;
      uint8_t* const b1 = stg_base + STAGING_PER_WARP;
      const bool want_d = p.epi == EPI_GELU_D;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        uint32_t w0[4], w1[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 x = make_float2(__uint_as_float(v[qq * 8 + 2 * j]), __uint_as_float(v[qq * 8 + 2 * j + 1]));
          float2 hv, dv;
          gelu2(x, hv, dv, want_d);
          w0[j] = want_d ? pack2(dv) : pack2(x);
          w1[j] = pack2(hv);
        }
        const uint32_t off = lane * 128 + ((qq ^ (lane & 7)) << 4);
        st_shared_v4(b0 + off, make_uint4(w0[0], w0[1], w0[2], w0[3]));
        st_shared_v4(b1 + off, make_uint4(w1[0], w1[1], w1[2], w1[3]));
      }
      store_plane(tmO, b0, col0);
      store_plane(tmO2, b1, col0);
    } else if (p.spread) {   // dW (no epilogue math): packed row -> full-column spread
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) pk[j] = pack_bf16(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
      spread_chunk(pk, col0);
    } else {
      staging_free();
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        uint32_t w[4];
        const uint32_t a4[4] = {pin[qq].x, pin[qq].y, pin[qq].z, pin[qq].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 x = make_float2(__uint_as_float(v[qq * 8 + 2 * j]), __uint_as_float(v[qq * 8 + 2 * j + 1]));
          if (has_aux) {
            // G1 = dH * GeLU'(pre_in)  (EPI_MUL: aux already holds GeLU'(pre))
            const float2 a = unpack2(a4[j]);
            if (p.epi == EPI_GELU_GRAD) {
              float2 hv, dv;
              gelu2(a, hv, dv, true);
              x = __fmul2_rn(x, dv);
            } else {
              x = __fmul2_rn(x, a);
            }
          }
          w[j] = pack2(x);
        }
        st_shared_v4(stg + lane * 128 + ((qq ^ (lane & 7)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
      }
      store_plane(tmO, stg, col0);
    }
  }
}

// Shared prologue of both kernels: barriers, TMEM allocation, then the PDL
// handshake.  Returns the TMEM base address.
template <int CG>
__device__ __forceinline__ uint32_t kernel_prologue(uint64_t* full, uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                                                    uint32_t* tmem_slot, int warp) {
  using C = Cfg<CG>;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS * CG);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2)
      tmem_alloc_cg2(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  return *tmem_slot;
}

template <int CG>
__device__ __forceinline__ void kernel_teardown(uint32_t tmem_base, int warp) {
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (CG == 2)
      tmem_dealloc_cg2(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}

template <int KIND, int CG, bool AG, bool BG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    ztp_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2,
                    const __grid_constant__ CUtensorMap tmW, const GemmParams p) {
  using C = Cfg<CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* staging = smem + C::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = (CG == 2 || p.cs > 1) ? cluster_ctarank() : 0u;   // rank in the cluster
  const int rank = CG == 2 ? (int)(crank & 1u) : 0;                         // CTA rank in the pair
  const bool leader = rank == 0;
  const uint16_t pmask = (uint16_t)(0x3u << (crank & ~1u));   // this pair's CTAs (commit multicast)
  const int csplit = p.cs > 1 ? (int)crank / CG : 0;          // cluster split-K: this pair's K-slice
  const int pair = blockIdx.x / CG, npairs = gridDim.x / CG;
  unsigned long long* const cst = p.cta_stamps ? p.cta_stamps + (size_t)blockIdx.x * 8 : nullptr;
  if (cst && threadIdx.x == 0) cst[0] = globaltimer();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (p.fo_target && blockIdx.x == 0 && threadIdx.x == 0) {
    // this launch's share of the slot's cumulative target, also added to the
    // column blocks it does not produce (so every block of the slot keeps
    // pace with the target); before CTA 0 can trigger a consumer
    atomicAdd(p.fo_target, p.fo_T);
    for (int nb = p.fo_nb; nb < FLAG_NB; ++nb) atomicAdd(p.fo_flags + nb, p.fo_T);
    __threadfence();
  }
  const uint32_t tmem_base = kernel_prologue<CG>(full, empty, tfull, tempty, tmem_slot, warp);
  // prologue done (barriers, TMEM, descriptor prefetch): wait for the
  // preceding kernel's results, let the next kernel begin its own prologue.
  // pdl_late (a dW GEMM right after the dX GEMM it does not depend on): run
  // now, wait for the predecessor only before exiting, so successors still
  // see it complete (its own inputs were complete before the dX started).
  // flag consumer: only B comes from the preceding kernel, and it is waited
  // for per column block; the PDL wait (and, after it, the trigger -- so a
  // successor launched off it sees everything up to the producer complete)
  // is left to warp 3
  const bool fcons = !AG && !BG && p.fi_flags != nullptr;
  const bool early = !fcons && p.a_early && !AG && !BG && !p.pdl_late && p.cs <= 1;   // producer waits in unit 1
  if (fcons) {
    if (warp == 3) {
      pdl_wait();
      pdl_trigger();
    }
  } else {
    if (!p.pdl_late && !(early && warp == 0)) pdl_wait();
    if (!(early && warp == 0)) pdl_trigger();
  }
  if (cst && threadIdx.x == 0) cst[1] = globaltimer();
  if (p.stamp != nullptr && threadIdx.x == 0) atomicMin(p.stamp, (unsigned long long)globaltimer());
  if (p.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p.prof_stamp, ~(unsigned long long)globaltimer());

  const Sched<KIND, C::TM> sc(p);
  // persistent round-robin over work units; cluster split-K: exactly one unit,
  // K-slice `csplit` of the cluster's tile
  int u_first = pair, u_step = npairs;
  if (p.cs > 1) {
    u_first = csplit * sc.tiles_c + (int)(blockIdx.x / (CG * p.cs));
    u_step = sc.num_units;
  }
  Pipe ps;
  if (warp == 0) {
    bool waited = !early;
    const unsigned long long ftgt = fcons ? ld_acquire_u64(p.fi_target) : 0ull;
    for (int u = u_first; u < sc.num_units; u += u_step) {
      const Work wk = sc.get(u);
      if (wk.zero) continue;
      if (!waited) {
        if constexpr (!AG && !BG)
          produce_unit_early<KIND, CG>(&tmA, &tmB, p, wk, rank, leader, lane, ring, full, empty, ps);
        waited = true;
      } else {
        produce_unit<KIND, CG, AG, BG>(&tmA, &tmB, p, wk, rank, leader, lane, ring, full, empty, ps, ftgt);
      }
    }
    if (!waited) {
      pdl_wait();
      pdl_trigger();
    }
  } else if (warp == 1 && leader) {
    unsigned long long* f = cst ? cst + 2 : nullptr;
    for (int u = u_first; u < sc.num_units; u += u_step) {
      const Work wk = sc.get(u);
      if (!wk.zero) mma_unit<KIND, CG>(wk, lane, pmask, ring, full, empty, tfull, tempty, tmem_base, ps, &f);
    }
    if (cst && lane == 0) cst[3] = globaltimer();
  } else if (warp >= 4 && p.cs > 1) {
    // cluster split-K: this pair's K-slice is accumulated; reduced below
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
  } else if (warp >= 4) {
    unsigned long long* f = (cst && warp == 4) ? cst + 4 : nullptr;
    // flag producer: a unit's column block is counted once its stores are
    // performed -- checked one unit later (at most the last unit's bulk
    // groups still pending), so the epilogue never stalls on its own stores
    int pend0 = -1, pend1 = -1;
    const bool two = p.epi == EPI_GELU || p.epi == EPI_GELU_D;
    for (int u = u_first; u < sc.num_units; u += u_step) {
      const Work wk = sc.get(u);
      if (p.fo_flags && pend1 >= 0) {
        if (lane < 8) {
          if (two)
            bulk_wait_n<4>();
          else
            bulk_wait_n<2>();
        }
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async_global();
          red_release_add_u64(p.fo_flags + pend1, 1ull);
        }
      }
      epilogue_unit<KIND, CG>(&tmO, &tmO2, &tmW, p, sc.S, wk, rank, warp - 4, lane, staging, tfull, tempty,
                              tmem_base, ps, &f);
      pend1 = pend0;
      pend0 = wk.n0 / BN;
    }
    if (cst && warp == 4 && lane == 0) cst[5] = globaltimer();
    if (lane < 8) bulk_wait0();   // all output writes performed before the CTA exits
    if (p.fo_flags) {
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_global();
        if (pend1 >= 0) red_release_add_u64(p.fo_flags + pend1, 1ull);
        if (pend0 >= 0) red_release_add_u64(p.fo_flags + pend0, 1ull);
      }
    }
    if (cst && warp == 4 && lane == 0) cst[6] = globaltimer();
  }

  if (p.cs > 1) {
    // ============ cluster split-K reduce through distributed shared memory
    // The S pairs of the cluster hold the S K-slice partials of one tile in
    // TMEM.  The tile's 256 columns are 8 chunks of 32; chunk j is owned by
    // split j % S.  Every CTA sends each chunk's fp32 partial (its 128 rows)
    // to the same-half CTA of the owner, into slot [source split][chunk] of
    // the owner's operand ring (idle once every slice is accumulated); the
    // owner sums the S slots in split order 0..S-1 (fixed order: the result
    // is deterministic), rounds to bf16 and stores its rows at the lineage
    // row map (rows past n_kept hold exact zeros).
    const int S = p.cs;
    const int slots = (8 + S - 1) / S;
    const int tile = (int)(blockIdx.x / (CG * S));
    const int m0 = (tile % sc.mc) * C::TM + BM * rank;
    const int n0 = (tile / sc.mc) * BN;
    const uint32_t rbuf = smem_u32(ring);
    const int ew = warp - 4, lq = ew & 3, ch = ew >> 2;
    const uint32_t row_off = (uint32_t)(lq * 32 + lane) * 128u;
    // #1: every slice of the cluster is accumulated (each epilogue waited its
    // tfull before arriving): all rings are free to receive
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp >= 4) {
      const uint32_t tb = tmem_base + ((uint32_t)(lq * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int j = ch * 4 + c;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tb + j * 32, v);
        tmem_ld_wait();
        const int owner = j % S, slot = j / S;
        const uint32_t dst = mapa_shared(rbuf + (uint32_t)((csplit * slots + slot) * 128) * 128u + row_off,
                                         (uint32_t)(owner * CG + rank));
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_cluster_v4(dst + ((uint32_t)(q ^ (lane & 7)) << 4), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
    // #2: every slot delivered (cluster barrier release / acquire)
    cluster_sync();
    if (warp >= 4) {
      const int m = m0 + lq * 32 + lane;
      int orow = -1;
      if (m < p.M) orow = p.out_dense ? m : (m < p.n_kept ? __ldg(p.kept + m) : __ldg(p.pruned + (m - p.n_kept)));
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int j = ch * 4 + c;
        if (j % S != csplit) continue;
        const int slot = j / S;
        float a[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = 0.f;
#pragma unroll 1
        for (int src = 0; src < S; ++src) {
          const uint32_t base = rbuf + (uint32_t)((src * slots + slot) * 128) * 128u + row_off;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 x = ld_shared_v4(base + ((uint32_t)(q ^ (lane & 7)) << 4));
            a[4 * q] += __uint_as_float(x.x);
            a[4 * q + 1] += __uint_as_float(x.y);
            a[4 * q + 2] += __uint_as_float(x.z);
            a[4 * q + 3] += __uint_as_float(x.w);
          }
        }
        if (orow >= 0 && !(p.dbg & 1)) {
          __nv_bfloat16* o = p.out + (int64_t)orow * p.ld_out + n0 + j * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int col = n0 + j * 32 + 8 * i;
            if (col < p.N)
              store_bf16x8(o + 8 * i,
                           make_uint4(pack_bf16(a[8 * i], a[8 * i + 1]), pack_bf16(a[8 * i + 2], a[8 * i + 3]),
                                      pack_bf16(a[8 * i + 4], a[8 * i + 5]), pack_bf16(a[8 * i + 6], a[8 * i + 7])),
                           p.N - col);
          }
        }
      }
      // rows of fully pruned tiles: Zero, one warp per row over the grid
      const int zr0 = sc.mc * C::TM;
      const int gw = (int)blockIdx.x * EPI_WARPS + ew, nw = (int)gridDim.x * EPI_WARPS;
      for (int zm = zr0 + gw; zm < p.M; zm += nw) {
        const int zr = p.out_dense ? zm : __ldg(p.pruned + (zm - p.n_kept));
        __nv_bfloat16* o = p.out + (int64_t)zr * p.ld_out;
        for (int col = lane * 8; col < p.N; col += 256) store_bf16x8(o + col, make_uint4(0u, 0u, 0u, 0u), p.N - col);
      }
    }
  }

  kernel_teardown<CG>(tmem_base, warp);
  if (p.pdl_late) pdl_wait();
  if (cst && threadIdx.x == 0) cst[7] = globaltimer();
  if (p.stamp != nullptr && threadIdx.x == 0) atomicMax(p.stamp + 1, (unsigned long long)globaltimer());
  if (p.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p.prof_stamp + 1, (unsigned long long)globaltimer());
}

// Two GEMM problems in ONE persistent launch (a linear's dX and dW, P:146:
// both need only G and the FWD operands): their work units share every CTA
// pair under a static longest-processing-time schedule built on the host,
// so neither GEMM's fill, tail or wave quantisation is exposed on its own
// and no SM split between two concurrent kernels is needed.
constexpr int GROUP_LIST_MAX = 256;   // work units of one pair in a grouped launch (smem-staged list)

struct GroupArgs {
  CUtensorMap a[2], b[2], o[2], o2[2], w[2];
  GemmParams p[2];
  const int32_t* sched;   // units of pair q: sched[off[q] .. off[q+1]), entry = problem << 24 | unit
  const int32_t* off;
};

template <int K0, int K1, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1) ztp_gemm_group_kernel(const __grid_constant__ GroupArgs g) {
  using C = Cfg<CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* staging = smem + C::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const int rank = CG == 2 ? (int)(crank & 1u) : 0;
  const bool leader = rank == 0;
  const uint16_t pmask = (uint16_t)(0x3u << (crank & ~1u));
  const int pair = blockIdx.x / CG;
  // this pair's unit list into shared memory (host-written before the
  // launch, so read before the PDL wait; made visible by the prologue's sync)
  int32_t* slist = reinterpret_cast<int32_t*>(smem + C::TOTAL - 1024);
  const int i0 = __ldg(g.off + pair), nu = __ldg(g.off + pair + 1) - i0;
  for (int i = threadIdx.x; i < nu; i += blockDim.x) slist[i] = __ldg(g.sched + i0 + i);
  if (warp == 0 && lane < 4) tma_prefetch_desc(lane < 2 ? &g.a[lane & 1] : &g.b[lane & 1]);
  const uint32_t tmem_base = kernel_prologue<CG>(full, empty, tfull, tempty, tmem_slot, warp);
  pdl_wait();
  pdl_trigger();
  const GemmParams& p0 = g.p[0];
  if (p0.stamp != nullptr && threadIdx.x == 0) atomicMin(p0.stamp, (unsigned long long)globaltimer());
  if (p0.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p0.prof_stamp, ~(unsigned long long)globaltimer());
  const Sched<K0, C::TM> s0(g.p[0]);
  const Sched<K1, C::TM> s1(g.p[1]);
  Pipe ps;
  if (warp == 0) {
    for (int i = 0; i < nu; ++i) {
      const int e = slist[i], u = e & 0xFFFFFF;
      if ((e >> 24) == 0) {
        const Work wk = s0.get(u);
        if (!wk.zero) produce_unit<K0, CG, false, false>(&g.a[0], &g.b[0], g.p[0], wk, rank, leader, lane, ring, full, empty, ps);
      } else {
        const Work wk = s1.get(u);
        if (!wk.zero) produce_unit<K1, CG, false, false>(&g.a[1], &g.b[1], g.p[1], wk, rank, leader, lane, ring, full, empty, ps);
      }
    }
  } else if (warp == 1 && leader) {
    for (int i = 0; i < nu; ++i) {
      const int e = slist[i], u = e & 0xFFFFFF;
      if ((e >> 24) == 0) {
        const Work wk = s0.get(u);
        if (!wk.zero) mma_unit<K0, CG>(wk, lane, pmask, ring, full, empty, tfull, tempty, tmem_base, ps);
      } else {
        const Work wk = s1.get(u);
        if (!wk.zero) mma_unit<K1, CG>(wk, lane, pmask, ring, full, empty, tfull, tempty, tmem_base, ps);
      }
    }
  } else if (warp >= 4) {
    for (int i = 0; i < nu; ++i) {
      const int e = slist[i], u = e & 0xFFFFFF;
      if ((e >> 24) == 0)
        epilogue_unit<K0, CG>(&g.o[0], &g.o2[0], &g.w[0], g.p[0], s0.S, s0.get(u), rank, warp - 4, lane, staging,
                              tfull, tempty, tmem_base, ps);
      else
        epilogue_unit<K1, CG>(&g.o[1], &g.o2[1], &g.w[1], g.p[1], s1.S, s1.get(u), rank, warp - 4, lane, staging,
                              tfull, tempty, tmem_base, ps);
    }
    if (lane < 8) bulk_wait0();
  }
  kernel_teardown<CG>(tmem_base, warp);
  if (p0.stamp != nullptr && threadIdx.x == 0) atomicMax(p0.stamp + 1, (unsigned long long)globaltimer());
  if (p0.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p0.prof_stamp + 1, (unsigned long long)globaltimer());
}

// Split-K reduction (fixed split order -> deterministic) fused with the
// epilogue the unsplit kernel applies: GeLU / GeLU', bf16 RNE, lineage row map
// and the Zero imputation of pruned rows.
template <int KIND>
__device__ __forceinline__ void splitk_reduce_body(const GemmParams& p) {
  // col_pos (DW with output pruning): output column j <- compact column
  // col_pos[j] of the partials, Zero where col_pos[j] < 0
  const int width = p.col_pos ? p.n_full : p.N;
  const int cpr = (width + 7) / 8;
  const int64_t total = (int64_t)p.M * cpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / cpr);
    const int col = (int)(i % cpr) * 8;
    const int nv = width - col;
    const bool computed = (KIND == KIND_FWD) || (m < p.n_kept);
    int orow;
    if (p.out_dense)
      orow = m;
    else if (KIND == KIND_FWD)
      orow = p.out_pos ? __ldg(p.out_pos + m) : m;
    else
      orow = computed ? __ldg(p.kept + m) : __ldg(p.pruned + (m - p.n_kept));
    if (orow < 0) continue;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (computed && p.col_pos) {
      int cc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) cc[q] = q < nv ? __ldg(p.col_pos + col + q) : -1;
      const float* src = p.ws + (int64_t)m * p.ld_ws;
      for (int s = 0; s < p.splits; ++s, src += p.ws_split_stride) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (cc[q] >= 0) v[q] += __ldg(src + cc[q]);   // L1: the 8 gathers of a group share sectors
      }
    } else if (computed) {
      const float* src = p.ws + (int64_t)m * p.ld_ws + col;
      for (int s = 0; s < p.splits; ++s) {
        const float4 a = *reinterpret_cast<const float4*>(src);
        const float4 b = *reinterpret_cast<const float4*>(src + 4);
        v[0] += a.x;
        v[1] += a.y;
        v[2] += a.z;
        v[3] += a.w;
        v[4] += b.x;
        v[5] += b.y;
        v[6] += b.z;
        v[7] += b.w;
        src += p.ws_split_stride;
      }
    }
    uint4 w;
    w.x = pack_bf16(v[0], v[1]);
    w.y = pack_bf16(v[2], v[3]);
    w.z = pack_bf16(v[4], v[5]);
    w.w = pack_bf16(v[6], v[7]);
    const int ar = p.aux_by_m ? m : orow;
    if ((p.epi == EPI_GELU_GRAD || p.epi == EPI_MUL) && computed) {
      const uint4 a = *reinterpret_cast<const uint4*>(p.aux + (int64_t)ar * p.ld_aux + col);
      const uint32_t a4[4] = {a.x, a.y, a.z, a.w};
      uint32_t o4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 x = make_float2(v[2 * j], v[2 * j + 1]);
        float2 g = unpack2(a4[j]), hv, dv;
        if (p.epi == EPI_GELU_GRAD) {
          gelu2(g, hv, dv, true);
          g = dv;
        }
        o4[j] = pack2(__fmul2_rn(x, g));
      }
      w = make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
    uint4 g = w;
    if (p.epi == EPI_GELU || p.epi == EPI_GELU_D) {
      uint32_t h4[4], d4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 hv, dv;
        gelu2(make_float2(v[2 * j], v[2 * j + 1]), hv, dv, p.epi == EPI_GELU_D);
        h4[j] = pack2(hv);
        d4[j] = pack2(dv);
      }
      g = make_uint4(h4[0], h4[1], h4[2], h4[3]);
      if (p.epi == EPI_GELU_D) w = make_uint4(d4[0], d4[1], d4[2], d4[3]);
    }
    store_bf16x8(p.out + (int64_t)orow * p.ld_out + col, w, nv);
    if (p.epi == EPI_GELU || p.epi == EPI_GELU_D) store_bf16x8(p.out2 + (int64_t)orow * p.ld_out2 + col, g, nv);
  }
}

template <int KIND>
__global__ void __launch_bounds__(256) ztp_splitk_reduce(const GemmParams p) {
  pdl_wait();
  pdl_trigger();
  splitk_reduce_body<KIND>(p);
  if (p.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p.prof_stamp + 1, (unsigned long long)globaltimer());
}

// Lean split-K reduce for dW (no epilogue math): S splits known at compile
// time, so every partial of an 8-column group is loaded before the fixed-order
// sum s = 0..S-1 (memory-level parallelism without predicated spare loads);
// COLPOS spreads compact columns to their units (output pruning).
template <int S, bool COLPOS>
__global__ void __launch_bounds__(256) ztp_dw_reduce(const GemmParams p) {
  pdl_wait();
  pdl_trigger();
  const int width = COLPOS ? p.n_full : p.N;
  const int cpr = (width + 7) / 8;
  const int64_t total = (int64_t)p.M * cpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / cpr);
    const int col = (int)(i % cpr) * 8;
    const int nv = width - col;
    const bool computed = m < p.n_kept;
    const int orow = p.out_dense ? m : (computed ? __ldg(p.kept + m) : __ldg(p.pruned + (m - p.n_kept)));
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (computed) {
      const float* src = p.ws + (int64_t)m * p.ld_ws;
      if constexpr (COLPOS) {
        int cc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cc[q] = q < nv ? __ldg(p.col_pos + col + q) : -1;
        // eight consecutive kept columns, e.g. the Q / K blocks of dWqkv under
        // V pruning: two float4 loads per split instead of eight gathers
        bool run = cc[0] >= 0 && (cc[0] & 3) == 0;
#pragma unroll
        for (int q = 1; q < 8; ++q) run = run && cc[q] == cc[0] + q;
        if (run) {
          float4 a[S], b[S];
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const float* q = src + s * p.ws_split_stride + cc[0];
            a[s] = __ldcg(reinterpret_cast<const float4*>(q));
            b[s] = __ldcg(reinterpret_cast<const float4*>(q + 4));
          }
#pragma unroll
          for (int s = 0; s < S; ++s) {
            v[0] += a[s].x;
            v[1] += a[s].y;
            v[2] += a[s].z;
            v[3] += a[s].w;
            v[4] += b[s].x;
            v[5] += b[s].y;
            v[6] += b[s].z;
            v[7] += b[s].w;
          }
        } else {
          float t[S][8];
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int q = 0; q < 8; ++q) t[s][q] = cc[q] >= 0 ? __ldg(src + s * p.ws_split_stride + cc[q]) : 0.f;
#pragma unroll
          for (int s = 0; s < S; ++s)
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] += t[s][q];
        }
      } else {
        float4 a[S], b[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const float* q = src + s * p.ws_split_stride + col;
          a[s] = __ldcg(reinterpret_cast<const float4*>(q));
          b[s] = __ldcg(reinterpret_cast<const float4*>(q + 4));
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          v[0] += a[s].x;
          v[1] += a[s].y;
          v[2] += a[s].z;
          v[3] += a[s].w;
          v[4] += b[s].x;
          v[5] += b[s].y;
          v[6] += b[s].z;
          v[7] += b[s].w;
        }
      }
    }
    uint4 w;
    w.x = pack_bf16(v[0], v[1]);
    w.y = pack_bf16(v[2], v[3]);
    w.z = pack_bf16(v[4], v[5]);
    w.w = pack_bf16(v[6], v[7]);
    store_bf16x8(p.out + (int64_t)orow * p.ld_out + col, w, nv);
  }
  if (p.prof_stamp != nullptr && threadIdx.x == 0) atomicMax(p.prof_stamp + 1, (unsigned long long)globaltimer());
}

template <int S>
static cudaError_t dw_reduce_launch(const GemmParams& p, int blocks, cudaStream_t st) {
  if (p.col_pos) return launch_k(ztp_dw_reduce<S, true>, blocks, 256, 0, st, p);
  return launch_k(ztp_dw_reduce<S, false>, blocks, 256, 0, st, p);
}

// ----------------------------------------------------------------- host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// Row-major [rows, cols] with leading dimension ld (elements); box = box_cols x box_rows.
static bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
                     uint32_t box_rows, bool f32 = false) {
  auto enc = get_encode();
  if (!enc) return false;
  const int64_t es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// fp32 split-K workspace [splits][rows][ld]: box 32 x 32 x 1 (128-byte rows).
static bool make_ws_map(CUtensorMap* m, const float* ptr, int64_t splits, int64_t rows, int64_t cols, int64_t ld) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(rows * ld * 4)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct Maps {
  CUtensorMap a, b, o, o2, w;
};

static int units_of(int kind, int cg, const GemmParams& p) {
  const int tm = BM * cg;
  const int m_tiles = (p.M + tm - 1) / tm, n_tiles = (p.N + BN - 1) / BN;
  int mc = m_tiles;
  if (kind != KIND_FWD) mc = std::min(m_tiles, (p.n_kept + tm - 1) / tm);
  return mc * n_tiles * p.splits + (p.splits == 1 && !p.skip_zero ? (m_tiles - mc) * n_tiles : 0) +
         (kind == KIND_FWD && p.splits == 1 ? p.tail_r : 0);
}

// FWD tail (2-CTA, unsplit, dense boxes): when the last round of tiles fills
// at most half of the CTA pairs, its tiles run as two 128-column halves on
// twice as many pairs -- the launch ends half a tile earlier (c2: QKV 320
// tiles = 4 x 74 + 24, FC1 256 = 3 x 74 + 34).  Returns the tile count.
static int tail_halves(int kind, int cg, const GemmParams& p, int num_sms, bool gathered) {
  if (kind != KIND_FWD || cg != 2 || p.splits != 1 || !p.tail_ok || gathered || p.fo_flags || p.fi_flags) return 0;
  const int m_tiles = (p.M + BM * cg - 1) / (BM * cg), n_tiles = (p.N + BN - 1) / BN;
  const int T = m_tiles * n_tiles, P = num_sms / cg;
  const int R = T >= P ? T % P : T;
  return (R > 0 && 2 * R <= P) ? R : 0;
}

// After a GEMM launch: the split-K reduce (fixed split order, the epilogue
// of the unsplit kernel; it also spreads output-pruned dW columns), or the
// column spread of an unsplit output-pruned dW.
template <int KIND>
static cudaError_t post_launch(const GemmParams& p, int num_sms, cudaStream_t st) {
  if (p.splits == 1 || p.cs > 1) {
    if (p.col_pos && !p.spread)   // compact columns written by the epilogue (scratch): spread them, Zero the rest
      return expand_cols_launch(p.out, p.ld_out, p.full_out, p.ld_full, p.kept, std::min(p.n_kept, p.M), p.pruned,
                                std::max(0, p.M - p.n_kept), p.col_pos, p.n_full, st);
    return cudaSuccess;
  }
  const int64_t chunks = (int64_t)p.M * (((p.col_pos ? p.n_full : p.N) + 7) / 8);
  const int blocks = (int)std::min<int64_t>((chunks + 255) / 256, (int64_t)num_sms * 8);
  if (KIND == KIND_DW && p.epi == EPI_NONE) {
    switch (p.splits) {
      case 2: return dw_reduce_launch<2>(p, blocks, st);
      case 3: return dw_reduce_launch<3>(p, blocks, st);
      case 4: return dw_reduce_launch<4>(p, blocks, st);
      default: break;   // more splits: the generic loop (measured faster at S = 8)
    }
  }
  return launch_k(ztp_splitk_reduce<KIND>, blocks, 256, 0, st, p);
}

template <int KIND, int CG, bool AG, bool BG>
static cudaError_t launch_kind(const Maps& mp, const GemmParams& p, int num_sms, cudaStream_t st) {
  const int smem = Cfg<CG>::TOTAL;
  auto kern = ztp_gemm_kernel<KIND, CG, AG, BG>;
  {
    cudaError_t e = ensure_smem_optin((const void*)kern, smem);
    if (e != cudaSuccess) return e;
  }
  GemmParams pl = p;
  pl.tail_r = tail_halves(KIND, CG, p, num_sms, AG || BG);
  const int units = units_of(KIND, CG, pl);
  const int pairs = pl.cs > 1 ? units : std::min(units, num_sms / CG);   // cluster split-K: one unit per pair
  if (pl.fo_flags) {
    const int n_tiles = (p.N + BN - 1) / BN;
    if (p.splits != 1 || p.cs > 1 || p.col_pos || n_tiles > FLAG_NB || units % n_tiles) {
      pl.fo_flags = nullptr;   // not a flag producer
      pl.fo_target = nullptr;
    } else {
      pl.fo_nb = n_tiles;
      pl.fo_T = (unsigned long long)(units / n_tiles) * EPI_WARPS * CG;
    }
  }
  if (pairs > 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pairs * CG);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG * (p.cs > 1 ? p.cs : 1);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    note_launch(st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mp.a, mp.b, mp.o, mp.o2, mp.w, pl);
    if (e != cudaSuccess) return e;
  }
  return post_launch<KIND>(p, num_sms, st);
}

int gemm_choose_cg(int kind, int M, int n_kept) {
  const int rows = kind == KIND_FWD ? M : std::min(M, n_kept);
  return rows > BM ? 2 : 1;
}

int gemm_choose_splits(int kind, int M, int N, int kdim, int n_kept, int num_sms) {
  const int cg = gemm_choose_cg(kind, M, n_kept);
  const int tm = BM * cg;
  const int m_tiles = (M + tm - 1) / tm, n_tiles = (N + BN - 1) / BN;
  int mc = m_tiles;
  if (kind != KIND_FWD) mc = std::min(m_tiles, (n_kept + tm - 1) / tm);
  const int tiles_c = std::max(1, mc * n_tiles);
  const int num_kb = (kdim + BK - 1) / BK;
  const int s = std::min((num_sms / cg) / tiles_c, num_kb / 16);  // each split keeps >= 1024 contraction elements
  return std::max(1, s);
}

// Cluster split-K (dW, no epilogue math): the `cs` K-slices of a tile run as
// one cluster of CG x cs CTAs (<= 8, portable) and reduce through DSMEM.  It
// needs every tile's cluster co-resident (one wave): checked against the
// occupancy API for this kernel's shared memory.  Opt-in: ZTP_CSPLIT=1.
int gemm_cluster_splits(int kind, int epi, int M, int N, int n_kept, int splits, int num_sms) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("ZTP_CSPLIT");
    enabled = e ? atoi(e) != 0 : 0;   // measured slower in the step graph: opt-in
  }
  if (!enabled || kind != KIND_DW || epi != EPI_NONE || splits < 2) return 0;
  const int cg = gemm_choose_cg(kind, M, n_kept);
  const int tm = BM * cg;
  const int m_tiles = (M + tm - 1) / tm, n_tiles = (N + BN - 1) / BN;
  const int tiles_c = std::min(m_tiles, (n_kept + tm - 1) / tm) * n_tiles;
  static int max_cl[3][9] = {};
  for (int cs = std::min(splits, 8 / cg); cs >= 2; --cs) {
    if (tiles_c * cs * cg > num_sms) continue;
    if (cs * ((8 + cs - 1) / cs) * BM * 128 > (cg == 2 ? Cfg<2>::RING : Cfg<1>::RING)) continue;   // DSMEM slots
    int& mc = max_cl[cg][cs];
    if (mc == 0) {
      const int smem = cg == 2 ? Cfg<2>::TOTAL : Cfg<1>::TOTAL;
      const void* kern = cg == 2 ? (const void*)ztp_gemm_kernel<KIND_DW, 2, false, false>
                                 : (const void*)ztp_gemm_kernel<KIND_DW, 1, false, false>;
      if (ensure_smem_optin(kern, smem) != cudaSuccess) return 0;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cg * cs * 64);
      cfg.blockDim = dim3(NUM_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cg * cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        n = -1;
      }
      mc = n > 0 ? n : -1;
    }
    if (mc > 0 && tiles_c <= mc) return cs;
  }
  return 0;
}

size_t gemm_ws_bytes(int kind, int M, int N, int n_kept, int splits) {
  if (splits <= 1) return 0;
  const int64_t rows = kind == KIND_FWD ? M : std::min(M, n_kept);
  const int64_t ld = (N + 7) / 8 * 8;
  return (size_t)splits * rows * ld * sizeof(float);
}

template <int KIND, int CG>
static cudaError_t dispatch(bool ag, bool bg, const Maps& mp, const GemmParams& p, int num_sms, cudaStream_t st) {
  if (KIND != KIND_FWD && bg) return cudaErrorInvalidValue;
  if (ag && bg) return launch_kind<KIND, CG, true, true>(mp, p, num_sms, st);
  if (ag) return launch_kind<KIND, CG, true, false>(mp, p, num_sms, st);
  if (bg) return launch_kind<KIND, CG, false, true>(mp, p, num_sms, st);
  return launch_kind<KIND, CG, false, false>(mp, p, num_sms, st);
}

// Operand, output and workspace tensor maps per kind (see the file header).
static bool build_maps(int kind, const GemmOperands& o, GemmParams& p, int cg, Maps& mp) {
  bool ok = true;
  const bool ag = o.a_gather, bg = o.b_gather;
  const uint32_t bnl = BN / cg;
  p.oob_row = (int)(o.a_rows > o.b_rows ? o.a_rows : o.b_rows);  // outside every gathered tensor
  p.oob_out = p.out_rows;                                        // TMA stores skip this row
  if (kind == KIND_FWD) {
    // A = W^T [K|K', n] MN-major; B = X^T [K|K', N] MN-major (same rows)
    ok &= make_map(&mp.a, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : 64);
    ok &= make_map(&mp.b, o.b, o.b_rows, o.b_cols, o.b_ld, 64, bg ? 1 : 64);
  } else if (kind == KIND_DX) {
    // A = W^T [K|K', n_out] K-major; B = G^T [n_out, N] MN-major 64 x 64 boxes
    ok &= make_map(&mp.a, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : BM);
    ok &= make_map(&mp.b, o.b, o.b_rows, o.b_cols, o.b_ld, 64, 64);
  } else {
    // A = X^T [K|K', N] K-major; B = G^T [n_out, N] K-major box 64 x BN/cg
    ok &= make_map(&mp.a, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : BM);
    ok &= make_map(&mp.b, o.b, o.b_rows, o.b_cols, o.b_ld, 64, bnl);
  }
  // outputs: dense box stores (32 rows x 64 columns) or 4-row scatters at the row map
  const bool dense_out = p.out_dense;
  ok &= make_map(&mp.o, p.out, p.out_rows, p.N, p.ld_out, 64, dense_out ? 32 : 1);
  if (p.epi == EPI_GELU || p.epi == EPI_GELU_D)
    ok &= make_map(&mp.o2, p.out2, p.out_rows, p.N, p.ld_out2, 64, dense_out ? 32 : 1);
  else
    mp.o2 = mp.o;
  if (p.splits > 1 && p.cs <= 1) {
    const int64_t rows = kind == KIND_FWD ? p.M : std::min(p.M, p.n_kept);
    ok &= make_ws_map(&mp.w, p.ws, p.splits, rows, p.N, p.ld_ws);
  } else {
    mp.w = mp.o;
  }
  return ok;
}

cudaError_t gemm_launch(int kind, const GemmOperands& o, GemmParams p, int num_sms, cudaStream_t st) {
  Maps mp;
  const bool ag = o.a_gather, bg = o.b_gather;
  const int cg = gemm_choose_cg(kind, p.M, p.n_kept);
  if (!build_maps(kind, o, p, cg, mp)) return cudaErrorInvalidValue;
  if (kind == KIND_FWD)
    return cg == 2 ? dispatch<KIND_FWD, 2>(ag, bg, mp, p, num_sms, st) : dispatch<KIND_FWD, 1>(ag, bg, mp, p, num_sms, st);
  if (kind == KIND_DX)
    return cg == 2 ? dispatch<KIND_DX, 2>(ag, bg, mp, p, num_sms, st) : dispatch<KIND_DX, 1>(ag, bg, mp, p, num_sms, st);
  return cg == 2 ? dispatch<KIND_DW, 2>(ag, bg, mp, p, num_sms, st) : dispatch<KIND_DW, 1>(ag, bg, mp, p, num_sms, st);
}

// ------------------------------------------------------- grouped dX + dW launch

// Host mirror of Sched: the work units of one problem and their cost in
// 64-deep k-blocks (+ an epilogue allowance: bf16 tile 2, fp32 split-K
// partial 3; an all-pruned Zero tile costs 1).
static void unit_costs(int kind, int cg, const GemmParams& p, std::vector<int>& cost, std::vector<char>& zero) {
  const int tm = BM * cg;
  const int m_tiles = (p.M + tm - 1) / tm, n_tiles = (p.N + BN - 1) / BN;
  const int num_kb = (p.kdim + BK - 1) / BK;
  int mc = m_tiles;
  if (kind != KIND_FWD) mc = std::min(m_tiles, (p.n_kept + tm - 1) / tm);
  const int tiles_c = mc * n_tiles, S = p.splits, kbs = p.kb_per_split;
  const int nz = S == 1 && !p.skip_zero ? (m_tiles - mc) * n_tiles : 0;
  cost.clear();
  zero.clear();
  for (int u = 0; u < nz; ++u) {
    cost.push_back(1);
    zero.push_back(1);
  }
  for (int u = 0; u < tiles_c * S; ++u) {
    const int s = u / tiles_c;
    const int kb0 = s * kbs, kb1 = std::min(num_kb, kb0 + kbs);
    cost.push_back(std::max(0, kb1 - kb0) + (S > 1 ? 3 : 2));
    zero.push_back(0);
  }
}

// Static schedule of a grouped launch: Zero tiles (epilogue only, ~3 k-blocks
// of time each) first, one per pair in turn -- LPT would pile the cheap ones
// onto the idle pairs -- then the computed units, longest first, each onto
// the least-loaded pair.  Returns the makespan in k-blocks.
struct GUnit {
  int cost, prob, idx;
  bool zero;
};
static int64_t lpt_schedule(std::vector<GUnit> us, int pairs, std::vector<std::vector<int32_t>>* lists) {
  std::stable_sort(us.begin(), us.end(), [](const GUnit& a, const GUnit& b) { return a.cost > b.cost; });
  std::vector<int64_t> load(pairs, 0);
  std::vector<std::vector<int32_t>> zl(pairs), rl(pairs);
  int zq = 0;
  for (const GUnit& u : us)
    if (u.zero) {
      zl[zq].push_back((u.prob << 24) | u.idx);
      load[zq] += 3;
      zq = (zq + 1) % pairs;
    }
  for (const GUnit& u : us) {
    if (u.zero) continue;
    int q = 0;
    for (int j = 1; j < pairs; ++j)
      if (load[j] < load[q]) q = j;
    load[q] += u.cost;
    rl[q].push_back((u.prob << 24) | u.idx);
  }
  if (lists) {
    lists->assign(pairs, {});
    for (int q = 0; q < pairs; ++q) {
      (*lists)[q] = zl[q];
      (*lists)[q].insert((*lists)[q].end(), rl[q].begin(), rl[q].end());
    }
  }
  return *std::max_element(load.begin(), load.end());
}

static std::vector<GUnit> group_units(int k0, const GemmParams& p0, int k1, const GemmParams& p1, int cg) {
  std::vector<int> c0, c1;
  std::vector<char> z0, z1;
  unit_costs(k0, cg, p0, c0, z0);
  unit_costs(k1, cg, p1, c1, z1);
  std::vector<GUnit> us;
  for (int i = 0; i < (int)c0.size(); ++i) us.push_back({c0[i], 0, i, z0[i] != 0});
  for (int i = 0; i < (int)c1.size(); ++i) us.push_back({c1[i], 1, i, z1[i] != 0});
  return us;
}

int gemm_group_splits(int M_dx, int N_dx, int kdim_dx, int n_kept_dx, int M_dw, int N_dw, int kdim_dw,
                      int n_kept_dw, int num_sms) {
  // the dW split count whose LPT schedule has the smallest makespan (fp32
  // partials and the reduce grow with the splits: ties go to fewer)
  const int cg = gemm_choose_cg(KIND_DX, M_dx, n_kept_dx);
  GemmParams px{}, pw{};
  px.M = M_dx; px.N = N_dx; px.kdim = kdim_dx; px.n_kept = n_kept_dx; px.splits = 1;
  px.kb_per_split = (kdim_dx + BK - 1) / BK;
  pw.M = M_dw; pw.N = N_dw; pw.kdim = kdim_dw; pw.n_kept = n_kept_dw;
  const int kb_dw = (kdim_dw + BK - 1) / BK;
  int best = 1;
  int64_t best_t = -1;
  for (int s = 1; s <= std::min(16, std::max(1, kb_dw / 8)); ++s) {
    pw.kb_per_split = (kb_dw + s - 1) / s;
    pw.splits = (kb_dw + pw.kb_per_split - 1) / pw.kb_per_split;
    if (pw.splits != s) continue;
    const auto us = group_units(KIND_DX, px, KIND_DW, pw, cg);
    const int pairs = std::max(1, std::min((int)us.size(), num_sms / cg));
    // each extra split adds the reduce's re-read of one fp32 partial (~1 k-block per pair)
    const int64_t t = lpt_schedule(us, pairs, nullptr) + (s > 1 ? s : 0);
    if (best_t < 0 || t < best_t) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

bool gemm_group_pays(int M_dx, int N_dx, int kdim_dx, int n_kept_dx, int M_dw, int N_dw, int kdim_dw, int n_kept_dw,
                     int num_sms) {
  // measured (profiles/r02_grouped_dx_dw_ab.txt): the grouped launch wins
  // only for small pairs (the O projection at c2: ~28 k-blocks per CTA pair),
  // where two concurrent kernels each run about one partial wave
  const int cg = gemm_choose_cg(KIND_DX, M_dx, n_kept_dx);
  const int tm = BM * cg;
  auto tiles = [&](int M, int N, int nk) { return ((std::min(M, nk) + tm - 1) / tm) * ((N + BN - 1) / BN); };
  const double total = (double)tiles(M_dx, N_dx, n_kept_dx) * ((kdim_dx + BK - 1) / BK) +
                       (double)tiles(M_dw, N_dw, n_kept_dw) * ((kdim_dw + BK - 1) / BK);
  return total / std::max(1, num_sms / cg) <= 32.0;
}

namespace {
struct SchedEntry {
  std::vector<int64_t> key;
  int32_t* d = nullptr;   // sched entries then offsets (device; kept for the process: captured graphs use it)
  int n = 0, pairs = 0;
};
std::vector<SchedEntry>& sched_cache() {
  static std::vector<SchedEntry> v;
  return v;
}
}  // namespace

cudaError_t gemm_group_launch(int k0, const GemmOperands& o0, GemmParams p0, int k1, const GemmOperands& o1,
                              GemmParams p1, int num_sms, cudaStream_t st) {
  if (k0 != KIND_DX || k1 != KIND_DW || o0.a_gather || o0.b_gather || o1.a_gather || o1.b_gather || p0.cs > 1 ||
      p1.cs > 1)
    return cudaErrorInvalidValue;
  const int cg = gemm_choose_cg(k0, p0.M, p0.n_kept);
  if (cg != gemm_choose_cg(k1, p1.M, p1.n_kept)) return cudaErrorInvalidValue;
  GroupArgs ga;
  Maps m0, m1;
  if (!build_maps(k0, o0, p0, cg, m0) || !build_maps(k1, o1, p1, cg, m1)) return cudaErrorInvalidValue;
  ga.a[0] = m0.a; ga.b[0] = m0.b; ga.o[0] = m0.o; ga.o2[0] = m0.o2; ga.w[0] = m0.w;
  ga.a[1] = m1.a; ga.b[1] = m1.b; ga.o[1] = m1.o; ga.o2[1] = m1.o2; ga.w[1] = m1.w;
  ga.p[0] = p0;
  ga.p[1] = p1;
  const int total = (int)group_units(k0, p0, k1, p1, cg).size();
  const int pairs = std::max(1, std::min(total, num_sms / cg));
  std::vector<int64_t> key = {k0, k1, cg, pairs, p0.M, p0.N, p0.kdim, p0.n_kept, p0.splits, p0.kb_per_split,
                              p1.M, p1.N, p1.kdim, p1.n_kept, p1.splits, p1.kb_per_split};
  SchedEntry* hit = nullptr;
  for (auto& e : sched_cache())
    if (e.key == key) hit = &e;
  if (!hit) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return cudaErrorStreamCaptureUnsupported;   // schedules are built by an eager (warm-up) call
    std::vector<std::vector<int32_t>> lists;
    lpt_schedule(group_units(k0, p0, k1, p1, cg), pairs, &lists);
    std::vector<int32_t> h;
    std::vector<int32_t> off(pairs + 1, 0);
    for (int q = 0; q < pairs; ++q) {
      off[q] = (int32_t)h.size();
      h.insert(h.end(), lists[q].begin(), lists[q].end());
    }
    off[pairs] = (int32_t)h.size();
    for (int q = 0; q < pairs; ++q)
      if (off[q + 1] - off[q] > GROUP_LIST_MAX) return cudaErrorInvalidConfiguration;   // caller: concurrent pair
    SchedEntry e;
    e.key = key;
    e.n = (int)h.size();
    e.pairs = pairs;
    cudaError_t err = cudaMalloc(&e.d, (h.size() + off.size()) * sizeof(int32_t));
    if (err != cudaSuccess) return err;
    err = cudaMemcpy(e.d, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
      err = cudaMemcpy(e.d + h.size(), off.data(), off.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) return err;
    sched_cache().push_back(e);
    hit = &sched_cache().back();
  }
  ga.sched = hit->d;
  ga.off = hit->d + hit->n;
  const int smem = (cg == 2 ? Cfg<2>::TOTAL : Cfg<1>::TOTAL) + GROUP_LIST_MAX * 4;
  auto kern = cg == 2 ? ztp_gemm_group_kernel<KIND_DX, KIND_DW, 2> : ztp_gemm_group_kernel<KIND_DX, KIND_DW, 1>;
  {
    cudaError_t e = ensure_smem_optin((const void*)kern, smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pairs * cg);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  note_launch(cfg.stream);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ga);
  if (e != cudaSuccess) return e;
  e = post_launch<KIND_DX>(p0, num_sms, st);
  if (e != cudaSuccess) return e;
  return post_launch<KIND_DW>(p1, num_sms, st);
}

}  // namespace ztp

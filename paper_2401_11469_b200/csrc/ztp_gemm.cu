// Resized GEMMs of one TP linear on sm_100a:
//   FWD  Y^T[j,t]  = sum_{k in S} W^T[k,j] X^T[k,t]
//   DX   dX^T[k,t] = sum_{j<n}   W^T[k,j] G^T[j,t], k in S
//   DW   dW^T[k,j] = sum_t       X^T[k,t] G^T[j,t], k in S
// with rows P of dX^T / dW^T imputed by Zero in the same kernel.
//
// Design: persistent, warp-specialised, 1-CTA
// tcgen05 kind::f16 128x256x16 MMAs accumulating in TMEM (2 x 256 columns,
// double-buffered so the epilogue of tile i overlaps the mainloop of i+1).
//   warp 0      TMA producer.  The pruned contraction rows are gathered
//               straight from HBM into the 128B-swizzled smem ring with
//               cp.async.bulk.tensor...tile::gather4 (4 rows per instruction,
//               32 lanes issuing in parallel) -- no compacted copy of X or W
//               is ever materialised (a4: "dimension extracting").
//   warp 1      MMA issuer (one thread), tcgen05.commit -> smem-slot release.
//   warp 2      TMEM allocator.
//   warps 4-7   epilogue: tcgen05.ld -> (GeLU | GeLU' | none) -> bf16 ->
//               swizzled smem staging -> 128-bit coalesced row stores at the
//               lineage row map (a6: scatter + Zero imputation).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "ztp_internal.h"
#include "ztp_ptx.cuh"

namespace ztp {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int NUM_THREADS = 256;
constexpr int A_BYTES = BM * BK * 2;              // 16 KB
constexpr int STAGING_PER_WARP = 32 * 128 * 2;    // two 32x64 bf16 planes (pre and H)

template <int BN>
struct Smem {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RING = STAGES * STAGE_BYTES;
  static constexpr int STAGING = 4 * STAGING_PER_WARP;
  static constexpr int BARS = (2 * STAGES + 4) * 8 + 16;
  static constexpr int TOTAL = 1024 + RING + STAGING + BARS;
};

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// GeLU tanh approximation and its derivative, fp32.
__device__ __forceinline__ float gelu_f(float x) {
  const float c = 0.7978845608028654f;
  float u = c * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c = 0.7978845608028654f;
  float u = c * (x + 0.044715f * x * x * x);
  float t = tanhf(u);
  float du = c * (1.0f + 3.0f * 0.044715f * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

template <int KIND>
__device__ __forceinline__ int gather_row_mk(const GemmParams& p, int m) {
  // K-major gathered operand (DX: W^T rows, DW: X^T rows): row m of the tile
  // is lineage row kept[m]; pruned rows read as zeros (OOB row -> TMA zero fill).
  return (m < p.n_kept) ? __ldg(p.kept + m) : p.oob_row;
}

// AG / BG: operand A / B gathered row-by-row with TMA gather4 through the
// lineage list (true) or loaded as dense TMA boxes from a compact, already
// row-selected tensor (false; rows past the compact extent are zero-filled).
template <int KIND, int BN, bool AG, bool BG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    ztp_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  using SM = Smem<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* staging = smem + SM::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + SM::STAGING);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (p.stamp != nullptr && threadIdx.x == 0) atomicMin(p.stamp, (unsigned long long)globaltimer());

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int m_tiles = (p.M + BM - 1) / BM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (p.kdim + BK - 1) / BK;
  // DX / DW: tiles whose rows are all pruned skip the MMA and write Zero.
  auto zero_tile = [&](int m0) { return (KIND != KIND_FWD) && (m0 >= p.n_kept); };

  if (warp == 0) {
    // ============================ TMA producer ============================
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile % m_tiles) * BM;
      const int n0 = (tile / m_tiles) * BN;
      if (zero_tile(m0)) continue;
      int ar0 = 0, ar1 = 0, ar2 = 0, ar3 = 0;
      if (KIND != KIND_FWD && AG) {
        const int mb = m0 + 4 * lane;
        ar0 = gather_row_mk<KIND>(p, mb + 0);
        ar1 = gather_row_mk<KIND>(p, mb + 1);
        ar2 = gather_row_mk<KIND>(p, mb + 2);
        ar3 = gather_row_mk<KIND>(p, mb + 3);
      }
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = ring + stage * SM::STAGE_BYTES;
        uint8_t* sb = sa + A_BYTES;
        if (lane == 0) mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
        __syncwarp();
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
            if (AG)
              tma_gather4(&tmA, &full[stage], sa + half * 8192 + g * 512, m0 + 64 * half, r[0], r[1], r[2], r[3]);
            if (BG) {
#pragma unroll
              for (int b = 2 * half; b < 2 * half + 2; ++b)
                if (b < BN / 64)
                  tma_gather4(&tmB, &full[stage], sb + b * 8192 + g * 512, n0 + 64 * b, r[0], r[1], r[2], r[3]);
            }
          }
          if (lane == 0) {
            if (!AG) {
              tma_load_2d(&tmA, &full[stage], sa, m0, kb * BK);
              tma_load_2d(&tmA, &full[stage], sa + 8192, m0 + 64, kb * BK);
            }
            if (!BG) {
#pragma unroll
              for (int b = 0; b < BN / 64; ++b) tma_load_2d(&tmB, &full[stage], sb + b * 8192, n0 + 64 * b, kb * BK);
            }
          }
        } else {
          // A: K-major rows (m) x 64 contraction columns
          if (AG) tma_gather4(&tmA, &full[stage], sa + lane * 512, kb * BK, ar0, ar1, ar2, ar3);
          if (lane == 0) {
            if (!AG) tma_load_2d(&tmA, &full[stage], sa, kb * BK, m0);
            if (KIND == KIND_DX) {
              // B = G^T [n, N] MN-major dense: 64 contraction rows x BN columns
#pragma unroll
              for (int b = 0; b < BN / 64; ++b) tma_load_2d(&tmB, &full[stage], sb + b * 8192, n0 + 64 * b, kb * BK);
            } else {
              // B = G^T [n, N] K-major dense: BN rows (output cols j) x 64 tokens
              tma_load_2d(&tmB, &full[stage], sb, kb * BK, n0);
            }
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    constexpr uint32_t IDESC = make_idesc_bf16(BM, BN, KIND == KIND_FWD ? 1 : 0, KIND == KIND_DW ? 0 : 1);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile % m_tiles) * BM;
      if (zero_tile(m0)) continue;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(ring + stage * SM::STAGE_BYTES);
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
            umma_bf16(d_tmem, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ============================ epilogue ================================
    const int ew = warp - 4;  // TMEM lane quarter == warp % 4
    uint8_t* stg = staging + ew * STAGING_PER_WARP;
    uint8_t* stg2 = stg + 32 * 128;
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile % m_tiles) * BM;
      const int n0 = (tile / m_tiles) * BN;
      const bool zt = zero_tile(m0);
      // output rows this lane stores: r = 4 i + lane / 8, i = 0..7
      int orow[8], arow[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + ew * 32 + 4 * i + (lane >> 3);
        int o = -1;
        if (m < p.M) {
          if (KIND == KIND_FWD)
            o = p.out_pos ? __ldg(p.out_pos + m) : m;   // producer-side compaction for the next layer
          else
            o = (m < p.n_kept) ? __ldg(p.kept + m) : __ldg(p.pruned + (m - p.n_kept));
        }
        orow[i] = o;
        arow[i] = p.aux_by_m ? m : o;
      }
      if (!zt) {
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
      }
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c) {
        uint32_t v0[32], v1[32];
        if (!zt) {
          tmem_ld_32x32b_x32(tbase + c * 64, v0);
          tmem_ld_32x32b_x32(tbase + c * 64 + 32, v1);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v0[i] = v1[i] = 0u;
        }
        // thread `lane` owns tile row ew*32 + lane: 64 fp32 -> 8 x 16B chunks
        const int r = lane;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int col = q * 8 + i;
            f[i] = __uint_as_float(col < 32 ? v0[col] : v1[col - 32]);
          }
          uint4 w;
          w.x = pack_bf16(f[0], f[1]);
          w.y = pack_bf16(f[2], f[3]);
          w.z = pack_bf16(f[4], f[5]);
          w.w = pack_bf16(f[6], f[7]);
          const int off = r * 128 + ((q ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(stg + off) = w;
          if (p.epi == EPI_GELU) {
            uint4 g;
            g.x = pack_bf16(gelu_f(f[0]), gelu_f(f[1]));
            g.y = pack_bf16(gelu_f(f[2]), gelu_f(f[3]));
            g.z = pack_bf16(gelu_f(f[4]), gelu_f(f[5]));
            g.w = pack_bf16(gelu_f(f[6]), gelu_f(f[7]));
            *reinterpret_cast<uint4*>(stg2 + off) = g;
          }
        }
        __syncwarp();
        const int q = lane & 7;
        const int col = n0 + c * 64 + q * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = 4 * i + (lane >> 3);
          const int off = rr * 128 + ((q ^ (rr & 7)) << 4);
          if (orow[i] >= 0 && col < p.N) {
            uint4 w = *reinterpret_cast<const uint4*>(stg + off);
            if (p.epi == EPI_GELU_GRAD && !zt) {
              // G1 = dH * GeLU'(pre_in) at the same (row, col) (row layer BWD)
              const uint4 pin = *reinterpret_cast<const uint4*>(p.aux + (int64_t)arow[i] * p.ld_aux + col);
              w.x = pack_bf16(bf16_lo(w.x) * gelu_grad_f(bf16_lo(pin.x)), bf16_hi(w.x) * gelu_grad_f(bf16_hi(pin.x)));
              w.y = pack_bf16(bf16_lo(w.y) * gelu_grad_f(bf16_lo(pin.y)), bf16_hi(w.y) * gelu_grad_f(bf16_hi(pin.y)));
              w.z = pack_bf16(bf16_lo(w.z) * gelu_grad_f(bf16_lo(pin.z)), bf16_hi(w.z) * gelu_grad_f(bf16_hi(pin.z)));
              w.w = pack_bf16(bf16_lo(w.w) * gelu_grad_f(bf16_lo(pin.w)), bf16_hi(w.w) * gelu_grad_f(bf16_hi(pin.w)));
            }
            st_global_v4(p.out + (int64_t)orow[i] * p.ld_out + col, w);
            if (p.epi == EPI_GELU) {
              const uint4 g = *reinterpret_cast<const uint4*>(stg2 + off);
              st_global_v4(p.out2 + (int64_t)orow[i] * p.ld_out2 + col, g);
            }
          }
        }
        __syncwarp();
      }
      if (!zt) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
  if (p.stamp != nullptr && threadIdx.x == 0) atomicMax(p.stamp + 1, (unsigned long long)globaltimer());
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

// bf16 row-major [rows, cols] with leading dimension ld (elements); box = box_cols x box_rows.
static bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
                     uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int KIND, int BN, bool AG, bool BG>
static cudaError_t launch_kind(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p, int num_sms,
                               cudaStream_t st) {
  static bool attr_set = false;
  const int smem = Smem<BN>::TOTAL;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(ztp_gemm_kernel<KIND, BN, AG, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  ztp_gemm_kernel<KIND, BN, AG, BG><<<grid, NUM_THREADS, smem, st>>>(a, b, p);
  return cudaGetLastError();
}

// Operand A / B tensor maps per kind (see the header comment of this file).
cudaError_t gemm_launch(int kind, const GemmOperands& o, GemmParams p, int num_sms, cudaStream_t st) {
  CUtensorMap ta, tb;
  bool ok = true;
  const bool ag = o.a_gather, bg = o.b_gather;
  p.oob_row = (int)(o.a_rows > o.b_rows ? o.a_rows : o.b_rows);  // outside every gathered tensor
  if (kind == KIND_FWD) {
    // A = W^T [K|K', n] MN-major; B = X^T [K|K', N] MN-major (same rows)
    ok &= make_map(&ta, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : 64);
    ok &= make_map(&tb, o.b, o.b_rows, o.b_cols, o.b_ld, 64, bg ? 1 : 64);
  } else if (kind == KIND_DX) {
    // A = W^T [K|K', n_out] K-major; B = G^T [n_out, N] MN-major 64 x 64 boxes
    ok &= make_map(&ta, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : BM);
    ok &= make_map(&tb, o.b, o.b_rows, o.b_cols, o.b_ld, 64, 64);
  } else {
    // A = X^T [K|K', N] K-major; B = G^T [n_out, N] K-major box 64 x 256
    ok &= make_map(&ta, o.a, o.a_rows, o.a_cols, o.a_ld, 64, ag ? 1 : BM);
    ok &= make_map(&tb, o.b, o.b_rows, o.b_cols, o.b_ld, 64, 256);
  }
  if (!ok) return cudaErrorInvalidValue;
#define ZTP_DISPATCH(K_)                                                          \
  if (ag && bg) return launch_kind<K_, 256, true, true>(ta, tb, p, num_sms, st);   \
  if (ag) return launch_kind<K_, 256, true, false>(ta, tb, p, num_sms, st);        \
  if (bg) return launch_kind<K_, 256, false, true>(ta, tb, p, num_sms, st);        \
  return launch_kind<K_, 256, false, false>(ta, tb, p, num_sms, st);
  if (kind == KIND_FWD) {
    ZTP_DISPATCH(KIND_FWD)
  }
  if (kind == KIND_DX) {
    if (bg) return cudaErrorInvalidValue;
    if (ag) return launch_kind<KIND_DX, 256, true, false>(ta, tb, p, num_sms, st);
    return launch_kind<KIND_DX, 256, false, false>(ta, tb, p, num_sms, st);
  }
  if (bg) return cudaErrorInvalidValue;
  if (ag) return launch_kind<KIND_DW, 256, true, false>(ta, tb, p, num_sms, st);
  return launch_kind<KIND_DW, 256, false, false>(ta, tb, p, num_sms, st);
#undef ZTP_DISPATCH
}

}  // namespace ztp

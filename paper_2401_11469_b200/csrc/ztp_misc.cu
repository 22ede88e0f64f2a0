// Small kernels of the path: straggler emulation (delay after each GEMM),
// the stand-in attention core (A-31), row fills, and the fp32 verification
// GEMM (SIMT FFMA with the same lineage semantics as the tcgen05 kernel).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ztp_internal.h"
#include "ztp_ptx.cuh"

namespace ztp {

// ------------------------------------------------------------ emulation
// The GEMM stamped [start_min, end_max] of its CTAs; spin until
// start + chi (end - start) so the rank's GEMM takes chi times longer (A-32),
// accumulate the (stretched) GEMM time into acc_ns[0] (M_i, A-6), reset stamps.
// Concurrent GEMMs (dX / dW on two streams, two stamp slots) are counted
// once where they overlap: acc_ns[1] is the latest end already accounted, and
// each delay adds only the part of [start, now] after it (the union of the
// GEMM intervals, up to the order in which two overlapping delays finish).
__global__ void ztp_delay_kernel(unsigned long long* stamp, double chi, unsigned long long* acc_ns) {
  pdl_wait();
  pdl_trigger();
  const unsigned long long s = stamp[0], e = stamp[1];
  if (s != ~0ull && e >= s) {
    const unsigned long long dur = e - s;
    const unsigned long long target = s + (unsigned long long)(chi * (double)dur);
    unsigned long long now = globaltimer();
    while (now < target) {
      __nanosleep(256);
      now = globaltimer();
    }
    if (acc_ns) {
      const unsigned long long seen = atomicMax(acc_ns + 1, now);
      const unsigned long long from = seen > s ? seen : s;
      if (now > from) atomicAdd(acc_ns, now - from);
    }
  }
  stamp[0] = ~0ull;
  stamp[1] = 0ull;
}

__global__ void ztp_stamp_reset_kernel(unsigned long long* stamp) {
  pdl_wait();
  pdl_trigger();
  stamp[0] = ~0ull;
  stamp[1] = 0ull;
}

cudaError_t delay_launch(unsigned long long* stamp, double chi, unsigned long long* acc_ns, cudaStream_t st) {
  return launch_k(ztp_delay_kernel, 1, 1, 0, st, stamp, chi, acc_ns);
}
cudaError_t stamp_reset_launch(unsigned long long* stamp, cudaStream_t st) {
  return launch_k(ztp_stamp_reset_kernel, 1, 1, 0, st, stamp);
}

// ------------------------------------------------------ stand-in core (A-31)
// FWD ctx[f,t] = q[f,t] + k[f,t] + v[f,t]; BWD q = k = v = dctx.  16-byte vectors.
// v_compact (A-36): the V block holds only the O projection's kept features
// (V row i <- feature rows[i]), FWD reads it at i, BWD writes dV there.
// BWD walks the 2 n_feat + n_v output rows once (each written once).
__global__ void ztp_core_bf16(int phase, const __nv_bfloat16* __restrict__ qkv_c, __nv_bfloat16* qkv, int64_t ld_qkv,
                              __nv_bfloat16* ctx, int64_t ld_ctx, int64_t feat, int64_t n_feat, int64_t N,
                              const int32_t* __restrict__ rows, int64_t n_v, int v_compact) {
  pdl_wait();
  pdl_trigger();
  const int64_t vec_per_row = N / 8;
  const int64_t total = (phase == 0 ? n_feat : 2 * n_feat + n_v) * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / vec_per_row, c = (i % vec_per_row) * 8;
    if (phase == 0) {
      const int64_t sf = rows ? (int64_t)__ldg(rows + f) : f;  // compact output row f <- feature sf
      const int64_t vr = v_compact ? 2 * feat + f : 2 * feat + sf;
      const uint4 a = *reinterpret_cast<const uint4*>(qkv_c + sf * ld_qkv + c);
      const uint4 b = *reinterpret_cast<const uint4*>(qkv_c + (feat + sf) * ld_qkv + c);
      const uint4 d = *reinterpret_cast<const uint4*>(qkv_c + vr * ld_qkv + c);
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
      const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&d);
      uint4 o;
      __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 x = __bfloat1622float2(pa[j]), y = __bfloat1622float2(pb[j]), z = __bfloat1622float2(pd[j]);
        po[j] = __floats2bfloat162_rn((x.x + y.x) + z.x, (x.y + y.y) + z.y);
      }
      *reinterpret_cast<uint4*>(ctx + f * ld_ctx + c) = o;
    } else {
      // output row f of g_qkv: Q rows [0, n_feat), K rows [feat, feat + n_feat), V rows from 2 feat
      int64_t orow, grow;
      if (f < n_feat) {
        orow = f;
        grow = f;
      } else if (f < 2 * n_feat) {
        orow = feat + (f - n_feat);
        grow = f - n_feat;
      } else {
        const int64_t j = f - 2 * n_feat;
        orow = 2 * feat + j;
        grow = v_compact ? (int64_t)__ldg(rows + j) : j;
      }
      *reinterpret_cast<uint4*>(qkv + orow * ld_qkv + c) = *reinterpret_cast<const uint4*>(ctx + grow * ld_ctx + c);
    }
  }
}

__global__ void ztp_core_f32(int phase, float* qkv, int64_t ld_qkv, float* ctx, int64_t ld_ctx, int64_t feat,
                             int64_t n_feat, int64_t N, const int32_t* __restrict__ rows, int64_t n_v, int v_compact) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (phase == 0 ? n_feat : 2 * n_feat + n_v) * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / N, c = i % N;
    if (phase == 0) {
      const int64_t sf = rows ? (int64_t)rows[f] : f;
      const int64_t vr = v_compact ? 2 * feat + f : 2 * feat + sf;
      ctx[f * ld_ctx + c] = (qkv[sf * ld_qkv + c] + qkv[(feat + sf) * ld_qkv + c]) + qkv[vr * ld_qkv + c];
    } else {
      int64_t orow, grow;
      if (f < n_feat) {
        orow = f;
        grow = f;
      } else if (f < 2 * n_feat) {
        orow = feat + (f - n_feat);
        grow = f - n_feat;
      } else {
        const int64_t j = f - 2 * n_feat;
        orow = 2 * feat + j;
        grow = v_compact ? (int64_t)rows[j] : j;
      }
      qkv[orow * ld_qkv + c] = ctx[grow * ld_ctx + c];
    }
  }
}

cudaError_t core_launch(int phase, const void* qkv, int64_t ld_qkv, void* ctx, int64_t ld_ctx, int64_t feat,
                        int64_t n_feat, int64_t N, int dtype, const int32_t* rows, int64_t n_v, int v_compact,
                        cudaStream_t st, bool pdl) {
  const int threads = 256;
  const int blocks = 148 * 8;
  if (dtype == 0)
    return launch_k_pdl(pdl, ztp_core_bf16, blocks, threads, 0, st, phase, (const __nv_bfloat16*)qkv,
                        (__nv_bfloat16*)qkv, ld_qkv, (__nv_bfloat16*)ctx, ld_ctx, feat, n_feat, N, rows, n_v, v_compact);
  return launch_k_pdl(pdl, ztp_core_f32, blocks, threads, 0, st, phase, (float*)qkv, ld_qkv, (float*)ctx, ld_ctx, feat,
                      n_feat, N, rows, n_v, v_compact);
}

// ------------------------------------------------- row compaction (a4 gather)
// dst[i, :] = src[idx[i], :] for i < n: the kept rows S of a feature-major
// tensor packed contiguously (producer-side "dimension extracting"), so
// the GEMM mainloop streams dense TMA boxes.  HBM-bound, 16-byte vectors.
__global__ void ztp_gather_rows(const uint8_t* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ idx,
                                int n, int64_t vec_per_row, uint8_t* __restrict__ dst, int64_t ld_dst) {
  pdl_wait();
  pdl_trigger();
  constexpr int U = 4;   // independent vectors in flight per thread
  const int64_t total = (int64_t)n * vec_per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < total; i0 += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        const int64_t r = i / vec_per_row, c = i % vec_per_row;
        v[u] = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)__ldg(idx + r) * ld_src) + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < total) {
        const int64_t r = i / vec_per_row, c = i % vec_per_row;
        reinterpret_cast<uint4*>(dst + r * ld_dst)[c] = v[u];
      }
    }
  }
}

// Rows whose width is not a multiple of 16 bytes: element-wise copy.
__global__ void ztp_gather_rows_elem(const uint8_t* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ idx,
                                     int n, int64_t cols, int64_t es, uint8_t* __restrict__ dst, int64_t ld_dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)n * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t sr = __ldg(idx + r);
    if (es == 2)
      reinterpret_cast<uint16_t*>(dst + r * ld_dst)[c] = reinterpret_cast<const uint16_t*>(src + sr * ld_src)[c];
    else
      reinterpret_cast<uint32_t*>(dst + r * ld_dst)[c] = reinterpret_cast<const uint32_t*>(src + sr * ld_src)[c];
  }
}

cudaError_t gather_rows_launch(const void* src, int64_t ld_src, const int32_t* idx, int n, int64_t cols, void* dst,
                               int64_t ld_dst, int dtype, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t es = dtype == 0 ? 2 : 4;
  const int64_t row_bytes = cols * es;
  if (row_bytes % 16) {
    const int64_t total = (int64_t)n * cols;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    return launch_k(ztp_gather_rows_elem, blocks, 256, 0, st, (const uint8_t*)src, ld_src * es, idx, n, cols, es,
                    (uint8_t*)dst, ld_dst * es);
  }
  const int64_t total = (int64_t)n * (row_bytes / 16);
  int blocks = (int)((total + 1023) / 1024);
  if (blocks > 148 * 8) blocks = 148 * 8;
  return launch_k(ztp_gather_rows, blocks, 256, 0, st, (const uint8_t*)src, ld_src * es, idx, n, row_bytes / 16,
                  (uint8_t*)dst, ld_dst * es);
}

// ------------------------------------ 2D compaction (output pruning, bf16)
// dst[r, c] = src[rows ? rows[r] : r, cols[c]] for r < n, c < nc: the weight
// block W^T[S, S'] a col layer needs when its consumer keeps only S' of its
// outputs.  Each thread builds 8 output columns (one 16-byte store) from the
// source row, which stays in L1 across the warp (cols ascending).
__global__ void ztp_gather_2d(const uint16_t* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ rows,
                              int n, const int32_t* __restrict__ cols, int nc, uint16_t* __restrict__ dst,
                              int64_t ld_dst) {
  pdl_wait();
  pdl_trigger();
  const int vpr = (nc + 7) / 8;
  const int64_t total = (int64_t)n * vpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / vpr), c0 = (int)(i % vpr) * 8;
    const uint16_t* s = src + (int64_t)(rows ? __ldg(rows + r) : r) * ld_src;
    uint16_t* d = dst + (int64_t)r * ld_dst + c0;
    if (c0 + 8 <= nc) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = (uint32_t)__ldg(s + __ldg(cols + c0 + 2 * q)) | ((uint32_t)__ldg(s + __ldg(cols + c0 + 2 * q + 1)) << 16);
      *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (int c = c0; c < nc; ++c) d[c - c0] = __ldg(s + __ldg(cols + c));
    }
  }
}

cudaError_t gather_2d_launch(const void* src, int64_t ld_src, const int32_t* rows, int n, const int32_t* cols, int nc,
                             void* dst, int64_t ld_dst, cudaStream_t st) {
  if (n <= 0 || nc <= 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0 || ld_dst % 8 != 0) return cudaErrorMisalignedAddress;
  const int64_t total = (int64_t)n * ((nc + 7) / 8);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(ztp_gather_2d, blocks, 256, 0, st, (const uint16_t*)src, ld_src, rows, n, cols, nc, (uint16_t*)dst,
                  ld_dst);
}

// Batched compaction of several operands (ztp_prepare): one launch over work
// items of (job, row, 1024-column chunk), one warp per item, so every SM
// keeps many independent 2 KB copies in flight (no shared memory: full
// occupancy).  Row copies stream 16-byte vectors, 4 per lane in flight; 2D
// jobs (a weight block W^T[S, S'], output pruning) gather the kept columns
// of the source row with 2-byte loads (the chunk's source window is a few KB,
// served by L1 after its first touch) and store 16-byte vectors.
constexpr int GM_CHUNK = 1024;   // output elements per work item

__device__ __forceinline__ uint32_t gm_pick2(const uint16_t* s, int a, int b) {
  return (uint32_t)__ldg(s + a) | ((uint32_t)__ldg(s + b) << 16);
}

__global__ void __launch_bounds__(256) ztp_gather_multi(const GatherJobs J) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < J.total; it += nw) {
    int j = 0;
#pragma unroll 1
    while (j + 1 < J.njobs && it >= J.job[j + 1].rbegin) ++j;
    const GatherJob& g = J.job[j];
    const int64_t li = it - g.rbegin;
    const int cpr = (g.nc + GM_CHUNK - 1) / GM_CHUNK;
    const int r = (int)(li / cpr), c0 = (int)(li % cpr) * GM_CHUNK;
    const int c1 = min(g.nc, c0 + GM_CHUNK);
    const uint16_t* s = g.src + (int64_t)(g.rows ? __ldg(g.rows + r) : r) * g.ld_src;
    uint16_t* d = g.dst + (int64_t)r * g.ld_dst;
    const int v1 = c0 + (c1 - c0) / 8 * 8;         // end of the 8-column groups
    if (!g.cols) {
      uint4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 8 * (lane + 32 * u);
        if (c < v1) w[u] = __ldg(reinterpret_cast<const uint4*>(s + c));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 8 * (lane + 32 * u);
        if (c < v1) *reinterpret_cast<uint4*>(d + c) = w[u];
      }
      for (int c = v1 + lane; c < c1; c += 32) d[c] = __ldg(s + c);
      continue;
    }
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) {
        int4 q0, q1;
        if ((reinterpret_cast<uintptr_t>(g.cols) & 15) == 0) {
          q0 = __ldg(reinterpret_cast<const int4*>(g.cols + c));
          q1 = __ldg(reinterpret_cast<const int4*>(g.cols + c + 4));
        } else {
          q0 = make_int4(__ldg(g.cols + c), __ldg(g.cols + c + 1), __ldg(g.cols + c + 2), __ldg(g.cols + c + 3));
          q1 = make_int4(__ldg(g.cols + c + 4), __ldg(g.cols + c + 5), __ldg(g.cols + c + 6), __ldg(g.cols + c + 7));
        }
        if ((q0.x & 7) == 0 && q0.y == q0.x + 1 && q0.z == q0.x + 2 && q0.w == q0.x + 3 && q1.x == q0.x + 4 &&
            q1.y == q0.x + 5 && q1.z == q0.x + 6 && q1.w == q0.x + 7)   // eight consecutive columns: one 16-byte load
          w[u] = __ldg(reinterpret_cast<const uint4*>(s + q0.x));
        else
          w[u] = make_uint4(gm_pick2(s, q0.x, q0.y), gm_pick2(s, q0.z, q0.w), gm_pick2(s, q1.x, q1.y),
                            gm_pick2(s, q1.z, q1.w));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) *reinterpret_cast<uint4*>(d + c) = w[u];
    }
    for (int c = v1 + lane; c < c1; c += 32) d[c] = __ldg(s + __ldg(g.cols + c));
  }
}

cudaError_t gather_multi_launch(const GatherJobs& j, cudaStream_t st) {
  if (j.total <= 0) return cudaSuccess;
  GatherJobs J = j;   // work items instead of rows
  int64_t items = 0;
  for (int i = 0; i < J.njobs; ++i) {
    GatherJob& g = J.job[i];
    if ((reinterpret_cast<uintptr_t>(g.src) & 15) || (reinterpret_cast<uintptr_t>(g.dst) & 15) || g.ld_src % 8 ||
        g.ld_dst % 8)
      return cudaErrorMisalignedAddress;
    if (g.cols && (g.src_cols <= 0 || g.src_cols > g.ld_src)) return cudaErrorInvalidValue;
    g.rbegin = items;
    items += (int64_t)g.n * ((g.nc + GM_CHUNK - 1) / GM_CHUNK);
  }
  J.total = items;
  const int64_t need = (items + 7) / 8;
  const int blocks = (int)std::min<int64_t>(need, (int64_t)148 * 8);
  return launch_k(ztp_gather_multi, blocks, 256, 0, st, J);
}

// Column expansion (output pruning, bf16), out of place, over the lineage
// rows: a kept row r = kept[i] gets dst[r, j] = pos[j] >= 0 ? src[r, pos[j]]
// : 0 (the Zero gradient of the consumer-pruned units), a pruned row
// r = pruned[i] (the Zero rows P) is written 0 without reading the
// scratch -- the dW GEMM computes no all-pruned units in this mode.  Work
// items of (row, 1024 output columns), one warp each: 8-column groups, pos
// read as 16-byte vectors, the compact source window gathered with 2-byte
// loads (L1), 16-byte stores.  (Within 1.1-1.6x of a device memcpy of the
// same bytes; CTA-tiled variants staging the windows in shared memory were
// slower: tools/bench_src/expand_bench.cu, profiles/r02_expand_variants.txt.)
__global__ void __launch_bounds__(256) ztp_expand_cols(const uint16_t* __restrict__ src, int64_t ld_src,
                                                       uint16_t* __restrict__ dst, int64_t ld_dst,
                                                       const int32_t* __restrict__ kept, int nk,
                                                       const int32_t* __restrict__ pruned, int np,
                                                       const int32_t* __restrict__ pos, int n_full) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int cpr = (n_full + GM_CHUNK - 1) / GM_CHUNK;
  const int64_t items = (int64_t)(nk + np) * cpr;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool pv = (reinterpret_cast<uintptr_t>(pos) & 15) == 0;
  const bool sv = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && ld_src % 8 == 0;   // 16-byte runs of src
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += nw) {
    const int i = (int)(it / cpr), c0 = (int)(it % cpr) * GM_CHUNK;
    const int c1 = min(n_full, c0 + GM_CHUNK);
    const int v1 = c0 + (c1 - c0) / 8 * 8;
    const bool zero_row = i >= nk;
    const int r = zero_row ? __ldg(pruned + (i - nk)) : (kept ? __ldg(kept + i) : i);
    const uint16_t* s = src + (int64_t)r * ld_src;
    uint16_t* d = dst + (int64_t)r * ld_dst;
    if (zero_row) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 8 * (lane + 32 * u);
        if (c < v1) *reinterpret_cast<uint4*>(d + c) = make_uint4(0u, 0u, 0u, 0u);
      }
      for (int c = v1 + lane; c < c1; c += 32) d[c] = 0;
      continue;
    }
    auto pick = [&](int q) -> uint32_t { return q >= 0 ? (uint32_t)__ldg(s + q) : 0u; };
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) {
        int4 q0, q1;
        if (pv) {
          q0 = __ldg(reinterpret_cast<const int4*>(pos + c));
          q1 = __ldg(reinterpret_cast<const int4*>(pos + c + 4));
        } else {
          q0 = make_int4(__ldg(pos + c), __ldg(pos + c + 1), __ldg(pos + c + 2), __ldg(pos + c + 3));
          q1 = make_int4(__ldg(pos + c + 4), __ldg(pos + c + 5), __ldg(pos + c + 6), __ldg(pos + c + 7));
        }
        if (sv && q0.x >= 0 && (q0.x & 7) == 0 && q0.y == q0.x + 1 && q0.z == q0.x + 2 && q0.w == q0.x + 3 &&
            q1.x == q0.x + 4 && q1.y == q0.x + 5 && q1.z == q0.x + 6 && q1.w == q0.x + 7)   // eight kept columns in a row
          w[u] = __ldg(reinterpret_cast<const uint4*>(s + q0.x));
        else
          w[u] = make_uint4(pick(q0.x) | (pick(q0.y) << 16), pick(q0.z) | (pick(q0.w) << 16),
                            pick(q1.x) | (pick(q1.y) << 16), pick(q1.z) | (pick(q1.w) << 16));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) *reinterpret_cast<uint4*>(d + c) = w[u];
    }
    for (int c = v1 + lane; c < c1; c += 32) d[c] = (uint16_t)pick(__ldg(pos + c));
  }
}

cudaError_t expand_cols_launch(const void* src, int64_t ld_src, void* dst, int64_t ld_dst, const int32_t* kept,
                               int nk, const int32_t* pruned, int np, const int32_t* pos, int n_full,
                               cudaStream_t st) {
  if (nk + np <= 0 || n_full <= 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0 || ld_dst % 8 != 0) return cudaErrorMisalignedAddress;
  if (np > 0 && !pruned) return cudaErrorInvalidValue;
  const int64_t items = (int64_t)(nk + np) * ((n_full + GM_CHUNK - 1) / GM_CHUNK);
  const int blocks = (int)std::min<int64_t>((items + 7) / 8, (int64_t)148 * 8);
  return launch_k(ztp_expand_cols, blocks, 256, 0, st, (const uint16_t*)src, ld_src, (uint16_t*)dst, ld_dst, kept,
                  nk, pruned, np, pos, n_full);
}

// ------------------------------------------ Average / Same imputation (NEXT-2)
// Average (A-10): the per-column mean over the kept rows S, in fp32
// with a fixed summation tree (deterministic), written to every row p in P
// (the GEMM's Zero rows are overwritten).  Same (A-11): out[p] <- hist[p].
template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }

// Local reduce (NEXT-3 migration: a helper's migrated contribution merged
// into its partial before the all-reduce; the root's sum of gathered
// partials): dst[r, c] (+)= sum_{q < nparts} src[q * part_stride + r, c], the
// parts added in order q = 0.. in fp32, one rounding.
template <typename T>
__global__ void __launch_bounds__(256) ztp_accumulate(T* dst, int64_t ld_dst, const T* src, int64_t ld_src,
                                                      int64_t rows, int64_t cols, int nparts, int64_t part_stride,
                                                      int overwrite) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    float a = overwrite ? 0.f : to_f<T>(dst[r * ld_dst + c]);
    for (int q = 0; q < nparts; ++q) a += to_f<T>(src[(q * part_stride + r) * ld_src + c]);
    dst[r * ld_dst + c] = from_f<T>(a);
  }
}

// Average, pass 1: one CTA per 32 columns; its 256 threads are 4 groups of 8
// columns x 64 row slices striding the kept rows S (4 loads in flight per
// thread); the 64 slices' fp32 partial sums are combined by a fixed tree
// (deterministic) and mean = sum / |S| is stored per column (fp32 workspace).
template <typename T>
__global__ void __launch_bounds__(256) ztp_impute_means(const T* out, int64_t ld, int64_t cols, const int32_t* kept,
                                                        int nk, float* means) {
  pdl_wait();
  pdl_trigger();
  __shared__ float part[64][33];
  const int cg = threadIdx.x & 3, sl = threadIdx.x >> 2;      // column group, row slice
  const int64_t c0 = (int64_t)blockIdx.x * 32 + cg * 8;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const bool full = c0 + 8 <= cols;
  for (int i0 = sl; i0 < nk; i0 += 64 * 4) {
    T v[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + 64 * u;
      if (i < nk) {
        const T* row = out + (int64_t)__ldg(kept + i) * ld + c0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[u][q] = (full || c0 + q < cols) ? row[q] : from_f<T>(0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + 64 * u < nk)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += to_f<T>(v[u][q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) part[sl][cg * 8 + q] = acc[q];
  __syncthreads();
  for (int w = 32; w > 0; w >>= 1) {           // fixed-order tree over the 64 row slices
    for (int j = threadIdx.x; j < w * 32; j += blockDim.x) part[j / 32][j % 32] += part[j / 32 + w][j % 32];
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
    if (c < cols) means[c] = part[0][threadIdx.x] * (1.0f / (float)nk);
  }
}

// Average, pass 2: rows P <- the column means, one warp per (row, 256
// columns), 8 columns per lane, 16-byte stores where the row allows.
template <typename T>
__global__ void __launch_bounds__(256) ztp_impute_fill(T* out, int64_t ld, int64_t cols, const int32_t* pruned, int np,
                                                       const float* means) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t cpr = (cols + 255) / 256, items = (int64_t)np * cpr;
  const bool vec = (sizeof(T) == 2) && ((ld * 2) % 16 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  for (int64_t it = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); it < items; it += (int64_t)gridDim.x * 8) {
    const int64_t r = __ldg(pruned + it / cpr), c = (it % cpr) * 256 + lane * 8;
    T* o = out + r * ld + c;
    if (vec && c + 8 <= cols) {
      const float4 a = *reinterpret_cast<const float4*>(means + c), b = *reinterpret_cast<const float4*>(means + c + 4);
      const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      T v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = from_f<T>(f[q]);
      *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(v);
    } else {
      for (int q = 0; q < 8 && c + q < cols; ++q) o[q] = from_f<T>(means[c + q]);
    }
  }
}

// Same: rows P copied from the history, 16-byte vectors (4 in flight per
// thread) when the row widths allow, else element-wise.
template <typename T>
__global__ void __launch_bounds__(256) ztp_impute_same(T* out, int64_t ld, int64_t cols, const int32_t* pruned, int np,
                                                       const T* hist, int64_t ld_hist, int vec) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    constexpr int E = 16 / sizeof(T);
    const int64_t vpr = cols / E, total = (int64_t)np * vpr;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < total; i0 += 4 * stride) {
      uint4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < total) {
          const int64_t r = __ldg(pruned + i / vpr), c = (i % vpr) * E;
          w[u] = __ldg(reinterpret_cast<const uint4*>(hist + r * ld_hist + c));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < total) {
          const int64_t r = __ldg(pruned + i / vpr), c = (i % vpr) * E;
          *reinterpret_cast<uint4*>(out + r * ld + c) = w[u];
        }
      }
    }
    return;
  }
  const int64_t total = (int64_t)np * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = __ldg(pruned + i / cols), c = i % cols;
    out[r * ld + c] = hist[r * ld_hist + c];
  }
}

cudaError_t impute_rows_launch(void* out, int64_t ld, int64_t cols, const int32_t* kept, int nk, const int32_t* pruned,
                               int np, int mode, const void* hist, int64_t ld_hist, int dtype, void* ws,
                               cudaStream_t st) {
  if (np <= 0 || cols <= 0) return cudaSuccess;
  if (mode == 1) {
    if (!ws) return cudaErrorInvalidValue;
    float* means = static_cast<float*>(ws);
    const int blocks = (int)((cols + 31) / 32);
    const int64_t items = (int64_t)np * ((cols + 255) / 256);
    const int fb = (int)std::min<int64_t>((items + 7) / 8, (int64_t)148 * 8);
    cudaError_t e;
    if (dtype == 0) {
      e = launch_k(ztp_impute_means<__nv_bfloat16>, blocks, 256, 0, st, (const __nv_bfloat16*)out, ld, cols, kept, nk,
                   means);
      if (e == cudaSuccess)
        e = launch_k(ztp_impute_fill<__nv_bfloat16>, fb, 256, 0, st, (__nv_bfloat16*)out, ld, cols, pruned, np,
                     (const float*)means);
      return e;
    }
    e = launch_k(ztp_impute_means<float>, blocks, 256, 0, st, (const float*)out, ld, cols, kept, nk, means);
    if (e == cudaSuccess)
      e = launch_k(ztp_impute_fill<float>, fb, 256, 0, st, (float*)out, ld, cols, pruned, np, (const float*)means);
    return e;
  }
  const int64_t es = dtype == 0 ? 2 : 4;
  const int vec = ((cols * es) % 16 == 0) && ((ld * es) % 16 == 0) && ((ld_hist * es) % 16 == 0) &&
                  ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(hist)) & 15) == 0;
  const int64_t work = vec ? (int64_t)np * cols / (16 / es) / 4 : (int64_t)np * cols;
  int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)148 * 8);
  blocks = std::max(blocks, 1);
  if (dtype == 0)
    return launch_k(ztp_impute_same<__nv_bfloat16>, blocks, 256, 0, st, (__nv_bfloat16*)out, ld, cols, pruned, np,
                    (const __nv_bfloat16*)hist, ld_hist, vec);
  return launch_k(ztp_impute_same<float>, blocks, 256, 0, st, (float*)out, ld, cols, pruned, np, (const float*)hist,
                  ld_hist, vec);
}

// ------------------------------------------- NEXT-1 priority maintenance
// One warp per row i of W^T: lanes stride the row in 8-element (16-byte)
// chunks, fp32 partial sums of |w - w_old| reduced by a fixed shuffle tree
// (deterministic), divided by n.  Rows pruned last epoch keep delta.
__global__ void ztp_priority_update_kernel(const uint16_t* __restrict__ w, int64_t ld_w,
                                           const uint16_t* __restrict__ wo, int64_t ld_o, int64_t K, int64_t n,
                                           const int32_t* __restrict__ pos_prev, float* delta, int32_t* count_above,
                                           float theta) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < K; i += warps) {
    float d;
    if (pos_prev && __ldg(pos_prev + i) < 0) {
      d = delta[i];                               // pruned last epoch: carried over
    } else {
      const uint16_t* a = w + i * ld_w;
      const uint16_t* b = wo + i * ld_o;
      float acc = 0.f;
      for (int64_t c = (int64_t)lane * 8; c < n; c += 256) {
        if (c + 8 <= n) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + c));
          const uint4 y = __ldg(reinterpret_cast<const uint4*>(b + c));
          const uint32_t xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc += fabsf(__uint_as_float(xa[q] << 16) - __uint_as_float(ya[q] << 16));
            acc += fabsf(__uint_as_float(xa[q] & 0xFFFF0000u) - __uint_as_float(ya[q] & 0xFFFF0000u));
          }
        } else {
          for (int64_t e = c; e < n; ++e)
            acc += fabsf(__uint_as_float((uint32_t)a[e] << 16) - __uint_as_float((uint32_t)b[e] << 16));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
      d = __shfl_sync(0xFFFFFFFFu, acc, 0) / (float)n;
      if (lane == 0) delta[i] = d;
    }
    if (count_above && lane == 0 && d > theta) atomicAdd(count_above, 1);
  }
}

cudaError_t priority_update_launch(const void* w, int64_t ld_w, const void* w_old, int64_t ld_old, int64_t K,
                                   int64_t n, const int32_t* pos_prev, float* delta, int32_t* count_above,
                                   float theta, cudaStream_t st) {
  if (K <= 0) return cudaSuccess;
  int blocks = (int)((K + 7) / 8);                   // 8 warps per block, one row each
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(ztp_priority_update_kernel, blocks, 256, 0, st, (const uint16_t*)w, ld_w, (const uint16_t*)w_old,
                  ld_old, K, n, pos_prev, delta, count_above, theta);
}

// ------------------------------------------------------------- row fill (Zero)
__global__ void ztp_fill_rows(uint8_t* out, int64_t ld_bytes, const int32_t* rows, int nrows, int64_t row_bytes) {
  pdl_wait();
  pdl_trigger();
  const int64_t per = row_bytes / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nrows * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per, c = i % per;
    reinterpret_cast<uint32_t*>(out + (int64_t)rows[r] * ld_bytes)[c] = 0u;
  }
}

cudaError_t fill_rows_launch(void* out, int64_t ld, const int32_t* rows, int nrows, int64_t cols, int dtype,
                             cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  const int64_t es = dtype == 0 ? 2 : 4;
  return launch_k(ztp_fill_rows, 148 * 4, 256, 0, st, (uint8_t*)out, ld * es, rows, nrows, cols * es);
}

// ------------------------------------------- fp32 verification GEMM (SIMT FFMA)
__device__ __forceinline__ float gelu_f32(float x) {
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f32(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * c * (1.0f + 3.0f * 0.044715f * x * x);
}

// 64x64 output tile, 256 threads, 4x4 register micro-tile, k in blocks of 16.
__global__ void __launch_bounds__(256) ztp_gemm_f32_kernel(const GemmParamsF32 p) {
  pdl_wait();
  pdl_trigger();
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  const bool zero_tile = (p.kind != KIND_FWD) && (m0 >= p.n_kept);
  if (!zero_tile) {
    for (int k0 = 0; k0 < p.kdim; k0 += 16) {
      for (int i = threadIdx.x; i < 16 * 64; i += 256) {
        const int kk = i / 64, mm = i % 64;
        const int k = k0 + kk, m = m0 + mm, n = n0 + mm;
        float a = 0.f, b = 0.f;
        if (k < p.kdim) {
          if (p.kind == KIND_FWD) {
            const int64_t kr = p.kept[k];
            if (m < p.M) a = p.w[kr * p.ld_w + m];
            if (n < p.N) b = p.x[(p.x_compact ? (int64_t)k : kr) * p.ld_x + n];
          } else if (p.kind == KIND_DX) {
            if (m < p.n_kept) a = p.w[(int64_t)p.kept[m] * p.ld_w + k];
            if (n < p.N) b = p.g[(int64_t)k * p.ld_g + n];
          } else {
            if (m < p.n_kept) a = p.x[(p.x_compact ? (int64_t)m : (int64_t)p.kept[m]) * p.ld_x + k];
            if (n < p.N) b = p.g[(int64_t)n * p.ld_g + k];
          }
        }
        As[kk][mm] = a;
        Bs[kk][mm] = b;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          av[i] = As[kk][ty * 4 + i];
          bv[i] = Bs[kk][tx * 4 + i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= p.M) continue;
    int64_t orow = m;
    if (p.kind != KIND_FWD)
      orow = (m < p.n_kept) ? p.kept[m] : p.pruned[m - p.n_kept];
    else if (p.out_pos)
      orow = p.out_pos[m];
    if (orow < 0) continue;
    const int64_t arow = p.aux_by_m ? (int64_t)m : orow;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= p.N) continue;
      float v = acc[i][j];
      if (p.epi == EPI_GELU || p.epi == EPI_GELU_D) {
        p.out[orow * p.ld_out + n] = p.epi == EPI_GELU ? v : gelu_grad_f32(v);
        p.out2[orow * p.ld_out2 + n] = gelu_f32(v);
      } else {
        if (p.epi == EPI_GELU_GRAD) v = v * gelu_grad_f32(p.aux[arow * p.ld_aux + n]);
        if (p.epi == EPI_MUL) v = v * p.aux[arow * p.ld_aux + n];
        p.out[orow * p.ld_out + n] = v;
      }
    }
  }
}

cudaError_t gemm_f32_launch(const GemmParamsF32& p, cudaStream_t st) {
  dim3 grid((p.N + 63) / 64, (p.M + 63) / 64);
  return launch_k(ztp_gemm_f32_kernel, grid, 256, 0, st, p);
}

}  // namespace ztp

namespace ztp {
cudaError_t accumulate_launch(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, int64_t rows, int64_t cols,
                              int dtype, int nparts, int64_t part_stride, int overwrite, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t total = rows * cols;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)148 * 16);
  if (dtype == 0)
    return launch_k(ztp_accumulate<__nv_bfloat16>, blocks, 256, 0, st, (__nv_bfloat16*)dst, ld_dst,
                    (const __nv_bfloat16*)src, ld_src, rows, cols, nparts, part_stride, overwrite);
  return launch_k(ztp_accumulate<float>, blocks, 256, 0, st, (float*)dst, ld_dst, (const float*)src, ld_src, rows,
                  cols, nparts, part_stride, overwrite);
}
}  // namespace ztp

namespace ztp {
// Transpose with column selection (the real attention core's layout changes,
// NEXT-4): dst[i, r] = src[r, cols ? cols[i] : i] for i < n, r < R.  32 x 32
// tiles through shared memory (+1 padding: conflict-free), 16-bit elements,
// coalesced reads along src rows and writes along dst rows.
__global__ void __launch_bounds__(256) ztp_transpose_k(const uint16_t* __restrict__ src, int64_t ld_src, int64_t R,
                                                       const int32_t* __restrict__ cols, int64_t n,
                                                       uint16_t* __restrict__ dst, int64_t ld_dst) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint16_t tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 rows of 32 lanes
  const int64_t i = i0 + tx;
  const int64_t c = i < n ? (cols ? (int64_t)__ldg(cols + i) : i) : -1;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k;
    tile[k][tx] = (r < R && c >= 0) ? src[r * ld_src + c] : (uint16_t)0;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t di = i0 + k, r = r0 + tx;
    if (di < n && r < R) dst[di * ld_dst + r] = tile[tx][k];
  }
}

cudaError_t transpose_launch(const void* src, int64_t ld_src, int64_t R, const int32_t* cols, int64_t n, void* dst,
                             int64_t ld_dst, cudaStream_t st) {
  if (R <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((R + 31) / 32));
  if (grid.y > 65535) return cudaErrorInvalidValue;
  return launch_k(ztp_transpose_k, grid, 256, 0, st, (const uint16_t*)src, ld_src, R, cols, n, (uint16_t*)dst,
                  ld_dst);
}
}  // namespace ztp

#include <map>
#include <mutex>
namespace ztp {
cudaError_t ensure_smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[{dev, kernel}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
}  // namespace ztp

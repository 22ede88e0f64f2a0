// a3. Priority select ("the one with small variation can be pruned";
// Alg.1 l.12-14 top-L_pri select + ascendSort; ties by ascending index, A-2).
//
// One CTA (1024 threads) per segment (= one rank-local linear).  The fp32
// score is mapped to an order-preserving 32-bit key (-0 canonicalised to +0),
// a 4 x 8-bit MSB radix select finds the key v of the n_prune-th smallest
// score and how many of the ties at v are pruned; one ordered pass then
// compacts indices into P (pruned) and S (kept) with warp ballot/popc and a
// block scan, so both lists come out ascending without a sort.  Segment sizes
// are <= tens of thousands of columns: the kernel is latency-bound, re-reading
// its scores from L2 on each pass.
#include <cuda_runtime.h>

#include <cstdint>

#include "ztp_internal.h"
#include "ztp_ptx.cuh"

namespace ztp {

__device__ __forceinline__ uint32_t ord32(float x, bool& nan) {
  uint32_t b = __float_as_uint(x);
  nan = ((b & 0x7F800000u) == 0x7F800000u) && (b & 0x007FFFFFu);
  if ((b & 0x7FFFFFFFu) == 0u) b = 0u;  // -0 == +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Block-wide exclusive scan of a 0/1 flag (blockDim = 1024 = 32 warps).
__device__ __forceinline__ int block_excl_scan(bool flag, int& total, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xFFFFFFFFu, flag);
  const int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    int v = warp_tot[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    warp_tot[32 + lane] = incl - v;           // exclusive
    if (lane == 31) warp_tot[64] = incl;      // total
  }
  __syncthreads();
  const int r = warp_tot[32 + w] + in_warp;
  total = warp_tot[64];
  __syncthreads();
  return r;
}

// Block-wide exclusive scan of an int (blockDim = 1024): two barriers.
__device__ __forceinline__ int block_excl_scan_int(int v, int& total, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int x = warp_tot[lane];
    int wi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += t;
    }
    warp_tot[32 + lane] = wi - x;
    if (lane == 31) warp_tot[64] = wi;
  }
  __syncthreads();
  total = warp_tot[64];
  return warp_tot[32 + w] + incl - v;
}

// Segments of up to 1024 * E columns: thread t holds keys [t E, t E + E) in
// registers; 4 radix passes with warp-aggregated histograms, then ONE scan of
// the per-thread tie counts and ONE of the per-thread prune counts give every
// element its place (instead of two block scans per 1024 elements).  Same
// result as the general path: prune (score asc, index asc), S and P ascending.
template <int E>
__device__ __forceinline__ void select_regs(const SelectSeg& s, const float* __restrict__ sc, int32_t* K, int32_t* P,
                                            int32_t* Q, int32_t* err_flag, uint32_t* hist, int* warp_tot,
                                            uint32_t* sel) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int i0 = tid * E;
  uint32_t key[E];
  bool saw_nan = false;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    bool nan = false;
    key[e] = (i0 + e < s.len) ? ord32(__ldg(sc + i0 + e), nan) : 0u;
    saw_nan |= nan;
  }
  if (saw_nan) atomicOr(err_flag, 1);
  uint32_t prefix = 0, mask = 0;
  int target = s.n_prune - 1;
  if (s.n_prune > 0) {
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      if (tid < 256) hist[tid] = 0;
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const bool hit = i0 + e < s.len && (key[e] & mask) == prefix;
        const uint32_t bin = hit ? (key[e] >> shift) & 255u : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        if (hit && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
      }
      __syncthreads();
      if (tid < 32) {
        uint32_t loc[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          loc[j] = hist[8 * lane + j];
          sum += loc[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - sum;
        if ((uint32_t)target >= excl && (uint32_t)target < incl) {
          uint32_t c = excl;
          for (int j = 0; j < 8; ++j) {
            if ((uint32_t)target < c + loc[j]) {
              sel[0] = 8 * lane + j;
              sel[1] = c;
              break;
            }
            c += loc[j];
          }
        }
      }
      __syncthreads();
      prefix |= sel[0] << shift;
      mask |= 0xFFu << shift;
      target -= (int)sel[1];
    }
  }
  const uint32_t v = prefix;
  const int t_need = target + 1;
  const bool any = s.n_prune > 0;
  int c_tie = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) c_tie += (any && i0 + e < s.len && key[e] == v) ? 1 : 0;
  int tot;
  int tr = block_excl_scan_int(c_tie, tot, warp_tot);
  bool isp[E];
  int c_p = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool valid = i0 + e < s.len;
    const bool tie = any && valid && key[e] == v;
    isp[e] = any && valid && (key[e] < v || (tie && tr < t_need));
    tr += tie ? 1 : 0;
    c_p += isp[e] ? 1 : 0;
  }
  int pr = block_excl_scan_int(c_p, tot, warp_tot);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = i0 + e;
    if (i < s.len) {
      if (isp[e]) {
        P[pr] = i;
        if (Q) Q[i] = -1;
        ++pr;
      } else {
        K[i - pr] = i;
        if (Q) Q[i] = i - pr;
      }
    }
  }
  const int nk = s.len - s.n_prune;
  for (int a = tid; a < s.append; a += blockDim.x) {
    K[nk + a] = s.len + a;
    if (Q) Q[s.len + a] = nk + a;
  }
}

__global__ void __launch_bounds__(1024) ztp_select_kernel(const SelectParams p, const float* __restrict__ scores,
                                                          int32_t* __restrict__ kept, int32_t* __restrict__ pruned,
                                                          int32_t* __restrict__ pos, int32_t* err_flag) {
  pdl_wait();
  pdl_trigger();
  const SelectSeg s = p.seg[blockIdx.x];
  const float* sc = scores + s.score_off;
  if (s.len <= 8 * 1024) {
    __shared__ uint32_t rhist[256];
    __shared__ int rwarp[65];
    __shared__ uint32_t rsel[2];
    int32_t* Kr = kept + s.kept_off;
    int32_t* Pr = pruned + s.pruned_off;
    int32_t* Qr = pos ? pos + s.pos_off : nullptr;
    if (s.len <= 1024)
      select_regs<1>(s, sc, Kr, Pr, Qr, err_flag, rhist, rwarp, rsel);
    else if (s.len <= 2048)
      select_regs<2>(s, sc, Kr, Pr, Qr, err_flag, rhist, rwarp, rsel);
    else if (s.len <= 4096)
      select_regs<4>(s, sc, Kr, Pr, Qr, err_flag, rhist, rwarp, rsel);
    else
      select_regs<8>(s, sc, Kr, Pr, Qr, err_flag, rhist, rwarp, rsel);
    return;
  }
  // keys staged in shared memory once when the segment fits (every pass and
  // the compaction then read smem instead of re-reading L2)
  extern __shared__ uint32_t skey[];
  const bool staged = s.len <= p.smem_keys;
  bool saw_nan = false;
  if (staged) {
    for (int i = threadIdx.x; i < s.len; i += blockDim.x) {
      bool nan;
      skey[i] = ord32(sc[i], nan);
      saw_nan |= nan;
    }
    __syncthreads();
  }
  auto key_at = [&](int i, bool& nan) -> uint32_t {
    if (staged) {
      nan = false;
      return skey[i];
    }
    return ord32(sc[i], nan);
  };
  int32_t* K = kept + s.kept_off;
  int32_t* P = pruned + s.pruned_off;
  int32_t* Q = pos ? pos + s.pos_off : nullptr;
  __shared__ uint32_t hist[256];
  __shared__ int warp_tot[65];
  __shared__ uint32_t sel_bin, sel_below;
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  uint32_t prefix = 0, mask = 0;
  int target = s.n_prune - 1;  // 0-based rank (by key) of the last pruned element
  if (s.n_prune > 0) {
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      // warp-aggregated histogram: scores cluster in few exponent bins, so
      // lanes with the same bin add once (__match_any_sync) instead of
      // serialising on one shared-memory address
      for (int base = 0; base < s.len; base += blockDim.x) {
        const int i = base + tid;
        bool nan = false;
        const uint32_t key = i < s.len ? key_at(i, nan) : 0u;
        saw_nan |= nan;
        const bool hit = i < s.len && (key & mask) == prefix;
        const uint32_t bin = hit ? (key >> shift) & 255u : 256u;   // 256 = no bin
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        if (hit && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
      }
      __syncthreads();
      if (tid < 32) {
        // lane l owns bins 8l..8l+7
        uint32_t loc[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          loc[j] = hist[8 * lane + j];
          sum += loc[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - sum;
        if ((uint32_t)target >= excl && (uint32_t)target < incl) {
          uint32_t c = excl;
          for (int j = 0; j < 8; ++j) {
            if ((uint32_t)target < c + loc[j]) {
              sel_bin = 8 * lane + j;
              sel_below = c;
              break;
            }
            c += loc[j];
          }
        }
      }
      __syncthreads();
      prefix |= sel_bin << shift;
      mask |= 0xFFu << shift;
      target -= (int)sel_below;
      __syncthreads();
    }
  } else if (!staged) {
    for (int i = tid; i < s.len; i += blockDim.x) {
      bool nan;
      (void)ord32(sc[i], nan);
      saw_nan |= nan;
    }
  }
  if (saw_nan) atomicOr(err_flag, 1);
  const uint32_t v = prefix;          // key of the n_prune-th smallest
  const int t_need = target + 1;      // ties at v that are pruned (ascending index)

  int carry_tie = 0, carry_p = 0;
  for (int base = 0; base < s.len; base += blockDim.x) {
    const int i = base + tid;
    const bool valid = i < s.len;
    bool nan;
    const uint32_t key = valid ? key_at(i, nan) : 0u;
    const bool less = valid && s.n_prune > 0 && key < v;
    const bool tie = valid && s.n_prune > 0 && key == v;
    int tot_tie, tot_p;
    const int tie_rank = carry_tie + block_excl_scan(tie, tot_tie, warp_tot);
    const bool isp = less || (tie && tie_rank < t_need);
    const int p_rank = carry_p + block_excl_scan(isp, tot_p, warp_tot);
    if (valid) {
      if (isp)
        P[p_rank] = i;
      else
        K[i - p_rank] = i;
      if (Q) Q[i] = isp ? -1 : i - p_rank;
    }
    carry_tie += tot_tie;
    carry_p += tot_p;
  }
  const int nk = s.len - s.n_prune;
  for (int a = tid; a < s.append; a += blockDim.x) {
    K[nk + a] = s.len + a;
    if (Q) Q[s.len + a] = nk + a;
  }
}

cudaError_t select_launch(const SelectParams& p, const float* scores, int32_t* kept, int32_t* pruned, int32_t* pos,
                          int32_t* err_flag, cudaStream_t st) {
  SelectParams q = p;
  int maxlen = 0;
  for (int i = 0; i < p.nseg; ++i) maxlen = p.seg[i].len > maxlen ? p.seg[i].len : maxlen;
  // stage keys in smem up to 48K keys (192 KB); longer segments re-read L2
  q.smem_keys = (maxlen > 8 * 1024 && maxlen <= SELECT_SMEM_KEYS) ? maxlen : 0;   // <= 8K: register path
  const int smem = q.smem_keys * 4;
  // the opt-in covers dynamic + static shared memory: raise it for any staged
  // launch (a 12288-key segment is exactly 48 KB dynamic, over the default
  // 48 KB limit once the kernel's static arrays are added)
  if (smem > 0) {
    cudaError_t e = ensure_smem_optin((const void*)ztp_select_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_k(ztp_select_kernel, p.nseg, 1024, smem, st, q, scores, kept, pruned, pos, err_flag);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace ztp

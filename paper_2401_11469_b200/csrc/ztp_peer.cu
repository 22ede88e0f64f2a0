// Peer-memory data plane (a7 collectives, a8 migration) over a symmetric
// window: every rank cudaMallocs one window, exports its IPC handle, and maps
// every peer's window (NVLink P2P loads on an NVSwitch box; the same device
// across processes in the one-GPU tests).  Tensors allocated from the window
// with ztp_sym_alloc sit at the same offset on every rank, so a peer's copy of
// a tensor is  peer_base + (ptr - own_base).
//
// Synchronisation: CTA b of rank r pairs with CTA b of every other rank
// through per-(rank, CTA) flags in the window: each barrier round the CTA
// stores its epoch into flags[r][b] of every peer (release, system scope) and
// waits until flags[q][b] of its own window reach the epoch for all q
// (acquire).  Epochs live in device memory (one counter per CTA slot), so a
// captured CUDA graph replays correctly.  A barrier that waits > 10 s sets an
// error flag (reported by ztp_sync) instead of hanging.
//
// All-reduce (A-14: the straggler's imputed partial is what is
// summed): two-shot.  Phase 1: rank r sums chunk r of every rank's partial in
// rank order 0..e-1 in fp32 (the oracle's left fold) and writes
// it to its own buffer; phase 2: rank r pulls chunk q from rank q.  Peer
// traffic per rank: 2 (e-1)/e of the payload, the ring's bus bytes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ztp_internal.h"
#include "ztp_ptx.cuh"

namespace ztp {

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// 16-byte load that bypasses L1 (peer data written during this launch)
__device__ __forceinline__ int4 ld_cg(const int4* p) { return __ldcg(p); }

// One barrier round of CTA `b` across the ranks (see file comment).
__device__ void peer_barrier(const PeerWin& w, int b) {
  __threadfence_system();   // every thread's writes before the round are published
  __syncthreads();
  __shared__ uint32_t s_ep;
  if (threadIdx.x == 0) {
    s_ep = w.ep[b] + 1;
    w.ep[b] = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const int q = threadIdx.x;
  if (q < w.world) {
    st_release_sys(w.flags[q] + w.rank * PEER_MAX_CTAS + b, ep);
    const uint32_t* f = w.flags[w.rank] + q * PEER_MAX_CTAS + b;
    const uint64_t t0 = globaltimer();
    int spins = 0;
    while ((int32_t)(ld_acquire_sys(f) - ep) < 0) {
      if (++spins > 64) __nanosleep(128);
      if ((spins & 1023) == 0 && globaltimer() - t0 > 10ull * 1000000000ull) {
        atomicExch(w.err, 2);   // peer barrier timeout
        break;
      }
    }
  }
  __syncthreads();
}

struct Bf16x8Acc {
  float v[8];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.f;
  }
  __device__ void add(const int4& x) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] += f.x;
      v[2 * i + 1] += f.y;
    }
  }
  __device__ int4 pack() const {
    int4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    return o;
  }
};

// in-place all-reduce (sum) of `nvec` 16-byte vectors at window offset `off`
template <bool F32>
__global__ void __launch_bounds__(512) ztp_peer_allreduce(const PeerWin w, int64_t off, int64_t nvec) {
  pdl_wait();
  const int b = blockIdx.x, nb = gridDim.x;
  const int e = w.world, r = w.rank;
  const int64_t cv = (nvec + e - 1) / e;
  peer_barrier(w, b);                       // every rank's partial is complete
  {
    const int64_t c0 = (int64_t)r * cv, c1 = c0 + cv < nvec ? c0 + cv : nvec;
    int4* mine = reinterpret_cast<int4*>(w.base[r] + off);
    for (int64_t i = c0 + (int64_t)b * blockDim.x + threadIdx.x; i < c1; i += (int64_t)nb * blockDim.x) {
      if constexpr (F32) {
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < e; ++q) {   // rank order: ((p0 + p1) + p2) + ...
          const int4 x = ld_cg(reinterpret_cast<const int4*>(w.base[q] + off) + i);
          const float* f = reinterpret_cast<const float*>(&x);
#pragma unroll
          for (int k = 0; k < 4; ++k) a[k] += f[k];
        }
        int4 o;
        float* fo = reinterpret_cast<float*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) fo[k] = a[k];
        mine[i] = o;
      } else {
        Bf16x8Acc acc;
        acc.zero();
        for (int q = 0; q < e; ++q) acc.add(ld_cg(reinterpret_cast<const int4*>(w.base[q] + off) + i));
        mine[i] = acc.pack();
      }
    }
  }
  peer_barrier(w, b);                       // every chunk is reduced
  for (int q = 0; q < e; ++q) {
    if (q == r) continue;
    const int64_t c0 = (int64_t)q * cv, c1 = c0 + cv < nvec ? c0 + cv : nvec;
    const int4* src = reinterpret_cast<const int4*>(w.base[q] + off);
    int4* dst = reinterpret_cast<int4*>(w.base[r] + off);
    for (int64_t i = c0 + (int64_t)b * blockDim.x + threadIdx.x; i < c1; i += (int64_t)nb * blockDim.x)
      dst[i] = ld_cg(src + i);
  }
  peer_barrier(w, b);                       // no rank overwrites a chunk a peer still reads
  pdl_trigger();
}

// all-gather of equal blocks: rank q's block q (blk_vec vectors at off + q blk)
// is pulled into every rank's buffer
__global__ void __launch_bounds__(512) ztp_peer_allgather(const PeerWin w, int64_t off, int64_t blk_vec) {
  pdl_wait();
  const int b = blockIdx.x, nb = gridDim.x;
  peer_barrier(w, b);
  for (int q = 0; q < w.world; ++q) {
    if (q == w.rank) continue;
    const int4* src = reinterpret_cast<const int4*>(w.base[q] + off) + (int64_t)q * blk_vec;
    int4* dst = reinterpret_cast<int4*>(w.base[w.rank] + off) + (int64_t)q * blk_vec;
    for (int64_t i = (int64_t)b * blockDim.x + threadIdx.x; i < blk_vec; i += (int64_t)nb * blockDim.x)
      dst[i] = ld_cg(src + i);
  }
  peer_barrier(w, b);
  pdl_trigger();
}

// broadcast from `root`: every other rank pulls root's tensor (nvec 16-byte
// vectors at window offset `off`) into its own copy
__global__ void __launch_bounds__(512) ztp_peer_bcast(const PeerWin w, int root, int64_t off, int64_t nvec) {
  pdl_wait();
  const int b = blockIdx.x, nb = gridDim.x;
  peer_barrier(w, b);                       // root's tensor is final
  if (w.rank != root) {
    const int4* src = reinterpret_cast<const int4*>(w.base[root] + off);
    int4* dst = reinterpret_cast<int4*>(w.base[w.rank] + off);
    for (int64_t i = (int64_t)b * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)nb * blockDim.x)
      dst[i] = ld_cg(src + i);
  }
  peer_barrier(w, b);                       // the root's copy is not reused while a peer reads it
  pdl_trigger();
}

// reduce (sum) to `root`: root sums every rank's tensor in rank order 0..e-1
// in fp32 (the oracle's left fold) into its own copy
template <bool F32>
__global__ void __launch_bounds__(512) ztp_peer_reduce(const PeerWin w, int root, int64_t off, int64_t nvec) {
  pdl_wait();
  const int b = blockIdx.x, nb = gridDim.x;
  peer_barrier(w, b);                       // every rank's partial is complete
  if (w.rank == root) {
    int4* mine = reinterpret_cast<int4*>(w.base[root] + off);
    for (int64_t i = (int64_t)b * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)nb * blockDim.x) {
      if constexpr (F32) {
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < w.world; ++q) {
          const int4 x = ld_cg(reinterpret_cast<const int4*>(w.base[q] + off) + i);
          const float* f = reinterpret_cast<const float*>(&x);
#pragma unroll
          for (int k = 0; k < 4; ++k) a[k] += f[k];
        }
        int4 o;
        float* fo = reinterpret_cast<float*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) fo[k] = a[k];
        mine[i] = o;
      } else {
        Bf16x8Acc acc;
        acc.zero();
        for (int q = 0; q < w.world; ++q) acc.add(ld_cg(reinterpret_cast<const int4*>(w.base[q] + off) + i));
        mine[i] = acc.pack();
      }
    }
  }
  peer_barrier(w, b);                       // no rank overwrites its partial while the root reads it
  pdl_trigger();
}

// one-sided pulls of shard slices (ztp_migrate): every transfer whose
// destination is this rank reads the source rank's window at the source's
// symmetric offset; one warp per destination row.
__global__ void __launch_bounds__(256) ztp_peer_pull(const PeerWin w, const PeerPulls P) {
  pdl_wait();
  const int b = blockIdx.x, nb = gridDim.x;
  peer_barrier(w, b);                       // sources are final on every rank
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = 0; t < P.n; ++t) {
    const PeerPull& x = P.x[t];
    const char* src = w.base[x.src_rank] + x.src_off;
    for (int64_t row = (int64_t)b * nw + warp; row < x.nr; row += (int64_t)nb * nw) {
      const char* s = src + (row + x.r0) * x.ld_src * x.es + x.c0 * x.es;
      char* d = static_cast<char*>(x.dst) + (row + x.dr0) * x.ld_dst * x.es + x.dc0 * x.es;
      const int64_t nbytes = x.nc * x.es;
      if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | nbytes) & 15) == 0) {
        for (int64_t i = lane; i < nbytes / 16; i += 32)
          reinterpret_cast<int4*>(d)[i] = ld_cg(reinterpret_cast<const int4*>(s) + i);
      } else if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | nbytes) & 3) == 0) {
        for (int64_t i = lane; i < nbytes / 4; i += 32)
          reinterpret_cast<uint32_t*>(d)[i] = __ldcg(reinterpret_cast<const unsigned int*>(s) + i);
      } else {
        for (int64_t i = lane; i < nbytes / 2; i += 32)
          reinterpret_cast<uint16_t*>(d)[i] = __ldcg(reinterpret_cast<const unsigned short*>(s) + i);
      }
    }
  }
  peer_barrier(w, b);                       // no source changes while a peer still reads it
  pdl_trigger();
}

// statistics exchange (Alg.1 l.1 / Alg.2 l.2): my (T, M) into slot r of every
// rank's window stats area, then one barrier round
__global__ void ztp_peer_stats(const PeerWin w, double T, double M) {
  pdl_wait();
  if (threadIdx.x < w.world) {
    double* s = reinterpret_cast<double*>(w.base[threadIdx.x] + PEER_STATS_OFF);
    s[2 * w.rank] = T;
    s[2 * w.rank + 1] = M;
  }
  peer_barrier(w, 0);
}

__global__ void ztp_peer_barrier_kernel(const PeerWin w) {
  pdl_wait();
  peer_barrier(w, blockIdx.x);
  pdl_trigger();
}

}  // namespace

cudaError_t peer_allreduce_launch(const PeerWin& w, int64_t off, int64_t bytes, int f32, int nctas, cudaStream_t st) {
  const int64_t nvec = bytes / 16;
  if (f32) return launch_k(ztp_peer_allreduce<true>, nctas, 512, 0, st, w, off, nvec);
  return launch_k(ztp_peer_allreduce<false>, nctas, 512, 0, st, w, off, nvec);
}
cudaError_t peer_allgather_launch(const PeerWin& w, int64_t off, int64_t blk_bytes, int nctas, cudaStream_t st) {
  return launch_k(ztp_peer_allgather, nctas, 512, 0, st, w, off, blk_bytes / 16);
}
cudaError_t peer_bcast_launch(const PeerWin& w, int root, int64_t off, int64_t bytes, int nctas, cudaStream_t st) {
  return launch_k(ztp_peer_bcast, nctas, 512, 0, st, w, root, off, bytes / 16);
}
cudaError_t peer_reduce_launch(const PeerWin& w, int root, int64_t off, int64_t bytes, int f32, int nctas,
                               cudaStream_t st) {
  if (f32) return launch_k(ztp_peer_reduce<true>, nctas, 512, 0, st, w, root, off, bytes / 16);
  return launch_k(ztp_peer_reduce<false>, nctas, 512, 0, st, w, root, off, bytes / 16);
}
cudaError_t peer_pull_launch(const PeerWin& w, const PeerPulls& p, int nctas, cudaStream_t st) {
  return launch_k(ztp_peer_pull, nctas, 256, 0, st, w, p);
}
cudaError_t peer_stats_launch(const PeerWin& w, double T, double M, cudaStream_t st) {
  return launch_k(ztp_peer_stats, 1, 32, 0, st, w, T, M);
}
cudaError_t peer_barrier_launch(const PeerWin& w, int nctas, cudaStream_t st) {
  return launch_k(ztp_peer_barrier_kernel, nctas, 32, 0, st, w);
}

}  // namespace ztp

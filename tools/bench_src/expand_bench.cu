// Standalone A/B of column-spread (output-pruned dW) kernel variants at the
// c4 shapes: dst[r, j] = pos[j] >= 0 ? src[r, pos[j]] : 0, bf16, r < R, j < F.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o expand_bench expand_bench.cu
// Run on a B200: ./expand_bench   (prints us per launch and GB/s of algorithmic bytes)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
constexpr int CH = 1024;

// A: the library's kernel (warp per (row, 1024-col chunk), 2-byte gathers from global)
__global__ void __launch_bounds__(256) kA(const uint16_t* __restrict__ src, int64_t lds, uint16_t* __restrict__ dst,
                                          int64_t ldd, int n, const int32_t* __restrict__ pos, int F) {
  const int lane = threadIdx.x & 31;
  const int cpr = (F + CH - 1) / CH;
  const int64_t items = (int64_t)n * cpr, nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += nw) {
    const int r = (int)(it / cpr), c0 = (int)(it % cpr) * CH, c1 = min(F, c0 + CH), v1 = c0 + (c1 - c0) / 8 * 8;
    const uint16_t* s = src + (int64_t)r * lds;
    uint16_t* d = dst + (int64_t)r * ldd;
    auto pick = [&](int q) -> uint32_t { return q >= 0 ? (uint32_t)__ldg(s + q) : 0u; };
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) {
        int4 q0 = __ldg(reinterpret_cast<const int4*>(pos + c)), q1 = __ldg(reinterpret_cast<const int4*>(pos + c + 4));
        w[u] = make_uint4(pick(q0.x) | (pick(q0.y) << 16), pick(q0.z) | (pick(q0.w) << 16),
                          pick(q1.x) | (pick(q1.y) << 16), pick(q1.z) | (pick(q1.w) << 16));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + 8 * (lane + 32 * u);
      if (c < v1) *reinterpret_cast<uint4*>(d + c) = w[u];
    }
  }
}

// D: CTA per (R-row block, 1024-col chunk).  Chunk's pos -> smem as window
// offsets once; the R rows' compact windows [lo, hi] staged with 16-byte
// loads (all in flight); threads build 16-byte outputs from smem.
template <int R>
__global__ void __launch_bounds__(256) kD(const uint16_t* __restrict__ src, int64_t lds, uint16_t* __restrict__ dst,
                                          int64_t ldd, int n, const int32_t* __restrict__ pos, int F) {
  __shared__ __align__(16) uint16_t win[R][CH + 16];
  __shared__ int16_t off[CH];
  __shared__ int s_lo, s_hi;
  const int cpr = (F + CH - 1) / CH;
  const int rb = blockIdx.x / cpr, ck = blockIdx.x % cpr;
  const int c0 = ck * CH, c1 = min(F, c0 + CH);
  if (threadIdx.x == 0) { s_lo = 0x7fffffff; s_hi = -1; }
  __syncthreads();
  int lo = 0x7fffffff, hi = -1;
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const int q = __ldg(pos + c);
    if (q >= 0) { lo = min(lo, q); hi = max(hi, q); }
  }
  lo = __reduce_min_sync(~0u, lo); hi = __reduce_max_sync(~0u, hi);
  if ((threadIdx.x & 31) == 0) { atomicMin(&s_lo, lo); atomicMax(&s_hi, hi); }
  __syncthreads();
  const int base = s_hi >= 0 ? (s_lo & ~7) : 0;
  const int nv = s_hi >= 0 ? (s_hi - base) / 8 + 1 : 0;   // 16-byte vectors of the window
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const int q = __ldg(pos + c);
    off[c - c0] = (int16_t)(q >= 0 ? q - base : -1);
  }
  const int r0 = rb * R;
  for (int i = threadIdx.x; i < R * nv; i += blockDim.x) {
    const int rr = i / nv, v = i - rr * nv;
    if (r0 + rr < n)
      *reinterpret_cast<uint4*>(&win[rr][8 * v]) = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)(r0 + rr) * lds + base) + v);
  }
  __syncthreads();
  const int ng = (c1 - c0) / 8;   // F % 8 == 0 here
  for (int i = threadIdx.x; i < R * ng; i += blockDim.x) {
    const int rr = i / ng, g = i - rr * ng;
    if (r0 + rr >= n) continue;
    uint32_t x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { const int o = off[8 * g + e]; x[e] = o >= 0 ? win[rr][o] : 0u; }
    *reinterpret_cast<uint4*>(dst + (int64_t)(r0 + rr) * ldd + c0 + 8 * g) =
        make_uint4(x[0] | (x[1] << 16), x[2] | (x[3] << 16), x[4] | (x[5] << 16), x[6] | (x[7] << 16));
  }
}

// E: like D, but rows whose lineage says "pruned" (zero rows) write zeros without reading.
template <int R>
__global__ void __launch_bounds__(256) kE(const uint16_t* __restrict__ src, int64_t lds, uint16_t* __restrict__ dst,
                                          int64_t ldd, int n, const int32_t* __restrict__ pos, int F,
                                          const uint8_t* __restrict__ rowkept) {
  __shared__ __align__(16) uint16_t win[R][CH + 16];
  __shared__ int16_t off[CH];
  __shared__ int s_lo, s_hi;
  const int cpr = (F + CH - 1) / CH;
  const int rb = blockIdx.x / cpr, ck = blockIdx.x % cpr;
  const int c0 = ck * CH, c1 = min(F, c0 + CH);
  if (threadIdx.x == 0) { s_lo = 0x7fffffff; s_hi = -1; }
  __syncthreads();
  int lo = 0x7fffffff, hi = -1;
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const int q = __ldg(pos + c);
    if (q >= 0) { lo = min(lo, q); hi = max(hi, q); }
  }
  lo = __reduce_min_sync(~0u, lo); hi = __reduce_max_sync(~0u, hi);
  if ((threadIdx.x & 31) == 0) { atomicMin(&s_lo, lo); atomicMax(&s_hi, hi); }
  __syncthreads();
  const int base = s_hi >= 0 ? (s_lo & ~7) : 0;
  const int nv = s_hi >= 0 ? (s_hi - base) / 8 + 1 : 0;
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const int q = __ldg(pos + c);
    off[c - c0] = (int16_t)(q >= 0 ? q - base : -1);
  }
  const int r0 = rb * R;
  for (int i = threadIdx.x; i < R * nv; i += blockDim.x) {
    const int rr = i / nv, v = i - rr * nv;
    if (r0 + rr < n && rowkept[r0 + rr])
      *reinterpret_cast<uint4*>(&win[rr][8 * v]) = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)(r0 + rr) * lds + base) + v);
  }
  __syncthreads();
  const int ng = (c1 - c0) / 8;
  for (int i = threadIdx.x; i < R * ng; i += blockDim.x) {
    const int rr = i / ng, g = i - rr * ng;
    if (r0 + rr >= n) continue;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (rowkept[r0 + rr]) {
      uint32_t x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) { const int o = off[8 * g + e]; x[e] = o >= 0 ? win[rr][o] : 0u; }
      w = make_uint4(x[0] | (x[1] << 16), x[2] | (x[3] << 16), x[4] | (x[5] << 16), x[6] | (x[7] << 16));
    }
    *reinterpret_cast<uint4*>(dst + (int64_t)(r0 + rr) * ldd + c0 + 8 * g) = w;
  }
}

int main() {
  struct Case { const char* name; int R, F, ident; };   // ident: leading columns always kept (Q, K of dWqkv)
  const Case cases[] = {{"c4 dW1 (R=4096, F=11008)", 4096, 11008, 0}, {"c4 dWqkv (R=4096, F=12288)", 4096, 12288, 8192},
                        {"c5 dW1 (R=5120, F=20480)", 5120, 20480, 0}};
  std::mt19937 rng(7);
  for (const Case& cs : cases) {
    std::vector<int> pos(cs.F, -1);
    std::vector<int> cand;
    for (int j = cs.ident; j < cs.F; ++j) cand.push_back(j);
    std::shuffle(cand.begin(), cand.end(), rng);
    std::vector<char> keep(cs.F, 0);
    for (int j = 0; j < cs.ident; ++j) keep[j] = 1;
    for (size_t i = 0; i < cand.size() / 2; ++i) keep[cand[i]] = 1;
    int C = 0;
    for (int j = 0; j < cs.F; ++j) if (keep[j]) pos[j] = C++;
    std::vector<uint8_t> rk(cs.R);
    for (int r = 0; r < cs.R; ++r) rk[r] = (r * 7 + 3) % 2;   // half the rows kept
    const int64_t lds = (C + 7) / 8 * 8, ldd = cs.F;
    uint16_t *src, *dst; int32_t* dpos; uint8_t* drk; void* flush;
    CK(cudaMalloc(&src, (size_t)cs.R * lds * 2)); CK(cudaMalloc(&dst, (size_t)cs.R * ldd * 2));
    CK(cudaMalloc(&dpos, cs.F * 4)); CK(cudaMalloc(&drk, cs.R)); CK(cudaMalloc(&flush, 256 << 20));
    CK(cudaMemcpy(dpos, pos.data(), cs.F * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drk, rk.data(), cs.R, cudaMemcpyHostToDevice));
    CK(cudaMemset(src, 0x3f, (size_t)cs.R * lds * 2));
    const double bytes = (double)cs.R * C * 2 + (double)cs.R * cs.F * 2;   // read compact + write full
    const double bytesE = (double)cs.R / 2 * C * 2 + (double)cs.R * cs.F * 2;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](const char* nm, auto launch, double b) {
      float best = 1e9, sum = 0; int k = 0;
      for (int it = 0; it < 12; ++it) {
        CK(cudaMemsetAsync(flush, it, 256 << 20));   // evict L2
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2) { best = std::min(best, ms); sum += ms; ++k; }
      }
      CK(cudaGetLastError());
      printf("  %-34s mean %7.1f us  best %7.1f us  %6.0f GB/s (mean)\n", nm, sum / k * 1e3, best * 1e3, b / (sum / k * 1e-3) / 1e9);
    };
    printf("%s: compact %d of %d columns\n", cs.name, C, cs.F);
    const int cpr = (cs.F + CH - 1) / CH;
    time("A library (warp/item, global gathers)", [&] {
      const int64_t items = (int64_t)cs.R * cpr; const int bl = (int)std::min<int64_t>((items + 7) / 8, 148 * 8);
      kA<<<bl, 256>>>(src, lds, dst, ldd, cs.R, dpos, cs.F); }, bytes);
    time("D4 CTA (4 rows x chunk, smem)", [&] { kD<4><<<(cs.R / 4) * cpr, 256>>>(src, lds, dst, ldd, cs.R, dpos, cs.F); }, bytes);
    time("D8 CTA (8 rows x chunk, smem)", [&] { kD<8><<<(cs.R / 8) * cpr, 256>>>(src, lds, dst, ldd, cs.R, dpos, cs.F); }, bytes);
    time("D16 CTA (16 rows x chunk, smem)", [&] { kD<16><<<(cs.R / 16) * cpr, 256>>>(src, lds, dst, ldd, cs.R, dpos, cs.F); }, bytes);
    time("E8 D8 + zero rows not read", [&] { kE<8><<<(cs.R / 8) * cpr, 256>>>(src, lds, dst, ldd, cs.R, dpos, cs.F, drk); }, bytesE);
    time("copy (memcpy dst<-dst, same bytes)", [&] { CK(cudaMemcpyAsync(dst, dst + (size_t)cs.R * ldd / 2, (size_t)cs.R * ldd, cudaMemcpyDeviceToDevice)); }, (double)cs.R * ldd * 2);
    cudaFree(src); cudaFree(dst); cudaFree(dpos); cudaFree(drk); cudaFree(flush);
  }
  return 0;
}

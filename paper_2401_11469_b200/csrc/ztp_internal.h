// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <utility>

namespace ztp {

// Programmatic dependent launch (PDL) for every kernel of the path: the next
// kernel's CTAs start their prologue while this one drains; each kernel calls
// griddepcontrol.wait before touching memory (ztp_ptx.cuh pdl_wait).  Kept in
// CUDA graphs as programmatic edges.  ZTP_PDL=0 turns it off (A/B timing).
bool pdl_enabled();
// Every kernel launch of the library (all four launch sites) bumps this
// process-wide sequence: a GEMM may prefetch its A operand before its PDL wait
// only if the launch right before it (no other launch since) was a GEMM whose
// outputs are disjoint from that A (ztp_api.cu gemm, GemmParams::a_early).
inline std::atomic<uint64_t>& launch_seq() {
  static std::atomic<uint64_t> s{0};
  return s;
}
// ... and the sequence number of the last launch per stream: the kernel a
// launch on `st` is programmatically dependent on is the previous launch on
// `st` (other streams' launches do not matter for PDL).
struct StreamSeqs {
  std::mutex mu;
  cudaStream_t s[32];
  uint64_t seq[32];
  int n = 0;
};
inline StreamSeqs& stream_seqs() {
  static StreamSeqs x;
  return x;
}
inline void note_launch(cudaStream_t st) {
  const uint64_t q = launch_seq().fetch_add(1, std::memory_order_relaxed) + 1;
  StreamSeqs& x = stream_seqs();
  std::lock_guard<std::mutex> g(x.mu);
  for (int i = 0; i < x.n; ++i)
    if (x.s[i] == st) {
      x.seq[i] = q;
      return;
    }
  const int i = x.n < 32 ? x.n++ : (int)(q % 32);   // evicted streams read 0 (never a match)
  x.s[i] = st;
  x.seq[i] = q;
}
inline uint64_t last_launch_on(cudaStream_t st) {
  StreamSeqs& x = stream_seqs();
  std::lock_guard<std::mutex> g(x.mu);
  for (int i = 0; i < x.n; ++i)
    if (x.s[i] == st) return x.seq[i];
  return 0;
}
// launch_k_pdl(pdl = false): plain stream order.  Used where an early-
// launched elementwise kernel would occupy (squat) SMs while it waits: its
// CTAs would take the SMs a concurrent side-stream GEMM is waiting for.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  note_launch(st);
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  note_launch(st);
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Raise a kernel's dynamic shared-memory opt-in to >= bytes on the CURRENT
// device (function attributes are per device; cached per (device, kernel)).
cudaError_t ensure_smem_optin(const void* kernel, int bytes);

enum { KIND_FWD = 0, KIND_DX = 1, KIND_DW = 2 };
// EPI_GELU: out <- pre, out2 <- GeLU(pre).  EPI_GELU_D: out <- GeLU'(pre), out2 <- GeLU(pre).
// EPI_GELU_GRAD: out <- acc * GeLU'(aux).  EPI_MUL: out <- acc * aux (aux = GeLU'(pre)).
enum { EPI_NONE = 0, EPI_GELU = 1, EPI_GELU_GRAD = 2, EPI_GELU_D = 3, EPI_MUL = 4 };

constexpr int FLAG_NB = 64;   // column blocks (256 tokens) a flag slot covers
struct GemmParams {
  int M, N;            // output rows (M) and columns (N)
  int kdim;            // contraction length (FWD: n_kept; DX: n_out; DW: tokens)
  int n_kept;          // FWD: contraction rows; DX/DW: computed output rows (rest imputed)
  const int32_t* kept;    // FWD: contraction row list; DX/DW: row map of m < n_kept
  const int32_t* pruned;  // DX/DW: row map of m >= n_kept (Zero-imputed rows)
  int oob_row;         // a row index outside the gathered tensor (TMA zero fill)
  int epi;             // EPI_*
  __nv_bfloat16* out;
  int64_t ld_out;
  __nv_bfloat16* out2;  // EPI_GELU: GeLU(pre) (out holds pre)
  int64_t ld_out2;
  const __nv_bfloat16* aux;  // EPI_GELU_GRAD: pre-activation rows (row = output row, or m if aux_by_m)
  int64_t ld_aux;
  int aux_by_m;               // aux is compact (row m of the tile order) instead of at the output row
  const int32_t* out_pos;     // FWD: output row map (unit j -> row out_pos[j], dropped if < 0); NULL = identity
  unsigned long long* stamp;  // [start_min, end_max] %globaltimer of this launch (nullable)
  // split-K (set by gemm_launch): splits > 1 writes fp32 partials to ws and a
  // fixed-order reduce kernel applies the epilogue and the row map.
  int splits, kb_per_split;
  float* ws;
  int64_t ld_ws, ws_split_stride;
  int dbg;   // performance experiments only (ZTP_DEBUG_EPI): 1 skip stores, 2 skip the epilogue body
  int oob_out;   // a row index outside the output tensor (TMA stores skip it)
  int out_rows;  // rows of the output tensor(s)
  int out_dense; // the row map is the identity on m < M (set by the host): dense TMA box stores
  unsigned long long* prof_stamp;  // profiling: [max ~start, max end] %globaltimer (nullable)
  unsigned long long* cta_stamps;  // profiling mode 3: per CTA 8 %globaltimer stamps (CTA start, after the
                                   // PDL wait, first operand stage ready, last MMA commit, first accumulator
                                   // ready, last tile's stores issued, stores complete, CTA end) (nullable)
  const int32_t* col_pos;  // DW output pruning: full column j <- compact column col_pos[j] (< 0: Zero)
  int n_full;              // full output columns when col_pos is set (N = compact columns)
  int pdl_late;            // inputs do not depend on the preceding kernel: PDL wait deferred to exit
  int a_early;             // A is not written by the preceding kernel: the producer issues the first stages'
                           // A loads before the PDL wait (only B waits for the predecessor)
  // Tile-completion flags between consecutive GEMMs of a stream (ZTP_FLAGS):
  // a producer counts, per 256-column block of its output, the epilogue
  // warps whose stores of a tile are complete (fo_flags[nb] += 1 each, and
  // fo_target += fo_T once per launch: cumulative, never reset); a consumer
  // whose B operand is that output waits for fo_flags[nb] >= target before
  // loading B for a tile of column block nb, instead of the PDL wait.
  unsigned long long* fo_flags;
  unsigned long long* fo_target;
  unsigned long long fo_T;     // set by the launcher: units per column block x EPI_WARPS x CG
  int fo_nb;                   // column blocks of this launch
  const unsigned long long* fi_flags;
  const unsigned long long* fi_target;
  __nv_bfloat16* full_out; // DW output pruning without split-K: the epilogue writes compact columns to `out`
  int64_t ld_full;         // (a scratch) and the column spread writes full_out [out_rows, n_full]
  int cs;                  // DW cluster split-K: the `splits` K-slices of a tile run as one cluster and
                           // are reduced through distributed shared memory (no workspace, no reduce kernel)
  int spread;              // DW output pruning without split-K, written by the epilogue itself: each warp's
                           // staged 32 x 64 compact chunk goes out as the full-column row segments it owns
                           // (pruned units Zero) -- no scratch, no column-spread pass
  const int32_t* col_kept; // spread: compact column i -> full column col_kept[i] (ascending; col_pos inverse)
  int skip_zero;           // no all-pruned (Zero) units: the column-spread pass writes the Zero rows P itself
  int zero_generic;        // all-pruned units at a lineage row map written by generic 16-byte stores, not scatter4
  int tail_ok;             // FWD: the last partial round of tiles may run as 128-column halves (ZTP_OPT_TAIL_HALVES)
  int tail_r;              // set by the launcher: that many last tiles run as two halves each (0: off)
};
// Cluster split-K choice for a dW launch with `splits` K-slices: the split
// count to run as clusters (<= splits, cluster of cg x cs CTAs fits and every
// tile gets a co-resident cluster), or 0 when the mode does not apply.
int gemm_cluster_splits(int kind, int epi, int M, int N, int n_kept, int splits, int num_sms);

// Split-K choice for a launch and the fp32 workspace it needs (bytes).
int gemm_choose_splits(int kind, int M, int N, int kdim, int n_kept, int num_sms);
size_t gemm_ws_bytes(int kind, int M, int N, int n_kept, int splits);

// Operand tensors of one launch: row-major bf16 [rows, cols], pitch ld.
// *_gather: rows are fetched through the lineage list with TMA gather4;
// otherwise the tensor is compact (already row-selected) and loaded as boxes.
struct GemmOperands {
  const void* a;
  int64_t a_rows, a_cols, a_ld;
  bool a_gather;
  const void* b;
  int64_t b_rows, b_cols, b_ld;
  bool b_gather;
};

cudaError_t gemm_launch(int kind, const GemmOperands& o, GemmParams p, int num_sms, cudaStream_t st);
// A linear's dX (k0 = KIND_DX) and dW (k1 = KIND_DW) as ONE persistent launch
// (grouped, static LPT unit schedule), then their split-K reduces / column
// spreads.  Both must use the same CTA-group size and compact operands.  The
// unit schedule of a shape is built by the first (eager) call and cached;
// a cache miss during stream capture returns cudaErrorStreamCaptureUnsupported.
cudaError_t gemm_group_launch(int k0, const GemmOperands& o0, GemmParams p0, int k1, const GemmOperands& o1,
                              GemmParams p1, int num_sms, cudaStream_t st);
int gemm_choose_cg(int kind, int M, int n_kept);
bool gemm_group_pays(int M_dx, int N_dx, int kdim_dx, int n_kept_dx, int M_dw, int N_dw, int kdim_dw, int n_kept_dw,
                     int num_sms);
int gemm_group_splits(int M_dx, int N_dx, int kdim_dx, int n_kept_dx, int M_dw, int N_dw, int kdim_dw,
                      int n_kept_dw, int num_sms);

// fp32 verification GEMM (SIMT FFMA), same lineage semantics, fp32 tensors.
struct GemmParamsF32 {
  int kind, M, N, kdim, n_kept;
  int x_compact;            // X^T holds only the kept rows (row k / m instead of kept[.])
  int aux_by_m;
  const int32_t* out_pos;
  const int32_t* kept;
  const int32_t* pruned;
  const float* x;
  int64_t ld_x;
  const float* w;
  int64_t ld_w;
  const float* g;
  int64_t ld_g;
  float* out;
  int64_t ld_out;
  float* out2;
  int64_t ld_out2;
  const float* aux;
  int64_t ld_aux;
  int epi;
};
cudaError_t gemm_f32_launch(const GemmParamsF32& p, cudaStream_t st);

// Priority select (ztp_select.cu).
struct SelectSeg {
  int32_t len, n_prune, append;
  int32_t score_off, kept_off, pruned_off, pos_off;
};
constexpr int SELECT_MAX_SEGS = 64;
constexpr int SELECT_SMEM_KEYS = 48 * 1024;
struct SelectParams {
  int nseg;
  int smem_keys;   // segments up to this length stage their keys in shared memory (set by select_launch)
  SelectSeg seg[SELECT_MAX_SEGS];
};
cudaError_t select_launch(const SelectParams& p, const float* scores, int32_t* kept, int32_t* pruned, int32_t* pos,
                          int32_t* err_flag, cudaStream_t st);

// Straggler emulation (ztp_misc.cu).
cudaError_t delay_launch(unsigned long long* stamp, double chi, unsigned long long* acc_ns, cudaStream_t st);
cudaError_t stamp_reset_launch(unsigned long long* stamp, cudaStream_t st);
cudaError_t core_launch(int phase, const void* qkv, int64_t ld_qkv, void* ctx, int64_t ld_ctx, int64_t feat,
                        int64_t n_feat, int64_t N, int dtype, const int32_t* rows, int64_t n_v, int v_compact,
                        cudaStream_t st, bool pdl = true);
cudaError_t gather_rows_launch(const void* src, int64_t ld_src, const int32_t* idx, int n, int64_t cols, void* dst,
                               int64_t ld_dst, int dtype, cudaStream_t st);
cudaError_t gather_2d_launch(const void* src, int64_t ld_src, const int32_t* rows, int n, const int32_t* cols, int nc,
                             void* dst, int64_t ld_dst, cudaStream_t st);
// Batched compaction (ztp_prepare): dst[r, c] = src[rows ? rows[r] : r, cols ? cols[c] : c], bf16.
struct GatherJob {
  const uint16_t* src;
  int64_t ld_src;
  const int32_t* rows;   // nullable: identity
  const int32_t* cols;   // nullable: identity (16-byte vector copies)
  uint16_t* dst;
  int64_t ld_dst;
  int32_t n, nc;
  int64_t rbegin;        // first row of this job in the launch's row space
  int32_t src_cols;      // cols != NULL: logical width of the source rows (> every cols[c])
};
constexpr int GATHER_MAX_JOBS = 16;
struct GatherJobs {
  int njobs;
  int64_t total;         // rows over all jobs
  GatherJob job[GATHER_MAX_JOBS];
};
cudaError_t gather_multi_launch(const GatherJobs& j, cudaStream_t st);

// Average / Same imputation of rows P (NEXT-2): mode 1 = per-column
// mean over rows S of `out` (A-10), mode 2 = rows P copied from `hist` (A-11).
cudaError_t impute_rows_launch(void* out, int64_t ld, int64_t cols, const int32_t* kept, int nk, const int32_t* pruned,
                               int np, int mode, const void* hist, int64_t ld_hist, int dtype, void* ws,
                               cudaStream_t st);   // ws: cols floats (Average's column means)
// NEXT-1 column delta with carry-over (ztp_priority_update).
cudaError_t priority_update_launch(const void* w, int64_t ld_w, const void* w_old, int64_t ld_old, int64_t K,
                                   int64_t n, const int32_t* pos_prev, float* delta, int32_t* count_above,
                                   float theta, cudaStream_t st);
// out-of-place column spread over the lineage rows: for r = kept[i] (i < nk; kept NULL = identity)
// dst[r, j] = pos[j] >= 0 ? src[r, pos[j]] : 0, for r = pruned[i] (i < np) dst[r, :] = 0; j < n_full
cudaError_t expand_cols_launch(const void* src, int64_t ld_src, void* dst, int64_t ld_dst, const int32_t* kept,
                               int nk, const int32_t* pruned, int np, const int32_t* pos, int n_full,
                               cudaStream_t st);
// dst[i, r] = src[r, cols ? cols[i] : i], i < n, r < R (16-bit elements)
cudaError_t transpose_launch(const void* src, int64_t ld_src, int64_t R, const int32_t* cols, int64_t n, void* dst,
                             int64_t ld_dst, cudaStream_t st);
cudaError_t fill_rows_launch(void* out, int64_t ld, const int32_t* rows, int nrows, int64_t cols, int dtype,
                             cudaStream_t st);

// Peer-memory data plane (ztp_peer.cu): the symmetric window of every rank
// mapped into this process, per-(rank, CTA) barrier flags at its start.
constexpr int PEER_MAX_CTAS = 256;
constexpr int64_t PEER_FLAGS_OFF = 0;         // u32 flags[ZTP_MAX_RANKS][PEER_MAX_CTAS]
constexpr int64_t PEER_STATS_OFF = 8192;      // double stats[ZTP_MAX_RANKS][2]
constexpr int64_t PEER_RESERVED = 65536;      // ztp_sym_alloc starts here
struct PeerWin {
  int rank, world;
  char* base[8];         // window base of every rank, mapped here (base[rank] = own)
  uint32_t* flags[8];    // = base[q] + PEER_FLAGS_OFF
  uint32_t* ep;          // local: barrier epoch per CTA slot [PEER_MAX_CTAS]
  int32_t* err;          // local: 2 = peer barrier timeout
};
struct PeerPull {        // dst[dr0 +, dc0 +] <- window of src_rank at src_off [r0 +, c0 +], nr x nc elements
  int32_t src_rank, es;
  int64_t src_off, r0, c0, nr, nc, ld_src;
  void* dst;
  int64_t dr0, dc0, ld_dst;
};
constexpr int PEER_MAX_PULLS = 24;
struct PeerPulls {
  int n;
  PeerPull x[PEER_MAX_PULLS];
};
cudaError_t peer_allreduce_launch(const PeerWin& w, int64_t off, int64_t bytes, int f32, int nctas, cudaStream_t st);
cudaError_t peer_bcast_launch(const PeerWin& w, int root, int64_t off, int64_t bytes, int nctas, cudaStream_t st);
cudaError_t peer_reduce_launch(const PeerWin& w, int root, int64_t off, int64_t bytes, int f32, int nctas,
                               cudaStream_t st);
// dst += src (bf16 / f32 rows, fp32 add) and dst = sum of `nparts` row blocks of src (rank order)
cudaError_t accumulate_launch(void* dst, int64_t ld_dst, const void* src, int64_t ld_src, int64_t rows, int64_t cols,
                              int dtype, int nparts, int64_t part_stride, int overwrite, cudaStream_t st);
cudaError_t peer_allgather_launch(const PeerWin& w, int64_t off, int64_t blk_bytes, int nctas, cudaStream_t st);
cudaError_t peer_pull_launch(const PeerWin& w, const PeerPulls& p, int nctas, cudaStream_t st);
cudaError_t peer_stats_launch(const PeerWin& w, double T, double M, cudaStream_t st);
cudaError_t peer_barrier_launch(const PeerWin& w, int nctas, cudaStream_t st);

}  // namespace ztp

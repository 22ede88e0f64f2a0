// C ABI of libztp (include/ztp.h): context, select, resized linears with
// their collectives, stand-in core, migration, statistics, emulation.
// Host-side validation runs before anything is enqueued.
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ztp.h"
#include "ztp_internal.h"

namespace ztp {
thread_local std::string g_thread_err;
void set_thread_error(const std::string& msg) { g_thread_err = msg; }
}  // namespace ztp

struct LineageEntry {
  const int32_t* kept;
  const int32_t* pruned;
  int32_t nk, np;
};

struct ztp_ctx {
  int rank = 0, world = 1, device = 0, num_sms = 148;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // BWD: the dW GEMM runs on side_stream concurrently with the dX GEMM (they
  // are independent), so the two small-output GEMMs share the SMs
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_c = nullptr, ev_d = nullptr;
  int conc_bwd = 1;                    // ZTP_CONC (default 1): dW on the side stream, the SMs split by work
  // ZTP_DW_SHARE: weight of the dW GEMM's MMA work in that split.  dW carries
  // fixed costs dX does not (split-K partials + reduce, one unit per pair), so
  // it gets more SMs than its MMA share: 1.2 measured best (1.0 / 1.2 / 1.3 /
  // 1.4 / 1.5 / 1.6 / 0.8 swept, profiles/r01_dw_share_sweep_v*.txt)
  double dw_share = 1.2;
  int part_model = 1;                  // ZTP_PART: 0 work-proportional dX / dW partition, 1 wave-quantised
  double aux_weight = 1.0;             // ZTP_AUX_WEIGHT: dX work factor when its epilogue reads an aux operand
  // While a concurrent dW is pending, the (non-persistent) core kernel is
  // launched in plain stream order: under PDL its CTAs would sit resident on
  // every free SM waiting for the dX GEMM, and the side-stream dW GEMM could
  // not start on the SMs its predecessor frees (ZTP_SQUAT_GUARD=0: PDL anyway;
  // the same guard on the side stream's split-K reduces measured no better)
  int squat_guard = 1;
  // ZTP_GROUP: a linear's dX and dW as one grouped persistent launch on every
  // SM (ztp::gemm_group_launch) instead of two concurrent kernels (TP = 1 /
  // row layers; a col layer at TP > 1 keeps the concurrent pair so the dX
  // all-reduce overlaps its dW)
  // A-operand loads before the PDL wait when the preceding library launch was
  // a GEMM on the same stream whose outputs do not overlap A (ZTP_A_EARLY, default 1)
  int a_early = 1;
  int spread_epi = 0;         // output-pruned unsplit dW: column spread inside the GEMM epilogue (opt-in)
  int zero_generic = 1;       // Zero units at a lineage row map: generic stores instead of TMA scatter4
  int tail_halves = 1;        // FWD: a last round filling <= half the pairs runs as 128-column halves
  // MMA work queued on the side stream by a dw_side call and not yet part of
  // a dX / dW partition: work units, k-blocks per unit, CTA pairs it may use
  int side_bl_units = 0, side_bl_kps = 0, side_bl_pairs = 0;
  int64_t lg_id = -1;                  // ztp::launch_seq() right after the last eligible GEMM launch (-1: none)
  cudaStream_t lg_stream = nullptr;
  const char* lg_out[2] = {nullptr, nullptr};
  size_t lg_bytes[2] = {0, 0};
  int64_t lg_ld[2] = {0, 0}, lg_cols[2] = {0, 0};
  const char* lg_in[3] = {nullptr, nullptr, nullptr};   // its A, B and aux operands
  size_t lg_in_bytes[3] = {0, 0, 0};
  unsigned long long* lg_slot = nullptr;                // its tile-completion flag slot (nullptr: none)
  // Tile-completion flags between consecutive GEMMs of a stream (ZTP_FLAGS,
  // ZTP_OPT_FLAGS): slots of [target, FLAG_NB column-block counters],
  // cumulative (never reset), used round-robin
  // Each stream owns a partition of 16 slots (4 streams; further streams get
  // no flags), so two producers sharing a slot are always ordered on one
  // stream: a consumer's wait can only be on its own producer's tiles.
  int flags_opt = 0;
  static constexpr int FLAG_SLOTS = 64, FLAG_PART = 16;
  unsigned long long* d_tflags = nullptr;
  cudaStream_t flag_stream[FLAG_SLOTS / FLAG_PART] = {};
  int flag_next[FLAG_SLOTS / FLAG_PART] = {};
  int group_bwd = 0;                   // 0 never (default), 1 always, 2 small pairs only (measured: no net gain)
  int sm_cap = 0;                      // > 0: SMs a GEMM launch may use (concurrent dX / dW partition)
  bool side_pending = false;           // side-stream work not yet joined into a caller stream
  void* skws_side = nullptr;           // split-K partials of side-stream GEMMs
  size_t skws_side_cap = 0;
  std::string err;
  int64_t launches = 0;
  int32_t* d_flags = nullptr;               // [0]: NaN score seen
  unsigned long long* d_stamp = nullptr;    // [start_min, end_max]
  unsigned long long* d_gemm_ns = nullptr;  // accumulated GEMM (+delay) time
  double* d_stats = nullptr;                // 2 * world doubles
  double chi = 1.0;
  int stats = 0;
  std::map<std::pair<int, int>, LineageEntry> lineage;
  int32_t* d_iota = nullptr;
  int64_t iota_cap = 0;
  void* ws = nullptr;
  size_t ws_cap = 0;
  void* cws[2] = {nullptr, nullptr};   // compact-operand workspaces (x, w)
  size_t cws_cap[2] = {0, 0};
  int use_gather4 = 0;                 // 1: gather rows in the GEMM producer with TMA gather4
  int allow_splitk = 1;                // split-K for few-tile GEMMs (ZTP_SPLITK=0 disables)
  int dbg_epi = 0;                     // ZTP_DEBUG_EPI (performance experiments; results invalid)
  int dbg_skip = 0;                    // ZTP_DEBUG_SKIP bitmask (timing experiments only, results invalid):
                                       // 1 select, 2 compaction copies, 4 core, 16 GEMMs
  void* skws = nullptr;                // split-K fp32 partials
  void* xws[2] = {nullptr, nullptr};   // compact dW columns before the spread (main, side stream)
  void* mws[2] = {nullptr, nullptr};   // Average imputation's column means (main, side stream)
  size_t mws_cap[2] = {0, 0};
  size_t xws_cap[2] = {0, 0};
  size_t skws_cap = 0;
  // profiling (ztp_set_profile): event pairs around every kernel class
  struct ProfEv {
    cudaEvent_t a, b;
    int cat;
    double flops;
  };
  int prof_on = 0;
  unsigned long long* d_pstamp = nullptr;   // per-GEMM-launch kernel stamps while profiling
  int pstamp_used = 0;
  std::vector<double> pstamp_flops;         // algorithmic FLOPs of each stamped launch
  static constexpr int PSTAMP_CAP = 4096;
  static constexpr int CTASTAMP_LAUNCHES = 64, CTASTAMP_PER_LAUNCH = 160 * 8;   // mode 3: per-CTA stamps
  unsigned long long* d_ctastamp = nullptr;
  std::vector<ProfEv> prof;
  size_t prof_used = 0;
  // peer-memory data plane (ztp_window_*, ztp_sym_alloc; ztp_peer.cu)
  int transport = ZTP_TRANSPORT_NCCL;
  char* win = nullptr;                 // own symmetric window (cudaMalloc)
  size_t win_bytes = 0, win_used = 0;
  bool win_open = false;
  void* win_ipc[ZTP_MAX_RANKS] = {};   // peer windows opened through CUDA IPC (closed on destroy)
  ztp::PeerWin pw{};
  int peer_ctas = 32;                  // CTAs per peer collective (same on every rank)
  float* d_one = nullptr;              // NCCL barrier scratch
};

enum { PROF_GEMM = 0, PROF_OTHER = 1, PROF_COMM = 2 };

namespace {
int prof_begin(ztp_ctx* c, cudaStream_t st, int cat, double flops) {
  if (c->prof_on != 1) return -1;   // mode 2: kernel stamps only (capturable in CUDA graphs)
  if (c->prof_used == c->prof.size()) {
    ztp_ctx::ProfEv e{};
    if (cudaEventCreate(&e.a) != cudaSuccess || cudaEventCreate(&e.b) != cudaSuccess) return -1;
    c->prof.push_back(e);
  }
  const int i = (int)c->prof_used++;
  c->prof[i].cat = cat;
  c->prof[i].flops = flops;
  cudaEventRecord(c->prof[i].a, st);
  return i;
}
void prof_end(ztp_ctx* c, int i, cudaStream_t st) {
  if (i >= 0) cudaEventRecord(c->prof[i].b, st);
}
}  // namespace

namespace {

ztp_status fail(ztp_ctx* c, ztp_status s, const std::string& msg) {
  if (c) c->err = msg;
  ztp::set_thread_error(msg);
  return s;
}

#define CUDA_TRY(c, expr)                                                                  \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail(c, ZTP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_TRY(c, expr)                                                                  \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess) return fail(c, ZTP_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

std::string shp(const char* name, const ztp_mat& m) {
  char b[160];
  snprintf(b, sizeof b, "%s[%lld x %lld, ld %lld, %s]", name, (long long)m.rows, (long long)m.cols, (long long)m.ld,
           m.dtype == ZTP_F32 ? "f32" : "bf16");
  return b;
}

bool mat_ok(const ztp_mat& m) {
  if (!m.ptr || m.rows < 1 || m.cols < 1 || m.ld < m.cols) return false;
  if (m.dtype != ZTP_BF16 && m.dtype != ZTP_F32) return false;
  const int64_t align = m.dtype == ZTP_BF16 ? 8 : 4;
  if (m.ld % align != 0) return false;
  if (reinterpret_cast<uintptr_t>(m.ptr) % 16 != 0) return false;
  return true;
}

ztp_status ensure_iota(ztp_ctx* c, int64_t n) {
  if (n <= c->iota_cap) return ZTP_OK;
  int64_t cap = 1;
  while (cap < n) cap <<= 1;
  std::vector<int32_t> h(cap);
  for (int64_t i = 0; i < cap; ++i) h[i] = (int32_t)i;
  if (c->d_iota) cudaFree(c->d_iota);
  CUDA_TRY(c, cudaMalloc(&c->d_iota, cap * sizeof(int32_t)));
  CUDA_TRY(c, cudaMemcpy(c->d_iota, h.data(), cap * sizeof(int32_t), cudaMemcpyHostToDevice));
  c->iota_cap = cap;
  return ZTP_OK;
}

ztp_status ensure_ws(ztp_ctx* c, size_t bytes) {
  if (bytes <= c->ws_cap) return ZTP_OK;
  if (c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  CUDA_TRY(c, cudaMalloc(&c->ws, bytes));
  c->ws_cap = bytes;
  return ZTP_OK;
}

bool emulating(const ztp_ctx* c) { return c->chi > 1.0 || c->stats; }

// Stamp slot of a GEMM: the side stream (concurrent dW) has its own, so a
// slowed rank keeps the concurrent dX / dW schedule of an unslowed one.
unsigned long long* stamp_slot(ztp_ctx* c, cudaStream_t st) { return c->d_stamp + (st == c->side_stream ? 2 : 0); }

ztp_status after_gemm(ztp_ctx* c, cudaStream_t st) {
  if (!emulating(c)) return ZTP_OK;
  CUDA_TRY(c, ztp::delay_launch(stamp_slot(c, st), c->chi, c->d_gemm_ns, st));
  ++c->launches;
  return ZTP_OK;
}

ncclDataType_t nccl_type(int dtype) { return dtype == ZTP_F32 ? ncclFloat : ncclBfloat16; }

// Resolve the lineage entry: sel == NULL -> dense S = 0..K-1.
ztp_status resolve_sel(ztp_ctx* c, const ztp_sel* sel, int64_t K, const int32_t** kept, const int32_t** pruned,
                       int* nk, int* np) {
  if (sel == nullptr) {
    ztp_status s = ensure_iota(c, K);
    if (s != ZTP_OK) return s;
    *kept = c->d_iota;
    *pruned = nullptr;
    *nk = (int)K;
    *np = 0;
    return ZTP_OK;
  }
  if ((int64_t)sel->n_kept + sel->n_pruned != K)
    return fail(c, ZTP_ESHAPE,
                "lineage: n_kept + n_pruned = " + std::to_string(sel->n_kept + sel->n_pruned) + " != K = " +
                    std::to_string(K));
  if (sel->n_kept < 1) return fail(c, ZTP_EDEGENERATE, "lineage: nothing survives (#P >= K, S:64)");
  if (!sel->kept || (sel->n_pruned > 0 && !sel->pruned)) return fail(c, ZTP_EINVAL, "lineage: null index list");
  *kept = sel->kept;
  *pruned = sel->pruned;
  *nk = sel->n_kept;
  *np = sel->n_pruned;
  return ZTP_OK;
}

// Operand source of a GEMM: the full tensor (rows reached through the lineage
// list) or a compact tensor holding exactly the kept rows in lineage order.
struct Src {
  const ztp_mat* m;
  bool compact;
};

// Kernel parameters of one bf16 resized GEMM (operands, lineage, epilogue,
// split-K workspace).  force_splits > 0 overrides the split-K choice.
ztp_status gemm_build_bf16(ztp_ctx* c, int kind, Src A, Src B, int64_t n_out, const int32_t* kept,
                           const int32_t* pruned, int nk, const ztp_mat& out, const ztp_mat* out2, const ztp_mat* aux,
                           int aux_by_m, const int32_t* out_pos, int epi, cudaStream_t st, bool out_compact,
                           const int32_t* col_pos, int n_full, bool indep_of_prev, int M, int N, int kdim,
                           int force_splits, ztp::GemmOperands* po, ztp::GemmParams* pp,
                           const int32_t* col_kept = nullptr) {
  const ztp_mat& a = *A.m;
  const ztp_mat& b = *B.m;
  ztp::GemmOperands o{};
  o.a = a.ptr;
  o.a_ld = a.ld;
  o.a_gather = !A.compact;
  o.a_rows = A.compact ? nk : a.rows;
  o.a_cols = kind == ztp::KIND_DW ? a.cols : n_out;
  o.b = b.ptr;
  o.b_ld = b.ld;
  if (kind == ztp::KIND_FWD) {
    o.b_gather = !B.compact;
    o.b_rows = B.compact ? nk : b.rows;
    o.b_cols = b.cols;
  } else {
    o.b_gather = false;
    o.b_rows = n_out;
    o.b_cols = b.cols;
  }
  ztp::GemmParams p{};
  p.M = M;
  p.N = N;
  p.kdim = kdim;
  p.n_kept = nk;
  p.kept = kept;
  p.pruned = pruned;
  p.epi = epi;
  p.out = (__nv_bfloat16*)out.ptr;
  p.ld_out = out.ld;
  p.out_rows = (int)out.rows;
  if (out2 && out2->rows != out.rows)
    return fail(c, ZTP_ESHAPE, "gemm: " + shp("out2", *out2) + " must have the rows of " + shp("out", out));
  p.out2 = out2 ? (__nv_bfloat16*)out2->ptr : nullptr;
  p.ld_out2 = out2 ? out2->ld : 0;
  p.aux = aux ? (const __nv_bfloat16*)aux->ptr : nullptr;
  p.ld_aux = aux ? aux->ld : 0;
  p.aux_by_m = aux_by_m;
  p.out_pos = out_pos;
  // identity row map: compact outputs, or a dense lineage (S = 0..K-1)
  p.out_dense = out_compact || (kind == ztp::KIND_FWD ? out_pos == nullptr
                                                      : (kept == c->d_iota && pruned == nullptr && M <= nk));
  p.stamp = emulating(c) ? stamp_slot(c, st) : nullptr;
  p.dbg = c->dbg_epi;
  p.col_pos = col_pos;
  p.n_full = n_full;
  p.zero_generic = c->zero_generic;
  p.tail_ok = c->tail_halves;
  // early start (PDL wait at exit) only when nothing between the launches
  // depends on stamps (emulation) and the workspaces are disjoint (dW uses
  // its own split-K workspace)
  p.pdl_late = indep_of_prev && !emulating(c) && ztp::pdl_enabled();
  // split-K over the contraction when the output has too few tiles for 148 SMs
  const int nsm = c->sm_cap > 0 ? c->sm_cap : c->num_sms;
  p.splits = force_splits > 0 ? force_splits
                              : (c->allow_splitk ? ztp::gemm_choose_splits(kind, M, N, kdim, nk, nsm) : 1);
  if (p.splits > 1) {
    const int num_kb = (kdim + 63) / 64;
    // dW: the K-slices of a tile as one cluster reduced through DSMEM
    const int cs = force_splits > 0 ? 0 : ztp::gemm_cluster_splits(kind, epi, M, N, nk, p.splits, nsm);
    if (cs >= 2) p.splits = cs;
    p.kb_per_split = (num_kb + p.splits - 1) / p.splits;
    p.splits = (num_kb + p.kb_per_split - 1) / p.kb_per_split;
    p.cs = (cs >= 2 && p.splits == cs) ? cs : 0;
  }
  if (p.splits > 1 && p.cs > 1) {
    p.ws = nullptr;      // no workspace: partials never leave the cluster
  } else if (p.splits > 1) {
    const int num_kb = (kdim + 63) / 64;
    p.kb_per_split = (num_kb + p.splits - 1) / p.splits;
    p.splits = (num_kb + p.kb_per_split - 1) / p.kb_per_split;
    const size_t bytes = ztp::gemm_ws_bytes(kind, M, N, nk, p.splits);
    const bool side = st == c->side_stream || kind == ztp::KIND_DW;   // dW: its own workspace
    void*& wsp = side ? c->skws_side : c->skws;
    size_t& wcap = side ? c->skws_side_cap : c->skws_cap;
    if (wcap < bytes) {
      if (wsp) cudaFree(wsp);
      wsp = nullptr;
      wcap = 0;
      CUDA_TRY(c, cudaMalloc(&wsp, bytes));
      wcap = bytes;
    }
    p.ws = (float*)wsp;
    p.ld_ws = (N + 7) / 8 * 8;
    p.ws_split_stride = (int64_t)(kind == ztp::KIND_FWD ? M : std::min(M, nk)) * p.ld_ws;
  } else {
    p.splits = 1;
    p.kb_per_split = (kdim + 63) / 64;
  }
  if (col_pos && p.splits == 1 && c->spread_epi && col_kept) {
    // output pruning without split-K: the epilogue writes dW in full, its
    // kept columns from the staged tile and the Zero units in between
    p.spread = 1;
    p.col_kept = col_kept;
    p.full_out = p.out;
    p.ld_full = p.ld_out;
  } else if (col_pos && p.splits == 1) {
    // output pruning without split-K: the epilogue writes the compact
    // columns to a scratch (one per stream), the column spread writes dW in
    // full, Zero units included.  (Spreading inside the epilogue, by
    // row segments of full columns, measured slower: c4 step 0.87 -> 1.02 ms.)
    const int64_t ldc = (N + 7) / 8 * 8;
    const size_t bytes = (size_t)out.rows * ldc * 2;
    const int k = st == c->side_stream ? 1 : 0;
    if (c->xws_cap[k] < bytes) {
      if (c->xws[k]) cudaFree(c->xws[k]);
      c->xws[k] = nullptr;
      c->xws_cap[k] = 0;
      CUDA_TRY(c, cudaMalloc(&c->xws[k], bytes));
      c->xws_cap[k] = bytes;
    }
    p.full_out = p.out;
    p.ld_full = p.ld_out;
    p.out = (__nv_bfloat16*)c->xws[k];
    p.ld_out = ldc;
    p.skip_zero = 1;   // the spread writes the Zero rows P (no all-pruned units, no scratch reads for them)
  }
  *po = o;
  *pp = p;
  return ZTP_OK;
}

// Output rows M, columns N and contraction length of a GEMM of `kind`.
void gemm_dims(int kind, const ztp_mat& a, const ztp_mat& b, const ztp_mat& out, int64_t n_out, int nk, int* M,
               int* N, int* kdim) {
  if (kind == ztp::KIND_FWD) {
    *M = (int)n_out;
    *N = (int)b.cols;
    *kdim = nk;
  } else if (kind == ztp::KIND_DX) {
    *M = (int)out.rows;
    *N = (int)b.cols;
    *kdim = (int)n_out;
  } else {
    *M = (int)out.rows;
    *N = (int)n_out;
    *kdim = (int)a.cols;
  }
}

ztp_status gemm_check(ztp_ctx* c, int kind, Src A, Src B, int nk, const ztp_mat& out, const ztp_mat* out2,
                      const ztp_mat* aux) {
  const int dtype = A.m->dtype;
  const ztp_mat* need[3] = {A.m, B.m, &out};
  for (const ztp_mat* m : need)
    if (!mat_ok(*m) || m->dtype != dtype)
      return fail(c, ZTP_ESHAPE, "gemm: operand " + shp("m", *m) +
                                     " must be non-empty, 16-byte aligned with ld a multiple of 16 bytes, dtype "
                                     "matching");
  if (out2 && (!mat_ok(*out2) || out2->dtype != dtype)) return fail(c, ZTP_ESHAPE, "gemm: bad " + shp("out2", *out2));
  if (aux && (!mat_ok(*aux) || aux->dtype != dtype)) return fail(c, ZTP_ESHAPE, "gemm: bad " + shp("aux", *aux));
  if ((A.compact && A.m->rows < nk) || (kind == ztp::KIND_FWD && B.compact && B.m->rows < nk))
    return fail(c, ZTP_ESHAPE, "gemm: compact operand has fewer rows than n_kept");
  return ZTP_OK;
}

// One resized GEMM + (optional) emulated slowdown.
//   FWD: A = W^T source, B = X^T source     DX: A = W^T source, B = G^T
//   DW : A = X^T source, B = G^T
ztp_status gemm(ztp_ctx* c, int kind, Src A, Src B, int64_t n_out, const int32_t* kept, const int32_t* pruned,
                int nk, const ztp_mat& out, const ztp_mat* out2, const ztp_mat* aux, int aux_by_m,
                const int32_t* out_pos, int epi, cudaStream_t st, bool out_compact = false,
                const int32_t* col_pos = nullptr, int n_full = 0, bool indep_of_prev = false,
                const int32_t* col_kept = nullptr) {
  const int dtype = A.m->dtype;
  {
    const ztp_status cs = gemm_check(c, kind, A, B, nk, out, out2, aux);
    if (cs != ZTP_OK) return cs;
  }
  const ztp_mat& a = *A.m;
  const ztp_mat& b = *B.m;
  int M, N, kdim;
  gemm_dims(kind, a, b, out, n_out, nk, &M, &N, &kdim);
  const double tokens = (double)(kind == ztp::KIND_DW ? a.cols : b.cols);
  const int pe = prof_begin(c, st, PROF_GEMM, 2.0 * (double)nk * (double)n_out * tokens);
  if (dtype == ZTP_BF16) {
    ztp::GemmOperands o{};
    ztp::GemmParams p{};
    ztp_status bs = gemm_build_bf16(c, kind, A, B, n_out, kept, pruned, nk, out, out2, aux, aux_by_m, out_pos, epi, st,
                                    out_compact, col_pos, n_full, indep_of_prev, M, N, kdim, 0, &o, &p, col_kept);
    if (bs != ZTP_OK) return bs;
    if (c->prof_on && c->d_pstamp && c->pstamp_used < ztp_ctx::PSTAMP_CAP) {
      c->pstamp_flops.resize((size_t)c->pstamp_used + 1);
      c->pstamp_flops[c->pstamp_used] = 2.0 * (double)nk * (double)n_out * tokens;
      if (c->prof_on == 3 && c->d_ctastamp && c->pstamp_used < ztp_ctx::CTASTAMP_LAUNCHES)
        p.cta_stamps = c->d_ctastamp + (size_t)c->pstamp_used * ztp_ctx::CTASTAMP_PER_LAUNCH;
      p.prof_stamp = c->d_pstamp + 2 * (c->pstamp_used++);
    }
    const int nsm = c->sm_cap > 0 ? c->sm_cap : c->num_sms;
    // byte ranges this GEMM reads and writes
    const char* a0 = static_cast<const char*>(a.ptr);
    const size_t a_bytes = (size_t)(A.compact ? nk : a.rows) * a.ld * 2;
    const char* b0 = static_cast<const char*>(b.ptr);
    const int64_t b_rows = (kind == ztp::KIND_FWD && B.compact) ? nk : b.rows;
    const size_t b_bytes = (size_t)b_rows * b.ld * 2;
    const char* x0 = aux ? static_cast<const char*>(aux->ptr) : nullptr;
    const size_t x_bytes = aux ? (size_t)aux->rows * aux->ld * 2 : 0;
    const char* o0 = static_cast<const char*>(out.ptr);
    const size_t o_bytes = (size_t)out.rows * out.ld * 2;
    const char* o1 = out2 ? static_cast<const char*>(out2->ptr) : nullptr;
    const size_t o1_bytes = out2 ? (size_t)out2->rows * out2->ld * 2 : 0;
    auto ovl = [](const char* u, size_t nu, const char* v, size_t nv) { return u && v && u < v + nv && v < u + nu; };
    {
      // the previous launch on this stream -- the kernel this one is
      // programmatically dependent on -- is the GEMM recorded below (it
      // triggered this launch only after ITS predecessor completed)
      const bool chain = c->lg_id >= 0 && c->lg_stream == st && c->lg_id == (int64_t)ztp::last_launch_on(st) &&
                         !o.a_gather && !o.b_gather && !p.pdl_late;
      bool a_ok = chain;   // A untouched by that GEMM
      for (int k = 0; a_ok && k < 2; ++k)
        if (ovl(a0, a_bytes, c->lg_out[k], c->lg_bytes[k])) a_ok = false;
      // flag consumer: B is (a row range of) one of its outputs with the same
      // column origin and column blocks; nothing else read here is written
      // there, nothing written here is touched there
      int src = -1;
      if (chain && a_ok && c->flags_opt && c->lg_slot && kind != ztp::KIND_DW && p.cs <= 1)
        for (int k = 0; k < 2; ++k)
          if (c->lg_out[k] && b.ld == c->lg_ld[k] && b0 >= c->lg_out[k] &&
              b0 + b_bytes <= c->lg_out[k] + c->lg_bytes[k] && (size_t)(b0 - c->lg_out[k]) % (size_t)(b.ld * 2) == 0 &&
              b.cols <= c->lg_cols[k])
            src = k;
      bool fl = src >= 0;
      for (int k = 0; fl && k < 2; ++k)
        if (ovl(x0, x_bytes, c->lg_out[k], c->lg_bytes[k])) fl = false;
      for (int k = 0; fl && k < 3; ++k)
        if (ovl(o0, o_bytes, c->lg_in[k], c->lg_in_bytes[k]) || ovl(o1, o1_bytes, c->lg_in[k], c->lg_in_bytes[k]))
          fl = false;
      for (int k = 0; fl && k < 2; ++k)
        if (ovl(o0, o_bytes, c->lg_out[k], c->lg_bytes[k]) || ovl(o1, o1_bytes, c->lg_out[k], c->lg_bytes[k]))
          fl = false;
      if (fl) {
        p.fi_target = c->lg_slot;
        p.fi_flags = c->lg_slot + 1;
      }
      p.a_early = (c->a_early && a_ok && !fl) ? 1 : 0;
    }
    // a possible flag producer for the next GEMM of this stream (the launcher
    // drops the flags if its split-K / spread / width rules out a producer)
    const bool fprod = c->flags_opt && kind != ztp::KIND_DW && !p.pdl_late && !emulating(c) && p.splits == 1 &&
                       p.cs <= 1 && !p.col_pos && (N + 255) / 256 <= ztp::FLAG_NB;
    unsigned long long* slot = nullptr;
    if (fprod) {
      constexpr int NP = ztp_ctx::FLAG_SLOTS / ztp_ctx::FLAG_PART;
      int part = -1;
      for (int q = 0; q < NP && part < 0; ++q)
        if (c->flag_stream[q] == st && c->flag_next[q] > 0) part = q;
      for (int q = 0; q < NP && part < 0; ++q)
        if (c->flag_next[q] == 0) {
          part = q;
          c->flag_stream[q] = st;
        }
      if (part >= 0) {
        const int k = part * ztp_ctx::FLAG_PART + (c->flag_next[part]++ % ztp_ctx::FLAG_PART);
        slot = c->d_tflags + (size_t)k * (1 + ztp::FLAG_NB);
        p.fo_target = slot;
        p.fo_flags = slot + 1;
      }
    }
    const uint64_t seq0 = ztp::launch_seq().load();
    if (!(c->dbg_skip & 16)) CUDA_TRY(c, ztp::gemm_launch(kind, o, p, nsm, st));
    const bool extra = (p.splits > 1 && p.cs <= 1) || (p.col_pos && !p.spread);
    if (extra) ++c->launches;   // split-K reduce or column spread
    c->lg_id = -1;
    if (!extra && !p.pdl_late && !emulating(c) && ztp::launch_seq().load() == seq0 + 1) {   // exactly the GEMM
      // the launch the next GEMM may prefetch its A behind / wait on per column block
      c->lg_id = (int64_t)ztp::last_launch_on(st);
      c->lg_stream = st;
      c->lg_out[0] = o0;
      c->lg_bytes[0] = o_bytes;
      c->lg_ld[0] = out.ld;
      c->lg_cols[0] = out.cols;
      c->lg_out[1] = o1;
      c->lg_bytes[1] = o1_bytes;
      c->lg_ld[1] = out2 ? out2->ld : 0;
      c->lg_cols[1] = out2 ? out2->cols : 0;
      c->lg_in[0] = a0;
      c->lg_in_bytes[0] = a_bytes;
      c->lg_in[1] = b0;
      c->lg_in_bytes[1] = b_bytes;
      c->lg_in[2] = x0;
      c->lg_in_bytes[2] = x_bytes;
      c->lg_slot = slot;
    }
  } else {
    if (col_pos) return fail(c, ZTP_EUNSUPPORTED, "f32 path: output pruning");
    ztp::GemmParamsF32 p{};
    p.kind = kind;
    p.M = M;
    p.N = N;
    p.kdim = kdim;
    p.n_kept = nk;
    p.kept = kept;
    p.pruned = pruned;
    if (kind == ztp::KIND_FWD) {
      if (A.compact && kept != c->d_iota) return fail(c, ZTP_EUNSUPPORTED, "f32 path: compact weights");
      p.w = (const float*)a.ptr;
      p.ld_w = a.ld;
      p.x = (const float*)b.ptr;
      p.ld_x = b.ld;
      p.x_compact = B.compact ? 1 : 0;
    } else if (kind == ztp::KIND_DX) {
      if (A.compact && kept != c->d_iota) return fail(c, ZTP_EUNSUPPORTED, "f32 path: compact weights");
      p.w = (const float*)a.ptr;
      p.ld_w = a.ld;
      p.g = (const float*)b.ptr;
      p.ld_g = b.ld;
    } else {
      p.x = (const float*)a.ptr;
      p.ld_x = a.ld;
      p.x_compact = A.compact ? 1 : 0;
      p.g = (const float*)b.ptr;
      p.ld_g = b.ld;
    }
    if (out_compact) return fail(c, ZTP_EUNSUPPORTED, "f32 path: compact outputs");
    p.out = (float*)out.ptr;
    p.ld_out = out.ld;
    p.out2 = out2 ? (float*)out2->ptr : nullptr;
    p.ld_out2 = out2 ? out2->ld : 0;
    p.aux = aux ? (const float*)aux->ptr : nullptr;
    p.ld_aux = aux ? aux->ld : 0;
    p.aux_by_m = aux_by_m;
    p.out_pos = out_pos;
    p.epi = epi;
    CUDA_TRY(c, ztp::gemm_f32_launch(p, st));
  }
  ++c->launches;
  const ztp_status s = after_gemm(c, st);
  prof_end(c, pe, st);
  return s;
}

// A linear's dX and dW GEMMs as ONE grouped persistent launch (bf16): the
// two problems' work units share every CTA pair (ztp::gemm_group_launch).
// Returns ZTP_EUNSUPPORTED (nothing enqueued) when the pair does not qualify.
struct GemmSpec {
  int kind;
  Src A, B;
  int64_t n_out;
  const int32_t *kept, *pruned;
  int nk;
  ztp_mat out;
  const ztp_mat* aux;
  int aux_by_m, epi;
  bool out_compact;
  const int32_t* col_pos;
  int n_full;
  const int32_t* col_kept;
};
ztp_status gemm_group(ztp_ctx* c, const GemmSpec& x, const GemmSpec& w, cudaStream_t st) {
  for (const GemmSpec* g : {&x, &w}) {
    const ztp_status cs = gemm_check(c, g->kind, g->A, g->B, g->nk, g->out, nullptr, g->aux);
    if (cs != ZTP_OK) return cs;
    if (!g->A.compact || g->A.m->dtype != ZTP_BF16) return ZTP_EUNSUPPORTED;
  }
  int M0, N0, k0, M1, N1, k1;
  gemm_dims(x.kind, *x.A.m, *x.B.m, x.out, x.n_out, x.nk, &M0, &N0, &k0);
  gemm_dims(w.kind, *w.A.m, *w.B.m, w.out, w.n_out, w.nk, &M1, &N1, &k1);

  if (ztp::gemm_choose_cg(x.kind, M0, x.nk) != ztp::gemm_choose_cg(w.kind, M1, w.nk)) return ZTP_EUNSUPPORTED;
  const int sw = ztp::gemm_group_splits(M0, N0, k0, x.nk, M1, N1, k1, w.nk, c->num_sms);
  ztp::GemmOperands o0{}, o1{};
  ztp::GemmParams p0{}, p1{};
  ztp_status bs = gemm_build_bf16(c, x.kind, x.A, x.B, x.n_out, x.kept, x.pruned, x.nk, x.out, nullptr, x.aux,
                                  x.aux_by_m, nullptr, x.epi, st, x.out_compact, nullptr, 0, false, M0, N0, k0, 1, &o0,
                                  &p0);
  if (bs == ZTP_OK)
    bs = gemm_build_bf16(c, w.kind, w.A, w.B, w.n_out, w.kept, w.pruned, w.nk, w.out, nullptr, nullptr, 0, nullptr,
                         w.epi, st, false, w.col_pos, w.n_full, false, M1, N1, k1, sw, &o1, &p1, w.col_kept);
  if (bs != ZTP_OK) return bs;
  const double tok0 = (double)x.B.m->cols, tok1 = (double)w.A.m->cols;
  const double fl = 2.0 * x.nk * (double)x.n_out * tok0 + 2.0 * w.nk * (double)w.n_out * tok1;
  const int pe = prof_begin(c, st, PROF_GEMM, fl);
  if (c->prof_on && c->d_pstamp && c->pstamp_used < ztp_ctx::PSTAMP_CAP) {
    c->pstamp_flops.resize((size_t)c->pstamp_used + 1);
    c->pstamp_flops[c->pstamp_used] = fl;
    p0.prof_stamp = p1.prof_stamp = c->d_pstamp + 2 * (c->pstamp_used++);
  }
  if (!(c->dbg_skip & 16)) {
    const cudaError_t e = ztp::gemm_group_launch(x.kind, o0, p0, w.kind, o1, p1, c->num_sms, st);
    if (e == cudaErrorInvalidConfiguration) {   // too many units per pair: nothing enqueued, use the pair
      if (p0.prof_stamp) --c->pstamp_used;
      prof_end(c, pe, st);
      return ZTP_EUNSUPPORTED;
    }
    if (e == cudaErrorStreamCaptureUnsupported)
      return fail(c, ZTP_EUNSUPPORTED, "grouped dX/dW: unit schedule of this shape not built before capture "
                                       "(run the step once eagerly first)");
    CUDA_TRY(c, e);
  }
  c->launches += 1 + ((p1.splits > 1 || (p1.col_pos && !p1.spread)) ? 1 : 0) +
                 ((p0.splits > 1 || (p0.col_pos && !p0.spread)) ? 1 : 0);
  const ztp_status s = after_gemm(c, st);
  prof_end(c, pe, st);
  return s;
}

// Window offset of a tensor of `bytes` (peer transport): it must lie inside
// this rank's symmetric window, so every peer holds it at the same offset.
ztp_status win_offset(ztp_ctx* c, const void* p, size_t bytes, const char* what, int64_t* off) {
  if (!c->win_open) return fail(c, ZTP_EINVAL, std::string(what) + ": the peer transport needs ztp_window_open first");
  const char* q = static_cast<const char*>(p);
  if (q < c->win + ztp::PEER_RESERVED || q + bytes > c->win + c->win_bytes)
    return fail(c, ZTP_EINVAL, std::string(what) + ": tensor is not inside the symmetric window (ztp_sym_alloc)");
  *off = q - c->win;
  return ZTP_OK;
}

ztp_status allreduce(ztp_ctx* c, const ztp_mat& m, cudaStream_t st) {
  if (c->world == 1) return ZTP_OK;
  if (m.ld != m.cols) return fail(c, ZTP_ESHAPE, "all-reduce needs a contiguous tensor: " + shp("t", m));
  const size_t es = m.dtype == ZTP_F32 ? 4 : 2;
  const size_t bytes = (size_t)(m.rows * m.cols) * es;
  const int pe = prof_begin(c, st, PROF_COMM, 0.0);
  if (c->transport == ZTP_TRANSPORT_PEER) {
    int64_t off;
    ztp_status s = win_offset(c, m.ptr, bytes, "all-reduce", &off);
    if (s != ZTP_OK) return s;
    if (bytes % 16) return fail(c, ZTP_ESHAPE, "peer all-reduce: payload must be a multiple of 16 bytes");
    CUDA_TRY(c, ztp::peer_allreduce_launch(c->pw, off, (int64_t)bytes, m.dtype == ZTP_F32, c->peer_ctas, st));
    ++c->launches;
  } else {
    NCCL_TRY(c, ncclAllReduce(m.ptr, m.ptr, (size_t)(m.rows * m.cols), nccl_type(m.dtype), ncclSum, c->comm, st));
  }
  prof_end(c, pe, st);
  return ZTP_OK;
}

// In-place all-gather of `full` [world * blk_rows, cols] whose row block
// `rank` this rank has written (unpaired mode).
ztp_status allgather_rows(ztp_ctx* c, const ztp_mat& full, int64_t blk_rows, cudaStream_t st) {
  if (c->world == 1) return ZTP_OK;
  if (full.ld != full.cols) return fail(c, ZTP_ESHAPE, "all-gather needs a contiguous tensor: " + shp("t", full));
  const size_t es = full.dtype == ZTP_F32 ? 4 : 2;
  const size_t blk = (size_t)(blk_rows * full.cols) * es;
  const int pe = prof_begin(c, st, PROF_COMM, 0.0);
  if (c->transport == ZTP_TRANSPORT_PEER) {
    int64_t off;
    ztp_status s = win_offset(c, full.ptr, blk * c->world, "all-gather", &off);
    if (s != ZTP_OK) return s;
    if (blk % 16) return fail(c, ZTP_ESHAPE, "peer all-gather: block must be a multiple of 16 bytes");
    CUDA_TRY(c, ztp::peer_allgather_launch(c->pw, off, (int64_t)blk, c->peer_ctas, st));
    ++c->launches;
  } else {
    char* base = static_cast<char*>(full.ptr);
    NCCL_TRY(c, ncclAllGather(base + c->rank * blk, base, (size_t)(blk_rows * full.cols), nccl_type(full.dtype),
                              c->comm, st));
  }
  prof_end(c, pe, st);
  return ZTP_OK;
}

// Compact copy of the kept rows of `full` into `dst` (caller buffer or ctx
// workspace slot `slot`).  Returns the compact matrix in *out.
ztp_status compact_rows(ztp_ctx* c, const ztp_mat& full, const int32_t* kept, int nk, const ztp_mat& dst_in,
                        int slot, ztp_mat* out, cudaStream_t st) {
  ztp_mat d = dst_in;
  if (!d.ptr) {
    const size_t es = full.dtype == ZTP_F32 ? 4 : 2;
    const int64_t ld = (full.cols + 7) / 8 * 8;
    const size_t bytes = ((size_t)nk * ld * es + 1023) & ~size_t(1023);
    if (c->cws_cap[slot] < bytes) {
      if (c->cws[slot]) cudaFree(c->cws[slot]);
      c->cws[slot] = nullptr;
      c->cws_cap[slot] = 0;
      CUDA_TRY(c, cudaMalloc(&c->cws[slot], bytes));
      c->cws_cap[slot] = bytes;
    }
    d = ztp_mat{c->cws[slot], nk, full.cols, ld, full.dtype, 0};
  }
  if (!mat_ok(d) || d.rows < nk || d.cols < full.cols || d.dtype != full.dtype)
    return fail(c, ZTP_ESHAPE, "compact buffer " + shp("dst", d) + " too small for " + shp("src", full));
  const int pe = prof_begin(c, st, PROF_OTHER, 0.0);
  if (!(c->dbg_skip & 2))
    CUDA_TRY(c, ztp::gather_rows_launch(full.ptr, full.ld, kept, nk, full.cols, d.ptr, d.ld, full.dtype, st));
  prof_end(c, pe, st);
  ++c->launches;
  d.rows = nk;
  d.cols = full.cols;
  *out = d;
  return ZTP_OK;
}

// W^T[S, S'] (rows = this layer's kept S, or all rows when dense; columns =
// the consumer's kept S') into ws_t or ctx workspace slot 1 (output pruning).
// BWD (refill = false) reuses the copy FWD wrote into a caller ws_t.
ztp_status weight_2d(ztp_ctx* c, const ztp_mat& w, const int32_t* rows, int nk, const int32_t* cols, int n_y,
                     const ztp_mat& cbuf, bool refill, ztp_mat* tmp, Src* out, cudaStream_t st) {
  ztp_mat d = cbuf;
  if (d.ptr) {
    if (!mat_ok(d) || d.rows < nk || d.cols < n_y || d.dtype != w.dtype)
      return fail(c, ZTP_ESHAPE, "out_sel: compact weight " + shp("ws_t", d) + " needs [" + std::to_string(nk) +
                                     ", " + std::to_string(n_y) + "]");
  } else {
    const int64_t ld = (n_y + 7) / 8 * 8;
    const size_t bytes = ((size_t)nk * ld * 2 + 1023) & ~size_t(1023);
    if (c->cws_cap[1] < bytes) {
      if (c->cws[1]) cudaFree(c->cws[1]);
      c->cws[1] = nullptr;
      c->cws_cap[1] = 0;
      CUDA_TRY(c, cudaMalloc(&c->cws[1], bytes));
      c->cws_cap[1] = bytes;
    }
    d = ztp_mat{c->cws[1], nk, n_y, ld, w.dtype, 0};
    refill = true;
  }
  d.rows = nk;
  d.cols = n_y;
  if (refill) {
    const int pe = prof_begin(c, st, PROF_OTHER, 0.0);
    if (!(c->dbg_skip & 2)) CUDA_TRY(c, ztp::gather_2d_launch(w.ptr, w.ld, rows, nk, cols, n_y, d.ptr, d.ld, st));
    prof_end(c, pe, st);
    ++c->launches;
  }
  *tmp = d;
  *out = Src{tmp, true};
  return ZTP_OK;
}

// Average / Same imputation of rows P of a BWD output (NEXT-2; A-10,
// A-11) after the GEMM wrote rows S (and Zero rows P).
ztp_status impute(ztp_ctx* c, int policy, const ztp_mat& out, int64_t cols, const int32_t* kept, int nk,
                  const int32_t* pruned, int np, const ztp_mat* hist, cudaStream_t st) {
  if (policy == ZTP_IMPUTE_ZERO || np <= 0) return ZTP_OK;
  if (policy == ZTP_IMPUTE_SAME) {
    if (!hist || !hist->ptr) return fail(c, ZTP_EHISTORY, "Same imputation needs the previous step's values (S:74)");
    if (!mat_ok(*hist) || hist->rows != out.rows || hist->cols < cols || hist->dtype != out.dtype)
      return fail(c, ZTP_ESHAPE, "Same imputation: " + shp("hist", *hist) + " vs " + shp("out", out));
  }
  void* means = nullptr;
  if (policy == ZTP_IMPUTE_AVERAGE) {   // column means (fp32), a workspace per stream
    const int k = st == c->side_stream ? 1 : 0;
    const size_t bytes = (size_t)cols * sizeof(float);
    if (c->mws_cap[k] < bytes) {
      if (c->mws[k]) cudaFree(c->mws[k]);
      c->mws[k] = nullptr;
      c->mws_cap[k] = 0;
      CUDA_TRY(c, cudaMalloc(&c->mws[k], bytes));
      c->mws_cap[k] = bytes;
    }
    means = c->mws[k];
  }
  const int pe = prof_begin(c, st, PROF_OTHER, 0.0);
  CUDA_TRY(c, ztp::impute_rows_launch(out.ptr, out.ld, cols, kept, nk, pruned, np,
                                      policy == ZTP_IMPUTE_AVERAGE ? 1 : 2, hist ? hist->ptr : nullptr,
                                      hist ? hist->ld : 0, out.dtype, means, st));
  prof_end(c, pe, st);
  c->launches += policy == ZTP_IMPUTE_AVERAGE ? 2 : 1;
  return ZTP_OK;
}

enum { LAYER_COL = 0, LAYER_ROW = 1 };

// Source of the weight (or input) operand for this call.
ztp_status operand_src(ztp_ctx* c, bool dense_sel, bool caller_compact, const ztp_mat& full, const ztp_mat& cbuf,
                       bool refill, const int32_t* kept, int nk, int slot, ztp_mat* tmp, Src* out, cudaStream_t st) {
  if (dense_sel) {
    *out = Src{&full, true};
    return ZTP_OK;
  }
  if (caller_compact) {
    *out = Src{&full, true};
    return ZTP_OK;
  }
  if (full.dtype == ZTP_F32 || c->use_gather4) {
    *out = Src{&full, false};
    return ZTP_OK;
  }
  if (!refill && cbuf.ptr) {  // BWD: reuse the compact copy written by FWD (same lineage entry)
    *tmp = cbuf;
    tmp->rows = nk;
    *out = Src{tmp, true};
    return ZTP_OK;
  }
  ztp_status s = compact_rows(c, full, kept, nk, cbuf, slot, tmp, st);
  if (s != ZTP_OK) return s;
  *out = Src{tmp, true};
  return ZTP_OK;
}

ztp_status join_side(ztp_ctx* c, cudaStream_t st) {
  if (c->side_pending) {
    CUDA_TRY(c, cudaEventRecord(c->ev_d, c->side_stream));
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_d, 0));
    c->side_pending = false;
  }
  c->side_bl_units = c->side_bl_kps = c->side_bl_pairs = 0;
  return ZTP_OK;
}

ztp_status linear_impl(ztp_ctx* c, int layer, ztp_phase phase, const ztp_linear_args* a, cudaStream_t st);

ztp_mat row_block(const ztp_mat& m, int64_t r0, int64_t nr) {
  ztp_mat o = m;
  const size_t es = m.dtype == ZTP_F32 ? 4 : 2;
  o.ptr = static_cast<char*>(m.ptr) + (size_t)(r0 * m.ld) * es;
  o.rows = nr;
  return o;
}

// Unpaired mode (a column-parallel FWD whose output is needed whole,
// a row-parallel layer whose input is not split): the rank computes its row
// block of the full tensor and an all-gather completes it.
//   col FWD gather_output: y_t is [world n_out, N]; rows [rank n_out, ...) are
//     this rank's outputs, then all-gather of y_t.
//   row input_is_parallel = 0: x_t (and pre_in_t) are the full input [world K,
//     N], the rank uses rows [rank K, ...); BWD dx_t is [world K, N], the rank
//     computes its block (imputed rows P included, A-14), then all-gather.
ztp_status linear(ztp_ctx* c, int layer, ztp_phase phase, const ztp_linear_args* a, cudaStream_t st) {
  if (!c || !a) return fail(c, ZTP_EINVAL, "linear: null ctx/args");
  const bool gat = layer == LAYER_COL && a->gather_output;
  const bool unsplit_in = layer == LAYER_ROW && !a->input_is_parallel;
  if (!gat && !unsplit_in) return linear_impl(c, layer, phase, a, st);
  if (a->skip_collective) return fail(c, ZTP_EINVAL, "unpaired all-gather mode with skip_collective");
  if (a->out_sel || a->y_pos || a->x_compact || a->dx_compact || a->impute == ZTP_IMPUTE_SAME)
    return fail(c, ZTP_EUNSUPPORTED, "unpaired all-gather mode: no out_sel / y_pos / compact operands / Same");
  if (!mat_ok(a->w_t)) return fail(c, ZTP_ESHAPE, "linear: bad " + shp("w_t", a->w_t));
  ztp_linear_args b = *a;
  b.gather_output = 0;
  b.input_is_parallel = 1;
  const int e = c->world, r = c->rank;
  if (gat && phase == ZTP_BWD) {   // the gradient of a gathered output: this rank's row block of g_t
    const int64_t n_out = a->n_out > 0 ? a->n_out : a->w_t.cols;
    if (!mat_ok(a->g_t) || a->g_t.rows != e * n_out)
      return fail(c, ZTP_ESHAPE, "gather_output BWD: " + shp("g_t", a->g_t) + " must have world x n_out rows");
    b.g_t = row_block(a->g_t, r * n_out, n_out);
    return linear_impl(c, layer, phase, &b, st);
  }
  if (gat) {
    const int64_t n_out = a->n_out > 0 ? a->n_out : a->w_t.cols;
    if (!mat_ok(a->y_t) || a->y_t.rows != e * n_out)
      return fail(c, ZTP_ESHAPE, "gather_output: " + shp("y_t", a->y_t) + " must have world x n_out rows");
    b.y_t = row_block(a->y_t, r * n_out, n_out);
    ztp_status s = linear_impl(c, layer, phase, &b, st);
    if (s != ZTP_OK) return s;
    return allgather_rows(c, a->y_t, n_out, st);
  }
  const int64_t K = a->w_t.rows;
  if (!mat_ok(a->x_t) || a->x_t.rows != e * K)
    return fail(c, ZTP_ESHAPE, "input_is_parallel = 0: " + shp("x_t", a->x_t) + " must have world x K rows");
  b.x_t = row_block(a->x_t, r * K, K);
  if (a->pre_in_t.ptr) {
    if (a->pre_in_t.rows != e * K) return fail(c, ZTP_ESHAPE, "input_is_parallel = 0: " + shp("pre_in_t", a->pre_in_t));
    b.pre_in_t = row_block(a->pre_in_t, r * K, K);
  }
  if (phase == ZTP_BWD && a->dx_t.ptr) {
    if (!mat_ok(a->dx_t) || a->dx_t.rows != e * K)
      return fail(c, ZTP_ESHAPE, "input_is_parallel = 0: " + shp("dx_t", a->dx_t) + " must have world x K rows");
    b.dx_t = row_block(a->dx_t, r * K, K);
  }
  ztp_status s = linear_impl(c, layer, phase, &b, st);
  if (s != ZTP_OK) return s;
  if (phase == ZTP_BWD && a->dx_t.ptr) return allgather_rows(c, a->dx_t, K, st);
  return ZTP_OK;
}

ztp_status linear_impl(ztp_ctx* c, int layer, ztp_phase phase, const ztp_linear_args* a, cudaStream_t st) {
  if (phase == ZTP_FWD) {
    ztp_status js = join_side(c, st);   // a new step: earlier concurrent dW work is ordered before it
    if (js != ZTP_OK) return js;
  }
  const char* nm = layer == LAYER_COL ? "ztp_col_linear" : "ztp_row_linear";
  if (!mat_ok(a->w_t)) return fail(c, ZTP_ESHAPE, std::string(nm) + ": bad " + shp("w_t", a->w_t));
  const int64_t K = a->w_t.rows;
  const int64_t n_out = a->n_out > 0 ? a->n_out : a->w_t.cols;
  if (n_out > a->w_t.cols) return fail(c, ZTP_ESHAPE, std::string(nm) + ": n_out > w_t.cols");
  if (a->impute < ZTP_IMPUTE_ZERO || a->impute > ZTP_IMPUTE_SAME)
    return fail(c, ZTP_EINVAL, std::string(nm) + ": unknown imputation policy " + std::to_string(a->impute));
  if (a->impute != ZTP_IMPUTE_ZERO && (a->dx_compact || a->out_sel))
    return fail(c, ZTP_EUNSUPPORTED, std::string(nm) + ": dx_compact / out_sel imply Zero imputation (A-35)");
  const int dtype = a->w_t.dtype;
  const int32_t* kept;
  const int32_t* pruned;
  int nk, np;
  ztp_status s = resolve_sel(c, a->sel, K, &kept, &pruned, &nk, &np);
  if (s != ZTP_OK) return s;
  const bool dense_sel = a->sel == nullptr;
  // output pruning: only the consumer's kept outputs S' are computed / consumed
  const ztp_sel* os = a->out_sel;
  int64_t n_y = n_out;
  if (os) {
    if (dtype != ZTP_BF16) return fail(c, ZTP_EUNSUPPORTED, std::string(nm) + ": out_sel needs bf16");
    if ((int64_t)os->n_kept + os->n_pruned != n_out)
      return fail(c, ZTP_ESHAPE, std::string(nm) + ": out_sel n_kept + n_pruned != n_out " + std::to_string(n_out));
    if (os->n_kept < 1) return fail(c, ZTP_EDEGENERATE, std::string(nm) + ": out_sel keeps no output");
    if (!os->kept || !a->y_pos) return fail(c, ZTP_EINVAL, std::string(nm) + ": out_sel needs its kept list and y_pos");
    n_y = os->n_kept;
  }
  const bool dxc = a->dx_compact != 0 && !dense_sel;
  const std::pair<int, int> key = a->sel ? std::make_pair(a->sel->layer_id, a->sel->matrix_id) : std::make_pair(-1, -1);
  const bool xc = a->x_compact != 0;
  const int64_t x_rows_need = xc ? nk : K;
  ztp_mat tmpx{}, tmpw{};
  Src X{nullptr, false}, W{nullptr, false};

  if (phase == ZTP_FWD) {
    const ztp_mat& x = a->x_t;
    if (!mat_ok(x) || x.rows < x_rows_need || x.dtype != dtype || (!xc && x.rows != K))
      return fail(c, ZTP_ESHAPE, std::string(nm) + " FWD: " + shp("x_t", x) + " vs " + shp("w_t", a->w_t) +
                                     (xc ? " (compact x: needs n_kept rows)" : ""));
    const int64_t N = x.cols;
    const bool act = a->act == ZTP_ACT_GELU || a->act == ZTP_ACT_GELU_D;
    const int act_epi = a->act == ZTP_ACT_GELU_D ? ztp::EPI_GELU_D : ztp::EPI_GELU;
    const int64_t out_rows_need = os ? n_y : (a->y_pos ? 1 : n_out);
    if (!mat_ok(a->y_t) || a->y_t.rows < out_rows_need || a->y_t.cols != N || a->y_t.dtype != dtype)
      return fail(c, ZTP_ESHAPE, std::string(nm) + " FWD: " + shp("y_t", a->y_t) + " for n_out " + std::to_string(n_out));
    if (dtype == ZTP_BF16 && N % 8 != 0) return fail(c, ZTP_ESHAPE, "tokens N must be a multiple of 8");
    if (act && (!mat_ok(a->pre_t) || a->pre_t.rows < out_rows_need || a->pre_t.cols != N))
      return fail(c, ZTP_ESHAPE, std::string(nm) + " FWD GeLU: " + shp("pre_t", a->pre_t));
    if (layer == LAYER_ROW && a->y_pos && !a->skip_collective && c->world > 1)
      return fail(c, ZTP_EUNSUPPORTED, std::string(nm) + " FWD: an output row map (y_pos) needs TP = 1 or "
                                                          "skip_collective (the all-reduce sums full outputs)");
    if (a->sel) c->lineage[key] = LineageEntry{a->sel->kept, a->sel->pruned, a->sel->n_kept, a->sel->n_pruned};
    const bool fill_x = !(a->prepared & 1) || !a->xs_t.ptr;   // ztp_prepare wrote the copies already
    const bool fill_w = !(a->prepared & 2) || !a->ws_t.ptr;
    s = operand_src(c, dense_sel, xc, x, a->xs_t, fill_x, kept, nk, 0, &tmpx, &X, st);
    if (s != ZTP_OK) return s;
    if (os)
      s = weight_2d(c, a->w_t, dense_sel ? nullptr : kept, nk, os->kept, (int)n_y, a->ws_t, fill_w, &tmpw, &W, st);
    else
      s = operand_src(c, dense_sel, false, a->w_t, a->ws_t, fill_w, kept, nk, 1, &tmpw, &W, st);
    if (s != ZTP_OK) return s;
    s = gemm(c, ztp::KIND_FWD, W, X, n_y, kept, pruned, nk, act ? a->pre_t : a->y_t, act ? &a->y_t : nullptr,
             nullptr, 0, os ? nullptr : a->y_pos, act ? act_epi : ztp::EPI_NONE, st);
    if (s != ZTP_OK) return s;
    if (layer == LAYER_ROW && !a->skip_collective) return allreduce(c, a->y_t, st);
    return ZTP_OK;
  }
  // ----------------------------------------------------------------- BWD
  if (a->sel) {
    auto it = c->lineage.find(key);
    if (it == c->lineage.end() || it->second.kept != a->sel->kept || it->second.pruned != a->sel->pruned ||
        it->second.nk != a->sel->n_kept || it->second.np != a->sel->n_pruned)
      return fail(c, ZTP_ELINEAGE,
                  std::string(nm) + " BWD: no matching FWD lineage entry for <layer " +
                      std::to_string(key.first) + ", matrix " + std::to_string(key.second) + "> (S:400)");
  }
  const ztp_mat& g = a->g_t;
  if (!mat_ok(g) || g.rows < n_y || g.dtype != dtype)
    return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("g_t", g));
  const int64_t N = g.cols;
  if (dtype == ZTP_BF16 && N % 8 != 0) return fail(c, ZTP_ESHAPE, "tokens N must be a multiple of 8");
  const bool reduce_dx0 = layer == LAYER_COL && a->dx_t.ptr && !a->skip_collective && c->world > 1;
  if (c->group_bwd && a->dx_t.ptr && a->dw_t.ptr && dtype == ZTP_BF16 && !reduce_dx0 && !c->use_gather4 &&
      !(a->act_in != ZTP_ACT_NONE && layer != LAYER_ROW) &&
      (c->group_bwd == 1 || ztp::gemm_group_pays((int)(dxc ? nk : K), (int)N, (int)n_y, nk, (int)K, (int)n_y,
                                                 (int)N, nk, c->num_sms))) {
    // ---- grouped: dX and dW units in one persistent launch on every SM
    const ztp_mat& x = a->x_t;
    if (!mat_ok(a->dx_t) || (dxc ? a->dx_t.rows < nk : a->dx_t.rows != K) || a->dx_t.cols != N ||
        a->dx_t.dtype != dtype)
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("dx_t", a->dx_t) + " vs K " + std::to_string(K));
    if (dxc && a->act_in != ZTP_ACT_NONE && !xc)
      return fail(c, ZTP_EINVAL, std::string(nm) + " BWD: dx_compact with GeLU' needs x_compact pre_in_t");
    if (!mat_ok(x) || x.rows < x_rows_need || x.cols != N || x.dtype != dtype || (!xc && x.rows != K))
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("x_t", x) + " vs " + shp("g_t", g));
    if (!mat_ok(a->dw_t) || a->dw_t.rows != K || a->dw_t.cols < n_out || a->dw_t.dtype != dtype)
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("dw_t", a->dw_t));
    int epi = ztp::EPI_NONE;
    const ztp_mat* aux = nullptr;
    if (layer == LAYER_ROW && (a->act_in == ZTP_ACT_GELU || a->act_in == ZTP_ACT_GELU_D)) {
      if (!mat_ok(a->pre_in_t) || a->pre_in_t.rows < x_rows_need || a->pre_in_t.cols != N)
        return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD GeLU': " + shp("pre_in_t", a->pre_in_t));
      epi = a->act_in == ZTP_ACT_GELU_D ? ztp::EPI_MUL : ztp::EPI_GELU_GRAD;
      aux = &a->pre_in_t;
    }
    if (os)
      s = weight_2d(c, a->w_t, dense_sel ? nullptr : kept, nk, os->kept, (int)n_y, a->ws_t, false, &tmpw, &W, st);
    else
      s = operand_src(c, dense_sel, false, a->w_t, a->ws_t, false, kept, nk, 1, &tmpw, &W, st);
    if (s != ZTP_OK) return s;
    s = operand_src(c, dense_sel, xc, x, a->xs_t, false, kept, nk, 0, &tmpx, &X, st);
    if (s != ZTP_OK) return s;
    ztp_mat dx = a->dx_t;
    if (dxc) dx.rows = nk;   // rows P implied Zero, not written
    const GemmSpec sx{ztp::KIND_DX, W, Src{&g, true}, n_y, kept, dxc ? nullptr : pruned, nk, dx, aux, xc ? 1 : 0,
                      epi, dxc, nullptr, 0, nullptr};
    const GemmSpec sw{ztp::KIND_DW, X, Src{&g, true}, n_y, kept, pruned, nk, a->dw_t, nullptr, 0, ztp::EPI_NONE,
                      false, os ? a->y_pos : nullptr, (int)n_out, os ? os->kept : nullptr};
    s = gemm_group(c, sx, sw, st);
    if (s != ZTP_EUNSUPPORTED) {
      if (s != ZTP_OK) return s;
      if (!dense_sel) s = impute(c, a->impute, a->dx_t, N, kept, nk, pruned, np, a->hist_dx, st);
      if (s == ZTP_OK && !dense_sel) s = impute(c, a->impute, a->dw_t, n_out, kept, nk, pruned, np, a->hist_dw, st);
      if (s != ZTP_OK) return s;
      if (layer == LAYER_COL && !a->skip_collective && c->world > 1) return allreduce(c, a->dx_t, st);
      return ZTP_OK;
    }
    // not groupable (shapes): fall through to the concurrent pair
  }
  // dW concurrently with dX on the side stream (also on an emulated
  // straggler: each GEMM is stretched from its own stamp slot; not while
  // profiling with events, which times each GEMM alone)
  const bool conc = c->conc_bwd && c->prof_on != 1 && a->dx_t.ptr && a->dw_t.ptr && dtype == ZTP_BF16;
  // dW alone on the side stream (dw_side): it shares the GPU with what the
  // caller launches next on its stream (half the SMs for its persistent grid)
  const bool side_only = a->dw_side && !a->dx_t.ptr && a->dw_t.ptr && c->conc_bwd && c->prof_on != 1 &&
                         dtype == ZTP_BF16;
  cudaStream_t sw = st;
  int cap_dx = 0, cap_dw = 0;
  if (side_only) {
    CUDA_TRY(c, cudaEventRecord(c->ev_c, st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side_stream, c->ev_c, 0));
    sw = c->side_stream;
    cap_dw = 2 * ((c->num_sms / 2) / 2);
    // its work, for the next dX / dW partition (the side stream runs it first)
    const int cg = ztp::gemm_choose_cg(ztp::KIND_DW, (int)K, nk);
    const int tm = 128 * cg;
    const int mc = std::min(((int)K + tm - 1) / tm, (nk + tm - 1) / tm), nt = ((int)n_y + 255) / 256;
    const int sp = c->allow_splitk ? ztp::gemm_choose_splits(ztp::KIND_DW, (int)K, (int)n_y, (int)N, nk, cap_dw) : 1;
    const int kb = ((int)N + 63) / 64;
    c->side_bl_units += mc * nt * sp;
    c->side_bl_kps = std::max(c->side_bl_kps, (kb + sp - 1) / sp);
    c->side_bl_pairs = cap_dw / cg;
  }
  if (conc) {
    CUDA_TRY(c, cudaEventRecord(c->ev_c, st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side_stream, c->ev_c, 0));
    sw = c->side_stream;
    // partition the SMs (in CTA pairs) in proportion to the two GEMMs' MMA
    // work (tiles x 64-deep k-blocks; dW's weighted by dw_share), so both run
    // at once and each one's fill and tail overlap the other's mainloop
    const double rows = (double)std::min<int64_t>(nk, dxc ? nk : K);
    const double t_rows = std::ceil(rows / 256.0);
    // a GeLU' epilogue (reads pre_in_t per output element) costs dX more per
    // tile: weighted by aux_weight
    const bool dx_aux = layer == LAYER_ROW && (a->act_in == ZTP_ACT_GELU || a->act_in == ZTP_ACT_GELU_D);
    const double w_dx = t_rows * std::ceil((double)N / 256.0) * std::ceil((double)n_y / 64.0) *
                        (dx_aux ? c->aux_weight : 1.0);
    const double w_dw = t_rows * std::ceil((double)n_y / 256.0) * std::ceil((double)N / 64.0);
    const int pairs = c->num_sms / 2;
    int px = (int)std::lround(pairs * w_dx / (w_dx + c->dw_share * w_dw));
    px = std::max(1, std::min(pairs - 1, px));
    if (c->part_model >= 1) {
      // wave-quantised: each GEMM's time ~ ceil(units / CTA slots) x k-blocks
      // per unit (its split-K as gemm() will choose it for that many SMs);
      // the partition minimising the later finish, ties to the proportional one
      // The epilogue warps run beside the MMA: a pair's time is the longer
      // of its MMA k-blocks and its epilogue work -- computed tiles (~2 us,
      // EW k-blocks) plus the all-pruned Zero tiles, which have no MMA but
      // write a whole output tile (~2.5 us, ZW; the c0 TP = 8 gamma = 0.9
      // timeline, profiles/r02_zero_units_partition.txt).  Without the
      // epilogue term a heavily resized dX (few computed tiles, many Zero
      // rows) got few SMs and its Zero rows ran long after its MMAs.
      constexpr double EW = 5.0, ZW = 6.0;
      auto cost = [&](int kind, int M_, int N_, int kdim_, int nsm, double wgt, bool zero_units) {
        const int cg = ztp::gemm_choose_cg(kind, M_, nk);
        const int tm = 128 * cg;
        const int mt = (M_ + tm - 1) / tm;
        const int mc = std::min(mt, (nk + tm - 1) / tm), nt = (N_ + 255) / 256;
        const int sp = c->allow_splitk ? ztp::gemm_choose_splits(kind, M_, N_, kdim_, nk, nsm) : 1;
        const int kb = (kdim_ + 63) / 64, kps = (kb + sp - 1) / sp;
        const int slots = std::max(1, nsm / cg);
        const double rounds = std::ceil((double)mc * nt * sp / slots);
        const double zu = (zero_units && sp == 1) ? (double)(mt - mc) * nt : 0.0;
        if (c->part_model == 2) return rounds * kps * wgt;   // MMA work only (the model before the Zero term)
        return std::max(rounds * kps * wgt, rounds * EW + std::ceil(zu / slots) * ZW);
      };
      const int Mx = (int)(dxc ? nk : K);
      double best = 1e300;
      int bp = px;
      for (int q = 1; q < pairs; ++q) {
        // a dw_side GEMM queued on the side stream runs before this dW
        const double bl = c->side_bl_units > 0
                              ? std::ceil((double)c->side_bl_units / std::max(1, std::min(c->side_bl_pairs, pairs - q))) *
                                    c->side_bl_kps * c->dw_share
                              : 0.0;
        const double t =
            std::max(cost(ztp::KIND_DX, Mx, (int)N, (int)n_y, 2 * q, dx_aux ? c->aux_weight : 1.0, !dxc),
                     bl + cost(ztp::KIND_DW, (int)K, (int)n_y, (int)N, 2 * (pairs - q), c->dw_share, !os));
        if (t < best - 1e-9 || (t < best + 1e-9 && std::abs(q - px) < std::abs(bp - px))) {
          best = std::min(best, t);
          bp = q;
        }
      }
      px = bp;
    }
    cap_dx = 2 * px;
    cap_dw = 2 * (pairs - px);
    c->side_bl_units = c->side_bl_kps = c->side_bl_pairs = 0;   // accounted
  }
  if (a->dx_t.ptr) {
    if (!mat_ok(a->dx_t) || (dxc ? a->dx_t.rows < nk : a->dx_t.rows != K) || a->dx_t.cols != N ||
        a->dx_t.dtype != dtype)
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("dx_t", a->dx_t) + " vs K " + std::to_string(K) +
                                     (dxc ? " (compact dx: n_kept rows)" : ""));
    if (dxc && a->act_in != ZTP_ACT_NONE && !xc)
      return fail(c, ZTP_EINVAL, std::string(nm) + " BWD: dx_compact with GeLU' needs x_compact pre_in_t");
    int epi = ztp::EPI_NONE;
    const ztp_mat* aux = nullptr;
    if (layer == LAYER_ROW && (a->act_in == ZTP_ACT_GELU || a->act_in == ZTP_ACT_GELU_D)) {
      if (!mat_ok(a->pre_in_t) || a->pre_in_t.rows < x_rows_need || a->pre_in_t.cols != N)
        return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD GeLU': " + shp("pre_in_t", a->pre_in_t));
      epi = a->act_in == ZTP_ACT_GELU_D ? ztp::EPI_MUL : ztp::EPI_GELU_GRAD;
      aux = &a->pre_in_t;
    }
    if (os)
      s = weight_2d(c, a->w_t, dense_sel ? nullptr : kept, nk, os->kept, (int)n_y, a->ws_t, false, &tmpw, &W, st);
    else
      s = operand_src(c, dense_sel, false, a->w_t, a->ws_t, false, kept, nk, 1, &tmpw, &W, st);
    if (s != ZTP_OK) return s;
    ztp_mat dx = a->dx_t;
    if (dxc) dx.rows = nk;   // rows P implied Zero, not written
    c->sm_cap = cap_dx;
    s = gemm(c, ztp::KIND_DX, W, Src{&g, true}, n_y, kept, dxc ? nullptr : pruned, nk, dx, nullptr, aux, xc ? 1 : 0,
             nullptr, epi, st, dxc);
    c->sm_cap = 0;
    if (s != ZTP_OK) return s;
    // Average / Same on this rank's partial, before the all-reduce (A-14)
    if (!dense_sel) s = impute(c, a->impute, a->dx_t, N, kept, nk, pruned, np, a->hist_dx, st);
    if (s != ZTP_OK) return s;
  }
  const bool reduce_dx = layer == LAYER_COL && a->dx_t.ptr && !a->skip_collective && c->world > 1;
  if (reduce_dx) {
    // overlap the dX all-reduce with the dW GEMM: comm on a side stream
    CUDA_TRY(c, cudaEventRecord(c->ev_a, st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_a, 0));
    s = allreduce(c, a->dx_t, c->comm_stream);
    if (s != ZTP_OK) return s;
    CUDA_TRY(c, cudaEventRecord(c->ev_b, c->comm_stream));
  }
  if (a->dw_t.ptr) {
    const ztp_mat& x = a->x_t;
    if (!mat_ok(x) || x.rows < x_rows_need || x.cols != N || x.dtype != dtype || (!xc && x.rows != K))
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("x_t", x) + " vs " + shp("g_t", g));
    if (!mat_ok(a->dw_t) || a->dw_t.rows != K || a->dw_t.cols < n_out || a->dw_t.dtype != dtype)
      return fail(c, ZTP_ESHAPE, std::string(nm) + " BWD: " + shp("dw_t", a->dw_t));
    const int64_t l0 = c->launches;
    s = operand_src(c, dense_sel, xc, x, a->xs_t, false, kept, nk, 0, &tmpx, &X, sw);
    if (s != ZTP_OK) return s;
    const bool copied = c->launches != l0;   // a compaction kernel now precedes the dW GEMM
    // output pruning: the GEMM computes the compact columns S'; its split-K
    // reduce (or an expansion pass) spreads them to their units, P' <- Zero
    c->sm_cap = cap_dw;
    s = gemm(c, ztp::KIND_DW, X, Src{&g, true}, n_y, kept, pruned, nk, a->dw_t, nullptr, nullptr, 0, nullptr,
             ztp::EPI_NONE, sw, false, os ? a->y_pos : nullptr, (int)n_out,
             /*indep_of_prev=*/a->dx_t.ptr != nullptr && !copied && !conc && !reduce_dx &&
                 a->impute == ZTP_IMPUTE_ZERO,
             os ? os->kept : nullptr);
    c->sm_cap = 0;
    if (s != ZTP_OK) return s;
    if (!dense_sel) s = impute(c, a->impute, a->dw_t, n_out, kept, nk, pruned, np, a->hist_dw, sw);
    if (s != ZTP_OK) return s;
  }
  // the dW outputs feed nothing later in the step: the side stream is joined
  // by ztp_join (or the next FWD call), not here, so the next linear's dX
  // does not wait for this dW
  if (conc || side_only) c->side_pending = true;
  if (reduce_dx) CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_b, 0));
  return ZTP_OK;
}

}  // namespace

namespace ztp {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ZTP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace ztp

// =========================================================================== API

extern "C" {

const char* ztp_status_str(ztp_status s) {
  switch (s) {
    case ZTP_OK: return "ZTP_OK";
    case ZTP_EINVAL: return "ZTP_EINVAL";
    case ZTP_ESHAPE: return "ZTP_ESHAPE";
    case ZTP_EINDEX: return "ZTP_EINDEX";
    case ZTP_EDEGENERATE: return "ZTP_EDEGENERATE";
    case ZTP_ELINEAGE: return "ZTP_ELINEAGE";
    case ZTP_EHISTORY: return "ZTP_EHISTORY";
    case ZTP_ENOBASELINE: return "ZTP_ENOBASELINE";
    case ZTP_ENOHELPER: return "ZTP_ENOHELPER";
    case ZTP_ERECEIVERS: return "ZTP_ERECEIVERS";
    case ZTP_ECUDA: return "ZTP_ECUDA";
    case ZTP_ENCCL: return "ZTP_ENCCL";
    case ZTP_EUNSUPPORTED: return "ZTP_EUNSUPPORTED";
  }
  return "ZTP_?";
}

const char* ztp_last_error(const ztp_ctx* c) { return c ? c->err.c_str() : ztp::g_thread_err.c_str(); }

const char* ztp_version(void) { return "ztp 0.1 sm_100a (tcgen05 + TMA gather4 + NCCL)"; }

ztp_status ztp_get_unique_id(unsigned char uid[ZTP_UID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == ZTP_UID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_TRY(nullptr, ncclGetUniqueId(&id));
  std::memcpy(uid, &id, ZTP_UID_BYTES);
  return ZTP_OK;
}

ztp_status ztp_ctx_create(ztp_ctx** out, int rank, int world, const unsigned char* uid, int device) {
  if (!out) return fail(nullptr, ZTP_EINVAL, "ztp_ctx_create: out is NULL");
  *out = nullptr;
  if (world < 1 || world > ZTP_MAX_RANKS || rank < 0 || rank >= world)
    return fail(nullptr, ZTP_EINVAL, "ztp_ctx_create: rank/world out of range");
  CUDA_TRY(nullptr, cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(nullptr, cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(nullptr, ZTP_EUNSUPPORTED,
                std::string("libztp is built for sm_100a (B200) only; device is ") + prop.name + " sm_" +
                    std::to_string(prop.major) + std::to_string(prop.minor));
  ztp_ctx* c = new ztp_ctx();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (const char* g4 = getenv("ZTP_GATHER4")) c->use_gather4 = atoi(g4) != 0;
  if (const char* sk = getenv("ZTP_SPLITK")) c->allow_splitk = atoi(sk) != 0;
  if (const char* cc = getenv("ZTP_CONC")) c->conc_bwd = atoi(cc) != 0;
  if (const char* ds = getenv("ZTP_DW_SHARE")) c->dw_share = atof(ds);
  if (const char* aw = getenv("ZTP_AUX_WEIGHT")) c->aux_weight = atof(aw);
  if (const char* pm = getenv("ZTP_PART")) c->part_model = atoi(pm);
  if (const char* sg = getenv("ZTP_SQUAT_GUARD")) c->squat_guard = atoi(sg) != 0;
  if (const char* gb = getenv("ZTP_GROUP")) c->group_bwd = atoi(gb);
  if (const char* ae = getenv("ZTP_A_EARLY")) c->a_early = atoi(ae) != 0;
  if (const char* se = getenv("ZTP_SPREAD_EPI")) c->spread_epi = atoi(se) != 0;
  if (const char* zg = getenv("ZTP_ZERO_GENERIC")) c->zero_generic = atoi(zg) != 0;
  if (const char* th = getenv("ZTP_TAIL_HALVES")) c->tail_halves = atoi(th) != 0;
  if (const char* fl = getenv("ZTP_FLAGS")) c->flags_opt = atoi(fl) != 0;
  if (const char* de = getenv("ZTP_DEBUG_EPI")) c->dbg_epi = atoi(de);
  if (const char* ds = getenv("ZTP_DEBUG_SKIP")) c->dbg_skip = atoi(ds);
  auto cleanup = [&](ztp_status s) {
    ztp_ctx_destroy(c);
    return s;
  };
  if (cudaMalloc(&c->d_tflags, sizeof(unsigned long long) * ztp_ctx::FLAG_SLOTS * (1 + ztp::FLAG_NB)) != cudaSuccess ||
      cudaMemset(c->d_tflags, 0, sizeof(unsigned long long) * ztp_ctx::FLAG_SLOTS * (1 + ztp::FLAG_NB)) != cudaSuccess ||
      cudaMalloc(&c->d_flags, 64) != cudaSuccess || cudaMalloc(&c->d_stamp, 32) != cudaSuccess ||
      cudaMalloc(&c->d_gemm_ns, 16) != cudaSuccess || cudaMalloc(&c->d_stats, 2 * (ZTP_MAX_RANKS + 1) * sizeof(double)) != cudaSuccess)
    return cleanup(fail(nullptr, ZTP_ECUDA, "ztp_ctx_create: device allocation failed"));
  cudaMemset(c->d_flags, 0, 64);
  unsigned long long init_stamp[4] = {~0ull, 0ull, ~0ull, 0ull};
  cudaMemcpy(c->d_stamp, init_stamp, 32, cudaMemcpyHostToDevice);
  cudaMemset(c->d_gemm_ns, 0, 16);
  if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_c, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_d, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(fail(nullptr, ZTP_ECUDA, "ztp_ctx_create: stream/event creation failed"));
  if (ensure_iota(c, 1 << 16) != ZTP_OK) return cleanup(ZTP_ECUDA);
  c->transport = (world > 1 && !uid) ? ZTP_TRANSPORT_PEER : ZTP_TRANSPORT_NCCL;
  if (const char* pc = getenv("ZTP_PEER_CTAS")) c->peer_ctas = std::max(1, std::min(ztp::PEER_MAX_CTAS, atoi(pc)));
  if (world > 1 && uid) {
    ncclUniqueId id;
    std::memcpy(&id, uid, ZTP_UID_BYTES);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess)
      return cleanup(fail(nullptr, ZTP_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
  }
  *out = c;
  return ZTP_OK;
}

ztp_status ztp_ctx_destroy(ztp_ctx* c) {
  if (!c) return ZTP_OK;
  if (c->comm) ncclCommDestroy(c->comm);
  for (int q = 0; q < ZTP_MAX_RANKS; ++q)
    if (c->win_ipc[q]) cudaIpcCloseMemHandle(c->win_ipc[q]);
  if (c->win) cudaFree(c->win);
  if (c->pw.ep) cudaFree(c->pw.ep);
  if (c->d_one) cudaFree(c->d_one);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->ev_c) cudaEventDestroy(c->ev_c);
  if (c->ev_d) cudaEventDestroy(c->ev_d);
  if (c->skws_side) cudaFree(c->skws_side);
  if (c->d_pstamp) cudaFree(c->d_pstamp);
  if (c->d_ctastamp) cudaFree(c->d_ctastamp);
  cudaFree(c->d_flags);
  cudaFree(c->d_tflags);
  cudaFree(c->d_stamp);
  cudaFree(c->d_gemm_ns);
  cudaFree(c->d_stats);
  cudaFree(c->d_iota);
  cudaFree(c->ws);
  cudaFree(c->skws);
  cudaFree(c->cws[0]);
  cudaFree(c->cws[1]);
  cudaFree(c->xws[0]);
  cudaFree(c->xws[1]);
  cudaFree(c->mws[0]);
  cudaFree(c->mws[1]);
  for (auto& e : c->prof) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  delete c;
  return ZTP_OK;
}

ztp_status ztp_sync(ztp_ctx* c, void* stream) {
  if (!c) return fail(nullptr, ZTP_EINVAL, "ztp_sync: null ctx");
  CUDA_TRY(c, cudaStreamSynchronize((cudaStream_t)stream));
  CUDA_TRY(c, cudaGetLastError());
  int32_t flags[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpy(flags, c->d_flags, 8, cudaMemcpyDeviceToHost));
  if (flags[1]) {
    cudaMemset(c->d_flags + 1, 0, 4);
    return fail(c, ZTP_ECUDA, "peer barrier timed out (a rank did not reach the same collective within 10 s)");
  }
  if (flags[0]) {
    cudaMemset(c->d_flags, 0, 4);
    return fail(c, ZTP_EINVAL, "ztp_select saw a NaN score");
  }
  return ZTP_OK;
}

int64_t ztp_launch_count(const ztp_ctx* c) { return c ? c->launches : 0; }

ztp_status ztp_allgather_stats(ztp_ctx* c, double T_own, double M_own, double* T_all, double* M_all, void* stream) {
  if (!c || !T_all || !M_all) return fail(c, ZTP_EINVAL, "ztp_allgather_stats: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  double mine[2] = {T_own, M_own};
  if (c->world == 1) {
    T_all[0] = T_own;
    M_all[0] = M_own;
    return ZTP_OK;
  }
  double* d_send = c->d_stats + 2 * ZTP_MAX_RANKS;  // scratch after the gathered block
  std::vector<double> host(2 * c->world);
  if (c->transport == ZTP_TRANSPORT_PEER) {
    if (!c->win_open) return fail(c, ZTP_EINVAL, "ztp_allgather_stats: open the peer window first");
    CUDA_TRY(c, ztp::peer_stats_launch(c->pw, T_own, M_own, st));
    ++c->launches;
    CUDA_TRY(c, cudaMemcpyAsync(host.data(), c->win + ztp::PEER_STATS_OFF, 2 * c->world * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(d_send, mine, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
    NCCL_TRY(c, ncclAllGather(d_send, c->d_stats, 2, ncclDouble, c->comm, st));
    CUDA_TRY(c, cudaMemcpyAsync(host.data(), c->d_stats, 2 * c->world * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(c, cudaStreamSynchronize(st));
  for (int r = 0; r < c->world; ++r) {
    T_all[r] = host[2 * r];
    M_all[r] = host[2 * r + 1];
  }
  return ZTP_OK;
}

ztp_status ztp_select(ztp_ctx* c, int nseg, const int32_t* h_len, const int32_t* h_np, const int32_t* h_app,
                      const float* d_scores, int32_t* d_kept, int32_t* d_pruned, int32_t* d_pos, void* stream) {
  if (!c || !h_len || !h_np || !d_scores || !d_kept || !d_pruned || nseg < 1)
    return fail(c, ZTP_EINVAL, "ztp_select: null argument or nseg < 1");
  std::vector<ztp::SelectSeg> segs(nseg);
  int64_t so = 0, ko = 0, po = 0, qo = 0;
  for (int i = 0; i < nseg; ++i) {
    const int32_t app = h_app ? h_app[i] : 0;
    if (h_len[i] < 1 || h_np[i] < 0 || h_np[i] > h_len[i] - 1 || app < 0)
      return fail(c, ZTP_EINVAL,
                  "ztp_select: segment " + std::to_string(i) + " len " + std::to_string(h_len[i]) + " n_prune " +
                      std::to_string(h_np[i]) + " (need 0 <= n_prune <= len-1)");
    segs[i] = ztp::SelectSeg{h_len[i], h_np[i], app, (int32_t)so, (int32_t)ko, (int32_t)po, (int32_t)qo};
    so += h_len[i];
    qo += h_len[i] + app;
    ko += h_len[i] - h_np[i] + app;
    po += h_np[i];
  }
  if (so > INT32_MAX) return fail(c, ZTP_EINVAL, "ztp_select: too many columns");
  {  // a pending concurrent dW still reads the lineage lists this call rewrites
    ztp_status js = join_side(c, (cudaStream_t)stream);
    if (js != ZTP_OK) return js;
  }
  for (int b = 0; b < nseg; b += ztp::SELECT_MAX_SEGS) {
    ztp::SelectParams p{};
    p.nseg = std::min(ztp::SELECT_MAX_SEGS, nseg - b);
    for (int i = 0; i < p.nseg; ++i) p.seg[i] = segs[b + i];
    const int pe = prof_begin(c, (cudaStream_t)stream, PROF_OTHER, 0.0);
    if (!(c->dbg_skip & 1))
      CUDA_TRY(c, ztp::select_launch(p, d_scores, d_kept, d_pruned, d_pos, c->d_flags, (cudaStream_t)stream));
    prof_end(c, pe, (cudaStream_t)stream);
    ++c->launches;
  }
  return ZTP_OK;
}

ztp_status ztp_priority_update(ztp_ctx* c, const ztp_mat* w, const ztp_mat* wo, const int32_t* pos_prev, float* delta,
                               int32_t* count_above, float theta, void* stream) {
  if (!c || !w || !wo || !delta) return fail(c, ZTP_EINVAL, "ztp_priority_update: null argument");
  if (!mat_ok(*w) || !mat_ok(*wo) || w->rows != wo->rows || w->cols != wo->cols || w->dtype != ZTP_BF16 ||
      wo->dtype != ZTP_BF16)
    return fail(c, ZTP_ESHAPE, "ztp_priority_update: " + shp("w_t", *w) + " vs " + shp("w_old_t", *wo) + " (bf16)");
  cudaStream_t st = (cudaStream_t)stream;
  {  // the selection (pos_prev) and scores may still be read by a pending dW
    ztp_status js = join_side(c, st);
    if (js != ZTP_OK) return js;
  }
  const int pe = prof_begin(c, st, PROF_OTHER, 0.0);
  CUDA_TRY(c, ztp::priority_update_launch(w->ptr, w->ld, wo->ptr, wo->ld, w->rows, w->cols, pos_prev, delta,
                                          count_above, theta, st));
  prof_end(c, pe, st);
  ++c->launches;
  return ZTP_OK;
}

double ztp_pridiff_gamma(int64_t L, int64_t L_uni, double gamma_t, double alpha) {
  if (L <= 0) return 0.0;
  const double g = 1.0 - (double)L_uni / (double)L;
  const double f = alpha * gamma_t;
  return g > f ? g : f;
}

ztp_status ztp_prepare(ztp_ctx* c, int n, const ztp_linear_args* const* args, const int32_t* what, void* stream) {
  if (!c || n < 0 || (n > 0 && (!args || !what))) return fail(c, ZTP_EINVAL, "ztp_prepare: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  {  // the compact copies this call rewrites may still be read by a pending dW
    ztp_status js = join_side(c, st);
    if (js != ZTP_OK) return js;
  }
  ztp::GatherJobs J{};
  auto add = [&](const void* src, int64_t ld_src, const int32_t* rows, int nr, const int32_t* cols, int nc,
                 const ztp_mat& dst, int src_cols) -> ztp_status {
    if (J.njobs == ztp::GATHER_MAX_JOBS) return fail(c, ZTP_EINVAL, "ztp_prepare: more than 16 copies");
    if (!mat_ok(dst) || dst.rows < nr || dst.cols < nc || dst.dtype != ZTP_BF16)
      return fail(c, ZTP_ESHAPE, "ztp_prepare: destination " + shp("dst", dst) + " too small / not bf16");
    ztp::GatherJob& g = J.job[J.njobs++];
    g = ztp::GatherJob{(const uint16_t*)src, ld_src, rows, cols, (uint16_t*)dst.ptr, dst.ld, nr, nc, J.total,
                       src_cols};
    J.total += nr;
    return ZTP_OK;
  };
  for (int i = 0; i < n; ++i) {
    const ztp_linear_args* a = args[i];
    if (!a) return fail(c, ZTP_EINVAL, "ztp_prepare: null args");
    if (a->w_t.dtype != ZTP_BF16) return fail(c, ZTP_EUNSUPPORTED, "ztp_prepare: bf16 only");
    const int64_t K = a->w_t.rows;
    const int32_t* kept;
    const int32_t* pruned;
    int nk, np;
    ztp_status s = resolve_sel(c, a->sel, K, &kept, &pruned, &nk, &np);
    if (s != ZTP_OK) return s;
    const bool dense = a->sel == nullptr;
    if ((what[i] & 1) && !dense && !a->x_compact) {
      if (!mat_ok(a->x_t) || a->x_t.rows != K || a->x_t.dtype != ZTP_BF16)
        return fail(c, ZTP_ESHAPE, "ztp_prepare: " + shp("x_t", a->x_t));
      s = add(a->x_t.ptr, a->x_t.ld, kept, nk, nullptr, (int)a->x_t.cols, a->xs_t, 0);
      if (s != ZTP_OK) return s;
    }
    if (what[i] & 2) {
      const int64_t n_out = a->n_out > 0 ? a->n_out : a->w_t.cols;
      if (a->out_sel) {
        if ((int64_t)a->out_sel->n_kept + a->out_sel->n_pruned != n_out || !a->out_sel->kept)
          return fail(c, ZTP_ESHAPE, "ztp_prepare: out_sel does not cover n_out");
        s = add(a->w_t.ptr, a->w_t.ld, dense ? nullptr : kept, nk, a->out_sel->kept, a->out_sel->n_kept, a->ws_t,
                (int)n_out);
      } else if (!dense) {
        s = add(a->w_t.ptr, a->w_t.ld, kept, nk, nullptr, (int)a->w_t.cols, a->ws_t, 0);
      }
      if (s != ZTP_OK) return s;
    }
  }
  if (J.total == 0) return ZTP_OK;
  const int pe = prof_begin(c, st, PROF_OTHER, 0.0);
  if (!(c->dbg_skip & 2)) CUDA_TRY(c, ztp::gather_multi_launch(J, st));
  prof_end(c, pe, st);
  ++c->launches;
  return ZTP_OK;
}

ztp_status ztp_join(ztp_ctx* c, void* stream) {
  if (!c) return fail(c, ZTP_EINVAL, "ztp_join: null ctx");
  return join_side(c, (cudaStream_t)stream);
}

ztp_status ztp_col_linear(ztp_ctx* c, ztp_phase phase, const ztp_linear_args* a, void* stream) {
  return linear(c, LAYER_COL, phase, a, (cudaStream_t)stream);
}
ztp_status ztp_row_linear(ztp_ctx* c, ztp_phase phase, const ztp_linear_args* a, void* stream) {
  return linear(c, LAYER_ROW, phase, a, (cudaStream_t)stream);
}

ztp_status ztp_gemm(ztp_ctx* c, int kind, const ztp_linear_args* a, void* stream) {
  if (!c || !a || kind < 0 || kind > 2) return fail(c, ZTP_EINVAL, "ztp_gemm: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const ztp_mat& full_src = kind == ztp::KIND_DW ? a->x_t : a->w_t;
  const int64_t K = a->x_compact && kind == ztp::KIND_DW ? a->dw_t.rows : full_src.rows;
  const int64_t n_out = a->n_out > 0 ? a->n_out : (kind == ztp::KIND_DW ? a->dw_t.cols : a->w_t.cols);
  const int32_t* kept;
  const int32_t* pruned;
  int nk, np;
  ztp_status s = resolve_sel(c, a->sel, kind == ztp::KIND_FWD ? a->w_t.rows : (kind == ztp::KIND_DX ? a->w_t.rows : K),
                             &kept, &pruned, &nk, &np);
  if (s != ZTP_OK) return s;
  const bool dense_sel = a->sel == nullptr;
  ztp_mat tx{}, tw{};
  Src X{nullptr, false}, W{nullptr, false};
  if (kind == ztp::KIND_FWD) {
    const bool act = a->act == ZTP_ACT_GELU || a->act == ZTP_ACT_GELU_D;
    const int act_epi = a->act == ZTP_ACT_GELU_D ? ztp::EPI_GELU_D : ztp::EPI_GELU;
    s = operand_src(c, dense_sel, a->x_compact != 0, a->x_t, a->xs_t, true, kept, nk, 0, &tx, &X, st);
    if (s == ZTP_OK) s = operand_src(c, dense_sel, false, a->w_t, a->ws_t, true, kept, nk, 1, &tw, &W, st);
    if (s != ZTP_OK) return s;
    return gemm(c, kind, W, X, n_out, kept, pruned, nk, act ? a->pre_t : a->y_t, act ? &a->y_t : nullptr, nullptr,
                0, a->y_pos, act ? act_epi : ztp::EPI_NONE, st);
  }
  if (kind == ztp::KIND_DX) {
    const bool gg = a->act_in == ZTP_ACT_GELU || a->act_in == ZTP_ACT_GELU_D;
    const int gepi = a->act_in == ZTP_ACT_GELU_D ? ztp::EPI_MUL : ztp::EPI_GELU_GRAD;
    s = operand_src(c, dense_sel, false, a->w_t, a->ws_t, true, kept, nk, 1, &tw, &W, st);
    if (s != ZTP_OK) return s;
    return gemm(c, kind, W, Src{&a->g_t, true}, n_out, kept, pruned, nk, a->dx_t, nullptr,
                gg ? &a->pre_in_t : nullptr, a->x_compact ? 1 : 0, nullptr, gg ? gepi : ztp::EPI_NONE,
                st);
  }
  s = operand_src(c, dense_sel, a->x_compact != 0, a->x_t, a->xs_t, true, kept, nk, 0, &tx, &X, st);
  if (s != ZTP_OK) return s;
  return gemm(c, kind, X, Src{&a->g_t, true}, n_out, kept, pruned, nk, a->dw_t, nullptr, nullptr, 0, nullptr,
              ztp::EPI_NONE, st);
}

ztp_status ztp_core(ztp_ctx* c, ztp_phase phase, const ztp_mat* qkv, const ztp_mat* cx, int64_t feat, int64_t n_feat,
                    const int32_t* rows, int64_t n_rows, int32_t v_compact, void* stream) {
  if (!c || !qkv || !cx || !mat_ok(*qkv) || !mat_ok(*cx)) return fail(c, ZTP_ESHAPE, "ztp_core: bad matrices");
  if (v_compact && (!rows || n_rows < 1)) return fail(c, ZTP_EINVAL, "ztp_core: v_compact needs the kept list rows");
  const int64_t n_out = (phase == ZTP_FWD && rows) ? n_rows : n_feat;
  const int64_t n_v = v_compact ? n_rows : n_feat;
  const int64_t qkv_rows = v_compact ? 2 * feat + n_v : 3 * feat;
  if (qkv->rows < qkv_rows || n_feat > feat || cx->rows < n_out || cx->cols != qkv->cols || qkv->dtype != cx->dtype ||
      (rows && (n_rows < 1 || n_rows > n_feat)))
    return fail(c, ZTP_ESHAPE, "ztp_core: " + shp("qkv_t", *qkv) + " " + shp("ctx_t", *cx));
  if (qkv->dtype == ZTP_BF16 && qkv->cols % 8) return fail(c, ZTP_ESHAPE, "ztp_core: N % 8 != 0");
  const int pe = prof_begin(c, (cudaStream_t)stream, PROF_OTHER, 0.0);
  if (!(c->dbg_skip & 4)) {
    CUDA_TRY(c, ztp::core_launch(phase == ZTP_FWD ? 0 : 1, qkv->ptr, qkv->ld, cx->ptr, cx->ld, feat, n_out, qkv->cols,
                                 qkv->dtype, (phase == ZTP_FWD || v_compact) ? rows : nullptr, n_v, v_compact ? 1 : 0,
                                 (cudaStream_t)stream, !(c->side_pending && c->squat_guard)));
  }
  prof_end(c, pe, (cudaStream_t)stream);
  ++c->launches;
  return ZTP_OK;
}

ztp_status ztp_migrate(ztp_ctx* c, int n, const ztp_xfer* xs, void* stream) {
  if (!c || (n > 0 && !xs)) return fail(c, ZTP_EINVAL, "ztp_migrate: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  {
    ztp_status js = join_side(c, st);   // returned dW slices must be complete
    if (js != ZTP_OK) return js;
  }
  // one-sided peer pulls whenever the symmetric window is open (also under
  // the NCCL transport for the collectives): no staging copies
  const bool peer = c->world > 1 && (c->transport == ZTP_TRANSPORT_PEER || c->win_open);
  std::vector<size_t> off(n, 0);
  size_t total = 0;
  for (int i = 0; i < n; ++i) {
    const ztp_xfer& x = xs[i];
    if (x.src_rank < 0 || x.src_rank >= c->world || x.dst_rank < 0 || x.dst_rank >= c->world || x.nr < 0 || x.nc < 0)
      return fail(c, ZTP_EINVAL, "ztp_migrate: transfer " + std::to_string(i) + " has bad ranks/sizes");
    const bool me_src = x.src_rank == c->rank, me_dst = x.dst_rank == c->rank;
    if (me_src && (!mat_ok(x.src) || x.r0 + x.nr > x.src.rows || x.c0 + x.nc > x.src.cols))
      return fail(c, ZTP_ESHAPE, "ztp_migrate: source slice outside " + shp("src", x.src));
    if (me_dst && (!mat_ok(x.dst) || x.dr0 + x.nr > x.dst.rows || x.dc0 + x.nc > x.dst.cols))
      return fail(c, ZTP_ESHAPE, "ztp_migrate: destination slice outside " + shp("dst", x.dst));
    if (me_src && me_dst && x.src.dtype != x.dst.dtype) return fail(c, ZTP_ESHAPE, "ztp_migrate: dtype mismatch");
    const int dt = me_src ? x.src.dtype : x.dst.dtype;
    const size_t es = dt == ZTP_F32 ? 4 : 2;
    off[i] = total;
    if ((me_src || me_dst) && x.src_rank != x.dst_rank && !peer)
      total += ((size_t)x.nr * x.nc * es + 255) & ~size_t(255);
  }
  if (total && ensure_ws(c, total) != ZTP_OK) return ZTP_ECUDA;
  char* ws = (char*)c->ws;
  // local copies and packing of outgoing slices
  for (int i = 0; i < n; ++i) {
    const ztp_xfer& x = xs[i];
    if (x.nr == 0 || x.nc == 0) continue;
    const size_t es = (x.src_rank == c->rank ? x.src.dtype : x.dst.dtype) == ZTP_F32 ? 4 : 2;
    if (x.src_rank == c->rank && x.dst_rank == c->rank) {
      CUDA_TRY(c, cudaMemcpy2DAsync((char*)x.dst.ptr + (x.dr0 * x.dst.ld + x.dc0) * es, x.dst.ld * es,
                                    (const char*)x.src.ptr + (x.r0 * x.src.ld + x.c0) * es, x.src.ld * es, x.nc * es,
                                    x.nr, cudaMemcpyDeviceToDevice, st));
    } else if (x.src_rank == c->rank && !peer) {
      CUDA_TRY(c, cudaMemcpy2DAsync(ws + off[i], x.nc * es, (const char*)x.src.ptr + (x.r0 * x.src.ld + x.c0) * es,
                                    x.src.ld * es, x.nc * es, x.nr, cudaMemcpyDeviceToDevice, st));
    }
  }
  if (peer) {
    // one-sided pulls (P:237 peer copies): the destination reads the source
    // rank's window at the symmetric offset of its own counterpart of `src`;
    // no packing, no staging.  Every rank launches the same number of pull
    // rounds (computed from the common list) since they carry barriers.
    int per_rank[ZTP_MAX_RANKS] = {0};
    for (int i = 0; i < n; ++i)
      if (xs[i].nr > 0 && xs[i].nc > 0 && xs[i].src_rank != xs[i].dst_rank) ++per_rank[xs[i].dst_rank];
    int rounds = 0;
    for (int q = 0; q < c->world; ++q)
      rounds = std::max(rounds, (per_rank[q] + ztp::PEER_MAX_PULLS - 1) / ztp::PEER_MAX_PULLS);
    std::vector<ztp::PeerPull> mine;
    for (int i = 0; i < n; ++i) {
      const ztp_xfer& x = xs[i];
      if (x.nr == 0 || x.nc == 0 || x.src_rank == x.dst_rank || x.dst_rank != c->rank) continue;
      if (!mat_ok(x.src) || x.r0 + x.nr > x.src.rows || x.c0 + x.nc > x.src.cols || x.src.dtype != x.dst.dtype)
        return fail(c, ZTP_ESHAPE, "ztp_migrate (peer): the destination rank passes its own symmetric counterpart "
                                   "of the source, " + shp("src", x.src) + " does not cover the slice");
      const size_t es = x.dst.dtype == ZTP_F32 ? 4 : 2;
      int64_t off;
      ztp_status s = win_offset(c, x.src.ptr, (size_t)(x.src.rows * x.src.ld) * es, "ztp_migrate", &off);
      if (s != ZTP_OK) return s;
      mine.push_back(ztp::PeerPull{x.src_rank, (int32_t)es, off, x.r0, x.c0, x.nr, x.nc, x.src.ld, x.dst.ptr, x.dr0,
                                   x.dc0, x.dst.ld});
    }
    for (int rd = 0; rd < rounds; ++rd) {
      ztp::PeerPulls P{};
      for (int k = rd * ztp::PEER_MAX_PULLS; k < (int)mine.size() && P.n < ztp::PEER_MAX_PULLS; ++k) P.x[P.n++] = mine[k];
      CUDA_TRY(c, ztp::peer_pull_launch(c->pw, P, c->peer_ctas, st));
      ++c->launches;
    }
    return ZTP_OK;
  }
  if (c->world > 1) {
    NCCL_TRY(c, ncclGroupStart());
    for (int i = 0; i < n; ++i) {
      const ztp_xfer& x = xs[i];
      if (x.nr == 0 || x.nc == 0 || x.src_rank == x.dst_rank) continue;
      const int dt = x.src_rank == c->rank ? x.src.dtype : x.dst.dtype;
      const size_t cnt = (size_t)x.nr * x.nc;
      if (x.src_rank == c->rank) NCCL_TRY(c, ncclSend(ws + off[i], cnt, nccl_type(dt), x.dst_rank, c->comm, st));
      if (x.dst_rank == c->rank) NCCL_TRY(c, ncclRecv(ws + off[i], cnt, nccl_type(dt), x.src_rank, c->comm, st));
    }
    NCCL_TRY(c, ncclGroupEnd());
  }
  for (int i = 0; i < n; ++i) {
    const ztp_xfer& x = xs[i];
    if (x.nr == 0 || x.nc == 0 || x.src_rank == x.dst_rank || x.dst_rank != c->rank) continue;
    const size_t es = x.dst.dtype == ZTP_F32 ? 4 : 2;
    CUDA_TRY(c, cudaMemcpy2DAsync((char*)x.dst.ptr + (x.dr0 * x.dst.ld + x.dc0) * es, x.dst.ld * es, ws + off[i],
                                  x.nc * es, x.nc * es, x.nr, cudaMemcpyDeviceToDevice, st));
  }
  return ZTP_OK;
}

ztp_status ztp_window_create(ztp_ctx* c, size_t bytes, unsigned char handle[ZTP_IPC_BYTES]) {
  if (!c || !handle) return fail(c, ZTP_EINVAL, "ztp_window_create: null argument");
  if (c->win) return fail(c, ZTP_EINVAL, "ztp_window_create: the context already has a window");
  bytes = ((bytes + 4095) & ~size_t(4095)) + ztp::PEER_RESERVED;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMalloc(&c->win, bytes));
  CUDA_TRY(c, cudaMemset(c->win, 0, bytes));
  CUDA_TRY(c, cudaMalloc(&c->pw.ep, ztp::PEER_MAX_CTAS * sizeof(uint32_t)));
  CUDA_TRY(c, cudaMemset(c->pw.ep, 0, ztp::PEER_MAX_CTAS * sizeof(uint32_t)));
  c->win_bytes = bytes;
  c->win_used = ztp::PEER_RESERVED;
  std::memset(handle, 0, ZTP_IPC_BYTES);
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->win));
  static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "IPC handle size");
  std::memcpy(handle, &h, sizeof h);
  const uint64_t raw = reinterpret_cast<uint64_t>(c->win);
  const int32_t pid = (int32_t)getpid(), dev = c->device;
  const uint64_t nb = bytes;
  std::memcpy(handle + 64, &raw, 8);
  std::memcpy(handle + 72, &pid, 4);
  std::memcpy(handle + 76, &dev, 4);
  std::memcpy(handle + 80, &nb, 8);
  return ZTP_OK;
}

ztp_status ztp_window_open(ztp_ctx* c, const unsigned char* handles) {
  if (!c || !handles) return fail(c, ZTP_EINVAL, "ztp_window_open: null argument");
  if (!c->win) return fail(c, ZTP_EINVAL, "ztp_window_open: create the window first");
  if (c->win_open) return fail(c, ZTP_EINVAL, "ztp_window_open: already open");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int32_t mypid = (int32_t)getpid();
  ztp::PeerWin w{};
  w.rank = c->rank;
  w.world = c->world;
  for (int q = 0; q < c->world; ++q) {
    const unsigned char* h = handles + (size_t)q * ZTP_IPC_BYTES;
    uint64_t raw, nb;
    int32_t pid, dev;
    std::memcpy(&raw, h + 64, 8);
    std::memcpy(&pid, h + 72, 4);
    std::memcpy(&dev, h + 76, 4);
    std::memcpy(&nb, h + 80, 8);
    if (nb != c->win_bytes)
      return fail(c, ZTP_ESHAPE, "ztp_window_open: rank " + std::to_string(q) + "'s window has " +
                                     std::to_string(nb) + " bytes, mine " + std::to_string(c->win_bytes));
    if (q == c->rank) {
      w.base[q] = c->win;
    } else if (pid == mypid) {   // another context of this process: the pointer itself
      if (dev != c->device) {
        const cudaError_t pe = cudaDeviceEnablePeerAccess(dev, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
          return fail(c, ZTP_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(pe));
        cudaGetLastError();
      }
      w.base[q] = reinterpret_cast<char*>(raw);
    } else {
      cudaIpcMemHandle_t ih;
      std::memcpy(&ih, h, sizeof ih);
      void* p = nullptr;
      CUDA_TRY(c, cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
      c->win_ipc[q] = p;
      w.base[q] = static_cast<char*>(p);
    }
    w.flags[q] = reinterpret_cast<uint32_t*>(w.base[q] + ztp::PEER_FLAGS_OFF);
  }
  w.ep = c->pw.ep;
  w.err = c->d_flags + 1;
  c->pw = w;
  c->win_open = true;
  return ZTP_OK;
}

ztp_status ztp_sym_alloc(ztp_ctx* c, size_t bytes, void** ptr) {
  if (!c || !ptr) return fail(c, ZTP_EINVAL, "ztp_sym_alloc: null argument");
  *ptr = nullptr;
  if (!c->win) return fail(c, ZTP_EINVAL, "ztp_sym_alloc: create the window first");
  const size_t at = (c->win_used + 255) & ~size_t(255);
  if (at + bytes > c->win_bytes)
    return fail(c, ZTP_EINVAL, "ztp_sym_alloc: window exhausted (" + std::to_string(c->win_bytes - at) + " bytes left, " +
                                   std::to_string(bytes) + " asked)");
  c->win_used = at + bytes;
  *ptr = c->win + at;
  return ZTP_OK;
}

ztp_status ztp_set_transport(ztp_ctx* c, int transport) {
  if (!c || (transport != ZTP_TRANSPORT_NCCL && transport != ZTP_TRANSPORT_PEER))
    return fail(c, ZTP_EINVAL, "ztp_set_transport: unknown transport");
  if (transport == ZTP_TRANSPORT_NCCL && c->world > 1 && !c->comm)
    return fail(c, ZTP_EINVAL, "ztp_set_transport: this context has no NCCL communicator");
  c->transport = transport;
  return ZTP_OK;
}

ztp_status ztp_broadcast(ztp_ctx* c, int root, const ztp_mat* t, int mode, void* stream) {
  if (!c || !t) return fail(c, ZTP_EINVAL, "ztp_broadcast: null argument");
  if (root < 0 || root >= c->world || (mode != ZTP_COLL_TREE && mode != ZTP_COLL_P2P))
    return fail(c, ZTP_EINVAL, "ztp_broadcast: bad root / mode");
  if (!mat_ok(*t) || t->ld != t->cols) return fail(c, ZTP_ESHAPE, "ztp_broadcast: contiguous tensor needed, " + shp("t", *t));
  if (c->world == 1) return ZTP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = t->dtype == ZTP_F32 ? 4 : 2;
  const size_t n = (size_t)(t->rows * t->cols), bytes = n * es;
  const int pe = prof_begin(c, st, PROF_COMM, 0.0);
  if (c->transport == ZTP_TRANSPORT_PEER) {
    int64_t off;
    ztp_status s = win_offset(c, t->ptr, bytes, "ztp_broadcast", &off);
    if (s != ZTP_OK) return s;
    if (bytes % 16) return fail(c, ZTP_ESHAPE, "peer broadcast: payload must be a multiple of 16 bytes");
    CUDA_TRY(c, ztp::peer_bcast_launch(c->pw, root, off, (int64_t)bytes, c->peer_ctas, st));
    ++c->launches;
  } else if (mode == ZTP_COLL_TREE) {
    NCCL_TRY(c, ncclBroadcast(t->ptr, t->ptr, n, nccl_type(t->dtype), root, c->comm, st));
  } else {
    NCCL_TRY(c, ncclGroupStart());
    if (c->rank == root) {
      for (int q = 0; q < c->world; ++q)
        if (q != root) NCCL_TRY(c, ncclSend(t->ptr, n, nccl_type(t->dtype), q, c->comm, st));
    } else {
      NCCL_TRY(c, ncclRecv(t->ptr, n, nccl_type(t->dtype), root, c->comm, st));
    }
    NCCL_TRY(c, ncclGroupEnd());
  }
  prof_end(c, pe, st);
  return ZTP_OK;
}

ztp_status ztp_reduce(ztp_ctx* c, int root, const ztp_mat* t, int mode, void* stream) {
  if (!c || !t) return fail(c, ZTP_EINVAL, "ztp_reduce: null argument");
  if (root < 0 || root >= c->world || (mode != ZTP_COLL_TREE && mode != ZTP_COLL_P2P))
    return fail(c, ZTP_EINVAL, "ztp_reduce: bad root / mode");
  if (!mat_ok(*t) || t->ld != t->cols) return fail(c, ZTP_ESHAPE, "ztp_reduce: contiguous tensor needed, " + shp("t", *t));
  if (c->world == 1) return ZTP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = t->dtype == ZTP_F32 ? 4 : 2;
  const size_t n = (size_t)(t->rows * t->cols), bytes = n * es;
  const int pe = prof_begin(c, st, PROF_COMM, 0.0);
  if (c->transport == ZTP_TRANSPORT_PEER) {
    int64_t off;
    ztp_status s = win_offset(c, t->ptr, bytes, "ztp_reduce", &off);
    if (s != ZTP_OK) return s;
    if (bytes % 16) return fail(c, ZTP_ESHAPE, "peer reduce: payload must be a multiple of 16 bytes");
    CUDA_TRY(c, ztp::peer_reduce_launch(c->pw, root, off, (int64_t)bytes, t->dtype == ZTP_F32, c->peer_ctas, st));
    ++c->launches;
  } else if (mode == ZTP_COLL_TREE) {
    NCCL_TRY(c, ncclReduce(t->ptr, t->ptr, n, nccl_type(t->dtype), ncclSum, root, c->comm, st));
  } else {
    // gather every rank's tensor into the root's workspace, then the root
    // sums them in rank order (its own copy included) into t
    if (c->rank == root && ensure_ws(c, bytes * c->world) != ZTP_OK) return ZTP_ECUDA;
    char* ws = (char*)c->ws;
    if (c->rank == root)
      CUDA_TRY(c, cudaMemcpyAsync(ws + (size_t)root * bytes, t->ptr, bytes, cudaMemcpyDeviceToDevice, st));
    NCCL_TRY(c, ncclGroupStart());
    if (c->rank == root) {
      for (int q = 0; q < c->world; ++q)
        if (q != root) NCCL_TRY(c, ncclRecv(ws + (size_t)q * bytes, n, nccl_type(t->dtype), q, c->comm, st));
    } else {
      NCCL_TRY(c, ncclSend(t->ptr, n, nccl_type(t->dtype), root, c->comm, st));
    }
    NCCL_TRY(c, ncclGroupEnd());
    if (c->rank == root) {
      CUDA_TRY(c, ztp::accumulate_launch(t->ptr, t->cols, ws, t->cols, t->rows, t->cols, t->dtype, c->world, t->rows,
                                         1, st));
      ++c->launches;
    }
  }
  prof_end(c, pe, st);
  return ZTP_OK;
}

ztp_status ztp_allreduce(ztp_ctx* c, const ztp_mat* t, void* stream) {
  if (!c || !t) return fail(c, ZTP_EINVAL, "ztp_allreduce: null argument");
  if (!mat_ok(*t)) return fail(c, ZTP_ESHAPE, "ztp_allreduce: bad " + shp("t", *t));
  return allreduce(c, *t, (cudaStream_t)stream);
}

ztp_status ztp_accumulate(ztp_ctx* c, const ztp_mat* dst, const ztp_mat* src, void* stream) {
  if (!c || !dst || !src) return fail(c, ZTP_EINVAL, "ztp_accumulate: null argument");
  if (!mat_ok(*dst) || !mat_ok(*src) || dst->rows != src->rows || dst->cols != src->cols || dst->dtype != src->dtype)
    return fail(c, ZTP_ESHAPE, "ztp_accumulate: " + shp("dst", *dst) + " vs " + shp("src", *src));
  CUDA_TRY(c, ztp::accumulate_launch(dst->ptr, dst->ld, src->ptr, src->ld, dst->rows, dst->cols, dst->dtype, 1, 0, 0,
                                     (cudaStream_t)stream));
  ++c->launches;
  return ZTP_OK;
}

ztp_status ztp_transpose(ztp_ctx* c, const ztp_mat* src, const ztp_mat* dst, const int32_t* cols, int64_t n,
                         void* stream) {
  if (!c || !src || !dst) return fail(c, ZTP_EINVAL, "ztp_transpose: null argument");
  if (!mat_ok(*src) || !mat_ok(*dst) || src->dtype != ZTP_BF16 || dst->dtype != ZTP_BF16 || n < 0 ||
      dst->rows < n || dst->cols < src->rows || (!cols && n > src->cols))
    return fail(c, ZTP_ESHAPE, "ztp_transpose: " + shp("src", *src) + " -> " + shp("dst", *dst) + " n " +
                                   std::to_string(n));
  const int pe = prof_begin(c, (cudaStream_t)stream, PROF_OTHER, 0.0);
  CUDA_TRY(c, ztp::transpose_launch(src->ptr, src->ld, src->rows, cols, n, dst->ptr, dst->ld, (cudaStream_t)stream));
  prof_end(c, pe, (cudaStream_t)stream);
  ++c->launches;
  return ZTP_OK;
}

ztp_status ztp_set_option(ztp_ctx* c, ztp_option opt, double v) {
  if (!c) return fail(c, ZTP_EINVAL, "ztp_set_option: null ctx");
  if (!std::isfinite(v)) return fail(c, ZTP_EINVAL, "ztp_set_option: value must be finite");
  const int iv = (int)v;
  switch (opt) {
    case ZTP_OPT_CONC: c->conc_bwd = iv != 0; return ZTP_OK;
    case ZTP_OPT_DW_SHARE:
      if (!(v > 0.0)) return fail(c, ZTP_EINVAL, "ztp_set_option: dW share must be > 0");
      c->dw_share = v;
      return ZTP_OK;
    case ZTP_OPT_SQUAT_GUARD: c->squat_guard = iv != 0; return ZTP_OK;
    case ZTP_OPT_GATHER4: c->use_gather4 = iv != 0; return ZTP_OK;
    case ZTP_OPT_SPLITK: c->allow_splitk = iv != 0; return ZTP_OK;
    case ZTP_OPT_GROUP:
      if (iv < 0 || iv > 2) return fail(c, ZTP_EINVAL, "ztp_set_option: group mode is 0, 1 or 2");
      c->group_bwd = iv;
      return ZTP_OK;
    case ZTP_OPT_PEER_CTAS:
      if (iv < 1 || iv > ztp::PEER_MAX_CTAS) return fail(c, ZTP_EINVAL, "ztp_set_option: peer CTAs out of range");
      c->peer_ctas = iv;
      return ZTP_OK;
    case ZTP_OPT_A_EARLY: c->a_early = iv != 0; return ZTP_OK;
    case ZTP_OPT_PART:
      if (iv < 0 || iv > 2) return fail(c, ZTP_EINVAL, "ztp_set_option: partition model is 0, 1 or 2");
      c->part_model = iv;
      return ZTP_OK;
    case ZTP_OPT_AUX_WEIGHT:
      if (!(v > 0.0)) return fail(c, ZTP_EINVAL, "ztp_set_option: aux weight must be > 0");
      c->aux_weight = v;
      return ZTP_OK;
    case ZTP_OPT_FLAGS: c->flags_opt = iv != 0; return ZTP_OK;
    case ZTP_OPT_SPREAD_EPI: c->spread_epi = iv != 0; return ZTP_OK;
    case ZTP_OPT_ZERO_GENERIC: c->zero_generic = iv != 0; return ZTP_OK;
    case ZTP_OPT_TAIL_HALVES: c->tail_halves = iv != 0; return ZTP_OK;
  }
  return fail(c, ZTP_EINVAL, "ztp_set_option: unknown option " + std::to_string((int)opt));
}

ztp_status ztp_get_option(const ztp_ctx* c, ztp_option opt, double* v) {
  if (!c || !v) return fail(nullptr, ZTP_EINVAL, "ztp_get_option: null argument");
  switch (opt) {
    case ZTP_OPT_CONC: *v = c->conc_bwd; return ZTP_OK;
    case ZTP_OPT_DW_SHARE: *v = c->dw_share; return ZTP_OK;
    case ZTP_OPT_SQUAT_GUARD: *v = c->squat_guard; return ZTP_OK;
    case ZTP_OPT_GATHER4: *v = c->use_gather4; return ZTP_OK;
    case ZTP_OPT_SPLITK: *v = c->allow_splitk; return ZTP_OK;
    case ZTP_OPT_GROUP: *v = c->group_bwd; return ZTP_OK;
    case ZTP_OPT_PEER_CTAS: *v = c->peer_ctas; return ZTP_OK;
    case ZTP_OPT_A_EARLY: *v = c->a_early; return ZTP_OK;
    case ZTP_OPT_PART: *v = c->part_model; return ZTP_OK;
    case ZTP_OPT_AUX_WEIGHT: *v = c->aux_weight; return ZTP_OK;
    case ZTP_OPT_FLAGS: *v = c->flags_opt; return ZTP_OK;
    case ZTP_OPT_SPREAD_EPI: *v = c->spread_epi; return ZTP_OK;
    case ZTP_OPT_ZERO_GENERIC: *v = c->zero_generic; return ZTP_OK;
    case ZTP_OPT_TAIL_HALVES: *v = c->tail_halves; return ZTP_OK;
  }
  return fail(nullptr, ZTP_EINVAL, "ztp_get_option: unknown option " + std::to_string((int)opt));
}

ztp_status ztp_barrier(ztp_ctx* c, void* stream) {
  if (!c) return fail(c, ZTP_EINVAL, "ztp_barrier: null ctx");
  if (c->world == 1) return ZTP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (c->transport == ZTP_TRANSPORT_PEER) {
    if (!c->win_open) return fail(c, ZTP_EINVAL, "ztp_barrier: open the peer window first");
    CUDA_TRY(c, ztp::peer_barrier_launch(c->pw, 1, st));
    ++c->launches;
    return ZTP_OK;
  }
  if (!c->d_one) CUDA_TRY(c, cudaMalloc(&c->d_one, 16));
  NCCL_TRY(c, ncclAllReduce(c->d_one, c->d_one, 1, ncclFloat, ncclSum, c->comm, st));
  return ZTP_OK;
}

ztp_status ztp_set_profile(ztp_ctx* c, int on) {
  if (!c) return fail(c, ZTP_EINVAL, "ztp_set_profile: null ctx");
  c->prof_on = (on == 2 || on == 3) ? on : (on ? 1 : 0);
  if (on == 3 && !c->d_ctastamp) {
    const size_t bytes = (size_t)ztp_ctx::CTASTAMP_LAUNCHES * ztp_ctx::CTASTAMP_PER_LAUNCH * sizeof(unsigned long long);
    CUDA_TRY(c, cudaMalloc(&c->d_ctastamp, bytes));
    CUDA_TRY(c, cudaMemset(c->d_ctastamp, 0, bytes));
  }
  if (!on) c->pstamp_used = 0;
  if (on && !c->d_pstamp) CUDA_TRY(c, cudaMalloc(&c->d_pstamp, 2 * ztp_ctx::PSTAMP_CAP * sizeof(unsigned long long)));
  if (on) {
    CUDA_TRY(c, cudaMemset(c->d_pstamp, 0, 2 * ztp_ctx::PSTAMP_CAP * sizeof(unsigned long long)));
    c->pstamp_used = 0;
  }
  return ZTP_OK;
}

ztp_status ztp_read_profile(ztp_ctx* c, void* stream, ztp_profile* out) {
  if (!c || !out) return fail(c, ZTP_EINVAL, "ztp_read_profile: null argument");
  CUDA_TRY(c, cudaStreamSynchronize((cudaStream_t)stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->comm_stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->side_stream));
  std::memset(out, 0, sizeof(*out));
  for (size_t i = 0; i < c->prof_used; ++i) {
    float ms = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, c->prof[i].a, c->prof[i].b));
    if (c->prof[i].cat == PROF_GEMM) {
      out->gemm_ms += ms;
      out->gemm_flops += c->prof[i].flops;
      ++out->n_gemm;
    } else if (c->prof[i].cat == PROF_OTHER) {
      out->other_ms += ms;
      ++out->n_other;
    } else {
      out->comm_ms += ms;
      ++out->n_comm;
    }
  }
  c->prof_used = 0;
  if (c->pstamp_used > 0) {
    std::vector<unsigned long long> h(2 * (size_t)c->pstamp_used);
    CUDA_TRY(c, cudaMemcpy(h.data(), c->d_pstamp, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    // GEMM kernel time = length of the UNION of the launches' [start, end]
    // intervals (launches overlap under PDL; a sum would count it twice)
    std::vector<std::pair<unsigned long long, unsigned long long>> iv;
    for (int i = 0; i < c->pstamp_used; ++i) {
      const unsigned long long t0 = ~h[2 * i], t1 = h[2 * i + 1];
      if (h[2 * i] != 0 && t1 >= t0) {
        iv.emplace_back(t0, t1);
        if (c->prof_on >= 2) {
          out->gemm_flops += c->pstamp_flops[i];
          ++out->n_gemm;
        }
      }
    }
    std::sort(iv.begin(), iv.end());
    if (!iv.empty()) {
      unsigned long long cs = iv[0].first, ce = iv[0].second;
      for (size_t k = 1; k < iv.size(); ++k) {
        if (iv[k].first > ce) {
          out->gemm_kernel_ms += (double)(ce - cs) * 1e-6;
          cs = iv[k].first;
          ce = iv[k].second;
        } else if (iv[k].second > ce) {
          ce = iv[k].second;
        }
      }
      out->gemm_kernel_ms += (double)(ce - cs) * 1e-6;
    }
    CUDA_TRY(c, cudaMemset(c->d_pstamp, 0, h.size() * sizeof(unsigned long long)));
    // mode 2 keeps its slots: a captured graph writes the same ones every replay
    if (c->prof_on < 2) c->pstamp_used = 0;
  }
  return ZTP_OK;
}

int ztp_read_stamps(ztp_ctx* c, void* stream, unsigned long long* out, int max_launches) {
  if (!c || !out || max_launches < 0) return -1;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return -1;
  const int n = std::min(c->pstamp_used, max_launches);
  if (n <= 0 || !c->d_pstamp) return 0;
  if (cudaMemcpy(out, c->d_pstamp, 2 * (size_t)n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  for (int i = 0; i < n; ++i) out[2 * i] = ~out[2 * i];
  return n;
}

ztp_status ztp_set_slowdown(ztp_ctx* c, double chi) {
  if (!c || !(chi >= 1.0)) return fail(c, ZTP_EINVAL, "ztp_set_slowdown: chi must be >= 1");
  c->chi = chi;
  return ZTP_OK;
}

ztp_status ztp_set_stats(ztp_ctx* c, int on) {
  if (!c) return fail(c, ZTP_EINVAL, "ztp_set_stats: null ctx");
  c->stats = on ? 1 : 0;
  return ZTP_OK;
}

int ztp_read_cta_stamps(ztp_ctx* c, void* stream, unsigned long long* out, int max_launches) {
  if (!c || !out || max_launches < 0 || !c->d_ctastamp) return -1;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return -1;
  const int n = std::min(std::min(c->pstamp_used, max_launches), ztp_ctx::CTASTAMP_LAUNCHES);
  if (n <= 0) return 0;
  const size_t cnt = (size_t)n * ztp_ctx::CTASTAMP_PER_LAUNCH;
  if (cudaMemcpy(out, c->d_ctastamp, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

ztp_status ztp_read_gemm_ns(ztp_ctx* c, void* stream, double* ns) {
  if (!c || !ns) return fail(c, ZTP_EINVAL, "ztp_read_gemm_ns: null argument");
  CUDA_TRY(c, cudaStreamSynchronize((cudaStream_t)stream));
  unsigned long long v = 0;
  CUDA_TRY(c, cudaMemcpy(&v, c->d_gemm_ns, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemset(c->d_gemm_ns, 0, 8));
  *ns = (double)v;
  return ZTP_OK;
}

}  // extern "C"

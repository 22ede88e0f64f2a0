/*
 * ztp.h -- C ABI of the straggler-balanced 1D tensor-parallel linear layer
 * (ZERO-resizing + SEMI-migration, arXiv 2401.11469) on B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (Alg.1 l.k = P:202+k, Alg.2 l.k = P:293+k);
 * S:n = SPEC.md line n; A-n = the reading of an ambiguous passage listed in
 * DESIGN.md ("Readings").
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  - Indices are 0-based.  Ranks are 0..world-1.
 *  - Layout: every tensor indexed by the pruned
 *    contraction dimension K is stored with K as its OUTER (row) dimension:
 *      x_t  [K, N]   input, feature-major (paper's input [bs*sql, K] transposed)
 *      w_t  [K, n]   weight shard W^T     (paper's weight [n, K] transposed)
 *      y_t  [n, N]   output, g_t [n, N] upstream gradient (paper's grad_input)
 *      dx_t [K, N]   input gradient (paper's grad_output), dw_t [K, n]
 *    Row-major, `ld` = elements between consecutive rows (>= cols, multiple
 *    of 8 for bf16 so rows are 16-byte aligned), base pointer 16-byte aligned.
 *  - Ownership: the caller owns every buffer passed in (device memory for
 *    tensors and index lists, host memory for h_* arguments and results) and
 *    every stream.  The library never frees caller memory.  The context owns
 *    its NCCL communicator, cached TMA descriptors and workspaces.
 *  - Streams are `cudaStream_t` passed as `void*` (NULL = legacy default).
 *    Device work is enqueued asynchronously on that stream; host-side checks
 *    run before anything is enqueued, and on error NOTHING is enqueued and
 *    ztp_last_error() names the offending shapes/values.
 *  - Asynchronous CUDA / NCCL failures are reported as ZTP_ECUDA / ZTP_ENCCL
 *    by the next call that observes them (ztp_sync() forces the check).
 *  - There is no CPU fallback: every compute step runs in this library's
 *    CUDA kernels (or NCCL); a missing device is ZTP_ECUDA.
 */
#ifndef ZTP_H_
#define ZTP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZTP_MAX_RANKS 8
#define ZTP_UID_BYTES 128
#define ZTP_IPC_BYTES 128

typedef enum ztp_status {
  ZTP_OK = 0,
  ZTP_EINVAL = 1,        /* bad argument value (NaN score, < 2 cost samples, empty T: S:549) */
  ZTP_ESHAPE = 2,        /* shapes / leading dimensions inconsistent */
  ZTP_EINDEX = 3,        /* index outside [0, K) */
  ZTP_EDEGENERATE = 4,   /* #P >= K: nothing would survive */
  ZTP_ELINEAGE = 5,      /* BWD selection differs from the FWD lineage entry */
  ZTP_EHISTORY = 6,      /* Same imputation without history */
  ZTP_ENOBASELINE = 7,   /* M_i = 0 in Eq.1 */
  ZTP_ENOHELPER = 8,     /* migration with world = 1 */
  ZTP_ERECEIVERS = 9,    /* e - x = 0 receivers */
  ZTP_ECUDA = 10,
  ZTP_ENCCL = 11,
  ZTP_EUNSUPPORTED = 12
} ztp_status;

typedef enum ztp_dtype { ZTP_BF16 = 0, ZTP_F32 = 1 } ztp_dtype;

/* A row-major 2-D device matrix.  rows = outer dimension. */
typedef struct ztp_mat {
  void* ptr;
  int64_t rows, cols, ld;
  int32_t dtype;           /* ztp_dtype */
  int32_t _pad;
} ztp_mat;

typedef struct ztp_ctx ztp_ctx; /* one per rank / process / device */

const char* ztp_status_str(ztp_status s);
/* Last error message of `ctx` (ctx may be NULL: the calling thread's last
 * error from a context-free call).  Valid until the next call. */
const char* ztp_last_error(const ztp_ctx* ctx);
/* Version string, e.g. "ztp 0.1 sm_100a". */
const char* ztp_version(void);

/* ---------------------------------------------------------------------------
 * Context.  world == 1 needs no NCCL id (uid may be NULL).  For world > 1,
 * rank 0 calls ztp_get_unique_id() and the caller distributes the 128 bytes to
 * every rank (e.g. torch.distributed.broadcast); every rank then calls
 * ztp_ctx_create with its own rank and the CUDA device it owns.  Collective:
 * all ranks must call it.  The communicator is NCCL over NVLink/NVSwitch.
 * world > 1 with uid == NULL creates a context without NCCL whose data plane
 * is the peer-memory transport below (ztp_window_*).
 * ------------------------------------------------------------------------- */
ztp_status ztp_get_unique_id(unsigned char uid[ZTP_UID_BYTES]);
ztp_status ztp_ctx_create(ztp_ctx** out, int rank, int world,
                          const unsigned char* uid /* ZTP_UID_BYTES or NULL */, int device);
ztp_status ztp_ctx_destroy(ztp_ctx* ctx);
/* Blocks until `stream` drains and reports pending asynchronous errors
 * (including device-side flags such as a NaN score seen by ztp_select). */
ztp_status ztp_sync(ztp_ctx* ctx, void* stream);
/* Number of kernels this context launched so far (own kernels only). */
int64_t ztp_launch_count(const ztp_ctx* ctx);

/* ---------------------------------------------------------------------------
 * Peer-memory data plane (SURVEY §8(b) ztp_sym_alloc).
 * Every rank owns one symmetric window: ztp_window_create allocates it
 * (bytes + 64 KB of barrier flags) and writes a ZTP_IPC_BYTES handle (CUDA
 * IPC handle, pointer, pid, device, size); the caller all-gathers the handles
 * of every rank (rank order, e.g. torch.distributed.all_gather_object) and
 * calls ztp_window_open on every rank, which maps each peer's window (CUDA IPC
 * across processes, the pointer itself for contexts of one process, NVLink
 * P2P between GPUs).  ztp_sym_alloc carves caller tensors out of the window
 * (bump allocation, 256-byte aligned; the same call sequence on every rank
 * gives the same offsets, so a peer's copy of a tensor is found at the same
 * offset -- the library owns the memory, valid until ztp_ctx_destroy).
 * With ZTP_TRANSPORT_PEER (default for contexts created without an NCCL id):
 *   all-reduce (row FWD, col BWD) = two-shot over peer loads, summed
 *     in rank order 0..e-1 in fp32 (deterministic; the oracle's left fold);
 *   all-gather (unpaired mode) = pulls of the peers' row blocks;
 *   ztp_migrate = one-sided pulls of the source rank's slice, no
 *     staging copies;
 *   ztp_allgather_stats = stores into every peer's stats slot;
 * each a kernel whose CTA b meets CTA b of every peer at device-side
 * barriers (release / acquire, system scope), so it is graph-capturable; the
 * tensors involved must be window tensors (EINVAL otherwise).  A barrier not
 * met within 10 s raises a flag that ztp_sync reports as ZTP_ECUDA.
 * ZTP_TRANSPORT_NCCL: NCCL collectives and grouped send/recv.
 * Errors: EINVAL (no window / not open / exhausted / tensor outside it),
 * ESHAPE (window sizes differ across ranks), ECUDA.
 * ------------------------------------------------------------------------- */
enum { ZTP_TRANSPORT_NCCL = 0, ZTP_TRANSPORT_PEER = 1 };
ztp_status ztp_window_create(ztp_ctx* ctx, size_t bytes, unsigned char handle[ZTP_IPC_BYTES]);
ztp_status ztp_window_open(ztp_ctx* ctx, const unsigned char* handles /* world x ZTP_IPC_BYTES */);
ztp_status ztp_sym_alloc(ztp_ctx* ctx, size_t bytes, void** ptr);
ztp_status ztp_set_transport(ztp_ctx* ctx, int transport);
/* Device-side barrier of all ranks on `stream` (NCCL: a 1-element
 * all-reduce; peer: one barrier round).  Collective. */
ztp_status ztp_barrier(ztp_ctx* ctx, void* stream);

/* ---------------------------------------------------------------------------
 * Rooted collectives and the local reduce of the paper-literal migration
 * (NEXT-3; "sending-collecting migration", Table I).
 * Collective: every rank calls with the same root / shape / mode.
 * ztp_broadcast: every rank's t <- root's t.  ztp_reduce: root's t <- sum over
 * ranks of t (other ranks' t unchanged).  mode ZTP_COLL_TREE = the NCCL
 * collective (ncclBroadcast / ncclReduce: ring / tree / NVLS, many de facto
 * senders); ZTP_COLL_P2P = point to point (grouped ncclSend / ncclRecv: the
 * root sends the whole tensor to every rank / receives every rank's tensor
 * into the ctx workspace and sums them in rank order).  Under the peer
 * transport both modes are pulls (broadcast: every rank pulls the root's
 * window tensor; reduce: the root pulls every rank's and sums in rank order
 * 0..e-1 in fp32) and t must be a window tensor.  Contiguous t only (ld ==
 * cols).  Errors: EINVAL (root / mode / not in the window), ESHAPE, ENCCL.
 * ztp_accumulate: dst += src elementwise (same shape, fp32 add, one
 * rounding) -- a helper's migrated contribution merged into its own partial
 * before the all-reduce (the "reduce-merging" of P:248).
 * ------------------------------------------------------------------------- */
enum { ZTP_COLL_TREE = 0, ZTP_COLL_P2P = 1 };
ztp_status ztp_broadcast(ztp_ctx* ctx, int root, const ztp_mat* t, int mode, void* stream);
ztp_status ztp_reduce(ztp_ctx* ctx, int root, const ztp_mat* t, int mode, void* stream);
ztp_status ztp_accumulate(ztp_ctx* ctx, const ztp_mat* dst, const ztp_mat* src, void* stream);
/* The all-reduce (sum) the linears issue, for a caller that merges
 * extra contributions into its partial first (skip_collective = 1, then
 * ztp_accumulate, then this).  Contiguous t; peer transport: a window tensor. */
ztp_status ztp_allreduce(ztp_ctx* ctx, const ztp_mat* t, void* stream);

/* ---------------------------------------------------------------------------
 * Layout change for a token-major library kernel (the real attention core,
 * NEXT-4, runs cuDNN fused attention on [batch, seq, heads, head_dim]):
 *   dst[i, r] = src[r, cols ? cols[i] : i]   for i < n, r < src->rows
 * src [R, C], dst [>= n, >= R], bf16; cols (device, nullable) selects and
 * orders the source columns (e.g. the O projection's kept features S_o, so
 * the core's output lands compact in O's kept order).  Indices are not
 * range-checked on the device.  Errors: ESHAPE, ECUDA.
 * ------------------------------------------------------------------------- */
ztp_status ztp_transpose(ztp_ctx* ctx, const ztp_mat* src, const ztp_mat* dst, const int32_t* cols, int64_t n,
                         void* stream);

/* ---------------------------------------------------------------------------
 * Execution options of a context (performance scheduling only; results are
 * the same up to fp32 summation order within the stated tolerances).  Each
 * starts from its environment variable (read once by ztp_ctx_create) or the
 * default below; ztp_set_option overrides it for later calls.  Values are
 * doubles (integers for switches).  EINVAL on an unknown option / bad value.
 *   ZTP_OPT_CONC        (ZTP_CONC, 1)        dW GEMM on a side stream, concurrent with dX
 *   ZTP_OPT_DW_SHARE    (ZTP_DW_SHARE, 1.2)  weight of dW's MMA work in the dX / dW SM split
 *   ZTP_OPT_SQUAT_GUARD (ZTP_SQUAT_GUARD, 1) core kernel in stream order while a dW is pending
 *   ZTP_OPT_GATHER4     (ZTP_GATHER4, 0)     operand rows gathered by TMA gather4 inside the GEMM
 *   ZTP_OPT_SPLITK      (ZTP_SPLITK, 1)      split-K for few-tile GEMMs
 *   ZTP_OPT_GROUP       (ZTP_GROUP, 0)       0 / 1 / 2: dX + dW as one grouped launch never /
 *                                            always / only for small pairs
 *   ZTP_OPT_PEER_CTAS   (ZTP_PEER_CTAS, 32)  CTAs of a peer collective (same on every rank)
 *   ZTP_OPT_A_EARLY     (ZTP_A_EARLY, 1)     a GEMM right after a GEMM whose outputs do not overlap
 *                                            its A operand issues its first stages' A loads before
 *                                            the PDL wait (only B waits for the predecessor)
 *   ZTP_OPT_PART        (ZTP_PART, 1)        dX / dW SM partition: 0 work-proportional,
 *                                            1 wave-quantised (minimises the later finish of
 *                                            max(MMA k-blocks, epilogue incl. Zero tiles)),
 *                                            2 wave-quantised on MMA k-blocks only
 *   ZTP_OPT_AUX_WEIGHT  (ZTP_AUX_WEIGHT, 1.0) dX work factor in that partition when its epilogue
 *                                            reads an aux operand (GeLU')
 *   ZTP_OPT_FLAGS       (ZTP_FLAGS, 0)       a GEMM whose B operand is the output of the GEMM just
 *                                            before it on the stream waits per 256-column block
 *                                            on that GEMM's tile-completion counters instead of
 *                                            its PDL wait (measured slower: off by default)
 *   ZTP_OPT_SPREAD_EPI  (ZTP_SPREAD_EPI, 0)  an output-pruned dW without split-K (out_sel set) is
 *                                            written in full by the GEMM epilogue (lane = row: kept
 *                                            columns from the staged row, Zero units in between,
 *                                            16-byte stores); 0: compact scratch + a column-spread
 *                                            pass (measured: on par at c4, slower at c5 -- the
 *                                            scattered row stores make the epilogue L1-bound)
 *   ZTP_OPT_ZERO_GENERIC (ZTP_ZERO_GENERIC, 1) all-pruned (Zero) tiles of a dX / dW at a lineage row
 *                                            map are written by generic 16-byte stores (eight
 *                                            lanes per 128-byte row segment) instead of TMA
 *                                            scatter4 boxes
 *   ZTP_OPT_TAIL_HALVES (ZTP_TAIL_HALVES, 1) a FWD GEMM whose last round of 256 x 256 tiles fills at
 *                                            most half of the CTA pairs runs those tiles as two
 *                                            128-column halves each, on twice as many pairs
 * ------------------------------------------------------------------------- */
typedef enum ztp_option {
  ZTP_OPT_CONC = 0,
  ZTP_OPT_DW_SHARE = 1,
  ZTP_OPT_SQUAT_GUARD = 2,
  ZTP_OPT_GATHER4 = 3,
  ZTP_OPT_SPLITK = 4,
  ZTP_OPT_GROUP = 5,
  ZTP_OPT_PEER_CTAS = 6,
  ZTP_OPT_A_EARLY = 7,
  ZTP_OPT_PART = 8,
  ZTP_OPT_AUX_WEIGHT = 9,
  ZTP_OPT_FLAGS = 10,
  ZTP_OPT_SPREAD_EPI = 11,
  ZTP_OPT_ZERO_GENERIC = 12,
  ZTP_OPT_TAIL_HALVES = 13
} ztp_option;
ztp_status ztp_set_option(ztp_ctx* ctx, ztp_option opt, double value);
ztp_status ztp_get_option(const ztp_ctx* ctx, ztp_option opt, double* value);

/* ---------------------------------------------------------------------------
 * (1) Plan -- pure host, deterministic, no context, no device work.
 *
 * ztp_plan: per-rank runtimes T[e] and GEMM times M[e] (A-5, A-6) of the last
 * statistics window -> resize ratios and the migrate-or-resize decision.
 *   ZERO only (enable_migration = 0): Eq.1 with C = T_avg
 *     (zero_crit = AVG, Alg.1 l.1) or T_min (MIN); every rank with
 *     gamma > 0 resizes.
 *   SEMI (enable_migration = 1, Alg.2): stragglers are ranks with
 *     T > T_min (1 + eps) (A-17), ordered (T desc, rank asc) (A-21).
 *     z = 1: gamma <= gamma_tol -> resize; else beta by bisection on Eq.2
 *     (A-24), beta >= 1 - gamma_tol/gamma (A-23); phi = gamma beta,
 *     gamma_r = gamma (1-beta)/(1-gamma beta) (A-16).
 *     z > 1: Eq.3 scan (A-18..A-20): positions <= x migrate
 *     (phi = gamma), the rest resize with Eq.1 at T_min.
 *   L_ref: the reference column count of Eq.2/Eq.3 (A-25).
 * Every double is computed in a fixed order in IEEE fp64 without contraction,
 * so results are bit-identical on every rank and to the oracle.
 * Errors: EINVAL (world not in 1..8, T not finite / negative, cost function
 * with < 2 samples), ENOBASELINE (M_r <= 0 where Eq.1 is evaluated).
 * A-48: with costs given, a RESIZE rank whose Eq.1 saving gamma_r * M[r]
 * does not exceed costs->omega1 (the static resizing overhead) is
 * returned NORMAL with gamma 0 (timing noise above eps does not resize a
 * healthy task); costs == NULL or omega1 == 0 leaves the plan unfiltered.
 * ------------------------------------------------------------------------- */
typedef struct ztp_pwl {       /* piecewise linear, x ascending, linear extrapolation */
  int32_t n;
  const double* x;
  const double* y;
} ztp_pwl;

typedef struct ztp_costs {     /* Eq.2 / Eq.3 cost model (Alg.2 l.1 pretest) */
  double omega1;               /* static allocation overhead Omega_1 */
  ztp_pwl omega2;              /* dimension-extracting cost Omega_2(pruned columns) */
  ztp_pwl phi1;                /* communication cost Phi_1(migrated columns) */
  ztp_pwl phi2;                /* helper computation cost Phi_2(columns per helper) */
} ztp_costs;

typedef enum ztp_crit { ZTP_CRIT_AVG = 0, ZTP_CRIT_MIN = 1 } ztp_crit;

typedef struct ztp_plan_opts {
  int32_t enable_migration;    /* 0: ZERO-resizing only; 1: SEMI-migration */
  int32_t zero_crit;           /* ztp_crit for ZERO-only mode (A-7) */
  double gamma_max;            /* 0.9 (A-4) */
  double eps;                  /* 0.02 straggler tolerance (A-17) */
  double gamma_tol;            /* 0.5 resize-only bound (A-23) */
  int32_t bisect_iters;        /* 64 (A-24) */
  int32_t force_lambda;        /* -1 = Eq.3; >= 0 forces the migration group size */
} ztp_plan_opts;

typedef enum ztp_role { ZTP_NORMAL = 0, ZTP_RESIZE = 1, ZTP_MIGRATE = 2, ZTP_SPLIT = 3 } ztp_role;

typedef struct ztp_plan_t {
  int32_t world, z, x;
  int32_t order[ZTP_MAX_RANKS];       /* ranks sorted by (T desc, rank asc) */
  int32_t role[ZTP_MAX_RANKS];        /* ztp_role */
  double gamma[ZTP_MAX_RANKS];        /* Eq.1 ratio (clamped) */
  double beta[ZTP_MAX_RANKS];         /* migrated share of the shed work (Eq.2) */
  double phi[ZTP_MAX_RANKS];          /* migrated fraction of hidden units = gamma beta */
  double gamma_r[ZTP_MAX_RANKS];      /* prune ratio of the remaining work (A-16) */
} ztp_plan_t;

void ztp_plan_opts_default(ztp_plan_opts* o);
ztp_status ztp_plan(int world, const double* T, const double* M, double L_ref,
                    const ztp_costs* costs, const ztp_plan_opts* opts, ztp_plan_t* out);

/* ztp_plan_refine: statistics refresh of a plan (A-8, A-39, A-42, A-43).
 * The window (T, M measured WITH prev in effect) gives `fresh` = ztp_plan(...)
 * (ZERO-only) whose Eq.1 ratio is a fraction of the work the rank still
 * computes, so the kept fractions of prev's STRAGGLERS compose:
 *   RESIZE ranks of prev: gamma = gamma_r = min(1 - (1 - prev.gamma_r[r]) (1 - fresh.gamma_r[r]), gamma_max),
 *                   role RESIZE iff gamma > 0;
 *   MIGRATE / SPLIT ranks of prev (A-42): their whole shed fraction composes,
 *                   gamma = min(1 - (1 - prev.gamma[r]) (1 - fresh.gamma_r[r]), gamma_max), beta kept,
 *                   phi = gamma beta, gamma_r = gamma (1 - beta) / (1 - gamma beta), role kept;
 *   NORMAL ranks of prev (A-43): stay NORMAL with gamma = 0, whatever fresh
 *                   says -- Alg.2 resizes only the plan's stragglers
 *                   and a receiver's extra time is received, loss-free work
 *                   (P:233); only a new statistics window re-plans them.
 * fresh's tolerance eps is the dead band: a straggler within T_min (1 + eps)
 * of the fresh window has fresh.gamma_r = 0 and keeps its ratio.
 * z and x are prev's; order is prev's when prev migrates (same sender order),
 * else fresh's.  Host-only, bit-deterministic.
 * Errors: ZTP_EINVAL (null, world mismatch), ZTP_EUNSUPPORTED (fresh has a
 * MIGRATE / SPLIT role: the refresh plan must be ZERO-only). */
ztp_status ztp_plan_refine(const ztp_plan_t* prev, const ztp_plan_t* fresh, double gamma_max, ztp_plan_t* out);

/* ---------------------------------------------------------------------------
 * a1/a2 controller: the statistics-driven re-planning loop of P:171-178 and
 * Alg.2 l.2 (reading A-41), one call per step on every rank with the
 * all-gathered T, M of the step just run under ctl->plan.  Pure host state
 * machine (plain struct, copyable, bit-deterministic), so every rank holds the
 * same plan without further communication.
 *   WINDOW  the step ran un-resized (plan all NORMAL): ctl->plan = ztp_plan(T,
 *           M, L_ref, costs, opts->plan) (Eq.1 / Alg.2 are defined on
 *           un-resized runtimes); T_target = min T, T_wmax = max T -> FIRST.
 *   FIRST   first step under a plan: if it is off target (some rank below
 *           (1 - trigger) T_target or above (1 + trigger) T_wmax: the
 *           slowdowns changed while it was applied) the plan is lifted ->
 *           WINDOW.  Else, up to max_refines times, ztp_plan_refine(plan,
 *           ztp_plan(T, M, ZERO-only, T_min criterion)) (A-39, A-42, A-43);
 *           a changed plan stays in FIRST, an unchanged one sets T_ref = T
 *           -> MONITOR.
 *   MONITOR any rank with |T_r - T_ref_r| > trigger T_ref_r (P:178's "over-10%
 *           increase", either direction, A-8) lifts the plan -> WINDOW (a
 *           rank whose slowdown vanished must return to gamma = 0).
 * *action = ZTP_CTL_APPLY when ctl->plan changed (the caller applies it before
 * the next step: ztp_plan_counts, ztp_select, ztp_migrate), else KEEP.
 * Errors: EINVAL (null, T not finite or <= 0), and ztp_plan's errors. */
enum { ZTP_CTL_WINDOW = 0, ZTP_CTL_FIRST = 1, ZTP_CTL_MONITOR = 2 };
enum { ZTP_CTL_KEEP = 0, ZTP_CTL_APPLY = 1 };

typedef struct ztp_ctl_opts {
  ztp_plan_opts plan;          /* window plan (SEMI or ZERO-only, criterion, eps, gamma_max, ...) */
  double L_ref;                /* Eq.2 / Eq.3 reference column count (A-25) */
  double trigger;              /* 0.10 */
  int32_t max_refines;         /* refreshes of one plan before monitoring (1) */
  int32_t _pad;
} ztp_ctl_opts;

typedef struct ztp_ctl {
  int32_t world, state, refines, _pad;
  ztp_plan_t plan;             /* the plan in effect for the next step */
  double T_ref[ZTP_MAX_RANKS]; /* monitoring reference */
  double T_target, T_wmax;     /* the window's T_min and T_max */
  int64_t steps, windows, replans, refine_count, triggers;
} ztp_ctl;

void ztp_ctl_opts_default(ztp_ctl_opts* o);
ztp_status ztp_ctl_init(ztp_ctl* ctl, int world);
ztp_status ztp_ctl_step(ztp_ctl* ctl, const ztp_ctl_opts* opts, const ztp_costs* costs, const double* T,
                        const double* M, int32_t* action);

/* ztp_plan_counts: integer realisation of a plan for one linear of `rank`.
 *   K       contraction length of this rank's linear (col: d_in; row: d_in/e)
 *   n_units hidden units per rank that migration moves (MLP: f/e)
 *   unit    migration granularity (1 for MLP units)
 *   is_row  1 for a row-parallel linear (its K shrinks by the migrated units)
 * n_mig = unit floor((n_units/unit) phi + 0.5) (<= n_units - unit);
 * n_prune = floor(K_rem gamma_r + 0.5) clamped to K_rem - 1 (A-3, A-4);
 * helper ranges: receivers ordered by r' = (r - s + e) % e, equal
 * shares with the remainder to the lowest r' (A-28), contiguous inside the
 * migrated tail [n_units - n_mig, n_units) (A-27). */
typedef struct ztp_counts {
  int32_t n_prune, n_mig;
  int32_t n_out, out_dst[ZTP_MAX_RANKS];              /* my units [lo,hi) computed by out_dst */
  int64_t out_lo[ZTP_MAX_RANKS], out_hi[ZTP_MAX_RANKS];
  int32_t n_in, in_src[ZTP_MAX_RANKS];                /* in_src's units [lo,hi) computed by me */
  int64_t in_lo[ZTP_MAX_RANKS], in_hi[ZTP_MAX_RANKS];
} ztp_counts;

ztp_status ztp_plan_counts(const ztp_plan_t* plan, int rank, int64_t K, int64_t n_units,
                           int64_t unit, int is_row, ztp_counts* out);

/* ztp_layer_prune_counts: the four prune counts of one transformer layer of
 * `rank` (h hidden, a = h/e attention features, u = f/e MLP units per rank),
 * out = {QKV (K = h), O (K = a), FC1 (K = h), FC2 (K_rem = u - n_mig)}.
 * MLP: ztp_plan_counts with gamma_r (FC2 is a row layer).  Attention (A-37):
 * heads do not migrate in this build (A-26), so a MIGRATE / SPLIT rank
 * resizes QKV and O by its Eq.1 gamma -- its remaining attention work is
 * (1 - gamma), like its MLP's after migration; other ranks by gamma_r.
 * Host-only.  Errors: EINVAL (null, rank, sizes). */
ztp_status ztp_layer_prune_counts(const ztp_plan_t* plan, int rank, int64_t h, int64_t a, int64_t u,
                                  int32_t out[4]);

/* ztp_plan_uniform: every rank RESIZE with gamma (homogeneous resizing, the
 * paper's E2 setting P:344; NORMAL if gamma = 0).  EINVAL for gamma outside
 * [0, 1) or world outside 1..8. */
ztp_status ztp_plan_uniform(int world, double gamma, ztp_plan_t* out);

/* ztp_pridiff_counts: NEXT-1 PriDiff prune count of a segment of L columns
 * with L_uni columns above the variation threshold (Alg.1 l.9-11):
 * gamma_k = max(1 - L_uni / L, alpha gamma_t), clamped to [0, gamma_max]
 * (A-4), n_prune = floor(L gamma_k + 0.5) <= L - 1 (A-3, >= 1 survives).
 * Returns 0 for L < 1. */
int32_t ztp_pridiff_counts(int64_t L, int64_t L_uni, double gamma_t, double alpha, double gamma_max);

/* ztp_costs_fit: Alg.2 l.1 pretest samples -> the Eq.2 / Eq.3 cost model
 * (A-40).  omega: (pruned units n, extra non-GEMM time vs the dense step);
 * Omega_1 = the extra at the smallest n > 0 ("static space allocation
 * overhead", clamped >= 0), Omega_2(n) = extra(n) - Omega_1.  phi1: (migrated
 * units, time); phi2: (units received by one helper, time).  Each function
 * becomes non-decreasing piecewise linear through (0, 0): x ascending, x <= 0
 * and repeated x dropped, y the running max clamped at 0 (a cost cannot
 * shrink with more units; a dip is timing noise); a function without samples
 * is the zero line through (0,0), (1,0).  xs / ys: caller arrays of 3 cap
 * doubles that receive the points (function k at offset k cap); out's
 * ztp_pwl pointers point into them.  Errors: EINVAL (null, non-finite
 * sample, cap < max(n) + 2). */
ztp_status ztp_costs_fit(int n_omega, const double* omega_x, const double* omega_y, int n_phi1,
                         const double* phi1_x, const double* phi1_y, int n_phi2, const double* phi2_x,
                         const double* phi2_y, int cap, double* xs, double* ys, ztp_costs* out);

/* ---------------------------------------------------------------------------
 * a1. Statistics exchange (Alg.1 l.1 / Alg.2 l.2): all-gather of (T_i, M_i)
 * over the context's communicator, then a host copy.  Collective; blocks the
 * host (this is the one host sync per replan).  T_all, M_all: host
 * arrays of `world` doubles written in rank order.
 * ------------------------------------------------------------------------- */
ztp_status ztp_allgather_stats(ztp_ctx* ctx, double T_own, double M_own,
                               double* T_all, double* M_all, void* stream);

/* ---------------------------------------------------------------------------
 * (2) Priority select (Alg.1 l.12-14) -- device, stream-ordered.
 * nseg segments (one per rank-local linear); segment i has h_seg_len[i]
 * columns with fp32 scores (the per-column weight variation delta, Alg.1 l.4)
 * at d_scores + sum_{j<i} h_seg_len[j].  It prunes the h_n_prune[i] columns
 * with the smallest score, ties by ascending index (A-2); -0 == +0.
 * Outputs (both ascending, Alg.1 l.14):
 *   d_kept   segment i at offset sum_{j<i} (len_j - n_prune_j + append_j):
 *            the kept indices S followed by h_append[i] appended indices
 *            len_i, len_i+1, ... (migrated-in units on a helper, A-26);
 *   d_pruned segment i at offset sum_{j<i} n_prune_j: the pruned indices P.
 *   d_pos    (optional) segment i at offset sum_{j<i} (len_j + append_j):
 *            the inverse map -- pos[k] = position of column k in the kept
 *            list, -1 if pruned (used as the producer-side row map y_pos).
 * h_append may be NULL (no appends).  One CTA per segment: radix select over
 * the order-preserving 32-bit key of the score, ballot/popc compaction.
 * Errors: EINVAL (nseg < 1, len < 1, n_prune outside [0, len-1]); a NaN score
 * sets a device flag reported by ztp_sync() as EINVAL.
 * ------------------------------------------------------------------------- */
ztp_status ztp_select(ztp_ctx* ctx, int nseg, const int32_t* h_seg_len, const int32_t* h_n_prune,
                      const int32_t* h_append, const float* d_scores,
                      int32_t* d_kept, int32_t* d_pruned, int32_t* d_pos, void* stream);

/* ---------------------------------------------------------------------------
 * (3)(4) Resized linears.  Collective semantics: every rank calls
 * the same sequence.
 *
 * Lineage: `sel` = the entry <layer_id, matrix_id, P> -- device
 * index lists kept (n_kept) and pruned (n_pruned), each ascending, with
 * n_kept + n_pruned = K (appended units count as kept).  sel = NULL means
 * dense (S = 0..K-1).  FWD records (layer_id, matrix_id) -> (kept, pruned,
 * counts) in the context; BWD with a different entry returns ELINEAGE.
 *
 * FWD  y_t[j,t] = sum_{k in S} w_t[k,j] x_t[k,t]  for j < n_out
 *      act = GELU: pre_t <- that sum, y_t <- GeLU_tanh(pre)
 *      col layer: no collective (Megatron pairing) unless
 *                 gather_output (all-gather of y over ranks).
 *      row layer: y_t partial sums are all-reduced (sum) over ranks.
 * BWD  dx_t[k,t] = sum_{j < n_out} w_t[k,j] g_t[j,t]  for k in S
 *      dx_t[p,t]  = imputation for p in P: Zero (0, the paper's choice);
 *                   Average (per column t the mean of dx_t[k,t] over k in S,
 *                   A-10); Same (hist_dx[p,t], the previous step's values,
 *                   A-11; caller-owned [K, N]; missing -> ZTP_EHISTORY)
 *      dw_t[k,j]  = sum_t x_t[k,t] g_t[j,t]           for k in S, j < n_out
 *      dw_t[p,j]  = imputation for p in P (as dx_t; Same from hist_dw [K, n])
 *
 *      col layer: dx_t is all-reduced over ranks (the imputed rows
 *                 are applied to the partial BEFORE the sum, A-14).
 *      row layer: act_in = GELU multiplies dx_t by GeLU'(pre_in_t) (the
 *                 input of this row layer was GeLU(pre_in)); no collective
 *                 unless input_is_parallel == 0 (all-gather).
 * dx_t or dw_t may have ptr = NULL to skip that GEMM.
 * Shapes: x_t [K,N]; w_t [K, >= n_out]; y_t, pre_t [>= n_out, N];
 * g_t [>= n_out, N]; dx_t, pre_in_t [K, N]; dw_t [K, >= n_out]; bf16 except
 * ZTP_F32 verification mode (all fp32, SIMT FFMA, fp32 collectives).
 * Errors: ESHAPE, EINDEX (host-visible lists), EDEGENERATE (n_kept == 0),
 * ELINEAGE, EHISTORY, EUNSUPPORTED (dtype mix), ECUDA, ENCCL.
 * ------------------------------------------------------------------------- */
typedef enum ztp_phase { ZTP_FWD = 0, ZTP_BWD = 1 } ztp_phase;
typedef enum ztp_impute { ZTP_IMPUTE_ZERO = 0, ZTP_IMPUTE_AVERAGE = 1, ZTP_IMPUTE_SAME = 2 } ztp_impute;
/* GELU: FWD pre_t <- pre, BWD (act_in) dx *= GeLU'(pre_in_t).
 * GELU_D: FWD pre_t <- GeLU'(pre) -- the derivative the consumer's backward
 * needs, computed from the fp32 accumulator with the tanh the GeLU already
 * evaluates -- and BWD (act_in) dx *= pre_in_t.  Same results as GELU
 * (A-34); the backward epilogue is one multiply. */
typedef enum ztp_act { ZTP_ACT_NONE = 0, ZTP_ACT_GELU = 1, ZTP_ACT_GELU_D = 2 } ztp_act;

typedef struct ztp_sel {
  const int32_t* kept;
  const int32_t* pruned;
  int32_t n_kept, n_pruned;
  int32_t layer_id, matrix_id;
} ztp_sel;

typedef struct ztp_linear_args {
  ztp_mat x_t, w_t, y_t, pre_t, g_t, dx_t, dw_t, pre_in_t;
  /* Compact operand copies.  xs_t
   * [>= n_kept, N] receives x_t rows S in lineage order, ws_t [>= n_kept, n]
   * receives w_t rows S: FWD writes them, BWD of the same lineage entry reads
   * them (ptr NULL: context workspace, BWD re-gathers).  The GEMM mainloop
   * then streams dense TMA boxes. */
  ztp_mat xs_t, ws_t;
  const ztp_sel* sel;          /* lineage entry; NULL = dense */
  const int32_t* y_pos;        /* FWD, optional: output unit j is written to row y_pos[j] of y_t / pre_t
                                  and dropped if y_pos[j] < 0 -- the next layer's compaction done by this
                                  epilogue (device array of n_out entries).  With out_sel: required, the
                                  inverse of out_sel->kept (ztp_select's `pos` of that segment). */
  int32_t x_compact;           /* x_t (and pre_in_t) already hold only rows S, in lineage order */
  int32_t dx_compact;          /* row BWD: dx_t receives only rows S, row i <- unit kept[i]; the Zero
                                  rows P are implied, not written (consumed by the producer's out_sel) */
  /* Output-side lineage (col layer feeding a row layer, DESIGN.md "Output
   * pruning"): the consumer's entry over this layer's n_out outputs (its
   * kept S' and pruned P' units, S' + P' = n_out).  The consumer contracts
   * only over S' and Zero-imputes the gradient of P', so:
   *  FWD computes y / pre only for j in S' (row i <- unit S'[i], compact);
   *  BWD reads g_t compact (row i <- unit S'[i], the consumer's dx_compact),
   *      contracts dX over S' only, and writes dw_t[k, p] = 0 for p in P'.
   * Results are identical to the full-output computation.  NULL = off. */
  const ztp_sel* out_sel;
  /* FWD: compact copies already written by ztp_prepare for this lineage
   * entry -- bit 0: xs_t, bit 1: ws_t -- so this call does not refill them. */
  int32_t prepared;
  /* BWD with dw_t but no dx_t: 1 = run this dW GEMM on the context's side
   * stream, after the caller stream's current position, and return at once
   * (joined like a concurrent dW: ztp_join or the next FWD call).  The caller
   * launches its next work beside it -- e.g. the attention projection's dW
   * next to the QKV backward, after its dX ran alone on every SM. */
  int32_t dw_side;
  int64_t n_out;               /* output units computed (<= w_t.cols); 0 = w_t.cols */
  int32_t impute;              /* ztp_impute (Zero is the paper's choice) */
  int32_t act;                 /* FWD activation of this layer's output */
  int32_t act_in;              /* BWD (row layer): activation feeding this layer */
  int32_t gather_output;       /* col FWD: all-gather y over ranks */
  int32_t input_is_parallel;   /* row BWD: 0 -> all-gather dx over ranks */
  int32_t skip_collective;     /* 1: leave the all-reduce to the caller (fused later) */
  const ztp_mat* hist_dx;      /* Same imputation history for dx_t (or NULL) */
  const ztp_mat* hist_dw;      /* Same imputation history for dw_t (or NULL) */
} ztp_linear_args;

/* ---------------------------------------------------------------------------
 * NEXT-1 priority-score maintenance (Alg.1 l.4-11), once per epoch.
 * ztp_priority_update: for every row i of w_t [K, n] (the paper's weight
 * column i): delta[i] = sum_j |w_t[i,j] - w_old_t[i,j]| / n  (Alg.1 l.4; fp32,
 * fixed summation order -> deterministic), EXCEPT rows pruned in the previous
 * selection (pos_prev[i] < 0, the `pos` output of ztp_select), which keep
 * their delta (incremental update).  pos_prev NULL = first epoch.
 * If count_above != NULL, *count_above += #{i : delta[i] > theta} (L_uni,
 * Alg.1 l.9; device int32, exact).  delta [K] fp32 device, in/out; it is the
 * score array ztp_select consumes.  w_t, w_old_t bf16, same shape.
 * Errors: EINVAL (null), ESHAPE (shape / dtype mismatch), ECUDA.
 * ztp_pridiff_gamma (host): Alg.1 l.10-11, gamma_k = max(1 - L_uni / L,
 * alpha * gamma_t) (alpha = 0.8 in the paper). */
ztp_status ztp_priority_update(ztp_ctx* ctx, const ztp_mat* w_t, const ztp_mat* w_old_t, const int32_t* pos_prev,
                               float* delta, int32_t* count_above, float theta, void* stream);
double ztp_pridiff_gamma(int64_t L, int64_t L_uni, double gamma_t, double alpha);

/* a4, batched: the compact operand copies of several linears in ONE launch
 * (fewer kernel boundaries than one gather per linear).  For args[i] with a
 * lineage entry: what[i] bit 0 -> xs_t <- rows S of x_t (not with x_compact),
 * bit 1 -> ws_t <- rows S of w_t (with out_sel: W^T[S, S'], or W^T[:, S'] when
 * sel is NULL).  xs_t / ws_t must be caller buffers of sufficient size.  The
 * caller then sets args[i]->prepared to the same bits for the FWD call.
 * n <= 16 copies in total.  Errors: EINVAL, ESHAPE, EUNSUPPORTED (f32). */
ztp_status ztp_prepare(ztp_ctx* ctx, int n, const ztp_linear_args* const* args, const int32_t* what, void* stream);

/* ztp_join: make `stream` wait for the library's internal side-stream work.
 * With ZTP_CONC=1 (default) a BWD call runs its dW GEMM on an internal
 * stream concurrently with the dX GEMM (the SMs split in proportion to their
 * MMA work, dW's weighted by ZTP_DW_SHARE = 1.2 for its split-K costs) and
 * returns without joining it, so the next linear's dX is not held back;
 * while such work is pending, ztp_core launches in plain stream order (no
 * programmatic early launch that would hold SMs the dW needs;
 * ZTP_SQUAT_GUARD=0 disables that);
 * call ztp_join before reading dW on `stream` (a FWD call, ztp_migrate,
 * ztp_select, ztp_prepare and ztp_priority_update join automatically; a step
 * captured in a CUDA graph must end with it).  Until then the caller must not
 * modify a BWD call's inputs (x_t / xs_t, g_t) nor its lineage lists by
 * other means than these calls.
 * Errors: ZTP_EINVAL (null ctx), ZTP_ECUDA. */
ztp_status ztp_join(ztp_ctx* ctx, void* stream);

ztp_status ztp_col_linear(ztp_ctx* ctx, ztp_phase phase, const ztp_linear_args* a, void* stream);
ztp_status ztp_row_linear(ztp_ctx* ctx, ztp_phase phase, const ztp_linear_args* a, void* stream);

/* Stand-in attention core of the measurement layer (A-31): FWD ctx_t[f,t] =
 * q[f,t] + k[f,t] + v[f,t] with qkv_t = [Q; K; V] row blocks of `feat` rows
 * (the first n_feat of each block); BWD g_qkv_t = [dctx; dctx; dctx].
 * FWD with rows != NULL writes only features rows[0..n_rows) as compact rows
 * 0..n_rows-1 of ctx_t (the O projection's kept rows S, producer-side).
 * v_compact (A-36, output pruning of V): the V block of qkv_t holds only the
 * features rows[0..n_rows), compact (V row i <- feature rows[i]); FWD reads
 * it so, BWD writes dV compact (dQ, dK stay full).  qkv_t then has
 * 2 feat + n_rows rows. */
ztp_status ztp_core(ztp_ctx* ctx, ztp_phase phase, const ztp_mat* qkv_t, const ztp_mat* ctx_t,
                    int64_t feat, int64_t n_feat, const int32_t* rows, int64_t n_rows, int32_t v_compact,
                    void* stream);

/* ---------------------------------------------------------------------------
 * (5) Migration -- peer copies of shard slices (A-26).
 * Each transfer copies the sub-matrix src[r0:r0+nr, c0:c0+nc] held by
 * src_rank into dst[dr0:dr0+nr, dc0:dc0+nc] held by dst_rank.  Every rank
 * calls ztp_migrate with the SAME list; a rank acts only on transfers naming
 * it.  src_rank == dst_rank is a local device copy.  The slice is moved
 * exactly once over NVLink (the straggler's egress is the scarce resource;
 * helpers receive disjoint slices instead of full broadcasts).
 * Peer pulls (the peer transport, or any context whose window is open --
 * the NCCL transport then carries only the collectives): the destination
 * PULLS from the source rank's window --
 * `src` must be a window tensor, and on the destination rank `src` is its
 * OWN symmetric counterpart (same ztp_sym_alloc slot), whose window offset
 * locates the source's copy; one kernel per 24 pulls per rank, with device
 * barriers before (sources final) and after (sources not yet reused).
 * NCCL transport without a window: the slices are staged through a workspace and moved by
 * grouped ncclSend / ncclRecv (any pattern is deadlock-free).
 * ------------------------------------------------------------------------- */
typedef struct ztp_xfer {
  ztp_mat src;                 /* meaningful on src_rank only */
  ztp_mat dst;                 /* meaningful on dst_rank only */
  int64_t r0, c0, nr, nc, dr0, dc0;
  int32_t src_rank, dst_rank;
} ztp_xfer;

ztp_status ztp_migrate(ztp_ctx* ctx, int n, const ztp_xfer* xfers, void* stream);

/* ---------------------------------------------------------------------------
 * Straggler emulation and GEMM statistics (A-32).  chi > 1 makes every
 * GEMM this context launches run chi times longer: a one-thread delay kernel
 * after each GEMM spins until start + chi (end - start), where start/end are
 * the GEMM's own %globaltimer stamps (the side stream's concurrent dW GEMM
 * has its own stamp slot, so a slowed rank runs the same concurrent dX / dW
 * schedule as an unslowed one).  M (A-6) accumulates GEMM + delay time on the
 * device, overlapping GEMMs counted once (union of their intervals);
 * ztp_read_gemm_ns syncs `stream`, returns and resets it.
 * ------------------------------------------------------------------------- */
ztp_status ztp_set_slowdown(ztp_ctx* ctx, double chi);
/* on = 1: stamp every GEMM and accumulate M even when chi == 1 (statistics
 * window); off by default so unslowed ranks pay no extra launches. */
ztp_status ztp_set_stats(ztp_ctx* ctx, int on);
ztp_status ztp_read_gemm_ns(ztp_ctx* ctx, void* stream, double* ns);

/* Profiling with CUDA events recorded on the launching stream around every
 * kernel class this context issues (on = 1).  ztp_read_profile syncs `stream`,
 * returns the totals since the last read and resets them:
 *   gemm_ms     resized GEMM kernels (+ the emulated-slowdown delay after each)
 *   other_ms    select, row compaction, stand-in core
 *   comm_ms     collectives (NCCL) as seen on their stream
 *   gemm_flops  algorithmic FLOPs of the GEMMs: 2 n_kept n_out N per launch
 * T_i (A-5) = gemm_ms + other_ms (busy time, collective waits excluded) and
 * M_i (A-6) = gemm_ms of the statistics window. */
typedef struct ztp_profile {
  double gemm_ms, other_ms, comm_ms, gemm_flops;
  int64_t n_gemm, n_other, n_comm;
  /* length of the union over GEMM launches of [first CTA start, last CTA
   * end], from the kernels' own %globaltimer stamps (split-K reduce
   * included): GEMM kernel time without event / launch overheads, overlaps
   * between launches (PDL) counted once */
  double gemm_kernel_ms;
} ztp_profile;
/* on = 2: GEMM kernel stamps only (no events, no change to the launch
 * schedule), capturable: a graph captured in this mode writes the same stamp
 * slots on every replay, and each ztp_read_profile returns the GEMM kernel
 * time and FLOPs of the replays since the last read (one replay per read
 * gives per-step values).  on = 0 releases the slots. */
ztp_status ztp_set_profile(ztp_ctx* ctx, int on);
ztp_status ztp_read_profile(ztp_ctx* ctx, void* stream, ztp_profile* out);
/* Diagnostics: the raw [start, end] %globaltimer stamps (ns) of the stamped
 * GEMM launches (profiling on), in launch order, without resetting them;
 * returns how many pairs were written to out[2 * max_launches], -1 on error. */
int ztp_read_stamps(ztp_ctx* ctx, void* stream, unsigned long long* out, int max_launches);
/* Profiling mode 3 (ztp_set_profile(ctx, 3)): as mode 2, and every GEMM
 * launch (first 64) also records per CTA (<= 160) eight %globaltimer stamps:
 * CTA start, after the PDL wait, first operand stage ready (MMA issuer), last
 * MMA commit, first accumulator ready (epilogue), last tile's stores issued,
 * stores complete, CTA end; 0 = not recorded by that CTA.  Copies launches x
 * 160 x 8 values into out; returns the launch count or -1. */
int ztp_read_cta_stamps(ztp_ctx* ctx, void* stream, unsigned long long* out, int max_launches);

/* Raw resized GEMM (test / benchmark entry; the linears use it internally).
 * kind 0 = FWD (y = w[S]^T x[S]), 1 = dX (dx rows by sel), 2 = dW. */
ztp_status ztp_gemm(ztp_ctx* ctx, int kind, const ztp_linear_args* a, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ZTP_H_ */

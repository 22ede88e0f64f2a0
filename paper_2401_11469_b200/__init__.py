"""paper_2401_11469_b200 -- B200-native straggler-balanced 1D tensor-parallel
linear layer (ZERO-resizing + SEMI-migration, arXiv 2401.11469).

Python binding of the C ABI in include/ztp.h with the same names.  Every
function marshals arguments (torch tensors are used only as device memory)
and calls libztp.so; all compute runs in the library's sm_100a kernels and
NCCL.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

from . import _lib
from ._lib import (ACT_GELU, ACT_GELU_D, ACT_NONE, BF16, BWD, CRIT_AVG, CRIT_MIN, F32, FWD, IMPUTE_AVERAGE, IMPUTE_SAME,  # noqa
                   IMPUTE_ZERO, KIND_DW, KIND_DX, KIND_FWD, MIGRATE, NORMAL, RESIZE, SPLIT, Costs, Counts, Ctl, CtlOpts,
                   LinearArgs, Mat, PlanOpts, PlanT, Pwl, Sel, Xfer, ZtpError, check, lib)

__all__ = [
    "ztp_version", "ztp_get_unique_id", "ztp_ctx_create", "ztp_ctx_destroy", "ztp_sync", "ztp_launch_count",
    "ztp_plan", "ztp_plan_refine", "ztp_plan_counts", "ztp_allgather_stats", "ztp_select", "ztp_join", "ztp_col_linear", "ztp_row_linear",
    "ztp_core", "ztp_migrate", "ztp_set_slowdown", "ztp_set_stats", "ztp_read_gemm_ns", "ztp_gemm", "mat",
    "make_costs", "plan_opts", "ZtpError", "ztp_window_create", "ztp_window_open", "ztp_sym_alloc",
    "ztp_set_transport", "ztp_barrier", "TRANSPORT_NCCL", "TRANSPORT_PEER",
]
from ._lib import (TRANSPORT_NCCL, TRANSPORT_PEER, COLL_TREE, COLL_P2P, OPT_CONC, OPT_DW_SHARE, OPT_SQUAT_GUARD, OPT_GATHER4,  # noqa: E402
                   OPT_SPLITK, OPT_GROUP, OPT_PEER_CTAS, OPT_A_EARLY, OPT_PART, OPT_AUX_WEIGHT, OPT_FLAGS,
                   OPT_SPREAD_EPI, OPT_ZERO_GENERIC, OPT_TAIL_HALVES)


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def mat(t=None, rows: Optional[int] = None) -> Mat:
    """ztp_mat view of a 2-D torch tensor (row-major, unit column stride)."""
    if t is None:
        return Mat(None, 0, 0, 0, 0, 0)
    import torch
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("ztp_mat needs a 2-D tensor with unit column stride")
    dt = {torch.bfloat16: BF16, torch.float32: F32}[t.dtype]
    r = t.shape[0] if rows is None else rows
    return Mat(t.data_ptr(), r, t.shape[1], t.stride(0), dt, 0)


def ztp_version() -> str:
    return lib.ztp_version().decode()


def ztp_get_unique_id() -> bytes:
    buf = C.create_string_buffer(_lib.UID_BYTES)
    check(lib.ztp_get_unique_id(buf))
    return buf.raw


def ztp_ctx_create(rank: int = 0, world: int = 1, uid: Optional[bytes] = None, device: int = 0):
    h = C.c_void_p()
    check(lib.ztp_ctx_create(C.byref(h), rank, world, uid, device))
    return h


def ztp_ctx_destroy(ctx) -> None:
    check(lib.ztp_ctx_destroy(ctx))


def ztp_sync(ctx, stream=None) -> None:
    check(lib.ztp_sync(ctx, _stream(stream)), ctx)


def ztp_launch_count(ctx) -> int:
    return int(lib.ztp_launch_count(ctx))


# ------------------------------------------------------------------- plan (host)

def _pwl(points):
    xs, ys = points
    n = len(xs)
    xa = (C.c_double * n)(*xs)
    ya = (C.c_double * n)(*ys)
    return Pwl(n, xa, ya), (xa, ya)


def make_costs(omega1=0.0, omega2=((0.0, 1.0), (0.0, 0.0)), phi1=((0.0, 1.0), (0.0, 0.0)),
               phi2=((0.0, 1.0), (0.0, 0.0))):
    """ztp_costs from (xs, ys) sample points; returns (Costs, keepalive)."""
    o2, k1 = _pwl(omega2)
    p1, k2 = _pwl(phi1)
    p2, k3 = _pwl(phi2)
    return Costs(omega1, o2, p1, p2), (k1, k2, k3)


def plan_opts(**kw) -> PlanOpts:
    o = PlanOpts()
    lib.ztp_plan_opts_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def ztp_plan(T: Sequence[float], M: Sequence[float], L_ref: float, costs=None, opts: Optional[PlanOpts] = None
             ) -> PlanT:
    e = len(T)
    Ta = (C.c_double * max(e, 1))(*T)
    Ma = (C.c_double * max(e, 1))(*M)
    if costs is None:
        costs = make_costs()
    c, _keep = costs if isinstance(costs, tuple) else (costs, None)
    out = PlanT()
    check(lib.ztp_plan(e, Ta, Ma, L_ref, C.byref(c), C.byref(opts or plan_opts()), C.byref(out)))
    return out


def ztp_plan_refine(prev: PlanT, fresh: PlanT, gamma_max: float = 0.9) -> PlanT:
    out = PlanT()
    check(lib.ztp_plan_refine(C.byref(prev), C.byref(fresh), gamma_max, C.byref(out)))
    return out


CTL_WINDOW, CTL_FIRST, CTL_MONITOR = 0, 1, 2
CTL_KEEP, CTL_APPLY = 0, 1


def ctl_opts(L_ref: float = 1.0, trigger: float = 0.10, max_refines: int = 1, **plan_kw) -> CtlOpts:
    o = CtlOpts()
    lib.ztp_ctl_opts_default(C.byref(o))
    o.plan = plan_opts(**plan_kw)
    o.L_ref, o.trigger, o.max_refines = L_ref, trigger, max_refines
    return o


def ztp_ctl_init(world: int) -> Ctl:
    c = Ctl()
    check(lib.ztp_ctl_init(C.byref(c), world))
    return c


def ztp_ctl_step(ctl: Ctl, opts: CtlOpts, T: Sequence[float], M: Sequence[float], costs=None) -> int:
    """One controller step (include/ztp.h): T, M of the step just run under
    ctl.plan (all ranks', all-gathered); returns CTL_APPLY if ctl.plan changed."""
    e = ctl.world
    Ta = (C.c_double * e)(*T[:e])
    Ma = (C.c_double * e)(*M[:e])
    if costs is None:
        costs = make_costs()
    c, _keep = costs if isinstance(costs, tuple) else (costs, None)
    act = C.c_int32()
    check(lib.ztp_ctl_step(C.byref(ctl), C.byref(opts), C.byref(c), Ta, Ma, C.byref(act)))
    return int(act.value)


def ztp_plan_counts(plan: PlanT, rank: int, K: int, n_units: int, unit: int = 1, is_row: bool = False) -> Counts:
    out = Counts()
    check(lib.ztp_plan_counts(C.byref(plan), rank, K, n_units, unit, int(is_row), C.byref(out)))
    return out


SEGS = ("qkv", "o", "fc1", "fc2")


def ztp_layer_prune_counts(plan: PlanT, rank: int, h: int, a: int, u: int) -> dict:
    """{qkv, o, fc1, fc2} prune counts of one layer of `rank` (A-37 attention rule)."""
    out = (C.c_int32 * 4)()
    check(lib.ztp_layer_prune_counts(C.byref(plan), rank, h, a, u, out))
    return dict(zip(SEGS, (int(v) for v in out)))


def ztp_plan_uniform(world: int, gamma: float) -> PlanT:
    out = PlanT()
    check(lib.ztp_plan_uniform(world, gamma, C.byref(out)))
    return out


def ztp_pridiff_counts(L: int, L_uni: int, gamma_t: float, alpha: float = 0.8, gamma_max: float = 0.9) -> int:
    return int(lib.ztp_pridiff_counts(L, L_uni, gamma_t, alpha, gamma_max))


def ztp_costs_fit(omega, phi1, phi2):
    """Pretest samples [(x, y)] -> (Costs, keepalive, plain dict) via the C fit (A-40)."""
    def arr(pts, k):
        return (C.c_double * max(len(pts), 1))(*[float(p[k]) for p in pts])
    cap = max(len(omega), len(phi1), len(phi2)) + 2
    xs, ys = (C.c_double * (3 * cap))(), (C.c_double * (3 * cap))()
    out = Costs()
    keep = [arr(omega, 0), arr(omega, 1), arr(phi1, 0), arr(phi1, 1), arr(phi2, 0), arr(phi2, 1), xs, ys]
    check(lib.ztp_costs_fit(len(omega), keep[0], keep[1], len(phi1), keep[2], keep[3], len(phi2), keep[4],
                            keep[5], cap, xs, ys, C.byref(out)))
    plain = {"omega1": out.omega1}
    for name in ("omega2", "phi1", "phi2"):
        f = getattr(out, name)
        plain[name] = (tuple(f.x[i] for i in range(f.n)), tuple(f.y[i] for i in range(f.n)))
    return (out, keep), plain


def ztp_allgather_stats(ctx, T_own: float, M_own: float, world: int, stream=None):
    Ta = (C.c_double * world)()
    Ma = (C.c_double * world)()
    check(lib.ztp_allgather_stats(ctx, T_own, M_own, Ta, Ma, _stream(stream)), ctx)
    return list(Ta), list(Ma)


# ------------------------------------------------------------------ device calls

def ztp_join(ctx, stream=None) -> None:
    """Order the library's side-stream work (concurrent dW, ZTP_CONC) before
    later work on `stream`."""
    check(lib.ztp_join(ctx, _stream(stream)), ctx)


def ztp_select(ctx, seg_len: Sequence[int], n_prune: Sequence[int], scores, kept, pruned,
               append: Optional[Sequence[int]] = None, pos=None, stream=None) -> None:
    n = len(seg_len)
    la = (C.c_int32 * n)(*seg_len)
    pa = (C.c_int32 * n)(*n_prune)
    aa = (C.c_int32 * n)(*append) if append is not None else None
    check(lib.ztp_select(ctx, n, la, pa, aa, scores.data_ptr(), kept.data_ptr(), pruned.data_ptr(),
                         pos.data_ptr() if pos is not None else None, _stream(stream)), ctx)


def sel(kept, n_kept: int, pruned, n_pruned: int, layer_id: int, matrix_id: int) -> Sel:
    return Sel(kept.data_ptr() if kept is not None else None, pruned.data_ptr() if pruned is not None else None,
               n_kept, n_pruned, layer_id, matrix_id)


def linear_args(x_t=None, w_t=None, y_t=None, pre_t=None, g_t=None, dx_t=None, dw_t=None, pre_in_t=None,
                sel_: Optional[Sel] = None, n_out: int = 0, impute: int = IMPUTE_ZERO, act: int = ACT_NONE,
                act_in: int = ACT_NONE, skip_collective: int = 0, xs_t=None, ws_t=None, y_pos=None,
                x_compact: bool = False, dx_compact: bool = False, out_sel: Optional[Sel] = None,
                hist_dx=None, hist_dw=None, gather_output: bool = False, input_is_parallel: bool = True,
                dw_side: bool = False) -> LinearArgs:
    a = LinearArgs()
    a.x_t, a.w_t, a.y_t, a.pre_t = mat(x_t), mat(w_t), mat(y_t), mat(pre_t)
    a.g_t, a.dx_t, a.dw_t, a.pre_in_t = mat(g_t), mat(dx_t), mat(dw_t), mat(pre_in_t)
    a.xs_t, a.ws_t = mat(xs_t), mat(ws_t)
    a.y_pos = y_pos.data_ptr() if y_pos is not None else None
    a.x_compact = int(x_compact)
    a.dx_compact = int(dx_compact)
    a.sel = C.pointer(sel_) if sel_ is not None else None
    a.out_sel = C.pointer(out_sel) if out_sel is not None else None
    a.hist_dx = C.pointer(mat(hist_dx)) if hist_dx is not None else None
    a.hist_dw = C.pointer(mat(hist_dw)) if hist_dw is not None else None
    a.n_out = n_out
    a.impute = impute
    a.act = act
    a.act_in = act_in
    a.gather_output = int(gather_output)
    a.input_is_parallel = int(input_is_parallel)
    a.skip_collective = skip_collective
    a.dw_side = int(dw_side)
    return a


def ztp_col_linear(ctx, phase: int, args: LinearArgs, stream=None) -> None:
    check(lib.ztp_col_linear(ctx, phase, C.byref(args), _stream(stream)), ctx)


def ztp_row_linear(ctx, phase: int, args: LinearArgs, stream=None) -> None:
    check(lib.ztp_row_linear(ctx, phase, C.byref(args), _stream(stream)), ctx)


def ztp_priority_update(ctx, w_t, w_old_t, delta, pos_prev=None, count_above=None, theta: float = 0.0,
                        stream=None) -> None:
    """NEXT-1 (Alg.1 l.4-9): delta <- column variation of W^T rows, rows pruned
    last epoch (pos_prev < 0) carried over; count_above += #{delta > theta}."""
    wm, om = mat(w_t), mat(w_old_t)
    check(lib.ztp_priority_update(ctx, C.byref(wm), C.byref(om),
                                  pos_prev.data_ptr() if pos_prev is not None else None, delta.data_ptr(),
                                  count_above.data_ptr() if count_above is not None else None, float(theta),
                                  _stream(stream)), ctx)


def ztp_pridiff_gamma(L: int, L_uni: int, gamma_t: float, alpha: float = 0.8) -> float:
    return float(lib.ztp_pridiff_gamma(L, L_uni, gamma_t, alpha))


def ztp_prepare(ctx, items, stream=None) -> None:
    """items: [(LinearArgs, what_bits)] -> one batched compaction launch."""
    n = len(items)
    arr = (C.POINTER(LinearArgs) * n)(*[C.pointer(a) for a, _ in items])
    what = (C.c_int32 * n)(*[int(w) for _, w in items])
    check(lib.ztp_prepare(ctx, n, arr, what, _stream(stream)), ctx)


def ztp_gemm(ctx, kind: int, args: LinearArgs, stream=None) -> None:
    check(lib.ztp_gemm(ctx, kind, C.byref(args), _stream(stream)), ctx)


def ztp_core(ctx, phase: int, qkv_t, ctx_t, feat: int, n_feat: int, rows=None, n_rows: int = 0,
             stream=None, v_compact: bool = False) -> None:
    q, c = mat(qkv_t), mat(ctx_t)
    check(lib.ztp_core(ctx, phase, C.byref(q), C.byref(c), feat, n_feat,
                       rows.data_ptr() if rows is not None else None, n_rows, int(v_compact), _stream(stream)), ctx)


def ztp_migrate(ctx, xfers: Sequence[Xfer], stream=None) -> None:
    n = len(xfers)
    arr = (Xfer * max(n, 1))(*xfers)
    check(lib.ztp_migrate(ctx, n, arr, _stream(stream)), ctx)


def xfer(src=None, dst=None, r0=0, c0=0, nr=0, nc=0, dr0=0, dc0=0, src_rank=0, dst_rank=0) -> Xfer:
    return Xfer(mat(src), mat(dst), r0, c0, nr, nc, dr0, dc0, src_rank, dst_rank)


# ------------------------------------------------------- peer-memory data plane

def ztp_window_create(ctx, nbytes: int) -> bytes:
    """Allocate this rank's symmetric window; returns its IPC_BYTES handle."""
    buf = C.create_string_buffer(_lib.IPC_BYTES)
    check(lib.ztp_window_create(ctx, int(nbytes), buf), ctx)
    return buf.raw


def ztp_window_open(ctx, handles: Sequence[bytes]) -> None:
    """Map every rank's window (handles in rank order)."""
    blob = b"".join(handles)
    if len(blob) != len(handles) * _lib.IPC_BYTES:
        raise ValueError("ztp_window_open: every handle must be IPC_BYTES long")
    check(lib.ztp_window_open(ctx, blob), ctx)


class _DevPtr:
    """__cuda_array_interface__ of library-owned device memory (a window
    slice), so torch can view it without copying."""

    def __init__(self, ptr: int, nelem: int, typestr: str, device: int):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}
        self.device = device


def ztp_sym_alloc(ctx, rows: int, cols: int, dtype=None, device: int = 0):
    """A [rows, cols] tensor (row pitch padded to 16 bytes) carved out of the
    symmetric window: the same call sequence on every rank yields the same
    window offsets.  The library owns the memory (valid until
    ztp_ctx_destroy)."""
    import torch
    dtype = dtype or torch.bfloat16
    es = {torch.bfloat16: 2, torch.float32: 4}[dtype]
    ld = (cols * es + 15) // 16 * 16 // es
    p = C.c_void_p()
    n = max(rows, 1) * ld
    check(lib.ztp_sym_alloc(ctx, n * es, C.byref(p)), ctx)
    raw = torch.as_tensor(_DevPtr(p.value, n, "<i2" if es == 2 else "<f4", device), device=f"cuda:{device}")
    t = raw.view(dtype) if es == 2 else raw
    return t.view(max(rows, 1), ld)[:, :cols]


def ztp_set_transport(ctx, transport: int) -> None:
    check(lib.ztp_set_transport(ctx, transport), ctx)


def ztp_broadcast(ctx, root: int, t, mode: int = 0, stream=None) -> None:
    m = mat(t)
    check(lib.ztp_broadcast(ctx, root, C.byref(m), mode, _stream(stream)), ctx)


def ztp_reduce(ctx, root: int, t, mode: int = 0, stream=None) -> None:
    m = mat(t)
    check(lib.ztp_reduce(ctx, root, C.byref(m), mode, _stream(stream)), ctx)


def ztp_accumulate(ctx, dst, src, stream=None) -> None:
    d, s_ = mat(dst), mat(src)
    check(lib.ztp_accumulate(ctx, C.byref(d), C.byref(s_), _stream(stream)), ctx)


def ztp_allreduce(ctx, t, stream=None) -> None:
    m = mat(t)
    check(lib.ztp_allreduce(ctx, C.byref(m), _stream(stream)), ctx)


def ztp_transpose(ctx, src, dst, cols=None, n: Optional[int] = None, stream=None) -> None:
    """dst[i, r] = src[r, cols[i] if cols is not None else i] for i < n."""
    s_, d = mat(src), mat(dst)
    if n is None:
        n = int(cols.numel()) if cols is not None else src.shape[1]
    check(lib.ztp_transpose(ctx, C.byref(s_), C.byref(d), cols.data_ptr() if cols is not None else None, n,
                            _stream(stream)), ctx)


def ztp_set_option(ctx, opt: int, value: float) -> None:
    check(lib.ztp_set_option(ctx, int(opt), float(value)), ctx)


def ztp_get_option(ctx, opt: int) -> float:
    v = C.c_double()
    check(lib.ztp_get_option(ctx, int(opt), C.byref(v)), ctx)
    return v.value


def ztp_barrier(ctx, stream=None) -> None:
    check(lib.ztp_barrier(ctx, _stream(stream)), ctx)


def ztp_set_slowdown(ctx, chi: float) -> None:
    check(lib.ztp_set_slowdown(ctx, chi), ctx)


def ztp_set_stats(ctx, on: bool) -> None:
    check(lib.ztp_set_stats(ctx, int(on)), ctx)


def ztp_set_profile(ctx, on: bool) -> None:
    check(lib.ztp_set_profile(ctx, int(on)), ctx)


def ztp_read_profile(ctx, stream=None) -> dict:
    p = _lib.Profile()
    check(lib.ztp_read_profile(ctx, _stream(stream), C.byref(p)), ctx)
    return {k: getattr(p, k) for k, _ in _lib.Profile._fields_}


def ztp_read_stamps(ctx, stream=None, max_launches: int = 256):
    """[(start_ns, end_ns)] of the stamped GEMM launches (diagnostics)."""
    buf = (C.c_uint64 * (2 * max_launches))()
    n = lib.ztp_read_stamps(ctx, _stream(stream), buf, max_launches)
    if n < 0:
        raise ZtpError(-1, "ztp_read_stamps failed")
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n)]


def ztp_read_cta_stamps(ctx, stream=None, max_launches: int = 64):
    """Profiling mode 3: numpy [launches, 160, 8] per-CTA %globaltimer stamps."""
    import numpy as np
    buf = (C.c_uint64 * (max_launches * 160 * 8))()
    n = lib.ztp_read_cta_stamps(ctx, _stream(stream), buf, max_launches)
    if n < 0:
        raise ZtpError(-1, "ztp_read_cta_stamps failed (profiling mode 3 not enabled?)")
    return np.frombuffer(buf, dtype=np.uint64)[:n * 160 * 8].reshape(n, 160, 8).copy()


def ztp_read_gemm_ns(ctx, stream=None) -> float:
    v = C.c_double()
    check(lib.ztp_read_gemm_ns(ctx, _stream(stream), C.byref(v)), ctx)
    return v.value

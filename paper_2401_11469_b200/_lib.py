"""ctypes binding of libztp.so (include/ztp.h).  Argument marshalling only: no
arithmetic of the method lives in Python, and there is no CPU fallback -- if
the CUDA library is missing this module raises on import."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libztp.so")

MAX_RANKS = 8
UID_BYTES = 128
IPC_BYTES = 128
TRANSPORT_NCCL, TRANSPORT_PEER = 0, 1
COLL_TREE, COLL_P2P = 0, 1

# status codes (ztp_status)
STATUS = ["ZTP_OK", "ZTP_EINVAL", "ZTP_ESHAPE", "ZTP_EINDEX", "ZTP_EDEGENERATE", "ZTP_ELINEAGE", "ZTP_EHISTORY",
          "ZTP_ENOBASELINE", "ZTP_ENOHELPER", "ZTP_ERECEIVERS", "ZTP_ECUDA", "ZTP_ENCCL", "ZTP_EUNSUPPORTED"]
BF16, F32 = 0, 1
FWD, BWD = 0, 1
IMPUTE_ZERO, IMPUTE_AVERAGE, IMPUTE_SAME = 0, 1, 2
ACT_NONE, ACT_GELU, ACT_GELU_D = 0, 1, 2
CRIT_AVG, CRIT_MIN = 0, 1
NORMAL, RESIZE, MIGRATE, SPLIT = 0, 1, 2, 3
KIND_FWD, KIND_DX, KIND_DW = 0, 1, 2
(OPT_CONC, OPT_DW_SHARE, OPT_SQUAT_GUARD, OPT_GATHER4, OPT_SPLITK, OPT_GROUP, OPT_PEER_CTAS, OPT_A_EARLY, OPT_PART,
 OPT_AUX_WEIGHT, OPT_FLAGS, OPT_SPREAD_EPI, OPT_ZERO_GENERIC, OPT_TAIL_HALVES) = range(14)


class ZtpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.name = STATUS[code] if 0 <= code < len(STATUS) else f"ZTP_{code}"
        super().__init__(f"{self.name}: {msg}")


class Mat(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
                ("dtype", C.c_int32), ("_pad", C.c_int32)]


class Pwl(C.Structure):
    _fields_ = [("n", C.c_int32), ("x", C.POINTER(C.c_double)), ("y", C.POINTER(C.c_double))]


class Costs(C.Structure):
    _fields_ = [("omega1", C.c_double), ("omega2", Pwl), ("phi1", Pwl), ("phi2", Pwl)]


class PlanOpts(C.Structure):
    _fields_ = [("enable_migration", C.c_int32), ("zero_crit", C.c_int32), ("gamma_max", C.c_double),
                ("eps", C.c_double), ("gamma_tol", C.c_double), ("bisect_iters", C.c_int32),
                ("force_lambda", C.c_int32)]


class PlanT(C.Structure):
    _fields_ = [("world", C.c_int32), ("z", C.c_int32), ("x", C.c_int32), ("order", C.c_int32 * MAX_RANKS),
                ("role", C.c_int32 * MAX_RANKS), ("gamma", C.c_double * MAX_RANKS),
                ("beta", C.c_double * MAX_RANKS), ("phi", C.c_double * MAX_RANKS),
                ("gamma_r", C.c_double * MAX_RANKS)]


class CtlOpts(C.Structure):
    _fields_ = [("plan", PlanOpts), ("L_ref", C.c_double), ("trigger", C.c_double), ("max_refines", C.c_int32),
                ("_pad", C.c_int32)]


class Ctl(C.Structure):
    _fields_ = [("world", C.c_int32), ("state", C.c_int32), ("refines", C.c_int32), ("_pad", C.c_int32),
                ("plan", PlanT), ("T_ref", C.c_double * MAX_RANKS), ("T_target", C.c_double),
                ("T_wmax", C.c_double), ("steps", C.c_int64), ("windows", C.c_int64), ("replans", C.c_int64),
                ("refine_count", C.c_int64), ("triggers", C.c_int64)]


class Counts(C.Structure):
    _fields_ = [("n_prune", C.c_int32), ("n_mig", C.c_int32), ("n_out", C.c_int32),
                ("out_dst", C.c_int32 * MAX_RANKS), ("out_lo", C.c_int64 * MAX_RANKS),
                ("out_hi", C.c_int64 * MAX_RANKS), ("n_in", C.c_int32), ("in_src", C.c_int32 * MAX_RANKS),
                ("in_lo", C.c_int64 * MAX_RANKS), ("in_hi", C.c_int64 * MAX_RANKS)]


class Sel(C.Structure):
    _fields_ = [("kept", C.c_void_p), ("pruned", C.c_void_p), ("n_kept", C.c_int32), ("n_pruned", C.c_int32),
                ("layer_id", C.c_int32), ("matrix_id", C.c_int32)]


class LinearArgs(C.Structure):
    _fields_ = [("x_t", Mat), ("w_t", Mat), ("y_t", Mat), ("pre_t", Mat), ("g_t", Mat), ("dx_t", Mat),
                ("dw_t", Mat), ("pre_in_t", Mat), ("xs_t", Mat), ("ws_t", Mat), ("sel", C.POINTER(Sel)),
                ("y_pos", C.c_void_p), ("x_compact", C.c_int32), ("dx_compact", C.c_int32),
                ("out_sel", C.POINTER(Sel)), ("prepared", C.c_int32), ("dw_side", C.c_int32), ("n_out", C.c_int64),
                ("impute", C.c_int32), ("act", C.c_int32), ("act_in", C.c_int32), ("gather_output", C.c_int32),
                ("input_is_parallel", C.c_int32), ("skip_collective", C.c_int32),
                ("hist_dx", C.POINTER(Mat)), ("hist_dw", C.POINTER(Mat))]


class Profile(C.Structure):
    _fields_ = [("gemm_ms", C.c_double), ("other_ms", C.c_double), ("comm_ms", C.c_double),
                ("gemm_flops", C.c_double), ("n_gemm", C.c_int64), ("n_other", C.c_int64), ("n_comm", C.c_int64),
                ("gemm_kernel_ms", C.c_double)]


class Xfer(C.Structure):
    _fields_ = [("src", Mat), ("dst", Mat), ("r0", C.c_int64), ("c0", C.c_int64), ("nr", C.c_int64),
                ("nc", C.c_int64), ("dr0", C.c_int64), ("dc0", C.c_int64), ("src_rank", C.c_int32),
                ("dst_rank", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2401_11469_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    st = C.c_int
    vp = C.c_void_p
    sig = {
        "ztp_status_str": (C.c_char_p, [st]),
        "ztp_last_error": (C.c_char_p, [vp]),
        "ztp_version": (C.c_char_p, []),
        "ztp_get_unique_id": (st, [C.c_char_p]),
        "ztp_ctx_create": (st, [C.POINTER(vp), C.c_int, C.c_int, C.c_char_p, C.c_int]),
        "ztp_ctx_destroy": (st, [vp]),
        "ztp_sync": (st, [vp, vp]),
        "ztp_launch_count": (C.c_int64, [vp]),
        "ztp_plan_opts_default": (None, [C.POINTER(PlanOpts)]),
        "ztp_plan": (st, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double,
                          C.POINTER(Costs), C.POINTER(PlanOpts), C.POINTER(PlanT)]),
        "ztp_plan_refine": (st, [C.POINTER(PlanT), C.POINTER(PlanT), C.c_double, C.POINTER(PlanT)]),
        "ztp_ctl_opts_default": (None, [C.POINTER(CtlOpts)]),
        "ztp_ctl_init": (st, [C.POINTER(Ctl), C.c_int]),
        "ztp_ctl_step": (st, [C.POINTER(Ctl), C.POINTER(CtlOpts), C.POINTER(Costs), C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
        "ztp_layer_prune_counts": (st, [C.POINTER(PlanT), C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_int32)]),
        "ztp_plan_uniform": (st, [C.c_int, C.c_double, C.POINTER(PlanT)]),
        "ztp_pridiff_counts": (C.c_int32, [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double]),
        "ztp_costs_fit": (st, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int,
                               C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double),
                               C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(Costs)]),
        "ztp_plan_counts": (st, [C.POINTER(PlanT), C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                 C.POINTER(Counts)]),
        "ztp_allgather_stats": (st, [vp, C.c_double, C.c_double, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), vp]),
        "ztp_select": (st, [vp, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                            vp, vp, vp, vp, vp]),
        "ztp_join": (st, [vp, vp]),
        "ztp_col_linear": (st, [vp, C.c_int, C.POINTER(LinearArgs), vp]),
        "ztp_row_linear": (st, [vp, C.c_int, C.POINTER(LinearArgs), vp]),
        "ztp_core": (st, [vp, C.c_int, C.POINTER(Mat), C.POINTER(Mat), C.c_int64, C.c_int64, vp, C.c_int64,
                          C.c_int32, vp]),
        "ztp_migrate": (st, [vp, C.c_int, C.POINTER(Xfer), vp]),
        "ztp_set_slowdown": (st, [vp, C.c_double]),
        "ztp_set_stats": (st, [vp, C.c_int]),
        "ztp_read_gemm_ns": (st, [vp, vp, C.POINTER(C.c_double)]),
        "ztp_gemm": (st, [vp, C.c_int, C.POINTER(LinearArgs), vp]),
        "ztp_prepare": (st, [vp, C.c_int, C.POINTER(C.POINTER(LinearArgs)), C.POINTER(C.c_int32), vp]),
        "ztp_priority_update": (st, [vp, C.POINTER(Mat), C.POINTER(Mat), vp, vp, vp, C.c_float, vp]),
        "ztp_read_stamps": (C.c_int, [vp, vp, C.POINTER(C.c_uint64), C.c_int]),
        "ztp_read_cta_stamps": (C.c_int, [vp, vp, C.POINTER(C.c_uint64), C.c_int]),
        "ztp_pridiff_gamma": (C.c_double, [C.c_int64, C.c_int64, C.c_double, C.c_double]),
        "ztp_set_profile": (st, [vp, C.c_int]),
        "ztp_window_create": (st, [vp, C.c_size_t, C.c_char_p]),
        "ztp_window_open": (st, [vp, C.c_char_p]),
        "ztp_sym_alloc": (st, [vp, C.c_size_t, C.POINTER(vp)]),
        "ztp_set_transport": (st, [vp, C.c_int]),
        "ztp_barrier": (st, [vp, vp]),
        "ztp_set_option": (st, [vp, C.c_int, C.c_double]),
        "ztp_broadcast": (st, [vp, C.c_int, C.POINTER(Mat), C.c_int, vp]),
        "ztp_reduce": (st, [vp, C.c_int, C.POINTER(Mat), C.c_int, vp]),
        "ztp_accumulate": (st, [vp, C.POINTER(Mat), C.POINTER(Mat), vp]),
        "ztp_allreduce": (st, [vp, C.POINTER(Mat), vp]),
        "ztp_transpose": (st, [vp, C.POINTER(Mat), C.POINTER(Mat), vp, C.c_int64, vp]),
        "ztp_get_option": (st, [vp, C.c_int, C.POINTER(C.c_double)]),
        "ztp_read_profile": (st, [vp, vp, C.POINTER(Profile)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()

# every symbol include/ztp.h declares (checked by tests/test_abi.py)
EXPORTED = ("ztp_status_str", "ztp_last_error", "ztp_version", "ztp_get_unique_id", "ztp_ctx_create",
            "ztp_ctx_destroy", "ztp_sync", "ztp_launch_count", "ztp_plan_opts_default", "ztp_plan", "ztp_plan_refine",
            "ztp_ctl_opts_default", "ztp_ctl_init", "ztp_ctl_step", "ztp_plan_counts",
            "ztp_layer_prune_counts", "ztp_plan_uniform", "ztp_pridiff_counts", "ztp_costs_fit", "ztp_allgather_stats", "ztp_select", "ztp_join", "ztp_col_linear", "ztp_row_linear",
            "ztp_core", "ztp_migrate", "ztp_set_slowdown", "ztp_set_stats", "ztp_read_gemm_ns", "ztp_gemm", "ztp_prepare",
            "ztp_priority_update", "ztp_pridiff_gamma", "ztp_read_stamps",
            "ztp_set_profile", "ztp_read_profile", "ztp_window_create", "ztp_window_open", "ztp_sym_alloc",
            "ztp_set_transport", "ztp_barrier", "ztp_set_option", "ztp_get_option", "ztp_broadcast", "ztp_reduce",
            "ztp_accumulate", "ztp_allreduce", "ztp_transpose",
            "ztp_read_cta_stamps")


def check(code: int, ctx=None):
    if code != 0:
        msg = lib.ztp_last_error(ctx)
        raise ZtpError(code, msg.decode() if msg else "")

"""GEMM-only timing of the c2 (gamma = 0.5, output-pruned) GEMM shapes with
dense operands, per epilogue variant and ZTP_DEBUG_EPI mode (0 full, 1 no
stores, 2 no epilogue body) -- where the time of the small-K GEMMs goes.
Performance experiment only (dbg > 0 results are invalid by design)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402

N = 8192
bf = torch.bfloat16


def r(*s):
    return (torch.rand(*s, device="cuda") * 2 - 1).to(bf)


def cases():
    out = {}
    # FWD y[n, N] = W^T[K, n]^T X^T[K, N]
    for name, K, n, gelu in (("fc1_fwd_gelu", 512, 2048, True), ("fc1_fwd_plain", 512, 2048, False),
                             ("qkv_fwd", 512, 3072, False), ("fc2_fwd", 2048, 1024, False),
                             ("o_fwd", 512, 1024, False)):
        w, x = r(K, n), r(K, N)
        y, pre = torch.empty(n, N, device="cuda", dtype=bf), torch.empty(n, N, device="cuda", dtype=bf)
        a = Z.linear_args(x_t=x, w_t=w, y_t=y, pre_t=pre if gelu else None, act=Z.ACT_GELU if gelu else Z.ACT_NONE)
        out[name] = (Z.KIND_FWD, a, (w, x, y, pre))
    # DX dx[K, N] = W^T[K, n] G^T[n, N]
    for name, K, n, gg in (("fc2_dx_gelugrad", 2048, 1024, 1), ("fc2_dx_mul", 2048, 1024, 2),
                           ("fc2_dx_plain", 2048, 1024, 0), ("fc1_dx", 512, 2048, 0)):
        w, g = r(K, n), r(n, N)
        dx, pin = torch.empty(K, N, device="cuda", dtype=bf), r(K, N)
        a = Z.linear_args(w_t=w, g_t=g, dx_t=dx, pre_in_t=pin if gg else None,
                          act_in=[Z.ACT_NONE, Z.ACT_GELU, Z.ACT_GELU_D][gg])
        out[name] = (Z.KIND_DX, a, (w, g, dx, pin))
    # DW dw[K, n] = X^T[K, N] G^T[n, N]^T
    for name, K, n in (("fc2_dw", 2048, 1024), ("fc1_dw", 512, 2048), ("o_dw", 512, 1024), ("qkv_dw", 512, 3072)):
        x, g = r(K, N), r(n, N)
        dw = torch.empty(K, n, device="cuda", dtype=bf)
        a = Z.linear_args(x_t=x, g_t=g, dw_t=dw, w_t=dw)
        out[name] = (Z.KIND_DW, a, (x, g, dw))
    return out


def main():
    modes = [int(m) for m in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2").split(",")]
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    cs = cases()
    for dbg in modes:
        os.environ["ZTP_DEBUG_EPI"] = str(dbg)
        ctx = Z.ztp_ctx_create(0, 1, None, 0)
        for name, (kind, a, _) in cs.items():
            if only and name not in only:
                continue
            for _ in range(3):
                Z.ztp_gemm(ctx, kind, a)
            torch.cuda.synchronize()
            Z.ztp_read_profile(ctx)
            Z.ztp_set_profile(ctx, True)
            torch.cuda._sleep(int(1e8))
            for _ in range(20):
                Z.ztp_gemm(ctx, kind, a)
            prof = Z.ztp_read_profile(ctx)
            Z.ztp_set_profile(ctx, False)
            t = prof["gemm_kernel_ms"] / 20
            tf = prof["gemm_flops"] / 20 / (t * 1e-3) / 1e12
            print(f"dbg={dbg} {name:16s} {t * 1e3:7.1f} us {tf:7.1f} TF/s", flush=True)
        Z.ztp_ctx_destroy(ctx)


if __name__ == "__main__":
    main()

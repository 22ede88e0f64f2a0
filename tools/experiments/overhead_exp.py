"""Fixed vs per-tile cost of the tcgen05 GEMM: dense FWD with M = 256 (one
m-tile per CTA pair) and N = 256 * 74 * t tokens (t tiles per pair), K in
{128, 512, 2048}; kernel time from the GEMM's own %globaltimer stamps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402

bf = torch.bfloat16
ctx = Z.ztp_ctx_create(0, 1, None, 0)
peak_pair = 1604.9e12 / 74
for K in (128, 512, 2048):
    for t in (1, 2, 4):
        M, N = 256, 256 * 74 * t
        w = (torch.rand(K, M, device="cuda") - 0.5).to(bf)
        x = (torch.rand(K, N, device="cuda") - 0.5).to(bf)
        y = torch.empty(M, N, device="cuda", dtype=bf)
        for epi in ("plain", "gelu"):
            pre = torch.empty(M, N, device="cuda", dtype=bf) if epi == "gelu" else None
            a = Z.linear_args(x_t=x, w_t=w, y_t=y, pre_t=pre, act=Z.ACT_GELU_D if epi == "gelu" else Z.ACT_NONE)
            for _ in range(3):
                Z.ztp_gemm(ctx, Z.KIND_FWD, a)
            torch.cuda.synchronize()
            Z.ztp_read_profile(ctx)
            Z.ztp_set_profile(ctx, True)
            torch.cuda._sleep(int(5e7))
            for _ in range(20):
                Z.ztp_gemm(ctx, Z.KIND_FWD, a)
            prof = Z.ztp_read_profile(ctx)
            Z.ztp_set_profile(ctx, False)
            us = prof["gemm_kernel_ms"] / 20 * 1e3
            ideal = 2.0 * M * 256 * K * t / peak_pair * 1e6
            print(f"K={K:5d} tiles/pair={t} {epi:5s} kernel {us:6.2f} us  ideal {ideal:6.2f} us  "
                  f"overhead {us - ideal:6.2f} us", flush=True)
Z.ztp_ctx_destroy(ctx)

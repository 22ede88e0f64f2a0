"""Wave quantization check: the same GEMM at N = 8192 (tiles not a multiple of
74 pairs) and at N = 256 * 37 * k / ... (tiles a multiple of 74)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402

bf = torch.bfloat16
ctx = Z.ztp_ctx_create(0, 1, None, 0)
for (M, K) in ((2048, 512), (1024, 512), (512, 2048), (2560, 512)):
    for N in (8192, 9472, 7168):
        w = (torch.rand(K, M, device="cuda") - 0.5).to(bf)
        x = (torch.rand(K, N, device="cuda") - 0.5).to(bf)
        y = torch.empty(M, N, device="cuda", dtype=bf)
        a = Z.linear_args(x_t=x, w_t=w, y_t=y)
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
        tiles = (M // 256) * ((N + 255) // 256)
        print(f"M={M} K={K} N={N} tiles={tiles} ({tiles / 74:.2f} rounds) {us:6.1f} us "
              f"{2 * M * N * K / us / 1e6:7.1f} TF/s", flush=True)
Z.ztp_ctx_destroy(ctx)

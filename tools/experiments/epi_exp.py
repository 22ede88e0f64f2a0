"""Epilogue variants of the FWD GEMM at the c2 FC1 shape (K'=512): plain,
GeLU (two planes), output row map (scatter4), both.  GEMM-only time from the
library's CUDA-event profile."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402

K, n, N = 1024, 4096, 8192
ctx = Z.ztp_ctx_create(0, 1, None, 0)
x = torch.randn(K, N, device="cuda").bfloat16()
w = (torch.rand(K, n, device="cuda") * 2 - 1).mul_(1 / math.sqrt(K)).bfloat16()
npr = 512
perm = torch.randperm(K, generator=torch.Generator().manual_seed(1))
S = torch.sort(perm[npr:]).values.int().cuda()
P = torch.sort(perm[:npr]).values.int().cuda()
xs = torch.empty(K - npr, N, device="cuda", dtype=torch.bfloat16)
ws = torch.empty(K - npr, n, device="cuda", dtype=torch.bfloat16)
s = Z.sel(S, K - npr, P, npr, 0, 0)
y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
pre = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
pos = torch.full((n,), -1, dtype=torch.int32)
keep = torch.sort(torch.randperm(n, generator=torch.Generator().manual_seed(2))[: n // 2]).values
pos[keep] = torch.arange(n // 2, dtype=torch.int32)
pos = pos.cuda()
yc = torch.empty(n // 2, N, device="cuda", dtype=torch.bfloat16)
prec = torch.empty(n // 2, N, device="cuda", dtype=torch.bfloat16)
variants = {
    "plain": Z.linear_args(x_t=x, w_t=w, y_t=y, sel_=s, xs_t=xs, ws_t=ws),
    "gelu": Z.linear_args(x_t=x, w_t=w, y_t=y, pre_t=pre, sel_=s, xs_t=xs, ws_t=ws, act=Z.ACT_GELU),
    "ypos": Z.linear_args(x_t=x, w_t=w, y_t=yc, sel_=s, xs_t=xs, ws_t=ws, y_pos=pos),
    "gelu+ypos": Z.linear_args(x_t=x, w_t=w, y_t=yc, pre_t=prec, sel_=s, xs_t=xs, ws_t=ws, act=Z.ACT_GELU,
                               y_pos=pos),
}
for name, a in variants.items():
    for _ in range(3):
        Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    torch.cuda.synchronize()
    Z.ztp_read_profile(ctx)
    Z.ztp_set_profile(ctx, True)
    torch.cuda._sleep(int(1e8))
    for _ in range(20):
        Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    prof = Z.ztp_read_profile(ctx)
    Z.ztp_set_profile(ctx, False)
    t = prof["gemm_ms"] / 20
    print(f"{name:10s} {t * 1e3:7.1f} us  {prof['gemm_flops'] / 20 / (t * 1e-3) / 1e12:7.1f} TF/s", flush=True)

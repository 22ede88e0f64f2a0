"""Micro-benchmark of the resized GEMMs through the C ABI (CUDA events on the
launching stream, warm-up, inputs > L2 rotated).  Prints TFLOP/s per kind."""
import argparse
import json
import math

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2401_11469_b200 as Z


def run(K, n, N, gamma, iters=20, kinds=(0, 1, 2)):
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(K, N, device="cuda", generator=g).bfloat16()
    w = (torch.rand(K, n, device="cuda", generator=g) * 2 - 1).mul_(1 / math.sqrt(K)).bfloat16()
    gt = torch.randn(n, N, device="cuda", generator=g).bfloat16()
    y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
    dw = torch.empty(K, n, device="cuda", dtype=torch.bfloat16)
    npr = int(math.floor(K * gamma + 0.5))
    perm = torch.randperm(K, generator=torch.Generator().manual_seed(1))
    S = torch.sort(perm[npr:]).values.int().cuda()
    P = torch.sort(perm[:npr]).values.int().cuda() if npr else torch.zeros(1, dtype=torch.int32, device="cuda")
    s = Z.sel(S, K - npr, P, npr, 0, 0)
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=gt, dx_t=dx, dw_t=dw, sel_=s)
    out = {}
    for kind in kinds:
        for _ in range(3):
            Z.ztp_gemm(ctx, kind, a)
        torch.cuda.synchronize()
        Z.ztp_read_profile(ctx)
        Z.ztp_set_profile(ctx, True)
        for _ in range(iters):
            Z.ztp_gemm(ctx, kind, a)
        prof = Z.ztp_read_profile(ctx)
        Z.ztp_set_profile(ctx, False)
        t = prof["gemm_ms"] / iters * 1e-3           # GEMM kernel(s) only, CUDA events
        flops = prof["gemm_flops"] / iters
        out[["fwd", "dx", "dw"][kind]] = dict(ms=t * 1e3, tflops=flops / t / 1e12)
    Z.ztp_ctx_destroy(ctx)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="1024,4096,8192;4096,1024,8192;1024,3072,8192;1024,1024,8192")
    ap.add_argument("--gammas", default="0,0.5")
    args = ap.parse_args()
    for sh in args.shapes.split(";"):
        K, n, N = map(int, sh.split(","))
        for gm in map(float, args.gammas.split(",")):
            r = run(K, n, N, gm)
            print(json.dumps(dict(K=K, n=n, N=N, gamma=gm, **r)), flush=True)

"""Short driver for ncu captures of the resized GEMM kernels (one launch per
kind at the c2 TP=1 FC1 shapes, gamma=0.5, compact operands)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402

K, n, N = int(os.environ.get("K", 1024)), int(os.environ.get("NN", 4096)), int(os.environ.get("TOK", 8192))
gamma = float(os.environ.get("GAMMA", 0.5))
ctx = Z.ztp_ctx_create(0, 1, None, 0)
x = torch.randn(K, N, device="cuda").bfloat16()
w = (torch.rand(K, n, device="cuda") * 2 - 1).mul_(1 / math.sqrt(K)).bfloat16()
g = torch.randn(n, N, device="cuda").bfloat16()
y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
dx = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(K, n, device="cuda", dtype=torch.bfloat16)
npr = int(K * gamma + 0.5)
perm = torch.randperm(K, generator=torch.Generator().manual_seed(1))
S = torch.sort(perm[npr:]).values.int().cuda()
P = torch.sort(perm[:npr]).values.int().cuda() if npr else torch.zeros(1, dtype=torch.int32, device="cuda")
xs = torch.empty(K - npr, N, device="cuda", dtype=torch.bfloat16)
ws = torch.empty(K - npr, n, device="cuda", dtype=torch.bfloat16)
s = Z.sel(S, K - npr, P, npr, 0, 0)
act = os.environ.get("ACT", "")
pre = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
pin = torch.randn(K, N, device="cuda").bfloat16()
if act == "gelu":
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, pre_t=pre, g_t=g, dx_t=dx, dw_t=dw, sel_=s, xs_t=xs, ws_t=ws,
                      act=Z.ACT_GELU, act_in=Z.ACT_GELU, pre_in_t=pin)
else:
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=g, dx_t=dx, dw_t=dw, sel_=s, xs_t=xs, ws_t=ws)
for it in range(2):
    for kind in (Z.KIND_FWD, Z.KIND_DX, Z.KIND_DW):
        Z.ztp_gemm(ctx, kind, a)
torch.cuda.synchronize()
Z.ztp_ctx_destroy(ctx)
print("done")

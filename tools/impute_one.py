"""One col-linear BWD at c2 FC1 shapes (K = 1024 input rows, n = 4096,
N = 8192 tokens) with Average or Same imputation of the pruned rows
(NEXT-2): the launches ncu profiles for the impute kernels'
bandwidth (tools/gpu_nongemm.sh).  POLICY=average|same, GAMMA."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402

K, n, N = 1024, 4096, 8192
gamma = float(os.environ.get("GAMMA", "0.5"))
pol = {"average": Z.IMPUTE_AVERAGE, "same": Z.IMPUTE_SAME}[os.environ.get("POLICY", "average")]
ctx = Z.ztp_ctx_create(0, 1, None, 0)
x = torch.randn(K, N, device="cuda").bfloat16()
w = (torch.rand(K, n, device="cuda") * 2 - 1).mul_(1 / math.sqrt(K)).bfloat16()
g = torch.randn(n, N, device="cuda").bfloat16()
dx = torch.empty(K, N, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(K, n, device="cuda", dtype=torch.bfloat16)
hdx, hdw = torch.randn(K, N, device="cuda").bfloat16(), torch.randn(K, n, device="cuda").bfloat16()
npr = int(K * gamma + 0.5)
perm = torch.randperm(K, generator=torch.Generator().manual_seed(1))
S = torch.sort(perm[npr:]).values.int().cuda()
P = torch.sort(perm[:npr]).values.int().cuda()
s = Z.sel(S, K - npr, P, npr, 0, 0)
y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
fa = Z.linear_args(x_t=x, w_t=w, y_t=y, sel_=s)
ba = Z.linear_args(x_t=x, w_t=w, g_t=g, dx_t=dx, dw_t=dw, sel_=s, impute=pol, hist_dx=hdx, hist_dw=hdw)
for _ in range(3):
    Z.ztp_col_linear(ctx, Z.FWD, fa)
    Z.ztp_col_linear(ctx, Z.BWD, ba)
    Z.ztp_join(ctx)
torch.cuda.synchronize()
Z.ztp_ctx_destroy(ctx)
print("done")

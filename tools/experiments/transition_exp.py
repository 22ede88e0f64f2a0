"""Is a tile transition costly, or is it the clock?  Dense FWD, M = 256,
t tiles per pair, K per tile; one launch right after an idle gap (boost
clock) and 20 back-to-back launches; kernel time from %globaltimer stamps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402

bf = torch.bfloat16
ctx = Z.ztp_ctx_create(0, 1, None, 0)
print("ZTP_DEBUG_EPI", os.environ.get("ZTP_DEBUG_EPI", "0"))
peak_pair = 1604.9e12 / 74
for K, t in ((2048, 1), (8192, 1), (2048, 4), (512, 16), (8192, 4)):
    M, N = 256, 256 * 74 * t
    w = (torch.rand(K, M, device="cuda") - 0.5).to(bf)
    x = (torch.rand(K, N, device="cuda") - 0.5).to(bf)
    y = torch.empty(M, N, device="cuda", dtype=bf)
    a = Z.linear_args(x_t=x, w_t=w, y_t=y)
    for _ in range(3):
        Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    ideal = 2.0 * M * 256 * K * t / peak_pair * 1e6
    for reps in (1,):
        torch.cuda.synchronize()
        time_idle = 0.2
        torch.cuda._sleep(int(4e8))            # idle-ish gap (one SM spinning)
        torch.cuda.synchronize()
        Z.ztp_read_profile(ctx)
        Z.ztp_set_profile(ctx, True)
        for _ in range(reps):
            Z.ztp_gemm(ctx, Z.KIND_FWD, a)
        prof = Z.ztp_read_profile(ctx)
        Z.ztp_set_profile(ctx, False)
        us = prof["gemm_kernel_ms"] / reps * 1e3
        print(f"K={K:5d} tiles/pair={t:2d} reps={reps:2d} kernel {us:7.2f} us ideal {ideal:7.2f} "
              f"eff {ideal / us:5.3f}", flush=True)
Z.ztp_ctx_destroy(ctx)

"""ztp_select timing: c2 TP=1 segments {1024, 1024, 1024, 4096} at gamma 0.5,
100 back-to-back launches (CUDA events) and single launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402
from synth import inputs as I  # noqa: E402

ctx = Z.ztp_ctx_create(0, 1, None, 0)
lens = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024,4096").split(",")]
nps = [L // 2 for L in lens]
sc = torch.from_numpy(np.concatenate([I.lognormal_scores(1, f"s{i}", L) for i, L in enumerate(lens)])).cuda()
kept = torch.empty(sum(lens), dtype=torch.int32, device="cuda")
pr = torch.empty(sum(lens), dtype=torch.int32, device="cuda")
pos = torch.empty(sum(lens), dtype=torch.int32, device="cuda")
for _ in range(5):
    Z.ztp_select(ctx, lens, nps, sc, kept, pr, None, pos)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(1e8))
e0.record()
for _ in range(100):
    Z.ztp_select(ctx, lens, nps, sc, kept, pr, None, pos)
e1.record()
torch.cuda.synchronize()
print(f"lens {lens}: {e0.elapsed_time(e1) * 10:.2f} us per select (100 back-to-back)")
Z.ztp_ctx_destroy(ctx)

"""In-graph GEMM timeline of the c2 TP=1 gamma=0.5 step: the step captured
with stamp-only profiling, one replay, the 12 GEMM [start, end] intervals
relative to the replay start; gaps = the non-GEMM kernels (select, copies,
core, split-K reduces are inside the GEMM spans) and launch overheads."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth import inputs as I  # noqa: E402
import bench  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c2")]
h, f, N = cfg.h, cfg.f, cfg.N
ctx = Z.ztp_ctx_create(0, 1, None, 0)
sh = bench.rank_shards(cfg, 1, 0)
dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
L = ZtpLayer(ctx, h, f, N, 0, 1, dev)
sc = {s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, 0, {"qkv": h, "o": h, "fc1": h, "fc2": f}).items()}
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
p = Z.PlanT()
p.world = 1
p.role[0] = Z.RESIZE
p.gamma[0] = p.gamma_r[0] = 0.5
n_prune = {s: Z.ztp_plan_counts(p, 0, K, f, 1, s in ("o", "fc2")).n_prune
           for s, K in (("qkv", h), ("o", h), ("fc1", h), ("fc2", f))}
L.set_selection(n_prune, sc)
for _ in range(3):
    L.step(stream, select=False)
torch.cuda.synchronize()
Z.ztp_set_profile(ctx, 2)
g = L.capture(stream, select=False)   # selection once per plan
for _ in range(300):
    g.replay()
Z.ztp_read_profile(ctx, stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(50):
    g.replay()
Z.ztp_read_profile(ctx, stream)            # reset stamps after a warm run
e0.record(stream)
g.replay()
e1.record(stream)
st = Z.ztp_read_stamps(ctx, stream)
torch.cuda.synchronize()
names = ["QKV fwd", "O fwd", "FC1 fwd", "FC2 fwd", "FC2 dX", "FC2 dW", "FC1 dX", "FC1 dW", "O dX", "O dW",
         "QKV dX", "QKV dW"]
t0 = min(a for a, _ in st)
prev_end = t0
busy = 0
for i, (a, b) in enumerate(st):
    print(f"{names[i] if i < len(names) else i:8s} start {(a - t0) / 1e3:7.1f} us  end {(b - t0) / 1e3:7.1f} us  "
          f"len {(b - a) / 1e3:6.1f}  gap-before {(a - prev_end) / 1e3:6.1f}")
    prev_end = max(prev_end, b)
print(f"replay (events) {e0.elapsed_time(e1) * 1e3:.1f} us; first GEMM start .. last GEMM end "
      f"{(max(b for _, b in st) - t0) / 1e3:.1f} us")

"""c2 TP=1 gamma=0.5 layer: 2 warm-up steps then STEPS more (default 1),
un-captured -- the launch sequence ncu profiles (tools/gpu_profiles.sh)."""
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
L.X.copy_(torch.from_numpy(I.normal(cfg.seed, "x", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
L.G.copy_(torch.from_numpy(I.normal(cfg.seed, "g", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
sc = {s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, 0, {"qkv": h, "o": h, "fc1": h, "fc2": f}).items()}
p = Z.PlanT()
p.world = 1
p.role[0] = Z.RESIZE
p.gamma[0] = p.gamma_r[0] = float(os.environ.get("GAMMA", "0.5"))
n_prune = {s: Z.ztp_plan_counts(p, 0, K, f, 1, s in ("o", "fc2")).n_prune
           for s, K in (("qkv", h), ("o", h), ("fc1", h), ("fc2", f))}
L.set_selection(n_prune, sc)
for _ in range(2 + int(os.environ.get("STEPS", "1"))):
    L.step()
torch.cuda.synchronize()
print("flops", L.method_flops(), L.executed_flops())

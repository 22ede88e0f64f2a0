"""Per-CTA phases of every GEMM launch of one c2 TP=1 gamma=0.5 step,
inside the captured step graph (profiling mode 3): for each launch the
median / max over CTAs of  wait = PDL wait end - CTA start,  fill = first
operand stage ready - PDL wait end,  main = last MMA commit - first stage,
tail = stores complete - last MMA commit,  end = CTA end - stores complete,
and the launch span (first PDL-wait end .. last CTA end).  Under the A-operand
prefetch (ZTP_OPT_A_EARLY) the producer warp waits for the predecessor only
after issuing its first A loads, and thread 0 stamps the wait end before
that: such a launch's remaining PDL wait shows up in `fill` (e.g. FC2 FWD
right after FC1 FWD's long two-plane tail).
TP = e > 1 (env TP, GAMMA): rank 0's shard of a TP = e layer, collectives not run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
import bench  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c2")]
h, f, N = cfg.h, cfg.f, cfg.N
e = int(os.environ.get("TP", "1"))        # TP > 1: rank 0's shard of a TP = e layer (collectives not run)
a, u = h // e, f // e
gamma = float(os.environ.get("GAMMA", "0.5"))
ctx = Z.ztp_ctx_create(0, 1, None, 0)
sh = bench.rank_shards(cfg, e, 0)
dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
L = ZtpLayer(ctx, h, f, N, 0, e, dev)
L.X.normal_()
L.G.normal_()
sc = {s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, 0, {"qkv": h, "o": a, "fc1": h, "fc2": u}).items()}
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
if e == 1:
    L.set_selection(Z.ztp_layer_prune_counts(Z.ztp_plan_uniform(1, gamma), 0, h, h, f), sc)
else:
    from paper_2401_11469_b200.layer import layer_prune_counts
    p = Z.PlanT()
    p.world = e
    p.role[0] = Z.RESIZE if gamma > 0 else Z.NORMAL
    p.gamma[0] = p.gamma_r[0] = gamma
    L.set_selection(layer_prune_counts(p, 0, h, a, u), sc)
for _ in range(3):
    L.step(stream, select=False)
torch.cuda.synchronize()
Z.ztp_set_profile(ctx, 3)
g = L.capture(stream, select=False)
for _ in range(200):
    g.replay()
Z.ztp_read_profile(ctx, stream)
g.replay()
st = Z.ztp_read_cta_stamps(ctx, stream).astype(np.int64)
torch.cuda.synchronize()
names = ["QKV fwd", "O fwd", "FC1 fwd", "FC2 fwd", "FC2 dX", "FC2 dW", "FC1 dX", "FC1 dW", "O dX", "O dW",
         "QKV dX", "QKV dW"]
t0 = min(int(x[:, 1][x[:, 1] > 0].min()) for x in st if (x[:, 1] > 0).any())
print(f"{'GEMM':8s} {'CTAs':>4s} {'start':>7s} {'span':>6s} | median / max over CTAs (us): {'wait':>11s} {'fill':>11s}"
      f" {'main':>11s} {'tail':>11s} {'end':>11s}")
for i, x in enumerate(st):
    ok = np.nonzero(x[:, 0] > 0)[0]
    if not len(ok):
        continue
    lead = ok[(ok % 2 == 0) & (x[ok, 2] > 0)]               # 2-CTA pairs: the even CTA issues the MMAs
    fol = ok[x[ok & ~1, 3] > 0] if len(lead) else ok

    def q(a):
        return f"{np.median(a) / 1e3:5.2f}/{np.max(a) / 1e3:5.2f}" if len(a) else "    -"
    span = (x[ok, 7].max() - x[ok, 1].min()) / 1e3
    tail = x[fol, 6] - x[fol & ~1, 3]
    print(f"{names[i] if i < len(names) else i:8s} {len(ok):4d} {(x[ok, 1].min() - t0) / 1e3:7.1f} {span:6.1f} | "
          f"{q(x[ok, 1] - x[ok, 0]):>24s} {q(x[lead, 2] - x[lead, 1]):>11s} {q(x[lead, 3] - x[lead, 2]):>11s} "
          f"{q(tail):>11s} {q(x[ok, 7] - x[ok, 6]):>11s}")

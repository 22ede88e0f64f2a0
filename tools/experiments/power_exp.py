"""Step-time drift vs SM clock / power: the c2 TP=1 gamma=0.5 step graph
replayed in chunks of 100 steps for ~2 s while nvidia-smi samples clocks,
power and throttle reasons every 20 ms.  Diagnostics only."""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer, SEGS  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth import inputs as I  # noqa: E402
import bench  # noqa: E402

cfg = CONFIGS["c2"]
h, f, N = cfg.h, cfg.f, cfg.N
ctx = Z.ztp_ctx_create(0, 1, None, 0)
sh = bench.rank_shards(cfg, 1, 0)
dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
L = ZtpLayer(ctx, h, f, N, 0, 1, dev)
L.X.copy_(torch.from_numpy(I.normal(cfg.seed, "x", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
L.G.copy_(torch.from_numpy(I.normal(cfg.seed, "g", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
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
for _ in range(2):
    L.step(stream)
torch.cuda.synchronize()
g = L.capture(stream)
torch.cuda.synchronize()

samples = []
stop = threading.Event()


def sampler():
    cmd = ["nvidia-smi", "-i", "0", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active",
           "--format=csv,noheader,nounits", "-lms", "20"]
    pr = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    while not stop.is_set():
        line = pr.stdout.readline()
        if not line:
            break
        samples.append((time.time(), line.strip()))
    pr.kill()


th = threading.Thread(target=sampler, daemon=True)
th.start()
time.sleep(0.5)
t0 = time.time()
res = []
for chunk in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(100):
        g.replay()
    e1.record(stream)
    e1.synchronize()
    res.append((time.time() - t0, e0.elapsed_time(e1) / 100))
time.sleep(0.3)
stop.set()
th.join(timeout=2)
for t, ms in res:
    print(f"t={t:6.3f}s step {ms * 1e3:6.1f} us")
for ts, s in samples:
    print(f"smi t={ts - t0:6.3f} {s}")

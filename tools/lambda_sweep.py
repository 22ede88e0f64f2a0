"""NEXT-4 forced-lambda sweep, simulated on one GPU.

Eight TP ranks of the c4 layer (h = 4096, f = 11008, N = 2048) are simulated
with one context each on a single B200; four are slowed by chi = {8, 6, 4, 2}
(ranks 1, 3, 5, 7; the paper's multi-straggler setting) with the library's
delay kernel (A-32).  For lambda = 0..4 the SEMI plan is forced
(`force_lambda`): the lambda slowest stragglers migrate their Eq.1 share of MLP
units to the other ranks (A-26), the rest resize.  Each rank's step is timed
alone (graph replay, its own slowdown); a TP step cannot be faster than its
slowest rank, so the simulated step time is max_r T_r.  Collectives and
NVLink transfers are not simulated (one GPU): the all-reduce time is the same
for every lambda, the weight migration is a per-replan cost."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer, migration_io, layer_prune_counts, SEGS  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
import bench  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c4")]
e = 8
h, f, N = cfg.h, cfg.f, cfg.N
a, u = h // e, f // e
chi = {1: 8.0, 3: 6.0, 5: 4.0, 7: 2.0}
STEPS = int(os.environ.get("STEPS", "30"))


def time_rank(L, ctx, chi_r, steps=STEPS):
    stream = torch.cuda.Stream()
    Z.ztp_set_slowdown(ctx, chi_r)
    for _ in range(2):
        L.step(stream)
    torch.cuda.synchronize()
    g = L.capture(stream)
    with torch.cuda.stream(stream):      # replay() issues on the current stream
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    del g
    return e0.elapsed_time(e1) / steps


def main():
    ctxs = [Z.ztp_ctx_create(0, 1, None, 0) for _ in range(e)]
    shards = [bench.rank_shards(cfg, e, r) for r in range(e)]
    lens = {"qkv": h, "o": a, "fc1": h, "fc2": u}
    scores = [{s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, r, lens).items()} for r in range(e)]
    # statistics window: dense step per rank with its slowdown (A-5, A-6)
    cap = u                                         # spare capacity for received units
    layers = []
    for r in range(e):
        dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in shards[r].items()}
        L = ZtpLayer(ctxs[r], h, f, N, r, e, dev, mig_cap=cap)
        # single-GPU simulation: the per-step weight / dW peer copies of SEMI
        # (NVLink on a real box) are done once below as local copies
        L.migrate_weights = lambda stream=None: None
        L.return_grads = lambda stream=None: None
        L.X.normal_()
        L.G.normal_()
        layers.append(L)
    T, M = [], []
    for r, L in enumerate(layers):
        L.set_selection({s: 0 for s in SEGS}, scores[r])
        t = time_rank(L, ctxs[r], chi.get(r, 1.0))
        Z.ztp_set_stats(ctxs[r], True)
        Z.ztp_read_gemm_ns(ctxs[r])
        for _ in range(5):
            L.step()
        m = Z.ztp_read_gemm_ns(ctxs[r]) / 5 / 1e6
        Z.ztp_set_stats(ctxs[r], False)
        T.append(t)
        M.append(m)
    free = [time_rank(L, ctxs[r], 1.0) for r, L in enumerate(layers)]
    rows = []
    w1_0 = [L.w1_t.clone() for L in layers]
    w2_0 = [L.w2_t.clone() for L in layers]
    for lam in range(5):
        plan = Z.ztp_plan(T, M, float(u), None, Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN,
                                                               force_lambda=lam))
        per = []
        for r, L in enumerate(layers):
            L.w1_t.copy_(w1_0[r])
            L.w2_t.copy_(w2_0[r])
        mios = [migration_io(plan, r, e, u, h) for r in range(e)]
        for r, L in enumerate(layers):
            L.set_migration(mios[r])
        for (src, dst, lo, hi, off) in mios[0].all_xfers:       # local stand-in for ztp_migrate over NVLink
            Ls, Ld = layers[src], layers[dst]
            Ld.w1_t[:, u + off:u + off + hi - lo].copy_(Ls.w1_t[:, lo:hi])
            Ld.w2_t[u + off:u + off + hi - lo].copy_(Ls.w2_t[lo:hi])
        for r, L in enumerate(layers):
            L.set_selection(layer_prune_counts(plan, r, h, a, u), scores[r])
            per.append(time_rank(L, ctxs[r], chi.get(r, 1.0)))
        roles = ["NRMS"[int(x)] if int(x) < 4 else "?" for x in list(plan.role)[:e]]   # normal/resize/migrate/split
        rows.append({"lambda": lam, "x": plan.x, "z": plan.z, "roles": "".join(roles),
                     "gamma": [round(g, 3) for g in list(plan.gamma)[:e]],
                     "step_ms": max(per), "per_rank_ms": [round(p, 4) for p in per]})
        print(json.dumps(rows[-1]), flush=True)
    out = {"config": cfg.name, "tp": e, "chi": chi, "T_unbal_ms": max(T), "T_free_ms": max(free),
           "per_rank_unbal_ms": T, "sweep": rows,
           "note": "one-GPU simulation: each rank timed alone with its slowdown; TP step = max over ranks; "
                   "collectives not simulated"}
    best = min(rows, key=lambda r: r["step_ms"])
    print(json.dumps({"T_free_ms": out["T_free_ms"], "T_unbal_ms": out["T_unbal_ms"], "best_lambda": best["lambda"],
                      "best_step_ms": best["step_ms"], "recovery_best": out["T_free_ms"] / best["step_ms"]}))
    json.dump(out, open(os.environ.get("OUT", "gpurun_out/lambda_sweep.json"), "w"), indent=1)
    for c in ctxs:
        Z.ztp_ctx_destroy(c)


if __name__ == "__main__":
    main()

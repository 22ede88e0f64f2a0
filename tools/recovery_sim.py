"""Straggler recovery of the resized TP layer, simulated on one GPU
(BASELINE.json north_star target: one rank slowed 2x, the balanced step
recovers >= 85% of the straggler-free step time; SURVEY §8(d) timing protocol
steps 1-4).

The e TP ranks of a config are simulated with one context each on a single
B200; rank `strag` is slowed by chi with the library's delay kernel (A-32,
P:333).  Each rank's step (graph replay) is timed alone; a synchronous TP step
cannot finish before its slowest rank, so the compute part of a step is
max_r T_r.  The four all-reduces per layer step are not run (one
GPU); they are the same for every phase, and are added as a model: ring bus
bytes 2(e-1)/e x 2 N h B each at the measured 770 GB/s NVLink peer bandwidth,
un-overlapped.  Both recoveries (compute only, and with the modeled
collectives) are printed.

Phases (each rank timed alone, same seeded inputs):
  free    chi = 1 everywhere, dense
  unbal   chi on the straggler, dense; the statistics window gives T_i, M_i
          (A-5, A-6)
  bal     ztp_plan (ZERO with the T_min criterion, A-7; or SEMI) ->
          layer_prune_counts -> ztp_select; chi kept.  Then up to REFRESH
          statistics refreshes (P:178's 10% trigger, A-8): a new window with
          the plan in effect, ztp_plan on it, ztp_plan_refine (A-39).
Usage: CASES=c2:2:2,c2:4:2,c3:4:2,c4:8:2,c4:8:3s python tools/recovery_sim.py
(cfg:e:chi, suffix s = SEMI plan with migration)."""
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
from paper_2401_11469_b200.pretest import pretest  # noqa: E402

STEPS = int(os.environ.get("STEPS", "50"))
REFRESH = int(os.environ.get("REFRESH", "3"))
NVLINK_GBS = bench.NVLINK_GBS


def time_rank(L, ctx, chi_r, steps=STEPS):
    stream = torch.cuda.Stream()
    Z.ztp_set_slowdown(ctx, chi_r)
    for _ in range(2):
        L.step(stream)
    torch.cuda.synchronize()
    g = L.capture(stream)
    with torch.cuda.stream(stream):      # replay() issues on the current stream
        for _ in range(5):
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


def time_all(layers, ctxs, chis):
    """Per-rank step times, each the mean of a forward and a reverse sweep
    over the ranks (cancels the power/clock drift along one sweep)."""
    e = len(layers)
    fwd = [time_rank(L, ctxs[r], chis[r]) for r, L in enumerate(layers)]
    rev = [0.0] * e
    for r in reversed(range(e)):
        rev[r] = time_rank(layers[r], ctxs[r], chis[r])
    return [(a + b) / 2 for a, b in zip(fwd, rev)]


def gemm_ms(L, ctx):
    """M_i: GEMM time per step incl. the emulated slowdown (A-6)."""
    Z.ztp_set_stats(ctx, True)
    Z.ztp_read_gemm_ns(ctx)
    for _ in range(5):
        L.step()
    m = Z.ztp_read_gemm_ns(ctx) / 5 / 1e6
    Z.ztp_set_stats(ctx, False)
    return m


def run_case(cfg_name, e, chi, semi):
    cfg = CONFIGS[cfg_name]
    h, f, N = cfg.h, cfg.f, cfg.N
    a, u = h // e, f // e
    strag = e - 1
    chis = [chi if r == strag else 1.0 for r in range(e)]
    ctxs = [Z.ztp_ctx_create(0, 1, None, 0) for _ in range(e)]
    lens = {"qkv": h, "o": a, "fc1": h, "fc2": u}
    cap = u if semi else 0
    layers, scores = [], []
    for r in range(e):
        sh = bench.rank_shards(cfg, e, r)
        dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
        L = ZtpLayer(ctxs[r], h, f, N, r, e, dev, mig_cap=cap)
        # one GPU: the per-replan weight / dW peer copies of SEMI (NVLink on a
        # real box) are done once below as local copies
        L.migrate_weights = lambda stream=None: None
        L.return_grads = lambda stream=None: None
        L.X.normal_()
        L.G.normal_()
        layers.append(L)
        scores.append({s: torch.from_numpy(v).cuda() for s, v in bench.scores_for(cfg, r, lens).items()})
    for r, L in enumerate(layers):
        L.set_selection({s: 0 for s in SEGS}, scores[r])
    free = time_all(layers, ctxs, [1.0] * e)
    T = time_all(layers, ctxs, chis)
    M = [gemm_ms(L, ctxs[r]) for r, L in enumerate(layers)]
    costs, pre = None, None
    if semi:
        # Alg.2 l.1 pretest on a non-straggling rank (Phi_1 modelled over NVLink)
        costs, pre = pretest(layers[0], ctxs[0], scores[0], steps=10, link_gbs=NVLINK_GBS)
        for r, L in enumerate(layers):
            L.set_selection({s: 0 for s in SEGS}, scores[r])
    plan = Z.ztp_plan(T, M, float(u), costs, Z.plan_opts(enable_migration=1 if semi else 0, zero_crit=Z.CRIT_MIN))
    last_mios = []

    def apply(plan):
        if semi:
            mios = [migration_io(plan, r, e, u, h) for r in range(e)]
            last_mios[:] = mios
            for r, L in enumerate(layers):
                L.set_migration(mios[r])
            for (src, dst, lo, hi, off) in mios[0].all_xfers:      # local stand-in for ztp_migrate
                Ls, Ld = layers[src], layers[dst]
                Ld.w1_t[:, u + off:u + off + hi - lo].copy_(Ls.w1_t[:, lo:hi])
                Ld.w2_t[u + off:u + off + hi - lo].copy_(Ls.w2_t[lo:hi])
        cnt = [layer_prune_counts(plan, r, h, a, u) for r in range(e)]
        for r, L in enumerate(layers):
            L.set_selection(cnt[r], scores[r])
        return cnt
    counts = apply(plan)
    bal = time_all(layers, ctxs, chis)
    # statistics refresh (A-8): a rank whose runtime moved > 10% since
    # the window its plan came from triggers a new window; ZERO plans compose
    # with the fresh Eq.1 ratio (ztp_plan_refine, A-39)
    first = {"T_bal_ms": max(bal), "gamma": [round(g, 4) for g in list(plan.gamma)[:e]]}
    refresh = []
    T_last = T
    for _ in range(REFRESH):
        if max(abs(bal[r] - T_last[r]) / T_last[r] for r in range(e)) <= 0.10:
            break
        M_cur = [gemm_ms(L, ctxs[r]) for r, L in enumerate(layers)]
        fresh = Z.ztp_plan(bal, M_cur, float(u), None, Z.plan_opts(enable_migration=0, zero_crit=Z.CRIT_MIN))
        if fresh.z == 0:
            break
        T_last = bal
        plan = Z.ztp_plan_refine(plan, fresh)          # A-39 / A-42 (SEMI: shed fraction composes)
        counts = apply(plan)
        bal = time_all(layers, ctxs, chis)
        refresh.append({"gamma": [round(g, 4) for g in list(plan.gamma)[:e]], "T_bal_ms": max(bal),
                        "per_rank_ms": [round(x, 4) for x in bal]})
    t_comm = 4 * 2 * N * h * 2 * (e - 1) / e / (NVLINK_GBS * 1e9) * 1e3
    # per-step migration copies of a SEMI plan (weights out + dW back) from
    # the busiest sender's egress, modelled at NVLINK_GBS like the all-reduces
    t_mig = max([4 * m.n_mig * h * 2 / (NVLINK_GBS * 1e9) * 1e3 for m in last_mios] + [0.0])
    t_free, t_unbal, t_bal = max(free), max(T), max(bal) + t_mig
    roles = "".join("NRMS"[int(x)] for x in list(plan.role)[:e])
    out = {"config": cfg_name, "tp": e, "chi": chi, "straggler": strag, "plan": "SEMI" if semi else "ZERO (T_min)",
           "roles": roles, "gamma": [round(g, 4) for g in list(plan.gamma)[:e]],
           "beta": [round(b, 4) for b in list(plan.beta)[:e]],
           "n_prune_straggler": counts[strag],
           "T_free_ms": t_free, "T_unbal_ms": t_unbal, "T_bal_ms": t_bal,
           "recovery_compute": t_free / t_bal, "speedup_compute": t_unbal / t_bal,
           "t_allreduce_model_ms": t_comm, "t_migration_model_ms": t_mig,
           "recovery_with_comm": (t_free + t_comm) / (t_bal + t_comm),
           "speedup_with_comm": (t_unbal + t_comm) / (t_bal + t_comm),
           "per_rank_free_ms": [round(x, 4) for x in free], "per_rank_unbal_ms": [round(x, 4) for x in T],
           "per_rank_bal_ms": [round(x, 4) for x in bal], "M_ms": [round(x, 4) for x in M],
           "first_plan": first, "refresh": refresh, "pretest_costs": pre["costs"] if pre else None}
    for c in ctxs:
        Z.ztp_ctx_destroy(c)
    del layers
    torch.cuda.empty_cache()
    return out


def main():
    cases = os.environ.get("CASES", "c2:2:2,c2:4:2,c3:4:2,c4:8:2,c4:8:3s")
    rows = []
    for c in cases.split(","):
        name, e, chi = c.split(":")
        semi = chi.endswith("s")
        rows.append(run_case(name, int(e), float(chi.rstrip("s")), semi))
        print(json.dumps(rows[-1]), flush=True)
    json.dump({"note": "one-GPU simulation: each TP rank timed alone (graph replay, its own slowdown); "
                       "step = max over ranks; 4 all-reduces per layer step modeled at 770 GB/s ring bus bytes",
               "steps": STEPS, "cases": rows},
              open(os.environ.get("OUT", "gpurun_out/recovery_sim.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

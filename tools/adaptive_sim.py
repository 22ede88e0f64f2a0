"""c5 adaptive plan under time-varying slowdowns, simulated on one GPU
(BASELINE.json configs[4]: GPT-13B-shaped 4-layer stack, h=5120, ffn=20480,
seq 2048, TP=8, "time-varying per-rank slowdowns, adaptive resize/migrate
plan"; 40 steps, epoch = 10 steps).

Slowdown schedule (P:333 emulation, A-32), one phase per 10 steps:
  0-9    rank 0 x2                              (single light straggler)
  10-19  rank 3 x3                              (single heavy straggler: SEMI z=1)
  20-29  ranks 1,3,5,7 x 8,6,4,2                (the paper's multi-straggler setting; Eq.3)
  30-39  homogeneous                            (the plan must return to gamma = 0)

The 8 TP ranks are 8 library contexts on one B200, each with its own 4-layer
stack (fwd layers 0..3, bwd 3..0, one CUDA graph per rank and plan); each
rank's step is timed alone with its own slowdown and a synchronous TP step
lasts as long as its slowest rank: step = max_r T_r + the modelled
collectives (4 all-reduces per layer, ring bus bytes at the measured 770 GB/s
NVLink peer bandwidth, un-overlapped) + the modelled per-step migration
copies (weight slices out and dW slices back, bytes / 770 GB/s, from the
straggler's egress).

Controller (host, per step; Alg.2):
  * the first step, and the step after any trigger, is a STATISTICS WINDOW:
    the plan is lifted (dense, no migration) and every rank's T_i and M_i
    (A-5, A-6) are measured -- Eq.1 and Alg.2 are defined on un-resized
    runtimes;
  * plan = ztp_plan(T, M, u, costs, SEMI, T_min criterion) with the costs of
    the Alg.2 l.1 pretest (paper_2401_11469_b200/pretest.py, measured here at
    start-up, Phi_1 modelled over NVLink);
  * the first step under a new plan is the monitoring reference T_ref; a
    plan whose straggler is still detectably slower is refined once per
    window (ztp_plan_refine: A-39 for resizing ranks, A-42 for migrating
    ones -- their shed fraction composes, beta kept);
  * trigger: any rank's runtime moving > 10% from T_ref (A-8), or,
    on the first step under a plan, a rank running > 10% below the T_min the
    plan aimed at (its slowdown changed while the plan was being applied).
Output: per-step JSON (phase, mode, roles, gamma/beta, per-rank ms, step ms)
and per-phase means vs T_free.  Env: STEPS_PER_PHASE (10), REPLAYS (5), WARM (5), EPS (0.05),
OUT (gpurun_out/adaptive_sim.json), CFG (c5), TP (8)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer, migration_io, layer_prune_counts, MigrationIO, SEGS  # noqa: E402
from paper_2401_11469_b200.pretest import pretest  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth import inputs as I  # noqa: E402

NVLINK_GBS = 770.0
PER = int(os.environ.get("STEPS_PER_PHASE", "10"))
REPLAYS = int(os.environ.get("REPLAYS", "5"))
WARM = int(os.environ.get("WARM", "5"))       # replays after a (re)capture before timing
EPS = float(os.environ.get("EPS", "0.05"))    # A-17 straggler tolerance, above the one-GPU timing noise
TRIGGER = 0.10


def schedule(step, e):
    ph = step // PER
    chi = [1.0] * e
    if ph == 0:
        chi[0] = 2.0
    elif ph == 1:
        chi[3 % e] = 3.0
    elif ph == 2:
        for r, c in zip((1, 3, 5, 7), (8.0, 6.0, 4.0, 2.0)):
            if r < e:
                chi[r] = c
    return ph, chi


class Rank:
    def __init__(self, cfg, e, r, n_layers):
        self.ctx = Z.ztp_ctx_create(0, 1, None, 0)
        h, f, N = cfg.h, cfg.f, cfg.N
        a, u = h // e, f // e
        self.layers = []
        self.scores = []
        lens = {"qkv": h, "o": a, "fc1": h, "fc2": u}
        for li in range(n_layers):
            # timing only: device-random weights of the right scale (values do
            # not change the work; parity is covered by tests/test_gpu_layer.py)
            sh = {"qkv": torch.empty(h, 3 * a, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                  "o": torch.empty(a, h, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                  "w1": torch.empty(h, u, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                  "w2": torch.empty(u, h, device="cuda").uniform_(-f ** -0.5, f ** -0.5)}
            L = ZtpLayer(self.ctx, h, f, N, r, e, {k: v.to(torch.bfloat16) for k, v in sh.items()},
                         mig_cap=u, layer_id=li)
            L.migrate_weights = lambda stream=None: None     # modelled per step (NVLink), see module doc
            L.return_grads = lambda stream=None: None
            L.X.normal_()
            L.G.normal_()
            self.layers.append(L)
            self.scores.append({s: torch.from_numpy(I.lognormal_scores(cfg.seed, f"score.{s}.{li}", n, rank=r)).cuda()
                                for s, n in lens.items()})
        self.graph = None
        self.key = None

    def run(self, stream=None):
        for L in self.layers:
            L.run_select(stream)
        for L in self.layers:
            L.forward(stream)
        for L in reversed(self.layers):
            L.backward(stream)

    def time(self, chi, version):
        key = (chi, version)
        stream = getattr(self, "stream", None) or torch.cuda.Stream()
        self.stream = stream
        if self.key != key:
            self.graph = None
            Z.ztp_set_slowdown(self.ctx, chi)
            self.run(stream)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                self.run(stream)
            self.graph, self.key = g, key
            with torch.cuda.stream(stream):      # replay() issues on the current stream
                for _ in range(WARM):
                    self.graph.replay()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(REPLAYS):
                self.graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / REPLAYS

    def gemm_ms(self, chi):
        Z.ztp_set_slowdown(self.ctx, chi)
        Z.ztp_set_stats(self.ctx, True)
        Z.ztp_read_gemm_ns(self.ctx)
        self.run()
        m = Z.ztp_read_gemm_ns(self.ctx) / 1e6
        Z.ztp_set_stats(self.ctx, False)
        return m


def measure(ranks, chis, version):
    """Per-rank step times, each the mean of a forward (0..e-1) and a
    reverse pass: a rank's place in the sweep otherwise biases it by the
    board's power/clock drift (~10% over one sweep measured)."""
    e = len(ranks)
    fwd = [R.time(chis[r], version) for r, R in enumerate(ranks)]
    rev = [0.0] * e
    for r in reversed(range(e)):
        rev[r] = ranks[r].time(chis[r], version)
    return [(a + b) / 2 for a, b in zip(fwd, rev)]


def apply_plan(ranks, plan, e, h, a, u):
    """plan -> every rank's migration ranges and prune counts on all layers;
    the weight slices are copied locally (one GPU) once per plan."""
    mios = [migration_io(plan, r, e, u, h) if plan is not None else MigrationIO() for r in range(e)]
    for r, R in enumerate(ranks):
        counts = layer_prune_counts(plan, r, h, a, u) if plan is not None else {s: 0 for s in SEGS}
        for L in R.layers:
            L.set_migration(mios[r])
        for li, L in enumerate(R.layers):
            L.set_selection(counts, R.scores[li])
    for (src, dst, lo, hi, off) in mios[0].all_xfers:
        for li in range(len(ranks[0].layers)):
            Ls, Ld = ranks[src].layers[li], ranks[dst].layers[li]
            Ld.w1_t[:, u + off:u + off + hi - lo].copy_(Ls.w1_t[:, lo:hi])
            Ld.w2_t[u + off:u + off + hi - lo].copy_(Ls.w2_t[lo:hi])
    return mios


def mig_model_ms(mios, h, n_layers, elt=2):
    """Per-step migration copies (weights out + dW back) from each shedding
    rank's egress at NVLINK_GBS; the slowest shedder bounds the step."""
    worst = 0.0
    for m in mios:
        if m.n_mig:
            worst = max(worst, 4 * m.n_mig * h * elt * n_layers / (NVLINK_GBS * 1e9) * 1e3)
    return worst


def plan_summary(plan, e):
    if plan is None:
        return {"roles": "N" * e, "gamma": [0.0] * e, "beta": [0.0] * e, "z": 0, "x": 0}
    return {"roles": "".join("NRMS"[int(x)] for x in list(plan.role)[:e]),
            "gamma": [round(g, 4) for g in list(plan.gamma)[:e]],
            "gamma_r": [round(g, 4) for g in list(plan.gamma_r)[:e]],
            "beta": [round(b, 4) for b in list(plan.beta)[:e]], "z": int(plan.z), "x": int(plan.x)}


def main():
    cfg = CONFIGS[os.environ.get("CFG", "c5")]
    e = int(os.environ.get("TP", "8"))
    n_layers = cfg.layers
    h, f, N = cfg.h, cfg.f, cfg.N
    a, u = h // e, f // e
    t_start = time.time()
    ranks = [Rank(cfg, e, r, n_layers) for r in range(e)]
    # ---- Alg.2 l.1 pretest on rank 0's first layer, scaled to the stack
    L0 = ranks[0].layers[0]
    _, rep = pretest(L0, ranks[0].ctx, ranks[0].scores[0], steps=10, link_gbs=NVLINK_GBS)
    c = rep["costs"]
    sc = lambda p: (p[0], tuple(y * n_layers for y in p[1]))  # noqa: E731
    costs = Z.make_costs(c["omega1"] * n_layers, sc(c["omega2"]), sc(c["phi1"]), sc(c["phi2"]))
    opts = Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN, eps=EPS)
    zopts = Z.plan_opts(enable_migration=0, zero_crit=Z.CRIT_MIN, eps=EPS)
    t_comm = n_layers * 4 * 2 * N * h * 2 * (e - 1) / e / (NVLINK_GBS * 1e9) * 1e3
    # ---- T_free: everyone dense at chi = 1
    apply_plan(ranks, None, e, h, a, u)
    version = 0
    t_free = max(measure(ranks, [1.0] * e, version)) + t_comm

    plan, mios = None, [MigrationIO() for _ in range(e)]
    window, T_ref, refined = True, None, False
    T_target = T_window_max = 0.0
    series = []
    for step in range(4 * PER):
        ph, chis = schedule(step, e)
        rec = {"step": step, "phase": ph, "chi": chis}
        if window:
            if plan is not None:
                apply_plan(ranks, None, e, h, a, u)
                version += 1
                plan, mios = None, [MigrationIO() for _ in range(e)]
            T = measure(ranks, chis, version)
            M = [R.gemm_ms(chis[r]) for r, R in enumerate(ranks)]
            rec.update(mode="window", per_rank_ms=[round(x, 4) for x in T], M_ms=[round(x, 4) for x in M])
            rec["step_ms"] = max(T) + t_comm
            new = Z.ztp_plan(T, M, float(u), costs, opts)
            if int(new.z) > 0:
                plan = new
                mios = apply_plan(ranks, plan, e, h, a, u)
                version += 1
            window, T_ref, refined = False, None, False
            T_target = min(T)                       # the plan aims every rank at T_min
            T_window_max = max(T)
            rec["plan_after"] = plan_summary(plan, e)
        else:
            T = measure(ranks, chis, version)
            rec.update(mode="plan", per_rank_ms=[round(x, 4) for x in T])
            rec["step_ms"] = max(T) + t_comm + mig_model_ms(mios, h, n_layers)
            if T_ref is None and plan is not None and (min(T) < (1.0 - TRIGGER) * T_target or
                                                       max(T) > (1.0 + TRIGGER) * T_window_max):
                # on the first step under a plan, a rank runs > 10% below the
                # T_min the plan aimed at, or > 10% above the unbalanced window's
                # slowest rank: the slowdowns changed while the plan was being
                # applied -- a new window, not a refine
                window = True
                rec["trigger"] = "off target"
            elif T_ref is None:
                T_ref = T
                if plan is not None and not refined:
                    M = [R.gemm_ms(chis[r]) for r, R in enumerate(ranks)]
                    fresh = Z.ztp_plan(T, M, float(u), None, zopts)
                    # refine the plan's stragglers only: a normal task that is
                    # now slower carries received units (Alg.2 keeps normal
                    # tasks unpruned)
                    for r in range(e):
                        if int(plan.role[r]) == Z.NORMAL:
                            fresh.gamma[r] = fresh.gamma_r[r] = 0.0
                            fresh.role[r] = Z.NORMAL
                    if any(fresh.gamma_r[r] > 0.0 for r in range(e)):
                        plan = Z.ztp_plan_refine(plan, fresh)
                        mios = apply_plan(ranks, plan, e, h, a, u)
                        version += 1
                        T_ref, refined = None, True
                        rec["refined_to"] = plan_summary(plan, e)
            elif max(abs(T[r] - T_ref[r]) / T_ref[r] for r in range(e)) > TRIGGER:
                window = True
                rec["trigger"] = True
        rec["step_ms"] = round(rec["step_ms"], 4)
        series.append(rec)
        print(json.dumps({k: rec[k] for k in rec if k not in ("per_rank_ms", "M_ms")}), flush=True)
    phases = []
    for ph in range(4):
        rows = [s for s in series if s["phase"] == ph]
        steady = [s["step_ms"] for s in rows if s["mode"] == "plan"]
        allm = sum(s["step_ms"] for s in rows) / len(rows)
        phases.append({"phase": ph, "chi": rows[0]["chi"], "mean_step_ms": round(allm, 4),
                       "mean_planned_step_ms": round(sum(steady) / len(steady), 4) if steady else None,
                       "windows": sum(1 for s in rows if s["mode"] == "window"),
                       "recovery_all_steps": round(t_free / allm, 4),
                       "recovery_planned_steps": round(t_free * len(steady) / sum(steady), 4) if steady else None,
                       "last_plan": next((s.get("refined_to") or s.get("plan_after") for s in reversed(rows)
                                          if s.get("refined_to") or s.get("plan_after")), None)})
    unbal = {}
    # unbalanced reference per phase (dense, chi applied)
    apply_plan(ranks, None, e, h, a, u)
    version += 1
    for ph in range(4):
        _, chis = schedule(ph * PER, e)
        unbal[ph] = max(measure(ranks, chis, version)) + t_comm
        phases[ph]["unbal_step_ms"] = round(unbal[ph], 4)
        phases[ph]["speedup_planned_vs_unbal"] = (round(unbal[ph] / phases[ph]["mean_planned_step_ms"], 4)
                                                  if phases[ph]["mean_planned_step_ms"] else None)
    out = {"config": cfg.name, "tp": e, "layers": n_layers, "T_free_ms": round(t_free, 4), "eps": EPS,
           "replays": REPLAYS, "warm": WARM,
           "t_allreduce_model_ms": round(t_comm, 4), "pretest": rep, "phases": phases, "series": series,
           "wall_s": round(time.time() - t_start, 1),
           "note": "one-GPU simulation: each TP rank timed alone (graph replay of its 4-layer stack with its own "
                   "slowdown); step = max over ranks + modelled all-reduces and migration copies at 770 GB/s"}
    for p in phases:
        print(json.dumps(p), flush=True)
    json.dump(out, open(os.environ.get("OUT", "gpurun_out/adaptive_sim.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

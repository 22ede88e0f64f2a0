"""c5 adaptive plan under time-varying slowdowns, simulated on one GPU with
the library's controller (BASELINE.json configs[4]: GPT-13B-shaped 4-layer
stack, h=5120, ffn=20480, seq 2048, TP=8, "time-varying per-rank slowdowns,
adaptive resize/migrate plan"; 40 steps, 10 per phase).

Slowdown schedule (P:333 emulation, A-32), one phase per 10 steps:
  0-9    rank 0 x2                              (single light straggler)
  10-19  rank 3 x3                              (single heavy straggler: SEMI z=1)
  20-29  ranks 1,3,5,7 x 8,6,4,2                (the paper's multi-straggler setting; Eq.3)
  30-39  homogeneous                            (the plan must return to gamma = 0)

Harness tools/tp_sim.py (8 contexts on one B200, each rank's 4-layer stack
timed alone, step = max over ranks + modelled all-reduces and per-step
migration copies at 770 GB/s).  Every step's T_i, M_i go to ztp_ctl_step
(SEMI plans, T_min criterion, the Alg.2 l.1 pretest costs measured at
start-up); the plan it returns is applied before the next step.
Env: STEPS_PER_PHASE (10), REPLAYS (10), EPS (0.05), OUT, CFG (c5), TP (8),
SCHED=roundrobin (c0's schedule: rank 1 x2, rank 3 x4, rank 5 x8, homogeneous)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.pretest import pretest  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from tp_sim import SimTP, NVLINK_GBS  # noqa: E402

PER = int(os.environ.get("STEPS_PER_PHASE", "10"))
EPS = float(os.environ.get("EPS", "0.05"))


def schedule(step, e):
    ph = step // PER
    chi = [1.0] * e
    if os.environ.get("SCHED") == "roundrobin":
        # c0: the straggler rotates over the ranks with chi 2, 4, 8, then homogeneous
        if ph < 3:
            chi[(2 * ph + 1) % e] = (2.0, 4.0, 8.0)[ph]
        return chi
    if ph == 0:
        chi[0] = 2.0
    elif ph == 1:
        chi[3 % e] = 3.0
    elif ph == 2:
        for r, c in zip((1, 3, 5, 7), (8.0, 6.0, 4.0, 2.0)):
            if r < e:
                chi[r] = c
    return chi


def main():
    cfg = CONFIGS[os.environ.get("CFG", "c5")]
    e = int(os.environ.get("TP", "8"))
    t0 = time.time()
    sim = SimTP(cfg, e, n_layers=cfg.layers, semi=True, replays=int(os.environ.get("REPLAYS", "10")))
    nl = cfg.layers
    R0 = sim.ranks[0]
    _, rep = pretest(R0.layers[0], R0.ctx, R0.scores[0], steps=10, link_gbs=NVLINK_GBS)
    sim.apply(None)
    c = rep["costs"]
    scale = lambda p: (p[0], tuple(y * nl for y in p[1]))  # noqa: E731  (per layer -> the stack)
    costs = Z.make_costs(c["omega1"] * nl, scale(c["omega2"]), scale(c["phi1"]), scale(c["phi2"]))
    opts = Z.ctl_opts(L_ref=float(sim.u), trigger=0.10, max_refines=2, enable_migration=1, zero_crit=Z.CRIT_MIN,
                      eps=EPS)
    T_free, _ = sim.measure([1.0] * e, with_m=False)
    t_free = max(T_free) + sim.t_comm
    series, ctl = sim.run_controller(lambda k: schedule(k, e), 4 * PER, opts, costs,
                                     log=lambda r: print(json.dumps(r), flush=True))
    sim.apply(None)
    phases = []
    for ph in range(4):
        rows = [s for s in series if s["step"] // PER == ph]
        planned = [s["step_ms"] for s in rows if s["state"] != "window"]
        allm = sum(s["step_ms"] for s in rows) / len(rows)
        T_unbal, _ = sim.measure(schedule(ph * PER, e), with_m=False)
        unbal = max(T_unbal) + sim.t_comm
        mp = sum(planned) / len(planned) if planned else None
        phases.append({"phase": ph, "chi": rows[0]["chi"], "unbal_step_ms": round(unbal, 4),
                       "mean_step_ms": round(allm, 4), "mean_planned_step_ms": round(mp, 4) if mp else None,
                       "windows": sum(1 for s in rows if s["state"] == "window"),
                       "recovery_all_steps": round(t_free / allm, 4),
                       "recovery_planned_steps": round(t_free / mp, 4) if mp else None,
                       "speedup_planned_vs_unbal": round(unbal / mp, 4) if mp else None,
                       "last_plan": rows[-1]["plan"]})
    out = {"config": cfg.name, "tp": e, "layers": nl, "T_free_ms": round(t_free, 4), "eps": EPS,
           "t_allreduce_model_ms": round(sim.t_comm, 4), "pretest": rep, "phases": phases, "series": series,
           "controller": {"windows": ctl.windows, "replans": ctl.replans, "refines": ctl.refine_count,
                          "triggers": ctl.triggers},
           "wall_s": round(time.time() - t0, 1),
           "note": "one-GPU simulation driven by ztp_ctl_step: each TP rank timed alone (graph replay of its "
                   "4-layer stack with its own slowdown); step = max over ranks + modelled all-reduces and "
                   "migration copies at 770 GB/s"}
    for p in phases:
        print(json.dumps(p), flush=True)
    json.dump(out, open(os.environ.get("OUT", "gpurun_out/adaptive_sim.json"), "w"), indent=1)
    sim.destroy()


if __name__ == "__main__":
    main()

"""Straggler recovery of the resized TP layer, simulated on one GPU with the
library's controller (BASELINE.json north_star: one rank slowed 2x, the
balanced step recovers >= 85% of the straggler-free step time; SURVEY §8(d)
timing protocol steps 1-4).  Harness: tools/tp_sim.py (e contexts on one
B200, each rank timed alone, step = max over ranks + modelled all-reduces and
migration copies).

Per case: T_free (chi = 1, dense), T_unbal (chi on the straggler, dense),
then STEPS steps under ztp_ctl_step (window -> plan -> refresh -> monitor,
A-41/A-43) with the slowdown held; T_bal = mean of the monitored steps.
Usage: CASES=c2:2:2,c2:4:2,c3:4:2,c4:8:2,c4:8:3s python tools/recovery_sim.py
(cfg:e:chi, suffix s = SEMI plans with the pretest costs).  The E4 analog
(a chi sweep of one straggler on the paper's ViT-1B shape):
CASES=c0:8:1,c0:8:2,c0:8:3,c0:8:4,c0:8:6,c0:8:8,c0:8:4s,c0:8:8s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.pretest import pretest  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from tp_sim import SimTP, NVLINK_GBS, plan_summary  # noqa: E402

STEPS = int(os.environ.get("STEPS", "8"))
EPS = float(os.environ.get("EPS", "0.05"))     # A-17 tolerance above the one-GPU timing noise (~3%)
# Eq.1's criterion: T_min (A-7, the build's headline) or the paper-literal T_avg (CRIT=avg)
CRIT = {"min": Z.CRIT_MIN, "avg": Z.CRIT_AVG}[os.environ.get("CRIT", "min")]


def run_case(name, e, chi, semi):
    cfg = CONFIGS[name]
    sim = SimTP(cfg, e, semi=semi, replays=int(os.environ.get("REPLAYS", "30")))
    strag = e - 1
    chis = [chi if r == strag else 1.0 for r in range(e)]
    T_free, _ = sim.measure([1.0] * e, with_m=False)
    T_unbal, _ = sim.measure(chis, with_m=False)
    costs, pre = None, None
    if semi:
        R0 = sim.ranks[0]
        costs, pre = pretest(R0.layers[0], R0.ctx, R0.scores[0], steps=10, link_gbs=NVLINK_GBS)
        sim.apply(None)
    opts = Z.ctl_opts(L_ref=float(sim.u), trigger=0.10, max_refines=2, enable_migration=int(semi),
                      zero_crit=CRIT, eps=EPS)
    series, ctl = sim.run_controller(lambda k: chis, STEPS, opts, costs,
                                     log=lambda r: print(json.dumps(r), flush=True))
    mon = [s for s in series if s["state"] == "monitor"] or series[-1:]
    t_free = max(T_free) + sim.t_comm
    t_unbal = max(T_unbal) + sim.t_comm
    t_bal = sum(s["step_ms"] for s in mon) / len(mon)
    out = {"config": name, "tp": e, "chi": chi, "straggler": strag, "mode": ("SEMI" if semi else "ZERO") + (" (T_avg)" if CRIT == Z.CRIT_AVG else " (T_min)"),
           "eps": EPS, "T_free_ms": t_free, "T_unbal_ms": t_unbal, "T_bal_ms": t_bal,
           "recovery": t_free / t_bal, "speedup": t_unbal / t_bal,
           "recovery_compute_only": max(T_free) / (t_bal - sim.t_comm),
           "t_allreduce_model_ms": sim.t_comm, "final_plan": plan_summary(ctl.plan, e),
           "windows": ctl.windows, "refines": ctl.refine_count, "triggers": ctl.triggers,
           "per_rank_free_ms": [round(x, 4) for x in T_free], "per_rank_unbal_ms": [round(x, 4) for x in T_unbal],
           "series": series, "pretest_costs": pre["costs"] if pre else None}
    sim.destroy()
    return out


def main():
    cases = os.environ.get("CASES", "c2:2:2,c2:4:2,c3:4:2,c4:8:2,c4:8:3s")
    rows = []
    for c in cases.split(","):
        name, e, chi = c.split(":")
        semi = chi.endswith("s")
        rows.append(run_case(name, int(e), float(chi.rstrip("s")), semi))
        r = rows[-1]
        print(json.dumps({k: r[k] for k in r if k not in ("series", "pretest_costs")}), flush=True)
    json.dump({"note": "one-GPU simulation driven by ztp_ctl_step: each TP rank timed alone (graph replay, its own "
                       "slowdown); step = max over ranks + 4 all-reduces per layer (ring bytes at 770 GB/s) + "
                       "per-step migration copies (SEMI)", "steps": STEPS, "cases": rows},
              open(os.environ.get("OUT", "gpurun_out/recovery_sim.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

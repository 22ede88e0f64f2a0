"""Table I analog (NEXT-3 in SURVEY §8(f)), simulated on one GPU:
step time of the c4 Llama-2-7B-shaped layer at TP = 8 in a HOMOGENEOUS
environment when nu selected ranks migrate a fraction gamma of their MLP
hidden units to the others (gamma in {0, .25, .5, .75, 1}, nu in {1, 4}).

The paper compares broadcast-reduce and scatter-gather migration on V100s;
this build's policy is a third one for NVSwitch: each helper
pulls a disjoint slice of the shed units once (grouped send/recv), computes it
as extra units of its own FC1 / FC2 (merged accumulation, so the partial sums
ride the existing all-reduces: no reduce step), and returns the dW slices.

Measured: every rank's step (graph replay of the real library step with its
migration ranges: senders run u - n_mig units, receivers append theirs),
each timed alone; step = max over ranks + the layer's 4 all-reduces and the
per-step migration copies, both modelled at 770 GB/s (one GPU cannot time
NVLink): copies = max over ranks of max(egress, ingress) bytes, weights out
(W1^T columns + W2^T rows) and dW slices back, bf16.
Env: CFG (c4), TP (8), OUT (gpurun_out/migration_table.json)."""
import json
import os
import sys


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import migration_io, MigrationIO, SEGS  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from adaptive_sim import Rank, NVLINK_GBS, measure  # noqa: E402


def forced_plan(e, senders, gamma):
    """A SEMI plan with `senders` in role MIGRATE shedding a fraction gamma of
    their units (beta = 1, no resizing), everyone else NORMAL (receivers)."""
    p = Z.PlanT()
    p.world = e
    p.z = len(senders)
    p.x = len(senders)
    for r in range(e):
        p.order[r] = r
        p.role[r] = Z.MIGRATE if (r in senders and gamma > 0) else Z.NORMAL
        g = gamma if r in senders else 0.0
        p.gamma[r] = g
        p.beta[r] = 1.0 if g > 0 else 0.0
        p.phi[r] = g
        p.gamma_r[r] = 0.0
    return p


def main():
    cfg = CONFIGS[os.environ.get("CFG", "c4")]
    e = int(os.environ.get("TP", "8"))
    h, N = cfg.h, cfg.N
    u = cfg.f // e
    ranks = [Rank(cfg, e, r, 1) for r in range(e)]
    t_ar = 4 * 2 * N * h * 2 * (e - 1) / e / (NVLINK_GBS * 1e9) * 1e3
    rows = []
    version = 0
    for nu in (1, 4):
        senders = list(range(e - nu, e))
        for gamma in (0.0, 0.25, 0.5, 0.75, 1.0):
            plan = forced_plan(e, senders, gamma)
            mios = [migration_io(plan, r, e, u, h) if gamma > 0 else MigrationIO() for r in range(e)]
            for r, R in enumerate(ranks):
                L = R.layers[0]
                L.set_migration(mios[r])
                L.set_selection({s: 0 for s in SEGS}, R.scores[0])
            for (src, dst, lo, hi, off) in mios[0].all_xfers:
                Ls, Ld = ranks[src].layers[0], ranks[dst].layers[0]
                Ld.w1_t[:, u + off:u + off + hi - lo].copy_(Ls.w1_t[:, lo:hi])
                Ld.w2_t[u + off:u + off + hi - lo].copy_(Ls.w2_t[lo:hi])
            version += 1
            T = measure(ranks, [1.0] * e, version)
            egress = [0] * e
            ingress = [0] * e
            for (src, dst, lo, hi, off) in mios[0].all_xfers:
                b = 2 * (hi - lo) * h * 2          # W1^T columns + W2^T rows, bf16
                egress[src] += b
                ingress[dst] += b
                egress[dst] += b                   # dW slices back
                ingress[src] += b
            t_mig = max(max(a, b) for a, b in zip(egress, ingress)) / (NVLINK_GBS * 1e9) * 1e3
            row = {"nu": nu, "gamma": gamma, "units_moved_per_sender": mios[senders[0]].n_mig if gamma else 0,
                   "compute_ms": round(max(T), 4), "t_allreduce_model_ms": round(t_ar, 4),
                   "t_migration_model_ms": round(t_mig, 4), "step_ms": round(max(T) + t_ar + t_mig, 4),
                   "per_rank_ms": [round(x, 4) for x in T]}
            rows.append(row)
            print(json.dumps(row), flush=True)
    base = rows[0]["step_ms"]
    for r in rows:
        r["rel_to_gamma0"] = round(r["step_ms"] / base, 4)
    json.dump({"config": cfg.name, "tp": e, "note": __doc__.split("\n\n")[0], "rows": rows},
              open(os.environ.get("OUT", "gpurun_out/migration_table.json"), "w"), indent=1)
    print("nu gamma step_ms rel")
    for r in rows:
        print(r["nu"], r["gamma"], r["step_ms"], r["rel_to_gamma0"])


if __name__ == "__main__":
    main()

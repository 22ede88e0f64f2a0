"""One-GPU simulation of e tensor-parallel ranks driven by the library's
re-planning controller (ztp_ctl_step, include/ztp.h; Alg.2).

The e ranks of a config run as e library contexts on one B200, each with its
own layer stack (seeded synthetic weights).  Each rank's step (a CUDA graph
of its layers' FWD + BWD, the rank's emulated slowdown chi applied by the
delay kernel, A-32) is timed alone; a synchronous TP step cannot end before
its slowest rank, so the step's compute time is max_r T_r.  What one GPU
cannot run is added as a model, identical for every phase: the four
all-reduces per layer step (ring bus bytes 2 (e-1)/e x 2 N h at the measured
770 GB/s NVLink peer bandwidth, un-overlapped) and, under a SEMI plan, the
per-step migration copies (weights out + dW slices back) from the busiest
sender's egress.  Weight slices are copied locally once per plan (the
stand-in for ztp_migrate's peer pulls).

Per simulated step: measure every rank's T_i (mean of a forward and a reverse
sweep over the ranks, cancelling the board's power/clock drift) and M_i
(GEMM + delay time from the kernels' own stamps, A-6), feed the all-ranks
vectors to ztp_ctl_step, apply the plan it returns.  The selection runs once
per plan (selection is epoch-granular), not inside the timed step.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_11469_b200 as Z  # noqa: E402
from paper_2401_11469_b200.layer import ZtpLayer, migration_io, MigrationIO, SEGS  # noqa: E402
from synth import inputs as I  # noqa: E402

NVLINK_GBS = 770.0


class RankSim:
    def __init__(self, cfg, e, r, n_layers, cap, seeded=True):
        import bench
        self.ctx = Z.ztp_ctx_create(0, 1, None, 0)
        h, f, N = cfg.h, cfg.f, cfg.N
        a, u = h // e, f // e
        self.layers, self.scores = [], []
        lens = {"qkv": h, "o": a, "fc1": h, "fc2": u}
        for li in range(n_layers):
            if seeded and li == 0:
                sh = bench.rank_shards(cfg, e, r)
                dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
            else:   # timing only: device-random weights of the right scale
                dev = {"qkv": torch.empty(h, 3 * a, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                       "o": torch.empty(a, h, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                       "w1": torch.empty(h, u, device="cuda").uniform_(-h ** -0.5, h ** -0.5),
                       "w2": torch.empty(u, h, device="cuda").uniform_(-f ** -0.5, f ** -0.5)}
                dev = {k: v.to(torch.bfloat16) for k, v in dev.items()}
            L = ZtpLayer(self.ctx, h, f, N, r, e, dev, mig_cap=cap, layer_id=li)
            L.migrate_weights = lambda stream=None: None     # modelled per step (NVLink), see module doc
            L.return_grads = lambda stream=None: None
            L.X.normal_()
            L.G.normal_()
            self.layers.append(L)
            self.scores.append({s: torch.from_numpy(I.lognormal_scores(cfg.seed, f"score.{s}.{li}", n, rank=r)).cuda()
                                for s, n in lens.items()})
        self.stream = torch.cuda.Stream()
        self.graph, self.key = None, None

    def run(self, stream=None):
        for L in self.layers:
            L.forward(stream)
        for L in reversed(self.layers):
            L.backward(stream)

    def time(self, chi, version, replays, warm):
        key = (chi, version)
        st = self.stream
        if self.key != key:
            self.graph = None
            Z.ztp_set_slowdown(self.ctx, chi)
            with torch.cuda.stream(st):
                self.run(st)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                self.run(st)
            self.graph, self.key = g, key
            with torch.cuda.stream(st):
                for _ in range(warm):
                    self.graph.replay()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(replays):
                self.graph.replay()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / replays

    def gemm_ms(self, chi, steps=3):
        """M_i (A-6): GEMM (+ emulated delay) time per step, from the stamps."""
        Z.ztp_set_slowdown(self.ctx, chi)
        Z.ztp_set_stats(self.ctx, True)
        with torch.cuda.stream(self.stream):
            Z.ztp_read_gemm_ns(self.ctx, self.stream)
            for _ in range(steps):
                self.run(self.stream)
            m = Z.ztp_read_gemm_ns(self.ctx, self.stream) / steps / 1e6
        Z.ztp_set_stats(self.ctx, False)
        self.key = None                  # the cached graph was captured without statistics
        return m

    def destroy(self):
        self.graph = None
        Z.ztp_ctx_destroy(self.ctx)


class SimTP:
    def __init__(self, cfg, e, n_layers=1, semi=False, replays=20, warm=5):
        self.cfg, self.e, self.n_layers = cfg, e, n_layers
        self.h, self.a, self.u, self.N = cfg.h, cfg.h // e, cfg.f // e, cfg.N
        self.replays, self.warm = replays, warm
        self.ranks = [RankSim(cfg, e, r, n_layers, self.u if semi else 0) for r in range(e)]
        self.version = 0
        self.mios = [MigrationIO() for _ in range(e)]
        self.t_comm = n_layers * 4 * 2 * self.N * self.h * 2 * (e - 1) / e / (NVLINK_GBS * 1e9) * 1e3
        self.apply(None)

    def apply(self, plan):
        """A plan -> every rank's migration ranges, received weight slices
        (local copies, once per plan) and selection (ztp_select, once per plan)."""
        e, h, a, u = self.e, self.h, self.a, self.u
        self.mios = [migration_io(plan, r, e, u, h) if plan is not None else MigrationIO() for r in range(e)]
        for r, R in enumerate(self.ranks):
            counts = Z.ztp_layer_prune_counts(plan, r, h, a, u) if plan is not None else {s: 0 for s in SEGS}
            for li, L in enumerate(R.layers):
                L.set_migration(self.mios[r])
                L.set_selection(counts, R.scores[li])
        for (src, dst, lo, hi, off) in self.mios[0].all_xfers:
            for li in range(self.n_layers):
                Ls, Ld = self.ranks[src].layers[li], self.ranks[dst].layers[li]
                Ld.w1_t[:, u + off:u + off + hi - lo].copy_(Ls.w1_t[:, lo:hi])
                Ld.w2_t[u + off:u + off + hi - lo].copy_(Ls.w2_t[lo:hi])
        torch.cuda.synchronize()
        self.version += 1

    def mig_ms(self):
        """Per-step migration copies (weights out + dW back, bf16) from the
        busiest sender's egress at NVLINK_GBS."""
        worst = 0.0
        for m in self.mios:
            if m.n_mig:
                worst = max(worst, 4 * m.n_mig * self.h * 2 * self.n_layers / (NVLINK_GBS * 1e9) * 1e3)
        return worst

    def measure(self, chis, with_m=True):
        e = self.e
        fwd = [R.time(chis[r], self.version, self.replays, self.warm) for r, R in enumerate(self.ranks)]
        rev = [0.0] * e
        for r in reversed(range(e)):
            rev[r] = self.ranks[r].time(chis[r], self.version, self.replays, self.warm)
        T = [(x + y) / 2 for x, y in zip(fwd, rev)]
        M = [R.gemm_ms(chis[r]) for r, R in enumerate(self.ranks)] if with_m else None
        return T, M

    def step_ms(self, T):
        return max(T) + self.t_comm + self.mig_ms()

    def run_controller(self, chis_of_step, steps, opts, costs=None, log=None):
        """Drive ztp_ctl_step for `steps` simulated steps; returns the series."""
        ctl = Z.ztp_ctl_init(self.e)
        series = []
        for k in range(steps):
            chis = chis_of_step(k)
            state = ["window", "first", "monitor"][ctl.state]
            T, M = self.measure(chis)
            rec = {"step": k, "chi": chis, "state": state, "plan": plan_summary(ctl.plan, self.e),
                   "per_rank_ms": [round(x, 4) for x in T], "M_ms": [round(x, 4) for x in M],
                   "step_ms": round(self.step_ms(T), 4), "mig_model_ms": round(self.mig_ms(), 4)}
            act = Z.ztp_ctl_step(ctl, opts, T, M, costs)
            rec["action"] = "apply" if act == Z.CTL_APPLY else "keep"
            if act == Z.CTL_APPLY:
                self.apply(ctl.plan)
            series.append(rec)
            if log:
                log({kk: rec[kk] for kk in rec if kk not in ("per_rank_ms", "M_ms")})
        return series, ctl

    def destroy(self):
        for R in self.ranks:
            R.destroy()
        self.ranks = []
        torch.cuda.empty_cache()


def plan_summary(plan, e):
    return {"roles": "".join("NRMS"[int(x)] for x in list(plan.role)[:e]),
            "gamma": [round(g, 4) for g in list(plan.gamma)[:e]],
            "gamma_r": [round(g, 4) for g in list(plan.gamma_r)[:e]],
            "beta": [round(b, 4) for b in list(plan.beta)[:e]], "z": int(plan.z), "x": int(plan.x)}

"""bench.py -- resized-TP layer step on B200 (BASELINE.json metric).

python bench.py --gpus N --steps K --warmup W [--impl ztp|reference]
(N > 1: launched by torchrun, one rank per GPU; NCCL collectives over
NVLink, SEMI migration by one-sided peer pulls from symmetric windows.)

Workload (BASELINE.json configs[1]): one GPT-2-medium layer
(h=1024, 16 heads, ffn=4096, seq 1024 x batch 8 = 8192 tokens): attention-
projection block + MLP block, fwd + bwd, 1D TP over N ranks.
  N = 1: homogeneous ZERO-Pri resizing at gamma = 0.5 on every linear (the
         paper's homogeneous evaluation point) vs the dense step.
  N > 1: rank N-1 emulates a 2x straggler.  T_free (chi = 1, dense)
         -> T_unbal (chi = 2, dense) -> the library's re-planning controller
         (ztp_ctl_step: statistics window, Eq.1 with the T_min criterion,
         refresh of the plan's stragglers, monitoring, A-41, A-43)
         driven by every rank's measured T_i / M_i -> T_bal (timed headline).
         recovery = T_free / T_bal, speedup = T_unbal / T_bal.  `matrix` adds
         the other BASELINE configs that run at this N (N=4: c3; N=8: c4 with
         one 2x straggler, c4 SEMI with a 3x straggler and real migration, c5
         adaptive under time-varying slowdowns), each with its own recovery.
A step = FWD + BWD of the layer through the C ABI, replayed as one CUDA graph
(every kernel is libztp's; collectives NCCL).  The selection (ztp_select)
runs once per plan, as P:187 makes it epoch-granular, not per step.
value = executed GEMM TFLOP/s of the whole job: sum over ranks of the FLOPs
the step's GEMMs execute (A-35/A-36 output pruning included) / step time (max
over ranks).  `method_tflops` counts 6 N n K' per linear instead (SURVEY
§8(d)); the step time is the same.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "resized-TP layer step ms & TFLOP/s at TP=1/2/4/8 w/ 2× straggler; % of roofline"
NVLINK_GBS = 770.0   # measured peer copy per direction (B200_PROFILING.md)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.times = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        cmd = ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)
                self.times.append(time.time())
        p.kill()

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def median_mhz(self, t0: float, t1: float):
        """Median SM clock of the samples taken in [t0, t1] (None if none)."""
        v = [float(s[0]) for s, t in zip(self.samples, self.times) if t0 <= t <= t1 and
             s[0].replace(".", "").isdigit()]
        return float(np.median(v)) if v else None

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        load = [s for s in self.samples if s[6].isdigit() and int(s[6]) > 0] or self.samples
        sm = [float(s[0]) for s in load if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in load if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in load for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(load)}


# ------------------------------------------------------------ inputs (synth)
def rank_shards(cfg, e, r):
    """This rank's shards of the seeded dense layer weights (synth blocks)."""
    from synth import inputs as I
    h, f, seed = cfg.h, cfg.f, cfg.seed
    a, u = h // e, f // e
    F0, F1 = r * a, (r + 1) * a
    U0, U1 = r * u, (r + 1) * u
    bq = 1 / math.sqrt(h)
    qkv = np.concatenate([I.uniform_sym(seed, n, h, h, bq, c0=F0, c1=F1) for n in ("wq", "wk", "wv")], axis=1)
    o = I.uniform_sym(seed, "wo", h, h, bq, r0=F0, r1=F1)
    w1 = I.uniform_sym(seed, "w1", h, f, bq, c0=U0, c1=U1)
    w2 = I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f), r0=U0, r1=U1)
    return {"qkv": qkv, "o": o, "w1": w1, "w2": w2}


def scores_for(cfg, r, lens, layer: int = 0):
    from synth import inputs as I
    sfx = "" if layer == 0 else f".{layer}"
    return {s: I.lognormal_scores(cfg.seed, f"score.{s}{sfx}", L, rank=r) for s, L in lens.items()}


# ------------------------------------------------------------ distributed
class Dist:
    def __init__(self, n_gpus: int, share_gpu: bool):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != n_gpus:
            raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={self.world} (launch N>1 with torchrun)")
        # --share-gpu: every rank on cuda:0 (one-GPU validation of the N > 1
        # path; kernels of different processes time-slice, so its timings
        # mean nothing) -- the host plane then runs over gloo
        self.device = 0 if share_gpu else self.local
        torch.cuda.set_device(self.device)
        self.cpu = share_gpu
        if self.world > 1:
            if share_gpu:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))

    def _t(self, v, dtype=None):
        return self.torch.tensor([v], dtype=dtype or self.torch.float64, device="cpu" if self.cpu else "cuda")

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.all_reduce(self._t(1.0))
        self.torch.cuda.synchronize()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self._t(v)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self._t(v)
        self.dist.all_reduce(t)
        return float(t.item())

    def bcast_obj(self, o):
        if self.world == 1:
            return o
        obj = [o]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def allgather_obj(self, o):
        if self.world == 1:
            return [o]
        out = [None] * self.world
        self.dist.all_gather_object(out, o)
        return out


def timed(D, fn, steps: int, stream, tail=None) -> float:
    """Device time of `steps` calls of fn (CUDA events on the launching stream,
    barrier + synchronize on both sides), max over ranks, ms per step.  `tail`
    joins side streams into `stream` before the end event."""
    torch = D.torch
    D.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    if tail is not None:
        tail()
    e1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    return D.max(e0.elapsed_time(e1)) / steps


# ------------------------------------------------------------- oracle legs
_ORACLE_INPUTS = {}


def oracle_inputs(cfg, gamma: float, tokens: int):
    """Seeded inputs of the sampled workload, prepared once (not timed)."""
    key = (cfg.name, gamma, tokens)
    if key not in _ORACLE_INPUTS:
        from oracle import ztp_oracle as O
        from synth import inputs as I
        h, f = cfg.h, cfg.f
        d = rank_shards(cfg, 1, 0)
        sh = O.LayerShards([d["qkv"]], [d["o"]], [d["w1"]], [d["w2"]])
        X = I.normal(cfg.seed, "x", h, cfg.N, c1=tokens)
        G = I.normal(cfg.seed, "g", h, cfg.N, c1=tokens)
        lens = {"qkv": h, "o": h, "fc1": h, "fc2": f}
        sc = scores_for(cfg, 0, lens)
        _ORACLE_INPUTS[key] = (X, G, sh, lens, sc)
    return _ORACLE_INPUTS[key]


def oracle_sample(cfg, gamma: float, tokens: int, budget_s: float):
    """The fp64 oracle (as it stands) on a token sample of the same workload --
    select + layer step per run; returns (TFLOP/s, seconds, runs, FLOPs per
    run).  Baseline leg only."""
    from oracle import ztp_oracle as O
    X, G, sh, lens, sc = oracle_inputs(cfg, gamma, tokens)
    t0 = time.perf_counter()
    flops, runs = 0.0, 0
    while True:
        sel = [{s: O.select(sc[s], min(int(math.floor(L * gamma + 0.5)), L - 1)) for s, L in lens.items()}]
        out = O.layer_step(X, G, sh, sel)
        flops += sum(out["flops"])
        runs += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return flops / dt / 1e12, dt, runs, flops / runs


def reference_arm(args):
    """--impl reference: the oracle on the box's host cores, rank 0 only; each
    step is the layer step on a bounded token sample of the same workload."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from synth.configs import CONFIGS
    cfg = CONFIGS[args.config]
    tokens = args.ref_tokens
    for _ in range(args.warmup):
        oracle_sample(cfg, args.gamma, tokens, 0.0)
    t0 = time.perf_counter()
    fl = 0.0
    for _ in range(args.steps):
        _, _, _, f1 = oracle_sample(cfg, args.gamma, tokens, 0.0)
        fl += f1
    total = time.perf_counter() - t0
    value = fl / total / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded splitmix64, bf16-rounded values)",
            "config": {"workload": f"{cfg.note}: 1 transformer layer fwd+bwd, TP=1, gamma={args.gamma} "
                                   f"(fp64 oracle on {tokens} of {cfg.N} tokens per step)",
                       "tokens_per_step": tokens},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"fp64 numpy oracle layer_step, {tokens} tokens x {args.steps} steps"},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ cases
def c5_schedule(e, per):
    """c5 time-varying slowdowns: four phases."""
    out = []
    for ph in range(4):
        chi = [1.0] * e
        if ph == 0:
            chi[0] = 2.0
        elif ph == 1:
            chi[3 % e] = 3.0
        elif ph == 2:
            for r, c in zip((1, 3, 5, 7), (8.0, 6.0, 4.0, 2.0)):
                if r < e:
                    chi[r] = c
        out.append((chi, per))
    return out


def matrix_cases(e):
    """The other BASELINE configs that run at TP = e."""
    if e == 4:
        return [dict(name="c3", cfg="c3", chi={3: 2.0}, semi=False)]
    if e == 8:
        return [dict(name="c4 x2 ZERO", cfg="c4", chi={5: 2.0}, semi=False),
                dict(name="c4 x3 SEMI", cfg="c4", chi={5: 3.0}, semi=True),
                dict(name="c5 adaptive", cfg="c5", schedule="c5", semi=True)]
    return []


class Case:
    """One config at TP = D.world on this rank: a context (+ symmetric window
    at N > 1), the rank's layer stack, graphs and timings."""

    def __init__(self, D, args, cfg, semi: bool, stream, cap_units: float = 1.0):
        import torch
        import paper_2401_11469_b200 as Z
        from paper_2401_11469_b200.layer import ZtpLayer, ZtpStack, sym_allocator
        from synth import inputs as I
        self.D, self.args, self.cfg, self.semi, self.stream = D, args, cfg, semi, stream
        self.Z, self.torch = Z, torch
        e, r = D.world, D.rank
        self.e, self.r = e, r
        h, f, N = cfg.h, cfg.f, cfg.N
        self.h, self.f, self.N, self.a, self.u = h, f, N, h // e, f // e
        use_nccl = e > 1 and args.transport == "nccl" and not args.share_gpu
        uid = Z.ztp_get_unique_id() if (use_nccl and r == 0) else None
        uid = D.bcast_obj(uid) if use_nccl else None
        self.ctx = Z.ztp_ctx_create(r, e, uid, D.device)
        # receive capacity (MLP units) for migrated work: one straggler's whole
        # shard by default; forced plans (lambda sweep) can pile more on a rank
        self.cap = int(self.u * cap_units) if semi else 0
        nl = cfg.layers
        alloc = None
        if e > 1:
            nbytes = nl * ZtpLayer.window_bytes(h, f, N, e, self.cap) + 2 * h * N + (1 << 20)  # + e2e's dX
            hdl = Z.ztp_window_create(self.ctx, nbytes)
            Z.ztp_window_open(self.ctx, D.allgather_obj(hdl))
            alloc = sym_allocator(self.ctx, D.device)
        self.transport = "nccl" if use_nccl else ("peer" if e > 1 else "none")
        lens = {"qkv": h, "o": self.a, "fc1": h, "fc2": self.u}
        layers, self.scores = [], []
        gen = torch.Generator(device="cuda")
        for li in range(nl):
            if li == 0:
                sh = rank_shards(cfg, e, r)
                dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
            else:    # further layers of the stack: device-seeded weights of the same scale
                gen.manual_seed(cfg.seed * 1000 + li * 16 + r)
                a, u = self.a, self.u
                dev = {"qkv": (torch.rand(h, 3 * a, device="cuda", generator=gen) * 2 - 1) * h ** -0.5,
                       "o": (torch.rand(a, h, device="cuda", generator=gen) * 2 - 1) * h ** -0.5,
                       "w1": (torch.rand(h, u, device="cuda", generator=gen) * 2 - 1) * h ** -0.5,
                       "w2": (torch.rand(u, h, device="cuda", generator=gen) * 2 - 1) * f ** -0.5}
                dev = {k: v.to(torch.bfloat16) for k, v in dev.items()}
            attn = None
            if getattr(args, "attention", "standin") == "real":
                from paper_2401_11469_b200.layer import AttnSpec
                attn = AttnSpec(cfg.head_dim, cfg.seq, cfg.causal)
            L = ZtpLayer(self.ctx, h, f, N, r, e, dev, mig_cap=self.cap, layer_id=li, alloc=alloc, attn=attn)
            if li == 0:
                L.X.copy_(torch.from_numpy(I.normal(cfg.seed, "x", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
                L.G.copy_(torch.from_numpy(I.normal(cfg.seed, "g", h, N).astype(np.float32)).cuda().to(torch.bfloat16))
            else:
                L.X.copy_(layers[-1].Y)
                L.G.normal_(generator=gen)
            layers.append(L)
            self.scores.append({s: torch.from_numpy(v).cuda() for s, v in scores_for(cfg, r, lens, li).items()})
        self.stack = ZtpStack(layers)
        self.L0 = layers[0]
        self.graph, self.gkey, self.version = None, None, 0
        self.plan, self.chi = None, 1.0
        self.apply(None)

    # ------------------------------------------------------------ plumbing
    def apply(self, plan):
        """A plan -> this rank's migration ranges and prune counts (library:
        ztp_plan_counts, ztp_layer_prune_counts) and its selection (ztp_select,
        once per plan).  Every rank applies the same plan."""
        from paper_2401_11469_b200.layer import MigrationIO, migration_io, SEGS
        Z = self.Z
        mio = migration_io(plan, self.r, self.e, self.u, self.h) if plan is not None else MigrationIO()
        counts = (Z.ztp_layer_prune_counts(plan, self.r, self.h, self.a, self.u) if plan is not None
                  else {s: 0 for s in SEGS})
        for li, L in enumerate(self.stack.layers):
            L.set_migration(mio)
            L.set_selection(counts, self.scores[li], self.stream)
        self.plan = Z.PlanT.from_buffer_copy(plan) if plan is not None else None
        self.version += 1

    def set_chi(self, chi: float):
        self.Z.ztp_set_slowdown(self.ctx, chi)
        self.chi = chi

    def ensure_graph(self):
        """Capture the step for the current (plan, slowdown) after two eager
        warm-up steps (they size workspaces and set kernel attributes)."""
        key = (self.version, self.chi)
        if self.gkey == key:
            return self.graph
        torch, Z = self.torch, self.Z
        self.graph = None
        for _ in range(2):
            self.stack.step(self.stream)
        torch.cuda.synchronize()
        n0 = Z.ztp_launch_count(self.ctx)
        self.graph = self.stack.capture(self.stream)
        self.launches_per_step = Z.ztp_launch_count(self.ctx) - n0
        torch.cuda.synchronize()
        self.gkey = key
        return self.graph

    def run(self, steps: int, warm: int) -> float:
        """warm untimed replays (at least ~100 ms of them, so the timed steps
        start from the clock / power state of a running job), then `steps`
        timed replays; ms per step, max over ranks.  The warm-up count is
        agreed over ranks (max), since every replay runs collectives."""
        torch, D = self.torch, self.D
        g = self.ensure_graph()
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        per = max((time.time() - t0) / 3, 1e-6)
        n = int(D.max(float(max(warm, min(2000, math.ceil(0.1 / per))))))
        for i in range(3, n):
            g.replay()
            if i % 50 == 0:
                torch.cuda.synchronize()
        return timed(D, g.replay, steps, self.stream)

    def stats_window(self, n: int = 6):
        """Statistics of n eager steps (A-5, A-6): T_i = busy time of the
        rank's own kernels (GEMM + delay + the rest, collective waits
        excluded), M_i = GEMM (+ delay) time, all-gathered (ztp_allgather_stats)."""
        torch, Z = self.torch, self.Z
        Z.ztp_set_stats(self.ctx, True)
        Z.ztp_read_profile(self.ctx, self.stream)
        Z.ztp_set_profile(self.ctx, True)
        self.D.barrier()
        torch.cuda._sleep(int(2e8))   # hold the stream: the kernels then run back to back
        for _ in range(n):
            self.stack.step(self.stream)
        p = Z.ztp_read_profile(self.ctx, self.stream)
        Z.ztp_set_profile(self.ctx, False)
        Z.ztp_set_stats(self.ctx, False)
        T_own, M_own = (p["gemm_ms"] + p["other_ms"]) / n, p["gemm_ms"] / n
        return Z.ztp_allgather_stats(self.ctx, T_own, M_own, self.e, self.stream)

    def ingraph_gemm(self, reps: int = 10):
        """GEMM kernel time and executed FLOPs per step from the GEMMs' own
        %globaltimer stamps inside the captured step (no events, same launch
        schedule and PDL edges)."""
        torch, Z = self.torch, self.Z
        Z.ztp_set_profile(self.ctx, 2)
        gP = self.stack.capture(self.stream)
        for _ in range(5):
            gP.replay()
        Z.ztp_read_profile(self.ctx, self.stream)
        ms = fl = 0.0
        for _ in range(reps):
            gP.replay()
            pr = Z.ztp_read_profile(self.ctx, self.stream)
            ms += pr["gemm_kernel_ms"]
            fl += pr["gemm_flops"]
        Z.ztp_set_profile(self.ctx, 0)
        del gP
        torch.cuda.synchronize()
        return ms / reps, fl / reps

    def costs(self):
        """Alg.2 l.1 pretest on every rank in lockstep (its steps run the
        collectives), Phi_1 on real peer pulls; rank 0's functions are
        broadcast so every rank plans with identical costs."""
        from paper_2401_11469_b200.pretest import pretest
        Z = self.Z
        _, rep = pretest(self.L0, self.ctx, self.scores[0], steps=10, ctx_rank=self.r, world_pull=self.e > 1)
        self.apply(None)
        self.gkey = None
        c = self.D.bcast_obj(rep["costs"])
        nl = len(self.stack.layers)
        sc = lambda p: (p[0], tuple(y * nl for y in p[1]))  # noqa: E731  (per layer -> the stack)
        return Z.make_costs(c["omega1"] * nl, sc(c["omega2"]), sc(c["phi1"]), sc(c["phi2"])), c

    def destroy(self):
        self.graph = None
        self.torch.cuda.synchronize()
        self.D.barrier()
        self.Z.ztp_ctx_destroy(self.ctx)


def table1(D, args, stream):
    """Table I analog on this box's ranks: the
    paper-literal sending-collecting migration of one column linear (c4's FC1
    at TP = e: K = h, n = f / e, N tokens) in a homogeneous setting -- nu
    ranks each migrate a fraction gamma of their contraction rows to the
    normal ranks, broadcast-reduce (NCCL broadcast / reduce) vs
    scatter-gather (point-to-point) -- step (FWD + BWD) ms, max over ranks,
    and its ratio to gamma = 0."""
    import torch
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.kmig import KMigColLinear
    from paper_2401_11469_b200.layer import sym_allocator
    from synth.configs import CONFIGS
    e, r = D.world, D.rank
    cfg = CONFIGS["c4"]
    K, n, N = cfg.h, cfg.f // e, cfg.N
    use_nccl = args.transport == "nccl" and not args.share_gpu
    uid = D.bcast_obj(Z.ztp_get_unique_id() if (use_nccl and r == 0) else None) if use_nccl else None
    ctx = Z.ztp_ctx_create(r, e, uid, D.device)
    Z.ztp_window_open(ctx, D.allgather_obj(Z.ztp_window_create(ctx, 8 << 30)))
    alloc = sym_allocator(ctx, D.device)
    nus = sorted({1, min(4, e - 1)})
    rows = []
    for nu in nus:
        migr = list(range(e - nu, e))
        for mode, mname in ((Z.COLL_TREE, "broadcast-reduce"), (Z.COLL_P2P, "scatter-gather")):
            row = {"policy": mname, "nu": nu, "ms": {}}
            for g in (0.0, 0.25, 0.5, 0.75, 1.0):
                k = min(int(round(g * K)), K - 64)       # >= 64 contraction rows stay (A-4 analog)
                Lk = KMigColLinear(ctx, r, e, K, n, N, migr if k else [], k, mode, alloc=alloc)
                Lk.X.normal_()
                Lk.W.uniform_(-K ** -0.5, K ** -0.5)
                Lk.G.normal_()
                for _ in range(2):
                    Lk.step(stream)
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    Lk.step(stream)
                for _ in range(3):
                    gr.replay()
                row["ms"][str(g)] = timed(D, gr.replay, 20, stream)
                del gr, Lk
            base = row["ms"]["0.0"]
            row["ratio"] = {gk: v / base for gk, v in row["ms"].items()}
            rows.append(row)
    D.barrier()
    Z.ztp_ctx_destroy(ctx)
    return {"workload": f"c4 FC1 column linear at TP={e}: K={K}, n={n}, N={N}, fwd+bwd, homogeneous",
            "transport": "nccl collectives + peer pulls" if use_nccl else "peer", "rows": rows,
            "paper_v100_ratio_gamma1": {"broadcast-reduce(1)": 500 / 373, "scatter-gather(1)": 963 / 373,
                                        "broadcast-reduce(4)": 1113 / 373, "scatter-gather(4)": 1436 / 373}}


def lambda_sweep(D, args, stream):
    """NEXT-4's multi-straggler study: c4 at TP = 8
    with ranks 1, 3, 5, 7 slowed x8, x6, x4, x2 (the paper's setting), one
    statistics window, then the plan with Eq.3's migration bound forced to
    lambda = 0 .. 4 (force_lambda; lambda = 0 is ZERO for all four
    stragglers, lambda = 4 migration for all), each applied and timed; the
    automatic Eq.3 choice alongside."""
    import paper_2401_11469_b200 as Z
    from synth.configs import CONFIGS
    e = D.world
    C = Case(D, args, CONFIGS["c4"], True, stream, cap_units=2.0)
    chis = [1.0] * e
    for q, c in zip((1, 3, 5, 7), (8.0, 6.0, 4.0, 2.0)):
        if q < e:
            chis[q] = c
    C.set_chi(1.0)
    t_free = C.run(30, 3)
    costs, cplain = C.costs()
    C.set_chi(chis[D.rank])
    t_unbal = C.run(20, 3)
    T, M = C.stats_window()
    rows = []
    for lam in (-1, 0, 1, 2, 3, 4):
        opts = Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN, eps=args.eps, force_lambda=lam)
        plan = Z.ztp_plan(T, M, float(C.u), costs, opts)
        C.apply(plan)
        ms = C.run(20, 3)
        rows.append({"lambda": "auto (Eq.3)" if lam < 0 else lam, "x": int(plan.x), "ms": ms,
                     "recovery": t_free / ms, "speedup": t_unbal / ms, "plan": plan_summary(plan, e)})
    C.destroy()
    return {"workload": f"c4 at TP={e}, ranks 1,3,5,7 (those < TP) slowed x8,x6,x4,x2", "T_free_ms": t_free,
            "T_unbal_ms": t_unbal,
            "window_T_ms": T, "rows": rows, "pretest_costs": cplain}


def plan_summary(plan, e):
    if plan is None:
        return {"roles": "N" * e}
    return {"roles": "".join("NRMS"[int(x)] for x in list(plan.role)[:e]),
            "gamma": [round(g, 4) for g in list(plan.gamma)[:e]],
            "gamma_r": [round(g, 4) for g in list(plan.gamma_r)[:e]],
            "beta": [round(b, 4) for b in list(plan.beta)[:e]], "z": int(plan.z), "x": int(plan.x)}


def controller_run(C, args, schedule, semi, final_steps=0):
    """T_free, then per phase T_unbal and ztp_ctl_step steps under the
    phase's slowdowns; each controller step = the plan's graph replayed
    (timed, max over ranks) + a statistics window fed to ztp_ctl_step."""
    Z, e, r = C.Z, C.e, C.r
    C.apply(None)
    C.set_chi(1.0)
    t_free = C.run(args.steps if final_steps else 30, args.warmup)
    costs, cplain = (C.costs() if semi else (None, None))
    opts = Z.ctl_opts(L_ref=float(C.u), trigger=0.10, max_refines=2, enable_migration=int(semi),
                      zero_crit=Z.CRIT_AVG if args.criterion == "avg" else Z.CRIT_MIN, eps=args.eps)
    ctl = Z.ztp_ctl_init(e)
    phases, series = [], []
    for ph, (chis, nsteps) in enumerate(schedule):
        plan_keep = C.plan
        C.apply(None)
        C.set_chi(chis[r])
        t_unbal = C.run(30, 3)
        C.apply(plan_keep)
        rows = []
        for k in range(nsteps):
            state = ["window", "first", "monitor"][ctl.state]
            ms = C.run(20, 3)
            T, M = C.stats_window()
            act = Z.ztp_ctl_step(ctl, opts, T, M, costs)
            rec = {"phase": ph, "step": k, "state": state, "ms": round(ms, 4), "plan": plan_summary(C.plan, e),
                   "T_ms": [round(x, 4) for x in T], "M_ms": [round(x, 4) for x in M],
                   "action": "apply" if act == Z.CTL_APPLY else "keep"}
            if act == Z.CTL_APPLY:
                C.apply(ctl.plan if not _dense(ctl.plan, e) else None)
            rows.append(rec)
        series += rows
        mon = [x["ms"] for x in rows if x["state"] == "monitor"] or [rows[-1]["ms"]]
        phases.append({"chi": chis, "T_unbal_ms": t_unbal, "T_bal_ms": float(np.mean(mon)),
                       "recovery": t_free / float(np.mean(mon)), "speedup": t_unbal / float(np.mean(mon)),
                       "final_plan": plan_summary(C.plan, e)})
    out = {"T_free_ms": t_free, "phases": phases, "series": series, "pretest_costs": cplain,
           "controller": {"windows": ctl.windows, "replans": ctl.replans, "refines": ctl.refine_count,
                          "triggers": ctl.triggers}}
    if final_steps:
        out["T_bal_ms"] = C.run(final_steps, args.warmup)
    return out


def _dense(plan, e):
    return all(int(plan.role[q]) == 0 for q in range(e))


def case_summary(C, name, res, peak):
    g_ms, g_fl = C.ingraph_gemm(5)
    frac = C.D.allgather_obj(g_fl / (g_ms * 1e-3) / 1e12 / peak if g_ms > 0 else None)
    out = {"name": name, "config": C.cfg.note, "tp": C.e, "transport": C.transport,
           "T_free_ms": res["T_free_ms"], "phases": [{k: v for k, v in p.items()} for p in res["phases"]],
           "controller": res["controller"], "gemm_frac_per_rank": frac}
    if len(res["phases"]) == 1:
        p = res["phases"][0]
        out.update(T_unbal_ms=p["T_unbal_ms"], T_bal_ms=p["T_bal_ms"], recovery=p["recovery"],
                   speedup=p["speedup"], final_plan=p["final_plan"])
    return out


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ztp", choices=["ztp", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--gamma", type=float, default=0.5, help="N=1 homogeneous prune ratio")
    ap.add_argument("--chi", type=float, default=2.0, help="straggler slowdown (N>1)")
    ap.add_argument("--eps", type=float, default=0.05, help="A-17 straggler tolerance above timing noise")
    ap.add_argument("--criterion", default="min", choices=["min", "avg"],
                    help="N>1 Eq.1 criterion: T_min (A-7, headline) or the paper-literal T_avg")
    ap.add_argument("--ctl-steps", type=int, default=6, help="controller steps per phase (N>1)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"])
    ap.add_argument("--share-gpu", action="store_true", help="N>1 on one GPU (path validation only)")
    ap.add_argument("--no-matrix", action="store_true")
    ap.add_argument("--attention", default="standin", choices=["standin", "real"],
                    help="attention core: A-31's stand-in (default) or real fused attention (NEXT-4)")
    ap.add_argument("--extras", default="all", choices=["all", "table1", "lambda", "none"],
                    help="N>1 extras: Table I analog, forced-lambda sweep (N=8)")
    ap.add_argument("--ref-tokens", type=int, default=256)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import paper_2401_11469_b200 as Z
    from synth.configs import CONFIGS

    D = Dist(args.gpus, args.share_gpu)
    e, r = D.world, D.rank
    cfg = CONFIGS[args.config]
    h, f, N = cfg.h, cfg.f, cfg.N
    peak_burst, peak_sus, hbm, peak_src = load_peaks()
    sampler = ClockSampler(D.device)
    sampler.start()
    stream = torch.cuda.Stream()          # capture needs a non-default stream
    torch.cuda.set_stream(stream)
    C = Case(D, args, cfg, False, stream)
    plan_info, extra = {}, {}
    if e == 1:
        # ---- dense step, then homogeneous resize at gamma (P:344 E2 analog)
        C.set_chi(1.0)
        ms_free = C.run(args.steps, args.warmup)
        flops_dense = C.stack.executed_flops()
        C.apply(Z.ztp_plan_uniform(1, args.gamma))
        plan_info = {"gamma": [args.gamma], "mode": "homogeneous ZERO-Pri", "n_prune": dict(C.L0.n_prune)}
        ms_bal = C.run(args.steps, args.warmup)
    else:
        chis = [args.chi if q == e - 1 else 1.0 for q in range(e)]
        res = controller_run(C, args, [(chis, args.ctl_steps)], False, final_steps=args.steps)
        ms_free, ms_bal = res["T_free_ms"], res["T_bal_ms"]
        ph = res["phases"][0]
        flops_dense = None
        plan_info = {"final": ph["final_plan"], "controller": res["controller"], "criterion": "T_avg (paper-literal Eq.1)" if args.criterion == "avg" else "T_min (A-7)",
                     "eps": args.eps, "series": [{k: v for k, v in s.items() if k not in ("T_ms", "M_ms")}
                                                 for s in res["series"]]}
        extra = {"ms_unbal": ph["T_unbal_ms"], "recovery": ms_free / ms_bal, "speedup": ph["T_unbal_ms"] / ms_bal}
    launches = C.launches_per_step * args.steps
    # per-step distribution (median / p10 / p90 over 50 steps),
    # a separate pass after the timed region (the headline is the timed mean)
    g = C.ensure_graph()
    n_dist = 50
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_dist)]
    D.barrier()
    for a0, a1 in evs:
        a0.record(stream)
        g.replay()
        a1.record(stream)
    torch.cuda.synchronize()
    per_step = sorted(D.max(a0.elapsed_time(a1)) for a0, a1 in evs)
    step_dist = {"p10": per_step[n_dist // 10], "p50": per_step[n_dist // 2], "p90": per_step[(9 * n_dist) // 10],
                 "n": n_dist, "how": "one event pair per replay (launch gaps included), max over ranks"}
    flops_exec_rank = C.stack.executed_flops()
    flops_exec = D.sum(flops_exec_rank)
    flops_method = D.sum(C.stack.method_flops())
    value = flops_exec / (ms_bal * 1e-3) / 1e12
    t_g0 = time.time()
    gemm_ms, gemm_fl = C.ingraph_gemm(40)
    clk_gemm = sampler.median_mhz(t_g0, time.time())
    # the same measurement after 1 s idle: the board's power cap lowers SM
    # clocks during long replay runs, so the GEMM class is
    # also reported from a cool start (frac_after_idle); `frac` stays the
    # conservative, hot number taken right after the timed region
    torch.cuda.synchronize()
    time.sleep(1.0)
    gemm_ms_cool, gemm_fl_cool = C.ingraph_gemm()

    # ---- e2e: host buffers through the public API (pinned H2D of X, G; D2H of
    # dX every step), double-buffered like a prefetching input pipeline: step
    # i+1's H2D (copy stream) and step i-1's D2H (second copy stream) overlap
    # step i's compute; every copy of every step is inside the timed region.
    L = C.L0
    C.graph = None
    dX2 = L.alloc(h, N, torch.bfloat16) if L.alloc is not None else torch.empty_like(L.dX)  # all-reduce target
    Xd, Gd, dXd = [L.X, L.X.clone()], [L.G, L.G.clone()], [L.dX, dX2]
    Xp = [torch.empty((h, N), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    Gp = [torch.empty((h, N), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    dXp = [torch.empty((h, N), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    for k in range(2):
        Xp[k].copy_(L.X.cpu())
        Gp[k].copy_(L.G.cpu())
    gE = []
    for k in range(2):                      # one graph per buffer set
        L.X, L.G, L.dX = Xd[k], Gd[k], dXd[k]
        L._build_args()
        C.gkey = None
        gE.append(C.ensure_graph())
    L.X, L.G, L.dX = Xd[0], Gd[0], dXd[0]
    L._build_args()
    C.gkey = None
    cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    st = {"i": 0}

    def e2e_step():
        i, k = st["i"], st["i"] % 2
        if i == 0:                           # first H2D after the start event
            ev0 = torch.cuda.Event()
            ev0.record(stream)
            cin.wait_event(ev0)
        elif i >= 2:
            cin.wait_event(ev_comp[k])       # step i-2 is done with Xd[k], Gd[k]
        with torch.cuda.stream(cin):
            Xd[k].copy_(Xp[k], non_blocking=True)
            Gd[k].copy_(Gp[k], non_blocking=True)
        ev_in[k].record(cin)
        stream.wait_event(ev_in[k])
        if i >= 2:
            stream.wait_event(ev_out[k])     # D2H of step i-2 has read dXd[k]
        gE[k].replay()
        ev_comp[k].record(stream)
        cout.wait_event(ev_comp[k])
        with torch.cuda.stream(cout):
            dXp[k].copy_(dXd[k], non_blocking=True)
        ev_out[k].record(cout)
        st["i"] += 1

    def e2e_tail():
        for k in range(2):
            stream.wait_event(ev_out[k])

    for _ in range(3):                       # warm-up
        e2e_step()
    e2e_tail()
    torch.cuda.synchronize()
    st["i"] = 0
    e2e_steps = max(10, args.steps // 4)
    ms_e2e = timed(D, e2e_step, e2e_steps, stream, tail=e2e_tail)
    del gE
    clocks = sampler.stop()

    # ---- roofline of the dominant kernel (the resized tcgen05 GEMM): one
    # step's GEMM launches, kernel time from their own %globaltimer stamps
    # (first CTA start .. last CTA end, split-K reduce included)
    achieved = gemm_fl / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    timed_s = ms_bal * args.steps * 1e-3
    peak = peak_sus if timed_s >= 1.0 else peak_burst
    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = (tj.get("per_config", {}).get(f"{args.config}_tp{e}") or {}).get("bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "tensor", "kernel": "ztp_gemm_kernel (tcgen05 kind::f16, TMEM accum)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_source": f"{peak_src} {'sustained' if peak is peak_sus else 'burst'} bf16 (MEASURED_PEAKS.json)",
            "gemm_share_of_step": gemm_ms / ms_bal if ms_bal else None,
            "gemm_kernel_ms_per_step": gemm_ms, "gemm_executed_gflop_per_step": gemm_fl / 1e9,
            "frac_after_idle": (gemm_fl_cool / (gemm_ms_cool * 1e-3) / 1e12 / peak) if gemm_ms_cool > 0 else None,
            "sm_mhz_during_measure": clk_gemm,
            "frac_clock_normalized": (achieved / (peak * clk_gemm / 1965.0)) if (achieved and clk_gemm) else None,
            "gemm_kernel_ms_per_step_after_idle": gemm_ms_cool,
            "measured": "executed GEMM FLOPs / GEMM kernel time from the kernels' own %globaltimer stamps (first "
                        "CTA start after its PDL wait to last CTA end, split-K reduce included), union per step, "
                        "inside the captured step graph (10 replays after the timed region), rank 0"}
    # step roofline: max(GEMM at peak, collective bytes at NVLink) per rank,
    # on the FLOPs the GEMMs execute
    comm_bytes = 4 * 2 * N * h * 2 * (e - 1) / e * cfg.layers if e > 1 else 0.0
    t_ideal = max(flops_exec_rank / (peak_burst * 1e12), comm_bytes / (NVLINK_GBS * 1e9))
    cpu = None
    if r == 0 and e == 1 and not args.no_cpu:
        v, dt, runs, _ = oracle_sample(cfg, args.gamma, 512, args.cpu_budget)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"fp64 numpy oracle layer_step (TP=1, gamma={args.gamma}) on 512 of {N} tokens, "
                         f"{runs} runs in {dt:.1f} s"}
    matrix = []
    C.destroy()
    if e > 1 and not args.no_matrix:
        for mc in (matrix_cases(e) if args.extras == "all" else []):
            mcfg = CONFIGS[mc["cfg"]]
            M = Case(D, args, mcfg, mc["semi"], stream)
            if mc.get("schedule") == "c5":
                sched = c5_schedule(e, args.ctl_steps + 2)
            else:
                sched = [([mc["chi"].get(q, 1.0) for q in range(e)], args.ctl_steps)]
            res = controller_run(M, args, sched, mc["semi"])
            matrix.append(case_summary(M, mc["name"], res, peak_burst))
            M.destroy()
            torch.cuda.empty_cache()
        if args.extras in ("all", "table1"):
            extra["table1"] = table1(D, args, stream)
        if (e == 8 and args.extras == "all") or args.extras == "lambda":
            extra["lambda_sweep"] = lambda_sweep(D, args, stream)
        torch.cuda.empty_cache()
    h2d = 2 * h * N * 2
    d2h = h * N * 2
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": e, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_bal, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded splitmix64 inputs, random-init weights)",
        "config": {"workload": f"{cfg.note}: {cfg.layers} transformer layer(s) (attn-proj + MLP) fwd+bwd, TP={e}",
                   "tp": e, "tokens": N, "hidden": h, "ffn": f, "transport": C.transport,
                   "mode": ("homogeneous ZERO-Pri gamma=%.2f" % args.gamma) if e == 1 else
                           f"rank {e - 1} slowed {args.chi}x, ZERO-resizing (T_min), ztp_ctl_step controller",
                   "selection": "ztp_select once per plan (P:187 epoch granularity), not in the step",
                   "attention_core": ("real: cuDNN fused attention (torch SDPA) between ztp_transpose layout changes"
                                      if args.attention == "real" else "stand-in ctx = Q + K + V (A-31)"),
                   "l2": "no flush: per-step working set > 126 MB L2 (activations ~%d MB)" %
                         int((2 * h * N * 2 * 6 + 2 * (f // e) * N * 2 * 2) / 1e6)},
        "method_tflops": flops_method / (ms_bal * 1e-3) / 1e12,
        "flops_note": "value counts the FLOPs the GEMMs execute; method_tflops counts 6 N n K' per linear "
                      "(SURVEY §8(d)), which output pruning (A-35/A-36) partly avoids executing",
        "e2e": {"value": flops_exec / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "pipeline": "double-buffered: H2D(i+1) and D2H(i-1) on copy streams overlap compute(i)"},
        "gpu_launches": launches,
        "roofline": roof,
        "step_roofline": {"ideal_ms": t_ideal * 1e3, "frac": (t_ideal * 1e3) / ms_bal,
                          "rule": "max(rank executed GEMM FLOPs / burst peak, all-reduce ring bytes / 770 GB/s)"},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "step_ms_dist": step_dist,
        "ms_dense_free": ms_free,
        "plan": plan_info,
    }
    if e > 1:
        line.update(extra)
        line["matrix"] = matrix
        if args.share_gpu:
            line["note"] = "--share-gpu: all ranks on one GPU (path validation; timings are not meaningful)"
    else:
        line["dense_tflops"] = flops_dense / (ms_free * 1e-3) / 1e12
        line["speedup_vs_dense"] = ms_free / ms_bal
    if r == 0:
        print(json.dumps(line), flush=True)
    if e > 1:
        D.dist.destroy_process_group()


if __name__ == "__main__":
    main()

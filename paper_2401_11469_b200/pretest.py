"""Alg.2 l.1 "pretestDiffRatio(Omega_1, Omega_2, Phi_1)":
measure, before training, the cost functions Eq.2 / Eq.3 weigh against each
other, and hand them to ztp_plan as a ztp_costs (piecewise linear, SURVEY
§8(a) row a2, §8(d) timing protocol step 6).

  Omega_1     "static space allocation overhead for the submatrix with
              reduced dimensions": the extra non-GEMM time a step
              pays as soon as it resizes at all (select, compaction copies,
              imputation launches) -- measured at the smallest ratio.
  Omega_2(n)  "proportionally increased dimension extracting cost" of n
              pruned units: the extra non-GEMM time at n = L gamma pruned
              units, minus Omega_1.
  Phi_1(n)    "communication cost" of migrating n units: the weight
              slices out (W1^T columns, W2^T rows) and the dW slices back,
              per step, through ztp_migrate.
  Phi_2(m)    "computation cost" on a helper of m received units (P:258,
              P:280 infers it from the receiver's speed): measured directly
              as the step-time increase of a rank that appends m units.

x axes are MLP hidden units (L = u, the rank's FFN units, A-25); times are
milliseconds, the unit of the statistics T / M the plan receives.  Every
sample comes from CUDA-graph replays of the rank's real step through the C
ABI (select + GEMMs + epilogues), so the functions carry this box's fixed
costs, not a model.

Only host orchestration lives here (timing, sample bookkeeping); all work
runs in libztp.so.  The pure-host part (`fit_costs`) is unit-tested on CPU.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import paper_2401_11469_b200 as Z

GAMMAS = (0.0, 0.125, 0.25, 0.5, 0.75)
FRACS = (0.0, 0.125, 0.25, 0.5, 1.0)


def fit_costs(omega: Sequence[Tuple[float, float]], phi1: Sequence[Tuple[float, float]],
              phi2: Sequence[Tuple[float, float]]):
    """Raw pretest samples -> (ztp_costs keepalive tuple, plain dict), fitted
    by the library (ztp_costs_fit, A-40): omega = (pruned units n, extra
    non-GEMM ms vs the dense step), phi1 = (migrated units, ms), phi2 =
    (units received by one helper, ms)."""
    return Z.ztp_costs_fit(list(omega), list(phi1), list(phi2))


# ----------------------------------------------------------------- GPU side
def time_step(L, ctx, chi: float = 1.0, steps: int = 30, reps: int = 3) -> float:
    """Median over `reps` of the mean replay time (ms) of one captured step."""
    import torch
    stream = torch.cuda.Stream()
    Z.ztp_set_slowdown(ctx, chi)
    L.step(stream, select=False)          # selection: once per plan, not per step
    torch.cuda.synchronize()
    g = L.capture(stream, select=False)
    with torch.cuda.stream(stream):      # replay() issues on the current stream
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / steps)
    del g
    out.sort()
    return out[len(out) // 2]


def gemm_ms(L, ctx, steps: int = 5) -> float:
    """M (A-6): GEMM (+ emulated delay) time per step from the kernels' own
    stamps (statistics mode)."""
    Z.ztp_set_stats(ctx, True)
    Z.ztp_read_gemm_ns(ctx)
    for _ in range(steps):
        L.step(select=False)
    m = Z.ztp_read_gemm_ns(ctx) / steps / 1e6
    Z.ztp_set_stats(ctx, False)
    return m


def _homog_counts(L, g: float) -> Dict[str, int]:
    """The four prune counts of one homogeneous ratio (library: A-3, A-4)."""
    return Z.ztp_layer_prune_counts(Z.ztp_plan_uniform(1, g), 0, L.h, L.a, L.u)


def pretest(L, ctx, scores: Dict, *, gammas: Sequence[float] = GAMMAS, fracs: Sequence[float] = FRACS,
            steps: int = 30, link_gbs: Optional[float] = None, ctx_rank: int = 0, world_pull: bool = False):
    """Run the pretest on this rank's layer `L` (a ZtpLayer built with
    mig_cap >= L.u * max(fracs)) and return (costs, report).

    Phi_1's copies are local device copies through ztp_migrate (src = dst =
    ctx_rank, the rank of `ctx`): the one-GPU stand-in for the peer pulls of
    a multi-GPU box.  link_gbs: if given, Phi_1 is
    additionally modelled as bytes / link_gbs + the measured per-call fixed
    cost, and the MODEL is what the returned costs use (a one-GPU run cannot
    time NVLink; report["phi1_measured"] keeps the local copies).
    world_pull (TP > 1, every rank calls pretest in lockstep): Phi_1 is timed
    on real peer pulls between ranks (ztp_migrate), no model.
    The layer is left dense, without migration."""
    import torch
    from paper_2401_11469_b200.layer import MigrationIO

    u, h = L.u, L.h
    rep: Dict[str, List] = {"omega": [], "phi1_measured": [], "phi2": []}
    L.set_migration(MigrationIO())
    # ---- Omega: extra non-GEMM time of a resized step (gamma sweep)
    base = None
    for g in sorted(set([0.0] + list(gammas))):
        L.set_selection(_homog_counts(L, g), scores)
        T = time_step(L, ctx, 1.0, steps)
        M = gemm_ms(L, ctx)
        over = T - M
        if base is None:
            base = over
        n = L.n_prune["fc2"]
        rep["omega"].append({"gamma": g, "n_pruned": n, "T_ms": T, "M_ms": M, "extra_ms": over - base})
    # ---- Phi_2: a helper appending m units (merged accumulation, A-26)
    L.set_selection(_homog_counts(L, 0.0), scores)
    t0 = None
    src = (L.rank + 1) % max(L.world, 2)
    for fr in sorted(set([0.0] + list(fracs))):
        m = int(u * fr + 0.5)
        if m > L.cap:
            continue
        L.set_migration(MigrationIO(inc=[(src, 0, m)] if m > 0 else []))
        L.set_selection(_homog_counts(L, 0.0), scores)
        T = time_step(L, ctx, 1.0, steps)
        if t0 is None:
            t0 = T
        rep["phi2"].append({"units": m, "T_ms": T, "extra_ms": T - t0})
    L.set_migration(MigrationIO())
    L.set_selection(_homog_counts(L, 0.0), scores)
    # ---- Phi_1: weight slices out + dW slices back for n units
    stream = torch.cuda.Stream()
    fixed = None
    for fr in sorted(set(list(fracs))):
        n = int(u * fr + 0.5)
        if n == 0 or n > L.cap:
            continue
        xs = []
        # one GPU: local copies; TP > 1 (world_pull): every rank d pulls the
        # slices of rank d+1 -- n units cross every link, as they cross the
        # straggler's egress in a plan (collective: all ranks run it)
        pairs = ([((d + 1) % L.world, d) for d in range(L.world)] if world_pull and L.world > 1
                 else [(ctx_rank, ctx_rank)])
        for src_r, dst_r in pairs:
            for t, r0, c0, nr, nc, dr0, dc0 in ((L.w1_t, 0, 0, h, n, 0, u), (L.w2_t, 0, 0, n, h, u, 0),
                                               (L.dw1, 0, u, h, n, 0, 0), (L.dw2, u, 0, n, h, 0, 0)):
                xs.append(Z.xfer(t, t, r0=r0, c0=c0, nr=nr, nc=nc, dr0=dr0, dc0=dc0, src_rank=src_r, dst_rank=dst_r))
        for _ in range(3):
            Z.ztp_migrate(ctx, xs, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(reps):
                Z.ztp_migrate(ctx, xs, stream)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nbytes = 4 * n * h * L.w1_t.element_size()
        rep["phi1_measured"].append({"units": n, "ms": ms, "bytes": nbytes})
        fixed = ms if fixed is None else min(fixed, ms)
    if link_gbs:
        # bandwidth model over the link, with the smallest measured call as
        # its fixed cost (launch + latency), never below the measured copy
        rep["phi1"] = [{"units": d["units"], "ms": max(d["ms"], 0.5 * fixed + d["bytes"] / (link_gbs * 1e9) * 1e3),
                        "model": f"bytes / {link_gbs} GB/s + fixed"} for d in rep["phi1_measured"]]
    else:
        rep["phi1"] = rep["phi1_measured"]
    costs, plain = fit_costs([(d["n_pruned"], d["extra_ms"]) for d in rep["omega"]],
                             [(d["units"], d["ms"]) for d in rep["phi1"]],
                             [(d["units"], d["extra_ms"]) for d in rep["phi2"]])
    rep["costs"] = plain
    return costs, rep

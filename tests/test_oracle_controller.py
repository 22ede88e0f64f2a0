"""Pins of the oracle's statistics refresh and re-planning controller (P:171-178,
Alg.2; readings A-8, A-39, A-41, A-42, A-43) against what the paper fixes and
against closed-form runtime models -- not against the oracle itself.

The runtime model used here (a model, not a measurement) is the one Eq.1
assumes: a rank's step time is fixed work C plus GEMM time that scales
with the work it still computes; a slowed rank's GEMMs run chi times longer
(P:333); resizing or shedding adds a fixed overhead kappa (select, compaction,
copies); received units run at the receiver's speed.
"""
import random

import pytest

from oracle import ztp_oracle as O


class Model:
    """T_r = C + kappa [r resizes or sheds] + chi_r m (1 - shed_r) + m recv_r / u + noise_r,
    M_r = the GEMM part (chi_r m (1 - shed_r) + m recv_r / u).  shed_r is the rank's
    total shed fraction (gamma), recv_r the units it computes for others."""

    def __init__(self, e, u, m=1.0, C=0.4, kappa=0.02):
        self.e, self.u, self.m, self.C, self.kappa = e, u, m, C, kappa

    def run(self, plan, chis, noise):
        e, u, m = self.e, self.u, self.m
        recv = [0] * e
        shed = [0.0] * e
        for r in range(e):
            if plan.role[r] in (O.MIGRATE, O.SPLIT):
                shed[r] = plan.gamma[r]
                for (_, lo, hi) in O.plan_counts(plan, r, u, u, 1, True).out:
                    pass
            elif plan.role[r] == O.RESIZE:
                shed[r] = plan.gamma_r[r]
        for r in range(e):
            recv[r] = sum(hi - lo for (_, lo, hi) in O.plan_counts(plan, r, u, u, 1, True).inc)
        T, M = [], []
        for r in range(e):
            g = chis[r] * m * (1.0 - shed[r]) + m * recv[r] / u
            over = self.kappa if plan.role[r] != O.NORMAL else 0.0
            T.append(self.C + over + g + noise[r])
            M.append(g)
        return T, M


def _drive(model, ctl, opts, costs, chis_of_step, noise_of_step, steps):
    hist = []
    for k in range(steps):
        T, M = model.run(ctl.plan, chis_of_step(k), noise_of_step(k))
        act = ctl.step(T, M, opts, costs)
        hist.append((k, T, [x for x in ctl.plan.role], list(ctl.plan.gamma), act, ctl.state))
    return hist


FREE_MIG = O.Costs(0.0, ((0.0, 1.0), (0.0, 1.0)), ((0.0, 1.0), (0.0, 0.0)), ((0.0, 1.0), (0.0, 0.0)))


@pytest.mark.parametrize("seed", range(10))
def test_healthy_rank_at_2eps_stays_normal_through_refreshes_A43(seed):
    """A healthy rank whose runtime jitters up to T_min (1 + 2 eps) above the
    fastest rank is never resized by a refresh: A-43 refines the plan's
    stragglers only (Alg.2 resizes the z - x stragglers)."""
    rng = random.Random(seed)
    e, u, eps = 8, 1376, 0.02
    s = rng.randrange(e)
    mdl = Model(e, u, kappa=0.03)
    chis = [2.0 if r == s else 1.0 for r in range(e)]
    base = mdl.C + mdl.m
    # window noise below eps (so only the straggler is detected), then up to 2 eps
    noise0 = [0.0 if r == s else rng.uniform(0, 0.4 * eps) * base for r in range(e)]

    def noise(k):
        return noise0 if k == 0 else [0.0 if r == s else rng.uniform(0, 2 * eps) * base for r in range(e)]

    ctl = O.Controller(e)
    opts = O.CtlOpts(plan=O.PlanOpts(enable_migration=0, zero_crit=O.CRIT_MIN, eps=eps), L_ref=u, trigger=0.10,
                     max_refines=3)
    hist = _drive(mdl, ctl, opts, None, lambda k: chis, noise, 12)
    for (_, _, roles, gam, _, _) in hist:
        for r in range(e):
            if r != s:
                assert roles[r] == O.NORMAL and gam[r] == 0.0
    assert ctl.plan.role[s] == O.RESIZE and ctl.plan.gamma[s] > 0.0


def test_c4_tp8_chi2_zero_ends_with_ranks_0_to_6_unpruned():
    """c4 at TP = 8, rank 7 slowed 2x, ZERO-only with the
    T_min criterion and refreshes: ranks 0-6 end at gamma = 0 and the straggler
    lands within the overhead of T_min."""
    e, u, eps = 8, 1376, 0.02
    mdl = Model(e, u, kappa=0.03)
    chis = [1.0] * 7 + [2.0]
    rng = random.Random(3)
    ctl = O.Controller(e)
    opts = O.CtlOpts(plan=O.PlanOpts(enable_migration=0, zero_crit=O.CRIT_MIN, eps=eps), L_ref=u, trigger=0.10,
                     max_refines=3)
    _drive(mdl, ctl, opts, None, lambda k: chis,
           lambda k: [rng.uniform(0, 0.015) * (mdl.C + mdl.m) for _ in range(e)], 12)
    p = ctl.plan
    assert p.gamma[:7] == [0.0] * 7 and p.role[:7] == [O.NORMAL] * 7
    assert p.role[7] == O.RESIZE
    T, _ = mdl.run(p, chis, [0.0] * e)
    assert T[7] <= (mdl.C + mdl.m) * (1 + 2 * eps)          # within the dead band of T_min
    assert ctl.state == O.CTL_MONITOR


def test_c4_semi_chi3_helpers_stay_normal_A43():
    """c4 SEMI at TP = 8, rank 5 slowed 3x: gamma_MIN = 2/3 > gamma_tol, so the
    straggler migrates (free migration -> beta = 1); the seven helpers receive
    units, run longer than T_min, and must stay NORMAL (unpruned) through every
    refresh (A-43; P:233 loss-free migration)."""
    e, u = 8, 1376
    mdl = Model(e, u, kappa=0.03)
    chis = [1.0] * e
    chis[5] = 3.0
    ctl = O.Controller(e)
    opts = O.CtlOpts(plan=O.PlanOpts(enable_migration=1, zero_crit=O.CRIT_MIN, eps=0.02), L_ref=u, trigger=0.10,
                     max_refines=3)
    hist = _drive(mdl, ctl, opts, FREE_MIG, lambda k: chis, lambda k: [0.0] * e, 10)
    assert any(h[2][5] == O.MIGRATE for h in hist)
    for (_, _, roles, gam, _, _) in hist:
        for r in range(e):
            if r != 5:
                assert roles[r] == O.NORMAL and gam[r] == 0.0
    assert ctl.plan.role[5] == O.MIGRATE
    T, _ = mdl.run(ctl.plan, chis, [0.0] * e)
    T_free = mdl.C + mdl.m
    assert T_free / max(T) >= 0.85                        # north_star recovery, in this model


def test_controller_window_plan_refresh_monitor_sequence():
    """The state sequence of A-41: WINDOW -> (plan) FIRST -> (refresh) FIRST ->
    MONITOR; a >10% change lifts the plan to a window; when the
    slowdown vanishes the plan returns to gamma = 0 (temporariness)."""
    e, u = 4, 1024
    mdl = Model(e, u, kappa=0.05)
    ctl = O.Controller(e)
    opts = O.CtlOpts(plan=O.PlanOpts(enable_migration=0, zero_crit=O.CRIT_MIN, eps=0.02), L_ref=u, trigger=0.10,
                     max_refines=1)
    chis = [1.0, 1.0, 1.0, 2.0]
    assert ctl.state == O.CTL_WINDOW and ctl._dense(ctl.plan)
    T, M = mdl.run(ctl.plan, chis, [0.0] * e)
    assert ctl.step(T, M, opts) == O.CTL_APPLY                       # window -> plan
    assert ctl.state == O.CTL_FIRST and ctl.plan.gamma[3] == pytest.approx(0.5)
    T, M = mdl.run(ctl.plan, chis, [0.0] * e)                         # overshoot by kappa
    assert ctl.step(T, M, opts) == O.CTL_APPLY                       # one refresh (A-39)
    assert ctl.state == O.CTL_FIRST and ctl.plan.gamma[3] > 0.5 and ctl.refine_count == 1
    T, M = mdl.run(ctl.plan, chis, [0.0] * e)
    assert ctl.step(T, M, opts) == O.CTL_KEEP and ctl.state == O.CTL_MONITOR
    T, M = mdl.run(ctl.plan, chis, [0.0] * e)
    assert ctl.step(T, M, opts) == O.CTL_KEEP                        # steady: no trigger
    # the slowdown vanishes: rank 3 now runs faster by > 10% -> window (A-8)
    T, M = mdl.run(ctl.plan, [1.0] * e, [0.0] * e)
    assert ctl.step(T, M, opts) == O.CTL_APPLY and ctl.state == O.CTL_WINDOW and ctl._dense(ctl.plan)
    T, M = mdl.run(ctl.plan, [1.0] * e, [0.0] * e)
    assert ctl.step(T, M, opts) == O.CTL_KEEP and ctl._dense(ctl.plan)   # homogeneous: gamma = 0
    assert ctl.state == O.CTL_FIRST
    T, M = mdl.run(ctl.plan, [1.0] * e, [0.0] * e)
    ctl.step(T, M, opts)
    assert ctl.state == O.CTL_MONITOR and ctl.triggers == 1 and ctl.windows == 2


def test_controller_off_target_first_step_opens_window():
    """A-41: on the first step under a plan, a rank > 10% below the window's
    T_min (the straggler's slowdown vanished while the plan was applied) lifts
    the plan instead of refining it."""
    e, u = 2, 512
    mdl = Model(e, u, kappa=0.0)
    ctl = O.Controller(e)
    opts = O.CtlOpts(plan=O.PlanOpts(zero_crit=O.CRIT_MIN), L_ref=u)
    T, M = mdl.run(ctl.plan, [1.0, 3.0], [0.0, 0.0])
    ctl.step(T, M, opts)
    assert ctl.plan.role[1] == O.RESIZE
    T, M = mdl.run(ctl.plan, [1.0, 1.0], [0.0, 0.0])         # resized rank 1 without its slowdown
    assert ctl.step(T, M, opts) == O.CTL_APPLY and ctl.state == O.CTL_WINDOW and ctl._dense(ctl.plan)


def test_controller_errors():
    with pytest.raises(O.OracleError):
        O.Controller(0)
    ctl = O.Controller(2)
    with pytest.raises(O.OracleError):
        ctl.step([1.0, 0.0], [1.0, 1.0], O.CtlOpts())
    with pytest.raises(O.OracleError) as ei:                 # Eq.1 without a baseline
        ctl.step([1.0, 2.0], [1.0, 0.0], O.CtlOpts())
    assert ei.value.code == "ZTP_ENOBASELINE"


def test_refine_keeps_normal_ranks_normal_A43():
    """plan_refine: a NORMAL rank of prev is never resized by a refresh, a
    RESIZE rank inside the fresh dead band keeps its ratio exactly."""
    prev = O.plan([1.0, 1.0, 2.0], [0.5, 0.5, 1.5], 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_MIN))
    assert prev.role == [O.NORMAL, O.NORMAL, O.RESIZE]
    fresh = O.plan([1.3, 1.0, 1.01], [0.5, 0.5, 0.8], 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_MIN))
    assert fresh.role[0] == O.RESIZE and fresh.gamma_r[2] == 0.0
    out = O.plan_refine(prev, fresh)
    assert out.role == [O.NORMAL, O.NORMAL, O.RESIZE]
    assert out.gamma == [0.0, 0.0, prev.gamma[2]]
    assert out.z == prev.z

"""Pins of the oracle planner (Eq.1, Eq.2, Eq.3, Alg.2, renumbering) against
what the paper and the mathematics fix -- not against the oracle itself."""
import itertools
import math
import random

import numpy as np
import pytest

from conftest import golden
from oracle import ztp_oracle as O


def _costs_from(g, key):
    xs, ys = g[key]
    return (tuple(xs), tuple(ys))


def test_eq1_worked_example_S363():
    g = golden("eq1_worked.json")
    p = O.plan(g["T"], g["M"], 100.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_AVG))
    assert p.gamma == g["gamma"]                # exact: 5/16 is representable
    assert p.role == [O.NORMAL, O.RESIZE]


def test_c1_config_ratio_is_quarter():
    g = golden("c1_gamma.json")
    p = O.plan(g["T"], g["M"], 64.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_AVG))
    assert p.gamma == g["gamma"]


@pytest.mark.parametrize("seed", range(20))
def test_eq1_closed_form_uniform_synthetic(seed):
    """T_r = chi_r M + C with one straggler: gamma_AVG = (1-1/chi)(1-1/e),
    gamma_MIN = 1 - 1/chi (algebra of Eq.1)."""
    rng = random.Random(seed)
    e = rng.randint(2, 8)
    chi = rng.uniform(1.1, 2.5)
    M, C = rng.uniform(1, 100), rng.uniform(0, 50)
    s = rng.randrange(e)
    T = [M + C] * e
    Ms = [M] * e
    T[s] = chi * M + C
    Ms[s] = chi * M
    pa = O.plan(T, Ms, 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_AVG, gamma_max=1.0))
    pm = O.plan(T, Ms, 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_MIN, gamma_max=1.0))
    assert pa.gamma[s] == pytest.approx((1 - 1 / chi) * (1 - 1 / e), rel=1e-12)
    assert pm.gamma[s] == pytest.approx(1 - 1 / chi, rel=1e-12)
    for r in range(e):
        if r != s:
            assert pa.gamma[r] == 0.0 and pm.gamma[r] == 0.0


def test_eq1_clamp_and_errors():
    p = O.plan([1.0, 100.0], [1.0, 1.0], 1.0, O.Costs(), O.PlanOpts())
    assert p.gamma[1] == 0.9                     # A-4 clamp
    with pytest.raises(O.OracleError) as ei:
        O.plan([1.0, 2.0], [1.0, 0.0], 1.0, O.Costs(), O.PlanOpts())
    assert ei.value.code == "ZTP_ENOBASELINE"
    with pytest.raises(O.OracleError):
        O.plan([], [], 1.0, O.Costs(), O.PlanOpts())


def test_detection_tolerance_S562():
    p = O.plan([10.0, 10.1, 10.0, 10.0], [5.0] * 4, 1.0, O.Costs(),
               O.PlanOpts(enable_migration=1))
    assert p.z == 0 and all(r == O.NORMAL for r in p.role)
    p = O.plan([10.0, 20.0], [5.0, 10.0], 1.0, O.Costs(), O.PlanOpts(enable_migration=1))
    assert p.z == 1 and p.order[0] == 1


def test_zero_resizes_only_detected_stragglers_A38():
    """ZERO-only plans resize the ranks Alg.2 l.4 detects (T > T_min (1 + eps),
    A-17, A-38); eps = 0 gives Eq.1 literally for every rank."""
    T, M = [10.0, 10.1, 15.0], [5.0, 5.0, 10.0]
    p = O.plan(T, M, 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_MIN))
    assert p.gamma == [0.0, 0.0, 0.5] and p.role == [O.NORMAL, O.NORMAL, O.RESIZE] and p.z == 1
    p = O.plan(T, M, 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_MIN, eps=0.0))
    assert p.gamma[1] == pytest.approx(0.1 / 5.0, rel=1e-12) and p.gamma[2] == 0.5
    assert p.role == [O.NORMAL, O.RESIZE, O.RESIZE]
    # AVG criterion: the within-eps rank is below T_avg, so Eq.1 gives 0 anyway
    p = O.plan(T, M, 1.0, O.Costs(), O.PlanOpts(zero_crit=O.CRIT_AVG))
    T_avg = (10.0 + 10.1 + 15.0) / 3
    assert p.gamma[:2] == [0.0, 0.0] and p.gamma[2] == pytest.approx((15.0 - T_avg) / 10.0, rel=1e-12)


@pytest.mark.parametrize("seed", range(20))
def test_refine_reaches_Tmin_under_resize_overhead_A39(seed):
    """Eq.1 is exact for a rank whose GEMM time scales with the kept work
    (T = C + chi m (1 - gamma)), so a first plan lands on T_min.  With a fixed
    resize overhead kappa (select + compaction) the straggler overshoots by
    kappa; ONE refresh on the resized window (A-39 composition) brings its
    modelled runtime back to T_min exactly (algebra: keep = (1/chi)(1 - kappa/m))."""
    rng = random.Random(seed)
    e = rng.randint(2, 8)
    s = rng.randrange(e)
    m, C = rng.uniform(1, 10), rng.uniform(0, 5)
    chi = rng.uniform(1.5, 3.0)
    kappa = rng.uniform(0.05, 0.3) * m + 0.03 * (C + m)      # detectable (> eps T_min, A-17)
    chis = [chi if r == s else 1.0 for r in range(e)]

    def window(g):
        T = [C + (kappa if g[r] > 0 else 0.0) + chis[r] * m * (1 - g[r]) for r in range(e)]
        M = [chis[r] * m * (1 - g[r]) for r in range(e)]
        return T, M

    opts = O.PlanOpts(zero_crit=O.CRIT_MIN, gamma_max=1.0)
    p1 = O.plan(*window([0.0] * e), 1.0, O.Costs(), opts)
    assert p1.gamma[s] == pytest.approx(1 - 1 / chi, rel=1e-12)
    T1, _ = window(p1.gamma_r)
    assert T1[s] == pytest.approx(C + m + kappa, rel=1e-12)       # overshoot by the overhead
    p2 = O.plan_refine(p1, O.plan(*window(p1.gamma_r), 1.0, O.Costs(), opts), 1.0)
    T2, _ = window(p2.gamma_r)
    assert T2[s] == pytest.approx(C + m, rel=1e-12)                # = T_min
    assert [r for r in range(e) if p2.gamma[r] > 0] == [s]
    # a further refresh finds no straggler and changes nothing
    p3 = O.plan_refine(p2, O.plan(*window(p2.gamma_r), 1.0, O.Costs(), opts), 1.0)
    assert p3.gamma == p2.gamma


@pytest.mark.parametrize("seed", range(20))
def test_refine_semi_reaches_Tmin_A42(seed):
    """A-42: a migrating straggler whose remaining work (1 - gamma) runs at
    chi x (T = C + kappa + chi m (1 - gamma), kappa the fixed overhead of
    shedding) overshoots T_min by kappa under the first plan; ONE refresh
    composing its shed fraction lands it on T_min exactly, keeps beta, and the
    A-16 identity (1 - phi)(1 - gamma_r) = 1 - gamma holds for the new plan."""
    rng = random.Random(100 + seed)
    e = rng.randint(3, 8)
    s = rng.randrange(e)
    m, C = rng.uniform(1, 10), rng.uniform(0, 5)
    chi = rng.uniform(2.2, 4.0)                         # gamma > gamma_tol: SEMI migrates
    kappa = rng.uniform(0.05, 0.3) * m + 0.03 * (C + m)
    chis = [chi if r == s else 1.0 for r in range(e)]

    def window(gam):
        T = [C + (kappa if gam[r] > 0 else 0.0) + chis[r] * m * (1 - gam[r]) for r in range(e)]
        M = [chis[r] * m * (1 - gam[r]) for r in range(e)]
        return T, M

    lin = ((0.0, 1.0), (0.0, 0.0))
    costs = O.Costs(0.0, ((0.0, 1.0), (0.0, 1.0)), lin, lin)     # resizing costs, migration free: beta = 1
    p1 = O.plan(*window([0.0] * e), 1.0, costs, O.PlanOpts(enable_migration=1, zero_crit=O.CRIT_MIN, gamma_max=1.0))
    assert p1.role[s] == O.MIGRATE and p1.beta[s] == 1.0
    assert p1.gamma[s] == pytest.approx(1 - 1 / chi, rel=1e-12)
    zopts = O.PlanOpts(zero_crit=O.CRIT_MIN, gamma_max=1.0)
    T1, M1 = window(p1.gamma)
    assert T1[s] == pytest.approx(C + m + kappa, rel=1e-12)
    p2 = O.plan_refine(p1, O.plan(T1, M1, 1.0, O.Costs(), zopts), 1.0)
    T2, _ = window(p2.gamma)
    assert T2[s] == pytest.approx(C + m, rel=1e-12)
    assert p2.role[s] == O.MIGRATE and p2.beta[s] == 1.0 and p2.phi[s] == p2.gamma[s] and p2.gamma_r[s] == 0.0
    assert p2.x == p1.x and p2.order == p1.order
    # SPLIT: the A-16 identity for a fractional beta
    q = O.Plan(world=2, z=1, x=1, order=[1, 0], role=[O.NORMAL, O.SPLIT], gamma=[0.0, 0.6], beta=[0.0, 0.25],
               phi=[0.0, 0.15], gamma_r=[0.0, 0.6 * 0.75 / (1 - 0.15)])
    f = O.plan([1.0, 1.3], [1.0, 1.0], 1.0, O.Costs(), zopts)
    r2 = O.plan_refine(q, f, 1.0)
    assert r2.role[1] == O.SPLIT and r2.beta[1] == 0.25
    assert (1 - r2.phi[1]) * (1 - r2.gamma_r[1]) == pytest.approx(1 - r2.gamma[1], rel=1e-14)
    assert 1 - r2.gamma[1] == pytest.approx((1 - 0.6) * (1 - f.gamma_r[1]), rel=1e-14)


def test_eq2_worked_example_S572():
    g = golden("eq2_worked.json")
    c = O.Costs(g["omega1"], _costs_from(g, "omega2"), _costs_from(g, "phi1"), _costs_from(g, "phi2"))
    b = O.solve_beta(g["Lg"], c, g["e"], 64)
    assert abs(b - g["beta"]) <= g["tol"]
    # residual of Eq.2 at the solution
    lhs = c.omega1 + O.pwl_eval(c.omega2, g["Lg"] * (1 - b))
    rhs = O.pwl_eval(c.phi1, g["Lg"] * b) + O.pwl_eval(c.phi2, g["Lg"] * b / (g["e"] - 1))
    assert abs(lhs - rhs) <= 1e-6 * max(lhs, rhs)


def test_eq2_endpoints():
    zero = ((0.0, 1.0), (0.0, 0.0))
    lin = ((0.0, 1.0), (0.0, 1.0))
    # free migration -> beta = 1
    assert O.solve_beta(50.0, O.Costs(1.0, lin, zero, zero), 4, 64) == 1.0
    # free resizing, costly migration -> beta = 0
    assert O.solve_beta(50.0, O.Costs(0.0, zero, lin, lin), 4, 64) == 0.0


@pytest.mark.parametrize("seed", range(30))
def test_eq2_random_monotone_residual(seed):
    """For monotone piecewise-linear costs the bisection result brackets the
    root of LHS(b) - RHS(b) to 2^-64 (or is a valid endpoint)."""
    rng = random.Random(seed)

    def mono():
        xs = sorted({0.0} | {rng.uniform(1, 200) for _ in range(rng.randint(1, 4))})
        ys = [0.0]
        for _ in xs[1:]:
            ys.append(ys[-1] + rng.uniform(0, 5))
        return (tuple(xs), tuple(ys))
    c = O.Costs(rng.uniform(0, 3), mono(), mono(), mono())
    e = rng.randint(2, 8)
    Lg = rng.uniform(1, 300)
    b = O.solve_beta(Lg, c, e, 64)

    def gf(x):
        return (c.omega1 + O.pwl_eval(c.omega2, Lg * (1 - x))) - O.pwl_eval(c.phi1, Lg * x) \
            - O.pwl_eval(c.phi2, Lg * x / (e - 1))
    if b == 1.0:
        assert gf(1.0) >= 0
    elif b == 0.0:
        assert gf(0.0) <= 0
    else:
        assert gf(max(0.0, b - 1e-12)) >= -1e-9 and gf(min(1.0, b + 1e-12)) <= 1e-9


def test_eq3_worked_example_S582():
    g = golden("eq3_worked.json")
    c = O.Costs(0.0, ((0.0, 1.0), (0.0, 0.0)), _costs_from(g, "phi1"), ((0.0, 1.0), (0.0, 0.0)))
    T = g["T"]
    p = O.plan(T, [5.0] * 4, g["L"], c, O.PlanOpts(enable_migration=1, gamma_max=1.0))
    assert p.z == g["z"] and p.x == g["x"]
    assert p.role[0] == O.MIGRATE and p.role[1] == O.RESIZE
    assert p.role[2] == O.NORMAL and p.role[3] == O.NORMAL


def _f_bruteforce(T, x, L, phi1_per_col):
    """Eq.3 evaluated from scratch for one x with numpy (different code path)."""
    e = len(T)
    order = sorted(range(e), key=lambda r: (-T[r], r))
    Ts = np.array([T[r] for r in order])
    tmin = Ts.min()
    gam = float(np.sum(L * (Ts[:x] - tmin) / Ts[:x]))
    recv = np.max(gam / (e - x) * Ts[x:] / L)
    return (Ts[x - 1] - tmin) - phi1_per_col * gam - recv


@pytest.mark.parametrize("seed", range(100))
def test_eq3_bruteforce_random_S597(seed):
    rng = random.Random(1000 + seed)
    e = rng.randint(3, 8)
    T = [rng.choice([10.0, rng.uniform(10, 80)]) for _ in range(e)]
    T[rng.randrange(e)] = 10.0
    L = float(rng.choice([64, 100, 1024]))
    k = rng.uniform(0.0, 0.3)
    c = O.Costs(0.0, ((0.0, 1.0), (0.0, 0.0)), ((0.0, 1.0), (0.0, k)), ((0.0, 1.0), (0.0, 0.0)))
    p = O.plan(T, [4.0] * e, L, c, O.PlanOpts(enable_migration=1, eps=0.0, gamma_max=1.0))
    if p.z <= 1:
        return
    # brute force: x = length of the longest prefix with f > 0 (A-19)
    xb = 0
    for x in range(1, p.z + 1):
        if _f_bruteforce(T, x, L, k) > 0:
            xb = x
        else:
            break
    assert p.x == xb


def test_force_lambda_extremes_S592():
    T = [80.0, 10.0, 60.0, 10.0, 40.0, 10.0, 20.0, 10.0]     # chi = 8,6,4,2 on ranks 0,2,4,6
    M = [t - 5.0 for t in T]
    for lam, expect in ((0, [O.RESIZE] * 4), (4, [O.MIGRATE] * 4)):
        p = O.plan(T, M, 100.0, O.Costs(), O.PlanOpts(enable_migration=1, force_lambda=lam))
        assert [p.role[r] for r in (0, 2, 4, 6)] == expect


def test_renumbering_P267():
    g = golden("renumber.json")
    p = O.Plan(world=g["e"], order=[0, 1, 2], role=[O.MIGRATE, O.NORMAL, O.NORMAL],
               gamma=[0.5, 0, 0], beta=[1.0, 0, 0], phi=[0.5, 0, 0], gamma_r=[0.0, 0, 0])
    for r in (1, 2):
        c = O.plan_counts(p, r, 8, g["n_units"], 1, False)
        assert c.inc == [(0, *g["ranges"][str(r)])]
    c0 = O.plan_counts(p, 0, 8, g["n_units"], 1, False)
    assert c0.n_mig == g["n_mig"]
    # e=4, L_mig=5 -> (2,2,1) by virtual rank
    e, s = g["e2"], g["straggler2"]
    role = [O.NORMAL] * e
    role[s] = O.MIGRATE
    phi = [0.0] * e
    phi[s] = 0.5
    p = O.Plan(world=e, order=[s] + [r for r in range(e) if r != s], role=role,
               gamma=phi[:], beta=[1.0 if r == s else 0 for r in range(e)], phi=phi, gamma_r=[0.0] * e)
    loads = {}
    for r in range(e):
        for (src, lo, hi) in O.plan_counts(p, r, 16, g["n_units2"], 1, False).inc:
            loads[(r - s + e) % e] = hi - lo
    assert [loads[v] for v in (1, 2, 3)] == g["loads2_by_vrank"]


@pytest.mark.parametrize("e,s", [(e, s) for e in (2, 3, 4, 8) for s in range(e)])
def test_renumbering_bijection_and_partition(e, s):
    vr = [(r - s + e) % e for r in range(e)]
    assert sorted(vr) == list(range(e)) and vr[s] == 0
    role = [O.NORMAL] * e
    role[s] = O.MIGRATE
    phi = [0.0] * e
    phi[s] = 0.7
    p = O.Plan(world=e, order=[s] + [r for r in range(e) if r != s], role=role, gamma=phi[:],
               beta=[1.0 if r == s else 0 for r in range(e)], phi=phi, gamma_r=[0.0] * e)
    n_units, unit = 64, 4
    got = []
    for r in range(e):
        got += [(lo, hi) for (_, lo, hi) in O.plan_counts(p, r, 64, n_units, unit, True).inc]
    nm = O.plan_counts(p, s, 64, n_units, unit, True).n_mig
    cover = sorted(got)
    assert cover[0][0] == n_units - nm and cover[-1][1] == n_units
    for (a, b), (c, d) in zip(cover, cover[1:]):
        assert b == c                              # disjoint and contiguous
    assert all((hi - lo) % unit == 0 for lo, hi in got)


def test_counts_prune_rounding_and_floor():
    p = O.Plan(world=2, order=[1, 0], role=[O.NORMAL, O.RESIZE], gamma=[0, 0.25],
               beta=[0, 0], phi=[0, 0], gamma_r=[0.0, 0.25])
    assert O.plan_counts(p, 1, 64, 128, 1, False).n_prune == 16      # c1: FC1 16/64
    assert O.plan_counts(p, 1, 128, 128, 1, True).n_prune == 32      # c1: FC2 32/128
    assert O.plan_counts(p, 0, 64, 128, 1, False).n_prune == 0
    p.gamma_r[1] = 0.9999
    assert O.plan_counts(p, 1, 10, 10, 1, False).n_prune == 9        # >= 1 column survives (A-4)


def test_split_gamma_r_identity_A16():
    """gamma_r = gamma(1-beta)/(1-gamma beta): remaining work (1-phi)(1-gamma_r) = 1-gamma."""
    for g, b in itertools.product((0.55, 0.7, 0.9), (0.0, 0.3, 0.6, 1.0)):
        gr = (g * (1 - b)) / (1 - g * b)
        assert (1 - g * b) * (1 - gr) == pytest.approx(1 - g, abs=1e-15)


def test_semi_single_heavy_straggler_split():
    """z=1, gamma above gamma_tol: beta >= 1 - gamma_tol/gamma and role SPLIT/MIGRATE (A-23)."""
    T = [10.0] * 8
    M = [8.0] * 8
    T[5] = 26.0                 # chi=3 on GEMM time 8 -> gamma_MIN = 16/24 = 2/3
    M[5] = 24.0
    p = O.plan(T, M, 100.0, O.Costs(), O.PlanOpts(enable_migration=1))
    g = p.gamma[5]
    assert g == pytest.approx(2.0 / 3.0)
    assert p.beta[5] >= 1 - 0.5 / g - 1e-15
    assert p.role[5] in (O.SPLIT, O.MIGRATE)
    assert (1 - p.phi[5]) * (1 - p.gamma_r[5]) == pytest.approx(1 - g)


def test_pwl_eval_interpolation_S552():
    fn = ((0.0, 2.0, 4.0), (0.0, 1.0, 5.0))
    assert O.pwl_eval(fn, 2.0) == 1.0          # sample point returns its value exactly
    assert O.pwl_eval(fn, 1.0) == 0.5          # interpolation
    assert O.pwl_eval(fn, 3.0) == 3.0
    assert O.pwl_eval(fn, 6.0) == 9.0          # extrapolation of the last segment
    with pytest.raises(O.OracleError):
        O.pwl_eval(((0.0,), (0.0,)), 1.0)


def test_receivers_are_normal_tasks_A44():
    """A-44 ("evenly distributed across other normal tasks", P:233
    loss-free migration): in a multi-straggler plan (Eq.3 x migrators, z - x
    resizers) the migrated units go to NORMAL tasks only, which prune
    nothing; resize-group stragglers receive nothing."""
    e = 8
    T = [1.0, 8.0, 1.0, 6.0, 1.0, 4.0, 1.0, 2.0]     # c5 phase 3: ranks 1,3,5,7 x8,6,4,2
    M = [0.8 * t for t in T]
    costs = O.Costs(phi1=((0.0, 1.0), (0.0, 1e-4)))
    p = O.plan(T, M, 100.0, costs, O.PlanOpts(enable_migration=1, zero_crit=O.CRIT_MIN))
    assert p.x >= 1 and p.z == 4
    resizers = [r for r in range(e) if p.role[r] == O.RESIZE]
    normals = [r for r in range(e) if p.role[r] == O.NORMAL]
    assert normals == [0, 2, 4, 6]
    got = {r: O.plan_counts(p, r, 100, 100, 1, True) for r in range(e)}
    received = {r: sum(hi - lo for (_, lo, hi) in got[r].inc) for r in range(e)}
    sent = sum(got[r].n_mig for r in range(e))
    assert sum(received.values()) == sent > 0
    assert all(received[r] == 0 for r in resizers) and all(received[r] > 0 for r in normals)
    assert all(got[r].n_prune == 0 for r in normals)


def test_resize_only_when_it_pays_A48():
    """A-48: a rank just above the detection tolerance (timing noise) has an
    Eq.1 saving gamma M below the static resizing overhead Omega_1
    and stays NORMAL; the real straggler resizes as before; Omega_1 = 0 is
    the unfiltered plan."""
    T = [1.0, 1.06, 2.0]
    M = [0.8 * t for t in T]
    opts = O.PlanOpts(enable_migration=0, zero_crit=O.CRIT_MIN, eps=0.05)
    p0 = O.plan(T, M, 100.0, O.Costs(omega1=0.0), opts)
    assert p0.role[1] == O.RESIZE and p0.gamma_r[1] * M[1] == pytest.approx(0.06)
    p1 = O.plan(T, M, 100.0, O.Costs(omega1=0.1), opts)
    assert p1.role == [O.NORMAL, O.NORMAL, O.RESIZE] and p1.gamma[1] == 0.0
    assert p1.gamma[2] == p0.gamma[2] == pytest.approx(1.0 / 1.6)
    # SEMI multi-straggler: the noise rank drops out of the resize group, and
    # becomes a receiver (A-44)
    T = [1.0, 1.06, 1.0, 6.0, 1.0, 4.0, 1.0, 1.0]
    M = [0.8 * t for t in T]
    costs = O.Costs(omega1=0.1, phi1=((0.0, 1.0), (0.0, 1e-4)))
    p = O.plan(T, M, 100.0, costs, O.PlanOpts(enable_migration=1, zero_crit=O.CRIT_MIN, eps=0.05))
    assert p.role[1] == O.NORMAL and p.role[3] in (O.MIGRATE, O.SPLIT)
    got = {r: O.plan_counts(p, r, 100, 100, 1, True) for r in range(8)}
    assert sum(hi - lo for (_, lo, hi) in got[1].inc) > 0 or p.x == 0

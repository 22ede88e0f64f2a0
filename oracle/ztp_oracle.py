"""fp64 CPU oracle for the straggler-balanced 1D-TP layer (arXiv 2401.11469).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this module.
The product path (`paper_2401_11469_b200`) never imports it and shares no code
with it; the only shared module is `synth/` (seeded inputs, no arithmetic of
the method).

Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
Alg.1 l.k = P:202+k; Alg.2 l.k = P:293+k.  Readings of ambiguous passages are
numbered A-n as in SURVEY.md §8(c) and listed in DESIGN.md.

Layout: every tensor the method prunes along its contraction
dimension is stored feature-major, i.e. transposed w.r.t. the paper:
    Xt [K, N]  (paper's input  [bs*sql, K]),  Wt [K, n] (paper's weight [n, K]),
    Yt [n, N], Gt [n, N] (paper's grad_input, the upstream gradient),
    dXt [K, N] (paper's grad_output),  dWt [K, n] (paper's grad_weight^T).
Pruning a paper *column* k of input and weight = dropping *row* k here.

Parity status of every function is in its docstring; all are pinned by
tests/test_oracle_*.py except `pretest` costs (measured, "parity unpinned").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# status codes (mirror the names of include/ztp.h; values are the oracle's own)
# ----------------------------------------------------------------------------


class OracleError(Exception):
    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


# ----------------------------------------------------------------------------
# activation (GeLU via the tanh approximation with its exact derivative)
# ----------------------------------------------------------------------------

_C = math.sqrt(2.0 / math.pi)


def gelu_tanh(x):
    """GeLU(x) = 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + np.tanh(_C * (x + 0.044715 * x ** 3)))


def gelu_tanh_grad(x):
    """d/dx of gelu_tanh, differentiated analytically."""
    x = np.asarray(x, dtype=np.float64)
    u = _C * (x + 0.044715 * x ** 3)
    t = np.tanh(u)
    du = _C * (1.0 + 3.0 * 0.044715 * x ** 2)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * du


# ----------------------------------------------------------------------------
# a2. Plan: Eq.1, straggler detection, Eq.2, Eq.3, Alg.2, renumbering
# ----------------------------------------------------------------------------

NORMAL, RESIZE, MIGRATE, SPLIT = 0, 1, 2, 3
CRIT_AVG, CRIT_MIN = 0, 1


@dataclass
class Costs:
    """Eq.2/Eq.3 cost model: Omega1 constant, Omega2/Phi1/Phi2 piecewise
    linear through sampled points (A-24)."""
    omega1: float = 0.0
    omega2: tuple = ((0.0, 1.0), (0.0, 0.0))   # (xs, ys)
    phi1: tuple = ((0.0, 1.0), (0.0, 0.0))
    phi2: tuple = ((0.0, 1.0), (0.0, 0.0))


@dataclass
class PlanOpts:
    enable_migration: int = 0
    zero_crit: int = CRIT_MIN       # A-7: headline uses T_min; AVG = Eq.1 literal
    gamma_max: float = 0.9          # A-4
    eps: float = 0.02               # A-17
    gamma_tol: float = 0.5          # A-23
    bisect_iters: int = 64          # A-24
    force_lambda: int = -1          # NEXT-4 forced lambda; -1 = Eq.3


@dataclass
class Plan:
    world: int
    z: int = 0
    x: int = 0
    order: list = field(default_factory=list)
    role: list = field(default_factory=list)
    gamma: list = field(default_factory=list)
    beta: list = field(default_factory=list)
    phi: list = field(default_factory=list)
    gamma_r: list = field(default_factory=list)


def pwl_eval(fn, x: float) -> float:
    """Piecewise-linear cost function through points (xs, ys), xs ascending,
    linear extrapolation beyond both ends.  Segment j satisfies
    xs[j] <= x < xs[j+1]; the last segment extrapolates."""
    xs, ys = fn
    n = len(xs)
    if n < 2:
        raise OracleError("ZTP_EINVAL", "cost function needs >= 2 samples (S:549)")
    j = 0
    while j + 2 < n and x >= xs[j + 1]:
        j += 1
    return ys[j] + (ys[j + 1] - ys[j]) * ((x - xs[j]) / (xs[j + 1] - xs[j]))


def eq1_gamma(T_r: float, C: float, M_r: float, gamma_max: float) -> float:
    """Eq.1: gamma = (T_i - C) / M_i, C = T_avg (Eq.1) or T_min
    (P:284); clamped to [0, gamma_max] (A-4)."""
    if not (M_r > 0.0):
        raise OracleError("ZTP_ENOBASELINE", "M_i = 0 (S:360)")
    g = (T_r - C) / M_r
    if g < 0.0:
        g = 0.0
    if g > gamma_max:
        g = gamma_max
    return g


def plan_refine(prev: Plan, fresh: Plan, gamma_max: float = 0.9) -> Plan:
    """Statistics refresh of a plan ("over-10% increase ... update on
    demand", A-8; readings A-39, A-42).  `fresh` is Eq.1 (ZERO-only) on a
    window measured with `prev` in effect, so its ratio is a fraction of the
    work the rank still computes (the savings offset the remaining gap
    T_i - T_avg): kept fractions multiply, 1 - gamma = (1 - gamma_prev)
    (1 - gamma_fresh), clamped to gamma_max (A-4).
    A-42: a rank that sheds work by migration (MIGRATE / SPLIT) composes its
    whole shed fraction gamma the same way and keeps its Eq.2 split beta:
    phi = gamma beta, gamma_r = gamma (1 - beta) / (1 - gamma beta) (A-16);
    the plan keeps prev's migration group (x) and sender order.
    A-43: only prev's stragglers are refined.  A NORMAL task of prev stays
    NORMAL with gamma 0 whatever the fresh window says: Alg.2 resizes only the
    z - x stragglers, and a receiver's extra runtime is received work
    that migration makes loss-free.  The fresh plan's tolerance eps is
    the dead band (a straggler within T_min (1 + eps) gets fresh gamma 0)."""
    if prev.world != fresh.world:
        raise OracleError("ZTP_EINVAL", "world mismatch")
    e = fresh.world
    if any(x in (MIGRATE, SPLIT) for x in list(fresh.role[:e])):
        raise OracleError("ZTP_EUNSUPPORTED", "the refresh plan must be ZERO-only (A-39, A-42)")
    semi = any(x in (MIGRATE, SPLIT) for x in list(prev.role[:e]))
    out = Plan(world=e, z=prev.z, x=prev.x if semi else 0, order=list(prev.order if semi else fresh.order),
               role=[NORMAL] * e, gamma=[0.0] * e, beta=[0.0] * e, phi=[0.0] * e, gamma_r=[0.0] * e)
    for r in range(e):
        if prev.role[r] == NORMAL:
            continue                                   # A-43: stays NORMAL, gamma 0
        sheds = prev.role[r] in (MIGRATE, SPLIT)
        keep = (1.0 - (prev.gamma[r] if sheds else prev.gamma_r[r])) * (1.0 - fresh.gamma_r[r])
        g = 1.0 - keep
        if g > gamma_max:
            g = gamma_max
        if g < 0.0:
            g = 0.0
        out.gamma[r] = g
        if sheds:
            b = prev.beta[r]
            out.beta[r] = b
            out.phi[r] = g * b
            out.gamma_r[r] = 0.0 if b >= 1.0 else (g * (1.0 - b)) / (1.0 - g * b)
            out.role[r] = prev.role[r]
        else:
            out.gamma_r[r] = g
            out.role[r] = RESIZE if g > 0.0 else NORMAL
    return out


def solve_beta(Lg: float, costs: Costs, e: int, iters: int) -> float:
    """Eq.2: Omega1 + Omega2(L g (1-b)) = Phi1(L g b) + Phi2(L g b/(e-1)).
    g(b) = LHS - RHS is non-increasing; bisection with a fixed iteration count
    (A-24); endpoints per S:568."""
    def gfun(b):
        return ((costs.omega1 + pwl_eval(costs.omega2, Lg * (1.0 - b)))
                - pwl_eval(costs.phi1, Lg * b)) - pwl_eval(costs.phi2, (Lg * b) / float(e - 1))
    if gfun(1.0) >= 0.0:
        return 1.0
    if gfun(0.0) <= 0.0:
        return 0.0
    lo, hi = 0.0, 1.0
    for _ in range(iters):
        m = 0.5 * (lo + hi)
        if gfun(m) > 0.0:
            lo = m
        else:
            hi = m
    return 0.5 * (lo + hi)


def eq3_scan(T: list, order: list, z: int, T_min: float, L: float, costs: Costs) -> int:
    """Eq.3: Gamma(x) = sum_{k<=x} L (T_(k) - T_min)/T_(k);
    f(x) = (T_(x) - T_min) - Phi1(Gamma(x)) - max_{y in [x+1, e]} Gamma(x)/(e-x) * T_(y)/L.
    Scan x = 1..z, stop at the first f(x) <= 0 (A-19): x = that - 1; x = z if none."""
    e = len(T)
    gam = 0.0
    for xi in range(1, z + 1):
        Tk = T[order[xi - 1]]
        gam = gam + L * ((Tk - T_min) / Tk)
        if e - xi <= 0:
            raise OracleError("ZTP_ERECEIVERS", "e - x = 0 (S:579)")
        mx = -math.inf
        for y in range(xi + 1, e + 1):
            v = (gam / float(e - xi)) * (T[order[y - 1]] / L)
            if v > mx:
                mx = v
        f = ((Tk - T_min) - pwl_eval(costs.phi1, gam)) - mx
        if f <= 0.0:
            return xi - 1
    return z


def plan(T, M, L_ref: float, costs: Costs, opts: PlanOpts) -> Plan:
    """Alg.2 (below, plan_core) followed by reading A-48: a RESIZE rank whose
    Eq.1 saving gamma_r M does not exceed the static resizing overhead
    Omega_1 stays NORMAL with gamma 0.  No costs / Omega_1 = 0:
    unchanged."""
    p = plan_core(T, M, L_ref, costs, opts)
    if costs is not None and costs.omega1 > 0.0:
        for r in range(p.world):
            if p.role[r] == RESIZE and p.gamma_r[r] * M[r] <= costs.omega1:
                p.role[r] = NORMAL
                p.gamma[r] = 0.0
                p.gamma_r[r] = 0.0
    return p


def plan_core(T, M, L_ref: float, costs: Costs, opts: PlanOpts) -> Plan:
    """Alg.1 l.1-2 (ZERO-only) and Alg.2 (SEMI).

    Evaluation order is fixed (fp64, no FMA) so the GPU host planner must
    reproduce every double bit-exactly."""
    e = len(T)
    if e < 1 or e > 8 or len(M) != e:
        raise OracleError("ZTP_EINVAL", "world must be 1..8 and len(M) == len(T) (S:559)")
    for t in T:
        if not (math.isfinite(t) and t >= 0.0):
            raise OracleError("ZTP_EINVAL", "T must be finite and >= 0")
    p = Plan(world=e, order=sorted(range(e), key=lambda r: (-T[r], r)),
             role=[NORMAL] * e, gamma=[0.0] * e, beta=[0.0] * e, phi=[0.0] * e,
             gamma_r=[0.0] * e)
    acc = 0.0
    for r in range(e):                       # Alg.1 l.1: T_avg = all-reduce(T)/e
        acc = acc + T[r]
    T_avg = acc / float(e)
    T_min = T[0]
    for r in range(1, e):                    # Alg.2 l.3
        if T[r] < T_min:
            T_min = T[r]
    thr = T_min * (1.0 + opts.eps)           # Alg.2 l.4 with tolerance (A-17)
    stragglers = [r for r in p.order if T[r] > thr]
    p.z = len(stragglers)
    if not opts.enable_migration:
        # ZERO-resizing only (Alg.1 l.1-2): the detected stragglers (Alg.2
        # l.4 with tolerance eps, A-17) with gamma > 0 resize; a rank within
        # eps of T_min keeps its full shard (A-38).  eps = 0 is paper-literal:
        # the only excluded ranks sit at T_min, where Eq.1 gives 0 anyway.
        C = T_avg if opts.zero_crit == CRIT_AVG else T_min
        for r in range(e):
            g = eq1_gamma(T[r], C, M[r], opts.gamma_max)      # (raises on M_i = 0 for every rank)
            if not T[r] > thr:
                g = 0.0
            p.gamma[r] = g
            p.gamma_r[r] = g
            p.role[r] = RESIZE if g > 0.0 else NORMAL
        return p
    # SEMI (Alg.2): criterion T_min
    for r in stragglers:
        p.gamma[r] = eq1_gamma(T[r], T_min, M[r], opts.gamma_max)
    if p.z == 0:
        return p
    if p.z == 1:                              # Alg.2 l.7-12, A-15, A-16, A-23
        s = stragglers[0]
        g = p.gamma[s]
        if g <= opts.gamma_tol:
            p.role[s] = RESIZE if g > 0.0 else NORMAL
            p.gamma_r[s] = g
            return p
        b = solve_beta(L_ref * g, costs, e, opts.bisect_iters)
        floor_b = 1.0 - opts.gamma_tol / g
        if b < floor_b:
            b = floor_b
        p.beta[s] = b
        p.phi[s] = g * b
        p.gamma_r[s] = (g * (1.0 - b)) / (1.0 - g * b)
        p.role[s] = MIGRATE if b == 1.0 else (RESIZE if b == 0.0 else SPLIT)
        p.x = 1 if b > 0.0 else 0
        return p
    # several stragglers: Eq.3 scan (Alg.2 l.14-24, A-19..A-22)
    if opts.force_lambda >= 0:
        x = min(opts.force_lambda, p.z)
    else:
        x = eq3_scan(T, p.order, p.z, T_min, L_ref, costs)
    p.x = x
    for pos, r in enumerate(stragglers, start=1):
        if pos <= x:
            p.role[r] = MIGRATE
            p.beta[r] = 1.0
            p.phi[r] = p.gamma[r]
            p.gamma_r[r] = 0.0
        else:
            p.role[r] = RESIZE
            p.gamma_r[r] = p.gamma[r]
    return p


CTL_WINDOW, CTL_FIRST, CTL_MONITOR = 0, 1, 2
CTL_KEEP, CTL_APPLY = 0, 1


def dense_plan(e: int) -> Plan:
    return Plan(world=e, order=list(range(e)), role=[NORMAL] * e, gamma=[0.0] * e, beta=[0.0] * e,
                phi=[0.0] * e, gamma_r=[0.0] * e)


@dataclass
class CtlOpts:
    plan: PlanOpts = field(default_factory=PlanOpts)
    L_ref: float = 1.0
    trigger: float = 0.10          # P:178 "over-10% increase"
    max_refines: int = 1


class Controller:
    """The statistics-driven re-planning loop (Alg.2 l.2; reading
    A-41), written as the three-state machine it is:

    WINDOW   the step ran un-resized: plan = Alg.1/Alg.2 on its T, M (Eq.1 and
             Alg.2 are defined on un-resized runtimes); remember the window's
             T_min (the plan's target) and T_max.
    FIRST    first step under the plan.  Off target -- some rank below
             (1 - trigger) T_min or above (1 + trigger) T_max of the window: the
             slowdowns changed while the plan was applied -- lift it (WINDOW).
             Otherwise refresh it once (plan_refine on a ZERO-only T_min plan of
             this step, A-39/A-42/A-43); if the plan changed judge its first step
             again, else this step is the monitoring reference.
    MONITOR  a relative runtime change > trigger of any rank against the
             reference, in either direction (A-8), lifts the plan.

    step() returns CTL_APPLY when the plan for the next step changed."""

    def __init__(self, world: int):
        if not 1 <= world <= 8:
            raise OracleError("ZTP_EINVAL", "world outside 1..8")
        self.world = world
        self.state = CTL_WINDOW
        self.refines = 0
        self.plan = dense_plan(world)
        self.T_ref = [0.0] * world
        self.T_target = 0.0
        self.T_wmax = 0.0
        self.steps = self.windows = self.replans = self.refine_count = self.triggers = 0

    @staticmethod
    def _dense(p: Plan) -> bool:
        return all(x == NORMAL for x in p.role[:p.world])

    @staticmethod
    def _same(a: Plan, b: Plan) -> bool:
        e = a.world
        return (a.x == b.x and a.role[:e] == b.role[:e] and a.gamma[:e] == b.gamma[:e]
                and a.gamma_r[:e] == b.gamma_r[:e] and a.beta[:e] == b.beta[:e] and a.phi[:e] == b.phi[:e])

    def step(self, T, M, opts: CtlOpts, costs: Costs = None) -> int:
        e = self.world
        for t in T[:e]:
            if not (math.isfinite(t) and t > 0.0):
                raise OracleError("ZTP_EINVAL", "T must be finite and > 0")
        trig = opts.trigger
        self.steps += 1
        Tmin = min(T[:e])
        Tmax = max(T[:e])
        action = CTL_KEEP

        def lift():
            nonlocal action
            if not self._dense(self.plan):
                action = CTL_APPLY
            self.plan = dense_plan(e)
            self.state = CTL_WINDOW

        if self.state == CTL_WINDOW:
            p = plan(list(T[:e]), list(M[:e]), opts.L_ref, costs if costs is not None else Costs(), opts.plan)
            self.windows += 1
            if not self._dense(p):
                self.plan = p
                self.replans += 1
                action = CTL_APPLY
            self.T_target, self.T_wmax = Tmin, Tmax
            self.refines = 0
            self.state = CTL_FIRST
            return action
        if self.state == CTL_FIRST:
            if not self._dense(self.plan) and (Tmin < (1.0 - trig) * self.T_target or
                                               Tmax > (1.0 + trig) * self.T_wmax):
                lift()
                return action
            if not self._dense(self.plan) and self.refines < opts.max_refines:
                zo = PlanOpts(enable_migration=0, zero_crit=CRIT_MIN, gamma_max=opts.plan.gamma_max,
                              eps=opts.plan.eps, gamma_tol=opts.plan.gamma_tol, bisect_iters=opts.plan.bisect_iters,
                              force_lambda=opts.plan.force_lambda)
                fresh = plan(list(T[:e]), list(M[:e]), opts.L_ref, Costs(), zo)
                ref = plan_refine(self.plan, fresh, opts.plan.gamma_max)
                self.refines += 1
                if not self._same(ref, self.plan):
                    self.plan = ref
                    self.refine_count += 1
                    return CTL_APPLY
            self.T_ref = list(T[:e])
            self.state = CTL_MONITOR
            return action
        for r in range(e):
            if abs(T[r] - self.T_ref[r]) / self.T_ref[r] > trig:
                self.triggers += 1
                lift()
                return action
        return action


@dataclass
class Counts:
    n_prune: int = 0
    n_mig: int = 0
    out: list = field(default_factory=list)   # (dst, lo, hi): my units [lo, hi) computed by dst
    inc: list = field(default_factory=list)   # (src, lo, hi): src's units [lo, hi) computed by me


def plan_counts(p: Plan, rank: int, K: int, n_units: int, unit: int, is_row: bool) -> Counts:
    """Integer realisation of a plan for one linear of `rank`:
    n_mig = unit * floor((n_units/unit) * phi + 0.5); gamma_r = gamma(1-beta)/(1-gamma beta)
    (A-16); n_prune = floor(K_rem gamma_r + 0.5) (A-3) clamped so >= 1 survives (A-4);
    K_rem = K (column layer) or K - n_mig (row layer).  Helper ranges follow the
    virtual renumbering r' = (r + e - r_k) % e, remainder to the lowest r'
    (A-28), contiguous inside the tail J = [n_units - n_mig, n_units) (A-27)."""
    e = p.world
    if unit <= 0 or n_units % unit != 0 or K < 1:
        raise OracleError("ZTP_EINVAL", "bad unit / sizes")
    units = n_units // unit

    def nmig(s):
        if p.role[s] not in (MIGRATE, SPLIT):
            return 0
        nm = unit * int(math.floor(float(units) * p.phi[s] + 0.5))
        if nm > n_units - unit:
            nm = n_units - unit
        return nm

    c = Counts()
    c.n_mig = nmig(rank)
    K_rem = K - c.n_mig if is_row else K
    npr = int(math.floor(float(K_rem) * p.gamma_r[rank] + 0.5))
    if npr > K_rem - 1:
        npr = K_rem - 1
    if npr < 0:
        npr = 0
    c.n_prune = npr
    # receivers: the NORMAL tasks ("evenly distributed across other
    # normal tasks"; reading A-44) -- never resized, so migration stays
    # loss-free
    receivers = [r for r in range(e) if p.role[r] == NORMAL]
    for s in p.order:
        nm = nmig(s)
        if nm == 0:
            continue
        if not receivers:
            raise OracleError("ZTP_ERECEIVERS", "no receivers")
        R = sorted(receivers, key=lambda r: (r - s + e) % e)
        tot = nm // unit
        m, extra = tot // len(R), tot % len(R)
        lo = n_units - nm
        for i, r in enumerate(R):
            cnt = (m + (1 if i < extra else 0)) * unit
            if cnt > 0:
                if rank == s:
                    c.out.append((r, lo, lo + cnt))
                if rank == r:
                    c.inc.append((s, lo, lo + cnt))
            lo += cnt
    return c


def layer_prune_counts(p: Plan, rank: int, h: int, a: int, u: int) -> dict:
    """The four prune counts of one layer (SURVEY §8(a) layer): MLP by
    plan_counts (FC1 col over K = h, FC2 row over K_rem = u - n_mig).
    Attention, reading A-37: heads never migrate (A-26), so a rank that sheds
    MLP units (MIGRATE / SPLIT) keeps (1 - gamma) of its attention work by
    resizing QKV (K = h) and O (K = a) with its Eq.1 gamma; other ranks use
    gamma_r, as for FC1."""
    g_att = p.gamma[rank] if p.role[rank] in (MIGRATE, SPLIT) else p.gamma_r[rank]

    def att(K):
        n = int(math.floor(float(K) * g_att + 0.5))
        return max(0, min(n, K - 1))
    return {"qkv": att(h), "o": att(a),
            "fc1": plan_counts(p, rank, h, u, 1, False).n_prune,
            "fc2": plan_counts(p, rank, u, u, 1, True).n_prune}


def plan_uniform(e: int, gamma: float) -> Plan:
    """Homogeneous resizing (E2): every rank RESIZE with gamma."""
    if not (0.0 <= gamma < 1.0):
        raise OracleError("ZTP_EINVAL", "gamma outside [0, 1)")
    return Plan(world=e, order=list(range(e)), role=[RESIZE if gamma > 0 else NORMAL] * e, gamma=[gamma] * e,
                beta=[0.0] * e, phi=[0.0] * e, gamma_r=[gamma] * e)


def pridiff_counts(L: int, L_uni: int, gamma_t: float, alpha: float = 0.8, gamma_max: float = 0.9) -> int:
    """Alg.1 l.10-11 ratio max(1 - L_uni/L, alpha gamma_t), clamped to
    [0, gamma_max] (A-4), as a prune count floor(L g + 0.5) <= L - 1 (A-3)."""
    if L < 1:
        return 0
    g = max(1.0 - L_uni / L, alpha * gamma_t)
    g = min(max(g, 0.0), gamma_max)
    return min(int(math.floor(L * g + 0.5)), L - 1)


def costs_fit(omega, phi1, phi2):
    """Alg.2 l.1 pretest samples -> Costs (reading A-40).  Omega_1 is the extra
    cost at the smallest pruned count n > 0 ("static space allocation
    overhead"), clamped at 0; Omega_2(n) = extra(n) - Omega_1 (P:258
    "proportionally increased dimension extracting cost").  Every function
    passes through (0, 0) and is non-decreasing: samples with x <= 0 or an x
    already seen are dropped, y is the running maximum clamped at 0; a
    function without samples is the zero line (0,0)-(1,0)."""
    def mono(pts):
        xs, ys = [0.0], [0.0]
        for x, y in sorted((float(a), float(b)) for a, b in pts):
            if x > xs[-1]:
                xs.append(x)
                ys.append(max(ys[-1], y, 0.0))
        if len(xs) < 2:
            xs.append(1.0)
            ys.append(0.0)
        return (tuple(xs), tuple(ys))
    for pts in (omega, phi1, phi2):
        for x, y in pts:
            if not (math.isfinite(x) and math.isfinite(y)):
                raise OracleError("ZTP_EINVAL", "non-finite sample")
    pos = sorted(((float(x), float(y)) for x, y in omega if x > 0), key=lambda t: t[0])
    om1 = max(pos[0][1], 0.0) if pos else 0.0
    return Costs(om1, mono([(x, y - om1) for x, y in pos]), mono(phi1), mono(phi2))


# ----------------------------------------------------------------------------
# a3. Priority select (Alg.1 l.12-14, A-1, A-2)
# ----------------------------------------------------------------------------

def select(scores, n_prune: int):
    """Prune the n_prune columns with the smallest variation score ("the
    one with small variation can be pruned"), ties by ascending index (A-2);
    return (S kept, P pruned), both ascending (Alg.1 l.14 ascendSort)."""
    sc = np.asarray(scores, dtype=np.float32)
    L = sc.shape[0]
    if not (0 <= n_prune <= L):
        raise OracleError("ZTP_EINVAL", "n_prune out of range")
    if np.isnan(sc).any():
        raise OracleError("ZTP_EINVAL", "NaN score")
    keys = sorted(range(L), key=lambda k: (float(sc[k]), k))
    P = np.array(sorted(keys[:n_prune]), dtype=np.int64)
    S = np.array(sorted(keys[n_prune:]), dtype=np.int64)
    return S, P


# ----------------------------------------------------------------------------
# NEXT-1. Priority-score maintenance (Alg.1 l.4-11)
# ----------------------------------------------------------------------------

def column_delta(Wt_new, Wt_old):
    """Alg.1 l.4: delta_i = sum_{j=1..R} |w_ji^t - w_ji^{t-1}| / R, the average
    change of the paper's column i of the weight [R, L].  Here row i of Wt
    [K=L, n=R].  Pinned: S:87 worked example, constant-shift closed form."""
    a = np.asarray(Wt_new, dtype=np.float64)
    b = np.asarray(Wt_old, dtype=np.float64)
    if a.shape != b.shape:
        raise OracleError("ZTP_ESHAPE", "weights differ in shape")
    return np.abs(a - b).sum(axis=1) / a.shape[1]


def priority_update(delta_prev, Wt_new, Wt_old, P_prev=None):
    """Alg.1 l.4-8 with the incremental rule of P:190: every column's delta is
    recomputed except the columns pruned in the previous epoch, which keep their
    old value (their zero-imputed gradients would otherwise pin them as
    'small variation' forever -- the endless loop of P:190; A-1: 'index not in
    pri_list' = pruned).  P_prev None = first epoch (all recomputed)."""
    d = column_delta(Wt_new, Wt_old)
    if P_prev is not None and len(P_prev):
        P = np.asarray(P_prev, dtype=np.int64)
        d[P] = np.asarray(delta_prev, dtype=np.float64)[P]
    return d


def pridiff_gamma(delta, theta: float, gamma_t: float, alpha: float = 0.8) -> float:
    """Alg.1 l.9-11 (Differentiated Pruning Ratios): L_uni = #{i:
    delta_i > theta}; gamma_k = 1 - L_uni / L_k; de facto max(gamma_k,
    alpha * gamma_t).  theta = N_iter * theta_iter (theta_iter = 1e-3)."""
    d = np.asarray(delta, dtype=np.float64)
    L = d.shape[0]
    if L == 0:
        raise OracleError("ZTP_EINVAL", "empty segment")
    L_uni = int(np.count_nonzero(d > theta))
    return max(1.0 - L_uni / L, alpha * gamma_t)


# ----------------------------------------------------------------------------
# a4-a6. One resized linear: dual pruning + imputation (Fig. 2)
# ----------------------------------------------------------------------------

def impute_rows(out_S: np.ndarray, S, P, K: int, policy: str = "zero", hist=None):
    """Dimension recovery: place the compact rows back at S and fill
    rows P by Zero (0), Average (mean over surviving rows, per column: A-10,
    S:100) or Same (previous iteration's values; A-11: error without history)."""
    out = np.zeros((K, out_S.shape[1]), dtype=np.float64)
    S = np.asarray(S, dtype=np.int64)
    P = np.asarray(P, dtype=np.int64)
    if len(S) + len(P) != K:
        raise OracleError("ZTP_ESHAPE", "|S|+|P| != K")
    out[S] = out_S
    if len(P):
        if policy == "zero":
            out[P] = 0.0
        elif policy == "average":
            out[P] = out_S.mean(axis=0, keepdims=True)
        elif policy == "same":
            if hist is None:
                raise OracleError("ZTP_EHISTORY", "Same needs history (S:74)")
            out[P] = np.asarray(hist, dtype=np.float64)[P]
        else:
            raise OracleError("ZTP_EINVAL", policy)
    return out


# Summation order of every contraction of the layer ("fp64,
# naive loops ... every output element keeps one fixed summation order").
# "blas": numpy's product (fast, any order; results within the fp64 bound
# K 2^-53 sum|terms| of the exact sum).  "fixed": the naive loop over the
# contraction index in ascending order, each product and each add rounded
# once (no FMA) -- bit-reproducible, used where a pin needs exact equality.
_ORDER = ["blas"]


class fixed_order:
    """with fixed_order(): every contraction is the naive k-ascending loop."""

    def __enter__(self):
        self._prev = _ORDER[0]
        _ORDER[0] = "fixed"
        return self

    def __exit__(self, *exc):
        _ORDER[0] = self._prev
        return False


def contract(A, B):
    """A^T B = sum over the rows k of A and B (ascending) of outer(A[k], B[k])."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if _ORDER[0] == "blas":
        return A.T @ B
    acc = np.zeros((A.shape[1], B.shape[1]), dtype=np.float64)
    for k in range(A.shape[0]):
        acc = acc + np.multiply.outer(A[k], B[k])
    return acc


def linear_fwd(Wt, Xt, S=None):
    """Forward with dual pruning: drop rows P of Wt [K,n] and Xt [K,N]
    (the paper's columns), concatenate survivors in ascending order, multiply.
    Output keeps its unpruned shape [n, N]."""
    Wt = np.asarray(Wt, dtype=np.float64)
    Xt = np.asarray(Xt, dtype=np.float64)
    if S is None:
        return contract(Wt, Xt)
    S = np.asarray(S, dtype=np.int64)
    return contract(Wt[S], Xt[S])


def linear_bwd_dx(Wt, Gt, S=None, P=None, policy="zero", hist=None):
    """grad_output: the upstream gradient G is never pruned; the result
    has K(1-gamma) rows and is recovered to K rows via the lineage."""
    Wt = np.asarray(Wt, dtype=np.float64)
    Gt = np.asarray(Gt, dtype=np.float64)
    if S is None:
        return contract(Wt.T, Gt)
    return impute_rows(contract(Wt[np.asarray(S)].T, Gt), S, P, Wt.shape[0], policy, hist)


def linear_bwd_dw(Xt, Gt, S=None, P=None, policy="zero", hist=None):
    """grad_weight (Fig. 2 right): G^T times the pruned input gives
    [n, K(1-gamma)] (here [K', n]); re-placed via the lineage, P imputed."""
    Xt = np.asarray(Xt, dtype=np.float64)
    Gt = np.asarray(Gt, dtype=np.float64)
    if S is None:
        return contract(Xt.T, Gt.T)
    return impute_rows(contract(Xt[np.asarray(S)].T, Gt.T), S, P, Xt.shape[0], policy, hist)


def fold(parts):
    """All-reduce as a left fold over ranks 0..e-1."""
    acc = np.array(parts[0], dtype=np.float64, copy=True)
    for q in parts[1:]:
        acc = acc + q
    return acc


# ----------------------------------------------------------------------------
# The layer used for measurement: attention-projection block
# (QKV col -> stand-in core ctx = Q+K+V (A-31) -> O row -> all-reduce) and MLP
# block (FC1 col -> GeLU -> FC2 row -> all-reduce); step = fwd + bwd.
# ----------------------------------------------------------------------------

SEGMENTS = ("qkv", "o", "fc1", "fc2")


@dataclass
class LayerShards:
    """Per-rank shards of one transformer layer (1D Megatron TP).
    qkv_t[r] [h, 3h/e] = [W_Q^T[:,F_r] | W_K^T[:,F_r] | W_V^T[:,F_r]];
    o_t[r] [h/e, h] = W_O^T[F_r,:]; w1_t[r] [h, f/e]; w2_t[r] [f/e, h]."""
    qkv_t: list
    o_t: list
    w1_t: list
    w2_t: list


def shard_layer(WQt, WKt, WVt, WOt, W1t, W2t, e: int) -> LayerShards:
    h = WQt.shape[0]
    f = W1t.shape[1]
    a, u = h // e, f // e
    qkv, o, w1, w2 = [], [], [], []
    for r in range(e):
        F = slice(r * a, (r + 1) * a)
        U = slice(r * u, (r + 1) * u)
        qkv.append(np.concatenate([WQt[:, F], WKt[:, F], WVt[:, F]], axis=1))
        o.append(WOt[F, :])
        w1.append(W1t[:, U])
        w2.append(W2t[U, :])
    return LayerShards(qkv, o, w1, w2)


def dense_layer_step(Xt, Gt, WQt, WKt, WVt, WOt, W1t, W2t, blocks: int = 1):
    """The unsplit, unpruned layer written directly (no TP): the reference the
    TP layer must reproduce at gamma = 0 (BASELINE north_star).

    blocks = e: every contraction over a dimension 1D TP splits -- the O and
    FC2 forward inputs, FC1's and QKV's grad_output contractions -- is summed
    per block of e contiguous parts and the block sums are added in block
    order (the summation order of e ranks and a left-fold all-reduce).  With
    fixed_order() the TP layer at gamma = 0 equals this bit-for-bit; any two
    block counts agree within the fp64 bound."""
    h = Xt.shape[0]
    f = W1t.shape[1]
    a, u = h // blocks, f // blocks
    Fb = [slice(r * a, (r + 1) * a) for r in range(blocks)]
    Ub = [slice(r * u, (r + 1) * u) for r in range(blocks)]
    q, k, v = contract(WQt, Xt), contract(WKt, Xt), contract(WVt, Xt)
    ctx = (q + k) + v
    Y1 = fold([contract(WOt[F], ctx[F]) for F in Fb])
    pre = contract(W1t, Y1)
    H = gelu_tanh(pre)
    Y = fold([contract(W2t[U], H[U]) for U in Ub])
    # backward
    dW2t = contract(H.T, Gt.T)
    dH = contract(W2t.T, Gt)
    G1 = dH * gelu_tanh_grad(pre)
    dW1t = contract(Y1.T, G1.T)
    dY1 = fold([contract(W1t[:, U].T, G1[U]) for U in Ub])
    dWOt = contract(ctx.T, dY1.T)
    dctx = contract(WOt.T, dY1)
    dWQt = contract(Xt.T, dctx.T)
    # the QKV grad_output contracts over the concatenated [Q | K | V] outputs;
    # block r = [Q_r | K_r | V_r] (one rank's column shard)
    dX = fold([contract(np.concatenate([WQt[:, F], WKt[:, F], WVt[:, F]], axis=1).T,
                        np.concatenate([dctx[F], dctx[F], dctx[F]], axis=0)) for F in Fb])
    return dict(Y=Y, dX=dX, dWQt=dWQt, dWKt=dWQt.copy(), dWVt=dWQt.copy(),
                dWOt=dWOt, dW1t=dW1t, dW2t=dW2t)


@dataclass
class AttnCore:
    """The real attention core (NEXT-4; A-31's stand-in replaced): per rank
    heads = a / head_dim, tokens t = b * seq + s (batch-major), softmax
    attention per (batch, head) with scale 1/sqrt(head_dim), causal or not."""
    head_dim: int
    seq: int
    causal: bool = True


def attention_fwd(Qt, Kt, Vt, core: AttnCore):
    """ctx^T = per (batch, head): softmax(Q K^T / sqrt(d) [+ causal mask]) V,
    written out per query row in fp64 (feature-major [a, N] in and out).
    Returns ctx^T and the probabilities P[b][h] for the backward."""
    a, N = Qt.shape
    d, S = core.head_dim, core.seq
    H, B = a // d, N // S
    ctx = np.zeros((a, N))
    probs = {}
    for b in range(B):
        cols = slice(b * S, (b + 1) * S)
        for hh in range(H):
            rows = slice(hh * d, (hh + 1) * d)
            q, k, v = Qt[rows, cols].T, Kt[rows, cols].T, Vt[rows, cols].T        # [S, d]
            sc = (q @ k.T) / math.sqrt(d)
            if core.causal:
                sc = np.where(np.tril(np.ones((S, S), dtype=bool)), sc, -np.inf)
            m = sc.max(axis=1, keepdims=True)
            ex = np.exp(sc - m)
            P = ex / ex.sum(axis=1, keepdims=True)
            probs[(b, hh)] = P
            ctx[rows, cols] = (P @ v).T
    return ctx, probs


def attention_bwd(Qt, Kt, Vt, dctx, probs, core: AttnCore):
    """Gradients of attention_fwd: dV = P^T dO, dP = dO V^T,
    dS = P * (dP - rowsum(dP * P)), dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d)."""
    a, N = Qt.shape
    d, S = core.head_dim, core.seq
    H, B = a // d, N // S
    dQ, dK, dV = np.zeros((a, N)), np.zeros((a, N)), np.zeros((a, N))
    for b in range(B):
        cols = slice(b * S, (b + 1) * S)
        for hh in range(H):
            rows = slice(hh * d, (hh + 1) * d)
            q, k, v, do = Qt[rows, cols].T, Kt[rows, cols].T, Vt[rows, cols].T, dctx[rows, cols].T
            P = probs[(b, hh)]
            dv = P.T @ do
            dp = do @ v.T
            ds = P * (dp - (dp * P).sum(axis=1, keepdims=True))
            dQ[rows, cols] = (ds @ k / math.sqrt(d)).T
            dK[rows, cols] = (ds.T @ q / math.sqrt(d)).T
            dV[rows, cols] = dv.T
    return dQ, dK, dV


def layer_step(Xt, Gt, sh: LayerShards, sel=None, mig=None, merged=True, policy="zero", core=None):
    """One TP layer step (fwd + bwd) simulated for all e ranks in-process.

    sel[r][seg] = (S, P) per segment (None = dense) -- the lineage table
    <layer, matrix, P>; the same S serves FWD and BWD.
    mig = list of (s, r, lo, hi): straggler s's MLP hidden units [lo, hi) are
    computed by helper r (SEMI-migration; build reading A-26: hidden-
    unit slices, merged into the existing all-reduces).
    merged=False: explicit collection -- the helper's FC2 partial for J goes to
    a separate buffer that is added to the straggler's partial before the fold.

    Returns Y [h,N], dX [h,N] (after the all-reduce), per-rank weight grads in
    the owner's view (migrated slices returned), the all-reduce count and the
    executed FLOPs per rank.
    """
    e = len(sh.qkv_t)
    h, N = Xt.shape
    a = h // e
    n_s = sh.w1_t[0].shape[1]
    sel = sel or [dict() for _ in range(e)]
    mig = mig or []
    nar = 0
    flops = [0.0] * e

    def S_of(r, seg):
        sp = sel[r].get(seg)
        return (None, None) if sp is None else sp

    def kept_count(r, seg, K):
        S, _ = S_of(r, seg)
        return K if S is None else len(S)

    # units of each rank's MLP shard that it computes itself (A-27: tail migrates)
    own_hi = [n_s] * e
    for (s, r, lo, hi) in mig:
        own_hi[s] = min(own_hi[s], lo)
    # ---------------- forward: attention-projection block -------------------
    ctx = []
    attn_saved = []
    y1_parts = []
    for r in range(e):
        S, _ = S_of(r, "qkv")
        qkv = linear_fwd(sh.qkv_t[r], Xt, S)
        flops[r] += 2.0 * qkv.shape[0] * N * kept_count(r, "qkv", h)
        if core is None:
            c = (qkv[:a] + qkv[a:2 * a]) + qkv[2 * a:]          # stand-in core (A-31)
        else:
            c, pr = attention_fwd(qkv[:a], qkv[a:2 * a], qkv[2 * a:], core)
            attn_saved.append((qkv, pr))
        ctx.append(c)
        So, _ = S_of(r, "o")
        y1_parts.append(linear_fwd(sh.o_t[r], c, So))
        flops[r] += 2.0 * h * N * kept_count(r, "o", a)
    Y1 = fold(y1_parts)
    nar += 1
    # ---------------- forward: MLP block -------------------------------------
    pre, H = [], []
    y_parts = [None] * e
    for r in range(e):
        S, _ = S_of(r, "fc1")
        W1 = sh.w1_t[r][:, :own_hi[r]]
        p_ = linear_fwd(W1, Y1, S)
        flops[r] += 2.0 * own_hi[r] * N * kept_count(r, "fc1", h)
        pre.append(p_)
        H.append(gelu_tanh(p_))
        Sw, _ = S_of(r, "fc2")
        if Sw is not None and len(Sw) and max(Sw) >= own_hi[r]:
            raise OracleError("ZTP_EINVAL", "FC2 selection overlaps migrated units")
        W2 = sh.w2_t[r][:own_hi[r]]
        y_parts[r] = linear_fwd(W2, H[r], Sw)
        flops[r] += 2.0 * h * N * (own_hi[r] if Sw is None else len(Sw))
    # helpers: H_J and the merged (or explicit) FC2 contribution
    preJ, HJ = {}, {}
    extra_to_straggler = [np.zeros((h, N)) for _ in range(e)]
    for (s, r, lo, hi) in mig:
        # received units extend the helper's FC1 output columns, contracted over
        # the helper's own kept rows S_c (reading A-33), and are appended to its
        # FC2 contraction unpruned (A-26)
        Sr, _ = S_of(r, "fc1")
        pj = linear_fwd(sh.w1_t[s][:, lo:hi], Y1, Sr)
        preJ[(s, r)] = pj
        HJ[(s, r)] = gelu_tanh(pj)
        contrib = contract(sh.w2_t[s][lo:hi], HJ[(s, r)])
        flops[r] += 2.0 * (hi - lo) * N * (kept_count(r, "fc1", h) + h)
        if merged:
            y_parts[r] = y_parts[r] + contrib          # local reduce merged
        else:
            extra_to_straggler[s] = extra_to_straggler[s] + contrib
    if not merged:
        y_parts = [y_parts[r] + extra_to_straggler[r] for r in range(e)]
    Y = fold(y_parts)
    nar += 1
    # ---------------- backward: MLP block ------------------------------------
    dW1 = [np.zeros_like(w) for w in sh.w1_t]
    dW2 = [np.zeros_like(w) for w in sh.w2_t]
    dy1_parts = [None] * e
    for r in range(e):
        Sw, Pw = S_of(r, "fc2")
        nown = own_hi[r]
        W2 = sh.w2_t[r][:nown]
        dH = linear_bwd_dx(W2, Gt, Sw, Pw, policy)            # [nown, N]
        dW2[r][:nown] = linear_bwd_dw(H[r], Gt, Sw, Pw, policy)
        kw = nown if Sw is None else len(Sw)
        flops[r] += 2.0 * 2.0 * kw * h * N
        G1 = dH * gelu_tanh_grad(pre[r])
        S, P = S_of(r, "fc1")
        W1 = sh.w1_t[r][:, :nown]
        dy1_parts[r] = linear_bwd_dx(W1, G1, S, P, policy)
        dW1[r][:, :nown] = linear_bwd_dw(Y1, G1, S, P, policy)
        flops[r] += 2.0 * 2.0 * kept_count(r, "fc1", h) * nown * N
    for (s, r, lo, hi) in mig:
        dHJ = contract(sh.w2_t[s][lo:hi].T, Gt)
        dW2[s][lo:hi] = contract(HJ[(s, r)].T, Gt.T)       # returned to the owner
        G1J = dHJ * gelu_tanh_grad(preJ[(s, r)])
        Sr, Pr = S_of(r, "fc1")
        contrib = linear_bwd_dx(sh.w1_t[s][:, lo:hi], G1J, Sr, Pr, policy)
        dW1[s][:, lo:hi] = linear_bwd_dw(Y1, G1J, Sr, Pr, policy)   # returned to the owner
        flops[r] += 2.0 * (hi - lo) * N * (2.0 * h + 2.0 * kept_count(r, "fc1", h))
        if merged:
            dy1_parts[r] = dy1_parts[r] + contrib            # merged into the all-reduce
        else:
            dy1_parts[s] = dy1_parts[s] + contrib
    dY1 = fold(dy1_parts)
    nar += 1
    # ---------------- backward: attention-projection block -------------------
    dWqkv = [None] * e
    dWo = [None] * e
    dx_parts = []
    for r in range(e):
        So, Po = S_of(r, "o")
        dctx = linear_bwd_dx(sh.o_t[r], dY1, So, Po, policy)
        dWo[r] = linear_bwd_dw(ctx[r], dY1, So, Po, policy)
        flops[r] += 2.0 * 2.0 * kept_count(r, "o", a) * h * N
        if core is None:
            gq = np.concatenate([dctx, dctx, dctx], axis=0)   # stand-in core bwd: dQ=dK=dV=dctx
        else:
            qkv_r, pr = attn_saved[r]
            gq = np.concatenate(attention_bwd(qkv_r[:a], qkv_r[a:2 * a], qkv_r[2 * a:], dctx, pr, core), axis=0)
        S, P = S_of(r, "qkv")
        dx_parts.append(linear_bwd_dx(sh.qkv_t[r], gq, S, P, policy))
        dWqkv[r] = linear_bwd_dw(Xt, gq, S, P, policy)
        flops[r] += 2.0 * 2.0 * kept_count(r, "qkv", h) * 3 * a * N
    dX = fold(dx_parts)
    nar += 1
    return dict(Y=Y, dX=dX, Y1=Y1, dY1=dY1, dWqkv=dWqkv, dWo=dWo, dW1=dW1, dW2=dW2,
                allreduce_count=nar, flops=flops)


def layer_step_sampled(Xt, Gt, sh: LayerShards, sel, tok_idx, mig=None):
    """Sampled parity at full size: the layer computed only
    for the token columns `tok_idx`.  Every op of the layer except the weight-
    gradient reductions acts per token column (the stand-in core is per feature,
    A-31), so the sampled Y and dX are exactly the columns the full oracle
    would produce.  Weight gradients need all tokens and are not returned."""
    cols = np.asarray(tok_idx, dtype=np.int64)
    out = layer_step(Xt[:, cols], Gt[:, cols], sh, sel, mig)
    return dict(Y=out["Y"], dX=out["dX"], Y1=out["Y1"], dY1=out["dY1"])

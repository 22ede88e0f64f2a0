"""CPU tests of the C ABI: the library loads, exports every symbol include/ztp.h
declares, and its host planner (ztp_plan / ztp_plan_counts) matches the oracle
bit-exactly (plans and counts are bit-exact)."""
import ctypes as C
import os
import random
import re
import struct

import pytest

from conftest import ROOT
from oracle import ztp_oracle as O


@pytest.fixture(scope="module")
def Z():
    import paper_2401_11469_b200 as z
    return z


def test_header_symbols_exported(Z):
    hdr = open(os.path.join(ROOT, "include", "ztp.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(ztp_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    from paper_2401_11469_b200 import _lib
    for name in sorted(declared):
        assert hasattr(_lib.lib, name), f"{name} declared in ztp.h but not exported"
    assert set(_lib.EXPORTED) == declared


def test_status_strings_and_version(Z):
    from paper_2401_11469_b200 import _lib
    for i, nm in enumerate(_lib.STATUS):
        assert _lib.lib.ztp_status_str(i).decode() == nm
    assert "sm_100a" in Z.ztp_version()


def _bits(x):
    return struct.pack("<d", x)


def _costs_pair(Z, rng):
    def mono():
        xs = sorted({0.0} | {round(rng.uniform(1, 300), 3) for _ in range(rng.randint(1, 4))})
        ys = [0.0]
        for _ in xs[1:]:
            ys.append(ys[-1] + rng.uniform(0, 5))
        return (tuple(xs), tuple(ys))
    om1 = rng.uniform(0, 2)
    o2, p1, p2 = mono(), mono(), mono()
    return Z.make_costs(om1, o2, p1, p2), O.Costs(om1, o2, p1, p2)


def _compare(Z, T, M, L, costs_pair, kw):
    zc, oc = costs_pair
    oopts = O.PlanOpts(**kw)
    try:
        op = O.plan(T, M, L, oc, oopts)
        oerr = None
    except O.OracleError as e:
        oerr = e.code
    try:
        zp = Z.ztp_plan(T, M, L, zc, Z.plan_opts(**kw))
        zerr = None
    except Z.ZtpError as e:
        zerr = e.name
    assert oerr == zerr
    if oerr:
        return None
    e = len(T)
    assert zp.world == e and zp.z == op.z and zp.x == op.x
    assert list(zp.order)[:e] == op.order
    assert list(zp.role)[:e] == op.role
    for f in ("gamma", "beta", "phi", "gamma_r"):
        for r in range(e):
            assert _bits(getattr(zp, f)[r]) == _bits(getattr(op, f)[r]), (f, r)
    return zp, op


@pytest.mark.parametrize("seed", range(10))
def test_plan_bitexact_vs_oracle_randomized(Z, seed):
    """>= 1000 randomized instances in total (10 seeds x 120) across ZERO-AVG,
    ZERO-MIN and SEMI, with ties, clamps and forced lambda."""
    rng = random.Random(seed)
    for _ in range(120):
        e = rng.randint(1, 8)
        base = rng.uniform(1, 100)
        T, M = [], []
        for r in range(e):
            chi = rng.choice([1.0, 1.0, rng.uniform(1, 9)])
            m = rng.uniform(0.2, 0.9) * base
            T.append(base - m + chi * m if rng.random() < 0.9 else base)
            M.append(chi * m)
        if rng.random() < 0.05:
            M[rng.randrange(e)] = 0.0
        kw = dict(enable_migration=rng.randint(0, 1), zero_crit=rng.randint(0, 1),
                  gamma_max=rng.choice([0.9, 1.0, 0.5]), eps=rng.choice([0.0, 0.02]),
                  gamma_tol=rng.choice([0.5, 0.3]), bisect_iters=rng.choice([64, 20]),
                  force_lambda=rng.choice([-1, -1, -1, 0, 1, 3]))
        res = _compare(Z, T, M, rng.choice([64.0, 100.0, 4096.0]), _costs_pair(Z, rng), kw)
        if res is None:
            continue
        zp, op = res
        # counts for every rank and both layer kinds
        for r in range(e):
            for K, n_units, unit, is_row in ((1024, 512, 1, False), (512, 512, 1, True), (777, 128, 4, True)):
                try:
                    oc = O.plan_counts(op, r, K, n_units, unit, is_row)
                    oerr = None
                except O.OracleError as ex:
                    oerr = ex.code
                try:
                    zc = Z.ztp_plan_counts(zp, r, K, n_units, unit, is_row)
                    zerr = None
                except Z.ZtpError as ex:
                    zerr = ex.name
                assert oerr == zerr
                if oerr:
                    continue
                assert (zc.n_prune, zc.n_mig) == (oc.n_prune, oc.n_mig)
                assert [(zc.out_dst[i], zc.out_lo[i], zc.out_hi[i]) for i in range(zc.n_out)] == oc.out
                assert [(zc.in_src[i], zc.in_lo[i], zc.in_hi[i]) for i in range(zc.n_in)] == oc.inc


def test_plan_worked_examples_match(Z):
    zero = ((0.0, 1.0), (0.0, 0.0))
    lin = ((0.0, 1.0), (0.0, 1.0))
    pair = (Z.make_costs(0.0, lin, lin, lin), O.Costs(0.0, lin, lin, lin))
    _compare(Z, [10.0, 20.0], [16.0, 16.0], 100.0, pair, dict(zero_crit=O.CRIT_AVG))
    _compare(Z, [20.0, 36.0], [16.0, 32.0], 64.0, pair, dict(zero_crit=O.CRIT_AVG))
    p01 = ((0.0, 1.0), (0.0, 0.1))
    _compare(Z, [40.0, 30.0, 10.0, 10.0], [5.0] * 4, 100.0,
             (Z.make_costs(0.0, zero, p01, zero), O.Costs(0.0, zero, p01, zero)),
             dict(enable_migration=1, gamma_max=1.0))
    zp = Z.ztp_plan([20.0, 36.0], [16.0, 32.0], 64.0, opts=Z.plan_opts(zero_crit=Z.CRIT_AVG))
    assert zp.gamma[1] == 0.25
    assert Z.ztp_plan_counts(zp, 1, 64, 128, 1, False).n_prune == 16


def test_plan_errors(Z):
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_plan([], [], 1.0)
    assert ei.value.name == "ZTP_EINVAL"
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_plan([1.0, 2.0], [1.0, 0.0], 1.0)
    assert ei.value.name == "ZTP_ENOBASELINE"
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_plan([1.0, float("nan")], [1.0, 1.0], 1.0)
    assert ei.value.name == "ZTP_EINVAL"


def test_plan_refine_matches_oracle(Z):
    """ztp_plan_refine (A-39) bit-exact against the oracle on random ZERO
    plan pairs; SEMI roles are rejected by both."""
    import random
    rng = random.Random(7)
    for _ in range(300):
        e = rng.randint(1, 8)
        T1 = [rng.uniform(1, 3) for _ in range(e)]
        T2 = [rng.uniform(1, 3) for _ in range(e)]
        M = [rng.uniform(0.5, 2) for _ in range(e)]
        kw = dict(zero_crit=rng.randint(0, 1), gamma_max=rng.choice([0.9, 1.0]))
        zp1, zp2 = Z.ztp_plan(T1, M, 1.0, opts=Z.plan_opts(**kw)), Z.ztp_plan(T2, M, 1.0, opts=Z.plan_opts(**kw))
        op1, op2 = O.plan(T1, M, 1.0, O.Costs(), O.PlanOpts(**kw)), O.plan(T2, M, 1.0, O.Costs(), O.PlanOpts(**kw))
        zr = Z.ztp_plan_refine(zp1, zp2, kw["gamma_max"])
        orf = O.plan_refine(op1, op2, kw["gamma_max"])
        assert list(zr.role)[:e] == orf.role and zr.z == orf.z and list(zr.order)[:e] == orf.order
        for r in range(e):
            assert _bits(zr.gamma[r]) == _bits(orf.gamma[r]) and _bits(zr.gamma_r[r]) == _bits(orf.gamma_r[r])
    lin = ((0.0, 1.0), (0.0, 1.0))
    semi = Z.ztp_plan([10.0, 30.0], [10.0, 30.0], 100.0, Z.make_costs(0.0, lin, ((0.0, 1.0), (0.0, 0.0)), lin),
                      Z.plan_opts(enable_migration=1))
    assert semi.role[1] in (Z.MIGRATE, Z.SPLIT)
    with pytest.raises(Z.ZtpError) as ei:     # the refresh plan itself must be ZERO-only
        Z.ztp_plan_refine(semi, semi)
    assert ei.value.name == "ZTP_EUNSUPPORTED"


def test_plan_refine_semi_matches_oracle(Z):
    """A-42: refreshing a SEMI plan (MIGRATE / SPLIT ranks compose their shed
    fraction, keep beta) is bit-exact against the oracle on random plans."""
    import random
    rng = random.Random(11)
    seen = set()
    for _ in range(300):
        e = rng.randint(2, 8)
        T1 = [rng.uniform(1, 1.3) for _ in range(e)]
        for s in rng.sample(range(e), rng.randint(1, min(3, e - 1))):
            T1[s] = rng.uniform(2, 4)
        M = [rng.uniform(0.5, 1.0) * t for t in T1]
        T2 = [rng.uniform(1, 1.6) for _ in range(e)]
        xs = (0.0, 1.0)
        om2, p1, p2 = ((xs, (0.0, rng.uniform(0, 2))) for _ in range(3))
        om1 = rng.uniform(0, 0.2)
        zc, oc = Z.make_costs(om1, om2, p1, p2), O.Costs(om1, om2, p1, p2)
        kw = dict(enable_migration=1, zero_crit=1, gamma_max=rng.choice([0.9, 1.0]))
        zp1 = Z.ztp_plan(T1, M, 1.0, zc, Z.plan_opts(**kw))
        op1 = O.plan(T1, M, 1.0, oc, O.PlanOpts(**kw))
        kz = dict(zero_crit=1, gamma_max=kw["gamma_max"])
        zp2 = Z.ztp_plan(T2, M, 1.0, opts=Z.plan_opts(**kz))
        op2 = O.plan(T2, M, 1.0, O.Costs(), O.PlanOpts(**kz))
        zr = Z.ztp_plan_refine(zp1, zp2, kw["gamma_max"])
        orf = O.plan_refine(op1, op2, kw["gamma_max"])
        seen.update(orf.role)
        assert list(zr.role)[:e] == orf.role and zr.x == orf.x and list(zr.order)[:e] == orf.order[:e]
        for r in range(e):
            for k in ("gamma", "beta", "phi", "gamma_r"):
                assert _bits(getattr(zr, k)[r]) == _bits(getattr(orf, k)[r]), (k, r)
    assert {O.MIGRATE, O.RESIZE} <= seen or {O.SPLIT, O.RESIZE} <= seen


def test_no_cuda_device_is_an_error_not_a_fallback(Z):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_ctx_create()
    assert ei.value.name in ("ZTP_ECUDA", "ZTP_EUNSUPPORTED")


def test_pridiff_gamma_matches_oracle():
    """Alg.1 l.10-11 host function, bit-exact vs the oracle's rule."""
    import numpy as np
    from oracle import ztp_oracle as O
    import paper_2401_11469_b200 as Z
    rng = np.random.default_rng(9)
    for _ in range(300):
        L = int(rng.integers(1, 5000))
        d = rng.random(L) * 0.01
        theta = float(rng.choice([0.001, 0.005, 0.0]))
        g = float(rng.random() * 0.9)
        a = float(rng.choice([0.8, 1.0, 0.5]))
        L_uni = int(np.count_nonzero(d > theta))
        assert Z.ztp_pridiff_gamma(L, L_uni, g, a) == O.pridiff_gamma(d, theta, g, a)


def test_layer_prune_counts_attention_rule():
    """A-37: attention linears prune by gamma_r, except on ranks that shed MLP
    units (MIGRATE / SPLIT), which resize attention by their Eq.1 gamma; the
    MLP counts are ztp_plan_counts' (FC2 over its K_rem = u - n_mig)."""
    import math
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.layer import layer_prune_counts
    T = [10.0, 80.0, 10.0, 60.0, 10.0, 40.0, 10.0, 20.0]
    M = [8.0, 78.0, 8.0, 58.0, 8.0, 38.0, 8.0, 18.0]
    h, a, u = 4096, 512, 1376
    for lam in range(5):
        plan = Z.ztp_plan(T, M, float(u), None, Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN,
                                                               force_lambda=lam))
        for r in range(8):
            c = layer_prune_counts(plan, r, h, a, u)
            role = int(plan.role[r])
            g_att = plan.gamma[r] if role in (Z.MIGRATE, Z.SPLIT) else plan.gamma_r[r]
            for s, K in (("qkv", h), ("o", a)):
                want = min(max(int(math.floor(K * g_att + 0.5)), 0), K - 1)
                assert c[s] == want, (lam, r, s)
            assert c["fc1"] == Z.ztp_plan_counts(plan, r, h, u, 1, False).n_prune
            assert c["fc2"] == Z.ztp_plan_counts(plan, r, u, u, 1, True).n_prune
            if role == Z.MIGRATE:            # a migrating rank still sheds its attention excess
                assert c["qkv"] > 0 and c["o"] > 0


def _plan_bits_equal(zp, op, e):
    assert zp.world == op.world and zp.z == op.z and zp.x == op.x
    assert list(zp.role)[:e] == list(op.role[:e])
    assert list(zp.order)[:e] == list(op.order[:e])
    for k in ("gamma", "beta", "phi", "gamma_r"):
        for r in range(e):
            assert _bits(getattr(zp, k)[r]) == _bits(getattr(op, k)[r]), (k, r)


@pytest.mark.parametrize("semi", [0, 1])
def test_controller_matches_oracle_randomized(Z, semi):
    """ztp_ctl_step (the P:178 re-planning loop, A-41/A-43) bit-exact against
    the oracle's Controller on random runtime sequences: every plan, state,
    action and counter after every step."""
    rng = random.Random(17 + semi)
    seen = {"refine": 0, "trigger": 0, "apply": 0}
    for trial in range(60):
        e = rng.randint(1, 8)
        zc, oc = _costs_pair(Z, rng) if semi else (Z.make_costs(), O.Costs())
        kw = dict(enable_migration=semi, zero_crit=1 if semi else rng.randint(0, 1),
                  gamma_max=rng.choice([0.9, 1.0]), eps=rng.choice([0.0, 0.02, 0.05]))
        L = float(rng.choice([512, 1376, 2560]))
        trig = rng.choice([0.1, 0.05, 0.2])
        mr = rng.randint(0, 3)
        zo = Z.ctl_opts(L_ref=L, trigger=trig, max_refines=mr, **kw)
        oo = O.CtlOpts(plan=O.PlanOpts(**kw), L_ref=L, trigger=trig, max_refines=mr)
        zctl, octl = Z.ztp_ctl_init(e), O.Controller(e)
        chis = [1.0] * e
        for k in range(25):
            if rng.random() < 0.15:                     # the slowdowns change
                chis = [rng.choice([1.0, 1.0, 1.0, 2.0, 3.0, 8.0]) for _ in range(e)]
            T = [c * rng.uniform(0.9, 1.1) + rng.uniform(0.1, 0.3) for c in chis]
            M = [t * rng.uniform(0.5, 0.9) for t in T]
            try:
                oa = octl.step(T, M, oo, oc)
                oerr = None
            except O.OracleError as ex:
                oerr = ex.code
            try:
                za = Z.ztp_ctl_step(zctl, zo, T, M, zc)
                zerr = None
            except Z.ZtpError as ex:
                zerr = ex.name
            assert oerr == zerr, (trial, k)
            if oerr:
                break
            assert za == oa and zctl.state == octl.state and zctl.refines == octl.refines, (trial, k)
            _plan_bits_equal(zctl.plan, octl.plan, e)
            assert (zctl.windows, zctl.replans, zctl.refine_count, zctl.triggers) == \
                (octl.windows, octl.replans, octl.refine_count, octl.triggers)
            assert _bits(zctl.T_target) == _bits(octl.T_target) and _bits(zctl.T_wmax) == _bits(octl.T_wmax)
            seen["apply"] += za
        seen["refine"] += octl.refine_count
        seen["trigger"] += octl.triggers
    assert all(v > 0 for v in seen.values()), seen


def test_controller_errors_abi(Z):
    ctl = Z.ztp_ctl_init(2)
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_ctl_step(ctl, Z.ctl_opts(), [1.0, float("nan")], [1.0, 1.0])
    assert ei.value.name == "ZTP_EINVAL"
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_ctl_step(ctl, Z.ctl_opts(), [1.0, 2.0], [1.0, 0.0])
    assert ei.value.name == "ZTP_ENOBASELINE"
    with pytest.raises(Z.ZtpError):
        Z.ztp_ctl_init(9)


def test_layer_prune_counts_matches_oracle(Z):
    """ztp_layer_prune_counts (A-37 + MLP counts) equals the oracle's on random
    SEMI / ZERO plans for every rank; ztp_plan_uniform likewise."""
    rng = random.Random(23)
    for _ in range(200):
        e = rng.randint(1, 8)
        T = [rng.uniform(1, 1.2) for _ in range(e)]
        for s in rng.sample(range(e), rng.randint(0, max(0, e - 1))):
            T[s] = rng.uniform(1.5, 6.0)
        M = [t * rng.uniform(0.6, 0.9) for t in T]
        zc, oc = _costs_pair(Z, rng)
        kw = dict(enable_migration=rng.randint(0, 1) if e > 1 else 0, zero_crit=1)
        h = rng.choice([64, 1024, 4096])
        a, u = h // e, rng.choice([128, 1376, 2560])
        try:
            op = O.plan(T, M, float(u), oc, O.PlanOpts(**kw))
        except O.OracleError:
            continue
        zp = Z.ztp_plan(T, M, float(u), zc, Z.plan_opts(**kw))
        for r in range(e):
            assert Z.ztp_layer_prune_counts(zp, r, h, a, u) == O.layer_prune_counts(op, r, h, a, u)
    for g in (0.0, 0.25, 0.5, 0.9, 0.999):
        up, oup = Z.ztp_plan_uniform(4, g), O.plan_uniform(4, g)
        assert Z.ztp_layer_prune_counts(up, 2, 1024, 256, 1024) == O.layer_prune_counts(oup, 2, 1024, 256, 1024)
    with pytest.raises(Z.ZtpError):
        Z.ztp_plan_uniform(2, 1.0)


def test_pridiff_counts_matches_oracle(Z):
    rng = random.Random(29)
    for _ in range(500):
        L = rng.randint(1, 20000)
        L_uni = rng.randint(0, L)
        g, a, gm = rng.random(), rng.choice([0.5, 0.8, 1.0]), rng.choice([0.9, 1.0])
        assert Z.ztp_pridiff_counts(L, L_uni, g, a, gm) == O.pridiff_counts(L, L_uni, g, a, gm)
    assert Z.ztp_pridiff_counts(0, 0, 0.5) == 0


def test_costs_fit_matches_oracle(Z):
    """ztp_costs_fit (A-40) bit-exact vs the oracle's fit on random noisy
    samples (duplicates, negatives, dips)."""
    rng = random.Random(31)
    for _ in range(300):
        def pts(n, lo):
            return [(float(rng.choice([0, rng.randint(lo, 3000)])), rng.uniform(-0.01, 0.05)) for _ in range(n)]
        om, p1, p2 = pts(rng.randint(0, 7), 1), pts(rng.randint(0, 6), 1), pts(rng.randint(0, 6), 1)
        if rng.random() < 0.2 and om:
            om.append((om[0][0], om[0][1] + 0.001))          # repeated x
        (zc, _), plain = Z.ztp_costs_fit(om, p1, p2)
        oc = O.costs_fit(om, p1, p2)
        assert _bits(plain["omega1"]) == _bits(oc.omega1)
        for k in ("omega2", "phi1", "phi2"):
            zx, zy = plain[k]
            ox, oy = getattr(oc, k)
            assert len(zx) == len(ox) and all(_bits(p) == _bits(q) for p, q in zip(zx + zy, ox + oy)), k
    with pytest.raises(Z.ZtpError):
        Z.ztp_costs_fit([(1.0, float("nan"))], [], [])

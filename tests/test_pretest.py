"""Alg.2 l.1 pretest: the sample -> cost-function fitting on
CPU, the GPU measurement through the C ABI, and ztp_plan consuming the result
bit-exactly like the oracle's planner does with the same functions."""
import math

import numpy as np
import pytest

from oracle import ztp_oracle as O


@pytest.mark.parametrize("which", ["library", "oracle"])
def test_fit_costs_shape_and_monotone(which):
    """Omega_1 = extra cost at the smallest pruned count; Omega_2 / Phi_1 /
    Phi_2 pass through (0, 0), are non-decreasing (noise dips removed) and
    clamped at 0.  Hand-computed values (A-40), for the library's fit and the
    oracle's."""
    from paper_2401_11469_b200.pretest import fit_costs

    def oracle_fit(om, p1, p2):
        oc = O.costs_fit(om, p1, p2)
        return None, {"omega1": oc.omega1, "omega2": oc.omega2, "phi1": oc.phi1, "phi2": oc.phi2}
    fit = fit_costs if which == "library" else oracle_fit
    _, c = fit([(0, 0.0), (128, 0.010), (256, 0.012), (512, 0.011), (768, 0.020)],
                     [(128, 0.004), (64, 0.003), (1024, 0.020)],
                     [(0, 0.0), (128, -0.001), (256, 0.006), (512, 0.012)])
    assert c["omega1"] == pytest.approx(0.010)
    assert c["omega2"][0] == (0.0, 128.0, 256.0, 512.0, 768.0)
    assert c["omega2"][1] == pytest.approx((0.0, 0.0, 0.002, 0.002, 0.010))
    assert c["phi1"][0] == (0.0, 64.0, 128.0, 1024.0)
    assert c["phi1"][1] == pytest.approx((0.0, 0.003, 0.004, 0.020))
    assert c["phi2"][1] == pytest.approx((0.0, 0.0, 0.006, 0.012))
    for k in ("omega2", "phi1", "phi2"):
        ys = c[k][1]
        assert all(b >= a for a, b in zip(ys, ys[1:])) and min(ys) >= 0.0


def test_fit_costs_degenerate():
    """No positive samples -> Omega_1 = 0 and valid 2-point functions (ztp_pwl
    needs >= 2 samples)."""
    from paper_2401_11469_b200.pretest import fit_costs
    costs, c = fit_costs([(0, 0.0)], [], [])
    assert c["omega1"] == 0.0
    oc = O.costs_fit([(0, 0.0)], [], [])
    assert oc.omega1 == 0.0 and oc.phi1 == ((0.0, 1.0), (0.0, 0.0))
    for k in ("omega2", "phi1", "phi2"):
        assert len(c[k][0]) >= 2


def test_fitted_costs_drive_plan_like_oracle():
    """A fitted cost model through ztp_plan (SEMI, z = 1, heavy straggler)
    gives the oracle's plan bit-for-bit (Eq.2 bisection on the same
    piecewise-linear functions)."""
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.pretest import fit_costs
    costs, c = fit_costs([(0, 0.0), (256, 0.004), (512, 0.006), (768, 0.009)],
                         [(128, 0.010), (512, 0.030), (1024, 0.055)],
                         [(0, 0.0), (128, 0.020), (256, 0.040), (512, 0.080)])
    T = [1.0, 1.0, 1.0, 3.0]
    M = [0.8, 0.8, 0.8, 2.4]
    got = Z.ztp_plan(T, M, 1024.0, costs, Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN))
    oc = O.Costs(c["omega1"], c["omega2"], c["phi1"], c["phi2"])
    want = O.plan(T, M, 1024.0, oc, O.PlanOpts(enable_migration=1, zero_crit=O.CRIT_MIN))
    assert list(got.role[:4]) == list(want.role[:4])
    for k in ("gamma", "beta", "phi", "gamma_r"):
        assert list(getattr(got, k)[:4]) == list(getattr(want, k)[:4]), k
    assert 0.0 < got.beta[3] < 1.0 or got.beta[3] in (0.0, 1.0)


@pytest.mark.gpu
def test_pretest_on_gpu():
    """The pretest on a small layer through the C ABI: every sample finite,
    resizing saves GEMM time (M decreasing in gamma), a helper's extra time
    grows with the appended units, the copies grow with the units moved, and
    the fitted costs drive ztp_plan."""
    import torch
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.layer import ZtpLayer
    from paper_2401_11469_b200.pretest import pretest
    from synth import inputs as I
    h, f, N, seed = 512, 2048, 2048, 77
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    try:
        sh = {"qkv": I.uniform_sym(seed, "q", h, 3 * h, 0.04), "o": I.uniform_sym(seed, "o", h, h, 0.04),
              "w1": I.uniform_sym(seed, "w1", h, f, 0.04), "w2": I.uniform_sym(seed, "w2", f, h, 0.02)}
        dev = {k: torch.from_numpy(v.astype(np.float32)).cuda().to(torch.bfloat16) for k, v in sh.items()}
        L = ZtpLayer(ctx, h, f, N, 0, 1, dev, mig_cap=f)
        L.X.normal_()
        L.G.normal_()
        lens = {"qkv": h, "o": h, "fc1": h, "fc2": f}
        sc = {s: torch.from_numpy(I.lognormal_scores(seed, s, n)).cuda() for s, n in lens.items()}
        costs, rep = pretest(L, ctx, sc, steps=10, link_gbs=770.0)
        om = rep["omega"]
        assert all(math.isfinite(d["T_ms"]) and d["T_ms"] > 0 for d in om)
        assert om[-1]["M_ms"] < om[0]["M_ms"]                      # resizing saves GEMM time
        p2 = rep["phi2"]
        assert p2[-1]["extra_ms"] > 0.0 and p2[-1]["T_ms"] > p2[0]["T_ms"]
        p1 = rep["phi1_measured"]
        # copies of 1/8 .. all units: launch-dominated at this size, so only
        # positivity and a non-shrinking trend within timing noise
        assert all(d["ms"] > 0.0 for d in p1) and p1[-1]["ms"] >= 0.9 * p1[0]["ms"]
        assert p1[-1]["bytes"] == 8 * p1[0]["bytes"]
        plan = Z.ztp_plan([1.0, 3.0], [0.8, 2.4], float(f), costs,
                          Z.plan_opts(enable_migration=1, zero_crit=Z.CRIT_MIN))
        assert plan.z == 1 and 0.0 <= plan.beta[1] <= 1.0
        # the layer is left dense and still steps correctly
        assert L.n_prune["fc2"] == 0 and L.mig.n_mig == 0 and not L.mig.inc
        L.step()
        torch.cuda.synchronize()
        assert torch.isfinite(L.dX.float()).all()
    finally:
        Z.ztp_ctx_destroy(ctx)

"""Pins of the oracle's resized linear / layer step against closed forms, brute
force, finite differences and the paper's worked example (Fig. 2)."""
import math
import random

import numpy as np
import pytest

from conftest import golden
from oracle import ztp_oracle as O
from synth import inputs as I


def _rand(shape, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return I.round_bf16(rng.standard_normal(shape) * scale)


# ---------------------------------------------------------------- GeLU

def test_gelu_tanh_against_erf_gelu_and_fd():
    x = np.linspace(-6, 6, 2001)
    exact = 0.5 * x * (1 + np.vectorize(math.erf)(x / math.sqrt(2)))
    assert np.max(np.abs(O.gelu_tanh(x) - exact)) < 1e-3      # known tanh-approx bound
    assert O.gelu_tanh(0.0) == 0.0
    assert O.gelu_tanh(10.0) == pytest.approx(10.0, rel=1e-12)
    h = 1e-6
    fd = (O.gelu_tanh(x + h) - O.gelu_tanh(x - h)) / (2 * h)
    assert np.max(np.abs(O.gelu_tanh_grad(x) - fd)) < 1e-8
    assert O.gelu_tanh_grad(0.0) == 0.5


# ------------------------------------------------------- Fig. 2 shapes

def test_fig2_worked_example():
    g = golden("fig2.json")
    hs, e, Pp = g["hs"], g["e"], g["pruned"]
    N = 5
    S = [k for k in range(hs) if k not in Pp]
    Xt = _rand((hs, N), 1)
    Wt = _rand((hs, hs // e), 2)
    # pruned_input [N x hs(1-g)] and pruned_weight [hs/e x hs(1-g)] in the paper's view
    assert Xt[S].T.shape == (N, 2) and Wt[S].T.shape == (hs // e, 2)
    Y = O.linear_fwd(Wt, Xt, S)
    assert Y.T.shape == (N, hs // e)                           # output keeps its size
    Gt = _rand((hs // e, N), 3)
    dW = O.linear_bwd_dw(Xt, Gt, S, Pp)
    assert dW.T.shape == (hs // e, hs)                         # recovered grad_weight
    assert np.all(dW[Pp] == 0.0)                               # columns 2 and 4 zero
    dX = O.linear_bwd_dx(Wt, Gt, S, Pp)
    assert dX.shape == (hs, N) and np.all(dX[Pp] == 0.0)


# ------------------------------------------- Zero imputation == masked operands

def _kloop(A, B):
    """sum_k A[k]^T B[k] with k ascending, one add per k (fixed order)."""
    acc = np.zeros((A.shape[1], B.shape[1]))
    for k in range(A.shape[0]):
        acc = acc + np.outer(A[k], B[k])
    return acc


@pytest.mark.parametrize("seed", range(6))
def test_zero_resize_equals_dense_on_masked_operands_bitexact(seed):
    """pruning rows P of W^T and X^T and zero-imputing equals the
    dense computation on operands whose rows P are zero -- bit-exact under a
    fixed k order (adding exact zeros changes nothing)."""
    rng = random.Random(seed)
    K, n, N = rng.randint(3, 24), rng.randint(1, 9), rng.randint(1, 9)
    P = sorted(rng.sample(range(K), rng.randint(1, K - 1)))
    S = [k for k in range(K) if k not in P]
    Wt, Xt, Gt = _rand((K, n), seed), _rand((K, N), seed + 100), _rand((n, N), seed + 200)
    Wm, Xm = Wt.copy(), Xt.copy()
    Wm[P] = 0.0
    Xm[P] = 0.0
    assert np.array_equal(_kloop(Wt[S], Xt[S]), _kloop(Wm, Xm))              # fwd
    # dX rows: dX[k] = sum_j W[k,j] G[j]; dW rows: dW[k] = sum_t X[k,t] G[:,t]
    dx_c = O.impute_rows(_kloop(Wt[S].T, Gt), S, P, K)
    assert np.array_equal(dx_c, _kloop(Wm.T, Gt))
    dw_c = O.impute_rows(_kloop(Xt[S].T, Gt.T), S, P, K)
    assert np.array_equal(dw_c, _kloop(Xm.T, Gt.T))
    # the oracle's BLAS products agree with the fixed-order sums within the
    # fp64 bound  K * 2^-53 * sum|terms|
    for got, A, B in ((O.linear_fwd(Wt, Xt, S), Wt[S], Xt[S]),
                      (O.linear_bwd_dx(Wt, Gt, S, P)[S], Wt[S].T, Gt),
                      (O.linear_bwd_dw(Xt, Gt, S, P)[S], Xt[S].T, Gt.T)):
        ref = _kloop(A, B)
        bound = A.shape[0] * 2.0 ** -53 * _kloop(np.abs(A), np.abs(B))
        assert np.all(np.abs(got - ref) <= bound + 1e-300)
    assert np.all(O.linear_bwd_dx(Wt, Gt, S, P)[P] == 0.0)
    assert np.all(O.linear_bwd_dw(Xt, Gt, S, P)[P] == 0.0)


def test_dense_linear_bruteforce_triple_loop():
    K, n, N = 5, 3, 4
    Wt, Xt = _rand((K, n), 7), _rand((K, N), 8)
    Y = O.linear_fwd(Wt, Xt)
    for j in range(n):
        for t in range(N):
            s = math.fsum(Wt[k, j] * Xt[k, t] for k in range(K))
            assert abs(Y[j, t] - s) <= K * 2 ** -53 * sum(abs(Wt[k, j] * Xt[k, t]) for k in range(K))


# ------------------------------------------------------- imputation

def test_imputation_examples():
    g = golden("impute_worked.json")
    # paper view M = [[2,4]] (1 token row x 2 surviving features) -> ours is M^T
    surv = np.array(g["average_in_paper_view"], dtype=np.float64).T       # [2, 1]
    P = g["average_pruned"]
    out = O.impute_rows(surv, [0, 2], P, 3, "average")
    assert out.T.tolist() == g["average_out_paper_view"]
    z = O.impute_rows(np.array([[1.0], [3.0]]), [0, 2], [1, 3], 4, "zero")
    assert z.ravel().tolist() == [1.0, 0.0, 3.0, 0.0]
    M = _rand((6, 3), 9)
    S, P = [0, 2, 5], [1, 3, 4]
    assert np.array_equal(O.impute_rows(M[S], S, P, 6, "same", hist=M), M)  # round trip S:91
    with pytest.raises(O.OracleError) as ei:
        O.impute_rows(M[S], S, P, 6, "same")
    assert ei.value.code == "ZTP_EHISTORY"


# -------------------------------------------------------------- layer helpers

def _make(e, h=16, f=64, N=12, seed=0):
    Wq, Wk, Wv, Wo = (_rand((h, h), seed + i, 1 / math.sqrt(h)) for i in range(4))
    W1 = _rand((h, f), seed + 5, 1 / math.sqrt(h))
    W2 = _rand((f, h), seed + 6, 1 / math.sqrt(f))
    Xt, Gt = _rand((h, N), seed + 7), _rand((h, N), seed + 8)
    return (Xt, Gt, (Wq, Wk, Wv, Wo, W1, W2), O.shard_layer(Wq, Wk, Wv, Wo, W1, W2, e))


@pytest.mark.parametrize("e", [1, 2, 4])
def test_tp_equivalence_gamma0(e):
    """gamma = 0 and no migration reproduce the unsplit dense layer."""
    Xt, Gt, W, sh = _make(e)
    ref = O.dense_layer_step(Xt, Gt, *W)
    out = O.layer_step(Xt, Gt, sh)
    tol = 1e-12
    assert np.max(np.abs(out["Y"] - ref["Y"])) <= tol * np.max(np.abs(ref["Y"]))
    assert np.max(np.abs(out["dX"] - ref["dX"])) <= tol * np.max(np.abs(ref["dX"]))
    h, f = Xt.shape[0], W[4].shape[1]
    a, u = h // e, f // e
    for r in range(e):
        np.testing.assert_allclose(out["dW1"][r], ref["dW1t"][:, r * u:(r + 1) * u], rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["dW2"][r], ref["dW2t"][r * u:(r + 1) * u], rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["dWo"][r], ref["dWOt"][r * a:(r + 1) * a], rtol=0, atol=1e-12)
        np.testing.assert_allclose(out["dWqkv"][r][:, :a], ref["dWQt"][:, r * a:(r + 1) * a], rtol=0, atol=1e-12)
    assert out["allreduce_count"] == 4          # 2 per layer per direction (A-29)


@pytest.mark.parametrize("e", [1, 2, 4])
def test_tp_gamma0_reproduces_unsplit_bitexact_fixed_order(e):
    """BJ north_star "ratio 0 and no migration reproduce the unsplit full GEMM
    exactly" (SURVEY §8(c) pin 1): with every contraction the naive
    k-ascending loop, the e-rank layer at gamma = 0 equals, bit for bit, the
    unsplit dense layer summed per shard block and over blocks in rank order;
    and the block order differs from the textbook one-block order by no more
    than the fp64 bound."""
    Xt, Gt, W, sh = _make(e, h=16, f=32, N=6, seed=3 + e)
    with O.fixed_order():
        out = O.layer_step(Xt, Gt, sh)
        ref = O.dense_layer_step(Xt, Gt, *W, blocks=e)
        one = O.dense_layer_step(Xt, Gt, *W, blocks=1)
    h, f = Xt.shape[0], W[4].shape[1]
    a, u = h // e, f // e
    assert np.array_equal(out["Y"], ref["Y"]) and np.array_equal(out["dX"], ref["dX"])
    for r in range(e):
        assert np.array_equal(out["dW1"][r], ref["dW1t"][:, r * u:(r + 1) * u])
        assert np.array_equal(out["dW2"][r], ref["dW2t"][r * u:(r + 1) * u])
        assert np.array_equal(out["dWo"][r], ref["dWOt"][r * a:(r + 1) * a])
        assert np.array_equal(out["dWqkv"][r][:, :a], ref["dWQt"][:, r * a:(r + 1) * a])
    for k in ("Y", "dX"):
        sc = np.max(np.abs(one[k]))
        assert np.max(np.abs(ref[k] - one[k])) <= (h + f) * 2.0 ** -52 * sc * 8
    # the BLAS order agrees with the fixed order within the fp64 bound
    blas = O.layer_step(Xt, Gt, sh)
    for k in ("Y", "dX"):
        assert np.max(np.abs(blas[k] - out[k])) <= 1e-12 * np.max(np.abs(out[k]))


def test_fixed_order_contract_against_exact_sums():
    """The fixed-order contraction is the k-ascending loop: against math.fsum
    (exactly rounded) within K 2^-53 sum|terms|, and it reproduces a hand
    evaluation of the same loop bit for bit."""
    A, B = _rand((7, 3), 41), _rand((7, 4), 42)
    with O.fixed_order():
        C = O.contract(A, B)
    for j in range(3):
        for t in range(4):
            acc = 0.0
            for k in range(7):
                acc = acc + A[k, j] * B[k, t]
            assert C[j, t] == acc
            ex = math.fsum(A[k, j] * B[k, t] for k in range(7))
            assert abs(C[j, t] - ex) <= 7 * 2 ** -53 * sum(abs(A[k, j] * B[k, t]) for k in range(7))


def _loss(Xt, Gt, sh, sel=None, mig=None):
    return float(np.sum(O.layer_step(Xt, Gt, sh, sel, mig)["Y"] * Gt))


def _random_sel(e, h, f, seed, gamma=0.5):
    rng = np.random.default_rng(seed)
    sel = []
    for r in range(e):
        d = {}
        for seg, K in (("qkv", h), ("o", h // e), ("fc1", h), ("fc2", f // e)):
            npr = int(math.floor(K * gamma + 0.5))
            S, P = O.select(rng.random(K).astype(np.float32), min(npr, K - 1))
            d[seg] = (S, P)
        sel.append(d)
    return sel


@pytest.mark.parametrize("mode", ["dense", "pruned", "migrated", "pruned+migrated"])
def test_gradient_check_central_differences_S301(mode):
    """analytic gradients vs central differences (step 1e-5,
    rel 1e-5) on 32 coordinates.  The pruned layer is a function of its
    weights; its exact gradient has zeros at pruned rows -- which is what Zero
    imputation produces.  Migration is lossless."""
    e, h, f, N = 2, 8, 32, 6
    Xt, Gt, W, sh = _make(e, h, f, N, seed=11)
    mig = [(1, 0, 12, 16)] if "migrated" in mode else None
    if mode == "pruned":
        sel = _random_sel(e, h, f, 5)
    elif mode == "pruned+migrated":
        # SEMI split on the straggler (rank 1): units [12, 16) migrate to the
        # NORMAL helper (rank 0, unpruned, A-44) and the straggler resizes
        # its four linears, FC2 over its remaining 12 units
        sel = [{seg: (list(range(K)), []) for seg, K in (("qkv", h), ("o", h // e), ("fc1", h), ("fc2", f // e))}]
        rng = np.random.default_rng(6)
        d = {}
        for seg, K in (("qkv", h), ("o", h // e), ("fc1", h), ("fc2", 12)):
            d[seg] = O.select(rng.random(K).astype(np.float32), K // 2)
        sel.append(d)
    else:
        sel = None
    out = O.layer_step(Xt, Gt, sh, sel, mig)
    rng = random.Random(3)
    step = 1e-5
    checks = 0
    while checks < 32:
        which = rng.choice(["qkv", "o", "w1", "w2", "x"])
        r = rng.randrange(e)
        if which == "x":
            arr, grad = Xt, out["dX"]
        else:
            lst = {"qkv": sh.qkv_t, "o": sh.o_t, "w1": sh.w1_t, "w2": sh.w2_t}[which]
            arr = lst[r]
            grad = {"qkv": out["dWqkv"], "o": out["dWo"], "w1": out["dW1"], "w2": out["dW2"]}[which][r]
        i, j = rng.randrange(arr.shape[0]), rng.randrange(arr.shape[1])
        old = arr[i, j]
        arr[i, j] = old + step
        lp = _loss(Xt, Gt, sh, sel, mig)
        arr[i, j] = old - step
        lm = _loss(Xt, Gt, sh, sel, mig)
        arr[i, j] = old
        fd = (lp - lm) / (2 * step)
        an = grad[i, j]
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)), (which, r, i, j, fd, an)
        checks += 1


def test_migration_lossless_and_merge_equivalence_S501_S504():
    e, h, f, N = 4, 16, 64, 10
    Xt, Gt, W, sh = _make(e, h, f, N, seed=21)
    base = O.layer_step(Xt, Gt, sh)
    # straggler 2 sheds units [10,16) of its 16: helpers by r' = (r-2+4)%4 -> 3,0,1
    mig = [(2, 3, 10, 12), (2, 0, 12, 14), (2, 1, 14, 16)]
    m1 = O.layer_step(Xt, Gt, sh, mig=mig, merged=True)
    m2 = O.layer_step(Xt, Gt, sh, mig=mig, merged=False)
    for k in ("Y", "dX"):
        sc = np.max(np.abs(base[k]))
        assert np.max(np.abs(m1[k] - base[k])) <= 1e-12 * sc
        assert np.max(np.abs(m1[k] - m2[k])) <= 1e-12 * sc
    for r in range(e):
        for k in ("dW1", "dW2", "dWo", "dWqkv"):
            sc = max(1e-300, np.max(np.abs(base[k][r])))
            assert np.max(np.abs(m1[k][r] - base[k][r])) <= 1e-12 * sc
    assert m1["allreduce_count"] == 4 and m2["allreduce_count"] == 4
    # compute moved: the straggler's executed FLOPs drop, helpers' grow
    assert m1["flops"][2] < base["flops"][2]
    assert sum(m1["flops"]) == pytest.approx(sum(base["flops"]), rel=1e-12)


@pytest.mark.parametrize("gamma", [0.25, 0.5, 0.9])
def test_consistency_constraint_and_work_reduction(gamma):
    """all shapes unpruned; dW rows P exactly 0; executed
    FLOPs = (1-gamma) dense within 2/K."""
    e, h, f, N = 2, 16, 64, 8
    Xt, Gt, W, sh = _make(e, h, f, N, seed=31)
    sel = _random_sel(e, h, f, 9, gamma)
    out = O.layer_step(Xt, Gt, sh, sel)
    base = O.layer_step(Xt, Gt, sh)
    for k in ("Y", "dX"):
        assert out[k].shape == base[k].shape
    for r in range(e):
        for k, seg in (("dW1", "fc1"), ("dW2", "fc2"), ("dWo", "o"), ("dWqkv", "qkv")):
            assert out[k][r].shape == base[k][r].shape
            P = sel[r][seg][1]
            assert np.all(out[k][r][P] == 0.0)
            S = sel[r][seg][0]
            assert np.any(out[k][r][S] != 0.0)
    ratio = sum(out["flops"]) / sum(base["flops"])
    assert abs(ratio - (1 - gamma)) <= 2.0 / (f // e) + 1e-12


def test_sampled_columns_equal_full():
    e, h, f, N = 2, 16, 64, 20
    Xt, Gt, W, sh = _make(e, h, f, N, seed=41)
    sel = _random_sel(e, h, f, 3, 0.5)
    full = O.layer_step(Xt, Gt, sh, sel)
    cols = [0, 7, 19]
    smp = O.layer_step_sampled(Xt, Gt, sh, sel, cols)
    np.testing.assert_allclose(smp["Y"], full["Y"][:, cols], rtol=0, atol=1e-13)
    np.testing.assert_allclose(smp["dX"], full["dX"][:, cols], rtol=0, atol=1e-13)


def test_synth_shards_concatenate_to_dense():
    """The generator's block API gives shards that concatenate exactly."""
    d = I.uniform_sym(5, "w", 8, 12, 0.3)
    parts = [I.uniform_sym(5, "w", 8, 12, 0.3, c0=c, c1=c + 4) for c in (0, 4, 8)]
    assert np.array_equal(np.concatenate(parts, axis=1), d)
    z = I.normal(5, "x", 6, 10)
    assert np.array_equal(I.normal(5, "x", 6, 10, r0=2, r1=5), z[2:5])
    assert np.array_equal(I.round_bf16(z), z)


# ------------------------------------------------- real attention core (NEXT-4)

@pytest.mark.parametrize("causal", [True, False])
def test_attention_core_closed_forms(causal):
    """Q = 0 makes every allowed score equal: each query's output is the plain
    mean of V over the keys it may see -- the prefix mean (causal) or the
    sequence mean -- per batch and head; one-token sequences return V."""
    d, S, B, H = 4, 5, 2, 2
    core = O.AttnCore(head_dim=d, seq=S, causal=causal)
    V = _rand((H * d, B * S), 3)
    ctx, P = O.attention_fwd(np.zeros((H * d, B * S)), _rand((H * d, B * S), 4), V, core)
    for b in range(B):
        for i in range(S):
            lo, hi = b * S, b * S + (i + 1 if causal else S)
            np.testing.assert_allclose(ctx[:, b * S + i], V[:, lo:hi].mean(axis=1), rtol=0, atol=1e-15)
    for p in P.values():
        np.testing.assert_allclose(p.sum(axis=1), 1.0, rtol=0, atol=1e-15)
        if causal:
            assert np.all(np.triu(p, 1) == 0.0)
    one = O.AttnCore(head_dim=d, seq=1, causal=causal)
    Q1, K1, V1 = _rand((H * d, 3), 5), _rand((H * d, 3), 6), _rand((H * d, 3), 7)
    np.testing.assert_allclose(O.attention_fwd(Q1, K1, V1, one)[0], V1, rtol=0, atol=1e-15)


@pytest.mark.parametrize("mode", ["dense", "pruned"])
def test_attention_layer_gradient_check(mode):
    """The layer with the real attention core: analytic gradients of every
    weight and of X vs central differences (S:248/S:301 protocol)."""
    e, h, f, N = 2, 8, 16, 6
    core = O.AttnCore(head_dim=2, seq=3, causal=True)
    Xt, Gt, W, sh = _make(e, h, f, N, seed=13)
    sel = _random_sel(e, h, f, 8) if mode == "pruned" else None
    out = O.layer_step(Xt, Gt, sh, sel, core=core)
    loss = lambda: float(np.sum(O.layer_step(Xt, Gt, sh, sel, core=core)["Y"] * Gt))  # noqa: E731
    rng = random.Random(17)
    step = 1e-5
    for _ in range(24):
        which = rng.choice(["qkv", "o", "w1", "w2", "x"])
        r = rng.randrange(e)
        if which == "x":
            arr, grad = Xt, out["dX"]
        else:
            arr = {"qkv": sh.qkv_t, "o": sh.o_t, "w1": sh.w1_t, "w2": sh.w2_t}[which][r]
            grad = {"qkv": out["dWqkv"], "o": out["dWo"], "w1": out["dW1"], "w2": out["dW2"]}[which][r]
        i, j = rng.randrange(arr.shape[0]), rng.randrange(arr.shape[1])
        old = arr[i, j]
        arr[i, j] = old + step
        lp = loss()
        arr[i, j] = old - step
        lm = loss()
        arr[i, j] = old
        fd = (lp - lm) / (2 * step)
        assert abs(fd - grad[i, j]) <= 1e-5 * max(1.0, abs(grad[i, j])), (which, r, i, j, fd, grad[i, j])

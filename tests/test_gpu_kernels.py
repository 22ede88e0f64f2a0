"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle on
identical seeded inputs: select (bit-exact), resized GEMMs fwd/dX/dW with
ragged tiles and the Zero imputation (bf16: 2e-2 ||ref||_inf; imputed rows
exactly +0.0), fused GeLU / GeLU' epilogues, fp32 verification mode (1e-5)."""
import math

import numpy as np
import pytest

from oracle import ztp_oracle as O
from synth import inputs as I

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-5


@pytest.fixture(scope="module", params=["compact", "gather4"])
def env(request):
    """Both producer modes: compact operand copies + dense TMA boxes (default)
    and in-GEMM TMA gather4 of the lineage rows (ZTP_GATHER4=1)."""
    import os
    import torch
    import paper_2401_11469_b200 as Z
    assert torch.cuda.is_available(), "GPU tests need a B200"
    os.environ["ZTP_GATHER4"] = "1" if request.param == "gather4" else "0"
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    os.environ.pop("ZTP_GATHER4")
    yield Z, torch, ctx
    Z.ztp_ctx_destroy(ctx)


def dev(torch, a, dtype=None):
    """Device copy with the row pitch padded to a multiple of 8 elements (16 B);
    returns a view of the logical shape (exercises ld != cols)."""
    dtype = dtype or torch.bfloat16
    a = np.asarray(a, dtype=np.float32)
    if a.ndim == 1:
        return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)
    r, c = a.shape
    ld = (c + 7) // 8 * 8
    buf = torch.full((r, ld), float("nan"), device="cuda", dtype=dtype)
    buf[:, :c] = torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)
    return buf[:, :c]


def empty(torch, r, c, dtype):
    ld = (c + 7) // 8 * 8
    return torch.full((r, ld), float("nan"), device="cuda", dtype=dtype)[:, :c]


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def err_ok(got, ref, tol):
    scale = max(np.max(np.abs(ref)), 1e-30)
    return np.max(np.abs(got - ref)) <= tol * scale, np.max(np.abs(got - ref)) / scale


# ----------------------------------------------------------------- select

@pytest.mark.parametrize("seed", range(8))
def test_select_bitexact_random_segments(env, seed):
    Z, torch, ctx = env
    rng = np.random.default_rng(seed)
    nseg = int(rng.integers(1, 70))            # > 64 exercises the chunked launch
    lens = [int(rng.choice([1, 2, 7, 64, 333, 1024, 1376, 5000, 20480])) for _ in range(nseg)]
    nps = [int(rng.integers(0, L)) if L > 1 else 0 for L in lens]
    app = [int(rng.integers(0, 5)) for _ in range(nseg)]
    parts = []
    for i, L in enumerate(lens):
        kind = rng.integers(0, 3)
        if kind == 0:
            s = I.lognormal_scores(seed, f"s{i}", L)
        elif kind == 1:
            s = I.lognormal_scores(seed, f"s{i}", L, levels=16)       # tie stress (c3 variant)
        else:
            s = rng.standard_normal(L).astype(np.float32)
            s[rng.integers(0, L, size=max(1, L // 10))] = -0.0
        parts.append(s)
    scores = dev(torch, np.concatenate(parts), torch.float32)
    kept = torch.empty(sum(L - p + a for L, p, a in zip(lens, nps, app)), dtype=torch.int32, device="cuda")
    pruned = torch.empty(max(1, sum(nps)), dtype=torch.int32, device="cuda")
    Z.ztp_select(ctx, lens, nps, scores, kept, pruned, app)
    Z.ztp_sync(ctx)
    kh, ph = kept.cpu().numpy(), pruned.cpu().numpy()
    ko = po = 0
    for i, L in enumerate(lens):
        S, P = O.select(parts[i], nps[i])
        nk = L - nps[i]
        assert np.array_equal(kh[ko:ko + nk], S), f"segment {i} kept"
        assert np.array_equal(kh[ko + nk:ko + nk + app[i]], np.arange(L, L + app[i])), f"segment {i} appended"
        assert np.array_equal(ph[po:po + nps[i]], P), f"segment {i} pruned"
        ko += nk + app[i]
        po += nps[i]


@pytest.mark.parametrize("L", [8193, 12000, 12288, 49152, 49153])
def test_select_staging_boundaries(env, L):
    """Segment lengths around the shared-memory staging limits of the select
    kernel (register path <= 8K keys; staged keys up to 48K; 12288 keys =
    exactly 48 KB of dynamic smem, the c4 TP=1 derived V segment), each as
    the longest segment of its launch, bit-exact vs the oracle."""
    Z, torch, ctx = env
    lens = [L, 333]
    parts = [I.lognormal_scores(7, f"b{L}", L, levels=16), I.lognormal_scores(7, "small", 333)]
    nps = [L // 3, 100]
    scores = dev(torch, np.concatenate(parts), torch.float32)
    kept = torch.empty(sum(n - p for n, p in zip(lens, nps)), dtype=torch.int32, device="cuda")
    pruned = torch.empty(sum(nps), dtype=torch.int32, device="cuda")
    Z.ztp_select(ctx, lens, nps, scores, kept, pruned)
    Z.ztp_sync(ctx)
    kh, ph = kept.cpu().numpy(), pruned.cpu().numpy()
    ko = po = 0
    for i, n in enumerate(lens):
        S, P = O.select(parts[i], nps[i])
        assert np.array_equal(kh[ko:ko + n - nps[i]], S) and np.array_equal(ph[po:po + nps[i]], P), i
        ko += n - nps[i]
        po += nps[i]


def test_select_nan_flag(env):
    Z, torch, ctx = env
    s = dev(torch, np.array([1.0, np.nan, 2.0], dtype=np.float32), torch.float32)
    kept = torch.empty(3, dtype=torch.int32, device="cuda")
    pruned = torch.empty(3, dtype=torch.int32, device="cuda")
    Z.ztp_select(ctx, [3], [1], s, kept, pruned)
    with pytest.raises(Z.ZtpError) as ei:
        Z.ztp_sync(ctx)
    assert ei.value.name == "ZTP_EINVAL"
    Z.ztp_sync(ctx)  # flag cleared


def test_select_host_errors(env):
    Z, torch, ctx = env
    s = torch.zeros(4, device="cuda")
    k = torch.empty(4, dtype=torch.int32, device="cuda")
    with pytest.raises(Z.ZtpError):
        Z.ztp_select(ctx, [4], [4], s, k, k)     # nothing would survive


# ------------------------------------------------------------ resized GEMMs

def _case(K, n, N, gamma, seed):
    Xt = I.normal(seed, "x", K, N)
    Wt = I.uniform_sym(seed, "w", K, n, 1.0 / math.sqrt(K))
    Gt = I.normal(seed, "g", n, N)
    npr = int(math.floor(K * gamma + 0.5))
    npr = min(npr, K - 1)
    S, P = O.select(I.lognormal_scores(seed, "sc", K), npr)
    return Xt, Wt, Gt, S, P


def _sel_dev(Z, torch, S, P, lid=0, mid=0):
    kept = torch.tensor(np.asarray(S, dtype=np.int32), device="cuda")
    pruned = torch.tensor(np.asarray(P if len(P) else [0], dtype=np.int32), device="cuda")
    return Z.sel(kept, len(S), pruned, len(P), lid, mid), (kept, pruned)


SHAPES = [  # (K, n, N, gamma): ragged K' tails, partial M/N tiles, several tiles
    (200, 300, 328, 0.35),
    (64, 128, 256, 0.0),
    (1024, 512, 776, 0.5),
    (96, 40, 24, 0.9),
    (517, 264, 1032, 0.25),
]


@pytest.mark.parametrize("K,n,N,gamma", SHAPES)
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_fwd_dx_dw_parity(env, K, n, N, gamma, dtype):
    Z, torch, ctx = env
    Xt, Wt, Gt, S, P = _case(K, n, N, gamma, seed=K + n + N)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = TOL_BF16 if dtype == "bf16" else TOL_F32
    x, w, g = dev(torch, Xt, td), dev(torch, Wt, td), dev(torch, Gt, td)
    y = empty(torch, n, N, td)
    dx = empty(torch, K, N, td)
    dw = empty(torch, K, n, td)
    s, keep = _sel_dev(Z, torch, S, P)
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=g, dx_t=dx, dw_t=dw, sel_=s)
    Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    Z.ztp_gemm(ctx, Z.KIND_DX, a)
    Z.ztp_gemm(ctx, Z.KIND_DW, a)
    Z.ztp_sync(ctx)
    ref_y = O.linear_fwd(Wt, Xt, S)
    ref_dx = O.linear_bwd_dx(Wt, Gt, S, P)
    ref_dw = O.linear_bwd_dw(Xt, Gt, S, P)
    for name, got, ref in (("y", y, ref_y), ("dx", dx, ref_dx), ("dw", dw, ref_dw)):
        gh = host(got)
        assert np.isfinite(gh).all(), f"{name}: unwritten (NaN) elements"
        ok, e = err_ok(gh, ref, tol)
        assert ok, f"{name}: max|err|/||ref|| = {e:.3e}"
    # Zero imputation: rows P exactly +0.0 (bit pattern)
    if len(P):
        for t in (dx, dw):
            rows = t[torch.tensor(P, device="cuda")]
            assert torch.all(rows == 0) and not torch.any(torch.signbit(rows))


@pytest.mark.parametrize("act", ["gelu", "gelu_d"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_gelu_epilogues(env, dtype, act):
    """FWD: pre_t <- pre (GELU) or GeLU'(pre) (GELU_D), y <- GeLU(pre).
    Row-layer dX: G1 = dH * GeLU'(pre_in) (GELU) or dH * pre_in (GELU_D, where
    pre_in already holds GeLU'(pre))."""
    Z, torch, ctx = env
    K, n, N = 384, 272, 520
    Xt, Wt, Gt, S, P = _case(K, n, N, 0.4, seed=7)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = TOL_BF16 if dtype == "bf16" else TOL_F32
    A = Z.ACT_GELU if act == "gelu" else Z.ACT_GELU_D
    x, w = dev(torch, Xt, td), dev(torch, Wt, td)
    pre = empty(torch, n, N, td)
    h = empty(torch, n, N, td)
    s, keep = _sel_dev(Z, torch, S, P)
    Z.ztp_gemm(ctx, Z.KIND_FWD, Z.linear_args(x_t=x, w_t=w, y_t=h, pre_t=pre, sel_=s, act=A))
    K2, n2 = 272, 200
    W2 = I.uniform_sym(8, "w2", K2, n2, 1 / math.sqrt(K2))
    G2 = I.normal(8, "g2", n2, N)
    PreIn = I.normal(8, "pin", K2, N)
    S2, P2 = O.select(I.lognormal_scores(8, "s2", K2), 100)
    s2, keep2 = _sel_dev(Z, torch, S2, P2)
    g1 = empty(torch, K2, N, td)
    aux = PreIn if act == "gelu" else O.gelu_tanh_grad(PreIn)
    Z.ztp_gemm(ctx, Z.KIND_DX, Z.linear_args(w_t=dev(torch, W2, td), g_t=dev(torch, G2, td), dx_t=g1,
                                             pre_in_t=dev(torch, aux, td), sel_=s2, act_in=A))
    Z.ztp_sync(ctx)
    ref_pre = O.linear_fwd(Wt, Xt, S)
    ok, e = err_ok(host(pre), ref_pre if act == "gelu" else O.gelu_tanh_grad(ref_pre), tol)
    assert ok, e
    ok, e = err_ok(host(h), O.gelu_tanh(ref_pre), tol)
    assert ok, e
    ref_g1 = O.linear_bwd_dx(W2, G2, S2, P2) * O.gelu_tanh_grad(PreIn)
    ok, e = err_ok(host(g1), ref_g1, tol)
    assert ok, e


@pytest.mark.parametrize("case", ["fwd_gelu", "fwd_gelu_d", "dx_gelu_grad", "dx_mul", "dw"])
def test_gemm_splitk_paths(env, case):
    """Few output tiles + long contraction -> split-K partials + the fixed-order
    reduce kernel (epilogue, row map and Zero rows applied there)."""
    Z, torch, ctx = env
    if case.startswith("fwd_gelu"):
        K, n, N, gamma = 8192, 128, 256, 0.5            # 1 tile, 64 k-blocks
    elif case.startswith("dx"):
        K, n, N, gamma = 256, 2048, 256, 0.6            # 1 computed m-tile, kdim 2048
    else:
        K, n, N, gamma = 256, 200, 4096, 0.5            # 1 x 1 tiles, 64 token k-blocks
    Xt, Wt, Gt, S, P = _case(K, n, N, gamma, seed=31)
    x, w, g = dev(torch, Xt), dev(torch, Wt), dev(torch, Gt)
    s, keep = _sel_dev(Z, torch, S, P)
    if case.startswith("fwd_gelu"):
        gd = case == "fwd_gelu_d"
        pre, h = empty(torch, n, N, torch.bfloat16), empty(torch, n, N, torch.bfloat16)
        Z.ztp_gemm(ctx, Z.KIND_FWD, Z.linear_args(x_t=x, w_t=w, y_t=h, pre_t=pre, sel_=s,
                                                  act=Z.ACT_GELU_D if gd else Z.ACT_GELU))
        Z.ztp_sync(ctx)
        ref = O.linear_fwd(Wt, Xt, S)
        for got, want in ((pre, O.gelu_tanh_grad(ref) if gd else ref), (h, O.gelu_tanh(ref))):
            ok, e = err_ok(host(got), want, TOL_BF16)
            assert ok, e
    elif case.startswith("dx"):
        mul = case == "dx_mul"
        pin = I.normal(31, "pin", K, N)
        dx = empty(torch, K, N, torch.bfloat16)
        Z.ztp_gemm(ctx, Z.KIND_DX, Z.linear_args(w_t=w, g_t=g, dx_t=dx,
                                                 pre_in_t=dev(torch, O.gelu_tanh_grad(pin) if mul else pin), sel_=s,
                                                 act_in=Z.ACT_GELU_D if mul else Z.ACT_GELU))
        Z.ztp_sync(ctx)
        ref = O.linear_bwd_dx(Wt, Gt, S, P) * O.gelu_tanh_grad(pin)
        ok, e = err_ok(host(dx), ref, TOL_BF16)
        assert ok, e
        assert torch.all(dx[torch.tensor(P, device="cuda")] == 0)
    else:
        dw = empty(torch, K, n, torch.bfloat16)
        Z.ztp_gemm(ctx, Z.KIND_DW, Z.linear_args(x_t=x, w_t=w, g_t=g, dw_t=dw, sel_=s))
        Z.ztp_sync(ctx)
        ok, e = err_ok(host(dw), O.linear_bwd_dw(Xt, Gt, S, P), TOL_BF16)
        assert ok, e
        assert torch.all(dw[torch.tensor(P, device="cuda")] == 0)


@pytest.mark.parametrize("g1,g2,N", [(0.3, 0.45, 264), (0.0, 0.5, 264), (0.5, 0.0, 264), (0.3, 0.45, 4096)])
def test_output_pruning_col_row_pair(env, g1, g2, N):
    """FC1 (col, GeLU) -> FC2 (row) with out_sel = FC2's entry: FC1 computes
    only the units S2 FC2 keeps, FC2's dX is written compact (dx_compact) and
    FC1's backward contracts over S2 only and writes Zero columns P2 of dW1.
    Every result equals the full-output computation of the oracle."""
    Z, torch, ctx = env
    h, f = 200, 520          # N = 4096: dW1 split-K, the reduce spreads the compact columns
    seed = 41 + int(10 * g1) + int(100 * g2) + N
    X = I.normal(seed, "x", h, N)
    W1 = I.uniform_sym(seed, "w1", h, f, 1 / math.sqrt(h))
    W2 = I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f))
    G = I.normal(seed, "g", h, N)
    S1, P1 = O.select(I.lognormal_scores(seed, "s1", h), min(int(h * g1 + 0.5), h - 1))
    S2, P2 = O.select(I.lognormal_scores(seed, "s2", f), min(int(f * g2 + 0.5), f - 1))
    nk2 = len(S2)
    bf = torch.bfloat16
    x, w1, w2, g = dev(torch, X), dev(torch, W1), dev(torch, W2), dev(torch, G)
    s1, k1 = _sel_dev(Z, torch, S1, P1, 0, 2) if len(P1) else (None, None)
    s2, k2 = _sel_dev(Z, torch, S2, P2, 0, 3)
    pos = np.full(f, -1, dtype=np.int32)
    pos[np.asarray(S2)] = np.arange(nk2, dtype=np.int32)
    pos = torch.tensor(pos, device="cuda")
    hc, prec = empty(torch, nk2, N, bf), empty(torch, nk2, N, bf)
    y = empty(torch, h, N, bf)
    g1c = empty(torch, nk2, N, bf)
    dy1, dw1, dw2 = empty(torch, h, N, bf), empty(torch, h, f, bf), empty(torch, f, h, bf)
    ws1 = empty(torch, h, f, bf)
    a1 = Z.linear_args(x_t=x, w_t=w1, y_t=hc, pre_t=prec, ws_t=ws1, sel_=s1, act=Z.ACT_GELU, y_pos=pos,
                       out_sel=s2)
    a2 = Z.linear_args(x_t=hc, w_t=w2, y_t=y, g_t=g, dx_t=g1c, dw_t=dw2, pre_in_t=prec, sel_=s2,
                       act_in=Z.ACT_GELU, x_compact=True, dx_compact=True)
    b1 = Z.linear_args(x_t=x, w_t=w1, g_t=g1c, dx_t=dy1, dw_t=dw1, ws_t=ws1, sel_=s1, y_pos=pos, out_sel=s2)
    Z.ztp_col_linear(ctx, Z.FWD, a1)
    Z.ztp_row_linear(ctx, Z.FWD, a2)
    Z.ztp_row_linear(ctx, Z.BWD, a2)
    Z.ztp_col_linear(ctx, Z.BWD, b1)
    Z.ztp_sync(ctx)
    S2a = np.asarray(S2)
    pre_ref = O.linear_fwd(W1, X, S1)                       # full FC1 output
    H_ref = O.gelu_tanh(pre_ref)
    y_ref = O.linear_fwd(W2, H_ref, S2)
    G1_full = O.linear_bwd_dx(W2, G, S2, P2) * O.gelu_tanh_grad(pre_ref)   # rows P2 exactly 0
    checks = [("pre", prec, pre_ref[S2a]), ("H", hc, H_ref[S2a]), ("y", y, y_ref), ("G1", g1c, G1_full[S2a]),
              ("dW2", dw2, O.linear_bwd_dw(H_ref, G, S2, P2)), ("dY1", dy1, O.linear_bwd_dx(W1, G1_full, S1, P1)),
              ("dW1", dw1, O.linear_bwd_dw(X, G1_full, S1, P1))]
    for name, got, ref in checks:
        gh = host(got)
        assert np.isfinite(gh).all(), f"{name}: unwritten (NaN) elements"
        ok, e = err_ok(gh, ref, TOL_BF16)
        assert ok, f"{name}: max|err|/||ref|| = {e:.3e}"
    if len(P2):   # Zero columns P2 of dW1, bit pattern +0.0
        cols = dw1[:, torch.tensor(P2, device="cuda")]
        assert torch.all(cols == 0) and not torch.any(torch.signbit(cols))


def test_gemm_large_c2_shapes_sampled(env):
    """c2 e=1 FC1 shapes (K=1024, n=4096, N=8192) in the bench launch config,
    checked on sampled output rows/columns computed one by one in fp64."""
    Z, torch, ctx = env
    K, n, N = 1024, 4096, 8192
    Xt, Wt, Gt, S, P = _case(K, n, N, 0.5, seed=11)
    x, w, g = dev(torch, Xt), dev(torch, Wt), dev(torch, Gt)
    y = torch.empty((n, N), device="cuda", dtype=torch.bfloat16)
    dx = torch.empty((K, N), device="cuda", dtype=torch.bfloat16)
    dw = torch.empty((K, n), device="cuda", dtype=torch.bfloat16)
    s, keep = _sel_dev(Z, torch, S, P)
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=g, dx_t=dx, dw_t=dw, sel_=s)
    for kind in (Z.KIND_FWD, Z.KIND_DX, Z.KIND_DW):
        Z.ztp_gemm(ctx, kind, a)
    Z.ztp_sync(ctx)
    rng = np.random.default_rng(0)
    rows_n = rng.integers(0, n, 24)
    cols_N = rng.integers(0, N, 24)
    yh, dxh, dwh = host(y), host(dx), host(dw)
    ref = Wt[S][:, rows_n].T @ Xt[S][:, cols_N]
    ok, e = err_ok(yh[np.ix_(rows_n, cols_N)], ref, TOL_BF16)
    assert ok, e
    rk = rng.choice(S, 24)
    ok, e = err_ok(dxh[np.ix_(rk, cols_N)], Wt[rk] @ Gt[:, cols_N], TOL_BF16)
    assert ok, e
    ok, e = err_ok(dwh[np.ix_(rk, rows_n)], Xt[rk] @ Gt[rows_n].T, TOL_BF16)
    assert ok, e
    assert np.all(dxh[P] == 0) and np.all(dwh[P] == 0)


def test_prepare_batched_compaction(env):
    """ztp_prepare: one launch writes xs_t = x[S], ws_t = w[S] and the 2D block
    W^T[S, S'] (out_sel), bit-exact copies; ragged widths use the scalar path."""
    Z, torch, ctx = env
    K, n, N = 300, 523, 264
    X = I.normal(5, "x", K, N)
    W = I.uniform_sym(5, "w", K, n, 0.1)
    S, P = O.select(I.lognormal_scores(5, "s", K), 120)
    S2, P2 = O.select(I.lognormal_scores(5, "s2", n), 200)
    s, keep = _sel_dev(Z, torch, S, P)
    s2, keep2 = _sel_dev(Z, torch, S2, P2, 0, 1)
    x, w = dev(torch, X), dev(torch, W)
    xs, ws, w2 = empty(torch, K, N, torch.bfloat16), empty(torch, K, n, torch.bfloat16), empty(torch, K, n, torch.bfloat16)
    a1 = Z.linear_args(x_t=x, w_t=w, xs_t=xs, ws_t=ws, sel_=s)
    a2 = Z.linear_args(x_t=x, w_t=w, ws_t=w2, sel_=s, out_sel=s2)
    Z.ztp_prepare(ctx, [(a1, 3), (a2, 2)])
    Z.ztp_sync(ctx)
    Sa, S2a = np.asarray(S), np.asarray(S2)
    xb, wb = host(x), host(w)
    assert np.array_equal(host(xs[:len(S)]), xb[Sa])
    assert np.array_equal(host(ws[:len(S)]), wb[Sa])
    assert np.array_equal(host(w2[:len(S), :len(S2)]), wb[Sa][:, S2a])


@pytest.mark.parametrize("policy", ["average", "same"])
@pytest.mark.parametrize("layer", ["col", "row"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_bwd_imputation_average_same(env, policy, layer, dtype):
    """NEXT-2: rows P of dX and dW imputed by Average (per-column mean
    over rows S, A-10) or Same (previous step's values, A-11); rows S as the
    resized GEMM.  Same without history -> ZTP_EHISTORY."""
    Z, torch, ctx = env
    K, n, N = 300, 264, 520
    Xt, Wt, Gt, S, P = _case(K, n, N, 0.35, seed=61)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = TOL_BF16 if dtype == "bf16" else TOL_F32
    Hdx = I.normal(62, "hdx", K, N)
    Hdw = I.normal(62, "hdw", K, n)
    x, w, g = dev(torch, Xt, td), dev(torch, Wt, td), dev(torch, Gt, td)
    y = empty(torch, n, N, td)
    dx, dw = empty(torch, K, N, td), empty(torch, K, n, td)
    s, keep = _sel_dev(Z, torch, S, P, 3, 0 if layer == "col" else 1)
    pol = Z.IMPUTE_AVERAGE if policy == "average" else Z.IMPUTE_SAME
    hx, hw = (dev(torch, Hdx, td), dev(torch, Hdw, td)) if policy == "same" else (None, None)
    lin = Z.ztp_col_linear if layer == "col" else Z.ztp_row_linear
    a = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=g, dx_t=dx, dw_t=dw, sel_=s, impute=pol, hist_dx=hx, hist_dw=hw)
    lin(ctx, Z.FWD, a)
    lin(ctx, Z.BWD, a)
    Z.ztp_sync(ctx)
    hist_x = host(hx) if hx is not None else None
    hist_w = host(hw) if hw is not None else None
    ref_dx = O.linear_bwd_dx(Wt, Gt, S, P, policy, hist_x)
    ref_dw = O.linear_bwd_dw(Xt, Gt, S, P, policy, hist_w)
    for name, got, ref in (("dx", dx, ref_dx), ("dw", dw, ref_dw)):
        gh = host(got)
        assert np.isfinite(gh).all(), name
        ok, e = err_ok(gh, ref, tol)
        assert ok, f"{name}: {e:.3e}"
        Pa = np.asarray(P)
        if policy == "same":
            assert np.array_equal(gh[Pa], (hist_x if name == "dx" else hist_w)[Pa]), f"{name}: Same rows not copied"
    if policy == "same":
        b = Z.linear_args(x_t=x, w_t=w, y_t=y, g_t=g, dx_t=dx, dw_t=dw, sel_=s, impute=pol)
        with pytest.raises(Z.ZtpError) as ei:
            lin(ctx, Z.BWD, b)
        assert ei.value.name == "ZTP_EHISTORY"


@pytest.mark.parametrize("K,n", [(1024, 4096), (300, 523), (17, 8)])
def test_priority_update_next1(env, K, n):
    """NEXT-1 (Alg.1 l.4-9): GPU column deltas vs the oracle (fp32 sum
    of bf16 differences, 1e-4 relative: n * 2^-24 bound), pruned rows carried over bit-exactly,
    L_uni exact for the GPU's deltas, and the next selection on them equals the
    oracle's select on the same scores (bit-exact)."""
    Z, torch, ctx = env
    W0 = I.uniform_sym(71, "w0", K, n, 0.05)
    W1 = W0 + I.normal(71, "dw", K, n) * 1e-3
    W1 = I.round_bf16(W1)
    d_prev = I.lognormal_scores(71, "d0", K)
    S, P = O.select(d_prev, K // 3)
    pos = np.full(K, 0, dtype=np.int32)
    pos[np.asarray(P, dtype=np.int64)] = -1
    w1, w0 = dev(torch, W1), dev(torch, W0)
    delta = torch.tensor(d_prev, device="cuda", dtype=torch.float32)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    theta = 1e-3
    Z.ztp_priority_update(ctx, w1, w0, delta, pos_prev=torch.tensor(pos, device="cuda"), count_above=cnt,
                          theta=theta)
    Z.ztp_sync(ctx)
    got = delta.cpu().numpy()
    ref = O.priority_update(d_prev.astype(np.float64), host(w1), host(w0), P)
    Pa = np.asarray(P, dtype=np.int64)
    assert np.array_equal(got[Pa], d_prev[Pa])                     # carried over
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-12)
    assert int(cnt.item()) == int(np.count_nonzero(got > np.float32(theta)))
    # the epoch's selection on the maintained scores: GPU select == oracle select
    npr = int(math.floor(K * O.pridiff_gamma(got, theta, 0.5) + 0.5))
    npr = min(npr, K - 1)
    kept = torch.empty(K, dtype=torch.int32, device="cuda")
    pr = torch.empty(max(1, npr), dtype=torch.int32, device="cuda")
    Z.ztp_select(ctx, [K], [npr], delta, kept, pr)
    Z.ztp_sync(ctx)
    S2, P2 = O.select(got, npr)
    assert np.array_equal(kept.cpu().numpy()[:K - npr], S2)
    assert np.array_equal(pr.cpu().numpy()[:npr], P2)


@pytest.mark.parametrize("incremental", [True, False])
def test_anti_endless_loop_on_gpu_S410(env, incremental):
    """S:410 / P:190 scenario of tests/test_oracle_select.py driven through the
    GPU kernels (ztp_priority_update + ztp_select, bf16 weights): every
    epoch's GPU scores match the oracle's on the same weights (1e-4), its
    selection equals the oracle's select on the GPU scores bit for bit, and
    the incremental rule rotates the pruned set (>= 3 distinct in 10 epochs)
    where the naive update freezes on the first one."""
    Z, torch, ctx = env
    K, n, npr = 64, 32, 16
    rng = np.random.default_rng(410)
    W = I.round_bf16(rng.standard_normal((K, n)))
    d0 = rng.random(K).astype(np.float32)
    delta = torch.tensor(d0, device="cuda")
    kept = torch.empty(K, dtype=torch.int32, device="cuda")
    pr = torch.empty(npr, dtype=torch.int32, device="cuda")
    pos = torch.empty(K, dtype=torch.int32, device="cuda")
    Z.ztp_select(ctx, [K], [npr], delta, kept, pr, pos=pos)
    Z.ztp_sync(ctx)
    sets = [tuple(pr.cpu().tolist())]
    assert list(sets[0]) == list(O.select(d0, npr)[1])
    for _ in range(9):
        W_old = W
        scale = rng.lognormal(-3.0, 1.0, size=K)
        upd = rng.standard_normal((K, n)) * scale[:, None]
        upd[np.asarray(sets[-1])] = 0.0
        W = I.round_bf16(W + upd)
        prev = delta.cpu().numpy().astype(np.float64)
        Z.ztp_priority_update(ctx, dev(torch, W), dev(torch, W_old), delta,
                              pos_prev=pos if incremental else None)
        Z.ztp_sync(ctx)
        got = delta.cpu().numpy()
        ref = O.priority_update(prev, W, W_old, list(sets[-1]) if incremental else None)
        assert np.allclose(got, ref, rtol=1e-4, atol=1e-12)
        Z.ztp_select(ctx, [K], [npr], delta, kept, pr, pos=pos)
        Z.ztp_sync(ctx)
        sets.append(tuple(pr.cpu().tolist()))
        assert list(sets[-1]) == list(O.select(got, npr)[1])
    if incremental:
        assert len(set(sets)) >= 3
    else:
        assert all(sset == sets[0] for sset in sets)


# ------------------------------------------------------ guard bands (no OOB writes)

def _guarded(torch, r, c, dtype):
    """[r, c] view of a NaN-filled buffer with 3 extra rows and >= 24 extra
    columns of padding (ld a multiple of 8): writes outside the logical
    tensor would change the padding."""
    ld = (c + 24 + 7) // 8 * 8
    buf = torch.full((r + 3, ld), float("nan"), device="cuda", dtype=dtype)
    return buf, buf[:r, :c]


def _band_intact(buf, r, c):
    return bool(torch_isnan_all(buf[r:, :]) and torch_isnan_all(buf[:, c:]))


def torch_isnan_all(t):
    import torch
    return bool(torch.isnan(t.float()).all().item())


@pytest.mark.parametrize("opts", [{}, {"SPLITK": 0}, {"SPLITK": 0, "SPREAD_EPI": 1}, {"ZERO_GENERIC": 0},
                                  {"SPLITK": 0, "ZERO_GENERIC": 0}])
def test_outputs_stay_inside_their_tensors(env, opts):
    """Every output of the FC1 -> FC2 pair (GeLU epilogues, compact and
    lineage-mapped rows, Zero tiles, output-pruned dW1 through the split-K
    reduce, the column-spread pass or the spreading epilogue) is a view into a
    NaN buffer with guard rows and columns: results match the oracle and no
    byte outside the logical tensors is written (the compute-sanitizer is
    unavailable on the GPU pool; this is its stand-in for the write paths)."""
    Z, torch, ctx = env
    for k, v in opts.items():
        Z.ztp_set_option(ctx, getattr(Z, "OPT_" + k), v)
    try:
        h, f, N, seed = 264, 776, 1032, 4711
        X = I.normal(seed, "x", h, N)
        W1 = I.uniform_sym(seed, "w1", h, f, 1 / math.sqrt(h))
        W2 = I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f))
        G = I.normal(seed, "g", h, N)
        S1, P1 = O.select(I.lognormal_scores(seed, "s1", h), int(0.6 * h))
        S2, P2 = O.select(I.lognormal_scores(seed, "s2", f), int(0.5 * f))
        nk2 = len(S2)
        bf = torch.bfloat16
        x, w1, w2, g = dev(torch, X), dev(torch, W1), dev(torch, W2), dev(torch, G)
        s1, k1 = _sel_dev(Z, torch, S1, P1, 0, 2)
        s2, k2 = _sel_dev(Z, torch, S2, P2, 0, 3)
        pos = np.full(f, -1, dtype=np.int32)
        pos[np.asarray(S2)] = np.arange(nk2, dtype=np.int32)
        pos = torch.tensor(pos, device="cuda")
        outs = {}
        for name, (r, c) in {"hc": (nk2, N), "prec": (nk2, N), "y": (h, N), "g1c": (nk2, N), "dy1": (h, N),
                             "dw1": (h, f), "dw2": (f, h)}.items():
            outs[name] = _guarded(torch, r, c, bf) + (r, c)
        v = {k_: t[1] for k_, t in outs.items()}
        ws1 = empty(torch, h, f, bf)
        a1 = Z.linear_args(x_t=x, w_t=w1, y_t=v["hc"], pre_t=v["prec"], ws_t=ws1, sel_=s1, act=Z.ACT_GELU,
                           y_pos=pos, out_sel=s2)
        a2 = Z.linear_args(x_t=v["hc"], w_t=w2, y_t=v["y"], g_t=g, dx_t=v["g1c"], dw_t=v["dw2"], pre_in_t=v["prec"],
                           sel_=s2, act_in=Z.ACT_GELU, x_compact=True, dx_compact=True)
        b1 = Z.linear_args(x_t=x, w_t=w1, g_t=v["g1c"], dx_t=v["dy1"], dw_t=v["dw1"], ws_t=ws1, sel_=s1, y_pos=pos,
                           out_sel=s2)
        Z.ztp_col_linear(ctx, Z.FWD, a1)
        Z.ztp_row_linear(ctx, Z.FWD, a2)
        Z.ztp_row_linear(ctx, Z.BWD, a2)
        Z.ztp_col_linear(ctx, Z.BWD, b1)
        Z.ztp_join(ctx)
        Z.ztp_sync(ctx)
        S2a = np.asarray(S2)
        pre_ref = O.linear_fwd(W1, X, S1)
        H_ref = O.gelu_tanh(pre_ref)
        G1_full = O.linear_bwd_dx(W2, G, S2, P2) * O.gelu_tanh_grad(pre_ref)
        refs = {"prec": pre_ref[S2a], "hc": H_ref[S2a], "y": O.linear_fwd(W2, H_ref, S2), "g1c": G1_full[S2a],
                "dw2": O.linear_bwd_dw(H_ref, G, S2, P2), "dy1": O.linear_bwd_dx(W1, G1_full, S1, P1),
                "dw1": O.linear_bwd_dw(X, G1_full, S1, P1)}
        for name, (buf, view, r, c) in outs.items():
            gh = host(view)
            assert np.isfinite(gh).all(), f"{name}: unwritten (NaN) elements"
            ok, e = err_ok(gh, refs[name], TOL_BF16)
            assert ok, f"{name}: max|err|/||ref|| = {e:.3e}"
            assert _band_intact(buf, r, c), f"{name}: a write landed outside the tensor"
    finally:
        for k in opts:
            Z.ztp_set_option(ctx, getattr(Z, "OPT_" + k), {"SPLITK": 1, "SPREAD_EPI": 0, "ZERO_GENERIC": 1}[k])
